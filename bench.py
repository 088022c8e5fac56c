"""Benchmark: training images/s of the Zhang MNIST CNN (fwd + bwd + SGD), BASELINE.json configs[1].

Workload (N=1): the paper protocol -- 10k synthetic 28x28 images (synth::make_set(10000, 1)), batch 100,
lr 0.05, init_params(42).  One bench *step* = one epoch = 100 SGD groups of 100 images (one launch of the
persistent cooperative train kernel).  ``--steps 10`` times exactly the 10-epoch protocol (the timed run
starts from init_params(42), so its epoch losses are checked against the reference's golden values).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--mode fast|exact] [--impl ours|reference]

N > 1 (``--gpus N`` spawns N ranks under torch.distributed.run, one per GPU): weak scaling -- every rank
owns a 100-image shard of each global group of 100*N images (static_chunk, runtime.cpp:138-145) over a
10k*N-image corpus.  Default exchange: fused into the clustered train kernel over NVLink peer memory
(fixed-point gradient slices added into the owning rank's accumulator, no collective call); fallback
(all ranks together): shard kernel -> ncclAllReduce of the 3,904-float gradient sum -> sgd kernel.
Every N>1 line carries its own e2e (per-rank shard bytes in) and the rank-0 cpu_baseline.
``--impl reference`` times the reference's own CPU net::train (oracle/_ref, the unmodified tensorloom
library) with all host threads on the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training images/sec (fwd+bwd+SGD), Zhang MNIST CNN, batch 100 and batch sweep, 1/2/4/8 B200"
FLOP_PER_TRAIN_IMAGE = 1_048_320  # 524,160 MAC algorithmic
FP32_LANES_PER_SM = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["fast", "exact"], default="fast")
    ap.add_argument("--batch", type=int, default=100, help="per-GPU images per SGD group")
    ap.add_argument("--n", type=int, default=10000, help="per-GPU corpus size")
    ap.add_argument("--grid", type=int, default=0, help="CTAs of the persistent kernel (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-dp", action="store_true",
                    help="run the N>1 data-parallel step (shard kernel + NCCL allreduce + sgd) even at N=1")
    ap.add_argument("--no-graph", action="store_true", help="NCCL data-parallel step: plain launches, no CUDA graph")
    ap.add_argument("--plan", action="store_true",
                    help="print this rank's launch plan (rank, world, device) as JSON and exit (no GPU work)")
    ap.add_argument("--dp-mode", choices=["nvlink", "nccl"], default="nvlink",
                    help="N>1 step: fused clustered kernel over NVLink peer memory (default; falls back to "
                         "nccl when symmetric memory is unavailable or a peer times out) or NCCL allreduce")
    return ap.parse_args()


# ---- clocks sampled during the timed region (NVML) -------------------------------------------------
class ClockSampler:
    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
           "hw_power_brake_slowdown": 0x80}
    NOTE = {"sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv, self.err = None, str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self) -> dict:
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        reasons = [k for k, v in {**self.BAD, **self.NOTE}.items() if self.reasons & v]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def golden_losses():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "protocol.json")) as f:
            return [float(v) for v in json.load(f)["epoch_mean_loss"]]
    except Exception:
        return None


# ---- reference CPU path (oracle/_ref = the unmodified tensorloom library) ---------------------------
def reference_epochs(n: int, epochs_budget_s: float, max_epochs: int, batch: int, workers: int = 0):
    """Times the reference's own net::train (oracle/_ref) on whole epochs of its own synth::make_set(n, 1)
    from its own init_params(42), with `workers` host threads (0 = all); returns (img/s, info)."""
    from oracle import Reference  # reference arm / cpu_baseline only
    R = Reference()
    cores = workers or os.cpu_count() or 1
    R.set_workers(cores)
    images, labels = R.make_set(n, 1)
    p = R.init_params(42)
    done, t_total = 0, 0.0
    while done < max_epochs:
        t0 = time.perf_counter()
        p, _ = R.train(images, labels, p, rate=0.05, epochs=1, batch=batch)
        t_total += time.perf_counter() - t0
        done += 1
        if t_total >= epochs_budget_s:
            break
    return done * n / t_total, {"cores": cores, "epochs": done, "seconds": t_total}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def workload_config(args, world: int) -> dict:
    """The `config` object of BOTH arms (identical dicts, so the driver's same-config check holds)."""
    B, n_per = args.batch, args.n
    return {"workload": "Zhang CNN paper protocol (BASELINE configs[1]" + (", configs[3] batch sweep" if B > 100 else "")
                        + f"): 1 step = 1 epoch of {n_per} images/GPU at batch {B}/GPU, lr 0.05, init_params(42)",
            "batch_per_gpu": B, "global_batch": B * world, "n_images": n_per * world, "epochs_per_step": 1,
            "parallelism": f"dp{world}",
            "l2": "flushed between timed steps (256 MiB write outside the event pair)"}


def run_reference(args):
    """The reference's own CPU net::train (oracle/_ref = the unmodified tensorloom library): inputs and
    initial weights from the reference itself (synth::make_set, net::init_params), all host threads."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import Reference
    R = Reference()
    cores = os.cpu_count() or 1
    R.set_workers(cores)
    # one step = one epoch of the per-GPU corpus at the GLOBAL batch (batch-independent cost on the CPU
    # once batch >= workers); the full N-GPU corpus would only scale the sample, not the rate
    n = args.n
    images, labels = R.make_set(n, 1)
    batch = min(args.batch * world, n)
    p0 = R.init_params(42)
    p = p0
    for _ in range(args.warmup):
        p, _ = R.train(images, labels, p, rate=0.05, epochs=1, batch=batch)
    p = p0
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        p, _ = R.train(images, labels, p, rate=0.05, epochs=1, batch=batch)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = args.steps * n / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic: reference synth::make_set({n}, 1), reference init_params(42)",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} epoch(s) x {n} images at batch {batch}, reference net::train "
                                   f"(oracle/_ref) with set_global_config({{{cores},4096}})"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


NCU_CAPTURES = {  # (mode, batch, n) -> committed `ncu --set full` key metrics of that exact launch
    ("fast", 100, 10000): "profiles/r2/ncu_cluster_r2i_keymetrics.csv",         # train_cluster_kernel
    ("fast", 16384, 32768): "profiles/r2/ncu_batch16k_r2i_keymetrics.csv",     # train_batch_kernel<2,320,2,1>
}


def ncu_traffic(mode: str, batch: int, n: int, world: int):
    """(DRAM bytes per launch (read + write), source file) of the train kernel from the committed
    `ncu --set full` capture of this exact workload (one epoch per launch); (None, None) otherwise."""
    rel = NCU_CAPTURES.get((mode, batch, n)) if world == 1 else None
    path = os.path.join(ROOT, rel) if rel else None
    if not path or not os.path.exists(path):
        return None, None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total = 0.0
    import csv
    with open(path) as f:
        for row in csv.DictReader(f):
            if row["metric"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                total += float(row["value"]) * scale.get(row["unit"], 1)
    return total, rel


# ---- our arm ----------------------------------------------------------------------------------------
def shard_rows(n_total: int, global_batch: int, world: int, rank: int) -> np.ndarray:
    """Dataset rows of this rank's shards, group by group: static_chunk(m_g, world, rank) of every SGD group
    (runtime.cpp:138-145, network.cpp:228-234) -- the rank's local corpus in the shard layout
    (tlb_ctx_set_shard_layout), shard of group g at local row g * ceil(global_batch / world)."""
    from paper_1912_05234_b200.parallel import groups, static_chunk
    rows = []
    for g, (start, m) in enumerate(groups(n_total, global_batch)):
        lo, hi = static_chunk(m, world, rank)
        rows.append(np.arange(start + lo, start + hi))
    return np.concatenate(rows) if rows else np.zeros(0, np.int64)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1912_05234_b200 import Context
    from paper_1912_05234_b200.runtime import init_params, synth_make_digits, synth_make_set

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # TLB_BENCH_SAME_GPU=1 (developer check of the N>1 plumbing on a one-GPU box): every rank on cuda:0,
    # a gloo process group and CUDA-IPC-mapped DP workspaces; use a small --batch so all ranks' kernels
    # are co-resident.  Not a throughput number.
    same_gpu = os.environ.get("TLB_BENCH_SAME_GPU") == "1"
    local = 0 if same_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dp = world > 1 or args.force_dp
    real_stdout = None
    if dp:
        # NCCL / torch.distributed print banners on stdout while communicators come up (lazily, at the
        # first collective): send fd 1 to stderr until the JSON line, so stdout carries exactly one line.
        sys.stdout.flush()
        real_stdout = os.dup(1)
        os.dup2(2, 1)
        if "RANK" not in os.environ:  # --force-dp without torchrun: a one-rank NCCL group
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT="29517")
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    B, n_per = args.batch, args.n
    n_total = n_per * world
    Bg = B * world
    images, labels = synth_make_set(n_total, 1)
    rows = None
    if dp:  # weak scaling: each rank keeps only its shards (1/world of the corpus) in HBM
        rows = shard_rows(n_total, Bg, world, rank)
        images, labels = np.ascontiguousarray(images[rows]), np.ascontiguousarray(labels[rows])
    stream = torch.cuda.Stream(device=dev)  # a real stream: torch's default stream handle is 0
    torch.cuda.set_stream(stream)
    ctx = Context(local, mode=args.mode)
    ctx.set_stream(stream.cuda_stream)
    if args.grid:
        ctx.set_grid(args.grid)
    if dp:
        ctx.set_shard_layout(B)

    d_x = torch.from_numpy(images).to(dev)
    d_y = torch.from_numpy(labels).to(dev)
    p0 = init_params(42)
    d_p = torch.zeros(3904, device=dev)
    d_loss = torch.zeros(max(args.steps, args.warmup, 1) + 1, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def reset():
        d_p.zero_()
        d_p[:3898] = torch.from_numpy(p0).to(dev)

    dp_used, dp_note = None, None
    if not dp:
        def epoch(e):
            ctx.train_device(d_x.data_ptr(), d_y.data_ptr(), n_total, d_p.data_ptr(), 0.05, e, 1, B,
                             d_loss.data_ptr())
        launches_per_step = 1
    else:
        from paper_1912_05234_b200.parallel import DeviceShardStep
        from paper_1912_05234_b200.parallel import FusedDPStep
        step, dp_used, dp_note = None, "nccl", None
        if args.dp_mode == "nvlink" and args.mode == "fast":
            try:
                step = FusedDPStep(ctx, d_x, d_y, n_total, Bg, world, rank, ipc=same_gpu)
                dp_used = "nvlink"
            except Exception as exc:  # symmetric memory unavailable: NCCL path
                dp_note = f"fused NVLink step unavailable ({type(exc).__name__}: {exc}); NCCL fallback"
                print(dp_note, file=sys.stderr)
            # every rank must take the same path: if the fused step could not be set up on ANY rank, all
            # ranks use NCCL (a rank running the fused kernel alone would wait for peers that never arrive)
            agree = torch.tensor([0.0 if step is not None else 1.0], dtype=torch.float64,
                                 device="cpu" if same_gpu else dev)
            dist.all_reduce(agree, op=dist.ReduceOp.MAX)
            if float(agree) > 0 and step is not None:
                step, dp_used = None, "nccl"
                dp_note = "fused NVLink step unavailable on another rank; NCCL fallback on every rank"
                print(dp_note, file=sys.stderr)
        if step is None:
            step = DeviceShardStep(ctx, d_x, d_y, n_total, Bg, world, rank, graph=not (args.no_graph or same_gpu))

        def epoch(e):
            step.epoch(d_p, 0.05, d_loss, e)
        launches_per_step = 1 if dp_used == "nvlink" else 2 * step.groups_per_epoch

    def all_max(v: float) -> float:  # max over ranks (a CPU tensor for gloo, device for NCCL)
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if same_gpu else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    def fused_failed(ok: bool) -> bool:
        """Did ANY rank's fused step fail -- an argument error (e.g. a shard beyond the clustered kernel's
        co-resident capacity) or a peer-wait watchdog trip?  Every rank takes part, so all agree."""
        try:
            step.check()
        except RuntimeError:
            ok = False
        return all_max(0.0 if ok else 1.0) > 0

    def run_protocol():
        # warm-up (not timed), then the timed protocol from init_params(42)
        reset()
        ok = True
        try:
            for w in range(args.warmup):
                epoch(w % max(args.steps, 1))
            torch.cuda.synchronize()
        except Exception as exc:  # noqa: BLE001 -- only the fused step can fail here (NCCL path: re-raised)
            if not (dp and dp_used == "nvlink"):
                raise
            print(f"fused NVLink step failed in warm-up: {type(exc).__name__}: {exc}", file=sys.stderr)
            ok = False
        if dp and dp_used == "nvlink" and fused_failed(ok):
            return None, None
        reset()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if dp:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            for s in range(args.steps):
                flush.fill_(float(s))  # L2 flush between timed steps, outside the event pair
                starts[s].record(stream)
                epoch(s)
                ends[s].record(stream)
            torch.cuda.synchronize()
        if dp:
            dist.barrier()
        if dp and dp_used == "nvlink" and fused_failed(True):  # a trip during the timed epochs: re-measure
            return None, None
        return sum(a.elapsed_time(b) for a, b in zip(starts, ends)), clk

    total_ms, clk = run_protocol()
    if total_ms is None:  # the fused path failed on some rank: every rank moves to NCCL together
        dp_used = "nccl"
        dp_note = "fused NVLink step failed (argument error or peer-wait watchdog); NCCL fallback"
        print(dp_note, file=sys.stderr)
        step = DeviceShardStep(ctx, d_x, d_y, n_total, Bg, world, rank, graph=not (args.no_graph or same_gpu))
        launches_per_step = 2 * step.groups_per_epoch
        total_ms, clk = run_protocol()
    if dp:
        total_ms = all_max(total_ms)
    losses = d_loss[: args.steps].cpu().numpy().tolist()
    value = args.steps * n_total / (total_ms / 1e3)

    # roofline of the dominant kernel (the persistent train kernel = the whole step)
    info = ctx.info()
    peaks = measured_peaks()
    max_mhz = peaks.get("sm_max_mhz", 1965.0)
    fp32_nominal = info["sm_count"] * FP32_LANES_PER_SM * 2 * max_mhz * 1e6 / 1e12
    ffma = measured_ffma_peak()
    fp32_peak = ffma["tflops"] if ffma else fp32_nominal
    flop_per_launch = n_per * FLOP_PER_TRAIN_IMAGE
    achieved = flop_per_launch / (total_ms / args.steps / 1e3) / 1e12
    clocks = clk.summary()

    traffic, traffic_src = (None, None) if dp else ncu_traffic(args.mode, B, n_per, world)
    result = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic: synth::make_set({n_total}, 1) (reference generator restated in C++), init_params(42)"
                + ("; each rank holds its static_chunk shards of every group" if dp else ""),
        "config": workload_config(args, world),
        "impl_config": dict(mode=args.mode, grid=args.grid or "auto",
                       dp_step=None if not dp else (
                           "fused: one clustered launch per epoch, fixed-point gradient slices added into the owning "
                           "GPU's accumulator over NVLink peer memory (no collective call)" if dp_used == "nvlink" else
                           "shard kernel + NCCL allreduce + sgd per group" +
                           ("" if args.no_graph else ", epoch replayed as one CUDA graph")),
                       dp_note=dp_note),
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp32_peak, "traffic": traffic,
                     "traffic_note": (f"DRAM bytes/launch from {traffic_src}" if traffic_src else
                                      "no committed ncu capture of this exact launch") +
                                     f"; algorithmic input bytes/launch = {n_per * 3136}",
                     "per_launch": f"{n_per} images x {FLOP_PER_TRAIN_IMAGE} algorithmic FLOP",
                     "peak_source": (f"measured FFMA peak {ffma['tflops']:.2f} TFLOP/s ({ffma['source']}); nominal "
                                     f"{fp32_nominal:.2f} = {info['sm_count']} SMs x 128 lanes x 2 x {max_mhz} MHz"
                                     if ffma else
                                     f"{info['sm_count']} SMs x 128 FP32 lanes x 2 x sm_max_mhz {max_mhz} "
                                     "(MEASURED_PEAKS.json clocks)") + "; FFMA-bound path (no HBM/tensor bound)",
                     "frac_of_nominal": achieved / fp32_nominal},
        "clocks": clocks,
        "epoch_mean_loss": losses,
    }
    gl = golden_losses()
    if gl and world == 1 and 1 <= args.steps <= len(gl) and n_per == 10000 and B == 100:
        # the timed run starts from init_params(42): its epochs are the protocol's first `steps` epochs
        rel = max(abs(a - b) / abs(b) for a, b in zip(losses, gl[:args.steps]))
        result["parity"] = {"epoch_loss_max_rel_vs_reference": rel, "tolerance": 1e-4, "epochs_compared": args.steps,
                            "bitwise": all("%.17g" % a == "%.17g" % b for a, b in zip(losses, gl[:args.steps]))}

    # end-to-end through the public host API with host buffers, H2D + D2H inside the timed region
    if not args.no_e2e:
        # The e2e input is the corpus as a user holds it before decoding: the pixel BYTES of
        # synth::make_digits (= the IDX payload), which the byte ingestion (tlb_train_u8) moves over the link
        # and converts on the device -- bit-identical to the fp32 images (checked below).
        pix_all, _ = synth_make_digits(n_total, 1)
        pixels = np.ascontiguousarray(pix_all[rows]) if dp else pix_all
        assert np.array_equal(pixels.astype(np.float32) / np.float32(255.0), images.reshape(pixels.shape))
        pin_x = torch.from_numpy(images).pin_memory()
        pin_u8 = torch.from_numpy(pixels).pin_memory()
        pin_y = torch.from_numpy(labels).pin_memory()
        px, pu8, py = pin_x.numpy(), pin_u8.numpy(), pin_y.numpy()
        # this box's pinned host->device bandwidth for the step's image bytes (the e2e ingestion bound)
        d_probe = torch.empty_like(pin_x, device=dev)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d_probe.copy_(pin_x, non_blocking=True)
        h0.record()
        for _ in range(3):
            d_probe.copy_(pin_x, non_blocking=True)
        h1.record()
        torch.cuda.synchronize()
        h2d_gbps = 3 * images.nbytes / (h0.elapsed_time(h1) * 1e-3) / 1e9
        del d_probe
        times = []
        if not dp:  # net::train on host bytes (tlb_train_u8): pixels/labels/params in, params + losses out
            def timed(fn, src):
                p = p0.copy()
                fn(p, src, py, rate=0.05, epochs=1, batch=B)  # warm-up (allocations)
                torch.cuda.synchronize()
                p, ts = p0.copy(), []
                for s in range(args.steps):
                    flush.fill_(float(s))
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    p, _ = fn(p, src, py, rate=0.05, epochs=1, batch=B)
                    ts.append(time.perf_counter() - t0)
                return ts
            times = timed(ctx.train_u8, pu8)
            f32_times = timed(ctx.train, px)
            api = ("tlb_train_u8 (net::train on the corpus bytes; device-side /255) on pinned host buffers, wall clock "
                   "per call")
            h2d = pixels.nbytes + labels.nbytes + 3898 * 4
            d2h = 3898 * 4 + 8
            e2e_launches = 2 * args.steps  # conversion + train kernel (+ the same again for the fp32 variant)
            result["e2e_f32"] = {"value": args.steps * n_total / sum(f32_times), "unit": "images/s",
                                 "h2d_bytes_per_step": images.nbytes + labels.nbytes + 3898 * 4, "d2h_bytes_per_step": d2h,
                                 "api": "tlb_train (net::train on fp32 images) on pinned host buffers"}
        else:  # every rank: its shards H2D, the data-parallel epoch, loss (+ params on rank 0) D2H
            pin_p = torch.from_numpy(np.pad(p0, (0, 6))).pin_memory()
            out_p = torch.empty(3904).pin_memory()
            out_l = torch.empty(1, dtype=torch.float64).pin_memory()
            d_u8 = torch.empty(pixels.shape, dtype=torch.uint8, device=dev)
            for s in range(args.warmup + args.steps):
                flush.fill_(float(s))
                torch.cuda.synchronize()
                dist.barrier()
                t0 = time.perf_counter()
                d_u8.copy_(pin_u8, non_blocking=True)
                ctx.pixels_to_images_device(d_u8.data_ptr(), pixels.size, d_x.data_ptr())
                d_y.copy_(pin_y, non_blocking=True)
                d_p.copy_(pin_p, non_blocking=True)
                epoch(0)
                out_l.copy_(d_loss[0:1], non_blocking=True)
                if rank == 0:
                    out_p.copy_(d_p, non_blocking=True)
                torch.cuda.synchronize()
                if s >= args.warmup:
                    times.append(time.perf_counter() - t0)
            api = (f"per rank: its shards (1/{world} of the corpus) as pinned bytes H2D + device /255 + params H2D, "
                   "the data-parallel epoch, epoch loss D2H (+ params D2H on rank 0); wall clock per step, max over ranks")
            h2d = world * (pixels.nbytes + labels.nbytes + 3904 * 4)
            d2h = world * 8 + 3904 * 4
            e2e_launches = (launches_per_step + 1) * args.steps
        e2e_s = sum(times)
        if dp:
            e2e_s = all_max(e2e_s)
        result["e2e"] = {"value": args.steps * n_total / e2e_s, "unit": "images/s",
                         "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "api": api,
                         "h2d_GBps_measured": h2d_gbps,
                         "call_ms": {"median": 1e3 * sorted(times)[len(times) // 2], "min": 1e3 * min(times),
                                     "max": 1e3 * max(times)}}
        result["gpu_launches"] += e2e_launches
        if not dp:
            cpp = cpp_e2e(args, n_total, B)
            if cpp is not None:
                result["e2e_cpp"] = cpp
                result["gpu_launches"] += args.steps

    if not args.no_cpu_baseline:
        if rank == 0:  # the reference's net::train on this box's host cores, a bounded sample
            v, meta = reference_epochs(n_per, 10.0, 3, min(B * world, n_per))
            result["cpu_baseline"] = {"value": v, "unit": "images/s", "cores": meta["cores"], "kind": "reference",
                                      "sample": f"{meta['epochs']} epoch(s) x {n_per} images at batch "
                                                f"{min(B * world, n_per)}, reference net::train (oracle/_ref) with "
                                                f"{meta['cores']} workers, {meta['seconds']:.1f} s",
                                      "cpu_model": cpu_model()}
            # the reference at one worker too (a bounded sample: 1 epoch of <= 2000 images)
            n1 = min(n_per, 2000)
            v1, meta1 = reference_epochs(n1, 1.0, 1, min(B * world, n1), workers=1)
            result["cpu_baseline_w1"] = {"value": v1, "unit": "images/s", "cores": 1, "kind": "reference",
                                         "sample": f"1 epoch x {n1} images at batch {min(B * world, n1)}, reference "
                                                   f"net::train with 1 worker, {meta1['seconds']:.1f} s"}
        if dp:
            dist.barrier()
    if real_stdout is not None:
        sys.stdout.flush()
        os.dup2(real_stdout, 1)
    if rank == 0:
        print(json.dumps(result), flush=True)
    ctx.close()
    if dp:
        dist.destroy_process_group()


def cpp_e2e(args, n, batch):
    """The same epoch through the C++ drop-in (tloom::net::train on a host MnistSet in pageable memory, as the
    reference's callers hold it), timed by tools/e2e_bench.cpp in its own process: wall clock per call,
    dataset H2D and parameters D2H inside every call."""
    exe = os.path.join(ROOT, "paper_1912_05234_b200", "bin", "tloom-e2e-bench")
    if not os.path.exists(exe):
        return None
    cmd = [exe, "--n", str(n), "--batch", str(batch), "--steps", str(args.steps), "--warmup", str(args.warmup),
           "--mode", args.mode]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        rec = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:  # reported, never fatal to the bench line
        return {"error": f"{type(e).__name__}: {e}"[:300]}
    return {"value": rec["images_per_s"], "unit": "images/s", "h2d_bytes_per_step": rec["h2d_bytes_per_step"],
            "d2h_bytes_per_step": rec["d2h_bytes_per_step"], "api": rec["api"], "call_ms": rec["call_ms"],
            "epoch_loss": rec["epoch_loss"]}


def measured_ffma_peak():
    """The FP32 FMA roofline measured on this pool's B200 (scripts/ffma_peak.cu): the best of the scalar FFMA
    and the packed fma.rn.f32x2 (FFMA2) runs (profiles/r2/ffma_peak_r2k.json, profiles/r2/ffma2_peak_r2k.json);
    MEASURED_PEAKS.json (driver-written) has HBM and bf16 only."""
    best, src = None, []
    for name in ("ffma_peak_r2k.json", "ffma2_peak_r2k.json", "ffma_peak_r2a.json"):
        try:
            with open(os.path.join(ROOT, "profiles", "r2", name)) as f:
                rec = json.load(f)
            v = float(rec["tflops_best"])
            src.append(f"{rec.get('what', name)} {v:.2f}")
            best = v if best is None else max(best, v)
        except Exception:
            continue
    if best is None:
        return None
    return {"tflops": best, "source": "max of measured FP32 FMA peaks (best of 20 each): " + ", ".join(src) +
            " (profiles/r2/)"}


def ensure_ranks(args) -> None:
    """--gpus N: one process per GPU.  Without a torchrun environment and N > 1, re-launch this command
    under torch.distributed.run (N local ranks, rendezvous on 127.0.0.1); inside one, WORLD_SIZE must be
    N -- a mismatch is an error, never a silent single-rank run."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus > 1:
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            # the ranks get this command's arguments through the environment: torchrun's own parser would
            # claim abbreviations of its options (--n -> --nnodes / --nproc-per-node ...)
            os.environ["TLB_BENCH_ARGV"] = json.dumps(sys.argv[1:])
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)]
            sys.stdout.flush()
            os.execv(sys.executable, cmd)
        return
    if int(world) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
        sys.exit(2)


def main():
    if "TLB_BENCH_ARGV" in os.environ and len(sys.argv) == 1:  # a rank spawned by ensure_ranks
        sys.argv[1:] = json.loads(os.environ["TLB_BENCH_ARGV"])
    args = parse()
    if args.n < args.batch:  # configs[3] sweeps: at least two SGD groups per epoch per GPU
        args.n = 2 * args.batch
    ensure_ranks(args)
    if args.plan:
        print(json.dumps({"rank": int(os.environ.get("RANK", "0")), "world": int(os.environ.get("WORLD_SIZE", "1")),
                          "local_rank": int(os.environ.get("LOCAL_RANK", "0")), "gpus": args.gpus,
                          "impl": args.impl, "batch_per_gpu": args.batch, "n_per_gpu": args.n}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
