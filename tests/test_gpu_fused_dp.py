"""Fused data parallelism over NVLink peer memory (tlb_train_dp_device via parallel.FusedDPStep).

Only one GPU is available to this build: the protocol runs at world size 1 through
a real torch symmetric-memory workspace and process group: the slice owners, the system-scope fixed-point
adds, the per-slice arrival counters continuing across launches (seq_base) and the watchdog word all run
the code path a multi-GPU job runs.  The result must be bitwise identical to the single-GPU clustered
kernel (integer accumulation is order-independent) and within the tolerance of the reference."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import torch
    import torch.distributed as dist
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29631", world_size=1, rank=0,
                                device_id=torch.device("cuda:0"))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("n,batch", [(1000, 100), (1050, 100), (640, 64)])
def test_fused_dp_world1_equals_clustered_kernel(pg, n, batch):
    import torch
    from paper_1912_05234_b200 import Context
    from paper_1912_05234_b200.parallel import FusedDPStep
    from paper_1912_05234_b200.runtime import init_params, synth_make_set
    dev = torch.device("cuda:0")
    x, y = synth_make_set(n, 1)
    d_x, d_y = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    p0 = torch.zeros(3904, device=dev)
    p0[:3898] = torch.from_numpy(init_params(42)).to(dev)
    with Context(0, mode="fast") as c:
        s = torch.cuda.current_stream()
        c.set_stream(s.cuda_stream)
        ref_p, ref_l = p0.clone(), torch.zeros(3, dtype=torch.float64, device=dev)
        for e in range(3):
            c.train_device(d_x.data_ptr(), d_y.data_ptr(), n, ref_p.data_ptr(), 0.05, e, 1, batch, ref_l.data_ptr())
        step = FusedDPStep(c, d_x, d_y, n, batch, world=1, rank=0)
        got_p, got_l = p0.clone(), torch.zeros(3, dtype=torch.float64, device=dev)
        for e in range(3):  # three launches: the counters and buffer phase continue (seq_base)
            step.epoch(got_p, 0.05, got_l, e)
        torch.cuda.synchronize()
        step.check()
    assert torch.equal(got_p, ref_p)
    assert torch.equal(got_l, ref_l)
    assert step.seq == 3 * ((n + batch - 1) // batch)


@pytest.mark.parametrize("world", [2, 4])
def test_fused_dp_ranks_one_gpu_equal_single_gpu(tmp_path, world):
    """WORLD processes run the fused data-parallel protocol against each other on the one GPU (CUDA IPC
    mapped workspaces, gloo process group, system-scope atomics across processes; slice s owned by rank
    s % WORLD): every rank must end with identical parameters and losses, bitwise equal to the
    single-GPU clustered kernel on the same global groups (each rank's static_chunk of a group is two
    clusters' worth of examples, the same cluster partials as the single-GPU run)."""
    import socket
    import subprocess
    import sys

    import torch
    from paper_1912_05234_b200 import Context
    from paper_1912_05234_b200.runtime import init_params, synth_make_set
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = os.path.join(root, "tests", "_dp_ranks.py")
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    env = dict(os.environ, NCCL_DEBUG="WARN")
    procs = [subprocess.Popen([sys.executable, script, str(r), str(world), str(port), str(tmp_path)], cwd=root,
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = []
    for pr in procs:
        try:
            outs.append(pr.communicate(timeout=240)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for pr, out in zip(procs, outs):
        assert pr.returncode == 0, out[-3000:]
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    r0 = res[0]
    for r in res[1:]:
        assert np.array_equal(r0["params"], r["params"]) and np.array_equal(r0["loss"], r["loss"])

    n, batch, epochs = 480, 16 * world, 3
    dev = torch.device("cuda:0")
    x, y = synth_make_set(n, 1)
    d_x, d_y = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    p = torch.zeros(3904, device=dev)
    p[:3898] = torch.from_numpy(init_params(42)).to(dev)
    loss = torch.zeros(epochs, dtype=torch.float64, device=dev)
    with Context(0, mode="fast") as c:
        c.set_stream(torch.cuda.current_stream().cuda_stream)
        for e in range(epochs):
            c.train_device(d_x.data_ptr(), d_y.data_ptr(), n, p.data_ptr(), 0.05, e, 1, batch, loss.data_ptr())
        torch.cuda.synchronize()
    assert np.array_equal(r0["params"], p.cpu().numpy())
    assert np.array_equal(r0["loss"], loss.cpu().numpy())
