"""WORLD ranks of the fused data-parallel step on ONE GPU (driven by tests/test_gpu_fused_dp.py).

    python tests/_dp_ranks.py RANK WORLD PORT OUTDIR

Each process joins a WORLD-rank gloo process group, allocates its DP workspace and maps the peers'
(CUDA IPC handles exchanged over the process group: on the same device here instead of over NVLink),
and runs FusedDPStep epochs on its static_chunk of every global group -- the cross-rank protocol a
multi-GPU job runs: slice s's accumulator and arrival counter live on rank s % WORLD, system-scope
fixed-point adds and release/acquire counters, seq_base continuing across launches.  All ranks' kernels
must be co-resident on the one GPU, so the global batch is small (16 examples = two 8-CTA clusters per
rank).  Rank r writes its final parameters and epoch losses to OUTDIR/rank{r}.npz.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1912_05234_b200 import Context  # noqa: E402
from paper_1912_05234_b200.parallel import FusedDPStep  # noqa: E402
from paper_1912_05234_b200.runtime import init_params, synth_make_set  # noqa: E402

N, EPOCHS = 480, 3


def main() -> None:
    rank, world, port, outdir = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    batch = 16 * world
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", world_size=world, rank=rank)
    x, y = synth_make_set(N, 1)
    d_x, d_y = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    p = torch.zeros(3904, device=dev)
    p[:3898] = torch.from_numpy(init_params(42)).to(dev)
    loss = torch.zeros(EPOCHS, dtype=torch.float64, device=dev)
    with Context(0, mode="fast") as c:
        c.set_stream(torch.cuda.current_stream().cuda_stream)
        step = FusedDPStep(c, d_x, d_y, N, batch, world=world, rank=rank, timeout_s=5.0, ipc=True)
        for e in range(EPOCHS):
            step.epoch(p, 0.05, loss, e)
        torch.cuda.synchronize()
        step.check()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), params=p.cpu().numpy(), loss=loss.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
