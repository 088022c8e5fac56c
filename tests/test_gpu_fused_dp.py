"""Fused data parallelism over NVLink peer memory (tlb_train_dp_device via parallel.FusedDPStep).

Only one GPU is available to this build, so the multi-GPU protocol is exercised at world size 1 through
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
