"""bench.py's multi-GPU plumbing on CPU (no GPU work): `--gpus N` launches N ranks (one process per GPU, a
127.0.0.1 rendezvous), a WORLD_SIZE that disagrees with --gpus is an error (never a silent one-rank run),
and each rank's shard layout covers every SGD group's static_chunk (runtime.cpp:138-145) exactly once."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=e, timeout=300, cwd=ROOT)


def test_gpus_2_spawns_two_ranks():
    out = run(["--gpus", "2", "--plan", "--batch", "1024", "--n", "4096"])
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 and d["gpus"] == 2 for d in lines)
    assert sorted(d["local_rank"] for d in lines) == [0, 1]
    assert all(d["batch_per_gpu"] == 1024 and d["n_per_gpu"] == 4096 for d in lines)


def test_world_size_mismatch_is_an_error():
    out = run(["--gpus", "4", "--plan"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode == 2 and "WORLD_SIZE=2" in out.stderr


def test_reference_arm_plan_and_shard_rows():
    sys.path.insert(0, ROOT)
    import bench
    from paper_1912_05234_b200.parallel import groups, static_chunk
    for n_per, B, world in ((10000, 100, 4), (1030, 100, 3), (2048, 1024, 2), (7, 5, 8)):
        n_total, Bg = n_per * world, B * world
        seen = np.zeros(n_total, int)
        for r in range(world):
            rows = bench.shard_rows(n_total, Bg, world, r)
            seen[rows] += 1
            # the shard of group g starts at local row g * ceil(Bg / world) (tlb_ctx_set_shard_layout)
            stride = -(-Bg // world)
            off = 0
            for g, (start, m) in enumerate(groups(n_total, Bg)):
                lo, hi = static_chunk(m, world, r)
                if hi > lo:
                    assert off == g * stride
                    assert list(rows[off:off + hi - lo]) == list(range(start + lo, start + hi))
                off += hi - lo
        assert np.all(seen == 1)
