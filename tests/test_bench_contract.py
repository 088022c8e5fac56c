"""bench.py's reference arm runs on the CPU (the reference library compiled in oracle/_ref): its JSON line
keeps the driver contract (one line, the required keys, impl/reference fields).  Small workload."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtloom_ref.so")


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference library not built")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--n", "400"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "images/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_our_arm_json_line():
    """Our arm on the B200 (short run): one JSON line with the driver keys plus roofline (measured FP32 peak,
    ncu traffic), e2e through the C ABI on host bytes, e2e_cpp through the C++ drop-in, clocks, launch count,
    and the parity of the epoch losses against the reference's golden values."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "e2e_cpp", "clocks", "gpu_launches",
              "parity"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["value"] > 1e6
    r = d["roofline"]
    assert r["bound"] == "fp32" and 0 < r["frac"] < 1 and r["peak"] > 70 and r["traffic"] and r["traffic"] > 3e7
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e_cpp"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["parity"]["epoch_loss_max_rel_vs_reference"] <= 1e-4
