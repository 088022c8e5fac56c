"""compute-sanitizer regression guard: racecheck (shared memory incl. DSMEM), memcheck and synccheck
(barrier / mbarrier phase use) over the
persistent train kernels (clustered fast, flat fast, EXACT) on a few images -- 0 hazards, 0 errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool", ["racecheck", "memcheck", "synccheck"])
def test_train_kernels_clean_under_sanitizer(tool):
    out = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "9", sys.executable,
                          os.path.join(ROOT, "scripts", "sanitize.py"), "--only",
                          "train_fast_cluster,train_fast_flat,train_exact"],
                         capture_output=True, text=True, timeout=600)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-4000:]
    assert log.count(" ok") >= 3
    if tool == "racecheck":
        assert "0 hazards displayed (0 errors, 0 warnings)" in log, log[-4000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in log, log[-4000:]


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("cfg", ["", "p2x320x2"])
@pytest.mark.parametrize("tool", ["racecheck", "memcheck", "synccheck"])
def test_batched_kernel_clean_under_sanitizer(tool, cfg):
    """batch_train.cu (and the batched inference kernel): the default configuration below 8k images (4 images x 640 threads, one CTA per SM)
    and the two-CTAs-per-SM one (forced), whose full grid runs the SM-pair work mapping."""
    env = dict(os.environ, TLB_BATCH_CFG=cfg) if cfg else dict(os.environ)
    out = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "9", sys.executable,
                          os.path.join(ROOT, "scripts", "sanitize.py"), "--only", "train_batched,train_batched_big,eval"],
                         capture_output=True, text=True, timeout=900, env=env)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-4000:]
    assert log.count(" ok") >= 3
    if tool == "racecheck":
        assert "0 hazards displayed (0 errors, 0 warnings)" in log, log[-4000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in log, log[-4000:]
