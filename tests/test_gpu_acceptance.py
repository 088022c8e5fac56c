"""The reference's own release gate (proj/tests/acceptance.cpp + oracles.cpp, UNMODIFIED sources) compiled
against this repo's C++ headers (include/tloom/*.hpp) and linked to libtloom_b200.so, i.e. every
tloom::nn / tloom::net call inside it runs on the B200.  Built here by ``make -C oracle acceptance``
(the sources only exist in this container); the binary travels to the GPU box in oracle/_ref/."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(EXE), reason="acceptance_b200 not built (needs /root/reference at build time)")
@pytest.mark.parametrize("devices", [None, "0,0"])
def test_reference_acceptance_gate_on_b200(devices):
    """devices: TLOOM_B200_DEVICES -- the same gate through a multi-device context (net::train splits every
    group over the listed devices)."""
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_1912_05234_b200", "lib"))
    if devices:
        env["TLOOM_B200_DEVICES"] = devices
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    log_path = os.path.join(ROOT, "gpurun_out", "acceptance_b200%s.log" % ("_devices_" + devices.replace(",", "_")
                                                                            if devices else ""))
    # line-buffered straight into the log, so a stuck step is visible even when the timeout fires
    with open(log_path, "w") as f:
        try:
            rc = subprocess.run(["stdbuf", "-oL", "-eL", EXE], stdout=f, stderr=subprocess.STDOUT, timeout=180,
                                env=env).returncode
        except subprocess.TimeoutExpired:
            rc = None
    with open(log_path) as f:
        log = f.read()
    assert rc is not None, "acceptance gate timed out; partial log:\n" + log

    class _Out:
        stdout = log
        returncode = rc
    out = _Out()
    lines = [l for l in out.stdout.splitlines() if l[:1] == "A" and l[1:2].isdigit()]
    assert len(lines) == 7, log
    assert not [l for l in lines if ": FAIL" in l], log
    assert "ACCEPTANCE: 0 hard failure(s)" in out.stdout, log
    assert out.returncode == 0, log
