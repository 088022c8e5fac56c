"""The reference's command-line tools rebuilt over the B200 library (paper_1912_05234_b200/tools/):
`tensorloom train|bench|eval` and `tensorloom-datagen` (proj/tools/tensorloom_cli.cpp, datagen.cpp).

CPU tests: argument handling and exit codes (2 usage, 3 FormatError, 4 other), datagen bytes against
the reference generator.  GPU tests (marked): train -> checkpoint -> eval round trip, checked against
the unmodified reference library (oracle/_ref): same accuracy, and the TLM1 checkpoint written by the
B200 CLI is read by the reference's own load_params and equals the reference-trained weights bit for bit.
"""
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1912_05234_b200", "bin")
CLI = os.path.join(BIN, "tensorloom")
DATAGEN = os.path.join(BIN, "tensorloom-datagen")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtloom_ref.so")

needs_tools = pytest.mark.skipif(not (os.path.exists(CLI) and os.path.exists(DATAGEN)),
                                 reason="tools not built (python -m paper_1912_05234_b200.build)")


def run(args, **kw):
    return subprocess.run(args, capture_output=True, text=True, timeout=600, **kw)


@pytest.fixture(scope="module")
def corpus(tmp_path_factory):
    d = tmp_path_factory.mktemp("idx")
    r = run([DATAGEN, "--out", str(d), "--train-count", "600", "--test-count", "300", "--seed", "5"])
    assert r.returncode == 0, r.stderr
    return d


def files(d):
    return ["--train-images", str(d / "train-images-idx3-ubyte"), "--train-labels", str(d / "train-labels-idx1-ubyte"),
            "--test-images", str(d / "t10k-images-idx3-ubyte"), "--test-labels", str(d / "t10k-labels-idx1-ubyte")]


@needs_tools
def test_datagen_matches_reference_generator(corpus, orc):
    """IDX files = big-endian header + synth::make_digits bytes (seed, and seed+1 for the test set)."""
    for name, n, seed in (("train", 600, 5), ("t10k", 300, 6)):
        raw = (corpus / f"{name}-images-idx3-ubyte").read_bytes()
        assert struct.unpack(">iiii", raw[:16]) == (2051, n, 28, 28)
        px, lab = orc.make_digits(n, seed)
        assert raw[16:] == px.tobytes()
        rl = (corpus / f"{name}-labels-idx1-ubyte").read_bytes()
        assert struct.unpack(">ii", rl[:8]) == (2049, n)
        assert np.array_equal(np.frombuffer(rl[8:], np.uint8), lab.astype(np.uint8))


@needs_tools
@pytest.mark.parametrize("args", [[], ["train"], ["nope"], ["train", "--epochs", "-1"], ["train", "--batch", "0"],
                                  ["eval", "--test-images", "x"], ["bench", "--bench-workers", "0,2"],
                                  ["train", "--bogus", "1"], ["train", "--mt", "65"], ["train", "--mode", "fp16"]])
def test_cli_usage_errors_exit_2(args, corpus):
    extra = files(corpus) if args and args[0] in ("train", "bench") and len(args) > 1 else []
    r = run([CLI] + args + extra)
    assert r.returncode == 2, (r.returncode, r.stderr)


@needs_tools
def test_cli_help_exit_0():
    r = run([CLI, "--help"])
    assert r.returncode == 0 and "train" in r.stdout and "bench" in r.stdout and "eval" in r.stdout


@needs_tools
def test_cli_format_errors_exit_3(tmp_path, corpus):
    """A missing checkpoint / a corrupt IDX file is a FormatError before any device work (exit 3)."""
    r = run([CLI, "eval", "--checkpoint", str(tmp_path / "missing.tlm"), "--test-images",
             str(corpus / "t10k-images-idx3-ubyte"), "--test-labels", str(corpus / "t10k-labels-idx1-ubyte")])
    assert r.returncode == 3, r.stderr
    bad = tmp_path / "bad-images"
    bad.write_bytes(b"\x00\x00\x08\x04" + b"\x00" * 12)
    args = files(corpus)
    args[1] = str(bad)
    r = run([CLI, "train", "--epochs", "1"] + args)
    assert r.returncode == 3, r.stderr


@pytest.mark.gpu
@needs_tools
@pytest.mark.parametrize("devices", [None, "0,0", "0,0,0,0"])
def test_cli_train_checkpoint_eval_vs_reference(tmp_path, corpus, devices):
    """EXACT mode: the CLI's trained weights (TLM1 checkpoint) equal the reference library's own training
    run bit for bit, the reference's load_params reads the file, and train/eval report the reference's
    accuracy -- on one device and through tloom::net::train over a multi-device context
    (TLOOM_B200_DEVICES: every group split over the devices, reduced across them every step)."""
    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built")
    from oracle import Reference
    ref = Reference()
    ck = tmp_path / "w.tlm"
    env = dict(os.environ)
    if devices:
        env["TLOOM_B200_DEVICES"] = devices
    r = run([CLI, "train", "--epochs", "2", "--batch", "50", "--limit-train", "600", "--limit-test", "300",
             "--checkpoint", str(ck)] + files(corpus), env=env)
    assert r.returncode == 0, r.stderr
    out = dict(line.split() for line in r.stdout.strip().splitlines())
    tr_x, tr_y = ref.load_set(str(corpus / "train-images-idx3-ubyte"), str(corpus / "train-labels-idx1-ubyte"), 600)
    te_x, te_y = ref.load_set(str(corpus / "t10k-images-idx3-ubyte"), str(corpus / "t10k-labels-idx1-ubyte"), 300)
    want_p = ref.init_params(42)
    want_p, _ = ref.train(tr_x, tr_y, want_p, rate=0.05, epochs=2, batch=50)
    got_p = ref.load_params(str(ck))  # the reference's own TLM1 reader
    assert np.array_equal(got_p.view(np.uint32), want_p.view(np.uint32))
    want_acc = ref.evaluate(want_p, te_x, te_y)[0]
    assert out["final_test_accuracy"] == "%.6f" % want_acc
    r = run([CLI, "eval", "--checkpoint", str(ck), "--limit-test", "300", "--test-images",
             str(corpus / "t10k-images-idx3-ubyte"), "--test-labels", str(corpus / "t10k-labels-idx1-ubyte")])
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == "test_accuracy %.6f" % want_acc


@pytest.mark.gpu
@needs_tools
def test_cli_bench_csv_and_determinism(corpus):
    r = run([CLI, "bench", "--epochs", "1", "--limit-train", "300", "--limit-test", "100", "--bench-workers", "1,4"]
            + files(corpus))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "workers,seconds,speedup_vs_1" and [l.split(",")[0] for l in lines[1:]] == ["1", "4"]
    assert "determinism: final params identical" in r.stderr


E2E = os.path.join(BIN, "tloom-e2e-bench")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(E2E), reason="tools not built")
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_cpp_e2e_tool_trains_the_protocol(mode):
    """tools/e2e_bench.cpp drives tloom::net::train on a host MnistSet (pageable memory: the bounce-slot
    ingestion) one epoch per call from init_params(42): its 10 epoch losses are the reference's golden
    protocol losses -- bitwise in EXACT mode, within the north-star 1e-4 in FAST mode."""
    import json
    with open(os.path.join(ROOT, "tests", "golden", "protocol.json")) as f:
        want = [float(v) for v in json.load(f)["epoch_mean_loss"]]
    r = subprocess.run([E2E, "--steps", "10", "--warmup", "0", "--mode", mode], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    rec = json.loads(r.stdout.strip().splitlines()[-1])
    got = rec["epoch_loss"]
    assert len(got) == 10 and rec["images_per_s"] > 0
    if mode == "exact":
        assert got == want, (got, want)
    else:
        assert np.allclose(got, want, rtol=1e-4, atol=0), (got, want)
