"""Build libtloom_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_1912_05234_b200.build          # incremental
    python -m paper_1912_05234_b200.build --force

Objects go to paper_1912_05234_b200/_build/, the library to paper_1912_05234_b200/lib/.  Both are
git-ignored and travel to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libtloom_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
          "-I" + CSRC]
CU_FLAGS = ARCH + COMMON + ["-Xptxas", "-v", "--expt-relaxed-constexpr"]

SOURCES = ["zhang_kernels.cu", "batch_train.cu", "infer_kernels.cu", "nn_ops.cu", "wide_kernels.cu", "wide_tc.cu", "synth_device.cu", "capi.cu",
           "host_data.cpp"]
# C++ mirror of the reference headers (include/tloom/*.hpp): plain host code, g++ -std=gnu++20
HOST_SOURCES = ["host/tensor.cpp", "host/runtime.cpp", "host/nn.cpp", "host/network.cpp", "host/mnist.cpp",
                "host/synth.cpp"]
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-std=gnu++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
             "-I" + os.path.join(CSRC, "host")]
HEADERS = ["tlb_common.cuh", "train_common.cuh", "zhang_step.cuh", "tlb_launch.h", "tlb_capi_internal.h", "wide_kernels.cuh"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, force: bool) -> tuple[str, str]:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, os.path.splitext(src)[0].replace("/", "_") + ".o")
    if src.startswith("host/"):
        hdeps = [path, os.path.join(ROOT, "include", "tloom_b200.h"), os.path.join(CSRC, "host", "device.hpp")]
        hdeps += [os.path.join(ROOT, "include", "tloom", h) for h in os.listdir(os.path.join(ROOT, "include", "tloom"))]
        if not force and not _stale(obj, hdeps):
            return obj, ""
        cmd = [CXX] + CXX_FLAGS + ["-c", path, "-o", obj]
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(f"g++ failed for {src}:\n{' '.join(cmd)}\n{out.stdout}\n{out.stderr}")
        return obj, out.stderr
    deps = [path, os.path.join(ROOT, "include", "tloom_b200.h")] + [os.path.join(CSRC, h) for h in HEADERS]
    if not force and not _stale(obj, deps):
        return obj, ""
    flags = CU_FLAGS if src.endswith(".cu") else ARCH + COMMON
    cmd = [NVCC] + flags + ["-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC] + COMMON + ["-x", "cu", "-c", path, "-o", obj] + ARCH
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{out.stdout}\n{out.stderr}")
    return obj, out.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    with ThreadPoolExecutor(max_workers=8) as ex:
        results = list(ex.map(lambda s: _compile(s, force), SOURCES + HOST_SOURCES))
    objs = [r[0] for r in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if force or _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{out.stdout}\n{out.stderr}")
    return LIB


def build_variant(tag: str, defines: list[str], sources: tuple[str, ...] = ("zhang_kernels.cu",)) -> str:
    """Developer A/B builds: the library with `sources` (default zhang_kernels.cu) compiled under extra -D
    flags, written to lib/variants/libtloom_b200_<tag>.so (select at run time with TLB_LIB=<path>)."""
    lib = build()
    vdir = os.path.join(OBJ, "variant_" + tag)
    os.makedirs(vdir, exist_ok=True)
    objs = []
    for src in sources:
        obj = os.path.join(vdir, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC] + CU_FLAGS + ["-D" + d for d in defines] + ["-c", os.path.join(CSRC, src), "-o", obj]
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(f"variant build failed:\n{out.stderr}")
        objs.append(obj)
    objs += [os.path.join(OBJ, os.path.splitext(src)[0].replace("/", "_") + ".o")
             for src in SOURCES + HOST_SOURCES if src not in sources]
    os.makedirs(os.path.join(LIBDIR, "variants"), exist_ok=True)
    vlib = os.path.join(LIBDIR, "variants", f"libtloom_b200_{tag}.so")
    out = subprocess.run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", vlib] + objs, capture_output=True,
                         text=True)
    if out.returncode != 0:
        raise RuntimeError(f"variant link failed:\n{out.stderr}")
    return vlib


TOOLS = {"tensorloom": "tools/tensorloom_cli.cpp", "tensorloom-datagen": "tools/datagen.cpp",
         "tloom-e2e-bench": "tools/e2e_bench.cpp"}
BINDIR = os.path.join(PKG, "bin")


def build_tools(force: bool = False) -> list[str]:
    """The reference's CLI tools (proj/tools/) rebuilt over the C++ mirror + libtloom_b200.so."""
    os.makedirs(BINDIR, exist_ok=True)
    outs = []
    for name, src in TOOLS.items():
        path = os.path.join(PKG, src)
        exe = os.path.join(BINDIR, name)
        deps = [path, LIB] + [os.path.join(ROOT, "include", "tloom", h) for h in os.listdir(os.path.join(ROOT, "include", "tloom"))]
        if force or _stale(exe, deps):
            cmd = [CXX, "-std=gnu++20", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"), path, "-o", exe,
                   "-L" + LIBDIR, "-ltloom_b200", "-Wl,-rpath,$ORIGIN/../lib", "-lpthread"]
            out = subprocess.run(cmd, capture_output=True, text=True)
            if out.returncode != 0:
                raise RuntimeError(f"tool build failed for {name}:\n{' '.join(cmd)}\n{out.stderr}")
        outs.append(exe)
    return outs


def build_stage_bench() -> str:
    """Developer micro-benchmark of the per-image stages (not part of the library)."""
    os.makedirs(OBJ, exist_ok=True)
    exe = os.path.join(OBJ, "stage_bench")
    cmd = [NVCC] + ARCH + COMMON + ["-Xptxas", "-v", "--expt-relaxed-constexpr", os.path.join(CSRC, "stage_bench.cu"),
                                    "-o", exe]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"stage_bench build failed:\n{out.stderr}")
    return exe


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_tools(force="--force" in sys.argv))
    if "--bench" in sys.argv:
        print(build_stage_bench())
