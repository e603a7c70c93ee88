"""In-tree build of the CUDA library (sm_100a) and the C++ drop-in shim.

    python -m paper_2507_16165_b200.build        # or __graft_entry__.build()

Products (git-ignored, but they travel to the GPU box with the snapshot):
    paper_2507_16165_b200/libbhrt_b200.so   C ABI of include/bhrt_cuda.h
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libbhrt_b200.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: the kernels spell out every fused op with fma(); nothing else
# may be contracted, so integration arithmetic matches the oracle bit for bit
# (DESIGN.md §Parity).
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xptxas", "-v",
           "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-I" + os.path.join(ROOT, "include")]
SOURCES = ["trace_reference.cu", "trace_scene.cu", "table.cu", "shade.cu", "bhrt_cuda.cu",
           "fp64_peak.cu", "scene_text.cpp"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


DEBUG_LIB = os.path.join(PKG, "libbhrt_b200_debug.so")


def build(verbose: bool = False, force: bool = False, debug: bool = False) -> str:
    """libbhrt_b200.so; debug=True: libbhrt_b200_debug.so with device bounds
    checks (-DBHRT_DEBUG_BOUNDS), loaded by tests/test_gpu_debug_bounds.py."""
    target = DEBUG_LIB if debug else LIB
    flags = NVFLAGS + (["-DBHRT_DEBUG_BOUNDS"] if debug else [])
    tag = "_debug" if debug else ""
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "bhrt_cuda.h"))
    if force or _stale(target, deps):
        objs = []
        os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
        for src in SOURCES:
            obj = os.path.join(ROOT, "build", os.path.splitext(src)[0] + tag + ".o")
            cmd = [NVCC, *ARCH, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(obj)
        tmp = target + ".tmp"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, target)
    return target


REF = "/root/reference/proj"
DROPIN = os.path.join(PKG, "dropin")


def build_dropin(force: bool = False) -> bool:
    """Drop-in artefacts that compile against the reference's own headers
    and non-hot-path sources (only where /root/reference exists; the built
    files travel to the GPU box like the .so):

      dropin/libbhrt_render_b200.so   render.hpp surface over the C ABI
      dropin/bhrt_worker_b200         `bhrt worker` (BHRT protocol) on the GPU
      dropin/acceptance_b200          the reference's acceptance suite, its
                                      render.cpp replaced by render_shim.cpp
      dropin/bhrt_bench_b200          `bhrt bench`: the reference's sweep /
                                      CSV harness (bench.cpp) timing the GPU
    """
    if not os.path.isdir(os.path.join(REF, "src")):
        return False
    os.makedirs(DROPIN, exist_ok=True)
    shim = os.path.join(CSRC, "render_shim.cpp")
    worker = os.path.join(CSRC, "worker_main.cpp")
    benchm = os.path.join(CSRC, "bench_main.cpp")
    outs = [os.path.join(DROPIN, n) for n in
            ("libbhrt_render_b200.so", "bhrt_worker_b200", "acceptance_b200", "bhrt_bench_b200")]
    deps = [shim, worker, benchm, LIB, os.path.join(ROOT, "include", "bhrt_cuda.h")]
    if not force and all(not _stale(o, deps) for o in outs):
        return True
    cxx = ["g++", "-std=c++20", "-O2", "-fPIC", "-Wno-free-nonheap-object", "-include", "algorithm", "-I" + os.path.join(REF, "include"),
           "-I" + os.path.join(ROOT, "include")]
    # the reference's sources minus render.cpp (the replaced hot path)
    srcs = [os.path.join(REF, "src", f) for f in sorted(os.listdir(os.path.join(REF, "src")))
            if f.endswith(".cpp") and f != "render.cpp"]
    link = ["-L" + PKG, "-lbhrt_b200", "-Wl,-rpath," + PKG, "-Wl,-rpath,$ORIGIN/..", "-lpthread"]
    subprocess.run([*cxx, "-shared", "-o", outs[0], shim, *link], check=True)
    subprocess.run([*cxx, "-o", outs[1], worker, shim, *srcs, *link], check=True)
    subprocess.run([*cxx, f'-DBHRT_BINARY="{os.path.join("/root/repo", os.path.relpath(outs[1], ROOT))}"',
                    "-o", outs[2], os.path.join(REF, "tests", "acceptance.cpp"), shim, *srcs, *link],
                   check=True)
    subprocess.run([*cxx, "-o", outs[3], benchm, shim, *srcs, *link], check=True)
    return True


def build_oracle() -> None:
    """The CPU checker (oracle/liboracle.so) and, where /root/reference exists,
    the compiled reference (oracle/_ref). Test infrastructure, not product."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
    build(force="--force" in sys.argv, debug=True)
    build_dropin(force="--force" in sys.argv)
    build_oracle()
    print(LIB)
