"""Build libnimg_moe.so in-tree with nvcc for sm_100a (no torch JIT cache).

    python -m paper_2604_12163_b200._build
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libnimg_moe.so")
SOURCES = ["capi.cu", "route_kernels.cu", "grouped_gemm_sm100.cu", "grouped_gemm_simt.cu",
           "block_kernels.cu", "stack_kernels.cu", "backward_kernels.cu",
           "grouped_gemm_bwd_sm100.cu", "router_i8.cu", "f64_kernels.cu", "split_kernels.cu"]
HEADERS = ["common.cuh", "nimg_internal.h", os.path.join("..", "..", "include", "nimg_moe.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr", "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """out / defines: variant builds for A/B experiments (tools/), e.g.
    build(out=".../libnimg_moe_x.so", defines=("NIMG_X=1",))."""
    lib = out or LIB
    if not force and not out and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        tag = ("_%d" % abs(hash((lib,) + tuple(defines)))) if out else ""
        obj = os.path.join(CSRC, os.path.splitext(src)[0] + tag + ".o")
        cmd = [NVCC, *FLAGS, *(f"-D{d}" for d in defines), "-c", os.path.join(CSRC, src), "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        for src, obj, r in ex.map(compile_one, SOURCES):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(obj)
    tmp = lib + ".tmp"
    # --no-undefined: an unresolved internal symbol fails the build, not the dlopen
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-cudart", "static", "-Xlinker", "--no-undefined"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
