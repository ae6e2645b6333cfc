"""Builds libdllm.so in-tree with nvcc for sm_100a (no torch extension).

    python -m paper_2512_17077_b200.build        (or __graft_entry__.build())

Each .cu is compiled to an object in parallel, then linked into
paper_2512_17077_b200/libdllm.so (static cudart, -lineinfo for ncu).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
TRACE = os.environ.get("DLLM_TRACE_BUILD") == "1"       # dev: timestamped refresh kernel
VARIANT = os.environ.get("DLLM_VARIANT", "")              # dev: extra -D flags, e.g. "DLLM_POLY_PAIRS=2"
_tag = ("_trace" if TRACE else "") + ("_" + VARIANT.replace("=", "").replace(",", "_") if VARIANT else "")
BUILD = os.path.join(HERE, "_build" + _tag)
LIB = os.path.join(HERE, f"libdllm{_tag}.so")
EXTRA = (["-DDLLM_TRACE"] if TRACE else []) + [f"-D{v}" for v in VARIANT.split(",") if v]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(HERE, "..", "include")]
SOURCES = ["dllm_api.cu", "select.cu", "reuse_ws.cu", "reuse_tc.cu", "reuse_grp.cu", "lmhead.cu", "refresh_mma.cu", "refresh_tc2.cu"]


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    srcp = os.path.join(CSRC, src)
    deps = [srcp] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "dllm.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", srcp, "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB, *objs, "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
