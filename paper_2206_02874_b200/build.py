"""Build libtcx.so in-tree (nvcc, sm_100a only).  `python -m paper_2206_02874_b200.build`."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libtcx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

# no --use_fast_math, no -ftz: the epilogue's FP32 C-add must stay RNE with subnormals
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=true",
         "-I" + os.path.join(HERE, "..", "include")]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(HERE, "..", "include", "tcx.h"))
    return max(os.path.getmtime(h) for h in hs)


# debug variant: same sources, bounded barrier waits (ptx.cuh TCX_WATCHDOG) and the fault-injection
# hook of tcx_gemm_opts.reserved[0]; a separate library, never loaded unless TCX_LIB_PATH names it
DEBUG_LIB = os.path.join(HERE, "libtcx_debug.so")
DEBUG_FLAGS = ["-DTCX_WATCHDOG=1"]


def _compile(src, extra, build_dir=BUILD, force=False):
    obj = os.path.join(build_dir, os.path.basename(src) + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _headers_mtime()) and not force:
        return obj
    cmd = [NVCC] + FLAGS + extra + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False, extra=None, debug: bool = False) -> str:
    build_dir = os.path.join(BUILD, "debug") if debug else BUILD
    lib_path = DEBUG_LIB if debug else LIB
    os.makedirs(build_dir, exist_ok=True)
    extra = list(extra or [])
    flags = extra + (DEBUG_FLAGS if debug else [])
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, flags, build_dir, bool(extra)), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(lib_path) or os.path.getmtime(lib_path) < newest or extra:
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib_path] + objs + ["-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(lib_path)
    return lib_path


if __name__ == "__main__":
    args = sys.argv[1:]
    dbg = "--debug" in args
    build(verbose=True, extra=[a for a in args if a != "--debug"], debug=dbg)
