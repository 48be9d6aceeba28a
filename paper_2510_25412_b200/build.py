"""Build the in-tree C-ABI library paper_2510_25412_b200/libkvfs.so (host control plane in C++17 with g++,
data plane in CUDA for sm_100a with nvcc, cudart linked statically so the library loads without a GPU).

    python -m paper_2510_25412_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libkvfs.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter"]
NVFLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                  "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _sources():
    cc = sorted(glob.glob(os.path.join(CSRC, "host", "*.cc")))
    cu = sorted(glob.glob(os.path.join(CSRC, "cuda", "*.cu")))
    return cc, cu


def _headers():
    return (glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True)
            + glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
            + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _obj(src, out_dir):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(out_dir, rel + ".o")


def _compile(src, force, hdr_mtime, out_dir=OUT_DIR, defines=()):
    obj = _obj(src, out_dir)
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj, ""
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + ["-D" + d for d in defines] + ["-c", src, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-I" + os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB, out_dir: str = OUT_DIR) -> str:
    """Build `lib` (default: the in-tree libkvfs.so).  `defines` (e.g. KVFS_EXP_EMU=2) and another
    `lib`/`out_dir` are for tuning experiments only (loaded via KVFS_LIB_PATH)."""
    LIB = lib
    os.makedirs(out_dir, exist_ok=True)
    cc, cu = _sources()
    hdr_mtime = max([os.path.getmtime(h) for h in _headers()] + [0.0])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, hdr_mtime, out_dir, defines), cc + cu))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print(f"--- {os.path.basename(o)}\n{log}")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
