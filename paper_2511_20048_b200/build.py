"""Build libspa.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2511_20048_b200.build [--force] [--verbose] [--variant NAME --defs "-DX=1 ..."]

Objects go to build/ (git-ignored); the shared library lands next to this file so that
gpurun snapshots carry it to the GPU box.  A variant (performance experiments) builds the
same sources with extra defines into libspa_NAME.so; SPA_LIB=libspa_NAME.so selects it at
load time (paper_2511_20048_b200/spa.py).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libspa.so")
BUILD = os.path.join(ROOT, "build", "spa")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # noqa: WPS433

        inc = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    except ImportError:
        pass
    for cand in ("/usr/include", "/usr/local/include", "/usr/local/cuda/include"):
        if os.path.exists(os.path.join(cand, "nccl.h")):
            return cand
    raise RuntimeError("nccl.h not found")


DEFS: list[str] = []


def _flags():
    return ["-O3", "-std=c++17", "-Xcompiler", "-fPIC,-Wall", "-lineinfo", *ARCH, *DEFS,
            "-I", os.path.join(ROOT, "include"), "-I", _nccl_include()]


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [NVCC, *_flags(), "-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(BUILD, os.path.basename(src) + ".log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    if verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, variant: str = "", defs: str = "") -> str:
    global BUILD, OUT, DEFS
    if variant:
        BUILD = os.path.join(ROOT, "build", "spa_" + variant)
        OUT = os.path.join(HERE, f"libspa_{variant}.so")
        DEFS = defs.split()
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "*.cu")))
    if force:
        for o in glob.glob(os.path.join(BUILD, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if force or not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("--defs", default="")
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.variant, a.defs))
