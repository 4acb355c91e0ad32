"""Build libisoquant.so in-tree with nvcc for sm_100a.

Compiles every translation unit under csrc/ in parallel (one per
(variant, dtype) template block, plus the C ABI and the host parameter
builder) and links a self-contained shared library (static cudart) next to
this file.  Rebuilds only what changed.  No torch extension machinery: the
library has a plain C ABI (include/isoquant.h).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJDIR = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libisoquant.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", INCLUDE, "-I", CSRC] + ARCH


def _sources():
    out = []
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cu", ".cpp")):
            out.append(os.path.join(CSRC, f))
    return out


def _headers():
    hs = [os.path.join(INCLUDE, "isoquant.h")]
    for f in os.listdir(CSRC):
        if f.endswith((".h", ".cuh", ".inc")):
            hs.append(os.path.join(CSRC, f))
    return hs


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str, extra: list[str], verbose: bool, objdir: str = OBJDIR) -> str:
    obj = os.path.join(objdir, os.path.basename(src) + ".o")
    deps = [src] + _headers()
    if os.path.exists(obj) and os.path.getmtime(obj) >= _newest(deps):
        return obj
    cmd = [NVCC] + FLAGS + extra + ["-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False, jobs: int | None = None, extra: list[str] | None = None,
          lib: str = LIB, objdir: str = OBJDIR, only: list[str] | None = None) -> str:
    """Compile (incrementally) and link libisoquant.so; return its path.
    ``extra``/``lib``/``objdir`` build tuning variants (e.g. -DIQ_NWC=7) side by
    side for experiments; the product is the default build.  ``only``: the
    source basenames compiled with ``extra`` into ``objdir``; every other
    translation unit links the product build's object (a variant of one
    kernel family rebuilds one file)."""
    os.makedirs(objdir, exist_ok=True)
    extra = list(extra or [])
    srcs = _sources()
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))

    def one(src):
        if only is not None and os.path.basename(src) not in only:
            return _compile(src, [], verbose, OBJDIR)
        return _compile(src, extra, verbose, objdir)

    with ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(one, srcs))
    if not os.path.exists(lib) or os.path.getmtime(lib) < _newest(objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-cudart", "static"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
