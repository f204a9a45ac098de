"""Builds the in-tree CUDA library ``libslbm_b200.so`` for sm_100a.

``python -m paper_2408_06880_b200.build`` (or ``__graft_entry__.build()``)
compiles every ``csrc/*.cu`` with nvcc in parallel and links one shared
library next to this file, so it travels with the repository snapshot to
the GPU box.  Objects are rebuilt only when a source or header is newer.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libslbm_b200.so")
OBJDIR = os.path.join(ROOT, "build", "obj")


def _nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is not None and spec.submodule_search_locations:
        base = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    # bit-exact parity with the reference's numpy arithmetic: no FMA contraction
    "-fmad=false",
    "-Xcompiler",
    "-fPIC",
    "-Xptxas",
    "-v",
    "--expt-relaxed-constexpr",
    "-Wno-deprecated-gpu-targets",
]


# Optional build variants (environment, read at build time):
#   SLBM_EXPERIMENTAL_PAIR=1  compile csrc/pair.cu (temporally blocked AA pair
#                             kernel, off by default and slower)
#   SLBM_PROBES=1             allow tuning knob 0 = 2 (memory-pattern probe)
# Objects of another variant are rebuilt (the variant is part of the stamp).
def _variant() -> list[str]:
    defs = []
    if os.environ.get("SLBM_EXPERIMENTAL_PAIR") == "1":
        defs.append("-DSLBM_WITH_PAIR")
    if os.environ.get("SLBM_PROBES") == "1":
        defs.append("-DSLBM_PROBES")
    return defs


def _sources() -> list[str]:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if "-DSLBM_WITH_PAIR" not in _variant():
        srcs = [s for s in srcs if os.path.basename(s) != "pair.cu"]
    return srcs


def _stamp_ok() -> bool:
    stamp = os.path.join(OBJDIR, "variant.txt")
    want = " ".join(_variant())
    have = open(stamp).read() if os.path.exists(stamp) else None
    if have != want:
        for o in glob.glob(os.path.join(OBJDIR, "*.o")):
            os.remove(o)
        with open(stamp, "w") as fh:
            fh.write(want)
        return False
    return True


def _newest_header() -> float:
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    hdrs += glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hdrs), default=0.0)


def _compile(src: str, inc: str, verbose: bool) -> str:
    obj = os.path.join(OBJDIR, os.path.basename(src).replace(".cu", ".o"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _newest_header()):
        return obj
    cmd = [_nvcc(), *ARCH, *FLAGS, *_variant(), "-I", inc, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    log = os.path.join(OBJDIR, os.path.basename(src) + ".ptxas.log")
    with open(log, "w") as fh:
        fh.write(res.stderr)
    if verbose:
        print(f"[build] {os.path.basename(src)}", file=sys.stderr)
    return obj


def build(verbose: bool = True, force: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    inc, libdir = _nccl_dirs()
    sources = _sources()
    if force:
        for o in glob.glob(os.path.join(OBJDIR, "*.o")):
            os.remove(o)
    relink = not _stamp_ok()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, inc, verbose), sources))
    newest = max(os.path.getmtime(o) for o in objs)
    if not relink and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    ncclso = os.path.join(libdir, "libnccl.so.2")
    link = [
        _nvcc(),
        *ARCH,
        "-shared",
        "-o",
        LIB,
        *objs,
        f"-L{libdir}",
        "-l:libnccl.so.2" if os.path.exists(ncclso) else "-lnccl",
        f"-Xlinker=-rpath,{libdir}",
        "-lcudart",
    ]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    if verbose:
        print(f"[build] linked {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
