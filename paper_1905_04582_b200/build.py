"""Build libmds.so in-tree with nvcc for sm_100a (called by __graft_entry__.build()).

Each csrc/*.cu is one translation unit (the pass kernel is instantiated per
mode and precision in pass_m<MODE>_<prec>.cu), compiled in parallel to an
object, then linked into one shared library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmds.so")
ROOT = os.path.dirname(HERE)
OBJ = os.path.join(HERE, "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.inl")) + \
        glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(ROOT, "include", "*.h")) + [__file__]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, extra=(), out: str | None = None) -> str:
    """extra: additional nvcc flags (A/B variants, e.g. -DMDS_NO_FIRST_SPLIT) built to `out`."""
    lib = out or LIB
    if not force and not extra and out is None and not stale():
        return LIB
    objdir = OBJ if not extra else OBJ + "_" + "_".join(f.strip("-").replace("=", "") for f in extra)
    os.makedirs(objdir, exist_ok=True)
    srcs = sources()
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]

    def compile_one(so):
        src, obj = so
        cmd = [NVCC, *FLAGS, *extra, *(["-Xptxas", "-v"] if verbose else []), "-c", "-o", obj, src]
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, zip(srcs, objs)))
    tmp = lib + ".tmp%d" % os.getpid()
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                           "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [-v] [--variant NAME -DFLAG ...]  (variant -> libmds_ab_NAME.so)
    args = sys.argv[1:]
    if "--variant" in args:
        k = args.index("--variant")
        name, flags = args[k + 1], [a for a in args[k + 2:] if a.startswith("-D")]
        print(build(force=True, extra=flags, out=os.path.join(HERE, "libmds_ab_%s.so" % name)))
    else:
        build(force="--force" in args, verbose="-v" in args)
        print(LIB)
