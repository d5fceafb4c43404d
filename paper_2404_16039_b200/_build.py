"""Build libvb.so (all CUDA sources, sm_100a) in-tree with nvcc.  No GPU needed.

Each source compiles to its own object in parallel (build/obj/), then one link."""
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvb.so")
OBJ = os.path.join(HERE, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "-Xptxas", "-warn-spills"]
LFLAGS = [*ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fPIC"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "vb.h")]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in sources() + _deps())


def build(force=False, verbose=False, extra=(), out=None, only=None, objdir=None):
    """extra/out/only/objdir: an experimental variant (tools/build_variant.py): the sources named in
    `only` (basenames; default all) compile with `extra` flags into objdir, the rest reuse the default
    objects, and the library is linked to `out`."""
    if out is None and not force and not extra and not stale():
        return LIB
    if out is not None:
        build(verbose=verbose)   # default objects up to date
    os.makedirs(OBJ, exist_ok=True)
    if objdir:
        os.makedirs(objdir, exist_ok=True)
    hdr_t = max(os.path.getmtime(p) for p in _deps())

    def obj(src):
        mine = out is None or only is None or os.path.basename(src) in only
        o = os.path.join(objdir if (out is not None and mine) else OBJ, os.path.basename(src)[:-3] + ".o")
        if out is not None and not mine:
            return o
        if force or extra or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(src), hdr_t):
            cmd = [NVCC, *CFLAGS, *extra, "-c", "-o", o + ".tmp", src]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
            os.replace(o + ".tmp", o)
        return o

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(obj, sources()))
    target = out or LIB
    tmp = target + ".tmp%d" % os.getpid()
    subprocess.check_call([NVCC, *LFLAGS, "-o", tmp, *objs])
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
