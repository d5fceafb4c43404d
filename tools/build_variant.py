"""Build an experimental libvb.so variant with extra nvcc defines into tools/variants/
(A/B timing in one gpurun call: VB_LIBVB=tools/variants/<name>.so python bench.py ...).

usage: python tools/build_variant.py <name> [--only lattice.cu,...] -DVB_LAT_R=10 ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16039_b200 import _build  # noqa: E402

if __name__ == "__main__":
    name, args = sys.argv[1], sys.argv[2:]
    only = None
    if args[:1] == ["--only"]:
        only, args = set(args[1].split(",")), args[2:]
    out = os.path.join(ROOT, "tools", "variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    print(_build.build(extra=args, out=out, only=only, objdir=os.path.join(_build.HERE, "build", "obj_" + name)))
