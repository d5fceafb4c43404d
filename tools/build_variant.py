"""Build an experimental libvb.so variant with extra nvcc defines into tools/variants/
(A/B timing in one gpurun call: VB_LIBVB=tools/variants/<name>.so python bench.py ...).

usage: python tools/build_variant.py <name> -DVB_GATHER_U=8 ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16039_b200 import _build  # noqa: E402

if __name__ == "__main__":
    name, defines = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "tools", "variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.check_call([_build.NVCC, *_build.FLAGS, *defines, "-o", out, *_build.sources()])
    print(out)
