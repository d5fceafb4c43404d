#!/bin/bash
# A/B of lattice-kernel variants in one gpurun call: tools/ab_lattice.sh <variant> ...
# (variants built by tools/build_variant.py into tools/variants/; "base" = the in-tree libvb.so).
# Each variant: the lattice parity tests (bounded by timeout: a pipeline bug may hang), then the timing.
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then unset VB_LIBVB; else export VB_LIBVB=$PWD/tools/variants/$v.so; fi
  echo "== $v"
  timeout 300 python -m pytest tests/test_gpu_lattice.py -x -q -m gpu 2>&1 | tail -2
  timeout 120 python tools/time_lattice.py 128 2>&1 | tail -1
  timeout 120 python tools/time_lattice.py 128 2>&1 | tail -1
done
