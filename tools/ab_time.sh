#!/bin/bash
# timing only (knock-out variants give wrong results): tools/ab_time.sh <variant> ...
for v in "$@"; do
  if [ "$v" = base ]; then unset VB_LIBVB; else export VB_LIBVB=$PWD/tools/variants/$v.so; fi
  echo "== $v"; timeout 120 python tools/time_lattice.py 128 2>&1 | tail -1
done
