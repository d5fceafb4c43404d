#!/bin/bash
# run one command under several library variants: tools/ab_run.sh "<command>" <variant> ...  ("base" = in-tree libvb.so)
cmd=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then unset VB_LIBVB; else export VB_LIBVB=$PWD/tools/variants/$v.so; fi
  echo "== $v"; timeout 600 bash -c "$cmd" 2>&1 | tail -4
done
