#!/bin/bash
# ncu --set full capture of the lattice kernel of one variant: tools/lat_ncu.sh <variant> <tag>
v=$1; tag=$2
if [ "$v" != base ]; then export VB_LIBVB=$PWD/tools/variants/$v.so; fi
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:assemble_lattice -s 2 -c 1 -o gpurun_out/lat_$tag -f python tools/lat_one.py 128 128 128 > gpurun_out/ncu_lat_$tag.log 2>&1; tail -2 gpurun_out/ncu_lat_$tag.log
