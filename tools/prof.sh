#!/bin/bash
# one gpurun call: GPU tests, quick bench, then ncu launch list + one full capture of the top kernel.
# usage: tools/prof.sh <tag> [kernel-regex]
tag=${1:-r01}; kre=${2:-assemble_gather}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$tag.log 2>&1; tail -3 gpurun_out/gpu_tests_$tag.log
CMD="python bench.py --steps 20 --warmup 3 --quick --no-e2e --no-cpu"
$CMD > gpurun_out/bench_quick_$tag.json 2> gpurun_out/bench_quick_$tag.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$kre -s 3 -c 1 -o gpurun_out/prof_$tag -f $CMD > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu rc=$?"
cat gpurun_out/bench_quick_$tag.json
