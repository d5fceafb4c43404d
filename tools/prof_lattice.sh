tag=${1:-r02}
CMD="python bench.py --steps 20 --warmup 3 --quick --no-e2e --no-cpu"
$CMD > gpurun_out/bench_quick_$tag.json 2> gpurun_out/bench_quick_$tag.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assemble_lattice -s 3 -c 1 -o gpurun_out/prof_$tag -f $CMD > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu rc=$?"
cut -c1-300 gpurun_out/bench_quick_$tag.json
