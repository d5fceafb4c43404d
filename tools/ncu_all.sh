#!/bin/bash
# one ncu metric capture of every libvb kernel family (tools/prof_all.py; only the
# second, NVTX-marked call of each op is profiled); summary: tools/ncu_all_summary.py
mkdir -p gpurun_out
python tools/prof_all.py > gpurun_out/prof_all_plain.log 2>&1 || { echo "prof_all failed"; tail -5 gpurun_out/prof_all_plain.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
ncu --nvtx --nvtx-include "measured/" --metrics $M --clock-control none --csv --log-file gpurun_out/all_kernels.csv \
    python tools/prof_all.py > gpurun_out/ncu_all.log 2>&1
echo "ncu rc=$?"
