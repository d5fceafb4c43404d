"""Summarise an ncu report (run here, no GPU): key SOL metrics + stall reasons."""
import csv, io, subprocess, sys

def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum", "launch__occupancy_limit_shared_mem",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]

if __name__ == "__main__":
    for vals, units in raw(sys.argv[1]):
        for k in KEYS:
            if k in vals:
                print("%-70s %s %s" % (k, vals[k], units.get(k, "")))
        stalls = sorted(((float(v), k) for k, v in vals.items()
                         if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio")
                         and v not in ("", "n/a")), reverse=True)[:8]
        for v, k in stalls:
            print("  stall %-60s %.2f" % (k.replace("smsp__average_warp_latency_issue_stalled_", ""), v))
        stalls = sorted(((float(v.replace(",", "")), k) for k, v in vals.items()
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and v not in ("", "n/a")), reverse=True)[:10]
        for v, k in stalls:
            print("  pcsamp %-60s %.0f" % (k.replace("smsp__pcsamp_warps_issue_stalled_", ""), v))
