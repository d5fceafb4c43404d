"""Write the committed ncu evidence under profiles/ from gpurun_out/ (run here, no GPU).

usage: python tools/make_profile_summary.py <tag> <round> [--launches CSV] [--rep REP]...

* profiles/<round>/launches_<tag>.csv + launch_shares_<tag>.md: every launch of
  `bench.py --quick` with its device time (ncu --metrics gpu__time_duration.sum,
  cold-cache, serialised -- compare shares, not absolutes);
* profiles/<round>/<kernel>_<tag>.md: key metrics of one `ncu --set full`
  capture (DRAM bytes, throughput, occupancy, pipes, stall reasons);
* profiles/ncu_summary.json: dram bytes per launch per kernel (bench.py reads it
  for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory-unit throughput % (max unit)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared-memory wavefronts % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.sum", "FP64 warp instructions"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_shared_mem", "CTA limit by smem"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def ncu_csv(args):
    out = subprocess.check_output(["ncu", *args, "--csv"], stderr=subprocess.DEVNULL).decode()
    return list(csv.reader(io.StringIO(out)))


def sass_fp64_counts(rep):
    """Executed warp instructions of DFMA / DADD / DMUL (SASS source page) of a single-kernel report."""
    rows = ncu_csv(["-i", rep, "--page", "source", "--print-source=sass"])
    try:
        hdr = next(r for r in rows if "Instructions Executed" in r)
    except StopIteration:
        return None
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    out = {"dfma": 0, "dadd": 0, "dmul": 0}
    for r in rows[rows.index(hdr) + 1:]:
        try:
            n = int(r[i_ex])
        except (ValueError, IndexError):
            continue
        t = r[i_src].split()
        op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0].lower()
        if op in out:
            out[op] += n
    return out


def summarise_rep(rep, tag, outdir):
    rows = ncu_csv(["-i", rep, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    result = {}
    for r in rows[2:]:
        vals = dict(zip(hdr, r))
        name = vals.get("Kernel Name", "?")
        short = re.sub(r"^(void )?(vb::)?(<unnamed>::|unnamed>::)?", "", name).split("(")[0]
        lines = ["# ncu --set full: `%s` (%s)" % (short, tag), "",
                 "Report: `%s` (not committed; 4 MB).  Captured with `ncu --set full --clock-control none "
                 "--import-source on -k regex:<kernel> -s 3 -c 1` on `python bench.py --steps 20 --warmup 3 "
                 "--quick --no-e2e --no-cpu` (tools/prof.sh)." % os.path.basename(rep), "",
                 "| metric | value | unit |", "|---|---|---|"]
        for k, label in KEYS:
            if k in vals:
                lines.append("| %s (`%s`) | %s | %s |" % (label, k, vals[k], units[hdr.index(k)]))
        stalls = sorted(((float(v.replace(",", "")), k) for k, v in vals.items()
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
                         and v not in ("", "n/a")), reverse=True)[:8]
        if stalls:
            lines += ["", "Top warp-stall samples:", ""]
            for v, k in stalls:
                lines.append("- %s: %d" % (k.replace("smsp__pcsamp_warps_issue_stalled_", ""), v))
        unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(vals["dram__bytes_read.sum"].replace(",", "")) * unit_scale[units[hdr.index("dram__bytes_read.sum")]]
        wr = float(vals["dram__bytes_write.sum"].replace(",", "")) * unit_scale[units[hdr.index("dram__bytes_write.sum")]]
        result[short] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                         "duration": vals.get("gpu__time_duration.sum"), "tag": tag}
        ops = sass_fp64_counts(rep)
        if ops:
            result[short].update(ops)   # warp-level DFMA / DADD / DMUL executed (x 32 lanes ~ thread ops)
        with open(os.path.join(outdir, "%s_%s.md" % (re.sub(r"[^A-Za-z0-9_]+", "_", short).strip("_"), tag)), "w") as f:
            f.write("\n".join(lines) + "\n")
    return result


def summarise_launches(path, tag, outdir):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"^(void )?(vb::)?(<unnamed>::)?", "", r[ik]).split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = ["# Launch list `%s`" % tag, "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over `python bench.py --steps 20 --warmup 3 "
             "--quick --no-e2e --no-cpu`: the one-time plan build (fem_p1_pattern kernels) followed by 23 "
             "fem_p1_assemble launches (3 warm-up + 20 timed).  Cold-cache, serialised: compare shares.", "",
             "| launches | total us | share | kernel |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append("| %d | %.1f | %.1f%% | `%s` |" % (v[0], v[1] / 1e3, 100 * v[1] / tot, k))
    with open(os.path.join(outdir, "launch_shares_%s.md" % tag), "w") as f:
        f.write("\n".join(lines) + "\n")
    subprocess.check_call(["cp", path, os.path.join(outdir, "launches_%s.csv" % tag)])


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    outdir = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(outdir, exist_ok=True)
    args = sys.argv[3:]
    summary_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {"kernels": {}}
    i = 0
    while i < len(args):
        if args[i] == "--launches":
            summarise_launches(args[i + 1], tag, outdir)
        elif args[i] == "--rep":
            summary["kernels"].update(summarise_rep(args[i + 1], tag, outdir))
        i += 2
    with open(summary_path, "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
