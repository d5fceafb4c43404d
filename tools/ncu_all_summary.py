"""Summarise gpurun_out/all_kernels.csv (tools/ncu_all.sh) into
profiles/<round>/all_kernels_<tag>.md: per launch, DRAM GB/s and its fraction of
the measured HBM peak, sectors/request, FP64 pipe and shared-memory utilisation.
usage: python tools/ncu_all_summary.py <tag> <round>"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", "all_kernels.csv"))))
    hdr = None
    launches = {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = int(d["ID"])
        L = launches.setdefault(key, {"name": d["Kernel Name"], "grid": d.get("Grid Size", ""),
                                      "block": d.get("Block Size", "")})
        try:
            L[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6451.5
    out = ["# ncu metrics of every libvb kernel family (%s)" % tag, "",
           "`tools/ncu_all.sh`: `ncu --nvtx --nvtx-include measured/ --metrics ... --clock-control none` over "
           "`tools/prof_all.py` (BASELINE shapes: config 2 page ops n = 2..4 with N = 2^20, config 3 icosphere "
           "L10, config 5 Kuhn 128^3 pattern and assembly, config 4 2D 2048^2, NEXT-1/2/3).  Each op runs once "
           "warm, then once profiled; the profiled launch is cold in L2 only as far as ncu's replay makes it.  "
           "GB/s = DRAM bytes (read + write, measured) / duration; frac = GB/s / %.1f (MEASURED_PEAKS.json "
           "hbm_gbs).  Kernels bound by on-chip work show a low DRAM fraction by design (DESIGN.md §3)." % peak,
           "",
           "| # | kernel | grid x block | us | DRAM MB | GB/s | frac | sectors/req | FP64 pipe % | smem wavefronts % | warps active % |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for i, (key, L) in enumerate(sorted(launches.items())):
        name = re.sub(r"\(.*$", "", L["name"]).replace("void ", "").replace("vb::", "").replace("<unnamed>::", "")
        name = name.replace("unnamed>::", "")
        us = L.get("gpu__time_duration.sum", 0) / 1e3
        dram = L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
        gbs = dram / (us * 1e-6) / 1e9 if us else 0
        req = L.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", 0)
        spr = L.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 0) / req if req else float("nan")
        out.append("| %d | `%s` | %s x %s | %.1f | %.1f | %.0f | %.3f | %.1f | %.1f | %.1f | %.1f |" % (
            i, name, L["grid"], L["block"], us, dram / 1e6, gbs, gbs / peak, spr,
            L.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0),
            L.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 0),
            L.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0)))
    path = os.path.join(ROOT, "profiles", rnd, "all_kernels_%s.md" % tag)
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")
    print(path, len(launches), "launches")


if __name__ == "__main__":
    main()
