"""Per-CTA cycles of the VB_LAT_PROF build (tools/latprof_run.py output): balance and cycles per tile-layer by tile."""
import collections
import re
import statistics
import sys

txt = open(sys.argv[1]).read()
NK = int(sys.argv[2]) if len(sys.argv) > 2 else 129
chunk = txt.split("RUN")[-2]
recs = sorted(tuple(int(x) for x in m.groups())
              for m in re.finditer(r'LATPROF cta (\d+) sm (\d+) cycles (\d+) ns (\d+) g0 (\d+) g1 (\d+)', chunk))
cyc = [r[2] for r in recs]
print(len(recs), "CTAs: min", min(cyc), "mean", int(statistics.mean(cyc)), "max", max(cyc),
      "max/mean %.3f" % (max(cyc) / statistics.mean(cyc)))
by = collections.defaultdict(list)
for cta, sm, c, _, g0, g1 in recs:
    t0, t1 = g0 // NK, (g1 - 1) // NK
    if t0 == t1:
        by[t0].append(c / (g1 - g0))
    if "-v" in sys.argv:
        print(cta, sm, c, g1 - g0, "tiles", t0, t1, "%.0f cyc/layer" % (c / (g1 - g0)))
print("cycles per layer of the CTAs inside one tile:", {t: int(statistics.mean(v)) for t, v in sorted(by.items())})
worst = sorted(recs, key=lambda r: -r[2])[:8]
print("slowest:", [(r[0], r[2], r[4] // NK, (r[5] - 1) // NK, r[5] - r[4]) for r in worst])
best = sorted(recs, key=lambda r: r[2])[:8]
print("fastest:", [(r[0], r[2], r[4] // NK, (r[5] - 1) // NK, r[5] - r[4]) for r in best])
