import re, statistics, sys
txt = open(sys.argv[1]).read()
for chunk in txt.split("RUN")[:-1][-1:]:
    recs = [tuple(int(x) for x in m.groups()) for m in re.finditer(r'LATPROF cta (\d+) sm (\d+) cycles (\d+) ns (\d+) g0 (\d+) g1 (\d+)', chunk)]
    cyc = [r[2] for r in recs]
    print(len(recs), "min", min(cyc), "mean", int(statistics.mean(cyc)), "max", max(cyc))
    recs.sort()
    for r in recs[::10] + recs[-4:]:
        print(r)
