"""Stall samples and instruction counts of a kernel between its barrier-like instructions (BAR.SYNC,
SYNCS waits, DEPBAR) from an ncu report: python tools/ncu_phases.py <rep> [top-N sass]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if 'Instructions Executed' in r][0]
hdr, body = rows[hi], rows[hi + 1:]
tot = sum(int(r[2] or 0) for r in body)
print("sass", len(body), "inst", sum(int(r[5] or 0) for r in body), "samples", tot)
st = {hdr[j]: sum(int(r[j] or 0) for r in body) for j in range(29, 46)}
print("stalls:", sorted(st.items(), key=lambda x: -x[1])[:10])
marks = [i for i, r in enumerate(body) if ('BAR.SYNC' in r[1] or 'SYNCS' in r[1])]
cuts = [0] + [m + 1 for m in marks] + [len(body)]
for a, b in zip(cuts[:-1], cuts[1:]):
    s = sum(int(r[2] or 0) for r in body[a:b])
    n = sum(int(r[5] or 0) for r in body[a:b])
    if s * 200 < tot:
        continue
    stl = {hdr[j]: sum(int(r[j] or 0) for r in body[a:b]) for j in range(29, 46)}
    print("%5d-%5d samples %5d (%4.1f%%) inst %9d  %s | %s" % (a, b, s, 100 * s / tot, n, body[b - 1][1].strip()[:40],
          sorted(stl.items(), key=lambda x: -x[1])[:4]))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for i in sorted(range(len(body)), key=lambda i: -int(body[i][2] or 0))[:top]:
    r = body[i]
    rs = sorted(((int(r[j] or 0), hdr[j]) for j in range(29, 46)), reverse=True)[:2]
    print(i, r[2], r[5], r[1].strip()[:70], rs)
