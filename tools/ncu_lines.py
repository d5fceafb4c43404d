"""Per-source-line instruction counts / stall samples of one kernel in an ncu report (needs -lineinfo)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
SORT_STALL = len(sys.argv) > 3 and sys.argv[3] == "stall"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_ex = hdr.index("Instructions Executed")
start = rows.index(hdr) + 1
cur = None
per, ops, stalls = collections.OrderedDict(), collections.defaultdict(collections.Counter), collections.Counter()
for r in rows[start:]:
    if not r:
        continue
    if r[0] != "":
        try:
            cur = (int(r[0]), r[1][:80])
            per.setdefault(cur, 0)
        except ValueError:
            cur = None
        continue
    if cur is None:
        continue
    try:
        n = int(r[i_ex])
    except ValueError:
        continue
    per[cur] += n
    op = r[3].split()
    op = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
    ops[cur][op.split(".")[0]] += n
    stalls[cur] += int(r[4] or 0)
tot = sum(per.values())
print("total", tot, "stall samples", sum(stalls.values()))
for k, v in sorted(per.items(), key=lambda x: -(stalls[x[0]] if SORT_STALL else x[1]))[:top]:
    print("%4d %6.2f%% st%5d %-60s %s" % (k[0], 100 * v / tot, stalls[k], k[1][:60], dict(ops[k].most_common(4))))
