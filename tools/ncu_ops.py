"""SASS opcode mix of the kernel in an ncu report: totals and per-unit (argv[2] units, e.g. warp-steps)."""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and "Instructions Executed" in r)
i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tot, by = 0, collections.Counter()
for r in rows[rows.index(hdr) + 1:]:
    try:
        n = int(r[i_ex])
    except (ValueError, IndexError):
        continue
    t = r[i_src].split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    by[op.split(".")[0]] += n
    tot += n
print("total %d  per unit %.1f" % (tot, tot / units))
for op, n in by.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print("%-10s %10d %5.1f%%  per unit %.1f" % (op, n, 100 * n / tot, n / units))
