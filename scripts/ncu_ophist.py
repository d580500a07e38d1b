"""Executed-instruction histogram by SASS opcode (and stall samples) of one kernel in an .ncu-rep.
usage: python scripts/ncu_ophist.py REPORT.ncu-rep [top] [kernel-name substring]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
want = sys.argv[3] if len(sys.argv) > 3 else None
agg = defaultdict(lambda: [0.0, 0.0])
h, ci, take, seen = None, None, False, False
for r in rows:
    if r and r[0] == "Kernel Name":
        if seen and take:
            break
        take = (want is None and not seen) or (want is not None and want in r[1])
        seen = seen or take
        h = None
        continue
    if h is None:
        h = r
        ci = {k: i for i, k in enumerate(h)}
        continue
    if not take or len(r) < len(h):
        continue
    toks = r[1].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith('@') and len(toks) > 1 else toks[0]
    op = op.split('.')[0]
    try:
        agg[op][0] += float(r[ci['Instructions Executed']])
        agg[op][1] += float(r[ci['# Samples']])
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1.0
for op, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{op:10s} {int(v[0]):>12d} {100 * v[0] / tot:5.1f}%  samples {int(v[1])}")
