"""Opcode histogram (thread instructions per query) of an ncu SASS source dump:
python tools/sass_ops.py dump.csv QUERIES"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie, src = h.index("Instructions Executed"), h.index("Source")
thr = h.index("Thread Instructions Executed")
q = int(sys.argv[2])
c = Counter()
for r in rows[2:]:
    if len(r) > ie and r[ie]:
        tok = r[src].strip().split()
        op = tok[1] if tok[0].startswith("@") else tok[0]
        c[op.split(".")[0]] += int(r[thr])
tot = sum(c.values())
print(f"thread instructions per query: {tot / q:.1f}")
for k, v in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(f"  {k:10s} {v / q:6.2f}")
