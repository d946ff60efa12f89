"""Hot SASS lines of an ncu --page source --csv --print-source sass dump:
instructions executed, avg active threads, stall samples."""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie, src, samp, thr = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Avg. Threads Executed")
data = [(int(r[ie] or 0), r[src].strip(), int(r[samp] or 0), r[thr]) for r in rows[2:] if len(r) > ie]
tot = sum(d[0] for d in data)
tots = sum(d[2] for d in data)
print(f"total warp-inst {tot}  stall samples {tots}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if n:
    for i, (c, s, sm, t) in enumerate(data):
        if c * 1000 >= tot or sm * 200 >= tots:
            print(f"{i:5d} {c:11d} {sm:7d} thr={t:>5} {s}")
