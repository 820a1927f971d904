"""Hottest SASS instructions of one kernel by warp-stall samples (ncu --page source --csv --print-source sass).
Usage: python tools/ncu_src_hot.py src.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
ia, isrc, iall, ino = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Warp Stall Sampling (Not-issued Samples)")
recs = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        recs.append((int(r[iall] or 0), int(r[ino] or 0), r[ia], r[isrc]))
    except ValueError:
        pass
tot = sum(x[0] for x in recs)
print("total samples", tot)
byop = collections.Counter()
for a, n, ad, s in recs:
    byop[s.split()[0] if not s.startswith("@") else s.split()[1].split(".")[0]] += a
print("by opcode:", [(k, round(100 * v / tot, 1)) for k, v in byop.most_common(15)])
for a, n, ad, s in sorted(recs, reverse=True)[:top]:
    print(f"{100 * a / tot:5.1f}% {100 * n / tot:5.1f}% {ad} {s[:80]}")
