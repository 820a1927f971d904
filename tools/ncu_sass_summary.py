"""Summarise an ncu --page source --print-source=sass CSV (one or more kernels):
instructions executed and stall samples by opcode, plus the hottest instructions.
Usage: python tools/ncu_sass_summary.py f.csv [top]"""
import csv
import sys
from collections import defaultdict


def sections(rows):
    cur = None
    for r in rows:
        if r and r[0] == "Kernel Name":
            if cur:
                yield cur
            cur = {"name": r[1], "rows": []}
        elif cur is not None:
            cur["rows"].append(r)
    if cur:
        yield cur


def summarise(sec, top):
    rows = sec["rows"]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    by_op = defaultdict(lambda: [0.0, 0.0])
    lines = []
    tot_i = tot_s = 0.0
    for r in rows[1:]:
        if len(r) < len(hdr) or not r[ix["Address"]]:
            continue
        try:
            ie = float(r[ix["Instructions Executed"]] or 0)
            ss = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        src = r[ix["Source"]].strip()
        toks = src.split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
        op = op.split(".")[0]
        by_op[op][0] += ie
        by_op[op][1] += ss
        tot_i += ie
        tot_s += ss
        lines.append((ss, ie, src))
    print(f"== {sec['name'][:100]}\n   warp-instructions {tot_i:.4e}, stall samples {tot_s:.0f}")
    for op, (ie, ss) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"   {op:12s} inst {ie / max(tot_i, 1) * 100:6.2f}%  stall {ss / max(tot_s, 1) * 100:6.2f}%")
    print("   hottest (stall samples):")
    for ss, ie, src in sorted(lines, reverse=True)[:top]:
        print(f"   {ss:8.0f} {ie:12.0f} {src[:90]}")


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    for sec in sections(rows):
        summarise(sec, top)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
