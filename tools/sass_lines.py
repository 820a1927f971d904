"""Join ncu per-instruction SASS counts with source lines from the cubin's line table.

    python tools/sass_lines.py <ncu sass csv> <cubin> <kernel-substring> [top]

Offsets are taken relative to the first instruction of each kernel in the ncu export
and matched against `nvdisasm -g -c` offsets of the same function."""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def ncu_counts(path, ksub):
    rows = list(csv.reader(open(path)))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            secs.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    for s in secs:
        if ksub in s["name"]:
            hdr = s["rows"][0]
            ix = {h: i for i, h in enumerate(hdr)}
            out = []
            for r in s["rows"][1:]:
                if len(r) < len(hdr) or not r[ix["Address"]]:
                    continue
                try:
                    out.append((int(r[ix["Address"]], 16), float(r[ix["Instructions Executed"]] or 0),
                                float(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Source"]]))
                except ValueError:
                    pass
            return s["name"], out
    raise SystemExit("kernel not found")


def line_table(cubin, fn_mangled_sub):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    funcs, cur, line = {}, None, None
    for ln in txt.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = {}
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            line = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur is not None:
            funcs[cur][int(m.group(1), 16)] = line
    cands = [f for f in funcs if fn_mangled_sub in f]
    return funcs, cands


def main():
    path, cubin, ksub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    name, rows = ncu_counts(path, ksub)
    funcs, cands = line_table(cubin, sys.argv[5] if len(sys.argv) > 5 else ksub.split("<")[0])
    base = rows[0][0]
    best = None
    for f in cands:
        if len(funcs[f]) == len(rows):
            best = f
    best = best or (cands[0] if cands else None)
    print("kernel:", name[:100], "| cubin function:", best, "| n =", len(rows), len(funcs.get(best, {})))
    lt = funcs.get(best, {})
    agg = defaultdict(lambda: [0.0, 0.0])
    tot = sum(r[1] for r in rows)
    for addr, ie, ss, src in rows:
        key = lt.get(addr - base, ("?", 0))
        agg[key][0] += ie
        agg[key][1] += ss
    for (f, l), (ie, ss) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {ie / tot * 100:6.2f}%  stall {ss:7.0f}  {f}:{l}")


if __name__ == "__main__":
    main()
