"""Dynamic instruction counts and stall samples per source line of one kernel:
    python tools/ncu_line_attr.py <source csv (ncu --page source --csv --print-source sass)> <cubin>
        <kernel substring in the cubin> <first csv line of the kernel section> <voxels> [top]
The cubin must be built from the profiled source with -lineinfo."""
import collections
import csv
import re
import subprocess
import sys

path, cubin, ksub, start, nvox = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), float(sys.argv[5])
top = int(sys.argv[6]) if len(sys.argv) > 6 else 25
rows = list(csv.reader(open(path)))[start - 1:]
h = rows[1]
ie, isrc, ia, ist = (h.index("Instructions Executed"), h.index("Source"), h.index("Address"),
                     h.index("Warp Stall Sampling (All Samples)"))
recs = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) < len(h):
        continue
    try:
        recs.append((int(r[ia], 16), int(r[ie] or 0), int(r[ist] or 0), r[isrc].strip()))
    except ValueError:
        pass
recs.sort()
base = recs[0][0]
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cur = line = None
o2l, o2i = {}, {}
for l in out.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m and cur and ksub in cur:
        o2l[int(m.group(1), 16)] = line
        o2i[int(m.group(1), 16)] = m.group(2)
mism = sum(1 for a, n, st, src in recs if o2i.get(a - base, "").split()[:1] != src.split()[:1])
print(f"opcode mismatches {mism}/{len(recs)}; total {sum(r[1] for r in recs) * 32 / nvox:.1f} instr/voxel")
byl, bys = collections.Counter(), collections.Counter()
for a, n, st, src in recs:
    k = o2l.get(a - base)
    byl[k] += n
    bys[k] += st
srcs = {}
for k, v in byl.most_common(top):
    txt = ""
    if k:
        if k[0] not in srcs:
            try:
                srcs[k[0]] = open(k[0]).read().splitlines()
            except OSError:
                srcs[k[0]] = []
        L = srcs[k[0]]
        txt = L[k[1] - 1].strip()[:70] if k[1] - 1 < len(L) else ""
    name = f"{k[0].split('/')[-1]}:{k[1]}" if k else "?"
    print(f"{v * 32 / nvox:6.1f}/vox stall {bys[k]:6d} {name:26s} {txt}")
