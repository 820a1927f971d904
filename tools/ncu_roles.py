"""Instructions / stall samples of the fused LNCC kernel by warp role (sampler / moment /
waits), from an ncu source page and the cubin it was built from:
    python tools/ncu_roles.py src.csv cubin kernel-substring voxels"""
import collections
import csv
import re
import subprocess
import sys

path, cubin, ksub, nvox = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
src = open(re.sub(r"\.cubin$", "", cubin) and "/root/repo/paper_2509_25044_b200/csrc/step_lncc3.cu").read().splitlines()
# role boundaries from the source itself
def find(pat):
    return next(i + 1 for i, l in enumerate(src) if re.search(pat, l))
s_rows = find(r"void sampler_rows\(")
s_old = find(r"void sampler_warps\(")
m0 = find(r"float moment_warps\(")
k0 = find(r"k_lncc_fused\(const __grid_constant__")
rows = list(csv.reader(open(path)))
h = rows[1]
ie, ia, ist = h.index("Instructions Executed"), h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) < len(h):
        continue
    try:
        recs.append((int(r[ia], 16), int(r[ie] or 0), int(r[ist] or 0)))
    except ValueError:
        pass
recs.sort()
base = recs[0][0]
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cur = line = None
o2l = {}
for l in out.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m and cur and ksub in cur:
        o2l[int(m.group(1), 16)] = line


def role(k):
    if not k:
        return "?"
    f, n = k
    if f == "ffdp_common.cuh":
        return "sampler (common)"
    if f != "step_lncc3.cu":
        return f"intrinsics ({f})"
    if n < s_old - 1 and n > 100 and n < 200:
        return "helpers (mbar/quant)"
    if s_old <= n < s_rows:
        return "sampler (positions)"
    if s_rows <= n < m0:
        return "sampler (rows)"
    if m0 <= n < k0:
        return "moment"
    return "kernel/helpers"


I, S = collections.Counter(), collections.Counter()
for a, n, st in recs:
    r = role(o2l.get(a - base))
    I[r] += n
    S[r] += st
tot = sum(S.values())
print(f"total {sum(I.values()) * 32 / nvox:.1f} instr/voxel")
for r in sorted(I, key=lambda x: -I[x]):
    print(f"  {r:26s} {I[r] * 32 / nvox:7.1f} instr/voxel   {100 * S[r] / tot:5.1f}% of stall samples")
