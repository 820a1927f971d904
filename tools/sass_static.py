"""Static SASS instruction counts per source line inside an address range of one kernel.

    python tools/sass_static.py <cubin> <kernel-substring> [lo_hex hi_hex]

Uses `nvdisasm -g -c` line annotations (compile with -lineinfo)."""
import collections
import re
import subprocess
import sys

cubin, ksub = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 40
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cur_fn, line, cnt, ops = None, None, collections.Counter(), collections.defaultdict(collections.Counter)
for l in out.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", l)
    if m and cur_fn and ksub in cur_fn:
        a = int(m.group(1), 16)
        if lo <= a < hi:
            cnt[line] += 1
            ops[line][m.group(3).split(".")[0]] += 1
tot = sum(cnt.values())
print("total", tot)
for k, v in cnt.most_common(60):
    print(f"{v:5d} {k:28s} {dict(ops[k].most_common(6))}")
