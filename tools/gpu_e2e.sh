#!/bin/bash
# the default bench line (configs[4] headline, secondaries, CPU baseline) with the registered-host e2e
O=gpurun_out/${1:-e2e}; mkdir -p $O
free -g > $O/free.txt
start=$(date +%s); timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "rc=$? wall=$(( $(date +%s) - start ))s"
python - <<PY
import json
d = json.loads(open("$O/bench_default.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], json.dumps(d["e2e"]))
for s in d.get("secondary", []):
    print(s.get("config", {}).get("workload"), s.get("value"), json.dumps(s.get("e2e"))[:160])
PY
