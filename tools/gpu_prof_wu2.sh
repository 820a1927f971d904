#!/bin/bash
# ncu --set full (source counters) of the two warp-update kernels at 720x640x720, and their SASS source pages
O=gpurun_out/${1:-wu2}; mkdir -p $O
cat > /tmp/wu_run.py <<'PY'
import json, sys, os; sys.path.insert(0, os.getcwd()); import bench
hbm, kind = bench.peaks()
print(json.dumps(bench.run_warp_update((720, 640, 720), 5, hbm, kind)))
PY
python /tmp/wu_run.py > $O/wu_plain.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_smooth -s 6 -c 2 -o $O/wu python /tmp/wu_run.py > $O/wu.log 2>&1
ncu -i $O/wu.ncu-rep --page source --csv --print-source sass --kernel-name regex:"k_smooth<2" > $O/src_gp.csv 2>/dev/null
ncu -i $O/wu.ncu-rep --page source --csv --print-source sass --kernel-name regex:"k_smooth<3" > $O/src_adam.csv 2>/dev/null
ls -la $O
