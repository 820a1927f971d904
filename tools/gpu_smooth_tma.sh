#!/bin/bash
# k_smooth TMA plane loads: parity (the warp-update tests) and an A/B against the cp.async path
O=gpurun_out/${1:-stma}; mkdir -p $O
timeout 900 python -m pytest -q -x tests/test_gpu_smooth.py tests/test_gpu_plan.py tests/test_gpu_comm.py tests/test_gpu_dist.py "tests/test_gpu_fullsize.py::test_warp_update_720_sharded_bit_identical" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
cat > /tmp/wu_run.py <<'PY'
import json, sys, os; sys.path.insert(0, os.getcwd()); import bench
hbm, kind = bench.peaks()
d = bench.run_warp_update((720, 640, 720), 20, hbm, kind)
print(json.dumps(d))
PY
for i in 1 2; do
  python /tmp/wu_run.py > $O/tma$i.json 2>&1; tail -1 $O/tma$i.json | cut -c1-200
  FFDP_LIB=$PWD/exp/libffdp_smooth_cp.so python /tmp/wu_run.py > $O/cp$i.json 2>&1; tail -1 $O/cp$i.json | cut -c1-200
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_smooth -s 6 -c 2 -o $O/wu python /tmp/wu_run.py > $O/wu_ncu.log 2>&1
ls $O
