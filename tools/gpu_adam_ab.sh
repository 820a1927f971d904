#!/bin/bash
# sobolev_adam: Adam operand tiles by TMA into shared memory (ops) vs per-thread loads one plane ahead (noops)
O=gpurun_out/${1:-adam}; mkdir -p $O
timeout 900 python -m pytest -q -x tests/test_gpu_smooth.py tests/test_gpu_plan.py "tests/test_gpu_fullsize.py::test_warp_update_720_sharded_bit_identical" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
cat > /tmp/wu_run.py <<'PY'
import json, sys, os; sys.path.insert(0, os.getcwd()); import bench
hbm, kind = bench.peaks()
print(json.dumps(bench.run_warp_update((720, 640, 720), 20, hbm, kind)))
PY
for i in 1 2; do
  python /tmp/wu_run.py > $O/ops$i.json 2>&1; tail -1 $O/ops$i.json | cut -c1-170
  FFDP_LIB=$PWD/exp/libffdp_noops.so python /tmp/wu_run.py > $O/noops$i.json 2>&1; tail -1 $O/noops$i.json | cut -c1-170
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_smooth -s 6 -c 2 -o $O/wu python /tmp/wu_run.py > $O/wu_ncu.log 2>&1
