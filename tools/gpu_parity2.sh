#!/bin/bash
O=gpurun_out/${1:-parity2}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
set -x
free -g; nproc; nvidia-smi --query-gpu=name,memory.total --format=csv
timeout 2400 python -m pytest tests/test_gpu_refparity.py tests/test_gpu_shard.py::test_mi_slabs_straddle_fixed_point_switch tests/test_gpu_fullsize.py tests/test_gpu_plan.py -q -s -m gpu 2>&1 | grep -v "^$" | tail -60
