#!/bin/bash
# round-2 parity probe: box resources + the new reference / full-size parity tests
set -x
free -g; nproc; lscpu | grep -i "model name"; nvidia-smi --query-gpu=name,memory.total --format=csv
python -m pytest tests/test_gpu_refparity.py tests/test_gpu_shard.py::test_mi_slabs_straddle_fixed_point_switch \
  tests/test_gpu_fullsize.py -x -q -s -m gpu 2>&1 | tail -40
