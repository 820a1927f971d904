#!/bin/bash
# MI pass 2 bulk stream: 2 vs 3 input stages
O=gpurun_out/${1:-grs}; mkdir -p $O
run() { local n=$1 w=$2; shift 2
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 --workload $w > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/b_$n.err
}
run s_st2 mi256 X=1; run s_st3 mi256 FFDP_LIB=$PWD/exp/libffdp_st3.so
run big_st2a mi1760 X=1; run big_st3a mi1760 FFDP_LIB=$PWD/exp/libffdp_st3.so
run big_st2b mi1760 X=1; run big_st3b mi1760 FFDP_LIB=$PWD/exp/libffdp_st3.so
FFDP_LIB=$PWD/exp/libffdp_st3.so timeout 600 python -m pytest -q -x tests/test_gpu_fullsize.py -k mi > $O/pytest_st3.log 2>&1; tail -1 $O/pytest_st3.log
