#!/bin/bash
O=gpurun_out/${1:-c2}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
FFDP_LIB=$PWD/exp/libffdp_c2.so timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_mi.py -q -m gpu -x -k "mi" > $O/pytest_c2.log 2>&1; echo "rc=$?" >> $O/pytest_c2.log
run() { local n=$1; shift
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'])" || tail -3 $O/b_$n.err
}
for rep in 1 2; do
BARGS="--workload mi1760"; run big$rep X=1; run big_c2$rep FFDP_LIB=$PWD/exp/libffdp_c2.so
done
BARGS="--workload mi256"; run s X=1; run s_c2 FFDP_LIB=$PWD/exp/libffdp_c2.so
BARGS="--workload mi256 --jitter survey"; run ss X=1; run ss_c2 FFDP_LIB=$PWD/exp/libffdp_c2.so
tail -3 $O/pytest_c2.log
