#!/bin/bash
# MI pass 1 / record-free pass 2: L2 prefetch of the unit FFDP_MI_PF iterations ahead; parity under pf2
O=gpurun_out/${1:-mipf}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
FFDP_LIB=$PWD/exp/libffdp_pf2.so timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_plan.py -q -m gpu -x -k "mi" > $O/pytest_pf2.log 2>&1; echo "rc=$?" >> $O/pytest_pf2.log
run() { local n=$1; shift
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/b_$n.err
}
BARGS="--workload mi1760"; run big X=1; run big_pf1 FFDP_LIB=$PWD/exp/libffdp_pf1.so; run big_pf2 FFDP_LIB=$PWD/exp/libffdp_pf2.so; run big_pf4 FFDP_LIB=$PWD/exp/libffdp_pf4.so
run bignr FFDP_BENCH_NOREC=1; run bignr_pf2 FFDP_BENCH_NOREC=1 FFDP_LIB=$PWD/exp/libffdp_pf2.so
BARGS="--workload mi256"; run s X=1; run s_pf1 FFDP_LIB=$PWD/exp/libffdp_pf1.so; run s_pf2 FFDP_LIB=$PWD/exp/libffdp_pf2.so
tail -3 $O/pytest_pf2.log
