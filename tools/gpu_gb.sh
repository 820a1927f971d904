#!/bin/bash
O=gpurun_out/${1:-gb}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
timeout 600 python -m pytest tests/test_gpu_plan.py -q -m gpu -x -s -k "thin" > $O/pytest_thin.log 2>&1; echo "rc=$?" >> $O/pytest_thin.log
run() { local n=$1; shift
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/b_$n.err
}
BARGS="--workload mi1760"; run big X=1; for v in gb2 gb1; do run big_$v FFDP_LIB=$PWD/exp/libffdp_$v.so; done
BARGS="--workload mi256"; run s X=1; for v in gb2 gb1; do run s_$v FFDP_LIB=$PWD/exp/libffdp_$v.so; done
BARGS="--workload lncc1024"; run l1024 X=1
BARGS="--workload lncc128"; run l128 X=1
grep -E "thin|passed|failed" $O/pytest_thin.log | tail -5
