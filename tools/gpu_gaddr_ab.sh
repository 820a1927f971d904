#!/bin/bash
# A/B of gather_pad's OFF == 2 row-pointer form (FFDP_GADDR) at configs[4], alternating libraries
O=gpurun_out/${1:-gaddr}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1 || { tail -5 $O/smoke.log; exit 1; }
run() { local n=$1; shift
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 --workload mi1760 > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/b_$n.err
}
run base1 X=1; run gaddr1 FFDP_LIB=$PWD/exp/libffdp_gaddr.so; run base2 X=1; run gaddr2 FFDP_LIB=$PWD/exp/libffdp_gaddr.so
FFDP_LIB=$PWD/exp/libffdp_gaddr.so timeout 300 python -m pytest -q -x tests/test_gpu_fullsize.py -k "mi" > $O/pytest_gaddr.log 2>&1; tail -2 $O/pytest_gaddr.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mi1760.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary --workload mi1760 > $O/ncu_launch.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mi_hist_bs|k_step_mi_grad_rec" -s 6 -c 2 -o $O/full_mi1760 python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --workload mi1760 > $O/ncu_full_mi.out 2>&1
ls $O
