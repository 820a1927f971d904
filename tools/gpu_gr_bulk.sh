#!/bin/bash
# MI pass 2 from the records as a bulk-copy stream (FFDP_GR_TMA=1) vs the LDG form (gr_ldg): full GPU suite, then A/B
O=gpurun_out/${1:-grb}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1 || { tail -5 $O/smoke.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
run() { local n=$1 w=$2; shift 2
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 --workload $w > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/b_$n.err
}
run s_bulk mi256 X=1; run s_ldg mi256 FFDP_LIB=$PWD/exp/libffdp_gr_ldg.so
run big_bulk1 mi1760 X=1; run big_ldg1 mi1760 FFDP_LIB=$PWD/exp/libffdp_gr_ldg.so
run big_bulk2 mi1760 X=1; run big_ldg2 mi1760 FFDP_LIB=$PWD/exp/libffdp_gr_ldg.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_step_mi_grad_rec" -s 3 -c 1 -o $O/full_grb_mi1760 python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --workload mi1760 > $O/ncu_full.out 2>&1
ls $O
