#!/bin/bash
# MI unit order: plane-major (default) vs z-major, mi1760 (records) and mi256; parity under the variant
O=gpurun_out/${1:-miz}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
FFDP_LIB=$PWD/exp/libffdp_zord.so timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_plan.py -q -m gpu -x -k "mi" > $O/pytest_zord.log 2>&1; echo "rc=$?" >> $O/pytest_zord.log
run() { local n=$1; shift
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/b_$n.err
}
BARGS="--workload mi1760"; run big X=1; run big_z FFDP_LIB=$PWD/exp/libffdp_zord.so
BARGS="--workload mi256"; run s X=1; run s_z FFDP_LIB=$PWD/exp/libffdp_zord.so
FFDP_LIB=$PWD/exp/libffdp_zord.so timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_mi_hist_bs|k_step_mi_grad_rec" -s 6 -c 2 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --workload mi1760 > $O/ncu_z.csv 2> $O/ncu_z.err
grep -E "dram__bytes|lts__t_sector_hit|gpu__time" $O/ncu_z.csv | cut -c1-300
tail -3 $O/pytest_zord.log
