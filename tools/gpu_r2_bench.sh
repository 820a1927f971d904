#!/bin/bash
# round-2 default bench (headline + secondaries) and the launch list of the headline
O=gpurun_out/${1:-r2bench}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mi1760.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary --workload mi1760 > $O/ncu_launch.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lncc720.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary --workload lncc720 > $O/ncu_launch2.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mi_hist_bs|k_step_mi_grad_rec" -s 6 -c 2 -o $O/full_mi1760 python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --workload mi1760 > $O/ncu_full_mi.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lncc_fused -s 3 -c 1 -o $O/full_lncc_fused python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --workload lncc720 > $O/ncu_full_lncc.out 2>&1
python - <<PY
import json
d=json.loads(open('$O/bench_default.json').read().strip().splitlines()[-1])
print('HEAD', d['config']['workload'], d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d['step_roofline']['frac'], d.get('mi_records'), d['clocks'])
print('E2E', d['e2e']); print('CPU', d.get('cpu_baseline'))
for s in d.get('secondary', []): print('SEC', s['config']['workload'], s['config'].get('u_jitter'), s['value'], s['ms_per_step'], s['kernel_ms'], s['roofline']['frac'])
print('WU', d.get('warp_update', {}).get('ms'), 'REG', d.get('registration', {}).get('seconds'))
PY
ls $O
