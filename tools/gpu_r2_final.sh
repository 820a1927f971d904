#!/bin/bash
# round-2 final: smoke, the GPU suite, the default bench, the reference arm, launch lists and --set full of the headline
O=gpurun_out/${1:-r2final}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mi1760.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary --workload mi1760 > $O/ncu_launch.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lncc720.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary --workload lncc720 > $O/ncu_launch2.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mi_hist_bs|k_step_mi_grad_rec" -s 6 -c 2 -o $O/full_mi1760 python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --workload mi1760 > $O/ncu_full_mi.out 2>&1
tail -3 $O/smoke.log; tail -2 $O/pytest_gpu.log
python - <<PY
import json
d=json.loads(open('$O/bench_default.json').read().strip().splitlines()[-1])
print('HEAD', d['config']['workload'], d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d['step_roofline']['frac'], d['clocks'])
print('E2E', d['e2e']); print('CPU', d.get('cpu_baseline'))
for s in d.get('secondary', []): print('SEC', s['config']['workload'], s['config'].get('u_jitter'), s['value'], s['ms_per_step'], s['kernel_ms'], s['roofline']['frac'])
print('WU', d.get('warp_update', {}).get('ms'), d.get('warp_update', {}).get('kernel_ms'), 'REG', d.get('registration', {}).get('seconds'))
PY
tail -1 $O/bench_ref.json | cut -c1-300
