#!/bin/bash
# round-2 validation: smoke, the whole GPU suite, the default bench (headline + secondaries)
O=gpurun_out/${1:-r2full}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc" >> $O/smoke.log
if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
tail -3 $O/smoke.log; grep -E "passed|failed|FAILED|Error" $O/pytest_gpu.log | tail -12
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2full/bench_default.json').read().strip().splitlines()[-1])
print('HEAD', d['config']['workload'], d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d['step_roofline']['frac'], d.get('mi_records'), d['clocks'])
print('E2E', d['e2e']); print('CPU', d.get('cpu_baseline'))
for s in d.get('secondary', []): print('SEC', s['config']['workload'], s['config'].get('u_jitter'), s['value'], s['ms_per_step'], s['kernel_ms'], s['roofline']['frac'])
print('WU', d.get('warp_update', {}).get('ms'), 'REG', d.get('registration', {}).get('seconds'))
PY
