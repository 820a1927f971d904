#!/bin/bash
# reference driver through the binding; mi1760 with records; compute-sanitizer passes
O=gpurun_out/${1:-r2c}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc" >> $O/smoke.log
if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
timeout 600 python -m pytest tests/test_gpu_ref_backend.py -q -m gpu -s > $O/pytest_refbackend.log 2>&1; echo "rc=$?" >> $O/pytest_refbackend.log
timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 --workload mi1760 > $O/b_mi1760.json 2> $O/b_mi1760.err
python -c "import json; d=json.loads(open('$O/b_mi1760.json').read().strip().splitlines()[-1]); print('mi1760', d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline'], d['step_roofline'], d['clocks'], d['e2e'])" || tail -3 $O/b_mi1760.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/sanitize_$tool.log 2>&1; echo "rc=$?" >> $O/sanitize_$tool.log
  tail -3 $O/sanitize_$tool.log
done
tail -8 $O/pytest_refbackend.log
