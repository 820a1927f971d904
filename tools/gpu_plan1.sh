#!/bin/bash
# native plan tests + LNCC/MI bench after the addressing-mode split
O=gpurun_out/${1:-plan1}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_plan.py -q -m gpu -x -s > $O/pytest_plan.log 2>&1; echo "rc=$?" >> $O/pytest_plan.log
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_registration.py -q -m gpu -x > $O/pytest_step.log 2>&1; echo "rc=$?" >> $O/pytest_step.log
for wl in lncc720 mi1760 mi256; do
timeout 600 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 --workload $wl > $O/b_$wl.json 2> $O/b_$wl.err
python -c "import json; d=json.loads(open('$O/b_$wl.json').read().strip().splitlines()[-1]); print('$wl', d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d['step_roofline']['frac'], d['clocks'])" || tail -3 $O/b_$wl.err
done
grep -h "plan\|passed\|failed\|Error" $O/pytest_plan.log | tail -30; tail -3 $O/pytest_step.log
