#!/bin/bash
# after the MI table fix and the attribute mutex: MI parity, plan tests, local-group lines, MI lines
O=gpurun_out/${1:-r2f}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_step.py tests/test_gpu_fullsize.py -q -m gpu -k "plan or mi or first_use" -s > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for wl in mi256 lncc720; do for n in 2 4; do
timeout 200 python bench.py --gpus $n --transport local --workload $wl --steps 5 --warmup 3 > $O/b_local_${wl}_$n.json 2> $O/b_local_${wl}_$n.err; echo "rc=$?" >> $O/b_local_${wl}_$n.err
python -c "import json; d=json.loads(open('$O/b_local_${wl}_$n.json').read().strip().splitlines()[-1]); print('$wl N=$n', d['value'], d['ms_per_step'], d['scaling'], d['window'], d['config']['parallelism'])" || tail -12 $O/b_local_${wl}_$n.err
done; done
run() { local n=$1; shift
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/b_$n.err
}
BARGS="--workload mi1760"; run big X=1
BARGS="--workload mi256"; run s X=1
grep -E "passed|failed|FAILED|Error|plan " $O/pytest.log | tail -25
