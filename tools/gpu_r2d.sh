#!/bin/bash
# C++ suites (mirror incl. the sharded deformable_stage, the plan with threads / NCCL) and the
# bench's N > 1 path as ranks-as-threads on one device
O=gpurun_out/${1:-r2d}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
timeout 900 python -m pytest tests/test_cpp_api.py -q -m gpu -s > $O/pytest_cpp.log 2>&1; echo "rc=$?" >> $O/pytest_cpp.log
for wl in mi256 lncc720; do for n in 2 3; do
timeout 400 python bench.py --gpus $n --transport local --workload $wl --steps 5 --warmup 3 > $O/b_local_${wl}_$n.json 2> $O/b_local_${wl}_$n.err
python -c "import json; d=json.loads(open('$O/b_local_${wl}_$n.json').read().strip().splitlines()[-1]); print('$wl N=$n', d['value'], d['ms_per_step'], d['scaling'], d['window'], d['config']['parallelism'])" || tail -3 $O/b_local_${wl}_$n.err
done; done
grep -E "sharded stage|plan|NCCL|passed|failed|FAIL" $O/pytest_cpp.log | tail -30
