#!/bin/bash
# driver-like pass: smoke, GPU suite, reference arm, the plan path through torchrun at one rank
O=gpurun_out/${1:-r2g}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc" >> $O/smoke.log
if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
timeout 1800 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for wl in mi256 lncc720; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --force-plan --workload $wl --steps 5 --warmup 3 > $O/b_plan_$wl.json 2> $O/b_plan_$wl.err; echo "rc=$?" >> $O/b_plan_$wl.err
python -c "import json; d=json.loads(open('$O/b_plan_$wl.json').read().strip().splitlines()[-1]); print('plan', '$wl', d['value'], d['ms_per_step'], d['scaling'], d['window'], d['e2e'], d['config']['parallelism'])" || tail -15 $O/b_plan_$wl.err
done
tail -3 $O/smoke.log; tail -4 $O/pytest_gpu.log; tail -c 700 $O/bench_ref.json
