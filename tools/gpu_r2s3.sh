#!/bin/bash
# round-2 session-3 baseline: smoke, full GPU suite, default bench, lncc720 with both warp splits
O=gpurun_out/${1:-r2s3}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for nm in 256 128; do
FFDP_LNCC_NM=$nm timeout 300 python bench.py --workload lncc720 --no-secondary --no-cpu --steps 10 --warmup 3 > $O/bench_lncc720_$nm.json 2> $O/bench_lncc720_$nm.err
done
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err
tail -3 $O/smoke.log; tail -5 $O/pytest_gpu.log
for f in $O/bench_*.json; do echo "== $f"; tail -c 600 $f; done
