#!/bin/bash
# round-2 baseline on the GPU box: full GPU suite + default bench + the lncc720 bench line
O=gpurun_out/r02base; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --workload lncc720 --no-secondary --no-cpu > $O/bench_lncc720.json 2> $O/bench_lncc720.err
tail -3 $O/pytest_gpu.log; tail -c 3000 $O/bench_default.json; tail -c 2000 $O/bench_lncc720.json
