#!/bin/bash
# one-pass LNCC: smoke + LNCC parity tests + lncc720 bench + one ncu --set full capture
O=gpurun_out/${1:-l3b}; mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_shard.py tests/test_gpu_refparity.py tests/test_gpu_lncc.py tests/test_gpu_fullsize.py -q -m gpu -k "lncc" -s > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python bench.py --workload lncc720 --no-secondary --no-cpu --steps 10 --warmup 3 > $O/bench_new.json 2> $O/bench_new.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lncc_fused -s 3 -c 1 -o $O/full_lncc_fused python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --workload lncc720 > $O/ncu.out 2>&1
tail -3 $O/smoke.log; tail -4 $O/pytest.log; python -c "
import json; d=json.loads(open('$O/bench_new.json').read().strip().splitlines()[-1]); print('BENCH', d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'])"
