#!/bin/bash
# one-pass LNCC kernel: parity tests + smoke + lncc720 timing (new vs two-pass)
O=gpurun_out/l3; mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_shard.py tests/test_gpu_refparity.py tests/test_gpu_lncc.py tests/test_gpu_fullsize.py -q -m gpu -k "lncc" -s > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python bench.py --workload lncc720 --no-secondary --no-cpu --steps 10 --warmup 3 > $O/bench_new.json 2> $O/bench_new.err
FFDP_LNCC_IMPL=twopass timeout 300 python bench.py --workload lncc720 --no-secondary --no-cpu --steps 10 --warmup 3 > $O/bench_two.json 2> $O/bench_two.err
tail -3 $O/smoke.log; tail -15 $O/pytest.log; tail -c 1500 $O/bench_new.json; tail -5 $O/bench_new.err
