#!/bin/bash
# round-2 profiling pass: NaN test, two-pass LNCC comparison, ncu --set full of the fused
# LNCC kernel (lncc720) and of both MI passes at the headline mi1760
O=gpurun_out/${1:-r2prof}; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_registration.py -q -m gpu -x > $O/pytest_reg.log 2>&1; echo "rc=$?" >> $O/pytest_reg.log
for j in bench survey; do
FFDP_LNCC_IMPL=twopass timeout 300 python bench.py --workload lncc720 --jitter $j --no-secondary --no-cpu --steps 10 --warmup 3 > $O/bench_two_$j.json 2> $O/bench_two_$j.err
done
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lncc_fused -s 3 -c 1 -o $O/full_lncc_fused $B --workload lncc720 > $O/ncu_lncc.out 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_mi_hist_bs|k_step_mi_grad" -s 6 -c 2 -o $O/full_mi1760 $B --workload mi1760 > $O/ncu_mi.out 2>&1
tail -3 $O/pytest_reg.log
for j in bench survey; do python -c "
import json; d=json.loads(open('$O/bench_two_$j.json').read().strip().splitlines()[-1]); print('TWO $j', d['value'], d['ms_per_step'], d['kernel_ms'])"; done
ls -la $O
