#!/bin/bash
# fused LNCC warp layouts: 16 moment + 8 sampler warps (default) vs 8 + 8; parity first
O=gpurun_out/${1:-l6}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_shard.py tests/test_gpu_refparity.py tests/test_gpu_lncc.py tests/test_gpu_plan.py -q -m gpu -x -k "lncc" > $O/pytest_lncc.log 2>&1; echo "rc=$?" >> $O/pytest_lncc.log
run() { local n=$1; shift
  env "$@" timeout 600 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])" || tail -3 $O/b_$n.err
}
BARGS="--workload lncc720"; run nm512 X=1; run nm256 FFDP_LNCC_NM=256
BARGS="--workload lncc720 --jitter survey"; run nm512s X=1; run nm256s FFDP_LNCC_NM=256
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lncc_fused -s 3 -c 1 -o $O/full_lncc python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --workload lncc720 > $O/ncu.out 2>&1
tail -3 $O/pytest_lncc.log
