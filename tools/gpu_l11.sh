#!/bin/bash
# split finalize (sampler warps finish half the rows): parity under FFDP_LIB, then A/B
O=gpurun_out/${1:-l11}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
FFDP_LIB=$PWD/exp/libffdp_split.so timeout 120 python __graft_entry__.py smoke > $O/smoke_split.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke_split.log; exit 1; fi
FFDP_LIB=$PWD/exp/libffdp_split.so timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_shard.py tests/test_gpu_plan.py -q -m gpu -x -k "lncc" > $O/pytest_split.log 2>&1; echo "rc=$?" >> $O/pytest_split.log
run() { local n=$1; shift
  env "$@" timeout 240 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])" || tail -3 $O/b_$n.err
}
for rep in 1 2; do
BARGS="--workload lncc720"; run def$rep X=1; run split$rep FFDP_LIB=$PWD/exp/libffdp_split.so
done
BARGS="--workload lncc720 --jitter survey"; run defs X=1; run splits FFDP_LIB=$PWD/exp/libffdp_split.so
tail -3 $O/pytest_split.log
