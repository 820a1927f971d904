#!/bin/bash
# LNCC M-prefetch variants (bench + survey jitter); mi1760 records diagnostics
O=gpurun_out/${1:-l8}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
run() { local n=$1; shift
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'], d.get('mi_records'))" || tail -3 $O/b_$n.err
}
BARGS="--workload mi1760"; run big X=1
for j in bench survey; do BARGS="--workload lncc720 --jitter $j"
run l_def_$j X=1; for v in mpf2p mpf4 mpf6; do run l_${v}_$j FFDP_LIB=$PWD/exp/libffdp_$v.so; done; done
