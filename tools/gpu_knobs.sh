#!/bin/bash
O=gpurun_out/${1:-knobs}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
run() { local n=$1; shift
  env "$@" timeout 400 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['step_roofline']['frac'], d['clocks']['sm_mhz'])" || tail -3 $O/b_$n.err
}
BARGS="--workload lncc720"; run l_auto X=1; for zc in 40 60 80 90 144 180 240 360; do run l_zc$zc FFDP_LNCC_ZCHUNK=$zc; done
BARGS="--workload lncc1024"; run l1024_auto X=1; for zc in 64 128 256; do run l1024_zc$zc FFDP_LNCC_ZCHUNK=$zc; done
BARGS="--workload mi1760"; run big X=1; run big_nt896 FFDP_LIB=$PWD/exp/libffdp_nt896.so
BARGS="--workload mi256"; run s X=1; run s_nt896 FFDP_LIB=$PWD/exp/libffdp_nt896.so
