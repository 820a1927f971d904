#!/bin/bash
# A/B: MI pass 2 (k_mi_grad_bs vs the legacy resampling kernel, minBlocks 3/4) at mi1760 and
# the fused LNCC kernel's sampler backoff at lncc720; MI + LNCC step parity tests first
O=gpurun_out/${1:-ab2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py -q -m gpu -x -k "mi or lncc_parity" -s > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { # name env... -- bench args
  local n=$1; shift
  env "$@" timeout 600 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 $BARGS > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json; d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]); print('$n', d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d['step_roofline']['frac'])" || tail -3 $O/b_$n.err
}
BARGS="--workload lncc720"
for v in sleep0 sleep64 sleep1k; do run l_$v FFDP_LIB=$PWD/exp/libffdp_$v.so; done
run l_default X=1
BARGS="--workload mi1760"
run m_default X=1
run m_legacy FFDP_MI_GRAD_LEGACY=1
run m_g2m4 FFDP_LIB=$PWD/exp/libffdp_g2m4.so
tail -3 $O/pytest.log
