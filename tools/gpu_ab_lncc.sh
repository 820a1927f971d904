# A/B of library variants on the LNCC workload: gpu_ab_lncc.sh "<variants>" [bench args]
V=$1; shift
for rep in 1 2; do
for v in $V; do
  FFDP_LIB=$PWD/exp/libffdp_$v.so python bench.py --no-cpu --no-secondary --workload lncc720 --steps 10 "$@" > gpurun_out/abl_$v.json 2>gpurun_out/abl_$v.err
  python -c "import json; d=json.load(open('gpurun_out/abl_$v.json')); print('$v', d['value'], d['kernel_ms'])" || tail -3 gpurun_out/abl_$v.err
done
done
