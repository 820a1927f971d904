# A/B of library variants on the warp update at 720x640x720: wu_ab.sh "<variants>"
for rep in 1 2; do
for v in $1; do
  FFDP_LIB=$PWD/exp/libffdp_$v.so timeout 300 python -c "
import json, bench
hbm, kind = bench.peaks()
r = bench.run_warp_update((720, 640, 720), 20, hbm, kind)
print('$v', json.dumps(r['kernel_ms']), r.get('ms_per_update'))
" 2>&1 | tail -1
done
done
