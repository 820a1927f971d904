#!/bin/bash
# local-group bench lines (N ranks as threads on one device) + MI record streaming A/B
O=gpurun_out/${1:-r2e}; mkdir -p $O
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; rc=$?; if [ $rc -ne 0 ]; then tail -5 $O/smoke.log; exit 1; fi
for wl in mi256 lncc720; do for n in 2 3; do
timeout 200 python bench.py --gpus $n --transport local --workload $wl --steps 5 --warmup 3 > $O/b_local_${wl}_$n.json 2> $O/b_local_${wl}_$n.err; echo "rc=$?" >> $O/b_local_${wl}_$n.err
python -c "import json; d=json.loads(open('$O/b_local_${wl}_$n.json').read().strip().splitlines()[-1]); print('$wl N=$n', d['value'], d['ms_per_step'], d['scaling'], d['window'], d['config']['parallelism'])" || tail -12 $O/b_local_${wl}_$n.err
done; done
bash tools/gpu_mi_rec.sh mirec
