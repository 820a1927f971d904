# ncu evidence for the bench command (1 GPU): launch lists + one --set full capture per hot kernel
set -x
O=gpurun_out/${1:-r01}; mkdir -p $O
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mi256.csv $B > $O/launches_mi256.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lncc720.csv $B --workload lncc720 > $O/launches_lncc720.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mi_hist_bs -s 3 -c 1 -o $O/full_mi_hist_bs $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_mi_grad_rec -s 3 -c 1 -o $O/full_mi_grad_rec $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lncc_sample -s 3 -c 1 -o $O/full_lncc_sample $B --workload lncc720 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lncc_moments -s 3 -c 1 -o $O/full_lncc_moments $B --workload lncc720 > /dev/null 2>&1
# the warp update (720x640x720 lattice): both k_smooth kernels of one update
cat > /tmp/wu_prof.py <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import bench
hbm, kind = bench.peaks()
print(json.dumps(bench.run_warp_update((720, 640, 720), 3, hbm, kind)))
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_wu720.csv python /tmp/wu_prof.py > $O/launches_wu720.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_smooth -s 6 -c 2 -o $O/full_wu_smooth python /tmp/wu_prof.py > /dev/null 2>&1
ls -la $O
