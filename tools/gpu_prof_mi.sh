set -x
O=gpurun_out/r01; mkdir -p $O
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mi256.csv $B > $O/launches_mi256.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mi_hist_bs -s 3 -c 1 -o $O/full_mi_hist_bs $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_mi_grad_rec -s 3 -c 1 -o $O/full_mi_grad_rec $B > /dev/null 2>&1
ls -la $O
