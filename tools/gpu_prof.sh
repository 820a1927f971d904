# ncu evidence for the bench command (1 GPU): launch list + one --set full capture per hot kernel
set -x
O=gpurun_out/r01; mkdir -p $O
B="python bench.py --steps 3 --warmup 3 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mi256.csv $B --no-secondary > $O/launches_mi256.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lncc720.csv $B --workload lncc720 --no-secondary > $O/launches_lncc720.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_mi_hist -s 3 -c 1 -o $O/full_mi_hist $B --no-secondary > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_mi_grad -s 3 -c 1 -o $O/full_mi_grad $B --no-secondary > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_lncc -s 3 -c 1 -o $O/full_lncc $B --workload lncc720 --no-secondary > /dev/null 2>&1
ls -la $O
