# ncu --set full of the two MI step kernels (bench mi256)
O=gpurun_out/${1:-prof}; mkdir -p $O
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_mi_hist -s 3 -c 1 -o $O/full_mi_hist $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_mi_grad -s 3 -c 1 -o $O/full_mi_grad $B > /dev/null 2>&1
ls $O
