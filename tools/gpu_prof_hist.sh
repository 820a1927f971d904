# ncu --set full capture (with source) of the MI pass-1 kernel on the mi256 bench
O=gpurun_out/prof; mkdir -p $O
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mi_hist_bs -s 3 -c 1 -o $O/hist $B > $O/hist.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_mi_grad_rec -s 3 -c 1 -o $O/grad $B > $O/grad.log 2>&1
ls -la $O
