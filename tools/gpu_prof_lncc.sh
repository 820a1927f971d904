# ncu --set full of the fused LNCC step (bench lncc720)
O=gpurun_out/${1:-prof}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_lncc -s 3 -c 1 -o $O/full_lncc python bench.py --workload lncc720 --steps 3 --warmup 3 --no-cpu --no-secondary > /dev/null 2>&1
ls $O
