O=gpurun_out/${1:-l2p}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lncc_sample|k_lncc_moments" -s 6 -c 2 -o $O/full_lncc2 python bench.py --workload lncc720 --steps 3 --warmup 3 --no-cpu --no-secondary > /dev/null 2>&1
ls $O
