#!/bin/bash
# ncu --set full of the one-pass LNCC kernel at configs[2] (one launch)
O=gpurun_out/${1:-l3prof}; mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --workload lncc720"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lncc_fused -s 3 -c 1 -o $O/full_lncc_fused $B > $O/ncu.out 2>&1
ls -la $O
