# one ncu --set full capture of a kernel under a python snippet: gpu_prof_one.sh <regex> <skip> <count> <name> <python file>
O=gpurun_out/prof; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -o $O/$4 python $5 > $O/$4.log 2>&1
ls -la $O
