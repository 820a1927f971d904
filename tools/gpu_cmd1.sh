set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests.txt
python __graft_entry__.py smoke >> gpurun_out/gpu_tests.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 60 --csv --log-file gpurun_out/launches_mi256.csv python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_step -s 6 -c 2 -o gpurun_out/prof_mi256 python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_step_lncc -s 3 -c 1 -o gpurun_out/prof_lncc720 python bench.py --workload lncc720 --steps 3 --warmup 3 --no-secondary --no-cpu > /dev/null 2>&1
ls -la gpurun_out
