python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests.txt
timeout 600 python bench.py --no-cpu --steps 100 > gpurun_out/bench3.json 2> gpurun_out/bench3.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_step_lncc -s 3 -c 1 -o gpurun_out/prof_lncc720_v2 python bench.py --workload lncc720 --steps 3 --warmup 3 --no-secondary --no-cpu > /dev/null 2>&1
