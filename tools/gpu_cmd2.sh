set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests.txt
timeout 600 python bench.py --no-secondary --no-cpu > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_step -s 6 -c 2 -o gpurun_out/prof_mi256_v2 python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu > /dev/null 2>&1
