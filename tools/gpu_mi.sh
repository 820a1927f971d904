# MI iteration: GPU parity tests for MI + bench (mi256 only)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "mi or step or shard" > gpurun_out/gpu_tests_mi.txt 2>&1
timeout 300 python bench.py --no-secondary --no-cpu --steps 200 > gpurun_out/bench_mi.json 2> gpurun_out/bench_mi.err
