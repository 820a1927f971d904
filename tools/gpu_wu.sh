# warp update: GPU parity tests + timing at 720x640x720
timeout 600 python -m pytest tests/test_gpu_smooth.py tests/test_gpu_dist.py -x -q > gpurun_out/gpu_tests_wu.txt 2>&1
timeout 300 python -c "
import json, bench
hbm, kind = bench.peaks()
print(json.dumps(bench.run_warp_update((720, 640, 720), 20, hbm, kind)))
print(json.dumps(bench.run_warp_update((256, 256, 256), 50, hbm, kind)))
" > gpurun_out/wu.json 2> gpurun_out/wu.err
