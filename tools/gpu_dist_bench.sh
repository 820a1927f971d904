# functional check of the sharded bench path: 2 ranks on one GPU over gloo
for w in lncc128 mi256; do
FFDP_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --workload $w > gpurun_out/bench_gloo2_$w.json 2> gpurun_out/bench_gloo2_$w.err
done
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/gpu_tests_dist.txt 2>&1
