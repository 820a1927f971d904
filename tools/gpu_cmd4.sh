# round-1 check: GPU tests, N=1 bench, 2 ranks on one GPU over gloo (functional check of the sharded bench path)
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests4.txt
timeout 600 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err
for w in lncc128 mi256; do
FFDP_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --workload $w > gpurun_out/bench4_gloo2_$w.json 2> gpurun_out/bench4_gloo2_$w.err
done
