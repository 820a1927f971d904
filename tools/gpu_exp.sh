python bench.py --no-secondary --no-cpu --steps 100 > gpurun_out/exp_base.json 2>&1
FFDP_LIB=$PWD/exp/libffdp_noatomic.so python bench.py --no-secondary --no-cpu --steps 100 > gpurun_out/exp_noatomic.json 2>&1
