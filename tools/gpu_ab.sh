for v in ty8 ty16 ty8 ty16; do
  FFDP_LIB=$PWD/exp/libffdp_$v.so python bench.py --no-cpu --steps 50 > gpurun_out/ab_$v.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', d['value'], d['kernel_ms'], 'lncc', d['secondary']['value'], d['secondary']['kernel_ms'])"
done
