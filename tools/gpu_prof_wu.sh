# ncu --set full of the two warp-update kernels (256^3 lattice)
O=gpurun_out/prof; mkdir -p $O
cat > /tmp/wu_run.py <<'PY'
import json, sys, os; sys.path.insert(0, os.getcwd()); import bench
hbm, kind = bench.peaks()
print(json.dumps(bench.run_warp_update((256, 256, 256), 5, hbm, kind)))
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_smooth -s 6 -c 2 -o $O/wu python /tmp/wu_run.py > $O/wu.log 2>&1
ls -la $O
