import json, os, sys
sys.path.insert(0, os.getcwd())
import bench
hbm, kind = bench.peaks()
print(json.dumps(bench.run_warp_update((720, 640, 720), 3, hbm, kind)))
