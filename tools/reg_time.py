"""Time the configs[2] registration (bench.run_registration) three times in one process."""
import os, sys
sys.path.insert(0, os.getcwd())
import bench
r = bench.run_registration((720, 640, 720), [(4, 20), (2, 20), (1, 10)])
print(os.environ.get("FFDP_LIB", "in-tree").split("/")[-1], r["seconds_runs"], flush=True)
