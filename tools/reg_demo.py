"""The configs[2] registration line of bench.py alone (timing + loss per scale)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

print(json.dumps(bench.run_registration(bench.WORKLOADS["lncc720"][0], [(4, 20), (2, 20), (1, 10)])))
