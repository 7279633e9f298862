"""C3 alone (bench_configs.c3) -- a target for ncu captures of one insert-heavy batch's kernels."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_configs  # noqa: E402

print(json.dumps(bench_configs.c3())[:400])
