#!/usr/bin/env python
"""A short LRU Zipf(1.05) stream (bench_configs.lru_zipf's shape, 2^22 rows, 1M batches) for
profiling the rounds path: `ncu ... python tools/lru_zipf_profile.py [warm] [timed]`."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench  # noqa: E402
import paper_2602_17050_b200 as mz  # noqa: E402
from bench_configs import zipf_cdf, zipf_ranks  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 12
timed = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows, universe, B = 1 << 22, 1 << 27, 1 << 20
zipf_ranks.cdf = zipf_cdf(universe)
t = mz.MpzchTable(mz.TableConfig(mz.even_capacities(rows, 8), 128, 7))
t.set_path("rounds")
pol = mz.EvictionPolicy.lru()
st = torch.cuda.current_stream()
out_s = torch.empty(B, dtype=torch.int64, device="cuda")
out_o = torch.empty(B, dtype=torch.uint8, device="cuda")
for b in range(warm + timed):
    ids = bench.distinct_ids_t(2, zipf_ranks(B, 1.05, universe, 3000 + b)).contiguous()
    t.process_batch_device(ids, 10**6 + 60 * b, pol, None, out_s, out_o, None, st)
    s = t.last_stats()
    print(b, s["path"], s["rounds"], s["evicted"], flush=True)
