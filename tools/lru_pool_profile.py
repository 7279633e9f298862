#!/usr/bin/env python
"""Per-batch times of bench_configs.lru's stream (LRU, pool 1.2 x rows, 2^20 rows, 64K-position
batches): which path each batch took, its rounds, and its device time alone (event-timed, a
synchronize on both sides).  Run with MPZCH_DEBUG_ROUNDS=1 for the rounds kernel's counters, or
under `ncu --metrics gpu__time_duration.sum` for the per-kernel split.
`python tools/lru_pool_profile.py [pool_factor] [shards]`"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2602_17050_b200 as mz  # noqa: E402

pool_factor = float(sys.argv[1]) if len(sys.argv) > 1 else 1.2
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rows = 1 << 20
pool = int(pool_factor * rows)
ids_pool = bench.distinct_ids_t(9, torch.arange(pool, dtype=torch.int64, device="cuda"))
B, nb = 65536, 24
g = torch.Generator(device="cuda").manual_seed(9)
batches = [ids_pool[torch.randint(0, pool, (B,), generator=g, device="cuda")].contiguous() for _ in range(nb)]
t = mz.MpzchTable(mz.TableConfig(mz.even_capacities(rows, shards), 128, 7))
pol = mz.EvictionPolicy.lru()
st = torch.cuda.current_stream()
out_s = torch.empty(B, dtype=torch.int64, device="cuda")
out_o = torch.empty(B, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for b in range(nb):
    torch.cuda.synchronize()
    e0.record(st)
    t.process_batch_device(batches[b], 10 + b, pol, None, out_s, out_o, None, st)
    e1.record(st)
    torch.cuda.synchronize()
    s = t.last_stats()
    print(json.dumps(dict(batch=b, ms=e0.elapsed_time(e1), path=s["path"], rounds=s["rounds"], new_ids=s["new_ids"],
                          evicted=s["evicted"], inserted=s["inserted"])), flush=True)
