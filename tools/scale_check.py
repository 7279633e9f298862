"""Scale check on one B200: prefill a C5-sized table (default 2^30 rows, S=8, P=128) through the
API in 4M-id batches and, every 20 batches, verify with the read-only lookup that every id of
the batch is found at the slot the remap returned (or collided).  Catches memory-ordering bugs
that only appear at full size (it found the stream-0 ordering bug in round 1).

    python tools/scale_check.py [rows]
"""
import os
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'oracle'))
import numpy as np, torch
import paper_2602_17050_b200 as mz, bench
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
B = 1 << 22
caps = mz.even_capacities(rows, 8)
t = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
npre = int(0.8 * rows)
pol = mz.EvictionPolicy.disabled()
out_s = torch.empty(B, dtype=torch.int64, device='cuda'); out_o = torch.empty(B, dtype=torch.uint8, device='cuda')
ls = torch.empty(B, dtype=torch.int64, device='cuda'); lo = torch.empty(B, dtype=torch.uint8, device='cuda')
st = torch.cuda.current_stream()
t0 = time.perf_counter()
for bi, a in enumerate(range(0, npre, B)):
    ids = bench.distinct_ids_t(5, torch.arange(a, min(a + B, npre), dtype=torch.int64, device='cuda'))
    n = ids.numel()
    chk = ids.clone()
    try:
        t.process_batch_device(ids, 1, pol, None, out_s, out_o, None, st)
    except Exception as e:
        print("FAIL batch", bi, e, "ids[:4]", ids[:4].tolist(), "chk eq", bool((ids == chk).all()), flush=True)
        raise
    s = t.last_stats()
    if s['found'] + s['inserted'] + s['collision'] != n:
        print("COUNT MISMATCH", bi, s, flush=True)
    if not bool((ids == chk).all()):
        print("IDS CORRUPTED", bi, flush=True)
    if bi % 20 == 0 or bi > 195:
        t.lookup_device(ids, ls, lo, st)
        torch.cuda.synchronize()
        ok = (lo[:n] == 0) | ((lo[:n] == 3) & (out_o[:n] == 3))
        same = (ls[:n] == out_s[:n]) | (out_o[:n] == 3)
        print(f"batch {bi}: {time.perf_counter()-t0:.1f}s lookup-ok {bool(ok.all())} slot-same {bool(same.all())} {s}", flush=True)
print("prefill done", time.perf_counter() - t0)
