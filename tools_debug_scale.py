import sys, time, os
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, torch
import paper_2602_17050_b200 as mz, pyoracle, bench
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
check = len(sys.argv) > 3
caps = mz.even_capacities(rows, 8)
t = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
o = pyoracle.OracleTable(caps, 128, 7) if check else None
npre = int(0.8 * rows)
pol = mz.EvictionPolicy.disabled()
out_s = torch.empty(B, dtype=torch.int64, device='cuda'); out_o = torch.empty(B, dtype=torch.uint8, device='cuda')
st = torch.cuda.current_stream()
for a in range(0, npre, B):
    ids = bench.distinct_ids_t(5, torch.arange(a, min(a + B, npre), dtype=torch.int64, device='cuda'))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    t.process_batch_device(ids, 1, pol, None, out_s, out_o, None, st)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"batch@{a}: {dt*1e3:.2f} ms {t.last_stats()}", flush=True)
    if check:
        h = ids.cpu().numpy().view(np.uint64)
        s2, o2, _ = o.process_batch(h, 1, 0)
        n = h.size
        gs = out_s[:n].cpu().numpy().view(np.uint64); go = out_o[:n].cpu().numpy()
        bad = np.nonzero((gs != s2) | (go != o2))[0]
        print("  mismatches", bad.size, bad[:5], gs[bad[:3]], s2[bad[:3]], go[bad[:3]], o2[bad[:3]], flush=True)
if check:
    print("state equal", (t.identities_all() == o.identities_all()).all(), (t.metadata_all() == o.metadata_all()).all())
