"""Where does the e2e service loop lose against the PCIe copy-only ceiling?  Same loop as
bench.py's e2e (D buffer sets, H2D on s_in, remap on `stream`, D2H on s_out, host retires
step i-D) with parts switched off: copies only, H2D + remap, remap + D2H, everything."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
import paper_2602_17050_b200 as mz  # noqa: E402

dev = 0
rows = bench.ROWS
B = bench.BATCH
caps = mz.even_capacities(rows, bench.SHARDS)
t = mz.MpzchTable(mz.TableConfig(caps, bench.MAX_PROBE, bench.TABLE_SEED), device=dev)
pol = mz.EvictionPolicy.disabled()
stream = torch.cuda.current_stream(dev)
o_s = torch.empty(B, dtype=torch.int64, device=dev)
o_o = torch.empty(B, dtype=torch.uint8, device=dev)
npre = bench.prefill_count(rows)
for a in range(0, npre, B):
    ids = bench.distinct_ids_t(bench.ID_SEED, torch.arange(a, min(a + B, npre), dtype=torch.int64, device=dev))
    t.process_batch_device(ids, 1, pol, None, o_s, o_o, None, stream)
torch.cuda.synchronize()
steps = 24
fb = npre
host = []
for i in range(steps):
    idx, nf = bench.batch_indices(torch, dev, npre, B, i, fb, bench.SAMPLER_SEED)
    fb += nf
    host.append(bench.distinct_ids_t(bench.ID_SEED, idx).cpu().pin_memory())
D = 4
s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
d_ids = [torch.empty(B, dtype=torch.int64, device=dev) for _ in range(D)]
d_s = [torch.empty(B, dtype=torch.int64, device=dev) for _ in range(D)]
d_o = [torch.empty(B, dtype=torch.uint8, device=dev) for _ in range(D)]
h_s = [torch.empty(B, dtype=torch.int64).pin_memory() for _ in range(D)]
h_o = [torch.empty(B, dtype=torch.uint8).pin_memory() for _ in range(D)]


def loop(h2d, remap, d2h, now0):
    ev_in = [torch.cuda.Event() for _ in range(steps)]
    ev_cmp = [torch.cuda.Event() for _ in range(steps)]
    ev_out = [torch.cuda.Event() for _ in range(steps)]
    tk = [None] * steps
    torch.cuda.synchronize()
    t0 = time.perf_counter()

    def retire(k):
        if tk[k] is not None:
            t.wait(tk[k])
        ev_out[k].synchronize()

    for i in range(steps):
        j = i % D
        if i >= D:
            retire(i - D)
        with torch.cuda.stream(s_in):
            if h2d:
                d_ids[j].copy_(host[i], non_blocking=True)
            ev_in[i].record(s_in)
        stream.wait_event(ev_in[i])
        if remap:
            tk[i] = t.process_batch_device_async(d_ids[j] if h2d else d_ids[0], now0 + i, pol, None,
                                                 d_s[j], d_o[j], None, stream)
        ev_cmp[i].record(stream)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_cmp[i])
            if d2h:
                h_s[j].copy_(d_s[j], non_blocking=True)
                h_o[j].copy_(d_o[j], non_blocking=True)
            ev_out[i].record(s_out)
    for k in range(max(0, steps - D), steps):
        retire(k)
    return steps * B / (time.perf_counter() - t0) / 1e9


for name, a in [("copies only", (1, 0, 1)), ("h2d+remap", (1, 1, 0)), ("remap+d2h", (0, 1, 1)),
                ("remap only", (0, 1, 0)), ("all", (1, 1, 1)), ("copies only", (1, 0, 1)), ("all", (1, 1, 1))]:
    print(name, round(loop(*a, now0=10 + 100 * hash(name) % 1000), 3), "G positions/s", flush=True)
