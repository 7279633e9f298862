"""Does overlapping independent remap batches raise throughput?  Two 1B-slot C5 tables,
batches alternated over two streams ("two") vs all on one table ("one").  A probe of whether
the claim chain of one batch and the probe of the next could share the GPU profitably."""
import sys, time, torch
sys.path.insert(0, '/root/repo')
import bench, paper_2602_17050_b200 as mz
rows = 1 << 30
caps = mz.even_capacities(rows, 8)
pol = mz.EvictionPolicy.disabled()
B = bench.BATCH
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
tabs = [mz.MpzchTable(mz.TableConfig(caps, 128, 7), device=0) for _ in range(2)]
npre = bench.prefill_count(rows)
outs = [(torch.empty(B, dtype=torch.int64, device='cuda'), torch.empty(B, dtype=torch.uint8, device='cuda')) for _ in range(2)]
for ti, t in enumerate(tabs):
    for a in range(0, npre, B):
        with torch.cuda.stream(streams[ti]):
            ids = bench.distinct_ids_t(5, torch.arange(a, min(a + B, npre), dtype=torch.int64, device='cuda'))
            t.process_batch_device(ids, 1, pol, None, outs[ti][0], outs[ti][1], None, streams[ti])
torch.cuda.synchronize()
nb = 20
fb = npre


def make(k0):
    global fb
    out = []
    for b in range(k0, k0 + nb):
        idx, nf = bench.batch_indices(torch, 0, npre, B, b, fb, bench.SAMPLER_SEED)
        fb += nf
        out.append(bench.distinct_ids_t(5, idx).contiguous())
    torch.cuda.synchronize()
    return out


k0 = 0
for mode in ("one", "two", "one", "two"):
    batches = make(k0)  # fresh batches every run (same mix: 90% prefilled ids, 10% new)
    k0 += nb
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tk = []
    for b in range(nb):
        ti = 0 if mode == "one" else b % 2
        tk.append((ti, tabs[ti].process_batch_device_async(batches[b], 10 + k0 + b, pol, None, outs[ti][0],
                                                          outs[ti][1], None, streams[ti])))
    for ti, k in tk:
        tabs[ti].wait(k)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(mode, round(nb * B / dt / 1e9, 3), "G/s")
