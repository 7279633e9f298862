#!/usr/bin/env python
"""Per-batch cost of the row-sharded device protocol (csrc/sharded.cu) on ONE B200.

G ranks of one process share the GPU (each on its own stream; peer = same device), so their
remaps time-share the SMs and the total work equals the single table's: the difference to the
single table is the protocol's cost (the exchange kernels, the flag round trips between the
phases, the owners' remaps running as G smaller launches).  Two workloads:

  * C5 (default 2^30 rows, S=8, P=128, 0.8 load, 4M-position batches 90% hit / 10% fresh):
    device time per global batch, pipelined by ticket (every rank's batch enqueued by one
    host thread, then every ticket waited);
  * tiny batches (G x 64 positions): the latency floor of one protocol round (five phases for
    TTL, three for Disabled), i.e. the fixed cost a small batch pays per step.

Prints one JSON line per (G, workload); the single table (plain mpzch_process_batch_device_async)
is the G = 0 row.
"""
import argparse
import json
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2602_17050_b200 as mz  # noqa: E402


def c5_batches(npre, B, nb, fresh):
    out = []
    for b in range(nb):
        idx, nf = bench.batch_indices(torch, "cuda", npre, B, b, fresh, bench.SAMPLER_SEED)
        fresh += nf
        out.append(bench.distinct_ids_t(bench.ID_SEED, idx).contiguous())
    return out


def run_sharded(cfg, G, B, npre, batches, tiny, pol, steps, warm):
    ranks = [mz.ShardedRank(cfg, r, G, B, device=0) for r in range(G)]
    mz.ShardedRank.connect_local(ranks)
    streams = [torch.cuda.Stream() for _ in range(G)]
    outs = [(torch.empty(B, dtype=torch.int64, device="cuda"), torch.empty(B, dtype=torch.uint8, device="cuda"))
            for _ in range(G)]

    def enqueue(ids, now):
        n = ids.numel()
        tks = []
        for r in range(G):
            lo, hi = r * n // G, (r + 1) * n // G
            tks.append(ranks[r].process_batch_device_async(ids[lo:hi], now, pol, None, outs[r][0], outs[r][1],
                                                           None, streams[r]))
        return tks

    def wait(tks):
        for r in range(G):
            ranks[r].wait(tks[r])

    t0 = time.perf_counter()
    for a in range(0, npre, B):
        # (the tensor must outlive the ranks' streams' use of it: the caching allocator only
        # knows the current stream)
        chunk = bench.distinct_ids_t(bench.ID_SEED, torch.arange(a, min(a + B, npre), dtype=torch.int64,
                                                                 device="cuda"))
        torch.cuda.synchronize()  # written on the current stream, read on the ranks' streams
        wait(enqueue(chunk, 1))
        del chunk
    torch.cuda.synchronize()
    prefill_s = time.perf_counter() - t0
    res = {}
    for name, bl in (("c5", batches), ("tiny", tiny)):
        for b in range(warm):
            wait(enqueue(bl[b], 2 + b))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pend = [enqueue(bl[b], 2 + b) for b in range(warm, warm + steps)]
        for tks in pend:
            wait(tks)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / steps
        res[name] = ms
    hw = ranks[0].last_stats()["host_waits"]
    for r in ranks:
        r.close()
    del ranks
    torch.cuda.empty_cache()
    return res, prefill_s, hw


def run_single(cfg, B, npre, batches, tiny, pol, steps, warm):
    t = mz.MpzchTable(cfg)
    st = torch.cuda.current_stream()
    s_ = torch.empty(B, dtype=torch.int64, device="cuda")
    o_ = torch.empty(B, dtype=torch.uint8, device="cuda")
    for a in range(0, npre, B):
        ids = bench.distinct_ids_t(bench.ID_SEED, torch.arange(a, min(a + B, npre), dtype=torch.int64, device="cuda"))
        t.process_batch_device(ids, 1, pol, None, s_, o_, None, st)
    res = {}
    for name, bl in (("c5", batches), ("tiny", tiny)):
        for b in range(warm):
            t.process_batch_device(bl[b], 2 + b, pol, None, s_, o_, None, st)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tks = [t.process_batch_device_async(bl[b], 2 + b, pol, None, s_, o_, None, st)
               for b in range(warm, warm + steps)]
        for tk in tks:
            t.wait(tk)
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t0) * 1e3 / steps
    t.close()
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=bench.ROWS)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--worlds", default="1,2,4,8")
    args = ap.parse_args()
    B = bench.BATCH
    caps = mz.even_capacities(args.rows, bench.SHARDS)
    cfg = mz.TableConfig(caps, bench.MAX_PROBE, bench.TABLE_SEED)
    pol = mz.EvictionPolicy.disabled()
    npre = bench.prefill_count(args.rows)
    nb = args.warmup + args.steps
    batches = c5_batches(npre, B, nb, npre)
    gen = torch.Generator(device="cuda").manual_seed(5)
    tiny = [bench.distinct_ids_t(bench.ID_SEED, torch.randint(0, npre, (512,), generator=gen, device="cuda"))
            for _ in range(nb)]
    single = run_single(cfg, B, npre, batches, tiny, pol, args.steps, args.warmup)
    base = {"what": "row-sharded device protocol on ONE B200 (ranks time-share the GPU)",
            "rows": args.rows, "batch_positions": B, "tiny_positions": 512, "steps": args.steps}
    print(json.dumps(dict(base, world=0, mode="single table (mpzch_process_batch_device_async)",
                          c5_ms=single["c5"], tiny_ms=single["tiny"])), flush=True)
    for G in [int(x) for x in args.worlds.split(",")]:
        res, pre_s, hw = run_sharded(cfg, G, B, npre, batches, tiny, pol, args.steps, args.warmup)
        print(json.dumps(dict(base, world=G, mode="mpzch_sharded_* (connect_local, one stream per rank)",
                              c5_ms=res["c5"], tiny_ms=res["tiny"], c5_overhead_ms=res["c5"] - single["c5"],
                              tiny_overhead_ms=res["tiny"] - single["tiny"], host_waits_per_batch=hw,
                              prefill_s=pre_s)), flush=True)


if __name__ == "__main__":
    main()
