#!/usr/bin/env python
"""Measure every BASELINE.json config (C5 is bench.py) on one B200.

Prints one JSON object per config: device-timed positions/s (CUDA events on the launch
stream, inputs resident in HBM), per-batch kernel split from the in-library profiler,
outcome counts, and -- where a bounded sample is feasible -- the reference library
(oracle/_ref, OpenMP, all host cores) on the same stream.  Used for profiles/configs_r*.json.

  C1  2^20 rows, S=1 and S=8, P=128, Disabled, 64K-position batches uniform over a
      0.8*2^20 pool (run_latency_bench's sampler); cold fill (batches 0-15) and steady
      state (16 warm-up, 64 timed).
  C2  2^26 rows, S=8, P=128, TTL, Zipf(1.05) over 2^27 ranks, 1M-position batches,
      now = 1e6 + 60 t; TTL 42,000 s so live occupancy settles near 0.8 (reported).
  C3  2^28 rows, S=8, P=256, Disabled, prefilled to 0.95; (i) lookup-only 4M positions
      over the prefilled ids, (i') 50% absent, (ii) insert-heavy 4M positions 50% fresh.
  C4  2^27 rows, S=8, P=128, dim 128 fp32, init_seed 11, TTL 3600, prefill 0.8 at now=1,
      then 1M-position batches uniform over 2^27 fresh ids at now = 10000 + 600 t:
      evictions reset 512 B weights + 512 B momentum per row.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import bench  # noqa: E402  (id generators)
import paper_2602_17050_b200 as mz  # noqa: E402


def ev_time(fn, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def run_batches(t, batches, nows, pol, stream, timed_from=0, feats=None, split=True):
    """Synchronous batches after `timed_from` warm-up batches.  The first half of the timed
    batches runs with the in-library per-kernel event profiler (the split: probe / claim /
    tail), the second half without it (ids_per_s, ms_per_batch: no events between the
    kernels, so programmatic dependent launch can overlap them)."""
    n = max(b.numel() for b in batches)
    out_s = torch.empty(n, dtype=torch.int64, device="cuda")
    out_o = torch.empty(n, dtype=torch.uint8, device="cuda")
    out_e = torch.empty(n, dtype=torch.int64, device="cuda")
    for b in range(timed_from):
        t.process_batch_device(batches[b], nows[b], pol, None, out_s, out_o, out_e, stream)
    # split=False (non-stationary streams, e.g. LRU filling up): every timed batch unprofiled
    mid = timed_from + max((len(batches) - timed_from) // 2, 1) if split else timed_from
    stats = []

    def run(lo, hi):
        def body():
            for b in range(lo, hi):
                t.process_batch_device(batches[b], nows[b], pol, None, out_s, out_o, out_e, stream)
                stats.append(t.last_stats())
        return body
    t.set_profiling(True)
    ev_time(run(timed_from, mid), stream)
    prof = t.profile()
    t.set_profiling(False)
    ms = ev_time(run(mid, len(batches)), stream)
    pos = sum(b.numel() for b in batches[mid:])
    agg = {k: int(sum(s[k] for s in stats)) for k in ("found", "inserted", "evicted", "collision", "new_ids", "evicted_rows", "rounds")}
    nb = max(prof["batches"], 1)
    return dict(ids_per_s=pos / (ms / 1e3), ms_per_batch=ms / max(len(batches) - mid, 1),
                positions=sum(b.numel() for b in batches[timed_from:]),
                outcomes=agg, path=stats[-1]["path"] if stats else None,
                paths={p: sum(s["path"] == p for s in stats) for p in sorted({s["path"] for s in stats})},
                probe_ms=prof["probe_ms"] / nb, claim_ms=prof["claim_ms"] / nb,
                tail_ms=prof["tail_ms"] / nb,
                kernel_ms={k: prof[k] / nb for k in ("validate_ms", "dedup_ms", "claimk_ms", "commit_ms",
                                                     "finalize_ms")},
                probe_gbs=(prof["probe_bytes"] / nb) / (prof["probe_ms"] / nb / 1e3) / 1e9 if prof["probe_ms"] else None,
                batch_gbs=(prof["batch_bytes"] / nb) / (prof["batch_ms"] / nb / 1e3) / 1e9 if prof["batch_ms"] else None)


def run_batches_async(t, batches, nows, pol, stream, timed_from=0):
    """Same as run_batches but pipelined: enqueue every batch, then wait every ticket."""
    n = max(b.numel() for b in batches)
    out_s = torch.empty(n, dtype=torch.int64, device="cuda")
    out_o = torch.empty(n, dtype=torch.uint8, device="cuda")
    out_e = torch.empty(n, dtype=torch.int64, device="cuda")
    for b in range(timed_from):
        t.process_batch_device(batches[b], nows[b], pol, None, out_s, out_o, out_e, stream)

    def body():
        tks = [t.process_batch_device_async(batches[b], nows[b], pol, None, out_s, out_o, out_e, stream)
               for b in range(timed_from, len(batches))]
        for tk in tks:
            t.wait(tk)
    ms = ev_time(body, stream)
    pos = sum(b.numel() for b in batches[timed_from:])
    return dict(ids_per_s=pos / (ms / 1e3), ms_per_batch=ms / max(len(batches) - timed_from, 1))


def ref_time(caps, P, batches_np, nows, mode, ttl, dim=0, init_seed=0, warm=0):
    """The reference library on the same host stream (bounded)."""
    import pyoracle
    if not pyoracle.available("reference"):
        return None
    L = pyoracle.lib("reference")
    L["set_threads"](os.cpu_count() or 1)
    t = pyoracle.OracleTable(caps, P, 7, dim, init_seed, kind="reference")
    tot, pos = 0.0, 0
    for i, (b, now) in enumerate(zip(batches_np, nows)):
        s = time.perf_counter()
        t.process_batch(b, now, mode, ttl)
        if i >= warm:
            tot += time.perf_counter() - s
            pos += b.size
    return dict(ids_per_s=pos / tot, cores=os.cpu_count(), kind="reference")


def c1(shards):
    rows = 1 << 20
    pool = int(0.8 * rows)
    ids_pool = bench.distinct_ids_t(1, torch.arange(pool, dtype=torch.int64, device="cuda"))
    B, nb = 65536, 16 + 64
    k = torch.arange(nb * B, dtype=torch.int64, device="cuda")
    seed = int(bench.mix64_t(torch.tensor([1]), 0x5CA1AB1E).item()) & ((1 << 64) - 1)
    d = bench.splitmix_t(seed, k) & ((1 << 63) - 1)
    idx = d % pool
    batches = [ids_pool[idx[b * B:(b + 1) * B]].contiguous() for b in range(nb)]
    nows = [b + 1 for b in range(nb)]
    pol = mz.EvictionPolicy.disabled()
    st = torch.cuda.current_stream()
    caps = mz.even_capacities(rows, shards)
    t = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
    cold = run_batches(t, batches[:16], nows[:16], pol, st)
    t2 = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
    steady = run_batches(t2, batches, nows, pol, st, timed_from=16)
    t3 = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
    steady_async = run_batches_async(t3, batches, nows, pol, st, timed_from=16)
    bn = [b.cpu().numpy().view(np.uint64) for b in batches]
    ref = ref_time(caps, 128, bn, nows, 0, 0, warm=16)
    return dict(config=f"C1 S={shards}", cold_fill=cold, steady=steady, steady_pipelined=steady_async,
                reference=ref)


def zipf_cdf(universe, s=1.05):
    """The Zipf(s) CDF over `universe` ranks, computed on the host (sequential float64 sums) and
    moved to the GPU: a CUDA cumsum / sum of 2^27 doubles is not bitwise reproducible from run
    to run, which made the sampled streams (and their outcome counts) differ in a few positions
    between processes."""
    w = np.arange(1, universe + 1, dtype=np.float64) ** -s
    c = np.cumsum(w)
    c /= c[-1]
    return torch.from_numpy(c).cuda()


def zipf_ranks(n, s, universe, seed):
    # inverse CDF on a precomputed table, SplitMix64(3).next_unit()
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = torch.rand(n, generator=g, device="cuda", dtype=torch.float64)
    return torch.searchsorted(zipf_ranks.cdf, u).clamp_(max=universe - 1)


def c2():
    rows = 1 << 26
    universe = 1 << 27
    zipf_ranks.cdf = zipf_cdf(universe)
    B = 1 << 20
    # expected distinct ids of Zipf(1.05) over 2^27 reach 0.8 * 2^26 after ~700M draws, i.e.
    # ~700 batches at 60 s spacing: TTL 42,000 s targets a live occupancy near 0.8
    ttl = 42000
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(ttl))
    st = torch.cuda.current_stream()
    caps = mz.even_capacities(rows, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
    # warm up to steady state: 2 TTL periods of batches at 60 s spacing would be 2880
    # batches; run 1440 untimed batches, then time 64
    warm, timed = 1440, 64
    batches = []
    nows = []
    res = None
    for b in range(warm + timed):
        r = zipf_ranks(B, 1.05, universe, 1000 + b)
        batches.append(bench.distinct_ids_t(2, r).contiguous())
        nows.append(10**6 + 60 * b)
        if b == warm - 1:
            run_batches(t, batches, nows, pol, st)
            batches, nows = [], []
    res = run_batches(t, batches, nows, pol, st)
    live = int((torch.from_numpy(t.metadata_all().view(np.int64)) >= nows[-1]).sum())
    return dict(config="C2", ttl=ttl, live_occupancy=live / rows, steady=res)


def c2f():
    """Not a BASELINE config: C2 with three features carrying different TTLs (per-feature
    TTL: metadata values differ per feature, so batches take the A.4 rounds path)."""
    rows = 1 << 26
    universe = 1 << 27
    zipf_ranks.cdf = zipf_cdf(universe)
    B = 1 << 20
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(42000, {1: 21000, 2: 84000}))
    st = torch.cuda.current_stream()
    caps = mz.even_capacities(rows, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
    g = torch.Generator(device="cuda").manual_seed(77)
    warm, timed = 300, 16
    out_s = torch.empty(B, dtype=torch.int64, device="cuda")
    out_o = torch.empty(B, dtype=torch.uint8, device="cuda")
    for b in range(warm):
        r = zipf_ranks(B, 1.05, universe, 2000 + b)
        f = torch.randint(0, 3, (B,), generator=g, device="cuda", dtype=torch.int32)
        t.process_batch_device(bench.distinct_ids_t(2, r), 10**6 + 60 * b, pol, f, out_s, out_o, None, st)
    batches, feats, nows = [], [], []
    for b in range(warm, warm + timed):
        batches.append(bench.distinct_ids_t(2, zipf_ranks(B, 1.05, universe, 2000 + b)).contiguous())
        feats.append(torch.randint(0, 3, (B,), generator=g, device="cuda", dtype=torch.int32))
        nows.append(10**6 + 60 * b)
    torch.cuda.synchronize()

    def body():
        for b in range(timed):
            t.process_batch_device(batches[b], nows[b], pol, feats[b], out_s, out_o, None, st)
    ms = ev_time(body, st)
    return dict(config="C2 with per-feature TTL", ids_per_s=timed * B / (ms / 1e3),
                path=t.last_stats()["path"], rounds=t.last_stats()["rounds"])


def c3():
    rows = 1 << 28
    caps = mz.even_capacities(rows, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 256, 7))
    pol = mz.EvictionPolicy.disabled()
    st = torch.cuda.current_stream()
    npre = int(0.95 * rows)
    out_s = torch.empty(1 << 22, dtype=torch.int64, device="cuda")
    out_o = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
    t0 = time.perf_counter()
    for a in range(0, npre, 1 << 22):
        ids = bench.distinct_ids_t(3, torch.arange(a, min(a + (1 << 22), npre), dtype=torch.int64, device="cuda"))
        t.process_batch_device(ids, 1, pol, None, out_s, out_o, None, st)
    torch.cuda.synchronize()
    prefill_s = time.perf_counter() - t0
    B = 1 << 22
    g = torch.Generator(device="cuda").manual_seed(5)
    hit_idx = torch.randint(0, npre, (B,), generator=g, device="cuda")
    hits = bench.distinct_ids_t(3, hit_idx)
    half = torch.cat([hits[:B // 2], bench.distinct_ids_t(3, torch.arange(npre, npre + B // 2, device="cuda"))])

    def look(q):  # pipelined: 8 lookups enqueued, then every ticket waited
        t.wait(t.lookup_device_async(q, out_s, out_o, st))  # (warm-up: first-use scratch, kernel loads)

        def body():
            for tk in [t.lookup_device_async(q, out_s, out_o, st) for _ in range(8)]:
                t.wait(tk)
        return ev_time(body, st) / 8

    def look_sync(q):
        t.lookup_device(q, out_s, out_o, st)  # (warm-up)
        return ev_time(lambda: [t.lookup_device(q, out_s, out_o, st) for _ in range(8)], st) / 8
    lk = look(hits)
    lk_half = look(half)
    lk_sync = look_sync(hits)
    fresh = bench.distinct_ids_t(3, torch.arange(npre + B, npre + B + B // 2, device="cuda"))
    ins = [torch.cat([hits[:B // 2], fresh]).contiguous()]
    for i in range(1, 5):
        f2 = bench.distinct_ids_t(3, torch.arange(npre + (i + 1) * B, npre + (i + 1) * B + B // 2, device="cuda"))
        ins.append(torch.cat([hits[B // 2:], f2]).contiguous())
    r = run_batches(t, ins, [2 + i for i in range(5)], pol, st, timed_from=1)
    return dict(config="C3", prefill_s=prefill_s, lookup_ids_per_s=B / (lk / 1e3),
                lookup_50pct_absent_ids_per_s=B / (lk_half / 1e3),
                lookup_sync_call_ids_per_s=B / (lk_sync / 1e3), insert_heavy=r)


def c4():
    rows = 1 << 27
    caps = mz.even_capacities(rows, 8)
    t0 = time.perf_counter()
    t = mz.MpzchTable(mz.TableConfig(caps, 128, 7, 128, 11))
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(3600))
    st = torch.cuda.current_stream()
    npre = int(0.8 * rows)
    out_s = torch.empty(1 << 22, dtype=torch.int64, device="cuda")
    out_o = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
    for a in range(0, npre, 1 << 22):
        ids = bench.distinct_ids_t(4, torch.arange(a, min(a + (1 << 22), npre), dtype=torch.int64, device="cuda"))
        t.process_batch_device(ids, 1, pol, None, out_s, out_o, None, st)
    torch.cuda.synchronize()
    B = 1 << 20
    g = torch.Generator(device="cuda").manual_seed(41)
    batches = [bench.distinct_ids_t(41, torch.randint(0, 1 << 27, (B,), generator=g, device="cuda"))
               for _ in range(17)]
    nows = [10000 + 600 * i for i in range(17)]
    r = run_batches(t, batches, nows, pol, st, timed_from=1)
    reset_bytes = r["outcomes"]["evicted_rows"] * (128 * 8 + 1) / max(len(batches) - 1, 1)
    r["reset_bytes_per_batch"] = reset_bytes
    return dict(config="C4", init_draw_s=init_s, steady=r)


def lru(pool_factor=1.2):
    """Not a BASELINE config: C1-shaped LRU batches next to the reference on the same stream.
    pool_factor 0.8 (the C1 pool): no window fills, every batch runs the claim path;
    1.2: more ids than slots (full windows, LRU victims, double evictions) -- the claim
    attempt reverts and the A.4 rounds path runs."""
    rows = 1 << 20
    pool = int(pool_factor * rows)
    ids_pool = bench.distinct_ids_t(9, torch.arange(pool, dtype=torch.int64, device="cuda"))
    B, nb = 65536, 24
    g = torch.Generator(device="cuda").manual_seed(9)
    batches = [ids_pool[torch.randint(0, pool, (B,), generator=g, device="cuda")].contiguous()
               for _ in range(nb)]
    nows = [10 + b for b in range(nb)]
    st = torch.cuda.current_stream()
    out = {}
    bn = [b.cpu().numpy().view(np.uint64) for b in batches]
    for shards in (8, 64):
        caps = mz.even_capacities(rows, shards)
        t = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
        r = run_batches(t, batches, nows, mz.EvictionPolicy.lru(), st, timed_from=8, split=False)
        ref = ref_time(caps, 128, bn, nows, 2, 0, warm=8)
        out[f"lru_S{shards}"] = dict(gpu=r, reference=ref)
    return dict(config=f"LRU pool {pool_factor} x rows", **out)


def lru08():
    return lru(0.8)


def lru_zipf():
    """Not a BASELINE config: LRU under C2's Zipf(1.05) traffic over 2^27 ids on a 2^22-row table
    (8 shards, P=128, 1M-position batches): windows are full, so every batch evicts; the victims
    are cold tail ids, which the claim path places (K3b).  Beside it the same stream forced onto
    the rounds path."""
    rows, universe, B = 1 << 22, 1 << 27, 1 << 20
    zipf_ranks.cdf = zipf_cdf(universe)
    st = torch.cuda.current_stream()
    caps = mz.even_capacities(rows, 8)
    pol = mz.EvictionPolicy.lru()
    warm, timed = 48, 16
    batches = [bench.distinct_ids_t(2, zipf_ranks(B, 1.05, universe, 3000 + b)).contiguous()
               for b in range(warm + timed)]
    nows = [10**6 + 60 * b for b in range(warm + timed)]
    out = dict(config="LRU Zipf(1.05), 2^22 rows, 1M batches")
    for path in ("auto", "rounds"):
        t = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
        t.set_path(path)
        run_batches(t, batches[:warm], nows[:warm], pol, st, split=False)
        r = run_batches(t, batches[warm:], nows[warm:], pol, st, split=False)
        out[path] = r
    bn = [b.cpu().numpy().view(np.uint64) for b in batches]
    out["reference"] = ref_time(caps, 128, bn, nows, 2, 0, warm=warm)
    return out


def serve():
    """Not a BASELINE config: the frozen-replica read path -- batched lookup
    and fused lookup + row gather on a 2^24-row dim-128 table prefilled to 0.8, 1M-position
    batches (90% present ids, 10% absent)."""
    rows, dim, B = 1 << 24, 128, 1 << 20
    caps = mz.even_capacities(rows, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 128, 7, dim, 11))
    pol = mz.EvictionPolicy.disabled()
    st = torch.cuda.current_stream()
    npre = int(0.8 * rows)
    out_s = torch.empty(B, dtype=torch.int64, device="cuda")
    out_o = torch.empty(B, dtype=torch.uint8, device="cuda")
    for a in range(0, npre, B):
        ids = bench.distinct_ids_t(6, torch.arange(a, min(a + B, npre), dtype=torch.int64, device="cuda"))
        t.process_batch_device(ids, 1, pol, None, out_s, out_o, None, st)
    g = torch.Generator(device="cuda").manual_seed(6)
    nb = 10
    batches = [bench.distinct_ids_t(6, torch.randint(0, int(npre / 0.9), (B,), generator=g, device="cuda"))
               for _ in range(nb + 2)]
    torch.cuda.synchronize()
    rows_out = torch.empty((B, dim), dtype=torch.float32, device="cuda")
    trip = (out_s, out_o, rows_out)
    for b in range(2):
        t.lookup_device(batches[b], out_s, out_o, st)
        t.lookup_gather_device(batches[b], st, out=trip)
    def lookups():
        for tk in [t.lookup_device_async(batches[2 + b], out_s, out_o, st) for b in range(nb)]:
            t.wait(tk)
    ms_l = ev_time(lookups, st)
    ms_g = ev_time(lambda: [t.lookup_gather_device(batches[2 + b], st, out=trip) for b in range(nb)], st)
    found = int((out_o == 0).sum().item())
    return dict(config="serve (2^24 rows, dim 128, 1M-position lookups)", lookup_ids_per_s=nb * B / (ms_l / 1e3),
                lookup_gather_ids_per_s=nb * B / (ms_g / 1e3),
                gather_gbs=nb * B * dim * 4 * 2 / (ms_g / 1e3) / 1e9, found_fraction=found / B)


def publish():
    """Not a BASELINE config: publication images from HBM -- the .mpzc
    snapshot of a 2^22-row dim-128 table (2.1 GB image, CRC-32 on the device) and the .mpzd
    delta of the rows one 1M-position TTL batch dirtied."""
    rows, dim, B = 1 << 22, 128, 1 << 20
    caps = mz.even_capacities(rows, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 128, 7, dim, 11))
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(3600))
    st = torch.cuda.current_stream()
    npre = int(0.8 * rows)
    out_s = torch.empty(B, dtype=torch.int64, device="cuda")
    out_o = torch.empty(B, dtype=torch.uint8, device="cuda")
    for a in range(0, npre, B):
        ids = bench.distinct_ids_t(7, torch.arange(a, min(a + B, npre), dtype=torch.int64, device="cuda"))
        t.process_batch_device(ids, 1, pol, None, out_s, out_o, None, st)
    torch.cuda.synchronize()
    size = t.snapshot_size()
    buf = torch.empty(size, dtype=torch.uint8).pin_memory().numpy()  # page-locked image buffer
    t.serialize_snapshot_into(buf)  # warm (staging buffers)
    t0 = time.perf_counter()
    t.serialize_snapshot_into(buf)
    snap_s = time.perf_counter() - t0
    img = buf.tobytes()
    wts = torch.empty(rows * dim, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mz.crc32_device(wts)
    crc_s = time.perf_counter() - t0
    src = mz.DeltaSource(t, mz.snapshot_checksum(img))
    g = torch.Generator(device="cuda").manual_seed(7)
    ids = bench.distinct_ids_t(7, torch.randint(0, 2 * npre, (B,), generator=g, device="cuda"))
    t.process_batch_device(ids, 10000, pol, None, out_s, out_o, None, st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    delta = src.cut()
    delta_s = time.perf_counter() - t0
    return dict(config="publish (2^22 rows, dim 128)", snapshot_bytes=len(img), snapshot_s=snap_s,
                snapshot_gbs=len(img) / snap_s / 1e9, delta_bytes=len(delta), delta_s=delta_s,
                delta_gbs=len(delta) / delta_s / 1e9, crc32_device_gbs=rows * dim * 4 / crc_s / 1e9)


def train(reset_mode="eager", reference=True):
    """Not a BASELINE config: the reference's churn training loop (proj/src/experiments.cpp:86-125)
    at scale -- remap a batch (TTL evictions reset rows), then sgd_step over the distinct
    remapped rows -- on a 2^24-row dim-128 table (weights + momentum 16 GiB).  The reference
    runs the same loop (process_batch + sgd_step) on a 2^20-row sample.  reset_mode "deferred"
    fuses each evicted row's reset into its sgd_step."""
    rows, dim, B = 1 << 24, 128, 1 << 20
    caps = mz.even_capacities(rows, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 128, 7, dim, 11))
    t.set_reset_mode(reset_mode)
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(3600))
    st = torch.cuda.current_stream()
    npre = int(0.8 * rows)
    out_s = torch.empty(B, dtype=torch.int64, device="cuda")
    out_o = torch.empty(B, dtype=torch.uint8, device="cuda")
    for a in range(0, npre, B):
        ids = bench.distinct_ids_t(4, torch.arange(a, min(a + B, npre), dtype=torch.int64, device="cuda"))
        t.process_batch_device(ids, 1, pol, None, out_s, out_o, None, st)
    g = torch.Generator(device="cuda").manual_seed(5)
    nb = 12
    batches = [bench.distinct_ids_t(4, torch.randint(0, int(npre * 1.25), (B,), generator=g, device="cuda"))
               for _ in range(nb)]
    nows = [4000 + 400 * i for i in range(nb)]
    grads = (torch.rand((B, dim), generator=g, device="cuda") - 0.5).contiguous()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tm = {"remap": 0.0, "unique": 0.0, "sgd": 0.0}
    urows = 0
    evicted = 0
    for b in range(nb):
        ev[0].record(st)
        t.process_batch_device(batches[b], nows[b], pol, None, out_s, out_o, None, st)
        evicted += t.last_stats()["evicted_rows"]
        ev[1].record(st)
        rows_u = torch.unique(out_s)
        ev[2].record(st)
        t.sgd_step_device(rows_u, grads[:rows_u.numel()], 0.05, 0.9, st)
        ev[3].record(st)
        torch.cuda.synchronize()
        if b >= 2:
            tm["remap"] += ev[0].elapsed_time(ev[1])
            tm["unique"] += ev[1].elapsed_time(ev[2])
            tm["sgd"] += ev[2].elapsed_time(ev[3])
            urows += rows_u.numel()
    steps = nb - 2
    step_ms = sum(tm.values()) / steps
    sgd_bytes = urows / steps * dim * 4 * 5  # grad read + weights/momentum read and write
    out = dict(config=f"train (churn loop, 2^24 rows, dim 128, 1M-position batches, {reset_mode} resets)",
               ids_per_s=B / (step_ms / 1e3), step_ms=step_ms,
               split_ms={k: v / steps for k, v in tm.items()}, distinct_rows=urows / steps,
               evicted_rows=evicted / nb,
               sgd_gbs=sgd_bytes / (tm["sgd"] / steps / 1e3) / 1e9)
    # reference: the same loop on a 2^20-row sample, 64K-position batches
    import pyoracle
    if reference and pyoracle.available("reference"):
        pyoracle.lib("reference")["set_threads"](os.cpu_count() or 1)
        rrows, rB = 1 << 20, 1 << 16
        ref = pyoracle.OracleTable(mz.even_capacities(rrows, 8), 128, 7, dim, 11, kind="reference")
        pre = pyoracle.distinct_ids(4, 0, int(0.8 * rrows))
        for a in range(0, pre.size, 1 << 18):
            ref.process_batch(pre[a:a + (1 << 18)], 1, 1, 3600)
        rng = np.random.default_rng(5)
        gref = (rng.random((rB, dim), dtype=np.float32) - 0.5)
        tot, pos = 0.0, 0
        for b in range(6):
            ids = pyoracle.distinct_ids(4, 0, int(pre.size * 1.25))[rng.integers(0, int(pre.size * 1.25), rB)]
            s0 = time.perf_counter()
            sl, _, _ = ref.process_batch(ids, 4000 + 400 * b, 1, 3600)
            ur = np.unique(sl)
            ref.sgd_step(ur, gref[:ur.size], 0.05, 0.9)
            if b >= 1:
                tot += time.perf_counter() - s0
                pos += rB
        out["reference"] = dict(ids_per_s=pos / tot, cores=os.cpu_count(), kind="reference",
                                sample="2^20 rows, dim 128, 64K-position batches")
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c3", "c4"]
    out = []
    for w in which:
        torch.cuda.empty_cache()
        if w == "c1":
            res = [c1(1), c1(8)]
        elif w == "train_deferred":
            res = [train("deferred", reference=False)]
        else:
            res = [globals()[w]()]
        for r in res:
            out.append(r)
            print(json.dumps(r), flush=True)
