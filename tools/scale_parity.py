"""At-scale parity: replay a full-size stream through the B200 table and the
reference library (oracle/_ref, OpenMP) side by side; compare every batch's per-position slots
and outcomes and the canonical evicted list, then the final identity and metadata arrays (and,
with rows, the weights / momentum / trained flags).  Prints one JSON line per config.

    python tools/scale_parity.py c2 c3 lru_zipf c4s
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
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench  # noqa: E402
import paper_2602_17050_b200 as mz  # noqa: E402
import pyoracle  # noqa: E402
from bench_configs import zipf_cdf, zipf_ranks  # noqa: E402


def zipf_setup(universe):
    zipf_ranks.cdf = zipf_cdf(universe)


def replay(name, caps, P, dim, init_seed, mode, ttl, pf, batches, feats=None):
    """batches: list of (ids u64 numpy, now); feats: list of u32 arrays or None."""
    t = mz.MpzchTable(mz.TableConfig(caps, P, 7, dim, init_seed))
    L = pyoracle.lib("reference")
    L["set_threads"](os.cpu_count() or 1)
    o = pyoracle.OracleTable(caps, P, 7, dim, init_seed, kind="reference")
    pol = (mz.EvictionPolicy.ttl(mz.TtlPolicy(ttl, pf or {})) if mode == 1 else
           mz.EvictionPolicy.lru() if mode == 2 else mz.EvictionPolicy.disabled())
    paths, evicted, positions = {}, 0, 0
    t0 = time.perf_counter()
    for b, (ids, now) in enumerate(batches):
        f = feats[b] if feats else None
        gs, go, ge = t.process_batch(ids, now, pol, f)
        rs, ro, re_ = o.process_batch(ids, now, mode, ttl, pf or {}, f)
        st = t.last_stats()
        paths[st["path"]] = paths.get(st["path"], 0) + 1
        evicted += int(ge.size)
        positions += int(ids.size)
        if not ((gs == rs).all() and (go == ro).all() and ge.size == re_.size and (ge == re_).all()):
            bad = np.nonzero((gs != rs) | (go != ro))[0]
            return dict(config=name, ok=False, batch=b, differing_positions=int(bad.size),
                        evicted=[int(ge.size), int(re_.size)])
    state = {"identities": bool((t.identities_all() == o.identities_all()).all()),
             "metadata": bool((t.metadata_all() == o.metadata_all()).all())}
    if dim:
        state["weights"] = bool((t.weights().view(np.uint32) == o.weights().view(np.uint32)).all())
        state["momentum"] = bool((t.momentum().view(np.uint32) == o.momentum().view(np.uint32)).all())
        state["trained"] = bool((t.trained() == o.trained()).all())
    return dict(config=name, ok=all(state.values()), batches=sum(paths.values()), positions=positions,
                evicted_slots=evicted, paths=paths, final_state=state,
                seconds=round(time.perf_counter() - t0, 1))


def c2(nb=160):
    """C2 shape (2^26 rows, S=8, P=128, Zipf(1.05) over 2^27 ids, 1M batches, now += 60 s) with
    TTL 3,000 s so expiry starts after 50 batches."""
    universe = 1 << 27
    zipf_setup(universe)
    batches = [(bench.distinct_ids_t(2, zipf_ranks(1 << 20, 1.05, universe, 1000 + b)).cpu().numpy().view(np.uint64),
                10**6 + 60 * b) for b in range(nb)]
    return replay("C2-shaped TTL stream (2^26 rows, TTL 3000 s)", mz.even_capacities(1 << 26, 8), 128, 0, 0,
                  1, 3000, None, batches)


def c2f(nb=120):
    universe = 1 << 27
    zipf_setup(universe)
    g = np.random.default_rng(77)
    batches = [(bench.distinct_ids_t(2, zipf_ranks(1 << 20, 1.05, universe, 2000 + b)).cpu().numpy().view(np.uint64),
                10**6 + 60 * b) for b in range(nb)]
    feats = [g.integers(0, 3, 1 << 20).astype(np.uint32) for _ in range(nb)]
    return replay("C2-shaped per-feature TTL stream (2^26 rows, TTL 3000 / {1: 1500, 2: 6000})",
                  mz.even_capacities(1 << 26, 8), 128, 0, 0, 1, 3000, {1: 1500, 2: 6000}, batches, feats)


def c3(nb=6):
    """C3 (2^28 rows at 0.95, P=256): prefill through both, then insert-heavy batches."""
    rows = 1 << 28
    npre = int(0.95 * rows)
    B = 1 << 22
    batches = [(bench.distinct_ids_t(3, torch.arange(a, min(a + B, npre), dtype=torch.int64)).numpy().view(np.uint64), 1)
               for a in range(0, npre, B)]
    g = torch.Generator().manual_seed(5)
    for i in range(nb):
        hits = bench.distinct_ids_t(3, torch.randint(0, npre, (B // 2,), generator=g))
        fresh = bench.distinct_ids_t(3, torch.arange(npre + i * B, npre + i * B + B // 2))
        batches.append((torch.cat([hits, fresh]).numpy().view(np.uint64), 2 + i))
    return replay("C3 (2^28 rows prefilled to 0.95, P=256, insert-heavy batches)", mz.even_capacities(rows, 8),
                  256, 0, 0, 0, 0, None, batches)


def lru_zipf(nb=40):
    universe = 1 << 27
    zipf_setup(universe)
    batches = [(bench.distinct_ids_t(2, zipf_ranks(1 << 20, 1.05, universe, 3000 + b)).cpu().numpy().view(np.uint64),
                10**6 + 60 * b) for b in range(nb)]
    return replay("LRU Zipf (2^22 rows, 1M batches)", mz.even_capacities(1 << 22, 8), 128, 0, 0, 2, 0, None, batches)


def c4s(nb=12):
    """C4 shape at 2^23 rows (dim 128 fp32 rows, TTL 3600, prefill 0.8 at now=1, then uniform
    fresh ids at now = 10000 + 600 t): resets compared row for row."""
    rows = 1 << 23
    npre = int(0.8 * rows)
    B = 1 << 20
    batches = [(bench.distinct_ids_t(4, torch.arange(a, min(a + B, npre), dtype=torch.int64)).numpy().view(np.uint64), 1)
               for a in range(0, npre, B)]
    g = torch.Generator().manual_seed(41)
    for i in range(nb):
        batches.append((bench.distinct_ids_t(41, torch.randint(0, 1 << 27, (B,), generator=g)).numpy().view(np.uint64),
                        10000 + 600 * i))
    return replay("C4-shaped (2^23 rows, dim 128, TTL 3600 evictions + row resets)", mz.even_capacities(rows, 8),
                  128, 128, 11, 1, 3600, None, batches)


def c5(nb=8):
    """C5 at full size: 2^30 rows (S=8, P=128), prefilled to 0.8 through both, then the bench's
    4M-position batches (90% hits, 10% fresh)."""
    rows = bench.ROWS
    npre = bench.prefill_count(rows)
    B = bench.BATCH

    def gen():
        for a in range(0, npre, B):
            yield bench.distinct_ids_t(bench.ID_SEED, torch.arange(a, min(a + B, npre), dtype=torch.int64)).numpy().view(np.uint64), 1
        fresh = npre
        for b in range(nb):
            idx, nf = bench.batch_indices(torch, "cpu", npre, B, b, fresh, bench.SAMPLER_SEED)
            fresh += nf
            yield bench.distinct_ids_t(bench.ID_SEED, idx).numpy().view(np.uint64), 2 + b
    return replay("C5 (2^30 rows prefilled to 0.8, 4M-position batches 90% hit / 10% fresh)",
                  mz.even_capacities(rows, bench.SHARDS), bench.MAX_PROBE, 0, 0, 0, 0, None, gen())


if __name__ == "__main__":
    for w in sys.argv[1:] or ["c2", "c3", "lru_zipf", "c4s"]:
        print(json.dumps(globals()[w]()), flush=True)
