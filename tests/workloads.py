"""Seeded workload generators shared by the parity tests and the fixture generator.

Each generator restates one of the reference's own randomized test drivers
(paths relative to /root/reference/proj) with the same SplitMix64 draws:

* ``crit8_cases``   -- acceptance criterion 8, tests/acceptance_main.cpp:281-336
                       (multi-shard, heterogeneous capacities, Disabled/LRU/TTL with
                       per-feature TTL {1: 5}, features 0..2, embedding-backed configs)
* ``parallel_cases``-- "parallel and serial execution are bit-identical",
                       tests/test_table_batch.cpp:291-328
* ``oracle_cases``  -- make_oracle_case, tests/workloads.hpp:30-55 (single shard,
                       capacity <= 64, P <= 8, per-op TTL now+1..24)
* ``dense_cases``   -- the survey's high-contention regime (capacity
                       16-215, P <= 16, batch length up to capacity + 15)
"""
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from pyoracle import SplitMix64, distinct_ids

DISABLED, TTL, LRU = 0, 1, 2


@dataclass
class Batch:
    ids: np.ndarray
    features: Optional[np.ndarray]
    now: int
    default_ttl: int = 0            # TTL policy per batch (oracle_cases varies it per op)
    per_feature: Dict[int, int] = field(default_factory=dict)


@dataclass
class Case:
    name: str
    caps: List[int]
    max_probe: int
    seed: int
    dim: int
    init_seed: int
    mode: int
    batches: List[Batch]


def crit8_cases(seed=0x8A11E1, configs=50, batches=20):
    m = SplitMix64(seed)
    out = []
    for config in range(configs):
        shards = 2 + m.next_below(7)
        caps = [16 + m.next_below(81) for _ in range(shards)]
        P = 1 + m.next_below(8)
        tseed = m.next()
        dim = 2 if config % 2 == 0 else 0
        init_seed = m.next()
        mode = DISABLED
        if config % 3 == 1:
            mode = LRU
        if config % 3 == 2:
            mode = TTL
        total = sum(caps)
        universe = distinct_ids(m.next(), 0, total * 3 // 2)
        now = 1
        bl = []
        for _ in range(batches):
            now += 1 + m.next_below(8)
            length = 32 + m.next_below(225)
            ids = np.empty(length, dtype=np.uint64)
            f = np.empty(length, dtype=np.uint32)
            for k in range(length):
                ids[k] = universe[m.next_below(universe.size)]
                f[k] = m.next_below(3)
            bl.append(Batch(ids, f, now, 20 if mode == TTL else 0, {1: 5} if mode == TTL else {}))
        out.append(Case(f"crit8_{config}", caps, P, tseed, dim, init_seed, mode, bl))
    return out


def parallel_cases(seed=4096, rounds=8, batches=12):
    rng = SplitMix64(seed)
    out = []
    for rnd in range(rounds):
        shards = 1 + rng.next_below(6)
        caps = [8 + rng.next_below(56) for _ in range(shards)]
        P = 1 + rng.next_below(8)
        tseed = rng.next()
        init_seed = rng.next()
        mode = LRU if rnd % 2 == 0 else TTL
        universe = distinct_ids(rng.next(), 0, sum(caps) * 2)
        now = 1
        bl = []
        for _ in range(batches):
            now += 1 + rng.next_below(10)
            length = 1 + rng.next_below(96)
            ids = np.empty(length, dtype=np.uint64)
            f = np.empty(length, dtype=np.uint32)
            for k in range(length):
                ids[k] = universe[rng.next_below(universe.size)]
                f[k] = rng.next_below(2)
            bl.append(Batch(ids, f, now, 30 if mode == TTL else 0))
        out.append(Case(f"parallel_{rnd}", caps, P, tseed, 2, init_seed, mode, bl))
    return out


def oracle_cases(seed=0xACCE97, count=200):
    """Single-shard op sequences; each op becomes a singleton batch whose TTL policy
    reproduces the op's meta_in (workloads.hpp:51: meta_in = now + 1 + next_below(24))."""
    rng = SplitMix64(seed)
    out = []
    for c in range(count):
        cap = 1 + rng.next_below(64)
        P = 1 + rng.next_below(min(8, cap))
        tseed = rng.next()
        mode = [DISABLED, TTL, LRU][rng.next_below(3)]
        universe = 1 + rng.next_below(2 * cap)
        nops = 40 + rng.next_below(120)
        stream_seed = tseed ^ 0xABCDEF
        now = 1
        bl = []
        for _ in range(nops):
            now += rng.next_below(8)
            idx = rng.next_below(universe)
            meta = now + 1 + rng.next_below(24) if mode == TTL else now
            ids = distinct_ids(stream_seed, idx, 1)
            bl.append(Batch(ids, None, now, meta - now if mode == TTL else 0))
        out.append(Case(f"oracle_{c}", [cap], P, tseed, 0, 0, mode, bl))
    return out


def dense_cases(seed=0xDE45E, count=60, batches=12):
    rng = SplitMix64(seed)
    out = []
    for c in range(count):
        cap = 16 + rng.next_below(200)
        P = 1 + rng.next_below(16)
        P = min(P, cap)
        tseed = rng.next()
        mode = [DISABLED, TTL, LRU][c % 3]
        universe = distinct_ids(rng.next(), 0, cap * 2)
        with_feat = c % 2 == 1
        now = 1
        bl = []
        for _ in range(batches):
            now += rng.next_below(6)
            length = 1 + rng.next_below(cap + 15)
            ids = np.empty(length, dtype=np.uint64)
            f = np.zeros(length, dtype=np.uint32)
            for k in range(length):
                ids[k] = universe[rng.next_below(universe.size)]
                if with_feat:
                    f[k] = rng.next_below(3)
            bl.append(Batch(ids, f if with_feat else None, now, 9 if mode == TTL else 0,
                            {1: 5} if (mode == TTL and c % 4 == 1) else {}))
        out.append(Case(f"dense_{c}", [cap], P, tseed, 3 if c % 5 == 0 else 0, rng.next(), mode, bl))
    return out


def uniform_stream(pool_seed, pool, batch, nbatches, fresh_pct=0, sampler_seed=None, start_now=1):
    """SURVEY 8d sampler: positions uniform over DistinctIdStream(pool_seed)[0, pool), or a
    fresh index pool + k with probability fresh_pct/100.  Vectorised: SplitMix64 draws are
    generated in bulk from the stream state (same sequence as the scalar generator)."""
    from pyoracle import mix64_np, splitmix_stream
    seed = int(mix64_np(np.array([pool_seed], dtype=np.uint64), 0x5CA1AB1E)[0]) if sampler_seed is None else sampler_seed
    per = 2 if fresh_pct else 1
    draws = splitmix_stream(seed, batch * nbatches * per)
    out = []
    fresh_k = 0
    for b in range(nbatches):
        d = draws[b * batch * per:(b + 1) * batch * per]
        if fresh_pct:
            coin = d[0::2] % np.uint64(100)
            pick = d[1::2] % np.uint64(pool)
            fresh = coin < np.uint64(fresh_pct)
            idx = pick.copy()
            nf = int(fresh.sum())
            idx[fresh] = np.arange(pool + fresh_k, pool + fresh_k + nf, dtype=np.uint64)
            fresh_k += nf
        else:
            idx = d % np.uint64(pool)
        out.append(idx)
    return out
