"""GPU: the row-sharded table's device-side protocol (mpzch_sharded_*, csrc/sharded.cu).

G ranks in one process on the one B200 (each on its own stream, P2P = same device), connected
with mpzch_sharded_connect_local; every phase of a batch is enqueued by one host thread for all
ranks before any wait (so no rank's enqueue may block on the device), then each rank's ticket
is waited -- the Disabled / TTL fast path takes exactly one host wait.  Results must equal the
single table: every slice's slots and outcomes, the global canonical evicted list on every rank,
each rank's held rows, against the oracle (pinned to the reference in tests/test_oracle.py).
LRU (the host-synchronous fallback) runs one host thread per rank."""
import threading

import numpy as np
import pytest
import torch

import paper_2602_17050_b200 as mz

pytestmark = pytest.mark.gpu


def make_ranks(cfg, world, max_batch):
    ranks = [mz.ShardedRank(cfg, r, world, max_batch, device=0) for r in range(world)]
    mz.ShardedRank.connect_local(ranks)
    return ranks


def split(n, world, rng=None):
    """contiguous slices in rank order (uneven, some possibly empty)"""
    if rng is None:
        return np.array_split(np.arange(n), world)
    cuts = np.sort(rng.integers(0, n + 1, world - 1))
    return np.split(np.arange(n), cuts)


def run_batch(ranks, ids, feats, now, pol, slices, threads=False):
    world = len(ranks)
    streams = [torch.cuda.Stream() for _ in range(world)]
    bufs = []
    for r in range(world):
        sl = slices[r]
        ti = torch.from_numpy(ids[sl].view(np.int64).copy()).cuda()
        tf = None if feats is None else torch.from_numpy(feats[sl].view(np.int32).copy()).cuda()
        bufs.append((ti, tf, torch.empty(max(sl.size, 1), dtype=torch.int64, device="cuda"),
                     torch.empty(max(sl.size, 1), dtype=torch.uint8, device="cuda"),
                     torch.empty(ranks[r].max_batch, dtype=torch.int64, device="cuda")))
    torch.cuda.synchronize()
    nev = [None] * world
    errs = [None] * world
    if not threads:
        tks = [ranks[r].process_batch_device_async(bufs[r][0], now, pol, bufs[r][1], bufs[r][2], bufs[r][3],
                                                   bufs[r][4], streams[r]) for r in range(world)]
        for r in range(world):
            try:
                nev[r] = ranks[r].wait(tks[r])
            except mz.MpzchError as e:
                errs[r] = e
    else:
        def worker(r):
            try:
                nev[r] = ranks[r].process_batch_device(bufs[r][0], now, pol, bufs[r][1], bufs[r][2], bufs[r][3],
                                                       bufs[r][4], streams[r])
            except mz.MpzchError as e:
                errs[r] = e
        th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
    torch.cuda.synchronize()
    out = []
    for r in range(world):
        n = slices[r].size
        if errs[r] is not None:
            out.append(errs[r])
            continue
        out.append((bufs[r][2][:n].cpu().numpy().view(np.uint64), bufs[r][3][:n].cpu().numpy(),
                    bufs[r][4][:nev[r]].cpu().numpy().view(np.uint64)))
    return out


def check_state(ranks, o, dim):
    ident, meta = o.identities_all(), o.metadata_all()
    w = o.weights() if dim else None
    for rk in ranks:
        t = rk.table
        assert (t.identities_all() == ident[t.row_lo:t.row_hi]).all(), f"rank {rk.rank} identities"
        assert (t.metadata_all() == meta[t.row_lo:t.row_hi]).all(), f"rank {rk.rank} metadata"
        if dim:
            assert (t.weights(t.row_lo, t.held_rows).view(np.uint32) ==
                    w[t.row_lo:t.row_hi].view(np.uint32)).all(), f"rank {rk.rank} weights"


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mode", ["disabled", "ttl", "ttl_features", "lru"])
def test_device_protocol_equals_single_table(oracle, world, mode):
    rng = np.random.default_rng(world * 10 + len(mode))
    caps = mz.even_capacities(1 << 14, 8)
    dim = 8 if mode.startswith("ttl") else 0
    cfg = mz.TableConfig(caps, 32, 7, dim, 3)
    per = {1: 7, 2: 90} if mode == "ttl_features" else {}
    pol = {"disabled": mz.EvictionPolicy.disabled(), "lru": mz.EvictionPolicy.lru(),
           "ttl": mz.EvictionPolicy.ttl(mz.TtlPolicy(30)),
           "ttl_features": mz.EvictionPolicy.ttl(mz.TtlPolicy(30, per))}[mode]
    omode = {"disabled": 0, "ttl": 1, "ttl_features": 1, "lru": 2}[mode]
    ranks = make_ranks(cfg, world, 20000)
    if mode == "ttl" and world == 4:  # the owners' resets deferred (fused into later reads)
        for rk in ranks:
            rk.table.set_reset_mode("deferred")
    o = oracle.OracleTable(caps, 32, 7, dim, 3)
    uni = oracle.distinct_ids(40 + world, 0, int((1 << 14) * 1.3))
    total_ev = 0
    for b in range(8):
        n = int(rng.choice([3000, 12000, 20000]))
        ids = uni[rng.integers(0, uni.size, n)]
        feats = rng.integers(0, 3, n).astype(np.uint32) if mode == "ttl_features" or b % 3 == 2 else None
        now = 1 + 17 * b
        slices = split(n, world, rng if b % 2 else None)
        out = run_batch(ranks, ids, feats, now, pol, slices, threads=(mode == "lru"))
        os_, oo, oe = o.process_batch(ids, now, omode, 30 if omode == 1 else 0, per, feats)
        for r in range(world):
            assert not isinstance(out[r], Exception), f"rank {r}: {out[r]!r}"
            s_, o_, e_ = out[r]
            assert (s_ == os_[slices[r]]).all() and (o_ == oo[slices[r]]).all(), f"batch {b} rank {r}"
            assert e_.size == oe.size and (e_ == oe).all(), f"batch {b} rank {r}: evicted list"
        total_ev += oe.size
        if mode != "lru":
            assert all(rk.last_stats()["host_waits"] == 1 for rk in ranks)
    if mode != "disabled":
        assert total_ev > 0
    check_state(ranks, o, dim)
    for rk in ranks:
        rk.close()


def test_device_protocol_errors_agree(oracle):
    """An invalid id in rank 2's slice: every rank raises the reference's message with the GLOBAL
    position (batch_engine.cpp:90-94) and nothing changes; a slice over max_batch fails every
    rank; then batches run normally (the epochs stay in step)."""
    world = 4
    caps = mz.even_capacities(1 << 12, 4)
    cfg = mz.TableConfig(caps, 16, 7)
    ranks = make_ranks(cfg, world, 4000)
    pol = mz.EvictionPolicy.disabled()
    ids = oracle.distinct_ids(5, 0, 2000)
    bad = ids.copy()
    bad[1000 + 17] = np.uint64(1 << 63)
    bad[1500 + 3] = np.uint64((1 << 64) - 1)
    out = run_batch(ranks, bad, None, 5, pol, split(2000, world))
    for r in range(world):
        assert isinstance(out[r], mz.InvalidArgument) and str(out[r]) == "invalid id at batch position 1017", out[r]
    for rk in ranks:
        assert (rk.table.identities_all() == np.uint64((1 << 64) - 1)).all()
    big = oracle.distinct_ids(6, 0, 4100)
    out = run_batch(ranks, big, None, 6, pol, [np.arange(0, 4001)] + [np.arange(4001 + i, 4002 + i) for i in range(3)])
    for r in range(world):
        assert isinstance(out[r], mz.InvalidArgument) and "exchange capacity" in str(out[r]), out[r]
    o = oracle.OracleTable(caps, 16, 7)
    out = run_batch(ranks, ids, None, 7, pol, split(2000, world))
    os_, oo, _ = o.process_batch(ids, 7, 0, 0)
    assert (np.concatenate([x[0] for x in out]) == os_).all()
    check_state(ranks, o, 0)


def test_device_protocol_c5_shape_vs_single_table():
    """C5's shape (S = 8, P = 128, 0.8 load, 90% hit / 10% fresh) at 2^22 rows over G = 8 ranks
    against the single B200 table fed the whole batches: identical slots, outcomes and state."""
    import bench
    rows, world, B = 1 << 22, 8, 1 << 19
    caps = mz.even_capacities(rows, 8)
    cfg = mz.TableConfig(caps, 128, 7)
    single = mz.MpzchTable(cfg)
    ranks = make_ranks(cfg, world, 1 << 20)
    npre = bench.prefill_count(rows)
    pol = mz.EvictionPolicy.disabled()
    fresh = npre
    for b in range(-4, 4):
        if b < 0:  # prefill chunks
            lo = (b + 4) * (npre // 4)
            hi = npre if b == -1 else lo + npre // 4
            idx = torch.arange(lo, hi, dtype=torch.int64)
        else:
            idx, nf = bench.batch_indices(torch, "cpu", npre, B, b, fresh, bench.SAMPLER_SEED)
            fresh += nf
        ids = bench.distinct_ids_t(bench.ID_SEED, idx).numpy().view(np.uint64)
        now = 2 + b
        gs, go, _ = single.process_batch(ids, now, pol)
        slices = split(ids.size, world)
        assert ids.size <= (1 << 20)  # the ranks' max_batch
        out = run_batch(ranks, ids, None, now, pol, slices)
        assert (np.concatenate([x[0] for x in out]) == gs).all(), f"batch {b}"
        assert (np.concatenate([x[1] for x in out]) == go).all(), f"batch {b}"
    ident = single.identities_all()
    for rk in ranks:
        t = rk.table
        assert (t.identities_all() == ident[t.row_lo:t.row_hi]).all()


def test_device_protocol_two_processes(oracle, tmp_path):
    """Two ranks as two PROCESSES on the one B200 (torchrun; gloo carries the export records
    once), each mapping the other's exchange region by CUDA IPC: every slice, the global evicted
    list on both ranks, one host wait per batch."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29541",
           os.path.join(root, "tests", "sharded_ipc_worker.py"), str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    import sharded_ipc_worker as w
    caps, P, batches = w.workload(oracle)
    o = oracle.OracleTable(caps, P, 7, 4, 3)
    for b, (ids, f, now) in enumerate(batches):
        os_, oo, oe = o.process_batch(ids, now, 1, 40, {}, f)
        got = [np.load(tmp_path / f"r{r}_b{b}.npz") for r in range(2)]
        assert (np.concatenate([g["s"] for g in got]) == os_).all(), f"batch {b}"
        assert (np.concatenate([g["o"] for g in got]) == oo).all(), f"batch {b}"
        for g in got:
            assert (g["e"] == oe).all()
            assert int(g["hw"]) == 1


def test_device_protocol_ttl_overflow_and_precedence(oracle):
    """TTL expiry overflow (eviction.cpp:26-28) decided by every rank alike: a per-feature TTL that
    overflows at `now` for a feature present only in rank 1's slice fails every rank; a uniform
    TTL that overflows fails every rank; an invalid id anywhere takes precedence over the
    overflow (the reference validates first, batch_engine.cpp:90-94); nothing is mutated."""
    world = 2
    caps = mz.even_capacities(1 << 12, 4)
    cfg = mz.TableConfig(caps, 16, 7, 4, 3)
    ranks = make_ranks(cfg, world, 4000)
    ids = oracle.distinct_ids(8, 0, 1000)
    now = (1 << 64) - 100
    per = mz.EvictionPolicy.ttl(mz.TtlPolicy(10, {5: 1000}))   # feature 5 overflows, others do not
    feats = np.zeros(1000, np.uint32)
    feats[700] = 5                                               # rank 1's slice
    out = run_batch(ranks, ids, feats, now, per, split(1000, world), threads=True)
    for r in range(world):
        assert isinstance(out[r], mz.OverflowError_), out[r]
    feats[700] = 0
    out = run_batch(ranks, ids, feats, now, per, split(1000, world), threads=True)  # no overflowing feature present
    for r in range(world):
        assert not isinstance(out[r], Exception), out[r]
    uni = mz.EvictionPolicy.ttl(mz.TtlPolicy(1000))
    out = run_batch(ranks, oracle.distinct_ids(9, 0, 800), None, now, uni, split(800, world), threads=True)
    for r in range(world):
        assert isinstance(out[r], mz.OverflowError_), out[r]
    bad = oracle.distinct_ids(10, 0, 800)
    bad[650] = np.uint64((1 << 64) - 1)
    out = run_batch(ranks, bad, None, now, uni, split(800, world), threads=True)
    for r in range(world):
        assert isinstance(out[r], mz.InvalidArgument) and str(out[r]) == "invalid id at batch position 650", out[r]
    o = oracle.OracleTable(caps, 16, 7, 4, 3)
    o.process_batch(ids, now, 1, 10, {5: 1000}, feats)  # the one batch that went through
    check_state(ranks, o, 4)


@pytest.mark.parametrize("world", [2, 3])
def test_device_protocol_long_windows_tags(oracle, world):
    """max_probe 256 (the owners keep identity tags: tag walks, tag-guided claims) over uneven
    shard capacities (a rank's held rows start off a 128-row tag line), at high load, Disabled
    and TTL batches alternating: every slice and each rank's held state against the oracle."""
    rng = np.random.default_rng(300 + world)
    caps = [3001, 2500, 4100, 1777, 2999]
    cfg = mz.TableConfig(caps, 256, 11)
    ranks = make_ranks(cfg, world, 20000)
    o = oracle.OracleTable(caps, 256, 11)
    uni = oracle.distinct_ids(90 + world, 0, int(sum(caps) * 1.1))
    for b in range(8):
        mode = b % 2
        pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(5)) if mode else mz.EvictionPolicy.disabled()
        n = int(rng.choice([4000, 12000]))
        ids = uni[rng.integers(0, uni.size, n)]
        now = 1 + 3 * b
        slices = split(n, world, rng)
        out = run_batch(ranks, ids, None, now, pol, slices)
        os_, oo, oe = o.process_batch(ids, now, mode, 5 if mode else 0)
        for r in range(world):
            assert not isinstance(out[r], Exception), f"rank {r}: {out[r]!r}"
            s_, o_, e_ = out[r]
            assert (s_ == os_[slices[r]]).all() and (o_ == oo[slices[r]]).all(), f"batch {b} rank {r}"
            assert e_.size == oe.size and (e_ == oe).all(), f"batch {b} rank {r}: evicted list"
    check_state(ranks, o, 0)
    for rk in ranks:
        rk.close()
