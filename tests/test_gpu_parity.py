"""GPU parity: the sm_100a path, called through the C-ABI, against the oracle.

Every comparison is bit-exact (integer slots/outcomes/evicted lists, identity and
metadata words, fp32 weights/momentum bit patterns, trained flags, row generations).
Checkers: the reference's own recorded outputs (tests/golden/ref_streams.npz) and the
C restatement (oracle/, itself pinned by tests/test_oracle.py).
"""
import numpy as np
import pytest

import paper_2602_17050_b200 as mz
from test_oracle import _fixture, replay_fixture

pytestmark = pytest.mark.gpu

EMPTY = np.uint64((1 << 64) - 1)


def pol(mode, dttl=0, pf=None):
    if mode == 1:
        return mz.EvictionPolicy.ttl(mz.TtlPolicy(dttl, dict(pf or {})))
    return mz.EvictionPolicy.lru() if mode == 2 else mz.EvictionPolicy.disabled()


def gpu_state(t, dim):
    d = dict(ident=t.identities_all(), meta=t.metadata_all())
    if dim:
        d.update(weights=t.weights().view(np.uint32), momentum=t.momentum().view(np.uint32),
                 trained=t.trained())
    return d


def oracle_state(o, dim):
    d = dict(ident=o.identities_all(), meta=o.metadata_all())
    if dim:
        d.update(weights=o.weights().view(np.uint32), momentum=o.momentum().view(np.uint32),
                 trained=o.trained())
    return d


def assert_same_state(a, b, tag=""):
    for k in a:
        assert (a[k] == b[k]).all(), f"{tag} state {k} differs"


# ---------------------------------------------------------------- reference fixtures

@pytest.mark.parametrize("path", ["auto", "ordered", "rounds"])
def test_replay_reference_fixtures(path):
    z, man = _fixture()
    paths_seen = set()

    def make(c):
        t = mz.MpzchTable(mz.TableConfig(c["caps"], c["max_probe"], int(c["seed"]), c["dim"],
                                         int(c["init_seed"])))
        t.set_path(path)
        return t

    def run(t, c, ids, f, now, dttl, pf):
        r = t.process_batch(ids, now, pol(c["mode"], dttl, pf), f)
        paths_seen.add(t.last_stats()["path"])
        return r

    def state(t, c):
        d = dict(ident=t.identities_all(), meta=t.metadata_all())
        if c["dim"]:
            d.update(weights=t.weights(), momentum=t.momentum(), trained=t.trained())
        return d

    n = replay_fixture(make, run, state, z, man)
    assert n == len(z["batches"])
    if path == "auto":
        assert {"fast", "rounds"} <= paths_seen  # the claim and rounds paths really ran
    if path == "rounds":
        assert "rounds" in paths_seen


# ---------------------------------------------------------------- probe-core scenarios
# proj/tests/test_probe_core.cpp, expressed through the table API on one shard: the
# window is written raw (mpzch_write_slots), then one id is remapped.

def find_id_with_home(oracle, target, cap, seed, start=1):
    L = oracle.lib("port")
    i = start
    while True:
        if L["home_slot"](i, cap, seed) == target:
            return i
        i += 1


def scenario(oracle, cap, P, seed, mode, slots, idents, metas, id, now, meta_in):
    """Run one probe on GPU (fast path when the raw window is hole-free) and on the
    oracle probe core; compare result and both arrays."""
    t = mz.MpzchTable(mz.TableConfig([cap], P, seed))
    if len(slots):
        t.write_slots(0, slots, idents, metas)
    t.check_hole_free()
    I = np.full(cap, EMPTY, dtype=np.uint64)
    M = np.zeros(cap, dtype=np.uint64)
    I[list(slots)] = idents
    M[list(slots)] = metas
    s, o, I2, M2 = oracle.probe(id, meta_in, now, I, M, cap, P, seed, mode)
    p = pol(mode, meta_in - now if mode == 1 else 0)
    gs, go, _ = t.process_batch(np.array([id], dtype=np.uint64), now, p)
    assert (int(gs[0]), int(go[0])) == (s, o)
    assert (t.identities_all() == I2).all() and (t.metadata_all() == M2).all()
    return s, o


def test_insert_and_refresh(oracle):
    cap, P, seed = 32, 8, 11
    p = find_id_with_home(oracle, 9, cap, seed)
    assert scenario(oracle, cap, P, seed, 1, [], [], [], p, 10, 110) == (9, mz.INSERTED)
    assert scenario(oracle, cap, P, seed, 1, [9], [p], [110], p, 50, 150) == (9, mz.FOUND)


def test_probes_past_occupied(oracle):
    cap, P, seed = 32, 8, 23
    p = find_id_with_home(oracle, 4, cap, seed)
    assert scenario(oracle, cap, P, seed, 0, [4, 5], [p + 1000, p + 2000], [0, 0], p, 7, 7) == (6, 1)


def test_pass1_shields_existing_entry(oracle):
    cap, P, seed, now = 64, 8, 5, 100
    p = find_id_with_home(oracle, 20, cap, seed)
    slots = [20, 21, 22, 23, 24, 25]
    ids = [1_000_000 + o for o in range(5)] + [p]
    metas = [now + 50, now - 1, now + 50, now + 50, now + 50, now + 1]
    assert scenario(oracle, cap, P, seed, 1, slots, ids, metas, p, now, now + 10) == (25, mz.FOUND)


def test_ttl_first_expired_and_strict_boundary(oracle):
    cap, P, seed, now = 64, 8, 5, 100
    p = find_id_with_home(oracle, 20, cap, seed)
    slots = list(range(20, 28))
    ids = [1_000_000 + o for o in range(8)]
    metas = [now + 50] * 8
    metas[2] = now - 1
    metas[4] = now - 30
    assert scenario(oracle, cap, P, seed, 1, slots, ids, metas, p, now, now + 10) == (22, mz.EVICTED)
    cap, P, seed, now = 16, 2, 3, 50
    p = find_id_with_home(oracle, 6, cap, seed)
    assert scenario(oracle, cap, P, seed, 1, [6, 7], [p + 500, p + 600], [now, now + 1], p, now,
                    now + 10)[1] == mz.COLLISION
    assert scenario(oracle, cap, P, seed, 1, [6, 7], [p + 500, p + 600], [now - 1, now + 1], p, now,
                    now + 10) == (6, mz.EVICTED)


def test_expired_before_empty_and_full_window(oracle):
    cap, P, seed, now = 32, 4, 9, 40
    p = find_id_with_home(oracle, 12, cap, seed)
    assert scenario(oracle, cap, P, seed, 1, [12], [p + 100], [now - 2], p, now, now + 5) == (12, 2)
    cap, P, seed, now = 64, 4, 5, 100
    p = find_id_with_home(oracle, 30, cap, seed)
    assert scenario(oracle, cap, P, seed, 1, [30, 31, 32, 33], [2_000_000 + o for o in range(4)],
                    [now + 5 + o for o in range(4)], p, now, now + 10) == (30, mz.COLLISION)
    cap, P, seed, now = 16, 3, 2, 9
    p = find_id_with_home(oracle, 5, cap, seed)
    assert scenario(oracle, cap, P, seed, 0, [5, 6, 7], [3_000_000 + o for o in range(3)], [1] * 3, p,
                    now, now) == (5, mz.COLLISION)


def test_lru_oldest_and_ties(oracle):
    cap, P, seed = 64, 3, 5
    p = find_id_with_home(oracle, 40, cap, seed)
    ids = [4_000_000 + o for o in range(3)]
    assert scenario(oracle, cap, P, seed, 2, [40, 41, 42], ids, [5, 9, 3], p, 20, 20) == (42, 2)
    assert scenario(oracle, cap, P, seed, 2, [40, 41, 42], ids, [4, 4, 7], p, 20, 20) == (40, 2)


def test_wrap_around_and_hole_lookup(oracle):
    cap, P, seed = 13, 4, 17
    p = find_id_with_home(oracle, 11, cap, seed)
    assert scenario(oracle, cap, P, seed, 0, [11, 12], [9_000_000, 9_000_001], [0, 0], p, 1, 1) == (0, 1)
    # hole: id at offset 2 behind two EMPTY slots must still be Found by lookup
    # (test_probe_core.cpp:113-121)
    cap, P, seed = 16, 4, 77
    q = find_id_with_home(oracle, 3, cap, seed)
    t = mz.MpzchTable(mz.TableConfig([cap], P, seed))
    t.write_slots(0, [5], [q], [0])
    assert not t.check_hole_free()
    s, o = t.lookup(np.array([q], dtype=np.uint64))
    assert (int(s[0]), int(o[0])) == (5, mz.FOUND)
    t2 = mz.MpzchTable(mz.TableConfig([cap], P, seed))
    t2.write_slots(0, [3 + P], [q], [0])  # one past the window: invisible
    assert int(t2.lookup(np.array([q], dtype=np.uint64))[1][0]) == mz.COLLISION


# ---------------------------------------------------------------- table/batch scenarios
# proj/tests/test_table_batch.cpp

def test_duplicates_share_one_probe_and_cascade(oracle):
    t = mz.MpzchTable(mz.TableConfig.even(32, 1, 4, 13))
    L = oracle.lib("port")
    p = find_id_with_home(oracle, 7, 32, 13)
    q = find_id_with_home(oracle, 7, 32, 13, p + 1)
    s, o, _ = t.process_batch(np.array([p, q, p, p], dtype=np.uint64), 1, mz.EvictionPolicy.disabled())
    assert list(o) == [1, 1, 1, 1] and list(s) == [7, 8, 7, 7]


def test_dedup_key_is_id_feature(oracle):
    t = mz.MpzchTable(mz.TableConfig.even(64, 1, 4, 2))
    ids = np.array([11, 11, 12, 11], dtype=np.uint64)
    f = np.array([5, 2, 2, 5], dtype=np.uint32)
    s, o, _ = t.process_batch(ids, 100, mz.EvictionPolicy.ttl(mz.TtlPolicy(1000, {5: 60})), f)
    assert list(o) == [1, 0, 1, 1] and s[0] == s[1] == s[3]
    # per-feature TTL, last writer (the (11, 2) unique, rank 1) wins the metadata word
    assert t.metadata_all()[s[0]] == 1100 and t.metadata_all()[s[2]] == 1100


def test_validation_before_mutation():
    t = mz.MpzchTable(mz.TableConfig.even(16, 2, 2, 4))
    with pytest.raises(mz.InvalidArgument, match="invalid id at batch position 1"):
        t.process_batch(np.array([1, 1 << 63], dtype=np.uint64), 5, mz.EvictionPolicy.disabled())
    assert (t.identities_all() == EMPTY).all()
    with pytest.raises(mz.OverflowError_):
        t.process_batch(np.array([1], dtype=np.uint64), (1 << 64) - 6,
                        mz.EvictionPolicy.ttl(mz.TtlPolicy(1000)))
    assert (t.identities_all() == EMPTY).all() and (t.metadata_all() == 0).all()
    # invalid id wins over overflow (dedup validation runs first, batch_engine.cpp:149-158)
    with pytest.raises(mz.InvalidArgument):
        t.process_batch(np.array([1, (1 << 64) - 1], dtype=np.uint64), (1 << 64) - 6,
                        mz.EvictionPolicy.ttl(mz.TtlPolicy(1000)))
    with pytest.raises(mz.InvalidArgument, match="empty-slot sentinel"):
        t.lookup(np.array([5, (1 << 64) - 1], dtype=np.uint64))
    # an empty batch is a no-op
    s, o, e = t.process_batch(np.zeros(0, dtype=np.uint64), 5, mz.EvictionPolicy.disabled())
    assert s.size == 0 and e.size == 0


def test_singleton_batch_equals_single_id_path(oracle):
    cfg = mz.TableConfig.even(48, 4, 4, 31, 2, 7)
    a, b = mz.MpzchTable(cfg), mz.MpzchTable(cfg)
    p = mz.EvictionPolicy.ttl(mz.TtlPolicy(50))
    rng = oracle.SplitMix64(88)
    uni = oracle.distinct_ids(55, 0, 40)
    now = 1
    for _ in range(300):
        now += rng.next_below(4)
        i = int(uni[rng.next_below(40)])
        f = rng.next_below(3)
        s, o, _ = a.process_batch(np.array([i], dtype=np.uint64), now, p, np.array([f], dtype=np.uint32))
        assert (int(s[0]), int(o[0])) == b.lookup_or_insert(i, f, now, p)
    assert_same_state(gpu_state(a, 2), gpu_state(b, 2))


def test_eviction_resets_row_bit_exact(oracle):
    cfg = mz.TableConfig([4, 4], 4, 3, 4, 9)
    t, twin = mz.MpzchTable(cfg), mz.MpzchTable(cfg)
    fresh = twin.weights()
    lru = mz.EvictionPolicy.lru()
    L = oracle.lib("port")
    res, cur = [], 1
    while len(res) < 4:  # fill shard 0 (test_table_batch.cpp:80-88)
        i = cur
        while not (L["shard_of"](i, 2, 3) == 0 and L["home_slot"](i, 4, 3) == len(res) % 4):
            i += 1
        cur = i + 1
        s, o = t.lookup_or_insert(i, 0, 10 + len(res), lru)
        if o == mz.INSERTED:
            res.append(i)
    for r in range(4):
        t.write_row(r, np.full(4, 0.5, np.float32), np.full(4, 0.25, np.float32), 1)
    i = cur
    while not (L["shard_of"](i, 2, 3) == 0 and L["home_slot"](i, 4, 3) == 2):
        i += 1
    s, o = t.lookup_or_insert(i, 0, 100, lru)
    assert o == mz.EVICTED and s < 4
    assert t.identities_all()[s] == i
    assert t.trained()[s] == 0 and (t.momentum()[s] == 0).all()
    assert (t.weights()[s].view(np.uint32) == fresh[s].view(np.uint32)).all()
    assert (t.weights()[s] == oracle.draw_row(4, s, 9)).all()


def test_dirty_tracking(oracle):
    t = mz.MpzchTable(mz.TableConfig.even(8, 1, 2, 5, 2, 0))
    ttl = mz.EvictionPolicy.ttl(mz.TtlPolicy(100))
    c1 = t.make_cursor()
    assert t.dirty_rows_since(c1).size == 0
    a = find_id_with_home(oracle, 1, 8, 5)
    s, o = t.lookup_or_insert(a, 0, 10, ttl)
    assert o == mz.INSERTED and list(t.dirty_rows_since(c1)) == [s]
    c2 = t.make_cursor()
    assert t.lookup_or_insert(a, 0, 20, ttl)[1] == mz.FOUND
    assert t.dirty_rows_since(c2).size == 0
    with pytest.raises(mz.InvalidArgument, match="stale or unknown publication cursor"):
        t.dirty_rows_since(999)


def test_construction_errors():
    with pytest.raises(mz.InvalidArgument, match="layout needs at least one shard"):
        mz.MpzchTable(mz.TableConfig([], 1, 0))
    with pytest.raises(mz.InvalidArgument, match="shard capacity must be >= 1"):
        mz.MpzchTable(mz.TableConfig([4, 0], 1, 0))
    with pytest.raises(mz.InvalidArgument, match="max_probe must satisfy"):
        mz.MpzchTable(mz.TableConfig([4, 4], 5, 0))


def test_init_weights_bit_exact(oracle):
    for dim in (1, 3, 8, 100, 128):
        t = mz.MpzchTable(mz.TableConfig.even(96, 3, 4, 1, dim, 0xDEADBEEF))
        w = t.weights()
        o = oracle.OracleTable(t.shard_capacities, 4, 1, dim, 0xDEADBEEF)
        assert (w.view(np.uint32) == o.weights().view(np.uint32)).all(), dim


# ---------------------------------------------------------------- randomized streams

def run_stream(oracle, caps, P, seed, dim, init_seed, batches, mode, dttl=0, pf=None, path="auto",
               check_state_every=0):
    t = mz.MpzchTable(mz.TableConfig(caps, P, seed, dim, init_seed))
    t.set_path(path)
    o = oracle.OracleTable(caps, P, seed, dim, init_seed)
    p = pol(mode, dttl, pf)
    for bi, (ids, f, now) in enumerate(batches):
        gs, go, ge = t.process_batch(ids, now, p, f)
        os_, oo, oe = o.process_batch(ids, now, mode, dttl, pf, f)
        assert (gs == os_).all(), f"slots differ at batch {bi}"
        assert (go == oo).all(), f"outcomes differ at batch {bi}"
        assert (ge == oe).all(), f"evicted list differs at batch {bi}"
        if check_state_every and bi % check_state_every == 0:
            assert_same_state(gpu_state(t, dim), oracle_state(o, dim), f"batch {bi}")
    assert_same_state(gpu_state(t, dim), oracle_state(o, dim), "final")
    return t


def test_c1_shape_stream(oracle):
    """C1 at full table size (2^20 rows, P=128, 64K-position batches over a 0.8*2^20 pool,
    Disabled) for 24 batches: cold fill through ~90% hits."""
    import workloads
    rows = 1 << 20
    pool = int(0.8 * rows)
    ids_pool = oracle.distinct_ids(1, 0, pool)
    idx = workloads.uniform_stream(1, pool, 65536, 24)
    batches = [(ids_pool[x], None, b + 1) for b, x in enumerate(idx)]
    t = run_stream(oracle, [rows], 128, 7, 0, 0, batches, 0)
    assert t.last_stats()["path"] == "fast"


def test_c1_multi_shard_with_features(oracle):
    import workloads
    rows = 1 << 18
    pool = int(0.9 * rows)
    ids_pool = oracle.distinct_ids(11, 0, pool)
    idx = workloads.uniform_stream(11, pool, 32768, 12)
    rng = np.random.default_rng(3)
    batches = [(ids_pool[x], rng.integers(0, 3, x.size).astype(np.uint32), b + 1)
               for b, x in enumerate(idx)]
    run_stream(oracle, mz.even_capacities(rows, 8), 32, 7, 0, 0, batches, 0)


@pytest.mark.parametrize("path", ["auto", "ordered"])
def test_ttl_eviction_reset_stream(oracle, path):
    """C4 shape at reduced size: prefill 0.8 at now=1 (TTL 3600), then fresh ids at
    now = 10000 + 600 t evict expired rows; dim 16 resets must be bit-exact."""
    rows = 1 << 16
    caps = mz.even_capacities(rows, 8)
    pre = oracle.distinct_ids(4, 0, int(0.8 * rows))
    fresh = oracle.distinct_ids(41, 0, 1 << 17)
    rng = np.random.default_rng(5)
    batches = [(pre[i:i + 8192], None, 1) for i in range(0, pre.size, 8192)]
    for t_ in range(6):
        batches.append((fresh[rng.integers(0, fresh.size, 16384)], None, 10000 + 600 * t_))
    run_stream(oracle, caps, 128, 7, 16, 11, batches, 1, 3600, None, path)


def test_ttl_mixed_hits_and_expiry(oracle):
    """Zipf-like reuse with a short TTL: hits on live slots, refreshes of expired own
    slots contested by lower-rank new ids (the owner path), evictions, collisions."""
    rows = 1 << 12
    uni = oracle.distinct_ids(2, 0, rows * 2)
    rng = np.random.default_rng(9)
    w = 1.0 / np.arange(1, uni.size + 1) ** 1.05
    w /= w.sum()
    batches = []
    for b in range(40):
        batches.append((uni[rng.choice(uni.size, 3000, p=w)], None, 1000 + 7 * b))
    run_stream(oracle, mz.even_capacities(rows, 2), 16, 3, 0, 0, batches, 1, 20, None,
               check_state_every=5)


def test_lru_dense_stream(oracle):
    rows = 1 << 10
    uni = oracle.distinct_ids(8, 0, rows * 3)
    rng = np.random.default_rng(2)
    batches = [(uni[rng.integers(0, uni.size, 700)], rng.integers(0, 2, 700).astype(np.uint32),
                5 + b // 2) for b in range(30)]
    run_stream(oracle, [rows // 2, rows // 2], 8, 5, 4, 1, batches, 2)


def test_lookup_matches_oracle(oracle):
    rows = 1 << 16
    caps = mz.even_capacities(rows, 4)
    t = mz.MpzchTable(mz.TableConfig(caps, 64, 9))
    o = oracle.OracleTable(caps, 64, 9)
    ids = oracle.distinct_ids(3, 0, int(0.95 * rows))
    for i in range(0, ids.size, 8192):
        t.process_batch(ids[i:i + 8192], 1, mz.EvictionPolicy.disabled())
        o.process_batch(ids[i:i + 8192], 1, 0)
    q = np.concatenate([ids[::3], oracle.distinct_ids(3, ids.size, 20000)])
    gs, go = t.lookup(q)
    os_, oo = o.lookup(q)
    assert (gs == os_).all() and (go == oo).all()
    assert (t.identities_all() == o.identities_all()).all()


def test_lookup_long_walk_hand_over(oracle):
    """Synchronous lookups of >= 256K positions at max_probe 256 hand their long walks (after 4
    line rounds) to a resume launch: host-buffer and device-buffer calls, hits and misses at
    0.95 load, against the oracle; the ticketed call (no hand-over) agrees too."""
    import torch
    rows = 1 << 20
    caps = mz.even_capacities(rows, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 256, 9))
    o = oracle.OracleTable(caps, 256, 9)
    ids = oracle.distinct_ids(13, 0, int(0.95 * rows))
    for i in range(0, ids.size, 1 << 18):
        t.process_batch(ids[i:i + (1 << 18)], 1, mz.EvictionPolicy.disabled())
        o.process_batch(ids[i:i + (1 << 18)], 1, 0)
    q = np.concatenate([ids[::2], oracle.distinct_ids(13, ids.size, 150_000)])
    assert q.size >= 1 << 18
    os_, oo = o.lookup(q)
    gs, go = t.lookup(q)
    assert (gs == os_).all() and (go == oo).all()
    qd = torch.from_numpy(q.view(np.int64)).cuda()
    ds = torch.empty(q.size, dtype=torch.int64, device="cuda")
    do = torch.empty(q.size, dtype=torch.uint8, device="cuda")
    t.lookup_device(qd, ds, do)
    torch.cuda.synchronize()
    assert (ds.cpu().numpy().view(np.uint64) == os_).all() and (do.cpu().numpy() == oo).all()
    ds.zero_()
    t.wait(t.lookup_device_async(qd, ds, do))
    assert (ds.cpu().numpy().view(np.uint64) == os_).all() and (do.cpu().numpy() == oo).all()


def test_hole_import_uses_exact_path(oracle):
    """After a raw import with a hole, remaps follow the full two-pass semantics
    (pass 2 inserts at the EMPTY in front of an existing copy, probe_core.cpp:89-101)."""
    cap, P, seed = 16, 4, 77
    q = find_id_with_home(oracle, 3, cap, seed)
    t = mz.MpzchTable(mz.TableConfig([cap], P, seed))
    t.write_slots(0, [5], [q], [0])
    o = oracle.OracleTable([cap], P, seed)
    oracle_I = o  # port table: emulate the raw write through probe on arrays instead
    I = np.full(cap, EMPTY, dtype=np.uint64)
    M = np.zeros(cap, dtype=np.uint64)
    I[5] = q
    s, oc, I2, M2 = oracle.probe(q, 3, 3, I, M, cap, P, seed, 0)
    gs, go, _ = t.process_batch(np.array([q], dtype=np.uint64), 3, mz.EvictionPolicy.disabled())
    assert (int(gs[0]), int(go[0])) == (s, oc) == (3, mz.INSERTED)
    assert (t.identities_all() == I2).all()


def test_device_buffer_entry_point(oracle):
    import torch
    rows = 1 << 14
    t = mz.MpzchTable(mz.TableConfig.even(rows, 2, 32, 5))
    o = oracle.OracleTable(mz.even_capacities(rows, 2), 32, 5)
    ids = oracle.distinct_ids(6, 0, 9000)
    d = torch.from_numpy(ids.view(np.int64)).cuda()
    slots = torch.empty(ids.size, dtype=torch.int64, device="cuda")
    oc = torch.empty(ids.size, dtype=torch.uint8, device="cuda")
    ev = torch.empty(ids.size, dtype=torch.int64, device="cuda")
    nev = t.process_batch_device(d, 1, mz.EvictionPolicy.disabled(), None, slots, oc, ev)
    torch.cuda.synchronize()
    s, oo, e = o.process_batch(ids, 1, 0)
    assert nev == 0 and (slots.cpu().numpy().view(np.uint64) == s).all()
    assert (oc.cpu().numpy() == oo).all()
    assert t.kernel_launches() > 0


def test_default_stream_ordering(oracle):
    """ids produced by torch on its default stream (handle 0) immediately before the call
    must be seen complete: stream 0 means the legacy default stream, not a private one."""
    import torch
    import bench
    rows = 1 << 22
    t = mz.MpzchTable(mz.TableConfig.even(rows, 8, 128, 7))
    B = 1 << 20
    out_s = torch.empty(B, dtype=torch.int64, device="cuda")
    out_o = torch.empty(B, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for b in range(3):
        ids = bench.distinct_ids_t(5, torch.arange(b * B, (b + 1) * B, dtype=torch.int64, device="cuda"))
        t.process_batch_device(ids, 1, mz.EvictionPolicy.disabled(), None, out_s, out_o, None, st)
        assert t.last_stats()["found"] == 0  # fresh distinct ids are never found


def test_async_tickets_and_deferred_errors(oracle):
    """mpzch_process_batch_device_async: batches pipeline on one stream; each ticket's wait
    reports that batch's result or error; a failed batch mutates nothing."""
    import torch
    rows = 1 << 14
    caps = mz.even_capacities(rows, 4)
    t = mz.MpzchTable(mz.TableConfig(caps, 32, 5, 4, 2))
    o = oracle.OracleTable(caps, 32, 5, 4, 2)
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(30))
    uni = oracle.distinct_ids(6, 0, rows)
    rng = np.random.default_rng(4)
    host = []
    outs = []
    tickets = []
    for b in range(12):  # more batches than the 8-slot ring
        ids = uni[rng.integers(0, uni.size, 3000)].copy()
        if b == 5:
            ids[17] = np.uint64(1 << 63)
        host.append(ids)
        d = torch.from_numpy(ids.view(np.int64)).cuda()
        so = torch.empty(ids.size, dtype=torch.int64, device="cuda")
        oo = torch.empty(ids.size, dtype=torch.uint8, device="cuda")
        eo = torch.empty(ids.size, dtype=torch.int64, device="cuda")
        outs.append((d, so, oo, eo))
        tickets.append(t.process_batch_device_async(d, 10 + 20 * b, pol, None, so, oo, eo))
    for b, tk in enumerate(tickets):
        if b == 5:
            with pytest.raises(mz.InvalidArgument, match="invalid id at batch position 17"):
                t.wait(tk)
            with pytest.raises(oracle.OracleError):
                o.process_batch(host[b], 10 + 20 * b, 1, 30)
            continue
        nev = t.wait(tk)
        s, oc, e = o.process_batch(host[b], 10 + 20 * b, 1, 30)
        _, so, oo, eo = outs[b]
        assert (so.cpu().numpy().view(np.uint64) == s).all() and (oo.cpu().numpy() == oc).all()
        assert nev == e.size and (eo[:nev].cpu().numpy().view(np.uint64) == e).all()
    assert_same_state(gpu_state(t, 4), oracle_state(o, 4))
    with pytest.raises(mz.InvalidArgument, match="unknown or expired batch ticket"):
        t.wait(10 ** 9)


def test_lookup_gather_matches_lookup_then_gather(oracle):
    """fused lookup + gather == MpzchTable::lookup then gather of the rows."""
    import torch
    rows = 1 << 14
    caps = mz.even_capacities(rows, 4)
    for dim in (128, 3):
        t = mz.MpzchTable(mz.TableConfig(caps, 32, 9, dim, 5))
        o = oracle.OracleTable(caps, 32, 9, dim, 5)
        ids = oracle.distinct_ids(12, 0, 12000)
        t.process_batch(ids[:9000], 1, mz.EvictionPolicy.disabled())
        o.process_batch(ids[:9000], 1, 0)
        q = ids[::2].copy()
        s, oc, r = t.lookup_gather_device(torch.from_numpy(q.view(np.int64)).cuda())
        os_, oo = o.lookup(q)
        assert (s.cpu().numpy().view(np.uint64) == os_).all() and (oc.cpu().numpy() == oo).all()
        assert (r.cpu().numpy().view(np.uint32) == o.weights()[os_.astype(np.int64)].view(np.uint32)).all()
    t0 = mz.MpzchTable(mz.TableConfig(caps, 32, 9))
    with pytest.raises(mz.LogicError):
        t0.lookup_gather_device(torch.zeros(4, dtype=torch.int64, device="cuda"))


def test_delta_cut_matches_dirty_rows(oracle):
    """DeltaSource::cut on device -- rows dirtied since the cursor (inserts,
    evictions, training writes), with identities and weights, then a fresh cursor."""
    rows = 1 << 12
    caps = mz.even_capacities(rows, 4)
    t = mz.MpzchTable(mz.TableConfig(caps, 16, 3, 8, 4))
    o = oracle.OracleTable(caps, 16, 3, 8, 4)
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(20))
    ids = oracle.distinct_ids(13, 0, 6000)
    c = t.make_cursor()
    oc_ = o.make_cursor()
    rng = np.random.default_rng(1)
    for b in range(3):
        batch = ids[rng.integers(0, ids.size, 1500)]
        t.process_batch(batch, 100 + 30 * b, pol)
        o.process_batch(batch, 100 + 30 * b, 1, 20)
    r, idn, w, nxt = t.delta_cut(c)
    want = o.dirty_rows_since(oc_)
    assert (r == want).all() and r.size > 0
    assert (idn == o.identities_all()[want.astype(np.int64)]).all()
    assert (w.view(np.uint32) == o.weights()[want.astype(np.int64)].view(np.uint32)).all()
    # nothing dirtied since the new cursor
    r2, _, _, _ = t.delta_cut(nxt)
    assert r2.size == 0
    with pytest.raises(mz.InvalidArgument, match="stale or unknown publication cursor"):
        t.delta_cut(0)



@pytest.mark.parametrize("path", ["auto", "ordered", "rounds"])
@pytest.mark.parametrize("shards", [1, 8])
def test_lru_and_feature_ttl_streams_all_paths(oracle, path, shards):
    """LRU (full windows, double evictions) and per-feature TTL batches at a dense load: auto
    (LRU: the claim path with K3b evictions, or the rounds path when an eviction cannot be
    placed there; per-feature TTL: the claim path with the last-writer metadata pass), the
    ordered path and forced rounds agree with the oracle."""
    rows = 1 << 13
    caps = mz.even_capacities(rows, shards)
    uni = oracle.distinct_ids(21, 0, int(rows * 1.3))
    rng = np.random.default_rng(shards)
    for mode, dttl, pf in ((2, 0, None), (1, 40, {1: 7, 2: 90})):
        batches = []
        for b in range(12):
            n = 3000
            f = rng.integers(0, 3, n).astype(np.uint32) if mode == 1 or b % 2 else None
            batches.append((uni[rng.integers(0, uni.size, n)], f, 100 + 9 * b))
        t = run_stream(oracle, caps, 16, 5, 4, 3, batches, mode, dttl, pf, path, check_state_every=4)
        if path == "auto":
            assert t.last_stats()["path"] in (("fast", "rounds") if mode == 2 else ("fast",))


@pytest.mark.parametrize("line", [False, True])
def test_lru_claim_path_and_fallback(oracle, line):
    """LRU batches go to the claim path (metadata writes held back, then applied); a new id
    whose window is full -- before the batch (probe) or filled by lower ranks (claims) -- evicts
    there too when K3b can place the eviction exactly, else the batch reverts its claims on the
    device and runs the rounds path.  With features, against the oracle, state compared after
    every batch."""
    rows = 1 << 12
    caps = mz.even_capacities(rows, 4)
    uni = oracle.distinct_ids(31, 0, int(rows * 1.25))
    rng = np.random.default_rng(7)
    batches, fill = [], 0
    for b in range(16):
        n = 600
        lo = 0 if b < 6 else fill // 2   # early batches: a sparse table, no full window
        fill = min(uni.size, fill + 350)
        f = rng.integers(0, 2, n).astype(np.uint32) if b % 3 == 0 else None
        batches.append((uni[rng.integers(lo, max(fill, 1), n)], f, 50 + 3 * b))
    paths = []
    t = mz.MpzchTable(mz.TableConfig(caps, 8 if not line else 256, 5, 4, 9))
    o = oracle.OracleTable(caps, 8 if not line else 256, 5, 4, 9)
    p = mz.EvictionPolicy.lru()
    for bi, (ids, f, now) in enumerate(batches):
        gs, go, ge = t.process_batch(ids, now, p, f)
        os_, oo, oe = o.process_batch(ids, now, 2, 0, None, f)
        assert (gs == os_).all() and (go == oo).all() and (ge == oe).all(), f"batch {bi}"
        assert_same_state(gpu_state(t, 4), oracle_state(o, 4), f"batch {bi}")
        st = t.last_stats()
        paths.append((st["path"], st["evicted"] > 0))
    assert ("fast", False) in paths and any(e for _, e in paths), paths
    if not line:  # max_probe 8: evicting batches on the claim path
        assert ("fast", True) in paths, paths


def _lru_case(oracle, caps, P, batches, want_paths):
    t = mz.MpzchTable(mz.TableConfig(caps, P, 5, 4, 9))
    o = oracle.OracleTable(caps, P, 5, 4, 9)
    p = mz.EvictionPolicy.lru()
    got = []
    for bi, (ids, now) in enumerate(batches):
        ids = np.asarray(ids, dtype=np.uint64)
        gs, go, ge = t.process_batch(ids, now, p)
        os_, oo, oe = o.process_batch(ids, now, 2, 0, None, None)
        assert (gs == os_).all() and (go == oo).all() and (ge == oe).all(), f"batch {bi}"
        assert_same_state(gpu_state(t, 4), oracle_state(o, 4), f"batch {bi}")
        got.append(t.last_stats()["path"])
    assert got[-1] == want_paths, got


@pytest.mark.parametrize("case", ["untouched", "found_before", "found_after", "found_before_next_after",
                                  "same_victim", "tied_now", "repeated_evictor"])
def test_lru_eviction_cases(oracle, case):
    """The K3b exactness conditions one by one, on a single 8-slot shard with max_probe 8 (every
    window is the whole shard): one evictor on an untouched victim stays on the claim path, and
    so does one whose least recently used slot was Found earlier in the batch (it is `now` at the
    evictor's turn, the next oldest is evicted); a victim Found after the evictor (a cascade),
    two evictors on one victim, and metadata tied with `now` revert to the rounds path.
    Results, evicted lists, metadata and reset rows equal the oracle's in every case."""
    ids = [1000 + 17 * k for k in range(8)]
    fill = [([x], 1 + k) for k, x in enumerate(ids)]  # metadata 1..8: ids[0] is the LRU slot
    new1, new2 = 5_000_001, 5_000_003
    last = {
        "untouched": ([ids[3], new1, ids[5]], 20, "fast"),
        "found_before": ([ids[0], new1], 20, "fast"),
        "found_before_next_after": ([ids[0], new1, ids[1]], 20, "rounds"),
        "found_after": ([new1, ids[0]], 20, "rounds"),
        "same_victim": ([new1, new2], 20, "rounds"),
        "tied_now": ([new1], 5, "rounds"),
        "repeated_evictor": ([new1, ids[2], new1, ids[6]], 21, "fast"),
    }[case]
    if case == "tied_now":
        fill = [(ids, 5)]  # every slot's metadata equals the evicting batch's `now`
    _lru_case(oracle, [8], 8, fill + [(last[0], last[1])], last[2])


def test_lru_evictions_sector_probe(oracle):
    """Batches above 256K positions (per-thread sector probe) over a pool 1.25x the table under
    LRU: evictions on the claim path and, where K3b cannot place one, the rounds path; results
    and state against the oracle after every batch."""
    rows = 1 << 17
    caps = mz.even_capacities(rows, 4)
    uni = oracle.distinct_ids(61, 0, int(rows * 1.25))
    rng = np.random.default_rng(9)
    t = mz.MpzchTable(mz.TableConfig(caps, 16, 7, 0, 3))
    o = oracle.OracleTable(caps, 16, 7, 0, 3)
    p = mz.EvictionPolicy.lru()
    seen = set()
    for b in range(5):
        ids = uni[rng.integers(0, uni.size, 300_000)]
        now = 100 + 20 * b
        gs, go, ge = t.process_batch(ids, now, p)
        os_, oo, oe = o.process_batch(ids, now, 2, 0, None, None)
        assert (gs == os_).all() and (go == oo).all() and (ge == oe).all(), f"batch {b}"
        st = t.last_stats()
        seen.add((st["path"], st["evicted"] > 0))
        assert_same_state(gpu_state(t, 0), oracle_state(o, 0), f"batch {b}")
    assert any(e for _, e in seen), seen


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_large_batches_sector_probe(oracle, mode):
    """Batches above 256K positions take the per-thread sector probe (the C5 kernel; smaller
    batches and max_probe >= 256 take the quad line walk): Disabled, uniform TTL (expired
    owners, evictions) and eviction-free LRU against the oracle, state after every batch."""
    rows = 1 << 20
    caps = mz.even_capacities(rows, 4)
    uni = oracle.distinct_ids(51 + mode, 0, int(rows * 0.75))
    rng = np.random.default_rng(mode)
    n = 300_000
    t = mz.MpzchTable(mz.TableConfig(caps, 64, 7, 4 if mode == 1 else 0, 3))
    o = oracle.OracleTable(caps, 64, 7, 4 if mode == 1 else 0, 3)
    p = pol(mode, 30, None)
    hi = 250_000
    for b in range(4):
        hi = min(uni.size, hi + 120_000)
        ids = uni[rng.integers(0, hi, n)]
        now = 100 + 20 * b
        gs, go, ge = t.process_batch(ids, now, p)
        os_, oo, oe = o.process_batch(ids, now, mode, 30, None, None)
        assert (gs == os_).all() and (go == oo).all() and (ge == oe).all(), f"batch {b}"
        assert t.last_stats()["path"] == "fast"
        dim = 4 if mode == 1 else 0
        assert_same_state(gpu_state(t, dim), oracle_state(o, dim), f"batch {b}")


def test_lookup_async_tickets(oracle):
    """mpzch_lookup_device_async: results equal the oracle's lookup, tickets interleave with
    remap batches in enqueue order, and an invalid id is reported at wait with the reference's
    require_valid_id text."""
    import torch
    caps = mz.even_capacities(1 << 14, 4)
    t = mz.MpzchTable(mz.TableConfig(caps, 32, 7))
    o = oracle.OracleTable(caps, 32, 7, 0, 0)
    ids = oracle.distinct_ids(3, 0, 12000)
    rng = np.random.default_rng(5)
    p = mz.EvictionPolicy.disabled()
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    checks = []
    for b in range(6):
        ins = ids[rng.integers(0, 9000, 4000)]
        q = ids[rng.integers(0, 12000, 5000)]
        di = torch.from_numpy(ins.view(np.int64)).to(dev)
        dq = torch.from_numpy(q.view(np.int64)).to(dev)
        os_ = torch.empty(4000, dtype=torch.int64, device=dev)
        oo = torch.empty(4000, dtype=torch.uint8, device=dev)
        ls = torch.empty(5000, dtype=torch.int64, device=dev)
        lo = torch.empty(5000, dtype=torch.uint8, device=dev)
        torch.cuda.synchronize()
        t1 = t.process_batch_device_async(di, 10 + b, p, None, os_, oo, None, st)
        t2 = t.lookup_device_async(dq, ls, lo, st)
        o.process_batch(ins, 10 + b, 0, 0, None, None)
        ws, wo = o.lookup(q)
        checks.append((t1, t2, ls, lo, ws, wo))
    for t1, t2, ls, lo, ws, wo in checks:
        t.wait(t1)
        t.wait(t2)
        assert (ls.cpu().numpy().view(np.uint64) == ws).all() and (lo.cpu().numpy() == wo).all()
    bad = torch.tensor([5, -1, 7], dtype=torch.int64, device=dev)
    tk = t.lookup_device_async(bad, torch.empty(3, dtype=torch.int64, device=dev),
                               torch.empty(3, dtype=torch.uint8, device=dev), st)
    with pytest.raises(mz.InvalidArgument, match="empty-slot sentinel"):
        t.wait(tk)


@pytest.mark.parametrize("seed", range(40))
def test_random_configurations(oracle, seed):
    """Randomised configurations against the oracle: shard count and uneven capacities (not
    multiples of the 16-row line), max_probe from 1 up to the smallest capacity (whole-shard
    wrapping windows), all three policies incl. per-feature TTL, batch sizes on both sides of
    the line/sector probe switch, features on some batches; results and the full state after
    every batch."""
    rng = np.random.default_rng(1000 + seed)
    S = int(rng.integers(1, 9))
    caps = [int(c) for c in rng.integers(60, 20000, S)]
    P = int(min(min(caps), rng.choice([1, 3, 8, 16, 48, 128, 256])))
    mode = int(rng.integers(0, 3))
    pf = {1: int(rng.integers(1, 40)), 2: int(rng.integers(1, 40))} if (mode == 1 and seed % 2) else None
    dttl = int(rng.integers(1, 60))
    dim = int(rng.choice([0, 0, 4]))
    seed_tab = int(rng.integers(0, 1 << 32))
    t = mz.MpzchTable(mz.TableConfig(caps, P, seed_tab, dim, 9))
    o = oracle.OracleTable(caps, P, seed_tab, dim, 9)
    pool = oracle.distinct_ids(seed, 0, int(sum(caps) * float(rng.choice([0.5, 0.9, 1.3]))))
    p = pol(mode, dttl, pf)
    now = 1
    for b in range(5):
        n = int(rng.choice([1, 17, 5000, 70000, 300000]))
        ids = pool[rng.integers(0, pool.size, n)]
        f = rng.integers(0, 3, n).astype(np.uint32) if (b % 2 or pf) else None
        now += int(rng.integers(0, 25))
        gs, go, ge = t.process_batch(ids, now, p, f)
        os_, oo, oe = o.process_batch(ids, now, mode, dttl, pf, f)
        assert (gs == os_).all(), f"slots differ: batch {b}, S={S}, P={P}, mode={mode}"
        assert (go == oo).all(), f"outcomes differ: batch {b}"
        assert (ge == oe).all(), f"evicted list differs: batch {b}"
        assert_same_state(gpu_state(t, dim), oracle_state(o, dim), f"batch {b}")


@pytest.mark.parametrize("P", [256, 300])
def test_high_load_insert_heavy_long_windows(oracle, P):
    """C3's shape at 2^18 rows: prefilled to 0.95, then insert-heavy batches (50% fresh) with long
    windows -- the one-line-lookahead probe, the 4-sector claim scan, takeover chains and ~30%
    collisions -- over uneven shards (wrap-around at every shard end), against the oracle."""
    caps = [40000, 70001, 65536, 86607]
    rows = sum(caps)
    t = mz.MpzchTable(mz.TableConfig(caps, P, 17))
    o = oracle.OracleTable(caps, P, 17)
    pol = mz.EvictionPolicy.disabled()
    ids = oracle.distinct_ids(23, 0, rows + 200000)
    npre = int(0.95 * rows)
    for a in range(0, npre, 60000):
        t.process_batch(ids[a:min(a + 60000, npre)], 1, pol)
        o.process_batch(ids[a:min(a + 60000, npre)], 1, 0)
    rng = np.random.default_rng(P)
    fresh = npre
    for b in range(4):
        hits = ids[rng.integers(0, npre, 20000)]
        new = ids[fresh:fresh + 20000]
        fresh += 20000
        batch = np.concatenate([hits, new])[rng.permutation(40000)]
        gs, go, _ = t.process_batch(batch, 2 + b, pol)
        os_, oo, _ = o.process_batch(batch, 2 + b, 0)
        assert (gs == os_).all() and (go == oo).all(), f"batch {b}: {(gs != os_).sum()} slots differ"
        assert (oo == 3).sum() > 1000  # the windows are full for many new ids
    assert (t.identities_all() == o.identities_all()).all()
    assert (t.metadata_all() == o.metadata_all()).all()


# ---------------------------------------------------------------- identity tags (P >= 256)
# Tables with max_probe >= 256 keep one tag byte per slot; Disabled batches on the claim path
# walk the window past its first identity line on the tags (k_probe_tag).  Every identity
# writer keeps them: the claim path, the rounds and ordered paths (any policy), raw writes.

@pytest.mark.parametrize("P", [256, 300])
def test_tags_follow_every_writer(oracle, P):
    """Batches cycling through every policy and path on one long-window table at high load
    (TTL and LRU evictions rewrite identities; forced ordered / rounds paths write them their
    own way), each followed by Disabled claim-path batches that walk the tags; results and
    the full state against the oracle after every batch."""
    caps = [3001, 4100, 2500]
    rows = sum(caps)
    t = mz.MpzchTable(mz.TableConfig(caps, P, 31))
    o = oracle.OracleTable(caps, P, 31)
    pool = oracle.distinct_ids(77, 0, int(rows * 1.3))
    rng = np.random.default_rng(P)
    plan = [(0, "auto"), (1, "auto"), (0, "auto"), (2, "auto"), (0, "auto"), (1, "ordered"),
            (0, "auto"), (2, "rounds"), (0, "auto"), (0, "ordered"), (0, "auto"), (1, "rounds"),
            (0, "auto"), (2, "ordered"), (0, "auto"), (0, "auto")]
    now = 1
    for b, (mode, path) in enumerate(plan):
        t.set_path(path)
        n = int(rng.choice([3000, 9000]))
        ids = pool[rng.integers(0, pool.size, n)]
        now += int(rng.integers(1, 6))
        p = pol(mode, 7)
        gs, go, ge = t.process_batch(ids, now, p)
        os_, oo, oe = o.process_batch(ids, now, mode, 7)
        assert (gs == os_).all(), f"slots differ: batch {b} ({mode}, {path}), {(gs != os_).sum()}"
        assert (go == oo).all(), f"outcomes differ: batch {b} ({mode}, {path})"
        assert (ge == oe).all(), f"evicted list differs: batch {b}"
        assert_same_state(gpu_state(t, 0), oracle_state(o, 0), f"batch {b}")
    t.set_path("auto")
    # the tag walk itself: lookups of every pooled id match after all of it
    s, oc = t.lookup(pool)
    os_, oo = o.lookup(pool)
    assert (s == os_).all() and (oc == oo).all()


def test_tags_raw_writes(oracle):
    """Raw slot writes (mpzch_write_slots) retag their slots: an id written 40 slots past its
    home -- beyond the first identity line, so only the tag walk can reach it -- is Found there;
    overwritten by another id, it becomes absent and inserts at the first EMPTY."""
    cap, P, seed = 4096, 256, 5
    h = 100
    q = find_id_with_home(oracle, h, cap, seed)
    fill = [find_id_with_home(oracle, s, cap, seed, 1 << 20) for s in range(h, h + 40)]
    t = mz.MpzchTable(mz.TableConfig([cap], P, seed))
    t.write_slots(0, list(range(h, h + 40)) + [h + 40], fill + [q], [0] * 41)
    assert t.check_hole_free()
    r = find_id_with_home(oracle, h, cap, seed, q + 1)
    dis = mz.EvictionPolicy.disabled()
    s, oc, _ = t.process_batch(np.array([q, r], dtype=np.uint64), 1, dis)
    assert [int(x) for x in s] == [h + 40, h + 41] and [int(x) for x in oc] == [mz.FOUND, mz.INSERTED]
    z = find_id_with_home(oracle, h + 40, cap, seed, 1 << 21)
    t.write_slots(0, [h + 40], [z], [0])
    assert t.check_hole_free()
    s, oc, _ = t.process_batch(np.array([q, z], dtype=np.uint64), 2, dis)
    assert [int(x) for x in s] == [h + 42, h + 40] and [int(x) for x in oc] == [mz.INSERTED, mz.FOUND]
