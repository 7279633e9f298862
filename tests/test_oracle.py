"""CPU: pin the oracle before trusting it.

1. The C restatement (oracle/mpzch_oracle.c) against every golden vector the
   reference's tests hold for this path (tests/golden/known_answers.json).
2. The restatement against the reference library's own outputs on 238 seeded
   workloads (tests/golden/ref_streams.npz, produced by gen_golden.py from
   oracle/_ref): per-position slots/outcomes, evicted lists, final state.
3. When oracle/_ref is present, restatement vs reference live on fresh streams.
"""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
KA = json.load(open(os.path.join(HERE, "golden", "known_answers.json")))


def _kinds(oracle):
    return ["port"] + (["reference"] if oracle.available("reference") else [])


def test_mix64_golden(oracle):
    for kind in _kinds(oracle):
        L = oracle.lib(kind)
        for v in KA["mix64"]:
            assert L["mix64"](v["id"], v["seed"]) == int(v["out"], 16), (kind, v)


def test_home_and_shard_golden(oracle):
    for kind in _kinds(oracle):
        L = oracle.lib(kind)
        for v in KA["home_slot"]:
            assert L["home_slot"](v["id"], v["capacity"], v["seed"]) == v["out"]
        for v in KA["shard_of"]:
            assert L["shard_of"](v["id"], v["num_shards"], v["seed"]) == v["out"]


def test_distinct_stream_golden(oracle):
    for kind in _kinds(oracle):
        L = oracle.lib(kind)
        for v in KA["distinct_id_stream"]:
            assert L["distinct_id_at"](v["seed"], v["index"]) == int(v["out"], 16)


def test_make_metadata_golden(oracle):
    # make_metadata is observable through the metadata word a fresh insert writes
    for v in KA["make_metadata"]:
        mode = {"disabled": 0, "ttl": 1, "lru": 2}[v["mode"]]
        t = oracle.OracleTable([16], 4, 3, kind="port")
        pf = {int(k): x for k, x in v.get("per_feature", {}).items()}
        s, o = t.lookup_or_insert(77, v["feature"], v["now"], mode, v.get("default_ttl", 0), pf)
        assert o == 1
        assert t.metadata_all()[s] == v["out"], v


def test_even_layout_golden():
    from paper_2602_17050_b200 import even_capacities
    for v in KA["table_layout_even"]:
        assert even_capacities(v["total_rows"], v["num_shards"]) == v["capacities"]


def test_draw_row_is_bounded_and_seeded(oracle):
    a = oracle.draw_row(16, 5, 2024)
    b = oracle.draw_row(16, 5, 2024)
    assert (a == b).all() and (np.abs(a) <= 0.25).all() and (a < 0).any() and (a > 0).any()
    assert not (oracle.draw_row(16, 5, 2025) == a).all()


def _fixture():
    with np.load(os.path.join(HERE, "golden", "ref_streams.npz")) as f:
        z = {k: f[k] for k in f.files}  # decompress once (NpzFile re-reads per access)
    man = json.load(open(os.path.join(HERE, "golden", "ref_streams.json")))
    return z, man


def replay_fixture(make_table, run_batch, state_of, z, man, case_filter=None):
    """Replay every fixture case through (make_table, run_batch) and compare with the
    reference's recorded outputs.  Returns the number of batches checked."""
    bt = z["batches"].astype(np.int64)
    checked = 0
    by_case = {}
    for row in bt:
        by_case.setdefault(int(row[0]), []).append(row)
    soff = {k: 0 for k in ("ident", "meta", "weights", "momentum", "trained")}
    for ci, c in enumerate(man["cases"]):
        rows = by_case[ci]
        total = sum(c["caps"])
        sizes = dict(ident=total, meta=total, weights=total * c["dim"], momentum=total * c["dim"],
                     trained=total if c["dim"] else 0)
        want_state = {}
        for k, sz in sizes.items():
            want_state[k] = z["state_" + k][soff[k]:soff[k] + sz]
            soff[k] += sz
        if case_filter and not case_filter(c):
            continue
        t = make_table(c)
        pf = {int(k): int(v) for k, v in c["per_feature"].items()}
        for row in rows:
            _, p0, p1, e0, e1, now, dttl, has_f = [int(x) for x in row]
            ids = z["ids"][p0:p1]
            f = z["feats"][p0:p1] if has_f else None
            s, o, e = run_batch(t, c, ids, f, now, dttl, pf)
            assert (s == z["slots"][p0:p1]).all(), (c["name"], "slots", p0)
            assert (o == z["oc"][p0:p1]).all(), (c["name"], "outcomes", p0)
            assert (e == z["ev"][e0:e1]).all(), (c["name"], "evicted", p0)
            checked += 1
        got = state_of(t, c)
        for k, v in got.items():
            assert (v.reshape(-1) == want_state[k]).all(), (c["name"], k)
    return checked


def test_port_replays_reference_fixtures(oracle):
    z, man = _fixture()

    def make(c):
        return oracle.OracleTable(c["caps"], c["max_probe"], int(c["seed"]), c["dim"],
                                  int(c["init_seed"]), kind="port")

    def run(t, c, ids, f, now, dttl, pf):
        return t.process_batch(ids, now, c["mode"], dttl, pf, f)

    def state(t, c):
        d = dict(ident=t.identities_all(), meta=t.metadata_all())
        if c["dim"]:
            d.update(weights=t.weights(), momentum=t.momentum(), trained=t.trained())
        return d

    assert replay_fixture(make, run, state, z, man) == len(z["batches"])


def test_port_vs_reference_live(oracle):
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    rng = np.random.default_rng(7)
    for trial in range(40):
        caps = list(rng.integers(8, 90, size=int(rng.integers(1, 5))))
        P = int(rng.integers(1, min(caps) + 1))
        mode = trial % 3
        seed = int(rng.integers(0, 2**63))
        a = oracle.OracleTable(caps, P, seed, 2, 9, kind="port")
        b = oracle.OracleTable(caps, P, seed, 2, 9, kind="reference")
        now = 1
        for _ in range(15):
            now += int(rng.integers(0, 4))
            ids = rng.integers(0, sum(caps) * 2, size=int(rng.integers(1, 120))).astype(np.uint64)
            f = rng.integers(0, 3, size=ids.size).astype(np.uint32)
            ra = a.process_batch(ids, now, mode, 7, {2: 3}, f)
            rb = b.process_batch(ids, now, mode, 7, {2: 3}, f)
            for x, y in zip(ra, rb):
                assert (x == y).all()
        assert (a.identities_all() == b.identities_all()).all()
        assert (a.metadata_all() == b.metadata_all()).all()
        assert (a.weights() == b.weights()).all()


def test_port_error_order(oracle):
    t = oracle.OracleTable([8, 8], 2, 4, kind="port")
    with pytest.raises(oracle.OracleError) as e:
        t.process_batch(np.array([1, 1 << 63], dtype=np.uint64), 5, 0)
    assert e.value.code == 1 and "position 1" in e.value.msg
    with pytest.raises(oracle.OracleError) as e:
        t.process_batch(np.array([1], dtype=np.uint64), (1 << 64) - 6, 1, 1000)
    assert e.value.code == 2
    assert (t.identities_all() == np.uint64((1 << 64) - 1)).all()


# ------------------------------------------------------------------ sgd_step

def test_sgd_known_answers(oracle):
    """proj/tests/test_embedding.cpp:55-99 and :122-134 on MpzchTable (same row draws)."""
    for kind in _kinds(oracle):
        t = oracle.OracleTable([4], 1, 0, dim=2, init_seed=1, kind=kind)
        w0 = t.weights()[2].copy()
        t.sgd_step(np.array([2], np.uint64), np.array([[1.0, -2.0]], np.float32), 0.5, 0.5)
        assert t.momentum()[2].tolist() == [1.0, -2.0]
        assert np.allclose(t.weights()[2], w0 - np.array([0.5, -1.0], np.float32))
        assert t.trained().tolist() == [0, 0, 1, 0]
        t.sgd_step(np.array([2], np.uint64), np.array([[2.0, 2.0]], np.float32), 0.5, 0.5)
        assert t.momentum()[2].tolist() == [2.5, 1.0]
        assert np.allclose(t.weights()[2], w0 - np.array([0.5 + 1.25, -1.0 + 0.5], np.float32))
        good = np.zeros((1, 2), np.float32)
        one = np.array([0], np.uint64)
        for args, code in [((one, np.zeros((1, 3), np.float32), 0.1, 0.0), 1),
                           ((one, good, 0.0, 0.0), 1), ((one, good, -1.0, 0.0), 1),
                           ((one, good, float("nan"), 0.0), 1),
                           ((one, good, 0.1, 1.0), 1), ((one, good, 0.1, -0.1), 1),
                           ((np.array([4], np.uint64), good, 0.1, 0.0), 5)]:
            with pytest.raises(oracle.OracleError) as e:
                t.sgd_step(*args)
            assert e.value.code == code
        nodim = oracle.OracleTable([4], 1, 0, kind=kind)
        with pytest.raises(oracle.OracleError) as e:
            nodim.sgd_step(one, np.zeros((1, 0), np.float32), 0.1, 0.0)
        assert e.value.code == 4


def test_sgd_port_vs_reference_live(oracle):
    """Training steps interleaved with TTL batches (resets), repeated rows, and steps that fail
    part-way: port and reference agree bit for bit, dirty sets included."""
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    rng = np.random.default_rng(11)
    for trial in range(12):
        caps = list(rng.integers(8, 60, size=int(rng.integers(1, 4))))
        dim = int(rng.choice([1, 3, 4, 8]))
        seed = int(rng.integers(0, 2**63))
        T = [oracle.OracleTable(caps, 4, seed, dim, 5, kind=k) for k in ("port", "reference")]
        total = sum(caps)
        now = 1
        for step in range(10):
            now += 3
            ids = rng.integers(0, total * 2, size=int(rng.integers(1, 50))).astype(np.uint64)
            res = [t.process_batch(ids, now, 1, 4) for t in T]
            assert all((x == y).all() for x, y in zip(res[0], res[1]))
            rows = res[0][0].copy()
            if step % 4 == 3:
                rows[rng.integers(0, rows.size)] = total + 1  # fails part-way
            g = (rng.random((rows.size, dim)) - 0.5).astype(np.float32)
            lr, beta = float(rng.choice([0.01, 0.5])), float(rng.choice([0.0, 0.9]))
            cur = [t.make_cursor() for t in T]
            errs = []
            for t in T:
                try:
                    t.sgd_step(rows, g, lr, beta)
                    errs.append(0)
                except oracle.OracleError as e:
                    errs.append(e.code)
            assert errs[0] == errs[1]
            a, b = T
            assert (a.weights().view(np.uint32) == b.weights().view(np.uint32)).all()
            assert (a.momentum().view(np.uint32) == b.momentum().view(np.uint32)).all()
            assert (a.trained() == b.trained()).all()
            assert (a.dirty_rows_since(cur[0]) == b.dirty_rows_since(cur[1])).all()


# ------------------------------------------------------------------ publish

def test_crc32_known_answers(oracle):
    """proj/tests/test_publish.cpp:49-56; zlib's CRC-32 is the same code."""
    import zlib
    for kind in _kinds(oracle):
        assert oracle.crc32(b"123456789", kind) == 0xCBF43926
        assert oracle.crc32(b"", kind) == 0
        assert oracle.crc32(b"hello world", kind) != oracle.crc32(b"helmo world", kind)
    rng = np.random.default_rng(3)
    for n in (1, 7, 4096, 100003):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert oracle.crc32(b) == zlib.crc32(b)


def _busy(oracle, kind, seed, caps=(6, 5, 5), P=3, dim=4):
    """make_busy_table, proj/tests/test_publish.cpp:26-45."""
    t = oracle.OracleTable(list(caps), P, seed, dim, seed + 1, kind=kind)
    ids = oracle.distinct_ids(seed, 0, 64)
    touched = []
    for i, x in enumerate(ids):
        s, o = t.lookup_or_insert(int(x), 0, i + 2, mode=2)
        if o != 3:
            touched.append(s)
    t.sgd_step(np.array(touched, np.uint64), np.full((len(touched), dim), 0.125, np.float32),
               0.05, 0.9)
    return t


def test_snapshot_and_delta_port_vs_reference(oracle):
    import struct
    import zlib
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    for seed in (500, 77, 9):
        a, b = (_busy(oracle, k, seed) for k in ("port", "reference"))
        sa, sb = a.serialize_snapshot(), b.serialize_snapshot()
        assert sa == sb
        assert len(sa) == 48 + 8 * 3 + 8 * 16 + 4 * 4 * 16  # test_publish.cpp:58-66
        assert struct.unpack("<I", sa[-4:])[0] == zlib.crc32(sa[:-4])
        base = struct.unpack("<I", sa[-4:])[0]
        ca, cb = a.delta_source(base), b.delta_source(base)
        rng = np.random.default_rng(seed)
        for step in range(6):
            da, db = ca(), cb()
            assert da == db, step
            assert da[:4] == b"MPZD" and struct.unpack("<Q", da[12:20])[0] == step
            ids = rng.integers(0, 1 << 40, 12).astype(np.uint64)
            for t in (a, b):
                s, o, e = t.process_batch(ids, 100 + step, 1, 1)  # TTL 1: evictions
                if step % 2:
                    t.sgd_step(s[:3], np.ones((3, 4), np.float32), 0.1, 0.0)
    for kind in _kinds(oracle):
        nodim = oracle.OracleTable([4, 4], 2, 1, kind=kind)
        with pytest.raises(oracle.OracleError) as e:
            nodim.serialize_snapshot()
        assert e.value.code == 4
