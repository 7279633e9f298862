"""GPU parity for publishing: .mpzc snapshots and .mpzd delta logs built
from HBM with the CRC-32 on the device, byte-identical to the oracle (pinned to the reference's
serialize_snapshot / DeltaSource::cut + serialize_delta in tests/test_oracle.py)."""
import struct
import zlib

import numpy as np
import pytest

import paper_2602_17050_b200 as mz

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 4096, 16383, 16384, 16385, 3 * 16384 + 777,
                               (1 << 20) + 3, 10_000_019])
def test_crc32_device_matches_zlib(n):
    import torch
    g = torch.Generator(device="cuda").manual_seed(n)
    buf = torch.randint(0, 256, (n + 32,), dtype=torch.uint8, device="cuda", generator=g)
    host = buf.cpu().numpy().tobytes()
    for off in (0, 1, 7, 16, 19):
        view = buf[off:off + n]
        assert mz.crc32_device(view) == zlib.crc32(host[off:off + n]), (n, off)


def test_crc32_device_large():
    """1 GiB of HBM: the device CRC equals zlib's over the same bytes (full-size property)."""
    import torch
    n = (1 << 30) + 12345
    g = torch.Generator(device="cuda").manual_seed(3)
    buf = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g)
    assert mz.crc32_device(buf) == zlib.crc32(buf.cpu().numpy().tobytes())


def busy_pair(oracle, seed, caps=(6, 5, 5), P=3, dim=4):
    """make_busy_table (proj/tests/test_publish.cpp:26-45) on both sides."""
    t = mz.MpzchTable(mz.TableConfig(list(caps), P, seed, dim, seed + 1))
    o = oracle.OracleTable(list(caps), P, seed, dim, seed + 1)
    lru = mz.EvictionPolicy.lru()
    touched = []
    for i, x in enumerate(oracle.distinct_ids(seed, 0, 64)):
        s, oc = t.lookup_or_insert(int(x), 0, i + 2, lru)
        s2, oc2 = o.lookup_or_insert(int(x), 0, i + 2, mode=2)
        assert (s, oc) == (s2, oc2)
        if oc != 3:
            touched.append(s)
    g = np.full((len(touched), dim), 0.125, np.float32)
    t.sgd_step(np.array(touched, np.uint64), g, 0.05, 0.9)
    o.sgd_step(np.array(touched, np.uint64), g, 0.05, 0.9)
    return t, o


@pytest.mark.parametrize("seed", [500, 77, 9])
def test_snapshot_bytes_match_oracle(oracle, seed):
    t, o = busy_pair(oracle, seed)
    a, b = t.serialize_snapshot(), o.serialize_snapshot()
    assert a == b
    assert len(a) == 48 + 8 * 3 + 8 * 16 + 4 * 4 * 16
    assert mz.snapshot_checksum(a) == zlib.crc32(a[:-4])


def test_snapshot_large_table(oracle):
    """2^20 rows x dim 32 after a batch stream: image == oracle's (128 MiB, CRC on the GPU)."""
    rng = np.random.default_rng(1)
    caps = mz.even_capacities(1 << 20, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 16, 5, 32, 6))
    o = oracle.OracleTable(caps, 16, 5, 32, 6)
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(50))
    for b in range(6):
        ids = rng.integers(0, 1 << 40, 200_000).astype(np.uint64)
        s1, _, _ = t.process_batch(ids, 10 + 20 * b, pol)
        o.process_batch(ids, 10 + 20 * b, 1, 50)
        rows = np.unique(s1)[:50_000]
        g = (rng.random((rows.size, 32)) - 0.5).astype(np.float32)
        t.sgd_step(rows, g, 0.01, 0.9)
        o.sgd_step(rows, g, 0.01, 0.9)
    assert t.serialize_snapshot() == o.serialize_snapshot()


def test_delta_source_matches_oracle(oracle):
    t, o = busy_pair(oracle, 500)
    base = mz.snapshot_checksum(t.serialize_snapshot())
    src, osrc = mz.DeltaSource(t, base), o.delta_source(base)
    rng = np.random.default_rng(2)
    ttl = mz.EvictionPolicy.ttl(mz.TtlPolicy(1))
    for step in range(8):
        a, b = src.cut(), osrc()
        assert a == b, step
        d = mz.parse_delta(a)
        assert d["sequence"] == step and d["base_checksum"] == base and d["dim"] == 4
        if d["rows"].size:
            rows = d["rows"].astype(np.int64)
            assert (d["identities"] == t.identities_all()[rows]).all()
            assert (d["weights"].view(np.uint32) == t.weights()[rows].view(np.uint32)).all()
        ids = rng.integers(0, 1 << 40, 10).astype(np.uint64)
        s1, _, _ = t.process_batch(ids, 200 + step, ttl)
        o.process_batch(ids, 200 + step, 1, 1)
        if step % 2:
            t.sgd_step(s1[:3], np.ones((3, 4), np.float32), 0.1, 0.0)
            o.sgd_step(s1[:3], np.ones((3, 4), np.float32), 0.1, 0.0)


def test_publish_errors():
    nodim = mz.MpzchTable(mz.TableConfig([8, 8], 2, 1))
    with pytest.raises(mz.LogicError):
        nodim.serialize_snapshot()
    with pytest.raises(mz.LogicError):
        mz.DeltaSource(nodim, 0)
    sharded = mz.MpzchTable(mz.TableConfig([8, 8], 2, 1, 4, 1), shard_range=(1, 2))
    with pytest.raises(mz.InvalidArgument):
        sharded.serialize_snapshot()
    t = mz.MpzchTable(mz.TableConfig([8, 8], 2, 1, 4, 1))
    src = mz.DeltaSource(t, 7)
    src.cursor = 999
    with pytest.raises(mz.InvalidArgument):
        src.cut()
    empty = mz.DeltaSource(t, 7).cut()
    assert len(empty) == 36 and struct.unpack_from("<Q", empty, 24)[0] == 0
