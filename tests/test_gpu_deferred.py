"""GPU parity for the fused reset + sgd_step (MPZCH_RESET_DEFERRED).

A deferred-mode table marks its evicted rows reset-pending instead of writing them; the next
sgd_step of such a row starts from the closed-form draw_row and momentum 0 (one write of the
row), gathers draw pending rows, and every other reader flushes first.  Every observable value
must equal the reference's eager order (process_batch resets the row, table.cpp:142 ->
embedding_store.cpp:62-68; then sgd_step, embedding_store.cpp:70-93): checked bit for bit
against the oracle (pinned to the reference in tests/test_oracle.py) and against an eager
B200 table fed the same calls."""
import numpy as np
import pytest
import torch

import paper_2602_17050_b200 as mz

pytestmark = pytest.mark.gpu


def same_rows(t, o, rows=None):
    assert (t.weights().view(np.uint32) == o.weights().view(np.uint32)).all(), "weights differ"
    assert (t.momentum().view(np.uint32) == o.momentum().view(np.uint32)).all(), "momentum differs"
    assert (t.trained() == o.trained()).all(), "trained differs"


@pytest.mark.parametrize("dim", [3, 16, 128])
def test_deferred_ttl_stream_with_steps(oracle, dim):
    """TTL churn (most batches evict), a step over every batch's distinct rows plus rows that
    were evicted but are not stepped, and gathers between remap and step."""
    rng = np.random.default_rng(dim)
    caps = mz.even_capacities(1 << 13, 4)
    P, seed, init_seed, ttl = 64, 7, 11, 40
    d = mz.MpzchTable(mz.TableConfig(caps, P, seed, dim, init_seed))
    e = mz.MpzchTable(mz.TableConfig(caps, P, seed, dim, init_seed))
    o = oracle.OracleTable(caps, P, seed, dim, init_seed)
    d.set_reset_mode("deferred")
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(ttl))
    ids = oracle.distinct_ids(3, 0, 20000)
    total_ev = 0
    for b in range(10):
        now = 1 + 30 * b
        batch = ids[rng.integers(0, ids.size, 4096)]
        ds, do, de = d.process_batch(batch, now, pol)
        es, eo, ee = e.process_batch(batch, now, pol)
        os_, oo, oe = o.process_batch(batch, now, 1, ttl)
        assert (ds == os_).all() and (do == oo).all() and (de == oe).all()
        assert (es == os_).all() and (ee == oe).all()
        total_ev += de.size
        # the forward read of the batch's rows sees the reset rows (drawn, nothing flushed)
        rows = np.unique(ds)
        gd = d.gather(rows)
        assert (gd.view(np.uint32) == e.gather(rows).view(np.uint32)).all(), f"batch {b}: gather differs"
        assert (gd.view(np.uint32) == o.weights()[rows.astype(np.int64)].view(np.uint32)).all()
        # step most of the distinct rows (some evicted rows stay pending), with repeats
        keep = rows[rng.random(rows.size) < 0.8]
        step = np.concatenate([keep, keep[: keep.size // 10]]).astype(np.uint64)
        g = (rng.random((step.size, dim)) - 0.5).astype(np.float32)
        for t in (d, e):
            t.sgd_step(step, g, 0.05, 0.9)
        o.sgd_step(step, g, 0.05, 0.9)
        if b % 3 == 2:  # accessors flush; the next batch marks new rows pending again
            same_rows(d, o)
    assert total_ev > 1000
    same_rows(d, o)
    same_rows(e, o)
    assert d.state_equals(e)
    assert d.serialize_snapshot() == e.serialize_snapshot()


def test_deferred_device_path_and_lookup_gather(oracle):
    """process_batch_device -> lookup_gather_device -> sgd_step_device with a pending row
    stepped twice in one call (the ordered repeated-row path) and a row out of range."""
    dim = 8
    caps = mz.even_capacities(1 << 12, 2)
    d = mz.MpzchTable(mz.TableConfig(caps, 32, 5, dim, 3))
    o = oracle.OracleTable(caps, 32, 5, dim, 3)
    d.set_reset_mode("deferred")
    ids = oracle.distinct_ids(9, 0, 8000)
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(5))
    for b, now in enumerate((1, 2, 20, 21, 40)):
        batch = ids[b * 1500:(b + 1) * 1500 + 2000]
        bt = torch.from_numpy(batch.view(np.int64)).cuda()
        out_s = torch.empty(bt.numel(), dtype=torch.int64, device="cuda")
        out_o = torch.empty(bt.numel(), dtype=torch.uint8, device="cuda")
        d.process_batch_device(bt, now, pol, None, out_s, out_o, None)
        os_, oo, oe = o.process_batch(batch, now, 1, 5)
        assert (out_s.cpu().numpy().view(np.uint64) == os_).all()
        slots, oc, rows = d.lookup_gather_device(bt)
        assert (slots.cpu().numpy().view(np.uint64) == os_).all()
        assert (rows.cpu().numpy().view(np.uint32) ==
                o.weights()[os_.astype(np.int64)].view(np.uint32)).all(), f"batch {b}: lookup_gather"
        if oe.size:
            r = int(oe[0])
            step = np.array([r, r, oe[-1], r], dtype=np.uint64)
            g = np.arange(4 * dim, dtype=np.float32).reshape(4, dim) / 13
            d.sgd_step_device(torch.from_numpy(step.view(np.int64)).cuda(), torch.from_numpy(g).cuda(), 0.1, 0.5)
            torch.cuda.synchronize()
            o.sgd_step(step, g, 0.1, 0.5)
    # out of range at position 2: rows before it update from their drawn state
    fresh = oracle.distinct_ids(9, 10000, 900)  # every stored entry has expired by now = 100
    d.process_batch(fresh, 100, pol)
    _, _, oe2 = o.process_batch(fresh, 100, 1, 5)
    assert oe2.size > 2
    step = np.array([oe2[0], oe2[1], 1 << 40, oe2[2]], dtype=np.uint64)
    g = np.ones((4, dim), np.float32)
    with pytest.raises(mz.OutOfRange):
        d.sgd_step(step, g, 0.25, 0.0)
    with pytest.raises(Exception):
        o.sgd_step(step, g, 0.25, 0.0)
    same_rows(d, o)


def test_deferred_flush_on_mode_switch_and_raw_pointer(oracle):
    dim = 4
    caps = [2048]
    d = mz.MpzchTable(mz.TableConfig(caps, 16, 1, dim, 2))
    o = oracle.OracleTable(caps, 16, 1, dim, 2)
    d.set_reset_mode("deferred")
    ids = oracle.distinct_ids(4, 0, 4000)
    for now, lo in ((1, 0), (9, 1600), (30, 3000)):
        batch = ids[lo:lo + 1600]
        g = np.full((16, dim), 0.5, np.float32)
        d.process_batch(batch, now, mz.EvictionPolicy.ttl(mz.TtlPolicy(4)))
        o.process_batch(batch, now, 1, 4)
        rows = np.arange(16, dtype=np.uint64) * 101
        d.sgd_step(rows, g, 0.5, 0.25)
        o.sgd_step(rows, g, 0.5, 0.25)
    # raw weights pointer: flushed before it is handed out (CRC-32 of the device bytes)
    import zlib
    _, _, wptr = d.device_arrays()
    assert mz.crc32_device_ptr(wptr, 2048 * dim * 4) == zlib.crc32(o.weights().tobytes())
    d.set_reset_mode("eager")  # flushes; further batches write rows eagerly
    same_rows(d, o)
    d.process_batch(ids[:900], 50, mz.EvictionPolicy.ttl(mz.TtlPolicy(4)))
    o.process_batch(ids[:900], 50, 1, 4)
    same_rows(d, o)
