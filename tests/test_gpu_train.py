"""GPU parity for sgd_step: the sm_100a kernels through the C-ABI against the
oracle (itself pinned to the reference in tests/test_oracle.py::test_sgd_*), bit for bit:
weights/momentum fp32 patterns, trained flags, dirty rows, error codes and the partial update
a failing step leaves behind."""
import numpy as np
import pytest

import paper_2602_17050_b200 as mz

pytestmark = pytest.mark.gpu


def same_rows(t, o):
    assert (t.weights().view(np.uint32) == o.weights().view(np.uint32)).all(), "weights differ"
    assert (t.momentum().view(np.uint32) == o.momentum().view(np.uint32)).all(), "momentum differs"
    assert (t.trained() == o.trained()).all(), "trained differs"


def pair(oracle, caps, dim, seed=3, init_seed=9, P=8):
    t = mz.MpzchTable(mz.TableConfig(list(caps), P, seed, dim, init_seed))
    o = oracle.OracleTable(caps, P, seed, dim, init_seed)
    return t, o


@pytest.mark.parametrize("dim", [1, 3, 4, 8, 128])
def test_sgd_random_steps_with_repeats(oracle, dim):
    rng = np.random.default_rng(dim)
    caps = [300, 200, 500]
    t, o = pair(oracle, caps, dim)
    total = sum(caps)
    for step in range(8):
        n = int(rng.integers(1, 900))
        # a small hot set makes rows repeat (the per-row ordered path)
        rows = np.where(rng.random(n) < 0.3, rng.integers(0, 8, n), rng.integers(0, total, n))
        rows = rows.astype(np.uint64)
        g = (rng.random((n, dim)) - 0.5).astype(np.float32)
        lr, beta = float(rng.choice([0.01, 0.3])), float(rng.choice([0.0, 0.5, 0.9]))
        ct, co = t.make_cursor(), o.make_cursor()
        t.sgd_step(rows, g, lr, beta)
        o.sgd_step(rows, g, lr, beta)
        same_rows(t, o)
        assert (t.dirty_rows_since(ct) == o.dirty_rows_since(co)).all()


def test_sgd_errors_and_partial_update(oracle):
    t, o = pair(oracle, [64, 64], 4)
    one = np.array([3], np.uint64)
    good = np.ones((1, 4), np.float32)
    for args, exc in [((one, np.ones((1, 3), np.float32), 0.1, 0.0), mz.InvalidArgument),
                      ((one, good, 0.0, 0.0), mz.InvalidArgument),
                      ((one, good, float("nan"), 0.0), mz.InvalidArgument),
                      ((one, good, 0.1, 1.0), mz.InvalidArgument),
                      ((one, good, 0.1, -0.5), mz.InvalidArgument)]:
        with pytest.raises(exc):
            t.sgd_step(*args)
    same_rows(t, o)
    # out of range at position 3 of 6: positions 0-2 update (row 5 twice), nothing is stamped
    rows = np.array([5, 9, 5, 128, 9, 7], np.uint64)
    g = np.arange(24, dtype=np.float32).reshape(6, 4) / 7
    ct, co = t.make_cursor(), o.make_cursor()
    with pytest.raises(mz.OutOfRange, match="embedding row out of range"):
        t.sgd_step(rows, g, 0.2, 0.9)
    with pytest.raises(oracle.OracleError):
        o.sgd_step(rows, g, 0.2, 0.9)
    same_rows(t, o)
    assert t.dirty_rows_since(ct).size == 0 and o.dirty_rows_since(co).size == 0
    nodim = mz.MpzchTable(mz.TableConfig([16], 2, 1))
    with pytest.raises(mz.LogicError):
        nodim.sgd_step(one, np.zeros((1, 0), np.float32), 0.1, 0.0)


def test_sgd_device_tensors_and_unaligned_grads(oracle):
    import torch
    rng = np.random.default_rng(5)
    t, o = pair(oracle, [1000, 1000], 8)
    rows = rng.integers(0, 2000, 600).astype(np.uint64)
    g = (rng.random((600, 8)) - 0.5).astype(np.float32)
    t.sgd_step_device(torch.from_numpy(rows.view(np.int64)).cuda(), torch.from_numpy(g).cuda(),
                      0.1, 0.9)
    o.sgd_step(rows, g, 0.1, 0.9)
    torch.cuda.synchronize()
    same_rows(t, o)
    # grads starting 4 bytes into an allocation: not 16-byte aligned -> scalar lanes
    buf = torch.zeros(600 * 8 + 1, dtype=torch.float32, device="cuda")
    buf[1:] = torch.from_numpy(g).reshape(-1).cuda()
    t.sgd_step_device(torch.from_numpy(rows.view(np.int64)).cuda(), buf[1:].view(600, 8), 0.05, 0.5)
    o.sgd_step(rows, g, 0.05, 0.5)
    torch.cuda.synchronize()
    same_rows(t, o)


def test_sgd_after_ttl_evictions(oracle):
    """The churn loop (proj/src/experiments.cpp:86-125): remap a batch (evictions reset rows),
    train the remapped rows, repeat."""
    rng = np.random.default_rng(9)
    caps = [256, 256]
    t, o = pair(oracle, caps, 16, P=16)
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(5))
    now = 1
    for step in range(30):
        now += 2
        ids = rng.integers(0, 3000, 400).astype(np.uint64)
        s1, o1, e1 = t.process_batch(ids, now, pol)
        s2, o2, e2 = o.process_batch(ids, now, 1, 5)
        assert (s1 == s2).all() and (o1 == o2).all() and (e1 == e2).all()
        rows = np.unique(s1)  # the reference's step_rows (first occurrence order is irrelevant)
        g = (rng.random((rows.size, 16)) - 0.5).astype(np.float32)
        t.sgd_step(rows, g, 0.05, 0.9)
        o.sgd_step(rows, g, 0.05, 0.9)
    same_rows(t, o)


def test_sgd_large_unique_rows_numpy():
    """2^20 rows x dim 128, 2^18 distinct rows: the update equals numpy's float32 arithmetic
    (separately rounded mul/add) on those rows; untouched rows are unchanged."""
    import torch
    rows_total, dim, n = 1 << 20, 128, 1 << 18
    t = mz.MpzchTable(mz.TableConfig.even(rows_total, 8, 128, 7, dim, 3))
    rng = np.random.default_rng(1)
    rows = rng.choice(rows_total, n, replace=False).astype(np.uint64)
    g = (rng.random((n, dim), dtype=np.float32) - np.float32(0.5))
    w0 = t.weights()
    dr = torch.from_numpy(rows.view(np.int64)).cuda()
    dg = torch.from_numpy(g).cuda()
    t.sgd_step_device(dr, dg, 0.125, 0.75)
    t.sgd_step_device(dr, dg, 0.125, 0.75)
    torch.cuda.synchronize()
    lr, beta = np.float32(0.125), np.float32(0.75)
    m = np.zeros((n, dim), np.float32)
    w = w0[rows.astype(np.int64)].copy()
    for _ in range(2):
        m = (beta * m) + g
        w = w - (lr * m)
    w1 = t.weights()
    assert (w1[rows.astype(np.int64)].view(np.uint32) == w.view(np.uint32)).all()
    mask = np.ones(rows_total, bool)
    mask[rows.astype(np.int64)] = False
    assert (w1[mask].view(np.uint32) == w0[mask].view(np.uint32)).all()
    assert int(t.trained().sum()) == n
