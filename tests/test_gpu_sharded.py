"""GPU: the row-sharded mode end to end on real sharded handles (held shard ranges,
route kernel, marked remap), with G logical ranks as threads on one B200 (the run has
one GPU; the NCCL transport is the same protocol, tested over gloo on CPU).  Results
must equal the single-table path and the oracle for every G."""
import threading

import numpy as np
import pytest
import torch

import paper_2602_17050_b200 as mz
from paper_2602_17050_b200.sharded import ShardedMpzchTable, ThreadComm, held_shards

pytestmark = pytest.mark.gpu


def run_sharded(cfg, world, batches, pol, transport="collective"):
    comms = ThreadComm.group(world)
    out = [None] * world
    tables = [None] * world
    errs = []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = ShardedMpzchTable(cfg, comms[r], device=0, transport=transport)
            tables[r] = st
            res = []
            for ids, f, now in batches:
                sl = np.array_split(np.arange(ids.size), world)[r]
                ti = torch.from_numpy(ids[sl].view(np.int64).copy()).cuda()
                tf = None if f is None else torch.from_numpy(f[sl].astype(np.int32)).cuda()
                s, o, e = st.process_batch(ti, now, pol, tf)
                torch.cuda.synchronize()
                res.append((s.cpu().numpy().view(np.uint64), o.cpu().numpy(),
                            e.cpu().numpy().view(np.uint64)))
            out[r] = res
        except Exception as ex:  # surface worker failures, release the other ranks
            errs.append(repr(ex))
            comms[r].abort()
            raise

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out, tables


@pytest.mark.parametrize("transport", ["collective", "peer"])
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_sharded_equals_single_table(oracle, world, mode, transport):
    rows = 1 << 16
    caps = mz.even_capacities(rows, 8)
    cfg = mz.TableConfig(caps, 32, 7, 8 if mode == 1 else 0, 3)
    pol = (mz.EvictionPolicy.ttl(mz.TtlPolicy(50)) if mode == 1 else
           mz.EvictionPolicy.lru() if mode == 2 else mz.EvictionPolicy.disabled())
    uni = oracle.distinct_ids(9, 0, rows)
    rng = np.random.default_rng(world + 10 * mode)
    batches = [(uni[rng.integers(0, uni.size, 20000)],
                rng.integers(0, 3, 20000).astype(np.uint32) if b % 3 == 2 else None, 1 + 40 * b)
               for b in range(8)]
    out, tables = run_sharded(cfg, world, batches, pol, transport)
    single = mz.MpzchTable(cfg)
    o = oracle.OracleTable(caps, 32, 7, cfg.dim, 3)
    for b, (ids, f, now) in enumerate(batches):
        s, oc, e = single.process_batch(ids, now, pol, f)
        os_, oo, oe = o.process_batch(ids, now, mode, 50 if mode == 1 else 0, {}, f)
        assert (s == os_).all() and (oc == oo).all() and (e == oe).all()
        gs = np.concatenate([out[r][b][0] for r in range(world)])
        go = np.concatenate([out[r][b][1] for r in range(world)])
        assert (gs == s).all() and (go == oc).all(), f"batch {b}"
        for r in range(world):
            assert (out[r][b][2] == e).all()
    # the union of held rows equals the single table, word for word
    ident = single.identities_all()
    for r in range(world):
        t = tables[r].engine.table
        assert (t.identities_all() == ident[t.row_lo:t.row_hi]).all()
        if cfg.dim:
            assert (t.weights().view(np.uint32) ==
                    single.weights(t.row_lo, t.row_hi - t.row_lo).view(np.uint32)).all()


def test_foreign_id_is_rejected():
    caps = mz.even_capacities(1 << 12, 4)
    t = mz.MpzchTable(mz.TableConfig(caps, 8, 7), shard_range=held_shards(0, 4, 2))
    ids = np.arange(1, 200, dtype=np.uint64)
    with pytest.raises(mz.OutOfRange, match="routes to a shard this handle does not hold"):
        t.process_batch(ids, 1, mz.EvictionPolicy.disabled())
    assert (t.identities_all() == np.uint64((1 << 64) - 1)).all()


@pytest.mark.parametrize("transport", ["collective", "peer"])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_uneven_shards(oracle, world, transport):
    """Shard capacities that are not multiples of the 16-row line: every rank's held range
    starts and ends inside a line (line-aligned allocation base, masked line walks), with
    small batches (quad line walk) and one >256K-position batch (sector walk)."""
    caps = [1003, 2050, 777, 4093, 1500, 3001, 999, 2577]
    cfg = mz.TableConfig(caps, 24, 7, 4, 5)
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(30))
    uni = oracle.distinct_ids(17, 0, sum(caps))
    rng = np.random.default_rng(world)
    batches = [(uni[rng.integers(0, uni.size, 5000 if b < 5 else 300_000)], None, 1 + 20 * b)
               for b in range(6)]
    out, tables = run_sharded(cfg, world, batches, pol, transport)
    o = oracle.OracleTable(caps, 24, 7, 4, 5)
    for b, (ids, f, now) in enumerate(batches):
        os_, oo, oe = o.process_batch(ids, now, 1, 30, {}, f)
        gs = np.concatenate([out[r][b][0] for r in range(world)])
        go = np.concatenate([out[r][b][1] for r in range(world)])
        assert (gs == os_).all() and (go == oo).all(), f"batch {b}"
        for r in range(world):
            assert (out[r][b][2] == oe).all()
    ident = o.identities_all()
    for r in range(world):
        t = tables[r].engine.table
        assert (t.identities_all() == ident[t.row_lo:t.row_hi]).all()


@pytest.mark.parametrize("seed", range(8))
def test_sharded_random_configurations(oracle, seed):
    """Randomised row-sharded runs: S logical shards (uneven capacities) over G ranks, all
    policies, features on some batches; every rank's slice and the evicted list against the
    oracle, and each rank's held rows against the oracle state."""
    rng = np.random.default_rng(500 + seed)
    S = int(rng.choice([2, 4, 8]))
    world = int(rng.choice([w for w in (2, 4, 8) if w <= S]))
    caps = [int(c) for c in rng.integers(300, 5000, S)]
    P = int(min(min(caps), rng.choice([4, 16, 64])))
    mode = int(rng.integers(0, 3))
    dim = 4 if mode == 1 else 0
    cfg = mz.TableConfig(caps, P, 11, dim, 3)
    pol = (mz.EvictionPolicy.ttl(mz.TtlPolicy(35)) if mode == 1 else
           mz.EvictionPolicy.lru() if mode == 2 else mz.EvictionPolicy.disabled())
    uni = oracle.distinct_ids(60 + seed, 0, int(sum(caps) * 1.1))
    batches = []
    for b in range(5):
        n = int(rng.choice([3000, 20000]))
        f = rng.integers(0, 3, n).astype(np.uint32) if b % 2 else None
        batches.append((uni[rng.integers(0, uni.size, n)], f, 1 + 15 * b))
    out, tables = run_sharded(cfg, world, batches, pol, "peer" if seed % 2 else "collective")
    o = oracle.OracleTable(caps, P, 11, dim, 3)
    for b, (ids, f, now) in enumerate(batches):
        os_, oo, oe = o.process_batch(ids, now, mode, 35 if mode == 1 else 0, {}, f)
        gs = np.concatenate([out[r][b][0] for r in range(world)])
        go = np.concatenate([out[r][b][1] for r in range(world)])
        assert (gs == os_).all() and (go == oo).all(), f"batch {b} S={S} G={world} mode={mode}"
        for r in range(world):
            assert (out[r][b][2] == oe).all()
    ident = o.identities_all()
    for r in range(world):
        t = tables[r].engine.table
        assert (t.identities_all() == ident[t.row_lo:t.row_hi]).all()


def test_peer_transport_two_processes(oracle, tmp_path):
    """The peer transport across PROCESSES: two ranks (torchrun, gloo for the host barrier and
    the address exchange) share the one B200 and map each other's receive / result buffers
    with CUDA IPC (mpzch_ipc_export / mpzch_ipc_import) -- the same code path as one process
    per GPU on an NVLink box.  Every rank's slice and the evicted list against the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533",
           os.path.join(root, "tests", "peer_ipc_worker.py"), str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    import peer_ipc_worker as w
    caps, P, batches = w.workload(oracle)
    o = oracle.OracleTable(caps, P, 7, 4, 3)
    for b, (ids, f, now) in enumerate(batches):
        os_, oo, oe = o.process_batch(ids, now, 1, 40, {}, f)
        got = [np.load(tmp_path / f"r{r}_b{b}.npz") for r in range(2)]
        gs = np.concatenate([g["s"] for g in got])
        go = np.concatenate([g["o"] for g in got])
        assert (gs == os_).all() and (go == oo).all(), f"batch {b}"
        for g in got:
            assert (g["e"] == oe).all()


@pytest.mark.parametrize("transport", ["collective", "peer"])
def test_sharded_invalid_id_raises_everywhere(transport):
    """An invalid id in one rank's slice: every rank raises the reference's message with the
    GLOBAL position (batch_engine.cpp:90-94) and no rank's table changes."""
    world = 2
    caps = mz.even_capacities(1 << 12, 4)
    cfg = mz.TableConfig(caps, 16, 7)
    comms = ThreadComm.group(world)
    msgs = [None] * world
    tables = [None] * world

    def worker(r):
        torch.cuda.set_device(0)
        st = ShardedMpzchTable(cfg, comms[r], device=0, transport=transport)
        tables[r] = st
        ids = np.arange(1 + 1000 * r, 301 + 1000 * r, dtype=np.uint64)
        if r == 1:
            ids[17] = np.uint64((1 << 64) - 1)  # the EMPTY sentinel
        try:
            st.process_batch(torch.from_numpy(ids.view(np.int64)).cuda(), 5, mz.EvictionPolicy.disabled())
        except mz.InvalidArgument as e:
            msgs[r] = str(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert msgs == ["invalid id at batch position 317"] * world, msgs
    for r in range(world):
        assert (tables[r].engine.table.identities_all() == np.uint64((1 << 64) - 1)).all()
