"""CPU, world_size 2 and 3 over gloo: the row-sharded protocol (paper_2602_17050_b200/
sharded.py) reproduces the single-table reference result bit for bit -- per-position
slots and outcomes, the global canonical evicted list, the final state of every shard,
and the error agreement (first invalid GLOBAL position, TTL overflow) -- with the oracle
as each rank's engine (the GPU engine is covered by tests/test_gpu_sharded.py)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stream(seed, caps, nbatches, mode):
    import pyoracle
    rng = np.random.default_rng(seed)
    uni = pyoracle.distinct_ids(seed, 0, int(sum(caps) * 1.5))
    out = []
    now = 1
    for b in range(nbatches):
        now += int(rng.integers(1, 4))
        n = int(rng.integers(50, 400))
        ids = uni[rng.integers(0, uni.size, n)]
        f = rng.integers(0, 3, n).astype(np.uint32) if b % 2 else None
        out.append((ids, f, now))
    return out


def _worker(rank, world, port, mode, resq):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_2602_17050_b200 as mz
    from paper_2602_17050_b200.sharded import ShardedMpzchTable, TorchComm
    from sharded_engines import OracleEngine
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = mz.TableConfig([37, 51, 44, 29, 60, 33], 6, 12345, 2, 77)
    pol = (mz.EvictionPolicy.disabled(), mz.EvictionPolicy.ttl(mz.TtlPolicy(9, {1: 4})),
           mz.EvictionPolicy.lru())[mode]
    st = ShardedMpzchTable(cfg, TorchComm(), engine=OracleEngine(cfg))
    results = []
    for ids, f, now in _stream(100 + mode, cfg.shard_capacities, 14, mode):
        sl = np.array_split(np.arange(ids.size), world)[rank]
        t_ids = torch.from_numpy(ids[sl].view(np.int64).copy())
        t_f = None if f is None else torch.from_numpy(f[sl].astype(np.int32))
        s, o, ev = st.process_batch(t_ids, now, pol, t_f)
        results.append((s.numpy().view(np.uint64).copy(), o.numpy().copy(),
                        ev.numpy().view(np.uint64).copy()))
    # errors are agreed globally: the invalid id sits on the LAST rank's slice
    ids, _, now = _stream(7, cfg.shard_capacities, 1, 0)[0]
    ids = ids.copy()
    ids[-2] = np.uint64(1 << 63)
    sl = np.array_split(np.arange(ids.size), world)[rank]
    err = None
    try:
        st.process_batch(torch.from_numpy(ids[sl].view(np.int64).copy()), now + 100, pol)
    except mz.InvalidArgument as e:
        err = str(e)
    over = None
    try:
        st.process_batch(torch.from_numpy(ids[sl][:1].view(np.int64).copy() & 0xFFFF), (1 << 64) - 3,
                         mz.EvictionPolicy.ttl(mz.TtlPolicy(10)))
    except mz.OverflowError_ as e:
        over = str(e)
    state = (st.engine.t.identities_all(), st.engine.t.metadata_all())
    resq.put((rank, results, err, over, ids.size, state))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, 0), (2, 1), (3, 2), (3, 1)])
def test_sharded_protocol_matches_single_table(world, mode):
    import pyoracle
    import paper_2602_17050_b200 as mz
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(world):
        r = q.get(timeout=300)
        got[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
    cfg = mz.TableConfig([37, 51, 44, 29, 60, 33], 6, 12345, 2, 77)
    ref = pyoracle.OracleTable(cfg.shard_capacities, cfg.max_probe, cfg.seed, cfg.dim, cfg.init_seed)
    dt, pf = (0, {}) if mode != 1 else (9, {1: 4})
    for b, (ids, f, now) in enumerate(_stream(100 + mode, cfg.shard_capacities, 14, mode)):
        s, o, e = ref.process_batch(ids, now, mode, dt, pf, f)
        gs = np.concatenate([got[r][0][b][0] for r in range(world)])
        go = np.concatenate([got[r][0][b][1] for r in range(world)])
        assert (gs == s).all() and (go == o).all(), f"batch {b}"
        for r in range(world):
            assert (got[r][0][b][2] == e).all(), f"evicted list batch {b} rank {r}"
    n = got[0][3]
    for r in range(world):
        assert got[r][1] == f"invalid id at batch position {n - 2}"
        assert got[r][2] == "TTL expiry overflows the 64-bit timestamp range"
    # every rank's engine only ever touched its own shards: union == single table
    from paper_2602_17050_b200.sharded import shard_owner
    ident = ref.identities_all()
    meta = ref.metadata_all()
    offs = ref.offsets
    for s_ in range(len(cfg.shard_capacities)):
        r = shard_owner(s_, len(cfg.shard_capacities), world)
        a, b_ = int(offs[s_]), int(offs[s_ + 1])
        assert (got[r][4][0][a:b_] == ident[a:b_]).all()
        assert (got[r][4][1][a:b_] == meta[a:b_]).all()


def test_peer_offsets_lay_sources_out_in_rank_order():
    """peer_offsets: rank r's part-q positions start after every lower rank's part-q positions
    in owner q's receive buffer, and owner r receives column r of the count matrix."""
    from paper_2602_17050_b200.sharded import peer_offsets
    counts = [[3, 0, 5], [1, 4, 2], [0, 7, 6]]  # counts[source][owner]
    assert peer_offsets(counts, 0) == ([0, 0, 0], [3, 1, 0])
    assert peer_offsets(counts, 1) == ([3, 0, 5], [0, 4, 7])
    assert peer_offsets(counts, 2) == ([4, 4, 7], [5, 2, 6])
    for q in range(3):  # the sources tile each owner's buffer exactly
        spans = sorted((peer_offsets(counts, r)[0][q], counts[r][q]) for r in range(3))
        pos = 0
        for off, c in spans:
            assert off == pos
            pos += c
        assert pos == sum(counts[r][q] for r in range(3))
