"""GPU parity for LRU batches whose claim-vs-rounds decision is taken on the device.

An asynchronous call (mpzch_process_batch_device_async) never waits on the host: the LRU claim
attempt is followed on the stream by the rounds path, which runs only if the attempt aborted.
Both outcomes must equal the reference's sequential LRU (probe_core.cpp:114-129) exactly --
checked against the oracle (pinned to the reference in tests/test_oracle.py) for streams where
the attempt succeeds (windows with room), where it aborts (full windows, cascades), and mixed,
with every ticket waited only after the whole stream was enqueued."""
import numpy as np
import pytest
import torch

import paper_2602_17050_b200 as mz

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pool_factor", [0.5, 1.0, 1.6])
def test_lru_async_stream_matches_oracle(oracle, pool_factor):
    rows = 1 << 14
    caps = mz.even_capacities(rows, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 32, 7))
    o = oracle.OracleTable(caps, 32, 7)
    uni = oracle.distinct_ids(17, 0, int(rows * pool_factor))
    rng = np.random.default_rng(int(pool_factor * 10))
    pol = mz.EvictionPolicy.lru()
    st = torch.cuda.current_stream()
    nb, B = 12, 4096
    batches = [uni[rng.integers(0, uni.size, B)] for _ in range(nb)]
    dev = [torch.from_numpy(b.view(np.int64).copy()).cuda() for b in batches]
    outs = [(torch.empty(B, dtype=torch.int64, device="cuda"), torch.empty(B, dtype=torch.uint8, device="cuda"),
             torch.empty(B, dtype=torch.int64, device="cuda")) for _ in range(nb)]
    torch.cuda.synchronize()
    tks = [t.process_batch_device_async(dev[b], 5 + b, pol, None, outs[b][0], outs[b][1], outs[b][2], st)
           for b in range(nb)]
    paths = []
    for b in range(nb):
        nev = t.wait(tks[b])
        paths.append(t.last_stats()["path"])
        os_, oo, oe = o.process_batch(batches[b], 5 + b, 2, 0)
        assert (outs[b][0].cpu().numpy().view(np.uint64) == os_).all(), f"batch {b} slots"
        assert (outs[b][1].cpu().numpy() == oo).all(), f"batch {b} outcomes"
        assert nev == oe.size and (outs[b][2][:nev].cpu().numpy().view(np.uint64) == oe).all(), f"batch {b} evicted"
    assert (t.identities_all() == o.identities_all()).all()
    assert (t.metadata_all() == o.metadata_all()).all()
    if pool_factor < 0.8:
        assert set(paths) == {"fast"}
    if pool_factor > 1.2:
        assert "rounds" in paths
