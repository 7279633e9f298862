"""Parity at BASELINE scale, against the REFERENCE library (oracle/_ref) itself.

* C5 at its stated size: 2^30 rows (S=8, P=128, seed 7) prefilled to 0.8 with
  DistinctIdStream(5), then the bench's 4M-position batches (90% hit / 10% fresh, now = 2 + b).
  Every batch's slots and outcomes, then the final identity and metadata arrays, are compared
  word for word with the reference's process_batch on the same stream.  (A box with less than
  96 GiB of host memory runs the same stream at 2^28 rows.)
* C4 at its stated size: 2^27 rows x dim 128 fp32 (64 + 64 GiB on the device), TTL 3,600 s,
  prefill 0.8 at now = 1, then 1M-position batches of fresh ids (seed 41) at now = 10,000 + 600 t
  -- ~80% of new ids evict an expired entry.  Split so the CPU side stays affordable: the
  remap results (slots, outcomes, evicted list, identity, metadata) do not depend on dim, so
  the reference runs with dim = 0; the rows are checked in closed form.  Before the GPU batches
  run, every row the reference says will be evicted, plus random control rows, is trained one
  sgd_step (grad 1, lr 0.25), so a reset is visible: afterwards every evicted row must equal
  draw_row(row, 11) bit for bit (embedding_store.cpp:12-18, 62-68, table.cpp:142), with
  momentum 0 and trained 0, every control row that was not evicted must still hold its trained
  values, and the trained flags of all 2^27 rows must be exactly (perturbed \\ evicted).
"""
import os

import numpy as np
import pytest
import torch

import bench
import paper_2602_17050_b200 as mz

pytestmark = pytest.mark.gpu


def _ref():
    import pyoracle
    if not pyoracle.available("reference"):
        pytest.fail("oracle/_ref/libmpzch_ref.so missing (built by `make -C oracle` where "
                    "/root/reference exists; it ships to the GPU box)")
    pyoracle.lib("reference")["set_threads"](os.cpu_count() or 1)
    return pyoracle


def _host_gib():
    return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30


def _prefill_gpu(t, seed, npre, now, pol, chunk=1 << 22):
    out_s = torch.empty(chunk, dtype=torch.int64, device="cuda")
    out_o = torch.empty(chunk, dtype=torch.uint8, device="cuda")
    for a in range(0, npre, chunk):
        ids = bench.distinct_ids_t(seed, torch.arange(a, min(a + chunk, npre), dtype=torch.int64,
                                                      device="cuda"))
        t.process_batch_device(ids, now, pol, None, out_s, out_o, None)
    torch.cuda.synchronize()


def test_c5_full_scale_vs_reference():
    po = _ref()
    rows = bench.ROWS if _host_gib() >= 96 else 1 << 28
    caps = mz.even_capacities(rows, bench.SHARDS)
    npre = bench.prefill_count(rows)
    pol = mz.EvictionPolicy.disabled()
    t = mz.MpzchTable(mz.TableConfig(caps, bench.MAX_PROBE, bench.TABLE_SEED))
    _prefill_gpu(t, bench.ID_SEED, npre, 1, pol)
    o = po.OracleTable(caps, bench.MAX_PROBE, bench.TABLE_SEED, kind="reference")
    o.prefill_distinct(bench.ID_SEED, 0, npre, 1)
    fresh = npre
    kinds = np.zeros(4, dtype=np.int64)
    for b in range(4):
        idx, nf = bench.batch_indices(torch, "cpu", npre, bench.BATCH, b, fresh, bench.SAMPLER_SEED)
        fresh += nf
        ids = bench.distinct_ids_t(bench.ID_SEED, idx).numpy().view(np.uint64)
        gs, go, ge = t.process_batch(ids, 2 + b, pol)
        rs, ro, re_ = o.process_batch(ids, 2 + b, 0)
        assert (gs == rs).all() and (go == ro).all(), f"batch {b}: {(gs != rs).sum()} slots differ"
        assert ge.size == re_.size == 0
        kinds += np.bincount(go, minlength=4)
    assert kinds[0] > 0 and kinds[1] > 0  # hits and inserts (and the 0.8-load collisions)
    g = t.identities_all()
    r = o.identities_all()
    assert (g == r).all(), f"{(g != r).sum()} identity words differ"
    del g, r
    g = t.metadata_all()
    r = o.metadata_all()
    assert (g == r).all(), f"{(g != r).sum()} metadata words differ"


def test_c4_full_scale_resets():
    po = _ref()
    rows, S, P, dim, init_seed, ttl = 1 << 27, 8, 128, 128, 11, 3600
    caps = mz.even_capacities(rows, S)
    npre = int(0.8 * rows)
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(ttl))
    B, nb, lr = 1 << 20, 3, 0.25
    g = torch.Generator().manual_seed(41)
    batches = [(bench.distinct_ids_t(41, torch.randint(0, 1 << 27, (B,), generator=g)).numpy().view(np.uint64),
                10000 + 600 * i) for i in range(nb)]

    # 1. the reference (dim 0: the remap does not depend on dim)
    o = po.OracleTable(caps, P, 7, 0, 0, kind="reference")
    o.prefill_distinct(4, 0, npre, 1, mode=1, default_ttl=ttl)
    ref = [o.process_batch(ids, now, 1, ttl) for ids, now in batches]
    evicted = np.unique(np.concatenate([e for _, _, e in ref]))
    assert evicted.size > B // 2  # C4's shape: most new ids evict an expired entry

    # 2. the B200 table at full size, prefilled through the API
    t = mz.MpzchTable(mz.TableConfig(caps, P, 7, dim, init_seed))
    _prefill_gpu(t, 4, npre, 1, pol)

    # 3. make resets visible: one sgd_step (grad 1) on every row about to be evicted + controls
    rng = np.random.default_rng(7)
    controls = np.unique(rng.integers(0, rows, 1 << 16).astype(np.uint64))
    pert = np.union1d(evicted, controls)
    for a in range(0, pert.size, 1 << 20):
        r_ = torch.from_numpy(pert[a:a + (1 << 20)].view(np.int64)).cuda()
        t.sgd_step_device(r_, torch.ones(r_.numel(), dim, device="cuda"), lr, 0.5)
    torch.cuda.synchronize()

    # 4. the same batches on the device: every remap output identical to the reference's
    for b, (ids, now) in enumerate(batches):
        gs, go, ge = t.process_batch(ids, now, pol)
        rs, ro, re_ = ref[b]
        assert (gs == rs).all() and (go == ro).all(), f"batch {b}: {(gs != rs).sum()} slots differ"
        assert ge.size == re_.size and (ge == re_).all(), f"batch {b}: evicted lists differ"
    assert (t.identities_all() == o.identities_all()).all()
    assert (t.metadata_all() == o.metadata_all()).all()

    # 5. rows: evicted -> draw_row / 0 / untrained; controls not evicted -> still trained
    kept = np.setdiff1d(controls, evicted)
    trained = t.trained()
    want = np.zeros(rows, dtype=np.uint8)
    want[np.setdiff1d(pert, evicted)] = 1
    assert (trained == want).all(), f"{(trained != want).sum()} trained flags differ"
    fresh_rows = po.draw_rows(dim, evicted, init_seed)
    kept_w = po.draw_rows(dim, kept, init_seed) - np.float32(lr)  # w - lr * (beta * 0 + 1)
    CH = 1 << 20
    for a in range(0, rows, CH):
        w = t.weights(a, CH)
        m = t.momentum(a, CH)
        lo, hi = np.searchsorted(evicted, [a, a + CH])
        e = (evicted[lo:hi] - a).astype(np.int64)
        assert (w[e].view(np.uint32) == fresh_rows[lo:hi].view(np.uint32)).all(), f"reset rows differ near {a}"
        assert (m[e].view(np.uint32) == 0).all(), f"momentum of reset rows not zero near {a}"
        lo, hi = np.searchsorted(kept, [a, a + CH])
        k = (kept[lo:hi] - a).astype(np.int64)
        assert (w[k].view(np.uint32) == kept_w[lo:hi].view(np.uint32)).all(), f"control rows differ near {a}"
        assert (m[k] == 1.0).all()
