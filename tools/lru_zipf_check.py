"""Replay the lru_zipf stream (tools/bench_configs.py) through the GPU table and the reference
library side by side and report the first batch whose slots / outcomes / evicted list differ.
Usage: python tools/lru_zipf_check.py [rows_log2] [batches] [path]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
import bench  # noqa: E402
import paper_2602_17050_b200 as mz  # noqa: E402
import pyoracle  # noqa: E402
sys.path.insert(0, os.path.dirname(__file__))
from bench_configs import zipf_cdf, zipf_ranks  # noqa: E402


def main():
    rows = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    path = sys.argv[3] if len(sys.argv) > 3 else "auto"
    universe, B = 1 << 27, 1 << 20
    zipf_ranks.cdf = zipf_cdf(universe)
    caps = mz.even_capacities(rows, 8)
    t = mz.MpzchTable(mz.TableConfig(caps, 128, 7))
    t.set_path(path)
    L = pyoracle.lib("reference")
    L["set_threads"](os.cpu_count() or 1)
    o = pyoracle.OracleTable(caps, 128, 7, 0, 0, kind="reference")
    pol = mz.EvictionPolicy.lru()
    for b in range(nb):
        ids = bench.distinct_ids_t(2, zipf_ranks(B, 1.05, universe, 3000 + b)).cpu().numpy().view(np.uint64)
        now = 10**6 + 60 * b
        gs, go, ge = t.process_batch(ids, now, pol)
        rs, ro, re_ = o.process_batch(ids, now, 2, 0)
        st = t.last_stats()
        ok = (gs == rs).all() and (go == ro).all() and ge.size == re_.size and (ge == re_).all()
        print(f"batch {b}: path={st['path']} rounds={st['rounds']} evicted={st['evicted']} "
              f"{'ok' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            bad = np.nonzero((gs != rs) | (go != ro))[0]
            print(f"  {bad.size} positions differ; first {bad[:5]}, gpu {gs[bad[:5]]} {go[bad[:5]]} "
                  f"ref {rs[bad[:5]]} {ro[bad[:5]]}; evicted {ge.size} vs {re_.size}")
            sys.exit(1)
    same_state = (t.identities_all() == o.identities_all()).all() and (t.metadata_all() == o.metadata_all()).all()
    print("final state", "ok" if same_state else "MISMATCH")


if __name__ == "__main__":
    main()
