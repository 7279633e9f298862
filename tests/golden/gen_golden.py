"""Generate tests/golden/ref_streams.npz by running the REFERENCE library itself.

The reference (/root/reference/proj/src, compiled by oracle/Makefile into
oracle/_ref/libmpzch_ref.so, its own process_batch / lookup_or_insert code) is
fed the seeded workloads of tests/workloads.py; every input, every per-position
(slot, outcome), the canonical evicted list and the final table state are stored.
The GPU box has no /root/reference: the -m gpu tests replay these fixtures.

Run here (CPU):  python tests/golden/gen_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import pyoracle  # noqa: E402
import workloads  # noqa: E402


def run_case(case, kind="reference"):
    t = pyoracle.OracleTable(case.caps, case.max_probe, case.seed, case.dim, case.init_seed, kind=kind)
    outs = []
    for b in case.batches:
        s, o, e = t.process_batch(b.ids, b.now, case.mode, b.default_ttl, b.per_feature, b.features)
        outs.append((s, o, e))
    state = dict(ident=t.identities_all(), meta=t.metadata_all())
    if case.dim:
        state.update(weights=t.weights(), momentum=t.momentum(), trained=t.trained())
    return outs, state


def main():
    cases = (workloads.crit8_cases() + workloads.parallel_cases() + workloads.dense_cases() +
             workloads.oracle_cases(count=120))
    ids, feats, slots, ocs, evs = [], [], [], [], []
    bt = []  # per batch: case, pos0, pos1, ev0, ev1, now, default_ttl, has_f
    st = {k: [] for k in ("ident", "meta", "weights", "momentum", "trained")}
    manifest = []
    npos = nev = 0
    for ci, c in enumerate(cases):
        outs, state = run_case(c)
        pf = {}
        for b, (s, o, e) in zip(c.batches, outs):
            ids.append(b.ids)
            feats.append(b.features if b.features is not None else np.zeros(b.ids.size, np.uint32))
            slots.append(s)
            ocs.append(o)
            evs.append(e)
            bt.append([ci, npos, npos + b.ids.size, nev, nev + e.size, b.now, b.default_ttl,
                       int(b.features is not None)])
            npos += b.ids.size
            nev += e.size
            pf = b.per_feature
        manifest.append(dict(name=c.name, caps=c.caps, max_probe=c.max_probe, seed=str(c.seed),
                             dim=c.dim, init_seed=str(c.init_seed), mode=c.mode,
                             per_feature={str(x): y for x, y in pf.items()}))
        for k in st:
            if k in state:
                st[k].append(state[k].reshape(-1))
    arrays = dict(ids=np.concatenate(ids), feats=np.concatenate(feats), slots=np.concatenate(slots),
                  oc=np.concatenate(ocs), ev=np.concatenate(evs) if evs else np.zeros(0, np.uint64),
                  batches=np.array(bt, dtype=np.uint64))
    for k, v in st.items():
        arrays["state_" + k] = np.concatenate(v) if v else np.zeros(0)
    np.savez_compressed(os.path.join(HERE, "ref_streams.npz"), **arrays)
    with open(os.path.join(HERE, "ref_streams.json"), "w") as f:
        json.dump(dict(generator="tests/golden/gen_golden.py", source="oracle/_ref (reference library)",
                       cases=manifest), f, indent=0)
    print(f"{len(manifest)} cases, {len(bt)} batches, {npos} positions")


if __name__ == "__main__":
    main()
