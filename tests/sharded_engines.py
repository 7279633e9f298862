"""Test-only engine for the row-sharded protocol on CPU: the oracle (C restatement) plays
the owner's table so the host protocol (routing order, all-to-all, reassembly, evicted
list, error agreement) can be checked with gloo on CPU.  TEST INFRASTRUCTURE."""
import numpy as np
import torch

import pyoracle

EVICTED = 2


class OracleEngine:
    def __init__(self, cfg):
        self.cfg = cfg
        self.t = pyoracle.OracleTable(cfg.shard_capacities, cfg.max_probe, cfg.seed, cfg.dim,
                                      cfg.init_seed)
        self.S = len(cfg.shard_capacities)

    def validate(self, ids):
        a = ids.numpy().view(np.uint64)
        bad = np.nonzero(a >> np.uint64(63))[0]
        return int(bad[0]) if bad.size else None

    def route(self, ids, shard_to_part, parts):
        a = ids.numpy().view(np.uint64)
        shard = (pyoracle.mix64_np(a ^ np.uint64(0xD1B54A32D192ED03), self.cfg.seed) %
                 np.uint64(self.S)).astype(np.int64)
        part = np.asarray(shard_to_part, dtype=np.int64)[shard]
        perm = np.argsort(part, kind="stable").astype(np.int32)
        counts = np.bincount(part, minlength=parts).tolist()
        return torch.from_numpy(perm), counts

    def remap(self, ids, features, now, policy):
        a = ids.numpy().view(np.uint64)
        f = None if features is None else features.numpy().astype(np.uint32)
        mode = policy.mode
        s, o, _ = self.t.process_batch(a, now, mode, policy.ttl.default_ttl_seconds if mode == 1 else 0,
                                       dict(policy.ttl.per_feature_ttl) if mode == 1 else {}, f)
        # first position of every Evicted (id, feature) unique
        mark = np.zeros(a.size, dtype=np.uint8)
        seen = set()
        for i in range(a.size):
            key = (int(a[i]), 0 if f is None else int(f[i]))
            if key in seen:
                continue
            seen.add(key)
            if o[i] == EVICTED:
                mark[i] = 1
        return (torch.from_numpy(s.view(np.int64).copy()), torch.from_numpy(o.copy()),
                torch.from_numpy(mark))
