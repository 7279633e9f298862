"""Row-sharded MPZCH table over G ranks (one process per GPU) -- SURVEY 8e.

The S logical shards of one table layout (proj/include/mpzch/shard_router.hpp:13-29) are
spread over G ranks in contiguous blocks (rank r holds shards s with s*G//S == r).  Global
row numbers are those of the single-table layout, so every remapped slot is identical for
G = 1, 2, 4, 8.  A batch of N positions is split into G contiguous slices (rank r holds
positions [base_r, base_r + n_r)); one process_batch is:

  1. validate the slice (mpzch_validate_device) and agree on the first invalid GLOBAL
     position (all-reduce MIN): every rank raises the reference's
     "invalid id at batch position N" before anything is mutated
     (proj/src/batch_engine.cpp:90-94, 146-147);
  2. route: stable partition of the slice by owner (mpzch_route_device, shard_of
     proj/src/shard_router.cpp:42-46) and an all-to-all of (id, feature) -- NCCL over
     NVLink.  Because slices are rank-ordered and the partition is stable, each owner
     receives its positions in global first-occurrence order, which is exactly the
     order the reference's dedup gives (batch_engine.cpp:100-106), so the owner's claim
     ranks reproduce the single-table result with no sort;
  3. the owner remaps (mpzch_process_batch_device_marked) -- shards are independent
     (proj/include/mpzch/batch_engine.hpp:39-43), so no other exchange is needed;
  4. (slot, outcome, first-evicted mark) travel back by the reverse all-to-all and are
     scattered to the slice; the canonical evicted list is the rank-ordered
     concatenation of each rank's marked positions (an all-gather).

The communication and the per-rank engine are parameters, so the same protocol runs
with torch.distributed (NCCL on GPUs, gloo on CPU in the tests), with in-process
threads on one GPU (tests), and with any engine exposing validate/route/remap.

transport="peer" replaces both all-to-alls with stores into peer memory (PeerTransport):
step 2 becomes one kernel (mpzch_route_scatter_device) that partitions the slice and writes
every (id, feature, source position) straight into its owner's receive buffers over NVLink
(P2P / CUDA IPC mappings), at an offset the ranks agree on from an all-gather of the per-part
counts; step 4 becomes one kernel (mpzch_return_scatter_device) in which the owner writes
every result straight into the source rank's result buffers at the source position, so the
inverse permutation disappears too.  Phases are ordered by a stream sync + barrier.
"""
from __future__ import annotations

import threading
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import (EvictionPolicy, InvalidArgument, LengthError, MpzchTable, OverflowError_,
               TableConfig)

INF = (1 << 64) - 1


def shard_owner(shard: int, num_shards: int, parts: int) -> int:
    return shard * parts // num_shards


def held_shards(rank: int, num_shards: int, parts: int) -> Tuple[int, int]:
    """[lo, hi) of the contiguous shard block rank `rank` holds."""
    owned = [s for s in range(num_shards) if shard_owner(s, num_shards, parts) == rank]
    if not owned:
        raise InvalidArgument("row-sharded mode needs at least one logical shard per rank "
                              f"(S={num_shards}, G={parts})")
    return owned[0], owned[-1] + 1


# ------------------------------------------------------------------------------ comms

class TorchComm:
    """Collectives over torch.distributed: NCCL moves CUDA tensors directly (NVLink); with a
    gloo group, CUDA tensors are staged through host memory (used to exercise the
    multi-rank path on a single-GPU box)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.stage = dist.get_backend(group) == "gloo"

    def _dev(self, like):
        return "cpu" if self.stage else like.device

    def _to(self, t):
        return t.cpu() if self.stage and t.is_cuda else t

    def all_gather_int(self, x: int, like) -> List[int]:
        import torch
        t = torch.tensor([x], dtype=torch.int64, device=self._dev(like))
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(v.item()) for v in out]

    def all_reduce_min(self, x: int, like) -> int:
        import torch
        t = torch.tensor([x if x < (1 << 63) else (1 << 63) - 1], dtype=torch.int64,
                         device=self._dev(like))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        v = int(t.item())
        return INF if v == (1 << 63) - 1 else v

    def all_to_all(self, send, send_counts: Sequence[int], recv_counts: Sequence[int]):
        import torch
        src = self._to(send.contiguous())
        out = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype,
                          device=src.device)
        self.dist.all_to_all_single(out, src, list(recv_counts), list(send_counts),
                                    group=self.group)
        return out.to(send.device)

    in_process = False

    def barrier(self):
        self.dist.barrier(group=self.group)

    def all_gather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def all_gather_ints(self, xs: Sequence[int], like) -> List[List[int]]:
        """One small tensor all-gather (no pickling): every rank's int list."""
        import torch
        t = torch.tensor([int(x) for x in xs], dtype=torch.int64, device=self._dev(like))
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return torch.stack(out).cpu().tolist()

    def all_gather_v(self, t, counts: Sequence[int]):
        import torch
        m = max(counts) if counts else 0
        src = self._to(t)
        pad = torch.zeros(max(m, 1), dtype=t.dtype, device=src.device)
        pad[:src.numel()] = src
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad, group=self.group)
        return torch.cat([o[:c] for o, c in zip(outs, counts)]).to(t.device)


class ThreadComm:
    """In-process collectives for G logical ranks driven by G threads (one GPU tests)."""

    class _Hub:
        def __init__(self, world, timeout=600.0):
            self.world = world
            self.barrier = threading.Barrier(world, timeout=timeout)
            self.slots = [None] * world

    def __init__(self, hub: "_Hub", rank: int):
        self.hub = hub
        self.rank = rank
        self.world = hub.world

    @classmethod
    def group(cls, world: int):
        hub = cls._Hub(world)
        return [cls(hub, r) for r in range(world)]

    def abort(self):
        """Break the barrier so the other ranks fail instead of waiting forever."""
        self.hub.barrier.abort()

    def _exchange(self, obj):
        self.hub.barrier.wait()
        self.hub.slots[self.rank] = obj
        self.hub.barrier.wait()
        got = list(self.hub.slots)
        self.hub.barrier.wait()
        return got

    in_process = True  # every rank's buffers are addressable directly

    def barrier(self):
        self.hub.barrier.wait()

    def all_gather_object(self, obj):
        return self._exchange(obj)

    def all_gather_ints(self, xs, like):
        return [[int(v) for v in x] for x in self._exchange(list(xs))]

    def all_gather_int(self, x, like):
        return [int(v) for v in self._exchange(int(x))]

    def all_reduce_min(self, x, like):
        return min(self._exchange(int(x)))

    def all_to_all(self, send, send_counts, recv_counts):
        import torch
        offs = np.concatenate([[0], np.cumsum(send_counts)]).astype(np.int64)
        chunks = [send[offs[d]:offs[d + 1]] for d in range(self.world)]
        allc = self._exchange(chunks)
        return torch.cat([allc[src][self.rank] for src in range(self.world)])

    def all_gather_v(self, t, counts):
        import torch
        return torch.cat(self._exchange(t))


# ------------------------------------------------------------------------------ peer memory

class PeerTransport:
    """This rank's receive / result buffers and the device addresses of every rank's.

    Receive side (an owner's): ids u64, features u32, source positions u32 -- written by the
    sources' route-scatter kernels.  Result side (a source's): slots u64, outcomes u8, marks u8
    -- written by the owners' return-scatter kernels.  Buffers grow collectively (every rank
    reallocates and re-exchanges addresses when any rank needs more room)."""

    KEYS = (("ids", "int64"), ("feats", "int32"), ("src", "int32"), ("slots", "int64"),
            ("oc", "uint8"), ("mark", "uint8"))

    def __init__(self, comm, device: int):
        self.comm, self.device = comm, device
        self.cap = 0
        self.local = {}
        self.peers: List[dict] = []
        self._imported: List[int] = []

    def close(self):
        from . import ipc_close
        for a in self._imported:
            ipc_close(a)
        self._imported = []

    def ensure(self, want: int):
        """Collective when it grows: `want` must be the same on every rank."""
        import torch
        from . import ipc_export, ipc_import
        if want <= self.cap:
            return
        cap = 1024
        while cap < want:
            cap <<= 1
        self.close()
        self.local = {k: torch.empty(cap, dtype=getattr(torch, dt), device=f"cuda:{self.device}")
                      for k, dt in self.KEYS}
        if self.comm.in_process:
            self.peers = self.comm.all_gather_object({k: v.data_ptr() for k, v in self.local.items()})
        else:
            torch.cuda.synchronize(self.device)
            recs = self.comm.all_gather_object({k: ipc_export(v) for k, v in self.local.items()})
            self.peers = []
            for r, rec in enumerate(recs):
                if r == self.comm.rank:
                    self.peers.append({k: v.data_ptr() for k, v in self.local.items()})
                else:
                    addrs = {k: ipc_import(self.device, rec[k]) for k in rec}
                    self._imported += list(addrs.values())
                    self.peers.append(addrs)
        self.cap = cap

    def addrs(self, key: str) -> List[int]:
        return [p[key] for p in self.peers]


def peer_offsets(all_counts: Sequence[Sequence[int]], rank: int) -> Tuple[List[int], List[int]]:
    """(offsets of this rank's positions in every owner's receive buffer, received counts):
    sources are laid out in rank order, so owner q's buffer holds the global batch's part-q
    positions in global order."""
    world = len(all_counts)
    offset = [sum(int(all_counts[r][q]) for r in range(rank)) for q in range(world)]
    recv = [int(all_counts[r][rank]) for r in range(world)]
    return offset, recv


# ------------------------------------------------------------------------------ engines

class GpuEngine:
    """The per-rank engine: the rank's sm_100a table handle (held shards only)."""

    def __init__(self, cfg: TableConfig, rank: int, world: int, device: int):
        lo, hi = held_shards(rank, len(cfg.shard_capacities), world)
        self.table = MpzchTable(cfg, device=device, shard_range=(lo, hi))
        self.device = device

    def validate(self, ids) -> Optional[int]:
        return self.table.validate_device(ids)

    def route(self, ids, shard_to_part, parts):
        return self.table.route_device(ids, shard_to_part, parts)

    def route_count(self, ids, shard_to_part, parts):
        return self.table.route_count_device(ids, shard_to_part, parts)

    def route_scatter(self, ids, features, parts, ids_to, features_to, src_to, offset):
        self.table.route_scatter_device(ids, features, parts, ids_to, features_to, src_to, offset)

    def remap(self, ids, features, now, policy):
        return self.table.process_batch_device_marked(ids, now, policy, features)


# ------------------------------------------------------------------------------ protocol

class ShardedMpzchTable:
    """One rank's view of a row-sharded MpzchTable (proj/include/mpzch/table.hpp:41-131)."""

    def __init__(self, cfg: TableConfig, comm, engine=None, device: int = 0, transport: str = "collective"):
        if transport not in ("collective", "peer"):
            raise InvalidArgument("transport must be 'collective' or 'peer'")
        self.cfg = cfg
        self.comm = comm
        self.transport = transport
        self.device = device
        self.peer = PeerTransport(comm, device) if transport == "peer" else None
        self.rank, self.world = comm.rank, comm.world
        self.num_shards = len(cfg.shard_capacities)
        self.shard_to_part = np.array([shard_owner(s, self.num_shards, self.world)
                                       for s in range(self.num_shards)], dtype=np.uint32)
        self.engine = engine if engine is not None else GpuEngine(cfg, self.rank, self.world, device)

    def process_batch(self, ids, now: int, policy: EvictionPolicy, features=None):
        """Remap this rank's slice of the global batch.  Returns (slots, outcomes,
        evicted) where evicted is the GLOBAL canonical evicted list (identical on every
        rank)."""
        import torch
        if self.peer is not None:
            return self._process_peer(ids, features, now, policy)
        comm = self.comm
        n = ids.numel()
        sizes = comm.all_gather_int(n, ids)
        base = sum(sizes[:self.rank])
        if sum(sizes) > 0xFFFFFFFF:  # batch_engine.cpp:82-83
            raise LengthError("batch exceeds 2^32 - 1 positions")
        bad = self.engine.validate(ids) if n else None
        gbad = comm.all_reduce_min(INF if bad is None else base + bad, ids)
        if gbad != INF:
            raise InvalidArgument(f"invalid id at batch position {gbad}")
        if policy.mode == EvictionPolicy.TTL:
            # make_metadata (eviction.cpp:20-30) over the features present anywhere in the
            # batch: decided globally so every rank raises (or not) together
            limit = (1 << 64) - 1 - now
            present = [0] if features is None else [int(f) for f in torch.unique(features).tolist()]
            over = any(policy.ttl.ttl_for(f) > limit for f in present) if n else False
            if comm.all_reduce_min(0 if over else 1, ids) == 0:
                raise OverflowError_("TTL expiry overflows the 64-bit timestamp range")
        perm, send_counts = self.engine.route(ids, self.shard_to_part, self.world)
        recv_counts = self._exchange_counts(send_counts, ids)
        permi = perm.long()
        rid = comm.all_to_all(ids[permi], send_counts, recv_counts)
        rfeat = None
        if features is not None:
            rfeat = comm.all_to_all(features[permi], send_counts, recv_counts)
        rs, ro, rm = self.engine.remap(rid, rfeat, now, policy)
        bs = comm.all_to_all(rs, recv_counts, send_counts)
        bo = comm.all_to_all(ro, recv_counts, send_counts)
        bm = comm.all_to_all(rm, recv_counts, send_counts)
        slots = torch.empty_like(bs)
        oc = torch.empty_like(bo)
        mark = torch.empty_like(bm)
        slots[permi] = bs
        oc[permi] = bo
        mark[permi] = bm
        mine = slots[mark.bool()]
        counts = comm.all_gather_int(mine.numel(), ids)
        evicted = comm.all_gather_v(mine, counts)
        return slots, oc, evicted

    def close(self):
        """Unmap the other ranks' buffers (peer transport); call on every rank before the
        process group goes away.  (Process exit unmaps them too.)"""
        if self.peer is not None:
            self.peer.close()

    def _process_peer(self, ids, features, now, policy):
        """process_batch over peer memory in four host collectives: (1) one small all-gather
        carries every rank's slice size, first invalid position, TTL-overflow flag and
        per-part counts -- the errors are raised on every rank before anything moves; (2) a
        barrier after the route-scatter kernel; (3) after the owners' return-scatter, an
        all-gather of each owner's per-source count of first-evicted marks (it doubles as the
        barrier); (4) the all-gather of the marked slots (the canonical evicted list)."""
        import torch
        from . import return_scatter_device
        comm, tp, G = self.comm, self.peer, self.world
        n = ids.numel()
        bad = self.engine.validate(ids) if n else None
        over = 0
        if policy.mode == EvictionPolicy.TTL and n:  # make_metadata, eviction.cpp:20-30
            limit = (1 << 64) - 1 - now
            present = [0] if features is None else [int(f) for f in torch.unique(features).tolist()]
            over = int(any(policy.ttl.ttl_for(f) > limit for f in present))
        send_counts = self.engine.route_count(ids, self.shard_to_part, G)
        allv = comm.all_gather_ints([n, -1 if bad is None else bad, over] + send_counts, ids)
        sizes = [v[0] for v in allv]
        if sum(sizes) > 0xFFFFFFFF:  # batch_engine.cpp:82-83
            raise LengthError("batch exceeds 2^32 - 1 positions")
        bads = [sum(sizes[:r]) + v[1] for r, v in enumerate(allv) if v[1] >= 0]
        if bads:  # batch_engine.cpp:90-94: the first invalid GLOBAL position, on every rank
            raise InvalidArgument(f"invalid id at batch position {min(bads)}")
        if any(v[2] for v in allv):
            raise OverflowError_("TTL expiry overflows the 64-bit timestamp range")
        allc = [v[3:] for v in allv]
        offset, recv = peer_offsets(allc, self.rank)
        R = sum(recv)
        # room for the largest slice and the largest received set of any rank (same on all)
        tp.ensure(max(max(sizes), max(sum(col) for col in zip(*allc))))
        self.engine.route_scatter(ids, features, G, tp.addrs("ids"),
                                  tp.addrs("feats") if features is not None else None,
                                  tp.addrs("src"), offset)
        stream = torch.cuda.current_stream(self.device)
        stream.synchronize()
        comm.barrier()  # every source's stores have landed in this owner's buffers
        rid = tp.local["ids"][:R]
        rfeat = tp.local["feats"][:R] if features is not None else None
        rs, ro, rm = self.engine.remap(rid, rfeat, now, policy)
        roff = np.concatenate([[0], np.cumsum(recv)]).astype(np.uint64)
        return_scatter_device(self.device, rs, ro, rm, tp.local["src"][:R], roff, tp.addrs("slots"),
                              tp.addrs("oc"), tp.addrs("mark"))
        if R:
            src_rank = torch.repeat_interleave(torch.arange(G, device=rm.device),
                                               torch.tensor(recv, device=rm.device))
            per_src = torch.bincount(src_rank[rm.bool()], minlength=G).tolist()
        else:
            per_src = [0] * G
        stream.synchronize()
        marks = comm.all_gather_ints(per_src, ids)  # also: every owner's results have landed
        ev_counts = [sum(marks[o][r] for o in range(G)) for r in range(G)]
        slots = tp.local["slots"][:n].clone()
        oc = tp.local["oc"][:n].clone()
        mine = slots[tp.local["mark"][:n].bool()]
        return slots, oc, comm.all_gather_v(mine, ev_counts)

    def _exchange_counts(self, send_counts, like):
        import torch
        t = torch.tensor(send_counts, dtype=torch.int64, device=like.device)
        ones = [1] * self.world
        got = self.comm.all_to_all(t, ones, ones)
        return [int(v) for v in got.tolist()]
