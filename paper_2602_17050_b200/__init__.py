"""paper_2602_17050_b200 -- B200-native MPZCH batched ID remap.

Python mirror of the reference's C++ remap API (namespace ``mpzch``), over the
C-ABI of ``include/mpzch_b200.h`` implemented by the sm_100a library
``_lib/libmpzch_b200.so``.  Names, argument meaning and error behaviour follow
the reference (paths relative to /root/reference/):

=====================================  ==============================================
this module                            reference
=====================================  ==============================================
``TableConfig`` / ``TableConfig.even`` proj/include/mpzch/table.hpp:18-28
``EvictionPolicy.disabled/lru/ttl``    proj/include/mpzch/eviction.hpp:27-46
``TtlPolicy``                          proj/include/mpzch/eviction.hpp:13-23
``MpzchTable``                         proj/include/mpzch/table.hpp:41-131
``process_batch``                      proj/include/mpzch/batch_engine.hpp:44-46
``MpzchTable.lookup``                  proj/include/mpzch/table.hpp:65 (batched)
``MpzchTable.lookup_or_insert``        proj/include/mpzch/table.hpp:61-62
=====================================  ==============================================

Exceptions mirror the reference's std exception types (``InvalidArgument`` for
std::invalid_argument, ...).  There is no CPU fallback: importing this module
without the built CUDA library raises ``ImportError``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Dict, Iterable, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "FOUND", "INSERTED", "EVICTED", "COLLISION", "OUTCOME_NAMES",
    "MpzchError", "InvalidArgument", "OverflowError_", "LengthError", "LogicError", "OutOfRange",
    "CudaError", "TtlPolicy", "EvictionPolicy", "TableConfig", "MpzchTable", "process_batch",
    "lib_path", "load_library", "even_capacities",
]

FOUND, INSERTED, EVICTED, COLLISION = 0, 1, 2, 3
OUTCOME_NAMES = ("found", "inserted", "evicted", "collision")  # probe_core.cpp:17-25

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    # MPZCH_LIB_PATH: another build of the same sm_100a library (A/B measurements)
    return os.environ.get("MPZCH_LIB_PATH") or os.path.join(_HERE, "_lib", "libmpzch_b200.so")


class MpzchError(RuntimeError):
    pass


class InvalidArgument(MpzchError, ValueError):      # std::invalid_argument
    pass


class OverflowError_(MpzchError, OverflowError):     # std::overflow_error
    pass


class LengthError(MpzchError, ValueError):           # std::length_error
    pass


class LogicError(MpzchError):                        # std::logic_error
    pass


class OutOfRange(MpzchError, IndexError):            # std::out_of_range
    pass


class CudaError(MpzchError):
    pass


class OutOfMemory(MpzchError, MemoryError):
    pass


_STATUS = {1: InvalidArgument, 2: OverflowError_, 3: LengthError, 4: LogicError, 5: OutOfRange,
           6: CudaError, 7: OutOfMemory, 8: CudaError}


class _Policy(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("n_feat", ctypes.c_uint32),
                ("default_ttl", ctypes.c_uint64),
                ("feat_keys", ctypes.POINTER(ctypes.c_uint32)),
                ("feat_ttls", ctypes.POINTER(ctypes.c_uint64))]


class _Stats(ctypes.Structure):
    _fields_ = [("positions", ctypes.c_uint64), ("new_positions", ctypes.c_uint64),
                ("new_ids", ctypes.c_uint64), ("found", ctypes.c_uint64),
                ("inserted", ctypes.c_uint64), ("evicted", ctypes.c_uint64),
                ("collision", ctypes.c_uint64), ("evicted_rows", ctypes.c_uint64),
                ("path", ctypes.c_uint32), ("rounds", ctypes.c_uint32)]


class _Profile(ctypes.Structure):
    _fields_ = [("batches", ctypes.c_uint64), ("probe_launches", ctypes.c_uint64),
                ("probe_ms", ctypes.c_double), ("claim_ms", ctypes.c_double),
                ("tail_ms", ctypes.c_double), ("batch_ms", ctypes.c_double),
                ("probe_sectors", ctypes.c_uint64), ("probe_bytes", ctypes.c_uint64),
                ("batch_bytes", ctypes.c_uint64), ("validate_ms", ctypes.c_double),
                ("dedup_ms", ctypes.c_double), ("claimk_ms", ctypes.c_double),
                ("commit_ms", ctypes.c_double), ("finalize_ms", ctypes.c_double)]


_LIB = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_f32p = ctypes.POINTER(ctypes.c_float)
_vp = ctypes.c_void_p

# name -> (restype, argtypes); the exact exported surface of include/mpzch_b200.h
_SIGS = {
    "mpzch_table_create": (ctypes.c_int, [_u64p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                          ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                                          ctypes.POINTER(_vp)]),
    "mpzch_table_destroy": (ctypes.c_int, [_vp]),
    "mpzch_total_rows": (ctypes.c_uint64, [_vp]),
    "mpzch_num_shards": (ctypes.c_uint32, [_vp]),
    "mpzch_max_probe": (ctypes.c_uint32, [_vp]),
    "mpzch_dim": (ctypes.c_uint32, [_vp]),
    "mpzch_shard_layout": (ctypes.c_int, [_vp, _u64p, _u64p]),
    "mpzch_process_batch": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.POINTER(_Policy), _vp, _vp, _vp,
                                           ctypes.c_uint64, _u64p]),
    "mpzch_process_batch_device": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64, ctypes.c_uint64,
                                                  ctypes.POINTER(_Policy), _vp, _vp, _vp,
                                                  ctypes.c_uint64, _u64p, _vp]),
    "mpzch_process_batch_device_async": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64,
                                                        ctypes.c_uint64, ctypes.POINTER(_Policy),
                                                        _vp, _vp, _vp, ctypes.c_uint64, _vp, _u64p]),
    "mpzch_batch_wait": (ctypes.c_int, [_vp, ctypes.c_uint64, _u64p]),
    "mpzch_lookup": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp, _vp]),
    "mpzch_lookup_device": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp, _vp, _vp]),
    "mpzch_lookup_or_insert": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint32,
                                              ctypes.c_uint64, ctypes.POINTER(_Policy), _u64p,
                                              _u8p]),
    "mpzch_copy_identities": (ctypes.c_int, [_vp, _vp]),
    "mpzch_copy_metadata": (ctypes.c_int, [_vp, _vp]),
    "mpzch_copy_weights": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, _vp]),
    "mpzch_copy_momentum": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, _vp]),
    "mpzch_copy_trained": (ctypes.c_int, [_vp, _vp]),
    "mpzch_copy_row_generation": (ctypes.c_int, [_vp, _vp]),
    "mpzch_device_arrays": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                           ctypes.POINTER(_vp)]),
    "mpzch_write_slots": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp, _vp, _vp, ctypes.c_uint64]),
    "mpzch_check_hole_free": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int)]),
    "mpzch_write_row": (ctypes.c_int, [_vp, ctypes.c_uint64, _vp, _vp, ctypes.c_uint8]),
    "mpzch_make_cursor": (ctypes.c_int, [_vp, _u64p]),
    "mpzch_dirty_rows_since": (ctypes.c_int, [_vp, ctypes.c_uint64, _vp, ctypes.c_uint64, _u64p]),
    "mpzch_table_create_sharded": (ctypes.c_int, [_u64p, ctypes.c_uint32, ctypes.c_uint32,
                                                  ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                                  ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                                  ctypes.POINTER(_vp)]),
    "mpzch_held_rows": (ctypes.c_int, [_vp, _u64p, _u64p, _u32p, _u32p]),
    "mpzch_validate_device": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _u64p, _vp]),
    "mpzch_route_device": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _u32p, ctypes.c_uint32, _vp,
                                          _u64p, _vp]),
    "mpzch_route_count_device": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _u32p, ctypes.c_uint32,
                                                _u64p, _vp]),
    "mpzch_route_scatter_device": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64, ctypes.c_uint32,
                                                  _u64p, _u64p, _u64p, _u64p, _vp]),
    "mpzch_return_scatter_device": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, _vp, _vp, _vp, _vp,
                                                   ctypes.c_uint32, _u64p, _u64p, _u64p, _u64p, _vp]),
    "mpzch_ipc_export": (ctypes.c_int, [_vp, _vp]),
    "mpzch_ipc_import": (ctypes.c_int, [ctypes.c_int, _vp, _u64p]),
    "mpzch_ipc_close": (ctypes.c_int, [ctypes.c_uint64]),
    "mpzch_process_batch_device_marked": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64,
                                                         ctypes.c_uint64, ctypes.POINTER(_Policy),
                                                         _vp, _vp, _vp, _u64p, _vp]),
    "mpzch_lookup_gather_device": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp, _vp, _vp, _vp]),
    "mpzch_delta_cut": (ctypes.c_int, [_vp, ctypes.c_uint64, _vp, _vp, _vp, ctypes.c_uint64, _u64p,
                                       _u64p]),
    "mpzch_sgd_step": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp, ctypes.c_uint64, ctypes.c_float,
                                      ctypes.c_float]),
    "mpzch_sgd_step_device": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp, ctypes.c_uint64,
                                             ctypes.c_float, ctypes.c_float, _vp]),
    "mpzch_crc32_device": (ctypes.c_int, [_vp, ctypes.c_uint64, _u32p, _vp]),
    "mpzch_serialize_snapshot": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _u64p]),
    "mpzch_serialize_delta": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                             _vp, ctypes.c_uint64, _u64p, _u64p]),
    "mpzch_set_path": (ctypes.c_int, [_vp, ctypes.c_int]),
    "mpzch_set_reset_mode": (ctypes.c_int, [_vp, ctypes.c_int]),
    "mpzch_sharded_create": (ctypes.c_int, [_u64p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                            ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32,
                                            ctypes.c_uint32, ctypes.c_uint64, ctypes.POINTER(_vp)]),
    "mpzch_sharded_destroy": (ctypes.c_int, [_vp]),
    "mpzch_sharded_table": (_vp, [_vp]),
    "mpzch_sharded_held_shards": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_uint32),
                                                 ctypes.POINTER(ctypes.c_uint32)]),
    "mpzch_sharded_export": (ctypes.c_int, [_vp, _vp]),
    "mpzch_sharded_connect_ipc": (ctypes.c_int, [_vp, _vp]),
    "mpzch_sharded_connect_local": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_uint32]),
    "mpzch_sharded_process_batch_async": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64, ctypes.c_uint64, _vp,
                                                         _vp, _vp, _vp, ctypes.c_uint64, _vp, _u64p]),
    "mpzch_sharded_wait": (ctypes.c_int, [_vp, ctypes.c_uint64, _u64p]),
    "mpzch_sharded_process_batch": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64, ctypes.c_uint64, _vp,
                                                   _vp, _vp, _vp, ctypes.c_uint64, _u64p, _vp]),
    "mpzch_sharded_last_stats": (ctypes.c_int, [_vp, ctypes.POINTER(_Stats), ctypes.POINTER(ctypes.c_int)]),
    "mpzch_sharded_group_process_batch": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_uint32, _vp, _vp,
                                                         ctypes.c_uint64, ctypes.c_uint64, _vp, _vp, _vp, _vp,
                                                         ctypes.c_uint64, _u64p]),
    "mpzch_flush_resets": (ctypes.c_int, [_vp]),
    "mpzch_set_profiling": (ctypes.c_int, [_vp, ctypes.c_int]),
    "mpzch_get_profile": (ctypes.c_int, [_vp, ctypes.POINTER(_Profile)]),
    "mpzch_last_stats": (ctypes.c_int, [_vp, ctypes.POINTER(_Stats)]),
    "mpzch_lookup_device_async": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp, _vp, _vp, _u64p]),
    "mpzch_kernel_launches": (ctypes.c_uint64, [_vp]),
    "mpzch_process_shard_batch": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp, _vp, ctypes.c_uint64,
                                                 ctypes.c_uint64, ctypes.POINTER(_Policy), _vp, _vp]),
    "mpzch_dedup": (ctypes.c_int, [ctypes.c_int, _vp, _vp, ctypes.c_uint64, _vp, _vp, _vp, _u64p]),
    "mpzch_dedup_device": (ctypes.c_int, [ctypes.c_int, _vp, _vp, ctypes.c_uint64, _vp, _vp, _vp,
                                          _u64p, _vp]),
    "mpzch_reset_row": (ctypes.c_int, [_vp, ctypes.c_uint64]),
    "mpzch_state_equals": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(ctypes.c_int)]),
    "mpzch_read_identity": (ctypes.c_int, [_vp, ctypes.c_uint64, _u64p]),
    "mpzch_copy_identities_range": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, _vp]),
    "mpzch_copy_metadata_range": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, _vp]),
    "mpzch_copy_trained_range": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64, _vp]),
    "mpzch_gather": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp]),
    "mpzch_shard_config": (ctypes.c_int, [_vp, ctypes.c_uint32, _u64p, _u32p, _u64p]),
    "mpzch_last_error": (ctypes.c_char_p, []),
    "mpzch_build_info": (ctypes.c_char_p, []),
}


def load_library():
    """Load the sm_100a library; raise ImportError (no fallback) when it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(f"MPZCH CUDA library not built ({path}); run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def _check(rc: int):
    if rc != 0:
        msg = _LIB.mpzch_last_error().decode()
        raise _STATUS.get(rc, MpzchError)(msg)


def return_scatter_device(device: int, slots, outcomes, marks, src, recv_offset, slots_to,
                          outcomes_to, marks_to=None, stream=None):
    """Store received results into the source ranks' buffers (mpzch_return_scatter_device)."""
    import torch
    lib = load_library()
    st = stream if stream is not None else torch.cuda.current_stream(device)
    parts = len(recv_offset) - 1
    a = [np.ascontiguousarray(x, dtype=np.uint64) for x in (recv_offset, slots_to, outcomes_to)]
    mt = np.ascontiguousarray(marks_to, dtype=np.uint64) if marks_to is not None else None
    _check(lib.mpzch_return_scatter_device(
        device, slots.numel(), ctypes.c_void_p(slots.data_ptr()), ctypes.c_void_p(outcomes.data_ptr()),
        ctypes.c_void_p(marks.data_ptr()) if marks is not None else None, ctypes.c_void_p(src.data_ptr()),
        parts, *[x.ctypes.data_as(_u64p) for x in a], mt.ctypes.data_as(_u64p) if mt is not None else None,
        ctypes.c_void_p(st.cuda_stream)))


IPC_RECORD_BYTES = 72


def ipc_export(tensor) -> bytes:
    """CUDA IPC record of a device tensor's storage (allocation handle + offset)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(IPC_RECORD_BYTES)
    _check(lib.mpzch_ipc_export(ctypes.c_void_p(tensor.data_ptr()), buf))
    return buf.raw


def ipc_import(device: int, record: bytes) -> int:
    """Map another process's buffer; returns its device address in this process."""
    lib = load_library()
    out = ctypes.c_uint64(0)
    _check(lib.mpzch_ipc_import(device, ctypes.create_string_buffer(record, IPC_RECORD_BYTES), ctypes.byref(out)))
    return out.value


def ipc_close(addr: int):
    _check(load_library().mpzch_ipc_close(addr))


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else None


@dataclass
class TtlPolicy:
    """TtlPolicy, proj/include/mpzch/eviction.hpp:13-23."""
    default_ttl_seconds: int = 259200
    per_feature_ttl: Dict[int, int] = field(default_factory=dict)

    def ttl_for(self, feature: int) -> int:
        return self.per_feature_ttl.get(feature, self.default_ttl_seconds)

    def validate(self):  # eviction.cpp:8-18
        if self.default_ttl_seconds == 0:
            raise InvalidArgument("default TTL must be strictly positive")
        for f, t in self.per_feature_ttl.items():
            if t == 0:
                raise InvalidArgument(f"per-feature TTL must be strictly positive (feature {f})")


class EvictionPolicy:
    """EvictionPolicy, proj/include/mpzch/eviction.hpp:27-46 (mode 0/1/2 = Disabled/Ttl/Lru)."""
    DISABLED, TTL, LRU = 0, 1, 2

    def __init__(self, mode: int, ttl: Optional[TtlPolicy] = None):
        self.mode = mode
        self.ttl = ttl or TtlPolicy()
        keys = sorted(self.ttl.per_feature_ttl) if mode == self.TTL else []
        self._keys = np.array(keys, dtype=np.uint32)
        self._vals = np.array([self.ttl.per_feature_ttl[k] for k in keys], dtype=np.uint64)
        self._c = _Policy(mode, len(keys), self.ttl.default_ttl_seconds if mode == self.TTL else 0,
                          self._keys.ctypes.data_as(_u32p) if len(keys) else None,
                          self._vals.ctypes.data_as(_u64p) if len(keys) else None)

    @classmethod
    def disabled(cls):
        return cls(cls.DISABLED)

    @classmethod
    def lru(cls):
        return cls(cls.LRU)

    @classmethod
    def ttl(cls, cfg: Optional[TtlPolicy] = None, **kw):
        cfg = cfg or TtlPolicy(**kw)
        cfg.validate()
        return cls(cls.TTL, cfg)

    def meta_for(self, now: int, feature: int = 0) -> int:
        """make_metadata, proj/src/eviction.cpp:20-30."""
        if self.mode != self.TTL:
            return now
        t = self.ttl.ttl_for(feature)
        if t > (1 << 64) - 1 - now:
            raise OverflowError_("TTL expiry overflows the 64-bit timestamp range")
        return now + t


def even_capacities(total_rows: int, num_shards: int) -> list:
    """TableLayout::even, proj/src/shard_router.cpp:27-40."""
    if num_shards == 0:
        raise InvalidArgument("layout needs at least one shard")
    if total_rows < num_shards:
        raise InvalidArgument("fewer rows than shards")
    caps = [total_rows // num_shards] * num_shards
    for s in range(total_rows % num_shards):
        caps[s] += 1
    return caps


@dataclass
class TableConfig:
    """TableConfig, proj/include/mpzch/table.hpp:18-28."""
    shard_capacities: Sequence[int]
    max_probe: int = 1
    seed: int = 0
    dim: int = 0
    init_seed: int = 0

    @classmethod
    def even(cls, total_rows, num_shards, max_probe, seed, dim=0, init_seed=0):
        return cls(even_capacities(total_rows, num_shards), max_probe, seed, dim, init_seed)


class MpzchTable:
    """Device-resident MpzchTable (proj/include/mpzch/table.hpp:41-131) on one B200."""

    def __init__(self, cfg: TableConfig, device: int = 0, shard_range: Optional[Tuple[int, int]] = None):
        """shard_range=(lo, hi): row-sharded mode, hold only logical shards [lo, hi)."""
        lib = load_library()
        caps = np.ascontiguousarray(np.array(list(cfg.shard_capacities), dtype=np.uint64))
        h = _vp()
        cp = caps.ctypes.data_as(_u64p) if caps.size else None
        if shard_range is None:
            _check(lib.mpzch_table_create(cp, len(caps), cfg.max_probe, cfg.seed, cfg.dim,
                                          cfg.init_seed, device, ctypes.byref(h)))
        else:
            _check(lib.mpzch_table_create_sharded(cp, len(caps), cfg.max_probe, cfg.seed, cfg.dim,
                                                  cfg.init_seed, device, shard_range[0],
                                                  shard_range[1], ctypes.byref(h)))
        self._attach(h, lib, cfg, device, owned=True)

    @classmethod
    def _view(cls, h, cfg: TableConfig, device: int) -> "MpzchTable":
        """A non-owning wrapper of a handle another object owns (a row-sharded rank's table)."""
        t = cls.__new__(cls)
        t._attach(h, load_library(), cfg, device, owned=False)
        return t

    def _attach(self, h, lib, cfg: TableConfig, device: int, owned: bool):
        caps = np.ascontiguousarray(np.array(list(cfg.shard_capacities), dtype=np.uint64))
        self._h = h
        self._owned = owned
        self._lib = lib
        self.cfg = cfg
        self.device = device
        self.num_shards = len(caps)
        self.max_probe = cfg.max_probe
        self.dim = cfg.dim
        self.total_rows = int(lib.mpzch_total_rows(h))
        self.shard_capacities = caps.copy()
        offs = np.zeros(len(caps) + 1, dtype=np.uint64)
        _check(lib.mpzch_shard_layout(h, caps.ctypes.data_as(_u64p), offs.ctypes.data_as(_u64p)))
        self.shard_offsets = offs
        rl, rh = ctypes.c_uint64(0), ctypes.c_uint64(0)
        sl, sh = ctypes.c_uint32(0), ctypes.c_uint32(0)
        _check(lib.mpzch_held_rows(h, ctypes.byref(rl), ctypes.byref(rh), ctypes.byref(sl),
                                   ctypes.byref(sh)))
        self.row_lo, self.row_hi = rl.value, rh.value
        self.shard_lo, self.shard_hi = sl.value, sh.value
        self.held_rows = self.row_hi - self.row_lo

    def close(self):
        if getattr(self, "_h", None):
            if getattr(self, "_owned", True):
                self._lib.mpzch_table_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def has_embeddings(self) -> bool:
        return self.dim > 0

    # ---- hot path ------------------------------------------------------------------------
    def process_batch(self, ids, now: int, policy: EvictionPolicy, features=None,
                      evicted_cap: Optional[int] = None, out_slots=None, out_outcomes=None,
                      out_evicted=None) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """process_batch (batch_engine.cpp:141-221) on host buffers.

        Returns (slots u64[n] global rows, outcomes u8[n], evicted u64[k]) where evicted is the
        canonical evicted list (first-occurrence order, with multiplicity).  Output arrays may
        be supplied (e.g. page-locked) to avoid allocation."""
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        n = ids.size
        feats = None if features is None else np.ascontiguousarray(features, dtype=np.uint32)
        if feats is not None and feats.size != n:
            raise InvalidArgument("features must pair 1:1 with ids")
        slots = np.empty(n, dtype=np.uint64) if out_slots is None else out_slots
        oc = np.empty(n, dtype=np.uint8) if out_outcomes is None else out_outcomes
        assert slots.size >= n and oc.size >= n and slots.dtype == np.uint64 and oc.dtype == np.uint8
        cap = n if evicted_cap is None else evicted_cap
        ev = np.empty(max(cap, 1), dtype=np.uint64) if out_evicted is None else out_evicted
        cap = min(cap, ev.size)
        nev = ctypes.c_uint64(0)
        _check(self._lib.mpzch_process_batch(self._h, _ptr(ids), _ptr(feats), n, now,
                                             ctypes.byref(policy._c), _ptr(slots), _ptr(oc),
                                             _ptr(ev), cap, ctypes.byref(nev)))
        return slots[:n], oc[:n], ev[:min(nev.value, cap)].copy()

    def process_batch_device(self, ids, now: int, policy: EvictionPolicy, features=None,
                             out_slots=None, out_outcomes=None, out_evicted=None, stream=None):
        """process_batch on device tensors (torch, on this table's device).  Returns the
        evicted-list length; results land in out_slots / out_outcomes / out_evicted."""
        import torch
        n = ids.numel()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        nev = ctypes.c_uint64(0)
        _check(self._lib.mpzch_process_batch_device(
            self._h, ctypes.c_void_p(ids.data_ptr()),
            ctypes.c_void_p(features.data_ptr()) if features is not None else None, n, now,
            ctypes.byref(policy._c), ctypes.c_void_p(out_slots.data_ptr()),
            ctypes.c_void_p(out_outcomes.data_ptr()),
            ctypes.c_void_p(out_evicted.data_ptr()) if out_evicted is not None else None,
            out_evicted.numel() if out_evicted is not None else 0, ctypes.byref(nev),
            ctypes.c_void_p(st.cuda_stream)))
        return nev.value

    # ---- row-sharded helpers (device tensors) ------------------------------------------
    def validate_device(self, ids, stream=None) -> Optional[int]:
        """First invalid position of a device id tensor, or None."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        bad = ctypes.c_uint64(0)
        _check(self._lib.mpzch_validate_device(self._h, ctypes.c_void_p(ids.data_ptr()), ids.numel(),
                                               ctypes.byref(bad), ctypes.c_void_p(st.cuda_stream)))
        return None if bad.value == (1 << 64) - 1 else bad.value

    def route_device(self, ids, shard_to_part, parts: int, stream=None):
        """(perm int32 device tensor, counts list): positions grouped by owning part, stable."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        perm = torch.empty(ids.numel(), dtype=torch.int32, device=ids.device)
        s2p = np.ascontiguousarray(shard_to_part, dtype=np.uint32)
        counts = np.zeros(parts, dtype=np.uint64)
        _check(self._lib.mpzch_route_device(self._h, ctypes.c_void_p(ids.data_ptr()), ids.numel(),
                                            s2p.ctypes.data_as(_u32p), parts,
                                            ctypes.c_void_p(perm.data_ptr()),
                                            counts.ctypes.data_as(_u64p),
                                            ctypes.c_void_p(st.cuda_stream)))
        return perm, [int(c) for c in counts]

    def route_count_device(self, ids, shard_to_part, parts: int, stream=None):
        """Per-part counts of this rank's positions (count + scan of route_device); arms
        route_scatter_device for the same ids."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        s2p = np.ascontiguousarray(shard_to_part, dtype=np.uint32)
        counts = np.zeros(parts, dtype=np.uint64)
        _check(self._lib.mpzch_route_count_device(self._h, ctypes.c_void_p(ids.data_ptr()), ids.numel(),
                                                  s2p.ctypes.data_as(_u32p), parts,
                                                  counts.ctypes.data_as(_u64p), ctypes.c_void_p(st.cuda_stream)))
        return [int(c) for c in counts]

    def route_scatter_device(self, ids, features, parts: int, ids_to, features_to, src_to, offset,
                             stream=None):
        """Partition + store into the owners' receive buffers (device addresses per part)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        a = [np.ascontiguousarray(x, dtype=np.uint64) for x in (ids_to, features_to or [0] * parts, src_to, offset)]
        _check(self._lib.mpzch_route_scatter_device(
            self._h, ctypes.c_void_p(ids.data_ptr()),
            ctypes.c_void_p(features.data_ptr()) if features is not None else None, ids.numel(), parts,
            *[x.ctypes.data_as(_u64p) for x in a], ctypes.c_void_p(st.cuda_stream)))

    def process_batch_device_marked(self, ids, now: int, policy: EvictionPolicy, features=None,
                                    stream=None):
        """(slots, outcomes, first_evicted_marks) device tensors for device ids."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        n = ids.numel()
        slots = torch.empty(n, dtype=torch.int64, device=ids.device)
        oc = torch.empty(n, dtype=torch.uint8, device=ids.device)
        mark = torch.empty(n, dtype=torch.uint8, device=ids.device)
        nev = ctypes.c_uint64(0)
        _check(self._lib.mpzch_process_batch_device_marked(
            self._h, ctypes.c_void_p(ids.data_ptr()),
            ctypes.c_void_p(features.data_ptr()) if features is not None else None, n, now,
            ctypes.byref(policy._c), ctypes.c_void_p(slots.data_ptr()), ctypes.c_void_p(oc.data_ptr()),
            ctypes.c_void_p(mark.data_ptr()) if n else None, ctypes.byref(nev),
            ctypes.c_void_p(st.cuda_stream)))
        return slots, oc, mark

    def process_batch_device_async(self, ids, now: int, policy: EvictionPolicy, features=None,
                                   out_slots=None, out_outcomes=None, out_evicted=None,
                                   stream=None) -> int:
        """Enqueue process_batch on device tensors and return a ticket (see wait)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        tk = ctypes.c_uint64(0)
        _check(self._lib.mpzch_process_batch_device_async(
            self._h, ctypes.c_void_p(ids.data_ptr()),
            ctypes.c_void_p(features.data_ptr()) if features is not None else None, ids.numel(), now,
            ctypes.byref(policy._c), ctypes.c_void_p(out_slots.data_ptr()),
            ctypes.c_void_p(out_outcomes.data_ptr()),
            ctypes.c_void_p(out_evicted.data_ptr()) if out_evicted is not None else None,
            out_evicted.numel() if out_evicted is not None else 0, ctypes.c_void_p(st.cuda_stream),
            ctypes.byref(tk)))
        return tk.value

    def wait(self, ticket: int) -> int:
        """Block until the ticket's batch is done; raise its error; return its evicted count."""
        nev = ctypes.c_uint64(0)
        _check(self._lib.mpzch_batch_wait(self._h, ticket, ctypes.byref(nev)))
        return nev.value

    def lookup(self, ids) -> Tuple[np.ndarray, np.ndarray]:
        """Batched MpzchTable::lookup (table.cpp:150-156): (slots, outcomes), no writes."""
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        slots = np.empty(ids.size, dtype=np.uint64)
        oc = np.empty(ids.size, dtype=np.uint8)
        _check(self._lib.mpzch_lookup(self._h, _ptr(ids), ids.size, _ptr(slots), _ptr(oc)))
        return slots, oc

    def lookup_device(self, ids, out_slots, out_outcomes, stream=None):
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.mpzch_lookup_device(self._h, ctypes.c_void_p(ids.data_ptr()), ids.numel(),
                                             ctypes.c_void_p(out_slots.data_ptr()),
                                             ctypes.c_void_p(out_outcomes.data_ptr()),
                                             ctypes.c_void_p(st.cuda_stream)))

    def lookup_device_async(self, ids, out_slots, out_outcomes, stream=None) -> int:
        """Enqueue a batched lookup on device tensors; returns a ticket (see wait)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        tk = ctypes.c_uint64(0)
        _check(self._lib.mpzch_lookup_device_async(self._h, ctypes.c_void_p(ids.data_ptr()), ids.numel(),
                                                   ctypes.c_void_p(out_slots.data_ptr()),
                                                   ctypes.c_void_p(out_outcomes.data_ptr()),
                                                   ctypes.c_void_p(st.cuda_stream), ctypes.byref(tk)))
        return tk.value

    def lookup_or_insert(self, id: int, feature: int, now: int, policy: EvictionPolicy):
        """MpzchTable::lookup_or_insert (table.cpp:98-110): (global slot, outcome)."""
        slot = ctypes.c_uint64(0)
        oc = ctypes.c_uint8(0)
        _check(self._lib.mpzch_lookup_or_insert(self._h, id, feature, now, ctypes.byref(policy._c),
                                                ctypes.byref(slot), ctypes.byref(oc)))
        return slot.value, oc.value

    # ---- state (parity) ------------------------------------------------------------------
    def process_shard_batch(self, shard: int, ids, metas, now: int, policy: EvictionPolicy):
        """MpzchTable::process_shard_batch (table.cpp:112-148): shard's positions in order, each
        with its own metadata word.  Returns (slots, outcomes); on a bad metadata word the
        exception carries .partial = the results of the positions before it; on an invalid id,
        the results of the 256-position chunks before its chunk (the reference hoists the
        validating home_slot over each chunk, table.cpp:129-133)."""
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        metas = np.ascontiguousarray(metas, dtype=np.uint64)
        if metas.size != ids.size:
            raise InvalidArgument("batch spans disagree on length")
        slots = np.zeros(ids.size, dtype=np.uint64)
        oc = np.full(ids.size, 0xff, dtype=np.uint8)
        rc = self._lib.mpzch_process_shard_batch(self._h, shard, _ptr(ids), _ptr(metas), ids.size,
                                                 now, ctypes.byref(policy._c), _ptr(slots), _ptr(oc))
        if rc:
            k = int(np.argmax(oc == 0xff)) if (oc == 0xff).any() else ids.size
            try:
                _check(rc)
            except MpzchError as e:
                e.partial = (slots[:k], oc[:k])
                raise
        return slots, oc

    def reset_row(self, row: int):
        """MpzchTable::reset_row (table.cpp:181-186)."""
        _check(self._lib.mpzch_reset_row(self._h, row))

    def state_equals(self, other: "MpzchTable") -> bool:
        """MpzchTable::state_equals (table.cpp:249-260), compared on the device."""
        v = ctypes.c_int(0)
        _check(self._lib.mpzch_state_equals(self._h, other._h, ctypes.byref(v)))
        return bool(v.value)

    def row_identity(self, row: int) -> int:
        v = ctypes.c_uint64(0)
        _check(self._lib.mpzch_read_identity(self._h, row, ctypes.byref(v)))
        return v.value

    def gather(self, rows) -> np.ndarray:
        """MpzchTable::gather (table.cpp:158-163): one gather kernel, one copy."""
        r = np.ascontiguousarray(rows, dtype=np.uint64)
        out = np.empty((r.size, max(self.dim, 1)), dtype=np.float32)
        _check(self._lib.mpzch_gather(self._h, _ptr(r), r.size, _ptr(out)))
        return out

    def shard_config(self, shard: int) -> dict:
        cap, P, seed = ctypes.c_uint64(0), ctypes.c_uint32(0), ctypes.c_uint64(0)
        _check(self._lib.mpzch_shard_config(self._h, shard, ctypes.byref(cap), ctypes.byref(P),
                                            ctypes.byref(seed)))
        return {"capacity": cap.value, "max_probe": P.value, "shard_id": shard, "seed": seed.value}

    def identities_all(self) -> np.ndarray:
        """identity words of the held rows [row_lo, row_hi) (all rows unless sharded)."""
        out = np.empty(self.held_rows, dtype=np.uint64)
        _check(self._lib.mpzch_copy_identities(self._h, _ptr(out)))
        return out

    def metadata_all(self) -> np.ndarray:
        out = np.empty(self.held_rows, dtype=np.uint64)
        _check(self._lib.mpzch_copy_metadata(self._h, _ptr(out)))
        return out

    def identities(self, shard: int) -> np.ndarray:
        self._check_shard(shard)
        a, b = int(self.shard_offsets[shard]) - self.row_lo, int(self.shard_offsets[shard + 1]) - self.row_lo
        return self.identities_all()[a:b]

    def metadata(self, shard: int) -> np.ndarray:
        self._check_shard(shard)
        a, b = int(self.shard_offsets[shard]) - self.row_lo, int(self.shard_offsets[shard + 1]) - self.row_lo
        return self.metadata_all()[a:b]

    def _check_shard(self, shard):
        if shard < 0 or shard >= self.num_shards:
            raise OutOfRange("shard index out of range")
        if shard < self.shard_lo or shard >= self.shard_hi:
            raise OutOfRange("shard is not held by this handle")

    def weights(self, row0: Optional[int] = None, nrows: Optional[int] = None) -> np.ndarray:
        row0 = self.row_lo if row0 is None else row0
        nrows = self.row_hi - row0 if nrows is None else nrows
        out = np.empty((nrows, max(self.dim, 1)), dtype=np.float32)
        _check(self._lib.mpzch_copy_weights(self._h, row0, nrows, _ptr(out)))
        return out

    def momentum(self, row0: Optional[int] = None, nrows: Optional[int] = None) -> np.ndarray:
        row0 = self.row_lo if row0 is None else row0
        nrows = self.row_hi - row0 if nrows is None else nrows
        out = np.empty((nrows, max(self.dim, 1)), dtype=np.float32)
        _check(self._lib.mpzch_copy_momentum(self._h, row0, nrows, _ptr(out)))
        return out

    def trained(self) -> np.ndarray:
        out = np.empty(self.held_rows, dtype=np.uint8)
        _check(self._lib.mpzch_copy_trained(self._h, _ptr(out)))
        return out

    def row_generation(self) -> np.ndarray:
        out = np.empty(self.held_rows, dtype=np.uint64)
        _check(self._lib.mpzch_copy_row_generation(self._h, _ptr(out)))
        return out

    def device_arrays(self):
        """(identity, metadata, weights) device pointers as ints."""
        a, b, c = _vp(), _vp(), _vp()
        _check(self._lib.mpzch_device_arrays(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def write_slots(self, shard: int, local_slots, identities, metadata=None):
        s = np.ascontiguousarray(local_slots, dtype=np.uint64)
        i = np.ascontiguousarray(identities, dtype=np.uint64)
        m = None if metadata is None else np.ascontiguousarray(metadata, dtype=np.uint64)
        _check(self._lib.mpzch_write_slots(self._h, shard, _ptr(s), _ptr(i), _ptr(m), s.size))

    def check_hole_free(self) -> bool:
        v = ctypes.c_int(0)
        _check(self._lib.mpzch_check_hole_free(self._h, ctypes.byref(v)))
        return bool(v.value)

    def write_row(self, row: int, weights=None, momentum=None, trained: int = 1):
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float32)
        m = None if momentum is None else np.ascontiguousarray(momentum, dtype=np.float32)
        _check(self._lib.mpzch_write_row(self._h, row, _ptr(w), _ptr(m), trained))

    def sgd_step(self, rows, grads, lr: float, beta: float):
        """MpzchTable::sgd_step (table.cpp:174-179) with host arrays: rows[n], grads[n, dim]."""
        r = np.ascontiguousarray(rows, dtype=np.uint64)
        g = np.ascontiguousarray(grads, dtype=np.float32).reshape(-1)
        _check(self._lib.mpzch_sgd_step(self._h, _ptr(r), r.size, _ptr(g), g.size, lr, beta))

    def sgd_step_device(self, rows, grads, lr: float, beta: float, stream=None):
        """sgd_step on device tensors (rows int64 [n], grads float32 [n, dim]), stream-ordered."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        g = grads.contiguous()
        _check(self._lib.mpzch_sgd_step_device(
            self._h, ctypes.c_void_p(rows.data_ptr()), rows.numel(), ctypes.c_void_p(g.data_ptr()),
            g.numel(), lr, beta, ctypes.c_void_p(st.cuda_stream)))

    def lookup_gather_device(self, ids, stream=None, out=None):
        """Fused lookup + gather: (slots, outcomes, rows[n, dim]) device tensors (out: a
        preallocated (slots, outcomes, rows) triple to fill instead)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        n = ids.numel()
        if out is not None:
            slots, oc, rows = out
        else:
            slots = torch.empty(n, dtype=torch.int64, device=ids.device)
            oc = torch.empty(n, dtype=torch.uint8, device=ids.device)
            rows = torch.empty((n, self.dim), dtype=torch.float32, device=ids.device)
        _check(self._lib.mpzch_lookup_gather_device(
            self._h, ctypes.c_void_p(ids.data_ptr()), n, ctypes.c_void_p(slots.data_ptr()),
            ctypes.c_void_p(oc.data_ptr()), ctypes.c_void_p(rows.data_ptr()),
            ctypes.c_void_p(st.cuda_stream)))
        return slots, oc, rows

    def delta_cut(self, cursor: int):
        """DeltaSource::cut (publish.cpp:288-305) on device: (rows, identities, weights[k, dim],
        next_cursor)."""
        cap = self.held_rows
        rows = np.empty(cap, dtype=np.uint64)
        ids = np.empty(cap, dtype=np.uint64)
        w = np.empty((cap, max(self.dim, 1)), dtype=np.float32)
        n = ctypes.c_uint64(0)
        nxt = ctypes.c_uint64(0)
        _check(self._lib.mpzch_delta_cut(self._h, cursor, _ptr(rows), _ptr(ids), _ptr(w), cap,
                                         ctypes.byref(n), ctypes.byref(nxt)))
        k = n.value
        return rows[:k].copy(), ids[:k].copy(), w[:k].copy(), nxt.value

    def make_cursor(self) -> int:
        g = ctypes.c_uint64(0)
        _check(self._lib.mpzch_make_cursor(self._h, ctypes.byref(g)))
        return g.value

    def dirty_rows_since(self, cursor: int) -> np.ndarray:
        out = np.empty(self.held_rows, dtype=np.uint64)
        n = ctypes.c_uint64(0)
        _check(self._lib.mpzch_dirty_rows_since(self._h, cursor, _ptr(out), out.size, ctypes.byref(n)))
        return out[:n.value].copy()

    def set_path(self, path: str):
        _check(self._lib.mpzch_set_path(self._h, {"auto": 0, "ordered": 1, "rounds": 2}[path]))

    def set_reset_mode(self, mode: str):
        """'eager' (default: the batch writes every evicted row, as the reference does) or
        'deferred' (evicted rows are marked reset-pending; the next sgd_step of a row starts
        from the closed-form draw_row without reading it; gathers draw pending rows; every
        other reader flushes first -- observable state identical to 'eager')."""
        _check(self._lib.mpzch_set_reset_mode(self._h, {"eager": 0, "deferred": 1}[mode]))

    def flush_resets(self):
        _check(self._lib.mpzch_flush_resets(self._h))

    def last_stats(self) -> dict:
        s = _Stats()
        _check(self._lib.mpzch_last_stats(self._h, ctypes.byref(s)))
        d = {k: getattr(s, k) for k, _ in _Stats._fields_}
        d["path"] = {0: "fast", 1: "ordered", 2: "rounds"}[s.path]
        return d

    def set_profiling(self, on: bool = True):
        """CUDA events on the launch stream around the probe kernel / claims / whole batch."""
        _check(self._lib.mpzch_set_profiling(self._h, int(on)))

    def profile(self) -> dict:
        p = _Profile()
        _check(self._lib.mpzch_get_profile(self._h, ctypes.byref(p)))
        return {k: getattr(p, k) for k, _ in _Profile._fields_}

    def kernel_launches(self) -> int:
        return int(self._lib.mpzch_kernel_launches(self._h))

    def serialize_snapshot_into(self, out) -> int:
        """serialize_snapshot into a caller buffer (e.g. page-locked uint8 numpy); returns the
        image length.  The buffer must hold snapshot_size() bytes."""
        n = ctypes.c_uint64(0)
        _check(self._lib.mpzch_serialize_snapshot(self._h, _ptr(out), out.size, ctypes.byref(n)))
        return n.value

    def snapshot_size(self) -> int:
        n = ctypes.c_uint64(0)
        _check(self._lib.mpzch_serialize_snapshot(self._h, None, 0, ctypes.byref(n)))
        return n.value

    def serialize_snapshot(self) -> bytes:
        """serialize_snapshot (publish.cpp:126-155): the .mpzc image, CRC-32 on the device."""
        n = ctypes.c_uint64(0)
        _check(self._lib.mpzch_serialize_snapshot(self._h, None, 0, ctypes.byref(n)))
        out = np.empty(n.value, np.uint8)
        _check(self._lib.mpzch_serialize_snapshot(self._h, _ptr(out), out.size, ctypes.byref(n)))
        return out.tobytes()


class DeltaSource:
    """DeltaSource (proj/include/mpzch/publish.hpp:69-82): takes a cursor now; each cut()
    returns the serialized .mpzd log of the rows dirtied since the previous cut (records packed
    and checksummed on the device)."""

    def __init__(self, table: MpzchTable, base_checksum: int):
        if table.dim == 0:
            raise LogicError("index-only tables (dim = 0) cannot be published")
        self.table = table
        self.base_checksum = base_checksum
        self.sequence = 0
        self.cursor = table.make_cursor()

    def cut(self) -> bytes:
        t = self.table
        n, nxt = ctypes.c_uint64(0), ctypes.c_uint64(0)
        _check(t._lib.mpzch_serialize_delta(t._h, self.cursor, self.base_checksum, self.sequence,
                                            None, 0, ctypes.byref(n), ctypes.byref(nxt)))
        out = np.empty(n.value, np.uint8)
        _check(t._lib.mpzch_serialize_delta(t._h, self.cursor, self.base_checksum, self.sequence,
                                            _ptr(out), out.size, ctypes.byref(n), ctypes.byref(nxt)))
        self.cursor = nxt.value
        self.sequence += 1
        return out.tobytes()


def snapshot_checksum(image: bytes) -> int:
    """snapshot_checksum (publish.cpp:157-162): the trailer CRC, the lineage id."""
    if len(image) < 4:
        raise ValueError("truncated file")
    return int.from_bytes(image[-4:], "little")


def crc32_device(t) -> int:
    """crc32 (publish.cpp:110-124) of a CUDA tensor's bytes, computed on the device."""
    import torch
    c = ctypes.c_uint32(0)
    st = torch.cuda.current_stream(t.device)
    _check(load_library().mpzch_crc32_device(ctypes.c_void_p(t.data_ptr()),
                                             t.numel() * t.element_size(), ctypes.byref(c),
                                             ctypes.c_void_p(st.cuda_stream)))
    return c.value


SHARDED_RECORD_BYTES = 128


class ShardedRank:
    """One rank of a row-sharded table with the device-side protocol (mpzch_sharded_*):
    rank r of `world` holds the logical shards {s : s*world//S == r}; every process_batch is a
    collective over the ranks (each passes its contiguous slice of the global batch, slices in
    rank order), enqueued on the stream with one host wait.  Returns this slice's slots and
    outcomes and the GLOBAL canonical evicted list (identical on every rank).  Errors are raised
    on every rank with the reference's text (the GLOBAL position of the first invalid id)."""

    def __init__(self, cfg: TableConfig, rank: int, world: int, max_batch: int, device: int = 0):
        lib = load_library()
        caps = np.ascontiguousarray(np.array(list(cfg.shard_capacities), dtype=np.uint64))
        h = _vp()
        _check(lib.mpzch_sharded_create(caps.ctypes.data_as(_u64p), len(caps), cfg.max_probe, cfg.seed,
                                        cfg.dim, cfg.init_seed, device, rank, world, max_batch,
                                        ctypes.byref(h)))
        self._h, self._lib = h, lib
        self.rank, self.world, self.device, self.max_batch = rank, world, device, max_batch
        self.cfg = cfg
        self.table = MpzchTable._view(_vp(lib.mpzch_sharded_table(h)), cfg, device)

    def close(self):
        if getattr(self, "_h", None):
            self.table._h = None
            self._lib.mpzch_sharded_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self) -> bytes:
        buf = (ctypes.c_uint8 * SHARDED_RECORD_BYTES)()
        _check(self._lib.mpzch_sharded_export(self._h, buf))
        return bytes(buf)

    def connect_ipc(self, records):
        """records: every rank's export() in rank order (gathered by any host channel)."""
        blob = b"".join(records)
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(self._lib.mpzch_sharded_connect_ipc(self._h, buf))

    @staticmethod
    def connect_local(ranks):
        arr = (_vp * len(ranks))(*[r._h for r in ranks])
        _check(load_library().mpzch_sharded_connect_local(arr, len(ranks)))

    def process_batch_device_async(self, ids, now: int, policy: EvictionPolicy, features=None,
                                   out_slots=None, out_outcomes=None, out_evicted=None, stream=None) -> int:
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        tk = ctypes.c_uint64(0)
        _check(self._lib.mpzch_sharded_process_batch_async(
            self._h, ctypes.c_void_p(ids.data_ptr()),
            ctypes.c_void_p(features.data_ptr()) if features is not None else None, ids.numel(), now,
            ctypes.byref(policy._c), ctypes.c_void_p(out_slots.data_ptr()),
            ctypes.c_void_p(out_outcomes.data_ptr()),
            ctypes.c_void_p(out_evicted.data_ptr()) if out_evicted is not None else None,
            out_evicted.numel() if out_evicted is not None else 0, ctypes.c_void_p(st.cuda_stream),
            ctypes.byref(tk)))
        return tk.value

    def wait(self, ticket: int) -> int:
        nev = ctypes.c_uint64(0)
        _check(self._lib.mpzch_sharded_wait(self._h, ticket, ctypes.byref(nev)))
        return nev.value

    def process_batch_device(self, ids, now: int, policy: EvictionPolicy, features=None, out_slots=None,
                             out_outcomes=None, out_evicted=None, stream=None) -> int:
        return self.wait(self.process_batch_device_async(ids, now, policy, features, out_slots,
                                                         out_outcomes, out_evicted, stream))

    def process_batch(self, ids, now: int, policy: EvictionPolicy, features=None):
        """Host arrays in, host arrays out: (slots, outcomes, global evicted list)."""
        import torch
        dev = f"cuda:{self.device}"
        n = int(np.asarray(ids).size)
        ids_t = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.uint64).view(np.int64)).to(dev)
        f_t = None if features is None else torch.from_numpy(
            np.ascontiguousarray(features, dtype=np.uint32).view(np.int32)).to(dev)
        s_t = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        o_t = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        e_t = torch.empty(self.max_batch, dtype=torch.int64, device=dev)
        k = self.process_batch_device(ids_t, now, policy, f_t, s_t, o_t, e_t)
        return (s_t[:n].cpu().numpy().view(np.uint64), o_t[:n].cpu().numpy(),
                e_t[:min(k, self.max_batch)].cpu().numpy().view(np.uint64))

    def last_stats(self) -> dict:
        s = _Stats()
        hw = ctypes.c_int(0)
        _check(self._lib.mpzch_sharded_last_stats(self._h, ctypes.byref(s), ctypes.byref(hw)))
        d = {f: getattr(s, f) for f, _ in _Stats._fields_}
        d["host_waits"] = hw.value
        return d


def crc32_device_ptr(ptr: int, nbytes: int) -> int:
    """crc32 of `nbytes` device bytes at a raw device address (e.g. from device_arrays())."""
    c = ctypes.c_uint32(0)
    _check(load_library().mpzch_crc32_device(ctypes.c_void_p(ptr), nbytes, ctypes.byref(c), None))
    return c.value


def parse_delta(image: bytes) -> dict:
    """parse_delta (publish.cpp:232-252) on the host: header fields and records
    (rows, identities, weights[k, dim]); raises ValueError on a malformed image."""
    import struct
    import zlib
    if len(image) < 36 or image[:4] != b"MPZD":
        raise ValueError("bad magic; not a delta file")
    ver, base, seq, dim, count = struct.unpack_from("<IIQIQ", image, 4)
    rec = 16 + 4 * dim
    if ver != 1 or dim == 0 or len(image) != 36 + count * rec:
        raise ValueError("malformed delta")
    if int.from_bytes(image[-4:], "little") != zlib.crc32(image[:-4]):
        raise ValueError("checksum failure")
    body = np.frombuffer(image, np.uint8, count * rec, 32).reshape(count, rec)
    return dict(base_checksum=base, sequence=seq, dim=dim,
                rows=body[:, :8].copy().view(np.uint64).reshape(-1),
                identities=body[:, 8:16].copy().view(np.uint64).reshape(-1),
                weights=body[:, 16:].copy().view(np.float32).reshape(count, dim))


def dedup(ids, features=None, device: int = 0):
    """dedup (batch_engine.cpp:79-108, 133-139) on `device`: (unique ids, unique features,
    inverse u32[n]) in first-occurrence order of (id, feature)."""
    lib = load_library()
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    n = ids.size
    f = None if features is None else np.ascontiguousarray(features, dtype=np.uint32)
    uids = np.empty(max(n, 1), dtype=np.uint64)
    uf = np.empty(max(n, 1), dtype=np.uint32)
    inv = np.empty(max(n, 1), dtype=np.uint32)
    u = ctypes.c_uint64(0)
    _check(lib.mpzch_dedup(device, _ptr(ids), _ptr(f), n, _ptr(uids), _ptr(uf), _ptr(inv), ctypes.byref(u)))
    return uids[:u.value].copy(), uf[:u.value].copy(), inv[:n].copy()


def process_batch(table: MpzchTable, ids, now: int, policy: EvictionPolicy, features=None):
    """Free-function spelling of the reference's process_batch (batch_engine.hpp:44-46)."""
    return table.process_batch(ids, now, policy, features)


def build_info() -> str:
    return load_library().mpzch_build_info().decode()
