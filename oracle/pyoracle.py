"""pyoracle -- ctypes face of the CPU parity checkers.  TEST INFRASTRUCTURE ONLY.

Two interchangeable backends with one Python interface:

* ``kind="port"``      -> oracle/build/libmpzch_oracle.so, the plain-C restatement
                          (oracle/mpzch_oracle.c, every function cites its reference line);
* ``kind="reference"`` -> oracle/_ref/libmpzch_ref.so, the reference library itself,
                          compiled from /root/reference/proj/src by oracle/Makefile.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "build", "libmpzch_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libmpzch_ref.so")

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p

_LIBS = {}

EXC = {1: ValueError, 2: OverflowError, 3: ValueError, 4: RuntimeError, 5: IndexError, 7: MemoryError}


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code
        self.msg = msg


def build():
    """Compile the restatement (and the reference when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def available(kind: str) -> bool:
    return os.path.exists(REF_LIB if kind == "reference" else PORT_LIB)


def lib(kind: str = "port"):
    if kind in _LIBS:
        return _LIBS[kind]
    path = REF_LIB if kind == "reference" else PORT_LIB
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
    L = ctypes.CDLL(path)
    p = "ref_" if kind == "reference" else "orc_"
    sig = {
        "mix64": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint64]),
        "distinct_id_at": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint64]),
        "distinct_ids": (None, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _vp]),
        "home_slot": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]),
        "shard_of": (ctypes.c_uint32, [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]),
        "table_create": (ctypes.c_int, [_u64p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                        ctypes.c_uint32, ctypes.c_uint64, ctypes.POINTER(_vp)]),
        "table_destroy": (None, [_vp]),
        "total_rows": (ctypes.c_uint64, [_vp]),
        "shard_offset": (ctypes.c_uint64, [_vp, ctypes.c_uint32]),
        "process_batch": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, _vp, _vp,
                                         _vp, _vp, _vp, ctypes.c_uint64, _u64p]),
        "lookup": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp, _vp]),
        "lookup_or_insert": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                            ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, _vp,
                                            _vp, _u64p, _u8p]),
        "probe": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _vp, _vp,
                                 ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                                 _u64p, _u8p]),
        "probe_readonly": (ctypes.c_int, [ctypes.c_uint64, _vp, ctypes.c_uint64, ctypes.c_uint32,
                                          ctypes.c_uint64, _u64p, _u8p]),
        "copy_identities": (None, [_vp, _vp]),
        "copy_metadata": (None, [_vp, _vp]),
        "copy_weights": (None, [_vp, _vp]),
        "copy_momentum": (None, [_vp, _vp]),
        "copy_trained": (None, [_vp, _vp]),
        "make_cursor": (ctypes.c_uint64, [_vp]),
        "sgd_step": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp, ctypes.c_uint64, ctypes.c_float,
                                    ctypes.c_float]),
        "dirty_rows_since": (ctypes.c_int, [_vp, ctypes.c_uint64, _vp, ctypes.c_uint64, _u64p]),
        "last_error": (ctypes.c_char_p, []),
        "crc32": (ctypes.c_uint32, [_vp, ctypes.c_uint64]),
        "serialize_snapshot": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _u64p]),
    }
    if kind == "port":
        sig["serialize_delta"] = (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint32,
                                                 ctypes.c_uint64, _vp, ctypes.c_uint64, _u64p, _u64p])
        sig["draw_row"] = (None, [_vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64])
        sig["draw_rows"] = (None, [_vp, ctypes.c_uint32, _vp, ctypes.c_uint64, ctypes.c_uint64])
        sig["splitmix_next"] = (ctypes.c_uint64, [_u64p])
    else:
        sig["delta_source_create"] = (ctypes.c_int, [_vp, ctypes.c_uint32])
        sig["delta_source_cut"] = (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _u64p])
        sig["set_threads"] = (None, [ctypes.c_int])
        sig["max_threads"] = (ctypes.c_int, [])
        sig["process_batch_timed"] = (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, ctypes.c_uint64, _vp,
                                                     _vp, ctypes.POINTER(ctypes.c_double)])
        sig["prefill_distinct"] = (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_uint64,
                                                  ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                                  ctypes.c_int, ctypes.c_uint64])
    fns = {}
    for name, (res, args) in sig.items():
        f = getattr(L, p + name)
        f.restype = res
        f.argtypes = args
        fns[name] = f
    _LIBS[kind] = fns
    return fns


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else None


def _raise(L, rc):
    if rc:
        raise OracleError(rc, L["last_error"]().decode())


def policy_args(mode, default_ttl=0, per_feature=None):
    per_feature = per_feature or {}
    keys = np.array(sorted(per_feature), dtype=np.uint32)
    vals = np.array([per_feature[k] for k in sorted(per_feature)], dtype=np.uint64)
    return mode, default_ttl, keys, vals


def distinct_ids(seed: int, start: int, count: int, kind="port") -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib(kind)["distinct_ids"](seed, start, count, _ptr(out))
    return out


class OracleTable:
    """The reference MpzchTable (kind="reference") or its C restatement (kind="port")."""

    def __init__(self, caps, max_probe, seed, dim=0, init_seed=0, kind="port"):
        self.L = lib(kind)
        self.kind = kind
        c = np.ascontiguousarray(np.array(list(caps), dtype=np.uint64))
        h = _vp()
        _raise(self.L, self.L["table_create"](c.ctypes.data_as(_u64p) if c.size else None, len(c),
                                              max_probe, seed, dim, init_seed, ctypes.byref(h)))
        self.h = h
        self.dim = dim
        self.caps = c
        self.total_rows = int(self.L["total_rows"](h))
        self.offsets = np.array([self.L["shard_offset"](h, s) for s in range(len(c))] +
                                [self.total_rows], dtype=np.uint64)

    def __del__(self):
        try:
            if self.h:
                self.L["table_destroy"](self.h)
        except Exception:
            pass

    def process_batch(self, ids, now, mode=0, default_ttl=0, per_feature=None, features=None):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        n = ids.size
        f = None if features is None else np.ascontiguousarray(features, dtype=np.uint32)
        _, dt, keys, vals = policy_args(mode, default_ttl, per_feature)
        slots = np.empty(n, dtype=np.uint64)
        oc = np.empty(n, dtype=np.uint8)
        ev = np.empty(max(n, 1), dtype=np.uint64)
        nev = ctypes.c_uint64(0)
        _raise(self.L, self.L["process_batch"](self.h, _ptr(ids), _ptr(f), n, now, mode, dt,
                                               keys.size, _ptr(keys), _ptr(vals), _ptr(slots),
                                               _ptr(oc), _ptr(ev), n, ctypes.byref(nev)))
        return slots, oc, ev[:nev.value].copy()

    def process_batch_timed(self, ids, now, want_results=False):
        """Disabled process_batch with steady_clock around the call alone (reference only,
        proj/src/experiments.cpp:339-347).  Returns (seconds, slots, outcomes)."""
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        slots = np.empty(ids.size, dtype=np.uint64) if want_results else None
        oc = np.empty(ids.size, dtype=np.uint8) if want_results else None
        sec = ctypes.c_double(0)
        _raise(self.L, self.L["process_batch_timed"](self.h, _ptr(ids), ids.size, now, _ptr(slots),
                                                     _ptr(oc), ctypes.byref(sec)))
        return sec.value, slots, oc

    def prefill_distinct(self, id_seed, start, count, now, chunk=1 << 24, mode=0, default_ttl=0):
        """DistinctIdStream(id_seed).at([start, start+count)) at `now` under the policy (mode 0
        Disabled, 1 TTL with default_ttl, 2 LRU; feature 0), through process_shard_batch with the
        shards in parallel (reference only)."""
        _raise(self.L, self.L["prefill_distinct"](self.h, id_seed, start, count, now, chunk, mode,
                                                  default_ttl))

    def lookup(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        slots = np.empty(ids.size, dtype=np.uint64)
        oc = np.empty(ids.size, dtype=np.uint8)
        _raise(self.L, self.L["lookup"](self.h, _ptr(ids), ids.size, _ptr(slots), _ptr(oc)))
        return slots, oc

    def lookup_or_insert(self, id, feature, now, mode=0, default_ttl=0, per_feature=None):
        _, dt, keys, vals = policy_args(mode, default_ttl, per_feature)
        s = ctypes.c_uint64(0)
        o = ctypes.c_uint8(0)
        _raise(self.L, self.L["lookup_or_insert"](self.h, id, feature, now, mode, dt, keys.size,
                                                  _ptr(keys), _ptr(vals), ctypes.byref(s),
                                                  ctypes.byref(o)))
        return s.value, o.value

    def identities_all(self):
        out = np.empty(self.total_rows, dtype=np.uint64)
        self.L["copy_identities"](self.h, _ptr(out))
        return out

    def metadata_all(self):
        out = np.empty(self.total_rows, dtype=np.uint64)
        self.L["copy_metadata"](self.h, _ptr(out))
        return out

    def weights(self):
        out = np.empty((self.total_rows, max(self.dim, 1)), dtype=np.float32)
        if self.dim:
            self.L["copy_weights"](self.h, _ptr(out))
        return out

    def momentum(self):
        out = np.empty((self.total_rows, max(self.dim, 1)), dtype=np.float32)
        if self.dim:
            self.L["copy_momentum"](self.h, _ptr(out))
        return out

    def trained(self):
        out = np.zeros(self.total_rows, dtype=np.uint8)
        if self.dim:
            self.L["copy_trained"](self.h, _ptr(out))
        return out

    def make_cursor(self):
        return int(self.L["make_cursor"](self.h))

    def serialize_snapshot(self) -> bytes:
        n = ctypes.c_uint64(0)
        self.L["serialize_snapshot"](self.h, None, 0, ctypes.byref(n))
        if n.value == 0:
            _raise(self.L, self.L["serialize_snapshot"](self.h, None, 0, ctypes.byref(n)))
        out = np.empty(n.value, np.uint8)
        _raise(self.L, self.L["serialize_snapshot"](self.h, _ptr(out), out.size, ctypes.byref(n)))
        return out.tobytes()

    def delta_source(self, base_checksum: int):
        """DeltaSource(table, base) (publish.hpp:69-82): returns a cut() -> bytes callable
        (cut + serialize_delta)."""
        if self.kind == "reference":
            _raise(self.L, self.L["delta_source_create"](self.h, base_checksum))

            def cut():
                n = ctypes.c_uint64(0)
                cap = 64 + self.total_rows * (16 + 4 * self.dim)
                out = np.empty(cap, np.uint8)
                _raise(self.L, self.L["delta_source_cut"](self.h, _ptr(out), cap, ctypes.byref(n)))
                return out[:n.value].tobytes()
            return cut
        if self.dim == 0:
            raise OracleError(4, "index-only tables (dim = 0) cannot be published")
        state = {"cursor": self.make_cursor(), "seq": 0}

        def cut():
            n, nxt = ctypes.c_uint64(0), ctypes.c_uint64(0)
            cap = 64 + self.total_rows * (16 + 4 * self.dim)
            out = np.empty(cap, np.uint8)
            _raise(self.L, self.L["serialize_delta"](self.h, state["cursor"], base_checksum,
                                                     state["seq"], _ptr(out), cap,
                                                     ctypes.byref(n), ctypes.byref(nxt)))
            state["cursor"] = nxt.value
            state["seq"] += 1
            return out[:n.value].tobytes()
        return cut

    def sgd_step(self, rows, grads, lr, beta):
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        g = np.ascontiguousarray(grads, dtype=np.float32).reshape(-1)
        _raise(self.L, self.L["sgd_step"](self.h, _ptr(rows), rows.size, _ptr(g), g.size, lr, beta))

    def dirty_rows_since(self, cursor):
        out = np.empty(self.total_rows, dtype=np.uint64)
        n = ctypes.c_uint64(0)
        _raise(self.L, self.L["dirty_rows_since"](self.h, cursor, _ptr(out), out.size, ctypes.byref(n)))
        return out[:n.value].copy()


def crc32(data: bytes, kind="port") -> int:
    a = np.frombuffer(data, np.uint8)
    return int(lib(kind)["crc32"](_ptr(a), a.size))


def probe(id, meta_in, now, identities, metadata, capacity, max_probe, seed, mode, kind="port"):
    L = lib(kind)
    I = np.ascontiguousarray(identities, dtype=np.uint64)
    M = np.ascontiguousarray(metadata, dtype=np.uint64)
    s = ctypes.c_uint64(0)
    o = ctypes.c_uint8(0)
    _raise(L, L["probe"](id, meta_in, now, _ptr(I), _ptr(M), capacity, max_probe, seed, mode,
                         ctypes.byref(s), ctypes.byref(o)))
    return s.value, o.value, I, M


def probe_readonly(id, identities, capacity, max_probe, seed, kind="port"):
    L = lib(kind)
    I = np.ascontiguousarray(identities, dtype=np.uint64)
    s = ctypes.c_uint64(0)
    o = ctypes.c_uint8(0)
    _raise(L, L["probe_readonly"](id, _ptr(I), capacity, max_probe, seed, ctypes.byref(s),
                                  ctypes.byref(o)))
    return s.value, o.value


def draw_rows(dim, rows, init_seed):
    """draw_row for every row of `rows` (closed form, embedding_store.cpp:12-18): [n, dim]."""
    r = np.ascontiguousarray(rows, dtype=np.uint64)
    out = np.empty((r.size, dim), dtype=np.float32)
    lib("port")["draw_rows"](_ptr(out), dim, _ptr(r), r.size, init_seed)
    return out


def draw_row(dim, row, init_seed):
    out = np.empty(dim, dtype=np.float32)
    lib("port")["draw_row"](_ptr(out), dim, row, init_seed)
    return out


# ---- workload generators shared by tests and bench (SURVEY 8d synthetic inputs) ----------

class SplitMix64:
    """SplitMix64, proj/include/mpzch/rng.hpp:10-30 (pure Python; small streams only)."""
    M = (1 << 64) - 1

    def __init__(self, seed):
        self.state = seed & self.M

    def next(self):
        self.state = (self.state + 0x9E3779B97F4A7C15) & self.M
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def next_below(self, bound):
        return self.next() % bound

    def next_unit(self):
        return (self.next() >> 11) * 2.0 ** -53


def splitmix_stream(seed: int, count: int) -> np.ndarray:
    """count consecutive SplitMix64(seed).next() outputs, vectorised in numpy."""
    with np.errstate(over="ignore"):
        k = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def mix64_np(x: np.ndarray, seed: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x.astype(np.uint64) ^ np.uint64(seed)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xff51afd7ed558ccd)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xc4ceb9fe1a85ec53)
        x ^= x >> np.uint64(33)
        return x
