"""CPU ORACLE for the learned-join hot paths -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  It is
the checker, never the thing measured as the product: the package
``paper_2111_08824_b200`` never imports it and has no CPU fallback.

The arithmetic lives in ``lj_oracle.c`` (a plain-C restatement of the
reference ``learned_joins`` package, every function citing the reference
file:line it follows).  This module is a thin ctypes wrapper plus the one
piece of the reference that is numpy itself: the LSJ sampler
(``np.random.default_rng(seed).choice``, lsj.py:119-120), which we call
directly so that the oracle trains on exactly the reference's sample.

Pinned against golden vectors produced by importing the reference
(``oracle/make_golden.py`` -> ``tests/golden/``), see
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblj_oracle.so")
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64


class _Rmi(ctypes.Structure):
    _fields_ = [
        ("root_slope", ctypes.c_double),
        ("root_icpt", ctypes.c_double),
        ("m", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("slope", _f64p),
        ("icpt", _f64p),
        ("clamp_lo", _i64p),
        ("clamp_hi", _i64p),
        ("err_lo", _i64p),
        ("err_hi", _i64p),
    ]


class _Spline(ctypes.Structure):
    _fields_ = [
        ("npts", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("max_error", ctypes.c_int64),
        ("radix_bits", ctypes.c_int64),
        ("shift", ctypes.c_uint64),
        ("sk", _u64p),
        ("sr", _i64p),
        ("rt", _i64p),
    ]


def build() -> str:
    """Compile lj_oracle.c (make) and return the library path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        srcs = [os.path.join(_HERE, f) for f in ("lj_oracle.c", "lj_gen.c")]
        srcs.append(os.path.join(_HERE, "..", "include", "lj_gen.h"))
        if not os.path.exists(_LIB_PATH) or any(os.path.getmtime(_LIB_PATH) < os.path.getmtime(f)
                                                for f in srcs if os.path.exists(f)):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.orc_mix64.restype = ctypes.c_uint64
        _lib.orc_mix64.argtypes = [ctypes.c_uint64]
        _lib.orc_num_threads.restype = ctypes.c_int
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


# ------------------------------------------------------------------ util


def mix64(x):
    """util.py:30-44 (vectorised through the C finaliser)."""
    x = np.asarray(x, dtype=np.uint64)
    if x.ndim == 0:
        return np.uint64(lib().orc_mix64(int(x)))
    return np.array([lib().orc_mix64(int(v)) for v in x.ravel()], dtype=np.uint64).reshape(x.shape)


def make_payloads(n: int, seed: int) -> np.ndarray:
    """data.py:181-192 positional payload rule."""
    out = np.empty(n, dtype=np.uint64)
    lib().orc_make_payloads(_i64(n), ctypes.c_uint64(seed & (2**64 - 1)), _p(out, _u64p))
    return out


def chunk_bounds(n: int, workers: int) -> np.ndarray:
    out = np.empty(workers + 1, dtype=np.int64)
    lib().orc_chunk_bounds(_i64(n), _i64(workers), _p(out, _i64p))
    return out


def checksum_pairs(pr, ps) -> tuple[int, int, int]:
    """(count, sum, xor) of t = pr + ps mod 2^64 -- the result checksum."""
    pr = np.asarray(pr, dtype=np.uint64)
    ps = np.asarray(ps, dtype=np.uint64)
    with np.errstate(over="ignore"):
        t = pr + ps
    if t.size == 0:
        return (0, 0, 0)
    return (int(t.size), int(np.sum(t, dtype=np.uint64)), int(np.bitwise_xor.reduce(t)))


# ------------------------------------------------------------------ RMI


@dataclass
class Rmi:
    """Plain parameter bag of a two-level RMI (models.py:39-143)."""

    root_slope: float
    root_intercept: float
    trained_len: int
    leaf_slope: np.ndarray
    leaf_intercept: np.ndarray
    clamp_lo: np.ndarray
    clamp_hi: np.ndarray
    err_lo: np.ndarray
    err_hi: np.ndarray

    @property
    def fanout(self) -> int:
        return int(self.leaf_slope.size)

    @classmethod
    def from_model(cls, model) -> "Rmi":
        """Copy the parameters of any RMI-shaped object (reference or ours)."""
        return cls(
            float(model.root_slope),
            float(model.root_intercept),
            int(model.trained_len),
            np.ascontiguousarray(model.leaf_slope, dtype=np.float64),
            np.ascontiguousarray(model.leaf_intercept, dtype=np.float64),
            np.ascontiguousarray(model.clamp_lo, dtype=np.int64),
            np.ascontiguousarray(model.clamp_hi, dtype=np.int64),
            np.ascontiguousarray(model.err_lo, dtype=np.int64),
            np.ascontiguousarray(model.err_hi, dtype=np.int64),
        )

    def _c(self) -> _Rmi:
        return _Rmi(
            self.root_slope,
            self.root_intercept,
            self.fanout,
            self.trained_len,
            _p(self.leaf_slope, _f64p),
            _p(self.leaf_intercept, _f64p),
            _p(self.clamp_lo, _i64p),
            _p(self.clamp_hi, _i64p),
            _p(self.err_lo, _i64p),
            _p(self.err_hi, _i64p),
        )


def rmi_fit(sorted_keys, fanout: int) -> Rmi:
    keys = _u64(sorted_keys)
    m = int(fanout)
    arrs = [np.zeros(m, np.float64), np.zeros(m, np.float64)] + [np.zeros(m, np.int64) for _ in range(4)]
    c = _Rmi(0.0, 0.0, m, keys.size, _p(arrs[0], _f64p), _p(arrs[1], _f64p), _p(arrs[2], _i64p),
             _p(arrs[3], _i64p), _p(arrs[4], _i64p), _p(arrs[5], _i64p))
    if lib().orc_rmi_fit(_p(keys, _u64p), _i64(keys.size), _i64(m), ctypes.byref(c)) != 0:
        raise ValueError("cannot train on an empty key array")
    return Rmi(c.root_slope, c.root_icpt, keys.size, *arrs)


def rmi_predict(model: Rmi, keys):
    keys = _u64(keys)
    n = keys.size
    pos, lo, hi, leaf = (np.empty(n, np.int64) for _ in range(4))
    c = model._c()
    lib().orc_rmi_predict(ctypes.byref(c), _p(keys, _u64p), _i64(n), _p(pos, _i64p), _p(lo, _i64p),
                          _p(hi, _i64p), _p(leaf, _i64p))
    return pos, lo, hi, leaf


def rmi_partition_index(model: Rmi, keys, num_partitions: int) -> np.ndarray:
    keys = _u64(keys)
    out = np.empty(keys.size, np.int64)
    c = model._c()
    lib().orc_rmi_partition_index(ctypes.byref(c), _p(keys, _u64p), _i64(keys.size),
                                  _i64(num_partitions), _p(out, _i64p))
    return out


# ------------------------------------------------------------------ GRMI


def slot_count(gap_factor: float, n: int) -> int:
    """gapped.py:233  L = int(round(gap_factor * n)) (Python half-even)."""
    return int(round(float(gap_factor) * n))


@dataclass
class Grmi:
    model: Rmi
    n: int
    L: int
    gkeys: np.ndarray
    gpayloads: np.ndarray
    bitmap: np.ndarray


def grmi_build(keys, payloads, gap_factor: float, fanout: int, model: Rmi | None = None) -> Grmi:
    """gapped.py:221-256; `model` overrides the fit (e.g. the reference's)."""
    keys = _u64(keys)
    payloads = _u64(payloads)
    order = np.argsort(keys, kind="stable")
    sk, sp = np.ascontiguousarray(keys[order]), np.ascontiguousarray(payloads[order])
    n = sk.size
    if model is None:
        model = rmi_fit(sk, fanout)
    L = slot_count(gap_factor, n)
    g = np.empty(L, np.uint64)
    gp = np.empty(L, np.uint64)
    bm = np.empty(L, np.uint8)
    c = model._c()
    lib().orc_grmi_build(ctypes.byref(c), _p(sk, _u64p), _p(sp, _u64p), _i64(n), _i64(L),
                         _p(g, _u64p), _p(gp, _u64p), _p(bm, _u8p))
    return Grmi(model, n, L, g, gp, bm.astype(bool))


def grmi_predict_slots(idx: Grmi, keys) -> np.ndarray:
    keys = _u64(keys)
    out = np.empty(keys.size, np.int64)
    c = idx.model._c()
    lib().orc_grmi_predict_slots(ctypes.byref(c), _i64(idx.n), _i64(idx.L), _p(keys, _u64p),
                                 _i64(keys.size), _p(out, _i64p))
    return out


def exp_search(gkeys, slots0, keys):
    gkeys = _u64(gkeys)
    keys = _u64(keys)
    slots0 = np.ascontiguousarray(slots0, dtype=np.int64)
    slot = np.empty(keys.size, np.int64)
    probes = np.empty(keys.size, np.int64)
    lib().orc_exp_search(_p(gkeys, _u64p), _i64(gkeys.size), _p(slots0, _i64p), _p(keys, _u64p),
                         _i64(keys.size), _p(slot, _i64p), _p(probes, _i64p))
    return slot, probes


def match_runs(idx: Grmi, slots, keys):
    keys = _u64(keys)
    slots = np.ascontiguousarray(slots, dtype=np.int64)
    bm = np.ascontiguousarray(idx.bitmap, dtype=np.uint8)
    left = np.empty(keys.size, np.int64)
    count = np.empty(keys.size, np.int64)
    lib().orc_match_runs(_p(idx.gkeys, _u64p), _p(bm, _u8p), _i64(idx.L), _p(slots, _i64p),
                         _p(keys, _u64p), _i64(keys.size), _p(left, _i64p), _p(count, _i64p))
    return left, count


def grmi_join(idx: Grmi, s_keys, s_payloads, threads: int = 0):
    """-> (count, sum, xor, search_steps)"""
    sk = _u64(s_keys)
    sp = _u64(s_payloads)
    bm = np.ascontiguousarray(idx.bitmap, dtype=np.uint8)
    out = np.zeros(4, np.uint64)
    c = idx.model._c()
    lib().orc_grmi_join(ctypes.byref(c), _i64(idx.n), _i64(idx.L), _p(idx.gkeys, _u64p),
                        _p(idx.gpayloads, _u64p), _p(bm, _u8p), _p(sk, _u64p), _p(sp, _u64p),
                        _i64(sk.size), ctypes.c_int(threads), _p(out, _u64p))
    return tuple(int(v) for v in out)


def rmi_inlj(model: Rmi, sorted_keys, sorted_payloads, s_keys, s_payloads, threads: int = 0):
    """baselines.py:96-157 over sorted R -> (count, sum, xor, search_steps)."""
    rk = _u64(sorted_keys)
    rp = _u64(sorted_payloads)
    sk = _u64(s_keys)
    sp = _u64(s_payloads)
    out = np.zeros(4, np.uint64)
    c = model._c()
    lib().orc_rmi_inlj(ctypes.byref(c), _p(rk, _u64p), _p(rp, _u64p), _i64(rk.size), _p(sk, _u64p),
                       _p(sp, _u64p), _i64(sk.size), ctypes.c_int(threads), _p(out, _u64p))
    return tuple(int(v) for v in out)


# ------------------------------------------------------------ RadixSpline


@dataclass
class Spline:
    spline_keys: np.ndarray
    spline_ranks: np.ndarray
    radix_table: np.ndarray
    shift: int
    trained_len: int
    max_error: int
    radix_bits: int

    @classmethod
    def from_model(cls, model) -> "Spline":
        return cls(
            np.ascontiguousarray(model.spline_keys, dtype=np.uint64),
            np.ascontiguousarray(model.spline_ranks, dtype=np.int64),
            np.ascontiguousarray(model.radix_table, dtype=np.int64),
            int(model.shift),
            int(model.trained_len),
            int(model.max_error),
            int(model.radix_bits),
        )

    def _c(self) -> _Spline:
        return _Spline(self.spline_keys.size, self.trained_len, self.max_error, self.radix_bits,
                       self.shift, _p(self.spline_keys, _u64p), _p(self.spline_ranks, _i64p),
                       _p(self.radix_table, _i64p))


def spline_fit(sorted_keys, max_error: int, radix_bits: int) -> Spline:
    keys = _u64(sorted_keys)
    if keys.size == 0:
        raise ValueError("cannot train on an empty key array")
    n = keys.size
    sk = np.empty(n, np.uint64)
    sr = np.empty(n, np.int64)
    rt = np.empty((1 << radix_bits) + 1, np.int64)
    c = _Spline(0, 0, 0, 0, 0, _p(sk, _u64p), _p(sr, _i64p), _p(rt, _i64p))
    lib().orc_spline_fit(_p(keys, _u64p), _i64(n), _i64(max_error), _i64(radix_bits), ctypes.byref(c))
    k = c.npts
    return Spline(sk[:k].copy(), sr[:k].copy(), rt, int(c.shift), n, max_error, radix_bits)


def spline_predict(model: Spline, keys):
    keys = _u64(keys)
    n = keys.size
    pos, lo, hi = (np.empty(n, np.int64) for _ in range(3))
    c = model._c()
    lib().orc_spline_predict(ctypes.byref(c), _p(keys, _u64p), _i64(n), _p(pos, _i64p),
                             _p(lo, _i64p), _p(hi, _i64p))
    return pos, lo, hi


def spline_partition_index(model: Spline, keys, num_partitions: int) -> np.ndarray:
    keys = _u64(keys)
    out = np.empty(keys.size, np.int64)
    c = model._c()
    lib().orc_spline_partition_index(ctypes.byref(c), _p(keys, _u64p), _i64(keys.size),
                                     _i64(num_partitions), _p(out, _i64p))
    return out


@dataclass
class SplineHash:
    model: Spline
    table_len: int
    keys: np.ndarray
    payloads: np.ndarray
    starts: np.ndarray


def spline_hash_build(keys, payloads, max_error=32, radix_bits=18, table_factor=4.0,
                      model: Spline | None = None) -> SplineHash:
    """learned_hash.py:35-66"""
    keys = _u64(keys)
    payloads = _u64(payloads)
    n = keys.size
    if model is None:
        model = spline_fit(sort_u64(keys), max_error, radix_bits)
    P = max(1, int(round(float(table_factor) * n)))
    ek = np.empty(n, np.uint64)
    ep = np.empty(n, np.uint64)
    st = np.empty(P + 1, np.int64)
    c = model._c()
    lib().orc_spline_hash_build(ctypes.byref(c), _p(keys, _u64p), _p(payloads, _u64p), _i64(n),
                                _i64(P), _p(ek, _u64p), _p(ep, _u64p), _p(st, _i64p))
    return SplineHash(model, P, ek, ep, st)


def spline_hash_join(idx: SplineHash, s_keys, s_payloads, threads: int = 0):
    sk = _u64(s_keys)
    sp = _u64(s_payloads)
    out = np.zeros(4, np.uint64)
    c = idx.model._c()
    lib().orc_spline_hash_join(ctypes.byref(c), _i64(idx.table_len), _p(idx.keys, _u64p),
                               _p(idx.payloads, _u64p), _p(idx.starts, _i64p), _p(sk, _u64p),
                               _p(sp, _u64p), _i64(sk.size), ctypes.c_int(threads), _p(out, _u64p))
    return tuple(int(v) for v in out[:3])


# ------------------------------------------------------------------ LSJ


def lsj_sample_model(keys, sample_rate: float, seed: int, fanout: int | None = None) -> Rmi:
    """lsj.py:95-130: the reference's own sampler (numpy Generator.choice)
    and fanout rule, then the C fit.  The per-worker split of the sample
    positions does not change the sorted sample, so it is omitted."""
    keys = _u64(keys)
    n = keys.size
    total = int(round(sample_rate * n))
    if total == 0:
        return rmi_fit(np.sort(np.asarray([keys.min(), keys.max()], dtype=np.uint64)), 1)
    rng = np.random.default_rng(seed)
    positions = rng.choice(n, size=total, replace=False)
    sample = np.sort(keys[positions])
    if fanout is None:
        fanout = min(1000, max(1, total // 8))
    return rmi_fit(sample, fanout)


def lsj_join(rk, rp, sk, sp, workers=1, sample_rate=0.01, fanout=10000, seed=0x1D5EED,
             model_fanout=None, models=None):
    """lsj.py:373-405 -> ((count, sum, xor), (comparator_count, partitions_sorted))."""
    rk, rp, sk, sp = _u64(rk), _u64(rp), _u64(sk), _u64(sp)
    if rk.size == 0 or sk.size == 0:
        return (0, 0, 0), (0, 0)
    if models is None:
        mr = lsj_sample_model(rk, sample_rate, seed, model_fanout)
        ms = lsj_sample_model(sk, sample_rate, seed ^ 0x5DEECE66D, model_fanout)
    else:
        mr, ms = models
    out = np.zeros(3, np.uint64)
    stats = np.zeros(2, np.uint64)
    cr, cs = mr._c(), ms._c()
    lib().orc_lsj_join(_p(rk, _u64p), _p(rp, _u64p), _i64(rk.size), _p(sk, _u64p), _p(sp, _u64p),
                       _i64(sk.size), ctypes.byref(cr), ctypes.byref(cs), _i64(workers),
                       _i64(fanout), _p(out, _u64p), _p(stats, _u64p))
    return tuple(int(v) for v in out), tuple(int(v) for v in stats)


def sort_u64(keys) -> np.ndarray:
    """np.sort of uint64 keys (parallel radix sort in C; a sorted copy)."""
    out = np.array(keys, dtype=np.uint64, copy=True)
    if out.size > 1:
        lib().orc_sort_u64(_p(out, _u64p), _i64(out.size))
    return out


# ------------------------------------------------------- ground truth


def smj_checksum(rk, rp, sk, sp):
    rk, rp, sk, sp = _u64(rk), _u64(rp), _u64(sk), _u64(sp)
    out = np.zeros(3, np.uint64)
    lib().orc_smj_checksum(_p(rk, _u64p), _p(rp, _u64p), _i64(rk.size), _p(sk, _u64p),
                           _p(sp, _u64p), _i64(sk.size), _p(out, _u64p))
    return tuple(int(v) for v in out)


def nlj_checksum(rk, rp, sk, sp):
    rk, rp, sk, sp = _u64(rk), _u64(rp), _u64(sk), _u64(sp)
    out = np.zeros(3, np.uint64)
    lib().orc_nlj_checksum(_p(rk, _u64p), _p(rp, _u64p), _i64(rk.size), _p(sk, _u64p),
                           _p(sp, _u64p), _i64(sk.size), _p(out, _u64p))
    return tuple(int(v) for v in out)


def num_threads() -> int:
    return int(lib().orc_num_threads())
