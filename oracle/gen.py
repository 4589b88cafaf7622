"""HOST generator of the five BASELINE configurations -- TEST / BASELINE
INFRASTRUCTURE ONLY (see oracle/__init__.py).

A numpy restatement of ``paper_2111_08824_b200/configs.py`` on top of the
C primitives of ``oracle/lj_gen.c``, which evaluate the same portable
arithmetic (``include/lj_gen.h``) as the CUDA generator kernels.  It
produces the device inputs bit for bit without loading the CUDA library,
so ``bench.py --impl reference`` runs the reference path on exactly the
relations the GPU arm joins, and ``tests/test_gpu_fullsize.py`` pins the
device generator to it.

Every function returns numpy uint64 arrays ``(rk, rp, sk, sp)`` (C3 / C5
return S lazily: ``s_slice(lo, hi)``), plus the config's opts.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _i64, _p, _u64p, lib, sort_u64

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
MAX63 = (1 << 63) - 1
MAXKEY_F = float(2**63 - 1024)
_U53 = 1.0 / (1 << 53)


def _u(seed):
    return ctypes.c_uint64(int(seed) & (2**64 - 1))


def mix(n, seed, offset=0) -> np.ndarray:
    out = np.empty(int(n), np.uint64)
    if n:
        lib().orc_gen_mix(_p(out, _u64p), _i64(n), _i64(offset), _u(seed))
    return out


def payloads(n, seed, offset=0) -> np.ndarray:
    out = np.empty(int(n), np.uint64)
    if n:
        lib().orc_gen_payloads(_p(out, _u64p), _i64(n), _i64(offset), _u(seed))
    return out


def gather_uniform(src: np.ndarray, n, seed, offset=0) -> np.ndarray:
    src = np.ascontiguousarray(src, dtype=np.uint64)
    out = np.empty(int(n), np.uint64)
    if n:
        lib().orc_gen_gather_uniform(_p(out, _u64p), _i64(n), _i64(offset), _u(seed), _p(src, _u64p),
                                     _i64(src.size))
    return out


def normal(n, seed, offset=0) -> np.ndarray:
    out = np.empty(int(n), np.float64)
    if n:
        lib().orc_gen_normal(_p(out, _f64p), _i64(n), _i64(offset), _u(seed))
    return out


def lognormal_keys(n, seed, offset, sigma, scale) -> np.ndarray:
    out = np.empty(int(n), np.int64)
    if n:
        lib().orc_gen_lognormal(_p(out, _i64p), _i64(n), _i64(offset), _u(seed), ctypes.c_double(sigma),
                                ctypes.c_double(scale), ctypes.c_double(MAXKEY_F))
    return out.view(np.uint64)


def cluster_keys(n, seed, offset, centres: np.ndarray, sigma) -> np.ndarray:
    centres = np.ascontiguousarray(centres, dtype=np.float64)
    out = np.empty(int(n), np.int64)
    if n:
        lib().orc_gen_cluster(_p(out, _i64p), _i64(n), _i64(offset), _u(seed), _p(centres, _f64p),
                              ctypes.c_int(centres.size), ctypes.c_double(sigma), ctypes.c_double(MAXKEY_F))
    return out[out >= 0].view(np.uint64)


def uniform63(n, seed, offset=0) -> np.ndarray:
    return (mix(n, seed, offset) >> np.uint64(1)) & np.uint64(MAX63)


def unit(n, seed, offset=0) -> np.ndarray:
    m = mix(n, seed, offset)
    return ((m >> np.uint64(11)).astype(np.float64) + 0.5) * _U53


def first_occurrence(v: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.uint64)
    keep = np.empty(v.size, np.uint8)
    if v.size:
        lib().orc_first_occurrence(_p(v, _u64p), _i64(v.size), _p(keep, _u8p))
    return keep.astype(bool)


def distinct_first(draw, n) -> np.ndarray:
    """configs.distinct_first: the first n distinct values of the stream
    draw(count, offset), in draw order (chunking does not change it)."""
    have = np.empty(0, np.uint64)
    offset = 0
    need = n
    while need > 0:
        chunk = max(int(need * 1.05) + 1024, 4096)
        fresh = draw(chunk, offset)
        offset += chunk
        allv = np.concatenate([have, fresh])
        allv = allv[first_occurrence(allv)]
        have = allv[:n]
        need = n - have.size
    return have


def shuffle(t: np.ndarray, seed) -> np.ndarray:
    # configs.shuffle: argsort of signed int64 draws (no ties in practice)
    keys = np.ascontiguousarray(mix(t.size, seed).view(np.int64))
    order = np.empty(t.size, np.int64)
    if t.size:
        lib().orc_argsort_i64(_p(keys, _i64p), _i64(t.size), _p(order, _i64p))
    return t[order]


def searchsorted_left(cdf: np.ndarray, u: np.ndarray) -> np.ndarray:
    """np.searchsorted(cdf, u, side="left"), in parallel C."""
    cdf = np.ascontiguousarray(cdf, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty(u.size, np.int64)
    if u.size:
        lib().orc_searchsorted_f64(_p(cdf, _f64p), _i64(cdf.size), _p(u, _f64p), _i64(u.size), _p(out, _i64p))
    return out


def zipf_ranks(n, N, s, seed) -> np.ndarray:
    w = np.arange(1, N + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    u = unit(n, seed) * cdf[-1]
    return np.minimum(searchsorted_left(cdf, u), N - 1)


def not_in(sorted_r: np.ndarray, cand: np.ndarray) -> np.ndarray:
    sorted_r = np.ascontiguousarray(sorted_r, dtype=np.uint64)
    cand = np.ascontiguousarray(cand, dtype=np.uint64)
    pos = np.empty(cand.size, np.int64)
    if cand.size:
        lib().orc_searchsorted_u64(_p(sorted_r, _u64p), _i64(sorted_r.size), _p(cand, _u64p), _i64(cand.size),
                                   _p(pos, _i64p))
    pos = np.minimum(pos, sorted_r.size - 1)
    return cand[sorted_r[pos] != cand]


def mix_keys(keys: np.ndarray) -> np.ndarray:
    """mix64 of each key (configs._mix_keys, reference util.py:30-44)."""
    z = keys.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


@dataclass
class HostInputs:
    name: str
    rk: np.ndarray
    rp: np.ndarray
    n_s: int
    opts: dict
    algorithm: str
    s_slice: object = field(repr=False, default=None)  # (lo, hi) -> (sk, sp)

    def s(self):
        return self.s_slice(0, self.n_s)


def config1(scale: int = 0, seed: int = 0xC1, shard: int = 0) -> HostInputs:
    nr, ns = (1 << 20) >> scale, (1 << 22) >> scale
    with np.errstate(over="ignore"):
        rk = distinct_first(lambda c, o: uniform63(c, seed, o), nr)
        rp = mix_keys(rk)
    hits = int(round(0.9 * ns))
    ss = seed ^ (shard << 40)
    sk_hit = gather_uniform(rk, hits, ss ^ 0x51)
    srt = sort_u64(rk)
    miss = np.empty(0, np.uint64)
    off = 0
    while miss.size < ns - hits:
        c = not_in(srt, uniform63(2 * (ns - hits) + 1024, ss ^ 0x52, off))
        off += 2 * (ns - hits) + 1024
        miss = np.concatenate([miss, c])
    sk = shuffle(np.concatenate([sk_hit, miss[: ns - hits]]), ss ^ 0x53)
    sp = payloads(ns, ss ^ 0x54)
    return HostInputs("c1", rk, rp, ns, {"gap_factor": 2.0, "rmi_fanout": 1024}, "grmi-inlj",
                      lambda lo, hi: (sk[lo:hi], sp[lo:hi]))


def config2(scale: int = 0, seed: int = 0xC2, shard: int = 0) -> HostInputs:
    nr, ns = (1 << 24) >> scale, (1 << 28) >> scale
    leaves = (1 << 16) >> min(scale, 8)

    def draw(c, o):
        return lognormal_keys(c, seed, o, 2.0, 1e12)

    rk = distinct_first(draw, nr)
    rp = payloads(nr, seed ^ 0x11)
    srt = sort_u64(rk)
    hits = int(round(0.95 * ns))
    ss = seed ^ (shard << 40)
    sk_hit = srt[zipf_ranks(hits, nr, 0.8, ss ^ 0x21)]
    miss = np.empty(0, np.uint64)
    off = 0
    while miss.size < ns - hits:
        c = not_in(srt, draw(2 * (ns - hits) + 1024, (1 << 40) + (shard << 36) + off))
        off += 2 * (ns - hits) + 1024
        miss = np.concatenate([miss, c])
    sk = shuffle(np.concatenate([sk_hit, miss[: ns - hits]]), ss ^ 0x22)
    sp = payloads(ns, ss ^ 0x23)
    return HostInputs("c2", rk, rp, ns, {"gap_factor": 2.0, "rmi_fanout": leaves}, "grmi-inlj",
                      lambda lo, hi: (sk[lo:hi], sp[lo:hi]))


def config3(scale: int = 1, seed: int = 0xC3, shard: int = 0, shards: int = 1) -> HostInputs:
    """S is generated lazily: s_slice(lo, hi) draws probes lo..hi-1 of this
    shard (counter-based, so any slice is independent of the others)."""
    nr, ns_total = 200_000_000 // scale, 2_000_000_000 // scale
    lo_s = ns_total * shard // shards
    ns = ns_total * (shard + 1) // shards - lo_s
    centres = (uniform63(64, seed ^ 0x31) >> np.uint64(1)).astype(np.float64)

    def draw(c, o):
        return cluster_keys(c, seed, o, centres, float(2**40))

    rk = distinct_first(draw, nr)
    rp = payloads(nr, seed ^ 0x34)

    def s_slice(lo, hi):
        return (gather_uniform(rk, hi - lo, seed ^ 0x35, lo_s + lo), payloads(hi - lo, seed ^ 0x36, lo_s + lo))

    return HostInputs("c3", rk, rp, ns, {"spline_error": 32, "radix_bits": 18, "table_factor": 4.0},
                      "spline-hash-inlj", s_slice)


def config4(scale: int = 0, seed: int = 0xC4, shard: int = 0) -> HostInputs:
    nr = ns = (1 << 28) >> scale

    def draw(c, o):
        return lognormal_keys(c, seed, o, 1.5, float(2**40))

    rk = distinct_first(draw, nr)
    rp = payloads(nr, seed ^ 0x41)
    sk = sort_u64(rk)[zipf_ranks(ns, nr, 1.0, seed ^ 0x42 ^ (shard << 40))]
    sp = payloads(ns, seed ^ 0x43 ^ (shard << 40))
    return HostInputs("c4", rk, rp, ns, {"fanout": 4096, "sample_rate": 0.01}, "lsj",
                      lambda lo, hi: (sk[lo:hi], sp[lo:hi]))


def bijective63(i: np.ndarray, seed: int) -> np.ndarray:
    m = np.uint64(MAX63)
    x = (i.astype(np.uint64) + np.uint64(seed & MAX63)) & m
    for mul, sh in ((0x5851F42D4C957F2D, 29), (0x14057B7EF767814F, 31), (0x2545F4914F6CDD1D, 27)):
        x = (x * np.uint64(mul)) & m
        x = x ^ (x >> np.uint64(sh))
    return x


def config5(scale: int = 0, seed: int = 0xC5, shard: int = 0, shards: int = 1) -> HostInputs:
    n_total = 2_000_000_000 >> scale
    lo = n_total * shard // shards
    n = n_total * (shard + 1) // shards - lo
    with np.errstate(over="ignore"):
        rk = bijective63(np.arange(lo, lo + n, dtype=np.uint64), seed)
    rp = payloads(n, seed ^ 0x51, lo)

    def s_slice(a, b):
        j = mix(b - a, seed ^ 0x52, lo + a)
        sidx = (j >> np.uint64(1)) % np.uint64(n_total)
        with np.errstate(over="ignore"):
            return bijective63(sidx, seed), payloads(b - a, seed ^ 0x53, lo + a)

    return HostInputs("c5", rk, rp, n, {"fanout": 4096, "sample_rate": 0.01}, "lsj", s_slice)


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}
