"""Seeded synthetic inputs of the five BASELINE configurations, generated
on the device (BASELINE.json ``configs``).

Size interpretations (pinned): "16M" = 2^24, "256M" = 2^28, "200M" =
2*10^8, "2B" = 2*10^9.  Keys are uint64 < 2^63; payloads uint64.

Integer parts use counter-based SplitMix64 draws (``mix64(seed ^ i)``),
bit-identical anywhere.  The lognormal / normal draws (Box-Muller on two
counter draws) use the portable float64 arithmetic of ``include/lj_gen.h``
(IEEE + - * / sqrt only, no FMA), so the host generator ``oracle/gen.py``
regenerates every configuration bit for bit without the CUDA library (the
reference arm of bench.py does; ``tests/test_gpu_fullsize.py`` checks it).  Duplicates
are removed keeping the first draw, then topped up from the continuing
counter stream, and the draw order (already random) is kept.  A finite
Zipf(s) over N ranks is sampled by exact inverse-CDF lookup in the float64
cumulative weight table.  The paper's SOSD datasets are not available here;
these seeded generators stand in for them.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib
from .data import Relation, fill_payloads

MAX63 = (1 << 63) - 1
_U53 = 1.0 / (1 << 53)


def _mix(n: int, seed: int, offset: int = 0, device="cuda") -> torch.Tensor:
    out = torch.empty(int(n), dtype=torch.int64, device=device)
    if n:
        _lib.check(_lib.lib().lj_fill_mix64(_lib.ptr(out), int(n), int(offset), int(seed) & (2**64 - 1),
                                            _lib.stream_ptr()), "fill_mix64")
    return out


def _unit(n: int, seed: int, offset: int = 0, device="cuda") -> torch.Tensor:
    """Uniform float64 in (0, 1) from the top 53 bits of a counter draw."""
    m = _mix(n, seed, offset, device)
    return (((m >> 11) & ((1 << 53) - 1)).to(torch.float64) + 0.5) * _U53


def uniform63(n: int, seed: int, offset: int = 0, device="cuda") -> torch.Tensor:
    return (_mix(n, seed, offset, device) >> 1) & MAX63


def normal(n: int, seed: int, offset: int = 0, device="cuda") -> torch.Tensor:
    """Standard normal draws offset .. offset+n-1 of stream ``seed``
    (Box-Muller in the portable arithmetic of include/lj_gen.h: the host
    generator oracle/gen.py reproduces the same bits)."""
    out = torch.empty(int(n), dtype=torch.float64, device=device)
    if n:
        _lib.check(_lib.lib().lj_fill_normal(_lib.ptr(out), int(n), int(offset), int(seed) & (2**64 - 1),
                                             _lib.stream_ptr()), "fill_normal")
    return out


MAXKEY_F = float(2**63 - 1024)  # largest generated key (exact in float64)


def lognormal_keys(n: int, seed: int, offset: int, sigma: float, scale: float, device="cuda") -> torch.Tensor:
    """floor(scale * exp(sigma * normal)) clamped to [0, 2^63 - 1024]."""
    out = torch.empty(int(n), dtype=torch.int64, device=device)
    if n:
        _lib.check(_lib.lib().lj_fill_lognormal(_lib.ptr(out), int(n), int(offset), int(seed) & (2**64 - 1),
                                                float(sigma), float(scale), MAXKEY_F, _lib.stream_ptr()),
                   "fill_lognormal")
    return out


def cluster_keys(n: int, seed: int, offset: int, centres: torch.Tensor, sigma: float, device="cuda") -> torch.Tensor:
    """centre[cluster] + sigma * normal, draws outside [0, 2^63 - 1024) dropped
    (the kept draws stay in draw order)."""
    out = torch.empty(int(n), dtype=torch.int64, device=device)
    if n:
        _lib.check(_lib.lib().lj_fill_cluster(_lib.ptr(out), int(n), int(offset), int(seed) & (2**64 - 1),
                                              _lib.ptr(centres), centres.numel(), float(sigma), MAXKEY_F,
                                              _lib.stream_ptr()), "fill_cluster")
    return out[out >= 0]


def distinct_first(draw, n: int, device="cuda") -> torch.Tensor:
    """First ``n`` distinct values of the stream draw(count, offset), in
    draw order (data.py:92-124 semantics with a counter stream)."""
    have = torch.empty(0, dtype=torch.int64, device=device)
    offset = 0
    need = n
    while need > 0:
        chunk = max(int(need * 1.05) + 1024, 4096)
        fresh = draw(chunk, offset)
        offset += chunk
        allv = torch.cat([have, fresh])
        order = torch.sort(allv, stable=True).indices   # values < 2^63: signed order is fine
        sv = allv[order]
        dup = torch.zeros_like(sv, dtype=torch.bool)
        dup[1:] = sv[1:] == sv[:-1]
        keep = torch.ones_like(allv, dtype=torch.bool)
        keep[order[dup]] = False
        allv = allv[keep]
        have = allv[:n]
        need = n - have.numel()
    return have


def shuffle(t: torch.Tensor, seed: int) -> torch.Tensor:
    perm = torch.argsort(_mix(t.numel(), seed, 0, t.device))
    return t[perm]


def zipf_ranks(n: int, N: int, s: float, seed: int, device="cuda") -> torch.Tensor:
    """n ranks in [0, N) with P(k) proportional to (k+1)^-s (exact inverse CDF)."""
    # the cumulative weights are summed sequentially on the host: a device
    # scan's float rounding order is not fixed run to run, which would move
    # a few inverse-CDF boundaries and make the inputs irreproducible
    import numpy as np

    w = np.arange(1, N + 1, dtype=np.float64) ** (-s)
    cdf = torch.from_numpy(np.cumsum(w)).to(device)
    u = _unit(n, seed, 0, device) * cdf[-1]
    r = torch.searchsorted(cdf, u, right=False)
    return torch.clamp(r, max=N - 1)


def not_in(sorted_r: torch.Tensor, cand: torch.Tensor) -> torch.Tensor:
    pos = torch.searchsorted(sorted_r, cand).clamp(max=sorted_r.numel() - 1)
    return cand[sorted_r[pos] != cand]


@dataclass
class Inputs:
    name: str
    r: Relation
    s: Relation
    opts: dict
    algorithm: str
    description: str


def _gather_uniform(src: torch.Tensor, n: int, seed: int, offset: int = 0) -> torch.Tensor:
    out = torch.empty(int(n), dtype=torch.int64, device=src.device)
    if n:
        _lib.check(_lib.lib().lj_gather_uniform(_lib.ptr(out), int(n), int(offset), int(seed) & (2**64 - 1),
                                                _lib.ptr(src), src.numel(), _lib.stream_ptr()), "gather_uniform")
    return out


def config1(scale: int = 0, device="cuda", seed: int = 0xC1, shard: int = 0) -> Inputs:
    """C1: R = 2^20 unique uniform keys in [0, 2^63), payload = mix64(key);
    S = 2^22: round(0.9|S|) uniform with replacement from R, the rest uniform
    non-matching, shuffled; S payloads positional (data.py:181-192).
    ``scale`` shrinks both sides by 2^scale (parity tests)."""
    nr, ns = (1 << 20) >> scale, (1 << 22) >> scale
    rk = distinct_first(lambda c, o: uniform63(c, seed, o, device), nr, device)
    rp = _mix_keys(rk)  # "payload equal to a hash of the key"
    hits = int(round(0.9 * ns))
    ss = seed ^ (shard << 40)  # per-rank S shard (weak scaling), R shared
    sk_hit = _gather_uniform(rk, hits, ss ^ 0x51)
    srt = torch.sort(rk).values
    miss = torch.empty(0, dtype=torch.int64, device=device)
    off = 0
    while miss.numel() < ns - hits:
        c = not_in(srt, uniform63(2 * (ns - hits) + 1024, ss ^ 0x52, off, device))
        off += 2 * (ns - hits) + 1024
        miss = torch.cat([miss, c])
    sk = shuffle(torch.cat([sk_hit, miss[: ns - hits]]), ss ^ 0x53)
    s = Relation(sk, fill_payloads(ns, ss ^ 0x54, device=device), validate=False)
    return Inputs("c1", Relation(rk, rp, validate=False), s,
                  {"gap_factor": 2.0, "rmi_fanout": 1024}, "grmi-inlj",
                  f"GRMI INLJ: R={nr} uniform63 unique, S={ns} (90% hits), density 0.5, 1024 leaves")


def _mix_keys(keys: torch.Tensor) -> torch.Tensor:
    """mix64 (util.py:30-44) of each key, in wrapping int64 torch arithmetic
    with masked (logical) right shifts."""
    z = keys + torch.tensor(-7046029254386353131, dtype=torch.int64, device=keys.device)  # 0x9E3779B97F4A7C15
    z = (z ^ ((z >> 30) & ((1 << 34) - 1))) * torch.tensor(-4658895280553007687, dtype=torch.int64,
                                                           device=keys.device)  # 0xBF58476D1CE4E5B9
    z = (z ^ ((z >> 27) & ((1 << 37) - 1))) * torch.tensor(-7723592293110705685, dtype=torch.int64,
                                                           device=keys.device)  # 0x94D049BB133111EB
    return z ^ ((z >> 31) & ((1 << 33) - 1))


def config2(scale: int = 0, device="cuda", seed: int = 0xC2, shard: int = 0) -> Inputs:
    """C2: R = 2^24 unique floor(1e12 * lognormal(0, 2)); S = 2^28: 95%
    R keys at Zipf(0.8) ranks over R ascending, 5% non-matching; RMI with
    2^16 leaves, density 0.5."""
    nr, ns = (1 << 24) >> scale, (1 << 28) >> scale
    leaves = (1 << 16) >> min(scale, 8)

    def draw(c, o):
        return lognormal_keys(c, seed, o, 2.0, 1e12, device)

    rk = distinct_first(draw, nr, device)
    rp = fill_payloads(nr, seed ^ 0x11, device=device)
    srt = torch.sort(rk).values
    hits = int(round(0.95 * ns))
    ss = seed ^ (shard << 40)  # per-rank S shard (weak scaling), R shared
    sk_hit = srt[zipf_ranks(hits, nr, 0.8, ss ^ 0x21, device)]
    miss = torch.empty(0, dtype=torch.int64, device=device)
    off = 0
    while miss.numel() < ns - hits:
        c = not_in(srt, draw(2 * (ns - hits) + 1024, (1 << 40) + (shard << 36) + off))
        off += 2 * (ns - hits) + 1024
        miss = torch.cat([miss, c])
    sk = shuffle(torch.cat([sk_hit, miss[: ns - hits]]), ss ^ 0x22)
    del sk_hit, miss
    s = Relation(sk, fill_payloads(ns, ss ^ 0x23, device=device), validate=False)
    return Inputs("c2", Relation(rk, rp, validate=False), s,
                  {"gap_factor": 2.0, "rmi_fanout": leaves}, "grmi-inlj",
                  f"GRMI INLJ skewed: R={nr} lognormal(0,2)x1e12 unique, S={ns} (95% Zipf(0.8) hits), "
                  f"density 0.5, {leaves} leaves")


def config3(scale: int = 1, device="cuda", seed: int = 0xC3, shard: int = 0, shards: int = 1) -> Inputs:
    """C3: R = 2*10^8 unique keys from 64 normal clusters (centres uniform
    in [0, 2^62), sigma 2^40; draws outside [0, 2^63) rejected); S = 2*10^9
    keys drawn uniformly from R (counter sampler).  RadixSpline with 18 radix
    bits, max error 32, table_factor 4.  ``shards``/``shard`` give rank
    ``shard`` its contiguous 1/shards of S; ``scale`` divides both sides."""
    nr, ns_total = 200_000_000 // scale, 2_000_000_000 // scale
    lo_s = ns_total * shard // shards
    ns = ns_total * (shard + 1) // shards - lo_s
    centres = (uniform63(64, seed ^ 0x31, 0, device) >> 1).to(torch.float64)

    def draw(c, o):
        return cluster_keys(c, seed, o, centres, float(2**40), device)

    rk = distinct_first(draw, nr, device)
    rp = fill_payloads(nr, seed ^ 0x34, device=device)
    sk = _gather_uniform(rk, ns, seed ^ 0x35, lo_s)
    s = Relation(sk, fill_payloads(ns, seed ^ 0x36, offset=lo_s, device=device), validate=False)
    return Inputs("c3", Relation(rk, rp, validate=False), s,
                  {"spline_error": 32, "radix_bits": 18, "table_factor": 4.0}, "spline-hash-inlj",
                  f"RadixSpline learned-hash INLJ: R={nr} clustered-normal unique, S={ns} of {ns_total} "
                  f"uniform from R, 18 radix bits, max error 32, P=4|R|")


def config4(scale: int = 0, device="cuda", seed: int = 0xC4, shard: int = 0) -> Inputs:
    """C4: R = 2^28 unique floor(2^40 * lognormal(0, 1.5)); S = 2^28 keys
    R_sorted[Zipf(1.0) rank] (duplicates); LSJ with 4096 partitions and a
    1% sample per relation (per-relation models, as the reference)."""
    nr = ns = (1 << 28) >> scale

    def draw(c, o):
        return lognormal_keys(c, seed, o, 1.5, float(2**40), device)

    rk = distinct_first(draw, nr, device)
    rp = fill_payloads(nr, seed ^ 0x41, device=device)
    srt = torch.sort(rk).values
    sk = srt[zipf_ranks(ns, nr, 1.0, seed ^ 0x42 ^ (shard << 40), device)]
    del srt
    s = Relation(sk, fill_payloads(ns, seed ^ 0x43 ^ (shard << 40), device=device), validate=False)
    return Inputs("c4", Relation(rk, rp, validate=False), s,
                  {"fanout": 4096, "sample_rate": 0.01}, "lsj",
                  f"LSJ: R={nr} lognormal(0,1.5)x2^40 unique, S={ns} Zipf(1.0) over R ranks, 4096 partitions, "
                  f"1% sample models")


def bijective63(i: torch.Tensor, seed: int) -> torch.Tensor:
    """A bijection of [0, 2^63): odd multiplies, adds and xorshifts mod 2^63."""
    m = MAX63
    x = (i + (seed & m)) & m
    for mul, sh in ((0x5851F42D4C957F2D, 29), (0x14057B7EF767814F, 31), (0x2545F4914F6CDD1D, 27)):
        x = (x * mul) & m  # odd multiplier: a bijection mod 2^63 (int64 wraps mod 2^64)
        x = x ^ (x >> sh)
    return x


def config5(scale: int = 0, device="cuda", seed: int = 0xC5, shard: int = 0, shards: int = 1) -> Inputs:
    """C5: R = S = 2*10^9 (per all GPUs): R unique uniform keys by a
    bijective 63-bit mix of the counter (no dedup needed), S = R[idx] with a
    uniform counter draw; rank ``shard`` holds the contiguous 1/shards of
    both relations.  LSJ with one shared model in the multi-GPU path."""
    n_total = 2_000_000_000 >> scale
    lo = n_total * shard // shards
    n = n_total * (shard + 1) // shards - lo
    idx = torch.arange(lo, lo + n, dtype=torch.int64, device=device)
    rk = bijective63(idx, seed)
    rp = fill_payloads(n, seed ^ 0x51, offset=lo, device=device)
    j = _mix(n, seed ^ 0x52, lo, device)
    sidx = ((j >> 1) & MAX63) % n_total  # uniform over all of R (every rank's)
    sk = bijective63(sidx, seed)
    sp = fill_payloads(n, seed ^ 0x53, offset=lo, device=device)
    return Inputs("c5", Relation(rk, rp, validate=False), Relation(sk, sp, validate=False),
                  {"fanout": 4096, "sample_rate": 0.01}, "lsj",
                  f"LSJ: R=S={n} of {n_total} uniform unique (bijective mix) / uniform from R")


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}
