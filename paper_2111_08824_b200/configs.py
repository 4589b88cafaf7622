"""Seeded synthetic inputs of the five BASELINE configurations, generated
on the device (BASELINE.json ``configs``).

Size interpretations (pinned): "16M" = 2^24, "256M" = 2^28, "200M" =
2*10^8, "2B" = 2*10^9.  Keys are uint64 < 2^63; payloads uint64.

Integer parts use counter-based SplitMix64 draws (``mix64(seed ^ i)``),
bit-identical anywhere.  The lognormal / normal draws use float64 on the
device (Box-Muller on two counter draws), so the host never regenerates
them: parity tests copy the device inputs to the CPU oracle.  Duplicates
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
    u1 = _unit(n, seed ^ 0xA5A5, offset, device)
    u2 = _unit(n, seed ^ 0x5A5A, offset, device)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


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
    w = torch.arange(1, N + 1, dtype=torch.float64, device=device).pow(-s)
    cdf = torch.cumsum(w, 0)
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
        v = torch.floor(1e12 * torch.exp(2.0 * normal(c, seed, o, device)))
        return torch.clamp(v, 0, float(2**63 - 1024)).to(torch.int64)

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


CONFIGS = {"c1": config1, "c2": config2}
