"""Device-resident relations (reference data.py:65-89, 181-192).

A ``Relation`` holds two CUDA int64 tensors carrying uint64 keys and
payloads (struct-of-arrays, 8 B each per tuple).  Host inputs are copied to
the device once at construction; device tensors are adopted without a copy
(the zero-copy hand-off a GPU pipeline wants).  Keys equal to the reserved
sentinel are rejected exactly like the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .util import as_key_tensor, sort_pairs, to_device_u64, to_numpy_u64


class Relation:
    """Columnar key/payload store on the GPU.  Treated as immutable."""

    __slots__ = ("keys", "payloads")

    def __init__(self, keys, payloads, *, validate: bool = True):
        k = as_key_tensor(keys) if validate else to_device_u64(keys)
        p = to_device_u64(payloads, device=k.device)
        if k.shape != p.shape:
            raise ValueError("keys and payloads must have equal length")
        self.keys = k
        self.payloads = p

    def __len__(self) -> int:
        return int(self.keys.numel())

    @property
    def device(self):
        return self.keys.device

    def sorted_by_key(self) -> "Relation":
        k, p = sort_pairs(self.keys, self.payloads)
        return Relation(k, p, validate=False)

    def numpy(self) -> tuple[np.ndarray, np.ndarray]:
        return to_numpy_u64(self.keys), to_numpy_u64(self.payloads)

    def slice(self, lo: int, hi: int) -> "Relation":
        return Relation(self.keys[lo:hi], self.payloads[lo:hi], validate=False)

    def __repr__(self) -> str:
        return f"Relation(n={len(self)}, device={self.device})"


def fill_payloads(n: int, seed: int, offset: int = 0, device=None, stream=None) -> torch.Tensor:
    """data.py:181-192 positional payloads mix64(i + mix64(seed)) | 1."""
    out = torch.empty(int(n), dtype=torch.int64, device=device or "cuda")
    if n:
        lib = _lib.lib()
        _lib.check(lib.lj_fill_payloads(_lib.ptr(out), int(n), int(offset), int(seed) & (2**64 - 1),
                                        _lib.stream_ptr(stream)), "fill_payloads")
    return out


def make_relation(keys, seed: int) -> Relation:
    """Attach the reference's deterministic nonzero payloads to ``keys``."""
    k = as_key_tensor(keys)
    return Relation(k, fill_payloads(k.numel(), seed, device=k.device), validate=False)
