"""Device-array helpers (reference util.py): uint64 keys live in CUDA int64
tensors bit for bit; the reserved sentinel key; chunking and mixing."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

# util.py:8 reserved padding value; never a data key
SENTINEL_KEY = np.uint64(0xFFFF_FFFF_FFFF_FFFF)
_SIGN = -(2**63)


def to_device_u64(x, *, copy: bool = False, device=None) -> torch.Tensor:
    """numpy / list / torch -> contiguous CUDA int64 tensor holding the u64 bits."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype == torch.uint64:
            t = t.view(torch.int64)
        elif t.dtype != torch.int64:
            t = t.to(torch.int64)
        t = t.to(device or "cuda")
        t = t.contiguous()
        return t.clone() if copy and t.data_ptr() == x.data_ptr() else t
    a = np.ascontiguousarray(np.asarray(x, dtype=np.uint64)).reshape(-1)
    return torch.from_numpy(a.view(np.int64).copy()).to(device or "cuda")


def to_numpy_u64(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().to("cpu").contiguous().numpy().view(np.uint64)
    return np.asarray(t, dtype=np.uint64)


def as_key_tensor(keys, *, name: str = "keys", copy: bool = False) -> torch.Tensor:
    """util.py:15-22: 1-D uint64 keys, the reserved maximum key rejected."""
    if isinstance(keys, (np.ndarray, list, tuple)) and np.ndim(keys) != 1:
        raise ValueError(f"{name} must be one-dimensional")
    if isinstance(keys, torch.Tensor) and keys.dim() != 1:
        raise ValueError(f"{name} must be one-dimensional")
    t = to_device_u64(keys, copy=copy)
    if t.numel() and bool((t == -1).any()):
        raise ValueError(f"{name} may not contain the reserved maximum key")
    return t


def unsigned_order(t: torch.Tensor) -> torch.Tensor:
    """Signed view whose order equals the unsigned order of the u64 bits."""
    return t ^ _SIGN


def check_sorted(keys: torch.Tensor, *, name: str = "keys") -> None:
    if keys.numel() > 1:
        o = unsigned_order(keys)
        if bool((o[1:] < o[:-1]).any()):
            raise ValueError(f"{name} must be sorted ascending")


def chunk_bounds(n: int, workers: int) -> np.ndarray:
    """util.py:62-64 equal chunks: workers+1 offsets covering [0, n)."""
    step = n / workers
    b = np.array([int(i * step) for i in range(workers)] + [n], dtype=np.int64)
    return b


def sort_pairs(keys: torch.Tensor, payloads: torch.Tensor, stream=None):
    """Stable device sort of (key, payload) by unsigned key (data.py:84-86)."""
    lib = _lib.lib()
    n = keys.numel()
    ko = torch.empty_like(keys)
    po = torch.empty_like(payloads)
    if n == 0:
        return ko, po
    ws = _lib.workspace(lib.lj_sort_pairs_workspace_bytes(n), keys.device)
    _lib.check(lib.lj_sort_pairs(_lib.ptr(keys), _lib.ptr(payloads), _lib.ptr(ko), _lib.ptr(po), n, 0, 64,
                                 _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream)), "sort_pairs")
    return ko, po


def exclusive_offsets(counts: torch.Tensor):
    """counts -> (offsets[n], total) for materialisation (plumbing)."""
    if counts.numel() == 0:
        return counts.new_zeros(0), 0
    inc = torch.cumsum(counts, 0)
    return inc - counts, int(inc[-1].item())


def mix64(x):
    """util.py:30-44 SplitMix64 finaliser (host, numpy)."""
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return np.uint64(z) if np.ndim(x) == 0 else z
