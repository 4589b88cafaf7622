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

    @classmethod
    def on_host(cls, keys, payloads) -> "Relation":
        """A relation left in (pinned) HOST memory, as the reference's numpy
        relations are: the join runners copy it to the device inside their
        timed region (S streamed in chunks, overlapped with the probe) and
        validate its keys there.  ``keys``/``payloads``: numpy uint64 or CPU
        int64 tensors."""
        def host(x):
            if isinstance(x, torch.Tensor):
                t = x.view(torch.int64) if x.dtype == torch.uint64 else x
            else:
                t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.uint64)).view(np.int64))
            if t.device.type != "cpu" or t.dim() != 1:
                raise ValueError("host relations take 1-D CPU arrays")
            return t.contiguous() if t.is_pinned() else t.contiguous().pin_memory()

        self = cls.__new__(cls)
        self.keys, self.payloads = host(keys), host(payloads)
        if self.keys.shape != self.payloads.shape:
            raise ValueError("keys and payloads must have equal length")
        return self

    @property
    def is_host(self) -> bool:
        return self.keys.device.type == "cpu"

    def to_device(self, device=None) -> "Relation":
        """The device copy of a host relation (keys validated); a device
        relation is returned as is."""
        if not self.is_host:
            return self
        dev = device or "cuda"
        return Relation(self.keys.to(dev, non_blocking=True), self.payloads.to(dev, non_blocking=True))

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


class RecordRelation:
    """A relation held as n interleaved 16-B records {key, payload} on the
    GPU (an int64 [n, 2] tensor) -- what the range shuffle of the
    distributed LSJ delivers.  ``lsj_join`` partitions it in place
    (lj_lsj_partition_regions_rec); ``keys`` / ``payloads`` are strided views,
    ``columns()`` the contiguous copy every other consumer takes."""

    __slots__ = ("records",)

    def __init__(self, records: torch.Tensor):
        if records.dim() != 2 or records.shape[1] != 2 or records.dtype != torch.int64 or not records.is_cuda:
            raise ValueError("records must be a CUDA int64 [n, 2] tensor")
        self.records = records.contiguous()

    @property
    def keys(self) -> torch.Tensor:
        return self.records[:, 0]

    @property
    def payloads(self) -> torch.Tensor:
        return self.records[:, 1]

    def __len__(self) -> int:
        return int(self.records.shape[0])

    @property
    def device(self):
        return self.records.device

    def columns(self) -> "Relation":
        return Relation(self.records[:, 0].contiguous(), self.records[:, 1].contiguous(), validate=False)


def make_relation(keys, seed: int) -> Relation:
    """Attach the reference's deterministic nonzero payloads to ``keys``."""
    k = as_key_tensor(keys)
    return Relation(k, fill_payloads(k.numel(), seed, device=k.device), validate=False)


# ------------------------------------------------- key files (data.py:195-216)


class CorruptKeyFileError(ValueError):
    """data.py: a key file whose size disagrees with its count header."""


def write_keys_file(path, keys) -> None:
    """data.py:195-202: 8-byte LE count header plus LE uint64 keys."""
    k = to_numpy_u64(keys) if isinstance(keys, torch.Tensor) else np.ascontiguousarray(np.asarray(keys, np.uint64))
    with open(path, "wb") as fh:
        np.array([k.size], dtype="<u8").tofile(fh)
        k.astype("<u8").tofile(fh)


def load_keys_file(path, device=None) -> torch.Tensor:
    """data.py:205-216 loaded straight to the device: the file is read into
    pinned host memory and copied with one H2D transfer.  Returns the keys as
    a CUDA int64 tensor (uint64 bits), bit-exact."""
    import os

    size = os.path.getsize(path)
    if size < 8:
        raise CorruptKeyFileError(f"{path}: missing count header")
    with open(path, "rb") as fh:
        count = int(np.fromfile(fh, dtype="<u8", count=1)[0])
        if size != 8 + 8 * count:
            raise CorruptKeyFileError(f"{path}: header says {count} keys but file holds {(size - 8) // 8}")
        host = torch.empty(count, dtype=torch.int64, pin_memory=True)
        if count:
            fh.readinto(memoryview(host.numpy()).cast("B"))
    return host.to(device or "cuda", non_blocking=False)


def relation_from_keys_file(path, seed: int, device=None) -> Relation:
    """A relation over a key file with the positional payload rule
    (data.py:181-192), built on the device."""
    keys = load_keys_file(path, device)
    return Relation(keys, fill_payloads(keys.numel(), seed, device=keys.device))
