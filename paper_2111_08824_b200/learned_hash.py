"""Spline-keyed chained hash index on the GPU (reference learned_hash.py).

Chains are keyed by partition_index(spline, key, table_len) and keep
insertion order.  The build sorts (bucket, original index) pairs with a
stable device radix sort; the probe (K5) evaluates the spline, finds the
chain and scans it in one kernel, reducing to the checksum on device.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .data import Relation
from .models import RadixSplineIndex
from .util import as_key_tensor, exclusive_offsets, sort_pairs, to_device_u64, to_numpy_u64


class SplineHashIndex:
    """Bucket-chained hash table keyed by a scaled spline CDF prediction."""

    def __init__(self, max_error: int = 32, radix_bits: int = 18, table_factor: float = 4.0):
        if table_factor < 1.0:
            raise ValueError("table_factor must be >= 1")
        self.max_error = max_error
        self.radix_bits = radix_bits
        self.table_factor = float(table_factor)
        self.n = 0

    def get_params(self) -> dict:
        return {"max_error": self.max_error, "radix_bits": self.radix_bits, "table_factor": self.table_factor}

    def fit(self, relation: Relation, model: RadixSplineIndex | None = None) -> "SplineHashIndex":
        """learned_hash.py:35-40: spline on the sorted build keys, then chains."""
        if model is None:
            sk, _ = sort_pairs(relation.keys, relation.payloads)
            model = RadixSplineIndex(self.max_error, self.radix_bits).fit(sk)
        table_len = max(1, int(round(self.table_factor * len(relation))))
        return self._index_with(model, relation, table_len)

    @classmethod
    def from_model(cls, model, relation: Relation, table_len: int) -> "SplineHashIndex":
        """learned_hash.py:42-53: index under an externally trained model."""
        self = cls.__new__(cls)
        self.max_error = getattr(model, "max_error", 0)
        self.radix_bits = getattr(model, "radix_bits", 0)
        self.table_factor = table_len / max(1, len(relation))
        return self._index_with(model, relation, table_len)

    def _index_with(self, model, relation: Relation, table_len: int) -> "SplineHashIndex":
        self.model = model
        self.n = n = len(relation)
        self.table_len = P = int(table_len)
        self.stride = (P // n) if n and P % n == 0 else 1
        dev = relation.device
        self.entries = torch.empty(2 * max(n, 1), dtype=torch.int64, device=dev)
        self.starts = torch.zeros(P // self.stride + 1, dtype=torch.int32, device=dev)
        self.slots, self.nslots = None, 0
        if n == 0:
            return self
        lib = _lib.lib()
        ws = _lib.workspace(lib.lj_spline_hash_build_workspace_bytes(n, P), dev)
        c = model.c_struct()
        _lib.check(lib.lj_spline_hash_build(ctypes.byref(c), _lib.ptr(relation.keys), _lib.ptr(relation.payloads),
                                            n, P, _lib.ptr(self.entries), _lib.ptr(self.starts), _lib.ptr(ws),
                                            ws.numel(), _lib.stream_ptr()), "spline_hash_build")
        del ws
        self._build_slots(relation)
        return self

    build_slots = True  # class switch: the probe table never changes a result

    def _build_slots(self, relation: Relation) -> None:
        """The probe table (LjSplineHash.slots, lj_hash_staged.cu): the
        entries in key order at slot max(2 pos, previous + 1), gaps marked by
        payload 0 -- built only when every payload is nonzero (else the
        chains are probed)."""
        self.slots = None
        self.segs = None
        self.nslots = 0
        if not self.build_slots or self.model.trained_len != self.n:
            return
        lib = _lib.lib()
        dev = relation.device
        sk, sp = sort_pairs(relation.keys, relation.payloads)
        ws = _lib.workspace(lib.lj_spline_slots_workspace_bytes(self.n),
                            dev)
        plan = torch.zeros(3, dtype=torch.int64, device=dev)
        c = self.model.c_struct()
        _lib.check(lib.lj_spline_slots_plan(ctypes.byref(c), _lib.ptr(sk), _lib.ptr(sp), self.n, _lib.ptr(plan),
                                            _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "spline_slots_plan")
        nslots, zeros, dups = (int(v) for v in plan.cpu().tolist())
        if zeros:
            return
        self.slots_unique = int(dups == 0)
        self.segs = torch.empty(4 * self.model.spline_keys.size + 8, dtype=torch.float64, device=dev)
        _lib.check(lib.lj_spline_segments(ctypes.byref(c), _lib.ptr(self.segs), _lib.stream_ptr()), "spline_segments")
        self.slots = torch.empty(2 * nslots, dtype=torch.int64, device=dev)
        _lib.check(lib.lj_spline_slots_fill(_lib.ptr(sk), _lib.ptr(sp), self.n, _lib.ptr(self.slots), nslots,
                                            _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "spline_slots_fill")
        self.nslots = nslots

    def c_struct(self) -> _lib.LjSplineHash:
        slots = getattr(self, "slots", None)
        return _lib.LjSplineHash(self.model.c_struct(), self.n, self.table_len, self.stride,
                                 _lib.ptr(self.entries), _lib.ptr(self.starts), _lib.ptr(slots),
                                 getattr(self, "nslots", 0), getattr(self, "slots_unique", 0), 0,
                                 _lib.ptr(getattr(self, "segs", None)) if slots is not None else None)

    @property
    def _keys(self) -> np.ndarray:
        return to_numpy_u64(self.entries[0 : 2 * self.n : 2].contiguous())

    @property
    def _payloads(self) -> np.ndarray:
        return to_numpy_u64(self.entries[1 : 2 * self.n : 2].contiguous())

    def collision_fraction(self) -> float:
        """learned_hash.py:68-79: inserts that landed in an occupied bucket."""
        if self.n == 0:
            return 0.0
        st = self.starts.to(torch.int64)
        occupied = int((st[1:] != st[:-1]).sum().item())
        return (self.n - occupied) / self.n

    def join_checksum(self, s_keys: torch.Tensor, s_payloads: torch.Tensor, out: torch.Tensor | None = None,
                      accumulate: bool = False, stream=None) -> torch.Tensor:
        """K5 -> device int64[4] {count, sum, xor, 0}."""
        if out is None:
            out = torch.zeros(4, dtype=torch.int64, device=s_keys.device)
        c = self.c_struct()
        _lib.check(_lib.lib().lj_spline_hash_probe(ctypes.byref(c), _lib.ptr(s_keys), _lib.ptr(s_payloads),
                                                   s_keys.numel(), _lib.ptr(out), int(bool(accumulate)),
                                                   _lib.stream_ptr(stream)), "spline_hash_probe")
        return out

    def bucket_scratch(self, n: int, device=None) -> dict:
        lib = _lib.lib()
        dev = device or self.entries.device
        tl = self.model.trained_len
        cap = lib.lj_spline_hash_bucket_capacity(n, tl)
        nb = lib.lj_spline_hash_bucket_bins(tl)
        return {"pairs": torch.empty(2 * max(cap, 1), dtype=torch.int64, device=dev),
                "reg": torch.empty(2 * nb + 2, dtype=torch.int64, device=dev), "nbins": nb,
                "ws": _lib.workspace(max(lib.lj_spline_hash_bucket_est_workspace_bytes(ctypes.byref(self.c_struct()), n),
                                         8), dev)}

    def join_checksum_buffered(self, s_keys: torch.Tensor, s_payloads: torch.Tensor,
                               out: torch.Tensor | None = None, accumulate: bool = False, scratch: dict | None = None,
                               stream=None) -> torch.Tensor:
        """Group S by predicted-position window on device, then K5 over the
        grouped records (chain offsets and entries reused from L2).  Same
        result words as ``join_checksum``."""
        n = s_keys.numel()
        if out is None:
            out = torch.zeros(4, dtype=torch.int64, device=s_keys.device)
        if self.n == 0 or n == 0:
            if not accumulate:
                out.zero_()
            return out
        scratch = scratch or self.bucket_scratch(n, s_keys.device)
        self.bucket_records(s_keys, s_payloads, scratch, stream)
        self.probe_records(n, scratch, out, accumulate, stream)
        return out

    def bucket_records(self, s_keys: torch.Tensor, s_payloads: torch.Tensor, scratch: dict, stream=None) -> None:
        """S grouped by approximate-position window into scratch["pairs"]
        (one pass, estimated-capacity regions; scratch["reg"] = layout)."""
        lib = _lib.lib()
        c = self.c_struct()
        ws = scratch["ws"]
        if s_keys.data_ptr() % 16 or s_payloads.data_ptr() % 16:
            s_keys, s_payloads = s_keys.clone(), s_payloads.clone()
        _lib.check(lib.lj_spline_hash_bucket_est(ctypes.byref(c), _lib.ptr(s_keys), _lib.ptr(s_payloads),
                                                 s_keys.numel(), _lib.ptr(scratch["pairs"]), _lib.ptr(scratch["reg"]),
                                                 _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream)),
                   "spline_hash_bucket_est")

    def probe_records(self, n: int, scratch: dict, out: torch.Tensor, accumulate: bool = False, stream=None) -> None:
        """K5 over the grouped records bucket_records left in scratch (n is
        implied by the regions)."""
        c = self.c_struct()
        ws = scratch["ws"]
        _lib.check(_lib.lib().lj_spline_hash_probe_regions(ctypes.byref(c), _lib.ptr(scratch["pairs"]),
                                                           _lib.ptr(scratch["reg"]), scratch["nbins"], _lib.ptr(ws),
                                                           ws.numel(), _lib.ptr(out), int(bool(accumulate)),
                                                           _lib.stream_ptr(stream)), "spline_hash_probe_regions")
        return out

    def probe_batch(self, keys):
        """learned_hash.py:81-96 -> (payloads, source_index) device tensors;
        per probe, matches in chain (insertion) order."""
        k = as_key_tensor(keys)
        n = k.numel()
        if self.n == 0 or n == 0:
            e = torch.empty(0, dtype=torch.int64, device=k.device)
            return e, e.clone()
        lib = _lib.lib()
        c = self.c_struct()
        counts = torch.empty(n, dtype=torch.int64, device=k.device)
        _lib.check(lib.lj_spline_hash_count(ctypes.byref(c), _lib.ptr(k), n, _lib.ptr(counts), _lib.stream_ptr()),
                   "spline_hash_count")
        offsets, total = exclusive_offsets(counts)
        pays = torch.empty(total, dtype=torch.int64, device=k.device)
        src = torch.empty(total, dtype=torch.int64, device=k.device)
        if total:
            _lib.check(lib.lj_spline_hash_collect(ctypes.byref(c), _lib.ptr(k), n, _lib.ptr(offsets), _lib.ptr(pays),
                                                  _lib.ptr(src), _lib.stream_ptr()), "spline_hash_collect")
        return pays, src

    def probe(self, key) -> np.ndarray:
        pays, _ = self.probe_batch(np.asarray([key], dtype=np.uint64))
        return to_numpy_u64(pays)


def build_spline_hash(relation: Relation, max_error: int = 32, radix_bits: int = 18,
                      table_factor: float = 4.0) -> SplineHashIndex:
    return SplineHashIndex(max_error, radix_bits, table_factor).fit(relation)
