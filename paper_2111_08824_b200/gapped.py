"""Gapped RMI index on the GPU (reference gapped.py:206-342).

``fit`` sorts R on device, fits the RMI on device (K10) unless a model is
given, and places the entries by model-based insertion (K11).  The fused
probe (K1) joins a whole S relation against the index and reduces the
result to its checksum on device; ``search_from``/``lookup_batch``
materialise pairs with the reference's exact per-probe semantics.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from .data import Relation
from .models import RecursiveModelIndex
from .results import LookupStats
from .util import as_key_tensor, exclusive_offsets, sort_pairs, to_device_u64, to_numpy_u64


class GappedRmiIndex:
    """Gapped arrays filled by model-based insertion, probed via the RMI plus
    exponential search.  Read-only once fitted; concurrent probes are safe."""

    def __init__(self, gap_factor: float = 4.0, rmi_fanout: int = 1000):
        if gap_factor < 1.0:
            raise ValueError("gap_factor must be >= 1")
        self.gap_factor = float(gap_factor)
        self.rmi_fanout = int(rmi_fanout)
        self.n = 0
        self.slot_count = 0
        self.rmi = None

    def get_params(self) -> dict:
        return {"gap_factor": self.gap_factor, "rmi_fanout": self.rmi_fanout}

    def fit(self, relation: Relation, model: RecursiveModelIndex | None = None, stream=None) -> "GappedRmiIndex":
        n = len(relation)
        self.n = n
        if n == 0:
            self.rmi = None
            self.slot_count = 0
            return self
        sk, sp = sort_pairs(relation.keys, relation.payloads, stream)
        self.rmi = model if model is not None else RecursiveModelIndex(self.rmi_fanout).fit(sk, stream)
        L = int(round(self.gap_factor * n))  # gapped.py:233
        self.slot_count = L
        dev = sk.device
        self.slots = torch.empty(2 * L, dtype=torch.int64, device=dev)
        self.bitmap_words = torch.empty((L + 31) // 32, dtype=torch.int32, device=dev)
        flag = torch.empty(1, dtype=torch.int32, device=dev)
        lib = _lib.lib()
        ws = _lib.workspace(lib.lj_grmi_build_workspace_bytes(n, L), dev)
        c = self.rmi.c_struct()
        _lib.check(lib.lj_grmi_build(ctypes.byref(c), _lib.ptr(sk), _lib.ptr(sp), n, L, _lib.ptr(self.slots),
                                     _lib.ptr(self.bitmap_words), _lib.ptr(flag), _lib.ptr(ws), ws.numel(),
                                     _lib.stream_ptr(stream)), "grmi_build")
        self.payload_nonzero = int(flag.item())
        return self

    # -- reference attribute views (host copies, for inspection/tests) --
    @property
    def gkeys(self) -> np.ndarray:
        return to_numpy_u64(self.slots[0::2].contiguous())

    @property
    def gpayloads(self) -> np.ndarray:
        return to_numpy_u64(self.slots[1::2].contiguous())

    @property
    def bitmap(self) -> np.ndarray:
        w = self.bitmap_words.cpu().numpy().view(np.uint32)
        bits = np.unpackbits(w.view(np.uint8), bitorder="little")
        return bits[: self.slot_count].astype(bool)

    def c_struct(self) -> _lib.LjGrmi:
        return _lib.LjGrmi(self.rmi.c_struct(), self.n, self.slot_count, _lib.ptr(self.slots),
                           _lib.ptr(self.bitmap_words), self.payload_nonzero, 0)

    # -- probing --
    def join_checksum(self, s_keys: torch.Tensor, s_payloads: torch.Tensor, out: torch.Tensor | None = None,
                      accumulate: bool = False, stream=None) -> torch.Tensor:
        """K1: fused INLJ of S against the index -> device int64[4]
        {count, sum, xor, search_steps} (no host sync)."""
        if out is None:
            out = torch.zeros(4, dtype=torch.int64, device=s_keys.device)
        if self.n == 0:
            if not accumulate:
                out.zero_()
            return out
        c = self.c_struct()
        _lib.check(_lib.lib().lj_grmi_probe(ctypes.byref(c), _lib.ptr(s_keys), _lib.ptr(s_payloads),
                                            s_keys.numel(), _lib.ptr(out), int(bool(accumulate)),
                                            _lib.stream_ptr(stream)), "grmi_probe")
        return out

    def bucket_scratch(self, n: int, device=None) -> dict:
        """Preallocated device scratch for ``join_checksum_buffered`` over up
        to n probes (bucketed records + bin bounds + partition workspace)."""
        lib = _lib.lib()
        dev = device or self.slots.device
        L = self.slot_count
        return {"pairs": torch.empty(2 * max(lib.lj_leaf_bucket_capacity(n, L), 1), dtype=torch.int64, device=dev),
                "regions": torch.empty(lib.lj_leaf_bucket_regions(L), dtype=torch.int64, device=dev),
                "ws": _lib.workspace(lib.lj_leaf_bucket_workspace_bytes(n, L), dev),
                "work": torch.zeros(1, dtype=torch.int64, device=dev)}

    def join_checksum_buffered(self, s_keys: torch.Tensor, s_payloads: torch.Tensor,
                               out: torch.Tensor | None = None, accumulate: bool = False, scratch: dict | None = None,
                               stream=None) -> torch.Tensor:
        """Request-Buffer analogue (buffers.py:103-150): group S on device by
        the window of predicted gapped slots it will search (K4, shared-memory
        privatised partition), then run K1 over the grouped records, so each
        warp walks one index segment that stays in L1/L2.  Same result words
        as ``join_checksum``."""
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
        """K4: S grouped by key-range window into scratch["pairs"] / ["starts"]."""
        lib = _lib.lib()
        g = self.c_struct()
        ws = scratch["ws"]
        _lib.check(lib.lj_leaf_bucket(ctypes.byref(g), _lib.ptr(s_keys), _lib.ptr(s_payloads), s_keys.numel(),
                                      _lib.ptr(scratch["pairs"]), _lib.ptr(scratch["regions"]), _lib.ptr(ws),
                                      ws.numel(), _lib.stream_ptr(stream)), "leaf_bucket")

    # staging image (lj_grmi_stage_image_build) for indexes at least this
    # large: below it the 207 KB-per-window image costs more memory than the
    # staging it saves
    STAGE_IMAGE_MIN_SLOTS = 1 << 24

    def stage_image(self, stream=None):
        """The probe's per-window staging precomputed once (built on first
        use; None when the index is not probed through staged windows or is
        smaller than STAGE_IMAGE_MIN_SLOTS)."""
        img = getattr(self, "_stage_img", False)
        if img is not False:
            return img
        self._stage_img = None
        if self.slot_count >= self.STAGE_IMAGE_MIN_SLOTS and not os.environ.get("LJ_NO_STAGE_IMAGE"):
            lib = _lib.lib()
            g = self.c_struct()
            nbytes = lib.lj_grmi_stage_image_bytes(ctypes.byref(g))
            if nbytes:
                img = torch.empty(nbytes, dtype=torch.uint8, device=self.slots.device)
                _lib.check(lib.lj_grmi_stage_image_build(ctypes.byref(g), _lib.ptr(img), nbytes,
                                                         _lib.stream_ptr(stream)), "grmi_stage_image_build")
                self._stage_img = img
        return self._stage_img

    def probe_records(self, n: int, scratch: dict, out: torch.Tensor, accumulate: bool = False, stream=None,
                      count_steps: bool = True) -> None:
        """Staged K1 over the n records bucket_records left in scratch.
        ``count_steps=False`` leaves the reference's probe counter
        (search_steps, out[3]) out: the staged search never needs the model's
        prediction, so its evaluation goes with the counter (ablation; the
        checksum words are unchanged)."""
        g = self.c_struct()
        img = self.stage_image(stream)
        flags = int(bool(accumulate)) | (0 if count_steps else 2)
        _lib.check(_lib.lib().lj_grmi_probe_bucketed_img(ctypes.byref(g), _lib.ptr(scratch["pairs"]),
                                                         _lib.ptr(scratch["regions"]), _lib.ptr(scratch["work"]),
                                                         _lib.ptr(img), _lib.ptr(out), flags,
                                                         _lib.stream_ptr(stream)), "grmi_probe_bucketed")
        return out

    def _predict_slots(self, keys: torch.Tensor) -> torch.Tensor:
        out = torch.empty(keys.numel(), dtype=torch.int64, device=keys.device)
        c = self.c_struct()
        _lib.check(_lib.lib().lj_grmi_predict_slots(ctypes.byref(c), _lib.ptr(keys), keys.numel(), _lib.ptr(out),
                                                    _lib.stream_ptr()), "grmi_predict_slots")
        return out

    def predict_slots(self, keys) -> torch.Tensor:
        """gapped.py:290-292 model-predicted gapped slot of each probe key."""
        return self._predict_slots(as_key_tensor(keys))

    def leaf_of(self, keys) -> torch.Tensor:
        """gapped.py:263-265 leaf segment each key routes to."""
        return self.rmi.route_many(keys)

    def search(self, slots0, keys):
        """gapped.py:86-160 per-probe (slot or -1, probe count)."""
        k = to_device_u64(keys)
        s0 = to_device_u64(slots0)
        slot = torch.empty_like(k)
        probes = torch.empty_like(k)
        c = self.c_struct()
        _lib.check(_lib.lib().lj_grmi_search(ctypes.byref(c), _lib.ptr(s0), _lib.ptr(k), k.numel(),
                                             _lib.ptr(slot), _lib.ptr(probes), _lib.stream_ptr()), "grmi_search")
        return slot, probes

    def search_from(self, slots0, keys, stats: LookupStats | None = None):
        """gapped.py:294-321 -> (payloads, source_index, found) over all
        matches, as device tensors."""
        k = to_device_u64(keys)
        n = k.numel()
        s0 = None if slots0 is None else to_device_u64(slots0)
        lefts = torch.empty(n, dtype=torch.int64, device=k.device)
        counts = torch.empty_like(lefts)
        probes = torch.empty_like(lefts)
        lib = _lib.lib()
        c = self.c_struct()
        if n:
            _lib.check(lib.lj_grmi_count(ctypes.byref(c), _lib.ptr(s0), _lib.ptr(k), n, _lib.ptr(lefts),
                                         _lib.ptr(counts), _lib.ptr(probes), _lib.stream_ptr()), "grmi_count")
        offsets, total = exclusive_offsets(counts)
        pays = torch.empty(total, dtype=torch.int64, device=k.device)
        src = torch.empty(total, dtype=torch.int64, device=k.device)
        if total:
            _lib.check(lib.lj_grmi_collect(ctypes.byref(c), _lib.ptr(k), n, _lib.ptr(lefts), _lib.ptr(offsets),
                                           _lib.ptr(pays), _lib.ptr(src), _lib.stream_ptr()), "grmi_collect")
        if stats is not None:
            stats.search_steps += int(probes.sum().item()) if n else 0
            stats.predictions += n
        return pays, src, counts > 0

    def lookup_batch(self, keys, stats: LookupStats | None = None):
        """gapped.py:323-338 all matches for a probe batch."""
        k = as_key_tensor(keys)
        if self.n == 0 or k.numel() == 0:
            e = torch.empty(0, dtype=torch.int64, device=k.device)
            return e, e.clone(), torch.zeros(k.numel(), dtype=torch.bool, device=k.device)
        if stats is not None:
            leaf = self.leaf_of(k)
            stats.leaf_switches += int((leaf[1:] != leaf[:-1]).sum().item())
        return self.search_from(None, k, stats)

    def lookup(self, key, stats: LookupStats | None = None):
        """gapped.py:267-281 payload of the first real slot of ``key``, or None."""
        if self.n == 0:
            return None
        pays, _, found = self.lookup_batch(np.asarray([key], dtype=np.uint64), stats)
        if not bool(found[0]):
            return None
        return np.uint64(to_numpy_u64(pays[:1])[0])

    def lookup_range(self, key, stats: LookupStats | None = None) -> np.ndarray:
        """gapped.py:283-288 every payload stored under ``key``, left to right."""
        if self.n == 0:
            return np.empty(0, dtype=np.uint64)
        pays, _, _ = self.lookup_batch(np.asarray([key], dtype=np.uint64), stats)
        return to_numpy_u64(pays)


def build_grmi(relation: Relation, gap_factor: float = 4.0, rmi_fanout: int = 1000) -> GappedRmiIndex:
    return GappedRmiIndex(gap_factor=gap_factor, rmi_fanout=rmi_fanout).fit(relation)
