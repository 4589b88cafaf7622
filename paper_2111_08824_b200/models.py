"""CDF models on the GPU (reference models.py): the two-level linear RMI,
the RadixSpline, and the scaled partition mapping both share.

Parameters live in device memory in the layout the kernels read: RMI
leaves as 32-B records {slope, intercept, clamp_lo, clamp_hi} (one DRAM
sector per leaf lookup) and interleaved {err_lo, err_hi}; spline points as
keys u64 + ranks f64 + a u32 radix table.  Evaluation is bit-identical to
the reference's numpy arithmetic (see csrc/lj_common.cuh).
"""

from __future__ import annotations

import ctypes
import os
import uuid
from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from .util import as_key_tensor, check_sorted, to_device_u64, to_numpy_u64


class PosPrediction(NamedTuple):
    pos: int
    lo: int
    hi: int


def _keys_arg(keys):
    scalar = np.ndim(keys) == 0 and not isinstance(keys, torch.Tensor)
    t = to_device_u64(np.atleast_1d(np.asarray(keys, dtype=np.uint64)) if scalar or not isinstance(keys, torch.Tensor) else keys)
    return t, scalar


class RecursiveModelIndex:
    """Two-level RMI: linear root routing to ``fanout`` linear leaves, with
    per-leaf clamps and exact residual bounds (models.py:39-143)."""

    def __init__(self, fanout: int = 1000):
        if fanout < 1:
            raise ValueError("fanout must be >= 1")
        self.fanout = int(fanout)
        self.trained_len = 0
        self.tag = None
        self.root_slope = 0.0
        self.root_intercept = 0.0
        self.leaves = None  # (m, 4) int64 view of LjLeaf records
        self.err = None     # (m, 2) int64 {err_lo, err_hi}

    def get_params(self) -> dict:
        return {"fanout": self.fanout}

    def fit(self, sorted_keys, stream=None) -> "RecursiveModelIndex":
        """models.py:57-110 on device (K10)."""
        keys = as_key_tensor(sorted_keys)
        if keys.numel() == 0:
            raise ValueError("cannot train on an empty key array")
        check_sorted(keys)
        lib = _lib.lib()
        n, m = keys.numel(), self.fanout
        root = torch.empty(2, dtype=torch.float64, device=keys.device)
        self.leaves = torch.empty((m, 4), dtype=torch.int64, device=keys.device)
        self.err = torch.empty((m, 2), dtype=torch.int64, device=keys.device)
        ws = _lib.workspace(lib.lj_rmi_fit_workspace_bytes(n, m), keys.device)
        _lib.check(lib.lj_rmi_fit(_lib.ptr(keys), n, m, _lib.ptr(root), _lib.ptr(self.leaves),
                                  _lib.ptr(self.err), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream)),
                   "rmi_fit")
        rs, ri = root.tolist()
        self.root_slope, self.root_intercept = float(rs), float(ri)
        self.trained_len = int(n)
        self.tag = uuid.uuid4().hex
        return self

    @classmethod
    def from_params(cls, root_slope, root_intercept, trained_len, leaf_slope, leaf_intercept, clamp_lo,
                    clamp_hi, err_lo, err_hi, device=None) -> "RecursiveModelIndex":
        """Adopt externally fitted parameters (e.g. the reference's own)."""
        m = int(np.asarray(leaf_slope).size)
        self = cls(m)
        rec = np.empty((m, 4), dtype=np.int64)
        rec[:, 0] = np.asarray(leaf_slope, dtype=np.float64).view(np.int64)
        rec[:, 1] = np.asarray(leaf_intercept, dtype=np.float64).view(np.int64)
        rec[:, 2] = np.asarray(clamp_lo, dtype=np.int64)
        rec[:, 3] = np.asarray(clamp_hi, dtype=np.int64)
        err = np.stack([np.asarray(err_lo, np.int64), np.asarray(err_hi, np.int64)], axis=1)
        dev = device or "cuda"
        self.leaves = torch.from_numpy(rec).to(dev)
        self.err = torch.from_numpy(np.ascontiguousarray(err)).to(dev)
        self.root_slope, self.root_intercept = float(root_slope), float(root_intercept)
        self.trained_len = int(trained_len)
        self.tag = uuid.uuid4().hex
        return self

    # -- host views of the parameters (reference attribute names) --
    def _rec(self):
        return self.leaves.cpu().numpy()

    @property
    def leaf_slope(self):
        return self._rec()[:, 0].view(np.float64).copy()

    @property
    def leaf_intercept(self):
        return self._rec()[:, 1].view(np.float64).copy()

    @property
    def clamp_lo(self):
        return self._rec()[:, 2].copy()

    @property
    def clamp_hi(self):
        return self._rec()[:, 3].copy()

    @property
    def err_lo(self):
        return self.err.cpu().numpy()[:, 0].copy()

    @property
    def err_hi(self):
        return self.err.cpu().numpy()[:, 1].copy()

    def c_struct(self) -> _lib.LjRmi:
        self._check_fitted()
        return _lib.LjRmi(self.root_slope, self.root_intercept, self.fanout, self.trained_len,
                          _lib.ptr(self.leaves), _lib.ptr(self.err))

    def _check_fitted(self):
        if self.trained_len == 0:
            raise ValueError("model is not fitted")

    def _predict(self, keys, want_pos=True, want_bounds=True, want_leaf=False, stream=None):
        self._check_fitted()
        k = to_device_u64(keys)
        n = k.numel()
        dev = k.device
        pos = torch.empty(n, dtype=torch.int64, device=dev) if want_pos else None
        lo = torch.empty(n, dtype=torch.int64, device=dev) if want_bounds else None
        hi = torch.empty(n, dtype=torch.int64, device=dev) if want_bounds else None
        leaf = torch.empty(n, dtype=torch.int64, device=dev) if want_leaf else None
        c = self.c_struct()
        _lib.check(_lib.lib().lj_rmi_predict(ctypes.byref(c), _lib.ptr(k), n, _lib.ptr(pos), _lib.ptr(lo),
                                             _lib.ptr(hi), _lib.ptr(leaf), _lib.stream_ptr(stream)),
                   "rmi_predict")
        return pos, lo, hi, leaf

    def predict_many(self, keys):
        """models.py:126-135 -> (pos, lo, hi) device tensors, bounds inclusive."""
        pos, lo, hi, _ = self._predict(keys)
        return pos, lo, hi

    def route_many(self, keys) -> torch.Tensor:
        """models.py:116-119 leaf of each key."""
        return self._predict(keys, want_pos=False, want_bounds=False, want_leaf=True)[3]

    def predict(self, key) -> PosPrediction:
        pos, lo, hi = self.predict_many(np.asarray([key], dtype=np.uint64))
        return PosPrediction(int(pos[0]), int(lo[0]), int(hi[0]))


def train_rmi(sorted_keys, fanout: int) -> RecursiveModelIndex:
    return RecursiveModelIndex(fanout=fanout).fit(sorted_keys)


class RadixSplineIndex:
    """Greedy-corridor spline over the CDF with a radix table on top
    (models.py:150-256).  The corridor fit is sequential and runs on the
    host in C++ (lj_spline_fit_host); evaluation runs on the GPU."""

    def __init__(self, max_error: int = 32, radix_bits: int = 18):
        if max_error < 1:
            raise ValueError("max_error must be >= 1")
        if not 1 <= radix_bits <= 30:
            raise ValueError("radix_bits must be in [1, 30]")
        self.max_error = int(max_error)
        self.radix_bits = int(radix_bits)
        self.trained_len = 0
        self.tag = None

    def get_params(self) -> dict:
        return {"max_error": self.max_error, "radix_bits": self.radix_bits}

    def fit(self, sorted_keys) -> "RadixSplineIndex":
        if (isinstance(sorted_keys, torch.Tensor) and sorted_keys.is_cuda and sorted_keys.numel() > 0
                and not os.environ.get("LJ_HOST_SPLINE_FIT")):
            return self._fit_device(sorted_keys)
        if isinstance(sorted_keys, torch.Tensor):
            host = to_numpy_u64(sorted_keys)
        else:
            host = np.ascontiguousarray(np.asarray(sorted_keys, dtype=np.uint64))
        if host.size == 0:
            raise ValueError("cannot train on an empty key array")
        if host.max() == np.uint64(0xFFFF_FFFF_FFFF_FFFF):
            raise ValueError("keys may not contain the reserved maximum key")
        n = host.size
        sk = np.empty(n, np.uint64)
        sr = np.empty(n, np.int64)
        rt = np.empty((1 << self.radix_bits) + 1, np.int64)
        npts = ctypes.c_int64(0)
        shift = ctypes.c_uint64(0)
        lib = _lib.load()
        rc = lib.lj_spline_fit_host(host.ctypes.data, n, self.max_error, self.radix_bits, sk.ctypes.data,
                                    sr.ctypes.data, rt.ctypes.data, ctypes.byref(npts), ctypes.byref(shift))
        if rc == _lib.LJ_E_INVALID:
            raise ValueError("keys must be sorted ascending")
        _lib.check(rc, "spline_fit")
        k = npts.value
        return self._adopt(sk[:k], sr[:k], rt, shift.value, n)

    def _fit_device(self, keys: torch.Tensor) -> "RadixSplineIndex":
        """models.py:171-219 on the device (lj_spline_fit): speculative
        greedy runs per chunk, spliced where they converge -- the host
        fit's knots exactly."""
        k = keys.contiguous()
        if bool((k == -1).any()):
            raise ValueError("keys may not contain the reserved maximum key")
        check_sorted(k)
        n = k.numel()
        dev = k.device
        kk = torch.empty(n, dtype=torch.int64, device=dev)
        rr = torch.empty(n, dtype=torch.int64, device=dev)
        rt = torch.empty((1 << self.radix_bits) + 1, dtype=torch.int64, device=dev)
        lib = _lib.lib()
        ws = _lib.workspace(lib.lj_spline_fit_workspace_bytes(n), dev)
        npts = ctypes.c_int64(0)
        shift = ctypes.c_uint64(0)
        _lib.check(lib.lj_spline_fit(_lib.ptr(k), n, self.max_error, self.radix_bits, _lib.ptr(kk), _lib.ptr(rr),
                                     _lib.ptr(rt), ctypes.byref(npts), ctypes.byref(shift), _lib.ptr(ws), ws.numel(),
                                     _lib.stream_ptr()), "spline_fit")
        kn = npts.value
        return self._adopt(to_numpy_u64(kk[:kn]), rr[:kn].cpu().numpy(), rt.cpu().numpy(), shift.value, n, device=dev)

    def _adopt(self, spline_keys, spline_ranks, radix_table, shift, trained_len, device=None):
        dev = device or "cuda"
        self.spline_keys = np.ascontiguousarray(spline_keys, dtype=np.uint64)
        self.spline_ranks = np.ascontiguousarray(spline_ranks, dtype=np.int64)
        self.radix_table = np.ascontiguousarray(radix_table, dtype=np.int64)
        self.shift = np.uint64(shift)
        self.trained_len = int(trained_len)
        # two words of padding: the staged probe bulk-copies whole 16-B words
        K = self.spline_keys.size
        self._d_keys = to_device_u64(np.concatenate([self.spline_keys, np.zeros(2, np.uint64)]), device=dev)[:K]
        self._d_ranks = torch.from_numpy(np.concatenate([self.spline_ranks.astype(np.float64),
                                                         np.zeros(2)])).to(dev)[:K]
        self._d_radix = torch.from_numpy(self.radix_table.astype(np.uint32).view(np.int32)).to(dev)
        self._build_aux(dev)
        self.tag = uuid.uuid4().hex
        return self

    use_aux = True  # class switch: the accelerator never changes a result

    def _build_aux(self, dev):
        """Exact sub-radix accelerator of the bounded spline search
        (lj_spline_aux_host; see LjSpline.aux)."""
        self._d_aux = self._d_sub = None
        if not self.use_aux or self.spline_keys.size < 2:
            return
        lib = _lib.load()
        nb = 1 << self.radix_bits
        aux = np.zeros(nb, dtype=np.uint64)
        ln = ctypes.c_int64(0)
        args = (self.spline_keys.ctypes.data, self.spline_keys.size, self.radix_table.ctypes.data, self.radix_bits,
                int(self.shift))
        _lib.check(lib.lj_spline_aux_host(*args, aux.ctypes.data, None, ctypes.byref(ln)), "spline_aux")
        if ln.value == 0:
            return
        sub = np.zeros(ln.value, dtype=np.uint32)
        _lib.check(lib.lj_spline_aux_host(*args, aux.ctypes.data, sub.ctypes.data, ctypes.byref(ln)), "spline_aux")
        self._d_aux = torch.from_numpy(aux.view(np.int64)).to(dev)
        self._d_sub = torch.from_numpy(sub.view(np.int32)).to(dev)

    @classmethod
    def from_params(cls, spline_keys, spline_ranks, radix_table, shift, trained_len, max_error, radix_bits,
                    device=None) -> "RadixSplineIndex":
        self = cls(max_error, radix_bits)
        return self._adopt(spline_keys, spline_ranks, radix_table, shift, trained_len, device)

    def c_struct(self) -> _lib.LjSpline:
        self._check_fitted()
        return _lib.LjSpline(self.spline_keys.size, self.trained_len, self.max_error, self.radix_bits,
                             int(self.shift), _lib.ptr(self._d_keys), _lib.ptr(self._d_ranks),
                             _lib.ptr(self._d_radix), _lib.ptr(self._d_aux), _lib.ptr(self._d_sub),
                             0 if self._d_sub is None else self._d_sub.numel())

    def _check_fitted(self):
        if self.trained_len == 0:
            raise ValueError("model is not fitted")

    def predict_many(self, keys, stream=None):
        """models.py:221-248 -> (pos, lo, hi) device tensors."""
        self._check_fitted()
        k = to_device_u64(keys)
        n = k.numel()
        pos, lo, hi = (torch.empty(n, dtype=torch.int64, device=k.device) for _ in range(3))
        c = self.c_struct()
        _lib.check(_lib.lib().lj_spline_predict(ctypes.byref(c), _lib.ptr(k), n, _lib.ptr(pos), _lib.ptr(lo),
                                                _lib.ptr(hi), _lib.stream_ptr(stream)), "spline_predict")
        return pos, lo, hi

    def predict(self, key) -> PosPrediction:
        pos, lo, hi = self.predict_many(np.asarray([key], dtype=np.uint64))
        return PosPrediction(int(pos[0]), int(lo[0]), int(hi[0]))


def train_radix_spline(sorted_keys, max_error: int, radix_bits: int) -> RadixSplineIndex:
    return RadixSplineIndex(max_error=max_error, radix_bits=radix_bits).fit(sorted_keys)


def partition_index(model, keys, num_partitions: int, stream=None):
    """models.py:285-299: clip(pos * P // trained_len, 0, P-1) in exact
    int64 on device.  Scalar in, int out; array in, device tensor out."""
    if num_partitions < 1:
        raise ValueError("num_partitions must be >= 1")
    scalar = np.ndim(keys) == 0 and not isinstance(keys, torch.Tensor)
    k = to_device_u64(np.atleast_1d(np.asarray(keys, dtype=np.uint64)) if not isinstance(keys, torch.Tensor) else keys)
    out = torch.empty(k.numel(), dtype=torch.int64, device=k.device)
    c = model.c_struct()
    lib = _lib.lib()
    if isinstance(model, RecursiveModelIndex):
        rc = lib.lj_rmi_partition_index(ctypes.byref(c), _lib.ptr(k), k.numel(), int(num_partitions),
                                        _lib.ptr(out), _lib.stream_ptr(stream))
    else:
        rc = lib.lj_spline_partition_index(ctypes.byref(c), _lib.ptr(k), k.numel(), int(num_partitions),
                                           _lib.ptr(out), _lib.stream_ptr(stream))
    _lib.check(rc, "partition_index")
    return int(out[0]) if scalar else out
