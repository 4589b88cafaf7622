"""ctypes binding of the C ABI in ``include/lj_b200.h`` (csrc/liblj_b200.so).

There is no CPU fallback: every compute entry point of this package goes
through this library on a CUDA device, and fails loudly (``LjError`` /
``RuntimeError``) when the library or the device is missing.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .build import LIB

# diagnostics: load an alternative build of the same ABI (e.g. a tuning variant)
LIB = os.environ.get("LJ_LIB", LIB)

_c_void_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_size_t = ctypes.c_size_t

LJ_OK = 0
LJ_E_INVALID = -1
LJ_E_CUDA = -2
LJ_E_WORKSPACE = -3
LJ_E_NCCL = -4
LJ_E_UNSUPPORTED = -5

SENTINEL = 0xFFFF_FFFF_FFFF_FFFF


class LjError(RuntimeError):
    """A CUDA / workspace failure reported by the C library."""


class LjLeaf(ctypes.Structure):
    _fields_ = [("slope", ctypes.c_double), ("icpt", ctypes.c_double), ("clamp_lo", _i64), ("clamp_hi", _i64)]


class LjRmi(ctypes.Structure):
    _fields_ = [("root_slope", ctypes.c_double), ("root_icpt", ctypes.c_double), ("m", _i64), ("n", _i64),
                ("leaves", _c_void_p), ("err", _c_void_p), ("root_dev", _c_void_p)]


class LjGrmi(ctypes.Structure):
    _fields_ = [("model", LjRmi), ("n", _i64), ("L", _i64), ("slots", _c_void_p), ("bitmap", _c_void_p),
                ("payload_nonzero", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class LjSpline(ctypes.Structure):
    _fields_ = [("npts", _i64), ("n", _i64), ("max_error", _i64), ("radix_bits", _i64), ("shift", _u64),
                ("keys", _c_void_p), ("ranks", _c_void_p), ("radix", _c_void_p), ("aux", _c_void_p),
                ("sub", _c_void_p), ("nsub", _i64)]


class LjSplineHash(ctypes.Structure):
    _fields_ = [("model", LjSpline), ("n", _i64), ("table_len", _i64), ("stride", _i64),
                ("entries", _c_void_p), ("starts", _c_void_p), ("slots", _c_void_p), ("nslots", _i64),
                ("slots_unique", ctypes.c_int32), ("_pad", ctypes.c_int32), ("segs", _c_void_p)]


class LjLsjModel(ctypes.Structure):
    _fields_ = [("rmi", LjRmi), ("nbins", _i64), ("pb", _c_void_p), ("table", _c_void_p), ("sample", _c_void_p),
                ("nsample", _i64)]


# name -> (restype, argtypes); mirrors include/lj_b200.h one to one
_P = _c_void_p
SIGNATURES = {
    "lj_last_error": (ctypes.c_char_p, []),
    "lj_version": (_int, []),
    "lj_device_ok": (_int, []),
    "lj_fill_payloads": (_int, [_P, _i64, _i64, _u64, _P]),
    "lj_fill_mix64": (_int, [_P, _i64, _i64, _u64, _P]),
    "lj_gather_uniform": (_int, [_P, _i64, _i64, _u64, _P, _i64, _P]),
    "lj_fill_normal": (_int, [_P, _i64, _i64, _u64, _P]),
    "lj_spline_slots_workspace_bytes": (_size_t, [_i64]),
    "lj_lsj_run_workspace_bytes": (_size_t, [_i64, _i64, ctypes.c_double]),
    "lj_nccl_available": (_int, []),
    "lj_nccl_comm_init_all": (_int, [_int, _P, _P]),
    "lj_nccl_comm_destroy": (_int, [_P]),
    "lj_reduce_sums_workspace_bytes": (_size_t, [_int]),
    "lj_reduce_sums": (_int, [_int, _P, _P, _P, _P, _P]),
    "lj_lsj_run_multi_workspace_bytes": (_size_t, [_int, _i64, _i64, _i64, _i64, _i64, ctypes.c_double]),
    "lj_lsj_run_multi": (_int, [_int, _P, _P, _P, _P, _P, _P, _P, _P, _P, _i64, _i64, ctypes.c_double, _u64, _P, _P,
                                _P, _P]),
    "lj_lsj_run": (_int, [_P, _P, _i64, _P, _P, _i64, ctypes.c_double, _u64, _P, _P, _size_t, _P]),
    "lj_lsj_run_rec": (_int, [_P, _i64, _P, _i64, ctypes.c_double, _u64, _P, _P, _size_t, _P]),
    "lj_spline_segments": (_int, [ctypes.POINTER(LjSpline), _P, _P]),
    "lj_spline_slots_plan": (_int, [ctypes.POINTER(LjSpline), _P, _P, _i64, _P, _P, _size_t, _P]),
    "lj_spline_slots_fill": (_int, [_P, _P, _i64, _P, _i64, _P, _size_t, _P]),
    "lj_fill_lognormal": (_int, [_P, _i64, _i64, _u64, ctypes.c_double, ctypes.c_double, ctypes.c_double, _P]),
    "lj_fill_cluster": (_int, [_P, _i64, _i64, _u64, _P, _int, ctypes.c_double, ctypes.c_double, _P]),
    "lj_sort_pairs_workspace_bytes": (_size_t, [_i64]),
    "lj_sort_pairs": (_int, [_P, _P, _P, _P, _i64, _int, _int, _P, _size_t, _P]),
    "lj_rmi_fit_workspace_bytes": (_size_t, [_i64, _i64]),
    "lj_rmi_fit": (_int, [_P, _i64, _i64, _P, _P, _P, _P, _size_t, _P]),
    "lj_rmi_predict": (_int, [ctypes.POINTER(LjRmi), _P, _i64, _P, _P, _P, _P, _P]),
    "lj_rmi_partition_index": (_int, [ctypes.POINTER(LjRmi), _P, _i64, _i64, _P, _P]),
    "lj_rmi_probe": (_int, [ctypes.POINTER(LjRmi), _P, _P, _i64, _P, _P, _i64, _P, _int, _P]),
    "lj_grmi_build_workspace_bytes": (_size_t, [_i64, _i64]),
    "lj_grmi_build": (_int, [ctypes.POINTER(LjRmi), _P, _P, _i64, _i64, _P, _P, _P, _P, _size_t, _P]),
    "lj_grmi_predict_slots": (_int, [ctypes.POINTER(LjGrmi), _P, _i64, _P, _P]),
    "lj_grmi_search": (_int, [ctypes.POINTER(LjGrmi), _P, _P, _i64, _P, _P, _P]),
    "lj_grmi_probe": (_int, [ctypes.POINTER(LjGrmi), _P, _P, _i64, _P, _int, _P]),
    "lj_grmi_count": (_int, [ctypes.POINTER(LjGrmi), _P, _P, _i64, _P, _P, _P, _P]),
    "lj_grmi_collect": (_int, [ctypes.POINTER(LjGrmi), _P, _i64, _P, _P, _P, _P, _P]),
    "lj_leaf_bucket_bins": (_int, [_i64]),
    "lj_leaf_bucket_regions": (_int, [_i64]),
    "lj_leaf_bucket_capacity": (_i64, [_i64, _i64]),
    "lj_leaf_bucket_workspace_bytes": (_size_t, [_i64, _i64]),
    "lj_leaf_bucket": (_int, [ctypes.POINTER(LjGrmi), _P, _P, _i64, _P, _P, _P, _size_t, _P]),
    "lj_grmi_probe_bucketed": (_int, [ctypes.POINTER(LjGrmi), _P, _P, _P, _P, _int, _P]),
    "lj_grmi_stage_image_bytes": (_size_t, [ctypes.POINTER(LjGrmi)]),
    "lj_grmi_stage_image_build": (_int, [ctypes.POINTER(LjGrmi), _P, _size_t, _P]),
    "lj_grmi_probe_bucketed_img": (_int, [ctypes.POINTER(LjGrmi), _P, _P, _P, _P, _P, _int, _P]),
    "lj_grmi_probe_pairs": (_int, [ctypes.POINTER(LjGrmi), _P, _i64, _P, _int, _P]),
    "lj_spline_fit_host": (_int, [_P, _i64, _i64, _i64, _P, _P, _P, _P, _P]),
    "lj_spline_fit_workspace_bytes": (_size_t, [_i64]),
    "lj_spline_fit": (_int, [_P, _i64, _i64, _i64, _P, _P, _P, _P, _P, _P, _size_t, _P]),
    "lj_spline_aux_host": (_int, [_P, _i64, _P, _i64, _u64, _P, _P, _P]),
    "lj_spline_predict": (_int, [ctypes.POINTER(LjSpline), _P, _i64, _P, _P, _P, _P]),
    "lj_spline_partition_index": (_int, [ctypes.POINTER(LjSpline), _P, _i64, _i64, _P, _P]),
    "lj_spline_hash_build_workspace_bytes": (_size_t, [_i64, _i64]),
    "lj_spline_hash_build": (_int, [ctypes.POINTER(LjSpline), _P, _P, _i64, _i64, _P, _P, _P, _size_t, _P]),
    "lj_spline_hash_probe": (_int, [ctypes.POINTER(LjSplineHash), _P, _P, _i64, _P, _int, _P]),
    "lj_spline_hash_bucket_workspace_bytes": (_size_t, [_i64, _i64]),
    "lj_spline_hash_bucket": (_int, [ctypes.POINTER(LjSplineHash), _P, _P, _i64, _P, _P, _P, _size_t, _P]),
    "lj_spline_hash_probe_grouped": (_int, [ctypes.POINTER(LjSplineHash), _P, _i64, _P, _int, _P]),
    "lj_keybin_workspace_bytes": (_size_t, [_i64]),
    "lj_keybin_eval": (_int, [_P, _i64, _P, _i64, _P, _P, _size_t, _P]),
    "lj_lsj_key_bounds": (_int, [ctypes.POINTER(LjLsjModel), _P, _P, _size_t, _P]),
    "lj_lsj_shuffle_workspace_bytes": (_size_t, [_i64, _i64]),
    "lj_lsj_shuffle_count": (_int, [ctypes.POINTER(LjLsjModel), _P, _P, _i64, _P, _P, _size_t, _P]),
    "lj_lsj_shuffle_scatter": (_int, [ctypes.POINTER(LjLsjModel), _P, _P, _i64, _P, _P, _size_t, _P]),
    "lj_spline_hash_bucket_bins": (_i64, [_i64]),
    "lj_spline_hash_bucket_capacity": (_i64, [_i64, _i64]),
    "lj_spline_hash_bucket_est_workspace_bytes": (_size_t, [ctypes.POINTER(LjSplineHash), _i64]),
    "lj_spline_hash_bucket_est": (_int, [ctypes.POINTER(LjSplineHash), _P, _P, _i64, _P, _P, _P, _size_t, _P]),
    "lj_spline_hash_probe_regions": (_int, [ctypes.POINTER(LjSplineHash), _P, _P, _i64, _P, _size_t, _P, _int, _P]),
    "lj_spline_hash_count": (_int, [ctypes.POINTER(LjSplineHash), _P, _i64, _P, _P]),
    "lj_spline_hash_collect": (_int, [ctypes.POINTER(LjSplineHash), _P, _i64, _P, _P, _P, _P]),
    "lj_lsj_sample_workspace_bytes": (_size_t, [_i64]),
    "lj_lsj_sample": (_int, [_P, _i64, _i64, _u64, _P, _P, _size_t, _P]),
    "lj_lsj_sample_strided": (_int, [_P, _i64, _i64, _i64, _u64, _P, _P, _size_t, _P]),
    "lj_lsj_bins_workspace_bytes": (_size_t, [_i64]),
    "lj_lsj_bins": (_int, [ctypes.POINTER(LjRmi), _P, _i64, _i64, _P, _P, _P, _size_t, _P]),
    "lj_lsj_bins_from_bounds": (_int, [_P, _i64, _i64, _P, _P]),
    "lj_lsj_partition_workspace_bytes": (_size_t, [_i64, _i64]),
    "lj_lsj_partition": (_int, [ctypes.POINTER(LjLsjModel), _P, _P, _i64, _P, _P, _P, _size_t, _P]),
    "lj_lsj_sort_workspace_bytes": (_size_t, [_i64, _i64]),
    "lj_lsj_sort": (_int, [ctypes.POINTER(LjLsjModel), _P, _P, _i64, _P, _P, _size_t, _P, _P]),
    "lj_lsj_sort_regions": (_int, [ctypes.POINTER(LjLsjModel), _P, _P, _i64, _P, _P, _P, _size_t, _P, _P]),
    "lj_lsj_partition_regions": (_int, [ctypes.POINTER(LjLsjModel), _P, _P, _i64, _P, _P, _P, _size_t, _P]),
    "lj_lsj_partition_regions_rec": (_int, [ctypes.POINTER(LjLsjModel), _P, _i64, _P, _P, _P, _size_t, _P]),
    "lj_lsj_partition_regions_capacity": (_i64, [_i64, _i64]),
    "lj_lsj_partition_regions_workspace_bytes": (_size_t, [_i64, _i64]),
    "lj_lsj_ref_bounds": (_int, [ctypes.POINTER(LjRmi), _P, _i64, _i64, _P, _P]),
    "lj_lsj_join_workspace_bytes": (_size_t, [_i64]),
    "lj_lsj_join": (_int, [ctypes.POINTER(LjLsjModel), _P, _i64, _P, _P, _i64, _int, _P, _P, _P, _P, _P, _int,
                           _P, _size_t, _P]),
}

_lib = None


def load(build_if_missing: bool = False):
    """Load the library (no device needed).  Raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        if not build_if_missing:
            raise RuntimeError(
                f"CUDA library {LIB} is not built; run `python -m paper_2111_08824_b200.build` "
                "(there is no CPU fallback)"
            )
        from .build import build

        build()
    lib = ctypes.CDLL(LIB)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_device_checked = False


def lib():
    """The library, after checking that a CUDA device of cc 10.x is present."""
    global _device_checked
    lb = load()
    if not _device_checked:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2111_08824_b200 needs a CUDA device (B200, sm_100a); none is visible")
        torch.cuda.init()
        if lb.lj_device_ok() != 1:
            raise RuntimeError("paper_2111_08824_b200 is built for sm_100a; the visible device is not cc 10.x")
        _device_checked = True
    return lb


def check(rc: int, what: str = "") -> None:
    if rc == LJ_OK:
        return
    msg = (load().lj_last_error() or b"").decode(errors="replace")
    if rc == LJ_E_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise LjError(f"{what}: rc={rc}: {msg}")


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device arrays must be contiguous CUDA tensors"
    return int(t.data_ptr())


def workspace(nbytes: int, device=None) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device or "cuda")
