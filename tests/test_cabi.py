"""The C-ABI library loads without a GPU and exports exactly what
include/lj_b200.h declares; host-only entry points run on the CPU."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "lj_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lj_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2111_08824_b200 import _lib

    return _lib.load(build_if_missing=True)


def test_every_declared_symbol_is_exported(lib):
    from paper_2111_08824_b200 import _lib
    from paper_2111_08824_b200.build import LIB

    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(lj_[a-z0-9_]+)", out))
    declared = _declared()
    assert declared, "header parse failed"
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    # the ctypes binding covers the whole header, one to one
    assert sorted(_lib.SIGNATURES) == declared


def test_library_is_sm100a_only():
    from paper_2111_08824_b200.build import LIB

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_version_and_no_device(lib):
    assert lib.lj_version() == 1
    import torch

    if not torch.cuda.is_available():
        assert lib.lj_device_ok() == 0


def test_invalid_argument_codes_without_device(lib):
    from paper_2111_08824_b200 import _lib

    rc = lib.lj_rmi_fit(None, 0, 4, None, None, None, None, 0, None)
    assert rc == _lib.LJ_E_INVALID
    assert b"empty" in lib.lj_last_error()


@pytest.mark.parametrize("name", ["unif63", "lognorm1e12", "clusters", "seq_h", "dups", "linear", "tiny",
                                  "single", "dbl_collide"])
def test_host_spline_fit_matches_reference(golden, lib, name):
    """lj_spline_fit_host (models.py:171-219 in C++) picks exactly the
    reference's spline points, ranks and radix table."""
    from paper_2111_08824_b200.models import RadixSplineIndex

    d = golden("models")[name]
    keys = np.ascontiguousarray(d["keys"], dtype=np.uint64)
    me, rb = int(d["sp_max_error"]), int(d["sp_radix_bits"])
    n = keys.size
    sk = np.empty(n, np.uint64)
    sr = np.empty(n, np.int64)
    rt = np.empty((1 << rb) + 1, np.int64)
    npts, shift = ctypes.c_int64(0), ctypes.c_uint64(0)
    rc = lib.lj_spline_fit_host(keys.ctypes.data, n, me, rb, sk.ctypes.data, sr.ctypes.data, rt.ctypes.data,
                                ctypes.byref(npts), ctypes.byref(shift))
    assert rc == 0
    k = npts.value
    assert np.array_equal(sk[:k], d["sp_keys"])
    assert np.array_equal(sr[:k], d["sp_ranks"])
    assert np.array_equal(rt, d["sp_radix_table"])
    assert shift.value == int(d["sp_shift"])
    # and the oracle agrees with both
    sp = oracle.spline_fit(keys, me, rb)
    assert np.array_equal(sp.spline_keys, sk[:k])
    with pytest.raises(ValueError):
        RadixSplineIndex(me, rb).fit(keys[::-1].copy() if n > 1 else np.array([3, 1], np.uint64))
