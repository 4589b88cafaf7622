import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name: str) -> dict:
    """tests/golden/<name>.npz -> {case: {field: array}} (see oracle/make_golden.py)."""
    out: dict = {}
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        for key in z.files:
            if "/" in key:
                case, field = key.split("/", 1)
                out.setdefault(case, {})[field] = z[key]
            else:
                out[key] = z[key]
    return out


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get


def rmi_from_fixture(d, prefix=""):
    import oracle

    return oracle.Rmi(
        float(d[prefix + "root"][0]),
        float(d[prefix + "root"][1]),
        int(d[prefix + "trained_len"]),
        np.ascontiguousarray(d[prefix + "leaf_slope"]),
        np.ascontiguousarray(d[prefix + "leaf_intercept"]),
        np.ascontiguousarray(d[prefix + "clamp_lo"]),
        np.ascontiguousarray(d[prefix + "clamp_hi"]),
        np.ascontiguousarray(d[prefix + "err_lo"]),
        np.ascontiguousarray(d[prefix + "err_hi"]),
    )


def spline_from_fixture(d, n, max_error, radix_bits):
    import oracle

    return oracle.Spline(
        np.ascontiguousarray(d["sp_keys"], dtype=np.uint64),
        np.ascontiguousarray(d["sp_ranks"], dtype=np.int64),
        np.ascontiguousarray(d["sp_radix_table"], dtype=np.int64),
        int(d["sp_shift"]),
        int(n),
        int(max_error),
        int(radix_bits),
    )
