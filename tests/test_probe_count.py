"""Host check of the closed-form reference probe count used by the staged
GRMI probe (csrc/lj_probe_count.h): exhaustive over small arrays and all
(start, lb, re) placements, against the reference loop (gapped.py:86-160)."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None and not os.path.exists("/usr/bin/g++"), reason="no C++ compiler")
def test_closed_form_probe_count_matches_loop(tmp_path):
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    exe = tmp_path / "pcc"
    subprocess.run([cxx, "-O2", "-o", str(exe), os.path.join(ROOT, "tools", "probe_count_check.cpp")], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert out.startswith("OK"), out
