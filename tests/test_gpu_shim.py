"""The drop-in C++ API (include/mcf_gpu.hpp) against the reference itself.

oracle/_ref/shim_check is compiled (in the container that has the reference
tree) from tests/cpp/shim_check.cpp with the reference's headers and linked to
libmcf_b200.so: every mcf::gpu:: operator must reproduce mcf:: bit for bit.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "shim_check")


def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/shim_check not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "PASS" in r.stdout
