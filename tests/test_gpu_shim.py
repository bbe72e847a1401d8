"""The C++ drop-in shim (include/lutkan_b200.hpp) against the unmodified reference library:
tests/cpp/shim_parity.cpp swaps lutkan:: for lutkan_b200:: at the call sites of the reference's
own API and checks bytes, outputs, OobStats, argmax classes and exception types."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_parity")


@pytest.mark.gpu
def test_cpp_shim_against_reference_library():
    if not os.path.exists(BIN):
        pytest.skip("shim_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout and r.stdout.count("[PASS]") >= 10
