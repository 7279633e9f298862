"""GPU: the C++ drop-in surface (include/mpzch_b200.hpp) is source-compatible with the
reference's C++ API.  tests/cpp/drop_in_parity.cpp compiles ONE test body against
mpzch:: (the reference library, oracle/_ref) and mpzch_b200:: (this repo) and compares
every ProbeResult, the final identity/metadata arrays of every shard and the error text."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "drop_in_parity")


@pytest.mark.gpu
def test_cpp_drop_in_matches_reference_api():
    if not os.path.exists(BIN):
        pytest.skip("drop_in_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN, "90"], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
