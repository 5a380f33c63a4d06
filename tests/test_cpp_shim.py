"""INTEGRATION.md's C++ drop-in (include/treeattn_b200.hpp:
treeattn::b200::run_iteration over the C ABI) compiled against the reference's
own headers and run beside the reference's run_iteration on the same trees
and content (tests/cpp/shim_run_iteration.cpp, built by oracle/Makefile where
/root/reference exists; the binary travels with the repo)."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "shim_test")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/shim_test not built (needs /root/reference)")
def test_cpp_shim_matches_reference_run_iteration():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.strip().endswith("OK")
    assert r.stdout.count("relative_error") == 22
