"""GPU: the C++ drop-in shim (include/dic_b200/pipeline.hpp) compiled INSIDE
the reference build (oracle/_ref/shim_check, built by oracle/Makefile where
/root/reference exists) reproduces dic::analyze_pair and rethrows pair-level
errors as dic::Error; dic::b200::analyze_sequence reproduces
dic::analyze_sequence (both policies, serial and image-parallel, a pair-level
error mid-sequence)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "shim_check")


def test_cpp_shim_matches_reference_analyze_pair(gpu):
    if not os.path.exists(BIN):
        pytest.skip("shim_check not built (reference sources absent at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    # 3 integer + 3 fractional frame pairs, 4 sequences (2 policies x serial / image-parallel)
    assert r.stdout.count(" ok") == 10 and "dimension mismatch" in r.stdout
