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
    # 3 integer + 3 fractional frame pairs, 6 sequences (2 policies x serial / image-parallel / serial mPSO)
    assert r.stdout.count(" ok") == 12 and "dimension mismatch" in r.stdout


@pytest.mark.parametrize("chunk", ["1", "2", "3"])
def test_cpp_shim_chunked_sequence_calls(gpu, chunk):
    """The shim hands long sequences to the library in chunks of pairs (packing
    the next chunk while the device runs); forced here on the short check
    sequences: fields, pair indices, RNG keys (mPSO evaluations) and the
    mid-sequence pair error must be those of one call."""
    if not os.path.exists(BIN):
        pytest.skip("shim_check not built (reference sources absent at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300, env={**os.environ, "DICB200_SHIM_CHUNK": chunk})
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" ok") == 12
