"""The reference's own known-answer unit tests for the integer search
(test_integer_search.cpp:57-121), replayed through the device path on every
integer-search kernel: the CUDA-core tile kernel (small grids, or forced), the
tensor-core kernel and the block-sum kernel."""
import os

import numpy as np
import pytest

from paper_1905_06228_b200 import configs, dic, _abi
from paper_1905_06228_b200.dic import BfsDomain, GridParams, IntegerMethod, RunConfig, SearchConfig, SubpixelMethod

pytestmark = pytest.mark.gpu
PATHS = {"legacy": {"DICB200_BFS_LEGACY": "1"}, "tensor": {"DICB200_BFS_TC": "1"}, "default": {}}


def _run(a, b, cfg, path):
    keys = ("DICB200_BFS_LEGACY", "DICB200_BFS_TC", "DICB200_BFS_BS")
    for k in keys:
        os.environ.pop(k, None)
    os.environ.update(PATHS[path])
    try:
        return dic.analyze_pair(dic.GrayImage(a), dic.GrayImage(b, 1), cfg).records
    finally:
        for k in keys:
            os.environ.pop(k, None)


def _cfg(M, R, step):
    return RunConfig(integer_method=IntegerMethod.bfs, subpixel_method=SubpixelMethod.none,
                     search=SearchConfig(search_radius=R, bfs_domain=BfsDomain.window),
                     grid=GridParams(half_width=M, spacing=step))


def _speckle(w, h, seed, dtype=_abi.U8, maxv=255):
    if dtype == _abi.U8:
        return configs.FrameSpec(w, h, _abi.U8, 255, seed, w * h // 60, (2.0, 4.0), (60.0, 200.0)).render()
    return configs.FrameSpec(w, h, _abi.U16, maxv, seed, w * h // 42, (1.5, 3.5), (0.23 * maxv, 0.78 * maxv)).render()


@pytest.mark.parametrize("path", sorted(PATHS))
@pytest.mark.parametrize("dtype", [_abi.U8, _abi.U16], ids=["u8", "u16"])
def test_exact_integer_shift_everywhere(gpu, path, dtype):
    """test_integer_search.cpp:57-69: a pure integer shift is found at every
    POI, with the full window counted (no degenerate windows in speckle)."""
    ref = _speckle(420, 400, 17, dtype, 4095)
    tgt = np.roll(np.roll(ref, -2, axis=0), 3, axis=1)  # content moves by (+3, -2)
    cfg = _cfg(20, 12, 10)
    r = _run(ref, tgt, cfg, path)
    assert len(r) >= 1024  # large enough for the tensor-core / block-sum kernels
    inner = (r["x"] < 420 - 20 - 3) & (r["y"] >= 20 + 2)  # subsets not wrapped by np.roll
    assert inner.mean() > 0.9
    assert np.all(r["integer_dx"][inner] == 3) and np.all(r["integer_dy"][inner] == -2)
    assert np.all(np.abs(r["zncc"][inner] - 1.0) < 1e-12)
    assert np.all(r["evaluations"][inner] == 25 * 25)


@pytest.mark.parametrize("path", sorted(PATHS))
@pytest.mark.parametrize("dtype", [_abi.U8, _abi.U16], ids=["u8", "u16"])
def test_ties_break_toward_smallest_dy_dx(gpu, path, dtype):
    """test_integer_search.cpp:104-121: on a period-8 checkerboard every
    displacement that is a multiple of 8 on both axes (or 4 mod 8 on both)
    correlates perfectly; with R = 8 the winner is the smallest (dy, dx) =
    (-8, -8) at every POI (R = 12 would make it (-12, -12))."""
    y, x = np.mgrid[0:400, 0:420]
    cb = np.where(((x % 8) < 4) ^ ((y % 8) < 4), 200, 50)
    cb = cb.astype(np.uint8) if dtype == _abi.U8 else (cb * 16).astype(np.uint16)
    r = _run(cb, cb, _cfg(20, 8, 10), path)
    assert len(r) >= 1024
    assert np.all(r["integer_dx"] == -8) and np.all(r["integer_dy"] == -8)
    assert np.all(np.abs(r["zncc"] - 1.0) < 1e-12)


def test_small_grid_tie_break_reference_case(gpu):
    """The reference's own 32x32 checkerboard case (M = 7, R = 8, POI (16, 16))."""
    y, x = np.mgrid[0:32, 0:32]
    cb = np.where(((x % 8) < 4) ^ ((y % 8) < 4), 200, 50).astype(np.uint8)
    r = _run(cb, cb, _cfg(7, 8, 1), "default")
    k = np.nonzero((r["x"] == 16) & (r["y"] == 16))[0]
    assert len(k) == 1
    assert (r["integer_dx"][k[0]], r["integer_dy"][k[0]]) == (-8, -8)


def test_understated_bits_fail_loudly(gpu):
    """ADVICE r1 (host.cu bits trust): a caller declaring fewer significant bits
    than the data holds must not get silently overflowed u32 sums — the host
    entry point fails the pair, the device entry point marks every record."""
    import ctypes as C

    ref = _speckle(420, 400, 17, _abi.U16, 4095)
    tgt = np.roll(ref, 3, axis=1)
    cfg = _cfg(20, 12, 10)
    good = dic.analyze_pair(dic.GrayImage(ref), dic.GrayImage(tgt, 1), cfg).records
    assert np.all(good["status"] == 0)
    a, b = dic.GrayImage(ref).as_c(), dic.GrayImage(tgt, 1).as_c()
    a.bits = 8  # understated: the data holds 12 bits
    c = cfg.to_c()
    recs = np.zeros(len(good), dtype=_abi.record_dtype())
    cnt = C.c_size_t(0)
    st = dic.lib().dicb200_analyze_pair(C.byref(a), C.byref(b), C.byref(c), 0, recs.ctypes.data, len(recs), C.byref(cnt))
    assert st == 1 and b"declared dicb200_image.bits" in dic.lib().dicb200_last_error_message()
    assert np.all(recs["status"] == 12)
    # a correct declaration (12 bits) passes the guard and keeps the records
    a.bits = 12
    st = dic.lib().dicb200_analyze_pair(C.byref(a), C.byref(b), C.byref(c), 0, recs.ctypes.data, len(recs), C.byref(cnt))
    assert st == 0
    for f in ("integer_dx", "integer_dy", "evaluations", "status"):
        assert np.array_equal(recs[f], good[f]), f


def test_bits_guard_along_a_sequence(gpu):
    """The declared-width guard checks a repeated reference frame once per
    stream (cached flag) and every target: with a fixed-first sequence on the
    two compute streams, an understated target fails only its own pair, an
    understated reference fails every pair, and correct declarations pass."""
    import ctypes as C

    ref = _speckle(420, 400, 23, _abi.U16, 4095)
    frames = [ref] + [np.roll(ref, k, axis=1) for k in (1, 2, 3, 4, 5)]
    cfg = _cfg(20, 12, 10)
    cfg.reference_policy = dic.ReferencePolicy.fixed_first
    gi = [dic.GrayImage(f, i) for i, f in enumerate(frames)]
    good = dic.analyze_sequence(gi, cfg)
    assert all(not f.error and np.all(f.records["status"] == 0) for f in good)
    n = len(good[0].records)

    def run(bits):
        imgs = (_abi.Image * len(gi))()
        for i, g in enumerate(gi):
            imgs[i] = g.as_c()
            imgs[i].bits = bits[i]
        c = cfg.to_c()
        fields = (_abi.FieldC * (len(gi) - 1))()
        bufs = []
        for i in range(len(gi) - 1):
            b = np.zeros(n, dtype=_abi.record_dtype())
            bufs.append(b)
            fields[i].records = C.cast(b.ctypes.data, C.POINTER(_abi.PoiRecordC))
            fields[i].capacity = n
        st = dic.lib().dicb200_analyze_sequence(imgs, len(gi), C.byref(c), fields, len(gi) - 1)
        return st, [fields[i].status for i in range(len(gi) - 1)], bufs

    st, status, bufs = run([12] * 6)
    assert st == 0 and status == [0] * 5
    for i in range(5):
        for f in ("integer_dx", "integer_dy", "evaluations", "status"):
            assert np.array_equal(bufs[i][f], good[i].records[f]), (i, f)
    st, status, bufs = run([12, 12, 12, 8, 12, 12])  # frame 3 (pair 2) understated
    assert st == 0 and status == [0, 0, 1, 0, 0], status
    for i in (0, 1, 3, 4):
        assert np.array_equal(bufs[i]["integer_dx"], good[i].records["integer_dx"])
    st, status, _ = run([8, 12, 12, 12, 12, 12])  # the reference understated: every pair fails
    assert st == 0 and status == [1] * 5, status
