"""CPU: the C-ABI library loads, exports every symbol its headers declare, and
its host-side logic (grid, pairs, partitions, defaults, errors) matches the
reference. No compute calls here: without a GPU the analysis entry points must
refuse (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1905_06228_b200 import _abi, configs, dic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("dicb200.h", "dicb200_synth.h")]


def declared_symbols():
    names = set()
    for h in HEADERS:
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names |= set(re.findall(r"\b(dicb200_\w+)\s*\(", txt))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    L = dic.lib()
    syms = declared_symbols()
    assert "dicb200_analyze_pair" in syms and "dicb200_analyze_sequence" in syms
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {dic.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_abi_version_and_defaults():
    L = dic.lib()
    assert L.dicb200_abi_version() == 1
    c = _abi.RunConfigC()
    L.dicb200_default_config(C.byref(c))
    d = dic.RunConfig().to_c()  # the Python mirror of the reference defaults
    for f, _ in c._fields_:
        assert getattr(c, f) == getattr(d, f), f
    # reference defaults (integer_search.hpp:14-23, subpixel.hpp:41-44, pipeline.hpp:27-49)
    assert (c.search_radius, c.particle_count, c.max_generations, c.half_width, c.spacing, c.margin) == (25, 50, 5, 15, 10, -1)
    assert (c.stop_threshold, c.c1, c.c2, c.tol, c.max_iter) == (0.995, 2.0, 2.0, 0.01, 20)
    assert c.bfs_domain == _abi.BFS_WHOLE_IMAGE and c.integer_method == _abi.INT_MPSO


@pytest.mark.parametrize("w,h,m,s,mg", [(256, 256, 10, 16, 20), (100, 60, 15, 7, 0), (2048, 2048, 20, 5, 25),
                                        (512, 512, 15, 10, 30), (33, 47, 4, 3, 2), (31, 31, 15, 1, 15)])
def test_grid_matches_oracle(port, w, h, m, s, mg):
    got = np.array(dic.grid_subsets(w, h, m, s, mg), dtype=np.int32).reshape(-1, 2)
    assert np.array_equal(got, port.grid(w, h, m, s, mg))


def test_grid_errors():
    with pytest.raises(dic.DicError, match="half_width must be >= 1"):
        dic.grid_subsets(64, 64, 0, 5, 5)
    with pytest.raises(dic.DicError, match="spacing must be >= 1"):
        dic.grid_subsets(64, 64, 5, 0, 5)
    with pytest.raises(dic.DicError, match="image too small"):
        dic.grid_subsets(8, 8, 5, 1, 0)


def test_baseline_grid_sizes():
    # S per pair
    assert configs.c1().subsets_per_pair() == 196
    assert configs.c2().subsets_per_pair() == 2116
    assert configs.c3().subsets_per_pair() == 14400
    assert configs.c4().subsets_per_pair() == 160000
    assert configs.c5(2).subsets_per_pair() == 39601


def test_sequence_pairs_and_partitions():
    # pipeline.cpp:43-69; SPEC examples: 9 subsets over 4 workers -> {3,2,2,2}
    assert dic.sequence_pairs(dic.ReferencePolicy.update_every_pair, 4) == [(0, 1), (1, 2), (2, 3)]
    assert dic.sequence_pairs(dic.ReferencePolicy.fixed_first, 4) == [(0, 1), (0, 2), (0, 3)]
    assert [b - a for a, b in dic.partition_ranges(9, 4)] == [3, 2, 2, 2]
    assert dic.partition_ranges(8, 4) == [(0, 2), (2, 4), (4, 6), (6, 8)]
    assert dic.partition_ranges(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    with pytest.raises(dic.DicError):
        dic.partition_ranges(3, 0)
    with pytest.raises(dic.DicError, match="insufficient images"):
        dic.sequence_pairs(dic.ReferencePolicy.fixed_first, 1)


def test_dimension_mismatch_and_no_cpu_fallback():
    a = dic.GrayImage(np.zeros((40, 40), np.uint8))
    b = dic.GrayImage(np.zeros((40, 41), np.uint8))
    with pytest.raises(dic.DicError, match="dimension mismatch"):
        dic.analyze_pair(a, b, dic.RunConfig())
    if dic.lib().dicb200_device_count() == 0:
        # no GPU: the product refuses instead of computing on the CPU
        with pytest.raises(RuntimeError, match="no CUDA device"):
            dic.analyze_pair(a, a, dic.RunConfig(grid=dic.GridParams(5, 5, -1),
                                                  search=dic.SearchConfig(search_radius=3)))


def test_grayimage_gray_level_mapping():
    """Integer levels in [0, 65535] map losslessly to u8 / u16 (the exact
    integer kernels); any other finite levels stay doubles (the fp64 path, as
    the C++ shim passes them); non-finite levels are rejected (image.cpp:14-22)."""
    g = dic.GrayImage(np.full((8, 8), 300.0))
    assert g.pixels().dtype == np.uint16 and g.at(0, 0) == 300.0 and g.as_c().dtype == _abi.U16
    f = dic.GrayImage(np.array([[1.5, 0.0], [254.99609375, 17.25]]))
    assert f.pixels().dtype == np.float64 and f.at(0, 1) == 254.99609375 and f.as_c().dtype == _abi.F64
    for frac in (np.full((8, 8), 300.5), np.full((8, 8), -0.5), np.full((8, 8), 70000.0)):
        assert dic.GrayImage(frac).as_c().dtype == _abi.F64
    with pytest.raises(dic.DicError):
        dic.GrayImage(np.full((8, 8), np.nan))


def test_pack_gray_single_and_batch():
    """dicb200_pack_gray / _batch (the shim's GrayImage doubles -> u16 pass, AVX2
    when the host has it): lossless integers, per-frame maximum, fractional and
    out-of-range / NaN detection, odd widths (vector tail), row pitch."""
    L = dic.lib()
    L.dicb200_pack_gray.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32]
    L.dicb200_pack_gray_batch.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                          C.POINTER(C.c_void_p), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                          C.c_int32]
    rng = np.random.default_rng(7)
    w, h, n = 203, 157, 5
    frames = [rng.integers(0, 65536 if k else 256, (h, w)).astype(np.float64) for k in range(n)]
    frames[2][11, 17] = 65535.0
    outs = [np.zeros((h, w), np.uint16) for _ in range(n)]
    src = (C.c_void_p * n)(*[f.ctypes.data for f in frames])
    dst = (C.c_void_p * n)(*[o.ctypes.data for o in outs])
    frac = (C.c_int32 * n)()
    mx = (C.c_int32 * n)()
    for threads in (1, 4):
        assert L.dicb200_pack_gray_batch(src, n, w, h, 0, dst, frac, mx, threads) == 0
        for k in range(n):
            assert np.array_equal(outs[k], frames[k].astype(np.uint16)) and frac[k] == 0
            assert mx[k] == int(frames[k].max())
    # single-frame entry, with a source pitch wider than the row
    wide = np.zeros((h, w + 9))
    wide[:, :w] = frames[1]
    one = np.zeros((h, w), np.uint16)
    f1, m1 = C.c_int32(0), C.c_int32(0)
    assert L.dicb200_pack_gray(wide.ctypes.data, w, h, w + 9, 1, one.ctypes.data, C.byref(f1), C.byref(m1), 2) == 0
    assert np.array_equal(one, outs[1]) and f1.value == 0 and m1.value == mx[1]
    # a fractional level in the vector body and one in the scalar tail
    for (y, x) in ((3, 8), (h - 1, w - 1)):
        g = [f.copy() for f in frames]
        g[3][y, x] += 0.25
        src2 = (C.c_void_p * n)(*[f.ctypes.data for f in g])
        assert L.dicb200_pack_gray_batch(src2, n, w, h, 0, dst, frac, mx, 3) == 0
        assert [frac[k] for k in range(n)] == [0, 0, 0, 1, 0]
    for badv in (-1.0, 65536.0, np.nan, np.inf):
        g = [f.copy() for f in frames]
        g[4][5, 5] = badv
        src2 = (C.c_void_p * n)(*[f.ctypes.data for f in g])
        assert L.dicb200_pack_gray_batch(src2, n, w, h, 0, dst, frac, mx, 2) != 0


def test_synth_generator_is_deterministic_and_in_range():
    f = configs.crop(configs.get("c4"), 96, 96).frames[1]
    a, b = f.render(threads=1), f.render(threads=3)
    assert np.array_equal(a, b) and a.dtype == np.uint16 and a.max() <= 4095
    u8 = configs.crop(configs.get("c1"), 96, 96).frames[0].render()
    assert u8.dtype == np.uint8 and 40 < u8.mean() < 200
    # analytic re-render: an integer translation is an exact pixel shift
    w = configs.get("c1")
    r0, r1 = w.frames[0].render(), w.frames[1].render()
    assert np.array_equal(r1[40:200, 40:200], r0[45:205, 37:197])


def test_field_csv_format():
    recs = np.zeros(2, dtype=_abi.record_dtype())
    recs["x"] = [20, 36]
    recs["u"] = [3.0, 2.5]
    recs["zncc"] = [0.5, np.nan]
    recs["converged"] = [1, 0]
    recs["evaluations"] = [441, 0]
    s = dic.field_csv_string(dic.DisplacementField(0, 0, 1, recs, ""))
    assert s.splitlines()[0] == "x,y,u,v,zncc,converged,iterations,evaluations"
    assert s.splitlines()[1] == "20,0,3,0,0.5,1,0,441"
    assert s.splitlines()[2] == "36,0,2.5,0,nan,0,0,0"
