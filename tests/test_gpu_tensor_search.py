"""The tensor-core integer search (csrc/bfs_tc.cu) against the CUDA-core
kernel (csrc/bfs.cu, itself parity-checked against the reference) on the same
device: every integer decision — displacement, evaluation count, status — and
the ZNCC value of the winner must be bit-identical, across subset sizes (with
and without the row-major remainder stage), search radii, 8/12/16-bit pixels,
non-multiple-of-tile frames, windows clipped by the image border, row-sharded
launches and the PSO surface path."""
import os
from dataclasses import replace

import numpy as np
import pytest

from paper_1905_06228_b200 import _abi, configs, dic
from paper_1905_06228_b200.dic import (BfsDomain, GridParams, IntegerMethod, RefineConfig, RunConfig,
                                       SearchConfig, SubpixelMethod)

pytestmark = pytest.mark.gpu

FIELDS = ("x", "y", "u", "v", "zncc", "converged", "evaluations", "status", "integer_dx", "integer_dy")


def _frames(width, height, dtype, max_value, seed, u, v):
    if dtype == _abi.U8:
        f = configs.FrameSpec(width, height, _abi.U8, max_value, seed, width * height // 60, (2.0, 4.0),
                              (60.0, 200.0))
    else:
        peak = (0.23 * max_value, 0.78 * max_value)
        f = configs.FrameSpec(width, height, _abi.U16, max_value, seed, width * height // 42, (1.5, 3.5), peak)
    g = replace(f, field=_abi.FIELD_AFFINE, a=(u, 0.004, -0.003, v, 0.002, 0.005, width / 2.0, height / 2.0))
    return f.render(), g.render()


def _run(a, b, cfg, legacy, path=None):
    """path: None = the library's choice, "tc" = force the tensor-core kernel,
    "bs" = the block-sum kernel wherever it has an instantiation (also u8)."""
    for k in ("DICB200_BFS_LEGACY", "DICB200_BFS_TC", "DICB200_BFS_BS"):
        os.environ.pop(k, None)
    if legacy:
        os.environ["DICB200_BFS_LEGACY"] = "1"
    if path == "tc":
        os.environ["DICB200_BFS_TC"] = "1"
    if path == "bs":
        os.environ["DICB200_BFS_BS"] = "1"
    try:
        return dic.analyze_pair(dic.GrayImage(a, 0), dic.GrayImage(b, 1), cfg).records
    finally:
        for k in ("DICB200_BFS_LEGACY", "DICB200_BFS_TC", "DICB200_BFS_BS"):
            os.environ.pop(k, None)


def _cfg(M, R, step, method=IntegerMethod.bfs, margin=-1):
    return RunConfig(integer_method=method, subpixel_method=SubpixelMethod.none,
                     search=SearchConfig(search_radius=R, bfs_domain=BfsDomain.window, particle_count=20,
                                         max_generations=10),
                     refine=RefineConfig(tol=1e-4, max_iter=20),
                     grid=GridParams(half_width=M, spacing=step, margin=margin))


CASES = [
    # (width, height, dtype, max_value, M, R, step, u, v)
    (300, 260, _abi.U16, 4095, 20, 12, 6, 3.3, -2.1),   # side 41: row-major remainder stage
    (260, 230, _abi.U8, 255, 15, 15, 5, -4.6, 5.2),      # side 31: no remainder stage
    (250, 240, _abi.U16, 65535, 16, 7, 4, 1.2, 0.7),     # 16-bit full range, side 33 (remainder)
    (203, 187, _abi.U16, 1023, 10, 4, 3, -0.4, 2.9),     # 10-bit, odd frame, small window
    (230, 210, _abi.U8, 255, 7, 20, 5, 8.4, -6.1),       # large window vs subset, border clipping
]


@pytest.mark.parametrize("case", CASES, ids=[f"M{c[4]}R{c[5]}s{c[6]}d{c[2]}b{c[3]}" for c in CASES])
def test_tensor_search_bit_identical_to_cuda_core(gpu, case):
    width, height, dtype, maxv, M, R, step, u, v = case
    a, b = _frames(width, height, dtype, maxv, 11 + M, u, v)
    cfg = _cfg(M, R, step)
    # M < 8: the library's own choice is the reference-order fp64 search (host.cu kRefOrderBelowM);
    # the kernel-vs-kernel comparison forces the tensor-core kernel there
    got = _run(a, b, cfg, legacy=False, path="tc" if M < 8 else None)
    exp = _run(a, b, cfg, legacy=True)
    assert len(got) >= 1024  # the tensor-core path runs (smaller grids keep the CUDA-core kernel)
    for f in FIELDS:
        assert np.array_equal(got[f], exp[f], equal_nan=True), (f, np.nonzero(got[f] != exp[f])[0][:5])


def test_tensor_search_degenerate_and_constant_regions(gpu):
    """Constant target patches (skipped candidates, 'all positions degenerate')
    and a constant reference subset (no valid candidate) decide identically."""
    a, b = _frames(240, 240, _abi.U16, 4095, 5, 1.5, -0.5)
    b[:, :90] = 1234          # constant target band: degenerate windows
    a[100:150, 150:200] = 777  # constant reference block: sqrt(vf) == 0 subsets
    cfg = _cfg(12, 6, 4)
    got = _run(a, b, cfg, legacy=False)
    exp = _run(a, b, cfg, legacy=True)
    assert len(got) >= 1024
    assert (exp["status"] != 0).any() and (exp["evaluations"] < exp["evaluations"].max()).any()
    for f in FIELDS:
        assert np.array_equal(got[f], exp[f], equal_nan=True), f


def test_tensor_search_row_shards_equal_full(gpu):
    """Row-range launches (the subset-parallel sharding) equal one full launch."""
    import ctypes as C
    import torch

    a, b = _frames(256, 240, _abi.U16, 4095, 21, 2.2, 1.7)
    cfg = _cfg(20, 10, 5)
    full = _run(a, b, cfg, legacy=False)
    L = dic.lib()
    ta, tb = torch.from_numpy(a.copy()).cuda(), torch.from_numpy(b.copy()).cuda()
    ia, ib = dic.GrayImage(a, 0).as_c(), dic.GrayImage(b, 1).as_c()
    ia.data, ib.data = ta.data_ptr(), tb.data_ptr()
    n = C.c_size_t(0)
    L.dicb200_grid_size(a.shape[1], a.shape[0], C.byref(cfg.to_c()), C.byref(n))
    nx = len(np.unique(full["x"]))
    ny = n.value // nx
    parts = []
    for lo, hi in ((0, ny // 3), (ny // 3, ny)):
        out = torch.empty((hi - lo) * nx * C.sizeof(_abi.PoiRecordC), dtype=torch.uint8, device="cuda")
        cnt = C.c_size_t(0)
        st = L.dicb200_analyze_pair_device(C.byref(ia), C.byref(ib), C.byref(cfg.to_c()), 0, lo, hi,
                                           C.c_void_p(out.data_ptr()), (hi - lo) * nx, C.byref(cnt), None)
        assert st == 0
        torch.cuda.synchronize()
        parts.append(np.frombuffer(out.cpu().numpy().tobytes(), dtype=_abi.record_dtype()))
    sharded = np.concatenate(parts)
    for f in FIELDS:
        assert np.array_equal(sharded[f], full[f], equal_nan=True), f


def test_tensor_surface_matches_cuda_core_for_pso(gpu):
    """mPSO / PSO walk over the tensor-core ZNCC surface == over the CUDA-core surface."""
    a, b = _frames(260, 250, _abi.U8, 255, 31, -3.4, 2.6)
    for method in (IntegerMethod.mpso, IntegerMethod.pso):
        cfg = _cfg(15, 12, 5, method=method)
        got = _run(a, b, cfg, legacy=False)
        exp = _run(a, b, cfg, legacy=True)
        assert len(got) >= 1024
        for f in FIELDS:
            assert np.array_equal(got[f], exp[f], equal_nan=True), (method, f)


# Shared-block-sum kernel (csrc/bfs_bs.cu): lattices whose spacing / remainder
# match an instantiation; bit-identical to the tensor-core and CUDA-core kernels.
BS_CASES = [
    # (width, height, dtype, max_value, M, R, step, u, v, method)
    (420, 400, _abi.U16, 4095, 20, 12, 10, 2.6, -3.3, IntegerMethod.bfs),   # c5 shape (s 10, r 1)
    (337, 301, _abi.U16, 4095, 20, 5, 5, -1.4, 0.8, IntegerMethod.bfs),     # c4 shape (s 5, r 1), odd frame
    (300, 290, _abi.U16, 4095, 20, 10, 5, 6.3, -7.7, IntegerMethod.bfs),    # two dx chunks (EW 21 > DXC 11)
    (310, 300, _abi.U16, 4095, 20, 10, 5, -2.2, 1.9, IntegerMethod.pso),    # block sums feeding the PSO surface
    (420, 400, _abi.U8, 255, 15, 15, 10, 4.2, 3.1, IntegerMethod.bfs),      # c2 shape (u8, EW 31)
    (330, 320, _abi.U8, 255, 15, 20, 8, -6.3, 5.5, IntegerMethod.mpso),     # c3 shape (s 8, r 7), surface
]


@pytest.mark.parametrize("case", BS_CASES, ids=[f"bsM{c[4]}R{c[5]}s{c[6]}d{c[2]}{c[9].name}" for c in BS_CASES])
def test_block_sum_search_bit_identical(gpu, case):
    width, height, dtype, maxv, M, R, step, u, v, method = case
    a, b = _frames(width, height, dtype, maxv, 5 + M + R, u, v)
    cfg = _cfg(M, R, step, method=method)
    got = _run(a, b, cfg, legacy=False, path="bs")
    tc = _run(a, b, cfg, legacy=False, path="tc")
    exp = _run(a, b, cfg, legacy=True)
    assert len(got) >= 1024
    for f in FIELDS:
        assert np.array_equal(tc[f], exp[f], equal_nan=True), ("tc", f)
        assert np.array_equal(got[f], exp[f], equal_nan=True), ("bs", f, np.nonzero(got[f] != exp[f])[0][:5])


def test_block_sum_row_shards_and_degenerate(gpu):
    """Row-range launches and constant regions through the block-sum kernel."""
    a, b = _frames(420, 400, _abi.U16, 4095, 77, 1.2, -2.2)
    b[:, :80] = 2000
    a[120:180, 200:260] = 900
    cfg = _cfg(20, 12, 10)
    got = _run(a, b, cfg, legacy=False)
    exp = _run(a, b, cfg, legacy=True)
    assert (exp["status"] != 0).any()
    for f in FIELDS:
        assert np.array_equal(got[f], exp[f], equal_nan=True), f


@pytest.mark.parametrize("seed", range(6))
def test_block_sum_randomized_against_cuda_core(gpu, seed):
    """Randomised lattices matching the block-sum instantiations (spacing,
    remainder, q) with random radii, sizes, bit depths, displacements and
    flat patches: block-sum records == CUDA-core records, bit for bit."""
    rng = np.random.default_rng(1000 + seed)
    M, step = [(20, 10), (20, 5), (15, 10), (15, 8)][seed % 4]
    R = int(rng.integers(3, 16))
    w, h = int(rng.integers(420, 500)), int(rng.integers(420, 500))
    maxv = int(rng.choice([1023, 4095]))
    a, b = _frames(w, h, _abi.U16, maxv, 77 + seed, float(rng.uniform(-R + 1, R - 1)), float(rng.uniform(-R + 1, R - 1)))
    if seed % 2:
        b[rng.integers(0, h - 40):, : rng.integers(20, 80)] = maxv // 3  # a flat target patch
    cfg = _cfg(M, R, step)
    got = _run(a, b, cfg, legacy=False, path="bs")
    exp = _run(a, b, cfg, legacy=True)
    assert len(got) >= 1024
    for f in FIELDS:
        assert np.array_equal(got[f], exp[f], equal_nan=True), (seed, M, step, R, f)


def test_fused_block_sum_argmax_bit_identical(gpu):
    """DICB200_BS_FUSE=1: the block-sum search with the exact argmax fused into
    its second phase (no cross-term buffer; per-slice filter winners merged,
    near ties searched exactly) returns bit-identical records to the default
    two-kernel path, on a C5 crop and a C4 crop (16-lane segments)."""
    import copy
    import os

    from paper_1905_06228_b200 import configs, dic

    for w, k in ((configs.crop(configs.c5(8), 320, 288), 5), (configs.crop(configs.get("c4"), 256, 256), 1)):
        a, b = w.frames[0].render(), w.frames[k].render()
        cfg = copy.deepcopy(w.cfg)
        cfg.subpixel_method = dic.SubpixelMethod.none
        ref = dic.analyze_pair(dic.GrayImage(a), dic.GrayImage(b, 1), cfg).records
        os.environ["DICB200_BS_FUSE"] = "1"
        try:
            got = dic.analyze_pair(dic.GrayImage(a), dic.GrayImage(b, 1), cfg).records
        finally:
            os.environ.pop("DICB200_BS_FUSE", None)
        for f in ref.dtype.names:
            assert np.array_equal(got[f], ref[f], equal_nan=True), f
