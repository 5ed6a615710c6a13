"""f-4 accuracy sweep (accuracy.cpp:10-78) and its generators (synth.cpp).

CPU: the host restatement of synth_speckle / synth_warped_pair is pinned
bit-for-bit against the reference's own functions (oracle/_ref), plus the
reference's test_image.cpp cases for them (determinism, textureless rejection,
variance floor, identity / integer / half-pixel warps, out-of-bounds).
GPU: dic.run_accuracy_sweep (analysis on the device) against (a) the same
sweep computed with the reference's analyze_pair on the same quantized frames —
record-level parity, so the aggregate errors agree to the u/v tolerance — and
(b) the reference's own run_accuracy_sweep on its unquantized doubles."""
import copy

import numpy as np
import pytest

import oracle.pyoracle as po
from paper_1905_06228_b200 import dic
from paper_1905_06228_b200.dic import DicError, IntegerMethod as I, SubpixelMethod as S

needs_ref = pytest.mark.skipif(not po.available("reference"), reason="reference build absent")
UV_TOL = 1e-3  # north_star tolerance on u, v (px)


def _params(w, h, **kw):
    return dic.SpeckleParams(blob_count=dic.default_blob_count(w, h), **kw)


@needs_ref
@pytest.mark.parametrize("w,h,seed", [(64, 64, 11), (160, 160, 7), (31, 47, 3), (200, 90, 123456789)])
def test_speckle_bit_identical_to_reference(w, h, seed):
    p = _params(w, h)
    assert dic.synth_speckle(w, h, seed, p).tobytes() == po.ref_synth_speckle(w, h, seed, p).tobytes()
    q = _params(w, h, sigma_min=0.8, sigma_max=4.0, amp_min=20.0, background=100.0)
    assert dic.synth_speckle(w, h, seed, q).tobytes() == po.ref_synth_speckle(w, h, seed, q).tobytes()


def test_speckle_determinism_and_errors():
    """test_image.cpp:164-197."""
    p = _params(64, 64)
    a, b, c = dic.synth_speckle(64, 64, 11, p), dic.synth_speckle(64, 64, 11, p), dic.synth_speckle(64, 64, 12, p)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    with pytest.raises(DicError, match="textureless pattern"):
        dic.synth_speckle(64, 64, 1, dic.SpeckleParams(blob_count=0))
    with pytest.raises(DicError, match="invalid blob radius range"):
        dic.synth_speckle(64, 64, 1, _params(64, 64, sigma_min=2.0, sigma_max=1.0))
    with pytest.raises(DicError, match="zero-dimension image"):
        dic.synth_speckle(0, 5, 1, p)
    img = dic.synth_speckle(64, 64, 5, p)
    for oy in (0, 16, 33):
        for ox in (0, 16, 33):
            assert img[oy:oy + 31, ox:ox + 31].var() > p.variance_floor


@needs_ref
@pytest.mark.parametrize("warp", [
    dic.WarpSpec(1.25, -0.75), dic.WarpSpec(3, -2), dic.WarpSpec(-3.9, 3.9), dic.WarpSpec(0.1, -0.1),
    dic.WarpSpec(0.5, 0, 0.01, 0, 0, -0.02), dic.WarpSpec(-1.5, 2.25, 0.003, -0.004, 0.002, 0.005),
], ids=lambda w: f"{w.u}_{w.v}_{w.ux}")
def test_warped_pair_bit_identical_to_reference(warp):
    ref = dic.synth_speckle(120, 100, 9, _params(120, 100))
    t, m = dic.synth_warped_pair(ref, warp)
    t2, m2 = po.ref_synth_warped_pair(ref, warp)
    assert t.tobytes() == t2.tobytes() and np.array_equal(m, m2)


def test_warp_cases_from_reference_tests():
    """test_image.cpp:200-274: identity, exact integer shifts, half-pixel ramp,
    out-of-bounds and singular warps."""
    ref = dic.synth_speckle(48, 40, 2, _params(48, 40))
    t, m = dic.synth_warped_pair(ref, dic.WarpSpec())
    assert m.all() and np.array_equal(t, ref)
    for seed in range(20):
        ref = dic.synth_speckle(32, 28, seed, _params(32, 28))
        t, m = dic.synth_warped_pair(ref, dic.WarpSpec(3, -2))
        exp_m = np.zeros_like(m)
        exp_m[:26, 3:] = 1  # sx = x - 3 >= 0, sy = y + 2 <= 27
        assert np.array_equal(m, exp_m)
        assert np.array_equal(t[:26, 3:], ref[2:, :29])
    t, m = dic.synth_warped_pair(np.array([[10.0, 20.0, 30.0]]), dic.WarpSpec(u=0.5))
    assert m.tolist() == [[0, 1, 1]] and t[0, 1] == 15.0 and t[0, 2] == 25.0
    with pytest.raises(DicError, match="warp out of bounds"):
        dic.synth_warped_pair(ref, dic.WarpSpec(u=9999))
    with pytest.raises(DicError, match="warp not invertible"):
        dic.synth_warped_pair(ref, dic.WarpSpec(ux=-1.0))


# ---------------------------------------------------------------- GPU sweeps

COMBOS = [(I.bfs, S.none), (I.bfs, S.nr), (I.bfs, S.icgn), (I.mpso, S.nr), (I.pso, S.icgn), (I.mpso, S.none)]


def _sweep_cfg(gray_scale):
    cfg = dic.SweepConfig(gray_scale=gray_scale)
    cfg.base.search.bfs_domain = dic.BfsDomain.window
    cfg.base.search.search_radius = 8
    cfg.base.search.particle_count = 60
    cfg.base.search.max_generations = 12
    return cfg


def _reference_on_quantized(cfg, combos):
    """accuracy.cpp:10-78 computed with the reference's analyze_pair on the
    quantized frames the device sees (checker only)."""
    ref_o = po.Oracle("reference")
    sp = copy.deepcopy(cfg.speckle)
    if sp.blob_count <= 0:
        sp.blob_count = dic.default_blob_count(cfg.width, cfg.height)
    q = lambda a: np.round(a * cfg.gray_scale)  # noqa: E731
    ref = po.ref_synth_speckle(cfg.width, cfg.height, cfg.seed, sp)
    warps = [dic.WarpSpec(o + f, -(o + f)) for o in cfg.offsets for f in cfg.fractions]
    tgts = [q(po.ref_synth_warped_pair(ref, w)[0]) for w in warps]
    out = []
    for im, sm in combos:
        run = copy.deepcopy(cfg.base)
        run.integer_method, run.subpixel_method = im, sm
        err_sum, mx, n, unconv = 0.0, 0.0, 0, 0
        for k, (w, t) in enumerate(zip(warps, tgts)):
            for r in ref_o.analyze_pair(q(ref), t, run, pair_index=k):  # accuracy.cpp:52-60, same order
                eu, ev = abs(float(r["u"]) - w.u), abs(float(r["v"]) - w.v)
                mx = max(mx, eu, ev)
                err_sum += eu + ev
                n += 2
                unconv += int(r["converged"] == 0)
        out.append(dict(max_err=mx, mean_err=err_sum / n, measurements=n, unconverged=unconv))
    return out


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("gray_scale", [1, 256])
def test_sweep_matches_reference_on_same_frames(gpu, gray_scale):
    cfg = _sweep_cfg(gray_scale)
    rep = dic.run_accuracy_sweep(COMBOS, cfg)
    npoi = len(dic.grid_subsets(cfg.width, cfg.height, cfg.base.grid.half_width, cfg.base.grid.spacing,
                                cfg.base.effective_margin()))
    assert (rep.warp_count, rep.poi_count) == (15, npoi)
    exp = _reference_on_quantized(cfg, COMBOS)
    for got, e, combo in zip(rep.combos, exp, COMBOS):
        assert (got.integer_method, got.subpixel_method) == combo
        assert got.measurements == e["measurements"], combo
        assert got.unconverged == e["unconverged"], combo
        tol = 0.0 if combo[1] == S.none else UV_TOL
        assert abs(got.max_err - e["max_err"]) <= tol, (combo, got.max_err, e["max_err"])
        assert abs(got.mean_err - e["mean_err"]) <= tol, (combo, got.mean_err, e["mean_err"])


@pytest.mark.gpu
@needs_ref
def test_sweep_tracks_reference_sweep_on_doubles(gpu):
    """16-bit quantization keeps the reference's own sweep verdicts: same
    measurements, pass/flag and unconverged counts; errors within 2e-3 px."""
    cfg = _sweep_cfg(256)
    rep = dic.run_accuracy_sweep(COMBOS, cfg)
    exp, wc, pc, _ = po.ref_accuracy_sweep(COMBOS, cfg)
    assert (rep.warp_count, rep.poi_count) == (wc, pc)
    for got, e in zip(rep.combos, exp):
        assert got.measurements == e.measurements
        assert got.unconverged == e.unconverged
        assert got.passed == bool(e.pass_) and got.mean_flagged == bool(e.mean_flagged)
        assert abs(got.max_err - e.max_err) <= 2e-3 and abs(got.mean_err - e.mean_err) <= 2e-3


def _integer_only(cfg):
    import copy

    c = copy.deepcopy(cfg)
    c.subpixel_method = S.none
    return c


@pytest.mark.gpu
@needs_ref
def test_fractional_frames_track_reference_doubles(gpu):
    """The reference's own (non-integer) synthetic frames go through the exact
    fp64 path: the integer stage evaluates the reference's zncc in its own
    order, so evaluations (every mPSO trajectory included) and convergence
    equal the reference's on its doubles; u/v within the 1e-3 px tolerance."""
    ref = po.ref_synth_speckle(200, 180, 21, _params(200, 180))
    tgt, _ = po.ref_synth_warped_pair(ref, dic.WarpSpec(2.35, -1.6, 0.003, 0.0, 0.0, -0.002))
    oracle = po.Oracle("reference")
    for im, sm in ((I.bfs, S.icgn), (I.bfs, S.nr), (I.mpso, S.icgn)):
        cfg = _sweep_cfg(256).base
        cfg.integer_method, cfg.subpixel_method = im, sm
        got = dic.analyze_pair(dic.GrayImage(ref), dic.GrayImage(tgt, 1), cfg).records
        exp = oracle.analyze_pair(ref, tgt, cfg)
        assert len(got) == len(exp) and np.array_equal(got["x"], exp["x"]) and np.array_equal(got["y"], exp["y"])
        assert np.array_equal(got["converged"], exp["converged"]), (im, sm)
        assert np.array_equal(got["evaluations"], exp["evaluations"]), (im, sm)
        assert np.array_equal(got["update_evaluations"], exp["update_evaluations"]), (im, sm)
        iexp = oracle.analyze_pair(ref, tgt, _integer_only(cfg))  # the integer stage alone: exact values
        igot = dic.analyze_pair(dic.GrayImage(ref), dic.GrayImage(tgt, 1), _integer_only(cfg)).records
        for f in ("u", "v", "zncc", "evaluations"):
            assert np.array_equal(igot[f], iexp[f], equal_nan=True), (im, sm, f)
        ok = exp["converged"] == 1
        assert np.abs(got["u"] - exp["u"])[ok].max() < 1e-3 and np.abs(got["v"] - exp["v"])[ok].max() < 1e-3, (im, sm)


@pytest.mark.gpu
def test_float_image_dtypes_through_the_c_abi(gpu):
    """DICB200_F32 / DICB200_F64 images (host and device entry points) run on
    the fp64 path: bit-identical records to the same levels handed over as
    doubles (f32 widened exactly); non-finite levels are rejected on the host."""
    import ctypes as C

    import torch

    from paper_1905_06228_b200 import _abi

    ref = dic.synth_speckle(180, 170, 4, _params(180, 170))
    tgt, _ = dic.synth_warped_pair(ref, dic.WarpSpec(1.7, 2.2, -0.002, 0.0, 0.001, 0.0))
    cfg = _sweep_cfg(256).base
    cfg.subpixel_method = S.icgn
    exp = dic.analyze_pair(dic.GrayImage(ref), dic.GrayImage(tgt, 1), cfg).records
    L = dic.lib()
    n = len(exp)
    for dtype, npt in ((_abi.F64, np.float64), (_abi.F32, np.float32)):
        a, b = ref.astype(npt), tgt.astype(npt)
        if npt == np.float32:  # the f32-rounded levels as doubles
            exp32 = dic.analyze_pair(dic.GrayImage(a.astype(np.float64)), dic.GrayImage(b.astype(np.float64), 1),
                                     cfg).records
        else:
            exp32 = exp
        ims = []
        for arr, i in ((a, 0), (b, 1)):
            im = _abi.Image()
            im.width, im.height, im.pitch, im.dtype, im.id, im.bits = arr.shape[1], arr.shape[0], arr.shape[1], dtype, i, 0
            im.data = arr.ctypes.data
            ims.append(im)
        out = np.zeros(n, _abi.record_dtype())
        cnt = C.c_size_t(0)
        assert L.dicb200_analyze_pair(C.byref(ims[0]), C.byref(ims[1]), C.byref(cfg.to_c()), 0, out.ctypes.data, n,
                                      C.byref(cnt)) == 0
        for k in exp.dtype.names:
            assert np.array_equal(out[k], exp32[k], equal_nan=True), (dtype, k)
        # device entry point
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        ims[0].data, ims[1].data = ta.data_ptr(), tb.data_ptr()
        dout = torch.empty(n * C.sizeof(_abi.PoiRecordC), dtype=torch.uint8, device="cuda")
        assert L.dicb200_analyze_pair_device(C.byref(ims[0]), C.byref(ims[1]), C.byref(cfg.to_c()), 0, -1, -1,
                                             C.c_void_p(dout.data_ptr()), n, C.byref(cnt), None) == 0
        torch.cuda.synchronize()
        drec = np.frombuffer(dout.cpu().numpy().tobytes(), dtype=_abi.record_dtype())
        for k in exp.dtype.names:
            assert np.array_equal(drec[k], exp32[k], equal_nan=True), (dtype, "device", k)
    bad = ref.copy()
    bad[3, 3] = np.nan
    im = _abi.Image()
    im.width, im.height, im.pitch, im.dtype, im.id, im.bits = 180, 170, 180, _abi.F64, 0, 0
    im.data = bad.ctypes.data
    out = np.zeros(n, _abi.record_dtype())
    cnt = C.c_size_t(0)
    assert L.dicb200_analyze_pair(C.byref(im), C.byref(ims[1]), C.byref(cfg.to_c()), 0, out.ctypes.data, n,
                                  C.byref(cnt)) == 1
