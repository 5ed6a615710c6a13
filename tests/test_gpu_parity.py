"""GPU parity: the sm_100a path (through the C-ABI) against the oracle.

Tolerances (north star, BASELINE.json): integer displacements, evaluation
counts, per-POI status and `converged` identical on every subset; sub-pixel
u, v within 1e-3 px; ZNCC within 1e-5. Iteration counts may differ only where
a convergence test |du|,|dv| < tol sits at the rounding edge (<= 0.5% of POIs).
"""
import copy
import glob
import json
import os

import numpy as np
import pytest

from paper_1905_06228_b200 import _abi, configs, dic

pytestmark = pytest.mark.gpu

UV_TOL = 1e-3
ZNCC_TOL = 1e-5
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def run_device(a, b, cfg, pair_index=0):
    return dic.analyze_pair(dic.GrayImage(a), dic.GrayImage(b, 1), cfg, pair_index).records


def assert_parity(got, exp, iter_frac=0.005):
    """Integer stage bit-exact everywhere; sub-pixel values on every POI whose
    refinement converged in the oracle. A POI that does NOT converge (the
    iteration wanders for max_iter steps, e.g. a subset straddling a constant
    region) has no well-defined sub-pixel value: its converged flag must match,
    its (chaotic) u/v are not compared."""
    assert len(got) == len(exp)
    for f in ("x", "y", "evaluations", "update_evaluations", "converged"):
        assert np.array_equal(got[f], exp[f]), (f, np.nonzero(got[f] != exp[f])[0][:5])
    integer_ok = exp["evaluations"] > 0
    assert np.array_equal(np.isnan(got["zncc"]), np.isnan(exp["zncc"]))
    if "integer_dx" in exp.dtype.names and exp["integer_dx"].any():
        assert np.array_equal(got["integer_dx"][integer_ok], exp["integer_dx"][integer_ok])
        assert np.array_equal(got["integer_dy"][integer_ok], exp["integer_dy"][integer_ok])
    # integer-only runs: u, v are the integer displacement, bit-exact
    intonly = integer_ok & (exp["iterations"] == 0) & (exp["converged"] == 1)
    assert np.array_equal(got["u"][intonly], exp["u"][intonly])
    assert np.array_equal(got["v"][intonly], exp["v"][intonly])
    ok = (exp["converged"] == 1) & integer_ok
    du = np.abs(got["u"] - exp["u"])[ok]
    dv = np.abs(got["v"] - exp["v"])[ok]
    assert np.all(du < UV_TOL) and np.all(dv < UV_TOL), (du.max(initial=0), dv.max(initial=0))
    assert np.all(np.abs(got["zncc"][ok] - exp["zncc"][ok]) < ZNCC_TOL)
    # convergence-edge flips of |du|,|dv| < tol (fp32 gathers vs fp64): rare, never > tol apart
    assert np.sum(got["iterations"][ok] != exp["iterations"][ok]) <= max(2, iter_frac * len(exp))
    return float(max(du.max(initial=0), dv.max(initial=0)))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_device_matches_reference_golden(gpu, path):
    """Golden vectors produced by the reference's own sources (oracle/_ref)."""
    d = np.load(path)
    c = _abi.RunConfigC()
    for k, v in json.loads(str(d["config"])).items():
        setattr(c, k, v)
    cfg = dic.RunConfig(
        integer_method=dic.IntegerMethod(c.integer_method), subpixel_method=dic.SubpixelMethod(c.subpixel_method),
        search=dic.SearchConfig(c.search_radius, dic.BfsDomain(c.bfs_domain), c.particle_count, c.max_generations,
                                c.stop_threshold, c.c1, c.c2, c.rng_seed),
        refine=dic.RefineConfig(c.tol, c.max_iter), grid=dic.GridParams(c.half_width, c.spacing, c.margin))
    got = run_device(d["ref"], d["tgt"], cfg)
    exp = d["records"]
    # integer-stage fields the reference does not expose come from the u/v of integer-only runs
    assert_parity(got, exp)


@pytest.mark.parametrize("name,crop,pair", [
    ("c1", None, 1), ("c2", None, 1), ("c3", 256, 1), ("c3x", 256, 1), ("c4", 512, 1), ("c5", 384, 33),
    ("c5", 384, 64),
])
def test_config_parity_against_oracle(gpu, port, name, crop, pair):
    w = configs.get(name) if name != "c5" else configs.c5(64)
    if crop:
        w = configs.crop(w, crop, crop)
    a, b = w.frames[0].render(), w.frames[pair].render()
    exp = port.analyze_pair(a, b, w.cfg, pair_index=pair - 1)
    got = run_device(a, b, w.cfg, pair_index=pair - 1)
    assert_parity(got, exp)


def test_c1_exact_shift_everywhere(gpu):
    w = configs.c1()
    a, b = w.frames[0].render(), w.frames[1].render()
    got = run_device(a, b, w.cfg)
    assert len(got) == 196
    assert np.all(got["u"] == 3.0) and np.all(got["v"] == -5.0)
    assert np.all(got["evaluations"] == 441) and np.all(got["converged"] == 1)


def test_pso_and_mpso_parity_with_reference_defaults(gpu, port):
    w = configs.crop(configs.get("c3"), 192, 192)
    a, b = w.frames[0].render(), w.frames[1].render()
    for method in (dic.IntegerMethod.pso, dic.IntegerMethod.mpso):
        cfg = dic.RunConfig(integer_method=method, subpixel_method=dic.SubpixelMethod.none,
                            search=dic.SearchConfig(search_radius=20, bfs_domain=dic.BfsDomain.window, rng_seed=7),
                            grid=dic.GridParams(15, 9, -1))
        for pair_index in (0, 5):
            exp = port.analyze_pair(a, b, cfg, pair_index=pair_index)
            got = run_device(a, b, cfg, pair_index=pair_index)
            assert_parity(got, exp)
            assert np.array_equal(got["u"], exp["u"]) and np.array_equal(got["v"], exp["v"])


def test_u16_wide_values_use_exact_fp64_path(gpu, port):
    # 16-bit data: (2M+1)*max^2 >= 2^32 -> DFMA-exact accumulation path
    w = configs.crop(configs.get("c4"), 128, 128)
    a = (w.frames[0].render().astype(np.uint32) * 16).astype(np.uint16)
    b = (w.frames[1].render().astype(np.uint32) * 16).astype(np.uint16)
    exp = port.analyze_pair(a, b, w.cfg)
    got = run_device(a, b, w.cfg)
    assert_parity(got, exp)


def test_whole_image_domain(gpu, port):
    w = configs.crop(configs.get("c1"), 96, 80)
    a, b = w.frames[0].render(), w.frames[1].render()
    cfg = dic.RunConfig(integer_method=dic.IntegerMethod.bfs, subpixel_method=dic.SubpixelMethod.none,
                        search=dic.SearchConfig(search_radius=5, bfs_domain=dic.BfsDomain.whole_image),
                        grid=dic.GridParams(8, 13, -1))
    assert_parity(run_device(a, b, cfg), port.analyze_pair(a, b, cfg))


def test_large_radius_chunked_window(gpu, port):
    # R > 31 -> candidate window split over several CTAs + reduction kernel
    w = configs.crop(configs.get("c2"), 256, 256)
    a, b = w.frames[0].render(), w.frames[1].render()
    cfg = copy.deepcopy(w.cfg)
    cfg.search.search_radius = 40
    cfg.subpixel_method = dic.SubpixelMethod.none
    cfg.grid = dic.GridParams(12, 40, -1)
    assert_parity(run_device(a, b, cfg), port.analyze_pair(a, b, cfg))


def test_identical_images_refiners(gpu):
    # SPEC refine_nr / refine_icgn examples: identical images -> u=v=0, ZNCC=1, converged
    w = configs.crop(configs.get("c4"), 128, 128)
    a = w.frames[0].render()
    for sub in (dic.SubpixelMethod.nr, dic.SubpixelMethod.icgn):
        cfg = copy.deepcopy(w.cfg)
        cfg.subpixel_method = sub
        got = run_device(a, a, cfg)
        assert np.all(got["converged"] == 1)
        assert np.all(np.abs(got["u"]) < 1e-6) and np.all(np.abs(got["v"]) < 1e-6)
        assert np.all(np.abs(got["zncc"] - 1.0) < 1e-6)
        assert np.all(got["iterations"] == 1)


def test_row_sharding_equals_full(gpu):
    """Subset-parallel sharding over grid rows keeps global RNG keys (mPSO)."""
    import ctypes as C

    import torch

    w = configs.crop(configs.get("c3"), 256, 256)
    a, b = w.frames[0].render(), w.frames[1].render()
    full = run_device(a, b, w.cfg)
    L = dic.lib()
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    ia, ib = dic.GrayImage(a).as_c(), dic.GrayImage(b, 1).as_c()
    ia.data, ib.data = ta.data_ptr(), tb.data_ptr()
    nx = len({x for x, _ in dic.grid_subsets(256, 256, 15, 8, w.cfg.effective_margin())})
    ny = len(full) // nx
    parts = []
    for lo, hi in dic.partition_ranges(ny, 3):
        out = torch.empty((hi - lo) * nx * C.sizeof(_abi.PoiRecordC), dtype=torch.uint8, device="cuda")
        n = C.c_size_t(0)
        c = w.cfg.to_c()
        st = L.dicb200_analyze_pair_device(C.byref(ia), C.byref(ib), C.byref(c), 0, lo, hi,
                                           C.c_void_p(out.data_ptr()), (hi - lo) * nx, C.byref(n), None)
        assert st == 0
        torch.cuda.synchronize()
        parts.append(np.frombuffer(out.cpu().numpy().tobytes(), dtype=_abi.record_dtype()))
    sharded = np.concatenate(parts)
    for f in ("x", "y", "u", "v", "zncc", "evaluations", "update_evaluations", "iterations", "converged"):
        assert np.array_equal(sharded[f], full[f], equal_nan=True), f


def test_analyze_sequence_policies_and_pair_errors(gpu, port):
    w = configs.crop(configs.c5(4), 128, 128)
    frames = [f.render() for f in w.frames]
    imgs = [dic.GrayImage(f, i) for i, f in enumerate(frames)]
    for policy in (dic.ReferencePolicy.fixed_first, dic.ReferencePolicy.update_every_pair):
        cfg = copy.deepcopy(w.cfg)
        cfg.reference_policy = policy
        fields = dic.analyze_sequence(imgs, cfg)
        pairs = dic.sequence_pairs(policy, len(imgs))
        assert [f.pair_index for f in fields] == list(range(len(pairs)))
        for f, (ra, tb) in zip(fields, pairs):
            assert (f.ref_id, f.tgt_id) == (ra, tb) and not f.failed()
            assert_parity(f.records, port.analyze_pair(frames[ra], frames[tb], cfg, pair_index=f.pair_index))
    # a pair-level dic::Error lands in field.error, the sequence continues (pipeline.cpp:191-198)
    bad = imgs[:2] + [dic.GrayImage(np.zeros((64, 64), np.uint16), 9)]
    fields = dic.analyze_sequence(bad, w.cfg)
    assert not fields[0].failed() and fields[1].error == "dimension mismatch"


def test_analyze_sequence_pipeline_matches_pairwise(gpu):
    """The pipelined sequence (frame slots reused across pairs, uploads ahead of
    compute, read-back behind it) returns exactly what independent
    analyze_pair calls return, for both policies and across an invalid pair."""
    w = configs.crop(configs.c5(9), 160, 144)
    frames = [f.render() for f in w.frames]
    imgs = [dic.GrayImage(f, i) for i, f in enumerate(frames)]
    imgs[5] = dic.GrayImage(np.zeros((64, 64), np.uint16), 5)  # pairs touching frame 5 fail
    for policy in (dic.ReferencePolicy.fixed_first, dic.ReferencePolicy.update_every_pair):
        cfg = copy.deepcopy(w.cfg)
        cfg.reference_policy = policy
        fields = dic.analyze_sequence(imgs, cfg)
        for f, (ra, tb) in zip(fields, dic.sequence_pairs(policy, len(imgs))):
            if 5 in (ra, tb):
                assert f.error == "dimension mismatch" and len(f.records) == 0
                continue
            assert not f.failed()
            exp = run_device(frames[ra], frames[tb], cfg, pair_index=f.pair_index)
            for k in exp.dtype.names:
                assert np.array_equal(f.records[k], exp[k], equal_nan=True), (policy, f.pair_index, k)


def test_sequence_device_matches_pairwise(gpu):
    """dicb200_analyze_sequence_device (device-resident frames, reference-side
    inputs reused along the sequence) == independent analyze_pair calls, for
    both policies, BFS/IC-GN and mPSO/NR, with a pair-index offset (RNG keys)."""
    import ctypes as C
    import torch

    w = configs.crop(configs.c5(6), 170, 150)
    frames = [f.render() for f in w.frames]
    dev = [torch.from_numpy(f.astype(np.int16) if f.dtype == np.uint16 else f).cuda() for f in frames]
    L = dic.lib()
    L.dicb200_analyze_sequence_device.argtypes = [
        C.c_void_p, C.c_size_t, C.POINTER(_abi.RunConfigC), C.c_uint64, C.c_int32, C.c_int32, C.c_void_p,
        C.c_size_t, C.POINTER(C.c_size_t), C.c_void_p]
    ims = (_abi.Image * len(frames))()
    for i, t in enumerate(dev):
        im = dic.GrayImage(frames[i], i).as_c()
        im.data = t.data_ptr()
        ims[i] = im
    for policy in (dic.ReferencePolicy.fixed_first, dic.ReferencePolicy.update_every_pair):
        for im_, sm in ((dic.IntegerMethod.bfs, dic.SubpixelMethod.icgn), (dic.IntegerMethod.mpso, dic.SubpixelMethod.nr)):
            cfg = copy.deepcopy(w.cfg)
            cfg.reference_policy, cfg.integer_method, cfg.subpixel_method = policy, im_, sm
            n = len(dic.grid_subsets(170, 150, cfg.grid.half_width, cfg.grid.spacing, cfg.effective_margin()))
            out = torch.empty(len(frames) * n * C.sizeof(_abi.PoiRecordC), dtype=torch.uint8, device="cuda")
            cnt = C.c_size_t(0)
            assert L.dicb200_analyze_sequence_device(ims, len(frames), C.byref(cfg.to_c()), 7, -1, -1,
                                                     C.c_void_p(out.data_ptr()), n, C.byref(cnt), None) == 0
            torch.cuda.synchronize()
            recs = np.frombuffer(out.cpu().numpy().tobytes(), dtype=_abi.record_dtype())
            for k, (ra, tb) in enumerate(dic.sequence_pairs(policy, len(frames))):
                exp = run_device(frames[ra], frames[tb], cfg, pair_index=7 + k)
                got = recs[k * n:(k + 1) * n]
                for f in exp.dtype.names:
                    assert np.array_equal(got[f], exp[f], equal_nan=True), (policy, im_, k, f)


def test_failure_semantics_degenerate_target(gpu, port):
    """Constant target regions: skipped candidates, 'all positions degenerate',
    refine failures keep the integer fields (pipeline.cpp:82-133)."""
    w = configs.crop(configs.get("c4"), 160, 160)
    a, b = w.frames[0].render(), w.frames[1].render()
    b[:, :70] = 1000
    for sub in (dic.SubpixelMethod.nr, dic.SubpixelMethod.icgn):
        cfg = copy.deepcopy(w.cfg)
        cfg.subpixel_method = sub
        exp = port.analyze_pair(a, b, cfg)
        got = run_device(a, b, cfg)
        assert_parity(got, exp)
        # failure statuses agree wherever the refinement is not chaotic
        stable = (exp["converged"] == 1) | (exp["iterations"] == 0)
        assert np.mean(got["status"][stable] == exp["status"][stable]) > 0.97
        assert (exp["status"] != 0).any()


def test_sequence_mixed_bit_widths_reuse_reference_cache(gpu, port):
    """A fixed-first sequence whose targets change the pair's pixel range: the
    first pair (12-bit) runs the block-sum search, the second (13-bit target)
    the tensor-core search on the SAME cached reference frame, which then needs
    its strip images. Each field must equal an independent analyze_pair and the
    oracle (the per-stream reference cache is keyed on the kernel choice)."""
    w = configs.crop(configs.c5(4), 384, 384)
    frames = [f.render() for f in w.frames]
    for k in (3, 4):  # later targets: max 8190 -> 13 bits; pairs alternate over two compute streams
        frames[k] = (frames[k].astype(np.uint32) * 2).astype(np.uint16)
    imgs = [dic.GrayImage(f, i) for i, f in enumerate(frames)]
    assert imgs[1].bits() == 12 and imgs[3].bits() == 13
    fields = dic.analyze_sequence(imgs, w.cfg)
    for f, tb in zip(fields, (1, 2, 3, 4)):
        assert not f.failed()
        exp = run_device(frames[0], frames[tb], w.cfg, pair_index=f.pair_index)
        for k in exp.dtype.names:
            assert np.array_equal(f.records[k], exp[k], equal_nan=True), (tb, k)
        assert_parity(f.records, port.analyze_pair(frames[0], frames[tb], w.cfg, pair_index=f.pair_index))


def test_sequence_cb_chunks_equal_one_call(gpu):
    """dicb200_analyze_sequence_cb: a sequence handed over in two calls (first
    pair index 0 and 2) returns the fields of one call — pair indices, mPSO RNG
    keys (evaluations), every record — and calls field_ready once per field."""
    import ctypes as C

    w = configs.crop(configs.get("c3"), 192, 176)
    f0 = w.frames[0].render()
    frames = [f0] + [np.roll(f0, (k % 3 - 1, k), axis=(0, 1)) for k in (1, 2, 3, 4)]
    imgs = [dic.GrayImage(f, i) for i, f in enumerate(frames)]
    cfg = copy.deepcopy(w.cfg)
    cfg.reference_policy = dic.ReferencePolicy.fixed_first
    one = dic.analyze_sequence(imgs, cfg)
    n = len(one[0].records)
    L = dic.lib()
    CB = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t)
    L.dicb200_analyze_sequence_cb.argtypes = [C.POINTER(_abi.Image), C.c_size_t, C.POINTER(_abi.RunConfigC),
                                              C.POINTER(_abi.FieldC), C.c_size_t, C.c_uint64, CB, C.c_void_p]
    c = cfg.to_c()
    got, seen = {}, []
    for first, idx in ((0, [0, 1, 2]), (2, [0, 3, 4])):
        ims = (_abi.Image * 3)(*[imgs[i].as_c() for i in idx])
        fields = (_abi.FieldC * 2)()
        bufs = [np.zeros(n, dtype=_abi.record_dtype()) for _ in range(2)]
        for i in range(2):
            fields[i].records = C.cast(bufs[i].ctypes.data, C.POINTER(_abi.PoiRecordC))
            fields[i].capacity = n
        cb = CB(lambda user, i, first=first: seen.append(first + i))
        assert L.dicb200_analyze_sequence_cb(ims, 3, C.byref(c), fields, 2, first, cb, None) == 0
        for i in range(2):
            assert fields[i].status == 0 and fields[i].pair_index == first + i and fields[i].count == n
            got[first + i] = bufs[i]
    assert sorted(seen) == [0, 1, 2, 3]
    for k in range(4):
        for f in _abi.record_dtype().names:
            a, b = got[k][f], one[k].records[f]
            assert np.array_equal(a, b, equal_nan=True) if a.dtype.kind == "f" else np.array_equal(a, b), (k, f)
