"""CPU: pin the oracles. The C restatement (oracle/dic_oracle.c) must equal
the reference's own sources (oracle/_ref) bit-for-bit, reproduce the committed
golden fixtures (generated from the reference build by
tests/golden/make_golden.py) and the reference's known answers / unit-test
properties (proj/tests/test_correlation.cpp, test_integer_search.cpp)."""
import glob
import json
import os

import numpy as np
import pytest

from paper_1905_06228_b200 import _abi, configs
from paper_1905_06228_b200.dic import (BfsDomain, GridParams, IntegerMethod, RunConfig, SearchConfig,
                                       SubpixelMethod)

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
FIELDS_EXACT = ["x", "y", "u", "v", "zncc", "converged", "iterations", "evaluations", "update_evaluations"]


def cfg_from_json(s):
    c = _abi.RunConfigC()
    for k, v in json.loads(s).items():
        setattr(c, k, v)

    class Wrap:  # quacks like RunConfig for the oracle wrapper
        def __init__(self, c):
            self.c = c
            self.grid = GridParams(c.half_width, c.spacing, c.margin)

        def to_c(self):
            return self.c

        def effective_margin(self):
            return self.c.margin if self.c.margin >= 0 else self.c.half_width + self.c.search_radius

    return Wrap(c)


def speckle(w, h, seed):
    f = configs.FrameSpec(w, h, _abi.U8, 255, seed, w * h // 60, (2.0, 4.0), (60.0, 200.0))
    return f.render(threads=1).astype(np.float64)


# ---------------------------------------------------------------- known answers

@pytest.mark.parametrize("kind", ["port", "reference"])
def test_mt19937_64_known_answers(kind, request):
    orc = request.getfixturevalue(kind)
    # the 10000th output of a default-seeded mt19937_64 ([rand.predef])
    assert int(orc.mt64(5489, 10000)[-1]) == 9981545732273789042
    # derive_stream_seed (rng.hpp:20-27), SURVEY Appendix C.3
    assert orc.derive_stream_seed(1, 0, 0) == 8112600223918159332
    assert orc.uniform01(orc.derive_stream_seed(1, 0, 0), 1)[0] == 0.97839758413343236


def test_port_rng_matches_reference(port, reference):
    for seed in [0, 1, 2**63 + 5, 123456789]:
        assert np.array_equal(port.mt64(seed, 2000), reference.mt64(seed, 2000))
        for pair, subset in [(0, 0), (3, 7), (63, 160000)]:
            assert port.derive_stream_seed(seed, pair, subset) == reference.derive_stream_seed(seed, pair, subset)


# ---------------------------------------------------------------- golden fixtures

@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_port_reproduces_golden(port, path):
    d = np.load(path)
    cfg = cfg_from_json(str(d["config"]))
    got = port.analyze_pair(d["ref"], d["tgt"], cfg, threads=2)
    exp = d["records"]
    assert len(got) == len(exp)
    for f in FIELDS_EXACT:
        assert np.array_equal(got[f], exp[f], equal_nan=True), f


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_reference_build_reproduces_golden(reference, path):
    d = np.load(path)
    got = reference.analyze_pair(d["ref"], d["tgt"], cfg_from_json(str(d["config"])))
    for f in FIELDS_EXACT:
        assert np.array_equal(got[f], d["records"][f], equal_nan=True), f


@pytest.mark.parametrize("name,crop", [("c2", 112), ("c3", 112), ("c4", 112), ("c5", 112)])
def test_port_equals_reference_build(port, reference, name, crop):
    w = configs.crop(configs.get(name), crop, crop)
    a, b = w.frames[0].render(), w.frames[-1].render()
    x = port.analyze_pair(a, b, w.cfg)
    y = reference.analyze_pair(a, b, w.cfg)
    for f in FIELDS_EXACT:
        assert np.array_equal(x[f], y[f], equal_nan=True), f


def test_constant_inertia_variant_differs_only_in_w(port):
    # BASELINE's "inertia 0.7" (flagged extra): restated as w(t) = const
    w = configs.crop(configs.get("c3x"), 112, 112)
    a, b = w.frames[0].render(), w.frames[1].render()
    x = port.analyze_pair(a, b, w.cfg)
    w.cfg.inertia_mode = 0
    y = port.analyze_pair(a, b, w.cfg)
    assert not np.array_equal(x["evaluations"], y["evaluations"])


# ------------------------------------------------ reference unit-test properties

@pytest.mark.parametrize("kind", ["port", "reference"])
def test_zncc_properties(kind, request):
    orc = request.getfixturevalue(kind)
    img = speckle(64, 64, 21)
    # identity -> 1, inverted -> -1, affine gray invariance (test_correlation.cpp:57-90)
    assert abs(orc.zncc(img, img, 32, 32, 15, 0, 0) - 1.0) < 1e-12
    assert abs(orc.zncc(img, 255.0 - img, 32, 32, 15, 0, 0) + 1.0) < 1e-12
    base = orc.zncc(img, img, 32, 32, 15, 2, -1)
    assert abs(orc.zncc(img, 2.0 * img + 10.0, 32, 32, 15, 2, -1) - base) < 1e-9
    # symmetry at zero displacement (test_correlation.cpp:108-115)
    g = speckle(64, 64, 32)
    assert orc.zncc(img, g, 32, 32, 12, 0, 0) == orc.zncc(g, img, 32, 32, 12, 0, 0)


@pytest.mark.parametrize("kind", ["port", "reference"])
def test_zncc_error_strings(kind, request):
    from oracle.pyoracle import OracleError

    orc = request.getfixturevalue(kind)
    img = speckle(64, 64, 33)
    flat = np.full((64, 64), 50.0)
    with pytest.raises(OracleError, match="window out of range"):
        orc.zncc(img, img, 32, 32, 15, 20, 0)
    with pytest.raises(OracleError, match="degenerate target subset"):
        orc.zncc(img, flat, 32, 32, 15, 0, 0)
    with pytest.raises(OracleError, match="degenerate subset"):
        orc.zncc(flat, img, 32, 32, 15, 0, 0)


@pytest.mark.parametrize("kind", ["port", "reference"])
def test_bfs_exact_shift_and_tie_break(kind, request):
    orc = request.getfixturevalue(kind)
    ref = speckle(100, 100, 17)
    tgt = np.roll(np.roll(ref, -2, axis=0), 3, axis=1)  # content moves by (+3, -2)
    cfg = RunConfig(integer_method=IntegerMethod.bfs,
                    search=SearchConfig(search_radius=25, bfs_domain=BfsDomain.window))
    r = orc.integer_search(ref, tgt, 50, 50, 15, cfg, 0)
    assert (r["dx"], r["dy"]) == (3, -2)
    assert r["evaluations"] == 51 * 51  # test_integer_search.cpp:57-69
    # period-8 checkerboard: ties break toward the smallest (dy, dx) (:104-121)
    y, x = np.mgrid[0:32, 0:32]
    cb = np.where(((x % 8) < 4) ^ ((y % 8) < 4), 200.0, 50.0)
    cfg.search.search_radius = 8
    r = orc.integer_search(cb, cb, 16, 16, 7, cfg, 0)
    assert (r["dx"], r["dy"]) == (-8, -8)


@pytest.mark.parametrize("kind", ["port", "reference"])
def test_swarm_budgets_and_determinism(kind, request):
    orc = request.getfixturevalue(kind)
    ref, tgt = speckle(100, 100, 61), speckle(100, 100, 62)
    cfg = RunConfig()  # reference defaults: P=50, G=5
    for seed in range(4):
        s = orc.derive_stream_seed(seed, 0, 0)
        cfg.integer_method = IntegerMethod.pso
        a = orc.integer_search(ref, tgt, 50, 50, 15, cfg, s)
        b = orc.integer_search(ref, tgt, 50, 50, 15, cfg, s)
        assert a == b
        assert a["generations_used"] == 5 and a["evaluations"] <= 50 * 6  # :180-203
        cfg.integer_method = IntegerMethod.mpso
        m = orc.integer_search(ref, tgt, 50, 50, 15, cfg, s)
        assert m["evaluations"] <= 5 * 50 * 6 and m["update_evaluations"] <= 5 * 50 * 5


def test_grid_matches_reference(port, reference):
    for (w, h, m, s, mg) in [(256, 256, 10, 16, 20), (100, 60, 15, 7, 0), (2048, 2048, 20, 5, 25), (31, 31, 15, 1, 15)]:
        assert np.array_equal(port.grid(w, h, m, s, mg), reference.grid(w, h, m, s, mg))


def test_bicubic_restatement_known_answers(port):
    """The bicubic variant (B200 extension, parity unpinned: the reference has
    bilinear only): Keys cubic convolution reproduces polynomials of degree <= 2
    exactly away from the border, returns the node value on nodes, and its
    analytic gradient is exact on them too; out-of-domain samples fail like the
    bilinear pair (value [0, w-1], gradient [1, w-2])."""
    h, w = 24, 30
    y, x = np.mgrid[0:h, 0:w].astype(np.float64)
    cases = (
        (lambda a, b: 3.0 * a - 2.0 * b + 7.0, lambda a, b: (3.0, -2.0)),
        (lambda a, b: 0.5 * a * a + 0.25 * b * b + a * b, lambda a, b: (a + b, 0.5 * b + a)),
    )
    for f, grad in cases:
        img = f(x, y)
        for (sx, sy) in ((5.25, 7.5), (10.0, 11.0), (17.8, 3.3), (22.125, 16.9)):
            v, g = port.interp_bicubic(img, sx, sy)
            assert abs(v - f(sx, sy)) < 1e-9, (sx, sy, v)
            assert np.allclose(g, grad(sx, sy), atol=1e-9), (sx, sy, g)
    img = np.random.default_rng(3).integers(0, 4096, (h, w)).astype(np.float64)
    assert port.interp_bicubic(img, 9.0, 4.0)[0] == img[4, 9]
    assert port.interp_bicubic(img, -0.01, 4.0)[0] is None
    assert port.interp_bicubic(img, w - 1.0, h - 1.0)[0] == img[h - 1, w - 1]
    assert port.interp_bicubic(img, 0.5, 4.0)[1] is None  # gradient domain [1, w-2]
