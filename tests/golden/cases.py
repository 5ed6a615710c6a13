"""Golden-vector cases: (name, frame pair generator, RunConfig). Images are
small integer-valued frames; the expected records come from the reference's
own sources (oracle/_ref) — see make_golden.py."""
from __future__ import annotations

import copy

import numpy as np

from paper_1905_06228_b200 import configs
from paper_1905_06228_b200.dic import (BfsDomain, GridParams, IntegerMethod, RefineConfig, RunConfig,
                                       SearchConfig, SubpixelMethod)


def _cfg_case(name, crop=None, pair=1, mutate=None):
    def make():
        w = configs.get(name)
        if crop:
            w = configs.crop(w, crop, crop)
        a = w.frames[0].render(threads=1)
        b = w.frames[pair].render(threads=1)
        cfg = copy.deepcopy(w.cfg)
        if mutate:
            mutate(cfg)
        return a, b, cfg
    return make


def checkerboard():
    # test_integer_search.cpp:104-121: period-8 texture, ties -> smallest (dy, dx)
    y, x = np.mgrid[0:32, 0:32]
    img = np.where(((x % 8) < 4) ^ ((y % 8) < 4), 200, 50).astype(np.uint8)
    cfg = RunConfig(integer_method=IntegerMethod.bfs, subpixel_method=SubpixelMethod.none,
                    search=SearchConfig(search_radius=8, bfs_domain=BfsDomain.window),
                    grid=GridParams(half_width=7, spacing=4, margin=16))
    return img, img.copy(), cfg


def degenerate_half():
    # test_integer_search.cpp:123-146: left part of the target flat
    w = configs.crop(configs.get("c1"), 64, 64)
    a = w.frames[0].render(threads=1)
    b = a.copy()
    b[:, :36] = 100
    cfg = RunConfig(integer_method=IntegerMethod.bfs, subpixel_method=SubpixelMethod.nr,
                    search=SearchConfig(search_radius=10, bfs_domain=BfsDomain.window),
                    refine=RefineConfig(tol=1e-4, max_iter=30),
                    grid=GridParams(half_width=8, spacing=6, margin=-1))
    return a, b, cfg


def flat_target():
    # test_integer_search.cpp:148-158: every position degenerate
    w = configs.crop(configs.get("c1"), 40, 40)
    a = w.frames[0].render(threads=1)
    b = np.full_like(a, 99)
    cfg = RunConfig(integer_method=IntegerMethod.mpso, subpixel_method=SubpixelMethod.icgn,
                    search=SearchConfig(search_radius=5, bfs_domain=BfsDomain.window, rng_seed=3),
                    grid=GridParams(half_width=8, spacing=5, margin=-1))
    return a, b, cfg


def whole_image():
    # BfsDomain::whole_image (the reference default, integer_search.cpp:23-33)
    w = configs.crop(configs.get("c1"), 48, 40)
    a = w.frames[0].render(threads=1)
    b = w.frames[1].render(threads=1)
    cfg = RunConfig(integer_method=IntegerMethod.bfs, subpixel_method=SubpixelMethod.icgn,
                    search=SearchConfig(search_radius=4, bfs_domain=BfsDomain.whole_image),
                    refine=RefineConfig(tol=1e-3, max_iter=20),
                    grid=GridParams(half_width=6, spacing=9, margin=-1))
    return a, b, cfg


def pso_defaults():
    # reference SearchConfig defaults (P=50, G=5, c1=c2=2) with plain PSO
    w = configs.crop(configs.get("c3"), 128, 128)
    a = w.frames[0].render(threads=1)
    b = w.frames[1].render(threads=1)
    cfg = RunConfig(integer_method=IntegerMethod.pso, subpixel_method=SubpixelMethod.nr,
                    search=SearchConfig(search_radius=12, bfs_domain=BfsDomain.window, rng_seed=42),
                    refine=RefineConfig(tol=1e-3, max_iter=20),
                    grid=GridParams(half_width=10, spacing=12, margin=-1))
    return a, b, cfg


def _pso_plain(cfg):
    cfg.integer_method = IntegerMethod.pso


CASES = {
    "c1_full": _cfg_case("c1"),
    "c2_crop128": _cfg_case("c2", 128),
    "c3_crop128": _cfg_case("c3", 128),
    "c3_pso_crop128": _cfg_case("c3", 128, mutate=_pso_plain),
    "c4_crop128": _cfg_case("c4", 128),
    "c5_crop160_pair17": _cfg_case("c5", 160, pair=17),
    "checkerboard_tie": checkerboard,
    "degenerate_half": degenerate_half,
    "flat_target": flat_target,
    "whole_image": whole_image,
    "pso_defaults": pso_defaults,
}
