"""Randomised end-to-end parity: seeded random geometries (frame size, pixel
type, subset half-width, lattice step, search radius, margin), search methods
(BFS window / whole image, PSO, mPSO, both inertia modes), refiners (none, NR,
IC-GN; bilinear and bicubic) and deformation fields, through the C-ABI against
the C restatement of the reference (oracle "port": it also carries the two
BASELINE extras the reference build lacks, bicubic and constant inertia).

The BASELINE configurations pin five geometries; the kernels pick different
instantiations off them (fixed-geometry IC-GN strips only for known (M, step),
block sums only for 16-bit data and >= 1024 POIs, tensor-core search for u8
windows, chunked windows for R > 31, ...). These cases walk the dispatch
around those points with the same bar as test_gpu_parity.py.

FUZZ_CASES=<n> widens the sweep (default 40 seeds); FUZZ_SEED0 moves it.
"""
import os

import numpy as np
import pytest

from paper_1905_06228_b200 import _abi, configs, dic
from test_gpu_parity import assert_parity, run_device

pytestmark = pytest.mark.gpu

N = int(os.environ.get("FUZZ_CASES", "40"))
SEED0 = int(os.environ.get("FUZZ_SEED0", "0"))
MIN_M = int(os.environ.get("FUZZ_MIN_M", "5"))


def make_case(seed):
    r = np.random.default_rng(90000 + seed)
    u16 = bool(r.integers(0, 2))
    big = r.random() < 0.25  # enough POIs for the >= 1024-POI search paths
    M = int(r.integers(MIN_M, 23))
    step = int(r.integers(3, 18))
    if r.random() < 0.3:  # BASELINE's own (M, step) pairs: the fixed-geometry strips
        M, step = [(20, 10), (20, 5), (15, 10), (15, 8), (10, 16)][int(r.integers(0, 5))]
    R = int(r.integers(2, 15)) if r.random() < 0.9 else int(r.integers(32, 40))
    if big:
        step = min(step, 6)
        W, H = int(r.integers(300, 420)), int(r.integers(300, 420))
    else:
        W, H = int(r.integers(2 * (M + R) + 40, 2 * (M + R) + 200)), int(r.integers(2 * (M + R) + 40, 2 * (M + R) + 200))
    if u16:
        bits = int(r.choice([10, 12, 12, 14, 16]))
        mx = (1 << bits) - 1
        ref = configs.FrameSpec(W, H, _abi.U16, mx, 7000 + seed, W * H // 42, (1.5, 3.5), (0.23 * mx, 0.78 * mx))
    else:
        ref = configs.FrameSpec(W, H, _abi.U8, 255, 7000 + seed, W * H // 60, (2.0, 4.0), (60.0, 200.0))
    lim = min(R - 0.6, 6.0)
    if r.random() < 0.7:
        a = (float(r.uniform(-lim, lim)), float(r.uniform(-0.004, 0.004)), float(r.uniform(-0.004, 0.004)),
             float(r.uniform(-lim, lim)), float(r.uniform(-0.004, 0.004)), float(r.uniform(-0.004, 0.004)),
             (W - 1) / 2.0, (H - 1) / 2.0)
        tgt = configs.replace(ref, field=_abi.FIELD_AFFINE, a=a)
    else:
        amp = min(lim, 2.0)
        tgt = configs.replace(ref, field=_abi.FIELD_SINUSOID,
                              a=(amp, float(r.uniform(150, 600)), 0.5 * amp, float(r.uniform(150, 800)), 0, 0, 0, 0))
    im = [dic.IntegerMethod.bfs, dic.IntegerMethod.bfs, dic.IntegerMethod.pso, dic.IntegerMethod.mpso][int(r.integers(0, 4))]
    sp = [dic.SubpixelMethod.none, dic.SubpixelMethod.nr, dic.SubpixelMethod.icgn, dic.SubpixelMethod.icgn][int(r.integers(0, 4))]
    domain = dic.BfsDomain.window
    if im == dic.IntegerMethod.bfs and not big and r.random() < 0.15:
        domain = dic.BfsDomain.whole_image
        R = min(R, 6)
    cfg = dic.RunConfig(
        integer_method=im, subpixel_method=sp,
        search=dic.SearchConfig(search_radius=R, bfs_domain=domain, particle_count=int(r.integers(5, 40)),
                                max_generations=int(r.integers(3, 25)), stop_threshold=float(r.choice([0.9, 0.995, 2.0])),
                                c1=float(r.uniform(1.0, 2.2)), c2=float(r.uniform(1.0, 2.2)),
                                rng_seed=int(r.integers(0, 1 << 62))),
        refine=dic.RefineConfig(tol=float(r.choice([1e-2, 1e-3, 1e-4])), max_iter=int(r.integers(5, 40))),
        grid=dic.GridParams(half_width=M, spacing=step, margin=-1 if r.random() < 0.7 else int(r.integers(M, M + R + 6))),
    )
    if r.random() < 0.3:
        cfg.inertia_mode = dic.InertiaMode.constant
        cfg.inertia_constant = float(r.uniform(0.4, 0.9))
    if sp != dic.SubpixelMethod.none and r.random() < 0.3:
        cfg.interp = dic.Interp.bicubic
    return ref, tgt, cfg, int(r.integers(0, 70))


# seeds kept for what they found: 316 = mPSO + fixed-geometry IC-GN (M 20, step 5) with one integer
# estimate far from its strip's median (the node pass's hoisted shared-memory loads faulted)
REGRESSIONS = [316]


@pytest.mark.parametrize("seed", list(range(SEED0, SEED0 + N)) + [s for s in REGRESSIONS if not SEED0 <= s < SEED0 + N])
def test_random_geometry_parity(gpu, port, seed):
    ref, tgt, cfg, pair_index = make_case(seed)
    a, b = ref.render(), tgt.render()
    exp = port.analyze_pair(a, b, cfg, pair_index=pair_index)
    got = run_device(a, b, cfg, pair_index=pair_index)
    tag = (f"{ref.width}x{ref.height} {'u16' if ref.dtype == _abi.U16 else 'u8'} max {ref.max_value} M{cfg.grid.half_width} "
           f"s{cfg.grid.spacing} R{cfg.search.search_radius} m{cfg.grid.margin} {cfg.integer_method.name}/"
           f"{cfg.subpixel_method.name}/{cfg.interp.name} pois {len(exp)}")
    try:
        worst = assert_parity(got, exp, iter_frac=0.01)
    except AssertionError as e:
        raise AssertionError(f"seed {seed}: {tag}: {e}") from None
    print(f"seed {seed}: {tag}: max|du,dv| {worst:.2e}")
