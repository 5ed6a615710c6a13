"""The five BASELINE.json configurations, as synthetic frame
specs + reference RunConfigs. Values BASELINE leaves open are pinned here
(marked "pinned"), and recorded in DESIGN.md.

Parity runs use the reference semantics: bilinear interpolation (the reference
has no bicubic, subpixel.cpp:59-102), the reference inertia schedule
w(t)=0.9-t/(2G) (integer_search.cpp:35-37) and MT19937-64 streams
(rng.hpp:20-33). BASELINE's literal "inertia 0.7" is available as
InertiaMode.constant (flagged extra, C3X).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace
from typing import List, Optional, Tuple

import numpy as np

from . import _abi
from .dic import (
    BfsDomain, GrayImage, GridParams, InertiaMode, IntegerMethod, Interp, RefineConfig, ReferencePolicy,
    RunConfig, SearchConfig, SubpixelMethod, lib,
)


@dataclass
class FrameSpec:
    width: int
    height: int
    dtype: int
    max_value: int
    seed: int
    blob_count: int
    sigma: Tuple[float, float]
    peak: Tuple[float, float]
    background: float = 0.0
    field: int = _abi.FIELD_NONE
    a: Tuple[float, ...] = (0.0,) * 8

    def to_c(self) -> _abi.SynthSpecC:
        s = _abi.SynthSpecC()
        s.width, s.height, s.dtype, s.max_value = self.width, self.height, self.dtype, self.max_value
        s.seed = self.seed
        s.blob_count = self.blob_count
        s.field = self.field
        s.sigma_min, s.sigma_max = self.sigma
        s.peak_min, s.peak_max = self.peak
        s.background = self.background
        a = list(self.a) + [0.0] * (8 - len(self.a))
        for i in range(8):
            s.a[i] = a[i]
        return s

    def render(self, threads: int = 0) -> np.ndarray:
        out = np.zeros((self.height, self.width), np.uint8 if self.dtype == _abi.U8 else np.uint16)
        st = lib().dicb200_synth_render(C.byref(self.to_c()), out.ctypes.data, self.width, threads)
        if st:
            raise RuntimeError("synth_render failed")
        return out

    def displacement(self, x: float, y: float) -> Tuple[float, float]:
        dx, dy = C.c_double(), C.c_double()
        lib().dicb200_synth_displacement(C.byref(self.to_c()), x, y, C.byref(dx), C.byref(dy))
        return dx.value, dy.value


@dataclass
class Workload:
    name: str
    frames: List[FrameSpec]
    cfg: RunConfig
    pairs: List[Tuple[int, int]]
    description: str = ""

    def subsets_per_pair(self) -> int:
        from .dic import grid_subsets

        g = self.cfg.grid
        return len(grid_subsets(self.frames[0].width, self.frames[0].height, g.half_width, g.spacing,
                                self.cfg.effective_margin()))


def _u8_frame(w: int, h: int, seed: int) -> FrameSpec:
    # C1-C3 recipe: sigma ~ U[2,4], peak ~ U[60,200], background 0, count W*H/60 (pinned)
    return FrameSpec(w, h, _abi.U8, 255, seed, w * h // 60, (2.0, 4.0), (60.0, 200.0))


def _u16_frame(w: int, h: int, seed: int) -> FrameSpec:
    # C4-C5 12-bit recipe: sigma ~ U[1.5,3.5], peak ~ U[960,3200] (pinned), count W*H/42 (pinned)
    return FrameSpec(w, h, _abi.U16, 4095, seed, w * h // 42, (1.5, 3.5), (960.0, 3200.0))


def _translated(f: FrameSpec, u: float, v: float) -> FrameSpec:
    return replace(f, field=_abi.FIELD_AFFINE, a=(u, 0.0, 0.0, v, 0.0, 0.0, 0.0, 0.0))


def c1() -> Workload:
    ref = _u8_frame(256, 256, seed=1)
    cfg = RunConfig(
        integer_method=IntegerMethod.bfs, subpixel_method=SubpixelMethod.none,
        search=SearchConfig(search_radius=10, bfs_domain=BfsDomain.window),
        grid=GridParams(half_width=10, spacing=16, margin=-1),
    )
    return Workload("c1", [ref, _translated(ref, 3.0, -5.0)], cfg, [(0, 1)],
                    "BFS-ZNCC only, 256^2 u8, M=10, step 16, R=10, rigid (+3,-5)")


def c2() -> Workload:
    ref = _u8_frame(512, 512, seed=2)
    cfg = RunConfig(
        integer_method=IntegerMethod.bfs, subpixel_method=SubpixelMethod.nr,
        search=SearchConfig(search_radius=15, bfs_domain=BfsDomain.window),
        refine=RefineConfig(tol=1e-4, max_iter=50),
        grid=GridParams(half_width=15, spacing=10, margin=-1),
    )
    return Workload("c2", [ref, _translated(ref, 2.37, -1.62)], cfg, [(0, 1)],
                    "BFS + NR (bilinear), 512^2 u8, M=15, step 10, R=15, (2.37,-1.62)")


def c3(inertia_constant: Optional[float] = None) -> Workload:
    ref = _u8_frame(1024, 1024, seed=3)
    tgt = replace(ref, field=_abi.FIELD_AFFINE, a=(1.5, 0.002, -0.001, -0.8, 0.0005, 0.0015, 0.0, 0.0))
    cfg = RunConfig(
        integer_method=IntegerMethod.mpso, subpixel_method=SubpixelMethod.nr,
        search=SearchConfig(search_radius=20, bfs_domain=BfsDomain.window, particle_count=20,
                            max_generations=30, stop_threshold=0.995, c1=1.5, c2=1.5, rng_seed=1),
        refine=RefineConfig(tol=1e-4, max_iter=50),  # pinned (BASELINE gives none for C3)
        grid=GridParams(half_width=15, spacing=8, margin=-1),
    )
    name = "c3"
    if inertia_constant is not None:
        cfg.inertia_mode = InertiaMode.constant
        cfg.inertia_constant = inertia_constant
        name = "c3x"
    return Workload(name, [ref, tgt], cfg, [(0, 1)],
                    "mPSO (P=20,G=30,c1=c2=1.5) + NR, 1024^2 u8, M=15, step 8, R=20, affine")


def c4() -> Workload:
    ref = _u16_frame(2048, 2048, seed=4)
    tgt = replace(ref, field=_abi.FIELD_SINUSOID, a=(2.0, 512.0, 1.0, 768.0, 0.0, 0.0, 0.0, 0.0))
    cfg = RunConfig(
        integer_method=IntegerMethod.bfs, subpixel_method=SubpixelMethod.icgn,
        search=SearchConfig(search_radius=5, bfs_domain=BfsDomain.window),  # R=5 pinned
        refine=RefineConfig(tol=1e-4, max_iter=30),
        grid=GridParams(half_width=20, spacing=5, margin=-1),
    )
    return Workload("c4", [ref, tgt], cfg, [(0, 1)],
                    "BFS + IC-GN, 2048^2 u16 12-bit, M=20, step 5, R=5, sinusoidal field")


C5_STRAIN = (0.002, -0.001, 0.0005, 0.0015)  # (exx, exy, eyx, eyy), pinned


def c5_shift(k: int) -> Tuple[float, float]:
    """Rigid shift of frame k ~ U[-8,8]^2 from seed 1000+k (pinned)."""
    s = np.random.default_rng(1000 + k).uniform(-8.0, 8.0, size=2)
    return float(s[0]), float(s[1])


def c5(n_pairs: int = 64) -> Workload:
    ref = _u16_frame(2048, 2048, seed=5)
    cx, cy = (ref.width - 1) / 2.0, (ref.height - 1) / 2.0
    frames = [ref]
    for k in range(1, n_pairs + 1):
        sx, sy = c5_shift(k)
        e = [x * k / 64.0 for x in C5_STRAIN]
        frames.append(replace(ref, field=_abi.FIELD_AFFINE, a=(sx, e[0], e[1], sy, e[2], e[3], cx, cy)))
    cfg = RunConfig(
        integer_method=IntegerMethod.bfs, subpixel_method=SubpixelMethod.icgn,
        reference_policy=ReferencePolicy.fixed_first,
        search=SearchConfig(search_radius=12, bfs_domain=BfsDomain.window),
        refine=RefineConfig(tol=1e-4, max_iter=30),
        grid=GridParams(half_width=20, spacing=10, margin=-1),
    )
    return Workload("c5", frames, cfg, [(0, k) for k in range(1, n_pairs + 1)],
                    "image-parallel sequence: 64 pairs 2048^2 u16, BFS + IC-GN, M=20, step 10, R=12")


ALL = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def c2b() -> Workload:
    """C2 with BASELINE's literal bicubic interpolation (B200 extension; the
    reference, and so every parity run, uses bilinear)."""
    w = c2()
    w.cfg.interp = Interp.bicubic
    return replace(w, name="c2b", description="BFS + NR (bicubic), 512^2 u8, M=15, step 10, R=15, (2.37,-1.62)")


def get(name: str) -> Workload:
    if name == "c3x":
        return c3(inertia_constant=0.7)
    if name == "c2b":
        return c2b()
    return ALL[name]()


def crop(w: Workload, width: int, height: int) -> Workload:
    """Same recipe on a smaller frame (fast parity cases)."""
    frames = []
    for f in w.frames:
        scale = (width * height) / (f.width * f.height)
        a = list(f.a)
        if f.field == _abi.FIELD_AFFINE and a[6] != 0.0:
            a[6], a[7] = (width - 1) / 2.0, (height - 1) / 2.0
        frames.append(replace(f, width=width, height=height, blob_count=max(1, int(f.blob_count * scale)), a=tuple(a)))
    return replace(w, frames=frames, name=w.name + f"_{width}x{height}")
