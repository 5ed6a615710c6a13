"""ctypes wrapper over the two CPU oracles (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

from paper_1905_06228_b200 import _abi

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "port": os.path.join(HERE, "libdicoracle.so"),
    "reference": os.path.join(HERE, "_ref", "libdicref.so"),
}
PREFIX = {"port": "dco_", "reference": "dicref_"}
REFERENCE_SRC = "/root/reference/proj/core"


def build(verbose: bool = False) -> None:
    """Compile the port always; the reference build only where its sources exist."""
    targets = ["oracle"]
    if os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
        if os.path.exists(os.path.join(HERE, "..", "paper_1905_06228_b200", "libdicb200.so")):
            targets.append("shim")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


def available(kind: str) -> bool:
    return os.path.exists(PATHS[kind])


class OracleError(RuntimeError):
    pass


def _as_double(img: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(img, dtype=np.float64)


class Oracle:
    def __init__(self, kind: str = "port"):
        if not available(kind):
            raise FileNotFoundError(PATHS[kind])
        self.kind = kind
        self.L = C.CDLL(PATHS[kind])
        self.p = PREFIX[kind]
        f = self._f
        f("derive_stream_seed").restype = C.c_uint64
        f("derive_stream_seed").argtypes = [C.c_uint64] * 3
        f("interp_bilinear").restype = C.c_double
        f("interp_bilinear").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(C.c_int)]
        f("mt64").argtypes = [C.c_uint64, C.c_size_t, C.c_void_p]
        f("uniform01").argtypes = [C.c_uint64, C.c_size_t, C.c_void_p]
        f("integer_search").argtypes = [
            C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_abi.RunConfigC),
            C.c_uint64, C.c_void_p, C.POINTER(C.c_double), C.c_void_p, C.c_char_p, C.c_size_t,
        ]
        f("refine").argtypes = [
            C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
            C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t,
        ]
        f("zncc").argtypes = [
            C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
            C.POINTER(C.c_double), C.c_char_p, C.c_size_t,
        ]
        f("icgn_hessian").argtypes = [
            C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_double),
            C.c_char_p, C.c_size_t,
        ]
        f("grid").argtypes = [
            C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t),
            C.c_char_p, C.c_size_t,
        ]
        if kind == "port":
            f("analyze_pair").argtypes = [
                C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(_abi.RunConfigC), C.c_uint64, C.c_int,
                C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t,
            ]
            f("analyze_pair_rows").argtypes = [
                C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(_abi.RunConfigC), C.c_uint64, C.c_int,
                C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t,
            ]
        else:
            f("analyze_pair").argtypes = [
                C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(_abi.RunConfigC), C.c_uint64,
                C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t,
            ]
            f("analyze_pair_timed").argtypes = [
                C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(_abi.RunConfigC), C.c_uint64, C.c_int,
                C.POINTER(C.c_double), C.POINTER(C.c_size_t), C.c_void_p, C.c_size_t, C.c_char_p, C.c_size_t,
            ]
            f("analyze_sequence").argtypes = [
                C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.POINTER(_abi.RunConfigC), C.POINTER(_abi.FieldC),
                C.c_size_t, C.POINTER(C.c_double),
            ]
            f("hardware_threads").restype = C.c_uint

    def _f(self, name):
        return getattr(self.L, self.p + name)

    # -- pipeline ---------------------------------------------------------
    def grid(self, w: int, h: int, half_width: int, spacing: int, margin: int):
        n = C.c_size_t(0)
        err = C.create_string_buffer(160)
        if self._f("grid")(w, h, half_width, spacing, margin, None, 0, C.byref(n), err, 160):
            raise OracleError(err.value.decode())
        xy = np.zeros(2 * n.value, np.int32)
        self._f("grid")(w, h, half_width, spacing, margin, xy.ctypes.data, n.value, C.byref(n), err, 160)
        return xy.reshape(-1, 2)

    def analyze_pair(self, ref: np.ndarray, tgt: np.ndarray, cfg, pair_index: int = 0, threads: int = 0) -> np.ndarray:
        """cfg: paper_1905_06228_b200.dic.RunConfig. threads: port worker threads
        (0 = all cores); the reference build takes cfg.mode/worker_count."""
        a, b = _as_double(ref), _as_double(tgt)
        h, w = a.shape
        c = cfg.to_c()
        g = self.grid(w, h, cfg.grid.half_width, cfg.grid.spacing, cfg.effective_margin())
        out = np.zeros(len(g), dtype=_abi.record_dtype())
        n = C.c_size_t(0)
        err = C.create_string_buffer(160)
        if self.kind == "port":
            if threads <= 0:
                threads = os.cpu_count() or 1
            st = self._f("analyze_pair")(a.ctypes.data, b.ctypes.data, w, h, C.byref(c), pair_index, threads,
                                         out.ctypes.data, len(out), C.byref(n), err, 160)
        else:
            st = self._f("analyze_pair")(a.ctypes.data, b.ctypes.data, w, h, C.byref(c), pair_index,
                                         out.ctypes.data, len(out), C.byref(n), err, 160)
        if st:
            raise OracleError(err.value.decode())
        return out[: n.value]

    def analyze_pair_rows(self, ref, tgt, cfg, pair_index: int, row_begin: int, row_end: int, threads: int = 0):
        """Port only: grid rows [row_begin, row_end) with global subset indices."""
        a, b = _as_double(ref), _as_double(tgt)
        h, w = a.shape
        c = cfg.to_c()
        g = self.grid(w, h, cfg.grid.half_width, cfg.grid.spacing, cfg.effective_margin())
        out = np.zeros(len(g), dtype=_abi.record_dtype())
        n = C.c_size_t(0)
        err = C.create_string_buffer(160)
        if threads <= 0:
            threads = os.cpu_count() or 1
        if self._f("analyze_pair_rows")(a.ctypes.data, b.ctypes.data, w, h, C.byref(c), pair_index, threads,
                                        row_begin, row_end, out.ctypes.data, len(out), C.byref(n), err, 160):
            raise OracleError(err.value.decode())
        return out[: n.value]

    def analyze_pair_timed(self, ref, tgt, cfg, pair_index=0, repeats=1, records: bool = False):
        """Reference build only: seconds (best of repeats) of dic::analyze_pair
        alone, the POI count and (records=True) the last repeat's records."""
        a, b = _as_double(ref), _as_double(tgt)
        h, w = a.shape
        c = cfg.to_c()
        s = C.c_double(0)
        n = C.c_size_t(0)
        err = C.create_string_buffer(160)
        out, cap = None, 0
        if records:
            cap = len(self.grid(w, h, cfg.grid.half_width, cfg.grid.spacing, cfg.effective_margin()))
            out = np.zeros(cap, dtype=_abi.record_dtype())
        if self._f("analyze_pair_timed")(a.ctypes.data, b.ctypes.data, w, h, C.byref(c), pair_index, repeats,
                                         C.byref(s), C.byref(n), out.ctypes.data if records else None, cap,
                                         err, 160):
            raise OracleError(err.value.decode())
        if records:
            return s.value, n.value, out[: n.value]
        return s.value, n.value

    # -- per-subset pins ---------------------------------------------------
    def zncc(self, ref, tgt, cx, cy, m, dx, dy) -> float:
        a, b = _as_double(ref), _as_double(tgt)
        out = C.c_double(0)
        err = C.create_string_buffer(160)
        if self._f("zncc")(a.ctypes.data, b.ctypes.data, a.shape[1], a.shape[0], cx, cy, m, dx, dy, C.byref(out), err, 160):
            raise OracleError(err.value.decode())
        return out.value

    def integer_search(self, ref, tgt, cx, cy, m, cfg, stream_seed: int):
        a, b = _as_double(ref), _as_double(tgt)
        ires = np.zeros(3, np.int32)
        ev = np.zeros(2, np.int64)
        z = C.c_double(0)
        err = C.create_string_buffer(160)
        c = cfg.to_c()
        if self._f("integer_search")(a.ctypes.data, b.ctypes.data, a.shape[1], a.shape[0], cx, cy, m, C.byref(c),
                                     stream_seed, ires.ctypes.data, C.byref(z), ev.ctypes.data, err, 160):
            raise OracleError(err.value.decode())
        return dict(dx=int(ires[0]), dy=int(ires[1]), generations_used=int(ires[2]), zncc=z.value,
                    evaluations=int(ev[0]), update_evaluations=int(ev[1]))

    def refine(self, ref, tgt, cx, cy, m, init, method: str, tol: float, max_iter: int):
        a, b = _as_double(ref), _as_double(tgt)
        out = np.zeros(7)
        ic = np.zeros(2, np.int32)
        err = C.create_string_buffer(160)
        if self._f("refine")(a.ctypes.data, b.ctypes.data, a.shape[1], a.shape[0], cx, cy, m, init[0], init[1],
                             0 if method == "nr" else 1, tol, max_iter, out.ctypes.data, ic.ctypes.data, err, 160):
            raise OracleError(err.value.decode())
        return dict(u=out[0], v=out[1], zncc=out[2], ux=out[3], uy=out[4], vx=out[5], vy=out[6],
                    iterations=int(ic[0]), converged=bool(ic[1]))

    def icgn_hessian(self, ref, cx, cy, m):
        a = _as_double(ref)
        hs = np.zeros(36)
        cond = C.c_double(0)
        err = C.create_string_buffer(160)
        if self._f("icgn_hessian")(a.ctypes.data, a.shape[1], a.shape[0], cx, cy, m, hs.ctypes.data, C.byref(cond), err, 160):
            raise OracleError(err.value.decode())
        return hs.reshape(6, 6), cond.value

    def interp_bilinear(self, img, x, y) -> Optional[float]:
        a = _as_double(img)
        ok = C.c_int(0)
        v = self._f("interp_bilinear")(a.ctypes.data, a.shape[1], a.shape[0], x, y, C.byref(ok))
        return v if ok.value else None

    def interp_bicubic(self, img, x, y):
        """Port only: the bicubic variant (parity unpinned) -> (value or None, (gx, gy) or None)."""
        a = _as_double(img)
        L = self.L
        L.dco_interp_bicubic.restype = C.c_double
        L.dco_interp_bicubic.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(C.c_int)]
        L.dco_grad_bicubic.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        ok = C.c_int(0)
        v = L.dco_interp_bicubic(a.ctypes.data, a.shape[1], a.shape[0], x, y, C.byref(ok))
        gx, gy = C.c_double(), C.c_double()
        gok = L.dco_grad_bicubic(a.ctypes.data, a.shape[1], a.shape[0], x, y, C.byref(gx), C.byref(gy))
        return (v if ok.value else None), ((gx.value, gy.value) if gok else None)

    def derive_stream_seed(self, seed, pair, subset) -> int:
        return int(self._f("derive_stream_seed")(seed, pair, subset))

    def mt64(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self._f("mt64")(seed, n, out.ctypes.data)
        return out

    def uniform01(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.float64)
        self._f("uniform01")(seed, n, out.ctypes.data)
        return out


# -- f-4: the reference's generators and accuracy sweep (reference build only) ----
def _ref_lib():
    L = C.CDLL(PATHS["reference"])
    L.dicref_synth_speckle.argtypes = [C.c_int, C.c_int, C.c_uint64, C.POINTER(_abi.SpeckleParamsC), C.c_void_p,
                                       C.c_char_p, C.c_size_t]
    L.dicref_synth_warped_pair.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(_abi.WarpSpecC), C.c_void_p,
                                           C.c_void_p, C.c_char_p, C.c_size_t]
    L.dicref_accuracy_sweep.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(_abi.SweepConfigC),
                                        C.POINTER(_abi.ComboAccuracyC), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
    return L


def ref_synth_speckle(width: int, height: int, seed: int, params) -> np.ndarray:
    """dic::synth_speckle (synth.cpp:55-93); params: dic.SpeckleParams."""
    out = np.zeros((height, width), np.float64)
    err = C.create_string_buffer(160)
    if _ref_lib().dicref_synth_speckle(width, height, seed, C.byref(params.to_c()), out.ctypes.data, err, 160):
        raise OracleError(err.value.decode())
    return out


def ref_synth_warped_pair(reference: np.ndarray, warp) -> Tuple[np.ndarray, np.ndarray]:
    """dic::synth_warped_pair (synth.cpp:127-172); warp: dic.WarpSpec."""
    ref = _as_double(reference)
    tgt, mask = np.zeros_like(ref), np.zeros(ref.shape, np.uint8)
    err = C.create_string_buffer(160)
    if _ref_lib().dicref_synth_warped_pair(ref.ctypes.data, ref.shape[1], ref.shape[0], C.byref(warp.to_c()),
                                           tgt.ctypes.data, mask.ctypes.data, err, 160):
        raise OracleError(err.value.decode())
    return tgt, mask


def ref_accuracy_sweep(combos, cfg):
    """dic::run_accuracy_sweep (accuracy.cpp:10-78) on the reference's own
    double frames. Returns (list of ComboAccuracyC, warp_count, poi_count, elapsed_s)."""
    arr = np.array([[int(a), int(b)] for a, b in combos], np.int32)
    out = (_abi.ComboAccuracyC * len(combos))()
    c, keep = cfg.to_c()
    wc, pc, el = C.c_int(), C.c_int(), C.c_double()
    err = C.create_string_buffer(160)
    if _ref_lib().dicref_accuracy_sweep(arr.ctypes.data, len(combos), C.byref(c), out, C.byref(wc), C.byref(pc),
                                        C.byref(el), err, 160):
        raise OracleError(err.value.decode())
    return list(out), wc.value, pc.value, el.value


# -- synthetic frames without the product library (bench reference arm) -------
PATHS_SYNTH = os.path.join(HERE, "libdicsynth.so")


def render_rows(spec, row_begin: int = 0, row_end: Optional[int] = None, threads: int = 0) -> np.ndarray:
    """Rows [row_begin, row_end) of a configs.FrameSpec frame rendered by
    oracle/libdicsynth.so (the host generator synth.c built on its own): the
    same pixels as FrameSpec.render() / the device renderer, without loading
    libdicb200.so into the calling process."""
    L = C.CDLL(PATHS_SYNTH)
    L.dicb200_synth_render_rows.argtypes = [C.POINTER(_abi.SynthSpecC), C.c_void_p, C.c_int32, C.c_int32,
                                            C.c_int32, C.c_int32]
    if row_end is None:
        row_end = spec.height
    out = np.zeros((row_end - row_begin, spec.width), np.uint8 if spec.dtype == _abi.U8 else np.uint16)
    if L.dicb200_synth_render_rows(C.byref(spec.to_c()), out.ctypes.data, spec.width, row_begin, row_end, threads):
        raise OracleError("synth_render_rows failed")
    return out
