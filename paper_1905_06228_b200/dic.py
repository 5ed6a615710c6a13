"""Host-side mirror of the reference's `namespace dic` pipeline interface.

Same names, argument meaning and error behaviour as
/root/reference/proj/core/include/dic/{pipeline,integer_search,subpixel,image}.hpp,
so parity tests read like the reference's own tests. Every call goes through
the C-ABI library libdicb200.so (include/dicb200.h) onto the sm_100a kernels;
there is no CPU fallback: a missing library or a missing GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Sequence, Tuple

import numpy as np

from . import _abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DICB200_LIB") or os.path.join(_HERE, "libdicb200.so")  # override: A/B builds


class DicError(RuntimeError):
    """Mirror of dic::Error (error.hpp:10-13): recoverable engine failures."""


class IntegerMethod(IntEnum):  # pipeline.hpp:17
    bfs = 0
    pso = 1
    mpso = 2


class SubpixelMethod(IntEnum):  # pipeline.hpp:18
    nr = 0
    icgn = 1
    none = 2


class ExecMode(IntEnum):  # pipeline.hpp:19
    serial = 0
    subimage_parallel = 1
    image_parallel = 2


class ReferencePolicy(IntEnum):  # pipeline.hpp:20
    update_every_pair = 0
    fixed_first = 1


class BfsDomain(IntEnum):  # integer_search.hpp:12
    window = 0
    whole_image = 1


class InertiaMode(IntEnum):  # B200 extension (BASELINE asks for constant 0.7)
    reference_schedule = 0
    constant = 1


class Interp(IntEnum):  # B200 extension: BASELINE's "bicubic interpolation" (parity unpinned)
    bilinear = 0  # the reference's interp_bilinear / grad_bilinear (subpixel.cpp:59-128)
    bicubic = 1   # Keys cubic convolution a = -0.5, analytic gradient (include/dicb200.h)


@dataclass
class SearchConfig:  # integer_search.hpp:14-23
    search_radius: int = 25
    bfs_domain: BfsDomain = BfsDomain.whole_image
    particle_count: int = 50
    max_generations: int = 5
    stop_threshold: float = 0.995
    c1: float = 2.0
    c2: float = 2.0
    rng_seed: int = 0


@dataclass
class RefineConfig:  # subpixel.hpp:41-44
    tol: float = 0.01
    max_iter: int = 20


@dataclass
class GridParams:  # pipeline.hpp:27-31
    half_width: int = 15
    spacing: int = 10
    margin: int = -1


@dataclass
class RunConfig:  # pipeline.hpp:33-49
    integer_method: IntegerMethod = IntegerMethod.mpso
    subpixel_method: SubpixelMethod = SubpixelMethod.nr
    mode: ExecMode = ExecMode.serial
    reference_policy: ReferencePolicy = ReferencePolicy.update_every_pair
    worker_count: int = 1
    search: SearchConfig = field(default_factory=SearchConfig)
    refine: RefineConfig = field(default_factory=RefineConfig)
    grid: GridParams = field(default_factory=GridParams)
    inertia_mode: InertiaMode = InertiaMode.reference_schedule
    inertia_constant: float = 0.7
    interp: Interp = Interp.bilinear

    def effective_margin(self) -> int:
        return self.grid.margin if self.grid.margin >= 0 else self.grid.half_width + self.search.search_radius

    def effective_workers(self) -> int:
        return 1 if self.mode == ExecMode.serial else max(1, self.worker_count)

    def to_c(self) -> _abi.RunConfigC:
        c = _abi.RunConfigC()
        c.integer_method = int(self.integer_method)
        c.subpixel_method = int(self.subpixel_method)
        c.mode = int(self.mode)
        c.reference_policy = int(self.reference_policy)
        c.worker_count = int(self.worker_count)
        c.search_radius = int(self.search.search_radius)
        c.bfs_domain = int(self.search.bfs_domain)
        c.particle_count = int(self.search.particle_count)
        c.max_generations = int(self.search.max_generations)
        c.stop_threshold = float(self.search.stop_threshold)
        c.c1 = float(self.search.c1)
        c.c2 = float(self.search.c2)
        c.rng_seed = int(self.search.rng_seed) & 0xFFFFFFFFFFFFFFFF
        c.tol = float(self.refine.tol)
        c.max_iter = int(self.refine.max_iter)
        c.half_width = int(self.grid.half_width)
        c.spacing = int(self.grid.spacing)
        c.margin = int(self.grid.margin)
        c.inertia_mode = int(self.inertia_mode)
        c.inertia_constant = float(self.inertia_constant)
        c.interp = int(self.interp)
        return c


class GrayImage:
    """Immutable single-channel image (image.hpp:14-31).

    The reference stores doubles; the device path stores integer gray levels
    in [0, 65535] losslessly as uint8 / uint16 (the exact-integer search
    kernels). Any other finite levels — e.g. the reference's fractional
    synthetic frames — stay doubles and run on the exact fp64 path (the
    integer search evaluates the reference's zncc in its own order, bit for
    bit; the refiners gather fp32 from the fp64 image), as the C++ shim
    (include/dic_b200/pipeline.hpp) does. Non-finite levels raise DicError
    (image.cpp:14-22).
    """

    def __init__(self, pixels: np.ndarray, id: int = 0):
        a = np.asarray(pixels)
        if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
            raise DicError("zero-dimension image")
        if a.dtype == np.uint8 or a.dtype == np.uint16:
            px = np.ascontiguousarray(a)
        else:
            f = a.astype(np.float64)
            if not np.all(np.isfinite(f)):
                raise DicError("non-finite gray level")
            if np.all(f == np.round(f)) and f.min() >= 0 and f.max() <= 65535:
                px = np.ascontiguousarray(f.astype(np.uint8 if f.max() <= 255 else np.uint16))
            else:
                px = np.ascontiguousarray(f)  # fractional (or out-of-range) levels: fp64 path
        px.setflags(write=False)
        self._px = px
        self._id = int(id)

    def width(self) -> int:
        return self._px.shape[1]

    def height(self) -> int:
        return self._px.shape[0]

    def id(self) -> int:
        return self._id

    def pixels(self) -> np.ndarray:
        return self._px

    def at(self, x: int, y: int) -> float:
        return float(self._px[y, x])

    def as_c(self) -> _abi.Image:
        im = _abi.Image()
        im.width = self.width()
        im.height = self.height()
        im.pitch = self.width()
        im.dtype = {np.dtype(np.uint8): _abi.U8, np.dtype(np.uint16): _abi.U16}.get(self._px.dtype, _abi.F64)
        im.id = self._id
        im.bits = self.bits() if im.dtype != _abi.F64 else 0
        im.data = self._px.ctypes.data
        return im

    def bits(self) -> int:
        """Significant bits of the largest gray level (dicb200_image.bits): lets
        12-bit data in u16 storage take the exact 32-bit integer paths."""
        if not hasattr(self, "_bits"):
            self._bits = max(1, int(self._px.max()).bit_length())
        return self._bits


@dataclass
class DisplacementField:  # pipeline.hpp:61-67
    pair_index: int = 0
    ref_id: int = 0
    tgt_id: int = 0
    records: np.ndarray = None  # structured array, dtype = _abi.record_dtype()
    error: str = ""

    def failed(self) -> bool:
        return bool(self.error)


_lib_handle = None


def lib() -> C.CDLL:
    """The product library. Raises (never falls back) when it is missing."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = C.CDLL(LIB_PATH)
        L.dicb200_last_error_message.restype = C.c_char_p
        L.dicb200_launch_count.restype = C.c_uint64
        L.dicb200_analyze_pair.argtypes = [
            C.POINTER(_abi.Image), C.POINTER(_abi.Image), C.POINTER(_abi.RunConfigC), C.c_uint64,
            C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t),
        ]
        L.dicb200_analyze_pair_device.argtypes = [
            C.POINTER(_abi.Image), C.POINTER(_abi.Image), C.POINTER(_abi.RunConfigC), C.c_uint64,
            C.c_int32, C.c_int32, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t), C.c_void_p,
        ]
        L.dicb200_analyze_sequence.argtypes = [
            C.POINTER(_abi.Image), C.c_size_t, C.POINTER(_abi.RunConfigC), C.POINTER(_abi.FieldC), C.c_size_t,
        ]
        L.dicb200_grid_size.argtypes = [C.c_int32, C.c_int32, C.POINTER(_abi.RunConfigC), C.POINTER(C.c_size_t)]
        L.dicb200_grid.argtypes = [
            C.c_int32, C.c_int32, C.POINTER(_abi.RunConfigC), C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t),
        ]
        L.dicb200_sequence_pairs.argtypes = [C.c_int32, C.c_int32, C.c_void_p]
        L.dicb200_partition_ranges.argtypes = [C.c_size_t, C.c_int32, C.c_void_p]
        L.dicb200_synth_render.argtypes = [C.POINTER(_abi.SynthSpecC), C.c_void_p, C.c_int32, C.c_int32]
        L.dicb200_load_pgm.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_void_p, C.c_size_t]
        L.dicb200_save_pgm.argtypes = [C.c_char_p, C.POINTER(_abi.Image)]
        L.dicb200_sequence_files.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p, C.c_size_t,
                                             C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        L.dicb200_host_alloc.restype = C.c_void_p
        L.dicb200_host_alloc.argtypes = [C.c_size_t]
        L.dicb200_host_free.argtypes = [C.c_void_p]
        L.dicb200_synth_displacement.argtypes = [
            C.POINTER(_abi.SynthSpecC), C.c_double, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
        ]
        L.dicb200_synth_speckle.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.POINTER(_abi.SpeckleParamsC),
                                            C.c_void_p]
        L.dicb200_synth_warped_pair.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(_abi.WarpSpecC),
                                                C.c_void_p, C.c_void_p]
        L.dicb200_accuracy_sweep.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(_abi.SweepConfigC),
                                             C.POINTER(_abi.ComboAccuracyC), C.POINTER(C.c_int32),
                                             C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        L.dicb200_default_speckle.argtypes = [C.POINTER(_abi.SpeckleParamsC)]
        L.dicb200_default_sweep.argtypes = [C.POINTER(_abi.SweepConfigC)]
        L.dicb200_field_csv.argtypes = [C.POINTER(_abi.FieldC), C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.dicb200_write_field_csv.argtypes = [C.POINTER(_abi.FieldC), C.c_char_p]
        L.dicb200_field_filename.argtypes = [C.c_int32, C.c_char_p, C.c_size_t]
        L.dicb200_auto_repeats.argtypes = [C.c_double]
        L.dicb200_run_bench.argtypes = [C.POINTER(_abi.BenchCellC), C.c_size_t, C.c_char_p, C.c_char_p,
                                        C.POINTER(_abi.RunConfigC), C.c_int32, C.c_int32, C.c_char_p, C.c_int32,
                                        C.POINTER(_abi.BenchRecordC)]
        L.dicb200_derive_ratios.argtypes = [C.POINTER(_abi.BenchRecordC), C.c_size_t, C.c_char_p,
                                            C.POINTER(_abi.RatioRowC), C.c_size_t, C.POINTER(C.c_size_t)]
        L.dicb200_write_times_csv.argtypes = [C.POINTER(_abi.BenchRecordC), C.c_size_t, C.c_char_p, C.c_char_p]
        L.dicb200_write_records_csv.argtypes = [C.POINTER(_abi.BenchRecordC), C.c_size_t, C.c_char_p]
        L.dicb200_write_ratios_csv.argtypes = [C.POINTER(_abi.RatioRowC), C.c_size_t, C.c_char_p]
        _lib_handle = L
    return _lib_handle


def _raise(status: int) -> None:
    msg = lib().dicb200_last_error_message().decode()
    if status == 1:
        raise DicError(msg)
    raise RuntimeError(f"dicb200 status {status}: {msg}")


def load_image(path, allow_16bit: bool = False, id: int = 0) -> GrayImage:
    """image.cpp:60-96 (dic::load_image), native: P5/P2 graymaps, byte n -> gray
    level n; raises DicError with the reference's messages. allow_16bit also
    accepts maxval 256..65535 (the reference rejects it)."""
    L = lib()
    w, h, dt, mv = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    flags = 1 if allow_16bit else 0
    st = L.dicb200_load_pgm(str(path).encode(), flags, C.byref(w), C.byref(h), C.byref(dt), C.byref(mv), None, 0)
    if st:
        _raise(st)
    px = np.empty((h.value, w.value), np.uint8 if dt.value == _abi.U8 else np.uint16)
    st = L.dicb200_load_pgm(str(path).encode(), flags, C.byref(w), C.byref(h), C.byref(dt), C.byref(mv),
                            px.ctypes.data, px.size)
    if st:
        _raise(st)
    return GrayImage(px, id)


def save_pgm(img: GrayImage, path) -> None:
    """image.cpp:98-111 (dic::save_pgm): 8-bit P5, values clamped to 255."""
    im = img.as_c()
    st = lib().dicb200_save_pgm(str(path).encode(), C.byref(im))
    if st:
        _raise(st)


def sequence_files(directory, pattern: str) -> List[str]:
    """The file list of dic::load_sequence (image.cpp:113-138): regular files
    matching the glob, lexicographic by filename, at least two."""
    L = lib()
    need, cnt = C.c_size_t(), C.c_size_t()
    st = L.dicb200_sequence_files(str(directory).encode(), pattern.encode(), None, 0, C.byref(need), C.byref(cnt))
    if st:
        _raise(st)
    buf = C.create_string_buffer(need.value)
    st = L.dicb200_sequence_files(str(directory).encode(), pattern.encode(), buf, need.value, C.byref(need),
                                  C.byref(cnt))
    if st:
        _raise(st)
    return [n.decode() for n in buf.raw[: need.value].split(b"\0")[: cnt.value]]


class PinnedBlock:
    """Page-locked host memory from dicb200_host_alloc (cudaMallocHost), freed
    when the last array viewing it is collected. Frames in pinned memory are
    uploaded by analyze_sequence with asynchronous copies that overlap the
    previous pair's kernels."""

    def __init__(self, nbytes: int):
        self.nbytes = max(int(nbytes), 1)
        self.ptr = lib().dicb200_host_alloc(self.nbytes)
        if not self.ptr:
            raise DicError("pinned host allocation failed (%d bytes)" % self.nbytes)
        self.__array_interface__ = {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False),
                                    "version": 3}

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().dicb200_host_free(C.c_void_p(self.ptr))
            self.ptr = None

    def view(self, offset: int, shape, dtype) -> np.ndarray:
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        return np.asarray(self)[offset:offset + n].view(dtype).reshape(shape)


def _load_into(path, allow_16bit, out: np.ndarray, dtype_code: int):
    L = lib()
    w, h, dt, mv = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    st = L.dicb200_load_pgm(str(path).encode(), 1 if allow_16bit else 0, C.byref(w), C.byref(h), C.byref(dt),
                            C.byref(mv), out.ctypes.data, out.size)
    if st:
        _raise(st)
    assert dt.value == dtype_code


def load_sequence(directory, pattern: str, allow_16bit: bool = False, pinned: bool = False) -> List[GrayImage]:
    """image.cpp:113-138 (dic::load_sequence): ids are the sequence positions;
    frames must share dimensions ("dimension mismatch in sequence: <file>").
    pinned=True reads every frame straight into one page-locked host block."""
    names = sequence_files(directory, pattern)
    if pinned:
        return _load_sequence_pinned(directory, names, allow_16bit)
    images: List[GrayImage] = []
    for i, name in enumerate(names):
        path = os.path.join(str(directory), name)
        img = load_image(path, allow_16bit, id=i)
        if images and (img.width() != images[0].width() or img.height() != images[0].height()):
            raise DicError("dimension mismatch in sequence: " + path)
        images.append(img)
    return images


def _load_sequence_pinned(directory, names: List[str], allow_16bit: bool) -> List[GrayImage]:
    L = lib()
    heads = []
    for name in names:  # header pass: dimensions, sample width, error order as the reference
        path = os.path.join(str(directory), name)
        w, h, dt, mv = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        st = L.dicb200_load_pgm(path.encode(), 1 if allow_16bit else 0, C.byref(w), C.byref(h), C.byref(dt),
                                C.byref(mv), None, 0)
        if st:
            _raise(st)
        if heads and (w.value != heads[0][1] or h.value != heads[0][2]):
            raise DicError("dimension mismatch in sequence: " + path)
        heads.append((path, w.value, h.value, dt.value))
    sizes = [w * h * (1 if dt == _abi.U8 else 2) for _, w, h, dt in heads]
    offs = np.concatenate([[0], np.cumsum([(s + 255) // 256 * 256 for s in sizes])]).astype(np.int64)
    block = PinnedBlock(int(offs[-1]))
    images: List[GrayImage] = []
    for i, (path, w, h, dt) in enumerate(heads):
        arr = block.view(int(offs[i]), (h, w), np.uint8 if dt == _abi.U8 else np.uint16)
        _load_into(path, allow_16bit, arr, dt)
        images.append(GrayImage(arr, i))
    return images


def grid_subsets(width: int, height: int, half_width: int, spacing: int, margin: int) -> List[Tuple[int, int]]:
    """image.cpp:140-158 (through the C-ABI, no GPU needed)."""
    cfg = RunConfig()
    cfg.grid = GridParams(half_width, spacing, margin)
    c = cfg.to_c()
    n = C.c_size_t(0)
    st = lib().dicb200_grid_size(width, height, C.byref(c), C.byref(n))
    if st:
        _raise(st)
    xy = np.zeros(2 * n.value, np.int32)
    st = lib().dicb200_grid(width, height, C.byref(c), xy.ctypes.data, n.value, C.byref(n))
    if st:
        _raise(st)
    return [(int(xy[2 * i]), int(xy[2 * i + 1])) for i in range(n.value)]


def sequence_pairs(policy: ReferencePolicy, image_count: int) -> List[Tuple[int, int]]:
    """pipeline.cpp:43-54."""
    if image_count < 2:
        raise DicError("insufficient images")
    out = np.zeros(2 * (image_count - 1), np.int32)
    st = lib().dicb200_sequence_pairs(int(policy), image_count, out.ctypes.data)
    if st:
        _raise(st)
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(image_count - 1)]


def partition_ranges(n: int, workers: int) -> List[Tuple[int, int]]:
    """pipeline.cpp:56-69."""
    if workers < 1:
        raise DicError("worker count must be >= 1")
    out = np.zeros(2 * workers, np.uint64)
    st = lib().dicb200_partition_ranges(n, workers, out.ctypes.data)
    if st:
        _raise(st)
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(workers)]


def analyze_pair(reference: GrayImage, target: GrayImage, cfg: RunConfig, pair_index: int = 0) -> DisplacementField:
    """pipeline.hpp:76-77 / pipeline.cpp:147-180, on the GPU."""
    if reference.width() != target.width() or reference.height() != target.height():
        raise DicError("dimension mismatch")
    c = cfg.to_c()
    n = C.c_size_t(0)
    st = lib().dicb200_grid_size(reference.width(), reference.height(), C.byref(c), C.byref(n))
    if st:
        _raise(st)
    recs = np.zeros(n.value, dtype=_abi.record_dtype())
    a, b = reference.as_c(), target.as_c()
    cnt = C.c_size_t(0)
    st = lib().dicb200_analyze_pair(C.byref(a), C.byref(b), C.byref(c), pair_index, recs.ctypes.data, n.value, C.byref(cnt))
    if st:
        _raise(st)
    return DisplacementField(pair_index, reference.id(), target.id(), recs[: cnt.value], "")


def analyze_sequence(images: Sequence[GrayImage], cfg: RunConfig) -> List[DisplacementField]:
    """pipeline.hpp:79-80 / pipeline.cpp:182-214, on the GPU(s)."""
    pairs = sequence_pairs(cfg.reference_policy, len(images))
    c = cfg.to_c()
    imgs = (_abi.Image * len(images))(*[im.as_c() for im in images])
    fields = (_abi.FieldC * len(pairs))()
    bufs = []
    for i, (ra, tb) in enumerate(pairs):
        n = C.c_size_t(0)
        st = lib().dicb200_grid_size(images[ra].width(), images[ra].height(), C.byref(c), C.byref(n))
        cap = n.value if st == 0 else 0
        buf = np.zeros(max(cap, 1), dtype=_abi.record_dtype())
        bufs.append(buf)
        fields[i].records = C.cast(buf.ctypes.data, C.POINTER(_abi.PoiRecordC))
        fields[i].capacity = cap
    st = lib().dicb200_analyze_sequence(imgs, len(images), C.byref(c), fields, len(pairs))
    if st:
        _raise(st)
    out = []
    for i in range(len(pairs)):
        f = fields[i]
        out.append(DisplacementField(f.pair_index, f.ref_id, f.tgt_id, bufs[i][: f.count], f.error.decode()))
    return out


def _field_c(field_: DisplacementField):
    recs = np.ascontiguousarray(field_.records if field_.records is not None else
                                np.zeros(0, _abi.record_dtype()), dtype=_abi.record_dtype())
    f = _abi.FieldC()
    f.pair_index, f.ref_id, f.tgt_id = field_.pair_index, field_.ref_id, field_.tgt_id
    f.records = C.cast(recs.ctypes.data, C.POINTER(_abi.PoiRecordC))
    f.capacity = f.count = len(recs)
    return f, recs


def field_csv_string(field_: DisplacementField) -> str:
    """pipeline.cpp:222-231 (dic::field_csv_string), formatted natively with the
    reference's printf formats."""
    f, keep = _field_c(field_)
    need = C.c_size_t(0)
    lib().dicb200_field_csv(C.byref(f), None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    st = lib().dicb200_field_csv(C.byref(f), buf, need.value, C.byref(need))
    if st:
        _raise(st)
    return buf.value.decode()


def write_field_csv(field_: DisplacementField, path) -> None:
    """pipeline.cpp:233-238 (dic::write_field_csv)."""
    f, keep = _field_c(field_)
    st = lib().dicb200_write_field_csv(C.byref(f), str(path).encode())
    if st:
        _raise(st)


def field_filename(pair_index: int) -> str:
    """pipeline.cpp:216-220: field_%04d.csv."""
    buf = C.create_string_buffer(32)
    st = lib().dicb200_field_filename(pair_index, buf, 32)
    if st:
        _raise(st)
    return buf.value.decode()


# ---- f-4 accuracy sweep (accuracy.hpp / synth.hpp) --------------------------------


@dataclass
class SpeckleParams:  # synth.hpp:14-23
    blob_count: int = 0
    sigma_min: float = 1.0
    sigma_max: float = 2.5
    amp_min: float = 40.0
    amp_max: float = 140.0
    background: float = 128.0
    variance_floor: float = 25.0
    texture_window: int = 31

    def to_c(self) -> _abi.SpeckleParamsC:
        c = _abi.SpeckleParamsC()
        for k in ("blob_count", "sigma_min", "sigma_max", "amp_min", "amp_max", "background", "variance_floor",
                  "texture_window"):
            setattr(c, k, getattr(self, k))
        return c


@dataclass
class WarpSpec:  # synth.hpp:30-35
    u: float = 0.0
    v: float = 0.0
    ux: float = 0.0
    uy: float = 0.0
    vx: float = 0.0
    vy: float = 0.0

    def to_c(self) -> _abi.WarpSpecC:
        return _abi.WarpSpecC(self.u, self.v, self.ux, self.uy, self.vx, self.vy)


@dataclass
class SweepConfig:  # accuracy.hpp:15-23
    width: int = 160
    height: int = 160
    seed: int = 7
    speckle: SpeckleParams = field(default_factory=SpeckleParams)
    base: RunConfig = field(default_factory=RunConfig)
    fractions: List[float] = field(default_factory=lambda: [0.1, 0.25, 0.5, 0.75, 0.9])
    offsets: List[int] = field(default_factory=lambda: [-3, 0, 4])
    gray_scale: int = 256  # B200: integer gray levels round(v * scale); 1 = 8-bit PGM round trip

    def to_c(self):
        """(struct, keep-alive arrays)."""
        fr = (C.c_double * max(1, len(self.fractions)))(*self.fractions)
        of = (C.c_int32 * max(1, len(self.offsets)))(*self.offsets)
        c = _abi.SweepConfigC()
        c.width, c.height, c.seed = self.width, self.height, self.seed & 0xFFFFFFFFFFFFFFFF
        c.speckle = self.speckle.to_c()
        c.base = self.base.to_c()
        c.fractions, c.n_fractions = C.cast(fr, C.POINTER(C.c_double)), len(self.fractions)
        c.offsets, c.n_offsets = C.cast(of, C.POINTER(C.c_int32)), len(self.offsets)
        c.gray_scale = self.gray_scale
        return c, (fr, of)


@dataclass
class ComboAccuracy:  # accuracy.hpp:25-34
    integer_method: IntegerMethod = IntegerMethod.bfs
    subpixel_method: SubpixelMethod = SubpixelMethod.none
    max_err: float = 0.0
    mean_err: float = 0.0
    measurements: int = 0
    unconverged: int = 0
    passed: bool = False  # `pass` in the reference
    mean_flagged: bool = False


@dataclass
class SweepReport:  # accuracy.hpp:36-41
    combos: List[ComboAccuracy] = field(default_factory=list)
    warp_count: int = 0
    poi_count: int = 0
    elapsed_s: float = 0.0


def default_blob_count(width: int, height: int) -> int:
    """synth.cpp:14-16."""
    return int(lib().dicb200_default_blob_count(width, height))


def synth_speckle(width: int, height: int, seed: int, params: SpeckleParams) -> np.ndarray:
    """synth.cpp:55-93 (dic::synth_speckle): float64 frame, bit-identical to the
    reference's doubles. Raises DicError("textureless pattern") etc."""
    out = np.zeros((max(height, 0), max(width, 0)), np.float64)
    st = lib().dicb200_synth_speckle(width, height, seed & 0xFFFFFFFFFFFFFFFF, C.byref(params.to_c()),
                                     out.ctypes.data)
    if st:
        _raise(st)
    return out


def synth_warped_pair(reference: np.ndarray, warp: WarpSpec) -> Tuple[np.ndarray, np.ndarray]:
    """synth.cpp:127-172 (dic::synth_warped_pair): (target float64, valid mask u8)."""
    ref = np.ascontiguousarray(reference, np.float64)
    h, w = ref.shape
    tgt = np.zeros_like(ref)
    mask = np.zeros(ref.shape, np.uint8)
    st = lib().dicb200_synth_warped_pair(ref.ctypes.data, w, h, C.byref(warp.to_c()), tgt.ctypes.data,
                                         mask.ctypes.data)
    if st:
        _raise(st)
    return tgt, mask


def run_accuracy_sweep(combos: Sequence[Tuple[IntegerMethod, SubpixelMethod]], cfg: SweepConfig) -> SweepReport:
    """accuracy.cpp:10-78 (dic::run_accuracy_sweep) with every pair analysed on
    the GPU (one pipelined fixed-first sequence per combo)."""
    arr = np.array([[int(a), int(b)] for a, b in combos] or [[0, 0]], np.int32)
    out = (_abi.ComboAccuracyC * max(1, len(combos)))()
    c, keep = cfg.to_c()
    wc, pc, el = C.c_int32(), C.c_int32(), C.c_double()
    st = lib().dicb200_accuracy_sweep(arr.ctypes.data, len(combos), C.byref(c), out, C.byref(wc), C.byref(pc),
                                      C.byref(el))
    if st:
        _raise(st)
    rep = SweepReport(warp_count=wc.value, poi_count=pc.value, elapsed_s=el.value)
    for i in range(len(combos)):
        o = out[i]
        rep.combos.append(ComboAccuracy(IntegerMethod(o.integer_method), SubpixelMethod(o.subpixel_method), o.max_err,
                                        o.mean_err, o.measurements, o.unconverged, bool(o.pass_),
                                        bool(o.mean_flagged)))
    return rep


# ---- f-4 bench matrix (bench.hpp / bench.cpp) --------------------------------------


@dataclass
class BenchCell:  # bench.hpp:12-16
    integer_method: IntegerMethod = IntegerMethod.pso
    subpixel_method: SubpixelMethod = SubpixelMethod.nr
    mode: ExecMode = ExecMode.serial


@dataclass
class BenchRecord:  # bench.hpp:18-31
    cell: BenchCell = field(default_factory=BenchCell)
    dataset_id: str = ""
    repeats: int = 0
    pair_count: int = 0
    mean_s: float = 0.0
    stddev_s: float = 0.0
    per_pair_s: float = 0.0
    frame_rate_hz: float = 0.0
    total_evaluations: int = 0
    failed: bool = False
    error: str = ""

    def to_c(self) -> _abi.BenchRecordC:
        c = _abi.BenchRecordC()
        c.cell = _abi.BenchCellC(int(self.cell.integer_method), int(self.cell.subpixel_method), int(self.cell.mode))
        for k in ("repeats", "pair_count", "mean_s", "stddev_s", "per_pair_s", "frame_rate_hz", "total_evaluations"):
            setattr(c, k, getattr(self, k))
        c.failed = 1 if self.failed else 0
        c.dataset_id = self.dataset_id.encode()[:127]
        c.error = self.error.encode()[:159]
        return c

    @staticmethod
    def from_c(c: _abi.BenchRecordC) -> "BenchRecord":
        return BenchRecord(BenchCell(IntegerMethod(c.cell.integer_method), SubpixelMethod(c.cell.subpixel_method),
                                     ExecMode(c.cell.mode)), c.dataset_id.decode(), c.repeats, c.pair_count, c.mean_s,
                           c.stddev_s, c.per_pair_s, c.frame_rate_hz, c.total_evaluations, bool(c.failed),
                           c.error.decode())


@dataclass
class BenchReport:  # bench.hpp:33-42
    records: List[BenchRecord] = field(default_factory=list)
    dataset_id: str = ""
    cpu_model: str = ""
    hardware_threads: int = 0
    worker_count: int = 0
    timestamp: str = ""


@dataclass
class RepeatsPolicy:  # bench.hpp:44-47
    auto_bands: bool = True
    fixed: int = 1


@dataclass
class RatioRow:  # bench.hpp:56-61
    kind: str = ""
    detail: str = ""
    value: float = 0.0
    note: str = ""


def auto_repeats(warmup_seconds: float) -> int:
    """bench.cpp:14-19."""
    return int(lib().dicb200_auto_repeats(warmup_seconds))


def cpu_model_name() -> str:
    """bench.cpp:293-306 (/proc/cpuinfo "model name")."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name") and ":" in line:
                    name = line.split(":", 1)[1].rstrip("\n")
                    return name[1:] if name.startswith(" ") else name
    except OSError:
        pass
    return "unknown"


def timestamp_utc() -> str:
    """bench.cpp:308-315."""
    import time

    return time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())


def run_bench(cells: Sequence[BenchCell], dataset_dir, pattern: str, base: RunConfig,
              repeats: RepeatsPolicy = RepeatsPolicy(), scratch_dir=None, allow_16bit: bool = False) -> BenchReport:
    """bench.cpp:60-120 (dic::run_bench): cells in order, each repeat = load the
    sequence (native PGM loader, pinned), analyze it on the GPU, write the field
    CSVs under scratch_dir/cell-<int>-<sub>-<mode>/; host wall clock per repeat."""
    import tempfile

    if scratch_dir is None:
        scratch_dir = tempfile.mkdtemp(prefix="dicb200_bench_")
    arr = (_abi.BenchCellC * max(1, len(cells)))(
        *[_abi.BenchCellC(int(c.integer_method), int(c.subpixel_method), int(c.mode)) for c in cells])
    out = (_abi.BenchRecordC * max(1, len(cells)))()
    st = lib().dicb200_run_bench(arr, len(cells), str(dataset_dir).encode(), pattern.encode(), C.byref(base.to_c()),
                                 1 if repeats.auto_bands else 0, repeats.fixed, str(scratch_dir).encode(),
                                 1 if allow_16bit else 0, out)
    if st:
        _raise(st)
    d = str(dataset_dir)
    rep = BenchReport(dataset_id=os.path.basename(d) or d, cpu_model=cpu_model_name(),
                      hardware_threads=os.cpu_count() or 0, worker_count=base.worker_count, timestamp=timestamp_utc())
    rep.records = [BenchRecord.from_c(out[i]) for i in range(len(cells))]
    return rep


def _records_c(report: BenchReport):
    return (_abi.BenchRecordC * max(1, len(report.records)))(*[r.to_c() for r in report.records])


def derive_ratios(report: BenchReport) -> List[RatioRow]:
    """bench.cpp:142-208 (dic::derive_ratios)."""
    recs = _records_c(report)
    rows = (_abi.RatioRowC * 32)()
    n = C.c_size_t(0)
    st = lib().dicb200_derive_ratios(recs, len(report.records), report.dataset_id.encode(), rows, 32, C.byref(n))
    if st:
        _raise(st)
    return [RatioRow(rows[i].kind.decode(), rows[i].detail.decode(), rows[i].value, rows[i].note.decode())
            for i in range(n.value)]


def write_times_csv(report: BenchReport, path) -> None:
    """bench.cpp:210-251: one row per (integer, subpixel), one mean-seconds column per mode."""
    st = lib().dicb200_write_times_csv(_records_c(report), len(report.records), report.dataset_id.encode(),
                                       str(path).encode())
    if st:
        _raise(st)


def write_records_csv(report: BenchReport, path) -> None:
    """bench.cpp:253-269."""
    st = lib().dicb200_write_records_csv(_records_c(report), len(report.records), str(path).encode())
    if st:
        _raise(st)


def write_ratios_csv(rows: Sequence[RatioRow], path) -> None:
    """bench.cpp:271-283."""
    arr = (_abi.RatioRowC * max(1, len(rows)))()
    for i, r in enumerate(rows):
        arr[i].kind, arr[i].detail = r.kind.encode()[:31], r.detail.encode()[:159]
        arr[i].value, arr[i].note = r.value, r.note.encode()[:31]
    st = lib().dicb200_write_ratios_csv(arr, len(rows), str(path).encode())
    if st:
        _raise(st)


def write_manifest(entries: Sequence[Tuple[str, str]], path) -> None:
    """bench.cpp:285-291: "key = value" lines."""
    try:
        with open(path, "w") as f:
            for k, v in entries:
                f.write(f"{k} = {v}\n")
    except OSError:
        raise DicError("cannot open for writing: " + str(path))
