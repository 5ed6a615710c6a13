"""ctypes mirror of include/dicb200.h and include/dicb200_synth.h.

Plain C structs only; shared by the product wrapper (dic.py), the oracle
wrapper (oracle/pyoracle.py) and bench.py.
"""
from __future__ import annotations

import ctypes as C

U8, U16, F32, F64 = 0, 1, 2, 3  # dicb200_image.dtype (F32/F64: fractional levels, exact fp64 path)

INT_BFS, INT_PSO, INT_MPSO = 0, 1, 2
SUB_NR, SUB_ICGN, SUB_NONE = 0, 1, 2
MODE_SERIAL, MODE_SUBIMAGE, MODE_IMAGE = 0, 1, 2
POLICY_UPDATE, POLICY_FIXED_FIRST = 0, 1
BFS_WINDOW, BFS_WHOLE_IMAGE = 0, 1
INERTIA_REFERENCE, INERTIA_CONSTANT = 0, 1

FIELD_NONE, FIELD_AFFINE, FIELD_SINUSOID = 0, 1, 2

POI_STATUS = {
    0: "ok",
    1: "subset out of image bounds",
    2: "no valid search position",
    3: "all positions degenerate",
    4: "invalid swarm configuration",
    5: "degenerate subset",
    6: "drifted out of bounds",
    7: "degenerate target subset",
    8: "subset too close to border for gradients",
    9: "degenerate texture",
    10: "warp not invertible",
    11: "non-invertible warp increment",
    12: "pixel values exceed the declared dicb200_image.bits",  # B200 extension
}


class Image(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("pitch", C.c_int32),
        ("dtype", C.c_int32),
        ("id", C.c_int32),
        ("bits", C.c_int32),
        ("data", C.c_void_p),
    ]


class RunConfigC(C.Structure):
    _fields_ = [
        ("integer_method", C.c_int32),
        ("subpixel_method", C.c_int32),
        ("mode", C.c_int32),
        ("reference_policy", C.c_int32),
        ("worker_count", C.c_int32),
        ("search_radius", C.c_int32),
        ("bfs_domain", C.c_int32),
        ("particle_count", C.c_int32),
        ("max_generations", C.c_int32),
        ("pad0", C.c_int32),
        ("stop_threshold", C.c_double),
        ("c1", C.c_double),
        ("c2", C.c_double),
        ("rng_seed", C.c_uint64),
        ("tol", C.c_double),
        ("max_iter", C.c_int32),
        ("half_width", C.c_int32),
        ("spacing", C.c_int32),
        ("margin", C.c_int32),
        ("inertia_mode", C.c_int32),
        ("interp", C.c_int32),
        ("inertia_constant", C.c_double),
    ]


INTERP_BILINEAR, INTERP_BICUBIC = 0, 1  # dicb200_run_config.interp


class PoiRecordC(C.Structure):
    _fields_ = [
        ("x", C.c_int32),
        ("y", C.c_int32),
        ("u", C.c_double),
        ("v", C.c_double),
        ("zncc", C.c_double),
        ("converged", C.c_int32),
        ("iterations", C.c_int32),
        ("evaluations", C.c_int64),
        ("update_evaluations", C.c_int64),
        ("status", C.c_int32),
        ("integer_dx", C.c_int32),
        ("integer_dy", C.c_int32),
        ("pad", C.c_int32),
    ]


class FieldC(C.Structure):
    _fields_ = [
        ("pair_index", C.c_int32),
        ("ref_id", C.c_int32),
        ("tgt_id", C.c_int32),
        ("status", C.c_int32),
        ("records", C.POINTER(PoiRecordC)),
        ("capacity", C.c_size_t),
        ("count", C.c_size_t),
        ("error", C.c_char * 160),
    ]


class SynthSpecC(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("dtype", C.c_int32),
        ("max_value", C.c_int32),
        ("seed", C.c_uint64),
        ("blob_count", C.c_int32),
        ("field", C.c_int32),
        ("sigma_min", C.c_double),
        ("sigma_max", C.c_double),
        ("peak_min", C.c_double),
        ("peak_max", C.c_double),
        ("background", C.c_double),
        ("a", C.c_double * 8),
    ]


# numpy structured dtype with the exact layout of dicb200_poi_record
def record_dtype():
    import numpy as np

    return np.dtype(
        {
            "names": [f for f, _ in PoiRecordC._fields_],
            "formats": [
                np.int32, np.int32, np.float64, np.float64, np.float64, np.int32, np.int32,
                np.int64, np.int64, np.int32, np.int32, np.int32, np.int32,
            ],
            "offsets": [getattr(PoiRecordC, f).offset for f, _ in PoiRecordC._fields_],
            "itemsize": C.sizeof(PoiRecordC),
        }
    )


class SpeckleParamsC(C.Structure):  # dicb200_speckle_params (synth.hpp:14-23)
    _fields_ = [
        ("blob_count", C.c_int32),
        ("texture_window", C.c_int32),
        ("sigma_min", C.c_double),
        ("sigma_max", C.c_double),
        ("amp_min", C.c_double),
        ("amp_max", C.c_double),
        ("background", C.c_double),
        ("variance_floor", C.c_double),
    ]


class WarpSpecC(C.Structure):  # dicb200_warp_spec (synth.hpp:30-35)
    _fields_ = [(k, C.c_double) for k in ("u", "v", "ux", "uy", "vx", "vy")]


class SweepConfigC(C.Structure):  # dicb200_sweep_config (accuracy.hpp:15-23)
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("seed", C.c_uint64),
        ("speckle", SpeckleParamsC),
        ("base", RunConfigC),
        ("fractions", C.POINTER(C.c_double)),
        ("n_fractions", C.c_int32),
        ("n_offsets", C.c_int32),
        ("offsets", C.POINTER(C.c_int32)),
        ("gray_scale", C.c_int32),
        ("pad", C.c_int32),
    ]


class ComboAccuracyC(C.Structure):  # dicb200_combo_accuracy (accuracy.hpp:25-34)
    _fields_ = [
        ("integer_method", C.c_int32),
        ("subpixel_method", C.c_int32),
        ("max_err", C.c_double),
        ("mean_err", C.c_double),
        ("measurements", C.c_int32),
        ("unconverged", C.c_int32),
        ("pass_", C.c_int32),
        ("mean_flagged", C.c_int32),
    ]


class BenchCellC(C.Structure):  # dicb200_bench_cell (bench.hpp:12-16)
    _fields_ = [("integer_method", C.c_int32), ("subpixel_method", C.c_int32), ("mode", C.c_int32)]


class BenchRecordC(C.Structure):  # dicb200_bench_record (bench.hpp:18-31)
    _fields_ = [
        ("cell", BenchCellC),
        ("repeats", C.c_int32),
        ("pair_count", C.c_int32),
        ("failed", C.c_int32),
        ("mean_s", C.c_double),
        ("stddev_s", C.c_double),
        ("per_pair_s", C.c_double),
        ("frame_rate_hz", C.c_double),
        ("total_evaluations", C.c_int64),
        ("dataset_id", C.c_char * 128),
        ("error", C.c_char * 160),
    ]


class RatioRowC(C.Structure):  # dicb200_ratio_row (bench.hpp:56-61)
    _fields_ = [("kind", C.c_char * 32), ("detail", C.c_char * 160), ("value", C.c_double), ("note", C.c_char * 32)]
