"""f-3 field CSV and f-4 bench matrix (pipeline.cpp:216-238, bench.cpp:14-293)
against the reference build (oracle/_ref): byte-identical CSV layouts and ratio
rows for the same records, the same repeat bands, the same cell-failure
semantics; on the GPU, run_bench over a PGM dataset on disk reports the
reference's pair and evaluation counts and writes field CSVs that match the
reference's own (integer columns exact, u/v/zncc within tolerance)."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle.pyoracle as po
from paper_1905_06228_b200 import _abi, dic
from paper_1905_06228_b200.dic import BenchCell, BenchRecord, ExecMode as M, IntegerMethod as I, SubpixelMethod as S

needs_ref = pytest.mark.skipif(not po.available("reference"), reason="reference build absent")


def _ref():
    L = C.CDLL(po.PATHS["reference"])
    L.dicref_auto_repeats.argtypes = [C.c_double]
    L.dicref_field_csv.argtypes = [C.c_void_p, C.c_size_t, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
    L.dicref_bench_csvs.argtypes = [C.POINTER(_abi.BenchRecordC), C.c_size_t, C.c_char_p, C.c_char_p, C.c_char_p,
                                    C.c_char_p, C.c_char_p, C.c_size_t]
    L.dicref_run_bench.argtypes = [C.POINTER(_abi.BenchCellC), C.c_size_t, C.c_char_p, C.c_char_p,
                                   C.POINTER(_abi.RunConfigC), C.c_int, C.c_int, C.c_char_p,
                                   C.POINTER(_abi.BenchRecordC), C.c_char_p, C.c_size_t]
    return L


@needs_ref
def test_auto_repeats_bands():
    L = _ref()
    for s in (0.0, 0.5, 0.999, 1.0, 9.99, 10.0, 59.9, 60.0, 60.01, 500.0):
        assert dic.auto_repeats(s) == L.dicref_auto_repeats(s), s


@needs_ref
def test_field_csv_byte_identical():
    rng = np.random.default_rng(5)
    recs = np.zeros(40, _abi.record_dtype())
    recs["x"], recs["y"] = rng.integers(-5, 3000, 40), rng.integers(0, 3000, 40)
    recs["u"], recs["v"] = rng.normal(0, 30, 40), rng.normal(0, 1e-7, 40)
    recs["zncc"] = rng.uniform(-1, 1, 40)
    recs["zncc"][::7] = np.nan
    recs["u"][3], recs["v"][4] = 0.0, -0.0
    recs["converged"] = rng.integers(0, 2, 40)
    recs["iterations"] = rng.integers(0, 21, 40)
    recs["evaluations"] = rng.integers(0, 2 ** 40, 40)
    need = C.c_size_t(0)
    L = _ref()
    L.dicref_field_csv(recs.ctypes.data, len(recs), None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    L.dicref_field_csv(recs.ctypes.data, len(recs), buf, need.value, C.byref(need))
    assert dic.field_csv_string(dic.DisplacementField(0, 0, 1, recs, "")) == buf.value.decode()
    assert dic.field_filename(7) == "field_0007.csv" and dic.field_filename(12345) == "field_12345.csv"


def _records():
    """A report exercising every branch: failed and missing cells, all modes,
    the last-record-wins rule of the times table, NaN ratios."""
    R = []
    t = 1.0
    for im in (I.bfs, I.pso, I.mpso):
        for sm in (S.nr, S.icgn, S.none):
            for mode in (M.serial, M.subimage_parallel, M.image_parallel):
                if (im, sm, mode) in ((I.pso, S.icgn, M.image_parallel), (I.mpso, S.none, M.subimage_parallel)):
                    continue  # missing cells
                t *= 1.37
                r = BenchRecord(BenchCell(im, sm, mode), "seq-A", 250, 64, t % 7.3, t % 0.11, (t % 7.3) / 64,
                                64 / (t % 7.3), int(t * 1e6), False, "")
                if (im, sm, mode) == (I.bfs, S.none, M.image_parallel):
                    r.failed, r.error, r.mean_s = True, "dimension mismatch", 0.0
                R.append(r)
    R.append(BenchRecord(BenchCell(I.bfs, S.nr, M.serial), "seq-A", 25, 64, 0.123456789, 0.0, 0.002, 518.4, 99, False,
                         ""))
    return dic.BenchReport(records=R, dataset_id="seq-A")


@needs_ref
@pytest.mark.parametrize("subset", ["all", "bfs_only", "no_serial"])
def test_bench_csvs_and_ratios_byte_identical(tmp_path, subset):
    rep = _records()
    if subset == "bfs_only":
        rep.records = [r for r in rep.records if r.cell.integer_method == I.bfs]
    elif subset == "no_serial":
        rep.records = [r for r in rep.records if r.cell.mode != M.serial]
    dic.write_times_csv(rep, tmp_path / "t.csv")
    dic.write_records_csv(rep, tmp_path / "r.csv")
    dic.write_ratios_csv(dic.derive_ratios(rep), tmp_path / "q.csv")
    recs = (_abi.BenchRecordC * len(rep.records))(*[r.to_c() for r in rep.records])
    err = C.create_string_buffer(160)
    assert _ref().dicref_bench_csvs(recs, len(rep.records), b"seq-A", str(tmp_path / "t2.csv").encode(),
                                    str(tmp_path / "r2.csv").encode(), str(tmp_path / "q2.csv").encode(), err, 160) == 0
    for a in ("t", "r", "q"):
        assert (tmp_path / f"{a}.csv").read_bytes() == (tmp_path / f"{a}2.csv").read_bytes(), a
    rows = dic.derive_ratios(rep)
    if subset == "all":
        kinds = {r.kind for r in rows}
        assert kinds == {"bfs_vs_pso", "image_speedup_vs_serial", "subimage_speedup_vs_serial"}
        assert any(math.isnan(r.value) and r.note == "missing cell" for r in rows)


def test_run_bench_argument_errors_and_cpu_only_cells(tmp_path):
    with pytest.raises(dic.DicError, match="empty benchmark matrix"):
        dic.run_bench([], tmp_path, "*.pgm", dic.RunConfig(), scratch_dir=tmp_path)
    with pytest.raises(dic.DicError, match="repeats must be >= 1"):
        dic.run_bench([BenchCell()], tmp_path, "*.pgm", dic.RunConfig(), dic.RepeatsPolicy(False, 0), tmp_path)
    # a missing dataset fails the cell, not the call (bench.cpp:113-116)
    rep = dic.run_bench([BenchCell()], tmp_path / "nope", "*.pgm", dic.RunConfig(), dic.RepeatsPolicy(False, 1),
                        tmp_path / "scratch")
    assert rep.records[0].failed and "not a directory" in rep.records[0].error
    assert rep.dataset_id == "nope"


def _dataset(tmp_path, n=5):
    """A 5-frame 8-bit sequence on disk: reference speckle + growing sub-pixel warps."""
    d = tmp_path / "speckle-seq"
    d.mkdir()
    ref = dic.synth_speckle(128, 112, 3, dic.SpeckleParams(blob_count=dic.default_blob_count(128, 112)))
    for i in range(n):
        f = ref if i == 0 else dic.synth_warped_pair(ref, dic.WarpSpec(0.7 * i, -0.45 * i, 0.002 * i))[0]
        dic.save_pgm(dic.GrayImage(np.round(f).astype(np.uint8)), d / f"frame_{i:03d}.pgm")
    base = dic.RunConfig()
    base.grid = dic.GridParams(half_width=10, spacing=8)
    return d, base


@pytest.mark.gpu
@needs_ref
def test_run_bench_matches_reference_counts_and_fields(gpu, tmp_path):
    d, base = _dataset(tmp_path)
    base.search.search_radius = 6
    base.search.bfs_domain = dic.BfsDomain.window
    cells = [BenchCell(I.bfs, S.nr, M.serial), BenchCell(I.pso, S.icgn, M.serial),
             BenchCell(I.mpso, S.none, M.image_parallel)]
    rep = dic.run_bench(cells, d, "frame_*.pgm", base, dic.RepeatsPolicy(False, 2), tmp_path / "ours")
    arr = (_abi.BenchCellC * 3)(*[_abi.BenchCellC(int(c.integer_method), int(c.subpixel_method), int(c.mode))
                                  for c in cells])
    out = (_abi.BenchRecordC * 3)()
    err = C.create_string_buffer(160)
    assert _ref().dicref_run_bench(arr, 3, str(d).encode(), b"frame_*.pgm", C.byref(base.to_c()), 0, 1,
                                   str(tmp_path / "ref").encode(), out, err, 160) == 0
    for got, e, cell in zip(rep.records, out, cells):
        assert not got.failed and not e.failed, (got.error, e.error)
        assert (got.pair_count, got.total_evaluations, got.repeats) == (e.pair_count, e.total_evaluations, 2)
        assert got.mean_s > 0 and got.frame_rate_hz == pytest.approx(got.pair_count / got.mean_s)
        name = f"cell-{cell.integer_method.name}-{cell.subpixel_method.name}-" + \
            {M.serial: "serial", M.subimage_parallel: "subimage", M.image_parallel: "image"}[cell.mode]
        files = sorted(os.listdir(tmp_path / "ours" / name))
        assert files == sorted(os.listdir(tmp_path / "ref" / name)) and len(files) == got.pair_count
        for fn in files:
            a = np.genfromtxt(tmp_path / "ours" / name / fn, delimiter=",", names=True)
            b = np.genfromtxt(tmp_path / "ref" / name / fn, delimiter=",", names=True)
            for k in ("x", "y", "converged", "evaluations"):
                assert np.array_equal(a[k], b[k]), (fn, k)
            ok = np.isfinite(b["zncc"])
            assert np.abs(a["u"] - b["u"])[ok].max(initial=0) <= 1e-3 and np.abs(a["v"] - b["v"])[ok].max(initial=0) <= 1e-3
