"""f-4 evidence: the reference's bench matrix (bench.cpp run_bench ->
derive_ratios -> times/records/ratios CSVs) regenerated on B200 and, for the
same dataset and cells, by the reference build on the host CPU.

Dataset: an 8-bit PGM sequence written with the reference's own generators
(synth_speckle + synth_warped_pair, quantized like save_pgm), 512x512, 9 frames.
Writes <out>/{gpu,reference}_{times,records,ratios}.csv + manifest.txt."""
import argparse
import ctypes as C
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle.pyoracle as po  # noqa: E402
from paper_1905_06228_b200 import _abi, dic  # noqa: E402

I, S, M = dic.IntegerMethod, dic.SubpixelMethod, dic.ExecMode


def make_dataset(root, w=512, h=512, n=9):
    d = os.path.join(root, f"speckle{w}x{h}")
    os.makedirs(d, exist_ok=True)
    ref = dic.synth_speckle(w, h, 17, dic.SpeckleParams(blob_count=dic.default_blob_count(w, h)))
    for i in range(n):
        f = ref if i == 0 else dic.synth_warped_pair(ref, dic.WarpSpec(0.63 * i, -0.41 * i, 0.001 * i, 0, 0,
                                                                           -0.001 * i))[0]
        dic.save_pgm(dic.GrayImage(np.round(f).astype(np.uint8)), os.path.join(d, f"img_{i:03d}.pgm"))
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/bench_matrix")
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--reference-cells", type=int, default=3, help="cells the CPU reference also runs (slow)")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    tmp = tempfile.mkdtemp(prefix="dicb200_bm_")
    d = make_dataset(tmp)
    base = dic.RunConfig()
    base.search.bfs_domain = dic.BfsDomain.window
    base.search.search_radius = 10
    base.grid = dic.GridParams(half_width=15, spacing=10)
    cells = [dic.BenchCell(i, s, M.serial) for i in (I.bfs, I.pso, I.mpso) for s in (S.nr, S.icgn, S.none)]
    cells += [dic.BenchCell(I.bfs, S.icgn, M.image_parallel), dic.BenchCell(I.pso, S.icgn, M.image_parallel)]
    rep = dic.run_bench(cells, d, "img_*.pgm", base, dic.RepeatsPolicy(False, args.repeats), os.path.join(tmp, "g"))
    dic.write_times_csv(rep, os.path.join(args.out, "gpu_times.csv"))
    dic.write_records_csv(rep, os.path.join(args.out, "gpu_records.csv"))
    dic.write_ratios_csv(dic.derive_ratios(rep), os.path.join(args.out, "gpu_ratios.csv"))
    man = [("dataset", rep.dataset_id), ("frames", "9 x 512x512 u8 (synth_speckle + synth_warped_pair)"),
           ("cells", str(len(cells))), ("repeats", str(args.repeats)), ("cpu_model", rep.cpu_model),
           ("timestamp", rep.timestamp), ("timing", "bench.cpp boundary: load + analyze + write CSVs, host wall clock")]
    if po.available("reference") and args.reference_cells > 0:
        # the reference's own run_bench on the same dataset, first cells only (1 repeat)
        L = C.CDLL(po.PATHS["reference"])
        sub = [c for c in cells if c.integer_method != I.bfs][: args.reference_cells]
        sub = [dic.BenchCell(I.bfs, S.nr, M.serial)] + sub
        arr = (_abi.BenchCellC * len(sub))(*[_abi.BenchCellC(int(c.integer_method), int(c.subpixel_method),
                                                             int(c.mode)) for c in sub])
        out = (_abi.BenchRecordC * len(sub))()
        err = C.create_string_buffer(160)
        L.dicref_run_bench.argtypes = [C.POINTER(_abi.BenchCellC), C.c_size_t, C.c_char_p, C.c_char_p,
                                       C.POINTER(_abi.RunConfigC), C.c_int, C.c_int, C.c_char_p,
                                       C.POINTER(_abi.BenchRecordC), C.c_char_p, C.c_size_t]
        st = L.dicref_run_bench(arr, len(sub), d.encode(), b"img_*.pgm", C.byref(base.to_c()), 0, 1,
                                os.path.join(tmp, "r").encode(), out, err, 160)
        if st == 0:
            rr = dic.BenchReport(records=[dic.BenchRecord.from_c(out[i]) for i in range(len(sub))],
                                 dataset_id=rep.dataset_id)
            dic.write_times_csv(rr, os.path.join(args.out, "reference_times.csv"))
            dic.write_records_csv(rr, os.path.join(args.out, "reference_records.csv"))
            man.append(("reference", "oracle/_ref run_bench, 1 repeat, 1 host core"))
        else:
            man.append(("reference", "failed: " + err.value.decode()))
    dic.write_manifest(man, os.path.join(args.out, "manifest.txt"))
    for r in rep.records:
        print(f"{r.cell.integer_method.name:5s} {r.cell.subpixel_method.name:5s} {r.cell.mode.name:18s} "
              f"mean {r.mean_s * 1e3:8.2f} ms  {r.frame_rate_hz:9.1f} pairs/s  evals {r.total_evaluations} "
              f"{'FAILED ' + r.error if r.failed else ''}")


if __name__ == "__main__":
    main()
