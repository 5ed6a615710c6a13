"""f-4 evidence: dic.run_accuracy_sweep (GPU) next to the reference's own
dic::run_accuracy_sweep (oracle/_ref, CPU, unquantized doubles) for every
(integer, subpixel) combo, at the reference's SweepConfig defaults and at a
window-BFS configuration. Writes one JSON document (stdout or --out)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle.pyoracle as po  # noqa: E402
from paper_1905_06228_b200 import dic  # noqa: E402

I, S = dic.IntegerMethod, dic.SubpixelMethod
COMBOS = [(i, s) for i in (I.bfs, I.pso, I.mpso) for s in (S.nr, S.icgn, S.none)]


def configs():
    a = dic.SweepConfig()  # accuracy.hpp:15-23 defaults (whole-image BFS, radius 25)
    b = dic.SweepConfig()
    b.base.search.bfs_domain = dic.BfsDomain.window
    b.base.search.search_radius = 8
    b.base.search.particle_count = 60
    b.base.search.max_generations = 12
    return {"reference_defaults": a, "window_r8": b}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--no-reference", action="store_true")
    args = ap.parse_args()
    doc = {"combos": [f"{i.name}/{s.name}" for i, s in COMBOS], "runs": {}}
    for name, cfg in configs().items():
        run = {}
        for scale in (256, 1):
            cfg.gray_scale = scale
            dic.run_accuracy_sweep(COMBOS[:1], cfg)  # warm-up (context, module load)
            t = time.perf_counter()
            rep = dic.run_accuracy_sweep(COMBOS, cfg)
            wall = time.perf_counter() - t
            run[f"gpu_u{'16' if scale > 1 else '8'}"] = {
                "elapsed_s": rep.elapsed_s, "wall_s": wall, "warps": rep.warp_count, "pois": rep.poi_count,
                "combos": [dict(max_err=c.max_err, mean_err=c.mean_err, unconverged=c.unconverged, passed=c.passed,
                                mean_flagged=c.mean_flagged) for c in rep.combos]}
        if not args.no_reference and po.available("reference"):
            t = time.perf_counter()
            out, wc, pc, el = po.ref_accuracy_sweep(COMBOS, cfg)
            run["reference_cpu_1core"] = {
                "elapsed_s": el, "wall_s": time.perf_counter() - t, "warps": wc, "pois": pc,
                "combos": [dict(max_err=o.max_err, mean_err=o.mean_err, unconverged=o.unconverged,
                                passed=bool(o.pass_), mean_flagged=bool(o.mean_flagged)) for o in out]}
        doc["runs"][name] = run
    text = json.dumps(doc, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
