"""compute-sanitizer sweep over the hot-path kernels (SURVEY.md §5 race-detection
row): every integer-search kernel (K1 tiles, K1-TC tensor cores, K1-BS block
sums, the swarm walk), both refiners (generic and fixed-geometry IC-GN, NR,
bilinear and bicubic) and the pipelined sequence path, on crops small enough
for the instrumented run.

    python tools/sanitize.py OUTDIR [memcheck racecheck synccheck initcheck]

Each case runs in its own process (`python tools/sanitize.py --case NAME`)
under `compute-sanitizer --tool T`; the summary (case, tool, errors, seconds)
goes to OUTDIR/sanitize.json and the raw logs next to it.
"""
from __future__ import annotations

import json
import os
import re
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# name: (config, crop w, crop h, env, sequence pairs (0 = analyze_pair))
CASES = {
    "c1_k1_u8": ("c1", 160, 160, {}, 0),
    "c2_tc_nr": ("c2", 160, 160, {"DICB200_BFS_TC": "1"}, 0),
    "c2_bs_u8_nr": ("c2", 160, 160, {"DICB200_BFS_BS": "1"}, 0),
    "c2b_bicubic_nr": ("c2b", 128, 128, {}, 0),
    "c3_mpso_tc_surface": ("c3", 160, 160, {}, 0),
    "c3_mpso_bs_surface": ("c3", 160, 160, {"DICB200_BFS_BS": "1"}, 0),
    "c3x_pso_legacy": ("c3x", 144, 144, {"DICB200_BFS_LEGACY": "1"}, 0),
    "c4_bs_icgn": ("c4", 128, 128, {}, 0),
    "c4_tc_icgn_generic": ("c4", 128, 128, {"DICB200_BFS_TC": "1", "DICB200_REFINE_GENERIC": "1"}, 0),
    "c5_bs_icgn_fixed_tma": ("c5", 160, 160, {}, 0),
    "c5_bs_icgn_no_tma": ("c5", 160, 160, {"DICB200_NO_TMA": "1"}, 0),
    "c5_bs_fused_argmax": ("c5", 160, 160, {"DICB200_BS_FUSE": "1"}, 0),
    "c5_legacy_u16": ("c5", 128, 128, {"DICB200_BFS_LEGACY": "1"}, 0),
    "c5_sequence_3pairs": ("c5", 160, 160, {}, 3),
}


def run_case(name: str) -> None:
    from paper_1905_06228_b200 import configs, dic

    cfgname, w, h, _env, npairs = CASES[name]
    base = configs.c5(max(npairs, 1)) if cfgname == "c5" else configs.get(cfgname)
    wl = configs.crop(base, w, h)
    if npairs:
        frames = [dic.GrayImage(f.render(), i) for i, f in enumerate(wl.frames[: npairs + 1])]
        fields = dic.analyze_sequence(frames, wl.cfg)
        n = sum(len(f.records) for f in fields)
    else:
        a, b = (f.render() for f in wl.frames[:2])
        n = len(dic.analyze_pair(dic.GrayImage(a), dic.GrayImage(b, 1), wl.cfg).records)
    print(f"case {name}: {n} records")


def main() -> None:
    if len(sys.argv) > 2 and sys.argv[1] == "--case":
        run_case(sys.argv[2])
        return
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sanitize"
    tools = sys.argv[2:] or ["memcheck", "racecheck", "synccheck", "initcheck"]
    os.makedirs(out, exist_ok=True)
    only = os.environ.get("SANITIZE_CASES")
    names = only.split(",") if only else list(CASES)
    summary = []
    for tool in tools:
        for name in names:
            env = dict(os.environ, **CASES[name][3])
            log = os.path.join(out, f"{tool}_{name}.log")
            cmd = ["compute-sanitizer", "--tool", tool, "--print-limit", "20", "--error-exitcode", "9"]
            if tool == "memcheck":
                cmd += ["--leak-check", "no"]
            if tool == "racecheck":
                cmd += ["--racecheck-report", "all"]
            cmd += [sys.executable, os.path.abspath(__file__), "--case", name]
            t0 = time.time()
            try:
                p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=int(os.environ.get("SANITIZE_TIMEOUT", "600")))
                text, rc = p.stdout + p.stderr, p.returncode
            except subprocess.TimeoutExpired as e:
                out_ = e.stdout or ""
                text, rc = (out_.decode() if isinstance(out_, bytes) else out_) + "\nTIMEOUT", -1
            with open(log, "w") as f:
                f.write(text)
            m = re.search(r"ERROR SUMMARY: (\d+) error", text)
            hz = re.search(r"RACECHECK SUMMARY: (\d+) hazard", text)
            row = {"tool": tool, "case": name, "rc": rc, "errors": int(m.group(1)) if m else None,
                   "hazards": int(hz.group(1)) if hz else None, "ran": f"case {name}:" in text,
                   "seconds": round(time.time() - t0, 1)}
            summary.append(row)
            print(json.dumps(row), flush=True)
    with open(os.path.join(out, "sanitize.json"), "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
