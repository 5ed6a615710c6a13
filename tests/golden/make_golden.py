"""Regenerate tests/golden/*.npz from the reference's OWN sources
(oracle/_ref/libdicref.so, built from /root/reference/proj/core/src by
oracle/Makefile). Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Each fixture stores the exact input frames (so the test never depends on
the generator), the run configuration and the reference's records.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

from cases import CASES  # noqa: E402
from oracle import Oracle  # noqa: E402


def cfg_json(cfg):
    c = cfg.to_c()
    return json.dumps({f: getattr(c, f) for f, _ in c._fields_})


def main():
    ref = Oracle("reference")
    for name, make in CASES.items():
        a, b, cfg = make()
        recs = ref.analyze_pair(a, b, cfg)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), ref=a, tgt=b, records=recs,
                            config=np.array(cfg_json(cfg)))
        print(f"{name}: {a.shape} {a.dtype} -> {len(recs)} records")


if __name__ == "__main__":
    main()
