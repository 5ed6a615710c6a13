"""Iteration / status histogram of one configuration's records on the device."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1905_06228_b200 import configs, dic  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = configs.get(name)
a, b = w.frames[0].render(), w.frames[1].render()
r = dic.analyze_pair(dic.GrayImage(a), dic.GrayImage(b, 1), w.cfg).records
it = r["iterations"]
print(name, "POIs", len(r), "mean it %.2f" % it.mean())
print("iterations hist", np.bincount(it, minlength=max(it.max() + 1, 1)).tolist())
print("status", {int(s): int((r["status"] == s).sum()) for s in np.unique(r["status"])})
print("converged", int(r["converged"].sum()))
du = np.abs(r["u"] - r["integer_dx"]); dv = np.abs(r["v"] - r["integer_dy"])
print("|u - int| > 1:", int((du > 1).sum()), " > 2:", int((du > 2).sum()), "|v-int|>2:", int((dv > 2).sum()))
