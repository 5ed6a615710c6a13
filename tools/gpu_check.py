"""Quick device-vs-oracle comparison over the config shapes (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1905_06228_b200 import configs, dic
from oracle import Oracle

port = Oracle('port')
cases = sys.argv[1:] or ['c1', 'c2:160', 'c3:128', 'c4:160', 'c2', 'c4:512', 'c3:256']
for case in cases:
    name, _, crop = case.partition(':')
    w = configs.get(name)
    if crop:
        w = configs.crop(w, int(crop), int(crop))
    imgs = [f.render() for f in w.frames[:2]]
    t = time.time(); a = port.analyze_pair(imgs[0], imgs[1], w.cfg); tp = time.time() - t
    t = time.time(); d = dic.analyze_pair(dic.GrayImage(imgs[0]), dic.GrayImage(imgs[1], 1), w.cfg).records; td = time.time() - t
    ex = {f: int(np.sum(a[f] != d[f])) for f in ['x', 'y', 'integer_dx', 'integer_dy', 'evaluations', 'update_evaluations', 'status', 'converged', 'iterations']}
    du = np.nanmax(np.abs(a['u'] - d['u'])) if len(a) else 0
    dv = np.nanmax(np.abs(a['v'] - d['v'])) if len(a) else 0
    dz = np.nanmax(np.abs(a['zncc'] - d['zncc'])) if len(a) else 0
    print(f"{case:8s} n={len(a):6d} port {tp:6.2f}s dev {td:6.3f}s mismatches={ex} max|du|={du:.3g} |dv|={dv:.3g} |dz|={dz:.3g}", flush=True)
    bad = np.nonzero((a['integer_dx'] != d['integer_dx']) | (a['evaluations'] != d['evaluations']) | (a['status'] != d['status']))[0]
    for i in bad[:5]:
        print('   oracle', a[i]); print('   device', d[i])
