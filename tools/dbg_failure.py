import sys, copy; sys.path.insert(0,'.')
import numpy as np
from paper_1905_06228_b200 import configs, dic
from oracle import Oracle
port=Oracle('port')
w = configs.crop(configs.get("c4"), 160, 160)
a, b = w.frames[0].render(), w.frames[1].render()
b[:, :70] = 1000
for sub in (dic.SubpixelMethod.nr, dic.SubpixelMethod.icgn):
    cfg = copy.deepcopy(w.cfg); cfg.subpixel_method = sub
    exp = port.analyze_pair(a, b, cfg)
    got = dic.analyze_pair(dic.GrayImage(a), dic.GrayImage(b,1), cfg).records
    bad = np.nonzero((np.abs(got['u']-exp['u'])>1e-3) | (got['status']!=exp['status']) | (got['iterations']!=exp['iterations']))[0]
    print(sub.name, 'bad', len(bad))
    for i in bad[:6]:
        print(' exp', exp[i][['x','y','u','v','zncc','converged','iterations','status','integer_dx','integer_dy']])
        print(' got', got[i][['x','y','u','v','zncc','converged','iterations','status','integer_dx','integer_dy']])
