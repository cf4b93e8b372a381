import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1109_0545_b200 as phc
from synthetic import config_system
from synthetic.systems import system_from_terms
s, X = config_system("large", seed=1, points=1, workers=8)
def sub(n_eq, m):
    polys, coef = [], []
    for i in range(n_eq):
        ts = list(s.terms(i))[:m]
        polys.append([tl for _, tl in ts]); coef += [s.coeff[t] for t, _ in ts]
    return system_from_terms(n_eq, s.n_var, 4, polys, np.array(coef))
x = torch.from_numpy(X[0]).cuda()
def timed(fn, reps=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for n_eq, m in [(148, 256), (148, 224), (148, 192), (148, 160), (148, 128), (148, 64), (148, 32), (296, 128), (256, 256), (108, 256)]:
    ss = sub(n_eq, m)
    h = phc.System(ss)
    f = torch.empty((n_eq, 2, 4), dtype=torch.float64, device="cuda")
    j = torch.empty((n_eq, 256, 2, 4), dtype=torch.float64, device="cuda")
    us = timed(lambda: h.eval(x, f, j))
    print(json.dumps(dict(n_eq=n_eq, m=m, blocks_per_poly=m // 32, us=round(us, 1), us_per_blockwave=round(us / 1, 1))), flush=True)
