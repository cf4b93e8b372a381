import sys, time
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_1109_0545_b200 as phc
from synthetic import config_system
for name, P in [("batch", 65536), ("c3", 1), ("large", 1)]:
    s, X = config_system(name, seed=1, points=P)
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    h.newton_step(Xd); torch.cuda.synchronize()
    t = time.time(); Xn, r, st = h.newton_step(Xd); torch.cuda.synchronize(); dt = time.time() - t
    t = time.time(); h.eval_batch(Xd); torch.cuda.synchronize(); de = time.time() - t
    print(name, P, "newton step", dt, "eval only", de, "status", int(st.sum()), flush=True)
