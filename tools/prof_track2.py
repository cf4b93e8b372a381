import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np, paper_1109_0545_b200 as phc
from synthetic import total_degree_homotopy, real_limbs
s, cf, X0 = total_degree_homotopy(10, 2, seed=1)
h = phc.System(s, coeff_target=cf)
X = torch.from_numpy(X0).cuda()
T = torch.from_numpy(real_limbs([0.5] * X.shape[0], 2)).cuda()
def timed(fn, reps=50):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, (time.perf_counter() - t) / reps * 1e6
print("eval_homotopy 1024", timed(lambda: h.eval_homotopy_batch(X, T)))
print("newton_homotopy 1024", timed(lambda: h.newton_step_homotopy(X, T)))
print("eval plain 1024", timed(lambda: h.eval_batch(X)))
print(h.stats)
t = time.perf_counter(); Xe, st, stats = h.track(X); torch.cuda.synchronize(); print("track", time.perf_counter() - t, stats[:, 1].mean())
