import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, paper_1109_0545_b200 as phc
from synthetic import config_system, total_degree_homotopy
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
out = {"lib": os.environ.get("PHC_LIB", "default")}
for name, P in (("c3", 1024), ("c3", 4096), ("c2", 8192)):
    s, X = config_system(name, seed=1, points=P, workers=8)
    h = phc.System(s); Xd = torch.from_numpy(X).cuda()
    out[f"{name}x{P}_us_per_eval"] = round(timed(lambda: h.eval_batch(Xd)) / P, 3)
s, cf, X0 = total_degree_homotopy(10, 2, seed=1)
h = phc.System(s); X = torch.from_numpy(X0).cuda()
out["td10x1024_us"] = round(timed(lambda: h.eval_batch(X)), 1)
print(json.dumps(out))
