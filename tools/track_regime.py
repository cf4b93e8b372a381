import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch, paper_1109_0545_b200 as phc
from synthetic import total_degree_homotopy
for n in (8, 10):
    s, cf, X0 = total_degree_homotopy(n, 2, seed=1)
    h = phc.System(s, coeff_target=cf)
    X = torch.from_numpy(X0).cuda()
    h.track(X[:4]); torch.cuda.synchronize()
    for rep in range(2):
        t = time.perf_counter(); Xe, st, stats = h.track(X); torch.cuda.synchronize()
        print(json.dumps(dict(n=n, rep=rep, env=os.environ.get("PHC_DEBUG_NO_LATENCY_PATH", ""), s=round(time.perf_counter() - t, 3), steps=float(stats[:, 1].mean()))), flush=True)
