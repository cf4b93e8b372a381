import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_1109_0545_b200 as phc
from synthetic import total_degree_homotopy
s, cf, X0 = total_degree_homotopy(8, 2, seed=1)
h = phc.System(s, coeff_target=cf)
X = torch.from_numpy(X0).cuda()
Xe, st, stats = h.track(X[:64], max_steps=20)
torch.cuda.synchronize()
print("done")
