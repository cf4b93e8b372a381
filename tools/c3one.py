import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_1109_0545_b200 as phc
from synthetic import config_system
s, X = config_system(sys.argv[1] if len(sys.argv) > 1 else "c3", seed=1)
h = phc.System(s)
x = torch.from_numpy(X[0]).cuda()
for _ in range(5):
    f, j = h.eval(x)
torch.cuda.synchronize()
