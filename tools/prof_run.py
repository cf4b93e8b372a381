"""Small driver for ncu captures: evaluate `points` points of a config twice (warm-up + one)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "batch"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
s, X = config_system(name, seed=1, points=P, workers=8)
h = phc.System(s, device=0)
Xd = torch.from_numpy(X).cuda()
for _ in range(reps):
    F, J = h.eval_batch(Xd)
torch.cuda.synchronize()
print("ok", name, P, h.stats, float(F.abs().sum()))
