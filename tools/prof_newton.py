"""ncu driver: Newton steps on one point of a config (warm-up + reps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s, X = config_system(name, seed=1, points=P)
h = phc.System(s)
Xd = torch.from_numpy(X).cuda()
for _ in range(3):
    h.newton_step(Xd)
torch.cuda.synchronize()
print("ok")
