"""ncu driver: one Newton step of the batch config on 8,192 points (the CTA elimination)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system  # noqa: E402

s, X = config_system("batch", seed=1, points=8192)
h = phc.System(s)
Xd = torch.from_numpy(X).cuda()
for _ in range(2):
    h.newton_step(Xd)
torch.cuda.synchronize()
print("ok")
