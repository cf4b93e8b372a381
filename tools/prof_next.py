"""ncu driver for the NEXT-row kernels: common-support batch (monomial stage + coefficient
product), homotopy batch DD (block kernel HOM instantiation), one tracker run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import common_config, config_system, homotopy_target, random_t  # noqa: E402

what = sys.argv[1]
if what == "common":
    c, X = common_config("common_batch", seed=1, points=8192, workers=8)
    h = phc.System(c)
    Xd = torch.from_numpy(X).cuda()
    for _ in range(2):
        h.eval_batch(Xd)
elif what == "homotopy":
    s, X = config_system("batch", seed=1, points=8192, workers=8)
    h = phc.System(s, coeff_target=homotopy_target(s, seed=2, workers=8))
    Xd = torch.from_numpy(X).cuda()
    Td = torch.from_numpy(random_t(8192, 2, seed=3)).cuda()
    for _ in range(2):
        h.eval_homotopy_batch(Xd, Td)
torch.cuda.synchronize()
print("ok", what)
