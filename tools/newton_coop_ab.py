"""NEXT-1 large single point (n = 256, QD; cooperative elimination): Newton step time against
the cooperative grid size (PHC_NEWTON_COOP_CTAS), CUDA events after warm-up; bitwise check."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system  # noqa: E402

s, X = config_system("large", seed=1)
h = phc.System(s)
Xd = torch.from_numpy(X).cuda()
Xn = torch.empty_like(Xd)
ref = None
for g in ("148", "96", "74", "48", "32"):
    os.environ["PHC_NEWTON_COOP_CTAS"] = g
    for _ in range(2):
        h.newton_step(Xd, Xn)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        h.newton_step(Xd, Xn)
    b.record()
    b.synchronize()
    same = None if ref is None else bool(torch.equal(Xn, ref))
    ref = Xn.clone() if ref is None else ref
    print(json.dumps(dict(ctas=int(g), ms_step=a.elapsed_time(b) / 5, bitwise_equal_first=same)), flush=True)
