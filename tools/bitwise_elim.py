import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1109_0545_b200 as phc
from synthetic import config_system
for name, P in (("c3", 3), ("c2", 2)):
    s, X = config_system(name, seed=9, points=P)
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    os.environ["PHC_NEWTON_WARP"] = "0"
    os.environ.pop("PHC_NEWTON_GLOBAL", None)
    ref = [t.cpu().numpy() for t in h.newton_step(Xd)]
    os.environ["PHC_NEWTON_GLOBAL"] = "1"
    for coop in ("0", "1"):
        os.environ["PHC_NEWTON_COOP"] = coop
        out = [t.cpu().numpy() for t in h.newton_step(Xd)]
        for nm, a, b in zip(("x", "res", "st"), ref, out):
            if not np.array_equal(a, b):
                d = np.abs(a - b).max() if a.dtype != np.int32 else None
                print(name, "coop", coop, nm, "DIFF max", d, "count", int((a != b).sum()), "of", a.size, b.ravel()[:4] if nm=="st" else "")
            else:
                print(name, "coop", coop, nm, "equal")
