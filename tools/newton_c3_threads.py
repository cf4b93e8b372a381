"""NEXT-1 c3 single point (n = 40, QD): Newton step time against the CTA elimination's thread
count (PHC_NEWTON_THREADS; default 512 for few points), CUDA events after warm-up."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system  # noqa: E402

for name in ("c3", "c2"):
    s, X = config_system(name, seed=1)
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    Xn = torch.empty_like(Xd)
    ref = None
    for th in ("128", "256", "512", "768", "1024"):
        os.environ["PHC_NEWTON_THREADS"] = th
        os.environ["PHC_NEWTON_WARP"] = "0"
        try:
            for _ in range(3):
                h.newton_step(Xd, Xn)
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            print(json.dumps(dict(case=name, threads=int(th), error=str(e)[:80])), flush=True)
            continue
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            h.newton_step(Xd, Xn)
        b.record()
        b.synchronize()
        same = None if ref is None else bool(torch.equal(Xn, ref))
        ref = Xn.clone() if ref is None else ref
        print(json.dumps(dict(case=name, threads=int(th), ms_step=a.elapsed_time(b) / 50, bitwise_equal_first=same)),
              flush=True)
