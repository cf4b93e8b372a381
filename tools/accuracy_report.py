"""Print normwise relative errors (reading C9) of the GPU path vs the oracle for every config
(sampled rows/points for the big ones).  Evidence for DESIGN.md's error budget."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from _parity import compare_point, oracle_point  # noqa: E402
from synthetic import config_system  # noqa: E402

out = []
cases = [("tiny", None, None, "exact"), ("c2", None, None, "exact"), ("c3", None, None, "exact"),
         ("batch", [0, 65535], None, "exact"), ("large", [0], [0, 128, 255], "mp")]
for name, pts, rows, arith in cases:
    for seed in (1, 2):
        s, X = config_system(name, seed=seed)
        h = phc.System(s)
        Xd = torch.from_numpy(X).cuda()
        F, J = h.eval_batch(Xd)
        torch.cuda.synchronize()
        F, J = F.cpu().numpy(), J.cpu().numpy()
        for p in (pts or [0]):
            ar, Fr, Jr = oracle_point(s, X[p], rows=rows, arith=arith)
            ef, ej = compare_point(ar, Fr, Jr, F[p], J[p], s.limbs, rows)
            rec = dict(config=name, seed=seed, point=p, rows=rows or "all", err_F=ef, err_J=ej,
                       tol=1e-28 if s.limbs == 2 else 1e-60)
            out.append(rec)
            print(json.dumps(rec), flush=True)
