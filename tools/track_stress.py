"""Tracker stress: total-degree homotopies (n = 2..6, DD and QD, several seeds); every run with
window graphs must equal plain launches and window 1 bitwise; all paths should arrive."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import total_degree_homotopy  # noqa: E402

bad = 0
for n in (2, 3, 4, 5, 6):
    for L in (2, 4):
        if L == 4 and n > 4:
            continue
        for seed in range(3):
            s, cf, X0 = total_degree_homotopy(n, L, seed=100 + seed)
            h = phc.System(s, coeff_target=cf)
            outs = []
            for env in ({"PHC_TRACK_GRAPH": "1", "PHC_TRACK_WINDOW": "8"}, {"PHC_TRACK_GRAPH": "0", "PHC_TRACK_WINDOW": "8"},
                        {"PHC_TRACK_GRAPH": "0", "PHC_TRACK_WINDOW": "1"}):
                os.environ.update(env)
                Xe, st, stats = h.track(torch.from_numpy(X0).cuda())
                torch.cuda.synchronize()
                outs.append((Xe.cpu().numpy(), st, stats))
            same = all(np.array_equal(a, b) for o in outs[1:] for a, b in zip(outs[0], o))
            arrived = int((outs[0][1] == 1).sum())
            if not same:
                bad += 1
            print(n, L, seed, "bitwise" if same else "DIFFERENT", f"{arrived}/{X0.shape[0]} arrived", flush=True)
print("mismatches", bad)
