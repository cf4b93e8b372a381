"""NEXT-1 timing: one Newton step (evaluation + elimination + back substitution + update)
against the evaluation alone, CUDA events on the launching stream after warm-up."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import common_config, config_system  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = [("batch", 65536), ("c2", 1), ("c3", 1), ("large", 1), ("common", 1)]
for name, P in cases:
    s, X = common_config(name, seed=1, points=P) if name == "common" else config_system(name, seed=1, points=P)
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    Xn = torch.empty_like(Xd)
    reps = 3 if P > 1 or name == "large" else 50
    t_step = timed(lambda: h.newton_step(Xd, Xn), reps)
    t_eval = timed(lambda: h.eval_batch(Xd), reps)
    print(json.dumps(dict(config=name, points=P, ms_newton_step=round(t_step, 4), ms_eval=round(t_eval, 4),
                          ms_solve=round(t_step - t_eval, 4))), flush=True)
