import os, sys, subprocess, json
sys.path.insert(0, os.getcwd())
import numpy as np
which = sys.argv[1]
if which == "run":
    import torch, paper_1109_0545_b200 as phc
    from synthetic import config_system, common_config
    out = {}
    for name, P in (("c3", 1), ("c3", 64), ("large", 2)):
        s, X = config_system(name, seed=1, points=P)
        h = phc.System(s)
        F, J = h.eval_batch(torch.from_numpy(X).cuda())
        Xn, r, st = h.newton_step(torch.from_numpy(X).cuda())
        torch.cuda.synchronize()
        np.save(f"/tmp/{os.environ['TAG']}_{name}_{P}_F.npy", F.cpu().numpy()); np.save(f"/tmp/{os.environ['TAG']}_{name}_{P}_J.npy", J.cpu().numpy())
        np.save(f"/tmp/{os.environ['TAG']}_{name}_{P}_X.npy", Xn.cpu().numpy())
    print("saved", os.environ["TAG"])
else:
    for name, P in (("c3", 1), ("c3", 64), ("large", 2)):
        for q in "FJX":
            a = np.load(f"/tmp/old_{name}_{P}_{q}.npy"); b = np.load(f"/tmp/new_{name}_{P}_{q}.npy")
            print(name, P, q, "bitwise equal" if np.array_equal(a, b) else "DIFFERENT")
