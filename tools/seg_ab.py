"""A/B of the latency-path shapes on the QD single-point configs (DESIGN.md §4 "segmented
latency path"): for each PHC_SEG setting ("0" = the warp-scan kernel, "G" = the segmented
kernel with G lanes per term) a subprocess times `reps` warm back-to-back calls of phc_eval_jacobian and the median
of cold calls (L2 flushed before each), and reports the largest normwise difference of F and J
from the warp-scan kernel's result (both within the 1e-60 oracle tolerance of the parity tests).

    python tools/seg_ab.py c3 0 4 8 10 12 16
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(name, out):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import paper_1109_0545_b200 as phc
    from synthetic import config_system

    s, X = config_system(name, seed=1)
    h = phc.System(s)
    x = torch.from_numpy(X[0]).cuda()
    f = torch.empty((s.n_eq, 2, s.limbs), dtype=torch.float64, device="cuda")
    j = torch.empty((s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device="cuda")
    for _ in range(20):
        h.eval(x, f, j)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 400
    e0.record()
    for _ in range(reps):
        h.eval(x, f, j)
    e1.record()
    torch.cuda.synchronize()
    warm = e0.elapsed_time(e1) * 1e3 / reps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cold = []
    for _ in range(100):
        flush.fill_(1)
        e0.record()
        h.eval(x, f, j)
        e1.record()
        torch.cuda.synchronize()
        cold.append(e0.elapsed_time(e1) * 1e3)
    cold.sort()
    np.savez(out, F=f.cpu().numpy(), J=j.cpu().numpy())
    st = h.stats
    print(json.dumps(dict(config=name, seg=os.environ.get("PHC_SEG", ""), warm_us=warm, cold_us=cold[len(cold) // 2],
                          latency_exec_flops=st["latency_exec_flops_per_point"])), flush=True)


def value(a):
    """leading-limb magnitude per entry (normwise comparison)"""
    return np.sqrt(a[..., 0, 0] ** 2 + a[..., 1, 0] ** 2)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
        sys.exit(0)
    import numpy as np

    name, shapes = sys.argv[1], sys.argv[2:]
    tmp = tempfile.mkdtemp()
    base = None
    for sh in shapes:
        out = os.path.join(tmp, f"{sh}.npz")
        env = dict(os.environ, PHC_SEG=sh)
        r = subprocess.run([sys.executable, __file__, "--child", name, out], env=env, capture_output=True, text=True)
        if r.returncode:
            print(json.dumps(dict(config=name, seg=sh, error=r.stderr[-600:])), flush=True)
            continue
        rec = json.loads(r.stdout.strip().splitlines()[-1])
        g = np.load(out)
        if base is None:
            base = g
        else:
            for key in ("F", "J"):
                a, b = g[key], base[key]
                # limb-wise difference summed, relative to the largest entry (normwise)
                rec[f"diff_{key}"] = float(np.abs((a - b).sum(-1)).max() / value(b).max())
        print(json.dumps(rec), flush=True)
