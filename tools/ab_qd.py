"""A/B of library builds on the large QD config: single-point median latency (L2 flushed per
call), large x 4,096 throughput, and the normwise error of the single point against the
committed oracle values (tests/golden/large_seed1.npz, every F and J entry).
usage: python tools/ab_qd.py [lib ...]   (paths relative to paper_1109_0545_b200/; one
subprocess per library, PHC_LIB selects it)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import statistics

    import torch

    import paper_1109_0545_b200 as phc
    from _golden import load, to_mpc
    from oracle import MPArith, rel_errors
    from synthetic import config_system
    s, X = config_system("large_batch", seed=1, points=int(os.environ.get("AB_POINTS", "1024")))
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    x0 = Xd[0].contiguous()
    f = torch.empty((256, 2, 4), dtype=torch.float64, device="cuda")
    j = torch.empty((256, 256, 2, 4), dtype=torch.float64, device="cuda")
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(10):
        h.eval(x0, f, j)
    torch.cuda.synchronize()
    us = []
    for i in range(200):
        scrub.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.eval(x0, f, j)
        b.record()
        b.synchronize()
        us.append(a.elapsed_time(b) * 1e3)
    F, J = h.eval_batch(Xd)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        h.eval_batch(Xd, F, J)
    b.record()
    b.synchronize()
    eps = 3 * X.shape[0] / (a.elapsed_time(b) * 1e-3)
    sb, Xb = config_system("batch", seed=1)
    hb = phc.System(sb)
    Xbd = torch.from_numpy(Xb).cuda()
    Fb, Jb = hb.eval_batch(Xbd)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        hb.eval_batch(Xbd, Fb, Jb)
    b.record()
    b.synchronize()
    dd_eps = 10 * Xb.shape[0] / (a.elapsed_time(b) * 1e-3)
    del Fb, Jb, Xbd
    g = load()
    ar = MPArith(512)
    ef, _, _ = rel_errors(ar, to_mpc(g["F0"]), f.cpu().numpy())
    ej, _, _ = rel_errors(ar, to_mpc(g["J0"]), j.cpu().numpy().reshape(-1, 2, 4))
    print(json.dumps(dict(lib=os.environ.get("PHC_LIB", "libphc.so"), single_us_median=statistics.median(us),
                          single_us_min=min(us), batch_evals_per_s=eps, batch_dd_evals_per_s=dd_eps, err_F=ef, err_J=ej,
                          exec_flops_per_point=h.stats["exec_flops_per_point"])), flush=True)


if __name__ == "__main__":
    if os.environ.get("AB_CHILD"):
        child()
        sys.exit(0)
    libs = sys.argv[1:] or ["libphc.so"]
    for rep in range(2):
        for lib in libs:
            env = dict(os.environ, AB_CHILD="1", PHC_LIB=os.path.join(ROOT, "paper_1109_0545_b200", lib))
            r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True, timeout=900)
            print(r.stdout.strip() or r.stderr[-2000:], flush=True)
