import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, paper_1109_0545_b200 as phc
from synthetic import config_system
for name in ("tiny", "c2"):
    s, X = config_system(name, seed=1)
    h = phc.System(s)
    x = torch.from_numpy(X[0]).cuda()
    f = torch.empty((s.n_eq, 2, s.limbs), dtype=torch.float64, device="cuda")
    j = torch.empty((s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device="cuda")
    for _ in range(100): h.eval(x, f, j)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n): h.eval(x, f, j)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(name, "host us/call", round((t1 - t0) / n * 1e6, 2), "total us/call", round((t2 - t0) / n * 1e6, 2))
# the C ABI alone: pre-built ctypes arguments, no Python-side checks
import ctypes  # noqa: E402
from paper_1109_0545_b200 import _lib  # noqa: E402
lib = _lib.lib
for name in ("tiny", "c2"):
    s, X = config_system(name, seed=1)
    h = phc.System(s)
    x = torch.from_numpy(X[0]).cuda()
    f = torch.empty((s.n_eq, 2, s.limbs), dtype=torch.float64, device="cuda")
    j = torch.empty((s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device="cuda")
    args = (h._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(j.data_ptr()),
            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    for _ in range(100): lib.phc_eval_jacobian(*args)
    torch.cuda.synchronize()
    n = 5000
    t0 = time.perf_counter()
    for _ in range(n): lib.phc_eval_jacobian(*args)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(name, "C ABI only: host us/call", round((t1 - t0) / n * 1e6, 2))
