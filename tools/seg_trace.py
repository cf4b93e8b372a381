"""Phase timeline of the segmented latency kernel (diagnostic build with PHC_SEG_TRACE=1):
per-CTA %globaltimer stamps (start, power table ready, products done, rows summed, partial
written / arrival, merge done), printed as percentiles relative to the earliest CTA start.

    python -c "import __graft_entry__ as g; g.build('libphc_trace.so', ('PHC_SEG_TRACE=1',))"
    PHC_LIB=paper_1109_0545_b200/libphc_trace.so python tools/seg_trace.py c3
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from paper_1109_0545_b200 import _lib  # noqa: E402
from synthetic import config_system  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
s, X = config_system(name, seed=1)
h = phc.System(s)
x = torch.from_numpy(X[0]).cuda()
for _ in range(20):
    f, j = h.eval(x)
torch.cuda.synchronize()
lib = _lib.lib
fn = lib.phc_debug_seg_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
n = 4096
buf = np.zeros((n, 8), dtype=np.uint64)
for rep in range(3):
    h.eval(x)
    torch.cuda.synchronize()
    assert fn(buf.ctypes.data, n) == 0
    used = buf[:, 0] > 0
    b = buf[used].astype(np.int64)
    t0 = b[:, 0].min()
    print(f"rep {rep}: {used.sum()} CTAs on {len(set(b[:, 7].tolist()))} SMs")
    names = ["start", "table ready", "products", "rows summed", "partial/arrive", "merge end"]
    for k, nm in enumerate(names):
        v = b[:, k]
        v = v[v > 0] - t0
        if len(v):
            print(f"  {nm:15s} min {v.min()/1e3:7.2f}  p50 {np.median(v)/1e3:7.2f}  max {v.max()/1e3:7.2f} us  (n={len(v)})")
    buf[:] = 0
