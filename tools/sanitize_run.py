"""One small call of every kernel family, for compute-sanitizer:
block kernel (layouts 0/1/2, plain and homotopy), latency path (warp scan, split reduction),
generic path (k > 32), common-support path (both regimes), Newton (warp, CTA, cooperative,
multi-kernel), predictor, tracker (K = 2 lane placement, device-side control), arithmetic
self-test incl. the warp reciprocal, sharded calls (repeated devices)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import (common_support_system, config_system, homotopy_target, random_system, random_t,  # noqa: E402
                       system_from_terms, total_degree_homotopy)
from synthetic.systems import unit_circle_limbs  # noqa: E402

cuda = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
# block kernel layout 2 (DD) and the latency path (k = 16), plain + homotopy, sharded
s, X = config_system("batch", seed=1, points=700)
h = phc.System(s, coeff_target=homotopy_target(s, seed=2))
h.eval_batch(cuda(X), devices=[0, 0])
h.eval(cuda(X[0]))
h.eval_homotopy_batch(cuda(X), cuda(random_t(700, 2, seed=3)))
# layout 1 (c3 QD, latency path and block path)
s, X = config_system("c3", seed=1, points=8)
h = phc.System(s)
h.eval(cuda(X[0]))
h.eval_batch(cuda(X))
# layout 0 (QD, table in global memory): n = 160, k = 32
s, X = random_system(160, 32, 32, 6, 4, seed=2, points=2)
h = phc.System(s)
print("layout", h.stats["layout"])
h.eval_batch(cuda(X))
# generic path (k > 32)
rng = np.random.default_rng(1)
polys = [[[(v, 1) for v in range(34)]], [[(0, 2), (33, 1)], []]]
s = system_from_terms(2, 34, 2, polys, unit_circle_limbs(rng.uniform(0, 6, 3), 2, 1))
phc.System(s).eval_batch(cuda(unit_circle_limbs(rng.uniform(0, 6, (3, 34)), 2, 1)))
# common support, both regimes
c, X = common_support_system(10, 24, 1, 6, 3, 2, seed=3, points=600)
hc = phc.System(c)
hc.eval_batch(cuda(X[:1]))
hc.eval_batch(cuda(X))
# Newton: warp kernel (n = 8), CTA kernel (n = 40 QD), multi-kernel (n = 52 QD)
s, X = config_system("tiny", seed=1, points=4)
phc.System(s).newton_step(cuda(X))
s, X = config_system("c3", seed=1, points=2)
phc.System(s).newton_step(cuda(X))
s, X = random_system(52, 4, 3, 2, 4, seed=4, points=2)
phc.System(s).newton_step(cuda(X))            # cooperative (<= 4 points)
s, X = random_system(52, 4, 3, 2, 4, seed=4, points=6)
phc.System(s).newton_step(cuda(X))            # multi-kernel (> 4 points)
s, X = config_system("c2", seed=1, points=3)
phc.System(s).newton_solve(cuda(X), 1e-20, 6)  # Alg. 2 to tolerance
# tracker + predictor
s, cf, X0 = total_degree_homotopy(2, 2, seed=5)
phc.System(s, coeff_target=cf).track(cuda(X0), max_steps=40)
# arithmetic self-test
from paper_1109_0545_b200.system import _ptr  # noqa: E402
a = cuda(np.ones((64, 2, 4)))
o = torch.empty_like(a)
phc.phc_arith_test(5, 4, 64, _ptr(a), _ptr(a), _ptr(o), None)
phc.phc_arith_test(10, 4, 64, _ptr(a), _ptr(a), _ptr(o), None)
torch.cuda.synchronize()
print("sanitize run ok")
