"""ORACLE — test infrastructure, not product code.

A plain, slow, obviously-correct CPU evaluator of a sparse polynomial system and
its Jacobian, written from the definition the paper's method reaches exactly
(Verschelde & Yoffe 2011, §6 P:520-547 and Alg. 2 "Y").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_1109_0545_b200``) and imports nothing from it.
"""
from .naive import (  # noqa: F401
    ExactArith,
    MPArith,
    evaluate_rows,
    evaluate_system,
    monomial,
    derivative_monomial,
)
from .compare import rel_errors, exact_equal_limbs  # noqa: F401
from .newton import newton_step, solve_exact, solve_step_mp  # noqa: F401
from .homotopy import evaluate_homotopy_rows, evaluate_homotopy_dt  # noqa: F401
from .predictor import lagrange_value, predict_point  # noqa: F401
