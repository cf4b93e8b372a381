"""Pins of the predictor oracle (NEXT-4, oracle/predictor.py): SPEC's worked examples
(hand-derived there), exact reproduction of quadratic paths, partition of unity."""
from fractions import Fraction as Fr

import numpy as np

from oracle.predictor import lagrange_value, predict_point
from synthetic import real_limbs


def test_spec_examples():
    # quadratic: (0,0), (1,1), (2,4), tNew = 3 -> 9
    assert lagrange_value([Fr(2), Fr(1), Fr(0)], [(Fr(4), 0), (Fr(1), 0), (Fr(0), 0)], Fr(3)) == (9, 0)
    # z(t) = t^3 at 0.1, 0.2, 0.3, tNew = 0.4 -> 0.058
    ts = [Fr(3, 10), Fr(2, 10), Fr(1, 10)]
    assert lagrange_value(ts, [(t ** 3, 0) for t in ts], Fr(4, 10)) == (Fr(58, 1000), 0)
    # secant: (0,0), (0.5,1), tNew = 0.75 -> 1.5; t^2 at 0.4, 0.5, tNew = 0.6 -> 0.34
    assert lagrange_value([Fr(1, 2), Fr(0)], [(Fr(1), 0), (Fr(0), 0)], Fr(3, 4)) == (Fr(3, 2), 0)
    assert lagrange_value([Fr(5, 10), Fr(4, 10)], [(Fr(25, 100), 0), (Fr(16, 100), 0)], Fr(6, 10)) == (Fr(34, 100), 0)
    # constant (one point)
    assert lagrange_value([Fr(1, 3)], [(Fr(7), Fr(-2))], Fr(1, 2)) == (7, -2)


def test_exact_on_quadratic_paths():
    rng = np.random.Generator(np.random.PCG64(3))
    for _ in range(20):
        a, b, c = [(Fr(int(rng.integers(-99, 99)), 64), Fr(int(rng.integers(-99, 99)), 32)) for _ in range(3)]
        ts = sorted({Fr(int(rng.integers(0, 1000)), 1024) for _ in range(3)}, reverse=True)
        if len(ts) < 3:
            continue
        x = lambda t: (a[0] + b[0] * t + c[0] * t * t, a[1] + b[1] * t + c[1] * t * t)  # noqa: E731
        tau = ts[0] + Fr(int(rng.integers(1, 100)), 4096)
        assert lagrange_value(ts, [x(t) for t in ts], tau) == x(tau)


def test_partition_of_unity_and_limbs_path():
    ts = [Fr(7, 16), Fr(3, 8), Fr(1, 4)]
    assert lagrange_value(ts, [(Fr(1), Fr(0))] * 3, Fr(1, 2)) == (1, 0)
    th = real_limbs(ts, 2)
    xh = np.zeros((3, 1, 2, 2))
    xh[:, 0, 0, 0] = [1.0, 1.0, 1.0]
    assert predict_point(th, xh, 3, real_limbs([Fr(1, 2)], 2)[0]) == [(1, 0)]
