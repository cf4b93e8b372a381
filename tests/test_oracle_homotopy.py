"""Pins of the homotopy oracle (NEXT-3, oracle/homotopy.py) against things other than itself:
hand-derived worked examples (golden, cited), reduction to the plain evaluator at t = 0 and
t = 1, exact finite differences in t (h is affine in t), a closed form against mpmath, and
the t-as-variable expansion (the paper's "old" evaluator) evaluated by the plain
oracle."""
import json
import os
from dataclasses import replace
from fractions import Fraction

import mpmath
import numpy as np
import pytest

from oracle import ExactArith, evaluate_system
from oracle.homotopy import evaluate_homotopy_dt, evaluate_homotopy_rows
from synthetic import (config_system, homotopy_target, limbs_from_values, random_t, real_limbs,
                       system_from_terms)

GOLD = os.path.join(os.path.dirname(__file__), "golden", "homotopy_examples.json")
AR = ExactArith()


def _val(v):
    return AR.from_limbs(*limbs_from_values([complex(*v)], 2)[0])


def _golden_system(g, limbs=2):
    polys, cs, cf = [], [], []
    for poly in g["polys"]:
        terms = []
        for term in poly:
            terms.append([tuple(f) for f in term["f"]])
            cs.append(complex(*term["cs"]))
            cf.append(complex(*term["cf"]))
        polys.append(terms)
    s = system_from_terms(len(polys), g["n_var"], limbs, polys, limbs_from_values(cs, limbs))
    return s, limbs_from_values(cf, limbs)


def expand_t_as_variable(s, cf):
    """Test-side construction of the "old" representation: t becomes variable n_var and
    every term c x^a of the homotopy splits into c_s x^a - c_s t x^a + c_f t x^a."""
    polys, coeff = [], []
    for i in range(s.n_eq):
        terms = []
        for t, fac in s.terms(i):
            terms += [list(fac), list(fac) + [(s.n_var, 1)], list(fac) + [(s.n_var, 1)]]
            coeff += [s.coeff[t], -s.coeff[t], cf[t]]
        polys.append(terms)
    return system_from_terms(s.n_eq, s.n_var + 1, s.limbs, polys, np.asarray(coeff))


def test_golden_homotopy_examples():
    gold = json.load(open(GOLD))["systems"]
    for g in gold:
        s, cf = _golden_system(g)
        X = limbs_from_values([complex(*v) for v in g["x"]], 2)
        tl = real_limbs([Fraction(*g["t"])], 2)[0]
        ar, F, J = evaluate_homotopy_rows(s, cf, X, tl, arith="exact")
        _, D = evaluate_homotopy_dt(s, cf, X, arith="exact")
        for i in range(s.n_eq):
            assert AR.add(F[i], AR.scale_int(_val(g["F"][i]), -1))[:2] == (0, 0), g["cite"]
            assert AR.add(D[i], AR.scale_int(_val(g["dHdt"][i]), -1))[:2] == (0, 0), g["cite"]
            for v in range(s.n_var):
                assert AR.add(J[i][v], AR.scale_int(_val(g["J"][i][v]), -1))[:2] == (0, 0), g["cite"]


def _eq(a, b):
    return AR.add(a, AR.scale_int(b, -1))[:2] == (0, 0)


@pytest.mark.parametrize("name", ["tiny", "c2"])
def test_t0_and_t1_reduce_to_plain_systems(name):
    s, X = config_system(name, seed=2)
    cf = homotopy_target(s, seed=7)
    target = replace(s, coeff=cf)
    for tval, sysref in ((0, s), (1, target)):
        _, F, J = evaluate_homotopy_rows(s, cf, X[0], real_limbs([tval], s.limbs)[0], arith="exact")
        Fr, Jr = evaluate_system(sysref, X[0], arith="exact", workers=1)
        assert all(_eq(a, b) for a, b in zip(F, Fr))
        assert all(_eq(a, b) for ra, rb in zip(J, Jr) for a, b in zip(ra, rb))


def test_exact_finite_difference_in_t():
    """h is affine in t, so h(t1) - h(t0) = (t1 - t0) dh/dt exactly (rationals), for F and
    for every Jacobian entry (dJ/dt follows from the same identity per entry)."""
    s, X = config_system("tiny", seed=3)
    cf = homotopy_target(s, seed=9)
    t0, t1 = random_t(2, 2, seed=5)
    _, F0, J0 = evaluate_homotopy_rows(s, cf, X[0], t0, arith="exact")
    _, F1, J1 = evaluate_homotopy_rows(s, cf, X[0], t1, arith="exact")
    _, D = evaluate_homotopy_dt(s, cf, X[0], arith="exact")
    dt = AR.add(AR.from_limbs(t1, [0.0, 0.0]), AR.scale_int(AR.from_limbs(t0, [0.0, 0.0]), -1))
    for i in range(s.n_eq):
        assert _eq(AR.add(F1[i], AR.scale_int(F0[i], -1)), AR.mul(dt, D[i]))
    # J is affine in t as well: J(t) = J_start + t (J_target - J_start)
    Jt = evaluate_system(replace(s, coeff=cf), X[0], arith="exact", workers=1)[1]
    Js = evaluate_system(s, X[0], arith="exact", workers=1)[1]
    t0v = AR.from_limbs(t0, [0.0, 0.0])
    for i in range(s.n_eq):
        for v in range(s.n_var):
            want = AR.add(Js[i][v], AR.mul(t0v, AR.add(Jt[i][v], AR.scale_int(Js[i][v], -1))))
            assert _eq(J0[i][v], want)


def test_closed_form_single_monomial_mpmath():
    """h = c(t) x^d with c(t) = (1-t) c_s + t c_f: F = c(t) x^d, J = c(t) d x^(d-1) (mpmath)."""
    d = 7
    cs, cf = complex(0.75, -0.5), complex(-1.25, 2.0)
    x, t = complex(0.625, 0.375), 0.3125
    s = system_from_terms(1, 1, 4, [[[(0, d)]]], limbs_from_values([cs], 4))
    cfl = limbs_from_values([cf], 4)
    ar, F, J = evaluate_homotopy_rows(s, cfl, limbs_from_values([x], 4), real_limbs([t], 4)[0], arith="mp", prec=512)
    with mpmath.workprec(512):
        c = (1 - mpmath.mpf(t)) * mpmath.mpc(cs) + mpmath.mpf(t) * mpmath.mpc(cf)
        assert abs(F[0] - c * mpmath.power(mpmath.mpc(x), d)) < mpmath.mpf(2) ** -500
        assert abs(J[0][0] - c * d * mpmath.power(mpmath.mpc(x), d - 1)) < mpmath.mpf(2) ** -500


def test_old_t_as_variable_expansion_agrees():
    """The paper's "old" evaluator treats t as variable n+1: the expanded system
    evaluated by the plain oracle at (x, t) gives h, [dh/dx | dh/dt] exactly."""
    s, X = config_system("tiny", seed=1)
    cf = homotopy_target(s, seed=4)
    tl = random_t(1, 2, seed=8)[0]
    ex = expand_t_as_variable(s, cf)
    Xe = np.concatenate([X[0], np.zeros((1, 2, 2))])
    Xe[-1, 0, :] = tl
    Fe, Je = evaluate_system(ex, Xe, arith="exact", workers=1)
    _, F, J = evaluate_homotopy_rows(s, cf, X[0], tl, arith="exact")
    _, D = evaluate_homotopy_dt(s, cf, X[0], arith="exact")
    for i in range(s.n_eq):
        assert _eq(Fe[i], F[i])
        assert _eq(Je[i][s.n_var], D[i])
        assert all(_eq(Je[i][v], J[i][v]) for v in range(s.n_var))
