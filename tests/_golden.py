"""Loader of tests/golden/large_seed1.npz (written by tools/make_golden_large.py from oracle/
and synthetic/ only): the mp512 oracle values of the "large" config, as mpmath complex values."""
import hashlib
import os

import mpmath
import numpy as np

PATH = os.path.join(os.path.dirname(__file__), "golden", "large_seed1.npz")


def load():
    return np.load(PATH)


def digest(s, X):
    """SHA-256 of the system tables and the given points (tools/make_golden_large.input_digest)."""
    h = hashlib.sha256()
    for a in (s.poly_ptr, s.term_ptr, s.var_idx, s.exponent, s.coeff, X):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def to_mpc(limbs):
    """[N][2][10] stored limbs -> N mpmath complex values (exact limb sums at 1,100 bits)."""
    out = []
    with mpmath.workprec(1100):
        for v in np.asarray(limbs).reshape(-1, 2, limbs.shape[-1]):
            out.append(mpmath.mpc(mpmath.fsum(mpmath.mpf(float(d)) for d in v[0]),
                                  mpmath.fsum(mpmath.mpf(float(d)) for d in v[1])))
    return out
