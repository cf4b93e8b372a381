"""Test-only model of the paper's §6 scheme in exact arithmetic,
used to pin reading C1 (corrected omega indices) and the 3k-6 count
against the naive oracle.  Not used by the product path.
"""


class Counter:
    def __init__(self, ar):
        self.ar = ar
        self.mults = 0

    def mul(self, p, q):
        self.mults += 1
        return self.ar.mul(p, q)


def omega_products(cm, xv, literal=False):
    """omega_m = prod_{j != m} x_{i_j} via prefixes psi and suffixes phi.

    literal=True uses the indices exactly as printed (omega_1 = psi_{k-1},
    omega_k = phi_{k-1}, omega_m = psi_{m-1} phi_{k-m+2}); literal=False uses
    reading C1 (omega_1 = phi_{k-1}, omega_k = psi_{k-1}, omega_m = psi_{m-1} phi_{k-m}).
    Lists are 1-based via a dummy slot 0.
    """
    ar = cm.ar
    k = len(xv)
    if k == 0:
        return []
    if k == 1:
        return [ar.one()]
    psi = [None] * k
    phi = [None] * k
    psi[1] = xv[0]
    for m in range(2, k):  # psi_m = psi_{m-1} x_{i_m}
        psi[m] = cm.mul(psi[m - 1], xv[m - 1])
    phi[1] = xv[k - 1]
    for m in range(2, k):  # phi_m = phi_{m-1} x_{i_{k-m+1}}
        phi[m] = cm.mul(phi[m - 1], xv[k - m])
    om = [None] * (k + 1)
    if literal:
        om[1] = psi[k - 1]
        om[k] = phi[k - 1]
        for m in range(2, k):
            j = k - m + 2
            om[m] = cm.mul(psi[m - 1], phi[j] if j < k else ar.one())
    else:
        om[1] = phi[k - 1]
        om[k] = psi[k - 1]
        for m in range(2, k):
            om[m] = cm.mul(psi[m - 1], phi[k - m])
    return om[1:]


def ad_row(ar, xs, terms, coeffs, n_var, literal=False):
    """F_i and J row i by §6: common factor, omega, shifted monomials, value,
    coefficient stage with the exponent factor a_m (reading C3)."""
    cm = Counter(ar)
    f = ar.zero()
    jrow = [ar.zero() for _ in range(n_var)]
    omega_mults = []
    for factors, c in zip(terms, coeffs):
        if not factors:
            f = ar.add(f, c)
            continue
        cf = ar.one()
        for v, a in factors:  # step 1: x_{i1}^{a1-1} ... x_{ik}^{ak-1}
            for _ in range(a - 1):
                cf = cm.mul(cf, xs[v])
        before = cm.mults
        om = omega_products(cm, [xs[v] for v, _ in factors], literal)
        omega_mults.append((len(factors), cm.mults - before))
        shifted = [cm.mul(cf, w) for w in om]  # step 2
        value = cm.mul(shifted[0], xs[factors[0][0]])  # step 3
        f = ar.add(f, ar.mul(c, value))
        for (v, a), s in zip(factors, shifted):
            jrow[v] = ar.add(jrow[v], ar.mul(c, ar.scale_int(s, a)))
    return f, jrow, omega_mults
