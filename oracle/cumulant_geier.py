"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Independent CPU restatement of the D3Q27 cumulant collision with general
relaxation rates, written from the definitions in Geier, Schoenherr,
Pasquali, Krafczyk 2015 ("The cumulant lattice Boltzmann equation in three
dimensions: theory and validation", Comput. Math. Appl. 70) -- NOT from the
CUDA kernel (csrc/cumulant.cuh), whose route differs on purpose:

* here: raw moments M_abc = sum_q f_q c^abc / rho of the normalised
  distribution; cumulants of every order 1..6 from them by the general
  moment-cumulant formula over set partitions (singleton blocks included,
  so the first cumulants are the velocity); the relaxation of Geier 2015
  eqs. (57)-(77) in the combinations the paper relaxes, solved back with a
  linear solve; raw moments from the post-collision cumulants (same
  partition sums, coefficient 1); f* = rho V^-1 M* with the 27x27 raw-moment
  matrix V inverted numerically;
* the kernel: chimera transforms to central moments, generated closed-form
  relations without singleton blocks, closed-form back substitution.

The two agree to rounding (tests/test_cumulant.py: <= 1e-12 relative), which
pins the kernel's algebra to the paper's definitions; the physics tests
(shear and bulk wave decay, Galilean invariance) pin the model.  The
reference package has no cumulant model: parity UNPINNED.

Rates: omega = w1 (shear), bulk = w2, higher = (w3, ..., w10).
Equilibrium cumulants: C_200 = C_020 = C_002 = c_s^2 = 1/3, all other
second-order and every higher-order cumulant 0.
"""

from __future__ import annotations

from collections import defaultdict
from functools import lru_cache
from math import factorial

import numpy as np

INDICES = [(a, b, c) for c in range(3) for b in range(3) for a in range(3)]


def _set_partitions(items):
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for part in _set_partitions(rest):
        for i in range(len(part)):
            yield part[:i] + [[first] + part[i]] + part[i + 1:]
        yield [[first]] + part


@lru_cache(maxsize=None)
def _partition_terms(abc):
    """{(multi-indices of the blocks...): (n_blocks, multiplicity)} over all
    set partitions of the multiset {x^a, y^b, z^c}."""
    elems = [0] * abc[0] + [1] * abc[1] + [2] * abc[2]
    terms = defaultdict(int)
    nblocks = {}
    for part in _set_partitions(list(range(len(elems)))):
        key = tuple(sorted(tuple(sum(1 for i in b if elems[i] == ax) for ax in range(3))
                           for b in part))
        terms[key] += 1
        nblocks[key] = len(part)
    return {k: (nblocks[k], v) for k, v in terms.items()}


def cumulants_from_raw(M):
    """{abc: array} raw moments of a normalised distribution (M_000 = 1) ->
    {abc: array} cumulants, orders 1..6 (kappa = sum_pi (-1)^(|pi|-1)
    (|pi|-1)! prod_B M_B)."""
    K = {}
    for abc in INDICES:
        if sum(abc) == 0:
            continue
        acc = 0.0
        for key, (nb, mult) in _partition_terms(abc).items():
            prod = mult * (-1) ** (nb - 1) * factorial(nb - 1)
            for b in key:
                prod = prod * M[b]
            acc = acc + prod
        K[abc] = acc
    return K


def raw_from_cumulants(K):
    """Inverse: M_abc = sum_pi prod_B K_B."""
    M = {(0, 0, 0): np.ones_like(K[(1, 0, 0)])}
    for abc in INDICES:
        if sum(abc) == 0:
            continue
        acc = 0.0
        for key, (_, mult) in _partition_terms(abc).items():
            prod = float(mult)
            for b in key:
                prod = prod * K[b]
            acc = acc + prod
        M[abc] = acc
    return M


def _moment_matrix(st):
    c = st.c.astype(np.float64)
    return np.array([[c[q, 0] ** a * c[q, 1] ** b * c[q, 2] ** g for q in range(st.q)]
                     for (a, b, g) in INDICES])


def relax(K, omega, bulk, higher):
    """Geier 2015 relaxation of the normalised cumulants (in place copy)."""
    w3, w4, w5, w6, w7, w8, w9, w10 = (float(w) for w in higher)
    R = dict(K)
    # second order: off-diagonal and the two deviatoric differences with w1,
    # the trace towards 3 c_s^2 = 1 with w2; solved back for the diagonal
    for abc in ((1, 1, 0), (1, 0, 1), (0, 1, 1)):
        R[abc] = (1.0 - omega) * K[abc]
    d1 = (1.0 - omega) * (K[(2, 0, 0)] - K[(0, 2, 0)])
    d2 = (1.0 - omega) * (K[(2, 0, 0)] - K[(0, 0, 2)])
    tr = bulk * 1.0 + (1.0 - bulk) * (K[(2, 0, 0)] + K[(0, 2, 0)] + K[(0, 0, 2)])
    A = np.array([[1.0, -1.0, 0.0], [1.0, 0.0, -1.0], [1.0, 1.0, 1.0]])
    sol = np.linalg.solve(A, np.stack([d1, d2, tr]).reshape(3, -1))
    for i, abc in enumerate(((2, 0, 0), (0, 2, 0), (0, 0, 2))):
        R[abc] = sol[i].reshape(np.shape(d1))
    # third order: C_120 +/- C_102 (w3 / w4) and its cyclic partners, C_111 (w5)
    for p, q in (((1, 2, 0), (1, 0, 2)), ((2, 1, 0), (0, 1, 2)), ((2, 0, 1), (0, 2, 1))):
        s = (1.0 - w3) * (K[p] + K[q])
        d = (1.0 - w4) * (K[p] - K[q])
        R[p], R[q] = (s + d) / 2.0, (s - d) / 2.0
    R[(1, 1, 1)] = (1.0 - w5) * K[(1, 1, 1)]
    # fourth order: C_220 - 2 C_202 + C_022, C_220 + C_202 - 2 C_022 (w6),
    # C_220 + C_202 + C_022 (w7); C_211, C_121, C_112 (w8)
    B = np.array([[1.0, -2.0, 1.0], [1.0, 1.0, -2.0], [1.0, 1.0, 1.0]])
    v = np.stack([K[(2, 2, 0)], K[(2, 0, 2)], K[(0, 2, 2)]]).reshape(3, -1)
    comb = B @ v
    comb[0] *= 1.0 - w6
    comb[1] *= 1.0 - w6
    comb[2] *= 1.0 - w7
    sol = np.linalg.solve(B, comb)
    for i, abc in enumerate(((2, 2, 0), (2, 0, 2), (0, 2, 2))):
        R[abc] = sol[i].reshape(np.shape(d1))
    for abc in ((2, 1, 1), (1, 2, 1), (1, 1, 2)):
        R[abc] = (1.0 - w8) * K[abc]
    for abc in ((2, 2, 1), (2, 1, 2), (1, 2, 2)):
        R[abc] = (1.0 - w9) * K[abc]
    R[(2, 2, 2)] = (1.0 - w10) * K[(2, 2, 2)]
    return R


def cumulants_of(f, st):
    """(rho, {abc: normalised cumulant}) of (27, n) populations."""
    V = _moment_matrix(st)
    raw = V @ f
    rho = raw[0]
    M = {abc: raw[i] / rho for i, abc in enumerate(INDICES)}
    return rho, cumulants_from_raw(M)


def populations_of(rho, K, st):
    """Inverse of cumulants_of."""
    V = _moment_matrix(st)
    M = raw_from_cumulants(K)
    raw = np.stack([M[abc] for abc in INDICES]) * rho
    return np.linalg.solve(V, raw)


def collide_general(f, omega, bulk, higher, st):
    """(27, n) -> (27, n) post-collision populations."""
    assert st.q == 27
    higher = (1.0,) * 8 if higher is None else tuple(higher)
    rho, K = cumulants_of(f, st)
    return populations_of(rho, relax(K, omega, bulk, higher), st)


def equilibrium(rho, u, st):
    """Populations whose cumulants are the equilibrium ones (velocity u)."""
    n = np.shape(rho)
    K = {abc: np.zeros(n) for abc in INDICES if sum(abc)}
    for a in range(3):
        e = [0, 0, 0]
        e[a] = 1
        K[tuple(e)] = np.asarray(u[a], dtype=np.float64) * np.ones(n)
        e[a] = 2
        K[tuple(e)] = np.full(n, 1.0 / 3.0)
    return populations_of(np.asarray(rho, dtype=np.float64), K, st)
