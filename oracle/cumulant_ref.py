"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement of the D3Q27 cumulant collision implemented in
``paper_2408_06880_b200/csrc/cumulant.cuh``.  The reference package has no
cumulant model, so this is NOT pinned to the reference; it is
an independent numpy transcription of the same algorithm (Geier et al.
2015, non-parametrised: shear rate omega, bulk and all higher orders rate
1; the bulk rate is a parameter) with the identical floating-point operation order, so the CUDA kernel
can be checked bit for bit against it, and it is itself checked against
physics: mass/momentum conservation, the product-form equilibrium as a
fixed point, omega = 1 giving that equilibrium, and the shear-wave decay
rate nu = (1/omega - 1/2)/3 (tests/test_cumulant.py).
"""

from __future__ import annotations

import numpy as np


def _seeded_sum(t, weights):
    acc = None
    for k, w in enumerate(weights):
        if w == 0:
            continue
        if acc is None:
            acc = t[k].copy() if w > 0 else -t[k]
        else:
            acc = acc + t[k] if w > 0 else acc - t[k]
    return acc


def moments_seedless(t, st):
    """collide.cuh moments(): rho sequential in q order; u components are
    signed sums seeded with their first term, then divided by rho."""
    rho = t[0] + t[1]
    for k in range(2, st.q):
        rho = rho + t[k]
    u = [_seeded_sum(t, st.c[:, a]) / rho for a in range(st.dim)]
    return rho, u


def _coef(u):
    uu = u * u
    b0 = 2.0 * u
    return {"am": uu - u, "a0": 1.0 - uu, "ap": uu + u, "b0": b0, "bm": b0 - 1.0, "bp": b0 + 1.0}


def _back3(k0, k1, k2, c):
    fm = ((k0 * c["am"] + k1 * c["bm"]) + k2) * 0.5
    f0 = (k0 * c["a0"] - k1 * c["b0"]) - k2
    fp = ((k0 * c["ap"] + k1 * c["bp"]) + k2) * 0.5
    return fm, f0, fp


def _back3_even(k0, k2, c):
    return (k0 * c["am"] + k2) * 0.5, k0 * c["a0"] - k2, (k0 * c["ap"] + k2) * 0.5


def _back3_odd(k1, c):
    return (k1 * c["bm"]) * 0.5, -(k1 * c["b0"]), (k1 * c["bp"]) * 0.5


def cumulant_collide(t, omega, st, bulk=1.0):
    """(27, n) pre-collision values -> (27, n) post-collision values; shear
    rate omega, bulk rate ``bulk`` (trace of the second order), higher
    orders rate 1 (cumulant.cuh cumulant_collide, same operation order)."""
    assert st.q == 27
    rho, (ux, uy, uz) = moments_seedless(t, st)
    c = st.c
    pxx = _seeded_sum(t, c[:, 0] * c[:, 0])
    pyy = _seeded_sum(t, c[:, 1] * c[:, 1])
    pzz = _seeded_sum(t, c[:, 2] * c[:, 2])
    pxy = _seeded_sum(t, c[:, 0] * c[:, 1])
    pxz = _seeded_sum(t, c[:, 0] * c[:, 2])
    pyz = _seeded_sum(t, c[:, 1] * c[:, 2])
    jx, jy, jz = rho * ux, rho * uy, rho * uz
    kxx, kyy, kzz = pxx - jx * ux, pyy - jy * uy, pzz - jz * uz
    kxy, kxz, kyz = pxy - jx * uy, pxz - jx * uz, pyz - jy * uz
    om1 = 1.0 - omega
    dxy = om1 * (kxx - kyy)
    dxz = om1 * (kxx - kzz)
    tr = rho + (1.0 - bulk) * (((kxx + kyy) + kzz) - rho)
    sxx = ((tr + dxy) + dxz) / 3.0
    syy = sxx - dxy
    szz = sxx - dxz
    sxy, sxz, syz = om1 * kxy, om1 * kxz, om1 * kyz
    ir = 1.0 / rho
    k220 = (sxx * syy + 2.0 * (sxy * sxy)) * ir
    k202 = (sxx * szz + 2.0 * (sxz * sxz)) * ir
    k022 = (syy * szz + 2.0 * (syz * syz)) * ir
    k211 = (sxx * syz + 2.0 * (sxy * sxz)) * ir
    k121 = (syy * sxz + 2.0 * (sxy * syz)) * ir
    k112 = (szz * sxy + 2.0 * (sxz * syz)) * ir
    lin = ((sxx * k022 + syy * k202) + szz * k220) + 4.0 * ((syz * k211 + sxz * k121) + sxy * k112)
    cub = (16.0 * ((sxy * sxz) * syz)
           + 4.0 * (((sxz * sxz) * syy + (syz * syz) * sxx) + (sxy * sxy) * szz)) \
        + 2.0 * ((sxx * syy) * szz)
    k222 = lin * ir - cub * (ir * ir)

    cx, cy, cz = _coef(ux), _coef(uy), _coef(uz)
    G = [[[None] * 3 for _ in range(3)] for _ in range(3)]

    def put(b, cc, vals):
        for i in range(3):
            G[i][b][cc] = vals[i]

    put(0, 0, _back3_even(rho, sxx, cx))
    put(1, 0, _back3_odd(sxy, cx))
    put(2, 0, _back3_even(syy, k220, cx))
    put(0, 1, _back3_odd(sxz, cx))
    put(1, 1, _back3_even(syz, k211, cx))
    put(2, 1, _back3_odd(k121, cx))
    put(0, 2, _back3_even(szz, k202, cx))
    put(1, 2, _back3_odd(k112, cx))
    put(2, 2, _back3_even(k022, k222, cx))
    for i in range(3):
        for cc in range(3):
            a, b, d = _back3(G[i][0][cc], G[i][1][cc], G[i][2][cc], cy)
            G[i][0][cc], G[i][1][cc], G[i][2][cc] = a, b, d
    out = np.empty_like(t)
    index = {tuple(int(v) for v in st.c[k]): k for k in range(st.q)}
    for i in range(3):
        for j in range(3):
            vals = _back3(G[i][j][0], G[i][j][1], G[i][j][2], cz)
            for kk in range(3):
                out[index[(i - 1, j - 1, kk - 1)]] = vals[kk]
    return out


def product_equilibrium(rho, u, st):
    """D3Q27 product-form equilibrium rho * prod_a phi(c_a, u_a) with
    phi(-1) = (u^2 - u + 1/3)/2, phi(0) = 2/3 - u^2, phi(1) = (u^2 + u + 1/3)/2:
    the cumulant method's equilibrium (all central moments Maxwellian)."""
    phi = []
    for ua in u:
        phi.append({-1: 0.5 * (ua * ua - ua + 1.0 / 3.0), 0: 2.0 / 3.0 - ua * ua,
                    1: 0.5 * (ua * ua + ua + 1.0 / 3.0)})
    out = np.empty((st.q,) + np.shape(rho))
    for k in range(st.q):
        cx, cy, cz = (int(v) for v in st.c[k])
        out[k] = rho * phi[0][cx] * phi[1][cy] * phi[2][cz]
    return out
