"""Model of the index-list gather's memory transactions for two fluid-cell
orders on cell-wise random obstacle beds: distinct 32-B sectors per warp
request of the AA even sweep (neighbour's group slot, or the fold's own
group slot), reference lexicographic order vs brick orders.  CPU only.

    PYTHONPATH=. python tools/order_model.py
"""
import numpy as np
from paper_2408_06880_b200 import geometry
from paper_2408_06880_b200.lattice import make_stencil
st = make_stencil("d3q19")
C = np.array(st.c)
def sim(phi, order, N=96, B=4):
    rng = np.random.default_rng(1)
    fluid = rng.random((N, N, N)) < phi   # [z,y,x], periodic
    zz, yy, xx = np.nonzero(fluid)
    if order == "lex":
        key = (zz * N + yy) * N + xx
    else:
        key = ((((zz // B) * (N // B) + yy // B) * (N // B) + xx // B) * B**3
               + ((zz % B) * B + yy % B) * B + xx % B)
    o = np.argsort(key, kind="stable")
    zz, yy, xx = zz[o], yy[o], xx[o]
    nf = len(zz)
    cid = -np.ones((N, N, N), dtype=np.int64)
    cid[zz, yy, xx] = np.arange(nf)
    tot_sec = 0; tot_req = 0
    for q in range(1, 19):
        cx, cy, cz = C[q]
        nz, ny, nx = (zz - cz) % N, (yy - cy) % N, (xx - cx) % N
        nb = cid[nz, ny, nx]
        # slot address in doubles: group q of neighbour, or fold: group inv q of own
        addr = np.where(nb >= 0, q * nf + nb, (19 + q) * nf + np.arange(nf))
        sec = addr // 4
        w = np.arange(nf) // 32
        # distinct sectors per warp
        pairs = np.unique(np.stack([w, sec]), axis=1)
        tot_sec += pairs.shape[1]; tot_req += w.max() + 1
    return tot_sec / tot_req
for phi in (0.3, 0.6):
    print(phi, "lex", round(sim(phi, "lex"), 2), "brick4", round(sim(phi, "brick"), 2), "brick2", round(sim(phi, "brick", B=2),2))
