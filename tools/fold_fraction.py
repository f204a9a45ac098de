"""Fraction of (fluid cell, direction) pairs whose upwind neighbour is solid
(the no-slip folds of the index list) for the bench bed, C5 random
obstacles and the C4 artery.  Tuning aid (GPU box: the bed voxelizer runs
on the device):  python tools/fold_fraction.py"""
import sys; sys.path.insert(0, "/root/repo")
import numpy as np, bench
from paper_2408_06880_b200 import geometry
from paper_2408_06880_b200.lattice import make_stencil
st = make_stencil("d3q19"); C = np.array(st.c)
def fold_frac(fluid):
    tot = 0; folds = 0
    for q in range(1, 19):
        cx, cy, cz = C[q]
        up = np.roll(fluid, shift=(cz, cy, cx), axis=(0, 1, 2))
        folds += np.count_nonzero(fluid & ~up); tot += np.count_nonzero(fluid)
    return folds / tot
for name, fl in [("bed256", bench.make_flags(256, 0)),
                 ("obst0.3", geometry.obstacle_flags((96,)*3, 0.3, 1)),
                 ("obst0.6", geometry.obstacle_flags((96,)*3, 0.6, 1)),
                 ("obst0.05", geometry.obstacle_flags((96,)*3, 0.05, 1)),
                 ("obst0.9", geometry.obstacle_flags((96,)*3, 0.9, 1)),
                 ("artery", geometry.artery_flags((512,)*3, seed=0, r_root=40.0, r_min=14.0))]:
    fluid = fl.tags[1:-1, 1:-1, 1:-1] == 0
    print(name, round(fluid.mean(), 3), round(fold_frac(fluid), 3), flush=True)
