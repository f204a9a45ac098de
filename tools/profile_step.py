"""Short driver for ncu captures: builds the bench workload (512^3 periodic
bed, D3Q19 TRT AA) and issues a few individual sweeps.

    ncu --set full -k regex:k_aa -c 2 python tools/profile_step.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402


def main():
    edge = int(os.environ.get("EDGE", bench.EDGE))
    q = int(os.environ.get("Q", 19))
    model = os.environ.get("MODEL", "trt")
    steps = int(os.environ.get("STEPS", 6))
    st = make_stencil("d3q19" if q == 19 else "d3q27")
    p = CollisionParams(bench.OMEGA, model, bench.magic_lambda(bench.OMEGA))
    if os.environ.get("DENSE"):
        from paper_2408_06880_b200 import geometry
        from paper_2408_06880_b200.engine import DenseEngine

        phi = float(os.environ.get("PHI", 1.0))
        fl = geometry.obstacle_flags((edge,) * 3, phi, 1)
        eng = DenseEngine(fl, st, p, "aa", device=0, check="deferred")
    elif os.environ.get("ARTERY"):  # C4 vessel tree as one block
        from paper_2408_06880_b200 import geometry

        fl = geometry.artery_flags((edge,) * 3, seed=0, r_root=40.0, r_min=14.0)
        eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
    elif os.environ.get("OBSTACLE"):  # C5: cell-wise random obstacles at porosity PHI
        from paper_2408_06880_b200 import geometry

        fl = geometry.obstacle_flags((edge,) * 3, float(os.environ.get("PHI", 0.3)), 1)
        eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
    else:
        fl = bench.make_flags(edge, 0)
        eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
    eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
    for _ in range(steps):
        eng.refresh_boundary(eng.parity)
        eng.step()
        eng.finish_step()
    eng.poll()
    print("n_fluid", eng.n_fluid, "steps", steps)


if __name__ == "__main__":
    main()
