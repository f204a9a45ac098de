"""Does row/group alignment matter?  The bench bed as is (N_F % 32 != 0:
idx rows and PDF groups start mid-line) vs the same bed with N_F % 32 fluid
cells turned solid (every idx row and PDF group 256-B aligned).  Tuning aid."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_06880_b200 import geometry  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402
from paper_2408_06880_b200.tags import PERIODIC, make_flags  # noqa: E402

torch.cuda.set_device(0)
st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
dims = (512,) * 3
n = geometry.overlapping_sphere_count(dims, bench.DIAMETER, bench.POROSITY)
solid = geometry.voxelize_spheres(dims, geometry.sphere_centers(dims, bench.DIAMETER, n, bench.SEED),
                                  bench.DIAMETER, 0)


def pair(eng, reps=8):
    s = torch.cuda.ExternalStream(eng.stream())
    out = {0: [], 1: []}
    for _ in range(2 * reps):
        par = eng.parity.value
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        eng.step()
        b.record(s)
        eng.finish_step()
        b.synchronize()
        out[par].append(a.elapsed_time(b))
    return statistics.median(out[0]), statistics.median(out[1])


res = {}
hbm = bench.peaks()[0]
for rep in range(2):
    for name in ("as_is", "aligned"):
        sol = np.array(solid, dtype=bool, copy=True)
        if name == "aligned":
            flat = sol.reshape(-1)
            fluid_idx = np.flatnonzero(~flat)
            extra = fluid_idx.size % 32
            flat[np.random.default_rng(0).choice(fluid_idx, extra, replace=False)] = True
        fl = make_flags(dims, [(PERIODIC, PERIODIC)] * 3, solid=sol)
        eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
        eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
        te, to = pair(eng)
        res[f"{name}_{rep}"] = {"n_fluid": eng.n_fluid, "mod32": eng.n_fluid % 32,
                                "even_frac": round(eng.n_fluid * 376 / te / 1e6 / hbm, 4),
                                "odd_frac": round(eng.n_fluid * 304 / to / 1e6 / hbm, 4)}
        del eng
        torch.cuda.empty_cache()
print(json.dumps(res))
