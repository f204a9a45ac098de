"""Per-cell sweep throughput of slab-shaped engines: alone, two side by
side, and inside a Domain.  Tuning aid."""
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

torch.cuda.set_device(0)
st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))


def pair_times(e, reps=4):
    s = torch.cuda.ExternalStream(e.stream())
    out = {0: [], 1: []}
    for _ in range(2 * reps):
        par = e.parity.value
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        e.step()
        b.record(s)
        e.finish_step()
        b.synchronize()
        out[par].append(a.elapsed_time(b))
    ev, od = statistics.median(out[0]), statistics.median(out[1])
    return {"even_gbs": round(e.n_fluid * 376 / ev / 1e6, 1), "odd_gbs": round(e.n_fluid * 304 / od / 1e6, 1)}


res = {}
dims = tuple(int(x) for x in os.environ.get("DIMS", "512,512,256").split(","))
fl = geometry.packed_bed_flags(dims, 0.3, 16.0, 1, periodic=True, device=0)
e1 = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
e1.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
res["alone"] = pair_times(e1)
fl2 = geometry.packed_bed_flags(dims, 0.3, 16.0, 2, periodic=True, device=0)
e2 = SparseEngine(fl2, st, p, "aa", device=0, check="deferred")
e2.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
res["first_of_two"] = pair_times(e1)
res["second_of_two"] = pair_times(e2)
full = bench.make_flags(512, 0)
del e1, e2
torch.cuda.empty_cache()
e3 = SparseEngine(full, st, p, "aa", device=0, check="deferred")
e3.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
res["full_512"] = pair_times(e3)
print(json.dumps(res))
