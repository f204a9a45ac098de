"""Per-step duration of the index-list sweep over 80 steps on a C5 bed:
the clock drifts down under the board power cap, so a mean taken after
a few hundred steps (tools/bench_configs.py) sits below a burst median
(tools/variants.py).  Diagnostic:  python tools/c5_timing_check.py"""
import os, sys, statistics
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2408_06880_b200 import geometry
from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda
from paper_2408_06880_b200.engine import SparseEngine
from paper_2408_06880_b200.lattice import make_stencil
st = make_stencil("d3q19"); p = CollisionParams(1.2, "trt", trt_magic_lambda(1.2))
fl = geometry.obstacle_flags((384,) * 3, 0.6, 1)
eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
eng.init_equilibrium(1.0, np.array([0.005, 0.0, 0.0]))
eng.run(12)
s = torch.cuda.ExternalStream(eng.stream())
evs = [torch.cuda.Event(enable_timing=True) for _ in range(81)]
par = []
evs[0].record(s)
for k in range(80):
    par.append(eng.parity.value)
    eng.refresh_boundary(eng.parity); eng.step(); eng.finish_step()
    evs[k + 1].record(s)
evs[-1].synchronize()
per = [evs[k].elapsed_time(evs[k + 1]) for k in range(80)]
ev = [t for t, q in zip(per, par) if q == 0]
print("even per-step ms: mean", round(statistics.mean(ev), 4), "median", round(statistics.median(ev), 4), "min", round(min(ev), 4), "max", round(max(ev), 4))
print("first 10 even", [round(x, 3) for x in ev[:10]])
print("ctas", eng.sweep_ctas, "nf", eng.n_fluid)
