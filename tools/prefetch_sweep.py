"""Index-list sweep duration vs the idx L2 prefetch distance (knobs 2/3) and
CTAs per SM (knob 13) on C5 random-obstacle beds and the bench bed, burst,
interleaved medians.  Tuning aid:  python tools/prefetch_sweep.py"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_06880_b200 import geometry  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

torch.cuda.set_device(0)
st = make_stencil("d3q19")
p = CollisionParams(1.2, "trt", trt_magic_lambda(1.2))
PEAK = 6549.1e9


def even_ms(eng, n=6):
    s = torch.cuda.ExternalStream(eng.stream())
    out = []
    for _ in range(n):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(s)
        eng.refresh_boundary(eng.parity); eng.step(); eng.finish_step()
        b.record(s)
        eng.refresh_boundary(eng.parity); eng.step(); eng.finish_step()
        c.record(s)
        c.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


cases = [("c5 phi0.3", lambda: geometry.obstacle_flags((384,) * 3, 0.3, 1)),
         ("c5 phi0.4", lambda: geometry.obstacle_flags((384,) * 3, 0.4, 1)),
         ("c5 phi0.5", lambda: geometry.obstacle_flags((384,) * 3, 0.5, 1))]
variants = [(c, q, a) for c in (4, 5) for (q, a) in ((1, 0), (2, 0), (3, 0), (0, 74), (4, 0))]
for name, mk in cases:
    eng = SparseEngine(mk(), st, p, "aa", device=0, check="deferred")
    eng.init_equilibrium(1.0, np.array([0.005, 0.0, 0.0]))
    eng.run(12)
    res = {v: [] for v in variants}
    for rnd in range(3):
        for v in variants:
            eng.set_tuning(13, v[0]); eng.set_tuning(2, v[1]); eng.set_tuning(3, v[2])
            even_ms(eng, 2)
            res[v].append(even_ms(eng))
    n = eng.n_fluid
    for v in variants:
        ms = statistics.median(res[v])
        print(f"{name} ctas={v[0]} ahead_q={v[1]} ahead_ctas={v[2]}: {ms:.4f} ms frac "
              f"{n * 376 / (ms * 1e-3) / PEAK:.3f}", flush=True)
    del eng
    torch.cuda.empty_cache()
