"""Dense (direct-addressing) sweeps on a box of porosity PHI: per-kernel
times (CUDA events per step) and the fraction of the measured copy peak.

    python tools/dense_probe.py [edge] [phi] [steps] [lean odd 1|0]

Measured (384^3, phi 1.0): even 0.89, odd 0.85 of the copy peak; 5 or 6
CTAs/SM for the odd sweep (96 / 80 registers, spills) were slower (0.84 /
0.79).  The lean odd kernel (k_dense_odd, knob 9) then reached 0.97.  A lean
combined (even) step in the same style — per-direction constant offsets
recomputed at the store, predicated solid cells — compiled to 84 registers
without spills but ran at 0.60 (vs 0.85): the per-direction face-wrap
branches break up the batch of 19 loads.  An interior-only variant with
straight-line loads (face cells left to k_dense<1> in a frame pass) was
bitwise equal but also slower (0.59 vs 0.71 at phi 0.8).  Not kept.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2408_06880_b200 import geometry  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.engine import DenseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

edge = int(sys.argv[1]) if len(sys.argv) > 1 else 384
phi = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lean = int(sys.argv[4]) if len(sys.argv) > 4 else 1

torch.cuda.set_device(0)
from paper_2408_06880_b200 import _abi  # noqa: E402

_abi.load().slbm_set_tuning(9, lean)

st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
fl = geometry.obstacle_flags((edge,) * 3, phi, 1)
eng = DenseEngine(fl, st, p, "aa", device=0, check="deferred")
eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
eng.run(6)
s = torch.cuda.ExternalStream(eng.stream())
evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
par = []
torch.cuda.synchronize()
evs[0].record(s)
for k in range(steps):
    par.append(eng.parity.value)
    eng.refresh_boundary(eng.parity)
    eng.step()
    eng.finish_step()
    evs[k + 1].record(s)
evs[-1].synchronize()
per = [evs[k].elapsed_time(evs[k + 1]) for k in range(steps)]
even = statistics.mean(t for t, q in zip(per, par) if q == 0)
odd = statistics.mean(t for t, q in zip(per, par) if q == 1)
cells = edge ** 3
peak = bench.measured_peak_gbs() if hasattr(bench, "measured_peak_gbs") else 6549.1
gbs = lambda ms: cells * 304 / (ms / 1e3) / 1e9  # noqa: E731
import hashlib  # noqa: E402

digest = hashlib.sha256(eng.canonical_state().tobytes()).hexdigest()[:16]
print(json.dumps({"edge": edge, "phi": phi, "lean_odd": lean, "state_sha": digest, "even_ms": round(even, 4), "odd_ms": round(odd, 4),
                  "even_frac": round(gbs(even) / peak, 3), "odd_frac": round(gbs(odd) / peak, 3),
                  "mflups": round(cells * steps / (sum(per) / 1e3) / 1e6, 1)}))
