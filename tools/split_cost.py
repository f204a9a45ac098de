"""Cost of the interior/frame split used by the overlapped driver: one AA
step as a single sweep vs interior sweep + frame sweep (same engine, same
state), on the bench workload.  Tuning aid, not a bench line."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

edge = int(os.environ.get("EDGE", bench.EDGE))
st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
from paper_2408_06880_b200.engine import HaloWidths  # noqa: E402

fw = os.environ.get("FRAME", "1")
frame = int(fw) if "," not in fw else HaloWidths(int(x) for x in fw.split(","))
eng = SparseEngine(bench.make_flags(edge, 0), st, p, "aa", device=0, check="deferred",
                   frame_width=frame)
eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
stream = torch.cuda.ExternalStream(eng.stream())
res = {"frame": fw, "n_fluid": eng.n_fluid, "n_frame": eng.n_frame, "n_interior": eng.n_interior}
times = {}
for rep in range(6):
    for mode in ("whole", "split"):
        for par in (0, 1):
            a = torch.cuda.Event(enable_timing=True)
            m = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if mode == "whole":
                eng.step()
                m.record(stream)
            else:
                eng.step("interior")
                m.record(stream)
                eng.step("frame")
            b.record(stream)
            eng.finish_step()
            b.synchronize()
            tag = "even" if eng.parity.value == 1 else "odd"
            times.setdefault(f"{mode}_{tag}", []).append(a.elapsed_time(b))
            if mode == "split":
                times.setdefault(f"interior_{tag}", []).append(a.elapsed_time(m))
                times.setdefault(f"frame_{tag}", []).append(m.elapsed_time(b))
eng.poll()
for k, v in times.items():
    res[k + "_ms"] = round(statistics.median(v), 4)
print(json.dumps(res))
