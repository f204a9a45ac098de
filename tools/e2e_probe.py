"""Break the bench's e2e time into its parts (init H2D, drive loop,
macroscopic D2H) on the C2 workload; tuning aid, not a bench line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

torch.cuda.set_device(0)
st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
fl = bench.make_flags(bench.EDGE, 0)
eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
q, n = st.q, eng.n_fluid
host = torch.empty((q, n), dtype=torch.float64, pin_memory=True).numpy()
for r in range(q):
    host[r].fill(st.w[r])
out = {}
for rep in range(2):
    eng.check = "step"
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.init_canonical(host)
    t1 = time.perf_counter()
    for _ in range(200):
        eng.refresh_boundary(eng.parity)
        eng.step()
        eng.finish_step()
    t2 = time.perf_counter()
    rho, u = eng.macroscopic_fields()
    t3 = time.perf_counter()
    out[rep] = {"init_s": t1 - t0, "loop_s": t2 - t1, "macro_s": t3 - t2}
    del rho, u
print(json.dumps(out))
