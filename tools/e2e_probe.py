"""Break the bench's e2e time into its parts (init H2D, drive loop,
macroscopic D2H) on the C2 workload, for a few host-copy settings
(slbm_set_tuning knobs 10 = chunk MiB, 11 = threads); tuning aid only."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_06880_b200 import _abi  # noqa: E402
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
lib = _abi.load()
eng.init_canonical(host)
settings = [tuple(int(x) for x in s.split("x")) for s in
            os.environ.get("SETTINGS", "8x8,4x8,16x8,8x4,8x12,8x16,32x12").split(",")]
out = []
for chunk, threads in settings:
    lib.slbm_set_tuning(10, chunk)
    lib.slbm_set_tuning(11, threads)
    rho, u = eng.macroscopic_fields()  # lanes allocated outside the timing
    del rho, u
    for rep in range(2):
        eng.check = "step"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.init_canonical(host)
        t1 = time.perf_counter()
        for _ in range(20):
            eng.refresh_boundary(eng.parity)
            eng.step()
            eng.finish_step()
        t2 = time.perf_counter()
        rho, u = eng.macroscopic_fields()
        t3 = time.perf_counter()
        c = eng.canonical_state()
        t4 = time.perf_counter()
        out.append({"chunk_mib": chunk, "threads": threads, "rep": rep, "init_s": round(t1 - t0, 4),
                    "loop20_s": round(t2 - t1, 4), "macro_s": round(t3 - t2, 4),
                    "canonical_s": round(t4 - t3, 4)})
        print(json.dumps(out[-1]), flush=True)
        del rho, u, c
