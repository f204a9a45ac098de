"""Read-back of the box fields into pinned host buffers on the bench bed:
HBM staging + DMA copy (default) vs the field kernel writing straight into
mapped host memory (knob 12), a few repetitions each.

    python tools/fields_probe.py [reps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2408_06880_b200 import _abi  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
torch.cuda.set_device(0)
lib = _abi.load()
st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
eng = SparseEngine(bench.make_flags(bench.EDGE, 0), st, p, "aa", device=0, check="deferred")
eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
eng.run(4)
shape = tuple(reversed(eng.dims))
out = (torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy(),
       torch.empty(shape + (3,), dtype=torch.float64, pin_memory=True).numpy())
nbytes = out[0].nbytes + out[1].nbytes
res = {}
for mode in (0, 1, 0, 1):
    lib.slbm_set_tuning(12, mode)
    eng.macroscopic_fields(out=out)
    ts = []
    for _ in range(reps):
        eng.synchronize()
        t0 = time.perf_counter()
        eng.macroscopic_fields(out=out)
        ts.append(time.perf_counter() - t0)
    res.setdefault("mapped" if mode else "dma", []).append(round(min(ts), 4))
lib.slbm_set_tuning(12, 0)
print(json.dumps({"bytes": nbytes, "seconds_best": res,
                  "gbs_dma": round(nbytes / min(res["dma"]) / 1e9, 1),
                  "gbs_mapped": round(nbytes / min(res["mapped"]) / 1e9, 1)}))
