"""Debug probe of the pair kernel (pair.cu): per-launch time and the plan's
wait statistics (slbm_debug_pair_stats) on the bench bed.

    python tools/pair_debug.py [edge] [ahead] [slack] [hints]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2408_06880_b200 import _abi  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

lib = _abi.load()
lib.slbm_debug_pair_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint32)]
lib.slbm_set_tuning(5, 1)  # the pair kernel is off by default
torch.cuda.set_device(0)
st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
edge = int(sys.argv[1]) if len(sys.argv) > 1 else 512
if len(sys.argv) > 2:
    lib.slbm_set_tuning(7, int(sys.argv[2]))
if len(sys.argv) > 3:
    lib.slbm_set_tuning(6, int(sys.argv[3]))
if len(sys.argv) > 4:
    lib.slbm_set_tuning(8, int(sys.argv[4]))
fl = bench.make_flags(edge, 0)
e = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
e.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
s = torch.cuda.ExternalStream(e.stream())
prev = None
for k in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    e.run(2)
    e1.record(s)
    e1.synchronize()
    out = (C.c_uint32 * 16)()
    lib.slbm_debug_pair_stats(e._h, out)
    v = list(out)
    d = [v[4] - (prev[4] if prev else 0), v[5] - (prev[5] if prev else 0)]
    prev = v
    print(json.dumps({"edge": edge, "slack": sys.argv[3] if len(sys.argv) > 3 else "default",
                      "hints": sys.argv[4] if len(sys.argv) > 4 else "1", "launch": k, "ms": round(e0.elapsed_time(e1), 3),
                      "waits": d[0], "spins": d[1], "ctl": v[:4]}), flush=True)
