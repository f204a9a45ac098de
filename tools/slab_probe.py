"""Phase timing of the overlapped step on a slab domain (one GPU, device-
local halo): interior sweep, halo wait, frame sweep, per parity, through the
block group and through per-engine launches.  Tuning aid."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.domain import Domain, _cuda_engine, phase_for  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

torch.cuda.set_device(0)
edge = 512
st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
fl = bench.make_flags(edge, 0)
slabs = int(os.environ.get("SLABS", 2))
block = (edge, edge, edge // slabs)
res = {"block": block}
for mode in ("group", "engines"):
    kw = {} if mode == "group" else {"engine_factory": _cuda_engine}
    d = Domain(fl, block, st, p, pattern="aa", frame_width="halo", check="deferred", **kw)
    d.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
    d.run(2, driver="overlapped")
    s = torch.cuda.ExternalStream(d.stream())
    out = {}
    for _ in range(8):
        par = "even" if d.parity.value == 0 else "odd"
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        phase = phase_for(d.pattern, d.parity)
        ev[0].record(s)
        d._halo.start(phase, d._stream)
        d._refresh_all()
        ev[1].record(s)
        d._sweep("interior")
        ev[2].record(s)
        d._halo.wait(d._stream)
        ev[3].record(s)
        d._sweep("frame")
        ev[4].record(s)
        d._finish_all()
        ev[4].synchronize()
        for k, name in enumerate(("start_refresh", "interior", "wait", "frame")):
            out.setdefault(f"{mode}_{par}_{name}", []).append(ev[k].elapsed_time(ev[k + 1]))
    d.poll()
    res.update({k: round(statistics.median(v), 4) for k, v in out.items()})
    res[f"{mode}_n_fluid"] = d.total_fluid()
    del d
    torch.cuda.empty_cache()
print(json.dumps(res))
