"""Per-kernel device time of the C4 artery domain's overlapped step (CUPTI
through torch.profiler): where a strong-scaling step goes.  Tuning aid."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_06880_b200 import geometry  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda  # noqa: E402
from paper_2408_06880_b200.domain import Domain  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

torch.cuda.set_device(0)
DRIVER = os.environ.get("DRIVER", "overlapped")
fw = os.environ.get("FRAME", "1")
fw = int(fw) if fw.isdigit() else fw
fl = geometry.artery_flags((512, 512, 512), seed=0, r_root=40.0, r_min=14.0)
st = make_stencil("d3q19")
p = CollisionParams(1.7, "trt", trt_magic_lambda(1.7))
dom = Domain(fl, int(os.environ.get("BLOCK", 128)), st, p, pattern="aa", frame_width=fw,
             device=0, check="deferred")
dom.init_equilibrium()
dom.run(4, driver=DRIVER, use_graph=True)
dom.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

steps = 8
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    dom.run(steps, driver=DRIVER, use_graph=True)
    torch.cuda.synchronize()
agg = {}
for ev in prof.events():
    if ev.device_type.name == "CUDA":
        k = ev.name.replace("(anonymous namespace)::", "").split("(")[0][:70]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ev.device_time_total
s = torch.cuda.ExternalStream(dom.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
dom.run(40, driver=DRIVER, use_graph=True)
e1.record(s)
e1.synchronize()
ms = e0.elapsed_time(e1) / 40
nf = dom.total_fluid()
print(json.dumps({"driver": DRIVER, "frame": str(fw), "blocks": len(dom.blocks), "n_fluid": nf,
                  "ms_per_step": round(ms, 4), "mflups": round(nf / ms / 1e3, 1),
                  "kernels_us_per_step": {k: [n / steps, round(t / steps, 1)] for k, (n, t) in
                                          sorted(agg.items(), key=lambda kv: -kv[1][1])}}))
