"""C4 strong-scaling proxy on ONE GPU.

Builds the configs[3] artery (512^3 box, 128^3 blocks), measures the whole
domain, then the share one rank of an 8-GPU run holds: blocks go to 8
workers by the reference's Hilbert/greedy balance (domain.py:312-325) and
every cell outside worker 0's blocks is made solid, so the proxy runs worker
0's blocks at their real size and block count (its halo toward other ranks
becomes wall, a small part of the step).  Reports MFLUPS, the whole step's
fraction of the HBM roofline (340 B per fluid-cell update, pair average),
our kernel launches per step, and a per-kernel breakdown (torch.profiler).

    python tools/c4_share.py [--workers 8]
"""

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2408_06880_b200 import _abi, geometry  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda  # noqa: E402
from paper_2408_06880_b200.domain import Domain  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402
from paper_2408_06880_b200.tags import FlagField  # noqa: E402

STEPS = int(os.environ.get("STEPS", 200))


def measure(dom, label, profile=True):
    dom.init_equilibrium()
    dom.run(4, driver="overlapped", use_graph=True)
    dom.synchronize()
    s = torch.cuda.ExternalStream(dom.stream())
    c0 = _abi.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    dom.run(STEPS, driver="overlapped", use_graph=True)
    e1.record(s)
    e1.synchronize()
    launches = (_abi.launch_count() - c0) / STEPS
    ms = e0.elapsed_time(e1) / STEPS
    nf = dom.total_fluid()
    hbm = bench.peaks()[0]
    c = dom.counters()
    out = {"case": label, "blocks": len(dom.blocks), "n_fluid": nf, "ms_per_step": round(ms, 4),
           "n_ubb": sum(e.n_ubb_slots for e in dom.local_engines()),
           "n_outlet": sum(e.n_outlet_slots for e in dom.local_engines()),
           "halo_values_per_step": c.values_exchanged / max(c.steps, 1),
           "mflups": round(nf / ms / 1e3, 1),
           "step_frac": round(nf * 340 / (ms / 1e3) / 1e9 / hbm, 4),
           "launches_per_step": launches}
    if profile:
        from torch.profiler import ProfilerActivity, profile as prof_

        n = 8
        with prof_(activities=[ProfilerActivity.CUDA]) as prof:
            dom.run(n, driver="overlapped", use_graph=True)
            torch.cuda.synchronize()
        agg = {}
        seq = [(ev.name.replace("(anonymous namespace)::", "").split("(")[0][:40], round(ev.device_time_total, 1))
               for ev in prof.events() if ev.device_type.name == "CUDA"]
        out["first_launches_us"] = seq[:8]
        for ev in prof.events():
            if ev.device_type.name == "CUDA":
                k = ev.name.replace("(anonymous namespace)::", "").split("(")[0][:60]
                a = agg.setdefault(k, [0, 0.0])
                a[0] += 1
                a[1] += ev.device_time_total
        out["kernels_us_per_step"] = {k: [c / n, round(t / n, 1)] for k, (c, t) in agg.items()}
        out["kernel_sum_us_per_step"] = round(sum(t for _, t in agg.values()) / n, 1)
    dom.poll()
    print(json.dumps(out), flush=True)
    return out


def main():
    workers = int(sys.argv[sys.argv.index("--workers") + 1]) if "--workers" in sys.argv else 8
    torch.cuda.set_device(0)
    fl = geometry.artery_flags((512, 512, 512), seed=0, r_root=40.0, r_min=14.0)
    st = make_stencil("d3q19")
    p = CollisionParams(1.7, "trt", trt_magic_lambda(1.7))
    fw = os.environ.get("FRAME", "halo")
    if os.environ.get("BLOCK_SWEEP"):  # the same tree in blocks of 512 / 256 / 128
        for b in (512, 256, 128):
            dom = Domain(fl, b, st, p, pattern="aa", frame_width=fw, device=0, check="deferred")
            measure(dom, f"full, blocks of {b}^3")
            del dom
            torch.cuda.empty_cache()
        return
    dom = Domain(fl, 128, st, p, pattern="aa", frame_width=fw, device=0, check="deferred")
    measure(dom, "full")
    asg = dom.balance(workers)
    keep = np.zeros(tuple(reversed(fl.dims)), dtype=bool)
    for bid, w in asg.items():
        if w == 0:
            x0, y0, z0 = dom.blocks[bid].origin
            keep[z0:z0 + 128, y0:y0 + 128, x0:x0 + 128] = True
    del dom
    torch.cuda.empty_cache()
    tags = fl.tags.copy()
    inner = tags[1:-1, 1:-1, 1:-1]
    inner[~keep & (inner == 0)] = 1  # other ranks' cells -> solid
    proxy = FlagField(fl.dims, tags, fl.ubb_u, fl.periodic)
    dom = Domain(proxy, 128, st, p, pattern="aa", frame_width=fw, device=0, check="deferred")
    measure(dom, f"share 1/{workers} (worker 0)")


if __name__ == "__main__":
    main()
