"""One-GPU proxy for the weak-scaling step: the bench's 512^3 bed as one
block (plain engine) vs the same cells as z slabs driven by the overlapped
driver, with every halo edge a real NCCL message (loopback communicator) or
the device-local gather-scatter.  Shows what the exchange + split costs when
it is hidden behind the interior sweep.  Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.domain import Domain, DistributedDomain  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import torch.distributed as dist  # noqa: E402

dist.init_process_group("gloo", rank=0, world_size=1)
torch.cuda.set_device(0)
edge = int(os.environ.get("EDGE", bench.EDGE))
slabs = int(os.environ.get("SLABS", 2))
steps = int(os.environ.get("STEPS", 40))
st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
fl = bench.make_flags(edge, 0)
res = {"edge": edge, "slabs": slabs, "steps": steps}


def timed(run, stream, n):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    run(n)
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b)


eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
eng.run(4)
s = torch.cuda.ExternalStream(eng.stream())
ms = timed(eng.run, s, steps)
res["single_block_mflups"] = round(eng.n_fluid * steps / ms * 1e-3, 1)
n_fluid = eng.n_fluid
del eng
torch.cuda.empty_cache()

for name in ("local", "nccl_loopback", "p2p_loopback"):
    block = (edge, edge, edge // slabs)
    if name == "local":
        d = Domain(fl, block, st, p, pattern="aa", frame_width="halo", check="deferred")
    else:
        d = DistributedDomain(fl, block, st, p, pattern="aa", rank=0, world=1, device=0,
                              loopback=True, transport=name.split("_")[0])
    d.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
    d.run(4, driver="overlapped", use_graph=True)
    s = torch.cuda.ExternalStream(d.stream())
    ms = timed(lambda n: d.run(n, driver="overlapped", use_graph=True), s, steps)
    d.poll()
    res[f"{name}_overlapped_mflups"] = round(d.total_fluid() * steps / ms * 1e-3, 1)
    d.run(4, driver="sequential", use_graph=True)
    ms = timed(lambda n: d.run(n, driver="sequential", use_graph=True), s, steps)
    res[f"{name}_sequential_mflups"] = round(d.total_fluid() * steps / ms * 1e-3, 1)
    res[f"{name}_exchanged_values_per_step"] = int(
        sum(e.counters.values_exchanged for e in d.local_engines()) / max(d.steps_done, 1))
    del d
    torch.cuda.empty_cache()
# one block through the Domain (block-group kernels, no exchange)
d = Domain(fl, (edge, edge, edge), st, p, pattern="aa", frame_width="halo", check="deferred")
d.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
d.run(4, driver="overlapped", use_graph=True)
s = torch.cuda.ExternalStream(d.stream())
ms = timed(lambda n: d.run(n, driver="overlapped", use_graph=True), s, steps)
res["one_block_domain_mflups"] = round(d.total_fluid() * steps / ms * 1e-3, 1)
del d
torch.cuda.empty_cache()

if os.environ.get("KERNELS"):
    # per-kernel device time of the slab domain's overlapped step (CUPTI)
    from torch.profiler import ProfilerActivity, profile

    d = Domain(fl, (edge, edge, edge // slabs), st, p, pattern="aa", frame_width="halo",
               check="deferred")
    d.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
    d.run(2, driver="overlapped")
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        d.run(4, driver="overlapped")
        torch.cuda.synchronize()
    agg = {}
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            k = ev.name.replace("(anonymous namespace)::", "").split("(")[0][:90]
            agg.setdefault(k, [0, 0.0])
            agg[k][0] += 1
            agg[k][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    res["kernels_4_steps_us"] = {k: [n, round(t, 1)] for k, (n, t) in
                                 sorted(agg.items(), key=lambda kv: -kv[1][1])}
res["n_fluid"] = n_fluid
print(json.dumps(res))
