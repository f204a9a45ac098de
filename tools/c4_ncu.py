"""C4 artery (512^3, 128^3 blocks, one block group, direct local halo edges)
for ncu: builds and warms the domain outside the profiled range, then runs
STEPS steps (default 4) between cudaProfilerStart/Stop, so

    ncu --profile-from-start off --metrics gpu__time_duration.sum ... python tools/c4_ncu.py
    ncu --profile-from-start off --set full -k regex:k_group ... python tools/c4_ncu.py

see only the step kernels (the bench's own c4 line: bench.py impl_artery).
Prints the total fluid cells (N_FLUID for tools/ncu_summary.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_06880_b200 import geometry  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda  # noqa: E402
from paper_2408_06880_b200.domain import Domain  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

torch.cuda.set_device(0)
steps = int(os.environ.get("STEPS", 4))
fl = geometry.artery_flags((512, 512, 512), seed=0, r_root=40.0, r_min=14.0)
st = make_stencil("d3q19")
p = CollisionParams(1.7, "trt", trt_magic_lambda(1.7))
dom = Domain(fl, 128, st, p, pattern="aa", frame_width="halo", device=0, check="deferred")
dom.init_equilibrium()
dom.run(12, driver="overlapped", use_graph=True)
dom.synchronize()
torch.cuda.profiler.start()
dom.run(steps, driver="overlapped", use_graph=True)
dom.synchronize()
torch.cuda.profiler.stop()
dom.poll()
print("N_FLUID", sum(e.n_fluid for e in dom.local_engines()), "blocks", len(dom.local_engines()))
