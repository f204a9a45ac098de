"""Domain.gather_macroscopics wall time on the C4 artery (global box
assembled on the device + staged copies) and the host copy / fill costs
beside it.  Tuning aid:  python tools/gather_probe.py"""
import os, sys, time, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2408_06880_b200 import geometry, _abi
from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda
from paper_2408_06880_b200.domain import Domain
from paper_2408_06880_b200.lattice import make_stencil
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
fl = geometry.artery_flags((512,) * 3, seed=0, r_root=40.0, r_min=14.0)
dom = Domain(fl, 128, make_stencil("d3q19"), CollisionParams(1.7, "trt", trt_magic_lambda(1.7)), pattern="aa", frame_width="halo", check="deferred")
dom.init_equilibrium(); dom.run(2, use_graph=True); dom.synchronize()
for k in range(3):
    t = time.perf_counter(); rho, u = dom.gather_macroscopics(); t1 = time.perf_counter()
    print("gather", round(t1 - t, 3))
t = time.perf_counter(); a = np.empty((512, 512, 512, 3)); a.fill(0); print("host fill 3.2GB", round(time.perf_counter() - t, 3))
d = torch.zeros(512**3 * 3, dtype=torch.float64, device="cuda"); torch.cuda.synchronize()
import ctypes as C
b = np.empty((512, 512, 512, 3))
t = time.perf_counter(); _abi.call("slbm_copy_to_host", _abi.ptr(b, C.c_double), C.c_void_p(d.data_ptr()), b.nbytes, 0); print("copy fresh", round(time.perf_counter() - t, 3))
t = time.perf_counter(); _abi.call("slbm_copy_to_host", _abi.ptr(b, C.c_double), C.c_void_p(d.data_ptr()), b.nbytes, 0); print("copy touched", round(time.perf_counter() - t, 3))
