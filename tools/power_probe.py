"""Board power and SM clock while one sweep kind runs back to back on the
bench bed: the index-list (even) sweep repeated without finishing the step,
then the cell-local (odd) sweep the same way (the values are meaningless,
the traffic and instruction mix are the real ones).  Diagnostic for the
power-cap behaviour:  python tools/power_probe.py"""
import json
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
from paper_2408_06880_b200 import _abi  # noqa: E402

if os.environ.get("PROBE"):  # SLBM_PROBES=1 build: the even sweep's memory pattern only
    _abi.load().slbm_set_tuning(0, 2)
eng = SparseEngine(bench.make_flags(512, 0), st, p, "aa", device=0, check="deferred")
eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
eng.run(12, use_graph=False)
s = torch.cuda.ExternalStream(eng.stream())
out = {}
for kind in ("even", "odd", "even"):
    want = 0 if kind == "even" else 1
    if eng.parity.value != want:
        eng.step()
        eng.finish_step()
    samples, stop = [], False

    def sample():
        while not stop:
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True)
            samples.append([float(x) for x in r.stdout.strip().split(",")])
            time.sleep(0.05)

    th = threading.Thread(target=sample)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    th.start()
    a.record(s)
    n = 0
    t0 = time.time()
    while time.time() - t0 < 6.0:
        for _ in range(20):
            eng.step()  # same parity every time: the same kernel back to back
        n += 20
        torch.cuda.synchronize()
    b.record(s)
    b.synchronize()
    stop = True
    th.join()
    tail = samples[len(samples) // 2:]
    out[kind + ("2" if kind in out else "")] = {
        "ms_per_sweep": round(a.elapsed_time(b) / n, 4),
        "sm_mhz_median": statistics.median(x[0] for x in tail),
        "power_w_median": round(statistics.median(x[1] for x in tail), 1)}
print(json.dumps(out))
