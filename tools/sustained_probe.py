"""Per-step sweep times over a long back-to-back run (the bench's timed
loop) to see power-cap clock droop; prints means over windows of 20 steps
and nvidia-smi clock samples.  Tuning aid."""
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402

torch.cuda.set_device(0)
st = make_stencil("d3q19")
p = CollisionParams(bench.OMEGA, "trt", bench.magic_lambda(bench.OMEGA))
from paper_2408_06880_b200 import _abi  # noqa: E402

_abi.load().slbm_set_tuning(0, int(os.environ.get("VARIANT", 0)))
_abi.load().slbm_set_tuning(2, int(os.environ.get("AHEAD", 1)))  # idx prefetch, quarter waves
eng = SparseEngine(bench.make_flags(512, 0), st, p, "aa", device=0, check="deferred")
eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
eng.run(10)
steps = int(os.environ.get("STEPS", 600))
clocks = []
stop = False


def sample():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True)
        clocks.append(out.stdout.strip())
        time.sleep(0.05)


th = threading.Thread(target=sample)
th.start()
s = torch.cuda.ExternalStream(eng.stream())
evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
par = []
torch.cuda.synchronize()
evs[0].record(s)
for k in range(steps):
    par.append(eng.parity.value)
    eng.step()
    eng.finish_step()
    evs[k + 1].record(s)
evs[-1].synchronize()
stop = True
th.join()
per = [evs[k].elapsed_time(evs[k + 1]) for k in range(steps)]
win = []
for w in range(0, steps, 40):
    e = [t for t, q in zip(per[w:w + 40], par[w:w + 40]) if q == 0]
    o = [t for t, q in zip(per[w:w + 40], par[w:w + 40]) if q == 1]
    win.append((round(float(np.mean(e)), 4), round(float(np.mean(o)), 4)))
print(json.dumps({"variant": int(os.environ.get("VARIANT", 0)), "ahead": int(os.environ.get("AHEAD", 1)),
                  "mean_even_ms": round(float(np.mean([t for t, q in zip(per, par) if q == 0])), 4),
                  "mean_odd_ms": round(float(np.mean([t for t, q in zip(per, par) if q == 1])), 4),
                  "windows_even_odd_ms": win, "clock_samples": clocks[::4]}))
