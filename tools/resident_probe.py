"""Resident multi-step kernel (k_resident) vs the per-step graph path on
small blocks: MFLUPS of engine.run(n) for packed beds of growing size, to
place the knob-4 cap.  Timed with a device synchronize on both sides of
engine.run (the whole n-step run is one or a few launches).

    python tools/resident_probe.py [--steps 400]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=400)
    args = ap.parse_args()
    import numpy as np

    from paper_2408_06880_b200 import _abi, geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    lib = _abi.load()
    for name, model in (("d3q19", "trt"), ("d3q27", "cumulant")):
        st = make_stencil(name)
        for n in ([32, 64, 96, 128, 160, 192] if name == "d3q19" else [64, 96, 128]):
            fl = geometry.packed_bed_flags((n, n, n), 0.5, n / 10.0, 1, channel=False)
            for pattern in ("aa", "pull"):
                if pattern == "pull" and name != "d3q19":
                    continue
                rec = {"stencil": name, "model": model, "pattern": pattern, "n": n}
                p = CollisionParams(1.2, model, 0.9 if model == "trt" else None)
                e = SparseEngine(fl, st, p, pattern, check="deferred")
                e.init_equilibrium()
                rec["n_fluid"] = e.n_fluid
                for label, cap in (("graph", 0), ("resident", 1 << 40)):
                    lib.slbm_set_tuning(4, int(min(cap, 2**31 - 1)))
                    e.run(8)
                    e.synchronize()
                    best = 1e9
                    for _ in range(3):
                        t0 = time.perf_counter()
                        e.run(args.steps)
                        e.synchronize()
                        best = min(best, time.perf_counter() - t0)
                    rec[label + "_us_per_step"] = round(best / args.steps * 1e6, 3)
                    rec[label + "_mflups"] = round(e.n_fluid * args.steps / best / 1e6, 1)
                rec["speedup"] = round(rec["graph_us_per_step"] / rec["resident_us_per_step"], 3)
                print(json.dumps(rec), flush=True)
                e.close()
    lib.slbm_set_tuning(4, 1 << 19)


if __name__ == "__main__":
    main()
