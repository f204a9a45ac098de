"""Temporally blocked AA pair (pair.cu) vs the per-step sweeps on the bench
workload (512^3 packed bed, porosity 0.3, D3Q19 TRT): MFLUPS of
engine.run over `--pairs` step pairs (CUDA events on the engine stream),
and whether the two paths end bit-identical.

    python tools/pair_probe.py [--edge 512] [--pairs 50] [--slack 0]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edge", type=int, default=512)
    ap.add_argument("--pairs", type=int, default=50)
    ap.add_argument("--slack", type=int, nargs="*", default=[0])
    ap.add_argument("--model", default="trt")
    ap.add_argument("--stencil", default="d3q19")
    ap.add_argument("--porosity", type=float, default=0.3)
    args = ap.parse_args()
    import hashlib

    import numpy as np
    import torch

    import bench
    from paper_2408_06880_b200 import _abi
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    lib = _abi.load()
    torch.cuda.set_device(0)
    st = make_stencil(args.stencil)
    p = CollisionParams(bench.OMEGA, args.model,
                        bench.magic_lambda(bench.OMEGA) if args.model == "trt" else None)
    if args.porosity == 0.3:
        fl = bench.make_flags(args.edge, 0)
    else:
        from paper_2408_06880_b200 import geometry

        fl = geometry.packed_bed_flags((args.edge,) * 3, args.porosity, bench.DIAMETER, bench.SEED,
                                       device=0)

    def timed(eng, pairs):
        s = torch.cuda.ExternalStream(eng.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        eng.run(2 * pairs)
        e1.record(s)
        e1.synchronize()
        return e0.elapsed_time(e1)

    def digest(eng):
        rho, u = eng.macroscopic_fields()
        return hashlib.sha256(rho.tobytes() + u.tobytes()).hexdigest()[:16]

    eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
    n = eng.n_fluid
    out = {"edge": args.edge, "n_fluid": n, "model": args.model, "stencil": args.stencil}
    bpc = {19: 680, 27: 968}[st.q]
    variants = [("per_step", 0, 0)] + [("pair", 1, sl) for sl in args.slack]
    for label, pair, slack in variants:
        lib.slbm_set_tuning(5, pair)
        if True:
            lib.slbm_set_tuning(6, slack)
            if pair and eng._h is not None:
                eng.close()
                eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
            eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
            timed(eng, 3)
            ms = timed(eng, args.pairs)
            key = label if not pair else f"pair_s{slack}"
            out[key + "_ms_per_pair"] = round(ms / args.pairs, 4)
            out[key + "_mflups"] = round(2 * n * args.pairs / (ms / 1e3) / 1e6, 1)
            out[key + "_algorithmic_gbs"] = round(bpc * n / (ms / args.pairs / 1e3) / 1e9, 1)
            # same start, 10 steps -> compare
            eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
            eng.run(10)
            out[key + "_digest"] = digest(eng)
            print(json.dumps(out), flush=True)
    lib.slbm_set_tuning(5, 0)
    lib.slbm_set_tuning(6, 0)


if __name__ == "__main__":
    main()
