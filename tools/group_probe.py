"""A/B of the block-group sweep (k_group, group.cu) against the single-engine
sweep (k_index_sweep / k_aa_odd, kernels.cu) on the SAME engine: one 512^3
block (artery tree by default, BED=1 for the bench bed) driven alternately
through slbm_group_step and slbm_step, CUDA events on the engine stream.

    python tools/group_probe.py
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2408_06880_b200 import geometry  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda  # noqa: E402
from paper_2408_06880_b200.domain import BlockGroup  # noqa: E402
from paper_2408_06880_b200.engine import SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402


def main():
    torch.cuda.set_device(0)
    st = make_stencil("d3q19")
    p = CollisionParams(1.7, "trt", trt_magic_lambda(1.7))
    if os.environ.get("BED"):
        fl = bench.make_flags(512, 0)
    else:
        fl = geometry.artery_flags((512,) * 3, seed=0, r_root=40.0, r_min=14.0)
    eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
    eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
    grp = BlockGroup([eng])
    s = torch.cuda.ExternalStream(eng.stream())
    n = eng.n_fluid
    res = {"group": {0: [], 1: []}, "engine": {0: [], 1: []}}
    for rep in range(int(os.environ.get("REPS", 12))):
        for how, _ in (("group", 0), ("group", 1), ("engine", 0), ("engine", 1)):
            par = eng.parity.value
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            eng.refresh_boundary(eng.parity)
            a.record(s)
            if how == "group":
                grp.step("all", eng.stream())
            else:
                eng.step()
            b.record(s)
            if how == "group":
                grp.finish(eng.stream())
            else:
                eng.finish_step()
            b.synchronize()
            res[how][par].append(a.elapsed_time(b))
    hbm = bench.peaks()[0]
    out = {"n_fluid": n}
    for how, d in res.items():
        for par, name, by in ((0, "even", 376), (1, "odd", 304)):
            ms = statistics.median(d[par])
            out[f"{how}_{name}_ms"] = round(ms, 4)
            out[f"{how}_{name}_frac"] = round(n * by / ms / 1e6 / hbm, 4)
    eng.poll()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
