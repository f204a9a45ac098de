"""Measure BASELINE.json configs other than the headline (which bench.py owns)
on one B200 and print one JSON line per measurement.

    python tools/bench_configs.py [c1] [c3] [c3h] [c4] [c5] [--steps K]

c1  D3Q19 SRT, 64^3 periodic channel, overlapping-sphere bed porosity ~0.5,
    100 steps, pull and AA: GPU MFLUPS, bitwise parity with the reference's
    golden (SHA-256 of the final state), and the reference algorithm (oracle
    port) timed on the same full problem on this host.
c3  D3Q27 cumulant, 512^3 per GPU: particle bed (porosity ~0.35) in the lower
    half, free flow above, periodic x/y, no-slip floor, moving lid (N = 1
    here; the weak-scaling series runs through bench.py's DistributedDomain).
c3h the paper's hybrid riverbed: the C3 riverbed (D3Q19 TRT) in 128^3 blocks
    under the sparse, dense and hybrid layout policies (MFLUPS, memory).
c4  vessel-like branching tube tree, ~5% fluid, 512^3 box cut into 128^3
    blocks (empty blocks dropped), D3Q19 TRT, UBB inlet + fixed-density
    outlets; Domain on one GPU with the whole step pair captured as one CUDA
    graph (the strong-scaling baseline point).
c5  porosity sweep at 384^3 (cell-wise random obstacles, reference
    obstacle_flags), D3Q19 TRT AA: sparse MFLUPS vs the dense-equivalent
    roofline (304 B per cell update, model.py) and device memory vs the
    reference memory model (model.py:106-126).
"""

import hashlib
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2408_06880_b200 import geometry  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda  # noqa: E402
from paper_2408_06880_b200.engine import DenseEngine, SparseEngine  # noqa: E402
from paper_2408_06880_b200.lattice import make_stencil  # noqa: E402
from paper_2408_06880_b200.tags import PERIODIC, WALL, FaceKind, FaceSpec, make_flags  # noqa: E402

HBM = bench.peaks()[0]


def emit(d):
    print(json.dumps(d), flush=True)


def timed_run(eng, steps):
    stream = torch.cuda.ExternalStream(eng.stream())
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    eng.run(steps)
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b)


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def c1():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle.sparse_ref import OracleSparseEngine
    from test_oracle_golden import init_random_values

    for pattern in ("aa", "pull"):
        rec = dict(np.load(os.path.join(ROOT, "tests", "golden", f"bed_c1_64_srt_{pattern}.npz")))
        dims = (64, 64, 64)
        d = float(rec["diameter"])
        centers = geometry.sphere_centers(dims, d, int(rec["count"]), int(rec["seed"]))
        fl = geometry.channel_flags(dims, solid=geometry.voxelize_spheres(dims, centers, d, 0))
        st = make_stencil("d3q19")
        p = CollisionParams(1.2)
        eng = SparseEngine(fl, st, p, pattern, device=0, check="deferred")
        v0 = init_random_values(fl, st, eng, seed=7)
        eng.init_canonical(v0)
        eng.run(2)  # capture the step-pair graph outside the timed region
        eng.init_canonical(v0)
        ms = timed_run(eng, 100)
        eng.poll()
        ok = sha(eng.canonical_state()) == str(rec["final_sha"])
        # the same 100 steps with the reference algorithm on the host
        cpu = OracleSparseEngine(fl, st, p, pattern)
        cpu.init_canonical(v0)
        t0 = time.perf_counter()
        for _ in range(100):
            cpu.refresh_boundary(cpu.parity)
            cpu.step()
            cpu.finish_step()
        cpu_s = time.perf_counter() - t0
        cpu_ok = sha(cpu.canonical_state()) == str(rec["final_sha"])
        emit({"config": "c1", "pattern": pattern, "n_fluid": eng.n_fluid,
              "porosity": round(eng.n_fluid / 64**3, 4), "steps": 100,
              "gpu_mflups": round(eng.n_fluid * 100 / ms * 1e3 / 1e6, 1),
              "gpu_ms": round(ms, 3), "bitwise_equal_reference_golden": ok,
              "cpu_reference_mflups": round(eng.n_fluid * 100 / cpu_s / 1e6, 3),
              "cpu_reference_bitwise": cpu_ok, "cpu_cores": 1,
              "note": "GPU timed via engine.run: one resident cooperative launch for all steps (k_resident)"})


def c3(steps):
    edge = 512
    dims = (edge, edge, edge)
    st = make_stencil("d3q27")
    # particle bed in the lower half (porosity ~0.35), free flow above
    d = 16.0
    half = (edge, edge, edge // 2)
    n = geometry.overlapping_sphere_count(half, d, 0.35)
    centers = geometry.sphere_centers(half, d, n, 3)
    solid = geometry.voxelize_spheres(dims, centers, d, 0)
    lid = FaceSpec(FaceKind.WALL, velocity=(0.02, 0.0, 0.0))
    fl = make_flags(dims, [(PERIODIC, PERIODIC), (PERIODIC, PERIODIC), (WALL, lid)], solid=solid)
    for model in ("cumulant", "trt"):
        p = CollisionParams(1.6, model, trt_magic_lambda(1.6) if model == "trt" else None)
        eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
        eng.init_equilibrium(1.0, np.array([0.0, 0.0, 0.0]))
        eng.run(4)
        ms = timed_run(eng, steps)
        eng.poll()
        _, te, to = bench.timed_steps(eng, 20, torch, torch.cuda.ExternalStream(eng.stream()))
        be, bo = 2 * 27 * 8 + 26 * 4, 2 * 27 * 8
        nf = eng.n_fluid
        emit({"config": "c3", "model": model, "n_fluid": nf, "porosity": round(nf / edge**3, 4),
              "steps": steps, "mflups": round(nf * steps / ms * 1e3 / 1e6, 1),
              "even_frac": round(nf * be / te / 1e6 / HBM, 4),
              "odd_frac": round(nf * bo / to / 1e6 / HBM, 4),
              "pair_frac": round(nf * (be + bo) / (te + to) / 1e6 / HBM, 4),
              "n_ubb_slots": eng.n_ubb_slots, "device_gb": round(eng.device_bytes / 1e9, 2),
              "note": "D3Q27 AA 512^3/GPU, bed lower half + free flow, moving lid"})
        del eng


def c3h(steps):
    """The paper's hybrid riverbed on one GPU: the C3
    riverbed (D3Q19 TRT here) cut into 128^3 blocks, run with the sparse,
    dense and hybrid layout policies (hybrid: dense at block porosity >=
    phi_s = 0.8, domain.py:58-65).  All three give the same bits."""
    from paper_2408_06880_b200.domain import Domain

    edge = 512
    dims = (edge, edge, edge)
    d = 16.0
    half = (edge, edge, edge // 2)
    n = geometry.overlapping_sphere_count(half, d, 0.35)
    solid = geometry.voxelize_spheres(dims, geometry.sphere_centers(half, d, n, 3), d, 0)
    lid = FaceSpec(FaceKind.WALL, velocity=(0.02, 0.0, 0.0))
    fl = make_flags(dims, [(PERIODIC, PERIODIC), (PERIODIC, PERIODIC), (WALL, lid)], solid=solid)
    st = make_stencil("d3q19")
    p = CollisionParams(1.6, "trt", trt_magic_lambda(1.6))
    sums = {}
    for policy in ("sparse", "dense", "hybrid"):
        dom = Domain(fl, 128, st, p, pattern="aa", policy=policy, frame_width=1, device=0,
                     check="deferred")
        dom.init_equilibrium()
        dom.run(4, driver="overlapped", use_graph=True)
        stream = torch.cuda.ExternalStream(dom.stream())
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        dom.run(steps, driver="overlapped", use_graph=True)
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b)
        dom.poll()
        rho, _ = dom.gather_macroscopics()
        sums[policy] = float(np.abs(rho).sum())
        kinds = [blk.kind for blk in dom.blocks.values()]
        nf = dom.total_fluid()
        emit({"config": "c3h", "policy": policy, "n_fluid": nf, "blocks": len(kinds),
              "dense_blocks": kinds.count("dense"), "steps": steps,
              "mflups": round(nf * steps / ms * 1e3 / 1e6, 1),
              "device_gb": round(sum(e.device_bytes for e in dom.local_engines()) / 1e9, 2),
              "rho_abs_sum": sums[policy]})
        del dom
        torch.cuda.empty_cache()
    assert len(set(sums.values())) == 1, sums


def c4(steps):
    from paper_2408_06880_b200.domain import Domain

    edge, block = 512, 128
    t0 = time.perf_counter()
    fl = geometry.artery_flags((edge, edge, edge), seed=0, r_root=40.0, r_min=14.0)
    gen_s = time.perf_counter() - t0
    st = make_stencil("d3q19")
    p = CollisionParams(1.7, "trt", trt_magic_lambda(1.7))
    t0 = time.perf_counter()
    dom = Domain(fl, block, st, p, pattern="aa", frame_width=1, device=0, check="deferred")
    build_s = time.perf_counter() - t0
    dom.init_equilibrium()
    dom.run(4, driver="overlapped", use_graph=True)
    dom.synchronize()
    stream = torch.cuda.ExternalStream(dom.stream())
    out = {}
    for use_graph in (True, False):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        a.record(stream)
        dom.run(steps, driver="overlapped", use_graph=use_graph)
        b.record(stream)
        b.synchronize()
        wall = time.perf_counter() - t
        out[use_graph] = (a.elapsed_time(b), wall)
    dom.poll()
    nf = dom.total_fluid()
    rho, _ = dom.gather_macroscopics()
    emit({"config": "c4", "n_fluid": nf, "fluid_fraction": round(nf / edge**3, 4),
          "blocks": len(dom.blocks), "block": block, "edges": len(dom.edge_plans), "steps": steps,
          "mflups_graph": round(nf * steps / out[True][0] * 1e3 / 1e6, 1),
          "mflups_python_driver": round(nf * steps / (out[False][1] * 1e3) * 1e3 / 1e6, 1),
          "geometry_s": round(gen_s, 1), "build_s": round(build_s, 1),
          "mean_density_fluid": float(rho[fl.tags_interior == 0].mean()),
          "note": "one GPU, all blocks local; overlapped driver; strong-scaling baseline"})


def c5(steps):
    edge = 384
    st = make_stencil("d3q19")
    p = CollisionParams(1.2, "trt", trt_magic_lambda(1.2))
    dense_bpc = 304.0  # D3Q19 dense AA, GPU (reference model.py, test_acceptance.py:89-98)
    phis = os.environ.get("C5_PHIS", "0.05,0.1,0.2,0.3,0.4,0.5,0.6,0.7,0.8,0.9,1.0")
    for phi in (float(v) for v in phis.split(",")):
        fl = geometry.obstacle_flags((edge,) * 3, phi, 1)
        eng = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
        eng.init_equilibrium(1.0, np.array([0.005, 0.0, 0.0]))
        eng.run(12)  # the occupancy trials (kernels.cu sweep_ctas) end before timing
        ms = timed_run(eng, steps)
        eng.poll()
        nf = eng.n_fluid
        mfl = nf * steps / ms * 1e3 / 1e6
        # per-kernel: the reference loop with an event after every step
        stream = torch.cuda.ExternalStream(eng.stream())
        _, te, to = bench.timed_steps(eng, max(20, min(steps, 200)), torch, stream)
        even_frac = nf * bench.BYTES_EVEN / (te / 1e3) / 1e9 / HBM
        odd_frac = nf * bench.BYTES_ODD / (to / 1e3) / 1e9 / HBM
        sparse_bytes = eng.device_bytes
        ctas = eng.sweep_ctas
        del eng
        # measured dense (direct-addressing) engine on the same geometry
        den = DenseEngine(fl, st, p, "aa", device=0, check="deferred")
        den.init_equilibrium(1.0, np.array([0.005, 0.0, 0.0]))
        den.run(2)
        ms_d = timed_run(den, steps)
        den.poll()
        mfl_d = nf * steps / ms_d * 1e3 / 1e6
        dense_bytes = den.device_bytes
        del den
        dense_equiv = HBM * 1e9 / dense_bpc * phi / 1e6
        model_bytes = edge**3 * (19 * 8 + 18 * 4 + 5 * 8) * phi
        emit({"config": "c5", "porosity": phi, "n_fluid": nf, "mflups": round(mfl, 1),
              "sweep_ctas_per_sm": ctas,
              "dense_mflups_measured": round(mfl_d, 1),
              "dense_equivalent_mflups_model": round(dense_equiv, 1),
              "sparse_over_dense_measured": round(mfl / mfl_d, 3),
              "pair_frac": round(mfl * 1e6 * 340 / (HBM * 1e9), 4),
              "even_frac": round(even_frac, 4), "odd_frac": round(odd_frac, 4),
              "ms_even": round(te, 4), "ms_odd": round(to, 4),
              "device_bytes": sparse_bytes, "dense_device_bytes": dense_bytes,
              "model_memory_bytes": int(model_bytes),
              "device_bytes_per_fluid_cell": round(sparse_bytes / nf, 1)})


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    steps = 40
    if "--steps" in sys.argv:
        steps = int(sys.argv[sys.argv.index("--steps") + 1])
        args = [a for a in args if a != str(steps)]
    which = args or ["c1", "c3", "c4", "c5"]
    torch.cuda.set_device(0)
    for w in which:
        {"c1": lambda: c1(), "c3": lambda: c3(steps), "c3h": lambda: c3h(steps),
         "c4": lambda: c4(steps), "c5": lambda: c5(steps)}[w]()


if __name__ == "__main__":
    main()
