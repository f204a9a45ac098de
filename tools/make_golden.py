"""Generate tests/golden/*.npz by running the UNMODIFIED reference package.

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py

The reference is imported read-only from /root/reference/pkg/src (nothing
is copied into this repo).  Every fixture stores the exact inputs (tag box,
wall velocities, periodic flags, stencil, collision, pattern, initial
state) and the reference's outputs (index lists, slot tables, states after
N steps, macroscopic fields, EdgePlan slot lists, multi-block gathers), so
tests on the GPU box — where the reference is absent — can check the CUDA
engine and the oracle bit for bit.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _ref():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import slbm  # noqa: F401
    from slbm import core, domain, exchange, flags, geometry, sparse, stencil

    return core, domain, exchange, flags, geometry, sparse, stencil


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def seed_values(fl, st, seed, core, amplitude=0.01):
    """conftest.py:29-60 seed_state (values part)."""
    rng = np.random.default_rng(seed)
    shape = tuple(reversed(fl.dims))
    rho = 1.0 + amplitude * rng.standard_normal(shape)
    u = amplitude * rng.standard_normal((st.dim,) + shape)
    mask = fl.tags_interior == 0
    return core.equilibrium_fields(rho[mask], u.reshape(st.dim, -1)[:, mask.reshape(-1)], st)


def drive(eng, steps, ghost_slot=None, ghost_fill=None):
    """conftest.py:38-43; halo slots (if any) get fixed values before every
    step, standing in for a neighbour's canonical exchange."""
    for _ in range(steps):
        if ghost_slot is not None and ghost_slot.size:
            eng.write_slots(ghost_slot, ghost_fill)
        eng.refresh_boundary(eng.parity)
        eng.step()
        eng.finish_step()


def engine_case(name, fl, stname, model, omega, lam, steps_list, seed=11, frame_width=1):
    core, domain, exchange, flags, geometry, sparse, stencil = _ref()
    st = stencil.make_stencil(stname)
    p = core.CollisionParams(omega=omega, model=model, lambda_odd=lam)
    values = seed_values(fl, st, seed, core)
    rec = {
        "kind": np.array("engine"),
        "stencil": np.array(stname),
        "model": np.array(model),
        "omega": np.array(omega),
        "lambda_odd": np.array(lam if lam is not None else np.nan),
        "dims": np.array(fl.dims),
        "tags": fl.tags,
        "ubb_u": fl.ubb_u,
        "periodic": np.array(fl.periodic),
        "values0": values,
        "frame_width": np.array(frame_width),
    }
    eng = sparse.SparseEngine(fl, st, p, pattern="aa", frame_width=frame_width)
    rec["idx"] = eng.idx
    rec["base"] = eng.base
    rec["fluid_coords"] = eng.fluid_coords
    rec["ubb_slots"] = eng._ubb_slots
    rec["ubb_partner"] = eng._ubb_partner
    rec["ubb_corr"] = eng._ubb_corr
    items = sorted(eng._ghost_slots.items(), key=lambda kv: kv[1])
    rec["ghost_q"] = np.array([k[0] for k, _ in items], dtype=np.int64)
    rec["ghost_pflat"] = np.array([k[1] for k, _ in items], dtype=np.int64)
    rec["ghost_slot"] = np.array([v for _, v in items], dtype=np.int64)
    rec["interior"] = eng._cols["interior"]
    rec["frame"] = eng._cols["frame"]
    rec["total_slots"] = np.array(eng.total_slots)
    gq = rec["ghost_q"]
    ghost_fill = st.w[gq] * (1.0 + 0.001 * ((rec["ghost_slot"] * 37) % 11))
    rec["ghost_fill"] = ghost_fill
    for pattern in ("pull", "aa"):
        for steps in steps_list:
            e = sparse.SparseEngine(fl, st, p, pattern=pattern)
            e.init_canonical(values)
            drive(e, steps, rec["ghost_slot"], ghost_fill)
            rec[f"{pattern}_{steps}_state"] = e.canonical_state()
            rho, u = e.macroscopic_fields()
            rec[f"{pattern}_{steps}_rho"] = rho
            rec[f"{pattern}_{steps}_u"] = u
    rec["steps_list"] = np.array(steps_list)
    np.savez_compressed(os.path.join(OUT, f"engine_{name}.npz"), **rec)
    print("engine", name, "n_fluid", eng.n_fluid, "slots", eng.total_slots,
          "ubb", eng.n_ubb_slots, "ghost", eng.n_ghost_slots)


def domain_case(name, gf, block, stname, model, omega, lam, steps, seed=11, patterns=("pull", "aa")):
    core, domain, exchange, flags, geometry, sparse, stencil = _ref()
    st = stencil.make_stencil(stname)
    p = core.CollisionParams(omega=omega, model=model, lambda_odd=lam)
    rec = {
        "kind": np.array("domain"),
        "stencil": np.array(stname),
        "model": np.array(model),
        "omega": np.array(omega),
        "lambda_odd": np.array(lam if lam is not None else np.nan),
        "dims": np.array(gf.dims),
        "tags": gf.tags,
        "ubb_u": gf.ubb_u,
        "periodic": np.array(gf.periodic),
        "block": np.array(block),
        "seed": np.array(seed),
        "steps": np.array(steps),
    }
    for pattern in patterns:
        d = domain.Domain(gf, block, st, p, pattern=pattern, frame_width=1)
        d.init_random(seed)
        rec[f"{pattern}_init"] = d.gather_canonical()
        # EdgePlan slot lists (exchange.py:148-219), in edge order
        plans = []
        for plan in d.edge_plans:
            for ph, pp in plan.phases.items():
                plans.append((plan.src_bid, plan.dst_bid, plan.sigma, ph.value, pp))
        rec[f"{pattern}_edges"] = np.array(
            [[a, b, *sig, ph, pp.n_wire, len(pp.tgt_sel)] for a, b, sig, ph, pp in plans],
            dtype=np.int64,
        )
        rec[f"{pattern}_send"] = np.concatenate([pp.send_sel for *_, pp in plans]).astype(np.int64)
        rec[f"{pattern}_take"] = np.concatenate([pp.pos_from_sparse for *_, pp in plans]).astype(np.int64)
        rec[f"{pattern}_tgt"] = np.concatenate([pp.tgt_sel for *_, pp in plans]).astype(np.int64)
        d.run(steps, driver="overlapped")
        rec[f"{pattern}_final"] = d.gather_canonical()
        rho, u = d.gather_macroscopics()
        rec[f"{pattern}_rho"] = rho
        rec[f"{pattern}_u"] = u
        c = d.counters()
        rec[f"{pattern}_counters"] = np.array(
            [c.steps, c.cells_visited, c.cells_visited_interior, c.cells_visited_frame,
             c.pdf_accesses, c.idx_reads, c.values_exchanged, c.messages], dtype=np.int64)
        rec[f"{pattern}_blocks"] = np.array(sorted(d.blocks), dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, f"domain_{name}.npz"), **rec)
    print("domain", name, "blocks", len(d.blocks), "edges", len(d.edge_plans))


def bed_case(name, dims, porosity, diameter, seed, stname, model, omega, lam, steps, pattern,
             channel=True):
    """Larger packed bed: the geometry is regenerated from the recorded
    sphere centres (overlapping) through the reference voxelize; outputs
    are hashes + per-direction sums + sampled values (fixtures stay small)."""
    core, domain, exchange, flags, geometry, sparse, stencil = _ref()
    import math

    st = stencil.make_stencil(stname)
    p = core.CollisionParams(omega=omega, model=model, lambda_odd=lam)
    # Boolean model with centres drawn over the box grown by one radius per
    # side, so the bed is statistically uniform up to the faces
    vol = math.pi * diameter**3 / 6.0
    grown = np.asarray(dims, dtype=np.float64) + diameter
    count = int(round(-math.log(porosity) * float(np.prod(grown)) / vol))
    rng = np.random.default_rng(seed)
    centers = rng.random((count, 3)) * grown - diameter / 2.0
    pack = geometry.SpherePack(tuple(float(d) for d in dims), diameter, centers, seed)
    mask = geometry.voxelize(pack)
    if channel:
        fl = geometry.mask_flags(mask)
    else:
        P = flags.FaceSpec(flags.FaceKind.PERIODIC)
        fl = flags.make_flags(dims, [(P, P)] * 3, solid=mask.solid)
    rng2 = np.random.default_rng(seed + 1)
    d = domain.Domain(fl, dims, st, p, pattern=pattern)
    d.init_random(7)
    eng = d.blocks[0].engine
    values0 = eng.canonical_state()
    d.run(steps)
    final = eng.canonical_state()
    rho, u = eng.macroscopic_fields()
    sample_q = rng2.integers(0, st.q, 2000)
    sample_c = rng2.integers(0, eng.n_fluid, 2000)
    rec = {
        "kind": np.array("bed"),
        "stencil": np.array(stname),
        "model": np.array(model),
        "omega": np.array(omega),
        "lambda_odd": np.array(lam if lam is not None else np.nan),
        "dims": np.array(dims),
        "porosity_target": np.array(porosity),
        "diameter": np.array(diameter),
        "seed": np.array(seed),
        "count": np.array(count),
        "channel": np.array(channel),
        "pattern": np.array(pattern),
        "steps": np.array(steps),
        "solid_sha": np.array(sha(mask.solid.astype(np.uint8))),
        "tags_sha": np.array(sha(fl.tags)),
        "n_fluid": np.array(eng.n_fluid),
        "idx_sha": np.array(sha(eng.idx)),
        "values0_sha": np.array(sha(values0)),
        "final_sha": np.array(sha(final)),
        "rho_sha": np.array(sha(rho)),
        "u_sha": np.array(sha(u)),
        "final_sums": np.array([math.fsum(r) for r in final]),
        "sample_q": sample_q,
        "sample_c": sample_c,
        "sample_v": final[sample_q, sample_c],
        "mass0": np.array(math.fsum(values0.ravel())),
        "mass": np.array(math.fsum(final.ravel())),
    }
    np.savez_compressed(os.path.join(OUT, f"bed_{name}.npz"), **rec)
    print("bed", name, "n_fluid", eng.n_fluid, "porosity", eng.n_fluid / np.prod(dims))


def main():
    os.makedirs(OUT, exist_ok=True)
    core, domain, exchange, flags, geometry, sparse, stencil = _ref()
    FK, FS = flags.FaceKind, flags.FaceSpec
    P, W = FS(FK.PERIODIC), FS(FK.WALL)

    def lid_obstacle(dims=(12, 8), porosity=0.85, u_wall=0.04, seed=3):
        lid = FS(FK.WALL, velocity=(u_wall,) + (0.0,) * (len(dims) - 1))
        faces = [(P, P)] * (len(dims) - 1) + [(W, lid)]
        return flags.make_flags(dims, faces, solid=geometry.random_obstacles(dims, porosity, seed))

    trt = core.omega_from_viscosity(1 / 6)  # = 1.0
    lam316 = 1.0 / (3.0 / 16.0 / (1.0 / 1.2 - 0.5) + 0.5)
    # the reference's test CASES (tests/test_dense.py:14-25)
    engine_case("d2q9_lid", lid_obstacle(), "d2q9", "srt", 1.5, None, [4, 5])
    engine_case("d2q9_channel",
                geometry.channel_flags((10, 6), solid=geometry.random_obstacles((10, 6), 0.8, 8)),
                "d2q9", "srt", 1.5, None, [4, 5])
    engine_case("d3q19_periodic", geometry.obstacle_flags((6, 5, 4), 0.7, 5), "d3q19", "srt", 1.5,
                None, [4, 5])
    engine_case("d3q27_walled", geometry.obstacle_flags((5, 4, 4), 0.8, 9, periodic=False),
                "d3q27", "srt", 1.5, None, [4, 5])
    # TRT + moving lid (UBB) in 3-d
    engine_case("d3q19_couette_trt", geometry.riverbed_flags((8, 6, 8), (4, 3, 4), 0.5, 2, 0.05),
                "d3q19", "trt", 1.2, lam316, [6, 7])
    engine_case("d3q27_couette_trt", geometry.riverbed_flags((6, 6, 6), (3, 3, 3), 0.6, 4, 0.04),
                "d3q27", "trt", 1.3, 0.9, [4, 5])
    engine_case("d3q19_obstacles_trt", geometry.obstacle_flags((9, 7, 6), 0.6, 12), "d3q19", "trt",
                1.7, 1.1, [10, 11])
    # a partitioned block: EXCHANGE ghosts with in-block periodic wrap (F9)
    gf = geometry.obstacle_flags((8, 6, 5), 0.75, 21)
    dom = domain.Domain(gf, (4, 6, 5), stencil.make_stencil("d3q19"), core.CollisionParams(1.0))
    blk = dom.blocks[0]
    engine_case("d3q19_ghost_block", blk.flags, "d3q19", "srt", 1.3, None, [2, 3])
    gf2 = geometry.riverbed_flags((12, 8), (4, 4), 0.6, 5, 0.03)
    dom2 = domain.Domain(gf2, (4, 8), stencil.make_stencil("d2q9"), core.CollisionParams(1.0))
    engine_case("d2q9_ghost_block", dom2.blocks[1].flags, "d2q9", "trt", 1.4, 0.8, [2, 3])
    gf3 = geometry.obstacle_flags((6, 6, 6), 0.8, 33)
    dom3 = domain.Domain(gf3, (3, 6, 3), stencil.make_stencil("d3q27"), core.CollisionParams(1.0))
    engine_case("d3q27_ghost_block", dom3.blocks[2].flags, "d3q27", "srt", 1.1, None, [2, 3])

    # multi-block domains (decomposition + exchange + overlapped driver)
    domain_case("d2q9_riverbed", geometry.riverbed_flags((16, 16), (8, 8), 0.5, 3), (8, 8), "d2q9",
                "srt", 1.2, None, 6)
    domain_case("d3q19_2x2x2", geometry.obstacle_flags((8, 8, 8), 0.7, 4), (4, 4, 4), "d3q19",
                "trt", 1.2, lam316, 6)
    domain_case("d3q27_riverbed", geometry.riverbed_flags((8, 8, 8), (4, 4, 4), 0.6, 7, 0.03),
                (4, 8, 4), "d3q27", "srt", 1.4, None, 4)
    domain_case("d3q19_walled_strips", geometry.obstacle_flags((9, 6, 4), 0.8, 2, periodic=False),
                (3, 6, 2), "d3q19", "srt", 1.0, None, 5)

    # C1: 64^3 periodic channel, overlapping spheres d=8, porosity ~0.5, D3Q19 SRT, 100 steps
    bed_case("c1_64_srt_aa", (64, 64, 64), 0.5, 8.0, 42, "d3q19", "srt", 1.2, None, 100, "aa")
    bed_case("c1_64_srt_pull", (64, 64, 64), 0.5, 8.0, 42, "d3q19", "srt", 1.2, None, 100, "pull")
    # C2 law at reduced size: fully periodic bed porosity ~0.3, D3Q19 TRT AA
    bed_case("c2_48_trt_aa", (48, 48, 48), 0.3, 16.0 * 48 / 512 * 4, 5, "d3q19", "trt", 1.2, lam316,
             20, "aa", channel=False)
    print("trt magic lambda", lam316, trt)


def _state_digest(prefix, arr, mask_flat, rng, n_sample=4000):
    """SHA-256 + per-direction fsums + sampled values of a (q,)+box array
    (zeros at non-fluid cells) at random fluid positions."""
    import math

    q = arr.shape[0]
    flat = arr.reshape(q, -1)
    cells = np.flatnonzero(mask_flat)
    sq = rng.integers(0, q, n_sample)
    sc = cells[rng.integers(0, cells.size, n_sample)]
    return {
        f"{prefix}_sha": np.array(sha(arr)),
        f"{prefix}_sums": np.array([math.fsum(r) for r in flat]),
        f"{prefix}_sample_q": sq,
        f"{prefix}_sample_cell": sc,
        f"{prefix}_sample_v": flat[sq, sc],
    }


def config_domain_case(name, fl, block, stname, model, omega, lam, steps, recipe, seed=7,
                       pattern="aa", driver="overlapped", workers=8):
    """BASELINE config at reduced scale through the reference's own Domain
    (domain.py:69-268) and driver (exchange.py:330-374).  ``recipe`` records
    how the geometry is rebuilt on the GPU box (tests/test_gpu_configs.py);
    the tag box itself is pinned by its SHA.  Outputs are digests."""
    import math

    core, domain, exchange, flags, geometry, sparse, stencil = _ref()
    st = stencil.make_stencil(stname)
    p = core.CollisionParams(omega=omega, model=model, lambda_odd=lam)
    d = domain.Domain(fl, block, st, p, pattern=pattern, frame_width=1)
    d.init_random(seed)
    rng = np.random.default_rng(12345)
    mask = (fl.tags[tuple(slice(1, -1) for _ in fl.dims)] == 0).reshape(-1)
    rec = {
        "kind": np.array("config_domain"),
        "stencil": np.array(stname),
        "model": np.array(model),
        "omega": np.array(omega),
        "lambda_odd": np.array(lam if lam is not None else np.nan),
        "dims": np.array(fl.dims),
        "periodic": np.array(fl.periodic),
        "block": np.array(block),
        "seed": np.array(seed),
        "steps": np.array(steps),
        "pattern": np.array(pattern),
        "driver": np.array(driver),
        "recipe": np.array(json_dumps(recipe)),
        "tags_sha": np.array(sha(fl.tags)),
        "ubb_sha": np.array(sha(np.where((fl.tags == 2)[..., None], fl.ubb_u, 0.0))),
        "n_fluid": np.array(d.total_fluid()),
        "blocks": np.array(sorted(d.blocks), dtype=np.int64),
        "block_fluid": np.array([d.blocks[b].n_fluid for b in sorted(d.blocks)], dtype=np.int64),
        "n_edges": np.array(len(d.edge_plans)),
        "edge_wire": np.array([sum(pp.n_wire for pp in pl.phases.values()) for pl in d.edge_plans],
                              dtype=np.int64),
    }
    if workers and len(d.blocks) > 1:
        asg = d.balance(workers)
        rec["balance_bids"] = np.array(sorted(asg), dtype=np.int64)
        rec["balance_workers"] = np.array([asg[b] for b in sorted(asg)], dtype=np.int64)
    rec.update(_state_digest("init", d.gather_canonical(), mask, rng))
    d.run(steps, driver=driver)
    final = d.gather_canonical()
    rec.update(_state_digest("final", final, mask, rng))
    rec["mass"] = np.array(math.fsum(final.ravel()))
    rho, u = d.gather_macroscopics()
    rec["rho_sha"] = np.array(sha(rho))
    rec["u_sha"] = np.array(sha(u))
    c = d.counters()
    rec["counters"] = np.array(
        [c.steps, c.cells_visited, c.cells_visited_interior, c.cells_visited_frame,
         c.pdf_accesses, c.idx_reads, c.values_exchanged, c.messages], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, f"config_{name}.npz"), **rec)
    print("config", name, "n_fluid", d.total_fluid(), "blocks", len(d.blocks),
          "edges", len(d.edge_plans), flush=True)


def config_engine_case(name, fl, stname, model, omega, lam, steps, recipe, seed=11,
                       layouts=("sparse", "dense"), patterns=("aa", "pull")):
    """One block through the reference's SparseEngine / DenseEngine
    (sparse.py:48-383, dense.py:53-342) with the conftest drive loop."""
    core, domain, exchange, flags, geometry, sparse, stencil = _ref()
    from slbm import dense

    st = stencil.make_stencil(stname)
    p = core.CollisionParams(omega=omega, model=model, lambda_odd=lam)
    values = seed_values(fl, st, seed, core)
    rec = {
        "kind": np.array("config_engine"),
        "stencil": np.array(stname),
        "model": np.array(model),
        "omega": np.array(omega),
        "lambda_odd": np.array(lam if lam is not None else np.nan),
        "dims": np.array(fl.dims),
        "periodic": np.array(fl.periodic),
        "seed": np.array(seed),
        "steps": np.array(steps),
        "recipe": np.array(json_dumps(recipe)),
        "tags_sha": np.array(sha(fl.tags)),
        "values0_sha": np.array(sha(values)),
        "layouts": np.array(list(layouts)),
        "patterns": np.array(list(patterns)),
    }
    first = None
    for layout in layouts:
        cls = sparse.SparseEngine if layout == "sparse" else dense.DenseEngine
        for pattern in patterns:
            e = cls(fl, st, p, pattern=pattern)
            if layout == "sparse":
                rec["n_fluid"] = np.array(e.n_fluid)
                rec["idx_sha"] = np.array(sha(e.idx))
                rec["base"] = e.base
            e.init_canonical(values)
            drive(e, steps)
            final = e.canonical_state()
            rho, u = e.macroscopic_fields()
            key = f"{layout}_{pattern}"
            rec[f"{key}_final_sha"] = np.array(sha(final))
            rec[f"{key}_rho_sha"] = np.array(sha(rho))
            rec[f"{key}_u_sha"] = np.array(sha(u))
            rec[f"{key}_counters"] = np.array([e.counters.steps, e.counters.cells_visited,
                                               e.counters.pdf_accesses, e.counters.idx_reads],
                                              dtype=np.int64)
            if first is None:
                first = final
                rng = np.random.default_rng(99)
                rec["sample_q"] = rng.integers(0, st.q, 3000)
                rec["sample_c"] = rng.integers(0, final.shape[1], 3000)
            rec[f"{key}_sample_v"] = final[rec["sample_q"], rec["sample_c"]]
    np.savez_compressed(os.path.join(OUT, f"config_{name}.npz"), **rec)
    print("config", name, "n_fluid", int(rec["n_fluid"]), flush=True)


def json_dumps(obj):
    import json

    return json.dumps(obj, sort_keys=True)


def _sphere_solid(dims, diameter, porosity, seed, geometry, fill_dims=None):
    """Overlapping spheres through the reference's voxelize (geometry.py:
    150-178); centres drawn over ``fill_dims`` (default dims) grown by one
    radius per side (the law of bench.py / paper_2408_06880_b200.geometry)."""
    import math

    fill = tuple(fill_dims or dims)
    vol = math.pi * diameter**3 / 6.0
    grown = np.asarray(fill, dtype=np.float64) + diameter
    count = int(round(-math.log(porosity) * float(np.prod(grown)) / vol))
    rng = np.random.default_rng(seed)
    centers = rng.random((count, 3)) * grown - diameter / 2.0
    pack = geometry.SpherePack(tuple(float(d) for d in dims), diameter, centers, seed)
    return geometry.voxelize(pack).solid


def configs_main(which):
    """BASELINE configs pinned at reduced scale."""
    os.makedirs(OUT, exist_ok=True)
    core, domain, exchange, flags, geometry, sparse, stencil = _ref()
    FK, FS = flags.FaceKind, flags.FaceSpec
    P, W = FS(FK.PERIODIC), FS(FK.WALL)
    lam316 = 1.0 / (3.0 / 16.0 / (1.0 / 1.2 - 0.5) + 0.5)
    if "c2" in which:
        # C2 law (d = 16, porosity 0.30, fully periodic, TRT AA) at 128^3 and 256^3
        for edge in (128, 256):
            bed_case(f"c2_{edge}_trt_aa", (edge,) * 3, 0.3, 16.0, 1, "d3q19", "trt", 1.2, lam316,
                     20, "aa", channel=False)
    if "c5" in which:
        # C5 porosity sweep: obstacle_flags (geometry.py:250-260, 315-320), sparse and dense
        for phi in (0.05, 0.3, 0.6, 1.0):
            fl = geometry.obstacle_flags((96, 96, 96), phi, 1)
            config_engine_case(f"c5_96_phi{int(round(phi * 100)):03d}", fl, "d3q19", "trt", 1.2,
                               lam316, 6,
                               {"kind": "obstacle", "dims": [96, 96, 96], "porosity": phi,
                                "seed": 1})
    if "c3" in which:
        # C3 riverbed at 64^3 per block, 2x2x1 blocks, D3Q27 TRT, overlapped driver
        dims = (128, 128, 64)
        solid = _sphere_solid(dims, 16.0, 0.35, 3, geometry, fill_dims=(128, 128, 32))
        lid = FS(FK.WALL, velocity=(0.02, 0.0, 0.0))
        fl = flags.make_flags(dims, [(P, P), (P, P), (W, lid)], solid=solid)
        config_domain_case("c3_2x2x1_d3q27_trt", fl, (64, 64, 64), "d3q27", "trt", 1.6, 1.1, 8,
                           {"kind": "riverbed", "dims": list(dims), "diameter": 16.0,
                            "porosity": 0.35, "seed": 3, "fill": [128, 128, 32],
                            "lid": [0.02, 0.0, 0.0]})
    if "c4" in which:
        # C4 artery, quarter scale (128^3 box, radii / 4), 32^3 blocks, UBB inlet, no outlet
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        if root not in sys.path:
            sys.path.insert(0, root)
        from paper_2408_06880_b200 import geometry as mine  # the generator (unpinned, F13)

        dims = (128, 128, 128)
        fluid = mine.artery_tree(dims, seed=0, r_root=10.0, r_min=3.5)
        inlet = FS(FK.WALL, velocity=(0.02, 0.0, 0.0))
        fl = flags.make_flags(dims, [(inlet, W), (W, W), (W, W)], solid=~fluid)
        config_domain_case("c4_quarter_artery", fl, (32, 32, 32), "d3q19", "trt", 1.7,
                           1.0 / (3.0 / 16.0 / (1.0 / 1.7 - 0.5) + 0.5), 10,
                           {"kind": "artery", "dims": list(dims), "seed": 0, "r_root": 10.0,
                            "r_min": 3.5, "inlet": [0.02, 0.0, 0.0]})


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--configs":
        configs_main(sys.argv[2:] or ["c2", "c3", "c4", "c5"])
    else:
        main()
