"""BASELINE configs pinned against the reference at reduced scale.

``tools/make_golden.py --configs`` ran the UNMODIFIED reference (its
``SparseEngine`` / ``DenseEngine`` / ``Domain`` and overlapped driver) on:

* C5 -- ``obstacle_flags(96^3, phi, seed=1)`` (``geometry.py:250-260,
  315-320``) at phi in {0.05, 0.3, 0.6, 1.0}, D3Q19 TRT, sparse and dense,
  AA and pull;
* C3 -- the riverbed (overlapping-sphere bed in the lower half, free flow
  above, periodic x/y, no-slip floor, moving lid) at 64^3 per block, 2x2x1
  blocks, D3Q27 TRT, AA, overlapped driver (``exchange.py:349-374``);
* C4 -- the artery tree at quarter scale (128^3 box, radii / 4) in 32^3
  blocks (empty ones dropped), UBB inlet, D3Q19 TRT, AA, overlapped driver,
  plus the reference's ``balance(8)`` assignment (``domain.py:312-325``).

(The C2 law at 128^3 and 256^3 lives with C1 in ``bed_*.npz``, checked by
``test_gpu_engine.py::test_bed_runs_bit_exact``; here its CUDA-graph path.)

Here the geometry is rebuilt with this package's generators (the tag box is
pinned by its SHA-256), the same initial state is built, the GPU path runs,
and the SHA-256 of the final state, rho and u must equal the reference's:
bitwise parity, config by config.
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import drive, golden_files, load_golden, seed_values

pytestmark = pytest.mark.gpu

CONFIG = golden_files("config")
ENGINE_CFG = [p for p in CONFIG if "c5_" in os.path.basename(p)]
DOMAIN_CFG = [p for p in CONFIG if "c3_" in os.path.basename(p) or "c4_" in os.path.basename(p)]
BIG_BEDS = [p for p in golden_files("bed") if int(np.prod(np.load(p)["dims"])) >= 128 ** 3]


def _id(p):
    return os.path.basename(p)[:-4]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _params(rec):
    from paper_2408_06880_b200.collision import CollisionParams

    lam = float(rec["lambda_odd"])
    return CollisionParams(float(rec["omega"]), str(rec["model"]), None if math.isnan(lam) else lam)


def _flags(recipe):
    """The geometry of a config, rebuilt by this package's generators."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.tags import PERIODIC, WALL, FaceKind, FaceSpec, make_flags

    dims = tuple(recipe["dims"])
    kind = recipe["kind"]
    if kind == "obstacle":
        return geometry.obstacle_flags(dims, recipe["porosity"], recipe["seed"])
    if kind == "riverbed":
        fill, d = tuple(recipe["fill"]), recipe["diameter"]
        n = geometry.overlapping_sphere_count(fill, d, recipe["porosity"])
        centers = geometry.sphere_centers(fill, d, n, recipe["seed"])
        solid = geometry.voxelize_spheres(dims, centers, d, device=0)  # CUDA rasterizer
        lid = FaceSpec(FaceKind.WALL, velocity=tuple(recipe["lid"]))
        return make_flags(dims, [(PERIODIC, PERIODIC), (PERIODIC, PERIODIC), (WALL, lid)],
                          solid=solid)
    if kind == "artery":
        fluid = geometry.artery_tree(dims, seed=recipe["seed"], r_root=recipe["r_root"],
                                     r_min=recipe["r_min"])
        inlet = FaceSpec(FaceKind.WALL, velocity=tuple(recipe["inlet"]))
        return make_flags(dims, [(inlet, WALL), (WALL, WALL), (WALL, WALL)], solid=~fluid)
    raise AssertionError(kind)


def _check_flags(fl, rec):
    assert _sha(fl.tags) == str(rec["tags_sha"]), "geometry differs from the reference's"
    if "ubb_sha" in rec:
        ubb = np.where((fl.tags == 2)[..., None], np.asarray(fl.ubb_u), 0.0)
        assert _sha(ubb) == str(rec["ubb_sha"])


# ---------------------------------------------------------------- C5 engines


@pytest.mark.parametrize("path", ENGINE_CFG, ids=_id)
def test_c5_porosity_sweep_bit_exact(path, gpu_lib):
    from paper_2408_06880_b200.engine import DenseEngine, SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    rec = load_golden(path)
    recipe = json.loads(str(rec["recipe"]))
    fl = _flags(recipe)
    _check_flags(fl, rec)
    st = make_stencil(str(rec["stencil"]))
    p = _params(rec)
    values = seed_values(fl, st, int(rec["seed"]))
    assert _sha(values) == str(rec["values0_sha"])
    for layout in [str(x) for x in rec["layouts"]]:
        cls = SparseEngine if layout == "sparse" else DenseEngine
        for pattern in [str(x) for x in rec["patterns"]]:
            eng = cls(fl, st, p, pattern)
            if layout == "sparse":
                assert eng.n_fluid == int(rec["n_fluid"])
                assert _sha(eng.idx) == str(rec["idx_sha"])
                np.testing.assert_array_equal(eng.base, rec["base"])
            eng.init_canonical(values)
            drive(eng, int(rec["steps"]))
            key = f"{layout}_{pattern}"
            final = eng.canonical_state()
            np.testing.assert_array_equal(final[rec["sample_q"], rec["sample_c"]],
                                          rec[f"{key}_sample_v"])
            assert _sha(final) == str(rec[f"{key}_final_sha"]), key
            rho, u = eng.macroscopic_fields()
            assert _sha(rho) == str(rec[f"{key}_rho_sha"]), key
            assert _sha(u) == str(rec[f"{key}_u_sha"]), key
            c = eng.counters
            np.testing.assert_array_equal(
                [c.steps, c.cells_visited, c.pdf_accesses, c.idx_reads], rec[f"{key}_counters"])


@pytest.mark.parametrize("path", ENGINE_CFG, ids=_id)
def test_c5_device_loop_bit_exact(path, gpu_lib):
    """The same runs through engine.run (CUDA graph / resident kernel: the
    path the porosity-sweep benchmark times)."""
    from paper_2408_06880_b200.engine import DenseEngine, SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    rec = load_golden(path)
    fl = _flags(json.loads(str(rec["recipe"])))
    st = make_stencil(str(rec["stencil"]))
    values = seed_values(fl, st, int(rec["seed"]))
    for layout, cls in (("sparse", SparseEngine), ("dense", DenseEngine)):
        eng = cls(fl, st, _params(rec), "aa")
        eng.init_canonical(values)
        eng.run(int(rec["steps"]))
        assert _sha(eng.canonical_state()) == str(rec[f"{layout}_aa_final_sha"]), layout


# ---------------------------------------------------------------- C3 / C4 domains


def _domain_digest_check(dom, rec, prefix):
    g = dom.gather_canonical()
    q = g.shape[0]
    flat = g.reshape(q, -1)
    np.testing.assert_array_equal(flat[rec[f"{prefix}_sample_q"], rec[f"{prefix}_sample_cell"]],
                                  rec[f"{prefix}_sample_v"])
    assert _sha(g) == str(rec[f"{prefix}_sha"]), prefix


VARIANTS = ["reference-driver", "halo-frames-graph", "distributed-loopback"]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("path", DOMAIN_CFG, ids=_id)
def test_c3_c4_domains_bit_exact(path, variant, gpu_lib):
    """reference-driver: frame width 1 and the per-step overlapped driver,
    as the reference ran it (counters compared too); halo-frames-graph: the
    benchmark's layout (frames only toward other blocks, block group, one
    CUDA graph per step pair); distributed-loopback: DistributedDomain with
    a one-rank NCCL communicator exchanging every edge through NCCL."""
    from paper_2408_06880_b200.domain import DistributedDomain, Domain
    from paper_2408_06880_b200.lattice import make_stencil

    rec = load_golden(path)
    fl = _flags(json.loads(str(rec["recipe"])))
    _check_flags(fl, rec)
    st = make_stencil(str(rec["stencil"]))
    block = tuple(int(b) for b in rec["block"])
    pattern, driver = str(rec["pattern"]), str(rec["driver"])
    if variant == "reference-driver":
        dom = Domain(fl, block, st, _params(rec), pattern=pattern, frame_width=1)
    elif variant == "halo-frames-graph":
        dom = Domain(fl, block, st, _params(rec), pattern=pattern, frame_width="halo",
                     check="deferred")
    else:
        dom = DistributedDomain(fl, block, st, _params(rec), pattern=pattern, rank=0, world=1,
                                device=0, loopback=True)
    assert sorted(dom.blocks) == list(rec["blocks"])
    assert [dom.blocks[b].n_fluid for b in sorted(dom.blocks)] == list(rec["block_fluid"])
    assert len(dom.edge_plans) == int(rec["n_edges"])
    dom.init_random(int(rec["seed"]))
    _domain_digest_check(dom, rec, "init")
    steps = int(rec["steps"])
    if variant == "reference-driver":
        dom.run(steps, driver=driver)
    else:
        dom.run(steps, driver="overlapped", use_graph=True)
    _domain_digest_check(dom, rec, "final")
    rho, u = dom.gather_macroscopics()
    assert _sha(rho) == str(rec["rho_sha"]) and _sha(u) == str(rec["u_sha"])
    if variant == "reference-driver":
        c = dom.counters()
        np.testing.assert_array_equal(
            [c.steps, c.cells_visited, c.cells_visited_interior, c.cells_visited_frame,
             c.pdf_accesses, c.idx_reads, c.values_exchanged, c.messages], rec["counters"])
        wire = [sum(pp.n_wire for pp in pl.phases.values()) for pl in dom.edge_plans]
        np.testing.assert_array_equal(wire, rec["edge_wire"])
        if "balance_bids" in rec:
            asg = dom.balance(8)
            assert [asg[b] for b in rec["balance_bids"]] == list(rec["balance_workers"])


# ---------------------------------------------------------------- C2 law, graph path


@pytest.mark.parametrize("path", BIG_BEDS, ids=_id)
def test_c2_law_device_loop_bit_exact(path, gpu_lib):
    """The C2 law at 128^3 / 256^3 through engine.run -- the exact call the
    bench times (CUDA graph of a step pair) -- equals the reference."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.engine import SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil
    from paper_2408_06880_b200.tags import PERIODIC, make_flags
    from test_oracle_golden import init_random_values

    rec = load_golden(path)
    dims = tuple(int(d) for d in rec["dims"])
    d = float(rec["diameter"])
    n = geometry.overlapping_sphere_count(dims, d, float(rec["porosity_target"]))
    solid = geometry.voxelize_spheres(dims, geometry.sphere_centers(dims, d, n, int(rec["seed"])),
                                      d, device=0)
    fl = make_flags(dims, [(PERIODIC, PERIODIC)] * 3, solid=solid)
    assert _sha(fl.tags) == str(rec["tags_sha"])
    st = make_stencil(str(rec["stencil"]))
    eng = SparseEngine(fl, st, _params(rec), str(rec["pattern"]), check="deferred")
    eng.init_canonical(init_random_values(fl, st, eng, seed=7))
    eng.run(int(rec["steps"]))
    final = eng.canonical_state()
    np.testing.assert_array_equal(final[rec["sample_q"], rec["sample_c"]], rec["sample_v"])
    assert _sha(final) == str(rec["final_sha"])
    rho, u = eng.macroscopic_fields()
    assert _sha(rho) == str(rec["rho_sha"]) and _sha(u) == str(rec["u_sha"])
