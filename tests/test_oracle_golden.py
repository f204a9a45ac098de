"""Pins the CPU oracle to the reference: every golden vector produced by the
unmodified reference (tools/make_golden.py) must be reproduced bit for bit
by the numpy restatement in oracle/ (CPU only)."""

import hashlib
import math
import os

import numpy as np
import pytest

from conftest import drive, flags_of, golden_files, load_golden, params_of, stencil_of
from oracle.sparse_ref import OracleInstability, OracleSparseEngine, build_lists

ENGINE = golden_files("engine")
BED = golden_files("bed")
# the oracle steps the beds up to C1's 64^3 here; the C2 law at 128^3 / 256^3
# is pinned on the GPU only (tests/test_gpu_engine.py), the CPU suite stays fast
BED_CPU = [p for p in BED if int(np.prod(np.load(p)["dims"])) <= 64 ** 3]


def _id(p):
    return os.path.basename(p)[:-4]


@pytest.mark.parametrize("path", ENGINE, ids=_id)
def test_oracle_lists_match_reference(path):
    rec = load_golden(path)
    fl, st = flags_of(rec), stencil_of(rec)
    L = build_lists(fl, st)
    assert np.array_equal(L["idx"], rec["idx"]) and L["idx"].dtype == np.uint32
    assert np.array_equal(L["base"], rec["base"])
    assert np.array_equal(L["fluid_coords"], rec["fluid_coords"])
    assert np.array_equal(L["ubb_slots"], rec["ubb_slots"])
    assert np.array_equal(L["ubb_partner"], rec["ubb_partner"])
    assert np.array_equal(L["ubb_corr"], rec["ubb_corr"])
    items = sorted(L["ghost"].items(), key=lambda kv: kv[1])
    assert [k[0] for k, _ in items] == list(rec["ghost_q"])
    assert [k[1] for k, _ in items] == list(rec["ghost_pflat"])
    assert [v for _, v in items] == list(rec["ghost_slot"])
    eng = OracleSparseEngine(fl, st, params_of(rec), "aa", frame_width=int(rec["frame_width"]))
    assert np.array_equal(eng._sel["interior"], rec["interior"])
    assert np.array_equal(eng._sel["frame"], rec["frame"])


@pytest.mark.parametrize("pattern", ["pull", "aa"])
@pytest.mark.parametrize("path", ENGINE, ids=_id)
def test_oracle_states_match_reference(path, pattern):
    rec = load_golden(path)
    fl, st, p = flags_of(rec), stencil_of(rec), params_of(rec)
    for steps in rec["steps_list"]:
        eng = OracleSparseEngine(fl, st, p, pattern)
        eng.init_canonical(rec["values0"])
        drive(eng, int(steps), rec["ghost_slot"], rec["ghost_fill"])
        assert np.array_equal(eng.canonical_state(), rec[f"{pattern}_{steps}_state"])
        rho, u = eng.macroscopic_fields()
        assert np.array_equal(rho, rec[f"{pattern}_{steps}_rho"])
        assert np.array_equal(u, rec[f"{pattern}_{steps}_u"])


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("path", BED_CPU, ids=_id)
def test_oracle_bed_runs_match_reference(path):
    """C1 (64^3 channel bed, 100 steps) and the C2 law at 48^3: bitwise via
    SHA-256 of the full canonical state."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil
    from paper_2408_06880_b200.tags import PERIODIC, make_flags

    rec = load_golden(path)
    dims = tuple(int(d) for d in rec["dims"])
    d = float(rec["diameter"])
    centers = geometry.sphere_centers(dims, d, int(rec["count"]), int(rec["seed"]))
    solid = geometry.voxelize_spheres(dims, centers, d)
    if bool(rec["channel"]):
        fl = geometry.channel_flags(dims, solid=solid)
    else:
        fl = make_flags(dims, [(PERIODIC, PERIODIC)] * 3, solid=solid)
    assert _sha(fl.tags) == str(rec["tags_sha"])
    st = make_stencil(str(rec["stencil"]))
    lam = float(rec["lambda_odd"])
    p = CollisionParams(float(rec["omega"]), str(rec["model"]), None if math.isnan(lam) else lam)
    eng = OracleSparseEngine(fl, st, p, str(rec["pattern"]))
    assert eng.n_fluid == int(rec["n_fluid"])
    assert _sha(eng.idx) == str(rec["idx_sha"])
    values0 = init_random_values(fl, st, eng, seed=7)
    assert _sha(values0) == str(rec["values0_sha"])
    eng.init_canonical(values0)
    drive(eng, int(rec["steps"]))
    final = eng.canonical_state()
    assert _sha(final) == str(rec["final_sha"])
    rho, u = eng.macroscopic_fields()
    assert _sha(rho) == str(rec["rho_sha"]) and _sha(u) == str(rec["u_sha"])


def init_random_values(fl, st, eng, seed, amplitude=0.005):
    """domain.py:191-206 (Domain.init_random) for a single whole-box block."""
    from oracle.sparse_ref import equilibrium

    rng = np.random.default_rng(seed)
    shape = tuple(reversed(fl.dims))
    rho_g = 1.0 + amplitude * rng.standard_normal(shape)
    u_g = amplitude * rng.standard_normal((st.dim,) + shape)
    flat = np.ravel_multi_index(eng.fluid_coords[:, ::-1].T, shape)
    return equilibrium(rho_g.reshape(-1)[flat], u_g.reshape(st.dim, -1)[:, flat], st)


def test_oracle_flags_instability():
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.geometry import couette_flags
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d2q9")
    eng = OracleSparseEngine(couette_flags((8, 5), 0.05), st, CollisionParams(1.0))
    eng.init_equilibrium()
    with pytest.raises(OracleInstability):
        eng.step()
