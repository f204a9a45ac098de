"""CPU side of the reduced-scale BASELINE config goldens
(tools/make_golden.py --configs): this package's geometry generators rebuild
every config's tag box bit for bit (SHA-256 vs the reference's), and the
oracle reproduces the reference's C5 runs -- so the oracle the GPU tests
lean on is pinned on these configs too."""

import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import drive, golden_files, load_golden, seed_values

CONFIG = golden_files("config")


def _id(p):
    return os.path.basename(p)[:-4]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _flags(recipe):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.tags import PERIODIC, WALL, FaceKind, FaceSpec, make_flags

    dims = tuple(recipe["dims"])
    if recipe["kind"] == "obstacle":
        return geometry.obstacle_flags(dims, recipe["porosity"], recipe["seed"])
    if recipe["kind"] == "riverbed":
        fill, d = tuple(recipe["fill"]), recipe["diameter"]
        n = geometry.overlapping_sphere_count(fill, d, recipe["porosity"])
        solid = geometry.voxelize_spheres(dims, geometry.sphere_centers(fill, d, n, recipe["seed"]), d)
        lid = FaceSpec(FaceKind.WALL, velocity=tuple(recipe["lid"]))
        return make_flags(dims, [(PERIODIC, PERIODIC), (PERIODIC, PERIODIC), (WALL, lid)],
                          solid=solid)
    fluid = geometry.artery_tree(dims, seed=recipe["seed"], r_root=recipe["r_root"],
                                 r_min=recipe["r_min"])
    inlet = FaceSpec(FaceKind.WALL, velocity=tuple(recipe["inlet"]))
    return make_flags(dims, [(inlet, WALL), (WALL, WALL), (WALL, WALL)], solid=~fluid)


@pytest.mark.parametrize("path", CONFIG, ids=_id)
def test_config_geometry_matches_reference(path):
    rec = load_golden(path)
    fl = _flags(json.loads(str(rec["recipe"])))
    assert _sha(fl.tags) == str(rec["tags_sha"])
    if "ubb_sha" in rec:
        ubb = np.where((fl.tags == 2)[..., None], np.asarray(fl.ubb_u), 0.0)
        assert _sha(ubb) == str(rec["ubb_sha"])


@pytest.mark.parametrize("path", [p for p in CONFIG if "phi005" in p or "phi030" in p], ids=_id)
def test_oracle_reproduces_c5(path):
    from oracle.sparse_ref import OracleSparseEngine
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil

    rec = load_golden(path)
    fl = _flags(json.loads(str(rec["recipe"])))
    st = make_stencil(str(rec["stencil"]))
    lam = float(rec["lambda_odd"])
    p = CollisionParams(float(rec["omega"]), str(rec["model"]), None if math.isnan(lam) else lam)
    values = seed_values(fl, st, int(rec["seed"]))
    assert _sha(values) == str(rec["values0_sha"])
    eng = OracleSparseEngine(fl, st, p, "aa")
    assert _sha(eng.idx) == str(rec["idx_sha"])
    eng.init_canonical(values)
    drive(eng, int(rec["steps"]))
    assert _sha(eng.canonical_state()) == str(rec["sparse_aa_final_sha"])
