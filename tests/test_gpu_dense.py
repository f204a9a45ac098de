"""Direct-addressing (dense) GPU engine and the hybrid layout policy
(SURVEY §8f1): bit-identical to the reference goldens, like the reference's
own DenseEngine is to its SparseEngine (tests/test_sparse.py:49-65 of the
reference), and mixed sparse/dense decompositions give the same answer
(reference tests/test_domain.py:134-160)."""

import os

import numpy as np
import pytest

from conftest import (drive, flags_of, golden_files, load_golden, params_of, seed_values,
                      stencil_of)

pytestmark = pytest.mark.gpu

ENGINE = golden_files("engine")


def _id(p):
    return os.path.basename(p)[:-4]


@pytest.mark.parametrize("pattern", ["pull", "aa"])
@pytest.mark.parametrize("path", ENGINE, ids=_id)
def test_dense_engine_matches_reference_goldens(path, pattern, gpu_lib):
    from paper_2408_06880_b200.engine import DenseEngine

    rec = load_golden(path)
    fl, st, p = flags_of(rec), stencil_of(rec), params_of(rec)
    npad = int(np.prod(fl.tags.shape))
    ghost = rec["ghost_q"] * npad + rec["ghost_pflat"]  # halo slots of the dense layout
    for steps in rec["steps_list"]:
        eng = DenseEngine(fl, st, p, pattern)
        assert eng.layout == "dense" and eng.idx_element_count() == 0
        eng.init_canonical(rec["values0"])
        drive(eng, int(steps), ghost, rec["ghost_fill"])
        np.testing.assert_array_equal(eng.canonical_state(), rec[f"{pattern}_{steps}_state"])
        rho, u = eng.macroscopic_fields()
        np.testing.assert_array_equal(rho, rec[f"{pattern}_{steps}_rho"])
        np.testing.assert_array_equal(u, rec[f"{pattern}_{steps}_u"])
        box = int(np.prod(fl.dims))
        assert eng.counters.cells_visited == int(steps) * box
        assert eng.pdf_element_count() == (2 if pattern == "pull" else 1) * st.q * box


@pytest.mark.parametrize("pattern", ["pull", "aa"])
def test_layout_policies_never_change_the_answer(pattern, gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d2q9")
    gf = geometry.riverbed_flags((16, 16), (8, 8), bed_porosity=0.5, seed=3)
    p = CollisionParams(1.2)
    cases = [((16, 16), "dense"), ((16, 16), "sparse"), ((8, 16), "hybrid"), ((8, 8), "sparse"),
             ((4, 8), "hybrid"), ((8, 8), "dense")]
    out, kinds = [], []
    for block, policy in cases:
        d = Domain(gf, block, st, p, pattern=pattern, policy=policy, frame_width=1)
        d.init_random(11)
        d.run(6, driver="overlapped")
        out.append(d.gather_canonical())
        kinds.append({b.kind for b in d.blocks.values()})
    assert {"dense", "sparse"} in kinds  # a real hybrid mix was exercised
    for o in out[1:]:
        np.testing.assert_array_equal(o, out[0])
    gold = load_golden(os.path.join(os.path.dirname(ENGINE[0]), "domain_d2q9_riverbed.npz"))
    d = Domain(gf, (8, 8), st, p, pattern=pattern, policy="hybrid", frame_width=1)
    d.init_random(int(gold["seed"]))
    d.run(int(gold["steps"]), driver="overlapped")
    np.testing.assert_array_equal(d.gather_canonical(), gold[f"{pattern}_final"])


def test_dense_3d_with_moving_lid_and_split_sweeps(gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import DenseEngine, SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    for name, model in (("d3q19", "trt"), ("d3q27", "cumulant")):
        st = make_stencil(name)
        fl = geometry.riverbed_flags((14, 10, 12), (7, 5, 6), 0.6, 5, 0.04)
        p = CollisionParams(1.5, model, 0.8 if model == "trt" else None)
        a = SparseEngine(fl, st, p, "aa")
        b = DenseEngine(fl, st, p, "aa", frame_width=(2, 1, 1))
        a.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
        b.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
        for _ in range(9):
            a.refresh_boundary(a.parity)
            a.step()
            a.finish_step()
            b.refresh_boundary(b.parity)
            b.step("interior")
            b.step("frame")
            b.finish_step()
        np.testing.assert_array_equal(a.canonical_state(), b.canonical_state())
        assert b.n_interior + b.n_frame == int(np.prod(fl.dims))


@pytest.mark.parametrize("porosity", [0.55, 0.92])
@pytest.mark.parametrize("pattern", ["pull", "aa"])
def test_dense_mask_first_and_speculative_paths(porosity, pattern, gpu_lib):
    """Dense blocks below porosity 0.75 wait for the fold mask, denser ones
    load speculatively and re-read folded directions: both equal the sparse
    engine bit for bit (periodic bed with walls and a moving lid)."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import DenseEngine, SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    dims = (24, 20, 16)
    fl = geometry.packed_bed_flags(dims, porosity, 4.0, 9, channel=True)
    p = CollisionParams(1.3, "trt", 0.9)
    a = SparseEngine(fl, st, p, pattern)
    b = DenseEngine(fl, st, p, pattern)
    assert (a.n_fluid >= 0.75 * np.prod(dims)) == (porosity > 0.75)
    v = seed_values(fl, st, 3)
    a.init_canonical(v)
    b.init_canonical(v)
    for e in (a, b):
        for _ in range(6):
            e.refresh_boundary(e.parity)
            e.step()
            e.finish_step()
    np.testing.assert_array_equal(a.canonical_state(), b.canonical_state())
