"""Monitors (slbm_total_moments): mass and momentum from one device pass
with warp-shuffle reductions equal the canonical state's sums to rounding,
repeat bit for bit, and are conserved by the periodic AA/pull steps."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pattern", ["aa", "pull"])
@pytest.mark.parametrize("q", [19, 27])
def test_total_moments_match_state(pattern, q, gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil(f"d3q{q}")
    fl = geometry.obstacle_flags((40, 36, 32), 0.6, 3)
    eng = SparseEngine(fl, st, CollisionParams(1.1, "trt", 0.9), pattern)
    rng = np.random.default_rng(5)
    n = eng.n_fluid
    from oracle.sparse_ref import equilibrium

    eng.init_canonical(equilibrium(1.0 + 0.01 * rng.standard_normal(n),
                                   0.02 * rng.standard_normal((3, n)), st))
    for steps in (0, 1, 4):
        for _ in range(steps):
            eng.refresh_boundary(eng.parity)
            eng.step()
            eng.finish_step()
        m = eng.total_moments()
        f = eng.canonical_state()
        c = np.asarray(st.c, dtype=np.float64)
        want = np.concatenate([[f.sum()], c.T @ f.sum(axis=1)])
        np.testing.assert_allclose(m, want, rtol=1e-12, atol=1e-12 * want[0])
        assert np.array_equal(m, eng.total_moments())  # fixed reduction tree
        assert m[0] == eng.total_mass()


def test_domain_moments_conserved(gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.lattice import make_stencil

    fl = geometry.obstacle_flags((32, 32, 32), 0.7, 2)
    d = Domain(fl, (16, 16, 16), make_stencil("d3q19"), CollisionParams(1.2, "trt", 0.94),
               pattern="aa", frame_width=1)
    d.init_random(3)
    m0 = d.total_moments()
    d.run(10)
    m1 = d.total_moments()
    assert abs(m1[0] - m0[0]) <= 1e-12 * m0[0]
