"""The D3Q19 index-list sweep's occupancy (knob 13: 4 or 5 CTAs per SM, or
measured per engine on its first sweeps) changes the kernel's schedule, not
its arithmetic: every choice gives the same bits, for AA and pull, with and
without CUDA graphs (the graph path measures on eager steps first)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pattern", ["aa", "pull"])
def test_occupancy_choices_are_bit_identical(pattern, gpu_lib):
    from oracle.sparse_ref import equilibrium
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda
    from paper_2408_06880_b200.engine import SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    p = CollisionParams(1.2, "trt", trt_magic_lambda(1.2))
    fl = geometry.obstacle_flags((256, 256, 128), 0.5, 4)  # ~4.2 M fluid cells: measured
    rng = np.random.default_rng(1)
    states = []
    for knob, graph in ((4, False), (5, False), (0, False), (0, True)):
        e = SparseEngine(fl, st, p, pattern, device=0, check="deferred")
        assert e.n_fluid >= 1 << 22
        e.set_tuning(13, knob)
        n = e.n_fluid
        rng = np.random.default_rng(1)
        e.init_canonical(equilibrium(1.0 + 0.01 * rng.standard_normal(n),
                                     0.02 * rng.standard_normal((3, n)), st))
        if graph:
            e.run(12, use_graph=True)
        else:
            for _ in range(12):
                e.refresh_boundary(e.parity)
                e.step()
                e.finish_step()
        states.append(e.canonical_state())
        del e
    for s in states[1:]:
        assert np.array_equal(states[0], s)
