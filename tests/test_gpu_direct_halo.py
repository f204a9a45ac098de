"""Direct local halo edges (slbm_group_link_halo): an AA block group whose
device-local edges are served by direct addressing must hand back exactly
the copy program's state -- sources and ghosts, at both parities -- for any
mix of calls (single steps, CUDA-graph pairs, odd/even stops, both drivers),
and engine-level reads between calls must see the reference's state."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _domain(direct: bool, driver_frame=1):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.lattice import make_stencil

    os.environ["SLBM_DIRECT_HALO"] = "1" if direct else "0"
    try:
        gf = geometry.riverbed_flags((24, 16, 20), (8, 8, 10), 0.45, 7, 0.03)
        d = Domain(gf, (8, 8, 10), make_stencil("d3q19"), CollisionParams(1.25, "trt", 0.92),
                   pattern="aa", frame_width=driver_frame, check="deferred")
    finally:
        os.environ.pop("SLBM_DIRECT_HALO", None)
    d.init_random(11)
    return d


def _all_slots(d):
    return [b.engine.read_slots(np.arange(b.engine.total_slots)) for b in d.local_blocks()]


@pytest.mark.parametrize("driver", ["sequential", "overlapped"])
def test_direct_equals_copy_program(driver, gpu_lib):
    a, b = _domain(False), _domain(True)
    assert not a.direct_halo and b.direct_halo
    for n, graph in [(3, False), (5, True), (1, False), (4, True), (2, False), (7, True)]:
        a.run(n, driver=driver, use_graph=graph)
        b.run(n, driver=driver, use_graph=graph)
        # every slot of every block, ghosts included
        for x, y in zip(_all_slots(a), _all_slots(b)):
            np.testing.assert_array_equal(x, y)
        np.testing.assert_array_equal(a.gather_canonical(), b.gather_canonical())
        ra, ua = a.gather_macroscopics()
        rb, ub = b.gather_macroscopics()
        np.testing.assert_array_equal(ra, rb)
        np.testing.assert_array_equal(ua, ub)


def test_single_step_calls(gpu_lib):
    a, b = _domain(False), _domain(True)
    for _ in range(5):
        a.step_sequential()
        b.step_sequential()
        for x, y in zip(_all_slots(a), _all_slots(b)):
            np.testing.assert_array_equal(x, y)


def test_linked_engines_refuse_engine_level_steps(gpu_lib):
    from paper_2408_06880_b200 import errors

    d = _domain(True)
    e = d.local_blocks()[0].engine
    with pytest.raises(errors.error_class("ConfigurationError")):
        e.step()
    d.run(2)  # the domain still steps them


def test_many_block_group_equals_one_block(gpu_lib):
    """> 128 blocks: the boundary launch looks engines up in the device table
    (BoundaryTable), the sweep reads the 512-capacity parameter block; with
    a moving lid (UBB) and direct local edges the result equals one block."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    p = CollisionParams(1.3, "trt", 0.9)
    gf = geometry.riverbed_flags((48, 40, 48), (8, 8, 8), 0.5, 5, 0.03)
    many = Domain(gf, (8, 8, 8), st, p, pattern="aa", frame_width=1, check="deferred")
    assert len(many.local_blocks()) > 128 and many.direct_halo
    one = Domain(gf, (48, 40, 48), st, p, pattern="aa", frame_width=1, check="deferred")
    for d in (many, one):
        d.init_random(5)
        d.run(3, use_graph=True)
        d.run(5)  # an even total: odd-parity readouts are block-local (reference)
    np.testing.assert_array_equal(many.gather_canonical(), one.gather_canonical())
