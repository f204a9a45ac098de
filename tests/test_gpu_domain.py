"""Multi-block Domain on the GPU vs the reference's multi-block goldens:
decomposition, EdgePlan slot lists, device halo exchange (fused local
gather-scatter kernels), sequential and overlapped drivers — bit for bit."""

import os

import numpy as np
import pytest

from conftest import flags_of, golden_files, load_golden, params_of, stencil_of

pytestmark = pytest.mark.gpu

DOMAIN = golden_files("domain")


def _id(p):
    return os.path.basename(p)[:-4]


def _domain(rec, pattern, **kw):
    from paper_2408_06880_b200.domain import Domain

    return Domain(flags_of(rec), tuple(int(b) for b in rec["block"]), stencil_of(rec),
                  params_of(rec), pattern=pattern, frame_width=1, **kw)


@pytest.mark.parametrize("driver", ["overlapped", "sequential"])
@pytest.mark.parametrize("pattern", ["pull", "aa"])
@pytest.mark.parametrize("path", DOMAIN, ids=_id)
def test_domain_run_bit_exact(path, pattern, driver, gpu_lib):
    rec = load_golden(path)
    dom = _domain(rec, pattern)
    assert sorted(dom.blocks) == list(rec[f"{pattern}_blocks"])
    dom.init_random(int(rec["seed"]))
    np.testing.assert_array_equal(dom.gather_canonical(), rec[f"{pattern}_init"])
    rows, send, take, tgt = [], [], [], []
    for plan in dom.edge_plans:
        for ph, pp in plan.phases.items():
            rows.append([plan.src_bid, plan.dst_bid, *plan.sigma, ph.value, pp.n_wire, len(pp.tgt_sel)])
            send.append(pp.send_sel)
            take.append(pp.pos_from_sparse)
            tgt.append(pp.tgt_sel)
    assert np.array_equal(np.array(rows, dtype=np.int64), rec[f"{pattern}_edges"])
    assert np.array_equal(np.concatenate(send), rec[f"{pattern}_send"])
    assert np.array_equal(np.concatenate(take), rec[f"{pattern}_take"])
    assert np.array_equal(np.concatenate(tgt), rec[f"{pattern}_tgt"])
    dom.run(int(rec["steps"]), driver=driver)
    np.testing.assert_array_equal(dom.gather_canonical(), rec[f"{pattern}_final"])
    rho, u = dom.gather_macroscopics()
    np.testing.assert_array_equal(rho, rec[f"{pattern}_rho"])
    np.testing.assert_array_equal(u, rec[f"{pattern}_u"])
    c = dom.counters()
    got = [c.steps, c.cells_visited, c.cells_visited_interior, c.cells_visited_frame,
           c.pdf_accesses, c.idx_reads, c.values_exchanged, c.messages]
    if driver == "overlapped":
        assert got == list(rec[f"{pattern}_counters"])


def test_decomposition_invariance_and_aa_equals_pull(gpu_lib):
    """reference tests/test_domain.py:134-173 on the GPU: 1, 2, 4, 8 blocks give
    the same answer bitwise; AA pairs equal pull."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    gf = geometry.riverbed_flags((16, 16, 16), (8, 8, 8), 0.5, 3, 0.03)
    p = CollisionParams(1.3, "trt", 0.9)
    out = []
    for pattern in ("aa", "pull"):
        for block in [(16, 16, 16), (8, 16, 16), (8, 8, 16), (8, 8, 8)]:
            d = Domain(gf, block, st, p, pattern=pattern, frame_width=1)
            d.init_random(4)
            d.run(6, driver="overlapped" if block[0] == 8 else "sequential")
            out.append(d.gather_canonical())
    for o in out[1:]:
        np.testing.assert_array_equal(o, out[0])


def test_run_wraps_instability_with_the_step_number(gpu_lib):
    from paper_2408_06880_b200 import errors, geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.lattice import make_stencil

    gf = geometry.riverbed_flags((16, 16), (8, 8), seed=1, lid_speed=0.5)
    dom = Domain(gf, (8, 8), make_stencil("d2q9"), CollisionParams(omega=1.99))
    dom.init_random(1)
    with pytest.raises(errors.NumericalInstabilityError, match="unstable at step"):
        dom.run(100)


def test_driver_validation(gpu_lib):
    from paper_2408_06880_b200 import errors, geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.lattice import make_stencil

    dom = Domain(geometry.channel_flags((8, 4)), (4, 4), make_stencil("d2q9"), CollisionParams(1.0))
    dom.init_equilibrium()
    with pytest.raises(errors.ConfigurationError, match="frame_width"):
        dom.run(1, driver="overlapped")
    with pytest.raises(errors.ConfigurationError, match="unknown driver"):
        dom.run(1, driver="sideways")


@pytest.mark.parametrize("loopback", [False, True])
@pytest.mark.parametrize("pattern", ["aa", "pull"])
def test_graph_replay_matches_python_driver(pattern, loopback, gpu_lib):
    """Domain.run(use_graph=True) (one captured step pair of the whole
    domain, halo + all blocks, NCCL in loopback mode) == the Python driver."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain, DistributedDomain
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    gf = geometry.riverbed_flags((24, 16, 16), (8, 8, 8), 0.5, 7, 0.03)
    p = CollisionParams(1.4, "trt", 0.9)
    doms = []
    for use_graph in (False, True):
        if loopback:
            d = DistributedDomain(gf, (8, 8, 8), st, p, pattern=pattern, frame_width=1, rank=0,
                                  world=1, device=0, loopback=True)
        else:
            d = Domain(gf, (8, 8, 8), st, p, pattern=pattern, frame_width=1, check="deferred")
        d.init_random(3)
        d.run(3, driver="overlapped")
        d.run(8, driver="overlapped", use_graph=use_graph)
        d.run(1, driver="overlapped")
        # an odd number of eager steps between two graph runs: for pull the
        # buffers are swapped relative to the first capture
        d.run(2, driver="overlapped", use_graph=use_graph)
        d.run(1, driver="overlapped")
        d.run(4, driver="overlapped", use_graph=use_graph)
        doms.append(d)
    np.testing.assert_array_equal(doms[0].gather_canonical(), doms[1].gather_canonical())
    assert doms[0].counters().as_dict() == doms[1].counters().as_dict()
    assert doms[0].steps_done == doms[1].steps_done == 19


@pytest.mark.parametrize("pattern", ["aa", "pull"])
def test_halo_frame_slabs_match_sequential(pattern, gpu_lib):
    """frame_width="halo" on a z-slab decomposition (the weak-scaling
    layout): x/y wrap in-block, the frame is whole z planes, and the
    overlapped driver (loopback NCCL) equals the sequential single-block run."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain, DistributedDomain
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    gf = geometry.packed_bed_flags((16, 12, 24), 0.5, 5.0, 3, periodic=True)
    p = CollisionParams(1.2, "trt", 0.94)
    ref = Domain(gf, (16, 12, 24), st, p, pattern=pattern)
    ref.init_random(2)
    ref.run(6)
    d = DistributedDomain(gf, (16, 12, 8), st, p, pattern=pattern, rank=0, world=1, device=0,
                          loopback=True)
    assert d.frame_width == "halo"
    for e in d.local_engines():
        interior, frame = e.split_lists()
        z = e.fluid_coords[frame, 2]
        assert np.all((z == 0) | (z == 7))
        assert np.array_equal(interior, np.arange(interior[0], interior[-1] + 1))
    d.init_random(2)
    d.run(6, driver="overlapped")
    np.testing.assert_array_equal(d.gather_canonical(), ref.gather_canonical())


def test_gather_macroscopics_compact_and_box_paths(gpu_lib):
    """Domain.gather_macroscopics moves only fluid values for low-porosity
    sparse blocks and whole boxes otherwise; both equal one engine's
    macroscopic_fields bit for bit."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.engine import SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    gf = geometry.riverbed_flags((16, 16, 16), (8, 8, 8), 0.35, 5, 0.03)
    p = CollisionParams(1.3, "trt", 0.9)
    d = Domain(gf, (8, 8, 8), st, p, pattern="aa", frame_width=1)
    assert {b.porosity < 0.5 for b in d.blocks.values()} == {True, False}
    one = SparseEngine(gf, st, p, "aa")
    d.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
    one.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
    # an even step count: mid-pair (odd) readouts are block-local in the
    # reference too (domain.py:246-255 gathers without an exchange)
    d.run(6)
    for _ in range(6):
        one.refresh_boundary(one.parity)
        one.step()
        one.finish_step()
    rho_d, u_d = d.gather_macroscopics()
    rho_1, u_1 = one.macroscopic_fields()
    np.testing.assert_array_equal(rho_d, rho_1)
    np.testing.assert_array_equal(u_d, u_1)
    # at odd parity the compact path still equals the per-block box path
    d.run(1)
    rho_d, u_d = d.gather_macroscopics()
    rho_b, u_b = np.zeros_like(rho_d), np.zeros_like(u_d)
    for blk in d.local_blocks():
        r, v = blk.engine.macroscopic_fields()
        sel = tuple(slice(o, o + 8) for o in reversed(blk.origin))
        rho_b[sel] = r
        u_b[sel] = v
    np.testing.assert_array_equal(rho_d, rho_b)
    np.testing.assert_array_equal(u_d, u_b)


def test_overlap_ratio_tracing(gpu_lib):
    """domain.py:236-239 / exchange.py:333-374: with tracing on, each step adds
    (interior span, exchange window) from CUDA events; the overlapped driver
    with remote (loopback NCCL) edges reports a ratio in (0, 1], the
    sequential driver 0, and an untraced domain 0."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import DistributedDomain
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    gf = geometry.packed_bed_flags((32, 32, 64), 0.5, 6.0, 2, periodic=True)
    p = CollisionParams(1.2, "trt", 0.9)
    d = DistributedDomain(gf, (32, 32, 32), st, p, pattern="aa", rank=0, world=1, device=0,
                          loopback=True)
    d.init_random(1)
    d.run(4, driver="overlapped")
    assert d.overlap_ratio() == 0.0  # nothing traced yet
    d.trace = True
    d.run(6, driver="overlapped")
    r = d.overlap_ratio()
    assert 0.0 < r <= 1.0 and len(d.overlap_samples) == 6
    d.overlap_samples.clear()
    d.run(2, driver="sequential")
    assert d.overlap_ratio() == 0.0 and len(d.overlap_samples) == 2
