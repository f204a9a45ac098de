"""CUDA engine parity: lists, states and fields bit-identical to the
reference's golden vectors and to the oracle; protocol behaviour (errors,
counters, refresh idempotence, split sweeps) as in the reference's
tests/test_sparse.py."""

import hashlib
import math
import os

import numpy as np
import pytest

from conftest import drive, flags_of, golden_files, load_golden, params_of, seed_values, stencil_of

pytestmark = pytest.mark.gpu

ENGINE = golden_files("engine")
BED = golden_files("bed")


def _id(p):
    return os.path.basename(p)[:-4]


def _engine(*a, **k):
    from paper_2408_06880_b200.engine import SparseEngine

    return SparseEngine(*a, **k)


@pytest.mark.parametrize("path", ENGINE, ids=_id)
def test_lists_bit_exact(path, gpu_lib):
    rec = load_golden(path)
    eng = _engine(flags_of(rec), stencil_of(rec), params_of(rec), "aa",
                  frame_width=int(rec["frame_width"]))
    assert eng.idx.dtype == np.uint32
    assert np.array_equal(eng.idx, rec["idx"])
    assert np.array_equal(eng.base, rec["base"])
    assert eng.total_slots == int(rec["total_slots"])
    assert np.array_equal(eng.fluid_coords, rec["fluid_coords"])
    b = eng.export_boundary_lists()
    assert np.array_equal(b["ubb_slots"], rec["ubb_slots"])
    assert np.array_equal(b["ubb_partner"], rec["ubb_partner"])
    assert np.array_equal(b["ubb_corr"], rec["ubb_corr"])
    assert np.array_equal(b["ghost_q"], rec["ghost_q"])
    assert np.array_equal(b["ghost_pflat"], rec["ghost_pflat"])
    assert np.array_equal(b["ghost_slot"], rec["ghost_slot"])
    interior, frame = eng.split_lists()
    assert np.array_equal(interior, rec["interior"]) and np.array_equal(frame, rec["frame"])


@pytest.mark.parametrize("pattern", ["pull", "aa"])
@pytest.mark.parametrize("path", ENGINE, ids=_id)
def test_states_bit_exact(path, pattern, gpu_lib):
    rec = load_golden(path)
    fl, st, p = flags_of(rec), stencil_of(rec), params_of(rec)
    for steps in rec["steps_list"]:
        eng = _engine(fl, st, p, pattern)
        eng.init_canonical(rec["values0"])
        drive(eng, int(steps), rec["ghost_slot"], rec["ghost_fill"])
        np.testing.assert_array_equal(eng.canonical_state(), rec[f"{pattern}_{steps}_state"])
        rho, u = eng.macroscopic_fields()
        np.testing.assert_array_equal(rho, rec[f"{pattern}_{steps}_rho"])
        np.testing.assert_array_equal(u, rec[f"{pattern}_{steps}_u"])


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("path", BED, ids=_id)
def test_bed_runs_bit_exact(path, gpu_lib):
    """C1 = BASELINE configs[0] (64^3 channel bed, D3Q19 SRT, 100 steps) and
    the C2 law at 48^3 (D3Q19 TRT AA): SHA-256 of the whole final state
    equals the reference's."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil
    from paper_2408_06880_b200.tags import PERIODIC, make_flags
    from test_oracle_golden import init_random_values

    rec = load_golden(path)
    dims = tuple(int(d) for d in rec["dims"])
    d = float(rec["diameter"])
    centers = geometry.sphere_centers(dims, d, int(rec["count"]), int(rec["seed"]))
    solid = geometry.voxelize_spheres(dims, centers, d, device=0)  # CUDA rasterizer
    if bool(rec["channel"]):
        fl = geometry.channel_flags(dims, solid=solid)
    else:
        fl = make_flags(dims, [(PERIODIC, PERIODIC)] * 3, solid=solid)
    assert _sha(fl.tags) == str(rec["tags_sha"])
    st = make_stencil(str(rec["stencil"]))
    lam = float(rec["lambda_odd"])
    p = CollisionParams(float(rec["omega"]), str(rec["model"]), None if math.isnan(lam) else lam)
    eng = _engine(fl, st, p, str(rec["pattern"]))
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


@pytest.mark.parametrize("path", BED[:1], ids=_id)
def test_run_graph_matches_python_loop(path, gpu_lib):
    """engine.run (device loop + CUDA graph) == step-by-step driving."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil

    fl = geometry.packed_bed_flags((32, 24, 20), 0.5, 6.0, 3, channel=True)
    st = make_stencil("d3q19")
    p = CollisionParams(1.3, "trt", 0.9)
    for pattern in ("aa", "pull"):
        a = _engine(fl, st, p, pattern)
        b = _engine(fl, st, p, pattern)
        v = seed_values(fl, st, 5)
        a.init_canonical(v)
        b.init_canonical(v)
        a.run(1, use_graph=False)
        b.run(1, use_graph=False)
        a.run(9, use_graph=True)
        drive(b, 9)
        np.testing.assert_array_equal(a.canonical_state(), b.canonical_state())
        assert a.parity == b.parity and a.counters.as_dict() == b.counters.as_dict()


# -- protocol behaviour (reference tests/test_sparse.py) ------------------------------


def _d2q9():
    from paper_2408_06880_b200.lattice import make_stencil

    return make_stencil("d2q9")


def test_slot_budget_and_walls(gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    eng = _engine(geometry.obstacle_flags((6, 5, 4), 0.7, 5), st, CollisionParams(1.0))
    assert eng.n_ubb_slots == 0 and eng.n_ghost_slots == 0
    assert eng.total_slots == st.q * eng.n_fluid
    eng = _engine(geometry.channel_flags((8, 5)), _d2q9(), CollisionParams(1.0))
    assert eng.n_ubb_slots == 0 and eng.total_slots == 9 * eng.n_fluid
    eng = _engine(geometry.couette_flags((8, 5), 0.05), _d2q9(), CollisionParams(1.0))
    assert eng.n_ubb_slots == 3 * 8 and eng.total_slots == 9 * eng.n_fluid + 24
    assert eng.idx.shape == (8, eng.n_fluid)


def test_unrefreshed_moving_wall_slot_is_loud(gpu_lib):
    from paper_2408_06880_b200 import errors, geometry
    from paper_2408_06880_b200.collision import CollisionParams

    eng = _engine(geometry.couette_flags((8, 5), 0.05), _d2q9(), CollisionParams(1.0))
    eng.init_equilibrium()
    with pytest.raises(errors.NumericalInstabilityError):
        eng.step()


def test_refresh_is_idempotent(gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams

    st, p = _d2q9(), CollisionParams(1.2)
    fl = geometry.couette_flags((8, 5), 0.05)
    v = seed_values(fl, st, 9)
    a, b = _engine(fl, st, p, "aa"), _engine(fl, st, p, "aa")
    a.init_canonical(v)
    b.init_canonical(v)
    for _ in range(3):
        a.refresh_boundary(a.parity)
        a.step()
        a.finish_step()
        b.refresh_boundary(b.parity)
        b.refresh_boundary(b.parity)
        b.step()
        b.finish_step()
    np.testing.assert_array_equal(a.canonical_state(), b.canonical_state())


def test_counters(gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil

    st = _d2q9()
    fl = geometry.make_flags((12, 8), [(geometry.PERIODIC, geometry.PERIODIC),
                                       (geometry.WALL, geometry.WALL)],
                             solid=geometry.random_obstacles((12, 8), 0.6, 3))
    eng = _engine(fl, st, CollisionParams(1.0), "pull")
    eng.init_equilibrium()
    drive(eng, 3)
    nf = eng.n_fluid
    assert eng.counters.cells_visited == 3 * nf
    assert eng.counters.pdf_accesses == 3 * 2 * 9 * nf
    assert eng.counters.idx_reads == 3 * 8 * nf
    aa = _engine(fl, st, CollisionParams(1.0), "aa")
    aa.init_equilibrium()
    drive(aa, 1)
    assert aa.counters.idx_reads == 8 * nf
    drive(aa, 1)
    assert aa.counters.idx_reads == 8 * nf
    st19 = make_stencil("d3q19")
    fl3 = geometry.obstacle_flags((6, 5, 4), 0.5, 2)
    pull = _engine(fl3, st19, CollisionParams(1.0), "pull")
    aa3 = _engine(fl3, st19, CollisionParams(1.0), "aa")
    assert pull.pdf_element_count() == 2 * 19 * pull.n_fluid
    assert aa3.pdf_element_count() == 19 * aa3.n_fluid
    assert pull.idx_element_count() == 18 * pull.n_fluid


@pytest.mark.parametrize("pattern", ["pull", "aa"])
def test_interior_plus_frame_composes_bitwise(pattern, gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    fl = geometry.packed_bed_flags((20, 16, 12), 0.6, 5.0, 1, channel=True)
    p = CollisionParams(1.3, "trt", 0.8)
    v = seed_values(fl, st, 21)
    whole = _engine(fl, st, p, pattern, frame_width=1)
    split = _engine(fl, st, p, pattern, frame_width=(2, 1, 3))
    whole.init_canonical(v)
    split.init_canonical(v)
    for _ in range(4):
        whole.refresh_boundary(whole.parity)
        whole.step("all")
        whole.finish_step()
        split.refresh_boundary(split.parity)
        split.step("interior")
        split.step("frame")
        split.finish_step()
    np.testing.assert_array_equal(whole.canonical_state(), split.canonical_state())
    assert split.n_interior + split.n_frame == split.n_fluid


@pytest.mark.parametrize("widths", [(0, 0, 1), (0, 0, 2), (1, 0, 0), (0, 2, 1), (0, 0, 0)])
@pytest.mark.parametrize("pattern", ["pull", "aa"])
def test_halo_frame_widths(widths, pattern, gpu_lib):
    """HaloWidths (0 = no frame on that axis, domain-driver extension):
    frame = cells within the width of the faces of the non-zero axes;
    z-only frames are a cid prefix + suffix (contiguous interior range),
    others use the frame bitmask; either way interior + frame == whole."""
    from paper_2408_06880_b200 import errors, geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import HaloWidths
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    fl = geometry.packed_bed_flags((20, 16, 12), 0.6, 5.0, 2, periodic=True)
    p = CollisionParams(1.3, "trt", 0.8)
    v = seed_values(fl, st, 5)
    whole = _engine(fl, st, p, pattern)
    split = _engine(fl, st, p, pattern, frame_width=HaloWidths(widths))
    coords = split.fluid_coords
    want = np.zeros(split.n_fluid, bool)
    for a, w in enumerate(widths):
        if w:
            want |= (coords[:, a] < w) | (coords[:, a] >= fl.dims[a] - w)
    interior, frame = split.split_lists()
    np.testing.assert_array_equal(frame, np.flatnonzero(want))
    np.testing.assert_array_equal(interior, np.flatnonzero(~want))
    whole.init_canonical(v)
    split.init_canonical(v)
    for _ in range(4):
        whole.refresh_boundary(whole.parity)
        whole.step("all")
        whole.finish_step()
        split.refresh_boundary(split.parity)
        split.step("interior")
        split.step("frame")
        split.finish_step()
    np.testing.assert_array_equal(whole.canonical_state(), split.canonical_state())
    with pytest.raises(errors.ConfigurationError):
        _engine(fl, st, p, pattern, frame_width=(0, 0, 1))  # reference rule: >= 1


def test_errors(gpu_lib):
    from paper_2408_06880_b200 import errors, geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.tags import FLUID

    st = _d2q9()
    with pytest.raises(errors.ConfigurationError):
        _engine(geometry.channel_flags((6, 4)), st, CollisionParams(1.0), pattern="push")
    with pytest.raises(errors.ConfigurationError):
        _engine(geometry.obstacle_flags((4, 4, 4), 1.0, 0), st, CollisionParams(1.0))
    with pytest.raises(errors.EmptyBlockError):
        _engine(geometry.channel_flags((6, 4), solid=np.ones((4, 6), bool)), st, CollisionParams(1.0))
    eng = _engine(geometry.channel_flags((6, 4)), st, CollisionParams(1.0))
    with pytest.raises(errors.ConfigurationError):
        eng.init_canonical(np.zeros((9, 5)))
    with pytest.raises(errors.ConfigurationError):
        eng.step("frame")
    with pytest.raises(errors.ProtocolError):
        eng.ghost_slot_index(np.array([[-1, 0]]), np.array([1]))
    fl = geometry.make_flags((12, 8), [(geometry.PERIODIC, geometry.PERIODIC),
                                       (geometry.WALL, geometry.WALL)],
                             solid=geometry.random_obstacles((12, 8), 0.5, 3))
    eng = _engine(fl, st, CollisionParams(1.0))
    solid_rev = np.argwhere(fl.tags_interior != FLUID)[:1]
    with pytest.raises(errors.ProtocolError):
        eng.slot_index(solid_rev[:, ::-1], np.array([1]))


def test_macroscopic_zero_at_solids(gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams

    st = _d2q9()
    fl = geometry.make_flags((12, 8), [(geometry.PERIODIC, geometry.PERIODIC),
                                       (geometry.WALL, geometry.FaceSpec(geometry.FaceKind.WALL,
                                                                         (0.04, 0.0)))],
                             solid=geometry.random_obstacles((12, 8), 0.7, 3))
    eng = _engine(fl, st, CollisionParams(1.0))
    eng.init_canonical(seed_values(fl, st, 6))
    drive(eng, 2)
    rho, u = eng.macroscopic_fields()
    solid = fl.tags_interior != 0
    assert rho[solid].max() == 0.0 and np.abs(u[solid]).max() == 0.0
    assert rho[~solid].min() > 0.5


def test_slot_access_roundtrip(gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams

    st = _d2q9()
    fl = geometry.channel_flags((6, 4))
    eng = _engine(fl, st, CollisionParams(1.0))
    eng.init_equilibrium()
    s = eng.slot_index(np.array([[1, 1], [2, 3]]), np.array([3, 4]))
    assert list(s) == [int(eng.base[3]) + 7, int(eng.base[4]) + 20]
    eng.write_slots(s, np.array([0.5, 0.25]))
    assert list(eng.read_slots(s)) == [0.5, 0.25]


@pytest.mark.parametrize("chunk_mib,threads", [(4, 16), (1, 3)])
def test_staged_host_copies_roundtrip(chunk_mib, threads, gpu_lib):
    """Pageable NumPy arrays above 4 MB go through the multi-threaded pinned
    staging (hostcopy.cu): H2D (init_canonical) and D2H (canonical_state,
    macroscopic_fields) must be exact, including partial chunks and slices
    that do not divide evenly among the threads."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams

    lib = gpu_lib
    lib.slbm_set_tuning(10, chunk_mib)
    lib.slbm_set_tuning(11, threads)
    try:
        st = make_stencil_d3q19()
        fl = geometry.packed_bed_flags((96, 80, 72), 0.4, 8.0, 4, periodic=True)
        p = CollisionParams(1.1, "trt", 0.9)
        eng = _engine(fl, st, p, "aa")
        assert 19 * eng.n_fluid * 8 > (8 << 20)  # well above the staging threshold
        rng = np.random.default_rng(1)
        v = 0.05 + rng.random((19, eng.n_fluid))
        eng.init_canonical(v)  # pageable source: staged H2D
        np.testing.assert_array_equal(eng.canonical_state(), v)
        starts, _ = eng.pdf_layout()
        dev = eng.device_state().cpu().numpy()  # independent path (torch D2H)
        for r in range(19):
            np.testing.assert_array_equal(dev[starts[r]:starts[r] + eng.n_fluid], v[r])
        drive(eng, 3)
        rho, u = eng.macroscopic_fields()
        c = eng.canonical_state()
        x, y, z = eng.fluid_coords.T
        np.testing.assert_allclose(rho[z, y, x], c.sum(axis=0), rtol=1e-12)
        assert rho.sum() > 0 and np.isfinite(u).all()
    finally:
        lib.slbm_set_tuning(10, 4)
        lib.slbm_set_tuning(11, 16)


def test_macroscopic_fields_into_pinned_out(gpu_lib):
    """macroscopic_fields(out=...) with pinned buffers (one DMA) equals the
    default staged path; bad out arrays are rejected."""
    import torch

    from paper_2408_06880_b200 import errors, geometry
    from paper_2408_06880_b200.collision import CollisionParams

    st = make_stencil_d3q19()
    fl = geometry.packed_bed_flags((64, 48, 40), 0.5, 8.0, 2, periodic=True)
    eng = _engine(fl, st, CollisionParams(1.2, "trt", 0.9), "aa")
    eng.init_equilibrium(1.0, np.array([0.01, 0.0, 0.0]))
    drive(eng, 3)
    rho, u = eng.macroscopic_fields()
    shape = rho.shape
    out = (torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy(),
           torch.empty(shape + (3,), dtype=torch.float64, pin_memory=True).numpy())
    r2, u2 = eng.macroscopic_fields(out=out)
    assert r2 is out[0] and u2 is out[1]
    np.testing.assert_array_equal(r2, rho)
    np.testing.assert_array_equal(u2, u)
    with pytest.raises(errors.ConfigurationError):
        eng.macroscopic_fields(out=(np.empty(shape, np.float32), u2))


def make_stencil_d3q19():
    from paper_2408_06880_b200.lattice import make_stencil

    return make_stencil("d3q19")


def test_launch_count_is_graph_aware(gpu_lib):
    """slbm_launch_count (bench.py's gpu_launches): eager steps count their
    kernels, a CUDA-graph replay counts the kernels it captured, the
    resident path one cooperative launch; engine and domain graphs."""
    from paper_2408_06880_b200 import _abi, geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil("d3q19")
    p = CollisionParams(1.3, "trt", 0.9)
    fl = geometry.riverbed_flags((24, 16, 16), (8, 8, 8), 0.5, 7, 0.03)
    eng = _engine(fl, st, p, "aa")
    eng.set_tuning(4, 0)  # no resident kernel
    eng.init_equilibrium()
    c0 = _abi.launch_count()
    drive(eng, 2)
    eager = _abi.launch_count() - c0
    assert eager >= 4  # refresh + sweep + step counter per step (lid: refresh launches)
    c0 = _abi.launch_count()
    eng.run(10, use_graph=True)
    assert _abi.launch_count() - c0 == 5 * eager
    eng.set_tuning(4, 1 << 19)  # resident: n steps in one cooperative launch
    c0 = _abi.launch_count()
    eng.run(10, use_graph=True)
    assert _abi.launch_count() - c0 == 1
    dom = Domain(fl, (8, 8, 8), st, p, pattern="aa", frame_width=1, check="deferred")
    dom.init_equilibrium()
    c0 = _abi.launch_count()
    dom.run(2, driver="overlapped")
    eager = _abi.launch_count() - c0
    dom.run(6, driver="overlapped", use_graph=True)  # capture + first replay
    # run(n) replays (even, odd) pairs; a linked group's last pair of a call
    # is its own graph (with the call-boundary copy), so two more steps per
    # call are exactly one more replay of the mid-run pair
    c0 = _abi.launch_count()
    dom.run(4, driver="overlapped", use_graph=True)
    n4 = _abi.launch_count() - c0
    c0 = _abi.launch_count()
    dom.run(6, driver="overlapped", use_graph=True)
    pair = _abi.launch_count() - c0 - n4
    # one block group: one boundary launch + one sweep per step
    assert pair == 4 and eager >= 4
