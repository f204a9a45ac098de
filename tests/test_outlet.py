"""Fixed-density outlet (extension; the reference has no outlet, SURVEY F12 —
parity UNPINNED).  CPU: the oracle's restatement gives a pressure-driven
Poiseuille flow; GPU: the CUDA refresh kernel is bit-identical to it, and a
UBB-inlet / outlet channel reaches a steady through-flow."""

import numpy as np
import pytest

from oracle.sparse_ref import OracleSparseEngine
from paper_2408_06880_b200.collision import CollisionParams
from paper_2408_06880_b200.lattice import make_stencil
from paper_2408_06880_b200.tags import OUTLET, WALL, FaceKind, FaceSpec, make_flags


def pressure_channel(nx, ny, rho_in, rho_out, nz=None):
    inlet = FaceSpec(FaceKind.WALL, density=rho_in)
    outlet = FaceSpec(FaceKind.WALL, density=rho_out)
    faces = [(inlet, outlet), (WALL, WALL)] + ([(WALL, WALL)] if nz else [])
    return make_flags((nx, ny) + ((nz,) if nz else ()), faces)


def drive(e, n):
    for _ in range(n):
        e.refresh_boundary(e.parity)
        e.step()
        e.finish_step()


def test_outlet_tags_and_density_payload():
    fl = pressure_channel(6, 4, 1.01, 0.99)
    assert fl.tag_at((-1, 1)) == OUTLET and fl.tag_at((6, 2)) == OUTLET
    assert fl.ubb_at((-1, 1))[0] == 1.01 and fl.ubb_at((6, 2))[0] == 0.99
    # x is padded last, so the outlet face owns the corners (flags.py:12-15 rule)
    assert fl.tag_at((-1, -1)) == OUTLET
    eng = OracleSparseEngine(fl, make_stencil("d2q9"), CollisionParams(1.0), "aa")
    # every cell next to an outlet face reads 3 directions from it
    assert eng._lists["n_out"] == 2 * 3 * 4


@pytest.mark.parametrize("pattern", ["aa", "pull"])
def test_pressure_driven_poiseuille(pattern):
    nx, ny = 40, 15
    omega = 1.0
    drho = 0.002
    fl = pressure_channel(nx, ny, 1.0 + drho / 2, 1.0 - drho / 2)
    st = make_stencil("d2q9")
    eng = OracleSparseEngine(fl, st, CollisionParams(omega), pattern)
    eng.init_equilibrium()
    drive(eng, 3000)
    _, u = eng.macroscopic_fields()
    ux = u[:, :, 0]
    flux = ux.sum(axis=0)
    np.testing.assert_allclose(flux, flux.mean(), rtol=0.01)  # mass conservation along x
    prof = ux[:, nx // 2]
    y = np.arange(ny) + 0.5
    shape = y * (ny - y)
    fit = (prof * shape).sum() / (shape * shape).sum()
    assert np.abs(prof - fit * shape).max() < 0.03 * prof.max()
    # bulk: Poiseuille maximum from the measured interior pressure gradient
    rho, _ = eng.macroscopic_fields()
    x = np.arange(nx) + 0.5
    slope, icpt = np.polyfit(x[5:-5], rho[ny // 2, 5:-5], 1)
    nu = (1.0 / omega - 0.5) / 3.0
    umax_theory = (-slope / 3.0) * ny * ny / (8.0 * nu)
    assert abs(prof.max() - umax_theory) < 0.02 * umax_theory
    # boundaries: the imposed density drop is reproduced (anti-bounce-back
    # with first-order velocity estimate: within 10%)
    assert abs((-slope * nx) - drho) < 0.1 * drho


@pytest.mark.gpu
@pytest.mark.parametrize("name,pattern,model", [("d3q19", "aa", "trt"), ("d3q19", "pull", "srt"),
                                                ("d2q9", "aa", "srt"), ("d3q27", "aa", "cumulant")])
def test_gpu_outlet_bitwise_equals_restatement(name, pattern, model, gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.engine import SparseEngine

    st = make_stencil(name)
    dims = (14, 9) if st.dim == 2 else (12, 8, 7)
    inlet = FaceSpec(FaceKind.WALL, velocity=(0.02,) + (0.0,) * (st.dim - 1))
    outlet = FaceSpec(FaceKind.WALL, density=1.0)
    faces = [(inlet, outlet)] + [(WALL, WALL)] * (st.dim - 1)
    fl = make_flags(dims, faces, solid=geometry.random_obstacles(dims, 0.85, 3))
    p = CollisionParams(1.3, model, 0.9 if model == "trt" else None)
    gpu = SparseEngine(fl, st, p, pattern)
    cpu = OracleSparseEngine(fl, st, p, pattern)
    assert gpu.n_outlet_slots == cpu._lists["n_out"] > 0
    gpu.init_equilibrium()
    cpu.init_equilibrium()
    drive(gpu, 25)
    drive(cpu, 25)
    np.testing.assert_array_equal(gpu.canonical_state(), cpu.canonical_state())
    rg, ug = gpu.macroscopic_fields()
    rc, uc = cpu.macroscopic_fields()
    np.testing.assert_array_equal(rg, rc)
    np.testing.assert_array_equal(ug, uc)


@pytest.mark.gpu
@pytest.mark.parametrize("pattern", ["aa", "pull"])
def test_gpu_outlets_in_block_group_equal_single_block(pattern, gpu_lib):
    """Several blocks with inlet and outlet faces run as one block group
    (batched UBB and outlet refresh, group sweeps): same bits as one engine."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.domain import Domain
    from paper_2408_06880_b200.engine import SparseEngine

    st = make_stencil("d3q19")
    dims = (24, 8, 8)
    inlet = FaceSpec(FaceKind.WALL, velocity=(0.02, 0.0, 0.0))
    outlet = FaceSpec(FaceKind.WALL, density=1.0)
    fl = make_flags(dims, [(inlet, outlet), (WALL, WALL), (WALL, WALL)],
                    solid=geometry.random_obstacles(dims, 0.85, 5))
    p = CollisionParams(1.3, "trt", 0.9)
    one = SparseEngine(fl, st, p, pattern)
    one.init_equilibrium()
    drive(one, 12)
    dom = Domain(fl, (8, 8, 8), st, p, pattern=pattern, frame_width=1)
    assert dom._group is not None and len(dom.local_engines()) == 3
    dom.init_equilibrium()
    dom.run(12, driver="overlapped")
    rho_d, u_d = dom.gather_macroscopics()
    rho_1, u_1 = one.macroscopic_fields()
    np.testing.assert_array_equal(rho_d, rho_1)
    np.testing.assert_array_equal(u_d, u_1)
    box = dom.gather_canonical()  # (q, z, y, x) over the box
    x, y, z = one.fluid_coords.T
    np.testing.assert_array_equal(box[:, z, y, x], one.canonical_state())
