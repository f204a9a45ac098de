"""Cumulant collision (D3Q27): the CPU restatement's physics (CPU) and the
CUDA kernel's bitwise agreement with it (GPU).  Parity with the reference
is UNPINNED — the reference has no cumulant model."""

import numpy as np
import pytest

from oracle.cumulant_ref import cumulant_collide, moments_seedless, product_equilibrium
from paper_2408_06880_b200.lattice import make_stencil

ST = make_stencil("d3q27")


def _state(n, seed, amp=0.02):
    rng = np.random.default_rng(seed)
    rho = 1.0 + amp * rng.standard_normal(n)
    u = [amp * rng.standard_normal(n) for _ in range(3)]
    f = product_equilibrium(rho, u, ST)
    return f * (1.0 + 0.05 * rng.standard_normal(f.shape)), rho, u


def test_mass_and_momentum_are_conserved():
    f, _, _ = _state(500, 1)
    for omega in (0.6, 1.0, 1.3, 1.9):
        out = cumulant_collide(f, omega, ST)
        rho0, u0 = moments_seedless(f, ST)
        rho1, u1 = moments_seedless(out, ST)
        np.testing.assert_allclose(rho1, rho0, rtol=2e-15)
        for a in range(3):
            np.testing.assert_allclose(rho1 * u1[a], rho0 * u0[a], atol=2e-16 * 27)


def test_product_equilibrium_is_a_fixed_point():
    _, rho, u = _state(300, 2)
    feq = product_equilibrium(rho, u, ST)
    for omega in (0.7, 1.5):
        np.testing.assert_allclose(cumulant_collide(feq, omega, ST), feq, rtol=1e-13, atol=1e-16)


def test_omega_one_relaxes_to_the_equilibrium():
    f, _, _ = _state(300, 3)
    rho, u = moments_seedless(f, ST)
    np.testing.assert_allclose(cumulant_collide(f, 1.0, ST), product_equilibrium(rho, u, ST),
                               rtol=1e-13, atol=1e-16)


def test_second_order_moments_relax_with_omega():
    f, _, _ = _state(200, 4)
    omega = 1.4
    out = cumulant_collide(f, omega, ST)
    c = ST.c.astype(float)

    def central(g):
        rho, u = moments_seedless(g, ST)
        d = [c[:, a, None] - u[a][None, :] for a in range(3)]
        return rho, u, {(a, b): (d[a] * d[b] * g).sum(0) for a in range(3) for b in range(3)}

    _, _, k0 = central(f)
    _, _, k1 = central(out)
    np.testing.assert_allclose(k1[(0, 1)], (1 - omega) * k0[(0, 1)], atol=1e-14)
    np.testing.assert_allclose(k1[(0, 0)] - k1[(1, 1)], (1 - omega) * (k0[(0, 0)] - k0[(1, 1)]),
                               atol=1e-14)
    rho, _ = moments_seedless(f, ST)
    np.testing.assert_allclose(k1[(0, 0)] + k1[(1, 1)] + k1[(2, 2)], rho, rtol=1e-13)


def _shear_wave_decay(omega, n=32, t1=100, t2=300, amp=1e-4):
    """Periodic 1-d shear wave u_y(x) = A sin(kx) driven with the oracle
    engine; the kinematic viscosity from the decay between steps t1 and t2
    (after the start-up transient of the equilibrium initial state)."""
    from oracle.sparse_ref import OracleSparseEngine
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.tags import PERIODIC, make_flags

    fl = make_flags((n, 2, 2), [(PERIODIC, PERIODIC)] * 3)
    eng = OracleSparseEngine(fl, ST, CollisionParams(omega, "cumulant"), "aa")
    x = eng.fluid_coords[:, 0].astype(float)
    k = 2 * np.pi / n
    mode = np.sin(k * (x + 0.5))
    zero = np.zeros_like(x)
    eng.init_canonical(product_equilibrium(np.ones_like(x), [zero, amp * mode, zero], ST))
    cells = np.ravel_multi_index(eng.fluid_coords[:, ::-1].T, (2, 2, n))

    def amplitude():
        _, u = eng.macroscopic_fields()
        return (u[..., 1].reshape(-1)[cells] * mode).sum() / (mode ** 2).sum()

    done, amps = 0, []
    for target in (t1, t2):
        while done < target:
            eng.refresh_boundary(eng.parity)
            eng.step()
            eng.finish_step()
            done += 1
        amps.append(amplitude())
    return -np.log(amps[1] / amps[0]) / (k * k * (t2 - t1))


@pytest.mark.parametrize("omega", [0.8, 1.2, 1.7, 1.9])
def test_shear_wave_viscosity(omega):
    nu = _shear_wave_decay(omega)
    assert abs(nu - (1.0 / omega - 0.5) / 3.0) < 0.01 * (1.0 / omega - 0.5) / 3.0 + 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("pattern", ["aa", "pull"])
def test_gpu_cumulant_bitwise_equals_cpu_restatement(pattern, gpu_lib):
    from oracle.sparse_ref import OracleSparseEngine
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import SparseEngine

    fl = geometry.riverbed_flags((12, 10, 12), (6, 5, 6), 0.5, 4, 0.03)
    p = CollisionParams(1.6, "cumulant")
    gpu = SparseEngine(fl, ST, p, pattern)
    cpu = OracleSparseEngine(fl, ST, p, pattern)
    f, _, _ = _state(gpu.n_fluid, 9, amp=0.01)
    gpu.init_canonical(f)
    cpu.init_canonical(f)
    for _ in range(7):
        for e in (gpu, cpu):
            e.refresh_boundary(e.parity)
            e.step()
            e.finish_step()
    np.testing.assert_array_equal(gpu.canonical_state(), cpu.canonical_state())
