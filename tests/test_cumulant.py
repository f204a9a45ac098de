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


# ---------------------------------------------------------------- general rates
# (bulk and higher-order rates exposed, an independent
# restatement from Geier et al. 2015 -- oracle/cumulant_geier.py -- and
# physical validation: shear / bulk wave decay, Galilean invariance)

HIGHER = (0.9, 1.3, 1.1, 1.6, 0.8, 1.2, 1.4, 0.7)


def test_independent_restatement_matches_closed_form():
    """Two derivations of the same model agree to rounding: the closed form
    (higher rates 1, cumulant_ref = the kernel's op order) and the general
    partition-based restatement (cumulant_geier), for several bulk rates."""
    from oracle.cumulant_geier import collide_general

    f, _, _ = _state(400, 11, amp=0.03)
    for omega, bulk in ((1.3, 1.0), (0.9, 0.6), (1.8, 1.5)):
        a = collide_general(f, omega, bulk, None, ST)
        b = cumulant_collide(f, omega, ST, bulk)
        assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()


def test_general_rates_relax_each_cumulant_group():
    from oracle.cumulant_geier import collide_general, cumulants_of

    f, _, _ = _state(300, 12, amp=0.03)
    omega, bulk = 1.25, 0.8
    w3, w4, w5, w6, w7, w8, w9, w10 = HIGHER
    _, K0 = cumulants_of(f, ST)
    _, K1 = cumulants_of(collide_general(f, omega, bulk, HIGHER, ST), ST)
    tol = 1e-12

    def close(a, b):
        assert np.abs(a - b).max() <= tol

    close(K1[(1, 1, 0)], (1 - omega) * K0[(1, 1, 0)])
    close(K1[(2, 0, 0)] - K1[(0, 2, 0)], (1 - omega) * (K0[(2, 0, 0)] - K0[(0, 2, 0)]))
    tr = lambda K: K[(2, 0, 0)] + K[(0, 2, 0)] + K[(0, 0, 2)]  # noqa: E731
    close(tr(K1) - 1.0, (1 - bulk) * (tr(K0) - 1.0))
    close(K1[(1, 2, 0)] + K1[(1, 0, 2)], (1 - w3) * (K0[(1, 2, 0)] + K0[(1, 0, 2)]))
    close(K1[(2, 1, 0)] - K1[(0, 1, 2)], (1 - w4) * (K0[(2, 1, 0)] - K0[(0, 1, 2)]))
    close(K1[(1, 1, 1)], (1 - w5) * K0[(1, 1, 1)])
    iso = lambda K: K[(2, 2, 0)] + K[(2, 0, 2)] + K[(0, 2, 2)]  # noqa: E731
    close(iso(K1), (1 - w7) * iso(K0))
    dev = lambda K: K[(2, 2, 0)] - 2 * K[(2, 0, 2)] + K[(0, 2, 2)]  # noqa: E731
    close(dev(K1), (1 - w6) * dev(K0))
    close(K1[(2, 1, 1)], (1 - w8) * K0[(2, 1, 1)])
    close(K1[(1, 2, 2)], (1 - w9) * K0[(1, 2, 2)])
    close(K1[(2, 2, 2)], (1 - w10) * K0[(2, 2, 2)])
    # conserved: mass, momentum (first cumulants = velocity)
    rho0 = f.sum(0)
    out = collide_general(f, omega, bulk, HIGHER, ST)
    np.testing.assert_allclose(out.sum(0), rho0, rtol=1e-14)
    close(K1[(1, 0, 0)], K0[(1, 0, 0)])


def test_general_equilibrium_is_a_fixed_point():
    from oracle.cumulant_geier import collide_general, equilibrium

    _, rho, u = _state(200, 13)
    feq = equilibrium(rho, u, ST)
    np.testing.assert_allclose(feq, product_equilibrium(rho, u, ST), rtol=1e-13, atol=1e-16)
    out = collide_general(feq, 1.4, 0.7, HIGHER, ST)
    np.testing.assert_allclose(out, feq, rtol=1e-12, atol=1e-16)


def _wave_engine(make_engine, n, params, rho_mode, uy_mode, ux0=0.0):
    """1-d periodic (n, 2, 2) box; initial equilibrium with
    rho = 1 + rho_mode(x), u = (ux0, uy_mode(x), 0)."""
    from paper_2408_06880_b200.tags import PERIODIC, make_flags

    fl = make_flags((n, 2, 2), [(PERIODIC, PERIODIC)] * 3)
    eng = make_engine(fl, ST, params, "aa")
    x = eng.fluid_coords[:, 0].astype(float) + 0.5
    rho = 1.0 + rho_mode(x)
    eng.init_canonical(product_equilibrium(rho, [np.full_like(x, ux0), uy_mode(x), 0.0 * x], ST))
    cells = np.ravel_multi_index(eng.fluid_coords[:, ::-1].T, (2, 2, n))
    return eng, x, cells


def _advance(eng, steps):
    for _ in range(steps):
        eng.refresh_boundary(eng.parity)
        eng.step()
        eng.finish_step()


def measured_shear_viscosity(make_engine, params, n=48, t1=80, t2=400, ux0=0.0, amp=1e-4):
    """Shear wave u_y ~ sin(k (x - U t)): nu from the decay of its amplitude
    (projection on the advected sine and cosine, so a background velocity U
    along x -- the Galilean-invariance check -- moves the mode, not the
    measurement)."""
    k = 2 * np.pi / n
    eng, x, cells = _wave_engine(make_engine, n, params, lambda x: 0.0 * x,
                                 lambda x: amp * np.sin(k * x), ux0)
    done, amps = 0, []
    for t in (t1, t2):
        _advance(eng, t - done)
        done = t
        _, u = eng.macroscopic_fields()
        uy = u[..., 1].reshape(-1)[cells]
        ph = k * (x - ux0 * t)
        amps.append(np.hypot((uy * np.sin(ph)).sum(), (uy * np.cos(ph)).sum()) / (0.5 * x.size))
    return -np.log(amps[1] / amps[0]) / (k * k * (t2 - t1))


def measured_sound_attenuation(make_engine, params, n=64, steps=600, amp=1e-4):
    """Standing density wave rho = 1 + A cos(kx): the acoustic energy
    sum(c_s^2 rho'^2 + u^2) / 2 decays as exp(-2 alpha t); alpha / k^2 from a
    least-squares fit of log E over every step (averages the potential /
    kinetic exchange)."""
    k = 2 * np.pi / n
    eng, x, cells = _wave_engine(make_engine, n, params, lambda x: amp * np.cos(k * x),
                                 lambda x: 0.0 * x)
    ts, logs = [], []
    for t in range(1, steps + 1):
        _advance(eng, 1)
        if t < 50 or t % 2:
            continue  # AA: read at even steps; skip the start-up transient
        rho, u = eng.macroscopic_fields()
        r = rho.reshape(-1)[cells] - 1.0
        ux = u[..., 0].reshape(-1)[cells]
        ts.append(t)
        logs.append(np.log(((r * r) / 3.0 + ux * ux).sum()))
    slope = np.polyfit(ts, logs, 1)[0]
    return -slope / 2.0 / (k * k)


def _theory(omega, bulk):
    nu = (1.0 / omega - 0.5) / 3.0
    zeta = 2.0 / 9.0 * (1.0 / bulk - 0.5)
    return nu, 2.0 * nu / 3.0 + zeta / 2.0


def _oracle_engine(*a, **k):
    from oracle.sparse_ref import OracleSparseEngine

    return OracleSparseEngine(*a, **k)


@pytest.mark.parametrize("omega,bulk", [(1.2, 1.0), (1.2, 0.6), (1.6, 1.5)])
def test_sound_wave_attenuation_follows_bulk_viscosity(omega, bulk):
    """alpha = k^2 (2 nu / 3 + zeta / 2), zeta = 2/9 (1/w2 - 1/2) (isothermal
    linearised Navier-Stokes); 1 % tolerance (lattice dispersion at k dx =
    0.1 and the energy oscillation left after the fit)."""
    from paper_2408_06880_b200.collision import CollisionParams

    got = measured_sound_attenuation(_oracle_engine, CollisionParams(omega, "cumulant",
                                                                     bulk_omega=bulk))
    want = _theory(omega, bulk)[1]
    assert abs(got - want) < 0.01 * want, (got, want)


def test_shear_viscosity_with_general_rates():
    """Higher-order rates leave the shear viscosity (1/w1 - 1/2)/3 (1 %)."""
    from paper_2408_06880_b200.collision import CollisionParams

    p = CollisionParams(1.4, "cumulant", bulk_omega=0.9, higher_omegas=HIGHER)
    nu = measured_shear_viscosity(_oracle_engine, p, t2=300)
    want = _theory(1.4, 0.9)[0]
    assert abs(nu - want) < 0.01 * want, (nu, want)


# ---------------------------------------------------------------- GPU, general rates


def _gpu_engine(*a, **k):
    from paper_2408_06880_b200.engine import SparseEngine

    return SparseEngine(*a, **k)


@pytest.mark.gpu
@pytest.mark.parametrize("pattern", ["aa", "pull"])
def test_gpu_general_rates_match_independent_restatement(pattern, gpu_lib):
    """CUDA general-rate kernel vs oracle/cumulant_geier.py on a riverbed
    with walls and a moving lid, 6 steps: max |diff| <= 1e-12 * max |f|
    (different derivations, so rounding differs; not bitwise)."""
    from oracle.sparse_ref import OracleSparseEngine
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import SparseEngine

    fl = geometry.riverbed_flags((12, 10, 12), (6, 5, 6), 0.5, 4, 0.03)
    p = CollisionParams(1.5, "cumulant", bulk_omega=0.8, higher_omegas=HIGHER)
    gpu = SparseEngine(fl, ST, p, pattern)
    cpu = OracleSparseEngine(fl, ST, p, pattern)
    f, _, _ = _state(gpu.n_fluid, 21, amp=0.01)
    gpu.init_canonical(f)
    cpu.init_canonical(f)
    for _ in range(6):
        for e in (gpu, cpu):
            e.refresh_boundary(e.parity)
            e.step()
            e.finish_step()
    a, b = gpu.canonical_state(), cpu.canonical_state()
    assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()


@pytest.mark.gpu
def test_gpu_general_path_with_unit_rates_equals_closed_form(gpu_lib):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import SparseEngine

    fl = geometry.riverbed_flags((12, 10, 12), (6, 5, 6), 0.5, 4, 0.03)
    p = CollisionParams(1.5, "cumulant", bulk_omega=0.7)
    fast, gen = SparseEngine(fl, ST, p, "aa"), SparseEngine(fl, ST, p, "aa")
    gen.set_cumulant_rates(0.7, None, force_general=True)
    f, _, _ = _state(fast.n_fluid, 22, amp=0.01)
    for e in (fast, gen):
        e.init_canonical(f)
        e.run(6, use_graph=False)
    a, b = gen.canonical_state(), fast.canonical_state()
    assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()


@pytest.mark.gpu
@pytest.mark.parametrize("omega,bulk", [(1.2, 1.0), (1.2, 0.5), (1.7, 1.6)])
def test_gpu_sound_wave_attenuation(omega, bulk, gpu_lib):
    from paper_2408_06880_b200.collision import CollisionParams

    got = measured_sound_attenuation(_gpu_engine, CollisionParams(omega, "cumulant",
                                                                  bulk_omega=bulk),
                                     n=128, steps=1200)
    want = _theory(omega, bulk)[1]
    assert abs(got - want) < 0.01 * want, (got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("higher", [None, HIGHER])
def test_gpu_galilean_invariance_at_mach_0_1(higher, gpu_lib):
    """Shear-wave viscosity at rest and advected at Ma = U / c_s = 0.1 along
    the wave vector: both within 1 % of (1/w1 - 1/2)/3 and within 0.5 % of
    each other."""
    from paper_2408_06880_b200.collision import CollisionParams

    p = CollisionParams(1.6, "cumulant", bulk_omega=1.0, higher_omegas=higher)
    U = 0.1 / np.sqrt(3.0)
    nu0 = measured_shear_viscosity(_gpu_engine, p, n=96, t1=200, t2=2000)
    nuU = measured_shear_viscosity(_gpu_engine, p, n=96, t1=200, t2=2000, ux0=U)
    want = _theory(1.6, 1.0)[0]
    assert abs(nu0 - want) < 0.01 * want, (nu0, want)
    assert abs(nuU - want) < 0.01 * want, (nuU, want)
    assert abs(nuU - nu0) < 0.005 * want, (nu0, nuU)
