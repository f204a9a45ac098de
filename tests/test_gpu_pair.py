"""The experimental temporally blocked AA step pair (pair.cu k_pair, knob 5; engine.run on
sparse AA engines without halo slots) against the per-step path (refresh +
sweep + step counter per step, pinned to the goldens and the oracle):
bit-identical states, counters and first-unstable-step on the fuzz
geometries (every face kind incl. moving walls and outlets, all stencils
and models), on beds large enough for many completion chunks and for
tiles whose writers wrap around periodic faces, from both parities and
over repeated launches (the plan's counters carry over)."""

import ctypes as C

import numpy as np
import pytest

from conftest import seed_values
from test_gpu_fuzz import _case

pytestmark = pytest.mark.gpu

RESIDENT_CAP, PAIR = 4, 5


@pytest.fixture
def knobs(gpu_lib):
    """Per-engine switch to the pair kernel; the kernel is only in builds
    with SLBM_EXPERIMENTAL_PAIR=1 (paper_2408_06880_b200/build.py)."""
    from paper_2408_06880_b200 import _abi

    if _abi.load().slbm_set_tuning(PAIR, 0) != 0 or _abi.load().slbm_set_tuning(PAIR, 1) != 0:
        pytest.skip("pair kernel not built (SLBM_EXPERIMENTAL_PAIR=1)")
    _abi.load().slbm_set_tuning(PAIR, 0)

    def pair_path(eng, on):
        eng.set_tuning(RESIDENT_CAP, 0)  # small engines would run resident
        eng.set_tuning(PAIR, 1 if on else 0)

    return pair_path


def _engines(fl, st, p, seed, **kw):
    from paper_2408_06880_b200.engine import SparseEngine

    a = SparseEngine(fl, st, p, "aa", **kw)
    b = SparseEngine(fl, st, p, "aa", **kw)
    v = seed_values(fl, st, seed)
    a.init_canonical(v)
    b.init_canonical(v)
    return a, b


def _run(eng, n, knobs, pair):
    knobs(eng, pair)
    eng.run(n, use_graph=True)


def _same(a, b):
    np.testing.assert_array_equal(a.canonical_state(), b.canonical_state())
    assert a.parity == b.parity and a.counters.as_dict() == b.counters.as_dict()


@pytest.mark.parametrize("seed", range(24))
def test_pair_matches_per_step_path(seed, knobs):
    fl, st, p, _, _ = _case(seed)
    a, b = _engines(fl, st, p, seed)
    if seed % 2:
        a.run(1, use_graph=False)
        b.run(1, use_graph=False)
    n = 6 + seed % 3
    _run(a, n, knobs, True)
    _run(b, n, knobs, False)
    _same(a, b)
    for _ in range(3):  # repeated launches reuse the plan's counters
        _run(a, 4, knobs, True)
        _run(b, 4, knobs, False)
    _same(a, b)
    ra, ua = a.macroscopic_fields()
    rb, ub = b.macroscopic_fields()
    np.testing.assert_array_equal(ra, rb)
    np.testing.assert_array_equal(ua, ub)


@pytest.mark.parametrize("name,model,dims,channel", [
    ("d3q19", "trt", (96, 80, 72), False),   # periodic bed: wrap tiles on every face
    ("d3q19", "srt", (64, 48, 120), True),   # channel: walls, many chunks along z
    ("d3q27", "cumulant", (48, 40, 64), False),
])
def test_pair_on_beds(name, model, dims, channel, knobs):
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil

    st = make_stencil(name)
    fl = geometry.packed_bed_flags(dims, 0.45, 6.0, 11, channel=channel)
    p = CollisionParams(1.4, model, 0.8 if model == "trt" else None)
    a, b = _engines(fl, st, p, 2)
    for n in (2, 10, 7):
        _run(a, n, knobs, True)
        _run(b, n, knobs, False)
    _same(a, b)


def test_pair_with_moving_lid_and_outlet(knobs):
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil
    from paper_2408_06880_b200.tags import FaceKind, FaceSpec, make_flags

    st = make_stencil("d3q19")
    rng = np.random.default_rng(5)
    dims = (40, 36, 90)
    per = (FaceSpec(FaceKind.PERIODIC), FaceSpec(FaceKind.PERIODIC))
    kinds = [per,
             (FaceSpec(FaceKind.WALL), FaceSpec(FaceKind.WALL, velocity=(0.02, 0.0, 0.01))),
             (FaceSpec(FaceKind.WALL, velocity=(0.0, 0.0, 0.03)),
              FaceSpec(FaceKind.WALL, density=1.0))]
    solid = rng.random(tuple(reversed(dims))) < 0.2
    fl = make_flags(dims, kinds, solid=solid)
    p = CollisionParams(1.2, "trt", 0.25)
    a, b = _engines(fl, st, p, 9)
    assert a.n_ubb_slots > 0
    for n in (4, 9, 12):
        _run(a, n, knobs, True)
        _run(b, n, knobs, False)
    _same(a, b)


def test_pair_reports_first_unstable_step(knobs):
    from paper_2408_06880_b200 import _abi, geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.engine import SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    fl = geometry.packed_bed_flags((40, 32, 48), 0.6, 5.0, 7)
    st = make_stencil("d3q19")
    p = CollisionParams(1.3, "srt", None)
    got = []
    for pair in (True, False):
        e = SparseEngine(fl, st, p, "aa", check="deferred")
        e.init_canonical(seed_values(fl, st, 3))
        _run(e, 4, knobs, pair)
        v = e.canonical_state()
        v[:, 3000] = -1.0
        e.init_canonical(v)
        _run(e, 6, knobs, pair)
        bad = C.c_int64(-1)
        _abi.load().slbm_poll_instability(e._h, C.byref(bad))
        got.append(bad.value)
    assert got[0] == got[1] and got[0] >= 4
