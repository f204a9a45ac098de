"""The resident multi-step kernel (kernels.cu k_resident: slbm_run on small
engines, one cooperative launch for n steps) against the per-step path
(graph of refresh + sweep + step-counter launches, itself pinned to the
goldens and the oracle): bit-identical states, outlet velocity stores,
counters and first-unstable-step, over the fuzz geometries (every face
kind, all stencils / models / patterns), odd step counts and both
starting parities."""

import ctypes as C

import numpy as np
import pytest

from conftest import seed_values
from test_gpu_fuzz import _case

pytestmark = pytest.mark.gpu

CAP_KNOB = 4
DEFAULT_CAP = 1 << 19


@pytest.fixture
def cap(gpu_lib):
    """Per-engine resident cap (knob 4, slbm_engine_set_tuning)."""

    def set_cap(eng, v):
        eng.set_tuning(CAP_KNOB, int(v))

    return set_cap


def _pair(seed):
    from paper_2408_06880_b200.engine import SparseEngine

    fl, st, p, pattern, _ = _case(seed)
    a = SparseEngine(fl, st, p, pattern)
    b = SparseEngine(fl, st, p, pattern)
    v = seed_values(fl, st, seed)
    a.init_canonical(v)
    b.init_canonical(v)
    return a, b


def _run(eng, steps, cap, resident):
    cap(eng, DEFAULT_CAP if resident else 0)
    eng.run(steps, use_graph=True)


@pytest.mark.parametrize("seed", range(24))
def test_resident_matches_per_step_path(seed, cap):
    a, b = _pair(seed)
    if seed % 2:  # start the resident run at odd parity
        a.run(1, use_graph=False)
        b.run(1, use_graph=False)
    steps = 5 + seed % 4
    _run(a, steps, cap, True)
    _run(b, steps, cap, False)
    np.testing.assert_array_equal(a.canonical_state(), b.canonical_state())
    assert a.parity == b.parity and a.counters.as_dict() == b.counters.as_dict()
    # a second run continues from the same state (step counter, buffers)
    _run(a, 3, cap, True)
    _run(b, 3, cap, False)
    np.testing.assert_array_equal(a.canonical_state(), b.canonical_state())
    ra, ua = a.macroscopic_fields()
    rb, ub = b.macroscopic_fields()
    np.testing.assert_array_equal(ra, rb)
    np.testing.assert_array_equal(ua, ub)


@pytest.mark.parametrize("pattern", ["aa", "pull"])
def test_resident_reports_first_unstable_step(pattern, cap):
    """The instability flag carries the same step number in both paths."""
    from paper_2408_06880_b200 import geometry
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil

    fl = geometry.packed_bed_flags((24, 20, 16), 0.6, 4.0, 7, channel=True)
    st = make_stencil("d3q19")
    p = CollisionParams(1.3, "srt", None)
    steps = []
    for resident in (True, False):
        from paper_2408_06880_b200 import _abi
        from paper_2408_06880_b200.engine import SparseEngine

        e = SparseEngine(fl, st, p, pattern, check="deferred")
        e.init_canonical(seed_values(fl, st, 3))
        _run(e, 3, cap, resident)
        v = e.canonical_state()
        v[:, 10] = -1.0  # one cell with a negative density from step 3 on
        e.init_canonical(v)
        _run(e, 5, cap, resident)
        bad = C.c_int64(-1)
        _abi.load().slbm_poll_instability(e._h, C.byref(bad))
        steps.append(bad.value)
    assert steps[0] >= 0
    assert steps[0] == steps[1]


def test_cap_selects_path(cap):
    """Above the cap the per-step path runs; both give the same answer."""
    a, b = _pair(1)
    cap(a, 1)  # n_fluid > 1: per-step path
    a.run(6, use_graph=True)
    b.run(6, use_graph=True)  # default cap: resident
    np.testing.assert_array_equal(a.canonical_state(), b.canonical_state())
