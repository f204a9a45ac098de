"""Parity at BASELINE.json's full sizes (configs[1]: 512^3 packed bed,
porosity 0.3, D3Q19 TRT AA; configs[2]'s D3Q27 cumulant on the same bed)
through size-independent properties — the oracle cannot run these sizes in
seconds, so the checks are the ones the domain offers, evaluated on the
device without copying the 6-9 GB states to the host:

* the builder's slot ownership check passed (construction would raise) and
  a fully periodic bed has exactly Q * N_F slots;
* mass is conserved over 20 steps (bounce-back and periodic wrap conserve
  it; relative drift <= 1e-12 of fp64 round-off);
* 20 AA steps == 20 pull steps, bit for bit (sparse.py:232-241: an AA pair
  is two pull steps), over every slot;
* interior + frame sweeps (frame width 1) == whole sweeps, bit for bit.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EDGE = 512
STEPS = 20


def _bed():
    from paper_2408_06880_b200 import geometry

    return geometry.packed_bed_flags((EDGE,) * 3, 0.3, 16.0, 1, periodic=True, device=0)


def _init(eng, seed):
    rng = np.random.default_rng(seed)
    n = eng.n_fluid
    rho = 1.0 + 0.01 * rng.standard_normal(n)
    u = 0.02 * rng.standard_normal((3, n))
    eng.init_equilibrium(rho, u)


def _run(eng, steps, split=False):
    for _ in range(steps):
        eng.refresh_boundary(eng.parity)
        if split:
            eng.step("interior")
            eng.step("frame")
        else:
            eng.step()
        eng.finish_step()
    eng.poll()


@pytest.mark.parametrize("model", ["trt", "cumulant"])
def test_full_size_bed_properties(model, gpu_lib):
    import torch

    from paper_2408_06880_b200.collision import CollisionParams, trt_magic_lambda
    from paper_2408_06880_b200.engine import SparseEngine
    from paper_2408_06880_b200.lattice import make_stencil

    q = 19 if model == "trt" else 27
    st = make_stencil(f"d3q{q}")
    p = CollisionParams(1.2, model, trt_magic_lambda(1.2)) if model == "trt" else \
        CollisionParams(1.2, "cumulant")
    fl = _bed()
    aa = SparseEngine(fl, st, p, "aa", device=0, check="deferred")
    n = aa.n_fluid
    assert 0.29 < n / EDGE**3 < 0.31
    assert aa.total_slots == q * n and aa.n_ubb_slots == 0 and aa.n_ghost_slots == 0
    _init(aa, 5)
    m0 = aa.total_mass()
    _run(aa, STEPS)
    m1 = aa.total_mass()
    assert abs(m1 - m0) <= 1e-12 * m0, (m0, m1)
    starts, _ = aa.pdf_layout()  # group q: device slots starts[q] .. starts[q] + n
    ref = aa.device_state()

    def groups(view):
        return [view[int(starts[r]):int(starts[r]) + n] for r in range(q)]

    assert all(bool(torch.isfinite(g).all()) for g in groups(ref))

    def same(view):
        return all(torch.equal(a, b) for a, b in zip(groups(view), groups(ref)))

    pull = SparseEngine(fl, st, p, "pull", device=0, check="deferred")
    _init(pull, 5)
    _run(pull, STEPS)
    assert np.array_equal(pull.pdf_layout()[0], starts)
    assert same(pull.device_state())
    pull.close()
    del pull
    torch.cuda.empty_cache()

    if model == "trt":
        split = SparseEngine(fl, st, p, "aa", device=0, check="deferred", frame_width=1)
        assert split.n_interior + split.n_frame == n and split.n_frame > 0
        _init(split, 5)
        _run(split, STEPS, split=True)
        assert same(split.device_state())
        split.close()
    aa.close()
