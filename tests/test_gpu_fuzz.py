"""Randomised parity: GPU engine vs the CPU oracle (pinned bit for bit to
the reference, tests/test_oracle_golden.py) on seeded random geometries —
random solids, every face kind (periodic, no-slip, moving wall, outlet),
D2Q9 / D3Q19 / D3Q27, SRT / TRT / cumulant, pull / AA, with and without
interior/frame split sweeps and halo (ghost) slots fed with fixed values.
Covers the device layout (aligned groups, translated slot ids), the
prefetching sweeps and the boundary programs on shapes the goldens do not
pin individually."""

import numpy as np
import pytest

from conftest import drive, seed_values

pytestmark = pytest.mark.gpu

CASES = 24


def _case(seed):
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil
    from paper_2408_06880_b200.tags import FaceKind, FaceSpec, make_flags

    rng = np.random.default_rng(seed)
    name = ["d2q9", "d3q19", "d3q27"][seed % 3]
    st = make_stencil(name)
    dims = tuple(int(v) for v in rng.integers(5, 14, size=st.dim))
    kinds = []
    for a in range(st.dim):
        pick = rng.integers(0, 4)
        if pick == 0:
            kinds.append((FaceSpec(FaceKind.PERIODIC), FaceSpec(FaceKind.PERIODIC)))
            continue
        pair = []
        for _ in range(2):
            k = rng.integers(0, 3)
            if k == 0:
                pair.append(FaceSpec(FaceKind.WALL))
            elif k == 1:
                vel = tuple(float(v) for v in rng.uniform(-0.03, 0.03, size=st.dim))
                pair.append(FaceSpec(FaceKind.WALL, velocity=vel))
            else:
                pair.append(FaceSpec(FaceKind.WALL, density=float(rng.uniform(0.98, 1.02))))
        kinds.append(tuple(pair))
    solid = rng.random(tuple(reversed(dims))) < rng.uniform(0.0, 0.35)
    fl = make_flags(dims, kinds, solid=solid)
    model = ["srt", "trt", "cumulant"][int(rng.integers(0, 3 if st.q == 27 else 2))]
    omega = float(rng.uniform(0.8, 1.8))
    p = CollisionParams(omega, model, float(rng.uniform(0.6, 1.6)) if model == "trt" else None)
    pattern = ["pull", "aa"][int(rng.integers(0, 2))]
    frame = int(rng.integers(1, 3)) if rng.random() < 0.5 else None
    return fl, st, p, pattern, frame


@pytest.mark.parametrize("seed", range(CASES))
def test_gpu_matches_oracle_on_random_geometry(seed, gpu_lib):
    from oracle.sparse_ref import OracleSparseEngine
    from paper_2408_06880_b200.engine import SparseEngine

    fl, st, p, pattern, frame = _case(seed)
    if not np.any(fl.tags_interior == 0):
        pytest.skip("no fluid cell drawn")
    gpu = SparseEngine(fl, st, p, pattern, frame_width=frame)
    cpu = OracleSparseEngine(fl, st, p, pattern, frame_width=frame)
    np.testing.assert_array_equal(gpu.idx, cpu.idx)
    v = seed_values(fl, st, seed)
    gpu.init_canonical(v)
    cpu.init_canonical(v)
    steps = 5 + seed % 4
    if frame is None:
        drive(gpu, steps)
        drive(cpu, steps)
    else:
        for eng in (gpu, cpu):
            for _ in range(steps):
                eng.refresh_boundary(eng.parity)
                eng.step("interior")
                eng.step("frame")
                eng.finish_step()
    np.testing.assert_array_equal(gpu.canonical_state(), cpu.canonical_state())
    rg, ug = gpu.macroscopic_fields()
    rc, uc = cpu.macroscopic_fields()
    np.testing.assert_array_equal(rg, rc)
    np.testing.assert_array_equal(ug, uc)


def _domain_case(seed):
    from paper_2408_06880_b200.collision import CollisionParams
    from paper_2408_06880_b200.lattice import make_stencil
    from paper_2408_06880_b200.tags import FaceKind, FaceSpec, make_flags

    rng = np.random.default_rng(1000 + seed)
    st = make_stencil(["d2q9", "d3q19", "d3q27"][seed % 3])
    block = tuple(int(v) for v in rng.integers(3, 7, size=st.dim))
    grid = tuple(int(v) for v in rng.integers(1, 4, size=st.dim))
    dims = tuple(b * g for b, g in zip(block, grid))
    faces = []
    for a in range(st.dim):
        if rng.random() < 0.5:
            faces.append((FaceSpec(FaceKind.PERIODIC), FaceSpec(FaceKind.PERIODIC)))
        else:
            vel = tuple(float(v) for v in rng.uniform(-0.02, 0.02, size=st.dim))
            faces.append((FaceSpec(FaceKind.WALL), FaceSpec(FaceKind.WALL, velocity=vel)))
    solid = rng.random(tuple(reversed(dims))) < rng.uniform(0.0, 0.3)
    fl = make_flags(dims, faces, solid=solid)
    model = ["srt", "trt"][int(rng.integers(0, 2))]
    p = CollisionParams(float(rng.uniform(0.9, 1.7)), model, 0.9 if model == "trt" else None)
    pattern = ["pull", "aa"][int(rng.integers(0, 2))]
    mode = ["domain", "hybrid", "nccl", "p2p"][int(rng.integers(0, 4))]
    return fl, st, p, pattern, block, mode


@pytest.mark.parametrize("seed", range(CASES))
def test_gpu_domain_decomposition_matches_one_block(seed, gpu_lib):
    """Random block decompositions (device-local halo programs, block groups,
    dense/hybrid layouts, or every edge a loopback message over NCCL or the
    peer transport with per-face frames) equal one block, bit for bit, after
    an even number of steps (the reference's acceptance 05)."""
    from paper_2408_06880_b200.domain import Domain, DistributedDomain

    fl, st, p, pattern, block, mode = _domain_case(seed)
    if not np.any(fl.tags_interior == 0):
        pytest.skip("no fluid cell drawn")
    one = Domain(fl, fl.dims, st, p, pattern=pattern)
    if mode == "domain":
        dom = Domain(fl, block, st, p, pattern=pattern, frame_width=1)
    elif mode == "hybrid":
        dom = Domain(fl, block, st, p, pattern=pattern, frame_width=1, policy="hybrid", phi_s=0.85)
    else:
        dom = DistributedDomain(fl, block, st, p, pattern=pattern, rank=0, world=1, device=0,
                                loopback=True, transport=mode)
    for d in (one, dom):
        d.init_random(seed)
    steps = 4 + 2 * (seed % 2)
    one.run(steps)
    dom.run(steps, driver="overlapped" if seed % 3 else "sequential",
            use_graph=bool(seed % 2) and mode != "hybrid")
    np.testing.assert_array_equal(dom.gather_canonical(), one.gather_canonical())
