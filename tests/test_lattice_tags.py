"""Host-side types: stencil numbering, generated CUDA tables, flag painting
(CPU only)."""

import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import ROOT, golden_files, load_golden
from paper_2408_06880_b200 import errors, geometry
from paper_2408_06880_b200.lattice import emit_cuda_tables, make_stencil
from paper_2408_06880_b200.tags import (
    EXCHANGE,
    FLUID,
    NOSLIP,
    PERIODIC,
    UBB,
    WALL,
    FaceKind,
    FaceSpec,
    frame_mask,
    make_flags,
    ring_offset,
)

# SURVEY F8 (printed from the reference in-container)
D3Q19_C = [(0, 0, 0), (-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 1), (0, 1, 0), (1, 0, 0),
           (-1, -1, 0), (-1, 0, -1), (-1, 0, 1), (-1, 1, 0), (0, -1, -1), (0, -1, 1), (0, 1, -1),
           (0, 1, 1), (1, -1, 0), (1, 0, -1), (1, 0, 1), (1, 1, 0)]
D3Q19_INV = [0, 6, 5, 4, 3, 2, 1, 18, 17, 16, 15, 14, 13, 12, 11, 10, 9, 8, 7]


def test_d3q19_order_and_opposites():
    st = make_stencil("d3q19")
    assert [tuple(v) for v in st.c] == D3Q19_C
    assert list(st.inv) == D3Q19_INV


@pytest.mark.parametrize("name,q", [("d2q9", 9), ("d3q19", 19), ("d3q27", 27)])
def test_stencil_invariants(name, q):
    st = make_stencil(name)
    assert st.q == q
    assert sum(st.w_exact) == 1
    for i in range(q):
        assert np.array_equal(st.c[st.inv[i]], -st.c[i])
        assert st.w[i] == float(st.w_exact[i])
    # second-moment isotropy sum w c_a c_b = cs2 delta_ab
    for a in range(st.dim):
        for b in range(st.dim):
            m = sum(st.w_exact[i] * int(st.c[i, a]) * int(st.c[i, b]) for i in range(q))
            assert m == (Fraction(1, 3) if a == b else 0)


def test_d3q27_corners_follow_d3q19():
    st19, st27 = make_stencil("d3q19"), make_stencil("d3q27")
    assert np.array_equal(st27.c[:19], st19.c)
    assert [int(st27.inv[i]) for i in range(19, 27)] == [26, 25, 24, 23, 22, 21, 20, 19]


def test_unknown_stencil():
    with pytest.raises(errors.ConfigurationError):
        make_stencil("d3q15")


def test_generated_cuda_tables_are_current():
    path = os.path.join(ROOT, "paper_2408_06880_b200", "csrc", "lattice_tables.h")
    with open(path) as fh:
        assert fh.read().strip() == emit_cuda_tables().strip()


def test_make_flags_periodic_wrap_and_corners():
    lid = FaceSpec(FaceKind.WALL, velocity=(0.1, 0.0))
    fl = make_flags((4, 3), [(PERIODIC, PERIODIC), (WALL, lid)])
    # x periodic: ring column x=-1 mirrors x=3 (including painted y ring)
    assert np.array_equal(fl.tags[:, 0], fl.tags[:, 4])
    # y: bottom NOSLIP, top UBB; x ring padded after y -> corners are copies
    assert fl.tag_at((1, -1)) == NOSLIP and fl.tag_at((1, 3)) == UBB
    assert fl.tag_at((-1, 3)) == UBB
    assert fl.ubb_at((2, 3))[0] == 0.1 and fl.ubb_at((2, 1))[0] == 0.0
    walls = make_flags((3, 3), [(WALL, WALL), (WALL, lid)])
    # x padded last claims the corners: lid stops short of the side walls
    assert walls.tag_at((-1, 3)) == NOSLIP and walls.tag_at((0, 3)) == UBB


def test_make_flags_validation():
    with pytest.raises(errors.ConfigurationError):
        make_flags((4, 4), [(PERIODIC, WALL), (WALL, WALL)])
    with pytest.raises(errors.ConfigurationError):
        make_flags((4,), [(WALL, WALL)])
    with pytest.raises(errors.ConfigurationError):
        make_flags((4, 4), [(FaceSpec(FaceKind.PERIODIC, (1.0, 0.0)),) * 2, (WALL, WALL)])


def test_frame_mask_widths_and_clamp():
    m = frame_mask((6, 5, 4), (1, 2, 1))
    assert m.shape == (4, 5, 6)
    assert m[1:3, 2, 1:5].sum() == 0 and m[0].all() and m[:, 1].all()
    assert frame_mask((3, 3), 5).all()
    with pytest.raises(errors.ConfigurationError):
        frame_mask((3, 3), 0)


def test_ring_offset():
    assert ring_offset((-1, 2, 5), (4, 4, 5)) == (-1, 0, 1)


def _regen(name):
    """Rebuild the generator call behind each golden engine fixture."""
    lid = lambda d, s: FaceSpec(FaceKind.WALL, velocity=(s,) + (0.0,) * (len(d) - 1))  # noqa: E731
    table = {
        "engine_d2q9_lid": lambda: make_flags((12, 8), [(PERIODIC, PERIODIC), (WALL, lid((12, 8), 0.04))],
                                              solid=geometry.random_obstacles((12, 8), 0.85, 3)),
        "engine_d2q9_channel": lambda: geometry.channel_flags(
            (10, 6), solid=geometry.random_obstacles((10, 6), 0.8, 8)),
        "engine_d3q19_periodic": lambda: geometry.obstacle_flags((6, 5, 4), 0.7, 5),
        "engine_d3q27_walled": lambda: geometry.obstacle_flags((5, 4, 4), 0.8, 9, periodic=False),
        "engine_d3q19_couette_trt": lambda: geometry.riverbed_flags((8, 6, 8), (4, 3, 4), 0.5, 2, 0.05),
        "engine_d3q27_couette_trt": lambda: geometry.riverbed_flags((6, 6, 6), (3, 3, 3), 0.6, 4, 0.04),
        "engine_d3q19_obstacles_trt": lambda: geometry.obstacle_flags((9, 7, 6), 0.6, 12),
    }
    return table.get(name)


@pytest.mark.parametrize("path", golden_files("engine"), ids=lambda p: os.path.basename(p)[:-4])
def test_flag_generators_match_reference(path):
    mk = _regen(os.path.basename(path)[:-4])
    if mk is None:
        pytest.skip("fixture built from a partitioned block")
    rec = load_golden(path)
    fl = mk()
    assert np.array_equal(fl.tags, rec["tags"])
    assert np.array_equal(fl.ubb_u, rec["ubb_u"])
    assert fl.periodic == tuple(bool(p) for p in rec["periodic"])


@pytest.mark.parametrize("path", golden_files("bed"), ids=lambda p: os.path.basename(p)[:-4])
def test_sphere_bed_voxelization_matches_reference(path):
    import hashlib

    rec = load_golden(path)
    dims = tuple(int(d) for d in rec["dims"])
    d = float(rec["diameter"])
    n = geometry.overlapping_sphere_count(dims, d, float(rec["porosity_target"]))
    assert n == int(rec["count"])
    solid = geometry.voxelize_spheres(dims, geometry.sphere_centers(dims, d, n, int(rec["seed"])), d)
    assert hashlib.sha256(solid.astype(np.uint8).tobytes()).hexdigest() == str(rec["solid_sha"])


def test_tag_values_are_the_reference_contract():
    assert (FLUID, NOSLIP, UBB, EXCHANGE) == (0, 1, 2, 3)


def test_voxel_mask_roundtrip(tmp_path):
    mask = geometry.VoxelMask((5, 4, 3), geometry.random_obstacles((5, 4, 3), 0.6, 1))
    p = tmp_path / "m.vox"
    geometry.write_voxel_mask(p, mask)
    back = geometry.read_voxel_mask(p)
    assert back.dims == mask.dims and np.array_equal(back.solid, mask.solid)
    p.write_bytes(b"NOTAMASK" + bytes(12))
    with pytest.raises(errors.FormatError):
        geometry.read_voxel_mask(p)


def test_ring_field_equals_dense_painting():
    """make_flags(ring=True) keeps moving-wall values as a RingField
    (side-class table + tags); every window materialises to exactly the
    dense array make_flags paints, for every face combination drawn."""
    import numpy as np

    from paper_2408_06880_b200.tags import FaceKind, FaceSpec, RingField, make_flags

    rng = np.random.default_rng(3)
    for trial in range(60):
        nd = 2 + trial % 2
        dims = tuple(int(v) for v in rng.integers(1, 7, size=nd))
        faces = []
        for a in range(nd):
            if rng.random() < 0.3:
                faces.append((FaceSpec(FaceKind.PERIODIC), FaceSpec(FaceKind.PERIODIC)))
                continue
            pair = []
            for _ in range(2):
                k = rng.integers(0, 3)
                if k == 0:
                    pair.append(FaceSpec(FaceKind.WALL))
                elif k == 1:
                    pair.append(FaceSpec(FaceKind.WALL,
                                         velocity=tuple(float(v) for v in rng.normal(size=nd))))
                else:
                    pair.append(FaceSpec(FaceKind.WALL, density=float(rng.uniform(0.9, 1.1))))
            faces.append(tuple(pair))
        solid = rng.random(tuple(reversed(dims))) < 0.3
        dense = make_flags(dims, faces, solid=solid, ring=False)
        lazy = make_flags(dims, faces, solid=solid, ring=True)
        assert np.array_equal(dense.tags, lazy.tags)
        if not isinstance(lazy.ubb_u, RingField):
            continue  # no moving wall: both keep the zero view
        assert lazy.ubb_u.shape == dense.ubb_u.shape
        assert np.array_equal(np.asarray(lazy.ubb_u), dense.ubb_u)
        # a lazy window (a block slice) equals the dense slice
        sel = tuple(slice(int(rng.integers(0, s)), None) for s in dense.tags.shape)
        assert np.array_equal(np.asarray(lazy.ubb_u[sel]), dense.ubb_u[sel])
        c = tuple(int(rng.integers(0, d)) for d in dims)
        assert np.array_equal(lazy.ubb_at(c), dense.ubb_at(c))
