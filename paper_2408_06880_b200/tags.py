"""Cell tags and the padded flag box (input format of the list builder).

Same semantics as the reference (``pkg/src/slbm/flags.py``): a uint8 tag
per cell on a box padded by one ring cell per side, stored with axes in
reverse public order (``(z, y, x)`` for public ``(x, y, z)``), plus a
per-cell wall velocity that only matters where the tag is UBB.  Tag
values (``flags.py:27-30``) are part of the contract with the CUDA
builder.

Ring painting (``flags.py:196-249``): axes are padded in array order, so
for two meeting walls the later-padded axis wins the corner; periodic axes
copy the wrapped image of the opposite side (including already-painted
ring cells of earlier axes).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import errors

FLUID = 0
NOSLIP = 1
UBB = 2
EXCHANGE = 3
# extension beyond the reference (no outlet there): fixed-density
# outlet cell; its prescribed density is stored in ubb_u[..., 0]
OUTLET = 4
TAG_NAMES = {FLUID: "fluid", NOSLIP: "noslip", UBB: "ubb", EXCHANGE: "exchange", OUTLET: "outlet"}


class FaceKind(Enum):
    WALL = "wall"
    PERIODIC = "periodic"
    EXCHANGE = "exchange"


@dataclass(frozen=True)
class FaceSpec:
    """A face: WALL (resting, or moving with ``velocity`` -> UBB inlet, or
    with ``density`` -> fixed-density OUTLET) or PERIODIC."""

    kind: FaceKind
    velocity: tuple[float, ...] | None = None
    density: float | None = None


WALL = FaceSpec(FaceKind.WALL)
PERIODIC = FaceSpec(FaceKind.PERIODIC)


def rev_shape(dims) -> tuple[int, ...]:
    return tuple(int(d) for d in dims)[::-1]


def ring_offset(pos, dims) -> tuple[int, ...]:
    """-1 / 0 / +1 per public axis: below, inside, or above the box."""
    return tuple(-1 if p < 0 else (1 if p >= d else 0) for p, d in zip(pos, dims))


def frame_mask(dims, width) -> np.ndarray:
    """Cells within ``width`` (per public axis, clamped to the extent) of a
    box face, as a bool array over ``rev_shape(dims)``
    (``flags.py:83-108``)."""
    nd = len(dims)
    widths = (width,) * nd if isinstance(width, (int, np.integer)) else tuple(int(w) for w in width)
    if len(widths) != nd:
        raise errors.make(
            "ConfigurationError",
            f"need one frame width per axis, got {len(widths)} for {nd} axes",
        )
    if min(widths) < 1:
        raise errors.make("ConfigurationError", f"frame widths must be >= 1, got {widths}")
    grids = np.ogrid[tuple(slice(0, int(n)) for n in rev_shape(dims))]
    mask = np.zeros(rev_shape(dims), dtype=bool)
    for axis in range(nd):
        n = int(dims[axis])
        w = min(widths[axis], n)
        g = grids[nd - 1 - axis]
        mask |= (g < w) | (g >= n - w)
    return mask


@dataclass
class FlagField:
    dims: tuple[int, ...]
    tags: np.ndarray  # uint8, rev_shape(dims) + 2 per axis
    ubb_u: np.ndarray  # float64, tags.shape + (dim,)
    periodic: tuple[bool, ...]

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def core(self) -> tuple[slice, ...]:
        return tuple(slice(1, n + 1) for n in rev_shape(self.dims))

    @property
    def tags_interior(self) -> np.ndarray:
        return self.tags[self.core]

    def fluid_count(self) -> int:
        return int(np.count_nonzero(self.tags_interior == FLUID))

    def cell_count(self) -> int:
        return int(np.prod(self.dims, dtype=np.int64))

    def porosity(self) -> float:
        return self.fluid_count() / self.cell_count()

    def _padded_index(self, coord):
        return tuple(int(coord[a]) + 1 for a in reversed(range(self.ndim)))

    def tag_at(self, coord) -> int:
        return int(self.tags[self._padded_index(coord)])

    def ubb_at(self, coord) -> np.ndarray:
        return self.ubb_u[self._padded_index(coord)]


# boxes at least this large (padded cells) with moving walls / outlets keep
# ubb_u as a RingField instead of a dense float64 array (24 B per cell)
RING_MIN_CELLS = 1 << 27


class RingField:
    """``ubb_u`` of :func:`make_flags` without the dense (Z+2)(Y+2)(X+2) x dim
    float64 array.

    make_flags paints wall values face by face (flags.py:196-249), so a
    cell's value depends only on which side of each axis it sits on — low
    ring, interior or high ring — and on whether its final tag is UBB /
    OUTLET (everything else is zeroed).  The 3^dim side classes are painted
    once on a 1-cell box with the same faces (the same code path), and any
    window of the field is materialised on demand from that table and the
    tags.  Slicing with slices keeps a lazy window (block slices of a
    partition), ``np.asarray`` materialises.  Read-only."""

    def __init__(self, tags, table, origin=None, window=None):
        self._tags = tags
        self._table = table  # (3,) * nd + (nd,)
        nd = tags.ndim
        self._origin = tuple(origin) if origin is not None else (0,) * nd
        self._window = tuple(window) if window is not None else tuple(tags.shape)
        self.dtype = np.dtype(np.float64)
        self.shape = self._window + (nd,)
        self.ndim = len(self.shape)
        self.flags = type("Flags", (), {"writeable": False})()

    @property
    def nbytes(self) -> int:
        return int(np.prod(self.shape)) * 8

    def __array__(self, dtype=None, copy=None):
        # only cells on the global ring can be non-zero: start from zeros and
        # fill the (at most 2 per axis) ring planes crossing the window
        tags = self._tags
        nd = tags.ndim
        out = np.zeros(self._window + (nd,), dtype=np.float64)
        sides = []
        for a in range(nd):
            n_pad = tags.shape[a]
            c = np.arange(self._origin[a], self._origin[a] + self._window[a])
            sides.append(np.where(c == 0, 0, np.where(c == n_pad - 1, 2, 1)))
        table = self._table.reshape(-1, nd)
        for a in range(nd):
            for g in (0, tags.shape[a] - 1):
                k = g - self._origin[a]
                if not 0 <= k < self._window[a]:
                    continue
                cls = np.zeros([self._window[b] for b in range(nd) if b != a], dtype=np.int64)
                for b in range(nd):
                    side = sides[b] if b != a else np.array([0 if g == 0 else 2])
                    if b == a:
                        cls = cls * 3 + int(side[0])
                        continue
                    shape = [self._window[c] for c in range(nd) if c != a]
                    bb = b if b < a else b - 1
                    view = [1] * (nd - 1)
                    view[bb] = shape[bb]
                    cls = cls * 3 + side.reshape(view)
                sel = [slice(o, o + w) for o, w in zip(self._origin, self._window)]
                sel[a] = g
                t = tags[tuple(sel)]
                vals = table[cls]
                vals[(t != UBB) & (t != OUTLET)] = 0.0
                idx = [slice(None)] * nd
                idx[a] = k
                out[tuple(idx)] = vals
        return out if dtype is None else out.astype(dtype)

    def __getitem__(self, key):
        nd = self._tags.ndim
        if not isinstance(key, tuple):
            key = (key,)
        simple = all(isinstance(k, (int, np.integer)) or (isinstance(k, slice) and k.step in (None, 1))
                     for k in key)
        if len(key) <= nd and simple:
            origin, window = list(self._origin), list(self._window)
            for a, k in enumerate(key):
                if isinstance(k, slice):
                    lo, hi, _ = k.indices(self._window[a])
                else:
                    lo = int(k) + (self._window[a] if k < 0 else 0)
                    hi = lo + 1
                origin[a] = self._origin[a] + lo
                window[a] = max(hi - lo, 0)
            view = RingField(self._tags, self._table, origin, window)
            if all(isinstance(k, slice) for k in key):
                return view  # lazy window
            # integer axes: materialise only the small window, then drop them
            return np.asarray(view)[tuple(0 if not isinstance(k, slice) else slice(None)
                                          for k in key)]
        return np.asarray(self)[key]


def _wall_tag(spec: FaceSpec) -> int:
    if spec.density is not None:
        return OUTLET
    if spec.velocity is not None and any(float(v) != 0.0 for v in spec.velocity):
        return UBB
    return NOSLIP


def _face_value(spec: FaceSpec, nd: int):
    """per-cell payload painted with a wall face: UBB velocity, or the
    OUTLET density in component 0"""
    if spec.density is not None:
        return np.array([float(spec.density)] + [0.0] * (nd - 1))
    return 0.0 if spec.velocity is None else np.asarray(spec.velocity, np.float64)


def _check_faces(dims, faces):
    nd = len(dims)
    if len(faces) != nd:
        raise errors.make(
            "ConfigurationError", f"need one face pair per axis, got {len(faces)} for {nd} axes"
        )
    for axis, (lo, hi) in enumerate(faces):
        for spec in (lo, hi):
            if spec.kind is FaceKind.EXCHANGE:
                raise errors.make("ConfigurationError", "exchange faces only arise from partitioning")
            if spec.density is not None and (spec.kind is not FaceKind.WALL or spec.velocity is not None):
                raise errors.make("ConfigurationError", "density is only valid on resting wall faces")
            if spec.velocity is not None:
                if spec.kind is not FaceKind.WALL:
                    raise errors.make("ConfigurationError", "velocity is only valid on wall faces")
                if len(spec.velocity) != nd:
                    raise errors.make(
                        "ConfigurationError",
                        f"wall velocity needs {nd} components, got {len(spec.velocity)}",
                    )
        if (lo.kind is FaceKind.PERIODIC) ^ (hi.kind is FaceKind.PERIODIC):
            raise errors.make(
                "ConfigurationError", f"axis {axis}: periodic must be set on both sides or neither"
            )


def make_flags(dims, faces, solid: np.ndarray | None = None, ring: bool | None = None) -> FlagField:
    """Padded tag box for a domain with the given per-axis face pairs
    (``flags.py:196-249``).  ``ring`` (default: for boxes of at least
    RING_MIN_CELLS padded cells) keeps a moving-wall ``ubb_u`` as a
    :class:`RingField` instead of a dense array."""
    dims = tuple(int(d) for d in dims)
    nd = len(dims)
    if nd not in (2, 3):
        raise errors.make("ConfigurationError", f"dims must have 2 or 3 axes, got {nd}")
    if min(dims) < 1:
        raise errors.make("ConfigurationError", f"all extents must be positive, got {dims}")
    _check_faces(dims, faces)
    shape = rev_shape(dims)
    if solid is not None and tuple(solid.shape) != shape:
        raise errors.make("ConfigurationError", f"solid mask shape {solid.shape} != {shape}")

    padded = tuple(n + 2 for n in shape)
    tags = np.zeros(padded, dtype=np.uint8)
    moving = any(_wall_tag(s) in (UBB, OUTLET) for pair in faces for s in pair)
    if ring is None:
        ring = moving and int(np.prod(padded, dtype=np.int64)) >= RING_MIN_CELLS
    if moving and ring:
        # side-class table: the same painting on a 1-cell box, unmasked
        cls_vel = _paint_unmasked(faces, nd)
        moving = False  # tags only below; values come from the table
        vel = None
    elif moving:
        vel = np.zeros(padded + (nd,), dtype=np.float64)
    else:
        # no moving wall: a read-only zero view instead of 24 B/cell of zeros
        vel = np.broadcast_to(np.zeros((), dtype=np.float64), padded + (nd,))
    inner = tuple(slice(1, n + 1) for n in shape)
    if solid is not None:
        tags[inner][np.asarray(solid, dtype=bool)] = NOSLIP

    # grow the painted region one array axis at a time (z, then y, then x);
    # `done` tracks the extent already valid on every axis
    lo_idx = [1] * nd
    hi_idx = [n + 1 for n in shape]
    for arr_axis in range(nd):
        axis = nd - 1 - arr_axis
        lo, hi = faces[axis]
        region = [slice(lo_idx[a], hi_idx[a]) for a in range(nd)]
        n = shape[arr_axis]
        dst_lo = list(region)
        dst_hi = list(region)
        dst_lo[arr_axis] = slice(0, 1)
        dst_hi[arr_axis] = slice(n + 1, n + 2)
        if lo.kind is FaceKind.PERIODIC:
            src_lo = list(region)
            src_hi = list(region)
            src_lo[arr_axis] = slice(n, n + 1)
            src_hi[arr_axis] = slice(1, 2)
            tags[tuple(dst_lo)] = tags[tuple(src_lo)]
            tags[tuple(dst_hi)] = tags[tuple(src_hi)]
            if moving:
                vel[tuple(dst_lo)] = vel[tuple(src_lo)]
                vel[tuple(dst_hi)] = vel[tuple(src_hi)]
        else:
            tags[tuple(dst_lo)] = _wall_tag(lo)
            tags[tuple(dst_hi)] = _wall_tag(hi)
            if moving:
                vel[tuple(dst_lo)] = _face_value(lo, nd)
                vel[tuple(dst_hi)] = _face_value(hi, nd)
        lo_idx[arr_axis] = 0
        hi_idx[arr_axis] = n + 2
    if moving:
        vel[(tags != UBB) & (tags != OUTLET)] = 0.0
    if vel is None:
        vel = RingField(tags, cls_vel)
    periodic = tuple(faces[a][0].kind is FaceKind.PERIODIC for a in range(nd))
    return FlagField(dims=dims, tags=tags, ubb_u=vel, periodic=periodic)


def _paint_unmasked(faces, nd):
    """make_flags' value painting on a 1-cell box without the final masking:
    the value each side class (low ring / interior / high ring per axis)
    receives, whatever tag the real box ends up with there."""
    vel = np.zeros((3,) * nd + (nd,), dtype=np.float64)
    lo_idx, hi_idx = [1] * nd, [2] * nd
    for arr_axis in range(nd):
        lo, hi = faces[nd - 1 - arr_axis]
        region = [slice(lo_idx[a], hi_idx[a]) for a in range(nd)]
        dst_lo, dst_hi = list(region), list(region)
        dst_lo[arr_axis] = slice(0, 1)
        dst_hi[arr_axis] = slice(2, 3)
        if lo.kind is FaceKind.PERIODIC:
            src = list(region)
            src[arr_axis] = slice(1, 2)
            vel[tuple(dst_lo)] = vel[tuple(src)]
            vel[tuple(dst_hi)] = vel[tuple(src)]
        else:
            vel[tuple(dst_lo)] = _face_value(lo, nd)
            vel[tuple(dst_hi)] = _face_value(hi, nd)
        lo_idx[arr_axis], hi_idx[arr_axis] = 0, 3
    return vel
