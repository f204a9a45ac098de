"""Synthetic geometries and voxel-mask I/O (input side of the hot path).

Generators mirror the reference's (``pkg/src/slbm/geometry.py``) so both
sides of a parity test see identical tag boxes:

* ``random_obstacles``   geometry.py:250-260 (same seeded permutation)
* ``channel_flags`` / ``couette_flags`` / ``obstacle_flags`` /
  ``riverbed_flags`` / ``mask_flags``   geometry.py:301-344
* ``voxelize_spheres``   geometry.py:150-178 rasterization rule, with
  *overlapping* sphere centres (the reference packer jams at porosity
  ~0.69, so packed beds at 0.3-0.5 use overlapping spheres fed
  through the same rasterizer).  Large boxes rasterize on the GPU
  (``slbm_voxelize_spheres``), small ones in numpy — same bits.
* ``SLBMVOX1`` mask files  geometry.py:212-244.
* ``artery_tree``        new (no reference counterpart; unpinned): a
  branching capsule tree for the vessel-like benchmark.
"""

from __future__ import annotations

import ctypes as C
import math
import struct
from dataclasses import dataclass, field

import numpy as np

from . import errors
from .tags import PERIODIC, WALL, FaceKind, FaceSpec, make_flags, rev_shape

MASK_MAGIC = b"SLBMVOX1"
_MASK_HEADER = struct.Struct("<8s3I")


@dataclass
class VoxelMask:
    dims: tuple[int, ...]
    solid: np.ndarray = field(repr=False)

    def __post_init__(self) -> None:
        self.dims = tuple(int(d) for d in self.dims)
        if tuple(self.solid.shape) != rev_shape(self.dims):
            raise errors.make(
                "ConfigurationError", f"mask shape {self.solid.shape} does not match dims {self.dims}"
            )
        self.solid = self.solid.astype(bool)

    def cell_count(self) -> int:
        return int(np.prod(self.dims, dtype=np.int64))

    def fluid_count(self) -> int:
        return self.cell_count() - int(self.solid.sum())

    def porosity(self) -> float:
        return self.fluid_count() / self.cell_count()


# ---------------------------------------------------------------- obstacles


def random_obstacles(dims, porosity: float, seed) -> np.ndarray:
    if not 0.0 <= porosity <= 1.0:
        raise errors.make("ConfigurationError", f"porosity {porosity} outside [0, 1]")
    total = int(np.prod(dims, dtype=np.int64))
    n_solid = int(round((1.0 - porosity) * total))
    order = np.random.default_rng(seed).permutation(total)
    solid = np.zeros(total, dtype=bool)
    solid[order[:n_solid]] = True
    return solid.reshape(rev_shape(dims))


def riverbed_solids(dims, block_size, bed_porosity=0.35, seed=0, bed_fraction=0.5):
    nd = len(dims)
    if any(int(dims[a]) % int(block_size[a]) for a in range(nd)):
        raise errors.make("ConfigurationError", f"dims {dims} not divisible by block size {block_size}")
    solid = np.zeros(rev_shape(dims), dtype=bool)
    top = bed_fraction * dims[-1]
    grid = [int(dims[a]) // int(block_size[a]) for a in range(nd)]
    for flat in range(int(np.prod(grid))):
        pos, rem = [], flat
        for a in range(nd):
            pos.append(rem % grid[a])
            rem //= grid[a]
        if (pos[-1] + 1) * block_size[-1] > top:
            continue
        sel = tuple(slice(pos[a] * block_size[a], (pos[a] + 1) * block_size[a])
                    for a in reversed(range(nd)))
        solid[sel] = random_obstacles(block_size, bed_porosity, [seed, flat])
    return solid


def _lid(dims, speed):
    return FaceSpec(FaceKind.WALL, velocity=(float(speed),) + (0.0,) * (len(dims) - 1))


def channel_flags(dims, solid=None):
    """periodic x, resting walls elsewhere (geometry.py:309-312)"""
    return make_flags(dims, [(PERIODIC, PERIODIC)] + [(WALL, WALL)] * (len(dims) - 1), solid=solid)


def couette_flags(dims, u_wall):
    """periodic except the last axis: resting floor, moving lid (:301-306)"""
    faces = [(PERIODIC, PERIODIC)] * (len(dims) - 1) + [(WALL, _lid(dims, u_wall))]
    return make_flags(dims, faces)


def obstacle_flags(dims, porosity, seed, periodic=True):
    f = PERIODIC if periodic else WALL
    return make_flags(dims, [(f, f)] * len(dims), solid=random_obstacles(dims, porosity, seed))


def riverbed_flags(dims, block_size, bed_porosity=0.35, seed=0, lid_speed=0.02):
    faces = [(PERIODIC, PERIODIC)] * (len(dims) - 1) + [(WALL, _lid(dims, lid_speed))]
    return make_flags(dims, faces, solid=riverbed_solids(dims, block_size, bed_porosity, seed))


def mask_flags(mask: VoxelMask, periodic_x: bool = True):
    first = PERIODIC if periodic_x else WALL
    return make_flags(mask.dims, [(first, first)] + [(WALL, WALL)] * (len(mask.dims) - 1),
                      solid=mask.solid)


# ---------------------------------------------------------------- sphere beds


def overlapping_sphere_count(dims, diameter: float, porosity: float) -> int:
    """Boolean-model count, porosity = exp(-n V / |grown box|), where the
    centres are drawn over the box grown by one radius per side so the bed
    is statistically uniform right up to the faces."""
    vol = math.pi * diameter**3 / 6.0
    grown = np.asarray(dims, dtype=np.float64) + diameter
    return int(round(-math.log(porosity) * float(np.prod(grown)) / vol))


def sphere_centers(dims, diameter: float, count: int, seed: int) -> np.ndarray:
    """``count`` uniform centres (public order) over the grown box, overlap
    allowed (same draw as tools/make_golden.py)."""
    rng = np.random.default_rng(seed)
    grown = np.asarray(dims, dtype=np.float64) + diameter
    return rng.random((count, len(dims))) * grown - diameter / 2.0


def voxelize_spheres(dims, centers, diameter: float, device: int | None = None) -> np.ndarray:
    """Solid mask over rev_shape(dims): cell centre strictly inside a sphere
    (geometry.py:150-178 at resolution 1).  ``device`` selects the CUDA
    rasterizer (3-d only); None uses numpy."""
    dims = tuple(int(d) for d in dims)
    centers = np.ascontiguousarray(centers, dtype=np.float64)
    if device is not None and len(dims) == 3:
        from . import _abi

        out = np.zeros(rev_shape(dims), dtype=np.uint8)
        d32 = np.array(dims, dtype=np.int32)
        _abi.call("slbm_voxelize_spheres", _abi.ptr(d32, C.c_int32), _abi.ptr(centers, C.c_double),
                  centers.shape[0], float(diameter), int(device), _abi.ptr(out, C.c_uint8))
        return out.astype(bool)
    dim = len(dims)
    solid = np.zeros(rev_shape(dims), dtype=bool)
    r = diameter / 2.0
    r2 = r * r
    for ctr in centers:
        sel, axes = [], []
        for a in range(dim):
            lo = max(0, int(math.floor((ctr[a] - r) * 1.0 - 0.5)))
            hi = min(dims[a] - 1, int(math.ceil((ctr[a] + r) * 1.0 - 0.5)))
            if hi < lo:
                break
            sel.append(slice(lo, hi + 1))
            axes.append((np.arange(lo, hi + 1) + 0.5) / 1.0 - ctr[a])
        else:
            d2 = np.zeros(tuple(len(x) for x in reversed(axes)))
            for a, ax in enumerate(axes):
                shape = [1] * dim
                shape[dim - 1 - a] = len(ax)
                d2 = d2 + (ax * ax).reshape(shape)
            solid[tuple(reversed(sel))] |= d2 < r2
    return solid


def packed_bed_flags(dims, porosity: float, diameter: float, seed: int, periodic: bool = True,
                     device: int | None = None, channel: bool = False):
    """Overlapping-sphere bed: fully periodic box (``channel=False``) or the
    x-periodic channel of ``mask_flags`` (``channel=True``)."""
    n = overlapping_sphere_count(dims, diameter, porosity)
    solid = voxelize_spheres(dims, sphere_centers(dims, diameter, n, seed), diameter, device)
    if channel:
        return channel_flags(dims, solid=solid)
    f = PERIODIC if periodic else WALL
    return make_flags(dims, [(f, f)] * len(dims), solid=solid)


# ---------------------------------------------------------------- mask files


def write_voxel_mask(path, mask: VoxelMask) -> None:
    dims3 = tuple(mask.dims) + (1,) * (3 - len(mask.dims))
    payload = np.packbits(mask.solid.reshape(-1).astype(np.uint8), bitorder="little").tobytes()
    with open(path, "wb") as fh:
        fh.write(_MASK_HEADER.pack(MASK_MAGIC, *dims3))
        fh.write(payload)


def read_voxel_mask(path) -> VoxelMask:
    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < _MASK_HEADER.size:
        raise errors.make(
            "FormatError",
            f"voxel mask truncated at offset {len(data)}: header needs {_MASK_HEADER.size} bytes",
        )
    magic, nx, ny, nz = _MASK_HEADER.unpack_from(data, 0)
    if magic != MASK_MAGIC:
        raise errors.make("FormatError", f"bad magic {magic!r} at offset 0, want {MASK_MAGIC!r}")
    if min(nx, ny, nz) < 1:
        raise errors.make("FormatError", f"non-positive extent {(nx, ny, nz)} at offset 8")
    ncells = nx * ny * nz
    nbytes = (ncells + 7) // 8
    if len(data) < _MASK_HEADER.size + nbytes:
        raise errors.make(
            "FormatError",
            f"voxel mask truncated at offset {len(data)}: payload needs {nbytes} bytes for {ncells} cells",
        )
    raw = np.frombuffer(data, dtype=np.uint8, count=nbytes, offset=_MASK_HEADER.size)
    bits = np.unpackbits(raw, bitorder="little")[:ncells].astype(bool)
    dims = (nx, ny, nz) if nz > 1 else (nx, ny)
    return VoxelMask(dims, bits.reshape(rev_shape(dims)))


# ---------------------------------------------------------------- vessel tree


def artery_segments(dims, seed: int = 0, r_root: float = 20.0, r_min: float = 8.0,
                    levels: int = 5):
    """Capsule segments (p0, p1, radius) of a branching tube tree in the box
    ``dims`` (public order): a root enters through the x = 0 face at the
    centre of the y-z face, bifurcates ``levels`` times with Murray-law radii
    (r / 2^(1/3), clamped at ``r_min``) at 25-45 degrees in random planes,
    and the terminal branches run on until they leave the box.  New geometry
    (the reference has no vessel generator); deterministic in ``seed``."""
    rng = np.random.default_rng(seed)
    ext = np.asarray([float(d) for d in dims])
    seg_len = ext[0] / (levels + 1.5)
    segs = []
    stack = [(np.array([-1.0, ext[1] / 2, ext[2] / 2]), np.array([1.0, 0.0, 0.0]), r_root, 0)]
    while stack:
        p0, d, r, lvl = stack.pop()
        if lvl == levels:
            # terminal branch: continue straight until it exits the box
            p1 = p0 + d * (2.0 * float(ext.max()))
            segs.append((p0, p1, r))
            continue
        p1 = p0 + d * seg_len * (0.9 ** lvl)
        segs.append((p0, p1, r))
        rc = max(r / 2.0 ** (1.0 / 3.0), r_min)
        axis = rng.normal(size=3)
        axis -= axis.dot(d) * d
        axis /= np.linalg.norm(axis) + 1e-12
        for sgn in (1.0, -1.0):
            ang = math.radians(rng.uniform(25.0, 45.0))
            nd = math.cos(ang) * d + sgn * math.sin(ang) * axis
            nd[0] = max(nd[0], 0.35)  # keep the tree flowing towards +x
            nd /= np.linalg.norm(nd)
            stack.append((p1.copy(), nd, rc, lvl + 1))
    return segs


def artery_tree(dims, seed: int = 0, **kw) -> np.ndarray:
    """Fluid mask (True = fluid) over rev_shape(dims) of artery_segments:
    a cell is fluid iff its centre lies within a segment's radius."""
    dims = tuple(int(d) for d in dims)
    fluid = np.zeros(rev_shape(dims), dtype=bool)
    hi_box = np.asarray(dims) - 1
    for p0, p1, r in artery_segments(dims, seed, **kw):
        seg = p1 - p0
        L2 = float(seg.dot(seg)) or 1.0
        lo = np.maximum(np.floor(np.minimum(p0, p1) - r - 1).astype(np.int64), 0)
        hi = np.minimum(np.ceil(np.maximum(p0, p1) + r + 1).astype(np.int64), hi_box)
        if np.any(hi < lo):
            continue
        # march along x in slabs; each slab only scans the y-z box the
        # segment (plus radius) occupies inside that slab
        step = 16
        for x0 in range(int(lo[0]), int(hi[0]) + 1, step):
            x1 = min(int(hi[0]), x0 + step - 1)
            if abs(seg[0]) > 1e-9:
                ta = np.clip((x0 - r - 1.0 - p0[0]) / seg[0], 0.0, 1.0)
                tb = np.clip((x1 + 1.0 + r - p0[0]) / seg[0], 0.0, 1.0)
                pa, pb = p0 + ta * seg, p0 + tb * seg
                ylo = max(int(np.floor(min(pa[1], pb[1]) - r - 1)), int(lo[1]))
                yhi = min(int(np.ceil(max(pa[1], pb[1]) + r + 1)), int(hi[1]))
                zlo = max(int(np.floor(min(pa[2], pb[2]) - r - 1)), int(lo[2]))
                zhi = min(int(np.ceil(max(pa[2], pb[2]) + r + 1)), int(hi[2]))
            else:
                ylo, yhi, zlo, zhi = int(lo[1]), int(hi[1]), int(lo[2]), int(hi[2])
            if yhi < ylo or zhi < zlo:
                continue
            xs = np.arange(x0, x1 + 1) + 0.5
            ys = np.arange(ylo, yhi + 1) + 0.5
            zs = np.arange(zlo, zhi + 1) + 0.5
            zz, yy, xx = np.meshgrid(zs, ys, xs, indexing="ij")
            pts = np.stack([xx, yy, zz], axis=-1)
            tpar = np.clip(((pts - p0) @ seg) / L2, 0.0, 1.0)
            d2 = ((pts - (p0 + tpar[..., None] * seg)) ** 2).sum(-1)
            fluid[zlo:zhi + 1, ylo:yhi + 1, x0:x1 + 1] |= d2 < r * r
    return fluid


def artery_flags(dims, seed: int = 0, inlet_speed: float = 0.02, outlet_density: float = 1.0,
                 **kw):
    """Vessel-like benchmark geometry: tube-tree fluid in a solid box, UBB
    velocity inlet on the x-low face, fixed-density outlets on the other five
    faces (wherever a branch leaves the box)."""
    fluid = artery_tree(dims, seed=seed, **kw)
    inlet = FaceSpec(FaceKind.WALL, velocity=(float(inlet_speed), 0.0, 0.0))
    out = FaceSpec(FaceKind.WALL, density=float(outlet_density))
    faces = [(inlet, out), (out, out), (out, out)]
    return make_flags(dims, faces, solid=~fluid)
