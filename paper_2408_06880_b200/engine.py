"""GPU-backed sparse block engine: the drop-in for the reference's
``SparseEngine`` (``pkg/src/slbm/sparse.py:48-383``).

Same constructor, attributes, methods, error types and counter updates as
the reference engine protocol; every operation is one C-ABI
call into ``libslbm_b200.so`` (``include/slbm_b200.h``), which owns the PDF
buffers, the index list and the stream.  Nothing here computes LBM
arithmetic on the host; without the CUDA library the constructor raises.

Differences a caller can observe:

* ``check`` (keyword, default ``"step"``): after every ``step`` the
  instability flag written by the sweep kernel is polled, so
  ``NumericalInstabilityError`` surfaces on the same call as in the
  reference.  ``check="deferred"`` skips the per-step host sync; the flag
  is then reported by :meth:`poll` / :meth:`canonical_state` /
  :meth:`macroscopic_fields` with the first bad step number.
* ``run(n)`` advances ``n`` whole single-block steps without returning to
  Python (optionally via a captured CUDA graph of one step pair).
* ``fluid_coords`` and ``idx`` are exported from the device on first access.
* Extensions: ``macroscopic_fields(out=...)`` (pinned buffers are written
  directly by the field kernel), ``macroscopic_compact()``, ``set_frame``
  (per-face frames), ``device_state()`` / ``pdf_layout()`` (the device PDF
  array: 256-B aligned direction groups; slot ids elsewhere are the
  reference's), ``frame_width=HaloWidths(...)`` (0 = no frame on an axis).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _abi, errors
from .collision import cumulant_rates, is_even, params_code, parity_class
from .counters import Counters
from .lattice import stencil_code
from .tags import OUTLET, UBB, rev_shape

PATTERNS = ("pull", "aa")
_PHASE_CODE = {"all": 0, "interior": 1, "frame": 2}


def default_device() -> int:
    for key in ("SLBM_DEVICE", "LOCAL_RANK"):
        if key in os.environ:
            return int(os.environ[key])
    return 0


class HaloWidths(tuple):
    """Per-axis frame widths that may contain 0 = no frame on that axis.

    The reference's ``frame_mask`` requires every width >= 1 (flags.py:83-108)
    and so does this layer for plain ints/tuples.  The domain drivers use
    this type for blocks whose axes have no halo exchange (in-block periodic
    wrap or a single block along the axis): those faces need no frame, and
    dropping them leaves a frame of whole z planes whose cells are
    contiguous in cid order (profiles: x faces make the frame sweep a
    scattered gather)."""


def _widths(frame_width, dim):
    if frame_width is None:
        return None
    if isinstance(frame_width, HaloWidths):
        widths = tuple(int(w) for w in frame_width)
        if len(widths) != dim or min(widths) < 0:
            raise errors.make("ConfigurationError", f"bad halo frame widths {widths}")
        return widths
    if isinstance(frame_width, (int, np.integer)):
        widths = (int(frame_width),) * dim
    else:
        widths = tuple(int(w) for w in frame_width)
    if len(widths) != dim:
        raise errors.make(
            "ConfigurationError", f"need one frame width per axis, got {len(widths)} for {dim} axes"
        )
    if min(widths) < 1:
        raise errors.make("ConfigurationError", f"frame widths must be >= 1, got {widths}")
    return widths


class SparseEngine:
    layout = "sparse"
    _CREATE = "slbm_engine_create"

    def __init__(self, flags, stencil, params, pattern: str = "pull", frame_width=None,
                 device: int | None = None, check: str = "step"):
        if pattern not in PATTERNS:
            raise errors.make("ConfigurationError", f"unknown streaming pattern {pattern!r}")
        if len(flags.dims) != stencil.dim:
            raise errors.make(
                "ConfigurationError", f"{stencil.name} needs {stencil.dim}-d dims, got {flags.dims}"
            )
        if check not in ("step", "deferred"):
            raise errors.make("ConfigurationError", f"unknown check mode {check!r}")
        self.flags = flags
        self.stencil = stencil
        self.params = params
        self.pattern = pattern
        self.dims = tuple(int(d) for d in flags.dims)
        self.frame_width = frame_width
        self.check = check
        self.device = default_device() if device is None else int(device)
        self._h = None
        dim = stencil.dim
        widths = _widths(frame_width, dim)

        tags = np.ascontiguousarray(flags.tags, dtype=np.uint8)
        want = tuple(n + 2 for n in rev_shape(self.dims))
        if tags.shape != want:
            raise errors.make("ConfigurationError", f"tag box shape {tags.shape} != {want}")
        ubb = None
        if np.any((tags == UBB) | (tags == OUTLET)):
            ubb = np.ascontiguousarray(flags.ubb_u, dtype=np.float64)
            if ubb.shape != want + (dim,):
                raise errors.make("ConfigurationError", f"ubb_u shape {ubb.shape} != {want + (dim,)}")
        dims32 = np.array(list(self.dims) + [1] * (3 - dim), dtype=np.int32)
        per = np.array([1 if p else 0 for p in flags.periodic] + [0] * (3 - dim), dtype=np.uint8)
        fw = None if widths is None else np.array(list(widths) + [1] * (3 - dim), dtype=np.int32)
        model, omega, lam = params_code(params)
        handle = C.c_void_p()
        _abi.call(
            self._CREATE,
            _abi.ptr(tags, C.c_uint8),
            _abi.ptr(ubb, C.c_double),
            dim,
            _abi.ptr(dims32, C.c_int32),
            _abi.ptr(per, C.c_uint8),
            stencil_code(stencil),
            model,
            omega,
            lam,
            PATTERNS.index(pattern),
            _abi.ptr(fw, C.c_int32),
            self.device,
            C.byref(handle),
        )
        self._h = handle
        if getattr(params, "model", "srt") == "cumulant":
            bulk, higher = cumulant_rates(params)
            if bulk != 1.0 or higher is not None:
                self.set_cumulant_rates(bulk, higher)
        info = self.info()
        q = stencil.q
        self.n_fluid = int(info.n_fluid)
        self.total_slots = int(info.total_slots)
        self.n_ubb_slots = int(info.n_ubb_slots)
        self.n_ghost_slots = int(info.n_ghost_slots)
        self.n_outlet_slots = int(info.n_outlet_slots)
        self.base = np.array(info.base[: q + 1], dtype=np.int64)
        self._has_split = bool(info.has_split)
        self._n_interior = int(info.n_interior)
        self._n_frame = int(info.n_frame)
        self.parity = parity_class().EVEN
        self.counters = Counters()
        self._fluid_coords = None
        self._cid_map = None  # host copy for slot_index, fetched on first use
        self._idx = None
        self._padded_shape = want
        self._steps_issued = 0

    # -- lifetime ---------------------------------------------------------------

    def close(self) -> None:
        if self._h is not None and self._h.value:
            _abi.load().slbm_engine_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def info(self) -> _abi.SlbmInfo:
        info = _abi.SlbmInfo()
        _abi.call("slbm_engine_info", self._h, C.byref(info))
        return info

    # -- exported lists -----------------------------------------------------------

    @property
    def fluid_coords(self) -> np.ndarray:
        if self._fluid_coords is None:
            out = np.empty((self.n_fluid, self.stencil.dim), dtype=np.int64)
            _abi.call("slbm_export_lists", self._h, None, _abi.ptr(out, C.c_int64),
                      None, None, None, None, None, None)
            self._fluid_coords = out
        return self._fluid_coords

    @property
    def idx(self) -> np.ndarray:
        if self._idx is None:
            out = np.empty((self.stencil.q - 1, self.n_fluid), dtype=np.uint32)
            _abi.call("slbm_export_lists", self._h, _abi.ptr(out, C.c_uint32), None,
                      None, None, None, None, None, None)
            self._idx = out
        return self._idx

    def export_boundary_lists(self) -> dict:
        """UBB slots/partners/corrections and ghost (q, padded flat) -> slot
        entries, in the reference's order (sparse.py:157-191)."""
        nu, ng = self.n_ubb_slots, self.n_ghost_slots
        us = np.empty(nu, np.int64)
        up = np.empty(nu, np.int64)
        uc = np.empty(nu, np.float64)
        gq = np.empty(ng, np.int64)
        gp = np.empty(ng, np.int64)
        gs = np.empty(ng, np.int64)
        _abi.call("slbm_export_lists", self._h, None, None, _abi.ptr(us, C.c_int64),
                  _abi.ptr(up, C.c_int64), _abi.ptr(uc, C.c_double), _abi.ptr(gq, C.c_int64),
                  _abi.ptr(gp, C.c_int64), _abi.ptr(gs, C.c_int64))
        return {"ubb_slots": us, "ubb_partner": up, "ubb_corr": uc,
                "ghost_q": gq, "ghost_pflat": gp, "ghost_slot": gs}

    def set_frame(self, lo, hi) -> None:
        """Per-face interior/frame split (extension; the reference's
        frame_mask is lo == hi >= 1): frame cells lie within lo[a] of the low
        face or hi[a] of the high face of axis a, 0 meaning none.  Used by
        the domain drivers to frame only the faces with remote neighbours."""
        dim = self.stencil.dim
        lo32 = np.array(list(lo) + [0] * (3 - dim), dtype=np.int32)
        hi32 = np.array(list(hi) + [0] * (3 - dim), dtype=np.int32)
        _abi.call("slbm_engine_set_frame", self._h, _abi.ptr(lo32, C.c_int32),
                  _abi.ptr(hi32, C.c_int32))
        info = self.info()
        self._n_interior = int(info.n_interior)
        self._n_frame = int(info.n_frame)
        self._has_split = True

    def split_lists(self) -> tuple[np.ndarray, np.ndarray]:
        """(interior cids, frame cids) (sparse.py:80-88)."""
        a = np.empty(self._n_interior, np.int64)
        b = np.empty(self._n_frame, np.int64)
        _abi.call("slbm_export_split", self._h, _abi.ptr(a, C.c_int64), _abi.ptr(b, C.c_int64))
        return a, b

    # -- state init -----------------------------------------------------------------

    def init_canonical(self, values) -> None:
        values = np.ascontiguousarray(values, dtype=np.float64)
        if values.shape != (self.stencil.q, self.n_fluid):
            raise errors.make(
                "ConfigurationError",
                f"expected state shape {(self.stencil.q, self.n_fluid)}, got {values.shape}",
            )
        _abi.call("slbm_init_canonical", self._h, _abi.ptr(values, C.c_double))
        self.parity = parity_class().EVEN

    def init_canonical_device(self, dev_ptr: int) -> None:
        """init_canonical from a device buffer of (q, n_fluid) float64."""
        _abi.call("slbm_init_canonical_dev", self._h, C.c_void_p(dev_ptr))
        _abi.call("slbm_synchronize", self._h)
        self.parity = parity_class().EVEN

    def init_equilibrium(self, rho=1.0, u=None) -> None:
        dim, n = self.stencil.dim, self.n_fluid
        rho_a = np.ascontiguousarray(np.asarray(rho, dtype=np.float64).reshape(-1))
        rho_scalar = 1 if rho_a.size == 1 else 0
        if not rho_scalar and rho_a.size != n:
            rho_a = np.ascontiguousarray(np.broadcast_to(np.asarray(rho, np.float64), (n,)))
        if u is None:
            u_a = np.zeros(dim)
            u_scalar = 1
        else:
            u_in = np.asarray(u, dtype=np.float64)
            if u_in.ndim == 1:
                u_a, u_scalar = np.ascontiguousarray(u_in), 1
            else:
                u_a = np.ascontiguousarray(np.broadcast_to(u_in, (dim, n)))
                u_scalar = 0
        _abi.call("slbm_init_equilibrium", self._h, _abi.ptr(rho_a, C.c_double), rho_scalar,
                  _abi.ptr(u_a, C.c_double), u_scalar)
        self.parity = parity_class().EVEN

    # -- stepping -------------------------------------------------------------------

    def _phase_cells(self, phase: str) -> int:
        if phase == "all":
            return self.n_fluid
        if self._has_split and phase in ("interior", "frame"):
            return self._n_interior if phase == "interior" else self._n_frame
        raise errors.make(
            "ConfigurationError", f"{phase!r} sweep needs split lists; build with frame_width"
        )

    def step(self, phase: str = "all") -> None:
        cells = self._phase_cells(phase)
        _abi.call("slbm_step", self._h, _PHASE_CODE[phase])
        table_reads = self.pattern == "pull" or is_even(self.parity)
        self.counters.record_sweep(phase, cells, self.stencil.q, table_reads)
        if self.check == "step":
            self.poll()

    def finish_step(self) -> None:
        _abi.call("slbm_finish_step", self._h)
        if self.pattern == "aa":
            self.parity = self.parity.flipped()
        self.counters.steps += 1

    def refresh_boundary(self, parity) -> None:
        code = parity.value if hasattr(parity, "value") else int(parity)
        _abi.call("slbm_refresh_boundary", self._h, int(code))

    def run(self, steps: int, use_graph: bool = True) -> None:
        """``steps`` x (refresh_boundary, step("all"), finish_step) on the
        device without host round trips; counters advance as if driven
        step by step."""
        steps = int(steps)
        if steps <= 0:
            return
        q = self.stencil.q
        for _ in range(steps):
            table_reads = self.pattern == "pull" or is_even(self.parity)
            self.counters.record_sweep("all", self.n_fluid, q, table_reads)
            if self.pattern == "aa":
                self.parity = self.parity.flipped()
            self.counters.steps += 1
        _abi.call("slbm_run", self._h, steps, 1 if use_graph else 0)
        if self.check == "step":
            self.poll()

    def poll(self) -> None:
        """Raise NumericalInstabilityError if any sweep since the last poll
        saw a non-positive or non-finite density (synchronizes)."""
        bad = C.c_int64(-1)
        lib = _abi.load()
        status = lib.slbm_poll_instability(self._h, C.byref(bad))
        if status != 0:
            msg = lib.slbm_last_error().decode(errors="replace")
            if bad.value >= 0:
                msg = f"{msg} (engine step {bad.value})"
            errors.raise_for_status(status, msg)

    def synchronize(self) -> None:
        _abi.call("slbm_synchronize", self._h)

    def set_cumulant_rates(self, bulk: float = 1.0, higher=None, force_general: bool = False) -> None:
        """Cumulant model: bulk rate w2 and higher-order rates w3..w10
        (include/slbm_b200.h slbm_engine_set_cumulant_rates)."""
        arr = None
        if higher is not None:
            arr = np.ascontiguousarray(np.asarray(higher, dtype=np.float64).reshape(8))
        _abi.call("slbm_engine_set_cumulant_rates", self._h, float(bulk),
                  _abi.ptr(arr, C.c_double), 1 if force_general else 0)

    def set_tuning(self, knob: int, value: int) -> None:
        """Kernel-selection knob of THIS engine (include/slbm_b200.h, knobs
        0-9); drops the engine's captured step-pair graphs."""
        _abi.call("slbm_engine_set_tuning", self._h, int(knob), int(value))

    def buffer_state(self) -> int:
        """Pull: 1 when the second buffer is current, else 0; AA: 0."""
        st = C.c_int(0)
        _abi.call("slbm_buffer_state", self._h, C.byref(st))
        return int(st.value)

    def stream(self) -> int:
        s = C.c_void_p()
        _abi.call("slbm_engine_stream", self._h, C.byref(s))
        return s.value or 0

    def set_stream(self, stream: int | None) -> None:
        _abi.call("slbm_engine_set_stream", self._h, C.c_void_p(stream or 0))

    # -- inspection -----------------------------------------------------------------

    def canonical_state(self) -> np.ndarray:
        if self.check == "deferred":
            self.poll()
        out = np.empty((self.stencil.q, self.n_fluid), dtype=np.float64)
        _abi.call("slbm_canonical_state", self._h, _abi.ptr(out, C.c_double))
        return out

    def macroscopic_fields(self, out=None) -> tuple[np.ndarray, np.ndarray]:
        """sparse.py:323-331: (rho, u) over the block, zeros at solids.
        ``out=(rho, u)`` (extension) writes into caller-owned C-contiguous
        float64 arrays of those shapes — e.g. pinned host buffers, which the
        library reads back with one DMA instead of the staged copy."""
        if self.check == "deferred":
            self.poll()
        shape = rev_shape(self.dims)
        ushape = shape + (self.stencil.dim,)
        if out is None:
            rho = np.empty(shape, dtype=np.float64)
            u = np.empty(ushape, dtype=np.float64)
        else:
            rho, u = out
            for a, want in ((rho, shape), (u, ushape)):
                if (a.shape != want or a.dtype != np.float64 or not a.flags.c_contiguous
                        or not a.flags.writeable):
                    raise errors.make("ConfigurationError",
                                      f"out arrays must be writeable C-contiguous float64 of "
                                      f"shapes {shape} and {ushape}")
        _abi.call("slbm_macroscopic", self._h, _abi.ptr(rho, C.c_double), _abi.ptr(u, C.c_double))
        return rho, u

    def pdf_layout(self) -> tuple[np.ndarray, int]:
        """Device layout of the PDF array: direction-group starts (Q + 1) and
        the element count.  Sparse engines pad each group to 32 slots; slot
        ids in every other call are the reference's."""
        starts = np.zeros(self.stencil.q + 1, dtype=np.int64)
        n = C.c_int64()
        _abi.call("slbm_pdf_layout", self._h, _abi.ptr(starts, C.c_int64), C.byref(n))
        return starts, int(n.value)

    def device_state(self):
        """Zero-copy torch view (float64) of the active PDF buffer in its
        device layout (see :meth:`pdf_layout`; synchronizes first).  For
        device-side checks at full size."""
        import torch

        ptr = C.c_void_p()
        _abi.call("slbm_pdf_pointer", self._h, C.byref(ptr))
        self.synchronize()
        n = self.pdf_layout()[1]

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                        "data": (int(ptr.value or 0), False), "version": 3}

        return torch.as_tensor(_View(), device=f"cuda:{self.device}")

    def macroscopic_compact(self) -> tuple[np.ndarray, np.ndarray]:
        """(rho, u) per fluid cell in cid order, shapes (n_fluid,) and
        (n_fluid, dim): the values macroscopic_fields scatters into the box
        (pair with ``fluid_coords``)."""
        if self.check == "deferred":
            self.poll()
        rho = np.empty(self.n_fluid, dtype=np.float64)
        u = np.empty((self.n_fluid, self.stencil.dim), dtype=np.float64)
        _abi.call("slbm_macroscopic_compact", self._h, _abi.ptr(rho, C.c_double),
                  _abi.ptr(u, C.c_double))
        return rho, u

    def total_mass(self) -> float:
        m = C.c_double()
        _abi.call("slbm_total_mass", self._h, C.byref(m))
        return float(m.value)

    @property
    def sweep_ctas(self) -> int:
        """CTAs per SM of the index-list sweep (knob 13 or the engine's own
        measurement; 0 while undecided)."""
        v = C.c_int()
        _abi.call("slbm_engine_sweep_ctas", self._h, C.byref(v))
        return int(v.value)

    def total_moments(self) -> np.ndarray:
        """(mass, momentum x, y, z) of the canonical state: one device pass,
        warp-shuffle reductions in a fixed order (bit-reproducible)."""
        out = np.zeros(4)
        _abi.call("slbm_total_moments", self._h, _abi.ptr(out, C.c_double))
        return out

    # -- exchange access ------------------------------------------------------------

    def _pflat(self, coords: np.ndarray) -> np.ndarray:
        coords = np.asarray(coords, dtype=np.int64).reshape(-1, self.stencil.dim)
        p = np.zeros(coords.shape[0], dtype=np.int64)
        for arr_axis, extent in enumerate(self._padded_shape):
            axis = self.stencil.dim - 1 - arr_axis
            p = p * extent + (coords[:, axis] + 1)
        return p

    def _lookup(self, fn: str, coords, qs) -> np.ndarray:
        pflat = self._pflat(coords)
        qs = np.ascontiguousarray(np.broadcast_to(np.asarray(qs, dtype=np.int64).reshape(-1),
                                                  pflat.shape))
        out = np.empty(pflat.shape[0], dtype=np.int64)
        _abi.call(fn, self._h, _abi.ptr(qs, C.c_int64), _abi.ptr(pflat, C.c_int64),
                  pflat.shape[0], _abi.ptr(out, C.c_int64))
        return out

    def slot_index(self, coords, qs) -> np.ndarray:
        """sparse.py:335-343.  Sparse engines resolve it on the host from a
        copy of the device cid map (fetched once): halo planning asks for
        thousands of these, each a GPU round trip otherwise."""
        if self.layout != "sparse":
            return self._lookup("slbm_slot_index", coords, qs)
        if self._cid_map is None:
            cm = np.empty(int(np.prod(self._padded_shape)), dtype=np.int32)
            _abi.call("slbm_export_cid_map", self._h, _abi.ptr(cm, C.c_int32))
            self._cid_map = cm
        pflat = self._pflat(coords)
        qs = np.broadcast_to(np.asarray(qs, dtype=np.int64).reshape(-1), pflat.shape)
        ok = (qs >= 0) & (qs < self.stencil.q) & (pflat >= 0) & (pflat < self._cid_map.size)
        cid = np.full(pflat.shape, -1, dtype=np.int64)
        cid[ok] = self._cid_map[pflat[ok]]
        if not np.all(cid >= 0):
            raise errors.make("ProtocolError", "exchange addressed a non-fluid cell slot")
        return np.asarray(self.base, dtype=np.int64)[qs] + cid

    def ghost_slot_index(self, coords, qs) -> np.ndarray:
        """sparse.py:345-360"""
        return self._lookup("slbm_ghost_slot_index", coords, qs)

    def read_slots(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).reshape(-1))
        out = np.empty(idx.shape[0], dtype=np.float64)
        _abi.call("slbm_read_slots", self._h, _abi.ptr(idx, C.c_int64), idx.shape[0],
                  _abi.ptr(out, C.c_double))
        return out

    def write_slots(self, idx, values) -> None:
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).reshape(-1))
        vals = np.ascontiguousarray(np.broadcast_to(np.asarray(values, np.float64), idx.shape))
        _abi.call("slbm_write_slots", self._h, _abi.ptr(idx, C.c_int64), idx.shape[0],
                  _abi.ptr(vals, C.c_double))

    # -- bookkeeping ----------------------------------------------------------------

    def pdf_element_count(self) -> int:
        return (2 if self.pattern == "pull" else 1) * self.total_slots

    def idx_element_count(self) -> int:
        return (self.stencil.q - 1) * self.n_fluid

    @property
    def n_interior(self) -> int:
        return self._n_interior if self._has_split else self.n_fluid

    @property
    def n_frame(self) -> int:
        return self._n_frame if self._has_split else 0

    @property
    def device_bytes(self) -> int:
        return int(self.info().device_bytes)


class DenseEngine(SparseEngine):
    """GPU direct-addressing engine: the reference's ``DenseEngine``
    (``pkg/src/slbm/dense.py:52-342``), same protocol.  Storage is one
    plane per direction over the padded box (slot = q * npad + p), reads are
    computed from coordinates plus a per-cell wall-fold mask (no index list),
    and the counters count box cells like the reference (dense.py:290-297).
    Fluid results are bit-identical to :class:`SparseEngine`'s."""

    layout = "dense"
    _CREATE = "slbm_engine_create_dense"

    @property
    def idx(self):
        raise AttributeError("a dense engine has no index list")

    def _box_cells(self) -> int:
        return int(np.prod(self.dims))

    def _phase_cells(self, phase: str) -> int:
        if phase == "all":
            return self._box_cells()
        if self._has_split and phase in ("interior", "frame"):
            return self._n_interior if phase == "interior" else self._n_frame
        raise errors.make(
            "ConfigurationError", f"{phase!r} sweep needs split lists; build with frame_width"
        )

    def step(self, phase: str = "all") -> None:
        cells = self._phase_cells(phase)
        _abi.call("slbm_step", self._h, _PHASE_CODE[phase])
        self.counters.record_sweep(phase, cells, self.stencil.q, False)
        if self.check == "step":
            self.poll()

    def run(self, steps: int, use_graph: bool = True) -> None:
        steps = int(steps)
        if steps <= 0:
            return
        for _ in range(steps):
            self.counters.record_sweep("all", self._box_cells(), self.stencil.q, False)
            if self.pattern == "aa":
                self.parity = self.parity.flipped()
            self.counters.steps += 1
        _abi.call("slbm_run", self._h, steps, 1 if use_graph else 0)
        if self.check == "step":
            self.poll()

    def export_boundary_lists(self) -> dict:
        raise errors.make("ConfigurationError", "a dense engine resolves walls in its fold mask")

    def pdf_element_count(self) -> int:
        return (2 if self.pattern == "pull" else 1) * self.stencil.q * self._box_cells()

    def idx_element_count(self) -> int:
        return 0

    @property
    def n_interior(self) -> int:
        return self._n_interior if self._has_split else self._box_cells()

    @property
    def n_frame(self) -> int:
        return self._n_frame if self._has_split else 0
