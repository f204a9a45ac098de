"""Halo edge plans (host side) and the device exchange program.

``EdgePlan`` derives, for one directed edge (src block, dst block, offset
``sigma``) and each exchange phase, exactly the message layout of the
reference (``pkg/src/slbm/exchange.py:125-219``):

* entries enumerate the owner's boundary layer toward ``tau`` cell-major
  (z-major cell order), then the crossing direction subset in stencil
  order (``direction_subset``, exchange.py:52-66);
* CANONICAL (tau = sigma, owner = sender) ships the sender's fluid slots
  to the receiver's ghost slots; REVERSED (tau = -sigma, owner = receiver)
  ships the sender's ghost slots, where the combined AA step parked
  boundary-crossing values, to the receiver's interior opposite slots;
* only ``storable`` entries (both endpoint cells fluid, partner in the box)
  are written; the sparse wire carries ``owner_fluid`` (CANONICAL) or
  ``storable`` (REVERSED) entries.

Slot lists are resolved by whichever side owns the engine: the sender's
``send_sel`` needs the source engine, the receiver's ``tgt_sel`` the
destination engine, and the wire layout needs only the two flag boxes,
so a rank can plan its half of a cross-rank edge alone.

``DeviceHalo`` hands the resolved lists to the CUDA exchange program
(``slbm_halo_*``): local edges become one fused gather-scatter kernel per
phase, remote edges per-peer pack / ncclSend / ncclRecv / unpack on the
halo's comm stream.
"""

from __future__ import annotations

import ctypes as C
from enum import Enum

import numpy as np

from . import _abi, errors
from .collision import Parity
from .tags import FLUID


class Phase(Enum):
    CANONICAL = 0
    REVERSED = 1


def phase_for(pattern: str, parity) -> Phase:
    """exchange.py:313-316"""
    if pattern == "pull" or getattr(parity, "value", parity) == Parity.EVEN.value:
        return Phase.CANONICAL
    return Phase.REVERSED


def direction_subset(stencil, tau) -> tuple[int, ...]:
    """Directions whose nonzero components all agree with tau's nonzero
    components (exchange.py:52-66)."""
    if not any(tau):
        raise errors.make("ConfigurationError", "offset vector must be nonzero")
    fixed = [(a, t) for a, t in enumerate(tau) if t != 0]
    return tuple(k for k in range(1, stencil.q) if all(int(stencil.c[k][a]) == t for a, t in fixed))


def analytic_payload(dims, tau, stencil) -> int:
    n = len(direction_subset(stencil, tau))
    for axis, t in enumerate(tau):
        if t == 0:
            n *= int(dims[axis])
    return n


def layer_cells(dims, tau) -> np.ndarray:
    """Public coords of the boundary layer toward tau, z-major order
    (exchange.py:78-92)."""
    nd = len(dims)
    axes = []
    for arr_axis in range(nd):
        axis = nd - 1 - arr_axis
        t = tau[axis]
        axes.append(np.array([dims[axis] - 1]) if t == 1 else (np.array([0]) if t == -1 else np.arange(dims[axis])))
    mesh = np.meshgrid(*axes, indexing="ij")
    rev = np.stack([m.reshape(-1) for m in mesh], axis=1)
    return np.ascontiguousarray(rev[:, ::-1]).astype(np.int64)


def _tags_at(flags, coords) -> np.ndarray:
    pad = coords[:, ::-1] + 1
    return flags.tags[tuple(pad.T)]


class PhasePlan:
    __slots__ = ("subset", "n_full", "n_wire", "send_sel", "tgt_sel", "pos_from_full",
                 "pos_from_sparse", "sparse_in_full", "_send_cells", "_send_qs", "_tgt_cells",
                 "_tgt_qs", "n_msg", "take")
    # n_msg / take: message length and stored positions for THIS edge's
    # sender layout (whole layer for a dense sender, existing slots for a
    # sparse one; exchange.py:203-207, :242-247)


class EdgePlan:
    """exchange.py:125-219; engines may be None for the remote end."""

    def __init__(self, src_bid, dst_bid, sigma, stencil, src_flags, dst_flags, pattern,
                 src_engine=None, dst_engine=None, src_layout=None):
        for axis, t in enumerate(sigma):
            if t == 0 and src_flags.dims[axis] != dst_flags.dims[axis]:
                raise errors.make("ConfigurationError", "adjacent blocks must share extents on in-face axes")
        for e in (src_engine, dst_engine):
            if e is not None and e.pattern != pattern:
                raise errors.make("ConfigurationError", "blocks must share one streaming pattern")
        self.src_bid, self.dst_bid = src_bid, dst_bid
        self.sigma = tuple(int(s) for s in sigma)
        self.stencil = stencil
        self.src_flags, self.dst_flags = src_flags, dst_flags
        self.src_engine, self.dst_engine = src_engine, dst_engine
        self.pattern = pattern
        if src_layout is None:
            src_layout = getattr(src_engine, "layout", "sparse")
        self.src_layout = src_layout
        self.phases = {Phase.CANONICAL: self._build(Phase.CANONICAL)}
        if pattern == "aa":
            self.phases[Phase.REVERSED] = self._build(Phase.REVERSED)

    def _build(self, phase: Phase) -> PhasePlan:
        st = self.stencil
        canonical = phase is Phase.CANONICAL
        owner_fl = self.src_flags if canonical else self.dst_flags
        partner_fl = self.dst_flags if canonical else self.src_flags
        tau = self.sigma if canonical else tuple(-t for t in self.sigma)
        subset = direction_subset(st, tau)
        cells = layer_cells(owner_fl.dims, tau)
        ns = len(subset)
        ecells = np.repeat(cells, ns, axis=0)
        eqs = np.tile(np.asarray(subset, dtype=np.int64), cells.shape[0])
        n_full = eqs.shape[0]
        # owner layer seen from the partner block (its halo ring)
        shift = np.zeros(st.dim, dtype=np.int64)
        for axis, t in enumerate(self.sigma):
            if t == 1:
                shift[axis] = -self.src_flags.dims[axis]
            elif t == -1:
                shift[axis] = self.dst_flags.dims[axis]
        if not canonical:
            shift = -shift
        eimg = ecells + shift
        target = eimg + st.c[eqs]
        for axis, per in enumerate(partner_fl.periodic):
            if per:
                target[:, axis] %= partner_fl.dims[axis]
        in_box = np.all((target >= 0) & (target < np.asarray(partner_fl.dims)), axis=1)
        owner_fluid = _tags_at(owner_fl, ecells) == FLUID
        partner_fluid = np.zeros(n_full, dtype=bool)
        if in_box.any():
            partner_fluid[in_box] = _tags_at(partner_fl, target[in_box]) == FLUID
        storable = owner_fluid & in_box & partner_fluid
        wire = owner_fluid if canonical else storable

        pp = PhasePlan()
        pp.subset = subset
        pp.n_full = n_full
        pp.n_wire = int(wire.sum())
        pp.pos_from_full = np.nonzero(storable)[0]
        pp.pos_from_sparse = np.nonzero(storable[wire])[0]
        pp.sparse_in_full = np.nonzero(wire)[0]
        if self.src_layout == "dense":
            pp._send_cells = ecells if canonical else eimg
            pp._send_qs = eqs
            pp.n_msg, pp.take = n_full, pp.pos_from_full
        else:
            pp._send_cells = ecells[wire] if canonical else eimg[wire]
            pp._send_qs = eqs[wire]
            pp.n_msg, pp.take = pp.n_wire, pp.pos_from_sparse
        pp._tgt_cells = eimg[storable] if canonical else ecells[storable]
        pp._tgt_qs = eqs[storable]
        pp.send_sel = None
        pp.tgt_sel = None
        if self.src_engine is not None:
            lookup = self.src_engine.slot_index if canonical else self.src_engine.ghost_slot_index
            pp.send_sel = lookup(pp._send_cells, pp._send_qs) if pp.n_msg else np.empty(0, np.int64)
        if self.dst_engine is not None:
            lookup = self.dst_engine.ghost_slot_index if canonical else self.dst_engine.slot_index
            pp.tgt_sel = (lookup(pp._tgt_cells, pp._tgt_qs) if pp._tgt_qs.size
                          else np.empty(0, np.int64))
        return pp


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64).reshape(-1))


class DeviceHalo:
    """The CUDA exchange program of one process (slbm_halo_*).

    ``peer=(rank, world, group)`` selects the peer transport: remote
    messages are stored by the pack kernel straight into the peers' receive
    buffers (CUDA IPC over NVLink) with epoch flags instead of NCCL; the
    IPC handles and receive sections travel once through ``group`` (any
    torch.distributed backend; not used when world == 1)."""

    def __init__(self, device: int, peer: tuple | None = None):
        self.device = int(device)
        h = C.c_void_p()
        _abi.call("slbm_halo_create", self.device, C.byref(h))
        self._h = h
        self.committed = False
        self.has_remote = False
        self.peer = peer
        if peer is not None:
            _abi.call("slbm_halo_use_peer", self._h, int(peer[0]))

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _abi.load().slbm_halo_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def add_local(self, phase: Phase, src, dst, pp: PhasePlan):
        send, take, tgt = _i64(pp.send_sel), _i64(pp.take), _i64(pp.tgt_sel)
        _abi.call("slbm_halo_add_local", self._h, phase.value, src.handle, dst.handle,
                  _abi.ptr(send, C.c_int64), send.size, _abi.ptr(take, C.c_int64),
                  _abi.ptr(tgt, C.c_int64), tgt.size)

    def add_send(self, phase: Phase, src, peer: int, pp: PhasePlan):
        send = _i64(pp.send_sel)
        self.has_remote = True
        _abi.call("slbm_halo_add_send", self._h, phase.value, src.handle, int(peer),
                  _abi.ptr(send, C.c_int64), send.size)

    def add_recv(self, phase: Phase, dst, peer: int, pp: PhasePlan):
        take, tgt = _i64(pp.take), _i64(pp.tgt_sel)
        self.has_remote = True
        _abi.call("slbm_halo_add_recv", self._h, phase.value, dst.handle, int(peer), pp.n_msg,
                  _abi.ptr(take, C.c_int64), _abi.ptr(tgt, C.c_int64), tgt.size)

    def commit(self, nccl_comm: int | None = None):
        _abi.call("slbm_halo_commit", self._h, C.c_void_p(nccl_comm or 0))
        self.committed = True
        if self.peer is not None:
            self._connect_peers()

    def _connect_peers(self):
        rank, world, group = self.peer
        recv_h = (C.c_char * 64)()
        flag_h = (C.c_char * 64)()
        _abi.call("slbm_halo_ipc_handles", self._h, C.cast(recv_h, C.c_void_p),
                  C.cast(flag_h, C.c_void_p))
        # per sender s and phase: where s's message lands in this rank's buffer
        sections = {}
        for s in range(world):
            rows = []
            for ph in (Phase.CANONICAL, Phase.REVERSED):
                off, cnt = C.c_int64(), C.c_int64()
                _abi.call("slbm_halo_recv_section", self._h, ph.value, s, C.byref(off),
                          C.byref(cnt))
                rows.append((off.value, cnt.value))
            sections[s] = rows
        mine = {"rank": rank, "recv": bytes(recv_h), "flags": bytes(flag_h), "sections": sections}
        if world == 1:
            infos = [mine]
        else:
            import torch.distributed as dist

            infos = [None] * world
            dist.all_gather_object(infos, mine, group=group)
        for info in infos:
            r = info["rank"]
            to_r = info["sections"][rank]  # my message's place in r's buffer, per phase
            from_r = sections[r]           # r's message in my buffer
            if not any(c for _, c in to_r) and not any(c for _, c in from_r):
                continue
            off = np.array([o for o, _ in to_r], np.int64)
            cnt = np.array([c for _, c in to_r], np.int64)
            a = (C.c_char * 64).from_buffer_copy(info["recv"])
            b = (C.c_char * 64).from_buffer_copy(info["flags"])
            _abi.call("slbm_halo_connect", self._h, r, C.cast(a, C.c_void_p),
                      C.cast(b, C.c_void_p), _abi.ptr(off, C.c_int64), _abi.ptr(cnt, C.c_int64))

    def start(self, phase: Phase, after_stream: int | None, with_local: bool = True):
        _abi.call("slbm_halo_start_ex", self._h, phase.value, C.c_void_p(after_stream or 0),
                  1 if with_local else 0)

    def local_on(self, phase: Phase, stream: int | None):
        """Only the device-local edges, on ``stream``."""
        _abi.call("slbm_halo_local_on", self._h, phase.value, C.c_void_p(stream or 0))

    def wait(self, stream: int | None):
        _abi.call("slbm_halo_wait", self._h, C.c_void_p(stream or 0))

    def local_only(self, phase: Phase):
        _abi.call("slbm_halo_local", self._h, phase.value)

    def peer_sizes(self, phase: Phase, npeers: int):
        s = np.zeros(npeers, np.int64)
        r = np.zeros(npeers, np.int64)
        _abi.call("slbm_halo_peer_sizes", self._h, phase.value, npeers, _abi.ptr(s, C.c_int64),
                  _abi.ptr(r, C.c_int64))
        return s, r

    def pack_host(self, phase: Phase, peer: int, out: np.ndarray):
        _abi.call("slbm_halo_pack_host", self._h, phase.value, int(peer), _abi.ptr(out, C.c_double))

    def unpack_host(self, phase: Phase, peer: int, buf: np.ndarray):
        buf = np.ascontiguousarray(buf, dtype=np.float64)
        _abi.call("slbm_halo_unpack_host", self._h, phase.value, int(peer), _abi.ptr(buf, C.c_double))


class NcclComm:
    """NCCL communicator owned by the library (ncclCommInitRank); the
    unique id travels through any torch.distributed backend."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        uid = (C.c_char * 128)()
        if world == 1:
            # single-rank communicator (loopback tests): no rendezvous needed
            _abi.call("slbm_nccl_get_unique_id", C.cast(uid, C.c_void_p))
            rank = 0
        else:
            import torch.distributed as dist

            if rank == 0:
                _abi.call("slbm_nccl_get_unique_id", C.cast(uid, C.c_void_p))
            payload = [bytes(uid)]
            dist.broadcast_object_list(payload, src=0, group=group)
            uid = (C.c_char * 128).from_buffer_copy(payload[0])
        comm = C.c_void_p()
        _abi.call("slbm_nccl_comm_init", C.cast(uid, C.c_void_p), world, rank, device, C.byref(comm))
        self.handle = comm.value

    def close(self):
        if self.handle:
            _abi.load().slbm_nccl_comm_destroy(C.c_void_p(self.handle))
            self.handle = None
