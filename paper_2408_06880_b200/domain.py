"""Block decomposition and the time-step drivers on the GPU.

``Domain`` mirrors the reference's (``pkg/src/slbm/domain.py``): uniform
blocks cut from one padded global flag box, all-solid blocks dropped,
remote fluid in each block's ring retagged EXCHANGE (only on axes that do
not wrap inside the block), z-major block ids, edges over the stencil's
offsets, and the sequential / overlapped drivers of
``exchange.py:330-374``.  Every block engine is a CUDA
:class:`~paper_2408_06880_b200.engine.SparseEngine`; halo traffic is the
device exchange program of :class:`~paper_2408_06880_b200.halo.DeviceHalo`
(no host mailbox).

``DistributedDomain`` is the one-process-per-GPU version: every rank
derives the same partition and edge list, builds engines only for the
blocks assigned to it, and exchanges cross-rank edges with NCCL send/recv
(one message per peer per phase) on a comm stream that overlaps the
interior sweep.

Layout policies "sparse", "dense" and "hybrid" (dense at porosity >= phi_s)
follow the reference (``domain.py:58-65``); dense blocks are
:class:`~paper_2408_06880_b200.engine.DenseEngine` (direct addressing), and a
dense sender ships its whole layer (reference wire format), of which the
receiver stores the storable entries.
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field

import numpy as np

from . import errors
from .collision import is_even
from .counters import Counters
from .engine import DenseEngine, SparseEngine, default_device
from .halo import DeviceHalo, EdgePlan, NcclComm, Phase, phase_for
from .tags import EXCHANGE, FLUID, NOSLIP, FlagField, rev_shape

POLICIES = ("sparse", "dense", "hybrid")
DEFAULT_PHI_S = 0.8


@dataclass
class Block:
    bid: int
    grid_pos: tuple[int, ...]
    origin: tuple[int, ...]
    flags: FlagField
    n_fluid: int
    kind: str = "sparse"
    engine: object = None
    rank: int = 0
    neighbors: dict = field(default_factory=dict)

    @property
    def porosity(self) -> float:
        return self.n_fluid / self.flags.cell_count()


# ---------------------------------------------------------------- partition helpers


def grid_positions(grid):
    """z-major enumeration of block grid positions (domain.py:359-367)."""
    nd = len(grid)
    for flat in range(int(np.prod(grid))):
        pos, rem = [], flat
        for a in range(nd):
            pos.append(rem % grid[a])
            rem //= grid[a]
        yield tuple(pos)


def grid_linear(pos, grid) -> int:
    out = 0
    for a in reversed(range(len(grid))):
        out = out * grid[a] + pos[a]
    return out


def pad_to_multiple(gf: FlagField, block_size) -> FlagField:
    """NOSLIP filler up to a block multiple on walled axes (domain.py:407-429)."""
    nd = len(gf.dims)
    pads = []
    for a in range(nd):
        rem = gf.dims[a] % block_size[a]
        pad = 0 if rem == 0 else block_size[a] - rem
        if pad and gf.periodic[a]:
            raise errors.make(
                "ConfigurationError",
                f"axis {a} extent {gf.dims[a]} not divisible by block size {block_size[a]} and "
                "periodic; padding would break the wrap",
            )
        pads.append(pad)
    if not any(pads):
        return gf
    new_dims = tuple(gf.dims[a] + pads[a] for a in range(nd))
    tags = np.full(tuple(n + 2 for n in rev_shape(new_dims)), NOSLIP, dtype=np.uint8)
    ubb = np.zeros(tags.shape + (nd,))
    region = tuple(slice(0, s) for s in gf.tags.shape)
    tags[region] = gf.tags
    ubb[region] = gf.ubb_u
    return FlagField(dims=new_dims, tags=tags, ubb_u=ubb, periodic=gf.periodic)


def slice_block(gf: FlagField, origin, size, block_periodic) -> FlagField:
    nd = len(size)
    sel = tuple(slice(origin[a], origin[a] + size[a] + 2) for a in reversed(range(nd)))
    tags = gf.tags[sel].copy()
    ubb = gf.ubb_u[sel]  # a view: blocks never modify it, engines copy what they upload
    # halo fluid -> EXCHANGE on axes that leave the block (domain.py:390-404)
    ring = np.zeros(tags.shape, dtype=bool)
    for arr_axis in range(nd):
        if block_periodic[nd - 1 - arr_axis]:
            continue
        lo = [slice(None)] * nd
        lo[arr_axis] = 0
        ring[tuple(lo)] = True
        lo[arr_axis] = tags.shape[arr_axis] - 1
        ring[tuple(lo)] = True
    tags[ring & (tags == FLUID)] = EXCHANGE
    return FlagField(dims=tuple(size), tags=tags, ubb_u=ubb, periodic=tuple(block_periodic))


# ---------------------------------------------------------------- load balancing


def hilbert_key(coords, bits: int) -> int:
    """Position on the Hilbert curve of a 2**bits box (Skilling transpose)."""
    x = [int(c) for c in coords]
    n = len(x)
    top = 1 << (bits - 1)
    q = top
    while q > 1:
        p = q - 1
        for i in range(n):
            if x[i] & q:
                x[0] ^= p
            else:
                t = (x[0] ^ x[i]) & p
                x[0] ^= t
                x[i] ^= t
        q >>= 1
    for i in range(1, n):
        x[i] ^= x[i - 1]
    t = 0
    q = top
    while q > 1:
        if x[n - 1] & q:
            t ^= q - 1
        q >>= 1
    x = [v ^ t for v in x]
    h = 0
    for b in range(bits - 1, -1, -1):
        for v in x:
            h = (h << 1) | ((v >> b) & 1)
    return h


def morton_key(coords, bits: int) -> int:
    h = 0
    for b in range(bits - 1, -1, -1):
        for c in coords:
            h = (h << 1) | ((int(c) >> b) & 1)
    return h


def curve_key(pos, grid) -> int:
    """Hilbert over the non-trivial axes when they form an equal power-of-two
    box, Morton otherwise (domain.py:517-530)."""
    act = [a for a in range(len(grid)) if grid[a] > 1]
    if not act:
        return 0
    coords = [pos[a] for a in act]
    ext = [grid[a] for a in act]
    if len(coords) == 1:
        return coords[0]
    if len(set(ext)) == 1 and ext[0] & (ext[0] - 1) == 0:
        return hilbert_key(coords, ext[0].bit_length() - 1)
    return morton_key(coords, max(max(e - 1 for e in ext).bit_length(), 1))


def greedy_segments(loads, n_workers: int) -> list[int]:
    """Contiguous cuts against the running per-worker target
    (domain.py:446-465)."""
    seats = []
    remaining = float(sum(loads))
    left = n_workers
    target = remaining / left
    w, acc = 0, 0.0
    for load in loads:
        if w < n_workers - 1 and acc > 0 and acc + load / 2.0 > target:
            w += 1
            left -= 1
            target = remaining / left if left else 0.0
            acc = 0.0
        seats.append(w)
        acc += load
        remaining -= load
    return seats


# ---------------------------------------------------------------- domain


class Domain:
    """Whole-geometry solver on one GPU (all blocks in this process)."""

    def __init__(self, global_flags, block_size, stencil, params, pattern: str = "pull",
                 policy: str = "sparse", phi_s: float = DEFAULT_PHI_S, frame_width=None,
                 device: int | None = None, check: str = "step", _rank: int = 0, _world: int = 1,
                 _assignment=None, _comm=None, engine_factory=None, halo_factory=None):
        if policy not in POLICIES:
            raise errors.make("ConfigurationError", f"unknown layout policy {policy!r}")
        self.stencil, self.params, self.pattern = stencil, params, pattern
        self.policy, self.phi_s, self.frame_width = policy, phi_s, frame_width
        self.device = default_device() if device is None else int(device)
        self.check = check
        self.rank, self.world = _rank, _world
        dim = stencil.dim
        if isinstance(block_size, (int, np.integer)):
            block_size = (int(block_size),) * dim
        if len(block_size) != dim or min(block_size) < 1:
            raise errors.make("ConfigurationError", f"bad block size {block_size}")
        self.block_size = tuple(int(s) for s in block_size)
        gf = pad_to_multiple(global_flags, self.block_size)
        self.global_flags = gf
        self.global_dims = gf.dims
        self.periodic = gf.periodic
        self.grid = tuple(self.global_dims[a] // self.block_size[a] for a in range(dim))
        self._block_periodic = tuple(gf.periodic[a] and self.grid[a] == 1 for a in range(dim))

        self.blocks: dict[int, Block] = {}
        for pos in grid_positions(self.grid):
            bid = grid_linear(pos, self.grid)
            origin = tuple(pos[a] * self.block_size[a] for a in range(dim))
            fl = slice_block(gf, origin, self.block_size, self._block_periodic)
            nf = fl.fluid_count()
            if nf == 0:
                continue
            self.blocks[bid] = Block(bid, pos, origin, fl, nf)
        if not self.blocks:
            raise errors.make("ConfigurationError", "geometry has no fluid cells")

        self.assignment = dict(_assignment) if _assignment else {b: 0 for b in self.blocks}
        make_engine = engine_factory or _cuda_engine
        local = []
        for bid, blk in self.blocks.items():
            blk.rank = self.assignment.get(bid, 0)
            # hybrid picks dense at or above phi_s (domain.py:58-65, :109-114)
            blk.kind = classify_kind(blk.porosity, policy, phi_s)
            if blk.rank == self.rank:
                local.append(blk)

        def build(blk):
            return make_engine(blk.flags, stencil, params, pattern,
                               self._block_frame(frame_width), self.device, blk.kind)

        if engine_factory is None and len(local) > 1:
            # each engine builds its lists on its own stream and the C calls
            # release the GIL: several blocks build concurrently
            from concurrent.futures import ThreadPoolExecutor

            with ThreadPoolExecutor(max_workers=min(8, len(local))) as pool:
                for blk, eng in zip(local, pool.map(build, local)):
                    blk.engine = eng
        else:
            for blk in local:
                blk.engine = build(blk)
        engines = self.local_engines()
        self._stream = engines[0].stream() if engines and hasattr(engines[0], "stream") else 0
        for e in engines[1:]:
            if hasattr(e, "set_stream"):
                e.set_stream(self._stream)
        self._halo_factory = halo_factory or DeviceHalo

        self._edges = self._adjacency()
        self.edge_plans: list[EdgePlan] = []
        for a, b, sigma in self._edges:
            ba, bb = self.blocks[a], self.blocks[b]
            if ba.rank != self.rank and bb.rank != self.rank:
                continue
            self.edge_plans.append(EdgePlan(a, b, sigma, stencil, ba.flags, bb.flags, pattern,
                                            ba.engine, bb.engine, src_layout=ba.kind))
        self._comm = _comm
        self._halo = self._build_halo()
        self._face_frames = self._narrow_frames() if engine_factory is None else False
        self.direct_halo = False
        # direct local edges (linked group): steps left in the current call,
        # this one included (1 outside run()); see _stale_before
        self._left = 1
        self._stale_pending = False
        self._group = self._build_group() if engine_factory is None else None
        self.overlap_samples: list[tuple[float, float]] = []
        self.trace = False
        self._nvtx_open = False
        self._pending = []
        self._capturing = False
        self.steps_done = 0

    def _narrow_frames(self) -> bool:
        """``frame_width="halo"`` with remote edges: frame only the faces that
        have a neighbour on another rank (any stencil offset with that sign),
        per face, on sparse blocks.  Local edges then run on the compute
        stream before the interior sweep, so faces towards blocks of this
        rank need no frame.  Returns whether the driver must do so."""
        if not (isinstance(self.frame_width, str) and self.frame_width == "halo"):
            return False
        if not self._has_remote or not hasattr(self._halo, "local_on"):
            return False
        dim = self.stencil.dim
        loopback = getattr(self, "_loopback", False)
        for blk in self.local_blocks():
            if getattr(blk.engine, "layout", "") != "sparse":
                continue
            lo, hi = [0] * dim, [0] * dim
            for sigma, nbid in blk.neighbors.items():
                if not loopback and self.blocks[nbid].rank == self.rank:
                    continue
                for a in range(dim):
                    if sigma[a] < 0:
                        lo[a] = 1
                    elif sigma[a] > 0:
                        hi[a] = 1
            blk.engine.set_frame(lo, hi)
        return True

    def _block_frame(self, frame_width):
        """``frame_width="halo"`` (extension): width 1 only on axes with more
        than one block, 0 on axes every block wraps or spans alone (no halo
        there).  Anything else is passed through with the reference's rules."""
        if not (isinstance(frame_width, str) and frame_width == "halo"):
            return frame_width
        from .engine import HaloWidths

        return HaloWidths(1 if g > 1 else 0 for g in self.grid)

    def _build_group(self):
        """Batched block-table execution when this rank owns
        several sparse blocks: one launch per phase for all of them."""
        engines = self.local_engines()
        if len(engines) < 2 or any(getattr(e, "layout", "") != "sparse" for e in engines):
            return None
        group = BlockGroup(engines)
        # AA: device-local halo edges by direct addressing instead of copies
        # (slbm_group_link_halo; bit-identical).  SLBM_DIRECT_HALO=0 keeps
        # the copy program (A/B measurements).
        if (self.pattern == "aa" and type(self._halo) is DeviceHalo
                and os.environ.get("SLBM_DIRECT_HALO", "1") != "0"):
            self.direct_halo = group.link_halo(self._halo)
        return group

    # -- construction ------------------------------------------------------------

    def _adjacency(self):
        dim = self.stencil.dim
        offsets = sorted({tuple(0 if self._block_periodic[a] else int(self.stencil.c[k][a])
                                for a in range(dim)) for k in range(1, self.stencil.q)}
                         - {(0,) * dim})
        edges = []
        for bid, blk in sorted(self.blocks.items()):
            for sigma in offsets:
                npos = []
                for a in range(dim):
                    p = blk.grid_pos[a] + sigma[a]
                    if self.periodic[a]:
                        p %= self.grid[a]
                    elif not 0 <= p < self.grid[a]:
                        break
                    npos.append(p)
                else:
                    nbid = grid_linear(tuple(npos), self.grid)
                    if nbid in self.blocks:
                        blk.neighbors[sigma] = nbid
                        edges.append((bid, nbid, sigma))
        return edges

    def _build_halo(self):
        """Registers every planned edge, in edge order, with the exchange
        program.  Remote ends append to the peer's single per-phase message
        in this order on both ranks (one message per peer per phase)."""
        halo = self._halo_factory(self.device)
        loopback = getattr(self, "_loopback", False)
        for plan in self.edge_plans:
            src, dst = self.blocks[plan.src_bid], self.blocks[plan.dst_bid]
            for ph, pp in plan.phases.items():
                if loopback:
                    # test mode: every edge travels as a message to this rank
                    halo.add_send(ph, src.engine, self.rank, pp)
                    halo.add_recv(ph, dst.engine, self.rank, pp)
                elif src.rank == self.rank and dst.rank == self.rank:
                    halo.add_local(ph, src.engine, dst.engine, pp)
                elif src.rank == self.rank:
                    halo.add_send(ph, src.engine, dst.rank, pp)
                else:
                    halo.add_recv(ph, dst.engine, src.rank, pp)
        halo.commit(self._comm.handle if self._comm is not None else None)
        self._has_remote = loopback or any(
            (self.blocks[pl.src_bid].rank != self.rank) != (self.blocks[pl.dst_bid].rank != self.rank)
            for pl in self.edge_plans)
        return halo

    # -- access -----------------------------------------------------------------

    def local_blocks(self):
        return [b for _, b in sorted(self.blocks.items()) if b.rank == self.rank]

    def local_engines(self):
        return [b.engine for b in self.local_blocks()]

    def local_fluid(self) -> int:
        return sum(b.n_fluid for b in self.local_blocks())

    def total_fluid(self) -> int:
        return sum(b.n_fluid for b in self.blocks.values())

    @property
    def parity(self):
        return self.local_engines()[0].parity

    def stream(self) -> int:
        return self._stream

    # -- state init ---------------------------------------------------------------

    def init_equilibrium(self, rho: float = 1.0, u=None) -> None:
        for e in self.local_engines():
            e.init_equilibrium(rho, u)

    def init_random(self, seed: int, amplitude: float = 0.005) -> None:
        """domain.py:191-206: near-equilibrium state drawn over the global
        grid (decomposition-invariant); the equilibrium is evaluated on the
        device with the reference's operation order."""
        rng = np.random.default_rng(seed)
        shape = rev_shape(self.global_dims)
        rho_g = 1.0 + amplitude * rng.standard_normal(shape)
        u_g = amplitude * rng.standard_normal((self.stencil.dim,) + shape)
        for blk in self.local_blocks():
            coords = blk.engine.fluid_coords + np.asarray(blk.origin, dtype=np.int64)
            flat = np.ravel_multi_index(coords[:, ::-1].T, shape)
            blk.engine.init_equilibrium(rho_g.reshape(-1)[flat],
                                        u_g.reshape(self.stencil.dim, -1)[:, flat])

    # -- stepping -----------------------------------------------------------------

    def _count_exchange(self, phase: Phase):
        for plan in self.edge_plans:
            src = self.blocks[plan.src_bid]
            if src.rank == self.rank:
                src.engine.counters.values_exchanged += plan.phases[phase].n_wire
                src.engine.counters.messages += 1

    def _sweep(self, phase: str):
        if self._group is not None:
            self._group.step(phase, self._stream)
            return
        for e in self.local_engines():
            e.step(phase)

    def _refresh_all(self):
        if self._group is not None:
            self._group.refresh(self.parity, self._stream)
            return
        for e in self.local_engines():
            e.refresh_boundary(e.parity)

    def _finish_all(self):
        if self._group is not None:
            self._group.finish(self._stream)
            return
        for e in self.local_engines():
            e.finish_step()

    # -- tracing (exchange.py:333-374, domain.py:236-239) ----------------------
    # With ``trace = True`` the drivers record CUDA events on the compute
    # stream: exchange start, interior start / end, and the join after the
    # halo wait (= the later of interior end and exchange completion).  Like
    # the reference's perf_counter spans, a step contributes
    # (interior span, exchange window) to ``overlap_samples``; events are
    # resolved lazily (``overlap_ratio`` synchronises).  Off by default.

    def _mark(self, label: str | None = None):
        """CUDA event on the compute stream (and an NVTX range boundary named
        ``label`` for Nsight timelines) when tracing."""
        if not self.trace or self._capturing:
            return None
        import torch

        if self._nvtx_open:
            torch.cuda.nvtx.range_pop()
            self._nvtx_open = False
        if label:
            torch.cuda.nvtx.range_push(label)
            self._nvtx_open = True
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.ExternalStream(self._stream))
        return ev

    def _sample(self, e0, e1, e2, e3):
        if e0 is not None:
            self._pending.append((e0, e1, e2, e3))

    def overlap_ratio(self) -> float:
        """domain.py:236-239: interior time / exchange window over the
        traced steps (0 when nothing was traced)."""
        for e0, e1, e2, e3 in self._pending:
            e3.synchronize()
            inner = e1.elapsed_time(e2) / 1e3 if e1 is not None else 0.0
            self.overlap_samples.append((inner, e0.elapsed_time(e3) / 1e3))
        self._pending = []
        num = sum(s[0] for s in self.overlap_samples)
        den = sum(s[1] for s in self.overlap_samples)
        return num / den if den > 0 else 0.0

    def _fused_boundary(self) -> bool:
        """Local halo edges + refresh + step counters as one group launch."""
        return self._group is not None and type(self._halo) is DeviceHalo

    def _stale_before(self) -> None:
        """Linked group (direct local edges).  The copy program leaves, after
        an AA even step, the source slots of local edges stale (its REVERSED
        exchange delivers the even step's values before the odd step) and
        those values in the ghosts; the linked group writes the sources
        directly and never touches the ghosts.  So that every call hands back
        the copy program's state slot for slot, the even step that ends a
        call copies the stale sources into the ghosts first and swaps the
        two afterwards (the next odd step then starts with the REVERSED
        local exchange, ghost -> source), and the even step just before a
        call's last (odd) step copies its values into the ghosts.  Steps in
        the middle of a run do none of this."""
        if not self.direct_halo:
            return
        if is_even(self.parity):
            if self._left == 1:
                self._group.stale_copy(0, self._stream)
        elif self._stale_pending:
            self._group.stale_copy(2, self._stream)
            self._stale_pending = False

    def _stale_after(self) -> None:
        if not (self.direct_halo and is_even(self.parity)):
            return
        if self._left == 1:
            self._group.stale_copy(1, self._stream)
            self._stale_pending = True
        elif self._left == 2:
            self._group.stale_copy(0, self._stream)

    def step_sequential(self) -> None:
        """exchange.py:330-346 on the device: exchange, then whole-block sweeps."""
        self._stale_before()
        phase = phase_for(self.pattern, self.parity)
        e0 = self._mark("slbm.exchange")
        if not self._has_remote and self._fused_boundary():
            self._sample(e0, None, None, self._mark("slbm.sweep"))
            self._count_exchange(phase)
            self._group.boundary(self._halo, phase, self.parity, self._stream)
        else:
            self._halo.start(phase, self._stream)
            self._halo.wait(self._stream)
            self._sample(e0, None, None, self._mark("slbm.sweep"))
            self._count_exchange(phase)
            self._refresh_all()
        self._sweep("all")
        self._stale_after()
        self._finish_all()
        self._mark()  # closes the last NVTX range

    def step_overlapped(self) -> None:
        """exchange.py:349-374: pack/send/recv/unpack on the comm stream while
        the interior sweep runs on the compute stream; frame after the join.

        With no remote edge on this rank there is no transfer to hide: the
        device-local exchange program (one gather-scatter kernel) runs first
        and every block is swept whole, which is bitwise the same (F11) and
        avoids the split sweeps' cost (C4 artery: 0.51 -> 0.40 ms/step).
        Counters still record the interior/frame split the reference's
        overlapped driver reports."""
        self._stale_before()
        phase = phase_for(self.pattern, self.parity)
        e0 = self._mark("slbm.exchange_start")
        fused = self._fused_boundary() and (self._face_frames or not self._has_remote)
        if self._face_frames:
            # remote edges on the comm stream; local edges first on this one
            self._halo.start(phase, self._stream, with_local=False)
            if not fused:
                self._halo.local_on(phase, self._stream)
        elif not fused:
            self._halo.start(phase, self._stream)
        self._count_exchange(phase)
        if fused:  # local edges + refresh + step counters: one launch
            self._group.boundary(self._halo, phase, self.parity, self._stream)
        else:
            self._refresh_all()
        if not self._has_remote:
            if not fused:
                self._halo.wait(self._stream)
            self._sample(e0, None, None, self._mark("slbm.sweep"))
            self._sweep("all")
            for e in self.local_engines():
                e.counters.cells_visited_interior += e.n_interior
                e.counters.cells_visited_frame += e.n_frame
        else:
            e1 = self._mark("slbm.interior")
            self._sweep("interior")
            e2 = self._mark("slbm.halo_wait")
            self._halo.wait(self._stream)
            self._sample(e0, e1, e2, self._mark("slbm.frame"))
            self._sweep("frame")
        self._stale_after()
        self._finish_all()
        self._mark()  # closes the last NVTX range

    def run(self, steps: int, driver: str = "sequential", use_graph: bool = False) -> None:
        """``steps`` time steps.  ``use_graph`` (check="deferred" only) captures
        one step pair of the whole domain — halo program on the comm stream,
        every block's refresh and sweeps, NCCL included — into a CUDA graph
        and replays it, so many-block domains are not host-launch bound."""
        fn = self._driver(driver)
        steps = int(steps)
        try:
            if use_graph and self.check == "deferred" and self._graph_capable():
                # graphs hold (even, odd) pairs: an odd start runs one step
                # first; a linked group's last pair of a call is its own
                # graph (the call-boundary copy after the even step)
                if not is_even(self.parity) and steps >= 3:
                    self._left = steps
                    fn()
                    if self.check == "step":
                        self._poll_or_raise()
                    self.steps_done += 1
                    steps -= 1
                while steps >= 2 and is_even(self.parity):
                    self._left = steps
                    self._replay_pair(driver, fn)
                    steps -= 2
            for k in range(steps):
                self._left = steps - k
                fn()
                if self.check == "step":
                    self._poll_or_raise()
                self.steps_done += 1
        finally:
            self._left = 1

    def _graph_capable(self) -> bool:
        return bool(self._stream) and isinstance(self._halo, DeviceHalo)

    def _replay_pair(self, driver, fn):
        from . import _abi
        import ctypes as C

        # the captured pair bakes in buffer pointers: AA keys on parity, pull
        # on which of each engine's two buffers is current (finish_step swaps)
        key = (driver, getattr(self.parity, "value", self.parity),
               tuple(e.buffer_state() for e in self.local_engines()),
               self.direct_halo and self._left == 2)
        graphs = self.__dict__.setdefault("_graphs", {})
        if key not in graphs:
            engines = self.local_engines()
            snap = [(e.counters.copy(), e.parity) for e in engines]
            _abi.call("slbm_capture_begin", C.c_void_p(self._stream))
            self._capturing = True
            try:
                fn()
                fn()
            finally:
                self._capturing = False
                exec_ = C.c_void_p()
                _abi.call("slbm_capture_end", C.c_void_p(self._stream), C.byref(exec_))
            deltas = []
            for e, (c0, p0) in zip(engines, snap):
                d = {k: v - getattr(c0, k) for k, v in e.counters.as_dict().items()}
                deltas.append(d)
                e.counters = c0
                e.parity = p0
            graphs[key] = (exec_, deltas)
        exec_, deltas = graphs[key]
        from . import _abi as abi

        abi.call("slbm_graph_launch", exec_, C.c_void_p(self._stream))
        for e, d in zip(self.local_engines(), deltas):
            for k, v in d.items():
                setattr(e.counters, k, getattr(e.counters, k) + v)
        self.steps_done += 2

    def _driver(self, name: str):
        if name == "sequential":
            return self.step_sequential
        if name == "overlapped":
            if self.frame_width is None:
                raise errors.make("ConfigurationError", "overlapped driver needs frame_width at construction")
            return self.step_overlapped
        raise errors.make("ConfigurationError", f"unknown driver {name!r}")

    def _poll_or_raise(self):
        engines = self.local_engines()
        try:
            if engines and all(hasattr(e, "handle") for e in engines):
                _poll_engines(engines)  # one host round trip for all blocks
            else:
                for e in engines:
                    e.poll()
        except errors.error_class("NumericalInstabilityError") as exc:
            raise errors.make("NumericalInstabilityError", f"unstable at step {self.steps_done}: {exc}") from exc

    def poll(self) -> None:
        self._poll_or_raise()

    def synchronize(self) -> None:
        for e in self.local_engines():
            e.synchronize()

    # -- observation ----------------------------------------------------------------

    def fluid_mask(self) -> np.ndarray:
        return self.global_flags.tags_interior == FLUID

    def gather_macroscopics(self):
        """domain.py:246-268: global (rho, u) with zeros at solids.

        Sparse domains assemble the global box on the device -- every block
        writes its fluid cells' fields into one zeroed device box
        (slbm_macroscopic_global) -- and move it with one staged copy per
        field (slbm_copy_to_host).  A host-side scatter of the per-block
        values into a fresh multi-GB box is latency bound (C4 artery: ~1.7 s
        for 6.3 M cells into a 4.3 GB box, the device path ~0.2 s).  Other
        domains (dense blocks, or a box that does not fit the free device
        memory) gather per block on the host."""
        fast = self._gather_macroscopics_device()
        if fast is not None:
            return fast
        shape = rev_shape(self.global_dims)
        dim = self.stencil.dim
        rho = np.zeros(shape)
        u = np.zeros(shape + (dim,))
        for blk in self.local_blocks():
            e = blk.engine
            if getattr(e, "layout", "") == "sparse" and blk.porosity < 0.5 and hasattr(
                    e, "macroscopic_compact"):
                r, v = e.macroscopic_compact()
                g = tuple(e.fluid_coords[:, a] + blk.origin[a] for a in reversed(range(dim)))
                rho[g] = r
                u[g] = v
                continue
            r, v = e.macroscopic_fields()
            sel = tuple(slice(blk.origin[a], blk.origin[a] + self.block_size[a])
                        for a in reversed(range(dim)))
            rho[sel] = r
            u[sel] = v
        return rho, u

    def _gather_macroscopics_device(self):
        engines = [b.engine for b in self.local_blocks()]
        if not engines or any(getattr(e, "layout", "") != "sparse" or not hasattr(e, "handle")
                              for e in engines):
            return None
        import ctypes as C

        import torch

        from . import _abi

        shape = rev_shape(self.global_dims)
        dim = self.stencil.dim
        n = int(np.prod(shape))
        need = 8 * n * (1 + dim)
        dev = torch.device("cuda", int(engines[0].device))
        free, _ = torch.cuda.mem_get_info(dev)
        if need > free // 2:
            return None
        d_rho = torch.zeros(n, dtype=torch.float64, device=dev)
        d_u = torch.zeros(n * dim, dtype=torch.float64, device=dev)
        torch.cuda.synchronize(dev)
        gd = np.array(list(self.global_dims) + [1] * (3 - len(self.global_dims)), dtype=np.int64)
        for blk in self.local_blocks():
            org = np.array(list(blk.origin) + [0] * (3 - len(blk.origin)), dtype=np.int64)
            if blk.engine.check == "deferred":
                blk.engine.poll()  # raise a pending instability, as macroscopic_fields does
            _abi.call("slbm_macroscopic_global", blk.engine.handle, C.c_void_p(d_rho.data_ptr()),
                      C.c_void_p(d_u.data_ptr()), _abi.ptr(gd, C.c_int64), _abi.ptr(org, C.c_int64))
        rho = np.empty(shape)
        u = np.empty(shape + (dim,))
        _abi.call("slbm_copy_to_host", _abi.ptr(rho, C.c_double), C.c_void_p(d_rho.data_ptr()),
                  rho.nbytes, int(engines[0].device))
        _abi.call("slbm_copy_to_host", _abi.ptr(u, C.c_double), C.c_void_p(d_u.data_ptr()),
                  u.nbytes, int(engines[0].device))
        return rho, u

    def gather_canonical(self) -> np.ndarray:
        shape = rev_shape(self.global_dims)
        out = np.zeros((self.stencil.q,) + shape)
        flat_out = out.reshape(self.stencil.q, -1)
        for blk in self.local_blocks():
            coords = blk.engine.fluid_coords + np.asarray(blk.origin, dtype=np.int64)
            flat = np.ravel_multi_index(coords[:, ::-1].T, shape)
            flat_out[:, flat] = blk.engine.canonical_state()
        return out

    def total_moments(self) -> np.ndarray:
        """(mass, momentum x, y, z) over this rank's fluid cells (monitor):
        per block one device pass with warp-shuffle reductions, summed in
        block order."""
        tot = np.zeros(4)
        for e in self.local_engines():
            tot += e.total_moments()
        return tot

    def counters(self) -> Counters:
        total = Counters()
        for e in self.local_engines():
            total.add(e.counters)
        return total

    # -- balancing --------------------------------------------------------------------

    def workload(self, bid: int) -> int:
        """model.workload_sparse / workload_dense: Q x fluid cells, or Q x box
        cells for a dense block (domain.py:281-285)"""
        blk = self.blocks[bid]
        q = self.stencil.q
        if blk.kind == "dense":
            return 2 * q * 8 * blk.flags.cell_count()  # model.py workload_dense
        return (2 * q * 8 + (q - 1) * 4) * blk.n_fluid  # model.py workload_sparse

    def curve_order(self) -> list[int]:
        return sorted(self.blocks, key=lambda b: (curve_key(self.blocks[b].grid_pos, self.grid), b))

    def balance(self, n_workers: int) -> dict[int, int]:
        if n_workers < 1:
            raise errors.make("ConfigurationError", "need at least one worker")
        order = self.curve_order()
        seats = greedy_segments([self.workload(b) for b in order], n_workers)
        return {b: int(w) for b, w in zip(order, seats)}


class BlockGroup:
    """All sparse CUDA engines of one rank driven as one block table
    (slbm_group_*): refresh, each sweep phase and finish are single
    launches; the Python-side engine state (parity, counters) is advanced
    exactly as the per-engine calls would."""

    def __init__(self, engines):
        import ctypes as C

        from . import _abi

        self.engines = list(engines)
        arr = (C.c_void_p * len(self.engines))(*[e.handle.value for e in self.engines])
        h = C.c_void_p()
        _abi.call("slbm_group_create", arr, len(self.engines), C.byref(h))
        self._h = h

    def link_halo(self, halo) -> bool:
        """Serve ``halo``'s device-local edges by direct addressing
        (slbm_group_link_halo); False when not applicable (nothing changed)."""
        from . import _abi

        return _abi.load().slbm_group_link_halo(self._h, halo.handle) == 0

    def stale_copy(self, mode: int, stream):
        """slbm_group_stale_copy: local edges' source/ghost slots, mode 0
        ghost <- source, 1 swap, 2 source <- ghost."""
        import ctypes as C

        from . import _abi

        _abi.call("slbm_group_stale_copy", self._h, int(mode), C.c_void_p(stream or 0))

    def close(self):
        from . import _abi

        if getattr(self, "_h", None) is not None and self._h.value:
            _abi.load().slbm_group_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def refresh(self, parity, stream):
        import ctypes as C

        from . import _abi

        _abi.call("slbm_group_refresh", self._h, int(getattr(parity, "value", parity)),
                  C.c_void_p(stream or 0))

    def boundary(self, halo, phase, parity, stream):
        """refresh + the halo's device-local edges of ``phase``, one launch."""
        import ctypes as C

        from . import _abi

        _abi.call("slbm_group_boundary", self._h, halo.handle, int(phase.value),
                  int(getattr(parity, "value", parity)), C.c_void_p(stream or 0))

    def step(self, phase: str, stream):
        import ctypes as C

        from . import _abi
        from .engine import _PHASE_CODE

        cells = [e._phase_cells(phase) for e in self.engines]  # validates the phase
        _abi.call("slbm_group_step", self._h, _PHASE_CODE[phase], C.c_void_p(stream or 0))
        for e, n in zip(self.engines, cells):
            table = e.pattern == "pull" or is_even(e.parity)
            e.counters.record_sweep(phase, n, e.stencil.q, table)

    def finish(self, stream):
        import ctypes as C

        from . import _abi

        _abi.call("slbm_group_finish", self._h, C.c_void_p(stream or 0))
        for e in self.engines:
            if e.pattern == "aa":
                e.parity = e.parity.flipped()
            e.counters.steps += 1


def _poll_engines(engines):
    """slbm_poll_engines: every block's instability flag, one sync per stream."""
    import ctypes as C

    from . import _abi

    arr = (C.c_void_p * len(engines))(*[e.handle.value for e in engines])
    bad, which = C.c_int64(-1), C.c_int(-1)
    lib = _abi.load()
    status = lib.slbm_poll_engines(arr, len(engines), C.byref(bad), C.byref(which))
    if status != 0:
        msg = lib.slbm_last_error().decode(errors="replace")
        if bad.value >= 0:
            msg = f"{msg} (engine step {bad.value})"
        errors.raise_for_status(status, msg)


def _cuda_engine(flags, stencil, params, pattern, frame_width, device, kind="sparse"):
    cls = DenseEngine if kind == "dense" else SparseEngine
    return cls(flags, stencil, params, pattern=pattern, frame_width=frame_width, device=device,
               check="deferred")


def classify_kind(porosity: float, policy: str, phi_s: float = DEFAULT_PHI_S) -> str:
    """domain.py:58-65: hybrid is dense at or above phi_s (ties dense)."""
    if policy == "hybrid":
        return "dense" if porosity >= phi_s else "sparse"
    if policy in ("sparse", "dense"):
        return policy
    raise errors.make("ConfigurationError", f"unknown layout policy {policy!r}")


class HostStagedHalo:
    """DeviceHalo whose cross-rank messages travel through host memory and a
    torch.distributed (gloo) group instead of NCCL: for tests with several
    ranks on one GPU (NCCL refuses duplicate devices) and for hosts without
    peer access.  Same message layout and order as the NCCL path."""

    def __init__(self, device, group=None, world=1):
        self.inner = DeviceHalo(device)
        self.group = group
        self.world = world

    def add_local(self, *a):
        self.inner.add_local(*a)

    def add_send(self, *a):
        self.inner.add_send(*a)

    def add_recv(self, *a):
        self.inner.add_recv(*a)

    def commit(self, nccl_comm=None):
        self.inner.commit(None)

    def local_on(self, phase, stream):
        self.inner.local_on(phase, stream)

    def start(self, phase, after_stream, with_local=True):
        import torch
        import torch.distributed as dist

        _abi_sync_stream(after_stream)
        if with_local:
            self.inner.local_only(phase)
        sends, recvs = self.inner.peer_sizes(phase, self.world)
        reqs, bufs = [], {}
        for peer in range(self.world):
            if sends[peer]:
                out = np.empty(int(sends[peer]), dtype=np.float64)
                self.inner.pack_host(phase, peer, out)
                reqs.append(dist.isend(torch.from_numpy(out), dst=peer, group=self.group))
                bufs[("s", peer)] = out
            if recvs[peer]:
                buf = torch.empty(int(recvs[peer]), dtype=torch.float64)
                reqs.append(dist.irecv(buf, src=peer, group=self.group))
                bufs[("r", peer)] = buf
        for r in reqs:
            r.wait()
        for peer in range(self.world):
            if recvs[peer]:
                self.inner.unpack_host(phase, peer, bufs[("r", peer)].numpy())

    def wait(self, stream):
        self.inner.wait(stream)

    def close(self):
        self.inner.close()


def _abi_sync_stream(stream):
    """Wait until the compute stream has finished the previous sweep."""
    if stream:
        import ctypes as C

        _cudart().cudaStreamSynchronize(C.c_void_p(stream))


_CUDART = None


def _cudart():
    global _CUDART
    if _CUDART is None:
        import ctypes as C
        import ctypes.util

        for name in ("libcudart.so.12", "libcudart.so", ctypes.util.find_library("cudart")):
            if not name:
                continue
            try:
                _CUDART = C.CDLL(name)
                break
            except OSError:
                continue
    return _CUDART


class DistributedDomain(Domain):
    """One process per GPU.  Blocks go to ranks by ``assignment`` (default:
    the reference's Hilbert/greedy ``balance``); cross-rank edges use NCCL
    through the library's own communicator (``transport="nccl"``), peer
    memory — the pack kernel storing into the peers' buffers through CUDA IPC
    over NVLink, epoch flags instead of NCCL (``transport="p2p"``) — or host
    staging over a gloo group (``transport="host"``)."""

    def __init__(self, global_flags, block_size, stencil, params, pattern="aa", frame_width="halo",
                 rank: int | None = None, world: int | None = None, device: int | None = None,
                 assignment=None, check: str = "deferred", comm=None, transport: str = "nccl",
                 engine_factory=None, halo_factory=None, loopback: bool = False):
        import torch.distributed as dist

        rank = dist.get_rank() if rank is None else rank
        world = dist.get_world_size() if world is None else world
        # loopback (tests): all edges become NCCL messages from this rank to itself
        self._loopback = bool(loopback)
        if loopback and comm is None and transport == "nccl":
            comm = NcclComm(rank, 1, default_device() if device is None else device)
        if assignment is None:
            assignment = _balance_without_engines(global_flags, block_size, stencil, world)
        if transport not in ("nccl", "host", "p2p"):
            raise errors.make("ConfigurationError", f"unknown transport {transport!r}")
        if halo_factory is None and transport == "host":
            group = dist.new_group(backend="gloo") if dist.get_backend() != "gloo" else None
            halo_factory = lambda dev: HostStagedHalo(dev, group, world)  # noqa: E731
        if halo_factory is None and transport == "p2p":
            # peer memory over NVLink: loopback keeps every edge a message to itself
            peer = (0, 1, None) if loopback else (rank, world, None)
            halo_factory = lambda dev: DeviceHalo(dev, peer=peer)  # noqa: E731
        if comm is None and world > 1 and transport == "nccl" and halo_factory is None:
            comm = NcclComm(rank, world, default_device() if device is None else device)
        super().__init__(global_flags, block_size, stencil, params, pattern=pattern,
                         frame_width=frame_width, device=device, check=check, _rank=rank,
                         _world=world, _assignment=assignment, _comm=comm,
                         engine_factory=engine_factory, halo_factory=halo_factory)
        # NCCL sets up its peer connections on the first send/recv to a peer;
        # the first step pair of a graph run goes eagerly so that happens
        # outside stream capture
        self._eager_first = (world > 1 and transport == "nccl" and halo_factory is None
                             and not loopback)

    def gather_canonical_global(self) -> np.ndarray:
        """gather_canonical summed over ranks (rank 0 gets the full field)."""
        import torch
        import torch.distributed as dist

        local = torch.from_numpy(self.gather_canonical())
        if dist.get_backend() == "nccl":
            t = local.cuda()
            dist.all_reduce(t)
            return t.cpu().numpy()
        dist.all_reduce(local)
        return local.numpy()

    @classmethod
    def weak_scaling_bed(cls, block_edge, world, rank, stencil, params, porosity, diameter, seed,
                         device=None, transport="nccl"):
        """world slabs of ``block_edge`` stacked along z, fully periodic
        overlapping-sphere bed over the whole box, slab i on rank i.

        Slabs along z: each block exchanges with its two z neighbours only
        (one message per peer per phase over NVSwitch), x and y wrap inside
        the block, and with ``frame_width="halo"`` the frame is two whole z
        planes — a contiguous cid prefix and suffix — so the interior sweep
        is one cid range and the frame sweep stays coalesced."""
        from .geometry import packed_bed_flags

        bx, by, bz = block_edge
        dims = (bx, by, bz * world)
        fl = packed_bed_flags(dims, porosity, diameter, seed, periodic=True,
                              device=default_device() if device is None else device)
        assignment = {i: i for i in range(world)}
        return cls(fl, (bx, by, bz), stencil, params, pattern="aa", frame_width="halo",
                   rank=rank, world=world, device=device, assignment=assignment,
                   transport=transport)

    def run(self, steps: int, driver: str = "overlapped", use_graph: bool = False) -> None:
        steps = int(steps)
        if use_graph and steps > 0 and getattr(self, "_eager_first", False):
            first = min(steps, 2)
            super().run(first, driver, False)
            self._eager_first = False
            steps -= first
        super().run(steps, driver, use_graph)


def _balance_without_engines(gf, block_size, stencil, n_workers):
    dim = stencil.dim
    if isinstance(block_size, (int, np.integer)):
        block_size = (int(block_size),) * dim
    gf = pad_to_multiple(gf, tuple(block_size))
    grid = tuple(gf.dims[a] // block_size[a] for a in range(dim))
    loads = {}
    for pos in grid_positions(grid):
        sel = tuple(slice(1 + pos[a] * block_size[a], 1 + (pos[a] + 1) * block_size[a])
                    for a in reversed(range(dim)))
        nf = int(np.count_nonzero(gf.tags[sel] == FLUID))
        if nf:
            loads[grid_linear(pos, grid)] = (pos, nf)
    order = sorted(loads, key=lambda b: (curve_key(loads[b][0], grid), b))
    seats = greedy_segments([stencil.q * loads[b][1] for b in order], n_workers)
    return {b: int(w) for b, w in zip(order, seats)}
