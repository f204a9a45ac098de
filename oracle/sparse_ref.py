"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Numpy restatement of the reference's indirect-addressing engine:

* ``moments`` / ``equilibrium`` / ``collide``  <- core.py:96-170
  (row-by-row accumulation in stencil order, no BLAS, no pairwise sums —
  the fixed op order the CUDA kernels reproduce bit for bit);
* ``build_lists``                               <- sparse.py:97-195
* ``OracleSparseEngine`` steps / refresh / state <- sparse.py:199-383

Inputs are duck-typed (``dims``, ``tags``, ``ubb_u``, ``periodic`` on the
flag box; ``q``, ``dim``, ``c``, ``w``, ``inv`` on the stencil; ``omega``,
``model``, ``lambda_odd`` on the params) so the oracle accepts both this
repo's host types and the reference's.
"""

from __future__ import annotations

import numpy as np

CS2 = 1.0 / 3.0
FLUID, NOSLIP, UBB, EXCHANGE, OUTLET = 0, 1, 2, 3, 4


class OracleError(Exception):
    pass


class OracleInstability(OracleError):
    pass


# ---------------------------------------------------------------- collision


def moments(t, st, check=True):
    """core.py:96-124"""
    rho = t[0] + t[1]
    for k in range(2, st.q):
        rho += t[k]
    if check and ((rho <= 0.0).any() or not np.isfinite(rho).all()):
        raise OracleInstability("non-positive or non-finite density in collision input")
    u = np.zeros((st.dim, t.shape[1]))
    for a in range(st.dim):
        col = st.c[:, a]
        for k in range(st.q):
            if col[k] == 1:
                u[a] += t[k]
            elif col[k] == -1:
                u[a] -= t[k]
    u /= rho
    return rho, u


def _signed_sum(vectors, coeffs, like):
    acc = np.zeros_like(like)
    for v, s in zip(vectors, coeffs):
        if s == 1:
            acc += v
        elif s == -1:
            acc -= v
    return acc


def equilibrium(rho, u, st):
    """core.py:127-146"""
    rho = np.asarray(rho, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    usq = u[0] * u[0]
    for a in range(1, st.dim):
        usq = usq + u[a] * u[a]
    feq = np.empty((st.q, rho.shape[0]))
    for k in range(st.q):
        cu = _signed_sum(u, st.c[k], rho)
        feq[k] = st.w[k] * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq)
    return feq


def collide(t, params, st):
    """core.py:149-170 (SRT / TRT); "cumulant" -> oracle/cumulant_ref.py
    (not in the reference, unpinned)"""
    if params.model == "cumulant":
        moments(t, st)  # same instability check as every collision
        higher = getattr(params, "higher_omegas", None)
        bulk = float(getattr(params, "bulk_omega", 1.0))
        if higher is not None and any(float(w) != 1.0 for w in higher):
            # general rates: the independent restatement (tolerance, not bits)
            from .cumulant_geier import collide_general

            return collide_general(t, params.omega, bulk, higher, st)
        from .cumulant_ref import cumulant_collide

        return cumulant_collide(t, params.omega, st, bulk)
    rho, u = moments(t, st)
    feq = equilibrium(rho, u, st)
    if params.model == "srt":
        return t - params.omega * (t - feq)
    if params.model != "trt":
        raise OracleError(f"oracle has no {params.model!r} collision (reference: srt/trt only)")
    we, wo = params.omega, params.lambda_odd
    out = np.empty_like(t)
    for k in range(st.q):
        kb = st.inv[k]
        sym = 0.5 * (t[k] + t[kb])
        asym = 0.5 * (t[k] - t[kb])
        sym_eq = 0.5 * (feq[k] + feq[kb])
        asym_eq = 0.5 * (feq[k] - feq[kb])
        out[k] = t[k] - we * (sym - sym_eq) - wo * (asym - asym_eq)
    return out


def ubb_correction(st, k, u_wall):
    """core.py:173-188"""
    u_wall = np.asarray(u_wall, dtype=np.float64)
    cu = np.zeros(u_wall.shape[:-1])
    for a in range(st.dim):
        if st.c[k, a] == 1:
            cu += u_wall[..., a]
        elif st.c[k, a] == -1:
            cu -= u_wall[..., a]
    return 2.0 * st.w[k] * 1.0 * cu / CS2


# ---------------------------------------------------------------- list build


def _rev(dims):
    return tuple(int(d) for d in dims)[::-1]


def _ring(pos_pub, dims):
    return tuple(-1 if p < 0 else (1 if p >= d else 0) for p, d in zip(pos_pub, dims))


def build_lists(flags, st):
    """sparse.py:72-76 (cells) and :97-195 (lists).  Returns a dict with
    the reference's arrays: pos (rev coords), fluid_coords, idx (uint32),
    base, total_slots, n_ubb, n_ghost, ubb_slots/partner/corr, ghost
    {(q, p_flat): slot}, cid_map, padded_shape."""
    dims = tuple(int(d) for d in flags.dims)
    dim, q = st.dim, st.q
    inner = flags.tags[tuple(slice(1, n + 1) for n in _rev(dims))]
    pos = np.argwhere(inner == FLUID)
    n = pos.shape[0]
    if n == 0:
        raise OracleError(f"block {dims} has no fluid cells")
    padded = tuple(m + 2 for m in _rev(dims))
    tags_flat = flags.tags.reshape(-1)
    ubb_flat = flags.ubb_u.reshape(-1, dim)
    c_rev = st.c[:, ::-1]
    here_flat = np.ravel_multi_index((pos + 1).T, padded)
    cid_map = np.full(int(np.prod(padded)), -1, dtype=np.int64)
    cid_map[here_flat] = np.arange(n)

    upwind = np.zeros((q, n), dtype=np.int64)
    up_tag = np.zeros((q, n), dtype=np.uint8)
    for k in range(1, q):
        src = pos - c_rev[k]
        for axis in range(dim):
            if flags.periodic[axis]:
                col = dim - 1 - axis
                src[:, col] = np.mod(src[:, col], dims[axis])
        upwind[k] = np.ravel_multi_index((src + 1).T, padded)
        up_tag[k] = tags_flat[upwind[k]]

    n_ubb = np.array([0] + [int((up_tag[k] == UBB).sum()) for k in range(1, q)], dtype=np.int64)
    n_ghost = np.array([0] + [int((up_tag[k] == EXCHANGE).sum()) for k in range(1, q)],
                       dtype=np.int64)
    # OUTLET (extension, unpinned): slots appended after the ghost slots, so
    # layouts without outlets are exactly the reference's
    n_out = np.array([0] + [int((up_tag[k] == OUTLET).sum()) for k in range(1, q)], dtype=np.int64)
    sizes = n + n_ubb + n_ghost + n_out
    base = np.zeros(q + 1, dtype=np.int64)
    base[1:] = np.cumsum(sizes)
    total = int(base[-1])
    if total >= 2**32:
        raise OracleError("slot count exceeds the 4-byte table")

    idx = np.full((q - 1, n), -1, dtype=np.int64)
    ghost = {}
    ubb_s, ubb_p, ubb_c = [], [], []
    out_s, out_p, out_c, out_q, out_r = [], [], [], [], []
    for k in range(1, q):
        tag = up_tag[k]
        row = idx[k - 1]
        sel = np.nonzero(tag == FLUID)[0]
        src_cid = cid_map[upwind[k][sel]]
        if np.any(src_cid < 0):
            raise OracleError("fluid upwind cell missing from cell list")
        row[sel] = base[k] + src_cid
        sel = np.nonzero(tag == NOSLIP)[0]
        row[sel] = base[st.inv[k]] + sel
        sel = np.nonzero(tag == UBB)[0]
        slots = base[k] + n + np.arange(sel.size)
        row[sel] = slots
        ubb_s.append(slots)
        ubb_p.append(base[st.inv[k]] + sel)
        ubb_c.append(ubb_correction(st, k, ubb_flat[upwind[k][sel]]))
        sel = np.nonzero(tag == EXCHANGE)[0]
        if sel.size:
            pf = upwind[k][sel]
            pc = np.stack(np.unravel_index(pf, padded), axis=1)[:, ::-1] - 1
            keys = [(_ring(tuple(p), dims), int(f)) for p, f in zip(pc, pf)]
            order = sorted(range(sel.size), key=lambda i: keys[i])
            first = base[k] + n + n_ubb[k]
            for r, i in enumerate(order):
                row[sel[i]] = first + r
                ghost[(k, int(pf[i]))] = int(first + r)
        sel = np.nonzero(tag == OUTLET)[0]
        slots = base[k] + n + n_ubb[k] + n_ghost[k] + np.arange(sel.size)
        row[sel] = slots
        out_s.append(slots)
        out_p.append(base[st.inv[k]] + sel)
        out_c.append(sel)
        out_q.append(np.full(sel.size, k))
        out_r.append(ubb_flat[upwind[k][sel]][:, 0] if sel.size else np.empty(0))
    if np.any(idx < 0):
        raise OracleError("unknown tag upwind of a fluid cell")
    owned = np.concatenate((np.arange(n), idx.ravel()))
    if np.unique(owned).size != owned.size:
        raise OracleError("each slot must belong to exactly one (direction, cell) pair")
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.empty(0, dt))
    return {
        "pos": pos,
        "fluid_coords": np.ascontiguousarray(pos[:, ::-1]),
        "idx": idx.astype(np.uint32),
        "base": base,
        "total_slots": total,
        "n_ubb": int(n_ubb.sum()),
        "n_ghost": int(n_ghost.sum()),
        "ubb_slots": cat(ubb_s, np.int64),
        "ubb_partner": cat(ubb_p, np.int64),
        "ubb_corr": cat(ubb_c, np.float64),
        "n_out": int(n_out.sum()),
        "out_slots": cat(out_s, np.int64),
        "out_partner": cat(out_p, np.int64),
        "out_cell": cat(out_c, np.int64),
        "out_q": cat(out_q, np.int64),
        "out_rho": cat(out_r, np.float64),
        "ghost": ghost,
        "cid_map": cid_map,
        "padded_shape": padded,
    }


def frame_cells(dims, width, pos):
    """flags.py:83-108 evaluated at the fluid cells ``pos`` (rev coords)."""
    dim = len(dims)
    widths = (width,) * dim if isinstance(width, (int, np.integer)) else tuple(width)
    inside = np.zeros(pos.shape[0], dtype=bool)
    for axis in range(dim):
        w = min(int(widths[axis]), int(dims[axis]))
        col = pos[:, dim - 1 - axis]
        inside |= (col < w) | (col >= dims[axis] - w)
    return inside


# ---------------------------------------------------------------- engine


class _Counters:
    def __init__(self):
        self.steps = 0
        self.cells_visited = 0
        self.cells_visited_interior = 0
        self.cells_visited_frame = 0
        self.pdf_accesses = 0
        self.idx_reads = 0
        self.values_exchanged = 0
        self.messages = 0

    def as_dict(self):
        return dict(vars(self))


class OracleSparseEngine:
    """Protocol twin of the reference SparseEngine (sparse.py:48-383)."""

    layout = "sparse"

    def __init__(self, flags, stencil, params, pattern="pull", frame_width=None):
        if pattern not in ("pull", "aa"):
            raise OracleError(f"unknown streaming pattern {pattern!r}")
        self.flags, self.stencil, self.params, self.pattern = flags, stencil, params, pattern
        self.dims = tuple(int(d) for d in flags.dims)
        lists = build_lists(flags, stencil)
        self._lists = lists
        self.n_fluid = lists["pos"].shape[0]
        self.fluid_coords = lists["fluid_coords"]
        self.idx = lists["idx"]
        self.base = lists["base"]
        self.total_slots = lists["total_slots"]
        self.n_ubb_slots = lists["n_ubb"]
        self.n_ghost_slots = lists["n_ghost"]
        everything = np.arange(self.n_fluid)
        self._sel = {"all": everything}
        if frame_width is not None:
            fr = frame_cells(self.dims, frame_width, lists["pos"])
            self._sel["frame"] = everything[fr]
            self._sel["interior"] = everything[~fr]
        self._pdf = np.full(self.total_slots, np.nan)
        self._tmp = np.full(self.total_slots, np.nan) if pattern == "pull" else None
        self.parity = 0  # 0 EVEN, 1 ODD
        self.counters = _Counters()

    # state
    def init_canonical(self, values):
        values = np.asarray(values, dtype=np.float64)
        self._pdf.fill(np.nan)
        if self._tmp is not None:
            self._tmp.fill(np.nan)
        n = self.n_fluid
        for r in range(self.stencil.q):
            self._pdf[self.base[r]:self.base[r] + n] = values[r]
        self.parity = 0

    def init_equilibrium(self, rho=1.0, u=None):
        n, dim = self.n_fluid, self.stencil.dim
        rho_a = np.broadcast_to(np.asarray(rho, dtype=np.float64), (n,))
        if u is None:
            u_a = np.zeros((dim, n))
        else:
            u = np.asarray(u, dtype=np.float64)
            u_a = np.broadcast_to(u[:, None], (dim, n)) if u.ndim == 1 else u
        self.init_canonical(equilibrium(rho_a, u_a, self.stencil))

    # steps
    def step(self, phase="all"):
        cells = self._sel[phase]
        st = self.stencil
        table = True
        if cells.size:
            if self.pattern == "pull":
                t = self._gather(cells)
                out = collide(t, self.params, st)
                for r in range(st.q):
                    self._tmp[self.base[r] + cells] = out[r]
            elif self.parity == 0:
                t = self._gather(cells)
                out = collide(t, self.params, st)
                self._pdf[cells] = out[0]
                for r in range(1, st.q):
                    self._pdf[self.idx[r - 1, cells]] = out[st.inv[r]]
            else:
                table = False
                t = np.empty((st.q, cells.size))
                for r in range(st.q):
                    t[r] = self._pdf[self.base[st.inv[r]] + cells]
                out = collide(t, self.params, st)
                for r in range(st.q):
                    self._pdf[self.base[r] + cells] = out[r]
        elif self.pattern == "aa" and self.parity == 1:
            table = False
        c = self.counters
        m = int(cells.size)
        c.cells_visited += m
        if phase == "interior":
            c.cells_visited_interior += m
        elif phase == "frame":
            c.cells_visited_frame += m
        c.pdf_accesses += 2 * st.q * m
        if table:
            c.idx_reads += (st.q - 1) * m

    def _gather(self, cells):
        t = np.empty((self.stencil.q, cells.size))
        t[0] = self._pdf[cells]
        t[1:] = self._pdf[self.idx[:, cells]]
        return t

    def finish_step(self):
        if self.pattern == "pull":
            self._pdf, self._tmp = self._tmp, self._pdf
        else:
            self.parity = 1 - self.parity
        self.counters.steps += 1

    def refresh_boundary(self, parity):
        parity = getattr(parity, "value", parity)
        L = self._lists
        if L["ubb_slots"].size:
            if parity == 0:
                self._pdf[L["ubb_slots"]] = self._pdf[L["ubb_partner"]] + L["ubb_corr"]
            else:
                self._pdf[L["ubb_partner"]] = self._pdf[L["ubb_slots"]] + L["ubb_corr"]
        if L["n_out"]:
            self._refresh_outlet(parity)

    def _refresh_outlet(self, parity):
        """Fixed-density outlet (extension; csrc/kernels.cu k_outlet):
        anti-bounce-back f_q = 2 w_q rho_o (1 + 4.5 (c_q.u)^2 - 1.5 u^2) - f*_inv(q)
        with u the velocity of the adjacent fluid cell, evaluated from its
        EVEN-parity slots and kept for the following ODD refresh."""
        from .cumulant_ref import _seeded_sum

        L, st = self._lists, self.stencil
        cells = L["out_cell"]
        if not hasattr(self, "_out_u"):
            self._out_u = [np.zeros(cells.size) for _ in range(st.dim)]
        if parity == 0:
            t = np.stack([self._pdf[self.base[r] + cells] for r in range(st.q)])
            rho = t[0] + t[1]
            for r in range(2, st.q):
                rho = rho + t[r]
            self._out_u = [_seeded_sum(t, st.c[:, a]) / rho for a in range(st.dim)]
        u = self._out_u
        usq = u[0] * u[0]
        for a in range(1, st.dim):
            usq = usq + u[a] * u[a]
        cu = np.empty_like(usq)
        for i, k in enumerate(L["out_q"]):
            cu[i] = _seeded_sum([ua[i:i + 1] for ua in u], st.c[k])[0]
        w = st.w[L["out_q"]]
        feq_sym = (w * L["out_rho"]) * ((1.0 + (4.5 * cu) * cu) - 1.5 * usq)
        if parity == 0:
            self._pdf[L["out_slots"]] = 2.0 * feq_sym - self._pdf[L["out_partner"]]
        else:
            self._pdf[L["out_partner"]] = 2.0 * feq_sym - self._pdf[L["out_slots"]]

    # inspection
    def canonical_state(self):
        st, n = self.stencil, self.n_fluid
        t = np.empty((st.q, n))
        if self.parity == 1:
            self.refresh_boundary(1)
        for r in range(st.q):
            g = st.inv[r] if self.parity == 1 else r
            t[r] = self._pdf[self.base[g]:self.base[g] + n]
        return t

    def macroscopic_fields(self):
        rho, u = moments(self.canonical_state(), self.stencil)
        shape = _rev(self.dims)
        flat = np.ravel_multi_index(self._lists["pos"].T, shape)
        rf = np.zeros(shape)
        rf.reshape(-1)[flat] = rho
        uf = np.zeros(shape + (self.stencil.dim,))
        uf.reshape(-1, self.stencil.dim)[flat] = u.T
        return rf, uf

    # exchange access (sparse.py:335-366)
    def _pflat(self, coords):
        coords = np.asarray(coords, dtype=np.int64).reshape(-1, self.stencil.dim)
        return np.ravel_multi_index((coords[:, ::-1] + 1).T, self._lists["padded_shape"])

    def slot_index(self, coords, qs):
        cid = self._lists["cid_map"][self._pflat(coords)]
        if np.any(cid < 0):
            raise OracleError("exchange addressed a non-fluid cell slot")
        return self.base[np.asarray(qs, dtype=np.int64)] + cid

    def ghost_slot_index(self, coords, qs):
        flat = self._pflat(coords)
        qs = np.asarray(qs, dtype=np.int64).reshape(-1)
        g = self._lists["ghost"]
        try:
            return np.array([g[(int(k), int(f))] for k, f in zip(qs, flat)], dtype=np.int64)
        except KeyError as e:
            raise OracleError(f"unknown halo slot {e}") from None

    def read_slots(self, idx):
        return self._pdf[idx]

    def write_slots(self, idx, values):
        self._pdf[idx] = values

    def pdf_element_count(self):
        return (2 if self.pattern == "pull" else 1) * self.total_slots

    def idx_element_count(self):
        return (self.stencil.q - 1) * self.n_fluid

    @property
    def n_interior(self):
        return int(self._sel["interior"].size) if "interior" in self._sel else self.n_fluid

    @property
    def n_frame(self):
        return int(self._sel["frame"].size) if "frame" in self._sel else 0
