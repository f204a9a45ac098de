"""Partition + halo-plan logic (host side) against the reference's
multi-block goldens, with oracle engines standing in for the CUDA engines
(CPU only).  The GPU run of the same fixtures is tests/test_gpu_domain.py."""

import os

import numpy as np
import pytest

from conftest import flags_of, golden_files, load_golden, params_of, stencil_of
from oracle.sparse_ref import OracleSparseEngine
from paper_2408_06880_b200 import domain as D
from paper_2408_06880_b200.halo import EdgePlan, analytic_payload, direction_subset, layer_cells
from paper_2408_06880_b200.lattice import make_stencil

DOMAIN = golden_files("domain")


def _id(p):
    return os.path.basename(p)[:-4]


def partition(gf, block, st):
    block = tuple(int(b) for b in block)
    gf = D.pad_to_multiple(gf, block)
    grid = tuple(gf.dims[a] // block[a] for a in range(st.dim))
    bper = tuple(gf.periodic[a] and grid[a] == 1 for a in range(st.dim))
    blocks = {}
    for pos in D.grid_positions(grid):
        bid = D.grid_linear(pos, grid)
        origin = tuple(pos[a] * block[a] for a in range(st.dim))
        fl = D.slice_block(gf, origin, block, bper)
        if fl.fluid_count():
            blocks[bid] = (pos, origin, fl)
    return gf, grid, bper, blocks


def edges_of(gf, grid, bper, blocks, st):
    dim = st.dim
    offsets = sorted({tuple(0 if bper[a] else int(st.c[k][a]) for a in range(dim))
                      for k in range(1, st.q)} - {(0,) * dim})
    out = []
    for bid, (pos, _, _) in sorted(blocks.items()):
        for sigma in offsets:
            npos, ok = [], True
            for a in range(dim):
                p = pos[a] + sigma[a]
                if gf.periodic[a]:
                    p %= grid[a]
                elif not 0 <= p < grid[a]:
                    ok = False
                    break
                npos.append(p)
            if ok and D.grid_linear(tuple(npos), grid) in blocks:
                out.append((bid, D.grid_linear(tuple(npos), grid), sigma))
    return out


@pytest.mark.parametrize("pattern", ["pull", "aa"])
@pytest.mark.parametrize("path", DOMAIN, ids=_id)
def test_edge_plans_match_reference(path, pattern):
    rec = load_golden(path)
    gf, st, p = flags_of(rec), stencil_of(rec), params_of(rec)
    gf, grid, bper, blocks = partition(gf, rec["block"], st)
    assert sorted(blocks) == list(rec[f"{pattern}_blocks"])
    eng = {b: OracleSparseEngine(fl, st, p, pattern, frame_width=1) for b, (_, _, fl) in blocks.items()}
    edges = edges_of(gf, grid, bper, blocks, st)
    want = rec[f"{pattern}_edges"]
    rows, send, take, tgt = [], [], [], []
    for a, b, sigma in edges:
        plan = EdgePlan(a, b, sigma, st, blocks[a][2], blocks[b][2], pattern, eng[a], eng[b])
        for ph, pp in plan.phases.items():
            rows.append([a, b, *sigma, ph.value, pp.n_wire, len(pp.tgt_sel)])
            send.append(pp.send_sel)
            take.append(pp.pos_from_sparse)
            tgt.append(pp.tgt_sel)
    assert np.array_equal(np.array(rows, dtype=np.int64), want)
    assert np.array_equal(np.concatenate(send), rec[f"{pattern}_send"])
    assert np.array_equal(np.concatenate(take), rec[f"{pattern}_take"])
    assert np.array_equal(np.concatenate(tgt), rec[f"{pattern}_tgt"])


@pytest.mark.parametrize("path", DOMAIN, ids=_id)
def test_half_plans_need_only_flags(path):
    """A rank that owns only one end of an edge derives the same wire layout
    (n_wire, take) from the flag boxes alone."""
    rec = load_golden(path)
    gf, st, p = flags_of(rec), stencil_of(rec), params_of(rec)
    gf, grid, bper, blocks = partition(gf, rec["block"], st)
    eng = {b: OracleSparseEngine(fl, st, p, "aa") for b, (_, _, fl) in blocks.items()}
    for a, b, sigma in edges_of(gf, grid, bper, blocks, st)[:12]:
        full = EdgePlan(a, b, sigma, st, blocks[a][2], blocks[b][2], "aa", eng[a], eng[b])
        send_half = EdgePlan(a, b, sigma, st, blocks[a][2], blocks[b][2], "aa", eng[a], None)
        recv_half = EdgePlan(a, b, sigma, st, blocks[a][2], blocks[b][2], "aa", None, eng[b])
        for ph in full.phases:
            f, s, r = full.phases[ph], send_half.phases[ph], recv_half.phases[ph]
            assert np.array_equal(f.send_sel, s.send_sel) and r.send_sel is None
            assert np.array_equal(f.tgt_sel, r.tgt_sel) and s.tgt_sel is None
            assert f.n_wire == s.n_wire == r.n_wire
            assert np.array_equal(f.pos_from_sparse, r.pos_from_sparse)


@pytest.mark.parametrize("name,tau,count", [("d2q9", (1, 0), 3), ("d2q9", (1, 1), 1),
                                             ("d3q19", (1, 0, 0), 5), ("d3q19", (1, 1, 0), 1),
                                             ("d3q19", (1, 1, 1), 0), ("d3q27", (1, 0, 0), 9),
                                             ("d3q27", (1, 1, 0), 3), ("d3q27", (1, 1, 1), 1)])
def test_direction_subset_counts(name, tau, count):
    st = make_stencil(name)
    sub = direction_subset(st, tau)
    assert len(sub) == count
    for k in sub:
        assert all(int(st.c[k][a]) == t for a, t in enumerate(tau) if t)


def test_layer_and_payload():
    st = make_stencil("d3q19")
    cells = layer_cells((4, 3, 2), (1, 0, 0))
    assert cells.shape == (6, 3) and np.all(cells[:, 0] == 3)
    assert list(map(tuple, cells[:2])) == [(3, 0, 0), (3, 1, 0)]
    assert analytic_payload((4, 4, 4), (1, 0, 0), st) == 80


def test_balance_curves():
    assert D.hilbert_key((0, 0), 1) == 0
    keys = sorted(D.hilbert_key((x, y), 2) for x in range(4) for y in range(4))
    assert keys == list(range(16))
    assert D.morton_key((1, 0), 1) == 2 and D.morton_key((0, 1), 1) == 1
    assert D.greedy_segments([1, 1, 1, 1], 2) == [0, 0, 1, 1]
    assert D.greedy_segments([4, 1, 1, 1, 1], 2) == [0, 1, 1, 1, 1]
