// Shared pieces of the index-list sweeps (AA even, pull) used by the single-
// engine kernels (kernels.cu) and the block-group kernels (group.cu).
#pragma once

#include "collide.cuh"

namespace slbm {

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

// Index-list layout.  D3Q19 (the bench stencil) stores the Q-1 rows in
// interleaved pairs: for rows (2k, 2k+1) one uint2 per cell, rows of pairs
// `pitch` cells long — a cell's 18 slot ids are 9 64-bit loads instead of 18
// 32-bit ones, every warp load still one contiguous 256-B run (same bytes;
// even sweep 0.90 -> 0.97 of HBM burst, tools/variants.py).  Groups of four
// rows (uint4; 5 loads) measured 0.4 % slower than pairs in an alternating
// A/B.  D3Q27 keeps single rows (13 pair loads measured 5 % slower there:
// register pressure of the cumulant sweep).  idx_offset() is the uint32 position of (row r, cell c).
template <int QM1>
constexpr bool kPairedIdx = (QM1 == 18);

__host__ __device__ __forceinline__ size_t idx_offset(bool paired, uint32_t pitch, uint32_t r,
                                                      uint32_t c) {
  return paired ? size_t(r >> 1) * 2 * pitch + 2 * size_t(c) + (r & 1u)
                : size_t(r) * pitch + c;
}

// L2 prefetch of the index list of the CTA `ahead` CTAs later.
//
// The index-list sweep is latency bound: every PDF gather depends on an idx
// load, so each cell pays two dependent DRAM round trips (ncu r01: long
// scoreboard ~12 cycles per issue at 16 warps/SM).  Here CTA b touches the
// (Q-1) rows of CTA b+ahead's cells into L2 — one 128-byte line per thread,
// BLOCK*4/128 lines per row — so when that CTA starts, its idx loads hit L2
// and only the gather goes to DRAM.  Same DRAM bytes (the rows are read
// once either way), ~+7-9% sweep bandwidth measured (profiles/r01_*).
//
// Positions are sweep positions: with a cell list (frame sweeps) they index
// `cids` (the future CTA's first cell id of each line's run is read from
// it; call after the own gathers are issued, so that dependent load overlaps
// them), without one they are cell ids.  `first` is this CTA's first
// position, `end` one past the sweep's last.
template <int QM1, int BLOCK>
__device__ __forceinline__ void prefetch_idx_ahead(const uint32_t* idx, uint32_t pitch,
                                                   const uint32_t* cids, uint32_t end,
                                                   uint32_t first, uint32_t ahead) {
  constexpr bool kPaired = kPairedIdx<QM1>;
  constexpr int kRows = kPaired ? QM1 / 2 : QM1;
  constexpr int kCellsPerLine = kPaired ? 16 : 32;
  constexpr int kLines = BLOCK / kCellsPerLine;
  if (threadIdx.x >= kRows * kLines) return;
  const uint32_t row = threadIdx.x / kLines, line = threadIdx.x % kLines;
  const uint32_t pos = first + ahead * BLOCK + line * kCellsPerLine;
  if (pos >= end) return;
  const uint32_t cell = cids ? __ldcs(cids + pos) : pos;
  if constexpr (kPaired)
    prefetch_l2(reinterpret_cast<const uint2*>(idx) + size_t(row) * pitch + cell);
  else
    prefetch_l2(idx + size_t(row) * pitch + cell);
}

// one 128-B line of the index list of cells [c0, c0 + 32) per lane < Q-1
// (warp-granular prefetch: resident / pair kernels)
template <int QM1>
__device__ __forceinline__ void prefetch_idx_warp(const uint32_t* idx, uint32_t pitch,
                                                  uint32_t c0, uint32_t lane) {
  if (lane >= QM1) return;
  if constexpr (kPairedIdx<QM1>)
    prefetch_l2(reinterpret_cast<const uint2*>(idx) + size_t(lane >> 1) * pitch + c0 +
                (lane & 1u) * 16);
  else
    prefetch_l2(idx + size_t(lane) * pitch + c0);
}

// ---- per-cell bodies shared by the single-engine sweeps (kernels.cu) and
// the block-group sweeps (group.cu); `base` = the device group starts ----

// the cell's Q-1 slot ids (s[0] = c is the rest direction's own slot)
template <class L>
__device__ __forceinline__ void load_slots(uint32_t (&s)[L::Q], const uint32_t* idx,
                                           uint32_t pitch, uint32_t c) {
  s[0] = c;
  if constexpr (kPairedIdx<L::Q - 1>) {
    const uint2* p2 = reinterpret_cast<const uint2*>(idx);
    sfor<0, (L::Q - 1) / 2>([&](auto r) {
      constexpr int R = decltype(r)::value;
      const uint2 v = __ldcs(p2 + size_t(R) * pitch + c);
      s[1 + 2 * R] = v.x;
      s[2 + 2 * R] = v.y;
    });
  } else {
    sfor<1, L::Q>([&](auto q) { s[q] = __ldcs(idx + size_t(q - 1) * pitch + c); });
  }
}

template <class L>
__device__ __forceinline__ void gather(double (&t)[L::Q], const double* pdf,
                                       const uint32_t (&s)[L::Q]) {
  sfor<0, L::Q>([&](auto q) { t[q] = pdf[s[q]]; });
}

// collide the gathered values; AA even (sparse.py:264-271): out[q] goes back
// through the slot direction inv q was read from; pull (sparse.py:257-262):
// out[q] to the cell's own group q of the other buffer.  True if unstable.
template <class L, int MODEL, bool EVEN>
__device__ __forceinline__ bool collide_scatter(const double (&t)[L::Q], const uint32_t (&s)[L::Q],
                                                double* pdf, double* dst, const uint32_t* base,
                                                uint32_t c, double omega, double lam,
                                                const double* hr = nullptr) {
  if constexpr (EVEN) {
    return collide<L, MODEL>(t, omega, lam, [&](auto q, double v) {
      constexpr int qb = L::INV[decltype(q)::value];
      pdf[s[qb]] = v;
    }, hr);
  } else {
    return collide<L, MODEL>(t, omega, lam,
                             [&](auto q, double v) { dst[base[decltype(q)::value] + c] = v; }, hr);
  }
}

// L2-only load (ld.global.cg) for data another SM wrote during the same
// launch (pair.cu): the reading SM's L1 may hold a stale copy of the line
template <bool CG>
__device__ __forceinline__ double ld_pdf(const double* p) {
  if constexpr (CG)
    return __ldcg(p);
  else
    return *p;
}

// AA odd (cell-local reversed step, sparse.py:273-282): read the opposite
// groups, write the own groups — every access a coalesced row
template <class L, int MODEL, bool CG = false>
__device__ __forceinline__ bool cell_local(double* pdf, const uint32_t* base, uint32_t c,
                                           double omega, double lam, const double* hr = nullptr) {
  double t[L::Q];
  sfor<0, L::Q>([&](auto q) {
    constexpr int qb = L::INV[q];
    t[q] = ld_pdf<CG>(pdf + base[qb] + c);
  });
  return collide<L, MODEL>(t, omega, lam,
                           [&](auto q, double v) { pdf[base[decltype(q)::value] + c] = v; }, hr);
}

// Fixed-density outlet (extension; the reference has none).
// Anti-bounce-back for a read of direction q from an OUTLET cell:
//   f_q = 2 w_q rho_o (1 + 4.5 (c_q.u)^2 - 1.5 u.u) - f*_{inv q}
// u = velocity of the adjacent fluid cell from its EVEN-parity slots
// (post-collision, momentum conserving), kept for the following ODD refresh.
// EVEN fills the appended outlet slot, ODD the cell's partner slot, mirroring
// the UBB refresh (sparse.py:301-304).  CPU restatement:
// oracle/sparse_ref.py OracleSparseEngine._refresh_outlet (same op order).
// `base` = device group starts; `u_store` = this entry's 3 velocity words.
template <class L, bool CG = false>
__device__ __forceinline__ void outlet_entry(double* pdf, const uint32_t* base, uint32_t slot,
                                             uint32_t partner, uint32_t c, int qd, double rho_o,
                                             double* u_store, int parity) {
  double u[3];
  if (parity == SLBM_EVEN) {
    double t[L::Q];
    sfor<0, L::Q>([&](auto q) { t[q] = pdf[base[q] + c]; });
    double rho = t[0] + t[1];
    sfor<2, L::Q>([&](auto q) { rho = rho + t[q]; });
    u[0] = component_sum<L, 0>(t) / rho;
    u[1] = component_sum<L, 1>(t) / rho;
    u[2] = (L::DIM == 3) ? component_sum<L, 2>(t) / rho : 0.0;
    for (int k = 0; k < 3; ++k) u_store[k] = u[k];
  } else {
    for (int k = 0; k < 3; ++k) u[k] = u_store[k];
  }
  double usq = u[0] * u[0];
  usq = usq + u[1] * u[1];
  if constexpr (L::DIM == 3) usq = usq + u[2] * u[2];
  // c_q . u, seeded with the first nonzero component (x, y, z order)
  int cq[3] = {0, 0, 0};
  double w = 0.0;
  sfor<0, L::Q>([&](auto q) {
    if (qd == decltype(q)::value) {
      cq[0] = L::CX[q];
      cq[1] = L::CY[q];
      cq[2] = L::CZ[q];
      w = weight<L>(q);
    }
  });
  double cu = 0.0;
  bool any = false;
  for (int k = 0; k < L::DIM; ++k) {
    if (cq[k] == 0) continue;
    cu = any ? (cq[k] > 0 ? cu + u[k] : cu - u[k]) : (cq[k] > 0 ? u[k] : -u[k]);
    any = true;
  }
  const double feq_sym = (w * rho_o) * ((1.0 + (4.5 * cu) * cu) - 1.5 * usq);
  if (parity == SLBM_EVEN)
    pdf[slot] = 2.0 * feq_sym - pdf[partner];
  else
    pdf[partner] = 2.0 * feq_sym - ld_pdf<CG>(pdf + slot);
}

}  // namespace slbm
