// Shared pieces of the index-list sweeps (AA even, pull) used by the single-
// engine kernels (kernels.cu) and the block-group kernels (group.cu).
#pragma once

#include "common.cuh"

namespace slbm {

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
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
// `cids` (the future CTA's first cell id of each 32-cell run is read from
// it; call after the own gathers are issued, so that dependent load overlaps
// them), without one they are cell ids.  `first` is this CTA's first
// position, `end` one past the sweep's last.
template <int QM1, int BLOCK>
__device__ __forceinline__ void prefetch_idx_ahead(const uint32_t* idx, uint32_t pitch,
                                                   const uint32_t* cids, uint32_t end,
                                                   uint32_t first, uint32_t ahead) {
  constexpr int kLines = BLOCK * 4 / 128;
  if (threadIdx.x >= QM1 * kLines) return;
  const uint32_t row = threadIdx.x / kLines, line = threadIdx.x % kLines;
  const uint32_t pos = first + ahead * BLOCK + line * 32;
  if (pos >= end) return;
  const uint32_t cell = cids ? __ldcs(cids + pos) : pos;
  prefetch_l2(idx + size_t(row) * pitch + cell);
}

}  // namespace slbm
