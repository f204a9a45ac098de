// Batched block-table execution: every sparse engine a rank
// owns is swept by ONE launch per phase instead of one per block.  The
// reference only computes a block -> worker assignment (domain.py:302-325);
// here the blocks of a worker actually execute together.
//
// A group holds, per engine and phase, the engine's SweepArgs in a device
// table, and per phase the prefix sum of its CTA counts.  A CTA finds its
// engine by binary search over that prefix, stages the engine's SweepArgs in
// shared memory, and runs the same per-cell code as the single-engine sweep
// (identical arithmetic -> identical bits).  UBB refresh, outlet refresh and
// the step counters are batched the same way.  With the halo program this
// makes one domain step O(1) launches, which a CUDA graph then replays.
#include <algorithm>
#include <unordered_map>
#include <vector>

#include "collide.cuh"
#include <cstring>

#include "engine.cuh"
#include "sweep.cuh"

// per-engine sweep arguments of one phase, staged in shared memory by a CTA
namespace slbm {
struct GroupArgs {
  double* pdf;
  double* dst;
  const uint32_t* idx;
  const uint32_t* cids;
  const uint32_t* skip;  // interior: identity order minus the frame bits
  uint32_t offset;       // identity sweeps: first cell (contiguous interior), warp aligned
  uint32_t lo;           // cells below lo are skipped
  uint32_t n_cells;
  uint32_t n_fluid;
  uint32_t idx_pitch;
  uint32_t base[28];  // device group starts (pbase)
  unsigned long long* bad;
  const unsigned long long* step;
  // addressing of the index-list sweeps: the engine's own list and buffer,
  // or, with direct local halo edges (slbm_group_link_halo), the group's
  // rewritten list over the shared pdf pool (slots relative to spdf, a
  // cell's own rest slot at slot_off + c)
  const uint32_t* sidx;
  double* spdf;
  uint32_t slot_off;
};
// What an index-list CTA needs before its first load, per engine, held in
// the launch's kernel parameters (constant bank) together with the CTA
// prefix: finding the engine and its lists then costs constant-cache hits
// instead of a chain of dependent global loads (binary search over the
// prefix, then the table row) -- that chain held ~11 % of the group even
// sweep's stall samples and made it ~9 % slower than the single-engine
// sweep on the same block (tools/group_probe.py).
struct HotArgs {
  const uint32_t* idx;
  double* pdf;
  const uint32_t* cids;
  const uint32_t* skip;
  uint32_t offset, n_cells, idx_pitch, lo;
  uint32_t slot_off, pad;
};
template <int CAP>
struct GroupHot {
  uint32_t start[CAP + 1];
  HotArgs hot[CAP];
};
// the boundary launch's per-engine buffer and group starts, as kernel
// parameters (the UBB / outlet entries then need no table-row load)
template <int CAP>
struct BoundaryHot {
  double* pdf[CAP];
  uint32_t base[CAP][28];
  __device__ double* buf(int e) const { return pdf[e]; }
  __device__ const uint32_t* starts(int e) const { return base[e]; }
};
// ... and the same lookups through the device table (groups of > 128 blocks)
struct BoundaryTable {
  const GroupArgs* t;
  __device__ double* buf(int e) const { return t[e].pdf; }
  __device__ const uint32_t* starts(int e) const { return t[e].base; }
};
}  // namespace slbm

using namespace slbm;

struct SlbmGroup {
  int device = 0;
  int q = 19, model = SLBM_SRT, pattern = SLBM_AA;
  double omega = 1.0, lam = 1.0;
  const double* hr = nullptr;  // cumulant: higher-order rates of the first engine
  std::vector<SlbmEngine*> engines;
  // tables[phase][flip] -> device array of GroupArgs (one per engine)
  GroupArgs* table[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
  // the same per (phase, flip) as kernel-parameter blocks (index-list sweeps)
  GroupHot<16>* hot16[3][2] = {};
  GroupHot<128>* hot128[3][2] = {};
  GroupHot<512>* hot512[3][2] = {};
  // direct local halo edges (slbm_group_link_halo): every engine's pdf lives
  // in one pool, the index-list sweeps read a rewritten list whose ghost
  // entries of local edges address the source engine's slot in the pool
  bool direct = false;
  double* pool = nullptr;
  std::vector<uint32_t> pool_off;  // per engine, in pdf elements
  std::vector<uint32_t*> gidx;     // per engine, (q-1) x idx_pitch
  // the local edges as (source slot, ghost slot) pool offsets, for
  // slbm_group_stale_copy
  uint32_t* save_src = nullptr;
  uint32_t* save_dst = nullptr;
  int64_t n_save = 0;
  uint32_t* cta_start[3] = {nullptr, nullptr, nullptr};
  uint32_t n_cta[3] = {0, 0, 0};
  // the cell-local (odd) sweep: CTAs of kOddTiles tiles (own prefix)
  uint32_t* cta_start_odd[3] = {nullptr, nullptr, nullptr};
  uint32_t n_cta_odd[3] = {0, 0, 0};
  // batched UBB program
  uint16_t* ubb_eng = nullptr;
  uint32_t *ubb_slot = nullptr, *ubb_partner = nullptr;
  double* ubb_corr = nullptr;
  int64_t n_ubb = 0;
  unsigned long long** steps = nullptr;  // per engine d_step
  int flip = 0;  // pull: which buffer of each engine is current
  bool has_outlets = false;
  // batched outlet program: entry -> (engine, index in its outlet arrays)
  struct OutletTab* out_tab = nullptr;
  uint16_t* out_eng = nullptr;
  uint32_t* out_idx = nullptr;
  // the outlet program flattened in entry order (one coalesced load per
  // field instead of engine table -> arrays -> entry)
  uint32_t *fo_slot = nullptr, *fo_partner = nullptr, *fo_cell = nullptr;
  uint8_t* fo_dir = nullptr;
  double* fo_rho = nullptr;
  double** fo_u = nullptr;
  BoundaryHot<16>* bhot16[2] = {};
  BoundaryHot<128>* bhot128[2] = {};
  int64_t n_out = 0;
};

// an engine's outlet program arrays (kernels.cu k_outlet reads the same)
struct OutletTab {
  const uint32_t *slot, *partner, *cell;
  const uint8_t* dir;
  const double* rho;
  double* u;
};

namespace {

constexpr int kGB = 128;
// The odd sweep's CTAs stage their engine's table row in shared memory (one
// barrier per CTA); two 128-cell tiles per CTA halve that per-cell cost.
constexpr int kOddTiles = 2;
// index-list sweeps of the global-table kernel: one tile per CTA (two
// measured slower: the second tile spills and runs after the first)
constexpr int kEvenTiles = 1;

__device__ __forceinline__ int find_engine(const uint32_t* __restrict__ start, int n, uint32_t cta) {
  int lo = 0, hi = n;  // last e with start[e] <= cta
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (start[mid] <= cta)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// identity-order rows of CTA blockIdx + ahead of the group sweep
template <class L, int TILES>
__device__ __forceinline__ void prefetch_group_ahead(const GroupArgs* __restrict__ table,
                                                     const uint32_t* __restrict__ start,
                                                     int n_eng, int eng, uint32_t ahead) {
  constexpr int kPfThreads = (kPairedIdx<L::Q - 1> ? (L::Q - 1) / 2 : L::Q - 1) *
                             (kGB / (kPairedIdx<L::Q - 1> ? 16 : 32));
  const uint32_t tgt = blockIdx.x + ahead;
  if (threadIdx.x >= kPfThreads || tgt >= gridDim.x) return;
  const int e2 = (eng + 1 >= n_eng || tgt < start[eng + 1]) ? eng : find_engine(start, n_eng, tgt);
  const GroupArgs& b = table[e2];
  if (b.cids != nullptr) return;
#pragma unroll
  for (int t = 0; t < TILES; ++t)
    prefetch_idx_ahead<L::Q - 1, kGB>(gmem(b.sidx), b.idx_pitch, nullptr, b.offset + b.n_cells,
                                      b.offset + ((tgt - start[e2]) * TILES + t) * kGB, 0);
}

// index-list group sweep (AA even / pull) with the block table in the
// kernel parameters (GroupHot); bodies as k_index_sweep
template <class L, int MODEL, int KIND, int CAP>
__global__ void __launch_bounds__(kGB, 4)
    k_group_hot(const __grid_constant__ GroupHot<CAP> gh, const GroupArgs* __restrict__ table,
                int n_eng, double omega, double lam, const double* hr, uint32_t ahead) {
  static_assert(KIND != 2, "the cell-local sweep keeps the global table");
  int eng = 0;  // last e with start[e] <= blockIdx.x (constant-bank binary search)
  {
    int hi = n_eng;
    while (hi - eng > 1) {
      const int mid = (eng + hi) >> 1;
      if (gh.start[mid] <= blockIdx.x)
        eng = mid;
      else
        hi = mid;
    }
  }
  const HotArgs& a = gh.hot[eng];
  const uint32_t i = (blockIdx.x - gh.start[eng]) * kGB + threadIdx.x;
  const uint32_t* idx = gmem(a.idx);
  double* pdf = gmem(a.pdf);
  // identity sweeps: rows of CTA blockIdx + ahead (it may be the next engine's)
  {
    constexpr int kPfThreads = (kPairedIdx<L::Q - 1> ? (L::Q - 1) / 2 : L::Q - 1) *
                               (kGB / (kPairedIdx<L::Q - 1> ? 16 : 32));
    const uint32_t tgt = blockIdx.x + ahead;
    if (threadIdx.x < kPfThreads && tgt < gridDim.x) {
      int e2 = eng;
      while (e2 + 1 < n_eng && gh.start[e2 + 1] <= tgt) ++e2;
      const HotArgs& b = gh.hot[e2];
      if (b.cids == nullptr)
        prefetch_idx_ahead<L::Q - 1, kGB>(gmem(b.idx), b.idx_pitch, nullptr, b.offset + b.n_cells,
                                          b.offset + (tgt - gh.start[e2]) * kGB, 0);
    }
  }
  pdl_launch_dependents();
  pdl_wait();  // the boundary kernel's halo / wall values
  if (i >= a.n_cells) return;
  const uint32_t c = a.cids ? gmem(a.cids)[i] : a.offset + i;
  if (c < a.lo) return;
  const uint32_t skip_word = a.skip ? __ldg(gmem(a.skip) + (c >> 5)) : 0u;
  uint32_t s[L::Q];
  double t[L::Q];
  load_slots<L>(s, idx, a.idx_pitch, c);
  s[0] = a.slot_off + c;
  if ((skip_word >> (c & 31)) & 1u) return;
  gather<L>(t, pdf, s);
  if (a.cids)
    prefetch_idx_ahead<L::Q - 1, kGB>(idx, a.idx_pitch, gmem(a.cids), a.n_cells,
                                      (blockIdx.x - gh.start[eng]) * kGB, ahead);
  const GroupArgs& g = table[eng];
  double* dst = KIND == 0 ? gmem(g.dst) : nullptr;
  if (collide_scatter<L, MODEL, KIND == 1>(t, s, pdf, dst, g.base, c, omega, lam, hr))
    atomicMin(g.bad, *g.step - 1);  // the boundary kernel advanced the counter
}

template <class L, int MODEL, int KIND>
__global__ void __launch_bounds__(kGB, KIND == 2 ? 6 : 4) k_group(const GroupArgs* __restrict__ table,
                                                  const uint32_t* __restrict__ start, int n_eng,
                                                  double omega, double lam, const double* hr,
                                                  uint32_t ahead) {
  // every thread finds its engine and reads the (tiny, L1-resident) table
  // row itself: no single-thread staging + __syncthreads at CTA start, which
  // cost ~15% of the even sweep (measured, tools/slab_probe.py)
  // engine of this CTA: binary search over the (L1-resident) CTA prefix --
  // a per-CTA engine map measured slower (its line is an L2 round trip per
  // CTA, consecutive CTAs land on different SMs)
  // the cell-local sweep runs its CTAs last to first (as k_aa_odd): it
  // starts on the lines the index-list sweep before it left in L2
  const uint32_t bid = KIND == 2 ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
  const int eng = find_engine(start, n_eng, bid);
  const uint32_t first = start[eng];
  // the odd sweep addresses 2Q group rows through base[]: staged in shared
  // memory those offsets stay out of registers (77 vs 128 + spills)
  __shared__ GroupArgs staged;
  if constexpr (KIND == 2) {
    if (threadIdx.x == 0) staged = table[eng];
    __syncthreads();
  }
  const GroupArgs& a = KIND == 2 ? staged : table[eng];
  constexpr int kTiles = KIND == 2 ? kOddTiles : kEvenTiles;
  const uint32_t pos0 = (bid - first) * kGB * kTiles;  // this CTA's first sweep position
  const uint32_t* idx = gmem(a.sidx);
  const uint32_t* cids = a.cids ? gmem(a.cids) : nullptr;
  const uint32_t* skip = a.skip ? gmem(a.skip) : nullptr;
  double* pdf = KIND != 2 ? gmem(a.spdf) : nullptr;
  double* dst = KIND == 0 ? gmem(a.dst) : nullptr;  // pull only
  const uint32_t pitch = a.idx_pitch, n_cells = a.n_cells, offset = a.offset;
  pdl_launch_dependents();
  pdl_wait();  // the boundary kernel's halo / wall values (read-only lists above)
  bool bad = false;
#pragma unroll
  for (int tile = 0; tile < kTiles; ++tile) {
    const uint32_t i = pos0 + tile * kGB + threadIdx.x;
    if (i >= n_cells) break;
    const uint32_t c = cids ? cids[i] : offset + i;
    if (c < a.lo || (skip && ((__ldg(skip + (c >> 5)) >> (c & 31)) & 1u))) continue;
    if constexpr (KIND == 2) {
      bad |= cell_local<L, MODEL>(a.pdf, a.base, c, omega, lam, hr);
    } else {
      uint32_t s[L::Q];
      double t[L::Q];
      load_slots<L>(s, idx, pitch, c);
      s[0] = a.slot_off + c;
      gather<L>(t, pdf, s);
      // index-list rows of the CTA `ahead` CTAs later (sweep.cuh), issued
      // after this CTA's own loads: finding them takes dependent table
      // reads (the CTA may belong to the next engine -- a per-engine
      // distance left the first quarter wave of every block without it)
      if (tile == 0) prefetch_group_ahead<L, kTiles>(table, start, n_eng, eng, ahead);
      if (cids)
        prefetch_idx_ahead<L::Q - 1, kGB>(idx, pitch, cids, n_cells, pos0 + tile * kGB,
                                          ahead * kTiles);
      bad |= collide_scatter<L, MODEL, KIND == 1>(t, s, pdf, dst, a.base, c, omega, lam, hr);
    }
  }
  // the group's boundary kernel advanced the step counter before this sweep
  if (bad) atomicMin(a.bad, *a.step - 1);
}

// Everything a block group does between two sweeps, in ONE launch (the
// strong-scaling small-share path: per-step fixed costs):
//   * every engine's step counter += 1 (finish_step of the previous step's
//     device half: the sweeps report an instability at *step - 1);
//   * the device-local halo edges of this phase (exchange.py:222-253 for
//     blocks on this GPU);
//   * the UBB refresh (sparse.py:295-304) and the fixed-density outlet of
//     every block.
// The three programs touch disjoint slots -- a slot has exactly one upwind
// source (a fluid cell of the own block, a cell of another block, or a wall)
// -- and none reads a slot another writes, so they run concurrently; the
// per-engine path (halo kernel, then refresh) gives the same bits.
// Work split by CTA ranges (no section test per thread): halo CTAs and UBB
// CTAs copy kBItems entries per thread with all index and value loads of a
// thread issued before its stores (the program is latency bound: ~1.4 M
// 8-byte copies per phase for the C4 artery's 50 blocks), outlet CTAs one
// entry per thread.  The halo engines' pdf pointers are staged in shared
// memory (a divergent index into the kernel-parameter table serialises).
constexpr int kBT = 128;
constexpr int kBItems = 4;

// ---- direct local halo edges (slbm_group_link_halo) ----
__global__ void k_add_offset(uint32_t* out, const uint32_t* in, int64_t n, uint32_t off) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = in[i] + off;
}
// pos[slot] = uint32 position in the index list of the entry reading `slot`
// (a slot is read by at most one (cell, direction): the builder's check)
__global__ void k_slot_pos(uint32_t* pos, const uint32_t* idx, uint32_t pitch, uint32_t n_fluid,
                           int rows, int paired) {
  const int64_t n = int64_t(rows) * n_fluid;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = uint32_t(k / n_fluid), c = uint32_t(k % n_fluid);
    const size_t f = idx_offset(paired != 0, pitch, r, c);
    pos[idx[f]] = uint32_t(f);
  }
}
// mode 0: ghost <- source, 1: swap, 2: source <- ghost
__global__ void k_pool_copy(double* pool, const uint32_t* src, const uint32_t* dst, int64_t n,
                            int mode) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t a = mode == 2 ? dst[i] : src[i], b = mode == 2 ? src[i] : dst[i];
  const double v = pool[a];
  if (mode == 1) pool[a] = pool[b];
  pool[b] = v;
}
__global__ void k_rewrite(uint32_t* gidx, const uint32_t* pos, const uint32_t* ghost,
                          const uint32_t* val, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t p = pos[ghost[i]];
  if (p != 0xFFFFFFFFu) gidx[p] = val[i];
}

__global__ void k_flatten_outlet(const OutletTab* ot, const uint16_t* oeng, const uint32_t* oidx,
                                 int64_t n, uint32_t* slot, uint32_t* partner, uint32_t* cell,
                                 uint8_t* dir, double* rho, double** u) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const OutletTab& o = ot[oeng[i]];
  const uint32_t k = oidx[i];
  slot[i] = o.slot[k];
  partner[i] = o.partner[k];
  cell[i] = o.cell[k];
  dir[i] = o.dir[k];
  rho[i] = o.rho[k];
  u[i] = o.u + 3 * size_t(k);
}

// The boundary launch.  LK looks up an engine's buffer and group starts:
// BoundaryHot (kernel parameters, groups of <= 128 blocks) or BoundaryTable
// (the device table).  The outlet program is flattened in entry order, so
// every entry is one round of coalesced index loads, then its PDF loads.
template <class L, class LK>
__global__ void __launch_bounds__(kBT) k_group_boundary(
    const __grid_constant__ LK bh, const __grid_constant__ PdfTable lt,
    LocalEdges le, const uint16_t* __restrict__ ueng, const uint32_t* __restrict__ uslot,
    const uint32_t* __restrict__ upartner, const double* __restrict__ ucorr, int64_t n_ubb,
    const uint16_t* __restrict__ oeng, const uint32_t* __restrict__ fo_slot,
    const uint32_t* __restrict__ fo_partner, const uint32_t* __restrict__ fo_cell,
    const uint8_t* __restrict__ fo_dir, const double* __restrict__ fo_rho, double* const* fo_u,
    int64_t n_out, unsigned long long** steps, int n_eng, int parity, uint32_t cta_halo,
    uint32_t cta_ubb) {
  pdl_launch_dependents();
  const uint32_t b = blockIdx.x;
  if (b == 0) {
    pdl_wait();  // the previous sweep reads the step counters
    for (int e = threadIdx.x; e < n_eng; e += kBT) *steps[e] += 1;
  }
  if (b < cta_halo) {
    __shared__ double* sp[kMaxHaloEngines];
    for (int e = threadIdx.x; e < le.n_eng; e += kBT) sp[e] = gmem(lt.p[e]);
    __syncthreads();
    const int64_t i0 = int64_t(b) * kBT * kBItems + threadIdx.x;
    uint16_t se[kBItems], de[kBItems];
    uint32_t ss[kBItems], ds[kBItems];
    double v[kBItems];
#pragma unroll
    for (int k = 0; k < kBItems; ++k) {
      const int64_t i = i0 + k * kBT;
      if (i < le.n) {
        se[k] = le.se[i];
        ss[k] = le.ss[i];
        de[k] = le.de[i];
        ds[k] = le.ds[i];
      }
    }
    pdl_wait();
#pragma unroll
    for (int k = 0; k < kBItems; ++k)
      if (i0 + k * kBT < le.n) v[k] = gmem(sp[se[k]])[ss[k]];
#pragma unroll
    for (int k = 0; k < kBItems; ++k)
      if (i0 + k * kBT < le.n) gmem(sp[de[k]])[ds[k]] = v[k];
    return;
  }
  if (b < cta_halo + cta_ubb) {  // sparse.py:301-304
    const int64_t i0 = int64_t(b - cta_halo) * kBT * kBItems + threadIdx.x;
    double* pdf[kBItems];
    uint32_t from[kBItems], to[kBItems];
    double corr[kBItems], v[kBItems];
#pragma unroll
    for (int k = 0; k < kBItems; ++k) {
      const int64_t i = i0 + k * kBT;
      if (i < n_ubb) {
        pdf[k] = gmem(bh.buf(ueng[i]));
        from[k] = parity == SLBM_EVEN ? upartner[i] : uslot[i];
        to[k] = parity == SLBM_EVEN ? uslot[i] : upartner[i];
        corr[k] = ucorr[i];
      }
    }
    pdl_wait();
#pragma unroll
    for (int k = 0; k < kBItems; ++k)
      if (i0 + k * kBT < n_ubb) v[k] = pdf[k][from[k]];
#pragma unroll
    for (int k = 0; k < kBItems; ++k)
      if (i0 + k * kBT < n_ubb) pdf[k][to[k]] = v[k] + corr[k];
    return;
  }
  const int64_t i = int64_t(b - cta_halo - cta_ubb) * kBT + threadIdx.x;
  int e = 0;
  uint32_t slot = 0, partner = 0, cell = 0;
  int dir = 0;
  double rho = 0.0;
  double* u = nullptr;
  if (i < n_out) {
    e = oeng[i];
    slot = fo_slot[i];
    partner = fo_partner[i];
    cell = fo_cell[i];
    dir = fo_dir[i];
    rho = fo_rho[i];
    u = gmem(fo_u[i]);
  }
  pdl_wait();  // in every thread, so the chain's completion stays transitive
  if (i < n_out)
    outlet_entry<L>(gmem(bh.buf(e)), bh.starts(e), slot, partner, cell, dir, rho, u, parity);
}

// CTA prefix of a phase on the device: start[e] = first CTA of engine e
int upload_prefix(const std::vector<uint32_t>& start, uint32_t** out) {
  SLBM_CUDA_TRY(cudaMalloc(out, start.size() * sizeof(uint32_t)));
  SLBM_CUDA_TRY(cudaMemcpy(*out, start.data(), start.size() * sizeof(uint32_t),
                           cudaMemcpyHostToDevice));
  return SLBM_OK;
}

template <class F>
void on_lattice(int q, F&& f) {
  if (q == 9)
    f(LatD2Q9{});
  else if (q == 19)
    f(LatD3Q19{});
  else
    f(LatD3Q27{});
}

GroupArgs args_of(SlbmEngine* e, int phase, int flip) {
  GroupArgs a{};
  double* bufs[2] = {e->pdf, e->tmp};
  a.pdf = e->pattern == SLBM_PULL ? bufs[flip] : e->pdf;
  a.dst = e->pattern == SLBM_PULL ? bufs[1 - flip] : nullptr;
  a.idx = e->idx;
  a.n_fluid = uint32_t(e->n_fluid);
  a.cids = phase == SLBM_PHASE_FRAME ? e->frame_cids : nullptr;
  a.skip = nullptr;
  a.offset = 0;
  a.lo = 0;
  a.n_cells = uint32_t(phase == SLBM_PHASE_FRAME ? e->n_frame : e->n_fluid);
  if (phase == SLBM_PHASE_INTERIOR) {
    if (e->interior_lo >= 0) {
      a.lo = uint32_t(e->interior_lo);
      a.offset = a.lo & ~31u;
      a.n_cells = uint32_t(e->interior_lo + e->n_interior) - a.offset;
    } else {
      a.skip = e->frame_bits;
      if (e->n_interior == 0) a.n_cells = 0;
    }
  }
  a.idx_pitch = uint32_t(e->idx_pitch);
  for (int q = 0; q <= e->q && q < 28; ++q) a.base[q] = uint32_t(e->pbase[q]);
  a.bad = e->d_bad;
  a.step = e->d_step;
  a.sidx = a.idx;
  a.spdf = a.pdf;
  a.slot_off = 0;
  return a;
}

// engine i of the group: with direct local halo edges the index-list sweeps
// address the pool through the group's rewritten list (AA: one buffer)
GroupArgs gargs_of(const SlbmGroup* g, int i, int phase, int flip) {
  GroupArgs a = args_of(g->engines[i], phase, flip);
  if (g->direct) {
    a.sidx = g->gidx[i];
    a.spdf = g->pool;
    a.slot_off = g->pool_off[i];
  }
  return a;
}

template <int CAP>
void fill_hot(GroupHot<CAP>*& out, const SlbmGroup* g, int phase, int flip,
              const std::vector<uint32_t>& start) {
  const int n = int(g->engines.size());
  delete out;
  out = new GroupHot<CAP>();
  for (int i = 0; i <= n; ++i) out->start[i] = start[i];
  for (int i = 0; i < n; ++i) {
    const GroupArgs a = gargs_of(g, i, phase, flip);
    out->hot[i] = HotArgs{a.sidx,     a.spdf,      a.cids, a.skip, a.offset,
                          a.n_cells, a.idx_pitch, a.lo,   a.slot_off, 0};
  }
}

template <int CAP>
void fill_bhot(BoundaryHot<CAP>*& out, const SlbmGroup* g, int flip) {
  const int n = int(g->engines.size());
  delete out;
  out = new BoundaryHot<CAP>();
  for (int i = 0; i < n; ++i) {
    const GroupArgs a = args_of(g->engines[i], 0, flip);
    out->pdf[i] = a.pdf;
    for (int q = 0; q < 28; ++q) out->base[i][q] = a.base[q];
  }
}

// CTA prefixes, device tables and kernel-parameter blocks of every phase
int build_tables(SlbmGroup* g) {
  const int n = int(g->engines.size());
  for (int flip = 0; flip < 2; ++flip) {
    if (n <= 16)
      fill_bhot(g->bhot16[flip], g, flip);
    else if (n <= 128)
      fill_bhot(g->bhot128[flip], g, flip);
  }
  SlbmEngine* e0 = g->engines[0];
  for (int phase = 0; phase < 3; ++phase) {
    if (phase && !e0->has_split) continue;
    std::vector<uint32_t> start(n + 1, 0);
    for (int i = 0; i < n; ++i) {
      const GroupArgs a = args_of(g->engines[i], phase, 0);
      start[i + 1] = start[i] + (a.n_cells + kGB * kEvenTiles - 1) / (kGB * kEvenTiles);
    }
    g->n_cta[phase] = start[n];
    if (g->cta_start[phase]) cudaFree(g->cta_start[phase]);
    SLBM_TRY(upload_prefix(start, &g->cta_start[phase]));
    std::vector<uint32_t> odd(n + 1, 0);
    for (int i = 0; i < n; ++i) {
      const GroupArgs a = args_of(g->engines[i], phase, 0);
      odd[i + 1] = odd[i] + (a.n_cells + kGB * kOddTiles - 1) / (kGB * kOddTiles);
    }
    g->n_cta_odd[phase] = odd[n];
    if (g->cta_start_odd[phase]) cudaFree(g->cta_start_odd[phase]);
    SLBM_TRY(upload_prefix(odd, &g->cta_start_odd[phase]));
    for (int flip = 0; flip < 2; ++flip) {
      if (n <= 16)
        fill_hot(g->hot16[phase][flip], g, phase, flip, start);
      else if (n <= 128)
        fill_hot(g->hot128[phase][flip], g, phase, flip, start);
      else if (n <= 512)
        fill_hot(g->hot512[phase][flip], g, phase, flip, start);
    }
    for (int flip = 0; flip < 2; ++flip) {
      std::vector<GroupArgs> tab(n);
      for (int i = 0; i < n; ++i) tab[i] = gargs_of(g, i, phase, flip);
      if (g->table[phase][flip]) cudaFree(g->table[phase][flip]);
      SLBM_CUDA_TRY(cudaMalloc(&g->table[phase][flip], n * sizeof(GroupArgs)));
      SLBM_CUDA_TRY(cudaMemcpy(g->table[phase][flip], tab.data(), n * sizeof(GroupArgs),
                               cudaMemcpyHostToDevice));
    }
  }
  return SLBM_OK;
}


// everything of slbm_group_create past the checks (the caller destroys a
// partly built group on failure)
int init_group(SlbmGroup* g, SlbmEngine** engines, int n) {
  // pull: each engine's e->pdf is "current"; record the flip as 0
  SLBM_TRY(build_tables(g));
  // concatenated UBB program with engine ids
  for (int i = 0; i < n; ++i) g->n_ubb += engines[i]->n_ubb;
  for (int i = 0; i < n; ++i) g->has_outlets |= engines[i]->n_out > 0;
  if (g->has_outlets) {
    std::vector<OutletTab> tab(n);
    std::vector<uint16_t> oe;
    std::vector<uint32_t> oi;
    for (int i = 0; i < n; ++i) {
      SlbmEngine* e = engines[i];
      tab[i] = OutletTab{e->out_slot, e->out_partner, e->out_cell, e->out_dir, e->out_rho, e->out_u};
      // entries in cell order: the (up to 5 / 9) entries of one cell sit in
      // one warp and read its populations once (the engine's own order is by
      // direction; each entry is independent, so the order is free)
      std::vector<uint32_t> cell(size_t(e->n_out));
      if (e->n_out)
        SLBM_CUDA_TRY(cudaMemcpy(cell.data(), e->out_cell, e->n_out * sizeof(uint32_t),
                                 cudaMemcpyDeviceToHost));
      std::vector<uint32_t> order(size_t(e->n_out));
      for (int64_t k = 0; k < e->n_out; ++k) order[k] = uint32_t(k);
      std::stable_sort(order.begin(), order.end(),
                       [&](uint32_t a, uint32_t b) { return cell[a] < cell[b]; });
      for (uint32_t k : order) {
        oe.push_back(uint16_t(i));
        oi.push_back(k);
      }
    }
    g->n_out = int64_t(oe.size());
    SLBM_CUDA_TRY(cudaMalloc(&g->out_tab, n * sizeof(OutletTab)));
    SLBM_CUDA_TRY(cudaMemcpy(g->out_tab, tab.data(), n * sizeof(OutletTab), cudaMemcpyHostToDevice));
    SLBM_CUDA_TRY(cudaMalloc(&g->out_eng, oe.size() * sizeof(uint16_t)));
    SLBM_CUDA_TRY(cudaMemcpy(g->out_eng, oe.data(), oe.size() * 2, cudaMemcpyHostToDevice));
    SLBM_CUDA_TRY(cudaMalloc(&g->out_idx, oi.size() * sizeof(uint32_t)));
    SLBM_CUDA_TRY(cudaMemcpy(g->out_idx, oi.data(), oi.size() * 4, cudaMemcpyHostToDevice));
    const size_t m = oe.size();
    SLBM_CUDA_TRY(cudaMalloc(&g->fo_slot, m * 4));
    SLBM_CUDA_TRY(cudaMalloc(&g->fo_partner, m * 4));
    SLBM_CUDA_TRY(cudaMalloc(&g->fo_cell, m * 4));
    SLBM_CUDA_TRY(cudaMalloc(&g->fo_dir, m));
    SLBM_CUDA_TRY(cudaMalloc(&g->fo_rho, m * 8));
    SLBM_CUDA_TRY(cudaMalloc(&g->fo_u, m * sizeof(double*)));
    if (m) {
      k_flatten_outlet<<<unsigned((m + 255) / 256), 256>>>(g->out_tab, g->out_eng, g->out_idx,
                                                            int64_t(m), g->fo_slot, g->fo_partner,
                                                            g->fo_cell, g->fo_dir, g->fo_rho,
                                                            g->fo_u);
      slbm::count_launch();
      SLBM_CUDA_TRY(cudaDeviceSynchronize());
    }
  }
  if (g->n_ubb) {
    SLBM_CUDA_TRY(cudaMalloc(&g->ubb_eng, g->n_ubb * sizeof(uint16_t)));
    SLBM_CUDA_TRY(cudaMalloc(&g->ubb_slot, g->n_ubb * sizeof(uint32_t)));
    SLBM_CUDA_TRY(cudaMalloc(&g->ubb_partner, g->n_ubb * sizeof(uint32_t)));
    SLBM_CUDA_TRY(cudaMalloc(&g->ubb_corr, g->n_ubb * sizeof(double)));
    int64_t off = 0;
    for (int i = 0; i < n; ++i) {
      SlbmEngine* e = engines[i];
      if (!e->n_ubb) continue;
      std::vector<uint16_t> ids(e->n_ubb, uint16_t(i));
      SLBM_CUDA_TRY(cudaMemcpy(g->ubb_eng + off, ids.data(), e->n_ubb * 2, cudaMemcpyHostToDevice));
      SLBM_CUDA_TRY(cudaMemcpy(g->ubb_slot + off, e->ubb_slot, e->n_ubb * 4, cudaMemcpyDeviceToDevice));
      SLBM_CUDA_TRY(
          cudaMemcpy(g->ubb_partner + off, e->ubb_partner, e->n_ubb * 4, cudaMemcpyDeviceToDevice));
      SLBM_CUDA_TRY(cudaMemcpy(g->ubb_corr + off, e->ubb_corr, e->n_ubb * 8, cudaMemcpyDeviceToDevice));
      off += e->n_ubb;
    }
  }
  std::vector<unsigned long long*> st(n);
  for (int i = 0; i < n; ++i) st[i] = engines[i]->d_step;
  SLBM_CUDA_TRY(cudaMalloc(&g->steps, n * sizeof(unsigned long long*)));
  SLBM_CUDA_TRY(cudaMemcpy(g->steps, st.data(), n * sizeof(unsigned long long*),
                           cudaMemcpyHostToDevice));
  return SLBM_OK;
}

}  // namespace

extern "C" {

int slbm_group_create(SlbmEngine** engines, int n, SlbmGroup** out) {
  if (!engines || n < 1 || !out) return fail(SLBM_ECONFIG, "group needs engines");
  SlbmEngine* e0 = engines[0];
  for (int i = 0; i < n; ++i) {
    SlbmEngine* e = engines[i];
    if (!e) return fail(SLBM_ECONFIG, "null engine in group");
    if (e->layout != 0) return fail(SLBM_ECONFIG, "block groups hold sparse engines only");
    if (e->q != e0->q || e->model != e0->model || e->pattern != e0->pattern ||
        e->omega != e0->omega || e->lambda_odd != e0->lambda_odd || e->device != e0->device ||
        e->parity != e0->parity || e->has_split != e0->has_split ||
        std::memcmp(e->hr, e0->hr, sizeof(e->hr)) != 0)
      return fail(SLBM_ECONFIG, "group engines must share stencil, collision, pattern, device "
                                "and parity");
  }
  cudaSetDevice(e0->device);
  SlbmGroup* g = new SlbmGroup();
  g->device = e0->device;
  g->q = e0->q;
  g->model = e0->model;
  g->pattern = e0->pattern;
  g->omega = e0->omega;
  g->lam = e0->lambda_odd;
  g->hr = e0->d_hr;
  g->engines.assign(engines, engines + n);
  const int st = init_group(g, engines, n);
  if (st != SLBM_OK) {
    slbm_group_destroy(g);
    return st;
  }
  *out = g;
  return SLBM_OK;
}

// Direct local halo edges for an AA block group (extension of the group
// path; the reference copies every local edge twice a step pair,
// exchange.py:222-253).  Every engine's pdf moves into one pool, and the
// index-list sweeps read a rewritten copy of each engine's list in which a
// ghost slot fed by a local CANONICAL edge (B, s) -> (A, g) addresses B's
// slot s in the pool.  The combined AA step then reads the value the copy
// would have delivered and writes its result where the REVERSED copy would
// have taken it (the REVERSED program is checked to be the exact inverse),
// so both local copies disappear and the results are bit-identical.  Ghost
// slots of local edges are left unmaintained (internal buffers); remote
// edges keep their ghost slots and messages.  The halo's local program is
// switched off.
int slbm_group_link_halo(SlbmGroup* g, SlbmHalo* h) {
  if (!g || !h) return fail(SLBM_ECONFIG, "null group or halo");
  if (g->direct) return SLBM_OK;
  if (g->pattern != SLBM_AA) return fail(SLBM_ECONFIG, "direct local halo edges need the AA pattern");
  cudaSetDevice(g->device);
  const int n = int(g->engines.size());
  std::vector<SlbmEngine*> heng;
  std::vector<uint16_t> cse, cde, rse, rde;
  std::vector<uint32_t> css, cds, rss, rds;
  SLBM_TRY(halo_local_program(h, 0, &heng, &cse, &css, &cde, &cds));
  SLBM_TRY(halo_local_program(h, 1, &heng, &rse, &rss, &rde, &rds));
  if (cse.empty()) return fail(SLBM_ECONFIG, "the halo has no local edges");
  std::vector<int> gid(heng.size(), -1);
  for (size_t k = 0; k < heng.size(); ++k)
    for (int i = 0; i < n; ++i)
      if (heng[k] == g->engines[i]) gid[k] = i;
  auto key = [](uint64_t e, uint64_t slot) { return (e << 32) | slot; };
  std::unordered_map<uint64_t, uint64_t> fwd;  // (A, ghost g) -> (B, source s)
  fwd.reserve(cse.size() * 2);
  for (size_t k = 0; k < cse.size(); ++k) {
    if (gid[cse[k]] < 0 || gid[cde[k]] < 0)
      return fail(SLBM_ECONFIG, "local halo edge with an engine outside the group");
    if (!fwd.emplace(key(gid[cde[k]], cds[k]), key(gid[cse[k]], css[k])).second)
      return fail(SLBM_EPROTOCOL, "ghost slot fed twice");
  }
  if (rse.size() != cse.size()) return fail(SLBM_ECONFIG, "REVERSED local program is not the inverse");
  for (size_t k = 0; k < rse.size(); ++k) {
    if (gid[rse[k]] < 0 || gid[rde[k]] < 0)
      return fail(SLBM_ECONFIG, "local halo edge with an engine outside the group");
    auto it = fwd.find(key(gid[rse[k]], rss[k]));
    if (it == fwd.end() || it->second != key(gid[rde[k]], rds[k]))
      return fail(SLBM_ECONFIG, "REVERSED local program is not the inverse");
  }
  // pool layout: engines back to back, 32-element (256 B) aligned
  std::vector<uint32_t> off(n);
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    if (g->engines[i]->pool) return fail(SLBM_ECONFIG, "engine already pooled");
    off[i] = uint32_t(total);
    total += (g->engines[i]->phys_slots + 31) / 32 * 32;
    if (total >= (int64_t(1) << 32)) return fail(SLBM_ECONFIG, "group pool exceeds 2^32 slots");
  }
  SLBM_CUDA_TRY(cudaDeviceSynchronize());
  double* pool = nullptr;
  std::vector<uint32_t*> gidx(n, nullptr);
  uint32_t *pos = nullptr, *dg = nullptr, *dv = nullptr;
  // on failure everything allocated here is released and the group and its
  // engines are left as they were (the pdf buffers move only at the end)
  auto release = [&]() {
    for (void* p : {(void*)pos, (void*)dg, (void*)dv, (void*)g->save_src, (void*)g->save_dst,
                    (void*)pool})
      if (p) cudaFree(p);
    for (auto* p : gidx)
      if (p) cudaFree(p);
    g->save_src = g->save_dst = nullptr;
    g->n_save = 0;
  };
#define LINK_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      release();                                                                         \
      return fail(SLBM_ECUDA, std::string("slbm_group_link_halo: " #expr ": ") +         \
                                  cudaGetErrorString(_e));                               \
    }                                                                                    \
  } while (0)
  LINK_TRY(cudaMalloc(&pool, size_t(total) * sizeof(double)));
  for (int i = 0; i < n; ++i) {
    SlbmEngine* e = g->engines[i];
    const int64_t entries = int64_t(e->q - 1) * e->idx_pitch;
    LINK_TRY(cudaMalloc(&gidx[i], size_t(entries) * sizeof(uint32_t)));
    if (entries) {
      k_add_offset<<<1024, 256>>>(gidx[i], e->idx, entries, off[i]);
      slbm::count_launch();
    }
  }
  // the CANONICAL program in pool offsets (saving the stale source values)
  {
    std::vector<uint32_t> ss_(cse.size()), dd_(cse.size());
    for (size_t k = 0; k < cse.size(); ++k) {
      ss_[k] = off[gid[cse[k]]] + css[k];
      dd_[k] = off[gid[cde[k]]] + cds[k];
    }
    LINK_TRY(cudaMalloc(&g->save_src, ss_.size() * 4));
    LINK_TRY(cudaMalloc(&g->save_dst, dd_.size() * 4));
    LINK_TRY(cudaMemcpy(g->save_src, ss_.data(), ss_.size() * 4, cudaMemcpyHostToDevice));
    LINK_TRY(cudaMemcpy(g->save_dst, dd_.data(), dd_.size() * 4, cudaMemcpyHostToDevice));
    g->n_save = int64_t(ss_.size());
  }
  // rewrite the ghost entries of local edges, per destination engine
  std::vector<std::vector<uint32_t>> ghost(n), val(n);
  for (size_t k = 0; k < cse.size(); ++k) {
    const int a = gid[cde[k]], b = gid[cse[k]];
    ghost[a].push_back(cds[k]);
    val[a].push_back(off[b] + css[k]);
  }
  for (int i = 0; i < n; ++i) {
    if (ghost[i].empty()) continue;
    SlbmEngine* e = g->engines[i];
    const size_t m = ghost[i].size();
    LINK_TRY(cudaMalloc(&pos, size_t(e->phys_slots) * sizeof(uint32_t)));
    LINK_TRY(cudaMemset(pos, 0xFF, size_t(e->phys_slots) * sizeof(uint32_t)));
    k_slot_pos<<<1024, 256>>>(pos, e->idx, uint32_t(e->idx_pitch), uint32_t(e->n_fluid), e->q - 1,
                              (e->q == 19) ? 1 : 0);
    slbm::count_launch();
    LINK_TRY(cudaMalloc(&dg, m * sizeof(uint32_t)));
    LINK_TRY(cudaMalloc(&dv, m * sizeof(uint32_t)));
    LINK_TRY(cudaMemcpy(dg, ghost[i].data(), m * 4, cudaMemcpyHostToDevice));
    LINK_TRY(cudaMemcpy(dv, val[i].data(), m * 4, cudaMemcpyHostToDevice));
    k_rewrite<<<unsigned((m + 255) / 256), 256>>>(gidx[i], pos, dg, dv, int64_t(m));
    slbm::count_launch();
    LINK_TRY(cudaDeviceSynchronize());
    for (uint32_t** p : {&pos, &dg, &dv}) {
      cudaFree(*p);
      *p = nullptr;
    }
  }
  // copy every engine's pdf into the pool; the engines switch to it only
  // once all copies have succeeded
  for (int i = 0; i < n; ++i)
    LINK_TRY(cudaMemcpy(pool + off[i], g->engines[i]->pdf,
                        size_t(g->engines[i]->phys_slots) * sizeof(double),
                        cudaMemcpyDeviceToDevice));
  LINK_TRY(cudaGetLastError());
  LINK_TRY(cudaDeviceSynchronize());
#undef LINK_TRY
  PdfPool* ref = new PdfPool{pool, 0};
  for (int i = 0; i < n; ++i) {
    SlbmEngine* e = g->engines[i];
    cudaFree(e->pdf);
    e->pdf = pool + off[i];
    e->pool = ref;
    ++ref->refs;
    for (auto& gx : e->graph) {  // captured with the old buffer
      if (gx) cudaGraphExecDestroy(gx);
      gx = nullptr;
    }
  }
  g->direct = true;
  g->pool = pool;
  g->pool_off = off;
  g->gidx = gidx;
  halo_disable_local(h);
  SLBM_TRY(build_tables(g));
  SLBM_CUDA_TRY(cudaDeviceSynchronize());
  return SLBM_OK;
}

// the local edges' (source slot, ghost slot) pairs of a linked group, on
// `stream`: mode 0 ghost <- source, 1 swap, 2 source <- ghost
int slbm_group_stale_copy(SlbmGroup* g, int mode, void* stream) {
  if (!g) return fail(SLBM_ECONFIG, "null group");
  if (mode < 0 || mode > 2) return fail(SLBM_ECONFIG, "stale copy mode 0, 1 or 2");
  if (!g->direct || !g->n_save) return SLBM_OK;
  cudaSetDevice(g->device);
  { k_pool_copy<<<unsigned((g->n_save + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        g->pool, g->save_src, g->save_dst, g->n_save, mode); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int slbm_group_destroy(SlbmGroup* g) {
  if (!g) return SLBM_OK;
  cudaSetDevice(g->device);
  for (int p = 0; p < 3; ++p) {
    for (int f = 0; f < 2; ++f)
      if (g->table[p][f]) cudaFree(g->table[p][f]);
    if (g->cta_start[p]) cudaFree(g->cta_start[p]);
    if (g->cta_start_odd[p]) cudaFree(g->cta_start_odd[p]);
  }
  for (int p = 0; p < 3; ++p)
    for (int f = 0; f < 2; ++f) {
      delete g->hot16[p][f];
      delete g->hot128[p][f];
      delete g->hot512[p][f];
    }
  for (auto* p : g->gidx)
    if (p) cudaFree(p);
  if (g->save_src) cudaFree(g->save_src);
  if (g->save_dst) cudaFree(g->save_dst);
  for (int f = 0; f < 2; ++f) {
    delete g->bhot16[f];
    delete g->bhot128[f];
  }
  for (void* p : {(void*)g->fo_slot, (void*)g->fo_partner, (void*)g->fo_cell, (void*)g->fo_dir,
                  (void*)g->fo_rho, (void*)g->fo_u})
    if (p) cudaFree(p);
  void* ptrs[] = {g->ubb_eng, g->ubb_slot, g->ubb_partner, g->ubb_corr, g->steps,
                  g->out_tab, g->out_eng, g->out_idx};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete g;
  return SLBM_OK;
}

int group_boundary(SlbmGroup* g, SlbmHalo* halo, int phase, int parity, cudaStream_t s) {
  PdfTable lt{};
  LocalEdges le{};
  if (halo) SLBM_TRY(halo_local_edges(halo, phase, &lt, &le));
  const int flip = g->pattern == SLBM_PULL ? g->flip : 0;
  const int n = int(g->engines.size());
  constexpr int64_t kPer = kBT * kBItems;
  const uint32_t cta_halo = uint32_t((le.n + kPer - 1) / kPer);
  const uint32_t cta_ubb = uint32_t((g->n_ubb + kPer - 1) / kPer);
  const uint32_t cta_out = uint32_t((g->n_out + kBT - 1) / kBT);
  const uint32_t grid = std::max(1u, cta_halo + cta_ubb + cta_out);
  cudaError_t err = cudaSuccess;
  auto go = [&](const auto& lk) {
    using LK = std::decay_t<decltype(lk)>;
    on_lattice(g->q, [&](auto lat) {
      using L = decltype(lat);
      err = launch_pdl(k_group_boundary<L, LK>, dim3(grid), dim3(kBT), 0, s, lk, lt, le,
                       g->ubb_eng, g->ubb_slot, g->ubb_partner, g->ubb_corr, g->n_ubb, g->out_eng,
                       g->fo_slot, g->fo_partner, g->fo_cell, g->fo_dir, g->fo_rho, g->fo_u,
                       g->n_out, g->steps, n, parity, cta_halo, cta_ubb);
    });
  };
  if (g->bhot16[flip])
    go(*g->bhot16[flip]);
  else if (g->bhot128[flip])
    go(*g->bhot128[flip]);
  else
    go(BoundaryTable{g->table[0][flip]});
  SLBM_CUDA_TRY(err);
  return SLBM_OK;
}

// refresh_boundary of every engine (sparse.py:295-304) + the step counters,
// one launch on `stream` (k_group_boundary without halo edges)
int slbm_group_refresh(SlbmGroup* g, int parity, void* stream) {
  if (!g) return fail(SLBM_ECONFIG, "null group");
  return group_boundary(g, nullptr, 0, parity, (cudaStream_t)stream);
}

// ... and the device-local halo edges of `phase` of `halo` in the same launch
int slbm_group_boundary(SlbmGroup* g, SlbmHalo* halo, int phase, int parity, void* stream) {
  if (!g) return fail(SLBM_ECONFIG, "null group");
  return group_boundary(g, halo, phase, parity, (cudaStream_t)stream);
}

// one sweep of `phase` over every engine of the group, one launch
int slbm_group_step(SlbmGroup* g, int phase, void* stream) {
  if (!g) return fail(SLBM_ECONFIG, "null group");
  if (phase < 0 || phase > 2 || !g->cta_start[phase])
    return fail(SLBM_ECONFIG, "sweep needs split lists; build with frame_width");
  if (!g->n_cta[phase]) return SLBM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int parity = g->engines[0]->parity;
  const int kind = g->pattern == SLBM_PULL ? 0 : (parity == SLBM_EVEN ? 1 : 2);
  const int flip = g->pattern == SLBM_PULL ? g->flip : 0;
  const GroupArgs* tab = g->table[phase][flip];
  const int n = int(g->engines.size());
  cudaError_t err = cudaSuccess;
  on_lattice(g->q, [&](auto lat) {
    using L = decltype(lat);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t ahead = uint32_t(sms);  // one quarter wave at 4 CTAs/SM
    auto go = [&](auto mc) {
      constexpr int M = decltype(mc)::value;
      auto hot = [&](auto* gh) -> bool {  // kernel-parameter block table
        if (!gh || kind == 2) return false;
        constexpr int CAP = int(sizeof(gh->hot) / sizeof(HotArgs));
        if (kind == 0)
          err = launch_pdl(k_group_hot<L, M, 0, CAP>, dim3(g->n_cta[phase]), dim3(kGB), 0, s, *gh,
                           tab, n, g->omega, g->lam, g->hr, ahead);
        else
          err = launch_pdl(k_group_hot<L, M, 1, CAP>, dim3(g->n_cta[phase]), dim3(kGB), 0, s, *gh,
                           tab, n, g->omega, g->lam, g->hr, ahead);
        return true;
      };
      if (hot(g->hot16[phase][flip]) || hot(g->hot128[phase][flip]) ||
          hot(g->hot512[phase][flip]))
        return;
      if (kind == 0)
        err = launch_pdl(k_group<L, M, 0>, dim3(g->n_cta[phase]), dim3(kGB), 0, s, tab,
                         g->cta_start[phase], n, g->omega, g->lam, g->hr, ahead);
      else if (kind == 1)
        err = launch_pdl(k_group<L, M, 1>, dim3(g->n_cta[phase]), dim3(kGB), 0, s, tab,
                         g->cta_start[phase], n, g->omega, g->lam, g->hr, ahead);
      else
        err = launch_pdl(k_group<L, M, 2>, dim3(g->n_cta_odd[phase]), dim3(kGB), 0, s, tab,
                         g->cta_start_odd[phase], n, g->omega, g->lam, g->hr, ahead);
    };
    if (g->model == SLBM_SRT)
      go(std::integral_constant<int, SLBM_SRT>{});
    else if (g->model == SLBM_TRT)
      go(std::integral_constant<int, SLBM_TRT>{});
    else if constexpr (L::Q == 27) {
      if (g->model == SLBM_CUMULANT)
        go(std::integral_constant<int, SLBM_CUMULANT>{});
      else
        go(std::integral_constant<int, SLBM_CUMULANT_GEN>{});
    }
  });
  SLBM_CUDA_TRY(err);
  return SLBM_OK;
}

// finish_step of every engine (sparse.py:243-249): host state flips; the
// device step counters advance in the next step's boundary kernel
int slbm_group_finish(SlbmGroup* g, void* stream) {
  if (!g) return fail(SLBM_ECONFIG, "null group");
  for (SlbmEngine* e : g->engines) {
    if (e->pattern == SLBM_PULL)
      std::swap(e->pdf, e->tmp);
    else
      e->parity = 1 - e->parity;
    e->steps_done += 1;
  }
  if (g->pattern == SLBM_PULL) g->flip ^= 1;
  (void)stream;
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

}  // extern "C"
