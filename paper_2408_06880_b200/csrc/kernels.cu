// Stream-collide sweeps and the small per-step kernels.
//
// One thread per fluid cell; each thread owns a disjoint slot set (the
// builder's uniqueness check, sparse.py:182-185), so the in-place AA
// scatter needs no synchronisation and any cell subset (interior / frame)
// composes bitwise with the whole-block sweep.
//
//   k_index_sweep<kEven>  combined pull-collide-push step  sparse.py:264-271
//              t0 = pdf[c], t_q = pdf[idx[q-1][c]];  collide;
//              pdf[c] = out0, pdf[idx[q-1][c]] = out[inv q]
//              traffic 19x8 R + 19x8 W + 18x4 idx = 376 B/cell (D3Q19)
//   k_aa_odd   cell-local reversed step                  sparse.py:273-282
//              t_r = pdf[base[inv r] + c]; pdf[base[r] + c] = out_r
//              304 B/cell, every access coalesced
//   k_index_sweep<kPull>  two-buffer pull                 sparse.py:257-262
//              gather as the even step, dst[base[r] + c] = out_r; 376 B/cell
// base[] / idx hold device addresses (256-B aligned groups, engine.cuh).
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>

#include "collide.cuh"
#include "engine.cuh"
#include "sweep.cuh"

namespace slbm {

namespace cg = cooperative_groups;

struct SweepArgs {
  double* pdf;
  double* dst;
  const uint32_t* idx;
  const uint32_t* cids;  // nullptr: cell = offset + position
  const uint32_t* skip;  // identity sweep minus the cells whose bit is set (interior)
  uint32_t offset;       // first cell of an identity sweep (contiguous interior),
                         // rounded down to a warp boundary; cells below `lo` are skipped
  uint32_t lo;
  uint32_t n_cells;
  uint32_t n_fluid;
  uint32_t idx_pitch;  // elements per index-list row (256-B aligned rows)
  uint32_t base[28];   // device group starts (SlbmEngine::pbase)
  double omega, lam;
  const double* hr;  // cumulant: higher-order rates w3..w10 (device)
  unsigned long long* bad;
  const unsigned long long* step;
};

namespace {

constexpr int kBlock = 256;  // small kernels and the odd sweep
constexpr int kIB = 128;     // index-list sweeps: 128-thread CTAs, 4 per SM

__device__ __forceinline__ void flag_bad(const SweepArgs& a) {
  atomicMin(a.bad, *a.step);
}

int g_num_sms = 0;

enum Kind { kPull = 0, kEven = 1, kOdd = 2 };

// Index-list sweep: AA even (combined pull-collide-push, sparse.py:264-271)
// or pull (sparse.py:257-262).  One thread per cell; the Q-1 slot ids stay
// in registers through the collision so the even step scatters through the
// same slots it gathered from (opposite directions).
//
// Kernel-variant study (tools/variants.py, profiles/r01_variants_*.log):
// 256x2 vs 128x4 CTAs (+2% for 128x4); register caps 80/64 (spills, -10..-40%);
// re-reading idx before each store (RELOAD); cp.async gather into shared
// memory; persistent CTAs with a cp.async idx double buffer; a cell-major
// idx copy; ld.global.nc / L1::no_allocate PDF gathers (-40%: the gathers
// want L1 sector merging); st.global.cs stores (-4%); 5 or 6 CTAs/SM (94 /
// 80 + spill registers: -1% / -10%); __ldg gathers (same); L1::no_allocate,
// L1::evict_first or __ldlu gathers (-40%: evicting the line the thread is
// about to overwrite in place costs the store); a compressed index list
// (16-bit deltas against a per-32-cell base, escapes for folds/halo: 342
// instead of 376 B/cell, -4% burst / -2.5% sustained: more load
// instructions than bytes saved); FMA contraction (no change under the
// power cap, which costs the sweep ~6% of SM clock); round 2: the gather
// straight into shared memory (cp.async, one-pass moments from the staged
// column) at 6 CTAs/SM, 78-80 registers (bed 0.86 vs 0.97, C5 phi 0.3 0.81
// vs 0.82) or 8 CTAs/SM with spills (0.72 / 0.68) — all slower than the
// plain gather.  What pays is the L2 prefetch of the index list one quarter
// wave ahead (sweep.cuh): +7-9%.
template <class L, int MODEL, int KIND, int MINB, bool PF>
__global__ void __launch_bounds__(kIB, MINB) k_index_sweep(const SweepArgs a, uint32_t ahead) {
  const uint32_t first = blockIdx.x * kIB;
  if constexpr (PF) {
    if (a.cids == nullptr)
      prefetch_idx_ahead<L::Q - 1, kIB>(a.idx, a.idx_pitch, nullptr, a.offset + a.n_cells,
                                        a.offset + first, ahead);
  }
  const uint32_t i = first + threadIdx.x;
  if (i >= a.n_cells) return;
  const uint32_t c = a.cids ? a.cids[i] : a.offset + i;
  if (c < a.lo) return;
  uint32_t s[L::Q];
  double t[L::Q];
  // the skip word (interior sweep) is loaded alongside the index list, not
  // in front of it: a frame cell reads its idx row for nothing (~1% extra)
  // but no cell waits for the mask before its own loads start
  const uint32_t skip_word = a.skip ? __ldg(a.skip + (c >> 5)) : 0u;
  load_slots<L>(s, a.idx, a.idx_pitch, c);
  if ((skip_word >> (c & 31)) & 1u) return;
  gather<L>(t, a.pdf, s);
  if constexpr (PF) {
    if (a.cids != nullptr)
      prefetch_idx_ahead<L::Q - 1, kIB>(a.idx, a.idx_pitch, a.cids, a.n_cells, first, ahead);
  }
  if (collide_scatter<L, MODEL, KIND == kEven>(t, s, a.pdf, a.dst, a.base, c, a.omega, a.lam, a.hr))
    flag_bad(a);
}

// Memory-pattern probe (tuning only; does NOT compute LBM): the even sweep's
// gather + scatter through the same slots without the collision — the
// bandwidth ceiling of the access pattern itself.
template <class L>
__global__ void __launch_bounds__(kIB) k_probe(const SweepArgs a) {
  const uint32_t i = blockIdx.x * kIB + threadIdx.x;
  if (i >= a.n_cells) return;
  const uint32_t c = i;
  uint32_t s[L::Q];
  double t[L::Q];
  load_slots<L>(s, a.idx, a.idx_pitch, c);
  sfor<0, L::Q>([&](auto q) { t[q] = a.pdf[s[q]]; });
  sfor<0, L::Q>([&](auto q) { a.pdf[s[L::INV[q]]] = t[q]; });
}

// AA odd (cell-local reversed step, sparse.py:273-282): every access is a
// coalesced row of a direction group, no index list.
template <class L, int MODEL, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) k_aa_odd(const SweepArgs a) {
  // CTAs run from the last cells to the first: the index-list sweep before
  // ran first to last, so this sweep starts on the lines it left in L2, and
  // the next index-list sweep starts on the lines this one leaves
  const uint32_t i = (gridDim.x - 1 - blockIdx.x) * kBlock + threadIdx.x;
  if (i >= a.n_cells) return;
  const uint32_t c = a.cids ? a.cids[i] : a.offset + i;
  if (c < a.lo || (a.skip && ((__ldg(a.skip + (c >> 5)) >> (c & 31)) & 1u))) return;
  if (cell_local<L, MODEL>(a.pdf, a.base, c, a.omega, a.lam, a.hr)) flag_bad(a);
}

int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

template <class L, int MODEL, int KIND, int MINB, bool PF>
void launch_index(const SweepArgs& a, const SlbmTuning& t, cudaStream_t s) {
  static int resident = 0;  // CTAs per SM this instantiation actually gets
  if (!resident) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_index_sweep<L, MODEL, KIND, MINB, PF>,
                                                  kIB, 0);
    resident = std::max(resident, 1);
  }
  const uint32_t ahead = t.ahead_ctas > 0 ? uint32_t(t.ahead_ctas)
                                          : uint32_t(num_sms() * resident * t.ahead_quarters / 4);
  { k_index_sweep<L, MODEL, KIND, MINB, PF>
      <<<(a.n_cells + kIB - 1) / kIB, kIB, 0, s>>>(a, std::max(ahead, 1u)); slbm::count_launch(); }
}

template <class L, int MODEL>
void launch_kind(int kind, const SweepArgs& a, unsigned grid, const SlbmTuning& t, cudaStream_t s) {
  constexpr int MINB = L::Q == 9 ? 8 : 4;
  // D3Q19 index-list sweeps at 5 CTAs/SM (94 registers, no spills): more
  // gathers in flight pays on scattered geometries (C5 random obstacles
  // phi 0.3: 0.83 -> 0.86 of HBM) and costs on coherent ones (sphere bed
  // 0.97 -> 0.94); chosen per engine by measurement (sweep_ctas)
  constexpr bool kFive = L::Q == 19;
  const bool five = kFive && t.even_ctas == 5;
  if (kind == kPull) {
    if constexpr (kFive) {
      if (five) return launch_index<L, MODEL, kPull, 5, true>(a, t, s);
    }
    launch_index<L, MODEL, kPull, MINB, true>(a, t, s);
  } else if (kind == kEven) {
    if (t.even_variant == 1)
      launch_index<L, MODEL, kEven, MINB, false>(a, t, s);
#ifdef SLBM_PROBES
    else if (t.even_variant == 2)  // memory-pattern probe, not LBM
      { k_probe<L><<<(a.n_cells + kIB - 1) / kIB, kIB, 0, s>>>(a); slbm::count_launch(); }
#endif
    else if constexpr (kFive) {
      if (five)
        launch_index<L, MODEL, kEven, 5, true>(a, t, s);
      else
        launch_index<L, MODEL, kEven, MINB, true>(a, t, s);
    } else
      launch_index<L, MODEL, kEven, MINB, true>(a, t, s);
  } else {
    if (L::Q != 9 && t.odd_variant == 2)
      { k_aa_odd<L, MODEL, 4><<<grid, kBlock, 0, s>>>(a); slbm::count_launch(); }
    else
      { k_aa_odd<L, MODEL, L::Q == 9 ? 1 : 3><<<grid, kBlock, 0, s>>>(a); slbm::count_launch(); }
  }
}

template <class L>
void launch_model(int model, int kind, const SweepArgs& a, unsigned grid, const SlbmTuning& t,
                  cudaStream_t s) {
  if (model == SLBM_SRT)
    launch_kind<L, SLBM_SRT>(kind, a, grid, t, s);
  else if (model == SLBM_TRT)
    launch_kind<L, SLBM_TRT>(kind, a, grid, t, s);
  else if constexpr (L::Q == 27) {
    if (model == SLBM_CUMULANT)
      launch_kind<L, SLBM_CUMULANT>(kind, a, grid, t, s);
    else
      launch_kind<L, SLBM_CUMULANT_GEN>(kind, a, grid, t, s);
  }
}

__global__ void k_refresh(double* pdf, const uint32_t* slot, const uint32_t* partner,
                          const double* corr, uint32_t n, int parity) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // sparse.py:301-304
  if (parity == SLBM_EVEN)
    pdf[slot[i]] = pdf[partner[i]] + corr[i];
  else
    pdf[partner[i]] = pdf[slot[i]] + corr[i];
}

__global__ void k_advance(unsigned long long* step) { *step += 1; }

// Resident multi-step kernel for small engines (slbm_run, n_fluid <= the
// knob-4 cap): one cooperative launch runs n whole steps — refresh, outlet,
// sweep per step, a grid barrier between phases — instead of 2-3 launches
// per step.  A block whose lists fit in L2 sweeps in ~2 us, so the per-step
// launch latency (refresh + sweep + step counter ≈ 9 us in a graph, C1) was
// the cost.  Same per-cell bodies and phase order as sweep_once, hence
// bitwise identical; cells are strided over the resident threads.
struct ResidentArgs {
  const uint32_t* ubb_slot;
  const uint32_t* ubb_partner;
  const double* ubb_corr;
  uint32_t n_ubb;
  const uint32_t* out_slot;
  const uint32_t* out_partner;
  const uint32_t* out_cell;
  const uint8_t* out_dir;
  const double* out_rho;
  double* out_u;
  uint32_t n_out;
  uint32_t steps;
  int parity;  // AA parity of the first step
  int pull;
};

template <class L, int MODEL, int MINB>
__global__ void __launch_bounds__(kIB, MINB) k_resident(const SweepArgs a, const ResidentArgs r) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t tid = blockIdx.x * kIB + threadIdx.x;
  const uint32_t nth = gridDim.x * kIB;
  const unsigned long long step0 = *a.step;
  double* cur = a.pdf;
  double* oth = a.dst;
  int parity = r.parity;
  for (uint32_t k = 0; k < r.steps; ++k) {
    if (r.n_ubb) {  // sparse.py:301-304, as k_refresh
      for (uint32_t i = tid; i < r.n_ubb; i += nth) {
        if (parity == SLBM_EVEN)
          cur[r.ubb_slot[i]] = cur[r.ubb_partner[i]] + r.ubb_corr[i];
        else
          cur[r.ubb_partner[i]] = cur[r.ubb_slot[i]] + r.ubb_corr[i];
      }
      grid.sync();
    }
    if (r.n_out) {
      for (uint32_t i = tid; i < r.n_out; i += nth)
        outlet_entry<L>(cur, a.base, r.out_slot[i], r.out_partner[i], r.out_cell[i], r.out_dir[i],
                        r.out_rho[i], r.out_u + 3 * i, parity);
      grid.sync();
    }
    bool bad = false;
    if (r.pull || parity == SLBM_EVEN) {
      for (uint32_t c = tid; c < a.n_fluid; c += nth) {
        uint32_t s[L::Q];
        double t[L::Q];
        // idx rows of this warp's next cells into L2 (as the sweep kernels do)
        const uint32_t lane = threadIdx.x & 31, nxt = c - lane + nth;
        if (nxt < a.n_fluid) prefetch_idx_warp<L::Q - 1>(a.idx, a.idx_pitch, nxt, lane);
        load_slots<L>(s, a.idx, a.idx_pitch, c);
        gather<L>(t, cur, s);
        bad |= r.pull ? collide_scatter<L, MODEL, false>(t, s, cur, oth, a.base, c, a.omega, a.lam, a.hr)
                      : collide_scatter<L, MODEL, true>(t, s, cur, oth, a.base, c, a.omega, a.lam, a.hr);
      }
    } else {
      for (uint32_t c = tid; c < a.n_fluid; c += nth)
        bad |= cell_local<L, MODEL>(cur, a.base, c, a.omega, a.lam, a.hr);
    }
    if (bad) atomicMin(a.bad, step0 + k);
    grid.sync();
    if (r.pull) {
      double* t = cur;
      cur = oth;
      oth = t;
    } else {
      parity = 1 - parity;
    }
  }
  if (tid == 0) *const_cast<unsigned long long*>(a.step) = step0 + r.steps;
}

// Fixed-density outlet (extension; the reference has none):
// outlet_entry (sweep.cuh) per appended outlet slot.
template <class L>
__global__ void k_outlet(double* pdf, SweepArgs a, const uint32_t* slot, const uint32_t* partner,
                         const uint32_t* cell, const uint8_t* dir, const double* rho_o,
                         double* u_store, uint32_t n, int parity) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  outlet_entry<L>(pdf, a.base, slot[i], partner[i], cell[i], dir[i], rho_o[i], u_store + 3 * i,
                  parity);
}

// canonical (q, n) values per cell straight from the groups (sparse.py:308-321)
// out: gx == 0 -> the block's own box (or compact with x_flat == nullptr);
// gx > 0 -> a global box of row length gx, gy rows per plane, the block at
// origin (ox, oy, oz) (Domain.gather_macroscopics on the device)
struct MacroOut {
  int64_t gx = 0, gy = 0, ox = 0, oy = 0, oz = 0;
};

template <class L>
__global__ void k_macro(const double* pdf, SweepArgs a, int odd, Geometry g,
                        const uint32_t* x_flat, double* rho_f, double* u_f, int* bad,
                        MacroOut o) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.n_fluid) return;
  double t[L::Q];
  sfor<0, L::Q>([&](auto q) {
    constexpr int qb = L::INV[q];
    t[q] = pdf[a.base[odd ? qb : int(q)] + c];
  });
  const Moments<L> m = moments<L>(t);
  if (m.bad) atomicOr(bad, 1);
  int64_t f = c;  // compact output (one value per fluid cell) without x_flat
  if (x_flat) {
    int64_t x, y, z;
    g.coords(x_flat[c], x, y, z);
    f = o.gx ? ((z + o.oz) * o.gy + (y + o.oy)) * o.gx + (x + o.ox) : g.interior_flat(x, y, z);
  }
  rho_f[f] = m.rho;
  u_f[f * L::DIM + 0] = m.ux;
  u_f[f * L::DIM + 1] = m.uy;
  if constexpr (L::DIM == 3) u_f[f * L::DIM + 2] = m.uz;
}

// One thread per box cell (x fastest); cells that are not fluid (cid_map <
// 0) get zeros (sparse.py:323-331).  The interleaved u is transposed
// through shared memory so every warp store is one contiguous 256-B run of
// host memory — PCIe writes from SMs only stream at full width when
// coalesced.
constexpr int kMacroBlock = 256;

template <class L>
__global__ void __launch_bounds__(kMacroBlock) k_macro_box(const double* pdf, SweepArgs a, int odd,
                                                           Geometry g, const int32_t* cid_map,
                                                           double* rho_h, double* u_h, int* bad) {
  __shared__ double su[kMacroBlock * L::DIM];
  const int64_t cells = g.n_cells();
  const int64_t f0 = int64_t(blockIdx.x) * kMacroBlock;
  const int64_t f = f0 + threadIdx.x;
  double rho = 0.0, uv[3] = {0.0, 0.0, 0.0};
  if (f < cells) {
    const int64_t x = f % g.n[0];
    const int64_t r = f / g.n[0];
    const int64_t y = r % g.n[1];
    const int64_t z = r / g.n[1];
    const int32_t c = cid_map[g.padded_flat(x, y, z)];
    if (c >= 0) {
      double t[L::Q];
      sfor<0, L::Q>([&](auto q) {
        constexpr int qb = L::INV[q];
        t[q] = pdf[a.base[odd ? qb : int(q)] + uint32_t(c)];
      });
      const Moments<L> m = moments<L>(t);
      if (m.bad) atomicOr(bad, 1);
      rho = m.rho;
      uv[0] = m.ux;
      uv[1] = m.uy;
      uv[2] = m.uz;
    }
    rho_h[f] = rho;
  }
  for (int k = 0; k < L::DIM; ++k) su[threadIdx.x * L::DIM + k] = uv[k];
  __syncthreads();
  const int64_t n_here = std::min<int64_t>(kMacroBlock, cells - f0) * L::DIM;
  for (int k = threadIdx.x; k < n_here; k += kMacroBlock) u_h[f0 * L::DIM + k] = su[k];
}

template <class L>
__global__ void k_equilibrium(double* pdf, SweepArgs a, const double* rho, int rho_scalar,
                              const double* u, int u_scalar) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.n_fluid) return;
  const size_t n = a.n_fluid;
  // core.py:127-146 with the same usq accumulation order
  Moments<L> m;
  m.rho = rho[rho_scalar ? 0 : c];
  m.ux = u_scalar ? u[0] : u[c];
  m.uy = u_scalar ? u[1] : u[n + c];
  m.uz = (L::DIM == 3) ? (u_scalar ? u[2] : u[2 * n + c]) : 0.0;
  double usq = m.ux * m.ux;
  usq = usq + m.uy * m.uy;
  if constexpr (L::DIM == 3) usq = usq + m.uz * m.uz;
  m.usq = usq;
  m.bad = false;
  sfor<0, L::Q>([&](auto q) { pdf[a.base[q] + c] = feq<L, q>(m); });
}

__global__ void k_gather(const double* src, const uint32_t* slots, int64_t n, double* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[slots[i]];
}

__global__ void k_scatter(double* dst, const uint32_t* slots, int64_t n, const double* in) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[slots[i]] = in[i];
}

__global__ void k_fill(double* p, int64_t n, double v) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void k_slot_lookup(const int64_t* qs, const int64_t* pflat, int64_t n,
                              const int32_t* cid_map, int64_t n_pad, SweepArgs a, int q_max,
                              int64_t* out, int* err) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t q = qs[i], p = pflat[i];
  if (q < 0 || q >= q_max || p < 0 || p >= n_pad) {
    atomicOr(err, 1);
    return;
  }
  const int32_t cid = cid_map[p];
  if (cid < 0) {
    atomicOr(err, 1);
    return;
  }
  out[i] = int64_t(a.base[q]) + cid;
}

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  return unsigned(g > 0 ? g : 1);
}

SweepArgs sweep_args(SlbmEngine* e) {
  SweepArgs a{};
  a.pdf = e->pdf;
  a.dst = e->tmp;
  a.idx = e->idx;
  a.cids = nullptr;
  a.n_fluid = uint32_t(e->n_fluid);
  a.n_cells = uint32_t(e->n_fluid);
  a.idx_pitch = uint32_t(e->idx_pitch);
  for (int q = 0; q <= e->q && q < 28; ++q) a.base[q] = uint32_t(e->pbase[q]);
  a.omega = e->omega;
  a.lam = e->lambda_odd;
  a.hr = e->d_hr;
  a.bad = e->d_bad;
  a.step = e->d_step;
  return a;
}

template <class F>
void by_lattice(int q, F&& f) {
  if (q == 9)
    f(LatD2Q9{});
  else if (q == 19)
    f(LatD3Q19{});
  else
    f(LatD3Q27{});
}

}  // namespace

SlbmTuning g_tuning_defaults{};

int tuning_apply(SlbmTuning& t, int knob, int value) {
  switch (knob) {
    case 0:
#ifndef SLBM_PROBES
      if (value == 2) return fail(SLBM_ECONFIG, "knob 0 = 2 (memory probe) needs an SLBM_PROBES build");
#endif
      if (value < 0 || value > 2) return fail(SLBM_ECONFIG, "knob 0: variant 0, 1 or 2");
      t.even_variant = value;
      return SLBM_OK;
    case 1: t.odd_variant = value; return SLBM_OK;
    case 2:
      if (value < 0) return fail(SLBM_ECONFIG, "knob 2: distance >= 0");
      t.ahead_quarters = value;
      return SLBM_OK;
    case 3: t.ahead_ctas = value; return SLBM_OK;
    case 4: t.resident_cap = value; return SLBM_OK;
    case 5: case 6: case 7: case 8:
#ifndef SLBM_WITH_PAIR
      if (knob == 5 && value != 0)
        return fail(SLBM_ECONFIG, "the pair kernel is experimental: build with SLBM_EXPERIMENTAL_PAIR=1");
#endif
      (knob == 5 ? t.pair : knob == 6 ? t.pair_slack : knob == 7 ? t.pair_ahead : t.pair_hints) = value;
      return SLBM_OK;
    case 9: t.dense_lean_odd = value; return SLBM_OK;
    case 13:
      if (value != 0 && value != 4 && value != 5)
        return fail(SLBM_ECONFIG, "knob 13: 0 (measure), 4 or 5 CTAs per SM");
      t.even_ctas = value;
      return SLBM_OK;
    default: return fail(SLBM_ECONFIG, "unknown engine tuning knob " + std::to_string(knob));
  }
}

int set_tuning(int knob, int value) {
  if ((knob >= 0 && knob <= 9) || knob == 13) return tuning_apply(g_tuning_defaults, knob, value);
  if (knob == 10 || knob == 11 || knob == 12) return hostcopy_tune(knob, value);
  return fail(SLBM_ECONFIG, "unknown tuning knob " + std::to_string(knob));
}

int launch_slot_lookup(SlbmEngine* e, const int64_t* d_qs, const int64_t* d_pflat, int64_t n,
                       int64_t* d_out, int* d_err) {
  if (n == 0) return SLBM_OK;
  SweepArgs a = sweep_args(e);  // slot ids: the reference's layout, not the device one
  for (int q = 0; q <= e->q && q < 28; ++q) a.base[q] = uint32_t(e->base[q]);
  { k_slot_lookup<<<grid_for(n, 256), 256, 0, e->stream>>>(d_qs, d_pflat, n, e->cid_map,
                                                          e->geo.n_padded(), a, e->q, d_out,
                                                          d_err); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

// Occupancy of a D3Q19 engine's whole-block index-list sweep: the knob
// (tune.even_ctas 4 / 5) or, by default for blocks of >= 2^22 fluid cells,
// measured on the engine's own sweeps -- the first sweep warms up at 4
// CTAs/SM, the next four alternate 5, 4, 5, 4 between CUDA events, and the
// sixth compares the faster trial of each and keeps 5 only if it was
// >= 1.5 % faster.  Results are the same bits either way; during a stream
// capture an undecided engine uses 4.  *trial = the event pair to record
// around this launch, or -1.
int sweep_ctas(SlbmEngine* e, int* trial) {
  *trial = -1;
  if (e->q != 19 || e->tune.even_variant != 0) return 4;
  if (e->tune.even_ctas == 4 || e->tune.even_ctas == 5) return e->tune.even_ctas;
  if (e->even_ctas) return e->even_ctas;
  if (e->n_fluid < (int64_t(1) << 22)) return e->even_ctas = 4;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(e->stream, &cap);
  if (cap != cudaStreamCaptureStatusNone) return 4;
  const int k = e->even_trials++;
  if (k == 0) return 4;
  if (k <= 4) {
    for (auto& ev : e->even_ev)
      if (!ev && cudaEventCreate(&ev) != cudaSuccess) return e->even_ctas = 4;
    *trial = k - 1;
    return (k & 1) ? 5 : 4;
  }
  float t[4] = {0.f, 0.f, 0.f, 0.f};
  bool ok = cudaEventSynchronize(e->even_ev[7]) == cudaSuccess;
  for (int i = 0; i < 4 && ok; ++i)
    ok = cudaEventElapsedTime(&t[i], e->even_ev[2 * i], e->even_ev[2 * i + 1]) == cudaSuccess;
  const int pick = ok && std::min(t[0], t[2]) < 0.985f * std::min(t[1], t[3]) ? 5 : 4;
  for (auto& ev : e->even_ev) {
    if (ev) cudaEventDestroy(ev);
    ev = nullptr;
  }
  return e->even_ctas = pick;
}

int launch_step(SlbmEngine* e, int phase) {
  if (e->layout) return dense_step(e, phase);
  SweepArgs a = sweep_args(e);
  if (phase == SLBM_PHASE_INTERIOR) {
    if (e->interior_lo >= 0) {  // one contiguous cid range, warps aligned to 32 cells
      a.lo = uint32_t(e->interior_lo);
      a.offset = a.lo & ~31u;
      a.n_cells = uint32_t(e->interior_lo + e->n_interior) - a.offset;
    } else {  // all cells minus the frame (identity order)
      a.skip = e->frame_bits;
      if (e->n_interior == 0) a.n_cells = 0;
    }
  } else if (phase == SLBM_PHASE_FRAME) {
    a.cids = e->frame_cids;
    a.n_cells = uint32_t(e->n_frame);
  }
  if (a.n_cells == 0) return SLBM_OK;
  const int kind = e->pattern == SLBM_PULL ? kPull : (e->parity == SLBM_EVEN ? kEven : kOdd);
  const unsigned grid = grid_for(a.n_cells, kBlock);
  SlbmTuning t = e->tune;
  int trial = -1;  // event pair of a timed trial launch
  if (kind != kOdd && phase == SLBM_PHASE_ALL) t.even_ctas = sweep_ctas(e, &trial);
  if (trial >= 0) SLBM_CUDA_TRY(cudaEventRecord(e->even_ev[2 * trial], e->stream));
  by_lattice(e->q, [&](auto lat) {
    launch_model<decltype(lat)>(e->model, kind, a, grid, t, e->stream);
  });
  if (trial >= 0) SLBM_CUDA_TRY(cudaEventRecord(e->even_ev[2 * trial + 1], e->stream));
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_refresh(SlbmEngine* e, int parity) {
  if (e->n_ubb) {
    { k_refresh<<<grid_for(e->n_ubb, 256), 256, 0, e->stream>>>(
        e->pdf, e->ubb_slot, e->ubb_partner, e->ubb_corr, uint32_t(e->n_ubb), parity); slbm::count_launch(); }
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  if (e->n_out) {
    SweepArgs a = sweep_args(e);
    by_lattice(e->q, [&](auto lat) {
      using L = decltype(lat);
      { k_outlet<L><<<grid_for(e->n_out, 128), 128, 0, e->stream>>>(
          e->pdf, a, e->out_slot, e->out_partner, e->out_cell, e->out_dir, e->out_rho, e->out_u,
          uint32_t(e->n_out), parity); slbm::count_launch(); }
    });
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  return SLBM_OK;
}

int launch_advance(SlbmEngine* e) {
  { k_advance<<<1, 1, 0, e->stream>>>(e->d_step); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

namespace {
template <class L, int MODEL>
cudaError_t resident_launch(const SweepArgs& a, const ResidentArgs& r, cudaStream_t s) {
  constexpr int MINB = L::Q == 9 ? 8 : 4;
  auto fn = k_resident<L, MODEL, MINB>;
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kIB, 0);
    per_sm = std::max(per_sm, 1);
  }
  // no more CTAs than cells need: fewer CTAs make the grid barrier cheaper
  const int64_t need = (int64_t(a.n_fluid) + kIB - 1) / kIB;
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(per_sm) * num_sms())));
  void* args[] = {const_cast<SweepArgs*>(&a), const_cast<ResidentArgs*>(&r)};
  const cudaError_t err = cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kIB), args, 0, s);
  if (err == cudaSuccess) count_launch();
  return err;
}
}  // namespace

bool resident_eligible(const SlbmEngine* e, int64_t n) {
  return e->tune.resident_cap > 0 && n >= 2 && e->layout == 0 && e->n_fluid > 0 &&
         e->n_fluid <= e->tune.resident_cap;
}

// n whole steps in one cooperative launch (k_resident); the caller updates
// parity / buffers / steps_done as n calls of sweep_once would.
int launch_resident(SlbmEngine* e, int64_t n) {
  SweepArgs a = sweep_args(e);
  ResidentArgs r{};
  r.ubb_slot = e->ubb_slot;
  r.ubb_partner = e->ubb_partner;
  r.ubb_corr = e->ubb_corr;
  r.n_ubb = uint32_t(e->n_ubb);
  r.out_slot = e->out_slot;
  r.out_partner = e->out_partner;
  r.out_cell = e->out_cell;
  r.out_dir = e->out_dir;
  r.out_rho = e->out_rho;
  r.out_u = e->out_u;
  r.n_out = uint32_t(e->n_out);
  r.steps = uint32_t(n);
  r.parity = e->parity;
  r.pull = e->pattern == SLBM_PULL ? 1 : 0;
  cudaError_t ce = cudaSuccess;
  by_lattice(e->q, [&](auto lat) {
    using L = decltype(lat);
    if (e->model == SLBM_SRT)
      ce = resident_launch<L, SLBM_SRT>(a, r, e->stream);
    else if (e->model == SLBM_TRT)
      ce = resident_launch<L, SLBM_TRT>(a, r, e->stream);
    else if constexpr (L::Q == 27) {
      if (e->model == SLBM_CUMULANT)
        ce = resident_launch<L, SLBM_CUMULANT>(a, r, e->stream);
      else
        ce = resident_launch<L, SLBM_CUMULANT_GEN>(a, r, e->stream);
    }
  });
  if (ce != cudaSuccess) return fail(SLBM_ECUDA, std::string("resident sweep: ") + cudaGetErrorString(ce));
  return SLBM_OK;
}

// canonical: nullptr -> read the sparse groups of e->pdf at the current
// parity; else a (q, n_fluid) canonical array (dense engine)
int launch_macroscopic(SlbmEngine* e, const double* canonical, double* dev_rho, double* dev_u,
                       bool compact, const int64_t* gdims, const int64_t* origin) {
  SweepArgs a = sweep_args(e);
  const double* src = e->pdf;
  int odd = (e->pattern == SLBM_AA && e->parity == SLBM_ODD) ? 1 : 0;
  if (canonical) {
    for (int q = 0; q < 28; ++q) a.base[q] = uint32_t(q) * uint32_t(e->n_fluid);
    src = canonical;
    odd = 0;
  }
  int* bad = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&bad, sizeof(int), e->stream));
  SLBM_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), e->stream));
  by_lattice(e->q, [&](auto lat) {
    using L = decltype(lat);
    MacroOut o{};
    if (gdims) o = MacroOut{gdims[0], gdims[1], origin[0], origin[1], origin[2]};
    { k_macro<L><<<grid_for(e->n_fluid, 256), 256, 0, e->stream>>>(
        src, a, odd, e->geo, compact ? nullptr : e->x_flat, dev_rho, dev_u, bad, o); slbm::count_launch(); }
  });
  int h_bad = 0;
  SLBM_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
  SLBM_CUDA_TRY(cudaFreeAsync(bad, e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  if (h_bad) return fail(SLBM_EUNSTABLE, "non-positive or non-finite density in collision input");
  return SLBM_OK;
}

int launch_macroscopic_box(SlbmEngine* e, double* rho, double* u) {
  SweepArgs a = sweep_args(e);
  const int odd = (e->pattern == SLBM_AA && e->parity == SLBM_ODD) ? 1 : 0;
  int* bad = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&bad, sizeof(int), e->stream));
  SLBM_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), e->stream));
  by_lattice(e->q, [&](auto lat) {
    using L = decltype(lat);
    { k_macro_box<L><<<grid_for(e->geo.n_cells(), kMacroBlock), kMacroBlock, 0, e->stream>>>(
        e->pdf, a, odd, e->geo, e->cid_map, rho, u, bad); slbm::count_launch(); }
  });
  SLBM_CUDA_TRY(cudaGetLastError());
  int h_bad = 0;
  SLBM_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
  SLBM_CUDA_TRY(cudaFreeAsync(bad, e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  if (h_bad) return fail(SLBM_EUNSTABLE, "non-positive or non-finite density in collision input");
  return SLBM_OK;
}

int launch_equilibrium(SlbmEngine* e, const double* rho, int rho_scalar, const double* u,
                       int u_scalar, double* /*unused*/) {
  SweepArgs a = sweep_args(e);
  by_lattice(e->q, [&](auto lat) {
    using L = decltype(lat);
    { k_equilibrium<L><<<grid_for(e->n_fluid, 256), 256, 0, e->stream>>>(e->pdf, a, rho,
                                                                         rho_scalar, u, u_scalar); slbm::count_launch(); }
  });
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

// equilibrium into a (q, n_fluid) array (dense engine init)
int launch_equilibrium_qn(SlbmEngine* e, const double* rho, int rho_scalar, const double* u,
                          int u_scalar, double* out) {
  SweepArgs a = sweep_args(e);
  for (int q = 0; q < 28; ++q) a.base[q] = uint32_t(q) * uint32_t(e->n_fluid);
  by_lattice(e->q, [&](auto lat) {
    using L = decltype(lat);
    { k_equilibrium<L><<<grid_for(e->n_fluid, 256), 256, 0, e->stream>>>(out, a, rho, rho_scalar,
                                                                         u, u_scalar); slbm::count_launch(); }
  });
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_gather(const double* src, const uint32_t* slots, int64_t n, double* out,
                  cudaStream_t s) {
  if (n == 0) return SLBM_OK;
  { k_gather<<<grid_for(n, 256), 256, 0, s>>>(src, slots, n, out); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_scatter(double* dst, const uint32_t* slots, int64_t n, const double* in,
                   cudaStream_t s) {
  if (n == 0) return SLBM_OK;
  { k_scatter<<<grid_for(n, 256), 256, 0, s>>>(dst, slots, n, in); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_fill(double* p, int64_t n, double v, cudaStream_t s) {
  if (n == 0) return SLBM_OK;
  unsigned g = grid_for(n, 256);
  if (g > 148 * 32) g = 148 * 32;
  { k_fill<<<g, 256, 0, s>>>(p, n, v); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

// Deterministic reductions with warp shuffles: a fixed grid of kRedBlocks
// CTAs strides over the input (the assignment of elements to threads, and
// so the summation order, depends only on n), each CTA reduces its 256
// partial sums through __shfl_down_sync and one shared-memory step into one
// partial per CTA, and a single CTA reduces the kRedBlocks partials in the
// same fixed tree order.  Same input -> same bits on every run (an atomic
// accumulation would not be), no library kernel on the path.
constexpr int kRedBlocks = 592;  // 148 SMs x 4
constexpr int kRedThreads = 256;

template <int K>
__device__ __forceinline__ void block_reduce_store(double (&v)[K], double* out) {
  __shared__ double w[kRedThreads / 32][K];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < K; ++k)
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  if (lane == 0)
    for (int k = 0; k < K; ++k) w[warp][k] = v[k];
  __syncthreads();
  if (warp == 0) {
    for (int k = 0; k < K; ++k) {
      double x = lane < kRedThreads / 32 ? w[lane][k] : 0.0;
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      if (lane == 0) out[k] = x;
    }
  }
}

__global__ void __launch_bounds__(kRedThreads) k_sum_partial(const double* p, int64_t n,
                                                             double* part) {
  double v[1] = {0.0};
  for (int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kRedThreads)
    v[0] += p[i];
  block_reduce_store<1>(v, part + blockIdx.x);
}

// mass and momentum of every fluid cell from its canonical populations at
// the current parity (even: group q; odd: group inv q), one pass
template <class L>
__global__ void __launch_bounds__(kRedThreads) k_moments_partial(const double* pdf, SweepArgs a,
                                                                 int odd, double* part) {
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (uint32_t c = blockIdx.x * kRedThreads + threadIdx.x; c < a.n_fluid;
       c += gridDim.x * kRedThreads) {
    double rho = 0.0, j[3] = {0.0, 0.0, 0.0};
    sfor<0, L::Q>([&](auto q) {
      constexpr int qb = L::INV[q];
      const double f = pdf[a.base[odd ? qb : int(q)] + c];
      rho += f;
      if constexpr (L::CX[q] > 0) j[0] += f;
      if constexpr (L::CX[q] < 0) j[0] -= f;
      if constexpr (L::CY[q] > 0) j[1] += f;
      if constexpr (L::CY[q] < 0) j[1] -= f;
      if constexpr (L::CZ[q] > 0) j[2] += f;
      if constexpr (L::CZ[q] < 0) j[2] -= f;
    });
    v[0] += rho;
    v[1] += j[0];
    v[2] += j[1];
    v[3] += j[2];
  }
  block_reduce_store<4>(v, part + 4 * blockIdx.x);
}

// K sums of `n` strided partials (partial b of sum k at part[b * K + k])
template <int K>
__global__ void __launch_bounds__(kRedThreads) k_reduce_final(const double* part, int n,
                                                              double* out) {
  double v[K];
  for (int k = 0; k < K; ++k) v[k] = 0.0;
  for (int b = threadIdx.x; b < n; b += kRedThreads)
    for (int k = 0; k < K; ++k) v[k] += part[b * K + k];
  block_reduce_store<K>(v, out);
}

int launch_sum(const double* p, int64_t n, double* dev_out, cudaStream_t s) {
  double* part = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&part, kRedBlocks * sizeof(double), s));
  { k_sum_partial<<<kRedBlocks, kRedThreads, 0, s>>>(p, n, part); slbm::count_launch(); }
  { k_reduce_final<1><<<1, kRedThreads, 0, s>>>(part, kRedBlocks, dev_out); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  SLBM_CUDA_TRY(cudaFreeAsync(part, s));
  return SLBM_OK;
}

// total mass and momentum (4 doubles at dev_out) of a sparse engine
int launch_moments(SlbmEngine* e, double* dev_out) {
  SweepArgs a = sweep_args(e);
  const int odd = (e->pattern == SLBM_AA && e->parity == SLBM_ODD) ? 1 : 0;
  double* part = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&part, 4 * kRedBlocks * sizeof(double), e->stream));
  by_lattice(e->q, [&](auto lat) {
    using L = decltype(lat);
    { k_moments_partial<L><<<kRedBlocks, kRedThreads, 0, e->stream>>>(e->pdf, a, odd, part); slbm::count_launch(); }
  });
  { k_reduce_final<4><<<1, kRedThreads, 0, e->stream>>>(part, kRedBlocks, dev_out); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  SLBM_CUDA_TRY(cudaFreeAsync(part, e->stream));
  return SLBM_OK;
}

}  // namespace slbm
