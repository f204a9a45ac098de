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

template <class L, int MODEL, int KIND>
__global__ void __launch_bounds__(kGB, KIND == 2 ? 6 : 4) k_group(const GroupArgs* __restrict__ table,
                                                  const uint32_t* __restrict__ start, int n_eng,
                                                  double omega, double lam, const double* hr,
                                                  uint32_t ahead) {
  // every thread finds its engine and reads the (tiny, L1-resident) table
  // row itself: no single-thread staging + __syncthreads at CTA start, which
  // cost ~15% of the even sweep (measured, tools/slab_probe.py)
  const int eng = find_engine(start, n_eng, blockIdx.x);
  const uint32_t first = start[eng];
  // the odd sweep addresses 2Q group rows through base[]: staged in shared
  // memory those offsets stay out of registers (77 vs 128 + spills)
  __shared__ GroupArgs staged;
  if constexpr (KIND == 2) {
    if (threadIdx.x == 0) staged = table[eng];
    __syncthreads();
  }
  const GroupArgs& a = KIND == 2 ? staged : table[eng];
  constexpr int kTiles = KIND == 2 ? kOddTiles : 1;
  const uint32_t pos0 = (blockIdx.x - first) * kGB * kTiles;  // this CTA's first sweep position
  const uint32_t* idx = a.idx;
  const uint32_t* cids = a.cids;
  const uint32_t pitch = a.idx_pitch, n_cells = a.n_cells, offset = a.offset;
  // index-list rows of this engine's CTA `ahead` positions later (sweep.cuh),
  // issued first as in the single-engine sweep
  if (KIND != 2 && cids == nullptr)
    prefetch_idx_ahead<L::Q - 1, kGB>(idx, pitch, nullptr, offset + n_cells, offset + pos0,
                                      ahead);
  pdl_launch_dependents();
  pdl_wait();  // the boundary kernel's halo / wall values (read-only lists above)
  bool bad = false;
#pragma unroll
  for (int tile = 0; tile < kTiles; ++tile) {
    const uint32_t i = pos0 + tile * kGB + threadIdx.x;
    if (i >= n_cells) break;
    const uint32_t c = cids ? cids[i] : offset + i;
    if (c < a.lo || (a.skip && ((__ldg(a.skip + (c >> 5)) >> (c & 31)) & 1u))) continue;
    if constexpr (KIND == 2) {
      bad |= cell_local<L, MODEL>(a.pdf, a.base, c, omega, lam, hr);
    } else {
      uint32_t s[L::Q];
      double t[L::Q];
      load_slots<L>(s, idx, pitch, c);
      gather<L>(t, a.pdf, s);
      if (cids) prefetch_idx_ahead<L::Q - 1, kGB>(idx, pitch, cids, n_cells, pos0, ahead);
      bad |= collide_scatter<L, MODEL, KIND == 1>(t, s, a.pdf, a.dst, a.base, c, omega, lam, hr);
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
template <class L>
__global__ void k_group_boundary(PdfTable lt, LocalEdges le, const GroupArgs* table,
                                 const uint16_t* ueng, const uint32_t* uslot,
                                 const uint32_t* upartner, const double* ucorr, int64_t n_ubb,
                                 const OutletTab* ot, const uint16_t* oeng, const uint32_t* oidx,
                                 int64_t n_out, unsigned long long** steps, int n_eng, int parity) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  pdl_launch_dependents();
  pdl_wait();  // the previous sweep
  if (i < n_eng) *steps[i] += 1;
  if (i < le.n) {
    lt.p[le.de[i]][le.ds[i]] = lt.p[le.se[i]][le.ss[i]];
    return;
  }
  i -= le.n;
  if (i < n_ubb) {
    double* pdf = table[ueng[i]].pdf;
    if (parity == SLBM_EVEN)
      pdf[uslot[i]] = pdf[upartner[i]] + ucorr[i];
    else
      pdf[upartner[i]] = pdf[uslot[i]] + ucorr[i];
    return;
  }
  i -= n_ubb;
  if (i < n_out) {
    const int e = oeng[i];
    const uint32_t k = oidx[i];
    const OutletTab& o = ot[e];
    const GroupArgs& a = table[e];
    outlet_entry<L>(a.pdf, a.base, o.slot[k], o.partner[k], o.cell[k], o.dir[k], o.rho[k],
                    o.u + 3 * size_t(k), parity);
  }
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
  return a;
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
  // pull: each engine's e->pdf is "current"; record the flip as 0
  for (int phase = 0; phase < 3; ++phase) {
    if (phase && !e0->has_split) continue;
    std::vector<uint32_t> start(n + 1, 0);
    for (int i = 0; i < n; ++i) {
      const GroupArgs a = args_of(engines[i], phase, 0);
      start[i + 1] = start[i] + (a.n_cells + kGB - 1) / kGB;
    }
    g->n_cta[phase] = start[n];
    SLBM_CUDA_TRY(cudaMalloc(&g->cta_start[phase], (n + 1) * sizeof(uint32_t)));
    SLBM_CUDA_TRY(cudaMemcpy(g->cta_start[phase], start.data(), (n + 1) * sizeof(uint32_t),
                             cudaMemcpyHostToDevice));
    std::vector<uint32_t> odd(n + 1, 0);
    for (int i = 0; i < n; ++i) {
      const GroupArgs a = args_of(engines[i], phase, 0);
      odd[i + 1] = odd[i] + (a.n_cells + kGB * kOddTiles - 1) / (kGB * kOddTiles);
    }
    g->n_cta_odd[phase] = odd[n];
    SLBM_CUDA_TRY(cudaMalloc(&g->cta_start_odd[phase], (n + 1) * sizeof(uint32_t)));
    SLBM_CUDA_TRY(cudaMemcpy(g->cta_start_odd[phase], odd.data(), (n + 1) * sizeof(uint32_t),
                             cudaMemcpyHostToDevice));
    for (int flip = 0; flip < 2; ++flip) {
      std::vector<GroupArgs> tab(n);
      for (int i = 0; i < n; ++i) tab[i] = args_of(engines[i], phase, flip);
      SLBM_CUDA_TRY(cudaMalloc(&g->table[phase][flip], n * sizeof(GroupArgs)));
      SLBM_CUDA_TRY(cudaMemcpy(g->table[phase][flip], tab.data(), n * sizeof(GroupArgs),
                               cudaMemcpyHostToDevice));
    }
  }
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
  *out = g;
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
  const int64_t work = std::max<int64_t>(n, le.n + g->n_ubb + g->n_out);
  cudaError_t err = cudaSuccess;
  on_lattice(g->q, [&](auto lat) {
    using L = decltype(lat);
    err = launch_pdl(k_group_boundary<L>, dim3(unsigned((work + 127) / 128)), dim3(128), 0, s,
                     lt, le, g->table[0][flip], g->ubb_eng, g->ubb_slot, g->ubb_partner,
                     g->ubb_corr, g->n_ubb, g->out_tab, g->out_eng, g->out_idx, g->n_out,
                     g->steps, n, parity);
  });
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
