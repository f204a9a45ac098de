// Stream-collide sweeps and the small per-step kernels.
//
// One thread per fluid cell; each thread owns a disjoint slot set (the
// builder's uniqueness check, sparse.py:182-185), so the in-place AA
// scatter needs no synchronisation and any cell subset (interior / frame)
// composes bitwise with the whole-block sweep.
//
//   k_aa_even  combined pull-collide-push step   sparse.py:264-271
//              t0 = pdf[c], t_q = pdf[idx[q-1][c]];  collide;
//              pdf[c] = out0, pdf[idx[q-1][c]] = out[inv q]
//              traffic 19x8 R + 19x8 W + 18x4 idx = 376 B/cell (D3Q19)
//   k_aa_odd   cell-local reversed step          sparse.py:273-282
//              t_r = pdf[base[inv r] + c]; pdf[base[r] + c] = out_r
//              304 B/cell, every access coalesced
//   k_pull     two-buffer pull                   sparse.py:257-262
//              gather as k_aa_even, dst[base[r] + c] = out_r; 376 B/cell
#include <cub/cub.cuh>

#include <climits>

#include "collide.cuh"
#include "engine.cuh"

namespace slbm {

struct SweepArgs {
  double* pdf;
  double* dst;
  const uint32_t* idx;
  const uint32_t* cids;  // nullptr: identity (whole block)
  uint32_t n_cells;
  uint32_t n_fluid;
  uint32_t base[28];
  double omega, lam;
  unsigned long long* bad;
  const unsigned long long* step;
};

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ void flag_bad(const SweepArgs& a) {
  atomicMin(a.bad, *a.step);
}

template <class L, int MODEL>
__global__ void __launch_bounds__(kBlock) k_aa_even(const SweepArgs a) {
  const uint32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= a.n_cells) return;
  const uint32_t c = a.cids ? a.cids[i] : i;
  uint32_t s[L::Q];
  double t[L::Q];
  s[0] = c;
  sfor<1, L::Q>([&](auto q) { s[q] = __ldcs(a.idx + size_t(q - 1) * a.n_fluid + c); });
  sfor<0, L::Q>([&](auto q) { t[q] = a.pdf[s[q]]; });
  double* pdf = a.pdf;
  const bool bad = collide<L, MODEL>(t, a.omega, a.lam, [&](auto q, double v) {
    constexpr int qb = L::INV[decltype(q)::value];
    pdf[s[qb]] = v;
  });
  if (bad) flag_bad(a);
}

template <class L, int MODEL>
__global__ void __launch_bounds__(kBlock) k_aa_odd(const SweepArgs a) {
  const uint32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= a.n_cells) return;
  const uint32_t c = a.cids ? a.cids[i] : i;
  double t[L::Q];
  sfor<0, L::Q>([&](auto q) {
    constexpr int qb = L::INV[q];
    t[q] = a.pdf[a.base[qb] + c];
  });
  double* pdf = a.pdf;
  const bool bad = collide<L, MODEL>(t, a.omega, a.lam, [&](auto q, double v) {
    pdf[a.base[decltype(q)::value] + c] = v;
  });
  if (bad) flag_bad(a);
}

template <class L, int MODEL>
__global__ void __launch_bounds__(kBlock) k_pull(const SweepArgs a) {
  const uint32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= a.n_cells) return;
  const uint32_t c = a.cids ? a.cids[i] : i;
  double t[L::Q];
  t[0] = a.pdf[c];
  sfor<1, L::Q>([&](auto q) {
    t[q] = a.pdf[__ldcs(a.idx + size_t(q - 1) * a.n_fluid + c)];
  });
  double* dst = a.dst;
  const bool bad = collide<L, MODEL>(t, a.omega, a.lam, [&](auto q, double v) {
    dst[a.base[decltype(q)::value] + c] = v;
  });
  if (bad) flag_bad(a);
}

enum Kind { kPull = 0, kEven = 1, kOdd = 2 };

template <class L, int MODEL>
void launch_kind(int kind, const SweepArgs& a, unsigned grid, cudaStream_t s) {
  if (kind == kPull)
    k_pull<L, MODEL><<<grid, kBlock, 0, s>>>(a);
  else if (kind == kEven)
    k_aa_even<L, MODEL><<<grid, kBlock, 0, s>>>(a);
  else
    k_aa_odd<L, MODEL><<<grid, kBlock, 0, s>>>(a);
}

template <class L>
void launch_model(int model, int kind, const SweepArgs& a, unsigned grid, cudaStream_t s) {
  if (model == SLBM_SRT)
    launch_kind<L, SLBM_SRT>(kind, a, grid, s);
  else if (model == SLBM_TRT)
    launch_kind<L, SLBM_TRT>(kind, a, grid, s);
  else if constexpr (L::Q == 27)
    launch_kind<L, SLBM_CUMULANT>(kind, a, grid, s);
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

// canonical (q, n) values per cell straight from the groups (sparse.py:308-321)
template <class L>
__global__ void k_macro(const double* pdf, SweepArgs a, int odd, Geometry g,
                        const uint32_t* x_flat, double* rho_f, double* u_f, int* bad) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.n_fluid) return;
  double t[L::Q];
  sfor<0, L::Q>([&](auto q) {
    constexpr int qb = L::INV[q];
    t[q] = pdf[a.base[odd ? qb : int(q)] + c];
  });
  const Moments<L> m = moments<L>(t);
  if (m.bad) atomicOr(bad, 1);
  int64_t x, y, z;
  g.coords(x_flat[c], x, y, z);
  const int64_t f = g.interior_flat(x, y, z);
  rho_f[f] = m.rho;
  u_f[f * L::DIM + 0] = m.ux;
  u_f[f * L::DIM + 1] = m.uy;
  if constexpr (L::DIM == 3) u_f[f * L::DIM + 2] = m.uz;
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
  for (int q = 0; q <= e->q && q < 28; ++q) a.base[q] = uint32_t(e->base[q]);
  a.omega = e->omega;
  a.lam = e->lambda_odd;
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

int launch_slot_lookup(SlbmEngine* e, const int64_t* d_qs, const int64_t* d_pflat, int64_t n,
                       int64_t* d_out, int* d_err) {
  if (n == 0) return SLBM_OK;
  k_slot_lookup<<<grid_for(n, 256), 256, 0, e->stream>>>(d_qs, d_pflat, n, e->cid_map,
                                                          e->geo.n_padded(), sweep_args(e), e->q,
                                                          d_out, d_err);
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_step(SlbmEngine* e, int phase) {
  SweepArgs a = sweep_args(e);
  if (phase == SLBM_PHASE_INTERIOR) {
    a.cids = e->interior_cids;
    a.n_cells = uint32_t(e->n_interior);
  } else if (phase == SLBM_PHASE_FRAME) {
    a.cids = e->frame_cids;
    a.n_cells = uint32_t(e->n_frame);
  }
  if (a.n_cells == 0) return SLBM_OK;
  const int kind = e->pattern == SLBM_PULL ? kPull : (e->parity == SLBM_EVEN ? kEven : kOdd);
  const unsigned grid = grid_for(a.n_cells, kBlock);
  by_lattice(e->q, [&](auto lat) {
    launch_model<decltype(lat)>(e->model, kind, a, grid, e->stream);
  });
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_refresh(SlbmEngine* e, int parity) {
  if (e->n_ubb == 0) return SLBM_OK;
  k_refresh<<<grid_for(e->n_ubb, 256), 256, 0, e->stream>>>(
      e->pdf, e->ubb_slot, e->ubb_partner, e->ubb_corr, uint32_t(e->n_ubb), parity);
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_advance(SlbmEngine* e) {
  k_advance<<<1, 1, 0, e->stream>>>(e->d_step);
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_macroscopic(SlbmEngine* e, const double* /*unused*/, double* dev_rho, double* dev_u) {
  SweepArgs a = sweep_args(e);
  int* bad = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&bad, sizeof(int), e->stream));
  SLBM_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), e->stream));
  const int odd = (e->pattern == SLBM_AA && e->parity == SLBM_ODD) ? 1 : 0;
  by_lattice(e->q, [&](auto lat) {
    using L = decltype(lat);
    k_macro<L><<<grid_for(e->n_fluid, 256), 256, 0, e->stream>>>(e->pdf, a, odd, e->geo,
                                                                   e->x_flat, dev_rho, dev_u, bad);
  });
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
    k_equilibrium<L><<<grid_for(e->n_fluid, 256), 256, 0, e->stream>>>(e->pdf, a, rho,
                                                                         rho_scalar, u, u_scalar);
  });
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_gather(const double* src, const uint32_t* slots, int64_t n, double* out,
                  cudaStream_t s) {
  if (n == 0) return SLBM_OK;
  k_gather<<<grid_for(n, 256), 256, 0, s>>>(src, slots, n, out);
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_scatter(double* dst, const uint32_t* slots, int64_t n, const double* in,
                   cudaStream_t s) {
  if (n == 0) return SLBM_OK;
  k_scatter<<<grid_for(n, 256), 256, 0, s>>>(dst, slots, n, in);
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_fill(double* p, int64_t n, double v, cudaStream_t s) {
  if (n == 0) return SLBM_OK;
  unsigned g = grid_for(n, 256);
  if (g > 148 * 32) g = 148 * 32;
  k_fill<<<g, 256, 0, s>>>(p, n, v);
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int launch_sum(const double* p, int64_t n, double* dev_out, cudaStream_t s) {
  size_t tmp_bytes = 0;
  SLBM_CUDA_TRY(cub::DeviceReduce::Sum(nullptr, tmp_bytes, p, dev_out, n, s));
  void* tmp = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  SLBM_CUDA_TRY(cub::DeviceReduce::Sum(tmp, tmp_bytes, p, dev_out, n, s));
  SLBM_CUDA_TRY(cudaFreeAsync(tmp, s));
  return SLBM_OK;
}

}  // namespace slbm
