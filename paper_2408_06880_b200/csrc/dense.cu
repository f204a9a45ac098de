// Direct-addressing ("dense") block engine on the GPU — SURVEY §8f1, the
// reference's DenseEngine (pkg/src/slbm/dense.py).
//
// Storage is the reference's: one plane per direction over the padded block
// box, slot(q, p) = q * npad + p for padded flat index p (dense.py:95-97,
// :311-317), so halo plans address dense and sparse blocks alike and mixed
// ("hybrid") decompositions exchange with the reference's wire formats.
//
// Instead of the reference's precomputed (Q, cells) gather table, every
// read address is computed from the cell's coordinates: the neighbour slot
// q*npad + p - stride(q) (periodic in-block wrap only on boundary cells), or
// the cell's own opposite slot when the upwind cell is a wall — one 32-bit
// fold mask per box cell (bit q) built once on the device.  Moving-wall
// (UBB) folds add the reference's momentum term at the folded read and at
// the folded write of the combined step (dense.py:263-279); their few
// (cell, q) -> correction entries are found by binary search.  Solid cells
// carry the sentinel mask and are skipped: their slots are never read by a
// fluid cell, so fluid results are the same bits as the reference's full-box
// sweep (and as the sparse engine's).
//
// Traffic per fluid cell: 2 Q x 8 B of PDFs + 4 B of mask, no index list
// (D3Q19: 308 B vs 376 B for the sparse index-list step).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <vector>

#include "collide.cuh"
#include "engine.cuh"
#include "sweep.cuh"

namespace slbm {
namespace {

constexpr uint32_t kSolid = 0xffffffffu;
constexpr uint32_t kHasUbb = 0x80000000u;
constexpr uint8_t kFluidT = 0, kUbbT = 2, kExchT = 3, kOutT = 4;

struct DenseArgs {
  double* pdf;
  double* dst;
  const uint32_t* mask;     // per box cell
  const uint64_t* ubb_key;  // sorted (box cell << 5 | q)
  const double* ubb_corr;
  int64_t n_ubb;
  Geometry g;
  int64_t npad;
  int64_t stride[27];       // padded-flat offset of the upwind cell
  int32_t frame_w[3];
  int phase;                // SLBM_PHASE_*
  double omega, lam;
  const double* hr;         // cumulant: higher-order rates
  unsigned long long* bad;
  const unsigned long long* step;
};

__device__ __forceinline__ double ubb_corr_of(const DenseArgs& a, uint32_t cell, int q) {
  const uint64_t key = (uint64_t(cell) << 5) | uint64_t(q);
  int64_t lo = 0, hi = a.n_ubb;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a.ubb_key[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < a.n_ubb && a.ubb_key[lo] == key) ? a.ubb_corr[lo] : 0.0;
}

// Offset (in padded-flat units) to add to p - stride(q) when a direction-q
// read of face cell (x, y, z) wraps periodically inside the block
// (dense.py:126-131): +-extent along each periodic axis the upwind cell
// leaves.  Non-periodic faces read the padding ring (walls / halo), which
// p - stride(q) already addresses.
template <class L, int Q_>
__device__ __forceinline__ int32_t wrap_delta(const DenseArgs& a, int32_t x, int32_t y,
                                              int32_t z) {
  constexpr int cx = L::CX[Q_], cy = L::CY[Q_], cz = L::CZ[Q_];
  int32_t d = 0;
  if constexpr (cx != 0) {
    const int32_t s = x - cx, n = a.g.n[0];
    if (a.g.periodic[0]) d += s < 0 ? n : (s >= n ? -n : 0);
  }
  if constexpr (cy != 0) {
    const int32_t s = y - cy, n = a.g.n[1];
    if (a.g.periodic[1]) d += (s < 0 ? n : (s >= n ? -n : 0)) * int32_t(a.g.p[0]);
  }
  if constexpr (L::DIM == 3 && cz != 0) {
    const int32_t s = z - cz, n = a.g.n[2];
    if (a.g.periodic[2]) d += (s < 0 ? n : (s >= n ? -n : 0)) * int32_t(a.g.p[0] * a.g.p[1]);
  }
  return d;
}

__device__ __forceinline__ bool in_phase(const DenseArgs& a, int64_t x, int64_t y, int64_t z) {
  if (a.phase == SLBM_PHASE_ALL) return true;
  const int64_t v[3] = {x, y, z};
  bool frame = false;
  for (int k = 0; k < a.g.dim; ++k)
    frame |= (v[k] < a.frame_w[k]) || (v[k] >= a.g.n[k] - a.frame_w[k]);
  return (a.phase == SLBM_PHASE_FRAME) == frame;
}

// KIND 0 pull, 1 combined (AA even), 2 reversed (AA odd).
// Grid: 128 cells of one (y, z) row per CTA, chunks of a row on consecutive
// CTAs; slots are 32-bit (q * npad < 2^32 is checked at build).  Cells away from the block faces take the neighbour
// slot p - stride(q) directly; only face cells check the periodic wrap.
//
// Every cell first reads its fold mask, and every PDF address depends on it
// — one dependent DRAM round trip in front of the sweep's loads.  As in the
// sparse sweep's idx prefetch (sweep.cuh), each CTA touches into L2 the mask
// chunk of the row `ahead` rows later (4 lines of 128 B), so that CTA's mask
// load is an L2 hit.
//
// SPEC (blocks of porosity >= 0.75 — the ones the hybrid policy makes dense):
// the PDF loads do not wait for the mask.  The cell-local step loads its own
// slots and drops a solid cell's values afterwards; the index-free combined
// step loads every upwind neighbour's slot and re-reads only the folded
// directions (walls), which are rare in such blocks.
template <class L, int MODEL, int KIND, bool SPEC>
__global__ void __launch_bounds__(128, 4) k_dense(const DenseArgs a, uint32_t ahead) {
  const int32_t X = a.g.n[0], Y = a.g.n[1], Z = a.g.n[2];
  // CTA b -> (row, chunk) with the chunk fastest: consecutive CTAs sweep
  // consecutive memory of every direction plane (rows on the slow index
  // opened each DRAM page once per chunk column: -30 % measured)
  const uint32_t chunks = (uint32_t(X) + 127) / 128;
  const uint32_t row_u = blockIdx.x / chunks, chunk = blockIdx.x - row_u * chunks;
  const int32_t x = int32_t(chunk * 128 + threadIdx.x);
  const int32_t row = int32_t(row_u);  // z * Y + y
  if (threadIdx.x < 4) {
    const uint32_t fb = blockIdx.x + ahead;
    if (fb < gridDim.x) {
      const uint32_t fr = fb / chunks, fx = (fb - fr * chunks) * 128 + threadIdx.x * 32;
      if (fx < uint32_t(X)) prefetch_l2(a.mask + size_t(fr) * X + fx);
    }
  }
  if (x >= X) return;
  const int32_t y = row % Y, z = row / Y;
  const uint32_t i = uint32_t(row) * uint32_t(X) + uint32_t(x);
  const uint32_t m = a.mask[i];
  if (!SPEC && m == kSolid) return;
  if (!in_phase(a, x, y, z)) return;
  const uint32_t PX = uint32_t(a.g.p[0]), PY = uint32_t(a.g.p[1]);
  const uint32_t p = ((uint32_t(z + a.g.off[2]) * PY) + uint32_t(y + 1)) * PX + uint32_t(x + 1);
  const uint32_t np = uint32_t(a.npad);
  double* pdf = a.pdf;
  double t[L::Q];
  bool bad;
  if constexpr (KIND == 2) {
    sfor<0, L::Q>([&](auto q) {
      constexpr int qb = L::INV[q];
      t[q] = pdf[uint32_t(qb) * np + p];
    });
    if (SPEC && m == kSolid) return;  // loads above were harmless reads
    bad = collide<L, MODEL>(t, a.omega, a.lam, [&](auto q, double v) {
      pdf[uint32_t(decltype(q)::value) * np + p] = v;
    }, a.hr);
  } else {
    const bool face = x == 0 || x == X - 1 || y == 0 || y == Y - 1 ||
                      (L::DIM == 3 && (z == 0 || z == Z - 1));
    uint32_t addr[L::Q];
    addr[0] = p;
    // upwind slots (periodic in-block wrap only on face cells)
    if (!face) {
      sfor<1, L::Q>([&](auto q) { addr[q] = uint32_t(int(q)) * np + p - uint32_t(a.stride[q]); });
    } else {
      sfor<1, L::Q>([&](auto q) {
        addr[q] = uint32_t(int(q)) * np + p - uint32_t(a.stride[q]) +
                  uint32_t(wrap_delta<L, q>(a, x, y, z));
      });
    }
    constexpr uint32_t kFolds = (L::Q == 32 ? 0xffffffffu : ((1u << L::Q) - 1u)) & ~1u;
    if constexpr (SPEC) {
      sfor<0, L::Q>([&](auto q) { t[q] = pdf[addr[q]]; });
      if (m == kSolid) return;
      if (m & kFolds) {  // wall reads: the cell's own opposite slot instead
        sfor<1, L::Q>([&](auto q) {
          constexpr int qb = L::INV[q];
          if ((m >> q) & 1u) {
            addr[q] = uint32_t(qb) * np + p;
            t[q] = pdf[addr[q]];
          }
        });
      }
    } else {
      sfor<1, L::Q>([&](auto q) {
        constexpr int qb = L::INV[q];
        if ((m >> q) & 1u) addr[q] = uint32_t(qb) * np + p;
      });
      sfor<0, L::Q>([&](auto q) { t[q] = pdf[addr[q]]; });
    }
    if (m & kHasUbb) {
      sfor<1, L::Q>([&](auto q) {
        if ((m >> q) & 1u) t[q] += ubb_corr_of(a, i, q);
      });
    }
    if constexpr (KIND == 1) {
      bad = collide<L, MODEL>(t, a.omega, a.lam, [&](auto q, double v) {
        constexpr int qb = L::INV[decltype(q)::value];
        // out[q] lands at the read location of direction inv q; a folded
        // moving-wall read adds its term at that write too (dense.py:269-279)
        if constexpr (qb != 0) {
          if ((m & kHasUbb) && ((m >> qb) & 1u)) v = v + ubb_corr_of(a, i, qb);
        }
        pdf[addr[qb]] = v;
      }, a.hr);
    } else {
      double* dst = a.dst;
      bad = collide<L, MODEL>(t, a.omega, a.lam, [&](auto q, double v) {
        dst[uint32_t(decltype(q)::value) * np + p] = v;
      }, a.hr);
    }
  }
  if (bad) atomicMin(a.bad, *a.step);
}

// Lean AA odd (cell-local) sweep for whole-block phases: the same per-cell
// arithmetic as k_dense<KIND 2>, addressing every group through a table of
// 32-bit group starts (q * npad) that the compiler folds into the load
// instructions — k_dense<2> computes q * npad + p per direction and needs
// 122 registers at 4 CTAs/SM (80 + 128 B of spills at 6); this fits 80
// registers without spills, 6 CTAs/SM.
struct DenseOddArgs {
  double* pdf;
  const uint32_t* mask;
  uint32_t X, Y, PX, PY, offz;
  uint32_t base[28];  // q * npad
  double omega, lam;
  const double* hr;
  unsigned long long* bad;
  const unsigned long long* step;
};

template <class L, int MODEL>
__global__ void __launch_bounds__(128, L::Q == 27 ? 5 : 6) k_dense_odd(const DenseOddArgs a) {
  const uint32_t chunks = (a.X + 127) / 128;
  // CTAs last to first: the combined step before ran first to last, so this
  // sweep starts on the lines it left in L2 (as the sparse cell-local sweep)
  const uint32_t b = gridDim.x - 1 - blockIdx.x;
  const uint32_t row = b / chunks, chunk = b - row * chunks;
  const uint32_t x = chunk * 128 + threadIdx.x;
  if (x >= a.X) return;
  const uint32_t y = row % a.Y, z = row / a.Y;
  const uint32_t p = ((z + a.offz) * a.PY + y + 1) * a.PX + x + 1;
  double t[L::Q];
  sfor<0, L::Q>([&](auto q) {
    constexpr int qb = L::INV[q];
    t[q] = a.pdf[a.base[qb] + p];
  });
  // a solid cell's loads above were harmless reads; its results are dropped
  // (predicated stores: an early return here costs 128 B of spills)
  const bool fluid = a.mask[row * a.X + x] != kSolid;
  if (collide<L, MODEL>(t, a.omega, a.lam, [&](auto q, double v) {
        if (fluid) a.pdf[a.base[decltype(q)::value] + p] = v;
      }, a.hr) && fluid)
    atomicMin(a.bad, *a.step);
}

// fold mask per box cell and the number of UBB folds (for the entry list)
__global__ void k_dense_mask(const uint8_t* tags, Geometry g, DirTable d, uint32_t* mask,
                             unsigned long long* n_ubb, int* err) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.n_cells()) return;
  const int64_t x = i % g.n[0];
  const int64_t r = i / g.n[0];
  const int64_t y = r % g.n[1];
  const int64_t z = r / g.n[1];
  const uint8_t here = tags[g.padded_flat(x, y, z)];
  if (here != kFluidT) {
    mask[i] = kSolid;
    return;
  }
  uint32_t m = 0;
  unsigned nu = 0;
  for (int q = 1; q < d.q; ++q) {
    int64_t s[3] = {x - d.c[q][0], y - d.c[q][1], z - d.c[q][2]};
    for (int k = 0; k < 3; ++k)
      if (g.periodic[k]) s[k] = ((s[k] % g.n[k]) + g.n[k]) % g.n[k];
    const uint8_t tag = tags[g.padded_flat(s[0], s[1], s[2])];
    if (tag == kFluidT || tag == kExchT) continue;
    if (tag == kOutT) atomicOr(err, 1);
    m |= 1u << q;
    if (tag == kUbbT) {
      m |= kHasUbb;
      ++nu;
    }
  }
  mask[i] = m;
  if (nu) atomicAdd(n_ubb, (unsigned long long)nu);
}

__global__ void k_dense_ubb(const uint8_t* tags, Geometry g, DirTable d, const uint32_t* mask,
                            const uint32_t* wall_flat, const double* wall_u, int64_t n_wall,
                            unsigned long long* pos, uint64_t* keys, double* corr) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.n_cells()) return;
  const uint32_t m = mask[i];
  if (m == kSolid || !(m & kHasUbb)) return;
  const int64_t x = i % g.n[0];
  const int64_t r = i / g.n[0];
  const int64_t y = r % g.n[1];
  const int64_t z = r / g.n[1];
  for (int q = 1; q < d.q; ++q) {
    int64_t s[3] = {x - d.c[q][0], y - d.c[q][1], z - d.c[q][2]};
    for (int k = 0; k < 3; ++k)
      if (g.periodic[k]) s[k] = ((s[k] % g.n[k]) + g.n[k]) % g.n[k];
    const int64_t sp = g.padded_flat(s[0], s[1], s[2]);
    if (tags[sp] != kUbbT) continue;
    int64_t lo = 0, hi = n_wall;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (int64_t(wall_flat[mid]) < sp)
        lo = mid + 1;
      else
        hi = mid;
    }
    // core.py:173-188
    double cu = 0.0;
    for (int k = 0; k < g.dim; ++k) {
      if (d.c[q][k] == 1) cu = cu + wall_u[lo * 3 + k];
      if (d.c[q][k] == -1) cu = cu - wall_u[lo * 3 + k];
    }
    const unsigned long long at = atomicAdd(pos, 1ull);
    keys[at] = (uint64_t(i) << 5) | uint64_t(q);
    corr[at] = (((2.0 * d.w[q]) * 1.0) * cu) / (1.0 / 3.0);
  }
}

// resting weights in every box cell's slots (dense.py:208-209)
__global__ void k_dense_weights(double* pdf, Geometry g, int64_t npad, DirTable d) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.n_cells()) return;
  const int64_t x = i % g.n[0];
  const int64_t r = i / g.n[0];
  const int64_t p = g.padded_flat(x, r % g.n[1], r / g.n[1]);
  for (int q = 0; q < d.q; ++q) pdf[q * npad + p] = d.w[q];
}

// fluid-cell values <-> planes.  dir_map[q] = plane read for output row q
__global__ void k_dense_scatter(double* pdf, const uint32_t* x_flat, int64_t n, int64_t npad,
                                int q_count, const double* values) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n) return;
  for (int q = 0; q < q_count; ++q) pdf[q * npad + x_flat[c]] = values[q * n + c];
}

__global__ void k_dense_gather(const double* pdf, const uint32_t* x_flat, int64_t n, int64_t npad,
                               DirTable d, int odd, double* values) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n) return;
  for (int q = 0; q < d.q; ++q) values[q * n + c] = pdf[(odd ? d.inv[q] : q) * npad + x_flat[c]];
}

inline unsigned grid_of(int64_t n, int b) { return unsigned(std::max<int64_t>((n + b - 1) / b, 1)); }

template <class F>
void with_lattice(int q, F&& f) {
  if (q == 9)
    f(LatD2Q9{});
  else if (q == 19)
    f(LatD3Q19{});
  else
    f(LatD3Q27{});
}

DenseArgs dense_args(SlbmEngine* e) {
  DenseArgs a{};
  a.pdf = e->pdf;
  a.dst = e->tmp;
  a.mask = e->dense_mask;
  a.ubb_key = e->dense_ubb_key;
  a.ubb_corr = e->dense_ubb_corr;
  a.n_ubb = e->n_dense_ubb;
  a.g = e->geo;
  a.npad = e->geo.n_padded();
  for (int q = 0; q < e->q; ++q)
    a.stride[q] = (int64_t(e->dirs.c[q][2]) * e->geo.p[1] + e->dirs.c[q][1]) * e->geo.p[0] +
                  e->dirs.c[q][0];
  for (int k = 0; k < 3; ++k) a.frame_w[k] = e->dense_frame_w[k];
  a.phase = SLBM_PHASE_ALL;
  a.omega = e->omega;
  a.lam = e->lambda_odd;
  a.hr = e->d_hr;
  a.bad = e->d_bad;
  a.step = e->d_step;
  return a;
}

}  // namespace

int build_dense(SlbmEngine* e, const uint8_t* tags_pad, const double* ubb_u_pad,
                const int32_t* frame_width) {
  const Geometry& g = e->geo;
  cudaStream_t s = e->stream;
  const int64_t n_pad = g.n_padded(), cells = g.n_cells();
  std::vector<uint32_t> wall_flat;
  std::vector<double> wall_u;
  for (int64_t p = 0; p < n_pad; ++p) {
    if (tags_pad[p] != kUbbT) continue;
    if (!ubb_u_pad) return fail(SLBM_ECONFIG, "UBB tags present but no wall velocity array");
    wall_flat.push_back(uint32_t(p));
    for (int a = 0; a < 3; ++a) wall_u.push_back(a < g.dim ? ubb_u_pad[p * g.dim + a] : 0.0);
  }
  uint8_t* d_tags = nullptr;
  SLBM_CUDA_TRY(cudaMalloc(&d_tags, n_pad));
  SLBM_CUDA_TRY(cudaMemcpyAsync(d_tags, tags_pad, n_pad, cudaMemcpyHostToDevice, s));
  SLBM_CUDA_TRY(cudaMalloc(&e->dense_mask, cells * sizeof(uint32_t)));
  e->device_bytes += cells * 4;
  unsigned long long* d_cnt = nullptr;
  int* d_err = nullptr;
  SLBM_CUDA_TRY(cudaMalloc(&d_cnt, 2 * sizeof(unsigned long long)));
  SLBM_CUDA_TRY(cudaMalloc(&d_err, sizeof(int)));
  SLBM_CUDA_TRY(cudaMemsetAsync(d_cnt, 0, 2 * sizeof(unsigned long long), s));
  SLBM_CUDA_TRY(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  { k_dense_mask<<<grid_of(cells, 256), 256, 0, s>>>(d_tags, g, e->dirs, e->dense_mask, d_cnt,
                                                    d_err); slbm::count_launch(); }
  unsigned long long n_ubb = 0;
  int h_err = 0;
  SLBM_CUDA_TRY(cudaMemcpyAsync(&n_ubb, d_cnt, sizeof(n_ubb), cudaMemcpyDeviceToHost, s));
  SLBM_CUDA_TRY(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  SLBM_CUDA_TRY(cudaStreamSynchronize(s));
  if (h_err) {
    cudaFree(d_tags);
    return fail(SLBM_ECONFIG, "outlet boundaries are not supported by the dense engine");
  }
  e->n_dense_ubb = int64_t(n_ubb);
  if (n_ubb) {
    uint32_t* d_wf = nullptr;
    double* d_wu = nullptr;
    uint64_t* keys = nullptr;
    double* corr = nullptr;
    SLBM_CUDA_TRY(cudaMalloc(&d_wf, wall_flat.size() * 4));
    SLBM_CUDA_TRY(cudaMalloc(&d_wu, wall_u.size() * 8));
    SLBM_CUDA_TRY(cudaMemcpyAsync(d_wf, wall_flat.data(), wall_flat.size() * 4,
                                  cudaMemcpyHostToDevice, s));
    SLBM_CUDA_TRY(cudaMemcpyAsync(d_wu, wall_u.data(), wall_u.size() * 8, cudaMemcpyHostToDevice, s));
    SLBM_CUDA_TRY(cudaMalloc(&keys, n_ubb * 8));
    SLBM_CUDA_TRY(cudaMalloc(&corr, n_ubb * 8));
    SLBM_CUDA_TRY(cudaMalloc(&e->dense_ubb_key, n_ubb * 8));
    SLBM_CUDA_TRY(cudaMalloc(&e->dense_ubb_corr, n_ubb * 8));
    { k_dense_ubb<<<grid_of(cells, 256), 256, 0, s>>>(d_tags, g, e->dirs, e->dense_mask, d_wf, d_wu,
                                                     int64_t(wall_flat.size()), d_cnt + 1, keys,
                                                     corr); slbm::count_launch(); }
    size_t tmp_bytes = 0;
    SLBM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, e->dense_ubb_key, corr,
                                                  e->dense_ubb_corr, int64_t(n_ubb), 0, 64, s));
    void* tmp = nullptr;
    SLBM_CUDA_TRY(cudaMalloc(&tmp, tmp_bytes));
    SLBM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, e->dense_ubb_key, corr,
                                                  e->dense_ubb_corr, int64_t(n_ubb), 0, 64, s));
    SLBM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(tmp);
    cudaFree(keys);
    cudaFree(corr);
    cudaFree(d_wf);
    cudaFree(d_wu);
  }
  if (frame_width) {
    for (int k = 0; k < 3; ++k)
      e->dense_frame_w[k] = k < g.dim ? std::min<int32_t>(frame_width[k], g.n[k]) : 1;
    // interior / frame sizes in box cells (dense.py:330-341)
    int64_t inner = 1;
    for (int k = 0; k < g.dim; ++k) inner *= std::max<int64_t>(g.n[k] - 2 * e->dense_frame_w[k], 0);
    e->n_interior = inner;
    e->n_frame = cells - inner;
    e->has_split = true;
  }
  cudaFree(d_cnt);
  cudaFree(d_err);
  cudaFree(d_tags);
  e->total_slots = int64_t(e->q) * n_pad;
  e->phys_slots = e->total_slots;  // slot = q * npad + p is also the device address
  for (int q = 0; q <= e->q && q < 28; ++q) e->base[q] = e->pbase[q] = int64_t(q) * n_pad;
  if (e->total_slots >= (int64_t(1) << 32))
    return fail(SLBM_ECONFIG, "dense block too large: q * padded cells must be < 2^32");
  return SLBM_OK;
}

int dense_step(SlbmEngine* e, int phase) {
  DenseArgs a = dense_args(e);
  a.phase = phase;
  const int kind = e->pattern == SLBM_PULL ? 0 : (e->parity == SLBM_EVEN ? 1 : 2);
  const int64_t n_cta = e->geo.n[1] * e->geo.n[2] * ((e->geo.n[0] + 127) / 128);
  if (n_cta >= (int64_t(1) << 31)) return fail(SLBM_ECONFIG, "dense block too large for one grid");
  const dim3 grid{unsigned(n_cta), 1u, 1u};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t ahead = uint32_t(sms);  // ~ a quarter wave of 128-thread CTAs
  // speculative loads pay off when few box cells are solid
  const bool spec = double(e->n_fluid) >= 0.75 * double(e->geo.n_cells());
  DenseOddArgs oa{};
  oa.pdf = a.pdf;
  oa.mask = a.mask;
  oa.X = uint32_t(e->geo.n[0]);
  oa.Y = uint32_t(e->geo.n[1]);
  oa.PX = uint32_t(e->geo.p[0]);
  oa.PY = uint32_t(e->geo.p[1]);
  oa.offz = uint32_t(e->geo.off[2]);
  for (int q = 0; q < 28 && q < e->q; ++q) oa.base[q] = uint32_t(q) * uint32_t(a.npad);
  oa.omega = a.omega;
  oa.lam = a.lam;
  oa.hr = a.hr;
  oa.bad = a.bad;
  oa.step = a.step;
  with_lattice(e->q, [&](auto lat) {
    using L = decltype(lat);
    auto go = [&](auto model) {
      constexpr int M = decltype(model)::value;
      auto launch = [&](auto sp) {
        constexpr bool S = decltype(sp)::value;
        if (kind == 0)
          { k_dense<L, M, 0, S><<<grid, 128, 0, e->stream>>>(a, ahead); slbm::count_launch(); }
        else if (kind == 1)
          { k_dense<L, M, 1, S><<<grid, 128, 0, e->stream>>>(a, ahead); slbm::count_launch(); }
        else if (phase == SLBM_PHASE_ALL && e->tune.dense_lean_odd)
          { k_dense_odd<L, M><<<grid, 128, 0, e->stream>>>(oa); slbm::count_launch(); }
        else
          { k_dense<L, M, 2, S><<<grid, 128, 0, e->stream>>>(a, ahead); slbm::count_launch(); }
      };
      if (spec)
        launch(std::true_type{});
      else
        launch(std::false_type{});
    };
    if (e->model == SLBM_SRT)
      go(std::integral_constant<int, SLBM_SRT>{});
    else if (e->model == SLBM_TRT)
      go(std::integral_constant<int, SLBM_TRT>{});
    else if constexpr (L::Q == 27) {
      if (e->model == SLBM_CUMULANT)
        go(std::integral_constant<int, SLBM_CUMULANT>{});
      else
        go(std::integral_constant<int, SLBM_CUMULANT_GEN>{});
    }
  });
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

// init: NaN everywhere, resting weights in every box cell, values at fluid
int dense_init(SlbmEngine* e, const double* dev_values) {
  const int64_t npad = e->geo.n_padded();
  SLBM_TRY(launch_fill(e->pdf, e->total_slots, NAN, e->stream));
  if (e->tmp) SLBM_TRY(launch_fill(e->tmp, e->total_slots, NAN, e->stream));
  { k_dense_weights<<<grid_of(e->geo.n_cells(), 256), 256, 0, e->stream>>>(e->pdf, e->geo, npad,
                                                                          e->dirs); slbm::count_launch(); }
  { k_dense_scatter<<<grid_of(e->n_fluid, 256), 256, 0, e->stream>>>(e->pdf, e->x_flat, e->n_fluid,
                                                                    npad, e->q, dev_values); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  e->parity = SLBM_EVEN;
  return SLBM_OK;
}

int dense_canonical(SlbmEngine* e, double* dev_values) {
  const int odd = (e->pattern == SLBM_AA && e->parity == SLBM_ODD) ? 1 : 0;
  { k_dense_gather<<<grid_of(e->n_fluid, 256), 256, 0, e->stream>>>(
      e->pdf, e->x_flat, e->n_fluid, e->geo.n_padded(), e->dirs, odd, dev_values); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}


}  // namespace slbm
