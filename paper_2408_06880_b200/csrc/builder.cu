// GPU list builder: fluid enumeration, index list with no-slip folding,
// moving-wall (UBB) and halo (ghost) slot allocation, ownership check and
// interior/frame split.  Reproduces pkg/src/slbm/sparse.py:72-195 bit for
// bit:
//
//   cells      fluid cells of the interior in C order over (z, y, x)
//              (sparse.py:72-76)  -> cub::DeviceSelect over the interior
//   pass 1     upwind tag of every (q >= 1, cell) read, wrapping periodic
//              axes first (sparse.py:110-126) -> per-q UBB / ghost counts
//   base       prefix sum of N_F + n_ubb[q] + n_ghost[q] (sparse.py:128-137)
//   pass 2     FLUID  -> base[q] + cid(upwind)             (sparse.py:149-152)
//              NOSLIP -> base[inv q] + cid                  (:154-155)
//              UBB    -> base[q] + N_F + rank in cid order  (:157-164)
//              EXCH.  -> base[q] + N_F + n_ubb[q] + rank by (ring offset,
//                        padded flat index)                 (:166-179)
//   unique     every slot owned by exactly one (direction, cell) read
//              (:182-185) -> atomic bitset
//   split      frame = within the per-axis width of a face (flags.py:83-108)
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <climits>
#include <cstring>

#include "engine.cuh"
#include "sweep.cuh"

namespace slbm {
namespace {

constexpr uint8_t kFluid = 0, kNoslip = 1, kUbb = 2, kExchange = 3, kOutlet = 4;
constexpr int kCounters = 3 * 27;  // per q: UBB, ghost, outlet

__host__ __device__ inline int64_t wrap(int64_t v, int64_t n) {
  int64_t r = v % n;
  return r < 0 ? r + n : r;
}

struct Upwind {
  Geometry g;
  DirTable d;
  // padded flat index of the cell a direction-q read of (x, y, z) comes from
  __device__ __forceinline__ int64_t operator()(int q, int64_t x, int64_t y, int64_t z) const {
    int64_t s[3] = {x - d.c[q][0], y - d.c[q][1], z - d.c[q][2]};
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (g.periodic[a]) s[a] = wrap(s[a], g.n[a]);
    return g.padded_flat(s[0], s[1], s[2]);
  }
};

struct InteriorToPadded {
  Geometry g;
  __host__ __device__ uint32_t operator()(int64_t i) const {
    int64_t x = i % g.n[0];
    int64_t r = i / g.n[0];
    int64_t y = r % g.n[1];
    int64_t z = r / g.n[1];
    return uint32_t(g.padded_flat(x, y, z));
  }
};

struct FluidAt {
  const uint8_t* tags;
  __device__ bool operator()(uint32_t p) const { return tags[p] == kFluid; }
};

// selects cells whose direction-q read hits tag `want`
struct ReadsTag {
  const uint8_t* tags;
  const uint32_t* x_flat;
  Upwind up;
  int q;
  uint8_t want;
  __device__ bool operator()(uint32_t c) const {
    int64_t x, y, z;
    up.g.coords(x_flat[c], x, y, z);
    return tags[up(q, x, y, z)] == want;
  }
};

// frame cell: within lo[a] of the low face or hi[a] of the high face of any
// axis (flags.py:83-108 uses lo == hi)
struct InFrame {
  const uint32_t* x_flat;
  Geometry g;
  int32_t lo[3], hi[3];
  bool want;
  __device__ bool operator()(uint32_t c) const {
    int64_t v[3];
    g.coords(x_flat[c], v[0], v[1], v[2]);
    bool in = false;
    for (int a = 0; a < g.dim; ++a) in |= (v[a] < lo[a]) || (v[a] >= g.n[a] - hi[a]);
    return in == want;
  }
};

// one bit per cell, set for frame cells: the interior sweep runs over all
// cells in cid order and skips the set bits (one broadcast word per warp)
// instead of reading an explicit interior cell list (4 B/cell + a dependent
// load in front of the index list)
__global__ void k_frame_bits(InFrame fr, int64_t n, uint32_t* bits) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool in = c < n && fr(uint32_t(c));
  const unsigned word = __ballot_sync(0xffffffffu, in);
  if ((threadIdx.x & 31) == 0 && c < n) bits[c >> 5] = word;
}

__global__ void k_cid_map(const uint32_t* x_flat, int64_t n, int32_t* cid_map) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) cid_map[x_flat[i]] = int32_t(i);
}

// pass 1: per-direction UBB / ghost counts and sanity of every upwind tag
__global__ void k_count(const uint8_t* tags, const int32_t* cid_map, const uint32_t* x_flat,
                        int64_t n, Upwind up, unsigned long long* counts, int* err) {
  __shared__ unsigned int s_cnt[kCounters];
  for (int i = threadIdx.x; i < kCounters; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
       c += int64_t(gridDim.x) * blockDim.x) {
    int64_t x, y, z;
    up.g.coords(x_flat[c], x, y, z);
    for (int q = 1; q < up.d.q; ++q) {
      int64_t p = up(q, x, y, z);
      uint8_t tag = tags[p];
      if (tag == kUbb) {
        atomicAdd(&s_cnt[3 * q], 1u);
      } else if (tag == kExchange) {
        atomicAdd(&s_cnt[3 * q + 1], 1u);
      } else if (tag == kOutlet) {
        atomicAdd(&s_cnt[3 * q + 2], 1u);
      } else if (tag == kFluid) {
        if (cid_map[p] < 0) atomicOr(err, 1);
      } else if (tag != kNoslip) {
        atomicOr(err, 2);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kCounters; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(&counts[i], (unsigned long long)s_cnt[i]);
}

struct Bases {
  uint32_t b[28];
};

// pass 2 for in-list reads: FLUID -> neighbour slot, NOSLIP -> own opposite
// slot; UBB / EXCHANGE entries are assigned by the ranked passes below
__global__ void k_fill(const uint8_t* tags, const int32_t* cid_map, const uint32_t* x_flat,
                       int64_t n, Upwind up, Bases bases, uint32_t* idx) {
  int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n) return;
  int64_t x, y, z;
  up.g.coords(x_flat[c], x, y, z);
  for (int q = 1; q < up.d.q; ++q) {
    int64_t p = up(q, x, y, z);
    uint8_t tag = tags[p];
    uint32_t v = 0xffffffffu;
    if (tag == kFluid)
      v = bases.b[q] + uint32_t(cid_map[p]);
    else if (tag == kNoslip)
      v = bases.b[up.d.inv[q]] + uint32_t(c);
    idx[(q - 1) * n + c] = v;
  }
}

__device__ int64_t find_sorted(const uint32_t* keys, int64_t n, uint32_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < n && keys[lo] == key) ? lo : -1;
}

// UBB reads of direction q, `sel` = cells in cid order (sparse.py:157-164)
__global__ void k_ubb_assign(const uint32_t* sel, int64_t cnt, int q, const uint32_t* x_flat,
                             int64_t n, Upwind up, Bases bases, const uint32_t* wall_flat,
                             const double* wall_u, int64_t n_wall, uint32_t* idx,
                             uint32_t* ubb_slot, uint32_t* ubb_partner, double* ubb_corr,
                             int* err) {
  int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= cnt) return;
  uint32_t c = sel[k];
  uint32_t slot = bases.b[q] + uint32_t(n) + uint32_t(k);
  idx[(q - 1) * n + c] = slot;
  ubb_slot[k] = slot;
  ubb_partner[k] = bases.b[up.d.inv[q]] + c;
  int64_t x, y, z;
  up.g.coords(x_flat[c], x, y, z);
  uint32_t p = uint32_t(up(q, x, y, z));
  int64_t at = find_sorted(wall_flat, n_wall, p);
  if (at < 0) {
    atomicOr(err, 4);
    return;
  }
  // core.py:173-188: cu accumulated from 0 by +/- u_a; 2*w*rho_w*cu/cs2
  double cu = 0.0;
  for (int a = 0; a < up.g.dim; ++a) {
    if (up.d.c[q][a] == 1) cu = cu + wall_u[at * 3 + a];
    if (up.d.c[q][a] == -1) cu = cu - wall_u[at * 3 + a];
  }
  const double cs2 = 1.0 / 3.0;
  ubb_corr[k] = (((2.0 * up.d.w[q]) * 1.0) * cu) / cs2;
}

// OUTLET reads of direction q, `sel` = cells in cid order; the prescribed
// density sits in component 0 of the wall table
__global__ void k_outlet_assign(const uint32_t* sel, int64_t cnt, int q, const uint32_t* x_flat,
                                int64_t n, Upwind up, Bases bases, uint32_t first,
                                const uint32_t* wall_flat, const double* wall_u, int64_t n_wall,
                                uint32_t* idx, uint32_t* o_slot, uint32_t* o_partner,
                                uint32_t* o_cell, uint8_t* o_dir, double* o_rho, int* err) {
  int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= cnt) return;
  uint32_t c = sel[k];
  uint32_t slot = first + uint32_t(k);
  idx[(q - 1) * n + c] = slot;
  o_slot[k] = slot;
  o_partner[k] = bases.b[up.d.inv[q]] + c;
  o_cell[k] = c;
  o_dir[k] = uint8_t(q);
  int64_t x, y, z;
  up.g.coords(x_flat[c], x, y, z);
  int64_t at = find_sorted(wall_flat, n_wall, uint32_t(up(q, x, y, z)));
  if (at < 0) {
    atomicOr(err, 4);
    return;
  }
  o_rho[k] = wall_u[at * 3];
}

// ghost keys: (ring offset of the upwind halo cell, its padded flat index)
__global__ void k_ghost_keys(const uint32_t* sel, int64_t cnt, int q, const uint32_t* x_flat,
                             Upwind up, uint64_t* keys) {
  int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= cnt) return;
  int64_t x, y, z;
  up.g.coords(x_flat[sel[k]], x, y, z);
  int64_t p = up(q, x, y, z);
  int64_t v[3];
  up.g.coords(p, v[0], v[1], v[2]);
  int sig = 0;
  for (int a = 0; a < 3; ++a) {
    int s = 0;
    if (a < up.g.dim) s = v[a] < 0 ? -1 : (v[a] >= up.g.n[a] ? 1 : 0);
    sig = sig * 3 + (s + 1);
  }
  keys[k] = (uint64_t(sig) << 32) | uint64_t(p);
}

__global__ void k_ghost_assign(const uint32_t* sorted_cells, int64_t cnt, int q, int64_t n,
                               uint32_t first_slot, uint32_t* idx) {
  int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= cnt) return;
  idx[(q - 1) * n + sorted_cells[k]] = first_slot + uint32_t(k);
}

// reference slot ids -> device addresses (group g: pbase[g] + slot - base[g])
struct SlotMap {
  uint32_t base[28], pbase[28];
  int q;
  __device__ uint32_t operator()(uint32_t slot) const {
    int g = 0;
    while (g + 1 < q && base[g + 1] <= slot) ++g;
    return pbase[g] + (slot - base[g]);
  }
};

// logical (Q-1) x n index list -> physical addresses in rows of `pitch`
__global__ void k_physical_idx(const uint32_t* in, int64_t n, int64_t pitch, int64_t rows,
                               SlotMap m, uint32_t* out) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * n) return;
  const int64_t r = t / n, c = t - r * n;
  out[idx_offset(rows == 18, uint32_t(pitch), uint32_t(r), uint32_t(c))] = m(in[t]);
}

// physical rows of `pitch` -> the reference's contiguous (Q-1) x n slot ids
__global__ void k_logical_idx(const uint32_t* in, int64_t n, int64_t pitch, int64_t rows,
                              SlotMap inv, uint32_t* out) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * n) return;
  const int64_t r = t / n, c = t - r * n;
  out[t] = inv(in[idx_offset(rows == 18, uint32_t(pitch), uint32_t(r), uint32_t(c))]);
}

__global__ void k_physical_inplace(uint32_t* v, int64_t n, SlotMap m) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) v[t] = m(v[t]);
}

__global__ void k_unique(const uint32_t* idx, int64_t n, int q, uint64_t total,
                         unsigned int* bits, int* err) {
  int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= int64_t(q) * n) return;
  uint64_t slot = (t < n) ? uint64_t(t) : uint64_t(idx[t - n]);
  if (slot >= total) {
    atomicOr(err, 8);
    return;
  }
  unsigned int bit = 1u << (slot & 31);
  unsigned int old = atomicOr(&bits[slot >> 5], bit);
  if (old & bit) atomicOr(err, 16);
}

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  return unsigned(std::max<int64_t>(g, 1));
}

// cub select into `out` (capacity n); returns the count on the host
template <class InIt, class Pred, class T>
int select_if(InIt in, T* out, int64_t n, Pred pred, int64_t* count, cudaStream_t s) {
  int64_t* d_num = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&d_num, sizeof(int64_t), s));
  size_t tmp_bytes = 0;
  SLBM_CUDA_TRY(cub::DeviceSelect::If(nullptr, tmp_bytes, in, out, d_num, n, pred, s));
  void* tmp = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  SLBM_CUDA_TRY(cub::DeviceSelect::If(tmp, tmp_bytes, in, out, d_num, n, pred, s));
  SLBM_CUDA_TRY(cudaMemcpyAsync(count, d_num, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SLBM_CUDA_TRY(cudaFreeAsync(tmp, s));
  SLBM_CUDA_TRY(cudaFreeAsync(d_num, s));
  SLBM_CUDA_TRY(cudaStreamSynchronize(s));
  return SLBM_OK;
}

template <class T>
int dalloc(SlbmEngine* e, T** p, int64_t count) {
  size_t bytes = size_t(std::max<int64_t>(count, 1)) * sizeof(T);
  cudaError_t err = cudaMalloc(p, bytes);
  if (err != cudaSuccess)
    return fail(SLBM_ECUDA, std::string("cudaMalloc of ") + std::to_string(bytes) +
                                " bytes failed: " + cudaGetErrorString(err));
  e->device_bytes += int64_t(bytes);
  return SLBM_OK;
}

std::string dims_str(const Geometry& g) {
  std::string s = "(" + std::to_string(g.n[0]) + ", " + std::to_string(g.n[1]);
  if (g.dim == 3) s += ", " + std::to_string(g.n[2]);
  return s + ")";
}

}  // namespace

// fluid cells in C order over (z, y, x) -> e->x_flat, e->n_fluid (dense engine)
int enumerate_fluid(SlbmEngine* e, const uint8_t* tags_pad) {
  const Geometry& g = e->geo;
  cudaStream_t s = e->stream;
  const int64_t n_pad = g.n_padded(), n_cells = g.n_cells();
  if (n_pad >= (int64_t(1) << 32) - 1)
    return fail(SLBM_ECONFIG, "padded block has >= 2^32 cells; use smaller blocks");
  uint8_t* d_tags = nullptr;
  uint32_t* sel = nullptr;
  SLBM_CUDA_TRY(cudaMalloc(&d_tags, n_pad));
  SLBM_CUDA_TRY(cudaMemcpyAsync(d_tags, tags_pad, n_pad, cudaMemcpyHostToDevice, s));
  SLBM_CUDA_TRY(cudaMalloc(&sel, sizeof(uint32_t) * std::max<int64_t>(n_cells, 1)));
  auto interior = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0),
                                                  InteriorToPadded{g});
  int64_t n_fluid = 0;
  SLBM_TRY(select_if(interior, sel, n_cells, FluidAt{d_tags}, &n_fluid, s));
  if (n_fluid == 0) {
    cudaFree(sel);
    cudaFree(d_tags);
    return fail(SLBM_EEMPTY, "block " + dims_str(g) + " has no fluid cells");
  }
  e->n_fluid = n_fluid;
  SLBM_TRY(dalloc(e, &e->x_flat, n_fluid));
  SLBM_CUDA_TRY(cudaMemcpyAsync(e->x_flat, sel, n_fluid * sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, s));
  SLBM_CUDA_TRY(cudaStreamSynchronize(s));
  cudaFree(sel);
  cudaFree(d_tags);
  return SLBM_OK;
}

int build_lists(SlbmEngine* e, const uint8_t* tags_pad, const double* ubb_u_pad,
                const int32_t* frame_width) {
  const Geometry& g = e->geo;
  const DirTable& d = e->dirs;
  cudaStream_t s = e->stream;
  const int64_t n_pad = g.n_padded();
  if (n_pad >= (int64_t(1) << 32) - 1)
    return fail(SLBM_ECONFIG, "padded block has >= 2^32 cells; use smaller blocks");

  // moving-wall velocity table: padded positions tagged UBB, ascending
  std::vector<uint32_t> wall_flat;
  std::vector<double> wall_u;
  for (int64_t p = 0; p < n_pad; ++p) {
    if (tags_pad[p] != kUbb && tags_pad[p] != kOutlet) continue;
    if (!ubb_u_pad)
      return fail(SLBM_ECONFIG, "UBB/OUTLET tags present but no wall velocity/density array");
    wall_flat.push_back(uint32_t(p));
    for (int a = 0; a < 3; ++a) wall_u.push_back(a < g.dim ? ubb_u_pad[p * g.dim + a] : 0.0);
  }

  uint8_t* d_tags = nullptr;
  SLBM_CUDA_TRY(cudaMalloc(&d_tags, n_pad));
  SLBM_CUDA_TRY(cudaMemcpyAsync(d_tags, tags_pad, n_pad, cudaMemcpyHostToDevice, s));

  // -- fluid enumeration (sparse.py:72-76) --
  const int64_t n_cells = g.n_cells();
  uint32_t* sel_buf = nullptr;  // reused selection buffer, capacity max(n_cells, ...)
  SLBM_CUDA_TRY(cudaMalloc(&sel_buf, sizeof(uint32_t) * std::max<int64_t>(n_cells, 1)));
  auto interior = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0),
                                                  InteriorToPadded{g});
  int64_t n_fluid = 0;
  SLBM_TRY(select_if(interior, sel_buf, n_cells, FluidAt{d_tags}, &n_fluid, s));
  if (n_fluid == 0) {
    cudaFree(sel_buf);
    cudaFree(d_tags);
    return fail(SLBM_EEMPTY, "block " + dims_str(g) + " has no fluid cells");
  }
  e->n_fluid = n_fluid;
  const int64_t n = n_fluid;
  SLBM_TRY(dalloc(e, &e->x_flat, n));
  SLBM_CUDA_TRY(cudaMemcpyAsync(e->x_flat, sel_buf, n * sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, s));
  SLBM_TRY(dalloc(e, &e->cid_map, n_pad));
  SLBM_CUDA_TRY(cudaMemsetAsync(e->cid_map, 0xff, n_pad * sizeof(int32_t), s));
  { k_cid_map<<<grid_for(n, 256), 256, 0, s>>>(e->x_flat, n, e->cid_map); slbm::count_launch(); }

  // -- pass 1: counts --
  Upwind up{g, d};
  unsigned long long* d_counts = nullptr;
  int* d_err = nullptr;
  SLBM_CUDA_TRY(cudaMalloc(&d_counts, kCounters * sizeof(unsigned long long)));
  SLBM_CUDA_TRY(cudaMalloc(&d_err, sizeof(int)));
  SLBM_CUDA_TRY(cudaMemsetAsync(d_counts, 0, kCounters * sizeof(unsigned long long), s));
  SLBM_CUDA_TRY(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  {
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, e->device);
    unsigned blocks = std::min<unsigned>(grid_for(n, 256), unsigned(dev_sms) * 8);
    { k_count<<<blocks, 256, 0, s>>>(d_tags, e->cid_map, e->x_flat, n, up, d_counts, d_err); slbm::count_launch(); }
  }
  unsigned long long h_counts[kCounters];
  int h_err = 0;
  SLBM_CUDA_TRY(cudaMemcpyAsync(h_counts, d_counts, sizeof(h_counts), cudaMemcpyDeviceToHost, s));
  SLBM_CUDA_TRY(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  SLBM_CUDA_TRY(cudaStreamSynchronize(s));
  auto cleanup = [&]() {
    cudaFree(d_counts);
    cudaFree(d_err);
    cudaFree(sel_buf);
    cudaFree(d_tags);
  };
  if (h_err & 1) {
    cleanup();
    return fail(SLBM_ECONFIG, "fluid upwind cell missing from cell list (fluid tag in the ring "
                              "of a non-periodic axis)");
  }
  if (h_err & 2) {
    cleanup();
    return fail(SLBM_ECONFIG, "unknown tag value upwind of a fluid cell");
  }

  // -- slot budget (sparse.py:128-137) --
  int64_t total = 0;
  e->base[0] = 0;
  // outlet slots (extension; no reference counterpart) follow the ghost
  // slots, so blocks without outlets keep the reference layout exactly
  for (int q = 0; q < d.q; ++q) {
    int64_t nu = q ? int64_t(h_counts[3 * q]) : 0;
    int64_t ng = q ? int64_t(h_counts[3 * q + 1]) : 0;
    int64_t no = q ? int64_t(h_counts[3 * q + 2]) : 0;
    e->n_ubb_q[q] = nu;
    e->n_ghost_q[q] = ng;
    e->n_out_q[q] = no;
    total += n + nu + ng + no;
    e->base[q + 1] = total;
  }
  e->total_slots = total;
  e->n_ubb = e->n_ghost = e->n_out = 0;
  e->ubb_off[0] = e->ghost_off[0] = e->out_off[0] = 0;
  for (int q = 0; q < d.q; ++q) {
    e->n_ubb += e->n_ubb_q[q];
    e->n_ghost += e->n_ghost_q[q];
    e->n_out += e->n_out_q[q];
    e->ubb_off[q + 1] = e->n_ubb;
    e->ghost_off[q + 1] = e->n_ghost;
    e->out_off[q + 1] = e->n_out;
  }
  if (total >= (int64_t(1) << 32)) {
    cleanup();
    return fail(SLBM_ECONFIG, std::to_string(total) +
                                  " slots exceed the 4-byte location table range");
  }
  Bases bases{};
  for (int q = 0; q <= d.q && q < 28; ++q) bases.b[q] = uint32_t(e->base[q]);

  // -- pass 2: index list --
  SLBM_TRY(dalloc(e, &e->idx, int64_t(d.q - 1) * n));
  { k_fill<<<grid_for(n, 256), 256, 0, s>>>(d_tags, e->cid_map, e->x_flat, n, up, bases, e->idx); slbm::count_launch(); }

  SLBM_TRY(dalloc(e, &e->ubb_slot, e->n_ubb));
  SLBM_TRY(dalloc(e, &e->ubb_partner, e->n_ubb));
  SLBM_TRY(dalloc(e, &e->ubb_corr, e->n_ubb));
  uint32_t* d_wall_flat = nullptr;
  double* d_wall_u = nullptr;
  if (e->n_ubb || e->n_out) {
    SLBM_CUDA_TRY(cudaMalloc(&d_wall_flat, wall_flat.size() * sizeof(uint32_t)));
    SLBM_CUDA_TRY(cudaMalloc(&d_wall_u, wall_u.size() * sizeof(double)));
    SLBM_CUDA_TRY(cudaMemcpyAsync(d_wall_flat, wall_flat.data(),
                                  wall_flat.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    SLBM_CUDA_TRY(cudaMemcpyAsync(d_wall_u, wall_u.data(), wall_u.size() * sizeof(double),
                                  cudaMemcpyHostToDevice, s));
  }
  for (int q = 1; q < d.q; ++q) {
    if (!e->n_ubb_q[q]) continue;
    int64_t cnt = 0;
    SLBM_TRY(select_if(thrust::counting_iterator<uint32_t>(0), sel_buf, n,
                       ReadsTag{d_tags, e->x_flat, up, q, kUbb}, &cnt, s));
    { k_ubb_assign<<<grid_for(cnt, 256), 256, 0, s>>>(
        sel_buf, cnt, q, e->x_flat, n, up, bases, d_wall_flat, d_wall_u,
        int64_t(wall_flat.size()), e->idx, e->ubb_slot + e->ubb_off[q],
        e->ubb_partner + e->ubb_off[q], e->ubb_corr + e->ubb_off[q], d_err); slbm::count_launch(); }
  }

  SLBM_TRY(dalloc(e, &e->ghost_key, e->n_ghost));
  e->ghost_key_host.assign(size_t(e->n_ghost), 0);
  if (e->n_ghost) {
    int64_t max_g = 0;
    for (int q = 1; q < d.q; ++q) max_g = std::max(max_g, e->n_ghost_q[q]);
    uint64_t *k_in = nullptr, *k_out = nullptr;
    uint32_t* c_out = nullptr;
    SLBM_CUDA_TRY(cudaMalloc(&k_in, max_g * sizeof(uint64_t)));
    SLBM_CUDA_TRY(cudaMalloc(&k_out, max_g * sizeof(uint64_t)));
    SLBM_CUDA_TRY(cudaMalloc(&c_out, max_g * sizeof(uint32_t)));
    for (int q = 1; q < d.q; ++q) {
      if (!e->n_ghost_q[q]) continue;
      int64_t cnt = 0;
      SLBM_TRY(select_if(thrust::counting_iterator<uint32_t>(0), sel_buf, n,
                         ReadsTag{d_tags, e->x_flat, up, q, kExchange}, &cnt, s));
      { k_ghost_keys<<<grid_for(cnt, 256), 256, 0, s>>>(sel_buf, cnt, q, e->x_flat, up, k_in); slbm::count_launch(); }
      size_t tmp_bytes = 0;
      SLBM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, sel_buf,
                                                    c_out, cnt, 0, 37, s));
      void* tmp = nullptr;
      SLBM_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
      SLBM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, sel_buf, c_out,
                                                    cnt, 0, 37, s));
      SLBM_CUDA_TRY(cudaFreeAsync(tmp, s));
      uint32_t first = uint32_t(e->base[q] + n + e->n_ubb_q[q]);
      { k_ghost_assign<<<grid_for(cnt, 256), 256, 0, s>>>(c_out, cnt, q, n, first, e->idx); slbm::count_launch(); }
      SLBM_CUDA_TRY(cudaMemcpyAsync(e->ghost_key + e->ghost_off[q], k_out,
                                    cnt * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    }
    SLBM_CUDA_TRY(cudaMemcpyAsync(e->ghost_key_host.data(), e->ghost_key,
                                  e->n_ghost * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    SLBM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(k_in);
    cudaFree(k_out);
    cudaFree(c_out);
  }

  // -- fixed-density outlet reads (extension): cid order within q --
  SLBM_TRY(dalloc(e, &e->out_slot, e->n_out));
  SLBM_TRY(dalloc(e, &e->out_partner, e->n_out));
  SLBM_TRY(dalloc(e, &e->out_cell, e->n_out));
  SLBM_TRY(dalloc(e, &e->out_dir, e->n_out));
  SLBM_TRY(dalloc(e, &e->out_rho, e->n_out));
  SLBM_TRY(dalloc(e, &e->out_u, 3 * e->n_out));
  if (e->n_out) SLBM_CUDA_TRY(cudaMemsetAsync(e->out_u, 0, 3 * e->n_out * sizeof(double), s));
  for (int q = 1; q < d.q; ++q) {
    if (!e->n_out_q[q]) continue;
    int64_t cnt = 0;
    SLBM_TRY(select_if(thrust::counting_iterator<uint32_t>(0), sel_buf, n,
                       ReadsTag{d_tags, e->x_flat, up, q, kOutlet}, &cnt, s));
    const uint32_t first = uint32_t(e->base[q] + n + e->n_ubb_q[q] + e->n_ghost_q[q]);
    const int64_t off = e->out_off[q];
    { k_outlet_assign<<<grid_for(cnt, 256), 256, 0, s>>>(
        sel_buf, cnt, q, e->x_flat, n, up, bases, first, d_wall_flat, d_wall_u,
        int64_t(wall_flat.size()), e->idx, e->out_slot + off, e->out_partner + off,
        e->out_cell + off, e->out_dir + off, e->out_rho + off, d_err); slbm::count_launch(); }
  }

  // -- ownership uniqueness (sparse.py:182-185) --
  {
    unsigned int* bits = nullptr;
    int64_t words = (total + 31) / 32;
    SLBM_CUDA_TRY(cudaMalloc(&bits, words * sizeof(unsigned int)));
    SLBM_CUDA_TRY(cudaMemsetAsync(bits, 0, words * sizeof(unsigned int), s));
    int64_t entries = int64_t(d.q) * n;
    { k_unique<<<grid_for(entries, 256), 256, 0, s>>>(e->idx, n, d.q, uint64_t(total), bits,
                                                     d_err); slbm::count_launch(); }
    SLBM_CUDA_TRY(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    SLBM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(bits);
  }
  if (d_wall_flat) cudaFree(d_wall_flat);
  if (d_wall_u) cudaFree(d_wall_u);
  if (h_err & 4) {
    cleanup();
    return fail(SLBM_ECONFIG, "UBB tag without a wall velocity entry");
  }
  if (h_err & (8 | 16)) {
    cleanup();
    return fail(SLBM_ECONFIG, "each slot must belong to exactly one (direction, cell) pair");
  }

  // -- device layout: 256-B aligned direction groups and idx rows --
  {
    SlotMap m{};
    m.q = d.q;
    int64_t pb = 0;
    for (int q = 0; q <= d.q; ++q) {
      e->pbase[q] = pb;
      if (q < d.q) pb += (e->base[q + 1] - e->base[q] + 31) / 32 * 32;
    }
    for (int q = 0; q <= d.q && q < 28; ++q) {
      m.base[q] = uint32_t(e->base[q]);
      m.pbase[q] = uint32_t(e->pbase[q]);
    }
    e->phys_slots = e->pbase[d.q];
    if (e->phys_slots >= (int64_t(1) << 32)) {
      cleanup();
      return fail(SLBM_ECONFIG, std::to_string(e->phys_slots) +
                                    " aligned slots exceed the 4-byte location table range");
    }
    e->idx_pitch = (n + 31) / 32 * 32;
    uint32_t* logical = e->idx;
    e->idx = nullptr;
    if (dalloc(e, &e->idx, int64_t(d.q - 1) * e->idx_pitch) != SLBM_OK) {
      cudaFree(logical);
      cleanup();
      return SLBM_ECUDA;
    }
    e->device_bytes -= int64_t(d.q - 1) * n * 4;  // the logical list is freed below
    const int64_t entries = int64_t(d.q - 1) * n;
    if (entries)
      { k_physical_idx<<<grid_for(entries, 256), 256, 0, s>>>(logical, n, e->idx_pitch, d.q - 1, m,
                                                            e->idx); slbm::count_launch(); }
    if (e->n_ubb) {
      { k_physical_inplace<<<grid_for(e->n_ubb, 256), 256, 0, s>>>(e->ubb_slot, e->n_ubb, m); slbm::count_launch(); }
      { k_physical_inplace<<<grid_for(e->n_ubb, 256), 256, 0, s>>>(e->ubb_partner, e->n_ubb, m); slbm::count_launch(); }
    }
    if (e->n_out) {
      { k_physical_inplace<<<grid_for(e->n_out, 256), 256, 0, s>>>(e->out_slot, e->n_out, m); slbm::count_launch(); }
      { k_physical_inplace<<<grid_for(e->n_out, 256), 256, 0, s>>>(e->out_partner, e->n_out, m); slbm::count_launch(); }
    }
    SLBM_CUDA_TRY(cudaGetLastError());
    SLBM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(logical);
  }

  // -- interior / frame split (sparse.py:80-88) --
  int st = SLBM_OK;
  if (frame_width) {
    int32_t w[3];
    for (int a = 0; a < 3; ++a) w[a] = a < g.dim ? frame_width[a] : 1;
    st = build_split(e, w, w, sel_buf);
  }
  SLBM_CUDA_TRY(cudaStreamSynchronize(s));
  cleanup();
  return st;
}

// frame cids (explicit list) and the interior (one cid range, or the
// complement of a frame bitmask) for per-face widths; `scratch` holds n cids
int build_split(SlbmEngine* e, const int32_t* lo_w, const int32_t* hi_w, uint32_t* scratch) {
  const Geometry& g = e->geo;
  const int64_t n = e->n_fluid;
  cudaStream_t s = e->stream;
  InFrame fr{e->x_flat, g, {0, 0, 0}, {0, 0, 0}, true};
  for (int a = 0; a < 3; ++a) {
    fr.lo[a] = std::min<int32_t>(lo_w[a], g.n[a]);
    fr.hi[a] = std::min<int32_t>(hi_w[a], g.n[a]);
  }
  if (e->frame_cids) cudaFree(e->frame_cids);
  if (e->frame_bits) cudaFree(e->frame_bits);
  e->frame_cids = nullptr;
  e->frame_bits = nullptr;
  int64_t nf = 0;
  SLBM_TRY(select_if(thrust::counting_iterator<uint32_t>(0), scratch, n, fr, &nf, s));
  SLBM_TRY(dalloc(e, &e->frame_cids, nf));
  SLBM_CUDA_TRY(cudaMemcpyAsync(e->frame_cids, scratch, nf * sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, s));
  e->n_frame = nf;
  e->n_interior = n - nf;
  e->has_split = true;
  // frame = a cid prefix + a cid suffix (faces only across z, e.g. slab
  // decompositions): the interior is one contiguous cid range and needs
  // no mask at all
  std::vector<uint32_t> h(size_t(std::max<int64_t>(nf, 1)));
  if (nf)
    SLBM_CUDA_TRY(cudaMemcpyAsync(h.data(), e->frame_cids, nf * 4, cudaMemcpyDeviceToHost, s));
  SLBM_CUDA_TRY(cudaStreamSynchronize(s));
  int64_t lo = 0;
  while (lo < nf && int64_t(h[lo]) == lo) ++lo;
  const int64_t hi = n - (nf - lo);
  bool ranged = true;
  for (int64_t k = lo; k < nf && ranged; ++k) ranged = int64_t(h[k]) == hi + (k - lo);
  if (ranged) {
    e->interior_lo = lo;
  } else {
    e->interior_lo = -1;
    SLBM_TRY(dalloc(e, &e->frame_bits, (n + 31) / 32));
    { k_frame_bits<<<grid_for(n, 256), 256, 0, s>>>(fr, n, e->frame_bits); slbm::count_launch(); }
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  SLBM_CUDA_TRY(cudaStreamSynchronize(s));
  return SLBM_OK;
}

int set_frame(SlbmEngine* e, const int32_t* lo_w, const int32_t* hi_w) {
  uint32_t* scratch = nullptr;
  SLBM_CUDA_TRY(cudaMalloc(&scratch, size_t(std::max<int64_t>(e->n_fluid, 1)) * 4));
  const int st = build_split(e, lo_w, hi_w, scratch);
  cudaFree(scratch);
  return st;
}

// the index list in the reference's layout (slot ids, contiguous rows)
int export_idx_logical(SlbmEngine* e, uint32_t* host) {
  const int64_t n = e->n_fluid, rows = e->q - 1;
  if (rows * n == 0) return SLBM_OK;
  SlotMap inv{};
  inv.q = e->q;
  for (int q = 0; q <= e->q && q < 28; ++q) {
    inv.base[q] = uint32_t(e->pbase[q]);  // search the device layout ...
    inv.pbase[q] = uint32_t(e->base[q]);  // ... map back to slot ids
  }
  uint32_t* tmp = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&tmp, size_t(rows * n) * 4, e->stream));
  { k_logical_idx<<<grid_for(rows * n, 256), 256, 0, e->stream>>>(e->idx, n, e->idx_pitch, rows, inv,
                                                                tmp); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  SLBM_TRY(copy_d2h(host, tmp, size_t(rows * n) * 4, e->device, e->stream));
  SLBM_CUDA_TRY(cudaFreeAsync(tmp, e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SLBM_OK;
}

}  // namespace slbm
