// AA step pair in one launch, temporally blocked in L2 (slbm_run on sparse
// engines without halo slots).
//
// The even step (index list, sparse.py:264-271) of cell n writes into the
// slots of n's neighbours; the odd step (cell-local, sparse.py:273-282) of
// cell c reads and rewrites only c's own slots.  So odd(c) may run as soon
// as even(n) has run for every n that touches one of c's slots — in cid
// order (z-major) those are within about one z-plane of c.  Run separately,
// both sweeps stream the whole state through HBM (376 + 304 B/cell, D3Q19);
// here the odd step of a tile follows the even steps it depends on by about
// one plane + one wave of CTAs, while the values the even step wrote are
// still in the 126 MB L2: the odd reads hit L2 and the even writes are
// overwritten there before they are evicted.  Same per-cell bodies as the
// two sweeps (sweep.cuh), same order per slot, hence bitwise identical.
//
// Scheduling.  Work items are tiles of 128 cells, even or odd; CTAs take
// items in a precomputed order by an atomic ticket (not blockIdx), so an
// item is only ever handed out after every item it may wait for: an odd
// tile waits (spinning, L2-scope acquire) only for even tiles earlier in the
// order, which are held by running CTAs that never wait — deadlock free
// with any residency.  Even tiles publish completion per chunk of 32 tiles
// (monotonic counters, no reset between launches); odd tiles wait on the
// chunk range their writers span (computed once from the index list).
// Tiles whose writers wrap around a periodic boundary wait for all even
// tiles and are ordered last.  The odd UBB / outlet refresh
// (sparse.py:301-304) of an entry runs inside the odd tile of its partner
// cell, after the wait.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>

#include "collide.cuh"
#include "engine.cuh"
#include "sweep.cuh"

namespace slbm {

struct PairPlan {
  int64_t n_tiles = 0, n_chunks = 0, n_items = 0;
  int32_t* sched = nullptr;      // ticket -> item: t >= 0 even tile t, ~j odd tile j
  uint32_t* dep = nullptr;       // per odd tile: first, last chunk it waits for (kAll: all)
  uint32_t* chunk_done = nullptr;  // even tiles completed per chunk, cumulative over launches
  uint32_t* ctl = nullptr;       // [0] ticket, [1] finished items, [2] launch count
  unsigned long long* total_done = nullptr;  // even tiles completed, cumulative
  uint32_t* ubb_perm = nullptr;  // UBB entries grouped by odd tile of the partner cell
  uint32_t* ubb_start = nullptr;  // n_tiles + 1
  uint32_t* out_perm = nullptr;
  uint32_t* out_start = nullptr;
};

namespace {

constexpr int kPT = 128;            // cells per tile = threads per CTA
constexpr uint32_t kChunk = 32;     // tiles per completion counter
constexpr uint32_t kWide = 256;     // chunk span above which a tile waits for all
constexpr uint32_t kAll = 0xffffffffu;

int g_pair = 1;        // knob 5: 0 off
int g_pair_slack = 0;  // knob 6: extra tiles between an odd tile's writers and it (0: one wave)
int g_pair_persist = 1;  // knob 7: persistent CTAs (1) or one CTA per item (0)

struct PairArgs {
  double* pdf;
  const uint32_t* idx;
  uint32_t n_fluid, idx_pitch, n_tiles, n_items;
  uint32_t base[28];
  double omega, lam;
  unsigned long long* bad;
  unsigned long long* step;
  const int32_t* sched;
  const uint32_t* dep;
  uint32_t* chunk_done;
  uint32_t* ctl;
  unsigned long long* total_done;
  const uint32_t* ubb_slot;
  const uint32_t* ubb_partner;
  const double* ubb_corr;
  const uint32_t* ubb_perm;
  const uint32_t* ubb_start;
  const uint32_t* out_slot;
  const uint32_t* out_partner;
  const uint32_t* out_cell;
  const uint8_t* out_dir;
  const double* out_rho;
  const double* out_u;
  const uint32_t* out_perm;
  const uint32_t* out_start;
  uint32_t ahead;  // idx prefetch distance in tiles
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kEnd = INT_MIN;  // no more items

// even step of tile t (k_index_sweep<kEven> body), then publish completion
template <class L, int MODEL>
__device__ __forceinline__ void pair_even(const PairArgs& a, uint32_t t, unsigned long long step) {
  const uint32_t first = t * kPT;
  prefetch_idx_ahead<L::Q - 1, kPT>(a.idx, a.idx_pitch, nullptr, a.n_fluid, first, a.ahead);
  const uint32_t c = first + threadIdx.x;
  if (c < a.n_fluid) {
    uint32_t s[L::Q];
    double v[L::Q];
    load_slots<L>(s, a.idx, a.idx_pitch, c);
    gather<L>(v, a.pdf, s);
    if (collide_scatter<L, MODEL, true>(v, s, a.pdf, a.pdf, a.base, c, a.omega, a.lam))
      atomicMin(a.bad, step);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&a.chunk_done[t / kChunk], 1u);
    atomicAdd(a.total_done, 1ull);
  }
}

// odd step of tile j: wait for its writers, odd refresh of the boundary
// entries of its cells, cell-local sweep (loads from L2: written this launch)
template <class L, int MODEL>
__device__ __forceinline__ void pair_odd(const PairArgs& a, uint32_t j, uint32_t epoch,
                                         unsigned long long step) {
  if (threadIdx.x < 32) {
    const uint32_t lo = a.dep[2 * j], hi = a.dep[2 * j + 1];
    if (lo == kAll) {
      const unsigned long long target = (unsigned long long)(epoch + 1) * a.n_tiles;
      if (threadIdx.x == 0)
        while (ld_acquire(a.total_done) < target) __nanosleep(256);
    } else {
      for (uint32_t k0 = lo; k0 <= hi; k0 += 32) {
        const uint32_t k = k0 + threadIdx.x;
        if (k <= hi) {
          const uint32_t size = min(kChunk, a.n_tiles - k * kChunk);
          const uint32_t target = (epoch + 1) * size;
          while (ld_acquire(&a.chunk_done[k]) < target) __nanosleep(64);
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for (uint32_t i = a.ubb_start[j] + threadIdx.x; i < a.ubb_start[j + 1]; i += kPT) {
    const uint32_t e = a.ubb_perm[i];
    a.pdf[a.ubb_partner[e]] = __ldcg(a.pdf + a.ubb_slot[e]) + a.ubb_corr[e];
  }
  if (a.out_start) {
    for (uint32_t i = a.out_start[j] + threadIdx.x; i < a.out_start[j + 1]; i += kPT) {
      const uint32_t e = a.out_perm[i];
      outlet_entry<L, true>(a.pdf, a.base, a.out_slot[e], a.out_partner[e], a.out_cell[e],
                            a.out_dir[e], a.out_rho[e], const_cast<double*>(a.out_u) + 3 * e,
                            SLBM_ODD);
    }
  }
  __syncthreads();
  const uint32_t c = j * kPT + threadIdx.x;
  if (c < a.n_fluid && cell_local<L, MODEL, true>(a.pdf, a.base, c, a.omega, a.lam))
    atomicMin(a.bad, step + 1);
}

__device__ __forceinline__ void pair_item_done(const PairArgs& a, uint32_t epoch,
                                               unsigned long long step) {
  __threadfence();
  if (atomicAdd(&a.ctl[1], 1u) == a.n_items - 1) {  // last item of the launch
    a.ctl[2] = epoch + 1;
    *a.step = step + 2;
    __threadfence();
  }
}

// one CTA per item
template <class L, int MODEL, int MINB>
__global__ void __launch_bounds__(kPT, MINB) k_pair(const PairArgs a) {
  __shared__ int s_item;
  __shared__ uint32_t s_epoch;
  __shared__ unsigned long long s_step;
  if (threadIdx.x == 0) {
    s_item = a.sched[atomicAdd(&a.ctl[0], 1u)];
    s_epoch = *(volatile uint32_t*)&a.ctl[2];
    s_step = *(volatile unsigned long long*)a.step;
  }
  __syncthreads();
  const int item = s_item;
  if (item >= 0)
    pair_even<L, MODEL>(a, uint32_t(item), s_step);
  else
    pair_odd<L, MODEL>(a, ~uint32_t(item), s_epoch, s_step);
  __syncthreads();
  if (threadIdx.x == 0) pair_item_done(a, s_epoch, s_step);
}

// persistent CTAs (one wave); thread 0 fetches the ticket two items ahead
// and the item one ahead while the CTA works, so no item starts with a
// dependent ticket + schedule round trip.  Per-CTA tickets increase, so a
// waiting item only ever waits for smaller tickets held by CTAs that are
// not waiting on it: deadlock free.
template <class L, int MODEL, int MINB>
__global__ void __launch_bounds__(kPT, MINB) k_pair_persist(const PairArgs a) {
  __shared__ int s_item;
  __shared__ uint32_t s_epoch;
  __shared__ unsigned long long s_step;
  uint32_t tk = 0;  // thread 0: ticket of the next item
  if (threadIdx.x == 0) {
    const uint32_t t0 = atomicAdd(&a.ctl[0], 1u);
    s_item = t0 < a.n_items ? a.sched[t0] : kEnd;
    tk = atomicAdd(&a.ctl[0], 1u);
    s_epoch = *(volatile uint32_t*)&a.ctl[2];
    s_step = *(volatile unsigned long long*)a.step;
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const unsigned long long step = s_step;
  for (;;) {
    const int item = s_item;
    if (item == kEnd) break;
    int nxt = kEnd;
    uint32_t tk2 = 0;
    if (threadIdx.x == 0) {
      tk2 = atomicAdd(&a.ctl[0], 1u);  // overshoots past n_items; reset before each launch
      if (tk < a.n_items) nxt = __ldg(a.sched + tk);
    }
    if (item >= 0)
      pair_even<L, MODEL>(a, uint32_t(item), step);
    else
      pair_odd<L, MODEL>(a, ~uint32_t(item), epoch, step);
    __syncthreads();
    if (threadIdx.x == 0) {
      pair_item_done(a, epoch, step);
      s_item = nxt;
      tk = tk2;
    }
    __syncthreads();
  }
}

// ---- plan construction (once per engine, on first use) ----

__device__ __forceinline__ int64_t owner_cell(const uint32_t* pbase, int q, uint32_t n_fluid,
                                              uint32_t slot) {
  int g = 0;
  while (g + 1 < q && pbase[g + 1] <= slot) ++g;
  const uint32_t off = slot - pbase[g];
  return off < n_fluid ? int64_t(off) : -1;
}

struct Base28 {
  uint32_t v[28];
};

// writer chunk range of every odd tile: even(n) touches slot idx[q][n] (and
// n's own rest slot); a cell slot belongs to its cell, an appended UBB /
// outlet slot to the cell of the entry's partner slot (sorted_slot/entry:
// the appended slots in ascending order with their entry index)
__global__ void k_pair_deps(const uint32_t* idx, uint32_t pitch, uint32_t n_fluid, int q,
                            Base28 pb, const uint32_t* ubb_sorted, const uint32_t* ubb_entry,
                            const uint32_t* ubb_partner, uint32_t n_ubb,
                            const uint32_t* out_sorted, const uint32_t* out_entry,
                            const uint32_t* out_partner, uint32_t n_out, uint32_t* lo,
                            uint32_t* hi) {
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= n_fluid) return;
  const uint32_t wchunk = (n / kPT) / kChunk;
  auto add = [&](int64_t c) {
    const uint32_t t = uint32_t(c / kPT);
    atomicMin(lo + t, wchunk);
    atomicMax(hi + t, wchunk);
  };
  add(n);
  auto lookup = [&](const uint32_t* sorted, const uint32_t* entry, const uint32_t* partner,
                    uint32_t m, uint32_t s) -> int64_t {
    uint32_t l = 0, h = m;
    while (l < h) {
      const uint32_t mid = (l + h) / 2;
      if (sorted[mid] < s) l = mid + 1; else h = mid;
    }
    if (l < m && sorted[l] == s) return owner_cell(pb.v, q, n_fluid, partner[entry[l]]);
    return -2;
  };
  for (int r = 0; r < q - 1; ++r) {
    const uint32_t s = idx[size_t(r) * pitch + n];
    int64_t c = owner_cell(pb.v, q, n_fluid, s);
    if (c < 0) c = lookup(ubb_sorted, ubb_entry, ubb_partner, n_ubb, s);
    if (c == -2) c = lookup(out_sorted, out_entry, out_partner, n_out, s);
    if (c >= 0) add(c);
  }
}

// dep ranges (wide -> kAll) and the order key: the even tile after which
// an odd tile is handed out
__global__ void k_pair_keys(uint32_t* lo, uint32_t* hi, uint32_t n_tiles, uint32_t slack,
                            uint32_t* key, uint32_t* val) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_tiles) return;
  uint32_t l = lo[j], h = hi[j];
  uint32_t k;
  if (h - l > kWide) {
    lo[j] = kAll;
    k = n_tiles - 1;
  } else {
    const uint64_t last = uint64_t(h + 1) * kChunk - 1 + slack;
    k = uint32_t(std::min<uint64_t>(last, n_tiles - 1));
  }
  key[j] = k;
  val[j] = j;
}

// merge: odd item of sorted rank r goes after even tile key[r]
__global__ void k_pair_sched(const uint32_t* key_sorted, const uint32_t* odd_sorted,
                             uint32_t n_tiles, int32_t* sched) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_tiles) return;
  // odd item of rank i
  sched[key_sorted[i] + 1 + i] = ~int32_t(odd_sorted[i]);
  // even tile i: preceded by the odd items whose key < i
  uint32_t l = 0, h = n_tiles;
  while (l < h) {
    const uint32_t mid = (l + h) / 2;
    if (key_sorted[mid] < i) l = mid + 1; else h = mid;
  }
  sched[i + l] = int32_t(i);
}

__global__ void k_pair_dep_pack(const uint32_t* lo, const uint32_t* hi, uint32_t n_tiles,
                                uint32_t* dep) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_tiles) return;
  dep[2 * j] = lo[j];
  dep[2 * j + 1] = hi[j];
}

// entries -> (tile of the partner cell, entry); slot copy for the lookup
__global__ void k_entry_keys(const uint32_t* slot, const uint32_t* partner, uint32_t n,
                             uint32_t n_fluid, int q, Base28 pb, uint32_t* tile, uint32_t* ent,
                             uint32_t* slot_key) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int64_t c = owner_cell(pb.v, q, n_fluid, partner[e]);
  tile[e] = c >= 0 ? uint32_t(c / kPT) : 0u;
  ent[e] = e;
  slot_key[e] = slot[e];
}

__global__ void k_tile_starts(const uint32_t* tile_sorted, uint32_t n, uint32_t n_tiles,
                              uint32_t* start) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > n_tiles) return;
  uint32_t l = 0, h = n;
  while (l < h) {
    const uint32_t mid = (l + h) / 2;
    if (tile_sorted[mid] < t) l = mid + 1; else h = mid;
  }
  start[t] = l;
}

__global__ void k_fill_u32(uint32_t* p, uint32_t n, uint32_t v) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

inline unsigned blocks(int64_t n, int b = 256) { return unsigned(std::max<int64_t>(1, (n + b - 1) / b)); }

int num_sms_pair() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// entries of one boundary program grouped by the odd tile of their partner
// cell (perm, start) and sorted by their appended slot (for k_pair_deps)
int group_entries(SlbmEngine* e, const uint32_t* slot, const uint32_t* partner, int64_t n,
                  const Base28& pb, uint32_t n_tiles, uint32_t** perm, uint32_t** start,
                  uint32_t** slot_sorted, uint32_t** slot_entry, cudaStream_t s) {
  uint32_t *tile = nullptr, *tile2 = nullptr, *ent = nullptr, *skey = nullptr, *ent2 = nullptr;
  const size_t nb = size_t(std::max<int64_t>(n, 1)) * 4;
  SLBM_CUDA_TRY(cudaMallocAsync(&tile, nb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&tile2, nb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&ent, nb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&ent2, nb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&skey, nb, s));
  SLBM_CUDA_TRY(cudaMalloc(perm, nb));
  SLBM_CUDA_TRY(cudaMalloc(start, size_t(n_tiles + 1) * 4));
  SLBM_CUDA_TRY(cudaMallocAsync(slot_sorted, nb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(slot_entry, nb, s));
  if (n > 0) {
    k_entry_keys<<<blocks(n), 256, 0, s>>>(slot, partner, uint32_t(n), uint32_t(e->n_fluid), e->q,
                                           pb, tile, ent, skey);
    size_t tb = 0, tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, tile, tile2, ent, *perm, int(n), 0, 32, s);
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, skey, *slot_sorted, ent, ent2, int(n), 0, 32, s);
    void* tmp = nullptr;
    SLBM_CUDA_TRY(cudaMallocAsync(&tmp, std::max(tb, tb2), s));
    cub::DeviceRadixSort::SortPairs(tmp, tb, tile, tile2, ent, *perm, int(n), 0, 32, s);
    cub::DeviceRadixSort::SortPairs(tmp, tb2, skey, *slot_sorted, ent, *slot_entry, int(n), 0, 32, s);
    SLBM_CUDA_TRY(cudaFreeAsync(tmp, s));
  }
  k_tile_starts<<<blocks(n_tiles + 1), 256, 0, s>>>(tile2, uint32_t(n), n_tiles, *start);
  SLBM_CUDA_TRY(cudaFreeAsync(tile, s));
  SLBM_CUDA_TRY(cudaFreeAsync(tile2, s));
  SLBM_CUDA_TRY(cudaFreeAsync(ent, s));
  SLBM_CUDA_TRY(cudaFreeAsync(ent2, s));
  SLBM_CUDA_TRY(cudaFreeAsync(skey, s));
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

int build_pair_plan(SlbmEngine* e) {
  cudaStream_t s = e->stream;
  auto* p = new PairPlan();
  e->pair = p;
  const uint32_t n_tiles = uint32_t((e->n_fluid + kPT - 1) / kPT);
  p->n_tiles = n_tiles;
  p->n_chunks = (n_tiles + kChunk - 1) / kChunk;
  p->n_items = 2 * int64_t(n_tiles);
  Base28 pb{};
  for (int q = 0; q < 28; ++q) pb.v[q] = uint32_t(e->pbase[q]);

  uint32_t *u_sorted = nullptr, *u_entry = nullptr, *o_sorted = nullptr, *o_entry = nullptr;
  SLBM_TRY(group_entries(e, e->ubb_slot, e->ubb_partner, e->n_ubb, pb, n_tiles, &p->ubb_perm,
                         &p->ubb_start, &u_sorted, &u_entry, s));
  if (e->n_out)
    SLBM_TRY(group_entries(e, e->out_slot, e->out_partner, e->n_out, pb, n_tiles, &p->out_perm,
                           &p->out_start, &o_sorted, &o_entry, s));

  uint32_t *lo = nullptr, *hi = nullptr, *key = nullptr, *val = nullptr, *key2 = nullptr,
           *val2 = nullptr;
  const size_t tb = size_t(n_tiles) * 4;
  SLBM_CUDA_TRY(cudaMallocAsync(&lo, tb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&hi, tb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&key, tb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&val, tb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&key2, tb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&val2, tb, s));
  k_fill_u32<<<blocks(n_tiles), 256, 0, s>>>(lo, n_tiles, UINT_MAX);
  SLBM_CUDA_TRY(cudaMemsetAsync(hi, 0, tb, s));
  k_pair_deps<<<blocks(e->n_fluid), 256, 0, s>>>(
      e->idx, uint32_t(e->idx_pitch), uint32_t(e->n_fluid), e->q, pb, u_sorted, u_entry,
      e->ubb_partner, uint32_t(e->n_ubb), o_sorted, o_entry, e->out_partner, uint32_t(e->n_out),
      lo, hi);
  const uint32_t slack =
      g_pair_slack > 0 ? uint32_t(g_pair_slack) : uint32_t(num_sms_pair() * 4);
  k_pair_keys<<<blocks(n_tiles), 256, 0, s>>>(lo, hi, n_tiles, slack, key, val);
  size_t tmpb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmpb, key, key2, val, val2, int(n_tiles), 0, 32, s);
  void* tmp = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&tmp, tmpb, s));
  cub::DeviceRadixSort::SortPairs(tmp, tmpb, key, key2, val, val2, int(n_tiles), 0, 32, s);
  SLBM_CUDA_TRY(cudaMalloc(&p->sched, size_t(p->n_items) * 4));
  SLBM_CUDA_TRY(cudaMalloc(&p->dep, size_t(n_tiles) * 8));
  k_pair_sched<<<blocks(n_tiles), 256, 0, s>>>(key2, val2, n_tiles, p->sched);
  k_pair_dep_pack<<<blocks(n_tiles), 256, 0, s>>>(lo, hi, n_tiles, p->dep);
  SLBM_CUDA_TRY(cudaMalloc(&p->chunk_done, size_t(p->n_chunks) * 4));
  SLBM_CUDA_TRY(cudaMalloc(&p->ctl, 4 * 4));
  SLBM_CUDA_TRY(cudaMalloc(&p->total_done, 8));
  SLBM_CUDA_TRY(cudaMemsetAsync(p->chunk_done, 0, size_t(p->n_chunks) * 4, s));
  SLBM_CUDA_TRY(cudaMemsetAsync(p->ctl, 0, 16, s));
  SLBM_CUDA_TRY(cudaMemsetAsync(p->total_done, 0, 8, s));
  for (void* q : {(void*)lo, (void*)hi, (void*)key, (void*)val, (void*)key2, (void*)val2, tmp,
                  (void*)u_sorted, (void*)u_entry})
    SLBM_CUDA_TRY(cudaFreeAsync(q, s));
  if (o_sorted) SLBM_CUDA_TRY(cudaFreeAsync(o_sorted, s));
  if (o_entry) SLBM_CUDA_TRY(cudaFreeAsync(o_entry, s));
  SLBM_CUDA_TRY(cudaGetLastError());
  SLBM_CUDA_TRY(cudaStreamSynchronize(s));
  return SLBM_OK;
}

template <class L, int MODEL>
void pair_launch(const PairArgs& a, cudaStream_t s) {
  constexpr int MINB = L::Q == 9 ? 8 : 4;
  if (g_pair_persist) {
    static int per_sm = 0;
    if (!per_sm) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pair_persist<L, MODEL, MINB>, kPT, 0);
      per_sm = std::max(per_sm, 1);
    }
    const int64_t grid = std::min<int64_t>(a.n_items, int64_t(per_sm) * num_sms_pair());
    k_pair_persist<L, MODEL, MINB><<<unsigned(grid), kPT, 0, s>>>(a);
  } else {
    k_pair<L, MODEL, MINB><<<a.n_items, kPT, 0, s>>>(a);
  }
}

}  // namespace

int pair_tune(int knob, int value) {
  if (knob == 5) g_pair = value;
  else if (knob == 6) g_pair_slack = value;
  else g_pair_persist = value;
  return SLBM_OK;
}

bool pair_eligible(const SlbmEngine* e) {
  return g_pair && e->layout == 0 && e->pattern == SLBM_AA && e->n_ghost == 0 &&
         e->n_fluid > 0 && e->n_fluid < (int64_t(1) << 31) / 2;
}

void free_pair(SlbmEngine* e) {
  if (!e->pair) return;
  PairPlan* p = e->pair;
  for (void* q : {(void*)p->sched, (void*)p->dep, (void*)p->chunk_done, (void*)p->ctl,
                  (void*)p->total_done, (void*)p->ubb_perm, (void*)p->ubb_start,
                  (void*)p->out_perm, (void*)p->out_start})
    if (q) cudaFree(q);
  delete p;
  e->pair = nullptr;
}

// one AA step pair (even then odd) starting at EVEN parity: the EVEN
// refresh, then k_pair; parity unchanged, step counter +2 (in the kernel)
int launch_pair(SlbmEngine* e) {
  if (!e->pair) SLBM_TRY(build_pair_plan(e));
  SLBM_TRY(launch_refresh(e, SLBM_EVEN));
  PairPlan* p = e->pair;
  SLBM_CUDA_TRY(cudaMemsetAsync(p->ctl, 0, 2 * sizeof(uint32_t), e->stream));  // ticket, finished
  PairArgs a{};
  a.pdf = e->pdf;
  a.idx = e->idx;
  a.n_fluid = uint32_t(e->n_fluid);
  a.idx_pitch = uint32_t(e->idx_pitch);
  a.n_tiles = uint32_t(p->n_tiles);
  a.n_items = uint32_t(p->n_items);
  for (int q = 0; q < 28; ++q) a.base[q] = uint32_t(e->pbase[q]);
  a.omega = e->omega;
  a.lam = e->lambda_odd;
  a.bad = e->d_bad;
  a.step = e->d_step;
  a.sched = p->sched;
  a.dep = p->dep;
  a.chunk_done = p->chunk_done;
  a.ctl = p->ctl;
  a.total_done = p->total_done;
  a.ubb_slot = e->ubb_slot;
  a.ubb_partner = e->ubb_partner;
  a.ubb_corr = e->ubb_corr;
  a.ubb_perm = p->ubb_perm;
  a.ubb_start = p->ubb_start;
  a.out_slot = e->out_slot;
  a.out_partner = e->out_partner;
  a.out_cell = e->out_cell;
  a.out_dir = e->out_dir;
  a.out_rho = e->out_rho;
  a.out_u = e->out_u;
  a.out_perm = p->out_perm;
  a.out_start = p->out_start;
  a.ahead = uint32_t(num_sms_pair());
  if (e->q == 9)
    e->model == SLBM_SRT ? pair_launch<LatD2Q9, SLBM_SRT>(a, e->stream)
                         : pair_launch<LatD2Q9, SLBM_TRT>(a, e->stream);
  else if (e->q == 19)
    e->model == SLBM_SRT ? pair_launch<LatD3Q19, SLBM_SRT>(a, e->stream)
                         : pair_launch<LatD3Q19, SLBM_TRT>(a, e->stream);
  else if (e->model == SLBM_SRT)
    pair_launch<LatD3Q27, SLBM_SRT>(a, e->stream);
  else if (e->model == SLBM_TRT)
    pair_launch<LatD3Q27, SLBM_TRT>(a, e->stream);
  else
    pair_launch<LatD3Q27, SLBM_CUMULANT>(a, e->stream);
  SLBM_CUDA_TRY(cudaGetLastError());
  return SLBM_OK;
}

}  // namespace slbm
