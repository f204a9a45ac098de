// AA step pair in one launch, temporally blocked in L2 — EXPERIMENTAL,
// off by default (slbm_set_tuning knob 5 = 1 enables it for slbm_run on
// sparse AA engines without halo slots).  Bitwise identical to the per-step
// path (tests/test_gpu_pair.py) but slower on the bench bed; kept with the
// measurements below for the next attempt.
//
// Idea.  The even step (index list, sparse.py:264-271) of cell n writes into
// the slots of n's neighbours; the odd step (cell-local, sparse.py:273-282)
// of cell c reads and rewrites only c's own slots.  So odd(c) may run as
// soon as even(n) has run for every n that touches one of c's slots — in
// cid order (z-major) those lie within about one z-plane of c.  If the odd
// step of a tile follows its writers closely enough, the values the even
// step wrote are still in the 126 MB L2: odd reads hit L2 and the even
// writes are overwritten there before eviction (680 -> ~376 B/cell of HBM
// traffic per pair, D3Q19).
//
// Design.  Work items are 32-cell tiles (one warp), even or odd, in a
// precomputed order: odd tile j after the last even tile of its writers'
// chunks + `slack`.  Persistent warps take items by an atomic ticket (so
// the items in flight form a window near the frontier); even tiles publish
// per 128-tile chunk with red.release (no L1 invalidation; an acquire or
// __threadfence() emits CCTL.IVALL, which wiped the L1 the index gathers
// rely on: 5x slower); odd tiles poll their writer chunks (near range and
// the far range across a periodic wrap) with relaxed L2 loads and read the
// state with ld.global.cg.  The odd UBB / outlet refresh of an entry runs in
// the odd tile of its partner cell.  Deadlock free: tickets increase per
// warp, an item only waits for smaller positions, and a warp publishes its
// pending item before it spins.
//
// Measured (512^3 bed, tools/pair_debug.py, profiles/r01_pair.md): the
// ticket frontier advances ~500 tiles/us, so a few us of DRAM tail latency
// put thousands of positions between the oldest unfinished item and the
// newest; an odd tile only finds its writers done with slack >= ~6000
// tiles, and then ~190K cells (~130 MB of traffic) separate a write from its
// reuse — more than L2 holds.  Result: 24.4 GB of DRAM per pair instead of
// 27.4 and 5.2 ms instead of 4.4 ms for the two per-step sweeps (4.9 ms
// with L2 keep/drop hints on the even stores / odd loads, knob 8).  Per-CTA
// items (barrier stalls) reached 16.9 GB but 5.1 ms; static round robin let
// warps drift apart (38 ms).  A blocked cell order (short dependency
// distance) and a bounded frontier are the next things to try.
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
  uint32_t* dep = nullptr;       // per odd tile: near and far writer chunk ranges (4 words)
  uint32_t* chunk_done = nullptr;  // even tiles completed per chunk, cumulative over launches
  uint32_t* ctl = nullptr;       // [0] ticket, [1] finished items, [2] launch count
  uint32_t* ubb_perm = nullptr;  // UBB entries grouped by odd tile of the partner cell
  uint32_t* ubb_start = nullptr;  // n_tiles + 1
  uint32_t* out_perm = nullptr;
  uint32_t* out_start = nullptr;
};

namespace {

constexpr int kTile = 32;           // cells per tile = one warp
constexpr int kCTA = 128;           // threads per CTA (4 worker warps)
constexpr uint32_t kChunk = 128;    // tiles per completion counter (4096 cells)
constexpr uint32_t kWide = 512;     // chunk span above which a tile waits for all
constexpr uint32_t kBundle = 2;     // schedule positions per ticket
constexpr uint32_t kNone = 0xffffffffu;

// knobs 5-8 (SlbmTuning::pair*): use the pair kernel in slbm_run; extra
// tiles between an odd tile's writers and it (0: one wave); idx prefetch
// distance in tiles (-1: 4 per SM, 0: off); L2 keep/drop hints

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
  int hints;       // L2 eviction-priority hints (knob 8)
};

// Completion flags.  Release: fence.release / red.release (MEMBAR.ALL.GPU,
// no L1 invalidation — __threadfence() and every acquire operation also
// emit CCTL.IVALL, which wipes the SM's L1 and with it the sector merging
// the index-list gathers live on: 5x slower when done per tile).  Poll:
// ld.relaxed.gpu (L2).  The odd tile's data loads that follow are L2 loads
// as well (ld.global.cg, sweep.cuh ld_pdf<true>) issued after the poll
// observed the count, and the writer's release made its stores reach L2
// before the count: the L2 is the point of coherence for both.
__device__ __forceinline__ uint32_t ld_poll(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// L2 eviction priorities: lines the even step writes are kept (evict_last)
// until the odd step reads them (evict_first); the rest streams normally
__device__ __forceinline__ uint64_t policy_keep() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_drop() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ double ld_cg_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ void red_release(uint32_t* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

constexpr int kEnd = INT_MIN;  // no more items

// Publish the completion of the worker's previous even item: lanes' stores
// -> __syncwarp -> lane 0 fence + counter (the cooperative-groups grid
// barrier pattern).  Called after the NEXT item's loads are issued, so the
// fence's wait for outstanding memory operations overlaps loads the warp
// waits for anyway instead of stalling the warp on its own stores.
__device__ __forceinline__ void publish(const PairArgs& a, int& pend) {
  __syncwarp();
  if (pend >= 0 && (threadIdx.x & 31) == 0) {
    red_release(&a.chunk_done[uint32_t(pend) / kChunk]);
  }
  pend = -1;
}

__device__ __forceinline__ bool range_ready(const PairArgs& a, uint32_t lo, uint32_t hi,
                                            uint32_t epoch) {
  const uint32_t lane = threadIdx.x & 31;
  bool ok = true;
  for (uint32_t k0 = lo; k0 <= hi; k0 += 32) {
    const uint32_t k = k0 + lane;
    if (k <= hi) {
      const uint32_t size = min(kChunk, a.n_tiles - k * kChunk);
      ok &= ld_poll(&a.chunk_done[k]) >= (epoch + 1) * size;
    }
  }
  return ok;
}

// true when every even tile that writes into odd tile j's slots has
// completed: the chunks of its near writers (within kWide chunks) and of its
// far ones (across a periodic wrap), two ranges
__device__ __forceinline__ bool deps_ready(const PairArgs& a, uint32_t j, uint32_t epoch) {
  const uint4 d = reinterpret_cast<const uint4*>(a.dep)[j];
  bool ok = range_ready(a, d.x, d.y, epoch);
  if (d.z != kNone) ok &= range_ready(a, d.z, d.w, epoch);
  return __all_sync(0xffffffffu, ok);
}

// Persistent warps taking bundles of kBundle consecutive schedule positions
// by an atomic ticket (the ticket for the next bundle is fetched one bundle
// ahead, off the critical path).  Items are handed out in schedule order, so
// the items in flight form a window about one wave wide and an odd tile's
// writers (2 x slack positions earlier) are normally done when it starts;
// static round robin instead lets warps drift apart without bound (measured
// 8x slower).  Deadlock free: a warp's tickets increase, an odd item waits
// only for smaller positions, and a warp publishes its pending item before
// it spins.
template <class L, int MODEL, int MINB>
__global__ void __launch_bounds__(kCTA, MINB) k_pair(const PairArgs a) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t W = gridDim.x * (kCTA / 32);
  const uint32_t w = blockIdx.x * (kCTA / 32) + threadIdx.x / 32;
  const uint32_t epoch = *(volatile uint32_t*)&a.ctl[2];
  const unsigned long long step = *(volatile unsigned long long*)a.step;
  int pend = -1;  // even tile whose completion is not yet published
  bool bad = false, bad_odd = false;
  const bool hints = a.hints != 0;
  const uint64_t keep = policy_keep(), drop = policy_drop();
  uint32_t tk = 0;  // lane 0: ticket of the next item, fetched while this one's loads fly
  if (lane == 0) tk = atomicAdd(&a.ctl[0], 1u);
  uint32_t i = __shfl_sync(0xffffffffu, tk, 0);
  int item = i < a.n_items ? __ldg(a.sched + i) : kEnd;
  while (item != kEnd) {
    if (item >= 0) {
      const uint32_t t = uint32_t(item);
      if (a.ahead) {  // idx rows of the tile `ahead` tiles later into L2
        const uint32_t f = (t + a.ahead) * kTile;
        if (f < a.n_fluid) prefetch_idx_warp<L::Q - 1>(a.idx, a.idx_pitch, f, lane);
      }
      const uint32_t c = t * kTile + lane;
      const bool valid = c < a.n_fluid;
      uint32_t s[L::Q];
      double v[L::Q];
      if (valid) {
        load_slots<L>(s, a.idx, a.idx_pitch, c);
        gather<L>(v, a.pdf, s);
      }
      if (lane == 0) tk = atomicAdd(&a.ctl[0], 1u);  // overshoots at the end; reset per launch
      publish(a, pend);
      if (valid) {  // collide_scatter<EVEN> with the keep hint on the stores
        bad |= collide<L, MODEL>(v, a.omega, a.lam, [&](auto q, double x) {
          constexpr int qb = L::INV[decltype(q)::value];
          if (hints)
            st_hint(a.pdf + s[qb], x, keep);
          else
            a.pdf[s[qb]] = x;
        });
      }
      pend = item;
    } else {
      const uint32_t j = ~uint32_t(item);
      if (!deps_ready(a, j, epoch)) {
        publish(a, pend);
        uint32_t spins = 0;
        while (!deps_ready(a, j, epoch)) {
          __nanosleep(128);
          ++spins;
        }
        if (lane == 0) {  // debug statistics (slbm_debug_pair_stats)
          atomicAdd(&a.ctl[4], 1u);
          atomicAdd(&a.ctl[5], spins);
          if (atomicCAS(&a.ctl[6], 0u, 1u) == 0u) {
            a.ctl[7] = j;
            a.ctl[8] = a.dep[4 * j];
            a.ctl[9] = a.dep[4 * j + 1];
            a.ctl[10] = i;
            a.ctl[11] = w;
          a.ctl[12] = W;
          }
        }
      }
      __syncwarp();
      // odd refresh of the boundary entries whose partner slot is in this tile
      for (uint32_t k = a.ubb_start[j] + lane; k < a.ubb_start[j + 1]; k += 32) {
        const uint32_t e = a.ubb_perm[k];
        a.pdf[a.ubb_partner[e]] = __ldcg(a.pdf + a.ubb_slot[e]) + a.ubb_corr[e];
      }
      if (a.out_start) {
        for (uint32_t k = a.out_start[j] + lane; k < a.out_start[j + 1]; k += 32) {
          const uint32_t e = a.out_perm[k];
          outlet_entry<L, true>(a.pdf, a.base, a.out_slot[e], a.out_partner[e], a.out_cell[e],
                                a.out_dir[e], a.out_rho[e], const_cast<double*>(a.out_u) + 3 * e,
                                SLBM_ODD);
        }
      }
      __syncwarp();
      const uint32_t c = j * kTile + lane;
      const bool valid = c < a.n_fluid;
      double v[L::Q];
      if (valid) {
        sfor<0, L::Q>([&](auto q) {
          constexpr int qb = L::INV[q];
          v[q] = hints ? ld_cg_hint(a.pdf + a.base[qb] + c, drop) : __ldcg(a.pdf + a.base[qb] + c);
        });
      }
      if (lane == 0) tk = atomicAdd(&a.ctl[0], 1u);
      publish(a, pend);
      if (valid)
        bad_odd |= collide<L, MODEL>(v, a.omega, a.lam, [&](auto q, double x) {
          a.pdf[a.base[decltype(q)::value] + c] = x;
        });
    }
    i = __shfl_sync(0xffffffffu, tk, 0);
    item = i < a.n_items ? __ldg(a.sched + i) : kEnd;
  }
  publish(a, pend);
  if (bad) atomicMin(a.bad, step);
  if (bad_odd) atomicMin(a.bad, step + 1);
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(&a.ctl[1], 1u) == W - 1) {  // last warp of the launch
      a.ctl[2] = epoch + 1;
      *a.step = step + 2;
      __threadfence();
    }
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
                            const uint32_t* out_partner, uint32_t n_out, uint32_t* dep) {
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= n_fluid) return;
  const uint32_t wchunk = (n / kTile) / kChunk;
  auto add = [&](int64_t c) {  // near range (x, y), far range (z, w) of tile c / kTile
    const uint32_t t = uint32_t(c / kTile), tc = t / kChunk;
    const bool near = wchunk + kWide >= tc && wchunk <= tc + kWide;
    uint32_t* d = dep + 4 * size_t(t) + (near ? 0 : 2);
    atomicMin(d, wchunk);
    atomicMax(d + 1, wchunk);
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
    const uint32_t s = idx[idx_offset(q == 19, pitch, uint32_t(r), n)];
    int64_t c = owner_cell(pb.v, q, n_fluid, s);
    if (c < 0) c = lookup(ubb_sorted, ubb_entry, ubb_partner, n_ubb, s);
    if (c == -2) c = lookup(out_sorted, out_entry, out_partner, n_out, s);
    if (c >= 0) add(c);
  }
}

// order key of every odd tile: the even tile after which it is handed out
// (its last writer chunk's end + slack)
__global__ void k_pair_keys(const uint32_t* dep, uint32_t n_tiles, uint32_t slack, uint32_t* key,
                            uint32_t* val) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_tiles) return;
  uint32_t last = dep[4 * j + 1];
  if (dep[4 * j + 2] != kNone) last = max(last, dep[4 * j + 3]);
  const uint64_t k = uint64_t(last + 1) * kChunk - 1 + slack;
  key[j] = uint32_t(std::min<uint64_t>(k, n_tiles - 1));
  val[j] = j;
}

__global__ void k_pair_dep_init(uint32_t* dep, uint32_t n_tiles) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_tiles) return;
  reinterpret_cast<uint4*>(dep)[j] = make_uint4(kNone, 0u, kNone, 0u);
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

// entries -> (tile of the partner cell, entry); slot copy for the lookup
__global__ void k_entry_keys(const uint32_t* slot, const uint32_t* partner, uint32_t n,
                             uint32_t n_fluid, int q, Base28 pb, uint32_t* tile, uint32_t* ent,
                             uint32_t* slot_key) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int64_t c = owner_cell(pb.v, q, n_fluid, partner[e]);
  tile[e] = c >= 0 ? uint32_t(c / kTile) : 0u;
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
    { k_entry_keys<<<blocks(n), 256, 0, s>>>(slot, partner, uint32_t(n), uint32_t(e->n_fluid), e->q,
                                           pb, tile, ent, skey); slbm::count_launch(); }
    size_t tb = 0, tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, tile, tile2, ent, *perm, int(n), 0, 32, s);
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, skey, *slot_sorted, ent, ent2, int(n), 0, 32, s);
    void* tmp = nullptr;
    SLBM_CUDA_TRY(cudaMallocAsync(&tmp, std::max(tb, tb2), s));
    cub::DeviceRadixSort::SortPairs(tmp, tb, tile, tile2, ent, *perm, int(n), 0, 32, s);
    cub::DeviceRadixSort::SortPairs(tmp, tb2, skey, *slot_sorted, ent, *slot_entry, int(n), 0, 32, s);
    SLBM_CUDA_TRY(cudaFreeAsync(tmp, s));
  }
  { k_tile_starts<<<blocks(n_tiles + 1), 256, 0, s>>>(tile2, uint32_t(n), n_tiles, *start); slbm::count_launch(); }
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
  const uint32_t n_tiles = uint32_t((e->n_fluid + kTile - 1) / kTile);
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

  uint32_t *key = nullptr, *val = nullptr, *key2 = nullptr, *val2 = nullptr;
  const size_t tb = size_t(n_tiles) * 4;
  SLBM_CUDA_TRY(cudaMalloc(&p->dep, size_t(n_tiles) * 16));
  SLBM_CUDA_TRY(cudaMallocAsync(&key, tb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&val, tb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&key2, tb, s));
  SLBM_CUDA_TRY(cudaMallocAsync(&val2, tb, s));
  { k_pair_dep_init<<<blocks(n_tiles), 256, 0, s>>>(p->dep, n_tiles); slbm::count_launch(); }
  { k_pair_deps<<<blocks(e->n_fluid), 256, 0, s>>>(
      e->idx, uint32_t(e->idx_pitch), uint32_t(e->n_fluid), e->q, pb, u_sorted, u_entry,
      e->ubb_partner, uint32_t(e->n_ubb), o_sorted, o_entry, e->out_partner, uint32_t(e->n_out),
      p->dep); slbm::count_launch(); }
  const uint32_t slack =
      e->tune.pair_slack > 0 ? uint32_t(e->tune.pair_slack) : uint32_t(num_sms_pair() * 12);
  { k_pair_keys<<<blocks(n_tiles), 256, 0, s>>>(p->dep, n_tiles, slack, key, val); slbm::count_launch(); }
  size_t tmpb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmpb, key, key2, val, val2, int(n_tiles), 0, 32, s);
  void* tmp = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&tmp, tmpb, s));
  cub::DeviceRadixSort::SortPairs(tmp, tmpb, key, key2, val, val2, int(n_tiles), 0, 32, s);
  SLBM_CUDA_TRY(cudaMalloc(&p->sched, size_t(p->n_items) * 4));
  { k_pair_sched<<<blocks(n_tiles), 256, 0, s>>>(key2, val2, n_tiles, p->sched); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaMalloc(&p->chunk_done, size_t(p->n_chunks) * 4));
  SLBM_CUDA_TRY(cudaMalloc(&p->ctl, 16 * 4));
  SLBM_CUDA_TRY(cudaMemsetAsync(p->chunk_done, 0, size_t(p->n_chunks) * 4, s));
  SLBM_CUDA_TRY(cudaMemsetAsync(p->ctl, 0, 64, s));
  for (void* q : {(void*)key, (void*)val, (void*)key2, (void*)val2, tmp,
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
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pair<L, MODEL, MINB>, kCTA, 0);
    per_sm = std::max(per_sm, 1);
  }
  // one wave: every warp resident (the deadlock-freedom condition)
  const int64_t grid = std::min<int64_t>((a.n_items + kCTA / 32 - 1) / (kCTA / 32),
                                         int64_t(per_sm) * num_sms_pair());
  { k_pair<L, MODEL, MINB><<<unsigned(std::max<int64_t>(grid, 1)), kCTA, 0, s>>>(a); slbm::count_launch(); }
}

}  // namespace


bool pair_eligible(const SlbmEngine* e) {
  return e->tune.pair && e->model != SLBM_CUMULANT_GEN && e->layout == 0 && e->pattern == SLBM_AA && e->n_ghost == 0 &&
         e->n_fluid > 0 && e->n_fluid < (int64_t(1) << 31) / 2;
}

void free_pair(SlbmEngine* e) {
  if (!e->pair) return;
  PairPlan* p = e->pair;
  for (void* q : {(void*)p->sched, (void*)p->dep, (void*)p->chunk_done, (void*)p->ctl,
                  (void*)p->ubb_perm, (void*)p->ubb_start,
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
  SLBM_CUDA_TRY(cudaMemsetAsync(p->ctl, 0, 2 * sizeof(uint32_t), e->stream));  // finished warps
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
  a.hints = e->tune.pair_hints;
  a.ahead = e->tune.pair_ahead >= 0 ? uint32_t(e->tune.pair_ahead) : uint32_t(num_sms_pair() * 4);
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

// debug: the pair plan's wait statistics of the last launches (not in the header)
extern "C" int slbm_debug_pair_stats(SlbmEngine* e, uint32_t* out16) {
  if (!e || !e->pair || !out16) return 1;
  cudaStreamSynchronize(e->stream);
  cudaMemcpy(out16, e->pair->ctl, 64, cudaMemcpyDeviceToHost);
  return 0;
}
