// Internal state of one sparse block engine (the object behind SlbmEngine*).
#pragma once

#include <vector>

#include "common.cuh"

namespace slbm {
struct PairPlan;
// one device allocation holding the pdf buffers of several engines (block
// groups with direct local halo edges, group.cu); freed with its last engine
struct PdfPool {
  double* base = nullptr;
  int refs = 0;
};
}

// Kernel-selection knobs (slbm_engine_set_tuning; include/slbm_b200.h).  Each
// engine owns a copy, taken from the process defaults (slbm_set_tuning) when
// it is created, so tuning one engine never changes another's kernels.
struct SlbmTuning {
  int even_variant = 0;            // 0: production, 1: no idx prefetch, 2: probe (SLBM_PROBES builds)
  int odd_variant = 0;             // cell-local sweep CTAs per SM (0: 3, 2: 4)
  int ahead_quarters = 1;          // idx L2 prefetch distance in quarter waves
  int ahead_ctas = 0;              // ... in CTAs when > 0
  int64_t resident_cap = 1 << 19;  // slbm_run: k_resident up to this n_fluid (0: off)
  int pair = 0;                    // slbm_run: temporally blocked pair kernel (SLBM_WITH_PAIR builds)
  int pair_slack = 0;
  int pair_ahead = -1;
  int pair_hints = 1;
  int dense_lean_odd = 1;          // dense engines: k_dense_odd
  int even_ctas = 0;               // D3Q19 index-list sweep CTAs/SM: 0 auto, 4 or 5
};

namespace slbm {
extern SlbmTuning g_tuning_defaults;
// knob -> field; SLBM_ECONFIG for unknown knobs or values this build refuses
int tuning_apply(SlbmTuning& t, int knob, int value);
}

struct SlbmEngine {
  int device = 0;
  int dim = 3, q = 19;
  int model = SLBM_SRT;
  double omega = 1.0, lambda_odd = 1.0;  // cumulant: lambda_odd holds the bulk rate
  double hr[8] = {1, 1, 1, 1, 1, 1, 1, 1};  // cumulant w3..w10 (host copy)
  double* d_hr = nullptr;                   // ... on the device (general cumulant only)
  int pattern = SLBM_PULL;
  int parity = SLBM_EVEN;
  SlbmTuning tune = slbm::g_tuning_defaults;
  slbm::Geometry geo{};
  slbm::DirTable dirs{};

  int64_t n_fluid = 0, total_slots = 0, n_ubb = 0, n_ghost = 0;
  int64_t n_interior = 0, n_frame = 0;
  bool has_split = false;
  int64_t base[28] = {0};   // slot-id layout of the reference (sparse.py:128-137)
  // Device layout: direction group q starts at pbase[q], each group padded to
  // a multiple of 32 slots (256 B), so every group row and idx row is
  // line-aligned (profiles: +1% index sweep, +2% cell-local sweep).  The
  // index list and the boundary programs hold physical addresses; slot ids
  // crossing the C-ABI are the reference's and translated (phys_slot).
  int64_t pbase[28] = {0};
  int64_t phys_slots = 0;   // pdf elements allocated (>= total_slots)
  int64_t idx_pitch = 0;    // elements per idx row (n_fluid rounded up to 32)
  int64_t n_ubb_q[27] = {0}, n_ghost_q[27] = {0};
  int64_t ubb_off[28] = {0}, ghost_off[28] = {0};
  int64_t n_out = 0, n_out_q[27] = {0}, out_off[28] = {0};

  // device memory
  double* pdf = nullptr;   // active buffer
  slbm::PdfPool* pool = nullptr;  // pdf lives in this pool (not freed on its own)
  double* tmp = nullptr;   // pull: second buffer
  int layout = 0;  // 0 sparse (index list), 1 dense (direct addressing)
  uint32_t* dense_mask = nullptr;       // per box cell fold mask (dense)
  uint64_t* dense_ubb_key = nullptr;    // sorted (box cell << 5 | q)
  double* dense_ubb_corr = nullptr;
  int64_t n_dense_ubb = 0;
  int32_t dense_frame_w[3] = {1, 1, 1};
  uint32_t* idx = nullptr;  // (q-1) x n_fluid
  uint32_t* x_flat = nullptr;  // cid -> padded flat
  int32_t* cid_map = nullptr;  // padded flat -> cid or -1
  uint32_t* ubb_slot = nullptr;
  uint32_t* ubb_partner = nullptr;
  double* ubb_corr = nullptr;
  uint32_t* out_slot = nullptr;     // fixed-density outlet program
  uint32_t* out_partner = nullptr;
  uint32_t* out_cell = nullptr;
  uint8_t* out_dir = nullptr;
  double* out_rho = nullptr;
  double* out_u = nullptr;          // 3 x n_out, velocity kept EVEN -> ODD
  uint64_t* ghost_key = nullptr;  // per q sorted (sigma_key << 32 | pflat)
  std::vector<uint64_t> ghost_key_host;
  uint32_t* frame_cids = nullptr;
  uint32_t* frame_bits = nullptr;  // bit c set <=> cell c is a frame cell
  int64_t interior_lo = -1;        // >= 0: interior = cids [lo, lo + n_interior), no mask
  unsigned long long* d_bad = nullptr;   // first unstable step (ULLONG_MAX = none)
  unsigned long long* d_step = nullptr;  // step counter read by the sweeps
  double* d_scratch = nullptr;           // staging for host transfers
  size_t scratch_bytes = 0;
  int64_t device_bytes = 0;

  unsigned long long* h_bad = nullptr;   // pinned copy for polling

  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;

  // CUDA graphs of one step pair, keyed by starting state (0/1)
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  long long graph_kernels[2] = {0, 0};  // library kernels per replay (slbm_launch_count)
  int64_t steps_done = 0;
  slbm::PairPlan* pair = nullptr;  // pair.cu: temporally blocked AA step pair
  // index-list sweep occupancy chosen by measurement (kernels.cu
  // sweep_ctas): 0 undecided, else 4 or 5 CTAs per SM
  int even_ctas = 0;
  int even_trials = 0;
  cudaEvent_t even_ev[8] = {};

  int ensure_scratch(size_t bytes);

  // reference slot id -> device address (identity for dense engines)
  // inverse for a device address of a used slot
  int64_t slot_of(int64_t phys) const {
    if (layout) return phys;
    int g = 0;
    while (g + 1 < q && pbase[g + 1] <= phys) ++g;
    return base[g] + (phys - pbase[g]);
  }
  int64_t phys_slot(int64_t slot) const {
    if (layout) return slot;
    int g = 0;
    while (g + 1 < q && base[g + 1] <= slot) ++g;
    return pbase[g] + (slot - base[g]);
  }
};

namespace slbm {

// Device-local halo edges of one phase (halo.cu), for kernels that run them
// fused with other per-step work (group.cu k_group_boundary):
// pdf[de[i]][ds[i]] = pdf[se[i]][ss[i]], engines indexed by the halo.
constexpr int kMaxHaloEngines = 512;
struct PdfTable {
  double* p[kMaxHaloEngines];
};
struct LocalEdges {
  const uint16_t *se = nullptr, *de = nullptr;
  const uint32_t *ss = nullptr, *ds = nullptr;
  int64_t n = 0;
  int n_eng = 0;  // engines of the halo (entries of the PdfTable)
};
// committed local program of `phase`; the table holds the engines' current pdf
int halo_local_edges(SlbmHalo* h, int phase, PdfTable* table, LocalEdges* edges);
// host copy of the committed local program of `phase` (engine ids index
// `engines`), and switching it off (direct local edges, group.cu)
int halo_local_program(SlbmHalo* h, int phase, std::vector<SlbmEngine*>* engines,
                       std::vector<uint16_t>* se, std::vector<uint32_t>* ss,
                       std::vector<uint16_t>* de, std::vector<uint32_t>* ds);
void halo_disable_local(SlbmHalo* h);

// kernels / launchers implemented in kernels.cu
int launch_step(SlbmEngine* e, int phase);
int launch_refresh(SlbmEngine* e, int parity);
// small engines: n steps in one cooperative launch (kernels.cu k_resident)
constexpr int64_t kResidentChunk = 1 << 12;
bool resident_eligible(const SlbmEngine* e, int64_t n);
int launch_resident(SlbmEngine* e, int64_t n);
int launch_advance(SlbmEngine* e);
// pair.cu: one AA step pair (EVEN refresh + even + odd refresh + odd) in one
// launch, temporally blocked in L2; engines without halo slots
#ifdef SLBM_WITH_PAIR
bool pair_eligible(const SlbmEngine* e);
int launch_pair(SlbmEngine* e);
void free_pair(SlbmEngine* e);
#else  // pair.cu is experimental and left out of the shipped library
inline bool pair_eligible(const SlbmEngine*) { return false; }
inline int launch_pair(SlbmEngine*) { return SLBM_ECONFIG; }
inline void free_pair(SlbmEngine*) {}
#endif
int launch_canonical(SlbmEngine* e, double* dev_out);  // (q, n) at current parity
// box layout (zeros at solids must be pre-set) or compact: one value per fluid cell
// gdims/origin: write into a global box (rows of gdims[0], gdims[1] rows per
// plane) at the block's origin instead of the block's own box
int launch_macroscopic(SlbmEngine* e, const double* dev_canon, double* dev_rho, double* dev_u,
                       bool compact = false, const int64_t* gdims = nullptr,
                       const int64_t* origin = nullptr);
int launch_gather(const double* src, const uint32_t* slots, int64_t n, double* out,
                  cudaStream_t s);
int launch_scatter(double* dst, const uint32_t* slots, int64_t n, const double* in,
                   cudaStream_t s);
int launch_fill(double* p, int64_t n, double v, cudaStream_t s);
int launch_equilibrium(SlbmEngine* e, const double* rho, int rho_scalar, const double* u,
                       int u_scalar, double* dev_out);
int launch_sum(const double* p, int64_t n, double* dev_out, cudaStream_t s);
int launch_moments(SlbmEngine* e, double* dev_out);  // mass, momentum x/y/z (sparse)
int launch_equilibrium_qn(SlbmEngine* e, const double* rho, int rho_scalar, const double* u,
                          int u_scalar, double* out);
int launch_slot_lookup(SlbmEngine* e, const int64_t* d_qs, const int64_t* d_pflat, int64_t n,
                       int64_t* d_out, int* d_err);

int set_tuning(int knob, int value);

// hostcopy.cu: staged multi-threaded copies for pageable host arrays
// (synchronous; ordered after the work already queued on `s`)
int copy_d2h(void* host, const void* dev, size_t bytes, int device, cudaStream_t s);
int copy_h2d(void* dev, const void* host, size_t bytes, int device, cudaStream_t s);
int hostcopy_reserve(int device);
void* mapped_device_ptr(void* host);  // pinned host buffer -> device address, else nullptr
// macroscopic fields of every box cell written straight into (mapped) host
// memory: zeros at solids, no device staging
int launch_macroscopic_box(SlbmEngine* e, double* rho, double* u);
int hostcopy_tune(int knob, int value);  // 10: chunk MiB, 11: max threads, 12: mapped out
bool mapped_out_enabled();

// builder.cu
int build_lists(SlbmEngine* e, const uint8_t* tags_pad, const double* ubb_u_pad,
                const int32_t* frame_width);
int enumerate_fluid(SlbmEngine* e, const uint8_t* tags_pad);
int export_idx_logical(SlbmEngine* e, uint32_t* host);
int build_split(SlbmEngine* e, const int32_t* lo_w, const int32_t* hi_w, uint32_t* scratch);
int set_frame(SlbmEngine* e, const int32_t* lo_w, const int32_t* hi_w);

// dense.cu (direct-addressing engine)
int build_dense(SlbmEngine* e, const uint8_t* tags_pad, const double* ubb_u_pad,
                const int32_t* frame_width);
int dense_step(SlbmEngine* e, int phase);
int dense_init(SlbmEngine* e, const double* dev_values);
int dense_canonical(SlbmEngine* e, double* dev_values);

}  // namespace slbm
