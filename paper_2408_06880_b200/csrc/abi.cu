// extern "C" entry points of the engine (include/slbm_b200.h).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "engine.cuh"

namespace slbm {

std::atomic<long long> g_launches{0};
static thread_local long long t_capture_mark = 0;
static std::mutex g_graph_mu;
static std::unordered_map<void*, long long> g_graph_kernels;  // exec -> kernels per replay

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

}  // namespace slbm

using namespace slbm;

int SlbmEngine::ensure_scratch(size_t bytes) {
  if (bytes <= scratch_bytes) return SLBM_OK;
  if (d_scratch) cudaFree(d_scratch);
  d_scratch = nullptr;
  scratch_bytes = 0;
  SLBM_CUDA_TRY(cudaMalloc(&d_scratch, bytes));
  scratch_bytes = bytes;
  return SLBM_OK;
}

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

#define CHECK_ENGINE(e) \
  if (!(e)) return fail(SLBM_ECONFIG, "null engine handle")

DirTable make_dirs(int q) {
  DirTable d{};
  d.q = q;
  auto fill = [&](auto lat) {
    using L = decltype(lat);
    for (int i = 0; i < L::Q; ++i) {
      d.c[i][0] = int8_t(L::CX[i]);
      d.c[i][1] = int8_t(L::CY[i]);
      d.c[i][2] = int8_t(L::CZ[i]);
      d.inv[i] = int8_t(L::INV[i]);
      d.w[i] = double(L::WNUM[i]) / double(L::WDEN[i]);
    }
  };
  if (q == 9)
    fill(LatD2Q9{});
  else if (q == 19)
    fill(LatD3Q19{});
  else
    fill(LatD3Q27{});
  return d;
}

void free_engine(SlbmEngine* e) {
  if (!e) return;
  DeviceGuard g(e->device);
  // only the stream this engine created; a borrowed stream may already be gone
  if (e->own_stream) cudaStreamSynchronize(e->own_stream);
  for (auto& gx : e->graph)
    if (gx) cudaGraphExecDestroy(gx);
  free_pair(e);
  for (auto& ev : e->even_ev)
    if (ev) cudaEventDestroy(ev);
  if (e->pool) {  // the pdf is part of a group's pool: release this engine's share
    if (--e->pool->refs == 0) {
      cudaFree(e->pool->base);
      delete e->pool;
    }
    e->pdf = nullptr;
  }
  void* ptrs[] = {e->pdf,         e->tmp,          e->idx,       e->x_flat,
                  e->cid_map,     e->ubb_slot,     e->ubb_partner, e->ubb_corr,
                  e->ghost_key,   e->frame_cids,   e->frame_bits, e->d_bad,
                  e->out_slot,    e->out_partner,  e->out_cell,  e->out_dir,
                  e->out_rho,     e->out_u,        e->dense_mask,
                  e->dense_ubb_key, e->dense_ubb_corr,
                  e->d_step,      e->d_scratch};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (e->h_bad) cudaFreeHost(e->h_bad);
  if (e->d_hr) cudaFree(e->d_hr);
  if (e->own_stream) cudaStreamDestroy(e->own_stream);
  delete e;
}

int check_model(int q, int model) {
  if (model == SLBM_SRT || model == SLBM_TRT) return SLBM_OK;
  if (model == SLBM_CUMULANT) {  // general rates: slbm_engine_set_cumulant_rates
    if (q != 27) return fail(SLBM_ECONFIG, "cumulant collision needs the d3q27 stencil");
    return SLBM_OK;
  }
  return fail(SLBM_ECONFIG, "unknown collision model code " + std::to_string(model));
}

int upload_slots(SlbmEngine* e, const int64_t* slots, int64_t n, uint32_t** dev) {
  std::vector<uint32_t> s32(size_t(std::max<int64_t>(n, 1)));
  for (int64_t i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= e->total_slots)
      return fail(SLBM_EPROTOCOL, "slot " + std::to_string(slots[i]) + " outside [0, " +
                                      std::to_string(e->total_slots) + ")");
    s32[i] = uint32_t(e->phys_slot(slots[i]));
  }
  SLBM_CUDA_TRY(cudaMallocAsync(dev, s32.size() * sizeof(uint32_t), e->stream));
  SLBM_CUDA_TRY(cudaMemcpyAsync(*dev, s32.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                e->stream));
  return SLBM_OK;
}

// dense slot of (q, padded cell): q * npad + p, halo cells included
// (dense.py:311-322); no fluid check, like the reference
int dense_slots(const SlbmEngine* e, const int64_t* qs, const int64_t* pflat, int64_t n,
                int64_t* out) {
  const int64_t npad = e->geo.n_padded();
  for (int64_t i = 0; i < n; ++i) {
    if (qs[i] < 0 || qs[i] >= e->q || pflat[i] < 0 || pflat[i] >= npad)
      return fail(SLBM_EPROTOCOL, "dense slot outside the padded block");
    out[i] = qs[i] * npad + pflat[i];
  }
  return SLBM_OK;
}

int sweep_once(SlbmEngine* e) {
  SLBM_TRY(launch_refresh(e, e->parity));
  SLBM_TRY(launch_step(e, SLBM_PHASE_ALL));
  SLBM_TRY(slbm_finish_step(e));
  return SLBM_OK;
}

}  // namespace

extern "C" {

const char* slbm_last_error(void) { return last_error(); }
const char* slbm_version(void) { return "slbm_b200 0.1 sm_100a"; }

int slbm_set_tuning(int knob, int value) { return set_tuning(knob, value); }

int slbm_engine_set_tuning(SlbmEngine* e, int knob, int value) {
  CHECK_ENGINE(e);
  SlbmTuning t = e->tune;
  SLBM_TRY(tuning_apply(t, knob, value));
  e->tune = t;
  // captured step pairs baked in the previous kernel choice
  for (auto& g : e->graph)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  return SLBM_OK;
}

int slbm_capture_begin(void* stream) {
  if (!stream) return fail(SLBM_ECONFIG, "capture needs a non-default stream");
  SLBM_CUDA_TRY(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
  t_capture_mark = g_launches.load();
  return SLBM_OK;
}

int slbm_capture_end(void* stream, void** graph_exec) {
  if (!stream || !graph_exec) return fail(SLBM_ECONFIG, "null argument");
  const long long captured = g_launches.load() - t_capture_mark;
  g_launches.fetch_sub(captured);  // recorded, not launched: counted per replay
  cudaGraph_t graph = nullptr;
  SLBM_CUDA_TRY(cudaStreamEndCapture((cudaStream_t)stream, &graph));
  cudaGraphExec_t exec = nullptr;
  cudaError_t err = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (err != cudaSuccess)
    return fail(SLBM_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(err));
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    g_graph_kernels[(void*)exec] = captured;
  }
  *graph_exec = (void*)exec;
  return SLBM_OK;
}

int slbm_graph_launch(void* graph_exec, void* stream) {
  if (!graph_exec) return fail(SLBM_ECONFIG, "null graph");
  SLBM_CUDA_TRY(cudaGraphLaunch((cudaGraphExec_t)graph_exec, (cudaStream_t)stream));
  std::lock_guard<std::mutex> lk(g_graph_mu);
  auto it = g_graph_kernels.find(graph_exec);
  if (it != g_graph_kernels.end()) count_launch(it->second);
  return SLBM_OK;
}

int slbm_launch_count(int64_t* count) {
  if (!count) return fail(SLBM_ECONFIG, "null argument");
  *count = g_launches.load();
  return SLBM_OK;
}

int slbm_graph_destroy(void* graph_exec) {
  if (graph_exec) {
    cudaGraphExecDestroy((cudaGraphExec_t)graph_exec);
    std::lock_guard<std::mutex> lk(g_graph_mu);
    g_graph_kernels.erase(graph_exec);
  }
  return SLBM_OK;
}

static int create_engine(int layout, const uint8_t* tags_pad, const double* ubb_u_pad, int dim,
                         const int32_t* dims, const uint8_t* periodic, int q, int model,
                         double omega, double lambda_odd, int pattern,
                         const int32_t* frame_width, int device, SlbmEngine** out) {
  if (!out || !tags_pad || !dims || !periodic) return fail(SLBM_ECONFIG, "null argument");
  *out = nullptr;
  if (pattern != SLBM_PULL && pattern != SLBM_AA)
    return fail(SLBM_ECONFIG, "unknown streaming pattern code " + std::to_string(pattern));
  if (!((q == 9 && dim == 2) || ((q == 19 || q == 27) && dim == 3)))
    return fail(SLBM_ECONFIG, "stencil q=" + std::to_string(q) + " needs " +
                                  (q == 9 ? "2" : "3") + "-d dims, got " + std::to_string(dim) +
                                  "-d");
  SLBM_TRY(check_model(q, model));
  for (int a = 0; a < dim; ++a)
    if (dims[a] < 1) return fail(SLBM_ECONFIG, "all extents must be positive");
  if (frame_width)
    for (int a = 0; a < dim; ++a)
      // 0 = no frame on that axis (used for axes without halo exchange;
      // the reference's frame_mask requires >= 1, enforced by the host layer)
      if (frame_width[a] < 0) return fail(SLBM_ECONFIG, "frame widths must be >= 0");

  DeviceGuard guard(device);
  SlbmEngine* e = new SlbmEngine();
  e->device = device;
  e->dim = dim;
  e->q = q;
  e->model = model;
  e->omega = omega;
  e->lambda_odd = lambda_odd;
  e->pattern = pattern;
  e->dirs = make_dirs(q);
  Geometry& g = e->geo;
  g.dim = dim;
  for (int a = 0; a < 3; ++a) {
    const bool active = a < dim;
    g.n[a] = active ? dims[a] : 1;
    g.p[a] = active ? int64_t(dims[a]) + 2 : 1;
    g.off[a] = active ? 1 : 0;
    g.periodic[a] = active ? (periodic[a] ? 1 : 0) : 0;
  }
  cudaError_t err = cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking);
  if (err != cudaSuccess) {
    delete e;
    return fail(SLBM_ECUDA, std::string("stream create: ") + cudaGetErrorString(err));
  }
  e->stream = e->own_stream;
  e->layout = layout;
  int st = SLBM_OK;
  if (layout == 0) {
    st = build_lists(e, tags_pad, ubb_u_pad, frame_width);
  } else {
    st = enumerate_fluid(e, tags_pad);
    if (st == SLBM_OK) st = build_dense(e, tags_pad, ubb_u_pad, frame_width);
  }
  if (st != SLBM_OK) {
    std::string msg = last_error();
    free_engine(e);
    set_error(msg);
    return st;
  }
  // PDF buffers, NaN-poisoned (sparse.py:90-91)
  auto alloc = [&](double** p) -> int {
    cudaError_t er = cudaMalloc(p, size_t(e->phys_slots) * sizeof(double));
    if (er != cudaSuccess)
      return fail(SLBM_ECUDA, "PDF allocation of " + std::to_string(e->phys_slots * 8) +
                                  " bytes failed: " + cudaGetErrorString(er));
    e->device_bytes += e->phys_slots * 8;
    return launch_fill(*p, e->phys_slots, NAN, e->stream);
  };
  st = alloc(&e->pdf);
  if (st == SLBM_OK && pattern == SLBM_PULL) st = alloc(&e->tmp);
  if (st == SLBM_OK) {
    if (cudaMalloc(&e->d_bad, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&e->d_step, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMallocHost(&e->h_bad, sizeof(unsigned long long)) != cudaSuccess)
      st = fail(SLBM_ECUDA, "status allocation failed");
  }
  if (st == SLBM_OK) {
    cudaMemsetAsync(e->d_bad, 0xff, sizeof(unsigned long long), e->stream);
    cudaMemsetAsync(e->d_step, 0, sizeof(unsigned long long), e->stream);
    if (cudaStreamSynchronize(e->stream) != cudaSuccess)
      st = fail(SLBM_ECUDA, "engine init sync failed");
  }
  // large blocks will move GBs through init_canonical / canonical_state /
  // macroscopic_fields: set up the pinned staging lanes now, not in the
  // first transfer (hostcopy.cu)
  if (st == SLBM_OK && e->total_slots * 8 >= (int64_t(256) << 20)) st = hostcopy_reserve(e->device);
  if (st != SLBM_OK) {
    std::string msg = last_error();
    free_engine(e);
    set_error(msg);
    return st;
  }
  *out = e;
  return SLBM_OK;
}

int slbm_engine_create(const uint8_t* tags_pad, const double* ubb_u_pad, int dim,
                       const int32_t* dims, const uint8_t* periodic, int q, int model,
                       double omega, double lambda_odd, int pattern,
                       const int32_t* frame_width, int device, SlbmEngine** out) {
  return create_engine(0, tags_pad, ubb_u_pad, dim, dims, periodic, q, model, omega, lambda_odd,
                       pattern, frame_width, device, out);
}

int slbm_engine_create_dense(const uint8_t* tags_pad, const double* ubb_u_pad, int dim,
                             const int32_t* dims, const uint8_t* periodic, int q, int model,
                             double omega, double lambda_odd, int pattern,
                             const int32_t* frame_width, int device, SlbmEngine** out) {
  return create_engine(1, tags_pad, ubb_u_pad, dim, dims, periodic, q, model, omega, lambda_odd,
                       pattern, frame_width, device, out);
}

int slbm_engine_destroy(SlbmEngine* e) {
  free_engine(e);
  return SLBM_OK;
}

int slbm_engine_info(const SlbmEngine* e, SlbmInfo* info) {
  CHECK_ENGINE(e);
  if (!info) return fail(SLBM_ECONFIG, "null info");
  std::memset(info, 0, sizeof(*info));
  info->q = e->q;
  info->dim = e->dim;
  info->pattern = e->pattern;
  info->parity = e->parity;
  info->has_split = e->has_split ? 1 : 0;
  info->model = e->model;
  info->n_fluid = e->n_fluid;
  info->total_slots = e->total_slots;
  info->n_ubb_slots = e->n_ubb;
  info->n_ghost_slots = e->n_ghost;
  info->n_outlet_slots = e->n_out;
  info->layout = e->layout;
  info->n_interior = e->has_split ? e->n_interior : e->n_fluid;
  info->n_frame = e->has_split ? e->n_frame : 0;
  for (int q = 0; q <= e->q; ++q) info->base[q] = e->base[q];
  for (int q = 0; q < e->q; ++q) {
    info->n_ubb_q[q] = e->n_ubb_q[q];
    info->n_ghost_q[q] = e->n_ghost_q[q];
  }
  info->device_bytes = e->device_bytes;
  return SLBM_OK;
}

int slbm_engine_stream(const SlbmEngine* e, void** stream) {
  CHECK_ENGINE(e);
  *stream = (void*)e->stream;
  return SLBM_OK;
}

int slbm_engine_set_stream(SlbmEngine* e, void* stream) {
  CHECK_ENGINE(e);
  e->stream = stream ? (cudaStream_t)stream : e->own_stream;
  return SLBM_OK;
}

int slbm_engine_set_params(SlbmEngine* e, int model, double omega, double lambda_odd) {
  CHECK_ENGINE(e);
  SLBM_TRY(check_model(e->q, model));
  e->model = model;
  e->omega = omega;
  e->lambda_odd = lambda_odd;
  for (double& w : e->hr) w = 1.0;  // back to the closed-form cumulant
  for (auto& gx : e->graph)
    if (gx) {
      cudaGraphExecDestroy(gx);
      gx = nullptr;
    }
  return SLBM_OK;
}

int slbm_engine_set_cumulant_rates(SlbmEngine* e, double bulk, const double* higher,
                                   int force_general) {
  CHECK_ENGINE(e);
  if (e->model != SLBM_CUMULANT && e->model != SLBM_CUMULANT_GEN)
    return fail(SLBM_ECONFIG, "cumulant rates need an engine with the cumulant model");
  double hr[8] = {1, 1, 1, 1, 1, 1, 1, 1};
  if (higher)
    for (int k = 0; k < 8; ++k) hr[k] = higher[k];
  auto ok = [](double w) { return std::isfinite(w) && w > 0.0 && w < 2.0; };
  if (!ok(bulk)) return fail(SLBM_ECONFIG, "bulk rate must lie in (0, 2)");
  for (int k = 0; k < 8; ++k)
    if (!ok(hr[k])) return fail(SLBM_ECONFIG, "higher-order cumulant rates must lie in (0, 2)");
  bool general = force_general != 0;
  for (int k = 0; k < 8; ++k) general = general || hr[k] != 1.0;
  DeviceGuard guard(e->device);
  if (general && !e->d_hr) SLBM_CUDA_TRY(cudaMalloc(&e->d_hr, sizeof(hr)));
  if (e->d_hr) SLBM_CUDA_TRY(cudaMemcpy(e->d_hr, hr, sizeof(hr), cudaMemcpyHostToDevice));
  std::memcpy(e->hr, hr, sizeof(hr));
  e->lambda_odd = bulk;
  e->model = general ? SLBM_CUMULANT_GEN : SLBM_CUMULANT;
  for (auto& gx : e->graph)
    if (gx) {
      cudaGraphExecDestroy(gx);
      gx = nullptr;
    }
  return SLBM_OK;
}

int slbm_export_lists(const SlbmEngine* e, uint32_t* idx, int64_t* fluid_coords,
                      int64_t* ubb_slot, int64_t* ubb_partner, double* ubb_corr,
                      int64_t* ghost_q, int64_t* ghost_pflat, int64_t* ghost_slot) {
  CHECK_ENGINE(e);
  DeviceGuard guard(e->device);
  cudaStream_t s = e->stream;
  const int64_t n = e->n_fluid;
  if (idx && e->layout) return fail(SLBM_ECONFIG, "a dense engine has no index list");
  if (idx) SLBM_TRY(export_idx_logical(const_cast<SlbmEngine*>(e), idx));
  std::vector<uint32_t> xf;
  if (fluid_coords) {
    xf.resize(n);
    SLBM_CUDA_TRY(
        cudaMemcpyAsync(xf.data(), e->x_flat, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  }
  std::vector<uint32_t> us, up;
  if (e->n_ubb && (ubb_slot || ubb_partner)) {
    us.resize(e->n_ubb);
    up.resize(e->n_ubb);
    SLBM_CUDA_TRY(cudaMemcpyAsync(us.data(), e->ubb_slot, e->n_ubb * 4, cudaMemcpyDeviceToHost, s));
    SLBM_CUDA_TRY(
        cudaMemcpyAsync(up.data(), e->ubb_partner, e->n_ubb * 4, cudaMemcpyDeviceToHost, s));
  }
  if (e->n_ubb && ubb_corr)
    SLBM_CUDA_TRY(cudaMemcpyAsync(ubb_corr, e->ubb_corr, e->n_ubb * sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
  SLBM_CUDA_TRY(cudaStreamSynchronize(s));
  if (fluid_coords) {
    for (int64_t c = 0; c < n; ++c) {
      int64_t x, y, z;
      e->geo.coords(xf[c], x, y, z);
      fluid_coords[c * e->dim + 0] = x;
      fluid_coords[c * e->dim + 1] = y;
      if (e->dim == 3) fluid_coords[c * e->dim + 2] = z;
    }
  }
  for (int64_t i = 0; i < e->n_ubb; ++i) {  // device addresses -> slot ids
    if (ubb_slot) ubb_slot[i] = e->slot_of(us[i]);
    if (ubb_partner) ubb_partner[i] = e->slot_of(up[i]);
  }
  for (int q = 1; q < e->q; ++q) {
    for (int64_t k = 0; k < e->n_ghost_q[q]; ++k) {
      const int64_t at = e->ghost_off[q] + k;
      if (ghost_q) ghost_q[at] = q;
      if (ghost_pflat) ghost_pflat[at] = int64_t(e->ghost_key_host[at] & 0xffffffffull);
      if (ghost_slot) ghost_slot[at] = e->base[q] + n + e->n_ubb_q[q] + k;
    }
  }
  return SLBM_OK;
}

int slbm_engine_set_frame(SlbmEngine* e, const int32_t* lo, const int32_t* hi) {
  CHECK_ENGINE(e);
  if (e->layout) return fail(SLBM_ECONFIG, "per-face frames are for sparse engines");
  if (!lo || !hi) return fail(SLBM_ECONFIG, "null widths");
  int32_t l[3] = {0, 0, 0}, h[3] = {0, 0, 0};
  for (int a = 0; a < e->dim; ++a) {
    if (lo[a] < 0 || hi[a] < 0) return fail(SLBM_ECONFIG, "frame widths must be >= 0");
    l[a] = lo[a];
    h[a] = hi[a];
  }
  DeviceGuard guard(e->device);
  return set_frame(e, l, h);
}

int slbm_export_split(const SlbmEngine* e, int64_t* interior, int64_t* frame) {
  CHECK_ENGINE(e);
  if (!e->has_split) return fail(SLBM_ECONFIG, "engine has no split lists; build with frame_width");
  DeviceGuard guard(e->device);
  std::vector<uint32_t> b(size_t(std::max<int64_t>(e->n_frame, 1)));
  if (e->n_frame)
    SLBM_CUDA_TRY(cudaMemcpy(b.data(), e->frame_cids, e->n_frame * 4, cudaMemcpyDeviceToHost));
  if (frame)
    for (int64_t i = 0; i < e->n_frame; ++i) frame[i] = b[i];
  if (interior) {  // the complement of the (sorted) frame list
    int64_t k = 0, j = 0;
    for (int64_t c = 0; c < e->n_fluid; ++c) {
      if (j < e->n_frame && int64_t(b[j]) == c)
        ++j;
      else
        interior[k++] = c;
    }
  }
  return SLBM_OK;
}

int slbm_init_canonical_dev(SlbmEngine* e, const double* dev_values) {
  CHECK_ENGINE(e);
  DeviceGuard guard(e->device);
  if (e->layout) {  // dense.py:196-210
    SLBM_TRY(e->ensure_scratch(size_t(e->q) * e->n_fluid * sizeof(double)));
    SLBM_CUDA_TRY(cudaMemcpyAsync(e->d_scratch, dev_values,
                                  size_t(e->q) * e->n_fluid * sizeof(double), cudaMemcpyDefault,
                                  e->stream));
    return dense_init(e, e->d_scratch);
  }
  // sparse.py:205-210: poison everything, then write the Q direction groups
  SLBM_TRY(launch_fill(e->pdf, e->phys_slots, NAN, e->stream));
  if (e->tmp) SLBM_TRY(launch_fill(e->tmp, e->phys_slots, NAN, e->stream));
  for (int r = 0; r < e->q; ++r)
    SLBM_CUDA_TRY(cudaMemcpyAsync(e->pdf + e->pbase[r], dev_values + size_t(r) * e->n_fluid,
                                  e->n_fluid * sizeof(double), cudaMemcpyDefault, e->stream));
  e->parity = SLBM_EVEN;
  return SLBM_OK;
}

int slbm_init_canonical(SlbmEngine* e, const double* values) {
  CHECK_ENGINE(e);
  if (!values) return fail(SLBM_ECONFIG, "null values");
  DeviceGuard guard(e->device);
  if (e->layout) {
    SLBM_TRY(e->ensure_scratch(size_t(e->q) * e->n_fluid * sizeof(double)));
    SLBM_TRY(copy_h2d(e->d_scratch, values, size_t(e->q) * e->n_fluid * sizeof(double), e->device,
                      e->stream));
    SLBM_TRY(dense_init(e, e->d_scratch));
    SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return SLBM_OK;
  }
  // sparse.py:205-210: poison everything, then write the Q direction groups
  SLBM_TRY(launch_fill(e->pdf, e->phys_slots, NAN, e->stream));
  if (e->tmp) SLBM_TRY(launch_fill(e->tmp, e->phys_slots, NAN, e->stream));
  for (int r = 0; r < e->q; ++r)
    SLBM_TRY(copy_h2d(e->pdf + e->pbase[r], values + size_t(r) * e->n_fluid,
                      e->n_fluid * sizeof(double), e->device, e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  e->parity = SLBM_EVEN;
  return SLBM_OK;
}

int slbm_init_equilibrium(SlbmEngine* e, const double* rho, int rho_scalar, const double* u,
                          int u_scalar) {
  CHECK_ENGINE(e);
  if (!rho || !u) return fail(SLBM_ECONFIG, "null rho/u");
  DeviceGuard guard(e->device);
  const size_t nr = rho_scalar ? 1 : size_t(e->n_fluid);
  const size_t nu = u_scalar ? size_t(e->dim) : size_t(e->dim) * e->n_fluid;
  const size_t nq = e->layout ? size_t(e->q) * e->n_fluid : 0;
  SLBM_TRY(e->ensure_scratch((nr + nu + nq) * sizeof(double)));
  double* d_rho = e->d_scratch;
  double* d_u = e->d_scratch + nr;
  SLBM_CUDA_TRY(cudaMemcpyAsync(d_rho, rho, nr * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  SLBM_CUDA_TRY(cudaMemcpyAsync(d_u, u, nu * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  if (e->layout) {
    double* d_f = e->d_scratch + nr + nu;
    SLBM_TRY(launch_equilibrium_qn(e, d_rho, rho_scalar, d_u, u_scalar, d_f));
    SLBM_TRY(dense_init(e, d_f));
    SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return SLBM_OK;
  }
  SLBM_TRY(launch_fill(e->pdf, e->phys_slots, NAN, e->stream));
  if (e->tmp) SLBM_TRY(launch_fill(e->tmp, e->phys_slots, NAN, e->stream));
  SLBM_TRY(launch_equilibrium(e, d_rho, rho_scalar, d_u, u_scalar, nullptr));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  e->parity = SLBM_EVEN;
  return SLBM_OK;
}

int slbm_canonical_state(SlbmEngine* e, double* values) {
  CHECK_ENGINE(e);
  if (!values) return fail(SLBM_ECONFIG, "null values");
  DeviceGuard guard(e->device);
  if (e->layout) {  // dense.py:275-288
    SLBM_TRY(e->ensure_scratch(size_t(e->q) * e->n_fluid * sizeof(double)));
    SLBM_TRY(dense_canonical(e, e->d_scratch));
    return copy_d2h(values, e->d_scratch, size_t(e->q) * e->n_fluid * sizeof(double), e->device,
                    e->stream);
  }
  const bool odd = e->pattern == SLBM_AA && e->parity == SLBM_ODD;
  if (odd) SLBM_TRY(launch_refresh(e, SLBM_ODD));  // sparse.py:317
  for (int r = 0; r < e->q; ++r) {
    const int g = odd ? e->dirs.inv[r] : r;
    SLBM_TRY(copy_d2h(values + size_t(r) * e->n_fluid, e->pdf + e->pbase[g],
                      e->n_fluid * sizeof(double), e->device, e->stream));
  }
  return SLBM_OK;
}

int slbm_macroscopic(SlbmEngine* e, double* rho, double* u) {
  CHECK_ENGINE(e);
  if (!rho || !u) return fail(SLBM_ECONFIG, "null rho/u");
  DeviceGuard guard(e->device);
  const bool odd = e->pattern == SLBM_AA && e->parity == SLBM_ODD;
  if (odd) SLBM_TRY(launch_refresh(e, SLBM_ODD));
  const int64_t cells = e->geo.n_cells();
  if (!e->layout) {
    void* drho = mapped_device_ptr(rho);
    void* du = mapped_device_ptr(u);
    if (drho && du) {
      // pinned destinations
      if (mapped_out_enabled())  // the kernel writes straight into them over PCIe
        return launch_macroscopic_box(e, (double*)drho, (double*)du);
      // box fields into HBM (zeros at solids written by the kernel), then
      // one DMA copy each at the link rate
      SLBM_TRY(e->ensure_scratch(size_t(cells) * (1 + e->dim) * sizeof(double)));
      double* d_rho = e->d_scratch;
      double* d_u = e->d_scratch + cells;
      SLBM_TRY(launch_macroscopic_box(e, d_rho, d_u));
      SLBM_CUDA_TRY(cudaMemcpyAsync(rho, d_rho, size_t(cells) * sizeof(double),
                                    cudaMemcpyDeviceToHost, e->stream));
      SLBM_CUDA_TRY(cudaMemcpyAsync(u, d_u, size_t(cells) * e->dim * sizeof(double),
                                    cudaMemcpyDeviceToHost, e->stream));
      SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
      return SLBM_OK;
    }
  }
  const size_t nq = e->layout ? size_t(e->q) * e->n_fluid : 0;
  SLBM_TRY(e->ensure_scratch((size_t(cells) * (1 + e->dim) + nq) * sizeof(double)));
  double* d_rho = e->d_scratch;
  double* d_u = e->d_scratch + cells;
  SLBM_CUDA_TRY(cudaMemsetAsync(e->d_scratch, 0, size_t(cells) * (1 + e->dim) * sizeof(double),
                                e->stream));
  int st;
  if (e->layout) {
    double* d_f = e->d_scratch + size_t(cells) * (1 + e->dim);
    SLBM_TRY(dense_canonical(e, d_f));
    st = launch_macroscopic(e, d_f, d_rho, d_u);
  } else {
    st = launch_macroscopic(e, nullptr, d_rho, d_u);
  }
  if (st != SLBM_OK) return st;
  SLBM_TRY(copy_d2h(rho, d_rho, cells * sizeof(double), e->device, e->stream));
  return copy_d2h(u, d_u, cells * e->dim * sizeof(double), e->device, e->stream);
}

int slbm_macroscopic_compact(SlbmEngine* e, double* rho, double* u) {
  CHECK_ENGINE(e);
  if (!rho || !u) return fail(SLBM_ECONFIG, "null rho/u");
  DeviceGuard guard(e->device);
  const bool odd = e->pattern == SLBM_AA && e->parity == SLBM_ODD;
  if (odd) SLBM_TRY(launch_refresh(e, SLBM_ODD));
  const size_t n = size_t(e->n_fluid);
  const size_t nq = e->layout ? size_t(e->q) * n : 0;
  SLBM_TRY(e->ensure_scratch((n * (1 + e->dim) + nq) * sizeof(double)));
  double* d_rho = e->d_scratch;
  double* d_u = e->d_scratch + n;
  int st;
  if (e->layout) {
    double* d_f = e->d_scratch + n * (1 + e->dim);
    SLBM_TRY(dense_canonical(e, d_f));
    st = launch_macroscopic(e, d_f, d_rho, d_u, true);
  } else {
    st = launch_macroscopic(e, nullptr, d_rho, d_u, true);
  }
  if (st != SLBM_OK) return st;
  SLBM_TRY(copy_d2h(rho, d_rho, n * sizeof(double), e->device, e->stream));
  return copy_d2h(u, d_u, n * e->dim * sizeof(double), e->device, e->stream);
}

int slbm_macroscopic_global(SlbmEngine* e, double* dev_rho, double* dev_u,
                            const int64_t* gdims, const int64_t* origin) {
  CHECK_ENGINE(e);
  if (!dev_rho || !dev_u || !gdims || !origin) return fail(SLBM_ECONFIG, "null argument");
  if (e->layout) return fail(SLBM_ECONFIG, "global-box read-out: sparse engines only");
  for (int k = 0; k < 3; ++k)
    if (origin[k] < 0 || (k < e->dim && origin[k] + e->geo.n[k] > gdims[k]))
      return fail(SLBM_ECONFIG, "block outside the global box");
  DeviceGuard guard(e->device);
  const bool odd = e->pattern == SLBM_AA && e->parity == SLBM_ODD;
  if (odd) SLBM_TRY(launch_refresh(e, SLBM_ODD));
  return launch_macroscopic(e, nullptr, dev_rho, dev_u, false, gdims, origin);
}

int slbm_engine_sweep_ctas(const SlbmEngine* e, int* ctas) {
  CHECK_ENGINE(e);
  if (!ctas) return fail(SLBM_ECONFIG, "null output");
  *ctas = e->tune.even_ctas ? e->tune.even_ctas : e->even_ctas;  // 0: not decided yet
  return SLBM_OK;
}

int slbm_copy_to_host(void* host, const void* dev, int64_t bytes, int device) {
  if (!host || !dev || bytes < 0) return fail(SLBM_ECONFIG, "bad copy arguments");
  DeviceGuard guard(device);
  return copy_d2h(host, dev, size_t(bytes), device, nullptr);
}

int slbm_total_moments(SlbmEngine* e, double* out4) {
  CHECK_ENGINE(e);
  if (!out4) return fail(SLBM_ECONFIG, "null output");
  DeviceGuard guard(e->device);
  const bool odd = e->pattern == SLBM_AA && e->parity == SLBM_ODD;
  if (odd) SLBM_TRY(launch_refresh(e, SLBM_ODD));
  if (e->layout) {  // dense: canonical (q, n) array, per-direction sums
    const size_t nq = size_t(e->q) * e->n_fluid;
    SLBM_TRY(e->ensure_scratch((size_t(e->q) + nq) * sizeof(double)));
    double* d_f = e->d_scratch + e->q;
    SLBM_TRY(dense_canonical(e, d_f));
    for (int r = 0; r < e->q; ++r)
      SLBM_TRY(launch_sum(d_f + size_t(r) * e->n_fluid, e->n_fluid, e->d_scratch + r, e->stream));
    std::vector<double> parts(e->q);
    SLBM_CUDA_TRY(cudaMemcpyAsync(parts.data(), e->d_scratch, e->q * sizeof(double),
                                  cudaMemcpyDeviceToHost, e->stream));
    SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    for (int k = 0; k < 4; ++k) out4[k] = 0.0;
    for (int r = 0; r < e->q; ++r) {
      out4[0] += parts[r];
      for (int a = 0; a < 3; ++a)
        if (e->dirs.c[r][a] > 0)
          out4[1 + a] += parts[r];
        else if (e->dirs.c[r][a] < 0)
          out4[1 + a] -= parts[r];
    }
    return SLBM_OK;
  }
  SLBM_TRY(e->ensure_scratch(4 * sizeof(double)));
  SLBM_TRY(launch_moments(e, e->d_scratch));
  SLBM_CUDA_TRY(cudaMemcpyAsync(out4, e->d_scratch, 4 * sizeof(double), cudaMemcpyDeviceToHost,
                                e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SLBM_OK;
}

int slbm_total_mass(SlbmEngine* e, double* mass) {
  if (!mass) return fail(SLBM_ECONFIG, "null output");
  double m[4];
  SLBM_TRY(slbm_total_moments(e, m));
  *mass = m[0];
  return SLBM_OK;
}

int slbm_refresh_boundary(SlbmEngine* e, int parity) {
  CHECK_ENGINE(e);
  if (parity != SLBM_EVEN && parity != SLBM_ODD) return fail(SLBM_ECONFIG, "bad parity");
  DeviceGuard guard(e->device);
  return launch_refresh(e, parity);
}

// an engine of a linked block group reads other blocks' slots through the
// group's list; stepping it alone would read its unmaintained ghosts
#define CHECK_NOT_LINKED(e)                                                       \
  do {                                                                            \
    if ((e)->pool)                                                                \
      return fail(SLBM_ECONFIG, "engine belongs to a linked block group: step it " \
                                "through the group (Domain)");                    \
  } while (0)

int slbm_step(SlbmEngine* e, int phase) {
  CHECK_ENGINE(e);
  CHECK_NOT_LINKED(e);
  if (phase != SLBM_PHASE_ALL && phase != SLBM_PHASE_INTERIOR && phase != SLBM_PHASE_FRAME)
    return fail(SLBM_ECONFIG, "unknown sweep phase");
  if (phase != SLBM_PHASE_ALL && !e->has_split)
    return fail(SLBM_ECONFIG, "sweep needs split lists; build with frame_width");
  DeviceGuard guard(e->device);
  return launch_step(e, phase);
}

int slbm_finish_step(SlbmEngine* e) {
  CHECK_ENGINE(e);
  CHECK_NOT_LINKED(e);
  DeviceGuard guard(e->device);
  if (e->pattern == SLBM_PULL)
    std::swap(e->pdf, e->tmp);
  else
    e->parity = 1 - e->parity;
  e->steps_done += 1;
  return launch_advance(e);
}

int slbm_run(SlbmEngine* e, int64_t n, int use_graph) {
  CHECK_ENGINE(e);
  CHECK_NOT_LINKED(e);
  DeviceGuard guard(e->device);
  int64_t done = 0;
  if (use_graph && resident_eligible(e, n)) {  // small block: one launch for all n steps
    for (; done < n; done += kResidentChunk) {
      const int64_t k = std::min<int64_t>(kResidentChunk, n - done);
      SLBM_TRY(launch_resident(e, k));
      if (k & 1) {
        if (e->pattern == SLBM_PULL)
          std::swap(e->pdf, e->tmp);
        else
          e->parity = 1 - e->parity;
      }
      e->steps_done += k;
    }
    return SLBM_OK;
  }
  if (use_graph && n >= 2 && pair_eligible(e)) {  // temporally blocked step pairs
    if (e->parity == SLBM_ODD) {
      SLBM_TRY(sweep_once(e));
      done = 1;
    }
    for (; done + 2 <= n; done += 2) {
      SLBM_TRY(launch_pair(e));
      e->steps_done += 2;
    }
  }
  // a large D3Q19 engine measures its index-list sweep occupancy on its
  // first eager steps (kernels.cu sweep_ctas) before any graph bakes it in
  while (use_graph && done < n && e->q == 19 && e->even_ctas == 0 && e->tune.even_ctas == 0 &&
         e->tune.even_variant == 0 && e->n_fluid >= (int64_t(1) << 22) && e->layout == 0) {
    SLBM_TRY(sweep_once(e));
    ++done;
  }
  if (use_graph && n - done >= 2) {
    // state key: AA -> parity; pull -> which buffer is active (pdf < tmp)
    auto key = [&]() { return e->pattern == SLBM_AA ? e->parity : (e->pdf < e->tmp ? 0 : 1); };
    const int k = key();
    if (!e->graph[k]) {
      cudaGraph_t graph = nullptr;
      SLBM_CUDA_TRY(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
      const long long mark = g_launches.load();
      int st = sweep_once(e);
      if (st == SLBM_OK) st = sweep_once(e);
      e->graph_kernels[k] = g_launches.load() - mark;
      g_launches.fetch_sub(e->graph_kernels[k]);
      cudaError_t ce = cudaStreamEndCapture(e->stream, &graph);
      // the captured pair leaves the state where it started
      e->steps_done -= 2;
      if (st != SLBM_OK) return st;
      if (ce != cudaSuccess) return fail(SLBM_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
      ce = cudaGraphInstantiate(&e->graph[k], graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess) return fail(SLBM_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
    }
    int64_t pairs = 0;
    for (; done + 2 <= n; done += 2, pairs += 2) {
      SLBM_CUDA_TRY(cudaGraphLaunch(e->graph[k], e->stream));
      count_launch(e->graph_kernels[k]);
    }
    e->steps_done += pairs;
  }
  for (; done < n; ++done) SLBM_TRY(sweep_once(e));
  return SLBM_OK;
}

int slbm_poll_instability(SlbmEngine* e, int64_t* first_bad_step) {
  CHECK_ENGINE(e);
  DeviceGuard guard(e->device);
  SLBM_CUDA_TRY(cudaMemcpyAsync(e->h_bad, e->d_bad, sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  const unsigned long long v = *e->h_bad;
  if (v == ULLONG_MAX) {
    if (first_bad_step) *first_bad_step = -1;
    return SLBM_OK;
  }
  if (first_bad_step) *first_bad_step = int64_t(v);
  SLBM_CUDA_TRY(cudaMemsetAsync(e->d_bad, 0xff, sizeof(unsigned long long), e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return fail(SLBM_EUNSTABLE, "non-positive or non-finite density in collision input");
}

int slbm_poll_engines(SlbmEngine** engines, int n, int64_t* first_bad_step, int* which) {
  if (!engines || n < 0) return fail(SLBM_ECONFIG, "null engine list");
  if (first_bad_step) *first_bad_step = -1;
  if (which) *which = -1;
  // every flag read is queued first, each distinct stream synchronised once:
  // one host round trip for a whole block group instead of one per block
  std::vector<cudaStream_t> streams;
  for (int i = 0; i < n; ++i) {
    SlbmEngine* e = engines[i];
    CHECK_ENGINE(e);
    DeviceGuard guard(e->device);
    SLBM_CUDA_TRY(cudaMemcpyAsync(e->h_bad, e->d_bad, sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, e->stream));
    if (std::find(streams.begin(), streams.end(), e->stream) == streams.end())
      streams.push_back(e->stream);
  }
  for (cudaStream_t st : streams) SLBM_CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < n; ++i) {
    SlbmEngine* e = engines[i];
    if (*e->h_bad == ULLONG_MAX) continue;
    if (first_bad_step) *first_bad_step = int64_t(*e->h_bad);
    if (which) *which = i;
    DeviceGuard guard(e->device);
    SLBM_CUDA_TRY(cudaMemsetAsync(e->d_bad, 0xff, sizeof(unsigned long long), e->stream));
    SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return fail(SLBM_EUNSTABLE, "non-positive or non-finite density in collision input");
  }
  return SLBM_OK;
}

int slbm_synchronize(SlbmEngine* e) {
  CHECK_ENGINE(e);
  DeviceGuard guard(e->device);
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SLBM_OK;
}

int slbm_parity(const SlbmEngine* e, int* parity) {
  CHECK_ENGINE(e);
  *parity = e->parity;
  return SLBM_OK;
}

int slbm_buffer_state(const SlbmEngine* e, int* state) {
  CHECK_ENGINE(e);
  // pull: which of the two buffers is current (the pointers a captured graph
  // bakes in); AA: always 0 (one buffer, in place)
  *state = (e->pattern == SLBM_PULL && e->tmp != nullptr && e->tmp < e->pdf) ? 1 : 0;
  return SLBM_OK;
}

int slbm_set_parity(SlbmEngine* e, int parity) {
  CHECK_ENGINE(e);
  if (parity != SLBM_EVEN && parity != SLBM_ODD) return fail(SLBM_ECONFIG, "bad parity");
  e->parity = parity;
  return SLBM_OK;
}

int slbm_slot_index(const SlbmEngine* ce, const int64_t* qs, const int64_t* pflat, int64_t n,
                    int64_t* out) {
  CHECK_ENGINE(ce);
  if (n == 0) return SLBM_OK;
  if (ce->layout) return dense_slots(ce, qs, pflat, n, out);
  SlbmEngine* e = const_cast<SlbmEngine*>(ce);
  DeviceGuard guard(e->device);
  int64_t* d = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&d, size_t(n) * 3 * sizeof(int64_t) + sizeof(int), e->stream));
  int* d_err = reinterpret_cast<int*>(d + 3 * n);
  SLBM_CUDA_TRY(cudaMemcpyAsync(d, qs, n * sizeof(int64_t), cudaMemcpyHostToDevice, e->stream));
  SLBM_CUDA_TRY(cudaMemcpyAsync(d + n, pflat, n * sizeof(int64_t), cudaMemcpyHostToDevice, e->stream));
  SLBM_CUDA_TRY(cudaMemsetAsync(d_err, 0, sizeof(int), e->stream));
  SLBM_TRY(launch_slot_lookup(e, d, d + n, n, d + 2 * n, d_err));
  int h_err = 0;
  SLBM_CUDA_TRY(cudaMemcpyAsync(out, d + 2 * n, n * sizeof(int64_t), cudaMemcpyDeviceToHost, e->stream));
  SLBM_CUDA_TRY(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
  SLBM_CUDA_TRY(cudaFreeAsync(d, e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  if (h_err) return fail(SLBM_EPROTOCOL, "exchange addressed a non-fluid cell slot");
  return SLBM_OK;
}

int slbm_export_cid_map(const SlbmEngine* e, int32_t* out) {
  CHECK_ENGINE(e);
  if (!out) return fail(SLBM_ECONFIG, "null out");
  if (e->layout || !e->cid_map) return fail(SLBM_ECONFIG, "a dense engine has no cid map");
  DeviceGuard guard(e->device);
  return copy_d2h(out, e->cid_map, size_t(e->geo.n_padded()) * sizeof(int32_t), e->device,
                  e->stream);
}

int slbm_ghost_slot_index(const SlbmEngine* e, const int64_t* qs, const int64_t* pflat,
                          int64_t n, int64_t* out) {
  CHECK_ENGINE(e);
  if (e->layout) return dense_slots(e, qs, pflat, n, out);  // dense.py:319-322
  const Geometry& g = e->geo;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t q = qs[i];
    const int64_t p = pflat[i];
    bool ok = q >= 1 && q < e->q && p >= 0 && p < g.n_padded();
    int64_t slot = -1;
    if (ok) {
      int64_t v[3];
      g.coords(p, v[0], v[1], v[2]);
      int sig = 0;
      for (int a = 0; a < 3; ++a) {
        int s = 0;
        if (a < g.dim) s = v[a] < 0 ? -1 : (v[a] >= g.n[a] ? 1 : 0);
        sig = sig * 3 + (s + 1);
      }
      const uint64_t key = (uint64_t(sig) << 32) | uint64_t(p);
      auto b = e->ghost_key_host.begin() + e->ghost_off[q];
      auto en = e->ghost_key_host.begin() + e->ghost_off[q + 1];
      auto it = std::lower_bound(b, en, key);
      if (it != en && *it == key) slot = e->base[q] + e->n_fluid + e->n_ubb_q[q] + (it - b);
    }
    if (slot < 0)
      return fail(SLBM_EPROTOCOL, "exchange asked for halo slot (" + std::to_string(q) + ", " +
                                      std::to_string(p) + ") that no cell reads");
    out[i] = slot;
  }
  return SLBM_OK;
}

int slbm_read_slots(SlbmEngine* e, const int64_t* slots, int64_t n, double* outv) {
  CHECK_ENGINE(e);
  if (n == 0) return SLBM_OK;
  DeviceGuard guard(e->device);
  uint32_t* d_slots = nullptr;
  SLBM_TRY(upload_slots(e, slots, n, &d_slots));
  double* d_out = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&d_out, n * sizeof(double), e->stream));
  SLBM_TRY(launch_gather(e->pdf, d_slots, n, d_out, e->stream));
  SLBM_CUDA_TRY(cudaMemcpyAsync(outv, d_out, n * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  SLBM_CUDA_TRY(cudaFreeAsync(d_out, e->stream));
  SLBM_CUDA_TRY(cudaFreeAsync(d_slots, e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SLBM_OK;
}

int slbm_write_slots(SlbmEngine* e, const int64_t* slots, int64_t n, const double* in) {
  CHECK_ENGINE(e);
  if (n == 0) return SLBM_OK;
  DeviceGuard guard(e->device);
  uint32_t* d_slots = nullptr;
  SLBM_TRY(upload_slots(e, slots, n, &d_slots));
  double* d_in = nullptr;
  SLBM_CUDA_TRY(cudaMallocAsync(&d_in, n * sizeof(double), e->stream));
  SLBM_CUDA_TRY(cudaMemcpyAsync(d_in, in, n * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  SLBM_TRY(launch_scatter(e->pdf, d_slots, n, d_in, e->stream));
  SLBM_CUDA_TRY(cudaFreeAsync(d_in, e->stream));
  SLBM_CUDA_TRY(cudaFreeAsync(d_slots, e->stream));
  SLBM_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SLBM_OK;
}

int slbm_pdf_pointer(const SlbmEngine* e, double** dev_pdf) {
  CHECK_ENGINE(e);
  *dev_pdf = e->pdf;
  return SLBM_OK;
}

int slbm_pdf_layout(const SlbmEngine* e, int64_t* group_start, int64_t* n_elements) {
  CHECK_ENGINE(e);
  for (int q = 0; q <= e->q; ++q)
    if (group_start) group_start[q] = e->layout ? e->base[q] : e->pbase[q];
  if (n_elements) *n_elements = e->layout ? e->total_slots : e->phys_slots;
  return SLBM_OK;
}

}  // extern "C"
