// Shared device/host helpers of the slbm_b200 library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <type_traits>
#include <utility>

#include "../../include/slbm_b200.h"
#include "lattice_tables.h"

namespace slbm {

// ---- launch accounting (slbm_launch_count) ---------------------------------
// Every kernel launch site of the library calls count_launch() right after the
// launch; a stream capture takes its launches back out and the graph adds
// them again on every replay, so the counter is the number of this library's
// kernels that reached the GPU (cub / NCCL kernels are not counted).
extern std::atomic<long long> g_launches;
inline void count_launch(long long n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---- programmatic dependent launch (PDL) ---------------------------------
// Per-step kernel chains (boundary -> sweep -> boundary ...) are launched with
// programmatic stream serialization: a kernel's CTAs may be scheduled while
// its predecessor drains.  Every kernel launched this way calls
// pdl_launch_dependents() early and pdl_wait() in EVERY thread before it
// touches data the predecessor writes (and before any early return), so
// "completed" stays transitive along the chain.  Both are no-ops when the
// kernel was launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e == cudaSuccess) count_launch();
  return e;
}

// ---- address space of pointers read from device tables -------------------
// A pointer loaded from memory (a block table, a shared-memory staging copy)
// is generic to the compiler: its loads and stores become LD/ST with a
// run-time space check instead of LDG/STG, ~9 % on the group sweeps
// (tools/group_probe.py).  Every table pointer is a cudaMalloc address.
template <class T>
__device__ __forceinline__ T* gmem(T* p) {
  __builtin_assume(__isGlobal(p));
  return p;
}

// ---- error plumbing -------------------------------------------------------
void set_error(const std::string& msg);
const char* last_error();

struct Status {
  int code = SLBM_OK;
};

#define SLBM_CUDA_TRY(expr)                                                         \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::slbm::set_error(std::string("CUDA error at " __FILE__ ":") +                \
                        std::to_string(__LINE__) + " " #expr ": " +                 \
                        cudaGetErrorString(_e));                                    \
      return SLBM_ECUDA;                                                            \
    }                                                                               \
  } while (0)

#define SLBM_TRY(expr)            \
  do {                            \
    int _s = (expr);              \
    if (_s != SLBM_OK) return _s; \
  } while (0)

inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

// ---- compile-time loops ---------------------------------------------------
// Unrolls f(integral_constant<I>) for I in [B, E).  Keeps every stencil
// table access a compile-time constant, and the floating-point operation
// order exactly the order written in the loop body.
template <int B, int E, class F>
__host__ __device__ __forceinline__ void sfor(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    sfor<B + 1, E>(f);
  }
}

template <class L>
__host__ __device__ constexpr double weight(int q) {
  return double(L::WNUM[q]) / double(L::WDEN[q]);
}

// ---- block geometry -------------------------------------------------------
// Public extents (x, y, z) with z = 1 for 2-d blocks.  The padded box adds a
// one-cell ring on every *active* axis (z is inactive in 2-d), so a padded
// flat index equals the reference's np.ravel_multi_index over the padded
// tags array (sparse.py:105, :119) in both 2-d and 3-d.
struct Geometry {
  int32_t n[3];      // X, Y, Z
  int64_t p[3];      // padded extents X+2, Y+2, Z+2 (or 1 for inactive z)
  int32_t off[3];    // ring offset per axis (1, 1, 1 or 0)
  uint8_t periodic[3];
  int32_t dim;

  __host__ __device__ int64_t padded_flat(int64_t x, int64_t y, int64_t z) const {
    return ((z + off[2]) * p[1] + (y + off[1])) * p[0] + (x + off[0]);
  }
  // interior coords from a padded flat index
  __host__ __device__ void coords(int64_t pf, int64_t& x, int64_t& y, int64_t& z) const {
    int64_t px = pf % p[0];
    int64_t r = pf / p[0];
    int64_t py = r % p[1];
    int64_t pz = r / p[1];
    x = px - off[0];
    y = py - off[1];
    z = pz - off[2];
  }
  __host__ __device__ int64_t interior_flat(int64_t x, int64_t y, int64_t z) const {
    return (z * n[1] + y) * n[0] + x;
  }
  __host__ __device__ int64_t n_cells() const { return int64_t(n[0]) * n[1] * n[2]; }
  __host__ __device__ int64_t n_padded() const { return p[0] * p[1] * p[2]; }
};

// direction table passed by value to builder kernels (runtime q)
struct DirTable {
  int32_t q;
  int8_t c[27][3];
  int8_t inv[27];
  double w[27];
};

}  // namespace slbm
