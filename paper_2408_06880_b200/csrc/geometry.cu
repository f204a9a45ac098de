// Overlapping-sphere voxelizer (input generation for the packed-bed
// benchmarks).  Rasterization rule and floating-point evaluation order
// follow the reference voxelize (pkg/src/slbm/geometry.py:150-178) at
// resolution 1: per axis the candidate range is
//   [max(0, floor(c - r - 0.5)), min(n - 1, ceil(c + r - 0.5))],
// the cell centre is i + 0.5, and a cell is solid iff
//   ((0 + dx*dx) + dy*dy) + dz*dz < r*r.
// Spheres may overlap (the reference's non-overlapping packer
// cannot reach porosity 0.3-0.5).
#include <cmath>

#include "engine.cuh"

namespace {

__global__ void k_voxelize(const double* centers, int64_t n, double r, int3 dims,
                           uint8_t* solid) {
  const int64_t s = blockIdx.x;
  if (s >= n) return;
  const double c[3] = {centers[3 * s], centers[3 * s + 1], centers[3 * s + 2]};
  const int nd[3] = {dims.x, dims.y, dims.z};
  int lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = max(0, int(floor((c[a] - r) * 1.0 - 0.5)));
    hi[a] = min(nd[a] - 1, int(ceil((c[a] + r) * 1.0 - 0.5)));
    if (hi[a] < lo[a]) return;
  }
  const double r2 = r * r;
  const int ex = hi[0] - lo[0] + 1, ey = hi[1] - lo[1] + 1, ez = hi[2] - lo[2] + 1;
  const int64_t total = int64_t(ex) * ey * ez;
  for (int64_t i = threadIdx.x; i < total; i += blockDim.x) {
    const int x = lo[0] + int(i % ex);
    const int y = lo[1] + int((i / ex) % ey);
    const int z = lo[2] + int(i / (int64_t(ex) * ey));
    const double dx = (double(x) + 0.5) / 1.0 - c[0];
    const double dy = (double(y) + 0.5) / 1.0 - c[1];
    const double dz = (double(z) + 0.5) / 1.0 - c[2];
    double d2 = 0.0 + dx * dx;
    d2 = d2 + dy * dy;
    d2 = d2 + dz * dz;
    if (d2 < r2) solid[(int64_t(z) * nd[1] + y) * nd[0] + x] = 1;
  }
}

}  // namespace

extern "C" int slbm_voxelize_spheres(const int32_t* dims, const double* centers, int64_t n,
                                     double diameter, int device, uint8_t* solid) {
  using namespace slbm;
  if (!dims || !solid || (n && !centers)) return fail(SLBM_ECONFIG, "null argument");
  cudaSetDevice(device);
  const int64_t cells = int64_t(dims[0]) * dims[1] * dims[2];
  uint8_t* d_solid = nullptr;
  double* d_c = nullptr;
  SLBM_CUDA_TRY(cudaMalloc(&d_solid, cells));
  SLBM_CUDA_TRY(cudaMemset(d_solid, 0, cells));
  if (n) {
    SLBM_CUDA_TRY(cudaMalloc(&d_c, n * 3 * sizeof(double)));
    SLBM_CUDA_TRY(cudaMemcpy(d_c, centers, n * 3 * sizeof(double), cudaMemcpyHostToDevice));
    { k_voxelize<<<unsigned(n), 256>>>(d_c, n, diameter / 2.0, make_int3(dims[0], dims[1], dims[2]),
                                     d_solid); slbm::count_launch(); }
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  SLBM_CUDA_TRY(cudaMemcpy(solid, d_solid, cells, cudaMemcpyDeviceToHost));
  cudaFree(d_solid);
  if (d_c) cudaFree(d_c);
  return SLBM_OK;
}
