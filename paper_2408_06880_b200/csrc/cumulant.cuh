// Cumulant collision (D3Q27).  Not part of the reference package (SURVEY
// F12); placeholder until the implementation lands — the host rejects the
// model with SLBM_ECONFIG, so this body is never reached.
#pragma once

#include "common.cuh"

namespace slbm {

template <class L, class TV, class Sink>
__device__ __forceinline__ bool cumulant_collide(const TV& t, double omega, Sink&& sink) {
  sfor<0, L::Q>([&](auto q) { sink(q, t[q]); });
  return true;
}

}  // namespace slbm
