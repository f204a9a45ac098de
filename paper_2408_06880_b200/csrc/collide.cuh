// Collision arithmetic for one cell, fp64, operation order pinned to the
// reference so results are bit-identical.  The library is built
// with -fmad=false, so no multiply-add contraction changes the rounding.
//
//   moments           core.py:96-124   rho = t0 + t1, then += t2..; u_a is
//                                      accumulated from 0.0 by +/- t_q in q
//                                      order, then divided by rho
//   equilibrium       core.py:127-146  usq = ((ux*ux) + uy*uy) + uz*uz;
//                                      cu from 0.0 by +/- u_a;
//                                      (w*rho) * (((1 + 3cu) + (4.5cu)cu) - 1.5usq)
//   SRT               core.py:153-154  t - omega * (t - feq)
//   TRT               core.py:158-170  (t - we*(sym - sym_eq)) - wo*(asym - asym_eq)
//   instability       core.py:108-111  rho non-finite or <= 0
//
// The caller supplies a `sink(integral_constant<q>, value)` that stores the
// post-collision value of direction q wherever its streaming pattern wants
// it, so no output array has to stay live in registers.
#pragma once

#include "common.cuh"
#include "cumulant.cuh"

namespace slbm {

template <class L>
struct Moments {
  double rho, ux, uy, uz, usq;
  bool bad;
};

// `t` is anything indexable by direction: a register array, or a view onto
// the shared-memory staging buffer of the asynchronous gather kernel.
template <class L, class TV>
__device__ __forceinline__ Moments<L> moments(const TV& t) {
  Moments<L> m;
  double rho = t[0] + t[1];
  sfor<2, L::Q>([&](auto q) { rho = rho + t[q]; });
  m.bad = !isfinite(rho) || rho <= 0.0;
  double ux = 0.0, uy = 0.0, uz = 0.0;
  sfor<0, L::Q>([&](auto q) {
    if constexpr (L::CX[q] == 1) ux = ux + t[q];
    if constexpr (L::CX[q] == -1) ux = ux - t[q];
  });
  sfor<0, L::Q>([&](auto q) {
    if constexpr (L::CY[q] == 1) uy = uy + t[q];
    if constexpr (L::CY[q] == -1) uy = uy - t[q];
  });
  if constexpr (L::DIM == 3) {
    sfor<0, L::Q>([&](auto q) {
      if constexpr (L::CZ[q] == 1) uz = uz + t[q];
      if constexpr (L::CZ[q] == -1) uz = uz - t[q];
    });
  }
  m.rho = rho;
  m.ux = ux / rho;
  m.uy = uy / rho;
  m.uz = (L::DIM == 3) ? uz / rho : 0.0;
  double usq = m.ux * m.ux;
  usq = usq + m.uy * m.uy;
  if constexpr (L::DIM == 3) usq = usq + m.uz * m.uz;
  m.usq = usq;
  return m;
}

template <class L, int Q_>
__device__ __forceinline__ double feq(const Moments<L>& m) {
  double cu = 0.0;
  if constexpr (L::CX[Q_] == 1) cu = cu + m.ux;
  if constexpr (L::CX[Q_] == -1) cu = cu - m.ux;
  if constexpr (L::CY[Q_] == 1) cu = cu + m.uy;
  if constexpr (L::CY[Q_] == -1) cu = cu - m.uy;
  if constexpr (L::DIM == 3) {
    if constexpr (L::CZ[Q_] == 1) cu = cu + m.uz;
    if constexpr (L::CZ[Q_] == -1) cu = cu - m.uz;
  }
  constexpr double w = weight<L>(Q_);
  double poly = 1.0 + 3.0 * cu;
  poly = poly + (4.5 * cu) * cu;
  poly = poly - 1.5 * m.usq;
  return (w * m.rho) * poly;
}

// returns true when the cell is unstable (the values are still produced)
template <class L, int MODEL, class TV, class Sink>
__device__ __forceinline__ bool collide(const TV& t, double omega, double lam, Sink&& sink) {
  if constexpr (MODEL == SLBM_CUMULANT) {
    return cumulant_collide<L>(t, omega, sink);
  } else {
    const Moments<L> m = moments<L>(t);
    if constexpr (MODEL == SLBM_SRT) {
      sfor<0, L::Q>([&](auto q) {
        const double fe = feq<L, q>(m);
        sink(q, t[q] - omega * (t[q] - fe));
      });
    } else {
      // TRT: each direction pairs with its opposite; both outputs of a pair
      // come from the same two equilibria (same expressions as core.py:163-169).
      sfor<0, L::Q>([&](auto q) {
        constexpr int qb = L::INV[q];
        if constexpr (q <= qb) {
          const double fe = feq<L, q>(m);
          const double feb = feq<L, qb>(m);
          {
            const double sym = 0.5 * (t[q] + t[qb]);
            const double asym = 0.5 * (t[q] - t[qb]);
            const double sym_eq = 0.5 * (fe + feb);
            const double asym_eq = 0.5 * (fe - feb);
            sink(q, (t[q] - omega * (sym - sym_eq)) - lam * (asym - asym_eq));
          }
          if constexpr (q != qb) {
            const double sym = 0.5 * (t[qb] + t[q]);
            const double asym = 0.5 * (t[qb] - t[q]);
            const double sym_eq = 0.5 * (feb + fe);
            const double asym_eq = 0.5 * (feb - fe);
            sink(std::integral_constant<int, qb>{},
                 (t[qb] - omega * (sym - sym_eq)) - lam * (asym - asym_eq));
          }
        }
      });
    }
    return m.bad;
  }
}

}  // namespace slbm
