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

// Signed sums without the reference's 0.0 seed.
//
// The reference accumulates from 0.0 (`u = zeros; u[a] += / -= t[q]`,
// core.py:113-122; `cu = zeros_like(rho)`, :138-144).  Seeding with the
// first term instead is exact — 0.0 + x == x and 0.0 - x == -x in IEEE
// round-to-nearest — except for the sign of an exact zero (0.0 + -0.0 is
// +0.0).  A signed zero in u or cu cannot reach any output: u and cu enter
// the equilibrium only through 1 + 3cu, (4.5cu)cu and u*u, which are
// sign-of-zero invariant.  This drops one fp64 add per velocity component
// and per equilibrium direction.
template <class L, int A>
__host__ __device__ constexpr int comp(int q) {
  return A == 0 ? L::CX[q] : (A == 1 ? L::CY[q] : L::CZ[q]);
}

template <class L, int A>
__host__ __device__ constexpr int first_nonzero() {
  for (int q = 0; q < L::Q; ++q)
    if (comp<L, A>(q) != 0) return q;
  return -1;
}

template <class L, int A, class TV>
__device__ __forceinline__ double component_sum(const TV& t) {
  constexpr int first = first_nonzero<L, A>();
  double acc = 0.0;
  sfor<0, L::Q>([&](auto q) {
    constexpr int c = comp<L, A>(q);
    if constexpr (q == first) {
      acc = (c == 1) ? t[q] : -t[q];
    } else if constexpr (c == 1) {
      acc = acc + t[q];
    } else if constexpr (c == -1) {
      acc = acc - t[q];
    }
  });
  return acc;
}

// c_q . u with the same seeding rule, components in x, y, z order
template <class L, int Q_>
__device__ __forceinline__ double c_dot_u(const Moments<L>& m) {
  double acc = 0.0;
  bool any = false;
  auto add = [&](int c, double u) {
    if (c == 0) return;
    acc = any ? (c == 1 ? acc + u : acc - u) : (c == 1 ? u : -u);
    any = true;
  };
  add(L::CX[Q_], m.ux);
  add(L::CY[Q_], m.uy);
  if constexpr (L::DIM == 3) add(L::CZ[Q_], m.uz);
  return acc;
}

// `t` is anything indexable by direction: a register array, or a view onto
// the shared-memory staging buffer of the asynchronous gather kernel.
template <class L, class TV>
__device__ __forceinline__ Moments<L> moments(const TV& t) {
  Moments<L> m;
  double rho = t[0] + t[1];
  sfor<2, L::Q>([&](auto q) { rho = rho + t[q]; });
  m.bad = !isfinite(rho) || rho <= 0.0;
  const double ux = component_sum<L, 0>(t);
  const double uy = component_sum<L, 1>(t);
  const double uz = (L::DIM == 3) ? component_sum<L, 2>(t) : 0.0;
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
  const double cu = (Q_ == 0) ? 0.0 : c_dot_u<L, Q_>(m);
  constexpr double w = weight<L>(Q_);
  double poly = 1.0 + 3.0 * cu;
  poly = poly + (4.5 * cu) * cu;
  poly = poly - 1.5 * m.usq;
  return (w * m.rho) * poly;
}

// Equilibria of an opposite pair (q, inv q) from one c.u.  Exact because
// cu(inv q) = -cu(q) (RNE rounding is sign symmetric), so
//   1 + 3 cu_b        = 1 - 3 cu          (3 * -x == -(3 * x))
//   (4.5 cu_b) cu_b   = (4.5 cu) cu       (sign rule of products)
// and w(q) = w(inv q): two polynomials share 3cu, (4.5cu)cu, 1.5usq, w*rho.
template <class L, int Q_>
__device__ __forceinline__ void feq_pair(const Moments<L>& m, double& fe, double& feb) {
  const double cu = c_dot_u<L, Q_>(m);
  constexpr double w = weight<L>(Q_);
  const double wr = w * m.rho;
  const double a = 3.0 * cu;
  const double b = (4.5 * cu) * cu;
  const double c = 1.5 * m.usq;
  fe = wr * (((1.0 + a) + b) - c);
  feb = wr * (((1.0 - a) + b) - c);
}

// SRT / TRT relaxation given the cell's moments; true when unstable
template <class L, int MODEL, class TV, class Sink>
__device__ __forceinline__ bool relax(const TV& t, const Moments<L>& m, double omega, double lam,
                                      Sink&& sink) {
  static_assert(MODEL == SLBM_SRT || MODEL == SLBM_TRT, "cumulants relax in cumulant.cuh");
  {
    const double ho = 0.5 * omega, hl = 0.5 * lam;  // TRT: exact halvings
    // rest direction: cu = 0, so poly = (1 + 0) - 1.5usq exactly, and the
    // TRT form reduces to the SRT form (sym = t0, asym = +0) bit for bit
    {
      constexpr double w0 = weight<L>(0);
      const double fe0 = (w0 * m.rho) * (1.0 - 1.5 * m.usq);
      sink(std::integral_constant<int, 0>{}, t[0] - omega * (t[0] - fe0));
    }
    sfor<1, L::Q>([&](auto q) {
      constexpr int qb = L::INV[q];
      if constexpr (q < qb) {
        double fe, feb;
        feq_pair<L, q>(m, fe, feb);
        if constexpr (MODEL == SLBM_SRT) {
          sink(q, t[q] - omega * (t[q] - fe));
          sink(std::integral_constant<int, qb>{}, t[qb] - omega * (t[qb] - feb));
        } else {
          // TRT (core.py:158-170).  For the opposite member the reference's
          // sym, sym_eq are the same sums (addition commutes exactly) and
          // asym, asym_eq are exact negations, so
          //   out_q  = (t_q  - A) - B,   out_qb = (t_qb - A) + B
          // with A = we (sym - sym_eq), B = wo (asym - asym_eq).
          // Halving is exact and commutes with round-to-nearest, so
          //   we * (0.5 S - 0.5 Se) == (0.5 we) * (S - Se)
          // bit for bit (S = t_q + t_qb, Se = fe + feb, same for the
          // differences): 4 fp64 multiplies fewer per pair.  (Exact unless
          // S - Se is subnormal, which a difference of two PDFs >= 2^-970
          // in magnitude cannot be.)
          const double A = ho * ((t[q] + t[qb]) - (fe + feb));
          const double B = hl * ((t[q] - t[qb]) - (fe - feb));
          sink(q, (t[q] - A) - B);
          sink(std::integral_constant<int, qb>{}, (t[qb] - A) + B);
        }
      }
    });
    return m.bad;
  }
}

// returns true when the cell is unstable (the values are still produced).
// Cumulant models: `lam` is the bulk rate, `hr` the higher-order rates.
template <class L, int MODEL, class TV, class Sink>
__device__ __forceinline__ bool collide(const TV& t, double omega, double lam, Sink&& sink,
                                        const double* hr = nullptr) {
  if constexpr (MODEL == SLBM_CUMULANT) {
    return cumulant_collide<L>(t, omega, lam, sink);
  } else if constexpr (MODEL == SLBM_CUMULANT_GEN) {
    return cumulant_collide_general<L>(t, omega, lam, hr, sink);
  } else {
    return relax<L, MODEL>(t, moments<L>(t), omega, lam, sink);
  }
}

}  // namespace slbm
