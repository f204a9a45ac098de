// Cumulant collision, D3Q27 (Geier, Schoenherr, Pasquali, Krafczyk 2015,
// "The cumulant lattice Boltzmann equation in three dimensions").  Not in
// the reference package: parity is UNPINNED.  Checked against
// two CPU restatements: oracle/cumulant_ref.py (this fast
// path's operation order) and oracle/cumulant_geier.py (an independent
// restatement from the paper's definitions: raw moments, the general
// moment-cumulant formula, a 27x27 solve back), plus physical tests
// (conservation, shear and bulk wave decay, Galilean invariance).
//
// Relaxation rates (Geier 2015 §4): omega = w1 (shear: off-diagonal and
// deviatoric second-order cumulants), w2 = bulk (trace of the second
// order, towards rho c_s^2 * 3), w3/w4 (third order, sums / differences of
// the (120, 102)-type pairs), w5 (C_111), w6 / w7 (the two deviatoric / the
// isotropic combination of the (220, 202, 022) fourth-order cumulants), w8
// (C_211-type), w9 (fifth order), w10 (sixth order).  Equilibria: second
// order rho c_s^2 delta, everything of order >= 3 zero.
//
// Two paths:
//   * cumulant_collide      w3..w10 = 1 (the default, lbmpy's "non-
//     parametrised" cumulant method): post-collision cumulants of order >= 3
//     vanish, so the post-collision central moments follow from rho, u and
//     the six relaxed second-order central moments alone:
//       order 0/1: rho, 0          order 2: relaxed kappa_ab
//       order 3/5: 0               order 4: products of order-2 / rho
//       order 6  : kappa_222 from the cumulant->moment relation (C_222 = 0)
//     and one backward chimera transform (x, then y, then z) gives f*.
//   * cumulant_collide_general  any w3..w10: forward chimera transform (z,
//     y, x) to all 27 central moments, cumulants of order 4-6 from the
//     generated relations (cumulant_rel.h, tools/gen_cumulant.py), the
//     relaxation above, the inverse relations, backward chimera.
#pragma once

#include "common.cuh"
#include "cumulant_rel.h"

namespace slbm {

template <class L>
struct Moments;
template <class L, class TV>
__device__ __forceinline__ Moments<L> moments(const TV& t);

// direction index of velocity (cx, cy, cz) in lattice L (compile time)
template <class L>
__host__ __device__ constexpr int dir_of(int cx, int cy, int cz) {
  for (int q = 0; q < L::Q; ++q)
    if (L::CX[q] == cx && L::CY[q] == cy && L::CZ[q] == cz) return q;
  return -1;
}

// signed sum of t over directions weighted by s(q) in {-1, 0, 1}, q order,
// seeded with the first contributing term
template <class L, class TV, class S>
__device__ __forceinline__ double weighted_sum(const TV& t, S s) {
  double acc = 0.0;
  bool any = false;
  sfor<0, L::Q>([&](auto q) {
    constexpr int w = S::template at<decltype(q)::value>();
    if constexpr (w != 0) {
      if (!any) {
        acc = (w > 0) ? t[q] : -t[q];
      } else {
        acc = (w > 0) ? acc + t[q] : acc - t[q];
      }
      any = true;
    }
  });
  return acc;
}

template <class L, int A, int B>
struct SecondWeight {  // c_A * c_B
  template <int Q_>
  static constexpr int at() {
    constexpr int ca = A == 0 ? L::CX[Q_] : (A == 1 ? L::CY[Q_] : L::CZ[Q_]);
    constexpr int cb = B == 0 ? L::CX[Q_] : (B == 1 ? L::CY[Q_] : L::CZ[Q_]);
    return ca * cb;
  }
};

struct ChimeraCoef {
  double am, a0, ap, bm, b0, bp;
};

__device__ __forceinline__ ChimeraCoef chimera_coef(double u) {
  const double uu = u * u;
  ChimeraCoef c;
  c.am = uu - u;
  c.a0 = 1.0 - uu;
  c.ap = uu + u;
  c.b0 = 2.0 * u;
  c.bm = c.b0 - 1.0;
  c.bp = c.b0 + 1.0;
  return c;
}

// backward chimera step along one axis: (k0, k1, k2) central moments of
// order 0, 1, 2 in that axis -> values at c = -1, 0, +1
__device__ __forceinline__ void back3(double k0, double k1, double k2, const ChimeraCoef& c,
                                      double& fm, double& f0, double& fp) {
  fm = ((k0 * c.am + k1 * c.bm) + k2) * 0.5;
  f0 = (k0 * c.a0 - k1 * c.b0) - k2;
  fp = ((k0 * c.ap + k1 * c.bp) + k2) * 0.5;
}
// k1 == 0 structurally
__device__ __forceinline__ void back3_even(double k0, double k2, const ChimeraCoef& c, double& fm,
                                           double& f0, double& fp) {
  fm = (k0 * c.am + k2) * 0.5;
  f0 = k0 * c.a0 - k2;
  fp = (k0 * c.ap + k2) * 0.5;
}
// k0 == k2 == 0 structurally
__device__ __forceinline__ void back3_odd(double k1, const ChimeraCoef& c, double& fm, double& f0,
                                          double& fp) {
  fm = (k1 * c.bm) * 0.5;
  f0 = -(k1 * c.b0);
  fp = (k1 * c.bp) * 0.5;
}

template <class L, class TV, class Sink>
__device__ __forceinline__ bool cumulant_collide(const TV& t, double omega, double bulk,
                                                 Sink&& sink) {
  static_assert(L::Q == 27, "cumulant collision is defined on D3Q27");
  const Moments<L> m = moments<L>(t);
  const double rho = m.rho, ux = m.ux, uy = m.uy, uz = m.uz;

  // raw second moments P_ab = sum c_a c_b f, then central ones
  const double pxx = weighted_sum<L>(t, SecondWeight<L, 0, 0>{});
  const double pyy = weighted_sum<L>(t, SecondWeight<L, 1, 1>{});
  const double pzz = weighted_sum<L>(t, SecondWeight<L, 2, 2>{});
  const double pxy = weighted_sum<L>(t, SecondWeight<L, 0, 1>{});
  const double pxz = weighted_sum<L>(t, SecondWeight<L, 0, 2>{});
  const double pyz = weighted_sum<L>(t, SecondWeight<L, 1, 2>{});
  const double jx = rho * ux, jy = rho * uy, jz = rho * uz;
  const double kxx = pxx - jx * ux;
  const double kyy = pyy - jy * uy;
  const double kzz = pzz - jz * uz;
  const double kxy = pxy - jx * uy;
  const double kxz = pxz - jx * uz;
  const double kyz = pyz - jy * uz;

  // relaxation: deviatoric parts with omega, the trace towards its
  // equilibrium rho with the bulk rate (bulk == 1 gives rho exactly:
  // rho + 0 * (tr - rho))
  const double om1 = 1.0 - omega;
  const double dxy = om1 * (kxx - kyy);
  const double dxz = om1 * (kxx - kzz);
  const double tr = rho + (1.0 - bulk) * (((kxx + kyy) + kzz) - rho);
  const double sxx = ((tr + dxy) + dxz) / 3.0;
  const double syy = sxx - dxy;
  const double szz = sxx - dxz;
  const double sxy = om1 * kxy;
  const double sxz = om1 * kxz;
  const double syz = om1 * kyz;

  // post-collision central moments of order 4 and 6 (orders 3, 5 vanish)
  const double ir = 1.0 / rho;
  const double k220 = (sxx * syy + 2.0 * (sxy * sxy)) * ir;
  const double k202 = (sxx * szz + 2.0 * (sxz * sxz)) * ir;
  const double k022 = (syy * szz + 2.0 * (syz * syz)) * ir;
  const double k211 = (sxx * syz + 2.0 * (sxy * sxz)) * ir;
  const double k121 = (syy * sxz + 2.0 * (sxy * syz)) * ir;
  const double k112 = (szz * sxy + 2.0 * (sxz * syz)) * ir;
  const double lin = ((sxx * k022 + syy * k202) + szz * k220) +
                     4.0 * ((syz * k211 + sxz * k121) + sxy * k112);
  const double cub = (16.0 * ((sxy * sxz) * syz) +
                      4.0 * (((sxz * sxz) * syy + (syz * syz) * sxx) + (sxy * sxy) * szz)) +
                     2.0 * ((sxx * syy) * szz);
  const double k222 = lin * ir - cub * (ir * ir);

  // backward chimera: x lines (b, c) -> G[i][b][c]
  const ChimeraCoef cx = chimera_coef(ux), cy = chimera_coef(uy), cz = chimera_coef(uz);
  double G[3][3][3];
  back3_even(rho, sxx, cx, G[0][0][0], G[1][0][0], G[2][0][0]);
  back3_odd(sxy, cx, G[0][1][0], G[1][1][0], G[2][1][0]);
  back3_even(syy, k220, cx, G[0][2][0], G[1][2][0], G[2][2][0]);
  back3_odd(sxz, cx, G[0][0][1], G[1][0][1], G[2][0][1]);
  back3_even(syz, k211, cx, G[0][1][1], G[1][1][1], G[2][1][1]);
  back3_odd(k121, cx, G[0][2][1], G[1][2][1], G[2][2][1]);
  back3_even(szz, k202, cx, G[0][0][2], G[1][0][2], G[2][0][2]);
  back3_odd(k112, cx, G[0][1][2], G[1][1][2], G[2][1][2]);
  back3_even(k022, k222, cx, G[0][2][2], G[1][2][2], G[2][2][2]);
  // y lines (i, c) -> H[i][j][c], stored back into G
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double a, b, d;
      back3(G[i][0][c], G[i][1][c], G[i][2][c], cy, a, b, d);
      G[i][0][c] = a;
      G[i][1][c] = b;
      G[i][2][c] = d;
    }
  }
  // z lines (i, j) -> f[i][j][k]
  sfor<0, 9>([&](auto ij) {
    constexpr int i = decltype(ij)::value / 3, j = decltype(ij)::value % 3;
    double a, b, d;
    back3(G[i][j][0], G[i][j][1], G[i][j][2], cz, a, b, d);
    sink(std::integral_constant<int, dir_of<L>(i - 1, j - 1, -1)>{}, a);
    sink(std::integral_constant<int, dir_of<L>(i - 1, j - 1, 0)>{}, b);
    sink(std::integral_constant<int, dir_of<L>(i - 1, j - 1, 1)>{}, d);
  });
  return m.bad;
}

// forward chimera step along one axis: values at c = -1, 0, +1 -> central
// moments of order 0, 1, 2 about u
__device__ __forceinline__ void fwd3(double fm, double f0, double fp, double u, double& k0,
                                     double& k1, double& k2) {
  k0 = (fm + f0) + fp;
  const double d = fp - fm;
  k1 = d - u * k0;
  k2 = ((fp + fm) - 2.0 * (u * d)) + (u * u) * k0;
}

// General rates: hr = {w3, w4, w5, w6, w7, w8, w9, w10} (device memory).
template <class L, class TV, class Sink>
__device__ __forceinline__ bool cumulant_collide_general(const TV& t, double omega, double bulk,
                                                         const double* hr, Sink&& sink) {
  static_assert(L::Q == 27, "cumulant collision is defined on D3Q27");
  const Moments<L> mo = moments<L>(t);
  const double rho = mo.rho, ux = mo.ux, uy = mo.uy, uz = mo.uz;
  // forward chimera: z lines, then y, then x -> K[a][b][c] = kappa_abc
  double K[3][3][3];
  sfor<0, 9>([&](auto ij) {
    constexpr int i = decltype(ij)::value / 3, j = decltype(ij)::value % 3;
    fwd3(t[dir_of<L>(i - 1, j - 1, -1)], t[dir_of<L>(i - 1, j - 1, 0)],
         t[dir_of<L>(i - 1, j - 1, 1)], uz, K[i][j][0], K[i][j][1], K[i][j][2]);
  });
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) fwd3(K[i][0][c], K[i][1][c], K[i][2][c], uy, K[i][0][c], K[i][1][c], K[i][2][c]);
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int c = 0; c < 3; ++c) fwd3(K[0][b][c], K[1][b][c], K[2][b][c], ux, K[0][b][c], K[1][b][c], K[2][b][c]);
  const double ir = 1.0 / rho;
#define SLBM_M(a, b, c) const double m##a##b##c = K[a][b][c] * ir;
  SLBM_M(2, 0, 0) SLBM_M(0, 2, 0) SLBM_M(0, 0, 2) SLBM_M(1, 1, 0) SLBM_M(1, 0, 1) SLBM_M(0, 1, 1)
  SLBM_M(2, 1, 0) SLBM_M(2, 0, 1) SLBM_M(1, 2, 0) SLBM_M(0, 2, 1) SLBM_M(1, 0, 2) SLBM_M(0, 1, 2)
  SLBM_M(1, 1, 1) SLBM_M(2, 2, 0) SLBM_M(2, 0, 2) SLBM_M(0, 2, 2) SLBM_M(2, 1, 1) SLBM_M(1, 2, 1)
  SLBM_M(1, 1, 2) SLBM_M(2, 2, 1) SLBM_M(2, 1, 2) SLBM_M(1, 2, 2) SLBM_M(2, 2, 2)
#undef SLBM_M
  // cumulants of order 4..6 (k220, ..., k222) from the central moments
  SLBM_CUMULANTS_FROM_CENTRAL
  const double w3 = hr[0], w4 = hr[1], w5 = hr[2], w6 = hr[3], w7 = hr[4], w8 = hr[5],
               w9 = hr[6], w10 = hr[7];
  const double o1 = 1.0 - omega;
  // second order (normalised: equilibrium c_s^2 = 1/3 per diagonal, trace 1)
  const double k110 = o1 * m110, k101 = o1 * m101, k011 = o1 * m011;
  const double d1 = o1 * (m200 - m020), d2 = o1 * (m200 - m002);
  const double tr = 1.0 + (1.0 - bulk) * (((m200 + m020) + m002) - 1.0);
  const double k200 = ((tr + d1) + d2) / 3.0;
  const double k020 = k200 - d1, k002 = k200 - d2;
  // third order: sums (w3) and differences (w4) of the pairs, C_111 (w5)
  const double o3 = 1.0 - w3, o4 = 1.0 - w4;
  auto pair3 = [&](double a, double b, double& ra, double& rb) {
    const double s = o3 * (a + b), d = o4 * (a - b);
    ra = 0.5 * (s + d);
    rb = 0.5 * (s - d);
  };
  double k120, k102, k210, k012, k201, k021;
  pair3(m120, m102, k120, k102);
  pair3(m210, m012, k210, k012);
  pair3(m201, m021, k201, k021);
  const double k111 = (1.0 - w5) * m111;
  // fourth order: two deviatoric combinations (w6), the isotropic one (w7)
  const double e1 = (1.0 - w6) * ((k220 - 2.0 * k202) + k022);
  const double e2 = (1.0 - w6) * ((k220 + k202) - 2.0 * k022);
  const double e3 = (1.0 - w7) * ((k220 + k202) + k022);
  const double r022 = (e3 - e2) / 3.0, r202 = (e3 - e1) / 3.0;
  const double r220 = (e3 - r202) - r022;
  const double o8 = 1.0 - w8, o9 = 1.0 - w9;
  const double r211 = o8 * k211, r121 = o8 * k121, r112 = o8 * k112;
  const double r221 = o9 * k221, r212 = o9 * k212, r122 = o9 * k122;
  const double r222 = (1.0 - w10) * k222;
  {
    // post-collision central moments p_abc (normalised) of order 4..6
    const double k220 = r220, k202 = r202, k022 = r022, k211 = r211, k121 = r121, k112 = r112;
    const double k221 = r221, k212 = r212, k122 = r122, k222 = r222;
    SLBM_CENTRAL_FROM_CUMULANTS
    // kappa* = rho p, orders 0/1: rho, 0; backward chimera x, y, z
    const ChimeraCoef cx = chimera_coef(ux), cy = chimera_coef(uy), cz = chimera_coef(uz);
    double G[3][3][3];
    back3_even(rho, rho * k200, cx, G[0][0][0], G[1][0][0], G[2][0][0]);
    back3(0.0, rho * k110, rho * k210, cx, G[0][1][0], G[1][1][0], G[2][1][0]);
    back3(rho * k020, rho * k120, rho * p220, cx, G[0][2][0], G[1][2][0], G[2][2][0]);
    back3(0.0, rho * k101, rho * k201, cx, G[0][0][1], G[1][0][1], G[2][0][1]);
    back3(rho * k011, rho * k111, rho * p211, cx, G[0][1][1], G[1][1][1], G[2][1][1]);
    back3(rho * k021, rho * p121, rho * p221, cx, G[0][2][1], G[1][2][1], G[2][2][1]);
    back3(rho * k002, rho * k102, rho * p202, cx, G[0][0][2], G[1][0][2], G[2][0][2]);
    back3(rho * k012, rho * p112, rho * p212, cx, G[0][1][2], G[1][1][2], G[2][1][2]);
    back3(rho * p022, rho * p122, rho * p222, cx, G[0][2][2], G[1][2][2], G[2][2][2]);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double a, b, d;
        back3(G[i][0][c], G[i][1][c], G[i][2][c], cy, a, b, d);
        G[i][0][c] = a;
        G[i][1][c] = b;
        G[i][2][c] = d;
      }
    }
    sfor<0, 9>([&](auto ij) {
      constexpr int i = decltype(ij)::value / 3, j = decltype(ij)::value % 3;
      double a, b, d;
      back3(G[i][j][0], G[i][j][1], G[i][j][2], cz, a, b, d);
      sink(std::integral_constant<int, dir_of<L>(i - 1, j - 1, -1)>{}, a);
      sink(std::integral_constant<int, dir_of<L>(i - 1, j - 1, 0)>{}, b);
      sink(std::integral_constant<int, dir_of<L>(i - 1, j - 1, 1)>{}, d);
    });
  }
  return mo.bad;
}

}  // namespace slbm
