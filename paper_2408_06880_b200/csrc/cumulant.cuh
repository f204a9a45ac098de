// Cumulant collision, D3Q27 (Geier, Schoenherr, Pasquali, Krafczyk 2015,
// "The cumulant lattice Boltzmann equation in three dimensions").  Not in
// the reference package: parity is UNPINNED; the CPU
// restatement oracle/cumulant_ref.py uses the identical operation order and
// tests check conservation, the equilibrium fixed point and the shear-wave
// viscosity.
//
// Relaxation rates: shear omega (second-order deviatoric cumulants); bulk
// and every higher order relax with rate 1 (the non-parametrised cumulant
// method, lbmpy's default rates).  With higher-order rates 1 the
// post-collision cumulants of order >= 3 vanish, so the post-collision
// central moments follow from rho, u and the six relaxed second-order
// central moments alone:
//   order 0/1: rho, 0          order 2: relaxed kappa_ab
//   order 3/5: 0               order 4: products of order-2 / rho
//   order 6  : kappa_222 from the cumulant->moment relation (C_222 = 0)
// and one backward chimera transform (x, then y, then z) gives f*.
#pragma once

#include "common.cuh"

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
__device__ __forceinline__ bool cumulant_collide(const TV& t, double omega, Sink&& sink) {
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

  // relaxation: deviatoric parts with omega, trace to its equilibrium rho
  const double om1 = 1.0 - omega;
  const double dxy = om1 * (kxx - kyy);
  const double dxz = om1 * (kxx - kzz);
  const double sxx = ((rho + dxy) + dxz) / 3.0;
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

}  // namespace slbm
