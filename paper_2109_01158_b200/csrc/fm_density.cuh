// Batched densities of models.py, one element per thread, fp64 registers.
// The expressions keep the reference's operation order:
//   F            assembly.py:35-49  einsum 'rl,rl->r': (p0+p2)+(p1+p3) | (p0+p2)+p1
//   det          models.py:59-71    closed form, six terms left to right
//   cofactor     models.py:74-86
//   NH W         models.py:89-100   C1 (I1 - dim - 2 log det) + D1 (det-1)^2, +inf if det<=0
//   NH dW/dF     models.py:103-120  C1 (2F - (2/det) cof) + 2 D1 (det-1) cof
//   p-Laplace    models.py:123-138  |g|^p/p, |g|^(p-2) g (0 at g = 0 when p < 2)
// Every multiply / add here is an explicit round-to-nearest intrinsic, which
// the compiler never contracts into an FMA: the per-element values reproduce
// the reference bit-for-bit (up to libm ulps in log/pow) in any translation
// unit, while log/pow themselves keep their FMA-based implementations
// (SURVEY §7.2 H3).  The fused exact-gradient kernel uses its own FMA forms.
#pragma once

#include "fm_ctx.cuh"

namespace fm {

__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }

template <int NV>
__device__ __forceinline__ double einsum_row(const double (&a)[NV], const double (&b)[NV]) {
  if constexpr (NV == 4) {
    double p0 = rmul(a[0], b[0]), p1 = rmul(a[1], b[1]), p2 = rmul(a[2], b[2]),
           p3 = rmul(a[3], b[3]);
    return radd(radd(p0, p2), radd(p1, p3));
  } else {
    double p0 = rmul(a[0], b[0]), p1 = rmul(a[1], b[1]), p2 = rmul(a[2], b[2]);
    return radd(radd(p0, p2), p1);
  }
}

template <int DIM, int D>
__device__ __forceinline__ void grad_F(const double (&vv)[D][DIM + 1],
                                       const double (&g)[DIM][DIM + 1], double (&F)[D][DIM]) {
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int m = 0; m < DIM; ++m) F[j][m] = einsum_row<DIM + 1>(vv[j], g[m]);
}

template <int DIM>
__device__ __forceinline__ double det_F(const double (&F)[DIM][DIM]) {
  if constexpr (DIM == 2) {
    return rsub(rmul(F[0][0], F[1][1]), rmul(F[0][1], F[1][0]));
  } else {
    double a = rmul(rmul(F[0][0], F[1][1]), F[2][2]);
    double b = rmul(rmul(F[0][2], F[1][0]), F[2][1]);
    double c = rmul(rmul(F[0][1], F[1][2]), F[2][0]);
    double d = rmul(rmul(F[0][2], F[1][1]), F[2][0]);
    double e = rmul(rmul(F[0][1], F[1][0]), F[2][2]);
    double f = rmul(rmul(F[0][0], F[1][2]), F[2][1]);
    return rsub(rsub(rsub(radd(radd(a, b), c), d), e), f);
  }
}

template <int DIM>
__device__ __forceinline__ void cof_F(const double (&F)[DIM][DIM], double (&C)[DIM][DIM]) {
  if constexpr (DIM == 2) {
    C[0][0] = F[1][1];
    C[0][1] = -F[1][0];
    C[1][0] = -F[0][1];
    C[1][1] = F[0][0];
  } else {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int j1 = j == 0 ? 1 : 0, j2 = j == 2 ? 1 : 2;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int m1 = m == 0 ? 1 : 0, m2 = m == 2 ? 1 : 2;
        double minor = rsub(rmul(F[j1][m1], F[j2][m2]), rmul(F[j1][m2], F[j2][m1]));
        C[j][m] = ((j + m) & 1) ? -minor : minor;
      }
    }
  }
}

// W for the model; returns +inf for inadmissible Neo-Hookean states.
template <int DIM, int MODEL>
__device__ __forceinline__ double density(const double (&F)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
                                          const ModelArgs &m) {
  if constexpr (MODEL == FM_MODEL_NEOHOOKEAN) {
    double det = det_F<DIM>(F);
    double I1 = rmul(F[0][0], F[0][0]);
#pragma unroll
    for (int j = 0; j < DIM; ++j)
#pragma unroll
      for (int k = 0; k < DIM; ++k)
        if (j + k > 0) I1 = radd(I1, rmul(F[j][k], F[j][k]));
    if (!(det > 0.0)) return INFINITY;
    double ld = log(det);
    double dm1 = rsub(det, 1.0);
    return radd(rmul(m.C1, rsub(rsub(I1, (double)DIM), rmul(2.0, ld))),
                rmul(m.D1, rmul(dm1, dm1)));
  } else {
    double n2 = rmul(F[0][0], F[0][0]);
#pragma unroll
    for (int k = 1; k < DIM; ++k) n2 = radd(n2, rmul(F[0][k], F[0][k]));
    return np_scalar_pow(n2, m.e_w) / m.p;
  }
}

// dW/dF; sets bad when det <= 0 (Neo-Hookean).
template <int DIM, int MODEL>
__device__ __forceinline__ void ddensity(const double (&F)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
                                         const ModelArgs &m,
                                         double (&P)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
                                         bool &bad) {
  if constexpr (MODEL == FM_MODEL_NEOHOOKEAN) {
    double det = det_F<DIM>(F);
    bad = !(det > 0.0);
    double C[DIM][DIM];
    cof_F<DIM>(F, C);
    double dfac = rmul(rmul(2.0, m.D1), rsub(det, 1.0));
    double inv2 = 2.0 / det;
#pragma unroll
    for (int j = 0; j < DIM; ++j)
#pragma unroll
      for (int k = 0; k < DIM; ++k)
        P[j][k] = radd(rmul(m.C1, rsub(rmul(2.0, F[j][k]), rmul(inv2, C[j][k]))),
                       rmul(dfac, C[j][k]));
  } else {
    bad = false;
    double n2 = rmul(F[0][0], F[0][0]);
#pragma unroll
    for (int k = 1; k < DIM; ++k) n2 = radd(n2, rmul(F[0][k], F[0][k]));
    double fac;
    if (m.p >= 2.0)
      fac = np_scalar_pow(n2, m.e_dw);
    else
      fac = n2 > 0.0 ? pow(n2, m.e_dw) : 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) P[0][k] = rmul(fac, F[0][k]);
  }
}

// ---- FD states (gradients.py:84-121) from the unperturbed invariants ------
// states with det below this (absolute; det ~ 1 for the elastic configs) are
// recomputed in the reference's operation order by the caller
constexpr double FD_DET_NEAR = 1e-3;

// log1p(x) for |x| < 1e-3 (degree 7, relative truncation < 1.5e-19)
__device__ __forceinline__ double log1p_small(double x) {
  double p = fma(x, 1.0 / 7.0, -1.0 / 6.0);
  p = fma(p, x, 1.0 / 5.0);
  p = fma(p, x, -0.25);
  p = fma(p, x, 1.0 / 3.0);
  p = fma(p, x, -0.5);
  p = fma(p, x, 1.0);
  return p * x;
}

// |F|^2 in the reference's order (models.py:89-100: sequential sum of squares)
template <int DIM, int D>
__device__ __forceinline__ double sumsq_rn(const double (&F)[D][DIM]) {
  double s = rmul(F[0][0], F[0][0]);
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int k = 0; k < DIM; ++k)
      if (j + k > 0) s = radd(s, rmul(F[j][k], F[j][k]));
  return s;
}

// W of one perturbed state: row j of F moved by dl * dphi[:, l] (dl = the
// step the rounded perturbed value carries), so det = det0 + dl c,
// |F|^2 = I1_0 + dl (a + dl b), log det = log det0 + log1p(dl c / det0)
// (NH; p-Laplace: |g|^2 = n2_0 + dl (a + dl b)), W the reference's expression
// of those invariants (models.py:89-100, 123-126).  exact = true (W not
// computed): det near 0, the caller recomputes the state the reference's way.
template <int DIM, int MODEL>
__device__ __forceinline__ double fd_state_w(double dl, double cj, double aj, double bb,
                                             double base0, double rdet0, double ld0, double i10,
                                             const ModelArgs &m, bool &exact) {
  if constexpr (MODEL == FM_MODEL_NEOHOOKEAN) {
    const double det = fma(dl, cj, base0);
    if (!(det > FD_DET_NEAR)) {
      exact = true;
      return 0.0;
    }
    const double I1 = fma(dl, fma(dl, bb, aj), i10);
    const double x = (dl * cj) * rdet0;
    const double ld = fabs(x) < 1e-3 ? ld0 + log1p_small(x) : log(det);
    const double dm1 = det - 1.0;
    return m.C1 * ((I1 - (double)DIM) - 2.0 * ld) + m.D1 * (dm1 * dm1);
  } else {
    const double n2 = fmax(fma(dl, fma(dl, bb, aj), base0), 0.0);
    return np_scalar_pow(n2, m.e_w) / m.p;
  }
}

}  // namespace fm
