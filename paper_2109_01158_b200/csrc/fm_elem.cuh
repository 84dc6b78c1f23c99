// Element-level device functions and the shared-memory layout of the fused
// tile kernels (fm_eval_exact.cu: k_tile_exact; fm_eval_ws.cu: k_tile_ws).
#pragma once

#include "fm_ctx.cuh"
#include "fm_density.cuh"

namespace fm {

__host__ __device__ constexpr size_t r16(size_t x) { return (x + 15) / 16 * 16; }


template <int DIM, int CT>
struct PipeLayout {
  static constexpr int RB = RecBytes<DIM>::value;
  // stage: the chunk's records | their closure indices | its entry block
  // rec: bytes of the stage's record area — CT records, or only CT + 16 slot
  // bytes when every tile of the context is dictionary-coded (rec_area)
  __host__ __device__ static size_t rec_area(bool all_coded) {
    return all_coded ? r16((size_t)CT + 16) : r16((size_t)CT * RB);
  }
  __host__ __device__ static size_t loc_off(size_t rec = rec_area(false)) { return rec; }
  __host__ __device__ static size_t blk_off(size_t rec = rec_area(false)) {
    return loc_off(rec) + (size_t)(CT + 2) * 8;
  }
  __host__ __device__ static size_t stage(int blk_cap, size_t rec = rec_area(false)) {
    return blk_off(rec) + r16((size_t)blk_cap * 2);
  }
  __host__ __device__ static size_t nodev(int D, int clo_cap) { return r16((size_t)D * clo_cap * 8); }
  __host__ __device__ static size_t cids(int clo_cap) { return r16((size_t)clo_cap * 4); }
  // per-tile tables: node descriptors | exchange-item chunk starts
  // (+ the tile's record dictionary, DICT_MAX records)
  __host__ __device__ static size_t dict_off() { return (size_t)CT * 16 + XCH_STRIDE * 4; }
  __host__ __device__ static size_t tabs() { return dict_off() + (size_t)DICT_MAX * RB; }
  // contributions staging: [slot][component][row], except D = 2 (2D
  // Neo-Hookean): [slot][row][2] (one 16-B store / load per entry; cfg3 tile
  // kernel 0.1086 -> 0.1064 ms — the same with 4 padded doubles for D = 3
  // conflicts on the stores: 0.843 -> 0.975 ms at cfg4)
  static constexpr bool AOS(int D) { return D == 2; }
  // slot stride padded by SPD doubles (8 banks): the exchange items read the
  // slots of one row together, which would otherwise sit in the same bank
  // (cfg4 tile kernel 0.839 -> 0.830 ms)
  static constexpr int SPD = 4;
  __host__ __device__ static size_t slot_stride(int D) {
    return AOS(D) ? (size_t)(CT + SPD / 2) * D : (size_t)CT * D + SPD;
  }
  __host__ __device__ static size_t staging(int D) { return r16(slot_stride(D) * (DIM + 1) * 8); }
  // nb node-value buffers, tb table buffers (2: the next tile's tables load a
  // tile ahead)
  // (dn: node-value components per node, D; 2 D for the Hessian-vector
  // product, which gathers the direction's node values too)
  __host__ __device__ static size_t total(int D, int blk_cap, int clo_cap, int nb, int tb,
                                          int dn = 0, size_t rec = rec_area(false)) {
    return 2 * stage(blk_cap, rec) + nb * nodev(dn ? dn : D, clo_cap) + cids(clo_cap) +
           tb * tabs() + staging(D) + 32 * 8 + 8 * 8;
  }
};

// x^e for the fused kernels (x > 0): numpy's fast exponents, else
// exp2(e log2 x) — no extended-precision log as in pow(); |e log2 x| stays
// small for these fields, so the result is within a few ulps (1e-10 bars)
__device__ __forceinline__ double pow_fused(double x, double e) {
  if (e == 0.5) return sqrt(x);
  if (e == 1.5) return x * sqrt(x);
  if (e == 1.0) return x;
  if (e == 2.0) return x * x;
  if (e == -1.0) return 1.0 / x;
  if (e == 0.0) return 1.0;
  return exp2(e * log2(x));
}

// cofactors with one rounding per minor (fused; this kernel is not bound to
// the reference's operation order)
template <int DIM>
__device__ __forceinline__ void cof_F_fma(const double (&F)[DIM][DIM], double (&C)[DIM][DIM]) {
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
        const double minor = fma(F[j1][m1], F[j2][m2], -(F[j1][m2] * F[j2][m1]));
        C[j][m] = ((j + m) & 1) ? -minor : minor;
      }
    }
  }
}

// log(det) for the fused J: near 1 (|det - 1| < 1/8, the elastic states of the
// configs) by the atanh series 2 s (1 + z/3 + ... + z^7/15), s = (det-1)/(det+1),
// z = s^2 <= 0.0035 (truncation < 1e-18 relative; det - 1 is exact), Estrin
// evaluated, branch-free so that it interleaves with the contributions; states
// farther from 1 are corrected with libm's log after the contributions are
// staged (W += 2 C1 (series - log det)).  A few ulps, against J's 1e-10.
__device__ __forceinline__ double log_series(double det, double inv_dp1) {
  const double x = det - 1.0;
  const double s = x * inv_dp1;  // x / (det + 1)
  const double z = s * s, z2 = z * z, z4 = z2 * z2;
  const double a = fma(z, 1.0 / 3.0, 1.0), b = fma(z, 1.0 / 7.0, 1.0 / 5.0);
  const double c = fma(z, 1.0 / 11.0, 1.0 / 9.0), d = fma(z, 1.0 / 15.0, 1.0 / 13.0);
  const double p = fma(z4, fma(z2, d, c), fma(z2, b, a));
  return 2.0 * s * p;
}

// NH: P' = vol * dW/dF = a F + b cof with a = 2 C1 vol, b = vol (2 D1 (det-1) - 2 C1/det)
// (models.py:103-120 regrouped).  p-Laplace: P' = vol |g|^(p-2) g.
// Admissibility near det F = 0 follows the reference exactly: the FMA forms
// of F and det F differ from numpy's in the last bits, which only matters for
// the sign decision (J = +inf, models.py:94-99; the exact path's raise,
// models.py:107-110) when det F is tiny.  Below DET_NEAR the element's F is
// recomputed in einsum order (assembly.py:35-49) and det F as the six-term
// left-to-right expansion (models.py:59-71), bit for bit numpy's values, and
// that det decides and enters W and P'.  (A sign flip above DET_NEAR would need
// |F_ij| ~ 1e4, i.e. fma / numpy differences of 1e-3.)
constexpr double DET_NEAR = 1e-3;

// (vvf(out) refills the element's node values for the rare recompute: the
// callers either copy them from registers or re-read them from shared memory,
// so they need not stay live through the constitutive law)
template <int DIM, int MODEL, int D, class VVF>
__device__ __forceinline__ void element_P_f(const double (&F)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
                                          const VVF &vvf,
                                          const double (&g)[DIM][DIM + 1],
                                          double vol, const ModelArgs &m, bool want_w,
                                          double (&P)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
                                          double &W, bool &bad, bool &far, double &det_out,
                                          double &ls_out) {
  if constexpr (MODEL == FM_MODEL_NEOHOOKEAN) {
    double C[DIM][DIM];
    cof_F_fma<DIM>(F, C);
    double det = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) det = fma(F[0][k], C[0][k], det);
    if (!(det > DET_NEAR)) {  // rare: the reference's own det decides
      double vr[DIM][DIM + 1], Fr[DIM][DIM];
      vvf(vr);
      grad_F<DIM, DIM>(vr, g, Fr);
      det = det_F<DIM>(Fr);
    }
    bad = !(det > 0.0);
    // 1/det and (for J) 1/(det+1) from one division
    const double dp1 = det + 1.0;
    const double R = 1.0 / (det * dp1);
    const double rdet = dp1 * R;
    const double a = 2.0 * m.C1 * vol;
    const double bc = vol * (2.0 * m.D1 * (det - 1.0) - 2.0 * m.C1 * rdet);
#pragma unroll
    for (int j = 0; j < DIM; ++j)
#pragma unroll
      for (int k = 0; k < DIM; ++k) P[j][k] = fma(a, F[j][k], bc * C[j][k]);
    if (want_w) {
      double I1 = 0.0;
#pragma unroll
      for (int j = 0; j < DIM; ++j)
#pragma unroll
        for (int k = 0; k < DIM; ++k) I1 = fma(F[j][k], F[j][k], I1);
      const double dm1 = det - 1.0;
      const double ls = log_series(det, det * R);
      W = bad ? INFINITY : m.C1 * ((I1 - (double)DIM) - 2.0 * ls) + m.D1 * (dm1 * dm1);
      // far from 1: the caller adds 2 C1 (ls - log det) later
      far = !bad && !(fabs(dm1) < 0.125);
      det_out = det;
      ls_out = ls;
    }
  } else {
    bad = false;
    double n2 = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) n2 = fma(F[0][k], F[0][k], n2);
    double fac;
    if (m.p >= 2.0)
      fac = pow_fused(n2, m.e_dw);  // 0^e = 0 for e > 0 (exp2(-inf))
    else
      fac = n2 > 0.0 ? pow_fused(n2, m.e_dw) : 0.0;
    // W = |g|^p / p = |g|^(p-2) |g|^2 / p from the gradient's factor: no second
    // pow (a few ulps from pow(n2, p/2) / p; J is compared at 1e-10)
    if (want_w) W = fac * n2 / m.p;
    far = false;
    det_out = ls_out = 0.0;
    fac *= vol;
#pragma unroll
    for (int k = 0; k < DIM; ++k) P[0][k] = fac * F[0][k];
  }
}

template <int DIM, int MODEL, int D>
__device__ __forceinline__ void element_P(const double (&F)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
                                          const double (&vv)[D][DIM + 1],
                                          const double (&g)[DIM][DIM + 1],
                                          double vol, const ModelArgs &m, bool want_w,
                                          double (&P)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
                                          double &W, bool &bad, bool &far, double &det_out,
                                          double &ls_out) {
  element_P_f<DIM, MODEL, D>(
      F,
      [&](double (&o)[D][DIM + 1]) {
#pragma unroll
        for (int k = 0; k < D; ++k)
#pragma unroll
          for (int l = 0; l < DIM + 1; ++l) o[k][l] = vv[k][l];
      },
      g, vol, m, want_w, P, W, bad, far, det_out, ls_out);
}

// F = grad v as chained FMAs (one DMUL + NV-1 DFMA per entry; the edge-
// difference form sum_{l>=1} (v_l - v_0) dphi_l, one DADD fewer per entry and
// no dphi column 0, measured 2 % slower at cfg4)
template <int DIM, int D>
__device__ __forceinline__ void grad_F_fma(const double (&vv)[D][DIM + 1],
                                           const double (&g)[DIM][DIM + 1], double (&F)[D][DIM]) {
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      double s = vv[j][0] * g[m][0];
#pragma unroll
      for (int l = 1; l < DIM + 1; ++l) s = fma(vv[j][l], g[m][l], s);
      F[j][m] = s;
    }
}

// Position in this CTA's chunk stream: tile t, chunk offset c0.
template <int CT>
struct Cursor {
  int t, c0, ne;
  TileMeta tm;
  __device__ void load(const TileArgs &a) {
    if (t < a.n_tiles_all) {
      tm = a.meta[t];
      ne = tm.own_count;  // every element is computed once, by its owner tile
    } else {
      ne = 0;
    }
  }
  __device__ bool valid(const TileArgs &a) const { return t < a.n_tiles_all; }
  // next chunk of the stream; tiles without own elements have no chunks
  __device__ void advance(const TileArgs &a) {
    c0 += CT;
    while (c0 >= ne && t < a.n_tiles_all) {
      c0 = 0;
      t += gridDim.x;
      load(a);
    }
  }
};

}  // namespace fm
