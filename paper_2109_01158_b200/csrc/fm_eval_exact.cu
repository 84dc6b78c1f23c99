// Fused energy + exact gradient (gradients.py:124-149 with assembly.py:94-106)
// as one persistent, pipelined kernel; two 256-thread CTAs per SM.
//
// Each CTA walks its node tiles (t = blockIdx.x, += gridDim.x; tiles are in
// Morton order of their spatial boxes).  Every element is computed ONCE, by
// its owner tile (the tile of its first free node).  Per tile (<= CT free
// nodes, one node per thread):
//   tables        descriptors, entries and the exchange-item chunk starts by
//                 bulk copy (TB = 2: a tile ahead).
//   node values   the tile's node closure (sorted distinct nodes of its
//                 elements) gathered ONCE into shared memory (8-byte LDGSTS;
//                 NB = 2: a tile ahead); elements address it with 16-bit
//                 closure indices, so no per-element global gathers of v.
//   records       the own elements, chunks of CT, double-buffered and issued
//                 two chunks ahead: one 1D bulk copy (TMA engine, mbarrier
//                 complete_tx) for the records (80 B 3D / 48 B 2D: an odd
//                 number of 16-B chunks, so row-per-lane reads are bank-
//                 conflict free) and one for their closure indices.
//   compute       thread c: F = grad v, P' = vol * dW/dF = a F + b cof, the
//                 contributions P' . grad phi_l of its 4 (3) nodes, vol * W;
//                 contributions staged [slot][comp][row].
//   assemble      node threads add this chunk's entries of their own tile's
//                 elements (sorted by tile element; fixed order, no atomics);
//                 entries whose node belongs to another tile ("cross") are
//                 stored to the exchange buffer (coalesced: slots in owner-tile
//                 item order) and added by k_finish_cross.
// J: per-thread partials over a static tile assignment -> fixed block tree ->
// one partial per CTA (vol * W, and b.v of the tile nodes from the closure
// values), reduced in CTA order by the last block of k_finish_cross.
#include "fm_density.cuh"
#include "fm_elem.cuh"
#include "fm_kernels.h"
#include "fm_pipe.cuh"


// Phase timeline for profiling builds only (tools/trace_exact.py compiles this
// unit with -DFM_TRACE=1 into a separate library): clock64 stamps of warp
// leaders of CTAs 0..3 per chunk.
#ifndef FM_TRACE
#define FM_TRACE 0
#endif
#if FM_TRACE
constexpr int TR_CTAS = 4, TR_WARPS = 8, TR_CHUNKS = 160, TR_STAMPS = 8;
__device__ long long g_trace[TR_CTAS * TR_WARPS * TR_CHUNKS * TR_STAMPS];
#define TRACE(k)                                                                        \
  do {                                                                                  \
    if (blockIdx.x < TR_CTAS && (threadIdx.x & 31) == 0 && q < TR_CHUNKS)               \
      g_trace[((blockIdx.x * TR_WARPS + (threadIdx.x >> 5)) * TR_CHUNKS + q) * TR_STAMPS + \
              (k)] = clock64();                                                         \
  } while (0)
extern "C" int fm_trace_copy(long long *out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_trace, (size_t)n * sizeof(long long));
}
#else
#define TRACE(k) \
  do {           \
  } while (0)
#endif

namespace fm {

// Hessian-vector product per element: dP' = vol * d2W/dF2 : dF, the
// derivative of element_P's P' along dF = grad p (models.py:103-138
// differentiated once more).  NH: P' = a F + b C (a = 2 C1 vol, b = vol (2 D1
// (det-1) - 2 C1/det), C = cof F) -> dP' = a dF + db C + b dC with
// ddet = C : dF, db = vol (2 D1 + 2 C1/det^2) ddet, dC the cofactors'
// derivative (bilinear minors).  p-Laplace: P' = vol f g, f = |g|^(p-2) ->
// dP' = vol f (dg + (p-2) (g.dg)/|g|^2 g); at g = 0: vol f dg (f = [p == 2]).
template <int DIM, int MODEL>
__device__ __forceinline__ void element_dP(
    const double (&F)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
    const double (&dF)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM], double vol,
    const ModelArgs &m, double (&dP)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM], bool &bad) {
  if constexpr (MODEL == FM_MODEL_NEOHOOKEAN) {
    double C[DIM][DIM], dC[DIM][DIM];
    cof_F_fma<DIM>(F, C);
    if constexpr (DIM == 2) {
      cof_F_fma<DIM>(dF, dC);
    } else {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int j1 = j == 0 ? 1 : 0, j2 = j == 2 ? 1 : 2;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int k1 = k == 0 ? 1 : 0, k2 = k == 2 ? 1 : 2;
          const double t = fma(dF[j1][k1], F[j2][k2], F[j1][k1] * dF[j2][k2]) -
                           fma(dF[j1][k2], F[j2][k1], F[j1][k2] * dF[j2][k1]);
          dC[j][k] = ((j + k) & 1) ? -t : t;
        }
      }
    }
    double det = 0.0, ddet = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) det = fma(F[0][k], C[0][k], det);
#pragma unroll
    for (int j = 0; j < DIM; ++j)
#pragma unroll
      for (int k = 0; k < DIM; ++k) ddet = fma(C[j][k], dF[j][k], ddet);
    bad = !(det > 0.0);
    const double rdet = 1.0 / det;
    const double a = 2.0 * m.C1 * vol;
    const double bc = vol * (2.0 * m.D1 * (det - 1.0) - 2.0 * m.C1 * rdet);
    const double dbc = vol * (2.0 * m.D1 + 2.0 * m.C1 * rdet * rdet) * ddet;
#pragma unroll
    for (int j = 0; j < DIM; ++j)
#pragma unroll
      for (int k = 0; k < DIM; ++k) dP[j][k] = fma(a, dF[j][k], fma(dbc, C[j][k], bc * dC[j][k]));
  } else {
    bad = false;
    double n2 = 0.0, gd = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      n2 = fma(F[0][k], F[0][k], n2);
      gd = fma(F[0][k], dF[0][k], gd);
    }
    double fac;
    if (m.p >= 2.0)
      fac = pow_fused(n2, m.e_dw);
    else
      fac = n2 > 0.0 ? pow_fused(n2, m.e_dw) : 0.0;
    const double c2 = n2 > 0.0 ? (m.p - 2.0) * gd / n2 : 0.0;
    fac *= vol;
#pragma unroll
    for (int k = 0; k < DIM; ++k) dP[0][k] = fac * fma(c2, F[0][k], dF[0][k]);
  }
}

// Unperturbed invariants of an element for the FD states: F in einsum order
// (the reference's unperturbed F), det, 1/det, log det and |F|^2 in the
// reference's order (p-Laplace: |g|^2 in base0), and the rank-one
// coefficients a_jl = 2 F_j . dphi_l, c_jl = cof(F)_j . dphi_l and
// b_l = |dphi_l|^2 of every node l and component j.
template <int DIM, int MODEL, int D>
struct FdElem {
  static constexpr int NV = DIM + 1;
  static constexpr bool NH = MODEL == FM_MODEL_NEOHOOKEAN;
  double A[D][NV], Cc[NH ? D : 1][NV], BB[NV];
  double base0, rdet0 = 0.0, ld0 = 0.0, i10 = 0.0;
  __device__ __forceinline__ FdElem(const double (&vv)[D][NV], const Elem<DIM> &E) {
    double F[D][DIM];
    grad_F<DIM, D>(vv, E.g, F);
    double C[NH ? DIM : 1][DIM];
    if constexpr (NH) {
      base0 = det_F<DIM>(F);
      rdet0 = 1.0 / base0;
      // log det0 by the fused J's atanh series near 1 (<= 2 ulps; cfg4 FD
      // 2.096 -> 2.072 ms): it enters both W+- of every state of the element
      // and cancels in their difference
      if (fabs(base0 - 1.0) < 0.125)
        ld0 = log_series(base0, 1.0 / (base0 + 1.0));
      else
        ld0 = base0 > 0.0 ? log(base0) : NAN;
      i10 = sumsq_rn<DIM, D>(F);
      cof_F<DIM>(F, C);
    } else {
      base0 = sumsq_rn<DIM, D>(F);
    }
#pragma unroll
    for (int l = 0; l < NV; ++l) {
      double bb = E.g[0][l] * E.g[0][l];
#pragma unroll
      for (int q = 1; q < DIM; ++q) bb = fma(E.g[q][l], E.g[q][l], bb);
      BB[l] = bb;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double s2 = F[j][0] * E.g[0][l];
#pragma unroll
        for (int q = 1; q < DIM; ++q) s2 = fma(F[j][q], E.g[q][l], s2);
        A[j][l] = 2.0 * s2;
        if constexpr (NH) {
          double cj = C[j][0] * E.g[0][l];
#pragma unroll
          for (int q = 1; q < DIM; ++q) cj = fma(C[j][q], E.g[q][l], cj);
          Cc[j][l] = cj;
        }
      }
    }
  }
};

// Where the FD states of a tile-kernel element report to: the staging row,
// and the tile data that turns a non-finite state into the reference's
// offending-row key (gradients.py:77-81: sign, component, free rank of the
// node, element).
struct FdSink {
  double *st;       // staging of (slot 0, this row); slot l at st + l * sstride
  int sstride, cs;  // slot stride, component stride (doubles)
  const int32_t *closure, *rank_of, *s2o;
  int clo_begin;
  int64_t storage;  // the element's storage index
};

// The FD states of one element that the fast path left (det near 0, or
// |dl c / det0| >= 1e-4): both signs of every flagged (l, j) recomputed with
// the full rule of fd_state_w (the reference's own evaluation near det 0),
// the difference restaged; non-finite states latch their key.  Out of line
// and rare (flags: bit 2 (l D + j) + sg).
template <int DIM, int MODEL>
__device__ __noinline__ void fd_slow_states(unsigned flags, const unsigned char *stage, int row,
                                            const double *nv, int CAP, int4 cl,
                                            const ModelArgs &m, FdSink k,
                                            unsigned long long *key) {
  constexpr int NV = DIM + 1;
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  Elem<DIM> E;
  load_elem_smem<DIM>(stage, row, E);
  const int c[4] = {cl.x, cl.y, cl.z, cl.w};
  double vv[D][NV];
#pragma unroll
  for (int ll = 0; ll < NV; ++ll)
#pragma unroll
    for (int q = 0; q < D; ++q) vv[q][ll] = nv[q * CAP + c[ll]];
  const FdElem<DIM, MODEL, D> fe(vv, E);
#pragma unroll
  for (int l = 0; l < NV; ++l)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (!((flags >> (2 * (l * D + j))) & 3u)) continue;
      const double vl = vv[j][l];
      double w[2];
#pragma unroll
      for (int sg = 0; sg < 2; ++sg) {
        const double ve = radd(vl, sg ? m.eps : -m.eps);
        const double dl = ve - vl;
        bool exact = false;
        double cj = 0.0;
        if constexpr (FdElem<DIM, MODEL, D>::NH) cj = fe.Cc[j][l];
        double W = fd_state_w<DIM, MODEL>(dl, cj, fe.A[j][l], fe.BB[l], fe.base0, fe.rdet0,
                                          fe.ld0, fe.i10, m, exact);
        if (exact) {  // the reference's own evaluation: row j of F from ve
          double v2[D][NV];
#pragma unroll
          for (int ll = 0; ll < NV; ++ll)
#pragma unroll
            for (int q = 0; q < D; ++q) v2[q][ll] = vv[q][ll];
          v2[j][l] = ve;
          double F[D][DIM];
          grad_F<DIM, D>(v2, E.g, F);
          W = density<DIM, MODEL>(F, m);
        }
        if (!isfinite(W)) {
          const int node = __ldg(k.closure + k.clo_begin + c[l]);
          const int rk = __ldg(k.rank_of + node);
          if (rk >= 0) {  // a fixed node: the reference never perturbs it
            const unsigned long long kk = ((unsigned long long)sg << 63) |
                                          ((unsigned long long)j << 61) |
                                          ((unsigned long long)rk << 31) |
                                          (unsigned long long)__ldg(k.s2o + k.storage);
            *key = kk < *key ? kk : *key;
          }
        }
        w[sg] = rmul(E.vol, W);
      }
      k.st[l * k.sstride + j * k.cs] = w[1] - w[0];
    }
}

// FD contributions of one element (gradients.py:84-121 for the element's
// patch rows): per node l and component j the two perturbed states by
// rank-one updates of the unperturbed invariants (FdElem) and
// st[l][j] = vol W+ - vol W-.  The fast path (every state of the configs:
// det far from 0, |dl c / det0| < 1e-4) is branch-free; other states are
// flagged and redone by fd_slow_states with the full rule of fd_state_w.
template <int DIM, int MODEL, int D>
__device__ __forceinline__ void fd_element(const double (&vv)[D][DIM + 1], const Elem<DIM> &E,
                                           const ModelArgs &m, const FdSink &k,
                                           const unsigned char *stage, int row, const double *nv,
                                           int CAP, int4 cl, unsigned long long *key) {
  constexpr int NV = DIM + 1;
  constexpr bool NH = MODEL == FM_MODEL_NEOHOOKEAN;
  const FdElem<DIM, MODEL, D> fe(vv, E);
  const double eps = m.eps, vol = E.vol;
  const int c[4] = {cl.x, cl.y, cl.z, cl.w};
  unsigned flags = 0;
#pragma unroll
  for (int l = 0; l < NV; ++l)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double vl = nv[j * CAP + c[l]];  // re-read: vv and the gradients die after fe
      double cr = 0.0;                        // c_jl / det0
      if constexpr (NH) cr = fe.Cc[j][l] * fe.rdet0;
      double w[2];
#pragma unroll
      for (int sg = 0; sg < 2; ++sg) {
        const double ve = radd(vl, sg ? eps : -eps);  // the perturbed nodal value
        const double dl = ve - vl;                     // the step it carries
        double W;
        if constexpr (NH) {
          const double det = fma(dl, fe.Cc[j][l], fe.base0);
          const double I1 = fma(dl, fma(dl, fe.BB[l], fe.A[j][l]), fe.i10);
          const double x = dl * cr;
          // |x| < 1e-4 (dl ~ eps |v|: every state of the configs): log1p to x^4
          // (truncation x^4 / 5 < 2e-17 relative); otherwise the slow path
          if (!(det > FD_DET_NEAR) || !(fabs(x) < 1e-4)) flags |= 1u << (2 * (l * D + j) + sg);
          const double ld = fe.ld0 + x * fma(x, fma(x, fma(x, -0.25, 1.0 / 3.0), -0.5), 1.0);
          const double dm1 = det - 1.0;
          W = m.C1 * ((I1 - (double)DIM) - 2.0 * ld) + m.D1 * (dm1 * dm1);
        } else {
          const double n2 = fmax(fma(dl, fma(dl, fe.BB[l], fe.A[j][l]), fe.base0), 0.0);
          W = np_scalar_pow(n2, m.e_w) / m.p;
          if (!isfinite(W)) flags |= 1u << (2 * (l * D + j) + sg);  // non-finite input
        }
        w[sg] = rmul(vol, W);
      }
      k.st[l * k.sstride + j * k.cs] = w[1] - w[0];
    }
  if (flags) fd_slow_states<DIM, MODEL>(flags, stage, row, nv, CAP, cl, m, k, key);
}

// HV: Hessian-vector product instead of the gradient; b then holds the
// direction field p (full, zero on the Dirichlet dofs), there is no load term.
// EO: the energy alone (assembly.py:94-106) with WJ: each element's density in
// the reference's operation order (einsum F, the RN density of fm_density.cuh,
// bit for bit k_energy's values), optionally written to g as the per-element
// densities (reference element order); no staging, node sums or exchange, one
// barrier per chunk.
// FDM: the nodal-patch FD gradient (gradients.py:84-121) instead: every
// element, computed once by its owner tile, stages for each of its nodes l and
// components j the difference vol W(v + eps e_lj) - vol W(v - eps e_lj) of its
// two perturbed states (fd_element); the node sums, the cross-tile exchange
// and the finishing pass are the gradient's, and g = sum / (2 eps) - b.
template <int DIM, int MODEL, bool WJ, bool HV, bool FDM, bool EO, int CT, int NB, int TB,
          int MINB>
__global__ void __launch_bounds__(CT, MINB)
    k_tile_exact(TileArgs a, const double *__restrict__ v, const double *__restrict__ b,
                 double *__restrict__ g, double *__restrict__ jpart, double *__restrict__ bvpart,
                 unsigned long long *status, ModelArgs mdl) {
  constexpr int NV = DIM + 1;
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  constexpr int DG = HV ? 2 * D : D;  // node-value components gathered per node
  constexpr int RB = RecBytes<DIM>::value;
  constexpr int NCH = RB / 16;
  using L = PipeLayout<DIM, CT>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int CAP = a.clo_cap;
  const size_t REC = L::rec_area(a.all_coded != 0);  // record area of a stage
  const size_t SG = L::stage(a.blk_cap, REC);
  // stage s at smem + s * SG; node-value buffer k at nodev0 + k * nodev()
  auto stg = [&](int s) { return smem + s * SG; };
  auto nodev = [&](int k) {
    return reinterpret_cast<double *>(smem + 2 * SG + k * L::nodev(DG, CAP));
  };
  int32_t *cids = reinterpret_cast<int32_t *>(smem + 2 * SG + NB * L::nodev(DG, CAP));
  unsigned char *tabs0 = reinterpret_cast<unsigned char *>(cids) + L::cids(CAP);
  auto desc_of = [&](int k) { return reinterpret_cast<int4 *>(tabs0 + k * L::tabs()); };
  auto xch_of = [&](int k) {  // the tile's exchange-item chunk starts
    return reinterpret_cast<int *>(tabs0 + k * L::tabs() + (size_t)CT * 16);
  };
  auto dict_of = [&](int k) {  // the tile's record dictionary (dictionary-coded tiles)
    return reinterpret_cast<unsigned char *>(tabs0 + k * L::tabs() + L::dict_off());
  };
  double *stage_d = reinterpret_cast<double *>(tabs0 + TB * L::tabs());
  double *red = reinterpret_cast<double *>(reinterpret_cast<unsigned char *>(stage_d) +
                                           L::staging(D));
  // address of (slot, row) in the staging and the stride between components
  auto st_at = [&](int slot, int row) -> double * {
    return L::AOS(D) ? stage_d + slot * (int)L::slot_stride(D) + row * D
                     : stage_d + row + slot * (int)L::slot_stride(D);
  };
  constexpr int CS = L::AOS(D) ? 1 : CT;
  uint64_t *full = reinterpret_cast<uint64_t *>(red + 32);  // record stages
  uint64_t *nfull = full + 2;                               // node-value buffers
  uint64_t *cfull = nfull + 2;                              // closure ids
  uint64_t *tfull = cfull + 1;                              // tables (x TB)
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(full, 1);
    mbar_init(full + 1, 1);
    mbar_init(nfull, CT);
    mbar_init(nfull + 1, CT);
    mbar_init(cfull, 1);
    mbar_init(tfull, 1);
    mbar_init(tfull + 1, 1);
    fence_barrier_init();
  }
  __syncthreads();

  auto issue_clo = [&](int t) {  // closure ids of tile t -> cids
    if (tid == 0 && t < a.n_tiles_all) {
      const TileMeta tm = a.meta[t];
      const uint32_t bytes = (uint32_t)r16((size_t)tm.clo_count * 4);
      mbar_arrive_expect_tx(cfull, bytes);
      bulk_g2s(cids, a.closure + tm.clo_begin, bytes, cfull);
    }
  };
  // descriptors and exchange chunk starts of tile t -> table buffer k
  auto issue_tables = [&](int t, int k) {
    if (tid != 0 || t >= a.n_tiles_all) return;
    const TileMeta tm = a.meta[t];
    const uint32_t nb = (uint32_t)tm.node_count * 16;
    const uint32_t xb_ = t < a.n_tiles ? XCH_STRIDE * 4 : 0;
    const uint32_t db = (uint32_t)tm.dict_n * RB;
    mbar_arrive_expect_tx(tfull + k, nb + xb_ + db);
    if (nb) bulk_g2s(desc_of(k), a.node_desc + tm.node_begin, nb, tfull + k);
    if (xb_) bulk_g2s(xch_of(k), a.xchunk + (int64_t)t * XCH_STRIDE, xb_, tfull + k);
    if (db) bulk_g2s(dict_of(k), a.dict_rec + (int64_t)t * DICT_MAX * RB, db, tfull + k);
  };
  auto gather_nodev = [&](int clo_count, int k) {  // v of the closure -> nodev(k)
    double *dst = nodev(k);
    for (int i = tid; i < clo_count && !(FM_DBG(mdl) & 32); i += CT) {  // 32: probe without gathers
      const int64_t off = (int64_t)cids[i] * D;
#pragma unroll
      for (int kk = 0; kk < DG; ++kk)  // HV: components D.. are the direction's
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                         smem_u32(dst + kk * CAP + i)),
                     "l"(kk < D ? v + off + kk : b + off + (kk - D))
                     : "memory");
    }
    cp_async_arrive_noinc(nfull + k);
  };
  // own rows: records, their closure indices and the chunk's entry block, one
  // bulk copy each (the 8-byte index range is widened to 16-byte alignment:
  // row r sits at position r + (r0 & 1) of the stage's index array)
  auto issue_records = [&](const Cursor<CT> &x, int s) {
    if (!x.valid(a) || tid != 0) return;
    const int cnt = min(CT, x.ne - x.c0);
    const int64_t r0 = (int64_t)x.tm.own_begin + x.c0;
    const int64_t l0 = r0 & ~1ll;
    const uint32_t nl = (uint32_t)((cnt + (r0 - l0) + 1) & ~1);
    const uint32_t bb = (uint32_t)x.tm.blk_stride * 2;
    // records, or (dictionary-coded tile) their one-byte dictionary slots: the
    // byte range widened to 16-B alignment, row r at position r + (r0 & 15)
    const int64_t i0 = r0 & ~15ll;
    const uint32_t rbytes = x.tm.dict_n ? (uint32_t)((cnt + (r0 - i0) + 15) & ~15)
                                        : (uint32_t)cnt * RB;
    mbar_arrive_expect_tx(full + s, rbytes + nl * 8 + bb);
    if (cnt) {
      if (x.tm.dict_n)
        bulk_g2s(stg(s), a.eidx + i0, rbytes, full + s);
      else
        bulk_g2s(stg(s), a.aos + r0 * RB, rbytes, full + s);
      bulk_g2s(stg(s) + L::loc_off(REC), a.loc + l0, nl * 8, full + s);
    }
    if (bb)
      bulk_g2s(stg(s) + L::blk_off(REC),
               a.chunk_blocks + x.tm.blk_base + (int64_t)(x.c0 / CT) * x.tm.blk_stride, bb,
               full + s);
  };

  double jsum = 0.0, bvsum = 0.0;  // vol*W of own elements; b.v of the tile nodes' dofs
  bool bad_any = false;
  unsigned long long fdkey = ~0ull;  // FDM: smallest offending (sign, j, rank, element) key
  Cursor<CT> comp{(int)blockIdx.x, 0, 0, TileMeta{}};
  comp.load(a);
  if (comp.valid(a)) {
    // ---- prologue: tables (TB = 2), closure ids (+ node values with NB = 2),
    // chunk 0 and 1 records
    if (TB == 2) issue_tables(comp.t, 0);
    issue_clo(comp.t);
    if (NB == 2) {
      mbar_wait(cfull, 0);
      gather_nodev(comp.tm.clo_count, 0);
      fence_proxy_async();  // cids reads before the bulk refill
      __syncthreads();
      issue_clo(comp.t + gridDim.x);
    }
    // chunks 0 and 1 go out now; chunk q + 2 is issued into stage q & 1 as soon
    // as chunk q's records have been read (two chunks of lead, not one)
    Cursor<CT> iss = comp;
    iss.c0 = -CT;
    iss.advance(a);
    issue_records(iss, 0);
    iss.advance(a);
    issue_records(iss, 1);
    iss.advance(a);
    uint32_t q = 0, j = 0;

    while (comp.valid(a)) {
      const TileMeta tm = comp.tm;
      // every thread is done with the previous tile (its b.v reads of the node
      // values, its descriptor) before any buffer of it is refilled: the
      // node-value gather below overwrites the buffer that tile j - 1 (NB = 1)
      // or j - 2 ... read at its end, and a tile without chunks has no barrier
      if (j > 0) __syncthreads();
      TRACE(6);
      // ---- tile start: with TB = 1 the tables load now (previous tile done)
      const int tb = TB == 2 ? (int)(j & 1) : 0;
      if (TB == 1) issue_tables(comp.t, 0);
      const double *nv;
      if (NB == 2) {
        // node values of the NEXT tile (one tile of lead), then its successor's ids
        const int tn = comp.t + gridDim.x;
        if (tn < a.n_tiles_all) {
          mbar_wait(cfull, (j + 1) & 1);
          gather_nodev(a.meta[tn].clo_count, (j + 1) & 1);
          fence_proxy_async();
          __syncthreads();  // cids consumed
          issue_clo(tn + gridDim.x);
        }
        mbar_wait(nfull + (j & 1), (j >> 1) & 1);
        nv = nodev(j & 1);
      } else {
        // single buffer: gather this tile's node values now (previous tile done)
        mbar_wait(cfull, j & 1);
        gather_nodev(tm.clo_count, 0);
        mbar_wait(nfull, j & 1);
        fence_proxy_async();
        __syncthreads();  // cids consumed, every thread's copies visible
        issue_clo(comp.t + gridDim.x);
        nv = nodev(0);
      }
      mbar_wait(tfull + tb, TB == 2 ? (j >> 1) & 1 : j & 1);
      TRACE(7);
      const int4 *desc = desc_of(tb);
      const int *xch = xch_of(tb);
      const bool has_nodes = tm.node_count > 0;
      const bool my_node = tid < tm.node_count;
      int outw = 0, fmask = 0;
      bool cross = false;
      int4 nd = make_int4(0, 0, 0, 0);  // node descriptor (entry offset, per-chunk counts)
      double bj[D], acc[D];
#pragma unroll
      for (int k = 0; k < D; ++k) acc[k] = bj[k] = 0.0;
      int cl = 0;  // the node's index in this tile's closure (its v is in nv)
      if (my_node) {
        cl = __ldg(a.node_clo + tm.node_begin + tid);
        nd = desc[tid];
        outw = nd.w;
        fmask = desc_mask(nd);
        cross = ((unsigned)nd.x & CROSS_FLAG) != 0;
        if (b && !HV && !FDM) {  // FD: loaded at the tile end (not live through the tile)
#pragma unroll
          for (int k = 0; k < D; ++k) bj[k] = __ldg(b + (int64_t)nd.z * D + k);
        }
      }
      if (TB == 2) issue_tables(comp.t + gridDim.x, tb ^ 1);  // buffer of tile j - 1: done
      const int ne_t = comp.ne;
      for (int c0 = 0; c0 < ne_t; c0 += CT, ++q) {
        const int s = q & 1;
        // cross items of this chunk: contributions of own elements to nodes of
        // other tiles, written to xbuf for the finishing pass
        // (none in J-only orphan tiles); the first item of each thread is loaded
        // now, used after the first barrier
        int xb = 0, xe = 0;
        if (comp.t < a.n_tiles) {
          xb = xch[c0 / CT];
          xe = xch[c0 / CT + 1];
        }
        int xkey0 = 0;
        if (!EO && xb + tid < xe) xkey0 = __ldg(a.xkey + xb + tid);
        TRACE(0);
        mbar_wait(full + s, (q >> 1) & 1);
        TRACE(1);
        const int e = c0 + tid;
        const bool valid = e < ne_t && !(FM_DBG(mdl) & 8);  // 8: data-movement-only probe
        double P[D][DIM];
        double Wel = 0.0, det_el = 1.0, ls_el = 0.0;  // this element's W (J) and its log fix-up
        bool far = false;
        Elem<DIM> E;
        if (valid) {
          // the record: row tid of the stage, or the dictionary entry its slot byte names
          const unsigned char *rbase = stg(s);
          int ridx = tid;
          if (tm.dict_n) {
            ridx = rbase[((tm.own_begin + c0) & 15) + tid];
            rbase = dict_of(tb);
          }
          load_elem_smem<DIM>(rbase, ridx, E);
          decode_loc(*reinterpret_cast<const uint2 *>(stg(s) + L::loc_off(REC) +
                                                       (tid + ((tm.own_begin + c0) & 1)) * 8),
                     E.loc);
          double vv[D][NV];
#pragma unroll
          for (int l = 0; l < NV; ++l)
#pragma unroll
            for (int k = 0; k < D; ++k) vv[k][l] = nv[k * CAP + E.loc[l]];
          double F[D][DIM];
          if (!FDM && !EO) grad_F_fma<DIM, D>(vv, E.g, F);
          const bool own = true;
          if (EO) {
            grad_F<DIM, D>(vv, E.g, F);
            const double W = density<DIM, MODEL>(F, mdl);
            if (g) g[__ldg(a.s2o + (int64_t)tm.own_begin + e)] = W;
            jsum += E.vol * W;
          } else if (FDM) {
            if (has_nodes) {
              const FdSink sink{st_at(0, tid), (int)L::slot_stride(D), CS, a.closure, a.rank_of,
                                a.s2o, tm.clo_begin, (int64_t)tm.own_begin + c0 + tid};
              fd_element<DIM, MODEL, D>(vv, E, mdl, sink, rbase, ridx, nv, CAP,
                                        make_int4(E.loc[0], E.loc[1], E.loc[2],
                                                  DIM == 3 ? E.loc[DIM] : 0),
                                        &fdkey);
            }
          } else if (FM_DBG(mdl) & 1) {  // ablation: no constitutive work
#pragma unroll
            for (int k = 0; k < D; ++k)
#pragma unroll
              for (int m = 0; m < DIM; ++m) P[k][m] = F[k][m];
          } else if (HV && has_nodes) {
            double pp[D][NV];
#pragma unroll
            for (int l = 0; l < NV; ++l)
#pragma unroll
              for (int k = 0; k < D; ++k) pp[k][l] = nv[(D + k) * CAP + E.loc[l]];
            double dF[D][DIM];
            grad_F_fma<DIM, D>(pp, E.g, dF);
            bool bad;
            element_dP<DIM, MODEL>(F, dF, E.vol, mdl, P, bad);
            bad_any |= bad;
          } else if (has_nodes) {
            bool bad;
            element_P<DIM, MODEL, D>(F, vv, E.g, E.vol, mdl, WJ && own, P, Wel, bad, far, det_el,
                                     ls_el);
            bad_any |= bad;
          } else if (WJ) {
            jsum += E.vol * density<DIM, MODEL>(F, mdl);
          }
        }
        // contributions -> staging buffer (separate from the record stages, so
        // the TMA engine never overwrites generic-proxy writes: no proxy fence)
        if (!FDM && !EO && valid && has_nodes) {
#pragma unroll
          for (int l = 0; l < NV; ++l)
#pragma unroll
            for (int k = 0; k < D; ++k) {
              double sdot = P[k][0] * E.g[0][l];
#pragma unroll
              for (int m = 1; m < DIM; ++m) sdot = fma(P[k][m], E.g[m][l], sdot);
              st_at(l, tid)[k * CS] = sdot;
            }
          if (WJ) {
            if (far) Wel += 2.0 * mdl.C1 * (ls_el - log(det_el));
            jsum += E.vol * Wel;
          }
        }
        TRACE(2);
        __syncthreads();  // contributions staged; every record of stage s read
        TRACE(3);
        // stage s is free: records of chunk q + 2
        if (!EO && my_node && !(FM_DBG(mdl) & 2)) {
          // this node's entries of the chunk (its slice of the chunk's entry
          // block): the loads of two entries are issued together; the order
          // (ascending tile element) is the fixed summation order
          const uint16_t *blk = reinterpret_cast<const uint16_t *>(stg(s) + L::blk_off(REC));
          const int e_beg = blk[tid], n = blk[tid + 1] - e_beg;
          const uint16_t *ents = blk + blk_header(tm.node_count) + e_beg;
          int i = 0;
          for (; i + 1 < n; i += 2) {
            const int e0 = ents[i], e1 = ents[i + 1];
            if ((e1 >> 2) >= ne_t) break;  // cross entries (finishing pass) from here on
            const double *s0 = st_at(e0 & 3, (e0 >> 2) - c0);
            const double *s1 = st_at(e1 & 3, (e1 >> 2) - c0);
            double x0[D], x1[D];
#pragma unroll
            for (int k = 0; k < D; ++k) {
              x0[k] = s0[k * CS];
              x1[k] = s1[k * CS];
            }
#pragma unroll
            for (int k = 0; k < D; ++k) acc[k] = (acc[k] + x0[k]) + x1[k];
          }
          if (i < n) {
            const int e0 = ents[i];
            const double *s0 = st_at(e0 & 3, (e0 >> 2) - c0);
            if ((e0 >> 2) < ne_t) {
#pragma unroll
              for (int k = 0; k < D; ++k) acc[k] += s0[k * CS];
            }
          }
        }
        for (int i = xb + tid; !EO && i < xe; i += CT) {
          const int key = i == xb + tid ? xkey0 : (int)__ldg(a.xkey + i);
          const int64_t pos = i;  // item i -> exchange slot i (coalesced stores)
          const double *sp = st_at(key & 3, (key >> 2) - c0);
#pragma unroll
          for (int k = 0; k < D; ++k) a.xbuf[pos * D + k] = sp[k * CS];
        }
        // one staging buffer: it must be consumed before the next chunk writes
        // it; two: the next chunk's barrier already orders this consumption
        // before the write two chunks ahead
        TRACE(4);
        if (!EO) __syncthreads();  // stage s consumed: records of chunk q + 2 (EO: barrier 1)
        TRACE(5);
        issue_records(iss, s);
        iss.advance(a);
      }
      if (WJ && my_node && b) {
#pragma unroll
        for (int k = 0; k < D; ++k) bvsum += bj[k] * nv[k * CAP + cl];
      }
      if (my_node && !EO) {
        if (cross) {
          // cross entries follow in the finishing pass: dense partial by tile node
          // (FD: the plain difference sum; the scaling follows the cross entries)
#pragma unroll
          for (int k = 0; k < D; ++k)
            a.partial[(int64_t)(tm.node_begin + tid) * D + k] = FDM ? acc[k] : acc[k] - bj[k];
        } else if (FDM) {
          int o = outw;
          const double inv = 2.0 * mdl.eps;
#pragma unroll
          for (int k = 0; k < D; ++k)
            if (fmask & (1 << k)) {
              const double q = acc[k] / inv;
              g[o++] = b ? q - __ldg(b + (int64_t)nd.z * D + k) : q;
            }
        } else {
          int o = outw;
#pragma unroll
          for (int k = 0; k < D; ++k)
            if (fmask & (1 << k)) g[o++] = acc[k] - bj[k];
        }
      }
      ++j;
      comp.t += gridDim.x;  // every tile is visited (outputs), even without chunks
      comp.c0 = 0;
      comp.load(a);
    }
  }
  if (bad_any) atomicOr(status, 1ull);
  if (FDM && fdkey != ~0ull) atomicMin(status + 1, fdkey);
  if (WJ) {
    const double r = block_sum(jsum, red);
    const double r2 = block_sum(bvsum, red);
    if (tid == 0) {
      jpart[blockIdx.x] = r;
      bvpart[blockIdx.x] = r2;
    }
  }
}

// Finishing pass: a node's cross entries (elements owned by other tiles) were
// written by their owner tiles into xbuf at the node's dense exchange slots
// [xbase[k], xbase[k + 1]) (consecutive nodes back to back); the tile kernel
// left the node's own-element sum (minus b) in partial.  g = partial + the
// cross entries in ascending tile-element order.
// With J (jf.out): every block also adds b.v of its share of the nodes without
// a free dof (fixed block tree) into jf.fpart, and the last block to finish
// (atomic ticket) sums the tile kernel's per-CTA partials and these in index
// order: J = sum vol W - (b.v of tile nodes + b.v of fixed nodes).  The result
// does not depend on which block is last; the ticket is reset for the next call.
// FD (FDX): g = (partial + cross entries) / (2 eps) - b of the node (fdx.b at
// node_desc[tile node].z), as the tile kernel's own nodes.
struct FdFinish {
  double inv;            // 2 eps
  const double *b;       // load (may be null)
  const int4 *node_desc;
};

template <int D, bool FDX>
__global__ void __launch_bounds__(256) k_finish_cross(int64_t ntn,
                                                      const int4 *__restrict__ xdesc,
                                                      const int32_t *__restrict__ xinv,
                                                      const double *__restrict__ xbuf,
                                                      const double *__restrict__ partial,
                                                      double *__restrict__ g, JFinal jf,
                                                      FdFinish fdx) {
  // one thread per (node, component): the D threads of a node read adjacent
  // doubles of each exchange slot
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ntn * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / D;
    const int j = (int)(i - r * D);
    const int4 xd = __ldg(xdesc + r);  // {tile node, first slot, count | mask << 16, out}
    const int mask = xd.z >> 16, lo = xd.y, hi = lo + (xd.z & 0xffff);
    if (!(mask & (1 << j))) continue;
    double sum = partial[(int64_t)xd.x * D + j];
    // four entries per step (the last step predicated): their slot loads,
    // then their value loads, are issued back to back; the sum stays
    // sequential in entry order
    constexpr int U = 4;  // 8: cfg4 finishing pass 1 % slower
    for (int p = lo; p < hi; p += U) {
      int sl[U];
      double x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) sl[u] = p + u < hi ? __ldg(xinv + p + u) : -1;
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = sl[u] >= 0 ? __ldg(xbuf + (int64_t)sl[u] * D + j) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (p + u < hi) sum += x[u];
    }
    if (FDX) {
      const double q = sum / fdx.inv;
      sum = fdx.b ? q - __ldg(fdx.b + (int64_t)__ldg(&fdx.node_desc[xd.x].z) * D + j) : q;
    }
    g[xd.w + __popc(mask & ((1 << j) - 1))] = sum;
  }
  if (!jf.out) return;
  __shared__ double red[32];
  __shared__ bool last;
  double f = 0.0;
  if (jf.b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < jf.nfixed;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t q = (int64_t)__ldg(jf.fixed_nodes + i) * D;
#pragma unroll
      for (int j = 0; j < D; ++j) f += __ldg(jf.b + q + j) * __ldg(jf.v + q + j);
    }
  }
  f = block_sum(f, red);
  if (threadIdx.x == 0) {
    jf.fpart[blockIdx.x] = f;
    __threadfence();
    last = atomicAdd(jf.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a = 0.0, c = 0.0, ff = 0.0;
  for (int i = threadIdx.x; i < jf.njp; i += blockDim.x) a += jf.jp[i];
  if (jf.b) {
    for (int i = threadIdx.x; i < jf.njp; i += blockDim.x) c += jf.bvp[i];
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) ff += __ldcg(jf.fpart + i);
  }
  const double A = block_sum(a, red);
  const double C = block_sum(c, red);
  const double F = block_sum(ff, red);
  if (threadIdx.x == 0) {
    jf.out[0] = A - (C + F);
    jf.out[1] = A;
    jf.out[2] = C + F;
    *jf.ticket = 0u;
  }
}

int finish_cross_grid(int d, int64_t ntn) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((ntn * d + 255) / 256, finish_max_blocks()));
}

template <bool FDX>
static void finish_d(int d, int grid, int64_t ntn, const int4 *xdesc, const int32_t *xinv,
                     const double *xbuf, const double *partial, double *g, const JFinal &jf,
                     const FdFinish &fdx, cudaStream_t s) {
  if (d == 3)
    k_finish_cross<3, FDX><<<grid, 256, 0, s>>>(ntn, xdesc, xinv, xbuf, partial, g, jf, fdx);
  else if (d == 2)
    k_finish_cross<2, FDX><<<grid, 256, 0, s>>>(ntn, xdesc, xinv, xbuf, partial, g, jf, fdx);
  else
    k_finish_cross<1, FDX><<<grid, 256, 0, s>>>(ntn, xdesc, xinv, xbuf, partial, g, jf, fdx);
}

cudaError_t launch_finish_cross(int d, int64_t ntn, const int4 *xdesc, const int32_t *xinv,
                                const double *xbuf, const double *partial, double *g,
                                const JFinal &jf, cudaStream_t s) {
  // enough blocks for the cross nodes and for the b.v of the fixed nodes
  int grid = finish_cross_grid(d, ntn);
  if (jf.out && jf.b)
    grid = std::max<int>(grid, (int)std::min<int64_t>((jf.nfixed + 255) / 256, finish_max_blocks()));
  finish_d<false>(d, grid, ntn, xdesc, xinv, xbuf, partial, g, jf,
                  FdFinish{0.0, nullptr, nullptr}, s);
  return cudaGetLastError();
}

cudaError_t launch_finish_cross_fd(int d, int64_t ntn, const int4 *xdesc, const int32_t *xinv,
                                   const double *xbuf, const double *partial, double *g,
                                   double eps, const double *b, const int4 *node_desc,
                                   cudaStream_t s) {
  JFinal jf{};
  finish_d<true>(d, finish_cross_grid(d, ntn), ntn, xdesc, xinv, xbuf, partial, g, jf,
                 FdFinish{2.0 * eps, b, node_desc}, s);
  return cudaGetLastError();
}

template <int DIM, int CT>
static size_t smem_of(int d, int blk_cap, int clo_cap, int nb, int tb, int dn, bool all_coded) {
  using L = PipeLayout<DIM, CT>;
  return L::total(d, blk_cap, clo_cap, nb, tb, dn, L::rec_area(all_coded));
}

size_t tile_exact_smem(int dim, int d, int blk_cap, int clo_cap, int ct, int nb, int tb, int dn,
                       bool all_coded) {
  if (ct == 128)
    return dim == 3 ? smem_of<3, 128>(d, blk_cap, clo_cap, nb, tb, dn, all_coded)
                    : smem_of<2, 128>(d, blk_cap, clo_cap, nb, tb, dn, all_coded);
  return dim == 3 ? smem_of<3, 256>(d, blk_cap, clo_cap, nb, tb, dn, all_coded)
                  : smem_of<2, 256>(d, blk_cap, clo_cap, nb, tb, dn, all_coded);
}

template <int DIM, int MODEL, int CT, int NB, int TB>
static cudaError_t launch_cfg(const TileArgs &a, int grid, int mode, const double *v,
                              const double *b, double *g, double *jpart, double *bvpart,
                              unsigned long long *status, const ModelArgs &m, cudaStream_t s) {
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  constexpr int MINB = tile_exact_minb(DIM, CT), MINBF = tile_fd_minb(DIM, CT, MODEL);
  const size_t smem =
      smem_of<DIM, CT>(D, a.blk_cap, a.clo_cap, NB, TB, mode == 2 ? 2 * D : D, a.all_coded != 0);
  auto k = mode == 4   ? k_tile_exact<DIM, MODEL, true, false, false, true, CT, NB, TB, MINB>
           : mode == 3 ? k_tile_exact<DIM, MODEL, false, false, true, false, CT, NB, TB, MINBF>
           : mode == 2 ? k_tile_exact<DIM, MODEL, false, true, false, false, CT, NB, TB, MINB>
           : mode == 1 ? k_tile_exact<DIM, MODEL, true, false, false, false, CT, NB, TB, MINB>
                       : k_tile_exact<DIM, MODEL, false, false, false, false, CT, NB, TB, MINB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, CT, smem, s>>>(a, v, b, g, jpart, bvpart, status, m);
  return cudaGetLastError();
}

template <int DIM, int MODEL, int CT>
static cudaError_t launch_ct(const TileArgs &a, int grid, int nb, int ns, int mode,
                             const double *v, const double *b, double *g, double *jpart,
                             double *bvpart, unsigned long long *status, const ModelArgs &m,
                             cudaStream_t s) {
  if (nb == 2 && ns == 2)
    return launch_cfg<DIM, MODEL, CT, 2, 2>(a, grid, mode, v, b, g, jpart, bvpart, status, m, s);
  if (nb == 2) return launch_cfg<DIM, MODEL, CT, 2, 1>(a, grid, mode, v, b, g, jpart, bvpart, status, m, s);
  if (ns == 2) return launch_cfg<DIM, MODEL, CT, 1, 2>(a, grid, mode, v, b, g, jpart, bvpart, status, m, s);
  return launch_cfg<DIM, MODEL, CT, 1, 1>(a, grid, mode, v, b, g, jpart, bvpart, status, m, s);
}

template <int DIM, int MODEL>
static cudaError_t launch_exact_t(const TileArgs &a, int grid, int ct, int nb, int ns, int mode,
                                  const double *v, const double *b, double *g, double *jpart,
                                  double *bvpart, unsigned long long *status, const ModelArgs &m,
                                  cudaStream_t s) {
  if (ct == 128)
    return launch_ct<DIM, MODEL, 128>(a, grid, nb, ns, mode, v, b, g, jpart, bvpart, status, m, s);
  return launch_ct<DIM, MODEL, 256>(a, grid, nb, ns, mode, v, b, g, jpart, bvpart, status, m, s);
}

cudaError_t launch_tile_exact(int dim, int model, const TileArgs &a, int grid, int ct, int nb,
                              int ns, int mode, const double *v, const double *b, double *g,
                              double *jpart, double *bvpart, unsigned long long *status,
                              const ModelArgs &m, cudaStream_t s) {
  if (dim == 2 && model == FM_MODEL_PLAPLACE)
    return launch_exact_t<2, FM_MODEL_PLAPLACE>(a, grid, ct, nb, ns, mode, v, b, g, jpart, bvpart,
                                                status, m, s);
  if (dim == 3 && model == FM_MODEL_PLAPLACE)
    return launch_exact_t<3, FM_MODEL_PLAPLACE>(a, grid, ct, nb, ns, mode, v, b, g, jpart, bvpart,
                                                status, m, s);
  if (dim == 2)
    return launch_exact_t<2, FM_MODEL_NEOHOOKEAN>(a, grid, ct, nb, ns, mode, v, b, g, jpart,
                                                  bvpart, status, m, s);
  return launch_exact_t<3, FM_MODEL_NEOHOOKEAN>(a, grid, ct, nb, ns, mode, v, b, g, jpart, bvpart,
                                                status, m, s);
}

}  // namespace fm
