// Nodal-patch finite-difference gradient (gradients.py:84-121).
//
// The reference perturbs the nodal value v_l of component j by s = -/+eps,
// recomputes row j of F from the perturbed values (evaluate_GG,
// gradients.py:35-51; the other rows are the unperturbed F) and evaluates the
// density of every perturbed patch row; g = (sum vol W+ - sum vol W-)/(2 eps)
// - b.  Row j of the recomputed F is F0_j + dl * dphi[:, l] with dl =
// fl(v_l + s) - v_l the step the rounded perturbed value actually carries,
// and det F and |F|^2 are affine / quadratic in one row, so the perturbed
// state's invariants follow from the unperturbed ones (rank-one update):
//   det  = det0 + dl * c_jl,          c_jl = cof(F0)_j . dphi[:, l]
//   I1   = I1_0 + dl (a_jl + dl b_l), a_jl = 2 F0_j . dphi[:, l], b_l = |dphi[:, l]|^2
//   log det = log det0 + log1p(dl c_jl / det0)
//   (p-Laplace: |g|^2 = n2_0 + dl (a_l + dl b_l))
// and W is the reference's expression of those invariants (models.py:89-100,
// 123-126).  Each W+- is evaluated on its own and differenced afterwards, as
// the reference does; the per-state rounding (a few ulps of each term of W) is
// of the reference's own size and is what the FD tolerance allows for
// (tests/test_gpu_parity.py).  States whose det is near 0 are
// recomputed exactly the reference's way (einsum F, six-term det, the
// reference density), so admissibility and the first offending dof
// (gradients.py:77-81) are decided as in numpy.
//
// One CTA per node tile; its element list (own + halo, dealt order) in chunks
// of CT rows, three phases per chunk:
//  rows   thread r: record c0 + r, v of its nodes from the tile's closure
//         values (gathered once per tile), F0 in einsum order, det0 / I1_0 /
//         log det0 (reference order) and the per-slot coefficients c, a, b ->
//         a shared-memory row block (structure of arrays);
//  items  the chunk's entries in (row, slot) order (fd_items; consecutive
//         threads read consecutive rows), all D components and both signs per
//         item; vol W+ - vol W- to the entry's node-major slot;
//  nodes  node thread n sums its entries in ascending tile-element order;
//         g = S / (2 eps) - b.
// A non-finite density latches the smallest key (sign, j, free rank, element),
// i.e. the first offending stacked row in reference order (gradients.py:77-81).
#include "fm_density.cuh"
#include "fm_kernels.h"
#include "fm_pipe.cuh"

namespace fm {

// fields of the shared-memory row block ([field][row], doubles)
template <int DIM, int MODEL>
struct FdRow {
  static constexpr int NV = DIM + 1;
  static constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  static constexpr bool NH = MODEL == FM_MODEL_NEOHOOKEAN;
  static constexpr int VOL = 0;
  static constexpr int BASE = 1;   // det0 (NH) | n2_0 (p-Laplace)
  static constexpr int RDET = 2;   // NH: 1 / det0
  static constexpr int LD = 3;     // NH: log det0 (NaN if det0 <= 0)
  static constexpr int I1 = 4;     // NH: |F0|^2
  static constexpr int C0 = NH ? 5 : 2;              // c[j][l] (NH only)
  static constexpr int A0 = NH ? C0 + D * NV : C0;   // a[j][l]
  static constexpr int BB = A0 + D * NV;             // b[l]
  static constexpr int LW = BB + NV;                 // closure indices (u16 x 4, as bits)
  static constexpr int RF = LW + 1;
};

template <int DIM, int MODEL, int CT>
struct FdLayout {
  __host__ __device__ static size_t r16(size_t x) { return (x + 15) / 16 * 16; }
  __host__ __device__ static size_t nodev(int D, int cap) { return r16((size_t)D * cap * 8); }
  __host__ __device__ static size_t rows() { return (size_t)FdRow<DIM, MODEL>::RF * CT * 8; }
  __host__ __device__ static size_t stg(int D, int ech) { return r16((size_t)D * ech * 8); }
  __host__ __device__ static size_t hdr() { return r16((size_t)blk_header(CT) * 2); }
  __host__ __device__ static size_t items(int ech) { return r16((size_t)(ech + 8) * 4); }
  __host__ __device__ static size_t total(int D, int cap, int ech) {
    return nodev(D, cap) + rows() + stg(D, ech) + hdr() + items(ech);
  }
};

// states with det below this (absolute; det ~ 1 for the elastic configs) are
// recomputed in the reference's operation order (see the file header)
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

// The reference's own evaluation of one perturbed state (rare: near-singular
// states): row j of F recomputed from the perturbed value ve of slot l in
// einsum order, the other rows unperturbed, the reference density.
template <int DIM, int MODEL>
__device__ __noinline__ double fd_state_ref(const TileArgs &a, const TileMeta &tm, int te,
                                            const double *nodev, int CAP, uint64_t lw, int j,
                                            int l, double ve, const ModelArgs &mdl) {
  constexpr int NV = DIM + 1;
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  constexpr int NQ = RecBytes<DIM>::value / 16;
  const int64_t s = te < tm.own_count
                        ? (int64_t)tm.own_begin + te
                        : (int64_t)__ldg(a.halo_ids + tm.halo_begin + te - tm.own_count);
  const double2 *p = reinterpret_cast<const double2 *>(a.aos + s * RecBytes<DIM>::value);
  double2 q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = __ldg(p + k);
  Elem<DIM> E;
  decode_elem<DIM>(q, E);
  double vv[D][NV];
#pragma unroll
  for (int ll = 0; ll < NV; ++ll) {
    const int c = (int)((lw >> (16 * ll)) & 0xffffull);
#pragma unroll
    for (int k = 0; k < D; ++k) vv[k][ll] = nodev[k * CAP + c];
  }
#pragma unroll
  for (int k = 0; k < D; ++k)
    if (k == j) vv[k][l] = ve;
  double F[D][DIM];
  grad_F<DIM, D>(vv, E.g, F);
  return density<DIM, MODEL>(F, mdl);
}

// 3D: 2 x 256 threads per SM (<= 128 registers); 2D: 4 x 256 (<= 64)
template <int DIM, int MODEL, int CT>
__global__ void __launch_bounds__(CT, (DIM == 2 ? 1024 : 512) / CT)
    k_tile_fd(TileArgs a, const double *__restrict__ v, const double *__restrict__ b, double eps,
              double *__restrict__ g, unsigned long long *badkey, ModelArgs mdl, int ech) {
  using R = FdRow<DIM, MODEL>;
  constexpr int NV = DIM + 1;
  constexpr int D = R::D;
  constexpr int RB = RecBytes<DIM>::value;
  constexpr int NQ = RB / 16;
  using L = FdLayout<DIM, MODEL, CT>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int CAP = a.clo_cap;
  double *nodev = reinterpret_cast<double *>(smem);
  double *rowb = reinterpret_cast<double *>(smem + L::nodev(D, CAP));
  double *stg = reinterpret_cast<double *>(reinterpret_cast<unsigned char *>(rowb) + L::rows());
  uint16_t *hdr =
      reinterpret_cast<uint16_t *>(reinterpret_cast<unsigned char *>(stg) + L::stg(D, ech));
  uint32_t *its = reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned char *>(hdr) + L::hdr());
  auto fld = [&](int f, int r) -> double & { return rowb[f * CT + r]; };
  const int tid = threadIdx.x;

  const TileMeta tm = a.meta[blockIdx.x];
  if (tm.node_count == 0) return;  // orphan tile: no free node, nothing to differentiate
  // the tile's closure node values: ids first, then 8-byte LDGSTS per value
  for (int i = tid; i < tm.clo_count; i += CT) {
    const double *src = v + (int64_t)__ldg(a.closure + tm.clo_begin + i) * D;
#pragma unroll
    for (int k = 0; k < D; ++k)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(nodev + k * CAP + i)),
                   "l"(src + k)
                   : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  const bool my_node = tid < tm.node_count;
  int4 nd = make_int4(0, 0, 0, 0);
  if (my_node) nd = a.node_desc[tm.node_begin + tid];
  double acc[D];
#pragma unroll
  for (int j = 0; j < D; ++j) acc[j] = 0.0;
  unsigned long long mykey = ~0ull;
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  const int ne_t = tm.own_count + tm.halo_count;
  // storage id of this thread's row of the next chunk, loaded one chunk ahead
  auto row_src = [&](int e) -> int64_t {
    if (e >= ne_t) return -1;
    return e >= tm.own_count ? (int64_t)__ldg(a.halo_ids + tm.halo_begin + e - tm.own_count)
                             : (int64_t)tm.own_begin + e;
  };
  int64_t s_next = row_src(tid);
  const int H = blk_header(tm.node_count);
  // p-Laplace (small row block, registers to spare): this thread's row of the
  // NEXT chunk (record and closure indices) is loaded into registers right
  // after the current rows phase, so that the items and node-sum phases hide
  // its latency (cfg2 1.156 -> 1.109 ms).  Neo-Hookean keeps an L2 prefetch:
  // the extra live registers spill in its items loop (cfg4 4.51 -> 4.93 ms),
  // although the record loads are ~19 % of its time (profiling ablation
  // FM_FD_ABL_REC: 3.65 ms with every row reading one cached record).
  constexpr bool REGPF = MODEL == FM_MODEL_PLAPLACE;
  double2 qn[NQ];
  uint2 lwn = make_uint2(0, 0);
  auto fetch = [&](int e, int64_t st) {
    if (e >= ne_t) return;
    const double2 *p = reinterpret_cast<const double2 *>(a.aos + st * RB);
#pragma unroll
    for (int k = 0; k < NQ; ++k) qn[k] = ld_stream(p + k);
    lwn = e >= tm.own_count ? __ldg(a.halo_loc + tm.halo_begin + e - tm.own_count)
                            : __ldg(a.loc + st);
  };
  if constexpr (REGPF) fetch(tid, s_next);
  for (int c0 = 0, ch = 0; c0 < ne_t; c0 += CT, ++ch) {
    // ---- the chunk's node offsets (its entry block's header) and its
    // row-major items: asynchronous copies (LDGSTS), landing during the rows
    {
      const uint16_t *hsrc = a.chunk_blocks + tm.blk_base + (int64_t)ch * tm.blk_stride;
      const uint32_t *isrc = a.fd_items + tm.blk_base + (int64_t)ch * tm.blk_stride;
      const int nh = H / 8, ni = (tm.blk_stride - H) / 4;
      for (int i = tid; i < nh + ni; i += CT) {
        const void *src = i < nh ? (const void *)(hsrc + 8 * i) : (const void *)(isrc + 4 * (i - nh));
        void *dst = i < nh ? (void *)(hdr + 8 * i) : (void *)(its + 4 * (i - nh));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // ---- rows
    const int e = c0 + tid;
    const int64_t s = s_next;
    if (e < ne_t) {
      double2 q[NQ];
      uint2 lw;
      if constexpr (REGPF) {
#pragma unroll
        for (int k = 0; k < NQ; ++k) q[k] = qn[k];
        lw = lwn;
      } else {
        const bool halo = e >= tm.own_count;
        const int h = tm.halo_begin + e - tm.own_count;
#ifdef FM_FD_ABL_REC
        // profiling ablation: every row reads the tile's first record (cached)
        const int64_t sr = tm.own_begin;
#else
        const int64_t sr = s;
#endif
        const double2 *p = reinterpret_cast<const double2 *>(a.aos + sr * RB);
#pragma unroll
        for (int k = 0; k < NQ; ++k) q[k] = ld_stream(p + k);
        lw = halo ? __ldg(a.halo_loc + h) : __ldg(a.loc + s);
      }
      Elem<DIM> E;
      decode_elem<DIM>(q, E);
      decode_loc(lw, E.loc);
      double vv[D][NV];
#pragma unroll
      for (int l = 0; l < NV; ++l)
#pragma unroll
        for (int k = 0; k < D; ++k) vv[k][l] = nodev[k * CAP + E.loc[l]];
      double F[D][DIM];
      grad_F<DIM, D>(vv, E.g, F);  // einsum order: the reference's unperturbed F
      fld(R::VOL, tid) = E.vol;
      fld(R::LW, tid) = __longlong_as_double(
          (long long)(((unsigned long long)lw.y << 32) | (unsigned long long)lw.x));
#pragma unroll
      for (int l = 0; l < NV; ++l) {
        double bb = E.g[0][l] * E.g[0][l];
#pragma unroll
        for (int m = 1; m < DIM; ++m) bb = fma(E.g[m][l], E.g[m][l], bb);
        fld(R::BB + l, tid) = bb;
      }
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int l = 0; l < NV; ++l) {
          double s2 = F[j][0] * E.g[0][l];
#pragma unroll
          for (int m = 1; m < DIM; ++m) s2 = fma(F[j][m], E.g[m][l], s2);
          fld(R::A0 + j * NV + l, tid) = 2.0 * s2;
        }
      if constexpr (R::NH) {
        const double det0 = det_F<DIM>(F);
        fld(R::BASE, tid) = det0;
        fld(R::RDET, tid) = 1.0 / det0;
        fld(R::LD, tid) = det0 > 0.0 ? log(det0) : NAN;
        fld(R::I1, tid) = sumsq_rn<DIM, D>(F);
        double C[DIM][DIM];
        cof_F<DIM>(F, C);
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
          for (int l = 0; l < NV; ++l) {
            double c = C[j][0] * E.g[0][l];
#pragma unroll
            for (int m = 1; m < DIM; ++m) c = fma(C[j][m], E.g[m][l], c);
            fld(R::C0 + j * NV + l, tid) = c;
          }
      } else {
        fld(R::BASE, tid) = sumsq_rn<DIM, D>(F);
      }
    }
    // next chunk: its storage ids now, its records (into registers, or
    // towards L2)
    s_next = row_src(e + CT);
    if constexpr (REGPF) {
      fetch(e + CT, s_next);
    } else if (s_next >= 0) {
      const uint8_t *pn = a.aos + s_next * RB;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pn));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pn + RB - 1));
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // header and items landed; rows published
    const int base = my_node ? hdr[tid] : 0;
    const int cnt = my_node ? hdr[tid + 1] - base : 0;
    const int total = hdr[tm.node_count];
    // ---- items (row, slot): all D components, both signs
    for (int f = tid; f < total; f += CT) {
      const uint32_t it = its[f];
      const int r = (int)((it >> 2) & 0x3ffu), l = (int)(it & 3u), pos = (int)(it >> 16);
      const uint64_t lw = (uint64_t)__double_as_longlong(fld(R::LW, r));
      const int cl = (int)((lw >> (16 * l)) & 0xffffull);
      const double vol = fld(R::VOL, r), base0 = fld(R::BASE, r), bb = fld(R::BB + l, r);
      double rdet0 = 0.0, ld0 = 0.0, i10 = 0.0;
      if constexpr (R::NH) {
        rdet0 = fld(R::RDET, r);
        ld0 = fld(R::LD, r);
        i10 = fld(R::I1, r);
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double vl = nodev[j * CAP + cl];
        const double aj = fld(R::A0 + j * NV + l, r);
        const double cj = R::NH ? fld(R::C0 + j * NV + l, r) : 0.0;
        double w[2];
#pragma unroll
        for (int sg = 0; sg < 2; ++sg) {
          const double ve = radd(vl, sg ? eps : -eps);  // the perturbed nodal value
          const double dl = ve - vl;                     // the step it carries
          double W = 0.0;
          bool exact = false;
          if constexpr (R::NH) {
            const double det = fma(dl, cj, base0);
            if (!(det > FD_DET_NEAR)) {
              exact = true;
            } else {
              const double I1 = fma(dl, fma(dl, bb, aj), i10);
              const double x = (dl * cj) * rdet0;
              const double ld = fabs(x) < 1e-3 ? ld0 + log1p_small(x) : log(det);
              const double dm1 = det - 1.0;
              W = mdl.C1 * ((I1 - (double)DIM) - 2.0 * ld) + mdl.D1 * (dm1 * dm1);
            }
          } else {
            const double n2 = fmax(fma(dl, fma(dl, bb, aj), base0), 0.0);
            W = np_scalar_pow(n2, mdl.e_w) / mdl.p;
          }
          if (exact)
            W = fd_state_ref<DIM, MODEL>(a, tm, r + c0, nodev, CAP, lw, j, l, ve, mdl);
          if (!isfinite(W)) {
            const int node = __ldg(a.closure + tm.clo_begin + cl);
            const int te = r + c0;
            const int64_t st = te < tm.own_count
                                   ? (int64_t)tm.own_begin + te
                                   : (int64_t)__ldg(a.halo_ids + tm.halo_begin + te - tm.own_count);
            const unsigned long long key = ((unsigned long long)sg << 63) |
                                           ((unsigned long long)j << 61) |
                                           ((unsigned long long)__ldg(a.rank_of + node) << 31) |
                                           (unsigned long long)__ldg(a.s2o + st);
            mykey = key < mykey ? key : mykey;
          }
          w[sg] = rmul(vol, W);
        }
        stg[j * ech + pos] = w[1] - w[0];
      }
    }
    __syncthreads();
    // ---- nodes: ascending tile-element order
    if (my_node) {
      for (int k = 0; k < cnt; ++k)  // the D component sums advance together
#pragma unroll
        for (int j = 0; j < D; ++j) acc[j] += stg[j * ech + base + k];
    }
    __syncthreads();
  }
  if (mykey != ~0ull) atomicMin(badkey, mykey);
  if (my_node) {
    const int mask = desc_mask(nd);
    int o = nd.w;
    const double inv = 2.0 * eps;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (mask & (1 << j)) {
        const double q = acc[j] / inv;
        g[o++] = b ? q - __ldg(b + (int64_t)nd.z * D + j) : q;
      }
    }
  }
}

template <int DIM, int MODEL, int CT>
static size_t fd_smem_t(int clo_cap, int ech) {
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  return FdLayout<DIM, MODEL, CT>::total(D, clo_cap, ech);
}

size_t tile_fd_smem(int dim, int model, int clo_cap, int ech, int ct) {
  const bool nh = model == FM_MODEL_NEOHOOKEAN;
  if (ct == 128) {
    if (dim == 3)
      return nh ? fd_smem_t<3, FM_MODEL_NEOHOOKEAN, 128>(clo_cap, ech)
                : fd_smem_t<3, FM_MODEL_PLAPLACE, 128>(clo_cap, ech);
    return nh ? fd_smem_t<2, FM_MODEL_NEOHOOKEAN, 128>(clo_cap, ech)
              : fd_smem_t<2, FM_MODEL_PLAPLACE, 128>(clo_cap, ech);
  }
  if (dim == 3)
    return nh ? fd_smem_t<3, FM_MODEL_NEOHOOKEAN, 256>(clo_cap, ech)
              : fd_smem_t<3, FM_MODEL_PLAPLACE, 256>(clo_cap, ech);
  return nh ? fd_smem_t<2, FM_MODEL_NEOHOOKEAN, 256>(clo_cap, ech)
            : fd_smem_t<2, FM_MODEL_PLAPLACE, 256>(clo_cap, ech);
}

template <int DIM, int MODEL, int CT>
static cudaError_t fd_t(const TileArgs &a, int n_tiles, int ech, const double *v, const double *b,
                        double eps, double *g, unsigned long long *badkey, const ModelArgs &m,
                        cudaStream_t s) {
  const size_t smem = fd_smem_t<DIM, MODEL, CT>(a.clo_cap, ech);
  auto k = k_tile_fd<DIM, MODEL, CT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<n_tiles, CT, smem, s>>>(a, v, b, eps, g, badkey, m, ech);
  return cudaGetLastError();
}

template <int DIM, int MODEL>
static cudaError_t fd_ct(const TileArgs &a, int n_tiles, int ct, int ech, const double *v,
                         const double *b, double eps, double *g, unsigned long long *badkey,
                         const ModelArgs &m, cudaStream_t s) {
  if (ct == 128) return fd_t<DIM, MODEL, 128>(a, n_tiles, ech, v, b, eps, g, badkey, m, s);
  return fd_t<DIM, MODEL, 256>(a, n_tiles, ech, v, b, eps, g, badkey, m, s);
}

cudaError_t launch_tile_fd(int dim, int model, const TileArgs &a, int n_tiles, int ct, int ech,
                           const double *v, const double *b, double eps, double *g,
                           unsigned long long *badkey, const ModelArgs &m, cudaStream_t s) {
  if (dim == 2 && model == FM_MODEL_PLAPLACE)
    return fd_ct<2, FM_MODEL_PLAPLACE>(a, n_tiles, ct, ech, v, b, eps, g, badkey, m, s);
  if (dim == 3 && model == FM_MODEL_PLAPLACE)
    return fd_ct<3, FM_MODEL_PLAPLACE>(a, n_tiles, ct, ech, v, b, eps, g, badkey, m, s);
  if (dim == 2)
    return fd_ct<2, FM_MODEL_NEOHOOKEAN>(a, n_tiles, ct, ech, v, b, eps, g, badkey, m, s);
  return fd_ct<3, FM_MODEL_NEOHOOKEAN>(a, n_tiles, ct, ech, v, b, eps, g, badkey, m, s);
}

}  // namespace fm
