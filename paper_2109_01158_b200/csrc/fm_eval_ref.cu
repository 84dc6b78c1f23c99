// Energy-only streaming kernel and the nodal-patch finite-difference kernel.
// F, det, I1, W follow the reference's rounding order exactly through the
// explicit round-to-nearest forms of fm_density.cuh (assembly.py:35-49,
// models.py:59-126); only the libm ulps of log/pow differ from numpy.
#include "fm_density.cuh"
#include "fm_kernels.h"

namespace fm {

// ----------------------------------------------------------------- energy
// assembly.py:94-106: every element once in storage order; block b sums the
// fixed range [b*per, (b+1)*per) with a fixed tree -> partial[b].
template <int DIM, int MODEL>
__global__ void __launch_bounds__(256) k_energy(TileArgs a, int64_t ne, int64_t per,
                                                const double *__restrict__ v,
                                                double *__restrict__ part,
                                                double *__restrict__ dens, ModelArgs mdl) {
  constexpr int NV = DIM + 1;
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  __shared__ double red[32];
  const int64_t lo = blockIdx.x * per, hi = min(ne, lo + per);
  double acc = 0.0;
  for (int64_t s = lo + threadIdx.x; s < hi; s += blockDim.x) {
    Elem<DIM> E;
    load_elem<DIM>(a.aos, a.conn4, s, E);
    double vv[D][NV];
    gather_v<DIM, D>(v, E.c, vv);
    double F[D][DIM];
    grad_F<DIM, D>(vv, E.g, F);
    double W = density<DIM, MODEL>(F, mdl);
    if (dens) dens[a.s2o[s]] = W;
    acc += E.vol * W;
  }
  double r = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

// b.v over all dofs (assembly.py:89-91), fixed ranges per block.
__global__ void __launch_bounds__(256) k_dot(const double *__restrict__ a,
                                             const double *__restrict__ b, int64_t n, int64_t per,
                                             double *__restrict__ part) {
  __shared__ double red[32];
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += a[i] * b[i];
  double r = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

// J = sum(partials) - sum(dot partials), fixed order, one block.
__global__ void __launch_bounds__(1024) k_finalize(const double *__restrict__ jp, int nj,
                                                   const double *__restrict__ dp, int nd,
                                                   double *__restrict__ out) {
  __shared__ double red[32];
  double a = 0.0, c = 0.0;
  for (int i = threadIdx.x; i < nj; i += blockDim.x) a += jp[i];
  for (int i = threadIdx.x; i < nd; i += blockDim.x) c += dp[i];
  double A = block_sum(a, red);
  double C = block_sum(c, red);
  if (threadIdx.x == 0) {
    out[0] = A - C;
    out[1] = A;
    out[2] = C;
  }
}

// ----------------------------------------------------------------- FD
// gradients.py:84-121.  One CTA per node tile; its element list (own + halo,
// dealt order) in chunks of CT rows, three phases per chunk:
//  rows   thread r loads record c0 + r (halo rows take this tile's closure
//         indices from halo_loc), gathers v from the tile's node values
//         (closure gathered once per tile) and forms the unperturbed F
//         (einsum order); record and F go to shared memory.
//  items  the chunk's node entries (te << 2 | slot) flattened in node order (a
//         block scan of the per-chunk counts in node_desc), times the D
//         components.  Item (j, f) recomputes row j of F from the perturbed
//         nodal values v_l -/+ eps (gradients.py:105-106, einsum order); the
//         other rows are the unperturbed F (evaluate_GG, gradients.py:35-51);
//         vol*W of both signs is staged.  Work per thread is even whatever the
//         mix of own / halo elements and owned slots.
//  nodes  node thread n sums its entries' minus and plus values separately in
//         ascending tile-element order; g = (S+ - S-)/(2 eps) - b
//         (gradients.py:118-120).
// A non-finite density latches the smallest key (sign, j, free rank, element),
// i.e. the first offending stacked row in reference order (gradients.py:77-81).
template <int DIM, int CT>
struct FdLayout {
  // expanded shared-memory rows: vol | dphi[DIM][DIM + 1] | loc word
  // (2D: +1 pad double, an odd number of 8-byte words per row, so the
  // row-per-lane stores of the rows phase hit distinct bank pairs: cfg3 FD
  // 0.52 -> 0.45 ms; in 3D the pad was slower, 6.89 -> 7.08 ms)
  static constexpr int FRB = 8 * (2 + DIM * (DIM + 1) + (DIM == 2 ? 1 : 0));
  __host__ __device__ static size_t r16(size_t x) { return (x + 15) / 16 * 16; }
  __host__ __device__ static size_t nodev(int D, int cap) { return r16((size_t)D * cap * 8); }
  __host__ __device__ static size_t recs() { return (size_t)CT * FRB; }
  __host__ __device__ static size_t fbuf(int D) { return r16((size_t)CT * D * DIM * 8); }
  __host__ __device__ static size_t stg(int D, int ech) { return (size_t)D * ech * 16; }
  __host__ __device__ static size_t flat(int blk_cap) { return r16((size_t)blk_cap * 2); }
  // 3D Neo-Hookean: per row det0, 1/det0, log(det0) of the unperturbed F
  // (2D: register-bound at 4 CTAs per SM, the reuse spills; measured slower)
  __host__ __device__ static size_t lrow(int D) {
    return D == DIM && DIM == 3 ? (size_t)CT * 3 * 8 : 0;
  }
  __host__ __device__ static size_t total(int D, int cap, int ech, int blk_cap) {
    return nodev(D, cap) + recs() + fbuf(D) + lrow(D) + stg(D, ech) + flat(blk_cap) + 32 * 4;
  }
};

// exclusive block scan of x (CT threads); total in every thread
template <int CT>
__device__ __forceinline__ int block_excl_scan(int x, int *wsum, int &total) {
  constexpr int NW = CT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int t = lane < NW ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < NW) wsum[lane] = t;
  }
  __syncthreads();
  total = wsum[NW - 1];
  return (w ? wsum[w - 1] : 0) + incl - x;
}

#ifndef FM_FD_PREFETCH
#define FM_FD_PREFETCH 1
#endif

// 3D: 2 x 256 threads per SM (<= 128 registers); 2D: 4 x 256 (<= 64; FD at
// cfg2 3.59 ms with 2, 2.69 with 3, 2.34 with 4 CTAs per SM)
template <int DIM, int MODEL, int CT>
__global__ void __launch_bounds__(CT, (DIM == 2 ? 1024 : 512) / CT)
    k_tile_fd(TileArgs a, const double *__restrict__ v, const double *__restrict__ b, double eps,
              double *__restrict__ g, unsigned long long *badkey, ModelArgs mdl, int ech) {
  constexpr int NV = DIM + 1;
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  constexpr int RB = RecBytes<DIM>::value;
  constexpr int NQ = RB / 16;
  constexpr int NF = D * DIM;
  using L = FdLayout<DIM, CT>;
  constexpr int FRB = L::FRB;
  constexpr int LW = 1 + DIM * NV;  // shared row word holding the closure indices
  extern __shared__ __align__(16) unsigned char smem[];
  const int CAP = a.clo_cap;
  double *nodev = reinterpret_cast<double *>(smem);
  unsigned char *recs = smem + L::nodev(D, CAP);
  double *Fb = reinterpret_cast<double *>(recs + L::recs());
  double *lrow = reinterpret_cast<double *>(reinterpret_cast<unsigned char *>(Fb) + L::fbuf(D));
  double2 *stg = reinterpret_cast<double2 *>(reinterpret_cast<unsigned char *>(lrow) + L::lrow(D));
  uint16_t *flat = reinterpret_cast<uint16_t *>(reinterpret_cast<unsigned char *>(stg) +
                                                L::stg(D, ech));
  int *wsum = reinterpret_cast<int *>(reinterpret_cast<unsigned char *>(flat) + L::flat(a.blk_cap));
  (void)wsum;
  const int tid = threadIdx.x;

  const TileMeta tm = a.meta[blockIdx.x];
  if (tm.node_count == 0) return;  // orphan tile: no free node, nothing to differentiate
  for (int i = tid; i < tm.clo_count; i += CT) {
    const double *src = v + (int64_t)__ldg(a.closure + tm.clo_begin + i) * D;
#pragma unroll
    for (int k = 0; k < D; ++k) nodev[k * CAP + i] = __ldg(src + k);
  }
  const bool my_node = tid < tm.node_count;
  int4 nd = make_int4(0, 0, 0, 0);
  if (my_node) nd = a.node_desc[tm.node_begin + tid];
  double accm[D], accp[D];
#pragma unroll
  for (int j = 0; j < D; ++j) accm[j] = accp[j] = 0.0;
  unsigned long long mykey = ~0ull;
  __syncthreads();

  const int ne_t = tm.own_count + tm.halo_count;
  // storage id of this thread's row of the next chunk, loaded one chunk ahead
  auto row_src = [&](int e) -> int64_t {
    if (e >= ne_t) return -1;
    return e >= tm.own_count ? (int64_t)__ldg(a.halo_ids + tm.halo_begin + e - tm.own_count)
                             : (int64_t)tm.own_begin + e;
  };
  int64_t s_next = row_src(tid);
  for (int c0 = 0, ch = 0; c0 < ne_t; c0 += CT, ++ch) {
    // ---- rows: record + unperturbed F of tile element c0 + tid
    const int e = c0 + tid;
    const int64_t s = s_next;
    if (e < ne_t) {
      const bool halo = e >= tm.own_count;
      const int h = tm.halo_begin + e - tm.own_count;
      const double2 *p = reinterpret_cast<const double2 *>(a.aos + s * RB);
      double2 q[NQ];
#pragma unroll
      for (int k = 0; k < NQ; ++k) q[k] = ld_stream(p + k);
      const uint2 lw = halo ? __ldg(a.halo_loc + h) : __ldg(a.loc + s);
      Elem<DIM> E;
      decode_elem<DIM>(q, E);
      decode_loc(lw, E.loc);
      double *dst = reinterpret_cast<double *>(recs + tid * FRB);
      dst[0] = E.vol;
#pragma unroll
      for (int m = 0; m < DIM; ++m)
#pragma unroll
        for (int l = 0; l < NV; ++l) dst[1 + m * NV + l] = E.g[m][l];
      *reinterpret_cast<uint2 *>(dst + LW) = lw;
      double vv[D][NV];
#pragma unroll
      for (int l = 0; l < NV; ++l)
#pragma unroll
        for (int k = 0; k < D; ++k) vv[k][l] = nodev[k * CAP + E.loc[l]];
      double F[D][DIM];
      grad_F<DIM, D>(vv, E.g, F);
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int m = 0; m < DIM; ++m) Fb[tid * NF + j * DIM + m] = F[j][m];
      if constexpr (MODEL == FM_MODEL_NEOHOOKEAN && DIM == 3) {
        // the row's log(det F) once: the 2 D perturbed states of each of its
        // entries differ from it by O(eps) (log_near)
        const double det0 = det_F<DIM>(F);
        lrow[tid] = det0;
        lrow[CT + tid] = 1.0 / det0;
        lrow[2 * CT + tid] = det0 > 0.0 ? log(det0) : NAN;
      }
    }
    // next chunk: its storage ids now, its own records towards L2
    s_next = row_src(e + CT);
    if (FM_FD_PREFETCH && s_next >= 0 && e + CT < tm.own_count) {
      const uint8_t *pn = a.aos + s_next * RB;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pn));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pn + RB - 1));
    }
    // ---- this chunk's entries in node order: the chunk's entry block (node
    // offsets + entries), copied as is
    {
      const uint4 *src = reinterpret_cast<const uint4 *>(a.chunk_blocks + tm.blk_base +
                                                         (int64_t)ch * tm.blk_stride);
      uint4 *dst = reinterpret_cast<uint4 *>(flat);
      for (int i = tid; i < tm.blk_stride / 8; i += CT) dst[i] = __ldg(src + i);
    }
    __syncthreads();  // (also publishes the rows)
    const int H = blk_header(tm.node_count);
    const int base = my_node ? flat[tid] : 0;
    const int cnt = my_node ? flat[tid + 1] - base : 0;
    const int total = flat[tm.node_count];
    // ---- items f (one entry: element row r, slot l), all D components and both
    // signs.  The row's data (dphi, unperturbed F, closure indices) are read
    // once per entry; j is a compile-time constant of each unrolled pass (no
    // selects between rows), the slot l is not, so the words of slot l are
    // addressed directly.  Row j of F keeps the einsum order (p0+p2)+(p1+p3)
    // [NV = 3: (p0+p2)+p1]: the pair holding p_l is (p_l + partner), the other
    // pair is unperturbed, and IEEE addition is commutative, so only p_l
    // depends on the sign.
    for (int f = tid; f < total; f += CT) {
      const int en = flat[H + f];
      const int r = (en >> 2) - c0, l = en & 3;
      const unsigned char *rec = recs + r * FRB;
      const double *rd = reinterpret_cast<const double *>(rec);  // vol | dphi[m][k]
      const unsigned long long lw = *reinterpret_cast<const unsigned long long *>(rec + LW * 8);
      auto gat = [&](int m, int k) { return rd[1 + m * NV + k]; };
      double F0[D][DIM];
#pragma unroll
      for (int jj = 0; jj < D; ++jj)
#pragma unroll
        for (int m = 0; m < DIM; ++m) F0[jj][m] = Fb[r * NF + jj * DIM + m];
      int lp, la = 0, lb = 0;
      if constexpr (NV == 4) {
        lp = l ^ 2;
        la = (l + 1) & 3;
        lb = (l + 3) & 3;
      } else {
        lp = l == 1 ? 0 : 2 - l;
        la = l == 1 ? 2 : 1;
      }
      double gl[DIM];
#pragma unroll
      for (int m = 0; m < DIM; ++m) gl[m] = gat(m, l);
      const int cl = (int)((lw >> (16 * l)) & 0xffffull), cp = (int)((lw >> (16 * lp)) & 0xffffull);
      const int ca = (int)((lw >> (16 * la)) & 0xffffull), cb = (int)((lw >> (16 * lb)) & 0xffffull);
      const double vol = rd[0];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double *nvj = nodev + j * CAP;
        const double vl = nvj[cl];
        double q1[DIM], q2[DIM];
        if constexpr (NV == 4) {
          const double vp = nvj[cp], va = nvj[ca], vb = nvj[cb];
#pragma unroll
          for (int m = 0; m < DIM; ++m) {
            q1[m] = rmul(vp, gat(m, lp));                               // partner of p_l
            q2[m] = radd(rmul(va, gat(m, la)), rmul(vb, gat(m, lb)));  // the other pair
          }
        } else {
          const double vp = nvj[cp], vo = nvj[ca];
#pragma unroll
          for (int m = 0; m < DIM; ++m) {
            q1[m] = rmul(vp, gat(m, lp));
            q2[m] = rmul(vo, gat(m, la));
          }
        }
        double w[2];
#pragma unroll
        for (int sg = 0; sg < 2; ++sg) {
          const double ve = radd(vl, sg ? eps : -eps);
          double Fp[D][DIM];
#pragma unroll
          for (int jj = 0; jj < D; ++jj)
#pragma unroll
            for (int m = 0; m < DIM; ++m) Fp[jj][m] = F0[jj][m];
#pragma unroll
          for (int m = 0; m < DIM; ++m) {
            const double pl = rmul(ve, gl[m]);
            if constexpr (NV == 4) {
              Fp[j][m] = radd(radd(pl, q1[m]), q2[m]);
            } else {  // (p0+p2)+p1: l = 1 is the lone term
              Fp[j][m] = l == 1 ? radd(radd(q1[m], q2[m]), pl) : radd(radd(pl, q1[m]), q2[m]);
            }
          }
          double W;
          if constexpr (MODEL == FM_MODEL_NEOHOOKEAN && DIM == 3) {
            W = density_nh_near<DIM>(Fp, mdl, lrow[r], lrow[CT + r], lrow[2 * CT + r]);
          } else {
            W = density<DIM, MODEL>(Fp, mdl);
          }
          if (!isfinite(W)) {
            const int node = __ldg(a.closure + tm.clo_begin + cl);
            const int te = r + c0;
            const int64_t s = te < tm.own_count
                                  ? (int64_t)tm.own_begin + te
                                  : (int64_t)__ldg(a.halo_ids + tm.halo_begin + te - tm.own_count);
            const unsigned long long key = ((unsigned long long)sg << 63) |
                                           ((unsigned long long)j << 61) |
                                           ((unsigned long long)__ldg(a.rank_of + node) << 31) |
                                           (unsigned long long)__ldg(a.s2o + s);
            mykey = key < mykey ? key : mykey;
          }
          w[sg] = rmul(vol, W);
        }
        stg[j * ech + f] = make_double2(w[0], w[1]);
      }
    }
    __syncthreads();
    // ---- nodes: ascending tile-element order, minus and plus separately
    if (my_node) {
#pragma unroll
      for (int j = 0; j < D; ++j)
        for (int k = 0; k < cnt; ++k) {
          const double2 x = stg[j * ech + base + k];
          accm[j] += x.x;
          accp[j] += x.y;
        }
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
        const double q = (accp[j] - accm[j]) / inv;
        g[o++] = b ? q - __ldg(b + (int64_t)nd.z * D + j) : q;
      }
    }
  }
}

size_t tile_fd_smem(int dim, int d, int clo_cap, int ech, int ct, int blk_cap) {
  if (ct == 128)
    return dim == 3 ? FdLayout<3, 128>::total(d, clo_cap, ech, blk_cap) : FdLayout<2, 128>::total(d, clo_cap, ech, blk_cap);
  return dim == 3 ? FdLayout<3, 256>::total(d, clo_cap, ech, blk_cap) : FdLayout<2, 256>::total(d, clo_cap, ech, blk_cap);
}

// ----------------------------------------------------------------- descent
// free dof q (the order of g and dofs_minim) -> its position in v
__global__ void k_dof_pos(int64_t nfree, int d, const int32_t *free_node, const int32_t *free_out,
                          const uint8_t *free_mask, int32_t *dof_pos) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nfree;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = free_node[r];
    const int mask = free_mask[r];
    int o = free_out[r];
    for (int j = 0; j < d; ++j)
      if (mask & (1 << j)) dof_pos[o++] = (int32_t)(node * d + j);
  }
}

// v[dof_pos[q]] -= alpha g[q]: one thread per free dof, g read coalesced
__global__ void k_descent(int64_t nfd, const int32_t *__restrict__ dof_pos,
                          const double *__restrict__ g, double alpha, double *__restrict__ v) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nfd;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = __ldg(dof_pos + q);
    v[i] = rsub(v[i], rmul(alpha, __ldg(g + q)));
  }
}

// ----------------------------------------------------------------- launchers
template <int DIM, int MODEL>
static cudaError_t energy_t(const TileArgs &aos, int64_t ne, int nblocks, const double *v,
                            double *part, double *dens, const ModelArgs &m, cudaStream_t s) {
  int64_t per = (ne + nblocks - 1) / nblocks;
  k_energy<DIM, MODEL><<<nblocks, 256, 0, s>>>(aos, ne, per, v, part, dens, m);
  return cudaGetLastError();
}

cudaError_t launch_energy(int dim, int model, const TileArgs &aos, int64_t ne, int nblocks,
                          const double *v, double *part, double *dens, const ModelArgs &m,
                          cudaStream_t s) {
  if (dim == 2 && model == FM_MODEL_PLAPLACE)
    return energy_t<2, FM_MODEL_PLAPLACE>(aos, ne, nblocks, v, part, dens, m, s);
  if (dim == 3 && model == FM_MODEL_PLAPLACE)
    return energy_t<3, FM_MODEL_PLAPLACE>(aos, ne, nblocks, v, part, dens, m, s);
  if (dim == 2) return energy_t<2, FM_MODEL_NEOHOOKEAN>(aos, ne, nblocks, v, part, dens, m, s);
  return energy_t<3, FM_MODEL_NEOHOOKEAN>(aos, ne, nblocks, v, part, dens, m, s);
}

cudaError_t launch_dot(const double *a, const double *b, int64_t n, int nblocks, double *part,
                       cudaStream_t s) {
  int64_t per = (n + nblocks - 1) / nblocks;
  k_dot<<<nblocks, 256, 0, s>>>(a, b, n, per, part);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const double *jp, int nj, const double *dp, int nd, double *out,
                            cudaStream_t s) {
  k_finalize<<<1, 1024, 0, s>>>(jp, nj, dp, nd, out);
  return cudaGetLastError();
}

template <int DIM, int MODEL, int CT>
static cudaError_t fd_t(const TileArgs &a, int n_tiles, int ech, const double *v, const double *b,
                        double eps, double *g, unsigned long long *badkey, const ModelArgs &m,
                        cudaStream_t s) {
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  const size_t smem = FdLayout<DIM, CT>::total(D, a.clo_cap, ech, a.blk_cap);
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

cudaError_t launch_dof_pos(int64_t nfree, int d, const int32_t *free_node, const int32_t *free_out,
                           const uint8_t *free_mask, int32_t *dof_pos, cudaStream_t s) {
  k_dof_pos<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, d, free_node, free_out, free_mask, dof_pos);
  return cudaGetLastError();
}

cudaError_t launch_descent(int64_t nfd, const int32_t *dof_pos, const double *g, double alpha,
                           double *v, cudaStream_t s) {
  k_descent<<<grid_for(nfd, 256), 256, 0, s>>>(nfd, dof_pos, g, alpha, v);
  return cudaGetLastError();
}

}  // namespace fm

// ----------------------------------------------------------------- row batches
// The model plugin surface (models.py:59-138) on flat (rows) batches:
// F is stored as D*DIM arrays of n rows (F[j][m] at (j*DIM+m)*n).
namespace fm {

template <int DIM, int MODEL>
__global__ void k_rows(int64_t n, const double *__restrict__ Fs, double *__restrict__ W,
                       double *__restrict__ P, unsigned long long *nbad, ModelArgs mdl) {
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  unsigned long long bad_local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double F[D][DIM];
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int m = 0; m < DIM; ++m) F[j][m] = Fs[(int64_t)(j * DIM + m) * n + i];
    if (W) W[i] = density<DIM, MODEL>(F, mdl);
    if (P) {
      double Q[D][DIM];
      bool bad;
      ddensity<DIM, MODEL>(F, mdl, Q, bad);
      bad_local += bad;
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int m = 0; m < DIM; ++m) P[(int64_t)(j * DIM + m) * n + i] = Q[j][m];
    }
  }
  if (bad_local) atomicAdd(nbad, bad_local);
}

template <int DIM>
__global__ void k_det_rows(int64_t n, const double *__restrict__ Fs, double *__restrict__ det,
                           double *__restrict__ cof) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double F[DIM][DIM];
#pragma unroll
    for (int j = 0; j < DIM; ++j)
#pragma unroll
      for (int m = 0; m < DIM; ++m) F[j][m] = Fs[(int64_t)(j * DIM + m) * n + i];
    if (det) det[i] = det_F<DIM>(F);
    if (cof) {
      double Cf[DIM][DIM];
      cof_F<DIM>(F, Cf);
#pragma unroll
      for (int j = 0; j < DIM; ++j)
#pragma unroll
        for (int m = 0; m < DIM; ++m) cof[(int64_t)(j * DIM + m) * n + i] = Cf[j][m];
    }
  }
}

// evaluate_F (assembly.py:35-49): vals D x (rows, NV), dphi DIM x (rows, NV) -> F (D*DIM, rows)
template <int DIM>
__global__ void k_eval_F(int64_t rows, int D, const double *__restrict__ vals,
                         const double *__restrict__ dphi, double *__restrict__ F) {
  constexpr int NV = DIM + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows;
    const int j = (int)(i / rows);
    double a[NV];
#pragma unroll
    for (int l = 0; l < NV; ++l) a[l] = vals[((int64_t)j * rows + r) * NV + l];
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      double g[NV];
#pragma unroll
      for (int l = 0; l < NV; ++l) g[l] = dphi[((int64_t)m * rows + r) * NV + l];
      F[((int64_t)j * DIM + m) * rows + r] = einsum_row<NV>(a, g);
    }
  }
}

// segment_sums (patches.py:80-83) as direct fixed-order sums per segment.
__global__ void k_segment_sums(int64_t nseg, const double *__restrict__ vals,
                               const int64_t *__restrict__ indx, double *__restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nseg;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = k ? indx[k - 1] : 0, z = indx[k];
    double s = 0.0;
    for (int64_t q = a; q < z; ++q) s += vals[q];
    out[k] = s;
  }
}

}  // namespace fm

using namespace fm;

static ModelArgs rows_model(const fm_model *m) {
  ModelArgs a;
  a.kind = m->kind;
  a.p = m->p;
  a.C1 = m->C1;
  a.D1 = m->D1;
  a.e_w = m->p / 2.0;
  a.e_dw = (m->p - 2.0) / 2.0;
  return a;
}

extern "C" int fm_density_rows(const fm_model *m, int64_t n, const double *F, double *W,
                               double *P, int64_t *nbad_host, void *stream) {
  FM_NVTX("fm_density_rows");
  FM_ARG(m && F, "null argument");
  FM_ARG(m->dim == 2 || m->dim == 3, "dim must be 2 or 3");
  FM_ARG(m->kind == FM_MODEL_PLAPLACE || m->kind == FM_MODEL_NEOHOOKEAN, "unknown model kind");
  cudaStream_t s = as_stream(stream);
  Scratch bad;
  FM_CUDA(bad.alloc(8, s));
  FM_CUDA(cudaMemsetAsync(bad.p, 0, 8, s));
  ModelArgs a = rows_model(m);
  unsigned g = grid_for(n, 256);
  auto *nb = bad.as<unsigned long long>();
  if (m->dim == 2 && m->kind == FM_MODEL_PLAPLACE)
    k_rows<2, FM_MODEL_PLAPLACE><<<g, 256, 0, s>>>(n, F, W, P, nb, a);
  else if (m->dim == 3 && m->kind == FM_MODEL_PLAPLACE)
    k_rows<3, FM_MODEL_PLAPLACE><<<g, 256, 0, s>>>(n, F, W, P, nb, a);
  else if (m->dim == 2)
    k_rows<2, FM_MODEL_NEOHOOKEAN><<<g, 256, 0, s>>>(n, F, W, P, nb, a);
  else
    k_rows<3, FM_MODEL_NEOHOOKEAN><<<g, 256, 0, s>>>(n, F, W, P, nb, a);
  FM_CHECK_LAUNCH();
  unsigned long long h = 0;
  FM_CUDA(cudaMemcpyAsync(&h, bad.p, 8, cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  if (nbad_host) *nbad_host = (int64_t)h;
  return FM_OK;
}

extern "C" int fm_det_rows(int dim, int64_t n, const double *F, double *det, double *cof,
                           void *stream) {
  FM_NVTX("fm_det_rows");
  FM_ARG(dim == 2 || dim == 3, "dim must be 2 or 3");
  cudaStream_t s = as_stream(stream);
  if (dim == 2)
    k_det_rows<2><<<grid_for(n, 256), 256, 0, s>>>(n, F, det, cof);
  else
    k_det_rows<3><<<grid_for(n, 256), 256, 0, s>>>(n, F, det, cof);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

extern "C" int fm_eval_F(int dim, int d, int64_t rows, const double *vals, const double *dphi,
                         double *F, void *stream) {
  FM_NVTX("fm_eval_F");
  FM_ARG(dim == 2 || dim == 3, "dim must be 2 or 3");
  cudaStream_t s = as_stream(stream);
  if (dim == 2)
    k_eval_F<2><<<grid_for(rows * d, 256), 256, 0, s>>>(rows, d, vals, dphi, F);
  else
    k_eval_F<3><<<grid_for(rows * d, 256), 256, 0, s>>>(rows, d, vals, dphi, F);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

extern "C" int fm_segment_sums(int64_t nseg, const double *vals, const int64_t *indx,
                               double *out, void *stream) {
  FM_NVTX("fm_segment_sums");
  cudaStream_t s = as_stream(stream);
  k_segment_sums<<<grid_for(nseg, 256), 256, 0, s>>>(nseg, vals, indx, out);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

// linear_term (assembly.py:89-91): out[0] = a.b with the fixed-order partials.
extern "C" int fm_dot(int64_t n, const double *a, const double *b, double *out, void *stream) {
  FM_NVTX("fm_dot");
  FM_ARG(a && b && out, "null argument");
  cudaStream_t s = as_stream(stream);
  const int nb = sm_count() * 2;
  Scratch part;
  FM_CUDA(part.alloc(nb * sizeof(double), s));
  FM_CUDA(launch_dot(a, b, n, nb, part.as<double>(), s));
  FM_CUDA(launch_finalize(part.as<double>(), nb, part.as<double>(), 0, out, s));
  return FM_OK;
}
