// Fused energy + exact gradient (gradients.py:124-149 with assembly.py:94-106)
// as one persistent, multistage-pipelined kernel per SM.
//
// One CTA (256 threads) per SM walks its node tiles (t = blockIdx.x,
// += gridDim.x; tiles are in Morton order of their spatial boxes so concurrently
// running CTAs share halo elements and nodal values through L2).  The tile
// element list is processed in chunks of 256 (thread c <-> element c of the
// chunk) through a ring of STAGES shared-memory stages, STAGES-1 chunks ahead:
//
//   records   the tile's own elements are a contiguous storage range -> TMA 2D
//             tensor loads of 8..256 records with SWIZZLE_128B (3D) or one 1D
//             bulk copy (2D), issued by thread 0 and completing on the stage's
//             mbarrier; halo records (and a < 8 remainder) -> each thread copies
//             its own record with 16-byte LDGSTS into the same swizzled layout.
//   values    one chunk ahead, each thread gathers the nodal values v[conn] of
//             its element with 8-byte LDGSTS into the stage's value buffer.
//   compute   F = grad v, P' = vol * dW/dF = a F + b cof, the contributions
//             P' . grad phi_l of the four local nodes overwrite the thread's own
//             value slots; vol * W when the tile owns the element.
//   assemble  after one barrier each node thread consumes this chunk's entries
//             (sorted by tile element) into registers: a fixed summation order,
//             no floating-point atomics.
// Node descriptors and entries of the next tile are bulk-copied into a second
// tile buffer while the current tile runs.
//
// J: per-thread partials over a static tile assignment -> fixed block tree ->
// one partial per CTA, reduced in CTA order by k_finalize.
#include "fm_density.cuh"
#include "fm_kernels.h"
#include "fm_pipe.cuh"

namespace fm {

template <int DIM>
struct PipeLayout {
  static constexpr int RS = RecBytes<DIM>::smem;
  __host__ __device__ static size_t rec_bytes() {
    return ((size_t)CONSUMERS * RS + 1023) / 1024 * 1024;
  }
  // nodal values [NV*D][CONSUMERS] f64, overwritten by the contributions
  __host__ __device__ static size_t val_bytes(int D) {
    return (((size_t)CONSUMERS * (DIM + 1) * D * 8) + 1023) / 1024 * 1024;
  }
  __host__ __device__ static size_t stage_bytes(int D) { return rec_bytes() + val_bytes(D); }
  // tile buffer: node desc (256 x 16) | entries
  __host__ __device__ static size_t entries_off() { return (size_t)CONSUMERS * 16; }
  __host__ __device__ static size_t tile_bytes(int entry_cap) {
    return entries_off() + (((size_t)entry_cap * 2 + 15) / 16) * 16;
  }
  // + 1024 for aligning the dynamic shared memory base
  __host__ __device__ static size_t total(int stages, int entry_cap, int D) {
    return 1024 + stages * stage_bytes(D) + 2 * tile_bytes(entry_cap) + 32 * 8 +
           (stages + 2) * 8;
  }
};

// NH: P' = vol * dW/dF = a F + b cof with a = 2 C1 vol, b = vol (2 D1 (det-1) - 2 C1/det)
// (models.py:103-120 regrouped).  p-Laplace: P' = vol |g|^(p-2) g.
template <int DIM, int MODEL>
__device__ __forceinline__ void element_P(const double (&F)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
                                          double vol, const ModelArgs &m, bool want_w,
                                          double (&P)[MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1][DIM],
                                          double &W, bool &bad) {
  if constexpr (MODEL == FM_MODEL_NEOHOOKEAN) {
    double C[DIM][DIM];
    cof_F<DIM>(F, C);
    double det = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) det = fma(F[0][k], C[0][k], det);
    bad = !(det > 0.0);
    const double rdet = 1.0 / det;
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
      W = bad ? INFINITY : m.C1 * ((I1 - (double)DIM) - 2.0 * log(det)) + m.D1 * (dm1 * dm1);
    }
  } else {
    bad = false;
    double n2 = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) n2 = fma(F[0][k], F[0][k], n2);
    double fac;
    if (m.p >= 2.0)
      fac = np_scalar_pow(n2, m.e_dw);
    else
      fac = n2 > 0.0 ? pow(n2, m.e_dw) : 0.0;
    fac *= vol;
#pragma unroll
    for (int k = 0; k < DIM; ++k) P[0][k] = fac * F[0][k];
    if (want_w) W = np_scalar_pow(n2, m.e_w) / m.p;
  }
}

// Position in this CTA's chunk stream: tile t (j-th of the CTA), chunk offset c0.
struct Cursor {
  int t, j, c0, ne;
  TileMeta tm;
  __device__ void load(const TileArgs &a) {
    if (t < a.n_tiles_all) {
      tm = a.meta[t];
      ne = tm.own_count + tm.halo_count;
    } else {
      ne = 0;
    }
  }
  __device__ bool valid(const TileArgs &a) const { return t < a.n_tiles_all; }
  __device__ void advance(const TileArgs &a) {
    c0 += CONSUMERS;
    if (c0 >= ne) {
      c0 = 0;
      t += gridDim.x;
      ++j;
      load(a);
    }
  }
};

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int DIM, int MODEL, bool WJ, int STAGES>
__global__ void __launch_bounds__(CONSUMERS, 1)
    k_tile_exact(const __grid_constant__ TmaMaps tma, TileArgs a, const double *__restrict__ v,
                 const double *__restrict__ b, double *__restrict__ g,
                 double *__restrict__ jpart, unsigned long long *status, ModelArgs mdl) {
  constexpr int NV = DIM + 1;
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  constexpr int RB = RecBytes<DIM>::value;  // bytes of one record (global)
  constexpr int NCH = RB / 16;               // 16-B chunks per record
  using L = PipeLayout<DIM>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align to 1024 B (TMA 128-byte swizzle atom) while staying derived from the
  // __shared__ symbol, so that all accesses compile to LDS/STS, not generic LD/ST
  unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const size_t SB = L::stage_bytes(D);
  unsigned char *stage_base = smem;
  unsigned char *tile_base = stage_base + STAGES * SB;
  const size_t TB = L::tile_bytes(a.entry_cap);
  double *red = reinterpret_cast<double *>(tile_base + 2 * TB);
  uint64_t *full = reinterpret_cast<uint64_t *>(red + 32);  // TMA / bulk part of a stage
  uint64_t *tfull = full + STAGES;                          // tile buffers
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(full + s, 1);
    mbar_init(tfull, 1);
    mbar_init(tfull + 1, 1);
    fence_barrier_init();
  }
  __syncthreads();

  // tile buffer j&1 <- node descriptors + entries of tile t (thread 0)
  auto issue_tile = [&](int t, int j) {
    if (tid == 0 && t < a.n_tiles_all) {
      const TileMeta tm = a.meta[t];
      unsigned char *tb = tile_base + (j & 1) * TB;
      const uint32_t nb = (uint32_t)tm.node_count * 16;
      const uint32_t eb = (uint32_t)((tm.entry_count * 2 + 15) / 16) * 16;
      mbar_arrive_expect_tx(tfull + (j & 1), nb + eb);
      if (nb) bulk_g2s(tb, a.node_desc + tm.node_begin, nb, tfull + (j & 1));
      if (eb) bulk_g2s(tb + L::entries_off(), a.entries + tm.entry_begin, eb, tfull + (j & 1));
    }
  };
  // records of the chunk at cursor x into stage s; src = this thread's record id
  auto issue_records = [&](const Cursor &x, int s, int src) {
    if (x.valid(a)) {
      unsigned char *dst = stage_base + s * SB;
      const int cnt = min(CONSUMERS, x.ne - x.c0);
      const int n_own = max(0, min(cnt, x.tm.own_count - x.c0));
      const int n_bulk = DIM == 3 ? (n_own & ~7) : n_own;
      if (tid == 0) {
        mbar_arrive_expect_tx(full + s, (uint32_t)n_bulk * RB);
        if constexpr (DIM == 3) {
          int off = 0;
#pragma unroll 1
          for (int k = 5; k >= 0; --k) {
            const int rows = 8 << k;
            if (n_bulk - off >= rows) {
              tma_load_2d(dst + off * 128, &tma.box[k], 0, x.tm.own_begin + x.c0 + off, full + s);
              off += rows;
            }
          }
        } else {
          if (n_bulk)
            bulk_g2s(dst, a.aos + (int64_t)(x.tm.own_begin + x.c0) * RB, (uint32_t)n_bulk * RB,
                     full + s);
        }
      }
      if (tid >= n_bulk && tid < cnt) {
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          cp_async16(dst + rec_chunk_off<DIM>(tid, c), a.aos + (int64_t)src * RB + c * 16);
      }
    }
    cp_commit();
  };
  // record id of this thread's row at cursor x (halo ids are read from global)
  auto src_of = [&](const Cursor &x) -> int {
    if (!x.valid(a)) return 0;
    const int e = x.c0 + tid;
    if (e >= x.ne) return 0;
    return e < x.tm.own_count ? x.tm.own_begin + e
                              : __ldg(a.halo_ids + x.tm.halo_begin + e - x.tm.own_count);
  };
  // nodal values of this thread's element at cursor x (stage s) -> value buffer
  auto issue_values = [&](const Cursor &x, int s, uint32_t qq) {
    if (x.valid(a)) {
      mbar_wait(full + s, (qq / STAGES) & 1);
      if (x.c0 + tid < x.ne) {
        const int4 cc = *reinterpret_cast<const int4 *>(stage_base + s * SB +
                                                        rec_chunk_off<DIM>(tid, 0));
        const int c[4] = {cc.x, cc.y, cc.z, cc.w};
        double *vb = reinterpret_cast<double *>(stage_base + s * SB + L::rec_bytes());
#pragma unroll
        for (int l = 0; l < NV; ++l) {
          const double *src = v + (int64_t)c[l] * D;
#pragma unroll
          for (int k = 0; k < D; ++k)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                             smem_u32(vb + (l * D + k) * CONSUMERS + tid)),
                         "l"(src + k)
                         : "memory");
        }
      }
    }
    cp_commit();
  };

  double jsum = 0.0;
  bool bad_any = false;
  // ---- prologue: records of chunks 0..STAGES-2, values of chunk 0, tile 0/1 buffers
  Cursor comp{(int)blockIdx.x, 0, 0, 0, TileMeta{}};
  comp.load(a);
  Cursor iss = comp;
  issue_tile(comp.t, 0);
  issue_tile(comp.t + gridDim.x, 1);
  int src_next = src_of(iss);
  for (int k = 0; k < STAGES - 1; ++k) {
    issue_records(iss, k, src_next);
    iss.advance(a);
    src_next = src_of(iss);
  }
  cp_wait<STAGES - 2>();  // records of chunk 0 (own LDGSTS group)
  issue_values(comp, 0, 0);

  uint32_t q = 0;
  while (comp.valid(a)) {
    // ---- tile start
    const int j = comp.j;
    const TileMeta tm = comp.tm;
    const unsigned char *tb = tile_base + (j & 1) * TB;
    mbar_wait(tfull + (j & 1), (j >> 1) & 1);
    const int4 *desc = reinterpret_cast<const int4 *>(tb);
    const uint16_t *ents = reinterpret_cast<const uint16_t *>(tb + L::entries_off());
    const bool has_nodes = tm.node_count > 0;
    const bool my_node = tid < tm.node_count;
    int cur = 0, end = 0, outw = 0;
    double bj[D], acc[D];
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = bj[k] = 0.0;
    if (my_node) {
      const int4 nd = desc[tid];
      cur = nd.x;
      end = nd.x + nd.y;
      outw = nd.w;
      if (b) {
#pragma unroll
        for (int k = 0; k < D; ++k) bj[k] = __ldg(b + (int64_t)nd.z * D + k);
      }
    }
    const int ne_t = comp.ne;
    for (int c0 = 0; c0 < ne_t; c0 += CONSUMERS, ++q) {
      const int s = q % STAGES;
      // 1. records of chunk q+STAGES-1 into the stage freed by chunk q-1
      issue_records(iss, (q + STAGES - 1) % STAGES, src_next);
      iss.advance(a);
      src_next = src_of(iss);
      // 2. values of chunk q+1 (its records: TMA mbarrier + own LDGSTS group)
      Cursor nx = comp;
      nx.advance(a);
      cp_wait<2 * STAGES - 4>();
      issue_values(nx, (q + 1) % STAGES, q + 1);
      // 3. compute chunk q (its values: the group committed one iteration ago)
      cp_wait<2>();
      const unsigned char *stage = stage_base + s * SB;
      double *vb = reinterpret_cast<double *>(stage_base + s * SB + L::rec_bytes());
      const int e = c0 + tid;
      if (e < ne_t) {
        const bool own = e < tm.own_count;
        Elem<DIM> E;
        load_elem_smem<DIM>(stage, tid, E);
        double vv[D][NV];
#pragma unroll
        for (int l = 0; l < NV; ++l)
#pragma unroll
          for (int k = 0; k < D; ++k) vv[k][l] = vb[(l * D + k) * CONSUMERS + tid];
        double F[D][DIM];
        grad_F<DIM, D>(vv, E.g, F);
        if (has_nodes) {
          double P[D][DIM], W = 0.0;
          bool bad;
          element_P<DIM, MODEL>(F, E.vol, mdl, WJ && own, P, W, bad);
          bad_any |= bad;
          if (WJ && own) jsum += E.vol * W;
#pragma unroll
          for (int l = 0; l < NV; ++l)
#pragma unroll
            for (int k = 0; k < D; ++k) {
              double sdot = P[k][0] * E.g[0][l];
#pragma unroll
              for (int m = 1; m < DIM; ++m) sdot = fma(P[k][m], E.g[m][l], sdot);
              vb[(l * D + k) * CONSUMERS + tid] = sdot;  // own slots: [slot][comp][thread]
            }
        } else if (WJ) {
          jsum += E.vol * density<DIM, MODEL>(F, mdl);
        }
      }
      __syncthreads();  // contributions staged
      // 4. assemble: node threads consume this chunk's entries
      if (my_node) {
        const int lim = c0 + CONSUMERS;
        while (cur < end) {
          const int en = ents[cur];
          const int te = en >> 2;
          if (te >= lim) break;
          const double *src = vb + (te - c0) + (en & 3) * D * CONSUMERS;
#pragma unroll
          for (int k = 0; k < D; ++k) acc[k] += src[k * CONSUMERS];
          ++cur;
        }
      }
      __syncthreads();  // stage s free for chunk q+STAGES
      comp.advance(a);
    }
    if (my_node) {
      const int mask = (unsigned)outw >> OUT_MASK_SHIFT;
      int o = outw & ((1 << OUT_MASK_SHIFT) - 1);
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (mask & (1 << k)) g[o++] = acc[k] - bj[k];
    }
    // tile buffer j&1 is free (last barrier above): prefetch tile j+2 into it
    issue_tile(comp.t + gridDim.x, j + 2);
  }
  cp_wait<0>();
  if (bad_any) atomicOr(status, 1ull);
  if (WJ) {
    double r = block_sum(jsum, red);
    if (tid == 0) jpart[blockIdx.x] = r;
  }
}

template <int DIM, int MODEL>
static cudaError_t launch_exact_t(const TmaMaps &tma, const TileArgs &a, int grid, int stages,
                                  bool wj, const double *v, const double *b, double *g,
                                  double *jpart, unsigned long long *status, const ModelArgs &m,
                                  cudaStream_t s) {
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  const size_t smem = PipeLayout<DIM>::total(stages, a.entry_cap, D);
#define FM_LAUNCH(WJV, ST)                                                            \
  do {                                                                                \
    auto k = k_tile_exact<DIM, MODEL, WJV, ST>;                                       \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    k<<<grid, CONSUMERS, smem, s>>>(tma, a, v, b, g, jpart, status, m);               \
  } while (0)
  // the cp.async group accounting of the kernel (wait_group 2*STAGES-4) holds
  // for STAGES = 2 and 3
  if (stages == 3) {
    if (wj) FM_LAUNCH(true, 3); else FM_LAUNCH(false, 3);
  } else {
    if (wj) FM_LAUNCH(true, 2); else FM_LAUNCH(false, 2);
  }
#undef FM_LAUNCH
  return cudaGetLastError();
}

size_t tile_exact_smem(int dim, int d, int stages, int entry_cap, int halo_cap) {
  (void)halo_cap;
  return dim == 3 ? PipeLayout<3>::total(stages, entry_cap, d)
                  : PipeLayout<2>::total(stages, entry_cap, d);
}

cudaError_t launch_tile_exact(int dim, int model, const TmaMaps &tma, const TileArgs &a,
                              int grid, int stages, bool wj, const double *v, const double *b,
                              double *g, double *jpart, unsigned long long *status,
                              const ModelArgs &m, cudaStream_t s) {
  if (dim == 2 && model == FM_MODEL_PLAPLACE)
    return launch_exact_t<2, FM_MODEL_PLAPLACE>(tma, a, grid, stages, wj, v, b, g, jpart, status,
                                                m, s);
  if (dim == 3 && model == FM_MODEL_PLAPLACE)
    return launch_exact_t<3, FM_MODEL_PLAPLACE>(tma, a, grid, stages, wj, v, b, g, jpart, status,
                                                m, s);
  if (dim == 2)
    return launch_exact_t<2, FM_MODEL_NEOHOOKEAN>(tma, a, grid, stages, wj, v, b, g, jpart,
                                                  status, m, s);
  return launch_exact_t<3, FM_MODEL_NEOHOOKEAN>(tma, a, grid, stages, wj, v, b, g, jpart, status,
                                                m, s);
}

}  // namespace fm
