// Fused energy + exact gradient (gradients.py:124-149 with assembly.py:94-106)
// as one persistent, warp-specialised, mbarrier-pipelined kernel.
//
// One CTA per SM walks its node tiles (t = blockIdx.x, += gridDim.x; tiles are
// in Morton order of their spatial boxes so concurrently running CTAs share
// halo elements and nodal values through L2).  Per chunk of 256 tile elements
// a ring stage holds the element records and the gathered nodal values:
//
//   record producer  the tile's own elements are a contiguous storage range ->
//   (warp 8)         TMA 2D tensor loads (boxes of 8..256 records, SWIZZLE_128B)
//                    in 3D / one 1D bulk copy in 2D; halo records and the < 8
//                    remainder -> 16-byte LDGSTS by the 32 lanes into the same
//                    layout.  Per tile: node descriptors, node entries and halo
//                    ids -> double-buffered tile area (bulk copies).
//   8 consumer       thread c: gathers the nodal values of its element of the
//   warps            NEXT chunk into the stage's value buffer (8-byte LDGSTS,
//                    one commit group per chunk), then computes element c of
//                    this chunk from shared memory:
//                    F = grad v, P' = vol * dW/dF = a F + b cof, contributions
//                    P' . grad phi_l of the four local nodes, written over the
//                    (consumed) value buffer; vol * W when the tile owns the
//                    element.  Then as node threads they consume this chunk's
//                    entries (sorted by tile element) into registers: fixed
//                    summation order, no floating-point atomics.
//
// J: per-thread partials over a static tile assignment -> fixed block tree ->
// one partial per CTA, reduced in CTA order by k_finalize.
#include "fm_density.cuh"
#include "fm_kernels.h"
#include "fm_pipe.cuh"

namespace fm {

constexpr int PRODUCER_WARPS = 1;

template <int DIM>
struct PipeLayout {
  static constexpr int RS = RecBytes<DIM>::smem;
  __host__ __device__ static size_t rec_bytes() {
    return ((size_t)CONSUMERS * RS + 1023) / 1024 * 1024;
  }
  // nodal values [NV*D][CONSUMERS] f64, reused as the contribution staging
  __host__ __device__ static size_t val_bytes(int D) {
    return (((size_t)CONSUMERS * (DIM + 1) * D * 8) + 1023) / 1024 * 1024;
  }
  __host__ __device__ static size_t stage_bytes(int D) { return rec_bytes() + val_bytes(D); }
  // tile buffer: meta (64) | node desc (256 x 16) | entries | halo ids
  __host__ __device__ static size_t entries_off() { return 64 + (size_t)CONSUMERS * 16; }
  __host__ __device__ static size_t halo_off(int entry_cap) {
    return entries_off() + (((size_t)entry_cap * 2 + 15) / 16) * 16;
  }
  __host__ __device__ static size_t tile_bytes(int entry_cap, int halo_cap) {
    return halo_off(entry_cap) + (((size_t)halo_cap * 4 + 15) / 16) * 16;
  }
  // + 1024 for aligning the dynamic shared memory base
  __host__ __device__ static size_t total(int stages, int entry_cap, int halo_cap, int D) {
    return 1024 + stages * stage_bytes(D) + 2 * tile_bytes(entry_cap, halo_cap) + 32 * 8 +
           (3 * stages + 4) * 8;
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

template <int DIM, int MODEL, bool WJ, int STAGES>
__global__ void __launch_bounds__(CONSUMERS + 32 * PRODUCER_WARPS, 1)
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
  const size_t TB = L::tile_bytes(a.entry_cap, a.halo_cap);
  const size_t HO = L::halo_off(a.entry_cap);
  double *red = reinterpret_cast<double *>(tile_base + 2 * TB);
  uint64_t *full = reinterpret_cast<uint64_t *>(red + 32);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint64_t *tempty = tfull + 2;
  constexpr int CW = CONSUMERS / 32;  // consumer warps

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1 + 32);  // expect_tx arrival + one LDGSTS arrival per producer lane
      mbar_init(empty + s, CW);     // one arrival per consumer warp
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull + s, 1);
      mbar_init(tempty + s, 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  double jsum = 0.0;
  if (warp == CW) {
    // ------------------------------------------------------- record producer
    uint32_t q = 0, j = 0;
    for (int t = blockIdx.x; t < a.n_tiles_all; t += gridDim.x, ++j) {
      const TileMeta tm = a.meta[t];
      unsigned char *tb = tile_base + (j & 1) * TB;
      mbar_wait(tempty + (j & 1), ((j >> 1) & 1) ^ 1);
      const int32_t *halo_s = reinterpret_cast<const int32_t *>(tb + HO);
      if (lane == 0) {
        *reinterpret_cast<TileMeta *>(tb) = tm;
        const uint32_t nb = (uint32_t)tm.node_count * 16;
        const uint32_t eb = (uint32_t)((tm.entry_count * 2 + 15) / 16) * 16;
        const uint32_t hb = (uint32_t)((tm.halo_count * 4 + 15) / 16) * 16;
        mbar_arrive_expect_tx(tfull + (j & 1), nb + eb + hb);
        if (nb) bulk_g2s(tb + 64, a.node_desc + tm.node_begin, nb, tfull + (j & 1));
        if (eb) bulk_g2s(tb + L::entries_off(), a.entries + tm.entry_begin, eb, tfull + (j & 1));
        if (hb) bulk_g2s(tb + HO, a.halo_ids + tm.halo_begin, hb, tfull + (j & 1));
      }
      __syncwarp();
      bool halo_ready = false;
      const int ne_t = tm.own_count + tm.halo_count;
      for (int c0 = 0; c0 < ne_t; c0 += CONSUMERS, ++q) {
        const int s = q % STAGES;
        const int cnt = min(CONSUMERS, ne_t - c0);
        const int n_own = max(0, min(cnt, tm.own_count - c0));
        // 3D: TMA boxes cover the 8-aligned part of the own range; 2D: one bulk copy
        const int n_bulk = DIM == 3 ? (n_own & ~7) : n_own;
        if (!halo_ready && cnt > n_bulk && c0 + cnt > tm.own_count) {
          mbar_wait(tfull + (j & 1), (j >> 1) & 1);  // halo ids arrive with the tile buffer
          halo_ready = true;
        }
        mbar_wait(empty + s, ((q / STAGES) & 1) ^ 1);
        unsigned char *dst = stage_base + s * SB;
        if (lane == 0) {
          mbar_arrive_expect_tx(full + s, (uint32_t)n_bulk * RB);
          if constexpr (DIM == 3) {
            int off = 0;
#pragma unroll 1
            for (int k = 5; k >= 0; --k) {
              const int rows = 8 << k;
              if (n_bulk - off >= rows) {
                tma_load_2d(dst + off * 128, &tma.box[k], 0, tm.own_begin + c0 + off, full + s);
                off += rows;
              }
            }
          } else {
            if (n_bulk)
              bulk_g2s(dst, a.aos + (int64_t)(tm.own_begin + c0) * RB, (uint32_t)n_bulk * RB,
                       full + s);
          }
        }
        // remaining records of the chunk: 16-byte LDGSTS, lane-parallel
        for (int idx = lane; idx < (cnt - n_bulk) * NCH; idx += 32) {
          const int r = n_bulk + idx / NCH, c = idx % NCH;
          const int e = c0 + r;
          const int src = e < tm.own_count ? tm.own_begin + e : halo_s[e - tm.own_count];
          cp_async16(dst + rec_chunk_off<DIM>(r, c), a.aos + (int64_t)src * RB + c * 16);
        }
        cp_async_arrive_noinc(full + s);
      }
    }
  } else {
    // ------------------------------------------------------------- consumers
    // Flat stream over (tile, chunk).  Per chunk q: the nodal values of chunk
    // q+1 are gathered by each consumer thread for its own element with 8-byte
    // LDGSTS into the stage's value buffer (one commit group per chunk), so
    // they land while chunk q is computed; the thread then overwrites its own
    // value slots with its contributions (no barrier needed for that).
    bool bad_any = false;
    int t = blockIdx.x;
    uint32_t q = 0, j = 0;
    auto issue_values = [&](uint32_t qq, int c0, int ne) {
      const int s = qq % STAGES;
      mbar_wait(full + s, (qq / STAGES) & 1);
      if (c0 + tid < ne) {
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
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (t < a.n_tiles_all) {
      TileMeta tm = a.meta[t];
      issue_values(0, 0, tm.own_count + tm.halo_count);
      while (true) {
        // ---- tile start
        unsigned char *tb = tile_base + (j & 1) * TB;
        mbar_wait(tfull + (j & 1), (j >> 1) & 1);
        const int4 *desc = reinterpret_cast<const int4 *>(tb + 64);
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
        const int ne_t = tm.own_count + tm.halo_count;
        const int tn = t + gridDim.x;
        const TileMeta tmn = tn < a.n_tiles_all ? a.meta[tn] : TileMeta{};
        for (int c0 = 0; c0 < ne_t; c0 += CONSUMERS, ++q) {
          const int s = q % STAGES;
          const unsigned char *stage = stage_base + s * SB;
          double *vb = reinterpret_cast<double *>(stage_base + s * SB + L::rec_bytes());
          // prefetch the nodal values of the next chunk (this tile or the next one)
          if (c0 + CONSUMERS < ne_t)
            issue_values(q + 1, c0 + CONSUMERS, ne_t);
          else if (tn < a.n_tiles_all)
            issue_values(q + 1, 0, tmn.own_count + tmn.halo_count);
          else
            asm volatile("cp.async.commit_group;" ::: "memory");
          asm volatile("cp.async.wait_group 1;" ::: "memory");  // this chunk's values landed
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
          named_sync(1, CONSUMERS);  // contributions staged
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
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + s);  // this warp is done with the stage
        }
        if (my_node) {
          const int mask = (unsigned)outw >> OUT_MASK_SHIFT;
          int o = outw & ((1 << OUT_MASK_SHIFT) - 1);
#pragma unroll
          for (int k = 0; k < D; ++k)
            if (mask & (1 << k)) g[o++] = acc[k] - bj[k];
        }
        named_sync(1, CONSUMERS);  // all node threads done with the tile buffer
        if (tid == 0) mbar_arrive(tempty + (j & 1));
        ++j;
        t = tn;
        if (t >= a.n_tiles_all) break;
        tm = tmn;
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (bad_any) atomicOr(status, 1ull);
  }
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
  const size_t smem = PipeLayout<DIM>::total(stages, a.entry_cap, a.halo_cap, D);
  const int threads = CONSUMERS + 32 * PRODUCER_WARPS;
#define FM_LAUNCH(WJV, ST)                                                            \
  do {                                                                                \
    auto k = k_tile_exact<DIM, MODEL, WJV, ST>;                                       \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    k<<<grid, threads, smem, s>>>(tma, a, v, b, g, jpart, status, m);                 \
  } while (0)
  if (stages == 3) {
    if (wj) FM_LAUNCH(true, 3); else FM_LAUNCH(false, 3);
  } else if (stages == 2) {
    if (wj) FM_LAUNCH(true, 2); else FM_LAUNCH(false, 2);
  } else {
    if (wj) FM_LAUNCH(true, 4); else FM_LAUNCH(false, 4);
  }
#undef FM_LAUNCH
  return cudaGetLastError();
}

size_t tile_exact_smem(int dim, int d, int stages, int entry_cap, int halo_cap) {
  return dim == 3 ? PipeLayout<3>::total(stages, entry_cap, halo_cap, d)
                  : PipeLayout<2>::total(stages, entry_cap, halo_cap, d);
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
