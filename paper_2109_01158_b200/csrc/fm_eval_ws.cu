// Fused energy + exact gradient (gradients.py:124-149 with assembly.py:94-106),
// warp-specialised: ONE 800-thread CTA per SM, its warps split by role with
// their register budgets re-balanced (setmaxnreg):
//
//   node group    warps 0-7 (256 threads, 48 registers): one thread per tile
//                 node.  Per chunk it adds the node's entries from the staged
//                 contributions (fixed order) and stores the cross items to the
//                 exchange buffer; at the tile end the outputs and b.v.
//   element       warps 8-15 and 16-23 (2 x 256 threads, 96 registers): group
//   groups        gi takes the chunks q = gi (mod 2) of the CTA's chunk
//                 stream: F = grad v, P' = vol dW/dF, the contributions into
//                 the group's own staging buffer.
//   producer      warp 24: walks the CTA's tiles and chunks ahead of the
//                 others and requests everything they read from shared
//                 memory: per tile the tables (descriptors, exchange chunk
//                 starts: bulk copies), the closure ids and the gather of the
//                 closure's node values (8-byte LDGSTS by its 32 lanes); per
//                 chunk the records, closure indices and entry block (bulk
//                 copies, 4 record stages / 8 entry slots, four chunks ahead)
//                 and a chunk descriptor.  Only this warp waits on global
//                 memory latency (tile metadata).
//
// The element math, the staging layout, the per-node summation order, the
// exchange items and the outputs are k_tile_exact's (fm_eval_exact.cu): the
// gradient is bitwise the same; J's per-CTA partials are summed over another
// static assignment (one partial per CTA, reduced in CTA order by
// k_finish_cross as before).
//
// Hand-offs (mbarriers unless noted): full[s] records + closure indices +
// entry block + descriptor of chunk q in stage q & 3 / slot q & 7 (complete_tx);
// empty[s] the element threads have their records in registers; nfull[k] /
// tfull[k] node values / tables of tile j in buffer j % NBUF; tdone[k] the node
// group is done with tile j (its buffers may be refilled); named barriers
// STAGED + gi (element group arrives, node group waits) and FREE + gi (node
// group arrives, element group waits before it overwrites its staging buffer).
#include "fm_elem.cuh"
#include "fm_kernels.h"
#include "fm_pipe.cuh"

#if FM_WS_KERNEL  // experiment builds only (tools/ws_check.sh); the product library skips this unit

// Phase accounting for profiling builds only (-DFM_WS_TRACE=1, a separate
// library built by tools/ws_trace.py): per warp of CTAs 0..3 the clock64 cycles
// spent in each phase of its role, summed over the launch.
#ifndef FM_WS_TRACE
#define FM_WS_TRACE 0
#endif
#if FM_WS_TRACE
constexpr int WT_CTAS = 4, WT_WARPS = 25, WT_PH = 8;
__device__ long long g_wstrace[WT_CTAS * WT_WARPS * WT_PH];
extern "C" int fm_ws_trace_copy(long long *out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_wstrace, (size_t)n * sizeof(long long));
}
#define WT_DECL long long wt_acc[WT_PH] = {0, 0, 0, 0, 0, 0, 0, 0}, wt_last = clock64()
#define WT(k)                            \
  do {                                   \
    const long long wt_now = clock64();  \
    wt_acc[k] += wt_now - wt_last;       \
    wt_last = wt_now;                    \
  } while (0)
#define WT_FLUSH                                                                          \
  do {                                                                                    \
    if (blockIdx.x < WT_CTAS && (threadIdx.x & 31) == 0)                                  \
      for (int k = 0; k < WT_PH; ++k)                                                     \
        g_wstrace[(blockIdx.x * WT_WARPS + (threadIdx.x >> 5)) * WT_PH + k] = wt_acc[k]; \
  } while (0)
#else
#define WT_DECL \
  do {          \
  } while (0)
#define WT(k) \
  do {        \
  } while (0)
#define WT_FLUSH \
  do {           \
  } while (0)
#endif

namespace fm {

namespace {

constexpr int WS_CT = 256;       // chunk size = max tile nodes = threads per group
#ifndef WS_PRODUCER_WARPS
#define WS_PRODUCER_WARPS 4  // a whole warpgroup (setmaxnreg is warpgroup-aligned)
#endif
#ifndef WS_SETMAXNREG
#define WS_SETMAXNREG 1
#endif
constexpr int WS_THREADS = 768 + 32 * WS_PRODUCER_WARPS;  // node group + 2 element groups + producer
constexpr int WS_RSTAGES = 4;    // record stages
constexpr int WS_ESLOTS = 8;     // entry-block slots (a chunk's block lives until its node sums)
constexpr int BAR_STAGED = 1, BAR_FREE = 3;

__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// per-tile values the producer leaves with the tables
struct WsTileMeta {
  int node_count, own_count, node_begin, is_node_tile;
};

template <int DIM, int NBUF>
struct WsLayout {
  using L = PipeLayout<DIM, WS_CT>;
  __host__ __device__ static size_t rstage() { return L::blk_off(); }  // records | closure indices
  __host__ __device__ static size_t eslot(int blk_cap) { return r16((size_t)blk_cap * 2); }
  __host__ __device__ static size_t tabs() { return L::tabs() + 16; }  // + WsTileMeta
  __host__ __device__ static size_t total(int D, int blk_cap, int clo_cap) {
    return WS_RSTAGES * rstage() + WS_ESLOTS * eslot(blk_cap) + NBUF * L::nodev(D, clo_cap) +
           2 * L::cids(clo_cap) + NBUF * tabs() + 2 * L::staging(D) +
           (size_t)D * WS_CT * 8 /* load values of the tile nodes */ +
           WS_ESLOTS * 16 /* chunk descriptors */ + 32 * 8 + 32 * 8 +
           4 * sizeof(TileMeta);
  }
};

}  // namespace

template <int DIM, int MODEL, bool WJ, int NBUF>
__global__ void __launch_bounds__(WS_THREADS, 1)
    k_tile_ws(TileArgs a, const double *__restrict__ v, const double *__restrict__ b,
              double *__restrict__ g, double *__restrict__ jpart, double *__restrict__ bvpart,
              unsigned long long *status, ModelArgs mdl) {
  constexpr int CT = WS_CT;
  constexpr int NV = DIM + 1;
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  constexpr int RB = RecBytes<DIM>::value;
  using L = PipeLayout<DIM, CT>;
  using W = WsLayout<DIM, NBUF>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int CAP = a.clo_cap;
  const size_t RS = W::rstage(), ES = W::eslot(a.blk_cap), NVB = L::nodev(D, CAP);
  unsigned char *eslots = smem + WS_RSTAGES * RS;
  unsigned char *nodev0 = eslots + WS_ESLOTS * ES;
  auto nodev = [&](int k) { return reinterpret_cast<double *>(nodev0 + k * NVB); };
  unsigned char *cids0 = nodev0 + NBUF * NVB;
  unsigned char *tabs0 = cids0 + 2 * L::cids(CAP);
  unsigned char *stage0 = tabs0 + NBUF * W::tabs();
  double *bsm = reinterpret_cast<double *>(stage0 + 2 * L::staging(D));
  int4 *cdesc = reinterpret_cast<int4 *>(bsm + D * CT);  // {count, first-row parity, tile seq, has nodes}
  double *red = reinterpret_cast<double *>(cdesc + WS_ESLOTS);
  uint64_t *full = reinterpret_cast<uint64_t *>(red + 32);  // record stages (x 4)
  uint64_t *empty = full + WS_RSTAGES;                      // (x 4)
  uint64_t *nfull = empty + WS_RSTAGES;                     // node-value buffers (x NBUF)
  uint64_t *tfull = nfull + NBUF;                           // tables (x NBUF)
  uint64_t *tdone = tfull + NBUF;                           // (x NBUF)
  uint64_t *cfull = tdone + NBUF;                           // closure ids (x 2)
  TileMeta *metas = reinterpret_cast<TileMeta *>(full + 32);  // producer warps: 2 x 2 tiles
  constexpr int CS = L::AOS(D) ? 1 : CT;
  const int SST = (int)L::slot_stride(D);
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < WS_RSTAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CT);
    }
    for (int k = 0; k < NBUF; ++k) {
      mbar_init(nfull + k, 32);
      mbar_init(tfull + k, 1);
      mbar_init(tdone + k, CT);
    }
    mbar_init(cfull, 1);
    mbar_init(cfull + 1, 1);
    fence_barrier_init();
  }
  __syncthreads();

  double jsum = 0.0, bvsum = 0.0;
  bool bad_any = false;

  if (tid >= 3 * CT) {
    // ================= producer warpgroup =================
    // warp 24 requests the chunks, warp 25 prepares the tiles; warps 26 / 27
    // only lend their registers.  Each working warp keeps the metadata of its
    // current and next tile in shared memory (LDGSTS a tile ahead: no register
    // copies, no exposed load latency).
#if WS_SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;");
#endif
    const int lane = tid & 31;
    const int pw = (tid - 3 * CT) >> 5;
    if (pw < 2) {
      TileMeta *ring = metas + 2 * pw;
      auto fetch_meta = [&](int t, int k) {  // meta[t] -> ring[k] (one commit group)
        if (lane < 4 && t < a.n_tiles_all)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(
                           reinterpret_cast<unsigned char *>(ring + k) + lane * 16)),
                       "l"(reinterpret_cast<const unsigned char *>(a.meta + t) + lane * 16)
                       : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      int t = blockIdx.x;
      fetch_meta(t, 0);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      if (pw == 0) {
        // ---- chunk requests: records, closure indices, entry block, descriptor
        uint32_t q = 0, j = 0;
        for (; t < a.n_tiles_all; t += G, ++j) {
          fetch_meta(t + G, (j + 1) & 1);
          const TileMeta *m = ring + (j & 1);
          const int oc = m->own_count;
          for (int c0 = 0; c0 < oc; c0 += CT, ++q) {
            const int s = q & 3;
            if (q >= WS_RSTAGES) mbar_wait(empty + s, ((q >> 2) - 1) & 1);
            if (lane == 0) {
              const int cnt = min(CT, oc - c0);
              const int64_t r0 = (int64_t)m->own_begin + c0;
              const int64_t l0 = r0 & ~1ll;
              const uint32_t nl = (uint32_t)((cnt + (r0 - l0) + 1) & ~1);
              const uint32_t bb = (uint32_t)m->blk_stride * 2;
              cdesc[q & 7] = make_int4(cnt, (int)(r0 & 1), (int)j, m->node_count > 0);
              unsigned char *st = smem + s * RS;
              mbar_arrive_expect_tx(full + s, (uint32_t)cnt * RB + nl * 8 + bb);
              bulk_g2s(st, a.aos + r0 * RB, (uint32_t)cnt * RB, full + s);
              bulk_g2s(st + L::loc_off(), a.loc + l0, nl * 8, full + s);
              if (bb)
                bulk_g2s(eslots + (q & 7) * ES,
                         a.chunk_blocks + m->blk_base + (int64_t)(c0 / CT) * m->blk_stride, bb,
                         full + s);
            }
          }
          asm volatile("cp.async.wait_group 0;" ::: "memory");
          __syncwarp();
        }
        // end of the stream: an empty descriptor for each element group
        for (int k = 0; k < 2; ++k, ++q) {
          const int s = q & 3;
          if (q >= WS_RSTAGES) mbar_wait(empty + s, ((q >> 2) - 1) & 1);
          if (lane == 0) {
            cdesc[q & 7] = make_int4(0, 0, 0, 0);
            mbar_arrive(full + s);
          }
        }
      } else {
        // ---- tile preparation: tables, closure ids, node values
        auto cids = [&](int k) { return reinterpret_cast<int32_t *>(cids0 + k * L::cids(CAP)); };
        auto issue_clo = [&](const TileMeta *m, int k) {
          if (lane == 0) {
            const uint32_t bytes = (uint32_t)r16((size_t)m->clo_count * 4);
            mbar_arrive_expect_tx(cfull + k, bytes);
            bulk_g2s(cids(k), a.closure + m->clo_begin, bytes, cfull + k);
          }
        };
        uint32_t j = 0, jb = 0, ju = 0;  // tile sequence number, j % NBUF, j / NBUF
        issue_clo(ring, 0);
        for (; t < a.n_tiles_all; t += G, ++j) {
          fetch_meta(t + G, (j + 1) & 1);
          const TileMeta *m = ring + (j & 1);
          // buffers jb were tile j - NBUF's: the node group is done with it
          if (ju > 0) mbar_wait(tdone + jb, (ju - 1) & 1);
          unsigned char *tb = tabs0 + jb * W::tabs();
          if (lane == 0) {
            const int nc = m->node_count;
            *reinterpret_cast<WsTileMeta *>(tb + L::tabs()) =
                WsTileMeta{nc, m->own_count, m->node_begin, t < a.n_tiles ? 1 : 0};
            const uint32_t nb = (uint32_t)nc * 16;
            const uint32_t xb_ = t < a.n_tiles ? XCH_STRIDE * 4 : 0;
            mbar_arrive_expect_tx(tfull + jb, nb + xb_);
            if (nb) bulk_g2s(tb, a.node_desc + m->node_begin, nb, tfull + jb);
            if (xb_)
              bulk_g2s(tb + (size_t)CT * 16, a.xchunk + (int64_t)t * XCH_STRIDE, xb_, tfull + jb);
          }
          // node values of the tile's closure -> buffer jb
          mbar_wait(cfull + (j & 1), (j >> 1) & 1);
          {
            const int32_t *ci = cids(j & 1);
            double *dst = nodev(jb);
            const int nclo = m->clo_count;
            for (int i = lane; i < nclo; i += 32) {
              const int64_t off = (int64_t)ci[i] * D;
#pragma unroll
              for (int kk = 0; kk < D; ++kk)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                                 smem_u32(dst + kk * CAP + i)),
                             "l"(v + off + kk)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            cp_async_arrive_noinc(nfull + jb);
          }
          // the next tile's metadata has landed (the gather may still be in
          // flight); the other ids buffer was tile j - 1's, read a tile ago
          asm volatile("cp.async.wait_group 1;" ::: "memory");
          fence_proxy_async();
          __syncwarp();
          if (t + G < a.n_tiles_all) issue_clo(ring + ((j + 1) & 1), (j + 1) & 1);
          if (++jb == NBUF) {
            jb = 0;
            ++ju;
          }
        }
      }
    }
  } else if (tid >= CT) {
    // ================= element groups =================
#if WS_SETMAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 96;");
#endif
    const int gi = (tid >> 8) - 1;     // 0 / 1
    const int gt = tid & (CT - 1);     // thread in the group = row of the chunk
    double *stage_d = reinterpret_cast<double *>(stage0 + gi * L::staging(D));
    auto st_at = [&](int slot, int row) -> double * {
      return L::AOS(D) ? stage_d + slot * SST + row * D : stage_d + row + slot * SST;
    };
    uint32_t jn = 0, jnb = 0, jnu = 0;  // next tile whose node values have not been awaited
    WT_DECL;
    uint32_t q = gi;
    for (;; q += 2) {
      const int s = q & 3;
      WT(0);
      mbar_wait(full + s, (q >> 2) & 1);
      WT(2);  // record wait
      const int4 cd = cdesc[q & 7];
      if (cd.x == 0) break;
      const unsigned char *st = smem + s * RS;
      const bool valid = gt < cd.x;
      Elem<DIM> E;
      if (valid) {
        load_elem_smem<DIM>(st, gt, E);
        decode_loc(*reinterpret_cast<const uint2 *>(st + L::loc_off() + (gt + cd.y) * 8), E.loc);
      }
      mbar_arrive(empty + s);  // this thread's record is in registers
      WT(3);                   // record loads
      // node values of every tile up to this chunk's, in order (no skipped phase)
      int nb_cur = 0;
      while (jn <= (uint32_t)cd.z) {
        mbar_wait(nfull + jnb, jnu & 1);
        nb_cur = jnb;
        ++jn;
        if (++jnb == NBUF) {
          jnb = 0;
          ++jnu;
        }
      }
      if (jn > 0) nb_cur = (int)((jn - 1) % NBUF);
      const double *nv = nodev(nb_cur);
      WT(1);  // node-value wait
      const bool has_nodes = cd.w != 0;
      double P[D][DIM];
      double Wel = 0.0, det_el = 1.0, ls_el = 0.0;
      bool far = false;
      if (valid) {
        double vv[D][NV];
#pragma unroll
        for (int l = 0; l < NV; ++l)
#pragma unroll
          for (int k = 0; k < D; ++k) vv[k][l] = nv[k * CAP + E.loc[l]];
        double F[D][DIM];
        grad_F_fma<DIM, D>(vv, E.g, F);
        if (has_nodes) {
          bool bad;
          element_P_f<DIM, MODEL, D>(
              F,
              [&](double (&o)[D][NV]) {  // rare: re-read from shared memory
#pragma unroll
                for (int l = 0; l < NV; ++l)
#pragma unroll
                  for (int k = 0; k < D; ++k) o[k][l] = nv[k * CAP + E.loc[l]];
              },
              E.g, E.vol, mdl, WJ, P, Wel, bad, far, det_el, ls_el);
          bad_any |= bad;
        } else if (WJ) {
          jsum += E.vol * density<DIM, MODEL>(F, mdl);
        }
      }
      WT(5);  // element math
      // the node group is done with this buffer's previous chunk (q - 2)
      if (q >= 2) bar_sync(BAR_FREE + gi, 2 * CT);
      WT(6);  // staging-buffer wait
      if (valid && has_nodes) {
#pragma unroll
        for (int l = 0; l < NV; ++l)
#pragma unroll
          for (int k = 0; k < D; ++k) {
            double sdot = P[k][0] * E.g[0][l];
#pragma unroll
            for (int m = 1; m < DIM; ++m) sdot = fma(P[k][m], E.g[m][l], sdot);
            st_at(l, gt)[k * CS] = sdot;
          }
        if (WJ) {
          if (far) Wel += 2.0 * mdl.C1 * (ls_el - log(det_el));
          jsum += E.vol * Wel;
        }
      }
      bar_arrive(BAR_STAGED + gi, 2 * CT);
      WT(7);  // contributions staged
    }
    if (q >= 2) bar_sync(BAR_FREE + gi, 2 * CT);  // the node group's last arrival
    WT_FLUSH;
  } else {
    // ================= node group =================
#if WS_SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 48;");
#endif
    uint32_t q = 0, jb = 0, ju = 0;
    WT_DECL;
    for (int t = blockIdx.x; t < a.n_tiles_all; t += G) {
      WT(0);
      const unsigned char *tb = tabs0 + jb * W::tabs();
      mbar_wait(tfull + jb, ju & 1);
      WT(2);  // table wait
      const WsTileMeta tm = *reinterpret_cast<const WsTileMeta *>(tb + L::tabs());
      const int4 *desc = reinterpret_cast<const int4 *>(tb);
      const int *xch = reinterpret_cast<const int *>(tb + (size_t)CT * 16);
      const bool my_node = tid < tm.node_count;
      int outw = 0, fmask = 0, cl = 0;
      bool cross = false;
      double acc[D];
#pragma unroll
      for (int k = 0; k < D; ++k) acc[k] = 0.0;
      if (my_node) {
        const int4 nd = desc[tid];
        outw = nd.w;
        fmask = desc_mask(nd);
        cross = ((unsigned)nd.x & CROSS_FLAG) != 0;
        if (b) {  // the node's load values -> shared memory (read at the tile end)
#pragma unroll
          for (int k = 0; k < D; ++k)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                             smem_u32(bsm + k * CT + tid)),
                         "l"(b + (int64_t)nd.z * D + k)
                         : "memory");
        }
        if (WJ && b) cl = __ldg(a.node_clo + tm.node_begin + tid);
      }
      const int ne_t = tm.own_count;
      WT(1);  // tile start
      for (int c0 = 0; c0 < ne_t; c0 += CT, ++q) {
        const int gi = q & 1;
        int xb = 0, xe = 0;
        if (tm.is_node_tile) {
          xb = xch[c0 / CT];
          xe = xch[c0 / CT + 1];
        }
        int xkey0 = 0;
        if (xb + tid < xe) xkey0 = __ldg(a.xkey + xb + tid);
        const double *stage_d = reinterpret_cast<const double *>(stage0 + gi * L::staging(D));
        auto st_at = [&](int slot, int row) -> const double * {
          return L::AOS(D) ? stage_d + slot * SST + row * D : stage_d + row + slot * SST;
        };
        WT(3);  // chunk head
        bar_sync(BAR_STAGED + gi, 2 * CT);  // chunk q's contributions are staged
        WT(4);  // wait for the element group
        if (my_node) {
          // the node's entries of the chunk, four at a time (their loads issued
          // together); own entries come first (ascending tile element = the fixed
          // summation order), cross entries (tile element >= ne_t) are skipped
          const uint16_t *blk = reinterpret_cast<const uint16_t *>(eslots + (q & 7) * ES);
          const int e_beg = blk[tid], n = blk[tid + 1] - e_beg;
          const uint16_t *ents = blk + blk_header(tm.node_count) + e_beg;
          for (int i = 0; i < n; i += 4) {
            int e[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] = i + u < n ? (int)ents[i + u] : 0xffff;
            double x[4][D];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const bool ok = (e[u] >> 2) < ne_t;
              const double *sp = st_at(e[u] & 3, (e[u] >> 2) - c0);
#pragma unroll
              for (int k = 0; k < D; ++k) x[u][k] = ok ? sp[k * CS] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if ((e[u] >> 2) < ne_t) {
#pragma unroll
                for (int k = 0; k < D; ++k) acc[k] += x[u][k];
              }
            if ((e[3] >> 2) >= ne_t) break;
          }
        }
        WT(5);  // own-entry sums
        for (int i = xb + tid; i < xe; i += CT) {
          const int key = i == xb + tid ? xkey0 : (int)__ldg(a.xkey + i);
          const double *sp = st_at(key & 3, (key >> 2) - c0);
#pragma unroll
          for (int k = 0; k < D; ++k) a.xbuf[(int64_t)i * D + k] = sp[k * CS];
        }
        WT(6);  // cross items
        bar_arrive(BAR_FREE + gi, 2 * CT);  // staging buffer gi and entry slot q & 7 are free
      }
      WT(0);
      if (my_node) {
        double bj[D];
#pragma unroll
        for (int k = 0; k < D; ++k) bj[k] = 0.0;
        if (b) {
          asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
          for (int k = 0; k < D; ++k) bj[k] = bsm[k * CT + tid];
        }
        if (WJ && b) {
          mbar_wait(nfull + jb, ju & 1);  // (a tile without chunks: nobody waited yet)
          const double *nv = nodev(jb);
#pragma unroll
          for (int k = 0; k < D; ++k) bvsum += bj[k] * nv[k * CAP + cl];
        }
        if (cross) {
#pragma unroll
          for (int k = 0; k < D; ++k)
            a.partial[(int64_t)(tm.node_begin + tid) * D + k] = acc[k] - bj[k];
        } else {
          int o = outw;
#pragma unroll
          for (int k = 0; k < D; ++k)
            if (fmask & (1 << k)) g[o++] = acc[k] - bj[k];
        }
      }
      mbar_arrive(tdone + jb);  // the tile's tables and node values may be refilled
      if (++jb == NBUF) {
        jb = 0;
        ++ju;
      }
      WT(7);  // tile end
    }
    WT_FLUSH;
  }
  if (bad_any) atomicOr(status, 1ull);
  if (WJ) {
    const double r = block_sum(jsum, red);
    const double r2 = block_sum(bvsum, red);
    if (tid == 0) {
      jpart[blockIdx.x] = r;
      bvpart[blockIdx.x] = r2;
    }
  }
}

static int ws_nbuf(int dim, int d, int blk_cap, int clo_cap) {
  const size_t cap = (size_t)227 * 1024;
  const size_t s3 = dim == 3 ? WsLayout<3, 3>::total(d, blk_cap, clo_cap)
                             : WsLayout<2, 3>::total(d, blk_cap, clo_cap);
  if (s3 <= cap) return 3;
  const size_t s2 = dim == 3 ? WsLayout<3, 2>::total(d, blk_cap, clo_cap)
                             : WsLayout<2, 2>::total(d, blk_cap, clo_cap);
  return s2 <= cap ? 2 : 0;
}

// 0: the stages do not fit the SM's shared memory
size_t tile_ws_smem(int dim, int d, int blk_cap, int clo_cap) {
  const int nb = ws_nbuf(dim, d, blk_cap, clo_cap);
  if (nb == 0) return 0;
  if (dim == 3)
    return nb == 3 ? WsLayout<3, 3>::total(d, blk_cap, clo_cap)
                   : WsLayout<3, 2>::total(d, blk_cap, clo_cap);
  return nb == 3 ? WsLayout<2, 3>::total(d, blk_cap, clo_cap)
                 : WsLayout<2, 2>::total(d, blk_cap, clo_cap);
}

template <int DIM, int MODEL, int NBUF>
static cudaError_t launch_ws_n(const TileArgs &a, int grid, bool wj, const double *v,
                               const double *b, double *g, double *jpart, double *bvpart,
                               unsigned long long *status, const ModelArgs &m, cudaStream_t s) {
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  const size_t smem = WsLayout<DIM, NBUF>::total(D, a.blk_cap, a.clo_cap);
  auto k = wj ? k_tile_ws<DIM, MODEL, true, NBUF> : k_tile_ws<DIM, MODEL, false, NBUF>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, WS_THREADS, smem, s>>>(a, v, b, g, jpart, bvpart, status, m);
  return cudaGetLastError();
}

template <int DIM, int MODEL>
static cudaError_t launch_ws_t(const TileArgs &a, int grid, bool wj, const double *v,
                               const double *b, double *g, double *jpart, double *bvpart,
                               unsigned long long *status, const ModelArgs &m, cudaStream_t s) {
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  const int nb = ws_nbuf(DIM, D, a.blk_cap, a.clo_cap);
  if (nb == 3)
    return launch_ws_n<DIM, MODEL, 3>(a, grid, wj, v, b, g, jpart, bvpart, status, m, s);
  if (nb == 2)
    return launch_ws_n<DIM, MODEL, 2>(a, grid, wj, v, b, g, jpart, bvpart, status, m, s);
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_tile_ws(int dim, int model, const TileArgs &a, int grid, bool wj,
                           const double *v, const double *b, double *g, double *jpart,
                           double *bvpart, unsigned long long *status, const ModelArgs &m,
                           cudaStream_t s) {
  if (dim == 3 && model == FM_MODEL_NEOHOOKEAN)
    return launch_ws_t<3, FM_MODEL_NEOHOOKEAN>(a, grid, wj, v, b, g, jpart, bvpart, status, m, s);
  if (dim == 3)
    return launch_ws_t<3, FM_MODEL_PLAPLACE>(a, grid, wj, v, b, g, jpart, bvpart, status, m, s);
  if (model == FM_MODEL_NEOHOOKEAN)
    return launch_ws_t<2, FM_MODEL_NEOHOOKEAN>(a, grid, wj, v, b, g, jpart, bvpart, status, m, s);
  return launch_ws_t<2, FM_MODEL_PLAPLACE>(a, grid, wj, v, b, g, jpart, bvpart, status, m, s);
}

}  // namespace fm

#endif  // FM_WS_KERNEL
