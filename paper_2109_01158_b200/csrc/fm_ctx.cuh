// Device-side layout of an evaluation context (the frozen Mesh + Patches of
// mesh.py:31-53 / patches.py:22-34, re-laid out for sm_100a) and the device
// functions shared by the evaluation kernels.
//
// Element records (AoS, one per element, storage order = grouped by owner tile):
//   3D: 128 B = int32 conn[4] | f64 vol | f64 dphi[3][4] | int32 orig | pad
//   2D:  80 B = int32 conn[3] | int32 orig | f64 vol | f64 dphi[2][3] | pad
// A record is one 128-byte line (3D): a gather by element id costs one line and
// brings vol, dphi and conn together.  In shared memory 3D records are stored
// with a 144-byte stride (9 x 16 B, odd) so that lane i reading record i is
// bank-conflict free; 80 B (5 x 16 B) is already odd.
//
// Node tiles: each tile owns <= 256 free nodes of a spatial box.  Its element
// list is [own elements (contiguous storage range, the tile is their J owner)]
// + [halo elements (storage ids)], and its node entries (te_local << 2 | slot)
// are sorted by te_local per node so that a streaming pass over the element
// list can be consumed chunk by chunk.
#pragma once

#include <math.h>
#include <stdint.h>

#include "fm_common.cuh"

namespace fm {

constexpr int MAX_TILE_ELEMS = 16384;  // node entries store te_local in 14 bits
constexpr int CONSUMERS = 256;         // consumer threads = chunk size = max tile nodes
constexpr int OUT_MASK_SHIFT = 28;     // node_desc.w = out_offset | free_mask << 28

template <int DIM> struct RecBytes;
template <> struct RecBytes<2> { static constexpr int value = 80, smem = 80; };
template <> struct RecBytes<3> { static constexpr int value = 128, smem = 128; };

// 16-B chunk c of shared-memory record r: 3D records use the TMA 128-byte swizzle
// (chunk index XOR r mod 8, stage buffers 1024-B aligned), 2D records an odd stride.
template <int DIM>
__device__ __forceinline__ int rec_chunk_off(int r, int c) {
  if constexpr (DIM == 3) return r * 128 + ((c ^ (r & 7)) << 4);
  else return r * 80 + (c << 4);
}

struct TileMeta {
  int own_begin, own_count;      // storage range of the elements the tile owns
  int halo_begin, halo_count;    // range in halo_ids
  int node_begin, node_count;    // range in node_desc
  int entry_begin, entry_count;  // range in node_entries (entry_begin % 8 == 0)
  int elem_begin;                // range start in flags (own + halo)
  int pad[3];
};
static_assert(sizeof(TileMeta) == 48, "TileMeta layout");

template <int DIM> struct Elem {
  int c[DIM + 1];
  int orig;
  double vol;
  double g[DIM][DIM + 1];  // dphi[m][l]
};

// Element records read once per visit: stream them past L1.
__device__ __forceinline__ double2 ld_stream(const double2 *p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

template <int DIM>
__device__ __forceinline__ void decode_elem(const double2 (&q)[RecBytes<DIM>::value / 16],
                                            Elem<DIM> &E) {
  if constexpr (DIM == 3) {
    E.c[0] = __double2loint(q[0].x);
    E.c[1] = __double2hiint(q[0].x);
    E.c[2] = __double2loint(q[0].y);
    E.c[3] = __double2hiint(q[0].y);
    E.vol = q[1].x;
    const double f[12] = {q[1].y, q[2].x, q[2].y, q[3].x, q[3].y, q[4].x,
                          q[4].y, q[5].x, q[5].y, q[6].x, q[6].y, q[7].x};
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int l = 0; l < 4; ++l) E.g[m][l] = f[m * 4 + l];
    E.orig = __double2loint(q[7].y);
  } else {
    E.c[0] = __double2loint(q[0].x);
    E.c[1] = __double2hiint(q[0].x);
    E.c[2] = __double2loint(q[0].y);
    E.orig = __double2hiint(q[0].y);
    E.vol = q[1].x;
    E.g[0][0] = q[1].y;
    E.g[0][1] = q[2].x;
    E.g[0][2] = q[2].y;
    E.g[1][0] = q[3].x;
    E.g[1][1] = q[3].y;
    E.g[1][2] = q[4].x;
  }
}

template <int DIM>
__device__ __forceinline__ void load_elem(const uint8_t *__restrict__ aos, int64_t s,
                                          Elem<DIM> &E) {
  constexpr int NQ = RecBytes<DIM>::value / 16;
  const double2 *p = reinterpret_cast<const double2 *>(aos + s * (int64_t)RecBytes<DIM>::value);
  double2 q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = ld_stream(p + k);
  decode_elem<DIM>(q, E);
}

template <int DIM>
__device__ __forceinline__ void load_elem_smem(const uint8_t *stage, int r, Elem<DIM> &E) {
  constexpr int NQ = RecBytes<DIM>::value / 16;
  double2 q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k)
    q[k] = *reinterpret_cast<const double2 *>(stage + rec_chunk_off<DIM>(r, k));
  decode_elem<DIM>(q, E);
}

// CUtensorMap is a 128-byte, 64-byte aligned opaque descriptor; boxes of 8..256 rows.
struct alignas(64) TmaDesc {
  unsigned char bytes[128];
};
struct TmaMaps {
  TmaDesc box[6];  // rows 8 << k
};

// Gather the d components of the field at the element's nodes (v interleaved).
template <int DIM, int D>
__device__ __forceinline__ void gather_v(const double *__restrict__ v, const int (&c)[DIM + 1],
                                         double (&vv)[D][DIM + 1]) {
#pragma unroll
  for (int l = 0; l < DIM + 1; ++l) {
    const double *p = v + (int64_t)c[l] * D;
#pragma unroll
    for (int j = 0; j < D; ++j) vv[j][l] = __ldg(p + j);
  }
}

struct ModelArgs {
  int kind;  // FM_MODEL_*
  double p, C1, D1;
  // p-Laplace exponents classified like numpy's fast scalar power
  // (ndarray ** scalar: 0.5 -> sqrt, 1 -> copy, 2 -> square, -1 -> reciprocal)
  double e_w, e_dw;  // p/2 and (p-2)/2
};

__device__ __forceinline__ double np_scalar_pow(double x, double e) {
  if (e == 0.5) return sqrt(x);
  if (e == 1.0) return x;
  if (e == 2.0) return x * x;
  if (e == -1.0) return 1.0 / x;
  if (e == 0.0) return 1.0;
  return pow(x, e);
}

// Tile tables (built by fm_ctx_create).
struct TileArgs {
  const uint8_t *aos;
  const TileMeta *meta;      // n_tiles_all
  const int32_t *halo_ids;   // storage index of halo elements
  const uint8_t *flags;      // owned-slot mask per tile element (own then halo)
  const int4 *node_desc;     // {entry_off, entry_count, node id, out | mask << 28}
  const uint16_t *entries;   // te_local << 2 | slot, sorted by te_local per node
  const int32_t *rank_of;    // node -> free rank or -1
  int n_tiles;               // node tiles
  int n_tiles_all;           // + orphan tiles (J only)
  int entry_cap;             // max entries of one tile, rounded up to 8
  int halo_cap;              // max halo elements of one tile, rounded up to 4
};

// Deterministic block sum (fixed shuffle tree + fixed warp order).
__device__ __forceinline__ double block_sum(double x, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = x;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

}  // namespace fm

// Host-side context.
struct fm_ctx {
  int dim = 0, d = 0, nv = 0, tile_nodes = 0;
  int64_t nn = 0, ne = 0, nfree = 0, nfree_dofs = 0, p_total = 0;
  int32_t n_tiles = 0, n_tiles_all = 0;
  int64_t n_tile_elems = 0, n_node_entries = 0;
  int max_tile_elems = 0, max_tile_entries = 0, max_tile_nodes = 0, entry_cap = 0, halo_cap = 0;
  int n_sm = 148, stages = 4;
  uint8_t *aos = nullptr;
  fm::TileMeta *meta = nullptr;
  int32_t *halo_ids = nullptr;
  uint8_t *flags = nullptr;
  int4 *node_desc = nullptr;
  uint16_t *node_entries = nullptr;
  int32_t *free_node = nullptr, *free_out = nullptr, *rank_of = nullptr;
  int32_t *storage_to_orig = nullptr;
  uint8_t *free_mask = nullptr;
  // scratch
  double *jpart = nullptr;        // per CTA (fused) / per block (energy)
  double *dotpart = nullptr;      // b.v partials
  int n_dot_blocks = 0, n_energy_blocks = 0, n_part = 0;
  unsigned long long *status = nullptr;  // [0] exact inadmissible, [1] FD min key
  int64_t launches = 0;
  size_t bytes = 0;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;  // armed by fm_ctx_time_next
  fm::TmaMaps tma{};  // 3D element records as a 2D tensor (rows x 128 B), SWIZZLE_128B
  fm_ctx_stats stats{};

  fm::TileArgs tile_args() const {
    return fm::TileArgs{aos,     meta,    halo_ids,    flags,     node_desc, node_entries,
                        rank_of, n_tiles, n_tiles_all, entry_cap, halo_cap};
  }
};
