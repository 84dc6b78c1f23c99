// Device-side layout of an evaluation context (the frozen Mesh + Patches of
// mesh.py:31-53 / patches.py:22-34, re-laid out for sm_100a) and the device
// functions shared by the evaluation kernels.
//
// Element records (AoS, storage order = grouped by owner tile, 16-B multiples
// with an ODD number of 16-B chunks so that lane i reading record i from shared
// memory is bank-conflict free):
//   3D: 80 B = f64 vol | f64 dphi[3][1..3]
//   2D: 48 B = f64 vol | f64 dphi[2][1..2] | pad
// dphi[m][0] is not stored: compute_p1_gradients makes it -(sum of the other
// columns) (mesh.py:100-101), and the context build checks that identity bit
// for bit before dropping it, so decode_elem rebuilds the exact reference value.
// loc (u16 x 4 per element, storage order) are the element's nodes as indices
// into its OWNER tile's node closure (sorted distinct nodes of all elements the
// tile visits); global node ids live in conn4 (int4 per element, storage order)
// for the streaming kernels.
//
// Node tiles: each tile owns <= 256 free nodes of a spatial box.  Its element
// list is [own elements (contiguous storage range, the tile is their J owner)]
// + [halo elements (storage ids + loc w.r.t. this tile)], and its node entries
// (te_local << 2 | slot) are sorted by te_local per node so that a streaming
// pass over the element list can be consumed chunk by chunk.
#pragma once

#include <math.h>
#include <stdint.h>

#include "fm_common.cuh"

namespace fm {

constexpr int MAX_TILE_ELEMS = 16384;  // node entries store te_local in 14 bits
constexpr int CONSUMERS = 256;         // threads per tile CTA = chunk size = max tile nodes
// node_desc = {x: entry offset (bits 0..12) | chunk counts 0..2 (bits 13..27) |
//                 free-component mask (bits 28..30) | cross flag (bit 31),
//              y: chunk counts 3..8, z: node id, w: output offset (31 bits, so a
//              context holds up to 2^31 - 1 free dofs)}
constexpr int DESC_MASK_SHIFT = 28;        // node_desc.x: free-component mask
constexpr unsigned CROSS_FLAG = 1u << 31;  // node_desc.x: the node has cross entries
constexpr int MAX_CHUNKS = 9;          // per-chunk entry counts in node_desc.x/.y (5 bits each)
constexpr int ENTRY_OFF_MASK = (1 << 13) - 1;  // node_desc.x bits 0..12: tile-local entry offset
constexpr int XCH_STRIDE = 12;  // ints per tile in xchunk (MAX_CHUNKS + 1, padded to 16 B)
// Record dictionaries: a tile whose own elements share at most DICT_MAX distinct
// records (vol, dphi — bit patterns; structured meshes have a handful) keeps
// them as a per-tile table, and its elements as one byte each (the record's
// table slot, TileArgs::eidx).  The tile kernel then streams 1 B instead of
// 80 / 48 B per element and reads the record from the table in shared memory;
// the values are the same bits.  Tiles with more distinct records (unstructured
// meshes) stream their records as before.
constexpr int DICT_MAX = 16;

// entries of this node in chunk ch of its tile (node_desc packing, see k_node_desc)
__device__ __forceinline__ int chunk_count(int4 nd, int ch) {
  const unsigned long long cc =
      ((unsigned long long)(unsigned)nd.y << 15) | (((unsigned)nd.x >> 13) & 0x7fffu);
  return (int)((cc >> (5 * ch)) & 31ull);
}

// free components of the node (bit j: dof d*node+j is free)
__host__ __device__ __forceinline__ int desc_mask(int4 nd) {
  return (int)(((unsigned)nd.x >> DESC_MASK_SHIFT) & 7u);
}

template <int DIM> struct RecBytes;
template <> struct RecBytes<2> { static constexpr int value = 48; };
template <> struct RecBytes<3> { static constexpr int value = 80; };

struct TileMeta {
  int own_begin, own_count;      // storage range of the elements the tile owns
  int halo_begin, halo_count;    // range in halo_ids / halo_loc
  int node_begin, node_count;    // range in node_desc
  int entry_begin, entry_count;  // range in node_entries (entry_begin % 8 == 0)
  int elem_begin;                // range start in flags (own + halo)
  int clo_begin, clo_count;      // node closure (clo_begin % 4 == 0)
  int blk_stride;                // chunk entry blocks: u16 units per block (multiple of 8)
  int64_t blk_base;              // first block of the tile in chunk_blocks (u16 units)
  int dict_n;                    // distinct element records of the tile (0: not dictionary-coded)
  int pad;
};
static_assert(sizeof(TileMeta) == 64, "TileMeta layout");

// Chunk entry block (u16 units): [node offsets: node_count + 1, padded to 8]
// [the chunk's node entries (te << 2 | slot), node-major, te ascending per node]
__host__ __device__ __forceinline__ int blk_header(int node_count) {
  return (node_count + 1 + 7) / 8 * 8;
}

template <int DIM> struct Elem {
  int c[DIM + 1];  // global node ids (streaming kernels)
  int loc[4];      // closure indices (tile kernels; decode_loc)
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

__device__ __forceinline__ int4 ld_stream_i4(const int4 *p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// dphi[m][0] = -((dphi[m][1] + dphi[m][2]) + dphi[m][3]) as numpy's sum over
// the row (mesh.py:101); negation is exact
template <int DIM>
__device__ __forceinline__ double dphi0(const double (&g)[DIM + 1]) {
  if constexpr (DIM == 3)
    return -__dadd_rn(__dadd_rn(g[1], g[2]), g[3]);
  else
    return -__dadd_rn(g[1], g[2]);
}

template <int DIM>
__device__ __forceinline__ void decode_elem(const double2 (&q)[RecBytes<DIM>::value / 16],
                                            Elem<DIM> &E) {
  E.vol = q[0].x;
  if constexpr (DIM == 3) {
    const double f[9] = {q[0].y, q[1].x, q[1].y, q[2].x, q[2].y, q[3].x, q[3].y, q[4].x, q[4].y};
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int l = 1; l < 4; ++l) E.g[m][l] = f[m * 3 + l - 1];
  } else {
    const double f[4] = {q[0].y, q[1].x, q[1].y, q[2].x};
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int l = 1; l < 3; ++l) E.g[m][l] = f[m * 2 + l - 1];
  }
#pragma unroll
  for (int m = 0; m < DIM; ++m) E.g[m][0] = dphi0<DIM>(E.g[m]);
}

__device__ __forceinline__ void decode_loc(uint2 w, int (&loc)[4]) {
  loc[0] = (int)(w.x & 0xffffu);
  loc[1] = (int)(w.x >> 16);
  loc[2] = (int)(w.y & 0xffffu);
  loc[3] = (int)(w.y >> 16);
}

// record + global connectivity from global memory (streaming kernels)
template <int DIM>
__device__ __forceinline__ void load_elem(const uint8_t *__restrict__ aos,
                                          const int4 *__restrict__ conn4, int64_t s,
                                          Elem<DIM> &E) {
  constexpr int NQ = RecBytes<DIM>::value / 16;
  const double2 *p = reinterpret_cast<const double2 *>(aos + s * (int64_t)RecBytes<DIM>::value);
  double2 q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = ld_stream(p + k);
  decode_elem<DIM>(q, E);
  const int4 c = ld_stream_i4(conn4 + s);
  E.c[0] = c.x;
  E.c[1] = c.y;
  E.c[2] = c.z;
  if constexpr (DIM == 3) E.c[3] = c.w;
}

// record from a shared-memory stage (row r)
template <int DIM>
__device__ __forceinline__ void load_elem_smem(const uint8_t *stage, int r, Elem<DIM> &E) {
  constexpr int NQ = RecBytes<DIM>::value / 16;
  const double2 *p = reinterpret_cast<const double2 *>(stage + r * RecBytes<DIM>::value);
  double2 q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = p[k];
  decode_elem<DIM>(q, E);
}

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
  double eps;       // FD step (fm_grad_fd; 0 otherwise)
  int dbg;           // profiling ablations of the tile kernel, read through FM_DBG (FM_TILE_ABLATE,
                     // tools/ablate.py: 1 no constitutive, 2 no consume, 8 no compute, 32 no
                     // closure gathers; results are wrong on purpose), 0 = off
};

// The ablation switches exist only in profiling builds (-DFM_ABLATE=1, a
// separate library built by tools/ablate.py); in the product library FM_DBG
// is the constant 0 and the compiler drops every ablation branch.
#ifndef FM_ABLATE
#define FM_ABLATE 0
#endif
// the warp-specialised kernel experiment (fm_eval_ws.cu) is compiled only into
// the separate library tools/ws_check.sh builds (-DFM_WS_KERNEL=1)
#ifndef FM_WS_KERNEL
#define FM_WS_KERNEL 0
#endif
#define FM_DBG(m) (FM_ABLATE ? (m).dbg : 0)

// x ** e with numpy's fast scalar cases (-1, 0, 0.5, 1, 2) and, beyond numpy,
// 1.5 as x sqrt(x) (the p = 3 energy; <= 2 ulps of pow(x, 1.5), within the
// libm term of every tolerance); other exponents through pow
__device__ __forceinline__ double np_scalar_pow(double x, double e) {
  if (e == 0.5) return sqrt(x);
  if (e == 1.5) return x * sqrt(x);
  if (e == 1.0) return x;
  if (e == 2.0) return x * x;
  if (e == -1.0) return 1.0 / x;
  if (e == 0.0) return 1.0;
  return pow(x, e);
}

// Tile tables (built by fm_ctx_create).
struct TileArgs {
  const uint8_t *aos;
  const int4 *conn4;           // global node ids per element (storage order; 2D only)
  const int32_t *s2o;          // storage -> reference element id
  const TileMeta *meta;        // n_tiles_all
  const int32_t *halo_ids;     // storage index of halo elements (build only; null at run time)
  const uint2 *halo_loc;       // closure indices (u16 x 4) of halo elements (build only)
  const uint2 *loc;            // closure indices (u16 x 4) w.r.t. the owner tile, storage order
  const int32_t *closure;      // node ids of the tile closures
  const uint8_t *flags;        // owned-slot mask per tile element (build only)
  const int4 *node_desc;       // {entry_off | chunk counts, chunk counts, node id,
                               //  out offset} (see chunk_count, desc_mask)
  const uint16_t *entries;     // te_local << 2 | slot, sorted by te_local per node
  const uint16_t *chunk_blocks;  // per tile and chunk: node offsets + entries (see blk_header)
  const int32_t *rank_of;      // node -> free rank or -1
  // cross-tile exchange of the fused exact kernel (elements computed once, by
  // their owner tile): items (owner te << 2 | slot) -> exchange slot, sorted by
  // (owner tile, te); xchunk[t * XCH_STRIDE + c] = first item of chunk c
  // of tile t; xbuf[slot * D + k] receives the contributions (slots are dense
  // and node-major: a node's cross entries are consecutive, in te order)
  const uint16_t *xkey;
  const int32_t *xpos;          // node-major exchange slot -> item index (finishing pass)
  const int32_t *xchunk;
  double *xbuf;
  double *partial;             // tile node x D: own-element sums of nodes with cross entries
  const uint16_t *node_clo;    // tile node -> its index in the tile's node closure
  const uint8_t *eidx;         // dictionary slot of each element (storage order; see DICT_MAX)
  const uint8_t *dict_rec;     // per tile DICT_MAX records (tile t at t * DICT_MAX * record bytes)
  int n_tiles;                 // node tiles
  int n_tiles_all;             // + orphan tiles (J only)
  int entry_cap;               // max entries of one tile, rounded up to 8
  int blk_cap;                 // max chunk entry block, u16 units
  int clo_cap;                 // max closure size, rounded up to 4
  int all_coded;               // every tile with elements is dictionary-coded: the record
                               // area of a stage holds slot bytes only
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
  int max_tile_elems = 0, max_tile_entries = 0, max_tile_nodes = 0, entry_cap = 0, clo_cap = 0;
  int n_sm = 0, ctas_per_sm = 2, node_bufs = 2, table_bufs = 2;
  bool ws = false;  // experiment builds (FM_WS_KERNEL): fused J + gradient through fm_eval_ws.cu
  uint8_t *aos = nullptr;
  int4 *conn4 = nullptr;
  fm::TileMeta *meta = nullptr;
  int32_t *halo_ids = nullptr, *closure = nullptr;
  uint2 *halo_loc = nullptr, *loc = nullptr;
  uint8_t *flags = nullptr;
  int4 *node_desc = nullptr;
  uint16_t *node_entries = nullptr;
  int32_t *free_node = nullptr, *free_out = nullptr, *rank_of = nullptr;
  int32_t *storage_to_orig = nullptr;
  uint8_t *free_mask = nullptr;
  int32_t *dof_pos = nullptr;  // free dof q -> its index in v (descent update)
  uint16_t *xkey = nullptr;                        // cross-tile exchange (see TileArgs)
  int32_t *xpos = nullptr, *xchunk = nullptr;
  int32_t *node_xbase = nullptr, *node_xn = nullptr;  // per tile node: its cross entries
  int32_t *xnodes = nullptr;  // tile nodes with cross entries (build only)
  int4 *xdesc = nullptr;      // finishing pass, per tile node with cross entries:
                              // {tile node, first exchange slot, count | free mask << 16, out}
  int64_t n_xnodes = 0;
  double *xbuf = nullptr, *partial = nullptr;
  int32_t *node_outw = nullptr;  // per tile node: output offset (finishing pass)
  uint8_t *node_fmask = nullptr;  // per tile node: free-component mask (finishing pass)
  uint16_t *node_clo = nullptr;  // per tile node: index in its tile's closure
  uint8_t *eidx = nullptr, *dict_rec = nullptr;  // record dictionaries (see DICT_MAX)
  int64_t n_dict_tiles = 0;
  bool all_coded = false;  // every tile with elements is coded (small record stages)
  uint16_t *chunk_blocks = nullptr;  // chunk-major entry blocks (TileMeta blk_base / blk_stride)
  int blk_cap = 0;                   // max block size, u16 units
  int64_t blk_total = 0;             // size of chunk_blocks, u16 units
  int64_t n_cross = 0;
  int32_t *fixed_nodes = nullptr;  // nodes without a free dof (their b.v: finishing pass)
  int64_t n_fixed_nodes = 0;
  // scratch
  double *jpart = nullptr;        // per CTA (fused) / per block (energy)
  double *dotpart = nullptr;      // b.v partials
  int n_dot_blocks = 0, n_energy_blocks = 0, n_part = 0;
  unsigned long long *status = nullptr;  // [0] exact inadmissible, [1] FD min key
  double *fpart = nullptr;          // finishing pass: per-block b.v of fixed nodes
  unsigned int *ticket = nullptr;    // finishing pass: last-block ticket (0 between calls)
  int64_t launches = 0;
  size_t bytes = 0;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;  // armed by fm_ctx_time_next
  fm_ctx_stats stats{};

  fm::TileArgs tile_args() const {
    return fm::TileArgs{aos,     conn4,   storage_to_orig, meta,      halo_ids,    halo_loc,
                        loc,     closure, flags,   node_desc,       node_entries, chunk_blocks,
                        rank_of, xkey,
                        xpos,    xchunk,  xbuf,            partial,   node_clo,    eidx,
                        dict_rec, n_tiles,
                        n_tiles_all, entry_cap, blk_cap, clo_cap, all_coded ? 1 : 0};
  }
};
