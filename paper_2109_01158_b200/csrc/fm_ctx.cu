// Evaluation context: uploads/re-lays out the frozen Mesh + Patches once
// (mesh.py:31-53, patches.py:22-71) and exposes the evaluation entry points of
// include/femmin_b200.h.
//
// Context build (GPU, CUB radix sorts, deterministic; host only sees counts):
//   1. free-node ranks and output offsets of the restricted gradient
//      (gradients.py:68-74 _blocks_to_dofs order);
//   2. node tiles: free nodes bucketed into spatial boxes (edge = k * mesh width,
//      width from the mean element measure), boxes in Morton order, split to
//      <= 256 nodes and <= entry-cap node entries;
//   3. element owner tile = tile of its first free node (orphans: none);
//      storage order sorted by (owner tile, element) -> element records;
//   4. tile element lists = own elements (contiguous storage) + halo elements
//      (union of the tile nodes' patches, patches.py:37-71 rows, minus own),
//      slot masks OR-reduced by key;
//   5. node descriptors and entries (te_local << 2 | slot) sorted by te_local.
#include <cub/cub.cuh>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "fm_kernels.h"

namespace fm {

static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }

constexpr int ENTRY_CAP_DEFAULT = 8192;  // node entries per tile (16 KB of shared memory)

// ---------------------------------------------------------------- kernels
__global__ void k_ranks(int64_t nfree, int d, const int64_t *nodes_minim, const uint8_t *fixed,
                        int32_t *rank_of, int32_t *free_node, uint8_t *mask, int32_t *cnt) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nfree;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = nodes_minim[r];
    rank_of[n] = (int32_t)r;
    free_node[r] = (int32_t)n;
    int mk = 0, c = 0;
    for (int j = 0; j < d; ++j)
      if (!fixed[n * d + j]) {
        mk |= 1 << j;
        ++c;
      }
    mask[r] = (uint8_t)mk;
    cnt[r] = c;
  }
}

__device__ __forceinline__ unsigned long long ord_bits(double x) {
  unsigned long long u = __double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
static inline double from_ord(unsigned long long u) {
  unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
  double x;
  memcpy(&x, &b, 8);
  return x;
}

__global__ void k_bbox(int64_t n, int dim, const int64_t *nodes, const double *X,
                       unsigned long long *mn, unsigned long long *mx) {
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t node = nodes[r];
    for (int a = 0; a < dim; ++a) {
      unsigned long long o = ord_bits(X[node * dim + a]);
      lo[a] = o < lo[a] ? o : lo[a];
      hi[a] = o > hi[a] ? o : hi[a];
    }
  }
  for (int a = 0; a < dim; ++a) {
    atomicMin(mn + a, lo[a]);
    atomicMax(mx + a, hi[a]);
  }
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {  // 21 bits -> every 3rd bit
  x &= 0x1fffffull;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

__global__ void k_box_keys(int64_t nfree, int dim, const int64_t *nodes, const double *X,
                           double x0, double y0, double z0, double ex, double ey, double ez,
                           double hh, uint64_t *keys, int32_t *vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nfree;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t node = nodes[r];
    uint64_t ix = (uint64_t)floor((X[node * dim] - x0 + hh) / ex);
    uint64_t iy = (uint64_t)floor((X[node * dim + 1] - y0 + hh) / ey);
    uint64_t iz = dim == 3 ? (uint64_t)floor((X[node * dim + 2] - z0 + hh) / ez) : 0;
    keys[r] = spread3(ix) | (spread3(iy) << 1) | (spread3(iz) << 2);  // Morton order
    vals[r] = (int32_t)r;
  }
}

__global__ void k_sorted_lengths(int64_t n, const int32_t *ranks, const int64_t *prefix,
                                 int32_t *lens) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int r = ranks[k];
    lens[k] = (int32_t)(prefix[r] - (r ? prefix[r - 1] : 0));
  }
}

__global__ void k_tile_of_pos(int64_t ntn, int n_tiles, const int32_t *tile_node_ptr,
                              const int32_t *tile_node_rank, int32_t *tile_of_rank) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntn;
       k += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_tiles;  // largest t with ptr[t] <= k
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (tile_node_ptr[mid] <= k) lo = mid; else hi = mid;
    }
    tile_of_rank[tile_node_rank[k]] = lo;
  }
}

__global__ void k_owner(int64_t ne, int nv, const int64_t *conn, const int32_t *rank_of,
                        const int32_t *tile_of_rank, int n_tiles, uint32_t *okey,
                        int32_t *oval, int32_t *owner_of) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    // owner = the tile of the first free node (measured against the tile
    // holding most of the element's free nodes: 31 % fewer cross entries at
    // cfg4, but 5 % slower)
    int own = n_tiles;
    for (int l = 0; l < nv; ++l) {
      const int r = rank_of[conn[e * nv + l]];
      if (r >= 0) {
        own = tile_of_rank[r];
        break;
      }
    }
    okey[e] = (uint32_t)own;
    oval[e] = (int32_t)e;
    owner_of[e] = own;
  }
}

__global__ void k_inverse(int64_t n, const int32_t *perm, int32_t *inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    inv[perm[i]] = (int32_t)i;
}

// first index in the sorted array with value >= key, for keys t = 0..n
__global__ void k_lower_bounds_u32(int n, int64_t len, const uint32_t *sorted, int32_t *out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= n; t += gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = len;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (sorted[mid] < (uint32_t)t) lo = mid + 1; else hi = mid;
    }
    out[t] = (int32_t)lo;
  }
}

// dphi[m][:, 0] == -(dphi[m][:, 1:].sum()) bit for bit (mesh.py:100-101)?
template <int DIM>
__global__ void k_dphi0_check(int64_t ne, const double *dphi, unsigned long long *bad) {
  constexpr int NV = DIM + 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x)
    for (int m = 0; m < DIM; ++m) {
      const double *g = dphi + ((int64_t)m * ne + e) * NV;
      double r = __dadd_rn(g[1], g[2]);
      if (DIM == 3) r = __dadd_rn(r, g[3]);
      if (!(g[0] == -r)) atomicMin(bad, (unsigned long long)e);
    }
}

// records (vol | dphi[m][1..]) (+ conn4, 2D) in storage order
template <int DIM>
__global__ void k_build_aos(int64_t ne, const int32_t *s2o, const int64_t *conn, const double *vol,
                            const double *dphi, uint8_t *aos, int4 *conn4) {
  constexpr int NV = DIM + 1;
  constexpr int NF = RecBytes<DIM>::value / 8;  // f64 words per record
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < ne;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = s2o[s];
    double *dd = reinterpret_cast<double *>(aos + s * RecBytes<DIM>::value);
    dd[0] = vol[e];
    for (int m = 0; m < DIM; ++m)
      for (int l = 1; l < NV; ++l) dd[1 + m * DIM + l - 1] = dphi[((int64_t)m * ne + e) * NV + l];
    for (int k = 1 + DIM * DIM; k < NF; ++k) dd[k] = 0.0;
    if (DIM == 2) {  // 2D only: the streaming energy kernel's connectivity
      int4 c;
      c.x = (int)conn[e * NV];
      c.y = (int)conn[e * NV + 1];
      c.z = (int)conn[e * NV + 2];
      c.w = (int)e;
      conn4[s] = c;
    }
  }
}

// (tile, node) keys of every element a tile visits: node tiles from the unique
// (tile, halo?, element) list, orphan tiles from their own storage range
__global__ void k_closure_keys(int64_t i0, int64_t i1, int64_t M, const uint64_t *ukeys,
                               int64_t orph0, int n_tiles, int ot, const int32_t *s2o,
                               const int64_t *conn, int nv, uint64_t *keys) {
  for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < i1;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t t;
    int64_t e;
    if (i < M) {
      t = ukeys[i] >> 33;
      e = (int64_t)(ukeys[i] & 0xffffffffull);
    } else {
      const int64_t o = i - M;
      t = (uint64_t)(n_tiles + o / ot);
      e = s2o[orph0 + o];
    }
    for (int l = 0; l < nv; ++l) keys[(i - i0) * nv + l] = (t << 32) | (uint64_t)conn[e * nv + l];
  }
}

__global__ void k_lower_bounds_u64(int n, int64_t len, const uint64_t *sorted, int shift,
                                   int32_t *out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= n; t += gridDim.x * blockDim.x) {
    const uint64_t key = (uint64_t)t << shift;
    int64_t lo = 0, hi = len;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (sorted[mid] < key) lo = mid + 1; else hi = mid;
    }
    out[t] = (int32_t)lo;
  }
}

__global__ void k_closure_ids(int64_t C, const uint64_t *ckeys, const int32_t *cstart,
                              const int32_t *cbegin, int32_t *closure) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < C;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(ckeys[i] >> 32);
    closure[cbegin[t] + (i - cstart[t])] = (int32_t)(ckeys[i] & 0xffffffffull);
  }
}

// closure indices of every (tile, element): own -> record, halo -> halo_loc
template <int DIM>
__global__ void k_fill_loc(int64_t M, const uint64_t *ukeys, int64_t n_orph, int64_t orph0,
                           int n_tiles, int ot, const int32_t *s2o, const int32_t *o2s,
                           const int64_t *conn, const uint64_t *ckeys, const int32_t *cstart,
                           const int32_t *ptr, const int32_t *split, const int32_t *tpos,
                           const int32_t *halo_begin, uint2 *loc, uint2 *halo_loc,
                           unsigned long long *overflow) {
  constexpr int NV = DIM + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M + n_orph;
       i += (int64_t)gridDim.x * blockDim.x) {
    int t;
    int64_t e, s;
    bool halo = false;
    if (i < M) {
      t = (int)(ukeys[i] >> 33);
      halo = (ukeys[i] >> 32) & 1;
      e = (int64_t)(ukeys[i] & 0xffffffffull);
      s = o2s[e];
    } else {
      const int64_t o = i - M;
      t = n_tiles + (int)(o / ot);
      s = orph0 + o;
      e = s2o[s];
    }
    const int64_t lo0 = cstart[t], hi0 = cstart[t + 1];
    uint64_t packed = 0;
    for (int l = 0; l < NV; ++l) {
      const uint64_t key = ((uint64_t)t << 32) | (uint64_t)conn[e * NV + l];
      int64_t lo = lo0, hi = hi0;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (ckeys[mid] < key) lo = mid + 1; else hi = mid;
      }
      const int64_t idx = lo - lo0;
      if (idx > 0xffff || lo >= hi0 || ckeys[lo] != key) atomicAdd(overflow, 1ull);
      packed |= (uint64_t)(idx & 0xffff) << (16 * l);
    }
    if (halo) {
      halo_loc[halo_begin[t] + tpos[i] - (split[t] - ptr[t])] =
          make_uint2((unsigned)(packed & 0xffffffffull), (unsigned)(packed >> 32));
    } else {
      loc[s] = make_uint2((unsigned)(packed & 0xffffffffull), (unsigned)(packed >> 32));
    }
  }
}

__global__ void k_not_free(int64_t nn, const int32_t *rank_of, uint8_t *flag) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nn;
       n += (int64_t)gridDim.x * blockDim.x)
    flag[n] = rank_of[n] < 0;
}

// storage index -> owner tile (own ranges are contiguous per tile)
__global__ void k_storage_tile(int n_tiles, const int32_t *own_ptr, int32_t *stile) {
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x)
    for (int s = own_ptr[t] + threadIdx.x; s < own_ptr[t + 1]; s += blockDim.x) stile[s] = t;
}

// per tile node: its cross entries (element owned by another tile) are the tail
// of its sorted entry list, te >= own_count of its tile
__global__ void k_cross_count(int64_t ntn, const int32_t *tile_node_rank,
                              const int32_t *tile_of_rank, const TileMeta *meta, const int4 *desc,
                              const uint16_t *entries, const int32_t *entry_abs, int32_t *xbase,
                              int32_t *xn) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntn;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int t = tile_of_rank[tile_node_rank[k]];
    const int own = meta[t].own_count;
    const int4 nd = desc[k];
    int len = 0;
    for (int ch = 0; ch < MAX_CHUNKS; ++ch) len += chunk_count(nd, ch);
    const uint16_t *en = entries + entry_abs[k];
    int p = 0;
    while (p < len && (en[p] >> 2) < own) ++p;
    xbase[k] = entry_abs[k] + p;
    xn[k] = len - p;
  }
}

// tile node -> index of its node id in the tile's sorted node closure
__global__ void k_node_clo(int64_t ntn, const int32_t *tile_node_rank, const int32_t *tile_of_rank,
                           const TileMeta *meta, const int4 *desc, const int32_t *closure,
                           uint16_t *out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntn;
       k += (int64_t)gridDim.x * blockDim.x) {
    const TileMeta tm = meta[tile_of_rank[tile_node_rank[k]]];
    const int node = desc[k].z;
    int lo = 0, hi = tm.clo_count;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (closure[tm.clo_begin + mid] < node) lo = mid + 1; else hi = mid;
    }
    out[k] = (uint16_t)lo;
  }
}

__global__ void k_mark_cross(int64_t ntn, const int32_t *xn, int4 *desc, int32_t *outw,
                             uint8_t *fmask) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntn;
       k += (int64_t)gridDim.x * blockDim.x) {
    outw[k] = desc[k].w;
    fmask[k] = (uint8_t)desc_mask(desc[k]);
    if (xn[k]) desc[k].x = (int)((unsigned)desc[k].x | CROSS_FLAG);
  }
}

// the cross items: (owner tile, owner te, slot) -> entry index
__global__ void k_cross_items(int64_t ntn, const int32_t *tile_node_rank,
                              const int32_t *tile_of_rank, const TileMeta *meta,
                              const uint16_t *entries, const int32_t *xbase, const int32_t *xn,
                              const int32_t *xoff, const int32_t *halo_ids, const int32_t *stile,
                              uint64_t *keys, int32_t *vals) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntn;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int n = xn[k];
    if (!n) continue;
    const TileMeta tm = meta[tile_of_rank[tile_node_rank[k]]];
    for (int p = 0; p < n; ++p) {
      const int en = entries[xbase[k] + p];
      const int st = halo_ids[tm.halo_begin + (en >> 2) - tm.own_count];
      const int to = stile[st];
      const int te = st - meta[to].own_begin;
      keys[xoff[k] + p] = ((uint64_t)to << 16) | (uint64_t)((te << 2) | (en & 3));
      vals[xoff[k] + p] = xoff[k] + p;  // dense exchange slot, node-major
    }
  }
}

// finishing-pass descriptors of the tile nodes with cross entries (one 16-B
// load per node instead of four dependent ones)
__global__ void k_xdesc(int64_t n, const int32_t *xnodes, const int32_t *xbase,
                        const int32_t *outw, const uint8_t *fmask, int4 *xdesc) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int k = xnodes[r];
    const int lo = xbase[k], cnt = xbase[k + 1] - lo;
    xdesc[r] = make_int4(k, lo, cnt | ((int)fmask[k] << 16), outw[k]);
  }
}

__global__ void k_nonzero_flags(int64_t n, const int32_t *x, int32_t *flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = i < n && x[i] != 0;
}

__global__ void k_scatter_flagged(int64_t n, const int32_t *flag, const int32_t *pos,
                                  int32_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[pos[i]] = (int32_t)i;
}

// first item of every chunk of every tile
__global__ void k_xchunk(int n_tiles, int ct, int64_t X, const uint64_t *keys, int32_t *xchunk) {
  const int n = n_tiles * XCH_STRIDE;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t t = i / XCH_STRIDE, ch = min(i % XCH_STRIDE, MAX_CHUNKS);
    const uint64_t key = (t << 16) | ((ch * ct) << 2);
    int64_t lo = 0, hi = X;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    xchunk[i] = (int32_t)lo;
  }
}

__global__ void k_low16(int64_t n, const uint64_t *k, uint16_t *o) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = (uint16_t)(k[i] & 0xffffull);
}

// max over (tile, chunk) of the node entries falling in that chunk
__global__ void k_chunk_entry_max(int n_tiles, const TileMeta *meta, const int4 *desc,
                                  unsigned int *out, int32_t *per_chunk) {
  __shared__ unsigned int cnt[MAX_CHUNKS];
  const int t = blockIdx.x;
  if (threadIdx.x < MAX_CHUNKS) cnt[threadIdx.x] = 0;
  __syncthreads();
  const TileMeta tm = meta[t];
  for (int k = threadIdx.x; k < tm.node_count; k += blockDim.x) {
    const int4 nd = desc[tm.node_begin + k];
    for (int ch = 0; ch < MAX_CHUNKS; ++ch) atomicAdd(&cnt[ch], (unsigned)chunk_count(nd, ch));
  }
  __syncthreads();
  if (threadIdx.x < MAX_CHUNKS) {
    atomicMax(out, cnt[threadIdx.x]);
    per_chunk[t * MAX_CHUNKS + threadIdx.x] = (int32_t)cnt[threadIdx.x];
  }
}

// Chunk-major entry blocks: one CTA per tile, thread per node; per chunk a
// block scan of the nodes' counts gives the header offsets, then each node
// copies its entries of the chunk (they are contiguous in its te-sorted list).
__global__ void k_chunk_blocks(int n_tiles, const TileMeta *meta, const int4 *desc,
                               const uint16_t *entries, int ct, uint16_t *blocks) {
  __shared__ int wsum[32];
  const int t = blockIdx.x;
  const TileMeta tm = meta[t];
  // the own chunks only: the tile kernels compute each element once, by its
  // owner, and never load a block for the halo (cross) elements
  const int nch = (tm.own_count + ct - 1) / ct;
  const int k = threadIdx.x;  // blockDim.x >= node_count (<= 256)
  const bool my = k < tm.node_count;
  const int4 nd = my ? desc[tm.node_begin + k] : make_int4(0, 0, 0, 0);
  int cur = nd.x & ENTRY_OFF_MASK;
  const int H = blk_header(tm.node_count);
  const int lane = k & 31, w = k >> 5, nw = blockDim.x >> 5;
  for (int ch = 0; ch < nch; ++ch) {
    uint16_t *blk = blocks + tm.blk_base + (int64_t)ch * tm.blk_stride;
    const int cnt = my ? chunk_count(nd, ch) : 0;
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    int before = 0;
    for (int u = 0; u < w; ++u) before += wsum[u];
    int total = 0;
    for (int u = 0; u < nw; ++u) total += wsum[u];
    const int base = before + incl - cnt;
    if (my) {
      blk[k] = (uint16_t)base;
      for (int e = 0; e < cnt; ++e) blk[H + base + e] = entries[tm.entry_begin + cur + e];
      cur += cnt;
    }
    if (k == 0) blk[tm.node_count] = (uint16_t)total;
    __syncthreads();
  }
}

// (tile, halo?, element) keys of every patch row: te order = own first, then halo
__global__ void k_pair_keys(int64_t nfree, const int64_t *prefix, const int64_t *elems,
                            const int64_t *slot, const int32_t *tile_of_rank,
                            const int32_t *owner_of, uint64_t *keys, uint8_t *vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nfree;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = r ? prefix[r - 1] : 0, z = prefix[r];
    const int t = tile_of_rank[r];
    for (int64_t q = a; q < z; ++q) {
      const int64_t e = elems[q];
      const uint64_t halo = owner_of[e] != t;
      keys[q] = ((uint64_t)t << 33) | (halo << 32) | (uint64_t)e;
      vals[q] = (uint8_t)(1u << slot[q]);
    }
  }
}

struct OrOp {
  __device__ __forceinline__ uint8_t operator()(uint8_t a, uint8_t b) const { return a | b; }
};

// per tile: [ptr[t], split[t]) own pairs, [split[t], ptr[t+1]) halo pairs
__global__ void k_tile_bounds(int n_tiles, int64_t M, const uint64_t *ukeys, int32_t *ptr,
                              int32_t *split) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= n_tiles; t += gridDim.x * blockDim.x) {
    for (int w = 0; w < 2; ++w) {
      const uint64_t key = ((uint64_t)t << 33) | ((uint64_t)w << 32);
      int64_t lo = 0, hi = M;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (ukeys[mid] < key) lo = mid + 1; else hi = mid;
      }
      (w ? split : ptr)[t] = (int32_t)lo;
    }
  }
}

// Record dictionaries (DICT_MAX in fm_ctx.cuh): one block per tile.  Round k
// takes the first own element no earlier entry matched as entry k and marks
// every element whose record has the same bits; more than DICT_MAX distinct
// records leave the tile uncoded (dict_n = 0).  Deterministic: entries in the
// order of first occurrence.
template <int RB>
__global__ void k_tile_dict(int n_tiles_all, TileMeta *meta, const uint8_t *__restrict__ aos,
                            uint8_t *__restrict__ eidx, uint8_t *__restrict__ dict_rec) {
  constexpr int NQ = RB / 16;
  __shared__ int4 rep[NQ];
  __shared__ int first;
  const int t = blockIdx.x;
  if (t >= n_tiles_all) return;
  const int64_t e0 = meta[t].own_begin;
  const int n = meta[t].own_count;
  constexpr int PER = (MAX_TILE_ELEMS + 255) / 256;  // elements per thread (block of 256)
  unsigned long long pending = 0;  // bit i: element threadIdx.x + 256 i is unmatched
  for (int i = 0; i < PER; ++i)
    if ((int)threadIdx.x + 256 * i < n) pending |= 1ull << i;
  int k = 0;
  for (;; ++k) {
    if (threadIdx.x == 0) first = INT_MAX;
    __syncthreads();
    if (pending) atomicMin(&first, (int)threadIdx.x + 256 * (__ffsll((long long)pending) - 1));
    __syncthreads();
    const int f = first;
    if (f == INT_MAX) break;  // every element matched
    if (k == DICT_MAX) {      // too many distinct records: stream them
      k = 0;
      break;
    }
    if (threadIdx.x < NQ)
      rep[threadIdx.x] = reinterpret_cast<const int4 *>(aos + (e0 + f) * RB)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x < NQ)
      reinterpret_cast<int4 *>(dict_rec + ((int64_t)t * DICT_MAX + k) * RB)[threadIdx.x] =
          rep[threadIdx.x];
    for (unsigned long long m = pending; m; m &= m - 1) {
      const int i = __ffsll((long long)m) - 1;
      const int e = (int)threadIdx.x + 256 * i;
      const int4 *r = reinterpret_cast<const int4 *>(aos + (e0 + e) * RB);
      bool same = true;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int4 x = r[q], y = rep[q];
        same &= x.x == y.x && x.y == y.y && x.z == y.z && x.w == y.w;
      }
      if (same) {
        eidx[e0 + e] = (uint8_t)k;
        pending &= ~(1ull << i);
      }
    }
    __syncthreads();  // rep and first are rewritten next round
  }
  if (threadIdx.x == 0) meta[t].dict_n = k;
}

// Tile element positions ("dealt" order).  The sorted (tile, halo?, element)
// list puts spatial neighbours next to each other, so one node's elements
// would crowd into one or two chunks of ct rows and that chunk's consume
// step would wait on the node thread with the most entries.  Instead the
// r-th element of the own (resp. halo) range [A, B) goes to the r-th position
// of that range enumerated by (position mod ct, position div ct): consecutive
// elements land in consecutive chunks, so each node meets about
// (patch size / chunks) of its elements per chunk.  One block per tile,
// thread s = row s of every chunk.  deal == 0 keeps the sorted order.
__global__ void k_tile_deal(int n_tiles, const int32_t *ptr, const int32_t *split, int ct, int deal,
                            int32_t *tpos) {
  extern __shared__ int32_t cnt_s[];
  const int t = blockIdx.x;
  if (t >= n_tiles) return;
  const int no = split[t] - ptr[t], nh = ptr[t + 1] - split[t];
  for (int part = 0; part < 2; ++part) {
    const int A = part ? no : 0, B = part ? no + nh : no;
    const int64_t base = part ? split[t] : ptr[t];
    if (!deal) {
      for (int r = threadIdx.x; r < B - A; r += blockDim.x) tpos[base + r] = A + r;
      continue;
    }
    // rows s of chunks k with A <= s + ct k < B
    int kmin[4], kcnt[4];
    for (int u = 0; u < 4; ++u) {
      const int s = threadIdx.x + u * blockDim.x;
      kmin[u] = kcnt[u] = 0;
      if (s < ct) {
        const int k0 = A > s ? (A - s + ct - 1) / ct : 0;
        const int k1 = B - 1 >= s ? (B - 1 - s) / ct : -1;
        kmin[u] = k0;
        kcnt[u] = max(0, k1 - k0 + 1);
        cnt_s[s] = kcnt[u];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive scan over rows (ct <= 1024)
      int run = 0;
      for (int s = 0; s < ct; ++s) {
        const int x = cnt_s[s];
        cnt_s[s] = run;
        run += x;
      }
    }
    __syncthreads();
    for (int u = 0; u < 4; ++u) {
      const int s = threadIdx.x + u * blockDim.x;
      if (s < ct)
        for (int j = 0; j < kcnt[u]; ++j) tpos[base + cnt_s[s] + j] = s + ct * (kmin[u] + j);
    }
    __syncthreads();
  }
}

// own elements: storage position own_begin + tpos (storage order = dealt order)
__global__ void k_deal_storage(int64_t M, const uint64_t *ukeys, const int32_t *ptr,
                               const int32_t *own_ptr, const int32_t *tpos, int32_t *s2o) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = ukeys[i];
    if ((k >> 32) & 1) continue;
    const int t = (int)(k >> 33);
    s2o[own_ptr[t] + tpos[i]] = (int32_t)(k & 0xffffffffull);
  }
}

// owned-slot masks in tile element (dealt) order
__global__ void k_deal_flags(int64_t M, const uint64_t *ukeys, const int32_t *ptr,
                             const int32_t *tpos, const uint8_t *umask, uint8_t *flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(ukeys[i] >> 33);
    flags[ptr[t] + tpos[i]] = umask[i];
  }
}

__global__ void k_halo_ids(int64_t M, const uint64_t *ukeys, const int32_t *ptr,
                           const int32_t *split, const int32_t *tpos, const int32_t *halo_begin,
                           const int32_t *o2s, int32_t *halo_ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = ukeys[i];
    if (!((k >> 32) & 1)) continue;
    const int t = (int)(k >> 33);
    const int64_t e = (int64_t)(k & 0xffffffffull);
    halo_ids[halo_begin[t] + tpos[i] - (split[t] - ptr[t])] = o2s[e];
  }
}

__global__ void k_node_desc(int64_t ntn, const int32_t *tile_node_rank, const int32_t *tile_of_rank,
                            const int64_t *prefix, const int64_t *elems, const int64_t *slot,
                            const int32_t *owner_of, const uint64_t *ukeys, const int32_t *ptr,
                            const int32_t *tpos, const int32_t *entry_abs, const int32_t *entry_off,
                            const int32_t *free_node, const int32_t *free_out,
                            const uint8_t *free_mask, int ct, uint16_t *entries, int4 *desc,
                            unsigned long long *overflow) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntn;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int r = tile_node_rank[k];
    const int t = tile_of_rank[r];
    const int64_t a = r ? prefix[r - 1] : 0, z = prefix[r];
    const int64_t lo0 = ptr[t], hi0 = ptr[t + 1];
    uint16_t *out = entries + entry_abs[k];
    int n = 0;
    for (int64_t q = a; q < z; ++q) {
      const int64_t e = elems[q];
      const uint64_t key = ((uint64_t)t << 33) | ((uint64_t)(owner_of[e] != t) << 32) | (uint64_t)e;
      int64_t lo = lo0, hi = hi0;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (ukeys[mid] < key) lo = mid + 1; else hi = mid;
      }
      const bool found = lo < hi0 && ukeys[lo] == key;
      const int64_t te = found ? tpos[lo] : 0;
      if (!found) atomicOr(overflow, 1ull);               // internal: entry not in its tile
      if (te >= MAX_TILE_ELEMS) atomicOr(overflow, 2ull);  // capacity: tile too large
      uint16_t v = (uint16_t)((te << 2) | slot[q]);
      int p = n++;  // insertion sort by te (entries of one node are few)
      while (p > 0 && out[p - 1] > v) {
        out[p] = out[p - 1];
        --p;
      }
      out[p] = v;
    }
    const int fo = free_out[r];  // < 2^31 (checked on the host)
    // entries per chunk of ct tile elements (5 bits x MAX_CHUNKS) packed with the
    // tile-local entry offset (13 bits): x = off | c0..c2 << 13, y = c3..c8
    unsigned long long cc = 0;
    for (int p = 0; p < n; ++p) {
      const int ch = (out[p] >> 2) / ct;
      if (ch >= MAX_CHUNKS || ((cc >> (5 * ch)) & 31ull) == 31ull) {
        atomicOr(overflow, 2ull);  // capacity: > 9 chunks or > 31 entries in one chunk
        continue;
      }
      cc += 1ull << (5 * ch);
    }
    if (entry_off[k] >= (1 << 13)) atomicOr(overflow, 2ull);
    desc[k] = make_int4(entry_off[k] | (int)((cc & 0x7fffull) << 13) |
                            (int)((unsigned)free_mask[r] << DESC_MASK_SHIFT),
                        (int)(cc >> 15), free_node[r], fo);
  }
}

template <class T> static cudaError_t dmalloc(T **p, size_t n, size_t *acc) {
  *acc += n * sizeof(T);
  return cudaMalloc((void **)p, std::max<size_t>(n, 1) * sizeof(T));
}

// FM_DEBUG_MEM=1: device memory in use at the build stages (stderr)
static void memlog(const char *stage, cudaStream_t s) {
  static const bool on = getenv("FM_DEBUG_MEM") != nullptr;
  if (!on) return;
  cudaStreamSynchronize(s);
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  fprintf(stderr, "[fm mem] %-28s %8.2f GB in use\n", stage, (tot - fr) / 1e9);
}

static int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

static ModelArgs model_args(const fm_model *m) {
  ModelArgs a;
  a.kind = m->kind;
  a.p = m->p;
  a.C1 = m->C1;
  a.D1 = m->D1;
  a.e_w = m->p / 2.0;
  a.e_dw = (m->p - 2.0) / 2.0;
  a.eps = 0.0;
#if FM_ABLATE
  static const int ablate = [] {
    const char *e = getenv("FM_TILE_ABLATE");
    return e ? atoi(e) : 0;
  }();
  a.dbg = ablate;
#else
  a.dbg = 0;  // product build: no ablation switches (FM_DBG is 0)
#endif
  return a;
}

static int check_model(const fm_ctx *c, const fm_model *m) {
  FM_ARG(c && m, "null context or model");
  FM_ARG(m->kind == FM_MODEL_PLAPLACE || m->kind == FM_MODEL_NEOHOOKEAN, "unknown model kind");
  FM_ARG(m->dim == c->dim, "model dimension does not match the mesh");
  int d = m->kind == FM_MODEL_NEOHOOKEAN ? m->dim : 1;
  FM_ARG(d == c->d, "model component count does not match the mesh dof partition");
  if (m->kind == FM_MODEL_PLAPLACE) FM_ARG(m->p > 1.0, "p-Laplacian exponent must satisfy p > 1");
  return FM_OK;
}

template <class F> static cudaError_t cub_call(F f, cudaStream_t s) {
  size_t bytes = 0;
  cudaError_t e = f(nullptr, bytes);
  if (e != cudaSuccess) return e;
  Scratch tmp;
  e = tmp.alloc(bytes, s);
  if (e != cudaSuccess) return e;
  return f(tmp.p, bytes);
}

struct TimedLaunch {
  fm_ctx *c;
  cudaStream_t s;
  bool armed;
  TimedLaunch(fm_ctx *ctx, cudaStream_t st) : c(ctx), s(st), armed(ctx->ev_start && ctx->ev_stop) {
    if (armed) cudaEventRecord(c->ev_start, s);
  }
  ~TimedLaunch() {
    if (armed) {
      cudaEventRecord(c->ev_stop, s);
      c->ev_start = c->ev_stop = nullptr;
    }
  }
};

}  // namespace fm

using namespace fm;

extern "C" {

const char *fm_last_error(void) { return g_err.c_str(); }
int fm_version(void) { return 1; }

int fm_ctx_time_next(fm_ctx *c, void *ev_start, void *ev_stop) {
  FM_ARG(c, "null context");
  c->ev_start = reinterpret_cast<cudaEvent_t>(ev_start);
  c->ev_stop = reinterpret_cast<cudaEvent_t>(ev_stop);
  return FM_OK;
}

// One build attempt with the given tiling.  A per-tile capacity limit
// (closure > 2^16 nodes, > 16384 tile elements, > 9 chunks, > 31 entries of
// one node in a chunk, tables beyond shared memory) sets *cap and returns
// FM_INVALID_ARG; fm_ctx_create then retries with smaller tile boxes.
static int ctx_build(const fm_mesh_desc *m, const fm_tiling *tiling, void *stream, fm_ctx **out,
                     bool *cap) {
  *cap = false;
  FM_ARG(m && out, "null argument");
  FM_ARG(m->dim == 2 || m->dim == 3, "dim must be 2 or 3");
  FM_ARG(m->d >= 1 && m->d <= m->dim, "d must be 1..dim");
  FM_ARG(m->ne > 0 && m->nn > 0, "empty mesh");
  FM_ARG(m->ne < (1ll << 31) && m->nn < (1ll << 31) && m->p_total < (1ll << 31),
         "per-GPU mesh must fit 32-bit indices (shard larger meshes)");
  FM_ARG(m->nfree >= 0 && m->nfree * (int64_t)m->d < (1ll << 31),
         "per-GPU free dofs must be < 2^31 (shard larger meshes)");
  cudaStream_t s = as_stream(stream);
  const int dim = m->dim, nv = dim + 1, d = m->d;
  fm_ctx *c = new fm_ctx();
  *out = nullptr;
  auto fail = [&](int code) {
    fm_ctx_destroy(c);
    return code;
  };
  auto capacity = [&](const char *msg) {
    set_error(std::string(msg) + " (tile capacity)");
    *cap = true;
    return fail(FM_INVALID_ARG);
  };
  c->dim = dim;
  c->d = d;
  c->nv = nv;
  c->nn = m->nn;
  c->ne = m->ne;
  c->nfree = m->nfree;
  c->p_total = m->p_total;
  // tile = CTA width: 256 nodes (3D 8x8x4 boxes, 2D 16x16) or 128 (3D 8x4x4)
  int NT = (tiling && tiling->tile_nodes) ? tiling->tile_nodes : 256;
  NT = NT <= 128 ? 128 : 256;
  int box[3] = {dim == 3 ? 8 : 16, dim == 3 ? (NT == 128 ? 4 : 8) : 16, dim == 3 ? 4 : 1};
  if (tiling)
    for (int a = 0; a < 3; ++a)
      if (tiling->box[a] > 0) box[a] = tiling->box[a];
  c->tile_nodes = NT;
  const int64_t nfree = m->nfree, ne = m->ne, T = m->p_total;
  size_t &B = c->bytes;
  {
    c->n_sm = sm_count();
  }

#define CK(x)                                                     \
  do {                                                            \
    cudaError_t _e = (x);                                         \
    if (_e != cudaSuccess) {                                      \
      set_error(std::string(#x) + ": " + cudaGetErrorString(_e)); \
      return fail(FM_CUDA_ERROR);                                 \
    }                                                             \
  } while (0)

  memlog("1. ranks and output offset", s);
  // 1. ranks and output offsets ---------------------------------------------
  CK(dmalloc(&c->rank_of, m->nn, &B));
  CK(dmalloc(&c->free_node, nfree, &B));
  CK(dmalloc(&c->free_out, nfree + 1, &B));
  CK(dmalloc(&c->free_mask, nfree, &B));
  CK(cudaMemsetAsync(c->rank_of, 0xff, m->nn * 4, s));
  {
    Scratch cnt;
    CK(cnt.alloc((nfree + 1) * 4, s));
    CK(cudaMemsetAsync(cnt.p, 0, (nfree + 1) * 4, s));
    if (nfree)
      k_ranks<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, d, m->nodes_minim, m->fixed,
                                                   c->rank_of, c->free_node, c->free_mask,
                                                   cnt.as<int32_t>());
    CK(cudaGetLastError());
    int32_t *cp = cnt.as<int32_t>();
    CK(cub_call([&](void *t, size_t &b) {
      return cub::DeviceScan::ExclusiveSum(t, b, cp, c->free_out, nfree + 1, s);
    }, s));
    int32_t nfd = 0;
    CK(cudaMemcpyAsync(&nfd, c->free_out + nfree, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->nfree_dofs = nfd;
    CK(dmalloc(&c->dof_pos, std::max(nfd, 1), &B));
    CK(launch_dof_pos(nfree, d, c->free_node, c->free_out, c->free_mask, c->dof_pos, s));
    // nodes outside every tile (all components fixed): their b.v goes to the
    // fused path's finalize
    Scratch fl, nsel;
    CK(fl.alloc(m->nn, s));
    CK(nsel.alloc(8, s));
    CK(dmalloc(&c->fixed_nodes, m->nn - nfree + 1, &B));
    k_not_free<<<grid_for(m->nn, 256), 256, 0, s>>>(m->nn, c->rank_of, fl.as<uint8_t>());
    CK(cudaGetLastError());
    {
      cub::CountingInputIterator<int32_t> it(0);
      const uint8_t *flp = fl.as<uint8_t>();
      int32_t *ns = nsel.as<int32_t>();
      int32_t *outp = c->fixed_nodes;
      const int64_t nn = m->nn;
      CK(cub_call([&](void *t, size_t &b) {
        return cub::DeviceSelect::Flagged(t, b, it, flp, outp, ns, nn, s);
      }, s));
      int32_t hn = 0;
      CK(cudaMemcpyAsync(&hn, nsel.p, 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      c->n_fixed_nodes = hn;
    }
  }

  memlog("2. node tiles (Morton", s);
  // 2. node tiles (Morton-ordered boxes) -------------------------------------
  std::vector<int32_t> h_tnp{0};      // tile node ptr
  std::vector<int32_t> h_lens;        // patch length per sorted node
  Scratch s_tnr;                      // sorted ranks = tile node order
  CK(s_tnr.alloc(std::max<int64_t>(nfree, 1) * 4, s));
  if (nfree > 0) {
    double volsum = 0.0;
    {
      Scratch o;
      CK(o.alloc(8, s));
      const double *vp = m->volumes;
      double *op = o.as<double>();
      CK(cub_call([&](void *t, size_t &b) { return cub::DeviceReduce::Sum(t, b, vp, op, ne, s); },
                  s));
      CK(cudaMemcpyAsync(&volsum, o.p, 8, cudaMemcpyDeviceToHost, s));
    }
    unsigned long long hmn[3], hmx[3];
    {
      Scratch mm;
      CK(mm.alloc(48, s));
      CK(cudaMemsetAsync(mm.p, 0xff, 24, s));
      CK(cudaMemsetAsync(mm.as<uint8_t>() + 24, 0, 24, s));
      k_bbox<<<grid_for(nfree, 256, 8 * (int64_t)c->n_sm), 256, 0, s>>>(nfree, dim, m->nodes_minim, m->coords,
                                                        mm.as<unsigned long long>(),
                                                        mm.as<unsigned long long>() + 3);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(hmn, mm.p, 24, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(hmx, mm.as<uint8_t>() + 24, 24, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    const double fact = dim == 3 ? 6.0 : 2.0;
    const double h = std::pow(fact * volsum / (double)ne, 1.0 / dim);
    double x0[3] = {0, 0, 0}, edge[3] = {1, 1, 1};
    for (int a = 0; a < dim; ++a) {
      x0[a] = from_ord(hmn[a]);
      edge[a] = box[a] * h;
      double nb = std::floor((from_ord(hmx[a]) - x0[a] + 0.5 * h) / edge[a]) + 1;
      if (!(nb < 2e6)) {
        set_error("tiling box grid too large (> 2^21 boxes per axis)");
        return fail(FM_INVALID_ARG);  // smaller boxes would not help
      }
    }
    Scratch keys, keys2, vals2, lens;
    CK(keys.alloc(nfree * 8, s));
    CK(keys2.alloc(nfree * 8, s));
    CK(vals2.alloc(nfree * 4, s));
    CK(lens.alloc(nfree * 4, s));
    k_box_keys<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, dim, m->nodes_minim, m->coords, x0[0],
                                                    x0[1], x0[2], edge[0], edge[1], edge[2],
                                                    0.5 * h, keys.as<uint64_t>(),
                                                    s_tnr.as<int32_t>());
    CK(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> dk(keys.as<uint64_t>(), keys2.as<uint64_t>());
    cub::DoubleBuffer<int32_t> dv(s_tnr.as<int32_t>(), vals2.as<int32_t>());
    CK(cub_call([&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, nfree, 0, 63, s);
    }, s));
    if (dv.Current() != s_tnr.as<int32_t>())
      CK(cudaMemcpyAsync(s_tnr.p, dv.Current(), nfree * 4, cudaMemcpyDeviceToDevice, s));
    k_sorted_lengths<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, s_tnr.as<int32_t>(),
                                                          m->p_prefix, lens.as<int32_t>());
    CK(cudaGetLastError());
    std::vector<uint64_t> hkeys(nfree);
    h_lens.resize(nfree);
    CK(cudaMemcpyAsync(hkeys.data(), dk.Current(), nfree * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h_lens.data(), lens.p, nfree * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // split boxes into tiles of <= NT nodes and <= ENTRY_CAP entries
    int64_t i = 0;
    while (i < nfree) {
      int64_t j = i;
      while (j < nfree && hkeys[j] == hkeys[i]) ++j;
      const int64_t cnt = j - i;
      int64_t ent = 0;
      for (int64_t k = i; k < j; ++k) ent += h_lens[k];
      int64_t pieces = std::max<int64_t>((cnt + NT - 1) / NT,
                                         (ent + ENTRY_CAP_DEFAULT - 1) / ENTRY_CAP_DEFAULT);
      for (;; ++pieces) {
        bool ok = true;
        for (int64_t q = 0; q < pieces && ok; ++q) {
          int64_t a = i + cnt * q / pieces, z = i + cnt * (q + 1) / pieces, e2 = 0;
          for (int64_t k = a; k < z; ++k) e2 += h_lens[k];
          ok = (z - a) <= NT && e2 <= ENTRY_CAP_DEFAULT;
        }
        if (ok) break;
      }
      for (int64_t q = 1; q <= pieces; ++q) h_tnp.push_back((int32_t)(i + cnt * q / pieces));
      i = j;
    }
  }
  const int n_tiles = (int)h_tnp.size() - 1;
  c->n_tiles = n_tiles;
  c->max_tile_nodes = 0;
  for (int t = 0; t < n_tiles; ++t)
    c->max_tile_nodes = std::max(c->max_tile_nodes, h_tnp[t + 1] - h_tnp[t]);

  Scratch s_tor, d_tnp;  // tile_of_rank, tile node ptr
  CK(s_tor.alloc(std::max<int64_t>(nfree, 1) * 4, s));
  CK(d_tnp.alloc(h_tnp.size() * 4, s));
  CK(cudaMemcpyAsync(d_tnp.p, h_tnp.data(), h_tnp.size() * 4, cudaMemcpyHostToDevice, s));
  if (nfree)
    k_tile_of_pos<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, n_tiles, d_tnp.as<int32_t>(),
                                                       s_tnr.as<int32_t>(), s_tor.as<int32_t>());
  CK(cudaGetLastError());

  memlog("3. element owners", s);
  // 3. element owners and storage order ---------------------------------------
  Scratch okey, okey2, oval2, owner_of, o2s, own_ptr;
  CK(okey.alloc(ne * 4, s));
  CK(okey2.alloc(ne * 4, s));
  CK(oval2.alloc(ne * 4, s));
  CK(owner_of.alloc(ne * 4, s));
  CK(o2s.alloc(ne * 4, s));
  CK(own_ptr.alloc((n_tiles + 2) * 4, s));
  CK(dmalloc(&c->storage_to_orig, ne, &B));
  k_owner<<<grid_for(ne, 256), 256, 0, s>>>(ne, nv, m->conn, c->rank_of, s_tor.as<int32_t>(),
                                            n_tiles, okey.as<uint32_t>(), c->storage_to_orig,
                                            owner_of.as<int32_t>());
  CK(cudaGetLastError());
  {
    cub::DoubleBuffer<uint32_t> dk(okey.as<uint32_t>(), okey2.as<uint32_t>());
    cub::DoubleBuffer<int32_t> dv(c->storage_to_orig, oval2.as<int32_t>());
    const int end_bit = std::max(1, bits_for((uint64_t)n_tiles));
    CK(cub_call([&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, ne, 0, end_bit, s);
    }, s));
    if (dv.Current() != c->storage_to_orig)
      CK(cudaMemcpyAsync(c->storage_to_orig, dv.Current(), ne * 4, cudaMemcpyDeviceToDevice, s));
    k_lower_bounds_u32<<<grid_for(n_tiles + 2, 256), 256, 0, s>>>(n_tiles + 1, ne, dk.Current(),
                                                                  own_ptr.as<int32_t>());
    CK(cudaGetLastError());
  }
  okey.reset();  // owner keys and sort buffers are done
  okey2.reset();
  oval2.reset();
  std::vector<int32_t> h_own(n_tiles + 2);
  CK(cudaMemcpyAsync(h_own.data(), own_ptr.p, (n_tiles + 2) * 4, cudaMemcpyDeviceToHost, s));

  memlog("4. tile element lists", s);
  // 4. tile element lists (own + halo) ----------------------------------------
  int64_t M = 0;
  Scratch ukeys, umask, tptr, tsplit, tpos;
  CK(tptr.alloc((n_tiles + 1) * 4, s));
  CK(tsplit.alloc((n_tiles + 1) * 4, s));
  std::vector<int32_t> h_ptr(n_tiles + 1, 0), h_split(n_tiles + 1, 0);
  if (nfree > 0) {
    Scratch pk, pk2, pv, pv2, nsel;
    CK(pk.alloc(T * 8, s));
    CK(pk2.alloc(T * 8, s));
    CK(pv.alloc(T, s));
    CK(pv2.alloc(T, s));
    k_pair_keys<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, m->p_prefix, m->p_elems, m->p_slot,
                                                     s_tor.as<int32_t>(), owner_of.as<int32_t>(),
                                                     pk.as<uint64_t>(), pv.as<uint8_t>());
    CK(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> dk(pk.as<uint64_t>(), pk2.as<uint64_t>());
    cub::DoubleBuffer<uint8_t> dv(pv.as<uint8_t>(), pv2.as<uint8_t>());
    const int end_bit = 33 + bits_for((uint64_t)n_tiles);
    CK(cub_call([&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, T, 0, end_bit, s);
    }, s));
    CK(ukeys.alloc(T * 8, s));
    CK(umask.alloc(T, s));
    CK(nsel.alloc(8, s));
    uint64_t *uk = ukeys.as<uint64_t>();
    uint8_t *um = umask.as<uint8_t>();
    int64_t *ns = nsel.as<int64_t>();
    CK(cub_call([&](void *t, size_t &b) {
      return cub::DeviceReduce::ReduceByKey(t, b, dk.Current(), uk, dv.Current(), um, ns, OrOp(),
                                            T, s);
    }, s));
    CK(cudaMemcpyAsync(&M, nsel.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    memlog("4. after patch-pair sort", s);
    k_tile_bounds<<<grid_for(n_tiles + 1, 256), 256, 0, s>>>(n_tiles, M, uk, tptr.as<int32_t>(),
                                                             tsplit.as<int32_t>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h_ptr.data(), tptr.p, (n_tiles + 1) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h_split.data(), tsplit.p, (n_tiles + 1) * 4, cudaMemcpyDeviceToHost, s));
    // dealt tile element order; own elements are stored in it (FM_TILE_DEAL=0: sorted order)
    static const int deal = [] {
      const char *e = getenv("FM_TILE_DEAL");
      return e ? atoi(e) : 1;
    }();
    CK(tpos.alloc(M * 4, s));
    k_tile_deal<<<n_tiles, 256, NT * 4, s>>>(n_tiles, tptr.as<int32_t>(), tsplit.as<int32_t>(),
                                             NT, deal, tpos.as<int32_t>());
    CK(cudaGetLastError());
    k_deal_storage<<<grid_for(M, 256), 256, 0, s>>>(M, uk, tptr.as<int32_t>(),
                                                    own_ptr.as<int32_t>(), tpos.as<int32_t>(),
                                                    c->storage_to_orig);
    CK(cudaGetLastError());
  }
  k_inverse<<<grid_for(ne, 256), 256, 0, s>>>(ne, c->storage_to_orig, o2s.as<int32_t>());
  CK(cudaGetLastError());
  {
    Scratch bad;
    CK(bad.alloc(8, s));
    CK(cudaMemsetAsync(bad.p, 0xff, 8, s));
    if (dim == 3)
      k_dphi0_check<3><<<grid_for(ne, 256), 256, 0, s>>>(ne, m->dphi, bad.as<unsigned long long>());
    else
      k_dphi0_check<2><<<grid_for(ne, 256), 256, 0, s>>>(ne, m->dphi, bad.as<unsigned long long>());
    CK(cudaGetLastError());
    unsigned long long hb = 0;
    CK(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hb != ~0ull) {
      set_error("element " + std::to_string(hb) +
                ": dphi[m][k, 0] differs from -dphi[m][k, 1:].sum() (compute_p1_gradients, "
                "mesh.py:100-101, makes them equal; the records store only columns 1..dim)");
      return fail(FM_INVALID_ARG);
    }
  }
  const int rb = dim == 3 ? RecBytes<3>::value : RecBytes<2>::value;
  CK(dmalloc(&c->aos, (size_t)ne * rb, &B));
  CK(dmalloc(&c->loc, ne + 2, &B));
  CK(cudaMemsetAsync(c->loc, 0, (ne + 2) * 8, s));
  // global connectivity in storage order: only the 2D streaming energy kernel
  // reads it (3D energy runs through the tile pipeline: 16 B per element saved)
  CK(dmalloc(&c->conn4, dim == 2 ? ne : 1, &B));
  if (dim == 3)
    k_build_aos<3><<<grid_for(ne, 256), 256, 0, s>>>(ne, c->storage_to_orig, m->conn, m->volumes,
                                                     m->dphi, c->aos, c->conn4);
  else
    k_build_aos<2><<<grid_for(ne, 256), 256, 0, s>>>(ne, c->storage_to_orig, m->conn, m->volumes,
                                                     m->dphi, c->aos, c->conn4);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  const int64_t n_orph = (int64_t)ne - h_own[n_tiles];
  // host-side tile metadata
  std::vector<TileMeta> hm;
  std::vector<int32_t> h_halo_begin(n_tiles + 1, 0);
  int64_t halo_total = 0, entry_total = 0;
  std::vector<int32_t> h_entry_off(std::max<int64_t>(nfree, 1)), h_entry_abs(std::max<int64_t>(nfree, 1));
  c->max_tile_elems = 0;
  c->max_tile_entries = 0;
  int max_halo = 0;
  for (int t = 0; t < n_tiles; ++t) {
    TileMeta tm{};
    tm.own_begin = h_own[t];
    tm.own_count = h_own[t + 1] - h_own[t];
    if (tm.own_count != h_split[t] - h_ptr[t]) {
      set_error("internal error: owner partition and tile element lists disagree");
      return fail(FM_CUDA_ERROR);
    }
    tm.halo_count = h_ptr[t + 1] - h_split[t];
    tm.halo_begin = (int)halo_total;
    h_halo_begin[t] = (int)halo_total;
    halo_total += (tm.halo_count + 3) / 4 * 4;
    tm.node_begin = h_tnp[t];
    tm.node_count = h_tnp[t + 1] - h_tnp[t];
    tm.entry_begin = (int)entry_total;
    int off = 0;
    for (int k = h_tnp[t]; k < h_tnp[t + 1]; ++k) {
      h_entry_off[k] = off;
      h_entry_abs[k] = (int)entry_total + off;
      off += h_lens[k];
    }
    tm.entry_count = off;
    entry_total += (off + 7) / 8 * 8;
    tm.elem_begin = h_ptr[t];
    hm.push_back(tm);
    c->max_tile_elems = std::max(c->max_tile_elems, tm.own_count + tm.halo_count);
    c->max_tile_entries = std::max(c->max_tile_entries, off);
    max_halo = std::max(max_halo, tm.halo_count);
  }
  if (c->max_tile_elems > MAX_TILE_ELEMS) {
    return capacity("a node tile touches more than 16384 elements");
  }
  const int OT = 4 * CONSUMERS;  // orphan elements per J-only tile
  for (int64_t o = 0; o < n_orph; o += OT) {
    TileMeta tm{};
    tm.own_begin = (int)(h_own[n_tiles] + o);
    tm.own_count = (int)std::min<int64_t>(OT, n_orph - o);
    tm.halo_begin = (int)halo_total;
    tm.node_begin = h_tnp.back();
    tm.entry_begin = (int)entry_total;
    tm.elem_begin = (int)M;
    hm.push_back(tm);
  }
  c->n_tiles_all = (int)hm.size();
  c->n_tile_elems = M;
  c->entry_cap = (c->max_tile_entries + 7) / 8 * 8;
  (void)max_halo;
  CK(dmalloc(&c->halo_ids, halo_total + 4, &B));
  CK(dmalloc(&c->halo_loc, halo_total + 4, &B));
  CK(cudaMemsetAsync(c->halo_loc, 0, (halo_total + 4) * 8, s));

  memlog("4b. node closures", s);
  // 4b. node closures of every tile and the 16-bit closure indices ---------------
  {
    const int NTA = c->n_tiles_all;
    const int64_t NI = M + n_orph;
    // keys (tile << 32 | node) of the tile elements' nodes, sorted and
    // de-duplicated in batches of whole tiles (tile-major keys: the batches'
    // unique runs concatenate to the global result) so the sort buffers stay
    // small at config-5 scale; at most FM_CLOSURE_BATCH (default 2^25) elements
    int64_t cap = 1ll << 25;
    if (const char *e = getenv("FM_CLOSURE_BATCH")) cap = std::max<int64_t>(1, atoll(e));
    std::vector<int64_t> cuts{0};  // batch boundaries on tile boundaries
    {
      std::vector<int64_t> tb;  // tile starts in the element index space
      for (int t = 1; t < n_tiles; ++t) tb.push_back(h_ptr[t]);
      if (n_tiles > 0 && M < NI) tb.push_back(M);
      for (int64_t o = OT; o < n_orph; o += OT) tb.push_back(M + o);
      tb.push_back(NI);
      int64_t last = 0;
      for (size_t k = 0; k < tb.size(); ++k) {
        const bool end = k + 1 == tb.size();
        if (end || tb[k + 1] - cuts.back() > cap) {
          if (tb[k] > cuts.back()) cuts.push_back(tb[k]);
        }
        last = tb[k];
      }
      if (cuts.back() != last) cuts.push_back(last);
    }
    int64_t bmax = 0;
    for (size_t k = 0; k + 1 < cuts.size(); ++k) bmax = std::max(bmax, cuts[k + 1] - cuts[k]);
    const int64_t NKB = std::max<int64_t>(bmax * nv, 1);
    Scratch ck, ck2, nsel, cstart, cu;
    CK(nsel.alloc(8, s));
    CK(cstart.alloc((NTA + 1) * 4, s));
    const int end_bit = 32 + bits_for((uint64_t)NTA);
    int64_t C = 0;
    {
      CK(ck.alloc(NKB * 8, s));
      CK(ck2.alloc(NKB * 8, s));
      std::vector<std::unique_ptr<Scratch>> parts;
      std::vector<int64_t> part_n;
      for (size_t k = 0; k + 1 < cuts.size(); ++k) {
        const int64_t i0 = cuts[k], i1 = cuts[k + 1], nk = (i1 - i0) * nv;
        k_closure_keys<<<grid_for(i1 - i0, 256), 256, 0, s>>>(
            i0, i1, M, ukeys.as<uint64_t>(), h_own[n_tiles], n_tiles, OT, c->storage_to_orig,
            m->conn, nv, ck.as<uint64_t>());
        CK(cudaGetLastError());
        cub::DoubleBuffer<uint64_t> dk(ck.as<uint64_t>(), ck2.as<uint64_t>());
        CK(cub_call([&](void *t, size_t &b) {
          return cub::DeviceRadixSort::SortKeys(t, b, dk, nk, 0, end_bit, s);
        }, s));
        uint64_t *dst = dk.Current() == ck.as<uint64_t>() ? ck2.as<uint64_t>() : ck.as<uint64_t>();
        CK(cub_call([&](void *t, size_t &b) {
          return cub::DeviceSelect::Unique(t, b, dk.Current(), dst, nsel.as<int64_t>(), nk, s);
        }, s));
        int64_t cb_n = 0;
        CK(cudaMemcpyAsync(&cb_n, nsel.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        parts.emplace_back(new Scratch);
        CK(parts.back()->alloc(std::max<int64_t>(cb_n, 1) * 8, s));
        CK(cudaMemcpyAsync(parts.back()->p, dst, cb_n * 8, cudaMemcpyDeviceToDevice, s));
        part_n.push_back(cb_n);
        C += cb_n;
      }
      memlog("4b. after closure sorts", s);
      CK(cu.alloc(std::max<int64_t>(C, 1) * 8, s));
      int64_t off = 0;
      for (size_t k = 0; k < parts.size(); ++k) {
        CK(cudaMemcpyAsync(cu.as<uint64_t>() + off, parts[k]->p, part_n[k] * 8,
                           cudaMemcpyDeviceToDevice, s));
        off += part_n[k];
      }
    }
    uint64_t *cuk = cu.as<uint64_t>();
    k_lower_bounds_u64<<<grid_for(NTA + 1, 256), 256, 0, s>>>(NTA, C, cuk, 32,
                                                              cstart.as<int32_t>());
    CK(cudaGetLastError());
    std::vector<int32_t> h_cs(NTA + 1), h_cb(NTA + 1);
    CK(cudaMemcpyAsync(h_cs.data(), cstart.p, (NTA + 1) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int64_t ctot = 0;
    c->clo_cap = 0;
    for (int t = 0; t < NTA; ++t) {
      const int cnt = h_cs[t + 1] - h_cs[t];
      hm[t].clo_begin = (int)ctot;
      hm[t].clo_count = cnt;
      h_cb[t] = (int)ctot;
      ctot += (cnt + 3) / 4 * 4;
      c->clo_cap = std::max(c->clo_cap, cnt);
    }
    h_cb[NTA] = (int)ctot;
    c->clo_cap = (c->clo_cap + 3) / 4 * 4;
    if (c->clo_cap > 65536) {
      return capacity("a tile's node closure exceeds 65536 nodes");
    }
    CK(dmalloc(&c->closure, ctot + 4, &B));
    CK(cudaMemsetAsync(c->closure, 0, (ctot + 4) * 4, s));
    Scratch cb, hb, ovf;
    CK(cb.alloc((NTA + 1) * 4, s));
    CK(hb.alloc((n_tiles + 1) * 4, s));
    CK(ovf.alloc(8, s));
    CK(cudaMemsetAsync(ovf.p, 0, 8, s));
    CK(cudaMemcpyAsync(cb.p, h_cb.data(), (NTA + 1) * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(hb.p, h_halo_begin.data(), (n_tiles + 1) * 4, cudaMemcpyHostToDevice, s));
    k_closure_ids<<<grid_for(C, 256), 256, 0, s>>>(C, cuk, cstart.as<int32_t>(), cb.as<int32_t>(),
                                                   c->closure);
    if (dim == 3)
      k_fill_loc<3><<<grid_for(M + n_orph, 256), 256, 0, s>>>(
          M, ukeys.as<uint64_t>(), n_orph, h_own[n_tiles], n_tiles, OT, c->storage_to_orig,
          o2s.as<int32_t>(), m->conn, cuk, cstart.as<int32_t>(), tptr.as<int32_t>(),
          tsplit.as<int32_t>(), tpos.as<int32_t>(), hb.as<int32_t>(), c->loc, c->halo_loc,
          ovf.as<unsigned long long>());
    else
      k_fill_loc<2><<<grid_for(M + n_orph, 256), 256, 0, s>>>(
          M, ukeys.as<uint64_t>(), n_orph, h_own[n_tiles], n_tiles, OT, c->storage_to_orig,
          o2s.as<int32_t>(), m->conn, cuk, cstart.as<int32_t>(), tptr.as<int32_t>(),
          tsplit.as<int32_t>(), tpos.as<int32_t>(), hb.as<int32_t>(), c->loc, c->halo_loc,
          ovf.as<unsigned long long>());
    CK(cudaGetLastError());
    unsigned long long h_ovf = 0;
    CK(cudaMemcpyAsync(&h_ovf, ovf.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h_ovf) {
      set_error("internal error: element node missing from its tile closure");
      return fail(FM_CUDA_ERROR);
    }
  }
  CK(dmalloc(&c->meta, hm.size(), &B));
  CK(cudaMemcpyAsync(c->meta, hm.data(), hm.size() * sizeof(TileMeta), cudaMemcpyHostToDevice, s));
  CK(dmalloc(&c->flags, M + 16, &B));
  CK(dmalloc(&c->node_desc, std::max<int64_t>(nfree, 1), &B));
  if (c->max_tile_elems > MAX_CHUNKS * c->tile_nodes) {
    return capacity("a node tile has more than 9 chunks of elements");
  }
  CK(dmalloc(&c->node_entries, entry_total + 8, &B));
  c->n_node_entries = entry_total;
  CK(cudaMemsetAsync(c->halo_ids, 0, (halo_total + 4) * 4, s));
  CK(cudaMemsetAsync(c->node_entries, 0, (entry_total + 8) * 2, s));
  if (M) {
    k_deal_flags<<<grid_for(M, 256), 256, 0, s>>>(M, ukeys.as<uint64_t>(), tptr.as<int32_t>(),
                                                  tpos.as<int32_t>(), umask.as<uint8_t>(),
                                                  c->flags);
    CK(cudaGetLastError());
    Scratch hb;
    CK(hb.alloc((n_tiles + 1) * 4, s));
    CK(cudaMemcpyAsync(hb.p, h_halo_begin.data(), (n_tiles + 1) * 4, cudaMemcpyHostToDevice, s));
    k_halo_ids<<<grid_for(M, 256), 256, 0, s>>>(M, ukeys.as<uint64_t>(), tptr.as<int32_t>(),
                                                 tsplit.as<int32_t>(), tpos.as<int32_t>(),
                                                 hb.as<int32_t>(), o2s.as<int32_t>(),
                                                 c->halo_ids);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
  }
  o2s.reset();
  umask.reset();

  memlog("5. node descriptors", s);
  // 5. node descriptors and entries ---------------------------------------------
  if (nfree > 0) {
    Scratch eoff, eabs, ovf;
    CK(eoff.alloc(nfree * 4, s));
    CK(eabs.alloc(nfree * 4, s));
    CK(ovf.alloc(8, s));
    CK(cudaMemsetAsync(ovf.p, 0, 8, s));
    CK(cudaMemcpyAsync(eoff.p, h_entry_off.data(), nfree * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(eabs.p, h_entry_abs.data(), nfree * 4, cudaMemcpyHostToDevice, s));
    k_node_desc<<<grid_for(nfree, 256), 256, 0, s>>>(
        nfree, s_tnr.as<int32_t>(), s_tor.as<int32_t>(), m->p_prefix, m->p_elems, m->p_slot,
        owner_of.as<int32_t>(), ukeys.as<uint64_t>(), tptr.as<int32_t>(), tpos.as<int32_t>(),
        eabs.as<int32_t>(),
        eoff.as<int32_t>(), c->free_node, c->free_out, c->free_mask, c->tile_nodes,
        c->node_entries, c->node_desc, ovf.as<unsigned long long>());
    CK(cudaGetLastError());
    unsigned long long h_ovf = 0;
    CK(cudaMemcpyAsync(&h_ovf, ovf.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h_ovf & 1) {
      set_error("internal error: patch entry not found in its tile");
      return fail(FM_CUDA_ERROR);
    }
    if (h_ovf) return capacity("a tile node has more than 31 patch elements in one chunk of "
                               "its tile, or a tile more than 8192 node entries");
    ukeys.reset();  // tile element lists: consumed by the descriptors / entries
    tpos.reset();
    owner_of.reset();
    Scratch cmax, pch;
    CK(cmax.alloc(4, s));
    CK(pch.alloc((size_t)n_tiles * MAX_CHUNKS * 4, s));
    CK(cudaMemsetAsync(cmax.p, 0, 4, s));
    k_chunk_entry_max<<<n_tiles, 256, 0, s>>>(n_tiles, c->meta, c->node_desc,
                                               cmax.as<unsigned int>(), pch.as<int32_t>());
    CK(cudaGetLastError());
    unsigned int h_cmax = 0;
    std::vector<int32_t> h_pch((size_t)n_tiles * MAX_CHUNKS);
    CK(cudaMemcpyAsync(&h_cmax, cmax.p, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h_pch.data(), pch.p, h_pch.size() * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    (void)h_cmax;

    // 5a. chunk-major entry blocks (the tile kernels load a chunk's block with
    // its records): per tile a fixed stride = its largest block
    int64_t blk_total = 0;
    c->blk_cap = 0;
    for (int t = 0; t < n_tiles; ++t) {
      const int nch = (hm[t].own_count + c->tile_nodes - 1) / c->tile_nodes;  // own chunks
      int mx = 0;
      for (int ch = 0; ch < nch; ++ch) mx = std::max(mx, h_pch[(size_t)t * MAX_CHUNKS + ch]);
      const int stride = blk_header(hm[t].node_count) + (mx + 7) / 8 * 8;
      hm[t].blk_stride = stride;
      hm[t].blk_base = blk_total;
      blk_total += (int64_t)nch * stride;
      c->blk_cap = std::max(c->blk_cap, stride);
    }
    CK(cudaMemcpyAsync(c->meta, hm.data(), hm.size() * sizeof(TileMeta), cudaMemcpyHostToDevice, s));
    c->blk_total = blk_total;
    CK(dmalloc(&c->chunk_blocks, blk_total + 8, &B));
    CK(cudaMemsetAsync(c->chunk_blocks, 0, (blk_total + 8) * 2, s));
    k_chunk_blocks<<<n_tiles, c->tile_nodes, 0, s>>>(n_tiles, c->meta, c->node_desc,
                                                      c->node_entries, c->tile_nodes,
                                                      c->chunk_blocks);
    CK(cudaGetLastError());

    // 5b. cross-tile exchange of the fused exact kernel ---------------------------
    Scratch stile, xcnt, xoff, xk, xk2, xv, xv2, xsum;
    CK(stile.alloc(ne * 4, s));
    CK(cudaMemsetAsync(stile.p, 0, ne * 4, s));
    k_storage_tile<<<std::min(n_tiles, 65535), 256, 0, s>>>(n_tiles, own_ptr.as<int32_t>(),
                                                             stile.as<int32_t>());
    CK(cudaGetLastError());
    CK(dmalloc(&c->node_xbase, nfree + 1, &B));
    CK(dmalloc(&c->node_xn, nfree, &B));
    k_cross_count<<<grid_for(nfree, 256), 256, 0, s>>>(
        nfree, s_tnr.as<int32_t>(), s_tor.as<int32_t>(), c->meta, c->node_desc, c->node_entries,
        eabs.as<int32_t>(), c->node_xbase, c->node_xn);
    CK(cudaGetLastError());
    CK(xoff.alloc((nfree + 1) * 4, s));
    CK(xsum.alloc(8, s));
    {
      const int32_t *in = c->node_xn;
      int32_t *outp = xoff.as<int32_t>();
      CK(cub_call([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, in, outp, nfree, s);
      }, s));
      int32_t *tot = xsum.as<int32_t>();
      CK(cub_call([&](void *t, size_t &b) { return cub::DeviceReduce::Sum(t, b, in, tot, nfree, s); },
                  s));
    }
    int32_t hX = 0;
    CK(cudaMemcpyAsync(&hX, xsum.p, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int64_t X = hX;
    c->n_cross = X;
    CK(cudaMemcpyAsync(xoff.as<int32_t>() + nfree, xsum.p, 4, cudaMemcpyDeviceToDevice, s));
    CK(xk.alloc(std::max<int64_t>(X, 1) * 8, s));
    CK(xk2.alloc(std::max<int64_t>(X, 1) * 8, s));
    CK(xv.alloc(std::max<int64_t>(X, 1) * 4, s));
    CK(xv2.alloc(std::max<int64_t>(X, 1) * 4, s));
    k_cross_items<<<grid_for(nfree, 256), 256, 0, s>>>(
        nfree, s_tnr.as<int32_t>(), s_tor.as<int32_t>(), c->meta, c->node_entries, c->node_xbase,
        c->node_xn, xoff.as<int32_t>(), c->halo_ids, stile.as<int32_t>(), xk.as<uint64_t>(),
        xv.as<int32_t>());
    CK(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> dk(xk.as<uint64_t>(), xk2.as<uint64_t>());
    cub::DoubleBuffer<int32_t> dv(xv.as<int32_t>(), xv2.as<int32_t>());
    if (X) {
      const int end_bit = 16 + bits_for((uint64_t)n_tiles);
      CK(cub_call([&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, X, 0, end_bit, s);
      }, s));
    }
    CK(dmalloc(&c->xkey, X + 8, &B));
    CK(dmalloc(&c->xpos, X + 8, &B));
    CK(dmalloc(&c->xchunk, (size_t)n_tiles * XCH_STRIDE, &B));
    CK(dmalloc(&c->xbuf, (size_t)(X + 8) * d, &B));
    // the finishing pass reads each node's exchange slots from its dense offset
    CK(cudaMemcpyAsync(c->node_xbase, xoff.p, (nfree + 1) * 4, cudaMemcpyDeviceToDevice, s));
    // nodes with cross entries: flagged in their descriptor (the tile kernel
    // then leaves a dense partial sum instead of g), outputs for the finish
    CK(dmalloc(&c->node_outw, nfree, &B));
    CK(dmalloc(&c->node_fmask, nfree, &B));
    CK(dmalloc(&c->partial, (size_t)nfree * d, &B));
    k_mark_cross<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, c->node_xn, c->node_desc,
                                                       c->node_outw, c->node_fmask);
    CK(cudaGetLastError());
    // the finishing pass visits only the tile nodes with cross entries
    {
      Scratch xf, xs, xt;
      CK(xf.alloc((nfree + 1) * 4, s));
      CK(xs.alloc((nfree + 1) * 4, s));
      CK(xt.alloc(8, s));
      k_nonzero_flags<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, c->node_xn, xf.as<int32_t>());
      CK(cudaGetLastError());
      int32_t *fl = xf.as<int32_t>(), *ps = xs.as<int32_t>();
      CK(cub_call([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, fl, ps, nfree + 1, s);
      }, s));
      int32_t hn = 0;
      CK(cudaMemcpyAsync(&hn, ps + nfree, 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      c->n_xnodes = hn;
      CK(dmalloc(&c->xnodes, std::max(hn, 1), &B));
      k_scatter_flagged<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, fl, ps, c->xnodes);
      CK(cudaGetLastError());
      CK(dmalloc(&c->xdesc, std::max(hn, 1), &B));
      k_xdesc<<<grid_for(std::max(hn, 1), 256), 256, 0, s>>>(hn, c->xnodes, c->node_xbase,
                                                            c->node_outw, c->node_fmask,
                                                            c->xdesc);
      CK(cudaGetLastError());
    }
    CK(dmalloc(&c->node_clo, nfree + 8, &B));
    k_node_clo<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, s_tnr.as<int32_t>(), s_tor.as<int32_t>(),
                                                     c->meta, c->node_desc, c->closure,
                                                     c->node_clo);
    CK(cudaGetLastError());
    if (X) {
      k_low16<<<grid_for(X, 256), 256, 0, s>>>(X, dk.Current(), c->xkey);
      // the owner tiles write item i to xbuf slot i (coalesced); the finishing
      // pass reads node-major slot p through xinv[p] = i
      k_inverse<<<grid_for(X, 256), 256, 0, s>>>(X, dv.Current(), c->xpos);
      CK(cudaGetLastError());
    }
    k_xchunk<<<grid_for((int64_t)n_tiles * XCH_STRIDE, 256), 256, 0, s>>>(
        n_tiles, c->tile_nodes, X, dk.Current(), c->xchunk);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
  }

  // record dictionaries (DICT_MAX): per tile the distinct own-element records
  // and one slot byte per element; FM_TILE_DICT=0 streams the records of every tile
  {
    const char *de = getenv("FM_TILE_DICT");  // read per build (tests toggle it)
    const bool use_dict = !de || atoi(de) != 0;
    const int rbz = dim == 3 ? RecBytes<3>::value : RecBytes<2>::value;
    CK(dmalloc(&c->eidx, (size_t)ne + 32, &B));
    CK(cudaMemsetAsync(c->eidx, 0, (size_t)ne + 32, s));
    CK(dmalloc(&c->dict_rec, (size_t)std::max(1, c->n_tiles_all) * DICT_MAX * rbz, &B));
    c->n_dict_tiles = 0;
    if (use_dict && c->n_tiles_all > 0) {
      static_assert(MAX_TILE_ELEMS <= 64 * 256, "k_tile_dict: one pending bit per element");
      if (dim == 3)
        k_tile_dict<RecBytes<3>::value><<<c->n_tiles_all, 256, 0, s>>>(c->n_tiles_all, c->meta,
                                                                      c->aos, c->eidx, c->dict_rec);
      else
        k_tile_dict<RecBytes<2>::value><<<c->n_tiles_all, 256, 0, s>>>(c->n_tiles_all, c->meta,
                                                                      c->aos, c->eidx, c->dict_rec);
      CK(cudaGetLastError());
      std::vector<TileMeta> hm2(c->n_tiles_all);
      CK(cudaMemcpyAsync(hm2.data(), c->meta, hm2.size() * sizeof(TileMeta),
                         cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      bool all = true;
      for (const TileMeta &tm : hm2) {
        c->n_dict_tiles += tm.dict_n > 0;
        all &= tm.dict_n > 0 || tm.own_count == 0;
      }
      c->all_coded = all;  // the stages then hold slot bytes, not records
#if !FM_WS_KERNEL
      // no kernel reads the full records of a coded 3D context any more (its
      // energy runs through the tile pipeline too): 80 B per element back
      if (all && dim == 3) {
        CK(cudaFree(c->aos));
        c->aos = nullptr;
        B -= (size_t)ne * rbz;
      }
#endif
    }
  }

  // CTAs per SM: registers allow 4 x 128 / 2 x 256 threads (3D; 2D: 8 / 4,
  // tile_exact_minb); shared memory
  // (228 KB per SM, 1 KB reserved per CTA) decides, preferring two node-value
  // buffers (one tile of lead) when that does not cost a CTA
  {
    const int regs_cap = tile_exact_minb(dim, c->tile_nodes);
    auto fit = [&](int nb, int tb) {
      const size_t sm = tile_exact_smem(dim, d, c->blk_cap, c->clo_cap, c->tile_nodes, nb, tb, 0,
                                        c->all_coded);
      return sm > 227 * 1024 ? 0 : std::min<int>(regs_cap, (int)(228 * 1024 / (sm + 1024)));
    };
    // most CTAs per SM first, then the next tile's tables a tile ahead
    // (tb = 2); node values a tile ahead (nb = 2) measured better in 2D (many
    // small tiles, config 2/3) and, with streamed records, worse in 3D (config
    // 4: 0.874 vs 0.861 ms: 225 KB of shared memory leave no L1); with
    // dictionary-coded records the stages are small and nb = 2 wins there too
    // (config 4: 0.805 vs 0.818 ms); FM_TILE_CFG="nb,tb" forces a variant
    const int nb_pref = (dim == 2 || c->all_coded) ? 2 : 1;
    int best = -1;
    for (int nb = 2; nb >= 1; --nb)
      for (int tb = 2; tb >= 1; --tb) {
        const int f = fit(nb, tb);
        const int score = f * 8 + (tb == 2) * 2 + (nb == nb_pref);
        if (f > 0 && score > best) {
          best = score;
          c->node_bufs = nb;
          c->table_bufs = tb;
          c->ctas_per_sm = f;
        }
      }
    if (const char *e = getenv("FM_TILE_CFG")) {
      int nb = 0, tb = 0;
      if (sscanf(e, "%d,%d", &nb, &tb) == 2 && fit(nb, tb) > 0) {
        c->node_bufs = nb;
        c->table_bufs = tb;
        c->ctas_per_sm = fit(nb, tb);
      }
    }
    if (best < 0) {
      return capacity("tile tables exceed shared memory");
    }
#if FM_WS_KERNEL
    // experiment builds only (tools/ws_check.sh): the warp-specialised kernel of
    // fm_eval_ws.cu (one 896-thread CTA per SM) for FM_WS=1, 256-node tiles
    // whose stages fit the SM's shared memory
    c->ws = false;
    if (const char *e = getenv("FM_WS")) c->ws = atoi(e) != 0;
    if (c->tile_nodes != 256 || tile_ws_smem(dim, d, c->blk_cap, c->clo_cap) == 0)
      c->ws = false;
#endif
  }

  // build-only tables: the kernels read the chunk entry blocks instead of the
  // node-major entry lists, no kernel reads the owned-slot flags or the halo
  // lists (every element is computed once, by its owner tile), and the
  // finishing pass reads the packed xdesc instead of the per-node arrays
  CK(cudaStreamSynchronize(s));
  for (void **p : {(void **)&c->node_entries, (void **)&c->flags, (void **)&c->node_xbase,
                   (void **)&c->node_xn, (void **)&c->node_outw, (void **)&c->node_fmask,
                   (void **)&c->xnodes, (void **)&c->halo_ids, (void **)&c->halo_loc}) {
    if (*p) CK(cudaFree(*p));
    *p = nullptr;
  }

  memlog("scratch", s);
  // scratch ------------------------------------------------------------------
  c->n_energy_blocks = c->n_sm * 8;
  c->n_dot_blocks = c->n_sm * 2;
  c->n_part = std::max(c->n_sm, c->n_energy_blocks);
  CK(dmalloc(&c->jpart, c->n_part, &B));
  CK(dmalloc(&c->dotpart, std::max(c->n_part, c->n_dot_blocks), &B));
  CK(dmalloc(&c->status, 2, &B));
  CK(dmalloc(&c->fpart, finish_max_blocks(), &B));
  CK(dmalloc(&c->ticket, 1, &B));
  CK(cudaMemsetAsync(c->ticket, 0, sizeof(unsigned int), s));
  unsigned long long init[2] = {0ull, ~0ull};
  CK(cudaMemcpyAsync(c->status, init, 16, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
#undef CK

  fm_ctx_stats &st = c->stats;
  st.n_tiles = n_tiles;
  st.n_orphan_tiles = c->n_tiles_all - n_tiles;
  st.tile_elems_total = M + n_orph;
  st.node_entries_total = c->n_node_entries;
  st.max_tile_elems = c->max_tile_elems;
  st.max_tile_entries = c->max_tile_entries;
  st.bytes_device = (int64_t)c->bytes;
  st.redundancy = (double)(M + n_orph) / (double)ne;
  st.tile_threads = c->tile_nodes;
  st.ctas_per_sm = c->ctas_per_sm;
  st.node_bufs = c->node_bufs;
  st.table_bufs = c->table_bufs;
  st.entry_cap = c->entry_cap;
  st.closure_cap = c->clo_cap;
  st.cross_entries = c->n_cross;
  st.dict_tiles = c->n_dict_tiles;
  *out = c;
  return FM_OK;
}

int fm_ctx_create(const fm_mesh_desc *m, const fm_tiling *tiling, void *stream, fm_ctx **out) {
  FM_NVTX("fm_ctx_create");
  // FM_TILING="nodes,bx,by,bz" overrides the default tiling (tuning aid)
  fm_tiling til{};
  if (tiling) {
    til = *tiling;
  } else if (const char *e = getenv("FM_TILING")) {
    if (sscanf(e, "%d,%d,%d,%d", &til.tile_nodes, &til.box[0], &til.box[1], &til.box[2]) != 4)
      til = fm_tiling{};
  }
  FM_ARG(m && out, "null argument");
  const int dim = m->dim;
  int box[3] = {dim == 3 ? 8 : 16, dim == 3 ? 8 : 16, dim == 3 ? 4 : 1};
  if (til.tile_nodes > 0 && til.tile_nodes <= 128 && dim == 3) box[1] = 4;
  for (int a = 0; a < 3; ++a)
    if (til.box[a] > 0) box[a] = til.box[a];
  // capacity failures retry with the largest box edge halved (a mesh much
  // denser or more graded than the structured configs); other errors return
  std::string first_err;
  for (int attempt = 0;; ++attempt) {
    for (int a = 0; a < 3; ++a) til.box[a] = box[a];
    bool cap = false;
    const int st = ctx_build(m, &til, stream, out, &cap);
    if (st == FM_OK || !cap) return st;
    if (attempt == 0) first_err = fm_last_error();
    int big = 0;
    for (int a = 1; a < dim; ++a)
      if (box[a] > box[big]) big = a;
    if (box[big] <= 1) {
      set_error(first_err + "; no tiling down to single-width boxes fits");
      return FM_INVALID_ARG;
    }
    box[big] /= 2;
  }
}

int fm_ctx_destroy(fm_ctx *c) {
  FM_NVTX("fm_ctx_destroy");
  if (!c) return FM_OK;
  void *ptrs[] = {c->aos,       c->conn4,     c->meta,      c->halo_ids,  c->halo_loc, c->loc,
                  c->closure,   c->flags,     c->node_desc, c->node_entries, c->free_node,
                  c->free_out,  c->rank_of,   c->storage_to_orig, c->free_mask, c->jpart,
                  c->dotpart,   c->status,    c->xkey,      c->xpos,      c->xchunk,
                  c->node_xbase, c->node_xn,  c->xbuf,      c->fixed_nodes, c->node_outw, c->node_fmask,
                  c->partial,   c->node_clo,  c->chunk_blocks, c->fpart, c->ticket,
                  c->xnodes,    c->dof_pos,   c->xdesc,     c->eidx,      c->dict_rec};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  delete c;
  return FM_OK;
}

int fm_ctx_stats_get(const fm_ctx *c, fm_ctx_stats *out) {
  FM_ARG(c && out, "null argument");
  *out = c->stats;
  return FM_OK;
}

int64_t fm_ctx_launches(const fm_ctx *c) { return c ? c->launches : 0; }

#if FM_WS_KERNEL
// experiment builds only (tools/bank_probe.py): one tile's metadata, the
// closure indices of its own elements (u16 x 4 each, storage order), its
// closure's node ids and its chunk entry blocks, copied to the host
extern "C" int fm_debug_tile_records(const fm_ctx *c, int t, unsigned char *rec) {
  if (!c || t < 0 || t >= c->n_tiles_all) return FM_INVALID_ARG;
  TileMeta tm;
  if (cudaMemcpy(&tm, c->meta + t, sizeof(tm), cudaMemcpyDeviceToHost)) return FM_CUDA_ERROR;
  const size_t rb = c->dim == 3 ? 80 : 48;
  if (cudaMemcpy(rec, c->aos + (size_t)tm.own_begin * rb, (size_t)tm.own_count * rb,
                 cudaMemcpyDeviceToHost))
    return FM_CUDA_ERROR;
  return FM_OK;
}
extern "C" int fm_debug_tile(const fm_ctx *c, int t, int *meta16, unsigned short *loc4,
                             int *closure, unsigned short *blocks) {
  if (!c || t < 0 || t >= c->n_tiles_all) return FM_INVALID_ARG;
  TileMeta tm;
  if (cudaMemcpy(&tm, c->meta + t, sizeof(tm), cudaMemcpyDeviceToHost)) return FM_CUDA_ERROR;
  memcpy(meta16, &tm, sizeof(tm));
  if (loc4 && cudaMemcpy(loc4, c->loc + tm.own_begin, (size_t)tm.own_count * 8,
                         cudaMemcpyDeviceToHost))
    return FM_CUDA_ERROR;
  if (closure && cudaMemcpy(closure, c->closure + tm.clo_begin, (size_t)tm.clo_count * 4,
                            cudaMemcpyDeviceToHost))
    return FM_CUDA_ERROR;
  const int nch = (tm.own_count + c->tile_nodes - 1) / c->tile_nodes;
  if (blocks && cudaMemcpy(blocks, c->chunk_blocks + tm.blk_base,
                           (size_t)nch * tm.blk_stride * 2, cudaMemcpyDeviceToHost))
    return FM_CUDA_ERROR;
  return FM_OK;
}
#endif

int fm_energy(fm_ctx *c, const fm_model *model, const double *v, const double *b, double *J_out,
              double *densities, void *stream) {
  FM_NVTX("fm_energy");
  int st = check_model(c, model);
  if (st) return st;
  FM_ARG(v && J_out, "null field or output");
  cudaStream_t s = as_stream(stream);
  ModelArgs ma = model_args(model);
  if (c->dim == 3) {
    // 3D: the tile pipeline in energy-only mode (records by bulk copy, node
    // values from the tile closures; cfg4 0.59 -> 0.53 ms), then the fused
    // path's finalisation: b.v of the nodes without a free dof, J from the
    // per-CTA partials in order.  (2D: small tiles, the streaming kernel is
    // faster: cfg3 0.075 vs 0.087 ms, cfg2 0.33 vs 0.36 ms.)
    TileArgs ta = c->tile_args();
    const int grid = std::min(c->n_sm * c->ctas_per_sm, std::max(1, ta.n_tiles_all));
    if (ta.n_tiles_all > 0) {
      TimedLaunch tl(c, s);
      FM_CUDA(launch_tile_exact(c->dim, model->kind, ta, grid, c->tile_nodes, c->node_bufs,
                                c->table_bufs, 4, v, b, densities, c->jpart, c->dotpart,
                                c->status, ma, s));
      c->launches++;
    }
    JFinal jf{c->jpart, c->dotpart, ta.n_tiles_all > 0 ? grid : 0, c->fixed_nodes,
              c->n_fixed_nodes, b, v, c->fpart, c->ticket, J_out};
    FM_CUDA(launch_finish_cross(c->d, 0, c->xdesc, c->xpos, c->xbuf, c->partial, nullptr, jf, s));
    c->launches++;
    return FM_OK;
  }
  {
    TimedLaunch tl(c, s);
    FM_CUDA(launch_energy(c->dim, model->kind, c->tile_args(), c->ne, c->n_energy_blocks, v,
                          c->jpart, densities, ma, s));
  }
  int nd = 0;
  if (b) {
    FM_CUDA(launch_dot(v, b, c->nn * c->d, c->n_dot_blocks, c->dotpart, s));
    nd = c->n_dot_blocks;
    c->launches++;
  }
  FM_CUDA(launch_finalize(c->jpart, c->n_energy_blocks, c->dotpart, nd, J_out, s));
  c->launches += 2;
  return FM_OK;
}

int fm_grad_exact(fm_ctx *c, const fm_model *model, const double *v, const double *b, double *g,
                  double *J_out, void *stream) {
  FM_NVTX("fm_grad_exact");
  int st = check_model(c, model);
  if (st) return st;
  // an empty gradient (no free dof) may come as a null pointer
  FM_ARG(v && (g || c->nfree_dofs == 0), "null field or output");
  cudaStream_t s = as_stream(stream);
  ModelArgs ma = model_args(model);
  const bool wj = J_out != nullptr;
  TileArgs ta = c->tile_args();
  if (!wj) ta.n_tiles_all = c->n_tiles;  // J-only orphan tiles not needed
  const int grid =
      std::min(c->n_sm * (c->ws ? 1 : c->ctas_per_sm), std::max(1, ta.n_tiles_all));
  if (ta.n_tiles_all > 0) {
    TimedLaunch tl(c, s);
#if FM_WS_KERNEL
    if (c->ws)
      FM_CUDA(launch_tile_ws(c->dim, model->kind, ta, grid, wj, v, b, g, c->jpart, c->dotpart,
                             c->status, ma, s));
    else
#endif
      FM_CUDA(launch_tile_exact(c->dim, model->kind, ta, grid, c->tile_nodes, c->node_bufs,
                                c->table_bufs, wj ? 1 : 0, v, b, g, c->jpart, c->dotpart,
                                c->status, ma, s));
    c->launches++;
  }
  if (c->n_cross > 0 || wj) {
    // cross entries of the tile nodes, and with J its finalisation (b.v of the
    // tile nodes came with the tile kernel's partials; the nodes without a
    // free dof are added here)
    JFinal jf{c->jpart, c->dotpart, ta.n_tiles_all > 0 ? grid : 0, c->fixed_nodes,
              c->n_fixed_nodes, b, v, c->fpart, c->ticket, wj ? J_out : nullptr};
    FM_CUDA(launch_finish_cross(c->d, c->n_cross > 0 ? c->n_xnodes : 0, c->xdesc, c->xpos,
                                c->xbuf, c->partial, g, jf, s));
    c->launches++;
  }
  return FM_OK;
}

int fm_hvp_exact(fm_ctx *c, const fm_model *model, const double *v, const double *p, double *hp,
                 void *stream) {
  FM_NVTX("fm_hvp_exact");
  int st = check_model(c, model);
  if (st) return st;
  FM_ARG(v && p && (hp || c->nfree_dofs == 0), "null field, direction or output");
  cudaStream_t s = as_stream(stream);
  ModelArgs ma = model_args(model);
  TileArgs ta = c->tile_args();
  ta.n_tiles_all = c->n_tiles;  // no J: orphan tiles not needed
  if (tile_exact_smem(c->dim, c->d, c->blk_cap, c->clo_cap, c->tile_nodes, c->node_bufs,
                      c->table_bufs, 2 * c->d, c->all_coded) > 227 * 1024) {
    set_error("Hessian-vector tile staging exceeds shared memory; use smaller tiles");
    return FM_INVALID_ARG;
  }
  const int grid = std::min(c->n_sm * c->ctas_per_sm, std::max(1, ta.n_tiles_all));
  if (ta.n_tiles_all > 0) {
    TimedLaunch tl(c, s);
    FM_CUDA(launch_tile_exact(c->dim, model->kind, ta, grid, c->tile_nodes, c->node_bufs,
                              c->table_bufs, 2, v, p, hp, c->jpart, c->dotpart, c->status, ma,
                              s));
    c->launches++;
  }
  if (c->n_cross > 0) {
    JFinal jf{c->jpart, c->dotpart, 0, c->fixed_nodes, 0, nullptr, v, c->fpart, c->ticket,
              nullptr};
    FM_CUDA(launch_finish_cross(c->d, c->n_xnodes, c->xdesc, c->xpos, c->xbuf, c->partial, hp,
                                jf, s));
    c->launches++;
  }
  return FM_OK;
}

int fm_grad_fd(fm_ctx *c, const fm_model *model, const double *v, const double *b, double eps,
               double *g, void *stream) {
  FM_NVTX("fm_grad_fd");
  int st = check_model(c, model);
  if (st) return st;
  // an empty gradient (no free dof) may come as a null pointer
  FM_ARG(v && (g || c->nfree_dofs == 0), "null field or output");
  FM_ARG(eps > 0.0, "central-difference step must be positive");
  if (c->n_tiles == 0) return FM_OK;
  cudaStream_t s = as_stream(stream);
  ModelArgs ma = model_args(model);
  ma.eps = eps;
  // every element once, by its owner tile (the fused tile kernel in FD mode:
  // records by bulk copy, per-element perturbed states, the gradient's node
  // sums / cross-tile exchange), then the finishing pass scales by 1 / (2 eps)
  TileArgs ta = c->tile_args();
  ta.n_tiles_all = c->n_tiles;  // orphan tiles have no free node
  const int cps = std::min(c->ctas_per_sm, tile_fd_minb(c->dim, c->tile_nodes, model->kind));
  const int grid = std::min(c->n_sm * cps, std::max(1, c->n_tiles));
  {
    TimedLaunch tl(c, s);
    FM_CUDA(launch_tile_exact(c->dim, model->kind, ta, grid, c->tile_nodes, c->node_bufs,
                              c->table_bufs, 3, v, b, g, c->jpart, c->dotpart, c->status, ma, s));
    c->launches++;
  }
  if (c->n_cross > 0) {
    FM_CUDA(launch_finish_cross_fd(c->d, c->n_xnodes, c->xdesc, c->xpos, c->xbuf, c->partial, g,
                                   eps, b, c->node_desc, s));
    c->launches++;
  }
  return FM_OK;
}

int fm_descent_step(fm_ctx *c, double *v, const double *g, double alpha, void *stream) {
  FM_NVTX("fm_descent_step");
  FM_ARG(c && v && (g || c->nfree_dofs == 0), "null argument");
  FM_CUDA(launch_descent(c->nfree_dofs, c->dof_pos, g, alpha, v, as_stream(stream)));
  c->launches++;
  return FM_OK;
}

int fm_descent(fm_ctx *c, const fm_model *model, double *v, const double *b, double alpha,
               int iters, double *g, double *J_hist, void *stream) {
  FM_NVTX("fm_descent");
  FM_ARG(c && v && (g || c->nfree_dofs == 0), "null argument");
  FM_ARG(iters >= 0, "negative iteration count");
  // every iteration: (J,) grad J at v, then v_free -= alpha * g; the kernels
  // of consecutive iterations are ordered on the stream, nothing syncs
  for (int i = 0; i < iters; ++i) {
    int st = fm_grad_exact(c, model, v, b, g, J_hist ? J_hist + 3 * (int64_t)i : nullptr, stream);
    if (st) return st;
    st = fm_descent_step(c, v, g, alpha, stream);
    if (st) return st;
  }
  return FM_OK;
}

int fm_ctx_check(fm_ctx *c, void *stream, int64_t *index) {
  FM_NVTX("fm_ctx_check");
  FM_ARG(c && index, "null argument");
  cudaStream_t s = as_stream(stream);
  unsigned long long h[2];
  FM_CUDA(cudaMemcpyAsync(h, c->status, 16, cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  unsigned long long init[2] = {0ull, ~0ull};
  FM_CUDA(cudaMemcpyAsync(c->status, init, 16, cudaMemcpyHostToDevice, s));
  FM_CUDA(cudaStreamSynchronize(s));
  *index = -1;
  if (h[1] != ~0ull) {
    const unsigned long long key = h[1];
    const int j = (int)((key >> 61) & 3ull);
    const int64_t r = (int64_t)((key >> 31) & ((1ull << 30) - 1));
    int32_t node = 0;
    FM_CUDA(cudaMemcpy(&node, c->free_node + r, 4, cudaMemcpyDeviceToHost));
    *index = (int64_t)c->d * node + j;
    set_error("perturbed state inadmissible at dof " + std::to_string(*index));
    return FM_INADMISSIBLE;
  }
  if (h[0]) {
    set_error("nonpositive det F in the exact derivative path");
    return FM_INADMISSIBLE;
  }
  return FM_OK;
}

}  // extern "C"
