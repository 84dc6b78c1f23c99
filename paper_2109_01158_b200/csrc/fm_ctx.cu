// Evaluation context: uploads/re-lays out the frozen Mesh + Patches once
// (mesh.py:31-53, patches.py:22-71) and exposes the evaluation entry points of
// include/femmin_b200.h.
//
// Context build (all on the GPU, CUB radix sorts, deterministic):
//   1. free-node ranks, output offsets of the restricted gradient
//      (gradients.py:68-74 _blocks_to_dofs order);
//   2. node tiles: free nodes bucketed into spatial boxes (box edge = k * mesh
//      width, width from the mean element measure), boxes split to <= tile_nodes;
//   3. element owner tile = tile of its first free node (orphans: no free node);
//      storage order sorted by (owner tile, element) -> 128-byte records;
//   4. tile element lists = union of the tile nodes' patches (patches.py:37-71
//      rows), slot masks OR-reduced by key, J flag where the tile owns the element;
//   5. node entries (te_local << 2 | slot) in patch order (ascending element).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fm_kernels.h"

namespace fm {

static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }

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
__host__ __device__ inline double from_ord(unsigned long long u) {
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

__global__ void k_box_keys(int64_t nfree, int dim, const int64_t *nodes, const double *X,
                           double x0, double y0, double z0, double ex, double ey, double ez,
                           double hh, int64_t nbx, int64_t nby, uint64_t *keys, int32_t *vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nfree;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t node = nodes[r];
    int64_t ix = (int64_t)floor((X[node * dim] - x0 + hh) / ex);
    int64_t iy = (int64_t)floor((X[node * dim + 1] - y0 + hh) / ey);
    int64_t iz = dim == 3 ? (int64_t)floor((X[node * dim + 2] - z0 + hh) / ez) : 0;
    keys[r] = (uint64_t)(ix + nbx * (iy + nby * iz));
    vals[r] = (int32_t)r;
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
                        int32_t *oval, int32_t *owner_of, unsigned long long *n_orph) {
  unsigned long long cnt = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    int own = n_tiles;
    for (int l = 0; l < nv; ++l) {
      int r = rank_of[conn[e * nv + l]];
      if (r >= 0) {
        own = tile_of_rank[r];
        break;
      }
    }
    cnt += own == n_tiles;
    okey[e] = (uint32_t)own;
    oval[e] = (int32_t)e;
    owner_of[e] = own;
  }
  if (cnt) atomicAdd(n_orph, cnt);
}

__global__ void k_inverse(int64_t n, const int32_t *perm, int32_t *inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    inv[perm[i]] = (int32_t)i;
}

template <int DIM>
__global__ void k_build_aos(int64_t ne, const int32_t *s2o, const int64_t *conn, const double *vol,
                            const double *dphi, uint8_t *aos) {
  constexpr int NV = DIM + 1;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < ne;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = s2o[s];
    uint8_t *rec = aos + s * RecBytes<DIM>::value;
    int32_t *ci = reinterpret_cast<int32_t *>(rec);
    double *dd = reinterpret_cast<double *>(rec);
    for (int l = 0; l < NV; ++l) ci[l] = (int32_t)conn[e * NV + l];
    if (DIM == 3) {
      dd[2] = vol[e];
      for (int m = 0; m < 3; ++m)
        for (int l = 0; l < 4; ++l) dd[3 + m * 4 + l] = dphi[((int64_t)m * ne + e) * 4 + l];
      ci[30] = (int32_t)e;
      ci[31] = 0;
    } else {
      ci[3] = (int32_t)e;
      dd[2] = vol[e];
      for (int m = 0; m < 2; ++m)
        for (int l = 0; l < 3; ++l) dd[3 + m * 3 + l] = dphi[((int64_t)m * ne + e) * 3 + l];
      dd[9] = 0.0;
    }
  }
}

__global__ void k_pair_keys(int64_t nfree, const int64_t *prefix, const int64_t *elems,
                            const int64_t *slot, const int32_t *tile_of_rank, uint64_t *keys,
                            uint8_t *vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nfree;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = r ? prefix[r - 1] : 0, z = prefix[r];
    uint64_t t = (uint64_t)tile_of_rank[r] << 32;
    for (int64_t q = a; q < z; ++q) {
      keys[q] = t | (uint64_t)elems[q];
      vals[q] = (uint8_t)(1u << slot[q]);
    }
  }
}

struct OrOp {
  __device__ __forceinline__ uint8_t operator()(uint8_t a, uint8_t b) const { return a | b; }
};

__global__ void k_tile_elems(int64_t M, const uint64_t *ukeys, const uint8_t *umask,
                             const int32_t *o2s, const int32_t *owner_of, int32_t *tile_elems,
                             uint8_t *flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = ukeys[i];
    int t = (int)(k >> 32);
    int64_t e = (int64_t)(k & 0xffffffffull);
    tile_elems[i] = o2s[e];
    flags[i] = umask[i] | (owner_of[e] == t ? FLAG_J : 0);
  }
}

__global__ void k_tile_elem_ptr(int n_tiles, int64_t M, const uint64_t *ukeys, int32_t *ptr) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= n_tiles; t += gridDim.x * blockDim.x) {
    uint64_t key = (uint64_t)t << 32;
    int64_t lo = 0, hi = M;  // first index with ukeys >= key
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (ukeys[mid] < key) lo = mid + 1; else hi = mid;
    }
    ptr[t] = (int32_t)lo;
  }
}

__global__ void k_orphans(int64_t n_orph, int64_t first_storage, int64_t M, int32_t *tile_elems,
                          uint8_t *flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_orph;
       i += (int64_t)gridDim.x * blockDim.x) {
    tile_elems[M + i] = (int32_t)(first_storage + i);
    flags[M + i] = FLAG_J;
  }
}

__global__ void k_entry_lens(int64_t ntn, const int32_t *tile_node_rank, const int64_t *prefix,
                             int32_t *lens) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntn;
       k += (int64_t)gridDim.x * blockDim.x) {
    int r = tile_node_rank[k];
    lens[k] = (int32_t)(prefix[r] - (r ? prefix[r - 1] : 0));
  }
}

__global__ void k_entries(int64_t ntn, const int32_t *tile_node_rank, const int32_t *tile_of_rank,
                          const int64_t *prefix, const int64_t *elems, const int64_t *slot,
                          const uint64_t *ukeys, const int32_t *tile_elem_ptr,
                          const int32_t *entry_ptr, uint16_t *entries,
                          unsigned long long *overflow) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntn;
       k += (int64_t)gridDim.x * blockDim.x) {
    int r = tile_node_rank[k];
    int t = tile_of_rank[r];
    int64_t a = r ? prefix[r - 1] : 0, z = prefix[r];
    int64_t lo0 = tile_elem_ptr[t], hi0 = tile_elem_ptr[t + 1];
    int32_t o = entry_ptr[k];
    for (int64_t q = a; q < z; ++q) {
      uint64_t key = ((uint64_t)t << 32) | (uint64_t)elems[q];
      int64_t lo = lo0, hi = hi0;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (ukeys[mid] < key) lo = mid + 1; else hi = mid;
      }
      int64_t te = lo - lo0;
      if (te >= MAX_TILE_ELEMS || lo >= hi0 || ukeys[lo] != key) atomicAdd(overflow, 1ull);
      entries[o++] = (uint16_t)((te << 2) | slot[q]);
    }
  }
}

template <class T> static cudaError_t dmalloc(T **p, size_t n, size_t *acc) {
  *acc += n * sizeof(T);
  return cudaMalloc((void **)p, std::max<size_t>(n, 1) * sizeof(T));
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

int fm_ctx_time_next(fm_ctx *c, void *ev_start, void *ev_stop) {
  FM_ARG(c, "null context");
  c->ev_start = reinterpret_cast<cudaEvent_t>(ev_start);
  c->ev_stop = reinterpret_cast<cudaEvent_t>(ev_stop);
  return FM_OK;
}

const char *fm_last_error(void) { return g_err.c_str(); }
int fm_version(void) { return 1; }

int fm_ctx_create(const fm_mesh_desc *m, const fm_tiling *tiling, void *stream, fm_ctx **out) {
  FM_ARG(m && out, "null argument");
  FM_ARG(m->dim == 2 || m->dim == 3, "dim must be 2 or 3");
  FM_ARG(m->d >= 1 && m->d <= m->dim, "d must be 1..dim");
  FM_ARG(m->ne > 0 && m->nn > 0, "empty mesh");
  FM_ARG(m->ne < (1ll << 31) && m->nn < (1ll << 31) && m->p_total < (1ll << 31),
         "per-GPU mesh must fit 32-bit indices (shard larger meshes)");
  cudaStream_t s = as_stream(stream);
  const int dim = m->dim, nv = dim + 1, d = m->d;
  fm_ctx *c = new fm_ctx();
  *out = nullptr;
  auto fail = [&](int code) {
    fm_ctx_destroy(c);
    return code;
  };
  c->dim = dim;
  c->d = d;
  c->nv = nv;
  c->nn = m->nn;
  c->ne = m->ne;
  c->nfree = m->nfree;
  c->p_total = m->p_total;
  int NT = (tiling && tiling->tile_nodes) ? tiling->tile_nodes : (dim == 3 ? 256 : 512);
  NT = std::max(32, std::min(512, NT / 32 * 32));
  int box[3] = {dim == 3 ? 8 : 32, dim == 3 ? 8 : 16, dim == 3 ? 4 : 1};
  if (tiling)
    for (int a = 0; a < 3; ++a)
      if (tiling->box[a] > 0) box[a] = tiling->box[a];
  c->tile_nodes = NT;
  const int64_t nfree = m->nfree, ne = m->ne, T = m->p_total;
  size_t &B = c->bytes;

#define CK(x)                                                   \
  do {                                                          \
    cudaError_t _e = (x);                                       \
    if (_e != cudaSuccess) {                                    \
      set_error(std::string(#x) + ": " + cudaGetErrorString(_e)); \
      return fail(FM_CUDA_ERROR);                               \
    }                                                           \
  } while (0)

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
    k_ranks<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, d, m->nodes_minim, m->fixed, c->rank_of,
                                                 c->free_node, c->free_mask, cnt.as<int32_t>());
    CK(cudaGetLastError());
    size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.as<int32_t>(), c->free_out, nfree + 1,
                                     s));
    Scratch tmp;
    CK(tmp.alloc(bytes, s));
    CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.as<int32_t>(), c->free_out, nfree + 1, s));
    int32_t nfd = 0;
    CK(cudaMemcpyAsync(&nfd, c->free_out + nfree, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->nfree_dofs = nfd;
  }

  // 2. node tiles -----------------------------------------------------------
  std::vector<int32_t> h_tnp;  // tile node ptr (host)
  Scratch s_tnr;               // sorted ranks = tile_node_rank
  if (nfree > 0) {
    double volsum = 0.0;
    {
      Scratch out, tmp;
      CK(out.alloc(8, s));
      size_t bytes = 0;
      CK(cub::DeviceReduce::Sum(nullptr, bytes, m->volumes, out.as<double>(), ne, s));
      CK(tmp.alloc(bytes, s));
      CK(cub::DeviceReduce::Sum(tmp.p, bytes, m->volumes, out.as<double>(), ne, s));
      CK(cudaMemcpyAsync(&volsum, out.p, 8, cudaMemcpyDeviceToHost, s));
    }
    unsigned long long hmn[3], hmx[3];
    {
      Scratch mm;
      CK(mm.alloc(48, s));
      CK(cudaMemsetAsync(mm.p, 0xff, 24, s));
      CK(cudaMemsetAsync(mm.as<uint8_t>() + 24, 0, 24, s));
      k_bbox<<<grid_for(nfree, 256, 1184), 256, 0, s>>>(nfree, dim, m->nodes_minim, m->coords,
                                                        mm.as<unsigned long long>(),
                                                        mm.as<unsigned long long>() + 3);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(hmn, mm.p, 24, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(hmx, mm.as<uint8_t>() + 24, 24, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    const double fact = dim == 3 ? 6.0 : 2.0;
    const double h = std::pow(fact * volsum / (double)ne, 1.0 / dim);
    double x0[3] = {0, 0, 0}, ext[3] = {0, 0, 0}, edge[3] = {1, 1, 1};
    int64_t nb[3] = {1, 1, 1};
    for (int a = 0; a < dim; ++a) {
      x0[a] = from_ord(hmn[a]);
      ext[a] = from_ord(hmx[a]) - x0[a];
      edge[a] = box[a] * h;
      nb[a] = (int64_t)std::floor((ext[a] + 0.5 * h) / edge[a]) + 1;
    }
    if ((double)nb[0] * nb[1] * nb[2] > 4e18) {
      set_error("tiling box grid too large");
      return fail(FM_INVALID_ARG);
    }
    Scratch keys, keys2, vals2, runs, counts, nruns;
    CK(keys.alloc(nfree * 8, s));
    CK(keys2.alloc(nfree * 8, s));
    CK(s_tnr.alloc(nfree * 4, s));
    CK(vals2.alloc(nfree * 4, s));
    k_box_keys<<<grid_for(nfree, 256), 256, 0, s>>>(
        nfree, dim, m->nodes_minim, m->coords, x0[0], x0[1], x0[2], edge[0], edge[1], edge[2],
        0.5 * h, nb[0], nb[1], keys.as<uint64_t>(), s_tnr.as<int32_t>());
    CK(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> dk(keys.as<uint64_t>(), keys2.as<uint64_t>());
    cub::DoubleBuffer<int32_t> dv(s_tnr.as<int32_t>(), vals2.as<int32_t>());
    int end_bit = std::max(1, bits_for((uint64_t)(nb[0] * nb[1] * nb[2])));
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, nfree, 0, end_bit, s));
    {
      Scratch tmp;
      CK(tmp.alloc(bytes, s));
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, dk, dv, nfree, 0, end_bit, s));
    }
    if (dv.Current() != s_tnr.as<int32_t>())
      CK(cudaMemcpyAsync(s_tnr.p, dv.Current(), nfree * 4, cudaMemcpyDeviceToDevice, s));
    CK(runs.alloc(nfree * 8, s));
    CK(counts.alloc(nfree * 4, s));
    CK(nruns.alloc(8, s));
    bytes = 0;
    CK(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, dk.Current(), runs.as<uint64_t>(),
                                          counts.as<int32_t>(), nruns.as<int32_t>(), nfree, s));
    {
      Scratch tmp;
      CK(tmp.alloc(bytes, s));
      CK(cub::DeviceRunLengthEncode::Encode(tmp.p, bytes, dk.Current(), runs.as<uint64_t>(),
                                            counts.as<int32_t>(), nruns.as<int32_t>(), nfree,
                                            s));
    }
    int32_t nr = 0;
    CK(cudaMemcpyAsync(&nr, nruns.p, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<int32_t> cnts(nr);
    CK(cudaMemcpy(cnts.data(), counts.p, (size_t)nr * 4, cudaMemcpyDeviceToHost));
    h_tnp.push_back(0);
    int64_t pos = 0;
    for (int32_t cb : cnts) {
      int k = (cb + NT - 1) / NT;
      for (int q = 0; q < k; ++q) {
        int64_t sz = (int64_t)cb * (q + 1) / k - (int64_t)cb * q / k;
        pos += sz;
        h_tnp.push_back((int32_t)pos);
      }
    }
  } else {
    h_tnp.push_back(0);
  }
  const int n_tiles = (int)h_tnp.size() - 1;
  c->n_tiles = n_tiles;
  c->max_tile_nodes = 0;
  for (int t = 0; t < n_tiles; ++t)
    c->max_tile_nodes = std::max(c->max_tile_nodes, h_tnp[t + 1] - h_tnp[t]);

  Scratch s_tor;  // tile_of_rank
  CK(s_tor.alloc(std::max<int64_t>(nfree, 1) * 4, s));
  CK(dmalloc(&c->tile_node_rank, nfree, &B));
  if (nfree) CK(cudaMemcpyAsync(c->tile_node_rank, s_tnr.p, nfree * 4, cudaMemcpyDeviceToDevice, s));

  // 3. element owners and storage order ---------------------------------------
  Scratch okey, okey2, oval2, owner_of, o2s, cnt_orph;
  CK(okey.alloc(ne * 4, s));
  CK(okey2.alloc(ne * 4, s));
  CK(oval2.alloc(ne * 4, s));
  CK(owner_of.alloc(ne * 4, s));
  CK(o2s.alloc(ne * 4, s));
  CK(cnt_orph.alloc(8, s));
  CK(dmalloc(&c->storage_to_orig, ne, &B));
  CK(cudaMemsetAsync(cnt_orph.p, 0, 8, s));
  {
    Scratch d_tnp;
    CK(d_tnp.alloc(h_tnp.size() * 4, s));
    CK(cudaMemcpyAsync(d_tnp.p, h_tnp.data(), h_tnp.size() * 4, cudaMemcpyHostToDevice, s));
    if (nfree)
      k_tile_of_pos<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, n_tiles, d_tnp.as<int32_t>(),
                                                         c->tile_node_rank, s_tor.as<int32_t>());
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
  }
  k_owner<<<grid_for(ne, 256), 256, 0, s>>>(ne, nv, m->conn, c->rank_of, s_tor.as<int32_t>(),
                                            n_tiles, okey.as<uint32_t>(),
                                            c->storage_to_orig, owner_of.as<int32_t>(),
                                            cnt_orph.as<unsigned long long>());
  CK(cudaGetLastError());
  {
    cub::DoubleBuffer<uint32_t> dk(okey.as<uint32_t>(), okey2.as<uint32_t>());
    cub::DoubleBuffer<int32_t> dv(c->storage_to_orig, oval2.as<int32_t>());
    int end_bit = std::max(1, bits_for((uint64_t)n_tiles));
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, ne, 0, end_bit, s));
    Scratch tmp;
    CK(tmp.alloc(bytes, s));
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, dk, dv, ne, 0, end_bit, s));
    if (dv.Current() != c->storage_to_orig)
      CK(cudaMemcpyAsync(c->storage_to_orig, dv.Current(), ne * 4, cudaMemcpyDeviceToDevice, s));
  }
  k_inverse<<<grid_for(ne, 256), 256, 0, s>>>(ne, c->storage_to_orig, o2s.as<int32_t>());
  CK(cudaGetLastError());
  unsigned long long n_orph = 0;
  CK(cudaMemcpyAsync(&n_orph, cnt_orph.p, 8, cudaMemcpyDeviceToHost, s));

  // element records
  const int rb = dim == 3 ? RecBytes<3>::value : RecBytes<2>::value;
  CK(dmalloc(&c->aos, (size_t)ne * rb, &B));
  if (dim == 3)
    k_build_aos<3><<<grid_for(ne, 256), 256, 0, s>>>(ne, c->storage_to_orig, m->conn, m->volumes,
                                                     m->dphi, c->aos);
  else
    k_build_aos<2><<<grid_for(ne, 256), 256, 0, s>>>(ne, c->storage_to_orig, m->conn, m->volumes,
                                                     m->dphi, c->aos);
  CK(cudaGetLastError());

  // 4. tile element lists -------------------------------------------------------
  int64_t M = 0;
  Scratch ukeys, umask;
  if (nfree > 0) {
    Scratch pk, pk2, pv, pv2, nsel;
    CK(pk.alloc(T * 8, s));
    CK(pk2.alloc(T * 8, s));
    CK(pv.alloc(T, s));
    CK(pv2.alloc(T, s));
    k_pair_keys<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, m->p_prefix, m->p_elems, m->p_slot,
                                                     s_tor.as<int32_t>(), pk.as<uint64_t>(),
                                                     pv.as<uint8_t>());
    CK(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> dk(pk.as<uint64_t>(), pk2.as<uint64_t>());
    cub::DoubleBuffer<uint8_t> dv(pv.as<uint8_t>(), pv2.as<uint8_t>());
    int end_bit = 32 + bits_for((uint64_t)n_tiles);
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, T, 0, end_bit, s));
    {
      Scratch tmp;
      CK(tmp.alloc(bytes, s));
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, dk, dv, T, 0, end_bit, s));
    }
    CK(ukeys.alloc(T * 8, s));
    CK(umask.alloc(T, s));
    CK(nsel.alloc(8, s));
    bytes = 0;
    CK(cub::DeviceReduce::ReduceByKey(nullptr, bytes, dk.Current(), ukeys.as<uint64_t>(),
                                      dv.Current(), umask.as<uint8_t>(), nsel.as<int64_t>(),
                                      OrOp(), T, s));
    {
      Scratch tmp;
      CK(tmp.alloc(bytes, s));
      CK(cub::DeviceReduce::ReduceByKey(tmp.p, bytes, dk.Current(), ukeys.as<uint64_t>(),
                                        dv.Current(), umask.as<uint8_t>(), nsel.as<int64_t>(),
                                        OrOp(), T, s));
    }
    CK(cudaMemcpyAsync(&M, nsel.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  CK(cudaStreamSynchronize(s));
  const int OT = 4 * NT;  // orphan elements per orphan tile
  const int n_otiles = (int)((n_orph + OT - 1) / OT);
  c->n_tiles_all = n_tiles + n_otiles;
  c->n_tile_elems = M + (int64_t)n_orph;
  CK(dmalloc(&c->tile_elems, c->n_tile_elems, &B));
  CK(dmalloc(&c->tile_flags, c->n_tile_elems, &B));
  CK(dmalloc(&c->tile_elem_ptr, c->n_tiles_all + 1, &B));
  CK(dmalloc(&c->tile_node_ptr, c->n_tiles_all + 1, &B));
  if (M)
    k_tile_elems<<<grid_for(M, 256), 256, 0, s>>>(M, ukeys.as<uint64_t>(), umask.as<uint8_t>(),
                                                  o2s.as<int32_t>(), owner_of.as<int32_t>(),
                                                  c->tile_elems, c->tile_flags);
  if (n_tiles)
    k_tile_elem_ptr<<<grid_for(n_tiles + 1, 256), 256, 0, s>>>(n_tiles, M, ukeys.as<uint64_t>(),
                                                               c->tile_elem_ptr);
  if (n_orph)
    k_orphans<<<grid_for(n_orph, 256), 256, 0, s>>>((int64_t)n_orph, ne - (int64_t)n_orph, M,
                                                    c->tile_elems, c->tile_flags);
  CK(cudaGetLastError());
  {
    std::vector<int32_t> ext;
    for (int q = 1; q <= n_otiles; ++q)
      ext.push_back((int32_t)(M + std::min<int64_t>((int64_t)q * OT, (int64_t)n_orph)));
    if (n_tiles == 0) ext.insert(ext.begin(), 0);
    if (!ext.empty())
      CK(cudaMemcpyAsync(c->tile_elem_ptr + (n_tiles ? n_tiles + 1 : 0), ext.data(),
                         ext.size() * 4, cudaMemcpyHostToDevice, s));
    std::vector<int32_t> tnp(h_tnp);
    for (int q = 0; q < n_otiles; ++q) tnp.push_back(h_tnp.back());
    CK(cudaMemcpyAsync(c->tile_node_ptr, tnp.data(), tnp.size() * 4, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  std::vector<int32_t> h_tep(c->n_tiles_all + 1);
  CK(cudaMemcpy(h_tep.data(), c->tile_elem_ptr, h_tep.size() * 4, cudaMemcpyDeviceToHost));
  c->max_tile_elems = 0;
  for (int t = 0; t < c->n_tiles_all; ++t)
    c->max_tile_elems = std::max(c->max_tile_elems, h_tep[t + 1] - h_tep[t]);
  if (c->max_tile_elems > MAX_TILE_ELEMS) {
    set_error("a node tile touches more than 16384 elements; use smaller tiles");
    return fail(FM_INVALID_ARG);
  }

  // 5. node entries -------------------------------------------------------------
  CK(dmalloc(&c->node_entry_ptr, nfree + 1, &B));
  CK(dmalloc(&c->node_entries, T, &B));
  c->n_node_entries = T;
  if (nfree > 0) {
    Scratch lens, ovf;
    CK(lens.alloc((nfree + 1) * 4, s));
    CK(ovf.alloc(8, s));
    CK(cudaMemsetAsync(lens.p, 0, (nfree + 1) * 4, s));
    CK(cudaMemsetAsync(ovf.p, 0, 8, s));
    k_entry_lens<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, c->tile_node_rank, m->p_prefix,
                                                      lens.as<int32_t>());
    size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, lens.as<int32_t>(), c->node_entry_ptr,
                                     nfree + 1, s));
    {
      Scratch tmp;
      CK(tmp.alloc(bytes, s));
      CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, lens.as<int32_t>(), c->node_entry_ptr,
                                       nfree + 1, s));
    }
    k_entries<<<grid_for(nfree, 256), 256, 0, s>>>(
        nfree, c->tile_node_rank, s_tor.as<int32_t>(), m->p_prefix, m->p_elems, m->p_slot,
        ukeys.as<uint64_t>(), c->tile_elem_ptr, c->node_entry_ptr, c->node_entries,
        ovf.as<unsigned long long>());
    CK(cudaGetLastError());
    unsigned long long h_ovf = 0;
    CK(cudaMemcpyAsync(&h_ovf, ovf.p, 8, cudaMemcpyDeviceToHost, s));
    std::vector<int32_t> h_nep(nfree + 1);
    CK(cudaMemcpyAsync(h_nep.data(), c->node_entry_ptr, (nfree + 1) * 4, cudaMemcpyDeviceToHost,
                       s));
    CK(cudaStreamSynchronize(s));
    if (h_ovf) {
      set_error("internal error: patch entry not found in its tile");
      return fail(FM_CUDA_ERROR);
    }
    c->max_tile_entries = 0;
    for (int t = 0; t < n_tiles; ++t)
      c->max_tile_entries = std::max(c->max_tile_entries, h_nep[h_tnp[t + 1]] - h_nep[h_tnp[t]]);
  } else {
    CK(cudaMemsetAsync(c->node_entry_ptr, 0, 4, s));
  }

  // scratch ------------------------------------------------------------------
  c->n_energy_blocks = 148 * 8;
  c->n_dot_blocks = 148 * 2;
  CK(dmalloc(&c->jpart, std::max<int64_t>(c->n_tiles_all, c->n_energy_blocks), &B));
  CK(dmalloc(&c->dotpart, c->n_dot_blocks, &B));
  CK(dmalloc(&c->status, 2, &B));
  unsigned long long init[2] = {0ull, ~0ull};
  CK(cudaMemcpyAsync(c->status, init, 16, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
#undef CK

  fm_ctx_stats &st = c->stats;
  st.n_tiles = n_tiles;
  st.n_orphan_tiles = n_otiles;
  st.tile_elems_total = c->n_tile_elems;
  st.node_entries_total = c->n_node_entries;
  st.max_tile_elems = c->max_tile_elems;
  st.max_tile_entries = c->max_tile_entries;
  st.bytes_device = (int64_t)c->bytes;
  st.redundancy = (double)c->n_tile_elems / (double)ne;
  *out = c;
  return FM_OK;
}

int fm_ctx_destroy(fm_ctx *c) {
  if (!c) return FM_OK;
  void *ptrs[] = {c->aos,          c->tile_elem_ptr, c->tile_elems,   c->tile_node_ptr,
                  c->tile_node_rank, c->node_entry_ptr, c->tile_flags, c->node_entries,
                  c->free_node,    c->free_out,      c->rank_of,      c->storage_to_orig,
                  c->free_mask,    c->jpart,         c->dotpart,      c->status};
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

int fm_energy(fm_ctx *c, const fm_model *model, const double *v, const double *b, double *J_out,
              double *densities, void *stream) {
  int st = check_model(c, model);
  if (st) return st;
  FM_ARG(v && J_out, "null field or output");
  cudaStream_t s = as_stream(stream);
  ModelArgs ma = model_args(model);
  {
    TimedLaunch tl(c, s);
    FM_CUDA(launch_energy(c->dim, model->kind, c->aos, c->ne, c->n_energy_blocks, v, c->jpart,
                          densities, ma, s));
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
  int st = check_model(c, model);
  if (st) return st;
  FM_ARG(v && g, "null field or output");
  cudaStream_t s = as_stream(stream);
  ModelArgs ma = model_args(model);
  const bool wj = J_out != nullptr;
  const int nt = wj ? c->n_tiles_all : c->n_tiles;
  if (nt > 0) {
    TimedLaunch tl(c, s);
    FM_CUDA(launch_tile_exact(c->dim, model->kind, c->tile_args(), nt, c->tile_nodes,
                              (size_t)c->max_tile_entries * 2 + 16, wj, true, v, b, g, c->jpart,
                              c->status, ma, s));
    c->launches++;
  }
  if (wj) {
    int nd = 0;
    if (b) {
      FM_CUDA(launch_dot(v, b, c->nn * c->d, c->n_dot_blocks, c->dotpart, s));
      nd = c->n_dot_blocks;
      c->launches++;
    }
    FM_CUDA(launch_finalize(c->jpart, nt, c->dotpart, nd, J_out, s));
    c->launches++;
  }
  return FM_OK;
}

int fm_grad_fd(fm_ctx *c, const fm_model *model, const double *v, const double *b, double eps,
               double *g, void *stream) {
  int st = check_model(c, model);
  if (st) return st;
  FM_ARG(v && g, "null field or output");
  FM_ARG(eps > 0.0, "central-difference step must be positive");
  if (c->n_tiles == 0) return FM_OK;
  cudaStream_t s = as_stream(stream);
  ModelArgs ma = model_args(model);
  TimedLaunch tl(c, s);
  FM_CUDA(launch_tile_fd(c->dim, model->kind, c->tile_args(), c->n_tiles, c->tile_nodes,
                         (size_t)c->max_tile_entries * 2 + 16, v, b, eps, g, c->status + 1, ma,
                         s));
  c->launches++;
  return FM_OK;
}

int fm_descent_step(fm_ctx *c, double *v, const double *g, double alpha, void *stream) {
  FM_ARG(c && v && g, "null argument");
  FM_CUDA(launch_descent(c->nfree, c->d, c->free_node, c->free_out, c->free_mask, g, alpha, v,
                         as_stream(stream)));
  c->launches++;
  return FM_OK;
}

int fm_ctx_check(fm_ctx *c, void *stream, int64_t *index) {
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
