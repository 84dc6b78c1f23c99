// Hessian utilities (solver.py:344-398) on the GPU:
//   fm_hessian_pattern   hessian_sparsity: node adjacency of the elements,
//                        d x d dof blocks, restricted to the free dofs, CSR
//                        with ascending columns (scipy's canonical order)
//   fm_color_d2          distance-2 colouring of a symmetric pattern
//                        (columns sharing a row get distinct colours): rounds
//                        of "local priority maximum takes the smallest colour
//                        free in its distance-2 neighbourhood"
//   fm_hess_perturb / fm_hess_scatter / fm_hess_symmetrize
//                        colored_fd_hessian: one perturbed gradient per colour,
//                        (g(x + h e_C) - g(x)) / h scattered into the pattern's
//                        columns of that colour, then (H + H^T) / 2
// The gradient of a free dof only reads the dofs of its node patch, so with a
// distance-2 colouring every scattered difference is bit-identical to the
// single-column difference whatever the colouring.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "fm_common.cuh"

namespace fm {

template <class F> static cudaError_t cub_run(F f, cudaStream_t s) {
  size_t bytes = 0;
  cudaError_t e = f(nullptr, bytes);
  if (e != cudaSuccess) return e;
  Scratch tmp;
  e = tmp.alloc(bytes, s);
  if (e != cudaSuccess) return e;
  return f(tmp.p, bytes);
}

// node pair keys (a << 32 | b) of every element, a, b over its nodes
__global__ void k_node_pairs(int64_t ne, int nv, const int64_t *conn, uint64_t *keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x)
    for (int x = 0; x < nv; ++x)
      for (int y = 0; y < nv; ++y)
        keys[(e * nv + x) * nv + y] =
            ((uint64_t)conn[e * nv + x] << 32) | (uint64_t)conn[e * nv + y];
}

// dof -> free index (position in dofs_minim) or -1
__global__ void k_free_index(int64_t nfd, const int64_t *dofs_minim, int32_t *fidx) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nfd;
       q += (int64_t)gridDim.x * blockDim.x)
    fidx[dofs_minim[q]] = (int32_t)q;
}

// node a's neighbours are nb[aptr[a] .. aptr[a+1]) (sorted); first pass counts
// each free row's columns, second pass writes them
__global__ void k_pattern_rows(int64_t nfd, int d, const int64_t *dofs_minim,
                               const int64_t *aptr, const uint64_t *nb, const int32_t *fidx,
                               const int64_t *indptr, int64_t *cnt, int64_t *indices) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nfd;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = dofs_minim[q] / d;
    int64_t n = 0, o = indices ? indptr[q] : 0;
    for (int64_t p = aptr[a]; p < aptr[a + 1]; ++p) {
      const int64_t bn = (int64_t)(nb[p] & 0xffffffffull);
      for (int j = 0; j < d; ++j) {
        const int32_t c = fidx[bn * d + j];
        if (c < 0) continue;
        if (indices) indices[o + n] = c;
        ++n;
      }
    }
    if (cnt) cnt[q] = n;
  }
}

__global__ void k_node_starts(int64_t nn, int64_t len, const uint64_t *sorted, int64_t *aptr) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a <= nn;
       a += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = (uint64_t)a << 32;
    int64_t lo = 0, hi = len;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sorted[mid] < key) lo = mid + 1; else hi = mid;
    }
    aptr[a] = lo;
  }
}

// ---------------------------------------------------------------- colouring
__device__ __forceinline__ uint32_t prio_hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// one round: an uncoloured vertex whose (hash, index) beats every uncoloured
// vertex of its distance-2 neighbourhood takes the smallest colour not used
// there (colours >= 256 fall back to 256 + round)
__global__ void k_color_round(int64_t n, const int64_t *indptr, const int64_t *indices,
                              const int32_t *col_in, int32_t *col_out, int round,
                              unsigned long long *left) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t cv = col_in[v];
    col_out[v] = cv;
    if (cv >= 0) continue;
    const uint64_t pv = ((uint64_t)prio_hash((uint32_t)v) << 32) | (uint64_t)v;
    uint64_t used[4] = {0, 0, 0, 0};
    bool wins = true;
    for (int64_t p = indptr[v]; p < indptr[v + 1] && wins; ++p) {
      const int64_t r = indices[p];
      for (int64_t q = indptr[r]; q < indptr[r + 1]; ++q) {
        const int64_t u = indices[q];
        if (u == v) continue;
        const int32_t cu = col_in[u];
        if (cu < 0) {
          const uint64_t pu = ((uint64_t)prio_hash((uint32_t)u) << 32) | (uint64_t)u;
          if (pu > pv) {
            wins = false;
            break;
          }
        } else if (cu < 256) {
          used[cu >> 6] |= 1ull << (cu & 63);
        }
      }
    }
    if (!wins) {
      atomicAdd(left, 1ull);
      continue;
    }
    int c = 256 + round;
    for (int w = 0; w < 4; ++w)
      if (~used[w]) {
        c = w * 64 + __ffsll((long long)~used[w]) - 1;
        break;
      }
    col_out[v] = c;
  }
}

// ---------------------------------------------------------------- FD Hessian
__global__ void k_hess_perturb(int64_t nfd, const int64_t *dofs_minim, const int32_t *colors,
                               int color, double step, double *vp) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nfd;
       q += (int64_t)gridDim.x * blockDim.x)
    if (colors[q] == color) {
      const int64_t i = dofs_minim[q];
      vp[i] = __dadd_rn(vp[i], step);  // xp[cols] += step (solver.py:389)
    }
}

__global__ void k_hess_scatter(int64_t n, const int64_t *indptr, const int64_t *indices,
                               const int32_t *colors, int color, const double *gp,
                               const double *g0, double step, double *vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double diff = __ddiv_rn(__dsub_rn(gp[r], g0[r]), step);  // solver.py:390
    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p)
      if (colors[indices[p]] == color) vals[p] = diff;  // H[rows, col] = diff[rows]
  }
}

__global__ void k_hess_sym(int64_t n, const int64_t *indptr, const int64_t *indices,
                           const double *in, double *out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p) {
      const int64_t c = indices[p];
      int64_t lo = indptr[c], hi = indptr[c + 1];  // (c, r) in row c
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (indices[mid] < r) lo = mid + 1; else hi = mid;
      }
      out[p] = __dmul_rn(__dadd_rn(in[p], in[lo]), 0.5);  // (H + H.T) * 0.5
    }
}

}  // namespace fm

using namespace fm;

extern "C" {

int fm_hessian_pattern(int64_t nn, int64_t ne, int nv, int d, const int64_t *conn,
                       int64_t nfree_dofs, const int64_t *dofs_minim, int64_t *indptr,
                       int64_t *indices, int64_t *nnz_host, void *stream) {
  FM_NVTX("fm_hessian_pattern");
  FM_ARG(nn >= 0 && ne >= 0 && nv >= 1 && d >= 1 && nnz_host, "invalid pattern arguments");
  FM_ARG(nn < (1ll << 31), "node ids must fit 32 bits");
  cudaStream_t s = as_stream(stream);
  const int64_t NK = ne * nv * nv;
  Scratch k1, k2, uk, ns, fidx, aptr, cnt;
  FM_CUDA(k1.alloc(std::max<int64_t>(NK, 1) * 8, s));
  FM_CUDA(k2.alloc(std::max<int64_t>(NK, 1) * 8, s));
  FM_CUDA(uk.alloc(std::max<int64_t>(NK, 1) * 8, s));
  FM_CUDA(ns.alloc(8, s));
  FM_CUDA(fidx.alloc(std::max<int64_t>(nn * d, 1) * 4, s));
  FM_CUDA(aptr.alloc((nn + 1) * 8, s));
  FM_CUDA(cnt.alloc((nfree_dofs + 1) * 8, s));
  k_node_pairs<<<grid_for(ne, 256), 256, 0, s>>>(ne, nv, conn, k1.as<uint64_t>());
  FM_CHECK_LAUNCH();
  cub::DoubleBuffer<uint64_t> db(k1.as<uint64_t>(), k2.as<uint64_t>());
  FM_CUDA(cub_run([&](void *t, size_t &b) {
    return cub::DeviceRadixSort::SortKeys(t, b, db, NK, 0, 64, s);
  }, s));
  FM_CUDA(cub_run([&](void *t, size_t &b) {
    return cub::DeviceSelect::Unique(t, b, db.Current(), uk.as<uint64_t>(), ns.as<int64_t>(), NK,
                                     s);
  }, s));
  int64_t U = 0;
  FM_CUDA(cudaMemcpyAsync(&U, ns.p, 8, cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  k_node_starts<<<grid_for(nn + 1, 256), 256, 0, s>>>(nn, U, uk.as<uint64_t>(),
                                                       aptr.as<int64_t>());
  FM_CUDA(cudaMemsetAsync(fidx.p, 0xff, std::max<int64_t>(nn * d, 1) * 4, s));
  k_free_index<<<grid_for(nfree_dofs, 256), 256, 0, s>>>(nfree_dofs, dofs_minim,
                                                          fidx.as<int32_t>());
  FM_CHECK_LAUNCH();
  int64_t *c = cnt.as<int64_t>();
  FM_CUDA(cudaMemsetAsync(c + nfree_dofs, 0, 8, s));
  k_pattern_rows<<<grid_for(nfree_dofs, 256), 256, 0, s>>>(
      nfree_dofs, d, dofs_minim, aptr.as<int64_t>(), uk.as<uint64_t>(), fidx.as<int32_t>(),
      nullptr, c, nullptr);
  FM_CHECK_LAUNCH();
  // indptr = exclusive scan of the row counts (nfree_dofs + 1 entries)
  Scratch ip;
  int64_t *ipp = indptr;
  if (!indptr) {
    FM_CUDA(ip.alloc((nfree_dofs + 1) * 8, s));
    ipp = ip.as<int64_t>();
  }
  FM_CUDA(cub_run([&](void *t, size_t &b) {
    return cub::DeviceScan::ExclusiveSum(t, b, c, ipp, nfree_dofs + 1, s);
  }, s));
  FM_CUDA(cudaMemcpyAsync(nnz_host, ipp + nfree_dofs, 8, cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  if (indices) {
    k_pattern_rows<<<grid_for(nfree_dofs, 256), 256, 0, s>>>(
        nfree_dofs, d, dofs_minim, aptr.as<int64_t>(), uk.as<uint64_t>(), fidx.as<int32_t>(),
        ipp, nullptr, indices);
    FM_CHECK_LAUNCH();
    FM_CUDA(cudaStreamSynchronize(s));
  }
  return FM_OK;
}

int fm_color_d2(int64_t n, const int64_t *indptr, const int64_t *indices, int32_t *colors,
                int32_t *ncolors_host, void *stream) {
  FM_NVTX("fm_color_d2");
  FM_ARG(n >= 0 && ncolors_host, "invalid colouring arguments");
  cudaStream_t s = as_stream(stream);
  Scratch other, left;
  FM_CUDA(other.alloc(std::max<int64_t>(n, 1) * 4, s));
  FM_CUDA(left.alloc(8, s));
  FM_CUDA(cudaMemsetAsync(colors, 0xff, std::max<int64_t>(n, 1) * 4, s));
  int32_t *a = colors, *b = other.as<int32_t>();
  unsigned long long h = n > 0;
  int round = 0;
  while (h) {
    FM_CUDA(cudaMemsetAsync(left.p, 0, 8, s));
    k_color_round<<<grid_for(n, 256), 256, 0, s>>>(n, indptr, indices, a, b, round,
                                                   left.as<unsigned long long>());
    FM_CHECK_LAUNCH();
    FM_CUDA(cudaMemcpyAsync(&h, left.p, 8, cudaMemcpyDeviceToHost, s));
    FM_CUDA(cudaStreamSynchronize(s));
    std::swap(a, b);
    if (++round > 1 << 20) {
      set_error("distance-2 colouring did not converge");
      return FM_CUDA_ERROR;
    }
  }
  if (a != colors) FM_CUDA(cudaMemcpyAsync(colors, a, n * 4, cudaMemcpyDeviceToDevice, s));
  int32_t mx = -1;
  if (n > 0) {
    Scratch m;
    FM_CUDA(m.alloc(4, s));
    FM_CUDA(cub_run([&](void *t, size_t &bb) {
      return cub::DeviceReduce::Max(t, bb, colors, m.as<int32_t>(), n, s);
    }, s));
    FM_CUDA(cudaMemcpyAsync(&mx, m.p, 4, cudaMemcpyDeviceToHost, s));
    FM_CUDA(cudaStreamSynchronize(s));
  }
  *ncolors_host = mx + 1;
  return FM_OK;
}

int fm_hess_perturb(int64_t nfree_dofs, const int64_t *dofs_minim, const int32_t *colors,
                    int color, double step, double *vp, void *stream) {
  FM_NVTX("fm_hess_perturb");
  cudaStream_t s = as_stream(stream);
  k_hess_perturb<<<grid_for(nfree_dofs, 256), 256, 0, s>>>(nfree_dofs, dofs_minim, colors, color,
                                                           step, vp);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

int fm_hess_scatter(int64_t n, const int64_t *indptr, const int64_t *indices,
                    const int32_t *colors, int color, const double *g_pert, const double *g0,
                    double step, double *vals, void *stream) {
  FM_NVTX("fm_hess_scatter");
  cudaStream_t s = as_stream(stream);
  k_hess_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, indptr, indices, colors, color, g_pert, g0,
                                                  step, vals);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

int fm_hess_symmetrize(int64_t n, const int64_t *indptr, const int64_t *indices,
                       const double *vals, double *out, void *stream) {
  FM_NVTX("fm_hess_symmetrize");
  cudaStream_t s = as_stream(stream);
  k_hess_sym<<<grid_for(n, 256), 256, 0, s>>>(n, indptr, indices, vals, out);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

}  // extern "C"
