// Fused energy + exact gradient over node tiles (gradients.py:124-149 and
// assembly.py:94-106 in one pass).
//
// One CTA owns one tile of free nodes (a spatial box).  It visits every element
// incident to its nodes (its own elements plus a one-element halo), in chunks of
// blockDim elements, one element per thread:
//   phase A  gather record + nodal values, F = grad v, P = vol*dW/dF, and the
//            contributions vol * sum_m dW[j][m] dphi[m][l] for the slots l whose
//            node this tile owns -> shared-memory staging; vol*W for elements the
//            tile owns (each element counted in J exactly once).
//   phase B  each node thread consumes its staged entries in ascending element
//            order (the reference patch order, patches.py:51-53) into registers.
// No floating-point atomics: per-node sums are fixed-order, J is a fixed block
// tree into per-tile partials reduced by fm_finalize in tile order.
#include "fm_density.cuh"
#include "fm_kernels.h"

namespace fm {

template <int DIM, int MODEL, bool WJ, bool WG>
__global__ void __launch_bounds__(512) k_tile_exact(TileArgs a, const double *__restrict__ v,
                                                    const double *__restrict__ b,
                                                    double *__restrict__ g,
                                                    double *__restrict__ jpart,
                                                    unsigned long long *status, ModelArgs mdl) {
  constexpr int NV = DIM + 1;
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *stage = reinterpret_cast<double *>(smem_raw);              // [blockDim][NV][D]
  double *red = stage + (WG ? blockDim.x * NV * D : 0);               // [32]
  uint16_t *ents = reinterpret_cast<uint16_t *>(red + 32);            // tile node entries

  const int t = blockIdx.x;
  const int e0 = a.tile_elem_ptr[t], e1 = a.tile_elem_ptr[t + 1];
  const int n0 = a.tile_node_ptr[t], n1 = a.tile_node_ptr[t + 1];
  const int me = n0 + (int)threadIdx.x;
  const bool has_node = WG && me < n1;
  int cur = 0, end = 0;
  if (WG) {
    const int q0 = a.node_entry_ptr[n0], q1 = a.node_entry_ptr[n1];
    for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) ents[q - q0] = a.node_entries[q];
    if (has_node) {
      cur = a.node_entry_ptr[me] - q0;
      end = a.node_entry_ptr[me + 1] - q0;
    }
  }
  double acc[D];
#pragma unroll
  for (int j = 0; j < D; ++j) acc[j] = 0.0;
  double jsum = 0.0;
  bool bad_any = false;
  if (WG) __syncthreads();

  for (int c0 = e0; c0 < e1; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    if (i < e1) {
      const int s = a.tile_elems[i];
      const int fl = a.tile_flags[i];
      Elem<DIM> E;
      load_elem<DIM>(a.aos, s, E);
      double vv[D][NV];
      gather_v<DIM, D>(v, E, vv);
      double F[D][DIM];
      grad_F<DIM, D>(vv, E.g, F);
      if (WJ && (fl & FLAG_J)) jsum += E.vol * density<DIM, MODEL>(F, mdl);
      if (WG && (fl & 15)) {
        double P[D][DIM];
        bool bad;
        ddensity<DIM, MODEL>(F, mdl, P, bad);
        bad_any |= bad;
        double *row = stage + (size_t)threadIdx.x * NV * D;
#pragma unroll
        for (int l = 0; l < NV; ++l) {
          if (fl & (1 << l)) {
#pragma unroll
            for (int j = 0; j < D; ++j) {
              double sdot = P[j][0] * E.g[0][l];
#pragma unroll
              for (int k = 1; k < DIM; ++k) sdot = sdot + P[j][k] * E.g[k][l];
              row[l * D + j] = E.vol * sdot;
            }
          }
        }
      }
    }
    if (WG) {
      __syncthreads();
      if (has_node) {
        const int base = c0 - e0, lim = base + (int)blockDim.x;
        while (cur < end) {
          const int en = ents[cur];
          const int te = en >> 2;
          if (te >= lim) break;
          const double *src = stage + ((size_t)(te - base) * NV + (en & 3)) * D;
#pragma unroll
          for (int j = 0; j < D; ++j) acc[j] += src[j];
          ++cur;
        }
      }
      __syncthreads();
    }
  }

  if (WG) {
    if (bad_any) atomicOr(status, 1ull);
    if (has_node) {
      const int r = a.tile_node_rank[me];
      const int64_t node = a.free_node[r];
      const int mask = a.free_mask[r];
      int o = a.free_out[r];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (mask & (1 << j)) {
          double bj = b ? __ldg(b + node * D + j) : 0.0;
          g[o++] = acc[j] - bj;
        }
      }
    }
  }
  if (WJ) {
    double s = block_sum(jsum, red);
    if (threadIdx.x == 0) jpart[t] = s;
  }
}

template <int DIM, int MODEL>
static cudaError_t launch_exact_t(const TileArgs &a, int n_tiles, int threads, size_t smem_fixed,
                                  bool wj, bool wg, const double *v, const double *b, double *g,
                                  double *jpart, unsigned long long *status,
                                  const ModelArgs &m, cudaStream_t s) {
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  size_t smem = smem_fixed + 32 * sizeof(double) +
                (wg ? (size_t)threads * (DIM + 1) * D * sizeof(double) : 0);
  if (wj && wg) {
    auto k = k_tile_exact<DIM, MODEL, true, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<n_tiles, threads, smem, s>>>(a, v, b, g, jpart, status, m);
  } else if (wg) {
    auto k = k_tile_exact<DIM, MODEL, false, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<n_tiles, threads, smem, s>>>(a, v, b, g, jpart, status, m);
  } else {
    return cudaErrorInvalidValue;  // J alone streams elements once: k_energy
  }
  return cudaGetLastError();
}

cudaError_t launch_tile_exact(int dim, int model, const TileArgs &a, int n_tiles, int threads,
                              size_t smem_entries, bool wj, bool wg, const double *v,
                              const double *b, double *g, double *jpart,
                              unsigned long long *status, const ModelArgs &m, cudaStream_t s) {
  if (dim == 2 && model == FM_MODEL_PLAPLACE)
    return launch_exact_t<2, FM_MODEL_PLAPLACE>(a, n_tiles, threads, smem_entries, wj, wg, v, b,
                                                g, jpart, status, m, s);
  if (dim == 3 && model == FM_MODEL_PLAPLACE)
    return launch_exact_t<3, FM_MODEL_PLAPLACE>(a, n_tiles, threads, smem_entries, wj, wg, v, b,
                                                g, jpart, status, m, s);
  if (dim == 2)
    return launch_exact_t<2, FM_MODEL_NEOHOOKEAN>(a, n_tiles, threads, smem_entries, wj, wg, v,
                                                  b, g, jpart, status, m, s);
  return launch_exact_t<3, FM_MODEL_NEOHOOKEAN>(a, n_tiles, threads, smem_entries, wj, wg, v, b,
                                                g, jpart, status, m, s);
}

}  // namespace fm
