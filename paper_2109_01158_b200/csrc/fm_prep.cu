// GPU preprocessing: mesh generators, P1 gradients, Dirichlet
// partitions, nodal-patch CSR, constant loads and seeded fields.
//
// Index outputs are bit-exact with the reference femmin package:
//   generate_lshape_mesh_2d  mesh.py:200-221 (+ _grid_triangles 177-192,
//                            _compress_nodes 195-197, closed-form ranks)
//   generate_bar_mesh_3d     mesh.py:125-174 (Kuhn split, closed-form flips)
//   mark_dirichlet           mesh.py:289-322
//   build_patches            patches.py:37-71 (stable radix sort by (rank, elem))
// Coordinates follow numpy.linspace exactly: x_i = fl(fl(i*step) + start),
// last = stop (explicit __dmul_rn/__dadd_rn: no FMA contraction).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "fm_common.cuh"

namespace fm {

__device__ __forceinline__ double linspace_at(int64_t i, int64_t n, double start,
                                              double stop, double step) {
  if (i == n) return stop;
  return __dadd_rn(__dmul_rn((double)i, step), start);
}

// ---------------------------------------------------------------- L-shape
__global__ void k_lshape_coords(int64_t n, double step, int64_t nn, double *coords) {
  const int64_t half = n / 2, lower = half * (half + 1);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nn;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t ix, iy;
    if (r < lower) {
      iy = r / (half + 1);
      ix = r % (half + 1);
    } else {
      int64_t q = r - lower;
      iy = half + q / (n + 1);
      ix = q % (n + 1);
    }
    coords[2 * r] = linspace_at(ix, n, -1.0, 1.0, step);
    coords[2 * r + 1] = linspace_at(iy, n, -1.0, 1.0, step);
  }
}

__device__ __forceinline__ int64_t lshape_rank(int64_t ix, int64_t iy, int64_t n) {
  const int64_t half = n / 2;
  if (iy < half) return iy * (half + 1) + ix;
  return half * (half + 1) + (iy - half) * (n + 1) + ix;
}

__global__ void k_lshape_conn(int64_t n, int64_t ncells, int64_t *conn) {
  const int64_t half = n / 2, lower = half * half;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < ncells;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t ix, iy;
    if (q < lower) {
      iy = q / half;
      ix = q % half;
    } else {
      int64_t t = q - lower;
      iy = half + t / n;
      ix = t % n;
    }
    int64_t ll = lshape_rank(ix, iy, n), lr = lshape_rank(ix + 1, iy, n);
    int64_t ul = lshape_rank(ix, iy + 1, n), ur = lshape_rank(ix + 1, iy + 1, n);
    int64_t *c = conn + 6 * q;
    c[0] = ll; c[1] = lr; c[2] = ur;
    c[3] = ll; c[4] = ur; c[5] = ul;
  }
}

// ---------------------------------------------------------------- rectangle
__global__ void k_rect(int64_t nx, int64_t ny, double x0, double x1, double sx, double y0,
                       double y1, double sy, double *coords, int64_t *conn) {
  const int64_t nn = (nx + 1) * (ny + 1), nc = nx * ny;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn || i < nc;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nn) {
      int64_t ix = i % (nx + 1), iy = i / (nx + 1);
      coords[2 * i] = linspace_at(ix, nx, x0, x1, sx);
      coords[2 * i + 1] = linspace_at(iy, ny, y0, y1, sy);
    }
    if (i < nc) {
      int64_t ix = i % nx, iy = i / nx;
      int64_t ll = ix + (nx + 1) * iy;
      int64_t *c = conn + 6 * i;
      c[0] = ll; c[1] = ll + 1; c[2] = ll + nx + 2;
      c[3] = ll; c[4] = ll + nx + 2; c[5] = ll + nx + 1;
    }
  }
}

// ---------------------------------------------------------------- Kuhn beam
// itertools.permutations(range(3)) order; odd permutations (t = 1, 2, 5) are
// negatively oriented on a positive box and swap local nodes 2 <-> 3.
__constant__ int8_t c_kuhn_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                         {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

__global__ void k_beam_coords(int64_t nx, int64_t ny, int64_t nz, int64_t ix0, int64_t nxl,
                              double x0, double x1, double sx, double y0, double y1, double sy,
                              double z0, double z1, double sz, double *coords) {
  // slab [ix0, ix0 + nxl] of the global (nx, ny, nz) grid; global linspace
  const int64_t nn = (nxl + 1) * (ny + 1) * (nz + 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t ix = i % (nxl + 1), t = i / (nxl + 1);
    int64_t iy = t % (ny + 1), iz = t / (ny + 1);
    coords[3 * i] = linspace_at(ix + ix0, nx, x0, x1, sx);
    coords[3 * i + 1] = linspace_at(iy, ny, y0, y1, sy);
    coords[3 * i + 2] = linspace_at(iz, nz, z0, z1, sz);
  }
}

__global__ void k_beam_conn(int64_t nx, int64_t ny, int64_t nz, int64_t *conn) {
  const int64_t ncubes = nx * ny * nz, ne = 6 * ncubes;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = e / 6;
    int t = (int)(e % 6);
    int64_t cx = c % nx, r = c / nx;
    int64_t cy = r % ny, cz = r / ny;
    int64_t off[3] = {0, 0, 0};
    int64_t loc[4];
    loc[0] = cx + (nx + 1) * (cy + (ny + 1) * cz);
    for (int k = 0; k < 3; ++k) {
      off[c_kuhn_perm[t][k]] += 1;
      loc[k + 1] = (cx + off[0]) + (nx + 1) * ((cy + off[1]) + (ny + 1) * (cz + off[2]));
    }
    if (t == 1 || t == 2 || t == 5) {
      int64_t s = loc[2];
      loc[2] = loc[3];
      loc[3] = s;
    }
    int64_t *o = conn + 4 * e;
    o[0] = loc[0]; o[1] = loc[1]; o[2] = loc[2]; o[3] = loc[3];
  }
}

// ---------------------------------------------------------------- P1 gradients
template <int DIM>
__global__ void k_p1(int64_t ne, const double *__restrict__ X, const int64_t *__restrict__ conn,
                     double *__restrict__ vol, double *__restrict__ dphi,
                     unsigned long long *bad) {
  constexpr int NV = DIM + 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    double x[NV][DIM];
#pragma unroll
    for (int l = 0; l < NV; ++l) {
      int64_t n = conn[e * NV + l];
#pragma unroll
      for (int m = 0; m < DIM; ++m) x[l][m] = X[n * DIM + m];
    }
    double E[DIM][DIM];  // rows: x_l - x_0
#pragma unroll
    for (int r = 0; r < DIM; ++r)
#pragma unroll
      for (int m = 0; m < DIM; ++m) E[r][m] = x[r + 1][m] - x[0][m];
    double det, inv[DIM][DIM];
    if (DIM == 2) {
      det = E[0][0] * E[1][1] - E[0][1] * E[1][0];
      inv[0][0] = E[1][1] / det;
      inv[0][1] = -E[0][1] / det;
      inv[1][0] = -E[1][0] / det;
      inv[1][1] = E[0][0] / det;
    } else {
      double c00 = E[1][1] * E[2][2] - E[1][2] * E[2][1];
      double c01 = E[1][2] * E[2][0] - E[1][0] * E[2][2];
      double c02 = E[1][0] * E[2][1] - E[1][1] * E[2][0];
      det = E[0][0] * c00 + E[0][1] * c01 + E[0][2] * c02;
      double c10 = E[0][2] * E[2][1] - E[0][1] * E[2][2];
      double c11 = E[0][0] * E[2][2] - E[0][2] * E[2][0];
      double c12 = E[0][1] * E[2][0] - E[0][0] * E[2][1];
      double c20 = E[0][1] * E[1][2] - E[0][2] * E[1][1];
      double c21 = E[0][2] * E[1][0] - E[0][0] * E[1][2];
      double c22 = E[0][0] * E[1][1] - E[0][1] * E[1][0];
      // inv = adj / det, adj[i][j] = cof[j][i]
      inv[0][0] = c00 / det; inv[0][1] = c10 / det; inv[0][2] = c20 / det;
      inv[1][0] = c01 / det; inv[1][1] = c11 / det; inv[1][2] = c21 / det;
      inv[2][0] = c02 / det; inv[2][1] = c12 / det; inv[2][2] = c22 / det;
    }
    double v = det / (DIM == 2 ? 2.0 : 6.0);
    vol[e] = v;
    if (!(v > 0.0)) atomicMin(bad, (unsigned long long)e);
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      double s = 0.0;
#pragma unroll
      for (int l = 1; l < NV; ++l) {
        dphi[((int64_t)m * ne + e) * NV + l] = inv[m][l - 1];
        s += inv[m][l - 1];
      }
      dphi[((int64_t)m * ne + e) * NV] = -s;
    }
  }
}

// ---------------------------------------------------------------- Dirichlet
__global__ void k_predicate(int kind, int dim, int d, int64_t nn, const double *X, int axis,
                            double c, double tol, uint32_t compmask, uint8_t *fixed,
                            unsigned long long *matched) {
  unsigned long long cnt = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool hit;
    if (kind == 0) {
      hit = X[i * dim + axis] < tol;
    } else if (kind == 1) {
      hit = X[i * dim + axis] > c;  // c = coordinate - tol, computed by the host
    } else {
      double x = X[i * dim], y = X[i * dim + 1];
      bool outer = (fabs(x + 1.0) < tol) | (fabs(x - 1.0) < tol) | (fabs(y + 1.0) < tol) |
                   (fabs(y - 1.0) < tol);
      bool re = ((fabs(x) < tol) & (y < tol)) | ((fabs(y) < tol) & (x > -tol));
      hit = outer | re;
    }
    if (hit) {
      ++cnt;
      for (int j = 0; j < d; ++j)
        if (compmask & (1u << j)) fixed[i * d + j] = 1;
    }
  }
  if (cnt) atomicAdd(matched, cnt);
}

__global__ void k_dirichlet_flags(int64_t nn, int d, const uint8_t *fixed, uint8_t *node_fixed,
                                  uint8_t *node_free, uint8_t *dof_free) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool all = true;
    for (int j = 0; j < d; ++j) {
      bool f = fixed[i * d + j] != 0;
      all &= f;
      dof_free[i * d + j] = !f;
    }
    node_fixed[i] = all;
    node_free[i] = !all;
  }
}

__global__ void k_local_flags(int64_t nfree, int d, const int64_t *nodes_minim,
                              const uint8_t *fixed, uint8_t *flags) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nfree * d;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = q / d;
    int j = (int)(q % d);
    flags[q] = fixed[nodes_minim[k] * d + j] == 0;
  }
}

__global__ void k_not(int64_t n, const uint8_t *a, uint8_t *b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i] == 0;
}

// flatnonzero(flags) into out, count into *count (device)
static int select_indices(const uint8_t *flags, int64_t n, int64_t *out, int64_t *count_dev,
                          cudaStream_t st) {
  cub::CountingInputIterator<int64_t> it(0);
  size_t bytes = 0;
  FM_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, count_dev, n, st));
  Scratch tmp;
  FM_CUDA(tmp.alloc(bytes, st));
  FM_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, flags, out, count_dev, n, st));
  return FM_OK;
}

// ---------------------------------------------------------------- patches
__global__ void k_rank_of(int64_t nfree, const int64_t *nodes_minim, int64_t *rank_of) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nfree;
       r += (int64_t)gridDim.x * blockDim.x)
    rank_of[nodes_minim[r]] = r;
}

__global__ void k_patch_keys(int64_t nent, int nv, const int64_t *conn, const int64_t *rank_of,
                             int64_t nfree, uint64_t *keys, uint8_t *slots,
                             unsigned long long *lengths) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nent;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = q / nv;
    int s = (int)(q % nv);
    int64_t r = rank_of[conn[q]];
    if (r >= 0) {
      keys[q] = ((uint64_t)r << 32) | (uint64_t)e;
      atomicAdd(&lengths[r], 1ull);
    } else {
      keys[q] = (uint64_t)nfree << 32;
    }
    slots[q] = (uint8_t)s;
  }
}

__global__ void k_patch_unpack(int64_t total, const uint64_t *keys, const uint8_t *slots,
                               int64_t *elems, int64_t *slot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    elems[i] = (int64_t)(keys[i] & 0xffffffffull);
    slot[i] = slots[i];
  }
}

__global__ void k_first_empty(int64_t nfree, const int64_t *lengths,
                              unsigned long long *first) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nfree;
       r += (int64_t)gridDim.x * blockDim.x)
    if (lengths[r] == 0) atomicMin(first, (unsigned long long)r);
}

__global__ void k_node_volsum(int64_t nn, int64_t nent, const uint64_t *keys,
                              const int64_t *start, const double *vol, int nv, int d,
                              double f0, double f1, double f2, double *b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = start[i], z = (i + 1 < nn) ? start[i + 1] : nent;
    double s = 0.0;
    for (int64_t q = a; q < z; ++q) s += vol[keys[q] & 0xffffffffull];
    double row = s / (double)nv;
    double f[3] = {f0, f1, f2};
    for (int j = 0; j < d; ++j) b[i * d + j] = f[j] * row;
  }
}

// nodal f: b_i = sum_{k ∋ i} |T_k| (f_i + sum_b f_{k,b}) / (nv (nv+1)), the
// row of the exact local mass (1 + delta_ab) / (nv (nv+1)) |T| (assembly.py:52-62)
__global__ void k_node_load(int64_t nn, int64_t nent, const uint64_t *keys, const int64_t *start,
                            const double *vol, const int64_t *conn, int nv, int d,
                            const double *f, double *b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = start[i], z = (i + 1 < nn) ? start[i + 1] : nent;
    for (int j = 0; j < d; ++j) {
      double s = 0.0;
      for (int64_t q = a; q < z; ++q) {
        int64_t e = (int64_t)(keys[q] & 0xffffffffull);
        double fs = f[i * d + j];
        for (int l = 0; l < nv; ++l) fs += f[conn[e * nv + l] * d + j];
        s += vol[e] * fs;
      }
      b[i * d + j] = s / (double)(nv * (nv + 1));
    }
  }
}

__global__ void k_node_keys(int64_t nent, int nv, const int64_t *conn, uint64_t *keys,
                            unsigned long long *counts) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nent;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = conn[q];
    keys[q] = ((uint64_t)n << 32) | (uint64_t)(q / nv);
    atomicAdd(&counts[n], 1ull);
  }
}

// ---------------------------------------------------------------- fields
__device__ __forceinline__ uint64_t hash_index(int64_t dof, int d, const int64_t *gid) {
  return gid ? (uint64_t)(gid[dof / d] * d + dof % d) : (uint64_t)dof;
}

__global__ void k_field_uniform(int64_t nfd, const int64_t *dofs, int d, const int64_t *gid,
                                uint64_t base, double *v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nfd;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t dof = dofs[i];
    v[dof] = uniform01(base, hash_index(dof, d, gid));
  }
}

__global__ void k_field_nh(int64_t nfd, const int64_t *dofs, int d, const int64_t *gid,
                           uint64_t base, double amp, double *v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nfd;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t dof = dofs[i];
    double u = uniform01(base, hash_index(dof, d, gid));
    v[dof] = __dadd_rn(v[dof], __dmul_rn(amp, __dsub_rn(2.0 * u, 1.0)));
  }
}

static int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

}  // namespace fm

using namespace fm;

extern "C" {

int fm_lshape_sizes(int level, int64_t *nn, int64_t *ne) {
  FM_ARG(level >= 0, "level must be >= 0");
  FM_ARG(level <= 14, "level too large");
  int64_t n = (int64_t)1 << (level + 2), half = n / 2;
  *nn = (n + 1) * (n + 1) - half * half;
  *ne = 2 * (n * n - half * half);
  return FM_OK;
}

int fm_gen_lshape(int level, double *coords, int64_t *conn, void *stream) {
  FM_NVTX("fm_gen_lshape");
  int64_t nn, ne;
  int st = fm_lshape_sizes(level, &nn, &ne);
  if (st) return st;
  int64_t n = (int64_t)1 << (level + 2);
  double step = 2.0 / (double)n;  // numpy: delta / div with delta = 1 - (-1)
  cudaStream_t s = as_stream(stream);
  k_lshape_coords<<<grid_for(nn, 256), 256, 0, s>>>(n, step, nn, coords);
  k_lshape_conn<<<grid_for(ne / 2, 256), 256, 0, s>>>(n, ne / 2, conn);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

int fm_gen_rect(int nx, int ny, double x0, double x1, double y0, double y1, double *coords,
                int64_t *conn, void *stream) {
  FM_NVTX("fm_gen_rect");
  FM_ARG(nx > 0 && ny > 0, "grid sizes must be positive");
  int64_t n = std::max<int64_t>((int64_t)(nx + 1) * (ny + 1), (int64_t)nx * ny);
  k_rect<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(nx, ny, x0, x1, (x1 - x0) / nx, y0,
                                                           y1, (y1 - y0) / ny, coords, conn);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

int fm_gen_beam(int nx, int ny, int nz, const double *b, int ix0, int ix1, double *coords,
                int64_t *conn, void *stream) {
  FM_NVTX("fm_gen_beam");
  FM_ARG(nx > 0 && ny > 0 && nz > 0, "grid sizes must be positive");
  FM_ARG(b[1] > b[0] && b[3] > b[2] && b[5] > b[4], "bar dimensions must be positive");
  FM_ARG(0 <= ix0 && ix0 < ix1 && ix1 <= nx, "slab range must satisfy 0 <= ix0 < ix1 <= nx");
  cudaStream_t s = as_stream(stream);
  const int64_t nxl = ix1 - ix0;
  int64_t nn = (nxl + 1) * (ny + 1) * (nz + 1), ne = 6ll * nxl * ny * nz;
  k_beam_coords<<<grid_for(nn, 256), 256, 0, s>>>(nx, ny, nz, ix0, nxl, b[0], b[1],
                                                  (b[1] - b[0]) / nx, b[2], b[3],
                                                  (b[3] - b[2]) / ny, b[4], b[5],
                                                  (b[5] - b[4]) / nz, coords);
  k_beam_conn<<<grid_for(ne, 256), 256, 0, s>>>(nxl, ny, nz, conn);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

int fm_p1_gradients(int dim, int64_t nn, int64_t ne, const double *coords, const int64_t *conn,
                    double *volumes, double *dphi, int64_t *bad_elem_host, void *stream) {
  FM_NVTX("fm_p1_gradients");
  FM_ARG(dim == 2 || dim == 3, "dim must be 2 or 3");
  (void)nn;
  cudaStream_t s = as_stream(stream);
  Scratch bad;
  FM_CUDA(bad.alloc(8, s));
  FM_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, s));
  if (dim == 2)
    k_p1<2><<<grid_for(ne, 256), 256, 0, s>>>(ne, coords, conn, volumes, dphi,
                                              bad.as<unsigned long long>());
  else
    k_p1<3><<<grid_for(ne, 256), 256, 0, s>>>(ne, coords, conn, volumes, dphi,
                                              bad.as<unsigned long long>());
  FM_CHECK_LAUNCH();
  unsigned long long h = 0;
  FM_CUDA(cudaMemcpyAsync(&h, bad.p, 8, cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  if (h != ~0ull) {
    *bad_elem_host = (int64_t)h;
    double v = 0.0;
    FM_CUDA(cudaMemcpy(&v, volumes + h, 8, cudaMemcpyDeviceToHost));
    char buf[128];
    snprintf(buf, sizeof buf, "element %lld has nonpositive measure %.3e", (long long)h, v);
    set_error(buf);
    return FM_DEGENERATE;
  }
  *bad_elem_host = -1;
  return FM_OK;
}

int fm_dirichlet_predicate(int kind, int dim, int d, int64_t nn, const double *coords, int axis,
                           double c, double tol, const int32_t *comps, int ncomps,
                           uint8_t *fixed, int64_t *matched_host, void *stream) {
  FM_NVTX("fm_dirichlet_predicate");
  FM_ARG(kind >= 0 && kind <= 2, "unknown predicate kind");
  FM_ARG(axis >= 0 && axis < dim, "axis out of range");
  FM_ARG(d >= 1 && d <= 3, "d must be 1..3");
  uint32_t mask = 0;
  if (!comps || ncomps < 0) {
    mask = (1u << d) - 1;
  } else {
    for (int k = 0; k < ncomps; ++k) {
      FM_ARG(comps[k] >= 0 && comps[k] < d, "component out of range");
      mask |= 1u << comps[k];
    }
  }
  cudaStream_t s = as_stream(stream);
  Scratch cnt;
  FM_CUDA(cnt.alloc(8, s));
  FM_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
  k_predicate<<<grid_for(nn, 256), 256, 0, s>>>(kind, dim, d, nn, coords, axis, c, tol, mask,
                                                fixed, cnt.as<unsigned long long>());
  FM_CHECK_LAUNCH();
  unsigned long long h = 0;
  FM_CUDA(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  *matched_host = (int64_t)h;
  return FM_OK;
}

int fm_mark_dirichlet(int64_t nn, int d, const uint8_t *fixed, int64_t *nodes_dirichlet,
                      int64_t *nodes_minim, int64_t *dofs_dirichlet, int64_t *dofs_minim,
                      int64_t *dofs_minim_local, int64_t *counts_host, void *stream) {
  FM_NVTX("fm_mark_dirichlet");
  FM_ARG(d >= 1 && d <= 3, "d must be 1..3");
  cudaStream_t s = as_stream(stream);
  Scratch fl, cnt;
  FM_CUDA(fl.alloc((size_t)nn * (2 + 2 * d), s));
  FM_CUDA(cnt.alloc(5 * sizeof(int64_t), s));
  uint8_t *node_fixed = fl.as<uint8_t>(), *node_free = node_fixed + nn;
  uint8_t *dof_free = node_free + nn, *local = dof_free + nn * d;
  int64_t *c = cnt.as<int64_t>();
  k_dirichlet_flags<<<grid_for(nn, 256), 256, 0, s>>>(nn, d, fixed, node_fixed, node_free,
                                                      dof_free);
  FM_CHECK_LAUNCH();
  int st;
  if ((st = select_indices(node_fixed, nn, nodes_dirichlet, c + 0, s))) return st;
  if ((st = select_indices(node_free, nn, nodes_minim, c + 1, s))) return st;
  if ((st = select_indices(fixed, nn * d, dofs_dirichlet, c + 2, s))) return st;
  if ((st = select_indices(dof_free, nn * d, dofs_minim, c + 3, s))) return st;
  int64_t h[5];
  FM_CUDA(cudaMemcpyAsync(h, c, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  k_local_flags<<<grid_for(h[1] * d, 256), 256, 0, s>>>(h[1], d, nodes_minim, fixed, local);
  FM_CHECK_LAUNCH();
  if ((st = select_indices(local, h[1] * d, dofs_minim_local, c + 4, s))) return st;
  FM_CUDA(cudaMemcpyAsync(h + 4, c + 4, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < 5; ++k) counts_host[k] = h[k];
  return FM_OK;
}

int fm_build_patches(int64_t nn, int64_t ne, int nv, const int64_t *conn,
                     const int64_t *nodes_minim, int64_t nfree, int64_t *lengths,
                     int64_t *prefix, int64_t *elems, int64_t *slot, int64_t *total_host,
                     int64_t *bad_node_host, void *stream) {
  FM_NVTX("fm_build_patches");
  FM_ARG(nv >= 2 && nv <= 4, "nv must be 2..4");
  FM_ARG(ne < (1ll << 32) && nfree < (1ll << 31), "mesh too large for 32-bit patch keys");
  cudaStream_t s = as_stream(stream);
  const int64_t nent = ne * nv;
  *bad_node_host = -1;
  *total_host = 0;
  if (nfree == 0) return FM_OK;
  Scratch rk, keys, keys2, sl, sl2, len, misc;
  FM_CUDA(rk.alloc(nn * sizeof(int64_t), s));
  FM_CUDA(keys.alloc(nent * 8, s));
  FM_CUDA(keys2.alloc(nent * 8, s));
  FM_CUDA(sl.alloc(nent, s));
  FM_CUDA(sl2.alloc(nent, s));
  FM_CUDA(len.alloc(nfree * 8, s));
  FM_CUDA(misc.alloc(16, s));
  FM_CUDA(cudaMemsetAsync(rk.p, 0xff, nn * sizeof(int64_t), s));
  FM_CUDA(cudaMemsetAsync(len.p, 0, nfree * 8, s));
  FM_CUDA(cudaMemsetAsync(misc.p, 0xff, 8, s));
  k_rank_of<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, nodes_minim, rk.as<int64_t>());
  k_patch_keys<<<grid_for(nent, 256), 256, 0, s>>>(nent, nv, conn, rk.as<int64_t>(), nfree,
                                                   keys.as<uint64_t>(), sl.as<uint8_t>(),
                                                   len.as<unsigned long long>());
  FM_CHECK_LAUNCH();
  // stable LSD radix sort on (rank << 32 | elem): rows ascending, elems ascending
  int end_bit = 32 + bits_for((uint64_t)nfree);
  size_t bytes = 0;
  cub::DoubleBuffer<uint64_t> dk(keys.as<uint64_t>(), keys2.as<uint64_t>());
  cub::DoubleBuffer<uint8_t> dv(sl.as<uint8_t>(), sl2.as<uint8_t>());
  FM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, nent, 0, end_bit, s));
  {
    Scratch tmp;
    FM_CUDA(tmp.alloc(bytes, s));
    FM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, dk, dv, nent, 0, end_bit, s));
  }
  // lengths (int64), inclusive prefix, first empty patch
  FM_CUDA(cudaMemcpyAsync(lengths, len.p, nfree * 8, cudaMemcpyDeviceToDevice, s));
  bytes = 0;
  FM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, lengths, prefix, nfree, s));
  {
    Scratch tmp;
    FM_CUDA(tmp.alloc(bytes, s));
    FM_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, bytes, lengths, prefix, nfree, s));
  }
  k_first_empty<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, lengths,
                                                     misc.as<unsigned long long>());
  FM_CHECK_LAUNCH();
  int64_t total = 0;
  unsigned long long first = 0;
  FM_CUDA(cudaMemcpyAsync(&total, prefix + nfree - 1, 8, cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaMemcpyAsync(&first, misc.p, 8, cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  if (first != ~0ull) {
    int64_t node = 0;
    FM_CUDA(cudaMemcpy(&node, nodes_minim + first, 8, cudaMemcpyDeviceToHost));
    *bad_node_host = node;
    char buf[96];
    snprintf(buf, sizeof buf, "free node %lld has an empty patch", (long long)node);
    set_error(buf);
    return FM_PATCH_STRUCTURE;
  }
  k_patch_unpack<<<grid_for(total, 256), 256, 0, s>>>(total, dk.Current(), dv.Current(), elems,
                                                      slot);
  FM_CHECK_LAUNCH();
  *total_host = total;
  return FM_OK;
}

static int load_impl(int dim, int d, int64_t nn, int64_t ne, const int64_t *conn,
                     const double *volumes, const double *f, const double *f_nodal, double *b,
                     void *stream) {
  FM_ARG(dim == 2 || dim == 3, "dim must be 2 or 3");
  FM_ARG(d >= 1 && d <= 3, "d must be 1..3");
  FM_ARG(ne < (1ll << 32) && nn < (1ll << 31), "mesh too large");
  cudaStream_t s = as_stream(stream);
  const int nv = dim + 1;
  const int64_t nent = ne * nv;
  Scratch keys, keys2, cnt, start;
  FM_CUDA(keys.alloc(nent * 8, s));
  FM_CUDA(keys2.alloc(nent * 8, s));
  FM_CUDA(cnt.alloc(nn * 8, s));
  FM_CUDA(start.alloc(nn * 8, s));
  FM_CUDA(cudaMemsetAsync(cnt.p, 0, nn * 8, s));
  k_node_keys<<<grid_for(nent, 256), 256, 0, s>>>(nent, nv, conn, keys.as<uint64_t>(),
                                                  cnt.as<unsigned long long>());
  FM_CHECK_LAUNCH();
  size_t bytes = 0;
  int end_bit = 32 + bits_for((uint64_t)nn);
  cub::DoubleBuffer<uint64_t> dk(keys.as<uint64_t>(), keys2.as<uint64_t>());
  FM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, dk, nent, 0, end_bit, s));
  {
    Scratch tmp;
    FM_CUDA(tmp.alloc(bytes, s));
    FM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, dk, nent, 0, end_bit, s));
  }
  bytes = 0;
  FM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.as<int64_t>(), start.as<int64_t>(),
                                        nn, s));
  {
    Scratch tmp;
    FM_CUDA(tmp.alloc(bytes, s));
    FM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.as<int64_t>(),
                                          start.as<int64_t>(), nn, s));
  }
  if (f_nodal) {
    k_node_load<<<grid_for(nn, 256), 256, 0, s>>>(nn, nent, dk.Current(), start.as<int64_t>(),
                                                  volumes, conn, nv, d, f_nodal, b);
  } else {
    double fv[3] = {0, 0, 0};
    for (int j = 0; j < d; ++j) fv[j] = f[j];
    k_node_volsum<<<grid_for(nn, 256), 256, 0, s>>>(nn, nent, dk.Current(), start.as<int64_t>(),
                                                    volumes, nv, d, fv[0], fv[1], fv[2], b);
  }
  FM_CHECK_LAUNCH();
  return FM_OK;
}

int fm_load_constant(int dim, int d, int64_t nn, int64_t ne, const int64_t *conn,
                     const double *volumes, const double *f, double *b, void *stream) {
  FM_NVTX("fm_load_constant");
  return load_impl(dim, d, nn, ne, conn, volumes, f, nullptr, b, stream);
}

int fm_load_nodal(int dim, int d, int64_t nn, int64_t ne, const int64_t *conn,
                  const double *volumes, const double *f, double *b, void *stream) {
  FM_NVTX("fm_load_nodal");
  FM_ARG(f != nullptr, "null nodal load");
  return load_impl(dim, d, nn, ne, conn, volumes, nullptr, f, b, stream);
}

int fm_field_uniform(int64_t ndof, const int64_t *dofs, int64_t nfd, const int64_t *gid,
                     uint64_t seed, double *v, void *stream) {
  FM_NVTX("fm_field_uniform");
  cudaStream_t s = as_stream(stream);
  FM_CUDA(cudaMemsetAsync(v, 0, ndof * 8, s));
  if (nfd)
    k_field_uniform<<<grid_for(nfd, 256), 256, 0, s>>>(nfd, dofs, 1, gid, splitmix64(seed), v);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

int fm_field_nh(int64_t nn, int d, const double *coords, const int64_t *dofs, int64_t nfd,
                const int64_t *gid, uint64_t seed, double amp, double *v, void *stream) {
  FM_NVTX("fm_field_nh");
  cudaStream_t s = as_stream(stream);
  FM_CUDA(cudaMemcpyAsync(v, coords, nn * d * 8, cudaMemcpyDeviceToDevice, s));
  if (nfd)
    k_field_nh<<<grid_for(nfd, 256), 256, 0, s>>>(nfd, dofs, d, gid, splitmix64(seed), amp, v);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

}  // extern "C"
