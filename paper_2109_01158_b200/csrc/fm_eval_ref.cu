// Energy-only streaming kernel, the descent update and the row-batch model
// plugin (the nodal-patch finite-difference gradient is the fused tile kernel's
// FD mode, fm_eval_exact.cu).
// F, det, I1, W follow the reference's rounding order exactly through the
// explicit round-to-nearest forms of fm_density.cuh (assembly.py:35-49,
// models.py:59-126); only the libm ulps of log/pow differ from numpy.
#include "fm_density.cuh"
#include "fm_kernels.h"

namespace fm {

// ----------------------------------------------------------------- energy
// assembly.py:94-106: every element once in storage order; block b sums the
// fixed range [b*per, (b+1)*per) with a fixed tree -> partial[b].
template <int DIM, int MODEL>
__global__ void __launch_bounds__(256) k_energy(TileArgs a, int64_t ne, int64_t per,
                                                const double *__restrict__ v,
                                                double *__restrict__ part,
                                                double *__restrict__ dens, ModelArgs mdl) {
  constexpr int NV = DIM + 1;
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  __shared__ double red[32];
  const int64_t lo = blockIdx.x * per, hi = min(ne, lo + per);
  double acc = 0.0;
  for (int64_t s = lo + threadIdx.x; s < hi; s += blockDim.x) {
    Elem<DIM> E;
    load_elem<DIM>(a.aos, a.conn4, s, E);
    double vv[D][NV];
    gather_v<DIM, D>(v, E.c, vv);
    double F[D][DIM];
    grad_F<DIM, D>(vv, E.g, F);
    double W = density<DIM, MODEL>(F, mdl);
    if (dens) dens[a.s2o[s]] = W;
    acc += E.vol * W;
  }
  double r = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

// b.v over all dofs (assembly.py:89-91), fixed ranges per block.
__global__ void __launch_bounds__(256) k_dot(const double *__restrict__ a,
                                             const double *__restrict__ b, int64_t n, int64_t per,
                                             double *__restrict__ part) {
  __shared__ double red[32];
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += a[i] * b[i];
  double r = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

// J = sum(partials) - sum(dot partials), fixed order, one block.
__global__ void __launch_bounds__(1024) k_finalize(const double *__restrict__ jp, int nj,
                                                   const double *__restrict__ dp, int nd,
                                                   double *__restrict__ out) {
  __shared__ double red[32];
  double a = 0.0, c = 0.0;
  for (int i = threadIdx.x; i < nj; i += blockDim.x) a += jp[i];
  for (int i = threadIdx.x; i < nd; i += blockDim.x) c += dp[i];
  double A = block_sum(a, red);
  double C = block_sum(c, red);
  if (threadIdx.x == 0) {
    out[0] = A - C;
    out[1] = A;
    out[2] = C;
  }
}

// ----------------------------------------------------------------- descent
// free dof q (the order of g and dofs_minim) -> its position in v
__global__ void k_dof_pos(int64_t nfree, int d, const int32_t *free_node, const int32_t *free_out,
                          const uint8_t *free_mask, int32_t *dof_pos) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nfree;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = free_node[r];
    const int mask = free_mask[r];
    int o = free_out[r];
    for (int j = 0; j < d; ++j)
      if (mask & (1 << j)) dof_pos[o++] = (int32_t)(node * d + j);
  }
}

// v[dof_pos[q]] -= alpha g[q]: one thread per free dof, g read coalesced
__global__ void k_descent(int64_t nfd, const int32_t *__restrict__ dof_pos,
                          const double *__restrict__ g, double alpha, double *__restrict__ v) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nfd;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = __ldg(dof_pos + q);
    v[i] = rsub(v[i], rmul(alpha, __ldg(g + q)));
  }
}

// ----------------------------------------------------------------- launchers
template <int DIM, int MODEL>
static cudaError_t energy_t(const TileArgs &aos, int64_t ne, int nblocks, const double *v,
                            double *part, double *dens, const ModelArgs &m, cudaStream_t s) {
  int64_t per = (ne + nblocks - 1) / nblocks;
  k_energy<DIM, MODEL><<<nblocks, 256, 0, s>>>(aos, ne, per, v, part, dens, m);
  return cudaGetLastError();
}

cudaError_t launch_energy(int dim, int model, const TileArgs &aos, int64_t ne, int nblocks,
                          const double *v, double *part, double *dens, const ModelArgs &m,
                          cudaStream_t s) {
  if (dim == 2 && model == FM_MODEL_PLAPLACE)
    return energy_t<2, FM_MODEL_PLAPLACE>(aos, ne, nblocks, v, part, dens, m, s);
  if (dim == 3 && model == FM_MODEL_PLAPLACE)
    return energy_t<3, FM_MODEL_PLAPLACE>(aos, ne, nblocks, v, part, dens, m, s);
  if (dim == 2) return energy_t<2, FM_MODEL_NEOHOOKEAN>(aos, ne, nblocks, v, part, dens, m, s);
  return energy_t<3, FM_MODEL_NEOHOOKEAN>(aos, ne, nblocks, v, part, dens, m, s);
}

cudaError_t launch_dot(const double *a, const double *b, int64_t n, int nblocks, double *part,
                       cudaStream_t s) {
  int64_t per = (n + nblocks - 1) / nblocks;
  k_dot<<<nblocks, 256, 0, s>>>(a, b, n, per, part);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const double *jp, int nj, const double *dp, int nd, double *out,
                            cudaStream_t s) {
  k_finalize<<<1, 1024, 0, s>>>(jp, nj, dp, nd, out);
  return cudaGetLastError();
}

cudaError_t launch_dof_pos(int64_t nfree, int d, const int32_t *free_node, const int32_t *free_out,
                           const uint8_t *free_mask, int32_t *dof_pos, cudaStream_t s) {
  k_dof_pos<<<grid_for(nfree, 256), 256, 0, s>>>(nfree, d, free_node, free_out, free_mask, dof_pos);
  return cudaGetLastError();
}

cudaError_t launch_descent(int64_t nfd, const int32_t *dof_pos, const double *g, double alpha,
                           double *v, cudaStream_t s) {
  k_descent<<<grid_for(nfd, 256), 256, 0, s>>>(nfd, dof_pos, g, alpha, v);
  return cudaGetLastError();
}

}  // namespace fm

// ----------------------------------------------------------------- row batches
// The model plugin surface (models.py:59-138) on flat (rows) batches:
// F is stored as D*DIM arrays of n rows (F[j][m] at (j*DIM+m)*n).
namespace fm {

template <int DIM, int MODEL>
__global__ void k_rows(int64_t n, const double *__restrict__ Fs, double *__restrict__ W,
                       double *__restrict__ P, unsigned long long *nbad, ModelArgs mdl) {
  constexpr int D = MODEL == FM_MODEL_NEOHOOKEAN ? DIM : 1;
  unsigned long long bad_local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double F[D][DIM];
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int m = 0; m < DIM; ++m) F[j][m] = Fs[(int64_t)(j * DIM + m) * n + i];
    if (W) W[i] = density<DIM, MODEL>(F, mdl);
    if (P) {
      double Q[D][DIM];
      bool bad;
      ddensity<DIM, MODEL>(F, mdl, Q, bad);
      bad_local += bad;
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int m = 0; m < DIM; ++m) P[(int64_t)(j * DIM + m) * n + i] = Q[j][m];
    }
  }
  if (bad_local) atomicAdd(nbad, bad_local);
}

template <int DIM>
__global__ void k_det_rows(int64_t n, const double *__restrict__ Fs, double *__restrict__ det,
                           double *__restrict__ cof) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double F[DIM][DIM];
#pragma unroll
    for (int j = 0; j < DIM; ++j)
#pragma unroll
      for (int m = 0; m < DIM; ++m) F[j][m] = Fs[(int64_t)(j * DIM + m) * n + i];
    if (det) det[i] = det_F<DIM>(F);
    if (cof) {
      double Cf[DIM][DIM];
      cof_F<DIM>(F, Cf);
#pragma unroll
      for (int j = 0; j < DIM; ++j)
#pragma unroll
        for (int m = 0; m < DIM; ++m) cof[(int64_t)(j * DIM + m) * n + i] = Cf[j][m];
    }
  }
}

// evaluate_F (assembly.py:35-49): vals D x (rows, NV), dphi DIM x (rows, NV) -> F (D*DIM, rows)
template <int DIM>
__global__ void k_eval_F(int64_t rows, int D, const double *__restrict__ vals,
                         const double *__restrict__ dphi, double *__restrict__ F) {
  constexpr int NV = DIM + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows;
    const int j = (int)(i / rows);
    double a[NV];
#pragma unroll
    for (int l = 0; l < NV; ++l) a[l] = vals[((int64_t)j * rows + r) * NV + l];
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      double g[NV];
#pragma unroll
      for (int l = 0; l < NV; ++l) g[l] = dphi[((int64_t)m * rows + r) * NV + l];
      F[((int64_t)j * DIM + m) * rows + r] = einsum_row<NV>(a, g);
    }
  }
}

// segment_sums (patches.py:80-83) as direct fixed-order sums per segment.
__global__ void k_segment_sums(int64_t nseg, const double *__restrict__ vals,
                               const int64_t *__restrict__ indx, double *__restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nseg;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = k ? indx[k - 1] : 0, z = indx[k];
    double s = 0.0;
    for (int64_t q = a; q < z; ++q) s += vals[q];
    out[k] = s;
  }
}

}  // namespace fm

using namespace fm;

static ModelArgs rows_model(const fm_model *m) {
  ModelArgs a;
  a.kind = m->kind;
  a.p = m->p;
  a.C1 = m->C1;
  a.D1 = m->D1;
  a.e_w = m->p / 2.0;
  a.e_dw = (m->p - 2.0) / 2.0;
  return a;
}

extern "C" int fm_density_rows(const fm_model *m, int64_t n, const double *F, double *W,
                               double *P, int64_t *nbad_host, void *stream) {
  FM_NVTX("fm_density_rows");
  FM_ARG(m && F, "null argument");
  FM_ARG(m->dim == 2 || m->dim == 3, "dim must be 2 or 3");
  FM_ARG(m->kind == FM_MODEL_PLAPLACE || m->kind == FM_MODEL_NEOHOOKEAN, "unknown model kind");
  cudaStream_t s = as_stream(stream);
  Scratch bad;
  FM_CUDA(bad.alloc(8, s));
  FM_CUDA(cudaMemsetAsync(bad.p, 0, 8, s));
  ModelArgs a = rows_model(m);
  unsigned g = grid_for(n, 256);
  auto *nb = bad.as<unsigned long long>();
  if (m->dim == 2 && m->kind == FM_MODEL_PLAPLACE)
    k_rows<2, FM_MODEL_PLAPLACE><<<g, 256, 0, s>>>(n, F, W, P, nb, a);
  else if (m->dim == 3 && m->kind == FM_MODEL_PLAPLACE)
    k_rows<3, FM_MODEL_PLAPLACE><<<g, 256, 0, s>>>(n, F, W, P, nb, a);
  else if (m->dim == 2)
    k_rows<2, FM_MODEL_NEOHOOKEAN><<<g, 256, 0, s>>>(n, F, W, P, nb, a);
  else
    k_rows<3, FM_MODEL_NEOHOOKEAN><<<g, 256, 0, s>>>(n, F, W, P, nb, a);
  FM_CHECK_LAUNCH();
  unsigned long long h = 0;
  FM_CUDA(cudaMemcpyAsync(&h, bad.p, 8, cudaMemcpyDeviceToHost, s));
  FM_CUDA(cudaStreamSynchronize(s));
  if (nbad_host) *nbad_host = (int64_t)h;
  return FM_OK;
}

extern "C" int fm_det_rows(int dim, int64_t n, const double *F, double *det, double *cof,
                           void *stream) {
  FM_NVTX("fm_det_rows");
  FM_ARG(dim == 2 || dim == 3, "dim must be 2 or 3");
  cudaStream_t s = as_stream(stream);
  if (dim == 2)
    k_det_rows<2><<<grid_for(n, 256), 256, 0, s>>>(n, F, det, cof);
  else
    k_det_rows<3><<<grid_for(n, 256), 256, 0, s>>>(n, F, det, cof);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

extern "C" int fm_eval_F(int dim, int d, int64_t rows, const double *vals, const double *dphi,
                         double *F, void *stream) {
  FM_NVTX("fm_eval_F");
  FM_ARG(dim == 2 || dim == 3, "dim must be 2 or 3");
  cudaStream_t s = as_stream(stream);
  if (dim == 2)
    k_eval_F<2><<<grid_for(rows * d, 256), 256, 0, s>>>(rows, d, vals, dphi, F);
  else
    k_eval_F<3><<<grid_for(rows * d, 256), 256, 0, s>>>(rows, d, vals, dphi, F);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

extern "C" int fm_segment_sums(int64_t nseg, const double *vals, const int64_t *indx,
                               double *out, void *stream) {
  FM_NVTX("fm_segment_sums");
  cudaStream_t s = as_stream(stream);
  k_segment_sums<<<grid_for(nseg, 256), 256, 0, s>>>(nseg, vals, indx, out);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

// linear_term (assembly.py:89-91): out[0] = a.b with the fixed-order partials.
extern "C" int fm_dot(int64_t n, const double *a, const double *b, double *out, void *stream) {
  FM_NVTX("fm_dot");
  FM_ARG(a && b && out, "null argument");
  cudaStream_t s = as_stream(stream);
  const int nb = sm_count() * 2;
  Scratch part;
  FM_CUDA(part.alloc(nb * sizeof(double), s));
  FM_CUDA(launch_dot(a, b, n, nb, part.as<double>(), s));
  FM_CUDA(launch_finalize(part.as<double>(), nb, part.as<double>(), 0, out, s));
  return FM_OK;
}
