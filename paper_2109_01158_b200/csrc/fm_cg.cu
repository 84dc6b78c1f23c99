// Device-resident Steihaug truncated CG of the trust-region minimizer
// (solver.py:77-113).  The CG scalars (r.r, d.Hd, alpha,
// beta, |z_new|, the boundary step tau) live in a small device state array;
// every iteration is three fused vector kernels after the Hessian-vector
// product, each reducing its dot products with fixed per-block partials that
// the last block to finish (atomic ticket) sums in block order — deterministic
// and decided on the device, so the host reads one flag per iteration instead
// of synchronising on every scalar.  The vector arithmetic follows the
// reference's expressions (z + alpha d, r - alpha Hd, r + beta d,
// z + tau d; the FD product (g(x + h d) - g(x - h d)) / (2 h) with
// h = sqrt(eps) (1 + |x|) / |d|, solver.py:64-74).
#include "fm_density.cuh"
#include "fm_kernels.h"

namespace fm {

// state layout (doubles)
enum CgState {
  CG_RR = 0, CG_DHD, CG_ALPHA, CG_BETA, CG_RADIUS, CG_RTOL, CG_ZD, CG_DD, CG_ZZ, CG_TAU,
  CG_ZNEW2, CG_RRNEW, CG_H, CG_HSCALE, CG_MODE, CG_ITERS, CG_DONE, CG_HIT, CG_HFIX,
  CG_NSTATE = 32
};
// modes decided by the finalisers
constexpr double MODE_CONT = 0.0, MODE_TOL = 1.0, MODE_BOUNDARY = 2.0;

constexpr int CG_THREADS = 256;

// fixed-tree block sums of K values; the last block (ticket) reduces the
// per-block partials in block order and runs fin(sums) on thread 0
template <int K, class Fin>
__device__ __forceinline__ void cg_reduce(double (&x)[K], double *part, unsigned *ticket,
                                          Fin fin) {
  __shared__ double red[32];
  __shared__ bool last;
  double tot[K];
#pragma unroll
  for (int k = 0; k < K; ++k) tot[k] = block_sum(x[k], red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) part[k * gridDim.x + blockIdx.x] = tot[k];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double a = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) a += __ldcg(part + k * gridDim.x + i);
    s[k] = block_sum(a, red);
  }
  if (threadIdx.x == 0) {
    fin(s);
    *ticket = 0u;
  }
}

// z = 0, r = -g, d = r; rr = r.r; done if |r| <= rtol
__global__ void __launch_bounds__(CG_THREADS) k_cg_init(int64_t n, const double *__restrict__ g,
                                                        double *r, double *d, double *z,
                                                        double *st, double *part,
                                                        unsigned *ticket) {
  double x[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = -g[i];
    r[i] = ri;
    d[i] = ri;
    z[i] = 0.0;
    x[0] += ri * ri;
  }
  cg_reduce<1>(x, part, ticket, [&](const double (&s)[1]) {
    st[CG_RR] = s[0];
    st[CG_DD] = s[0];
    st[CG_DONE] = sqrt(s[0]) <= st[CG_RTOL] ? 1.0 : 0.0;
    st[CG_HIT] = 0.0;
    st[CG_MODE] = MODE_CONT;
    st[CG_ITERS] = 0.0;
    st[CG_H] = st[CG_HFIX] > 0.0 ? st[CG_HFIX] : st[CG_HSCALE] / sqrt(s[0]);
  });
}

// out[dof_pos[q]] = (x ? x[q] : 0) + sign * (use_h ? h : 1) * d[q]
__global__ void __launch_bounds__(CG_THREADS) k_cg_embed(int64_t n, const int32_t *__restrict__ dof_pos,
                                                         const double *__restrict__ x,
                                                         const double *__restrict__ d,
                                                         const double *__restrict__ st, int use_h,
                                                         double sign, double *out) {
  if (st[CG_DONE] != 0.0) return;
  const double h = use_h ? sign * st[CG_H] : sign;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double hd = __dmul_rn(h, d[q]);
    out[__ldg(dof_pos + q)] = x ? __dadd_rn(x[q], hd) : hd;
  }
}

// K1: Hd (from the FD gradients when gm != null), d.Hd, z.d, d.d, z.z; decide
// negative curvature (boundary) or alpha = rr / dHd
__global__ void __launch_bounds__(CG_THREADS) k_cg_curv(int64_t n, const double *__restrict__ gp,
                                                        const double *__restrict__ gm,
                                                        double *Hd, const double *__restrict__ d,
                                                        const double *__restrict__ z, double *st,
                                                        double *part, unsigned *ticket) {
  if (st[CG_DONE] != 0.0) return;
  const double inv2h = 2.0 * st[CG_H];
  double x[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double h;
    if (gm) {
      h = __ddiv_rn(__dsub_rn(gp[i], gm[i]), inv2h);
      Hd[i] = h;
    } else {
      h = Hd[i];
    }
    const double di = d[i], zi = z[i];
    x[0] += di * h;
    x[1] += zi * di;
    x[2] += di * di;
    x[3] += zi * zi;
  }
  cg_reduce<4>(x, part, ticket, [&](const double (&s)[4]) {
    st[CG_DHD] = s[0];
    st[CG_ZD] = s[1];
    st[CG_DD] = s[2];
    st[CG_ZZ] = s[3];
    const double R = st[CG_RADIUS];
    st[CG_TAU] = (-s[1] + sqrt(s[1] * s[1] + s[2] * (R * R - s[3]))) / s[2];
    if (s[0] <= 0.0) {
      st[CG_MODE] = MODE_BOUNDARY;
    } else {
      st[CG_ALPHA] = st[CG_RR] / s[0];
      st[CG_MODE] = MODE_CONT;
    }
  });
}

// K2: z_new = z + alpha d, r -= alpha Hd; |z_new|^2, r.r; decide boundary /
// tolerance / continue (beta)
__global__ void __launch_bounds__(CG_THREADS) k_cg_step(int64_t n, const double *__restrict__ z,
                                                        double *znew, double *r,
                                                        const double *__restrict__ d,
                                                        const double *__restrict__ Hd,
                                                        double *st, double *part,
                                                        unsigned *ticket) {
  if (st[CG_DONE] != 0.0 || st[CG_MODE] == MODE_BOUNDARY) return;
  const double alpha = st[CG_ALPHA];
  double x[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double zn = __dadd_rn(z[i], __dmul_rn(alpha, d[i]));
    znew[i] = zn;
    const double rn = __dsub_rn(r[i], __dmul_rn(alpha, Hd[i]));
    r[i] = rn;
    x[0] += zn * zn;
    x[1] += rn * rn;
  }
  cg_reduce<2>(x, part, ticket, [&](const double (&s)[2]) {
    st[CG_ZNEW2] = s[0];
    st[CG_RRNEW] = s[1];
    if (sqrt(s[0]) >= st[CG_RADIUS]) {
      st[CG_MODE] = MODE_BOUNDARY;
    } else if (sqrt(s[1]) <= st[CG_RTOL]) {
      st[CG_MODE] = MODE_TOL;
    } else {
      st[CG_BETA] = s[1] / st[CG_RR];
      st[CG_RR] = s[1];
      st[CG_MODE] = MODE_CONT;
    }
  });
}

// K3: apply the decision: continue (z = z_new, d = r + beta d, next h from
// |d|), tolerance (z = z_new, done) or boundary (z = z + tau d, done)
__global__ void __launch_bounds__(CG_THREADS) k_cg_update(int64_t n, double *z,
                                                          const double *__restrict__ znew,
                                                          const double *__restrict__ r, double *d,
                                                          double *st, double *part,
                                                          unsigned *ticket) {
  if (st[CG_DONE] != 0.0) return;
  const double mode = st[CG_MODE];
  const double beta = st[CG_BETA], tau = st[CG_TAU];
  double x[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (mode == MODE_BOUNDARY) {
      z[i] = __dadd_rn(z[i], __dmul_rn(tau, d[i]));
    } else {
      z[i] = znew[i];
      if (mode == MODE_CONT) {
        const double dn = __dadd_rn(r[i], __dmul_rn(beta, d[i]));
        d[i] = dn;
        x[0] += dn * dn;
      }
    }
  }
  cg_reduce<1>(x, part, ticket, [&](const double (&s)[1]) {
    st[CG_ITERS] += 1.0;
    if (mode == MODE_CONT) {
      st[CG_DD] = s[0];
      st[CG_H] = st[CG_HFIX] > 0.0 ? st[CG_HFIX] : st[CG_HSCALE] / sqrt(s[0]);
    } else {
      st[CG_DONE] = 1.0;
      st[CG_HIT] = mode == MODE_BOUNDARY ? 1.0 : 0.0;
    }
  });
}

}  // namespace fm

using namespace fm;

namespace {
int cg_grid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + CG_THREADS - 1) / CG_THREADS,
                                                     (int64_t)sm_count() * 4));
}
}  // namespace

extern "C" {

int fm_cg_scratch_doubles(void) { return 4 * sm_count() * 4; }

int fm_cg_init(int64_t n, const double *g, double *r, double *d, double *z, double *state,
               double *part, unsigned *ticket, void *stream) {
  FM_NVTX("fm_cg_init");
  FM_ARG(g && r && d && z && state && part && ticket, "null argument");
  FM_ARG(4 * cg_grid(n) <= fm_cg_scratch_doubles(), "CG scratch too small for this GPU");
  k_cg_init<<<cg_grid(n), CG_THREADS, 0, as_stream(stream)>>>(n, g, r, d, z, state, part,
                                                              ticket);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

int fm_cg_embed(fm_ctx *c, const double *x, const double *d, const double *state, int use_h,
                double sign, double *out, void *stream) {
  FM_ARG(c && d && state && out, "null argument");
  const int64_t n = c->nfree_dofs;
  k_cg_embed<<<cg_grid(n), CG_THREADS, 0, as_stream(stream)>>>(n, c->dof_pos, x, d, state, use_h,
                                                               sign, out);
  FM_CHECK_LAUNCH();
  c->launches++;
  return FM_OK;
}

int fm_cg_iterate(int64_t n, const double *gp, const double *gm, double *Hd, double *z,
                  double *znew, double *r, double *d, double *state, double *part,
                  unsigned *ticket, void *stream) {
  FM_NVTX("fm_cg_iterate");
  FM_ARG(gp || Hd, "null product");
  FM_ARG(Hd && z && znew && r && d && state && part && ticket, "null argument");
  cudaStream_t s = as_stream(stream);
  const int grid = cg_grid(n);
  k_cg_curv<<<grid, CG_THREADS, 0, s>>>(n, gp, gm, Hd, d, z, state, part, ticket);
  FM_CHECK_LAUNCH();
  k_cg_step<<<grid, CG_THREADS, 0, s>>>(n, z, znew, r, d, Hd, state, part, ticket);
  FM_CHECK_LAUNCH();
  k_cg_update<<<grid, CG_THREADS, 0, s>>>(n, z, znew, r, d, state, part, ticket);
  FM_CHECK_LAUNCH();
  return FM_OK;
}

}  // extern "C"
