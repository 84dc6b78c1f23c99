// Internal launcher declarations shared between translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fm_ctx.cuh"

namespace fm {

// persistent pipelined fused J + exact gradient; grid = ctas_per_sm * #SMs, CONSUMERS threads
// ct = threads per CTA = chunk size = max tile nodes (128 or 256); nb = node-value buffers
// tb = table buffers (2: the next tile's descriptors / entries load a tile ahead)
// mode 0: gradient, 1: gradient + J, 2: Hessian-vector product (b = direction),
// 3: nodal-patch FD gradient (m.eps; g = sum / (2 eps) - b, partials unscaled),
// 4: energy only (J partials; g = per-element densities or null)
cudaError_t launch_tile_exact(int dim, int model, const TileArgs &a, int grid, int ct, int nb,
                              int ns, int mode, const double *v, const double *b, double *g,
                              double *jpart, double *bvpart, unsigned long long *status,
                              const ModelArgs &m, cudaStream_t s);
// CTAs per SM the fused tile kernel is compiled for (__launch_bounds__ min
// blocks): 3D <= 128 registers per thread (2 x 256 threads); 2D elements need
// fewer: <= 64 registers gives 4 x 256 threads, 32 warps to hide latency
// (measured: 3 CTAs 0.865 ms, 4 CTAs 0.799 ms, 5 CTAs (spills) 0.862 ms at cfg2)
constexpr int tile_exact_minb(int dim, int ct) {
  return dim == 2 ? (ct == 128 ? 8 : 4) : (ct == 128 ? 4 : 2);
}
// the FD mode (mode 3) of the 2D Neo-Hookean kernel: 3 x 256 threads (<= 85
// registers; its per-element state loop spills at 64: cfg3 FD 0.222 ms at 3
// CTAs); p-Laplace keeps 4 (cfg2 0.94 ms at 4, 0.99 at 3)
constexpr int tile_fd_minb(int dim, int ct, int model) {
  return dim == 2 && model == FM_MODEL_NEOHOOKEAN ? (ct == 128 ? 6 : 3)
                                                  : tile_exact_minb(dim, ct);
}

// J finalisation carried by the finishing pass (see k_finish_cross)
struct JFinal {
  const double *jp, *bvp;      // tile kernel partials per CTA
  int njp;
  const int32_t *fixed_nodes;  // nodes without a free dof
  int64_t nfixed;
  const double *b, *v;
  double *fpart;               // finish_max_blocks()
  unsigned int *ticket;        // zero between calls
  double *out;                 // null: no J
};
// finishing-pass grid cap (32 blocks per SM); sizes the per-block b.v partials
inline int finish_max_blocks() { return sm_count() * 32; }
int finish_cross_grid(int d, int64_t ntn);
cudaError_t launch_finish_cross(int d, int64_t ntn, const int4 *xdesc, const int32_t *xinv,
                                const double *xbuf, const double *partial, double *g,
                                const JFinal &jf, cudaStream_t s);
// the FD gradient's finishing pass: g = (partial + cross entries) / (2 eps) - b
cudaError_t launch_finish_cross_fd(int d, int64_t ntn, const int4 *xdesc, const int32_t *xinv,
                                   const double *xbuf, const double *partial, double *g,
                                   double eps, const double *b, const int4 *node_desc,
                                   cudaStream_t s);
size_t tile_exact_smem(int dim, int d, int blk_cap, int clo_cap, int ct, int nb, int tb,
                       int dn = 0, bool all_coded = false);

// the warp-specialised variant of the fused J + exact gradient (fm_eval_ws.cu):
// one 768-thread CTA per SM (a node group and two element groups), 256-node
// tiles only; modes 0 / 1 of launch_tile_exact, bitwise the same gradient
cudaError_t launch_tile_ws(int dim, int model, const TileArgs &a, int grid, bool wj,
                           const double *v, const double *b, double *g, double *jpart,
                           double *bvpart, unsigned long long *status, const ModelArgs &m,
                           cudaStream_t s);
size_t tile_ws_smem(int dim, int d, int blk_cap, int clo_cap);


cudaError_t launch_energy(int dim, int model, const TileArgs &aos, int64_t ne, int nblocks,
                          const double *v, double *part, double *dens, const ModelArgs &m,
                          cudaStream_t s);

cudaError_t launch_dot(const double *a, const double *b, int64_t n, int nblocks, double *part,
                       cudaStream_t s);

cudaError_t launch_finalize(const double *jp, int nj, const double *dp, int nd, double *out,
                            cudaStream_t s);

cudaError_t launch_dof_pos(int64_t nfree, int d, const int32_t *free_node, const int32_t *free_out,
                           const uint8_t *free_mask, int32_t *dof_pos, cudaStream_t s);
cudaError_t launch_descent(int64_t nfd, const int32_t *dof_pos, const double *g, double alpha,
                           double *v, cudaStream_t s);

}  // namespace fm
