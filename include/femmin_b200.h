/*
 * femmin_b200.h — C ABI of the B200-native P1 energy / gradient engine.
 *
 * This is the drop-in boundary for the reference hot path
 * (/root/reference/pkg/src/femmin).  The reference has no FFI of its own (it is
 * pure numpy); each entry point below replaces the numpy body of the
 * reference function cited beside it, and the Python package
 * paper_2109_01158_b200 binds them through ctypes with the reference's own
 * names, argument meaning and exceptions.
 *
 * Conventions
 *   - Plain C types only.  Array arguments are DEVICE pointers (CUDA global
 *     memory) unless the name ends in _host.  `stream` is a cudaStream_t passed
 *     as void* (NULL = legacy default stream).
 *   - Index arrays follow the reference layout: 0-based int64, connectivity
 *     (ne, dim+1) row-major, dphi as dim stacked (ne, dim+1) arrays, fields
 *     interleaved v[d*i + j].
 *   - Every function returns an int status (fm_status_t); fm_last_error()
 *     returns a thread-local message for the last non-zero status.
 *   - Evaluation calls are asynchronous on `stream`; data-dependent conditions
 *     (inadmissible states) are latched in the context and read with
 *     fm_ctx_check(), which synchronises the stream.
 *   - A context is not re-entrant (one stream at a time); distinct contexts are
 *     independent.  fp64 throughout; results are deterministic (fixed-order
 *     reductions, no floating-point atomics).
 */
#ifndef FEMMIN_B200_H
#define FEMMIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FM_OK = 0,
  FM_INADMISSIBLE = 1,      /* models.py:107-110, gradients.py:110-114 */
  FM_INVALID_ARG = 2,       /* ValueError paths (assembly.py:41-46, gradients.py:28-32, models.py:27-31) */
  FM_CUDA_ERROR = 3,
  FM_DEGENERATE = 4,        /* mesh.py:92-96 DegenerateElementError */
  FM_PATCH_STRUCTURE = 5    /* patches.py:57-59 PatchStructureError */
} fm_status_t;

typedef enum { FM_MODEL_PLAPLACE = 0, FM_MODEL_NEOHOOKEAN = 1 } fm_model_kind;

/* Density plugin parameters: models.py:141-170 (NeoHookean / PLaplacian). */
typedef struct {
  int32_t kind;   /* fm_model_kind */
  int32_t dim;    /* spatial dimension 2 or 3 */
  double p;       /* p-Laplace exponent (p > 1)            models.py:50-56   */
  double C1, D1;  /* Neo-Hookean constants (duck-typed)     models.py:41-47   */
} fm_model;

const char *fm_last_error(void);
int fm_version(void);

/* ------------------------------------------------------------------------ */
/* Preprocessing (GPU).  Index outputs are bit-exact with the reference.      */

/* generate_lshape_mesh_2d (mesh.py:200-221): sizes, then coords (nn,2) and conn (ne,3). */
int fm_lshape_sizes(int level, int64_t *nn_host, int64_t *ne_host);
int fm_gen_lshape(int level, double *coords, int64_t *conn, void *stream);

/* _grid_triangles (mesh.py:177-192) on a linspace rectangle: nn=(nx+1)(ny+1), ne=2 nx ny. */
int fm_gen_rect(int nx, int ny, double x0, double x1, double y0, double y1,
                double *coords, int64_t *conn, void *stream);

/* generate_bar_mesh_3d (mesh.py:125-174) with free (nx,ny,nz) and box
 * {x0,x1,y0,y1,z0,z1}, restricted to the x1-slab of cubes [ix0, ix1) (full
 * mesh: 0, nx) with slab-local x-fastest numbering and the global linspace:
 * nn=(ix1-ix0+1)(ny+1)(nz+1), ne=6 (ix1-ix0) ny nz. */
int fm_gen_beam(int nx, int ny, int nz, const double *box_host, int ix0, int ix1,
                double *coords, int64_t *conn, void *stream);

/* compute_p1_gradients (mesh.py:79-104).  dphi: dim stacked (ne, dim+1).
 * Returns FM_DEGENERATE with *bad_elem_host = first element with vol <= 0. */
int fm_p1_gradients(int dim, int64_t nn, int64_t ne, const double *coords,
                    const int64_t *conn, double *volumes, double *dphi,
                    int64_t *bad_elem_host, void *stream);

/* Built-in Dirichlet predicates (bench.py:126-132, 155-166) writing a fixed
 * mask (nn*d uint8, 1 = fixed).  kind 0: x_axis < tol; kind 1: x_axis > c - tol;
 * kind 2: L-shape full boundary with tol.  Regions OR into the mask. */
int fm_dirichlet_predicate(int kind, int dim, int d, int64_t nn, const double *coords,
                           int axis, double c, double tol, const int32_t *comps_host,
                           int ncomps, uint8_t *fixed, int64_t *matched_host, void *stream);

/* mark_dirichlet partitions (mesh.py:307-313) from the fixed mask.  Output
 * buffers sized nn (node lists) and nn*d (dof lists); counts returned. */
int fm_mark_dirichlet(int64_t nn, int d, const uint8_t *fixed,
                      int64_t *nodes_dirichlet, int64_t *nodes_minim,
                      int64_t *dofs_dirichlet, int64_t *dofs_minim,
                      int64_t *dofs_minim_local, int64_t *counts_host /* [5] */,
                      void *stream);

/* build_patches (patches.py:37-71): CSR over free nodes.  elems/slot sized
 * ne*(dim+1) (upper bound); *total_host = ||T||.  lengths/prefix sized nfree.
 * FM_PATCH_STRUCTURE with *bad_node_host = first free node with no element. */
int fm_build_patches(int64_t nn, int64_t ne, int nv, const int64_t *conn,
                     const int64_t *nodes_minim, int64_t nfree, int64_t *lengths,
                     int64_t *prefix, int64_t *elems, int64_t *slot,
                     int64_t *total_host, int64_t *bad_node_host, void *stream);

/* LinearLoad.assemble for a constant f (assembly.py:65-82): b = M f with the
 * P1 mass row sums, b[d*i+j] = f_j * sum_{k ∋ i} |T_k| / (dim+1). */
int fm_load_constant(int dim, int d, int64_t nn, int64_t ne, const int64_t *conn,
                     const double *volumes, const double *f_host, double *b,
                     void *stream);

/* LinearLoad.assemble for a nodal f (nn, d) (device): b = M f with the exact
 * local mass (1 + delta_ab) |T| / (nv (nv+1)) (assembly.py:52-62). */
int fm_load_nodal(int dim, int d, int64_t nn, int64_t ne, const int64_t *conn,
                  const double *volumes, const double *f, double *b, void *stream);

/* Seeded trial fields (counter-based splitmix64, identical to the oracle).
 * The hash index of dof d*i+j is d*gid[i]+j (gid = global node id, NULL =
 * identity) so slabs of a partitioned mesh draw the global field.
 * uniform: v = U[0,1) on free dofs, 0 elsewhere (d = 1).
 * nh:      v = x + amp*(2U-1) on free dofs, v = x on fixed dofs (d = dim). */
int fm_field_uniform(int64_t ndof, const int64_t *dofs_minim, int64_t nfree_dofs,
                     const int64_t *gid, uint64_t seed, double *v, void *stream);
int fm_field_nh(int64_t nn, int d, const double *coords, const int64_t *dofs_minim,
                int64_t nfree_dofs, const int64_t *gid, uint64_t seed, double amp, double *v,
                void *stream);

/* ------------------------------------------------------------------------ */
/* Evaluation context: the frozen Mesh + Patches uploaded once (mesh.py:31-53,
 * patches.py:22-34), re-laid out as node tiles with 80-byte (3D) / 48-byte (2D)
 * element records. */

typedef struct fm_ctx fm_ctx;

typedef struct {
  int32_t dim, d;              /* spatial dim, components (model.d)            */
  int64_t nn, ne;
  const double *coords;        /* (nn, dim)                                     */
  const int64_t *conn;         /* (ne, dim+1)                                   */
  const double *volumes;       /* (ne,)                                         */
  const double *dphi;          /* dim x (ne, dim+1)                             */
  int64_t nfree;               /* |nodes_minim|                                 */
  const int64_t *nodes_minim;  /* (nfree,) ascending                            */
  const uint8_t *fixed;        /* (nn*d) 1 = Dirichlet dof                      */
  const int64_t *p_prefix;     /* (nfree,) inclusive patch prefix p_i           */
  const int64_t *p_elems;      /* (||T||,) ascending per patch                  */
  const int64_t *p_slot;       /* (||T||,) owner slot = argmax(logical)         */
  int64_t p_total;             /* ||T||                                         */
} fm_mesh_desc;

typedef struct {
  int32_t tile_nodes;          /* nodes per tile (<= 512); 0 = default          */
  int32_t box[3];              /* box edge in mesh widths per axis; 0 = default */
} fm_tiling;

typedef struct {
  int64_t n_tiles, n_orphan_tiles, tile_elems_total, node_entries_total;
  int64_t max_tile_elems, max_tile_entries, bytes_device;
  double redundancy;           /* tile element visits / ne                      */
  int32_t tile_threads, ctas_per_sm, node_bufs, table_bufs;  /* tile-kernel launch shape */
  int32_t entry_cap, closure_cap;                            /* per-tile table capacities */
  int64_t cross_entries;       /* node entries whose element another tile computes */
  int64_t dict_tiles;          /* tiles whose element records are dictionary-coded (<= 16
                                  distinct records: 1 B per element streamed instead of 80 / 48) */
} fm_ctx_stats;

int fm_ctx_create(const fm_mesh_desc *desc, const fm_tiling *tiling, void *stream,
                  fm_ctx **out);
int fm_ctx_destroy(fm_ctx *ctx);
int fm_ctx_stats_get(const fm_ctx *ctx, fm_ctx_stats *out);

/* energy (assembly.py:94-106): J_out[0] = vol.W - b.v (device double[3]:
 * J, sum vol W, b.v).  b may be NULL (no load).  densities (ne,) optional
 * (reference element order); det <= 0 gives +inf like models.py:94-99. */
int fm_energy(fm_ctx *ctx, const fm_model *model, const double *v, const double *b,
              double *J_out, double *densities, void *stream);

/* exact_gradient (gradients.py:124-149) into g_out (|dofs_minim|,), optionally
 * fused with the energy (J_out non-NULL, same layout as fm_energy). */
int fm_grad_exact(fm_ctx *ctx, const fm_model *model, const double *v, const double *b,
                  double *g_out, double *J_out, void *stream);

/* Exact Hessian-vector product (new; SURVEY §8f row 4 "exact HVP via d2W"):
 * hp_out (|dofs_minim|,) = d(grad J)(v)[p] = sum_k vol_k d2W/dF2(F_k) : grad p
 * contracted with the basis gradients, on the free dofs; p is a full field
 * (d*nn) that must be zero on the Dirichlet dofs.  det F <= 0 latches like
 * fm_grad_exact.  One fused launch (+ the finishing pass), the same tiles. */
int fm_hvp_exact(fm_ctx *ctx, const fm_model *model, const double *v, const double *p,
                 double *hp_out, void *stream);

/* numeric_gradient (gradients.py:84-121): nodal-patch central differences. */
int fm_grad_fd(fm_ctx *ctx, const fm_model *model, const double *v, const double *b,
               double eps, double *g_out, void *stream);

/* Masked descent v_free <- v_free - alpha * g (config 5 loop; new, not in the
 * reference).  g indexed like dofs_minim. */
int fm_descent_step(fm_ctx *ctx, double *v, const double *g, double alpha, void *stream);

/* First-order descent loop of config 5 (BASELINE.json configs[4]; new, the
 * reference has no such loop — its callers are the minimizers, solver.py):
 * `iters` times { J_hist[3i..3i+2] = J(v) (fm_energy layout); g = grad J(v)
 * (gradients.py:124-149); v_free <- v_free - alpha * g }.  J_hist may be NULL
 * (gradient-only kernels); g (|dofs_minim|,) holds the last gradient.  Fully
 * asynchronous on `stream`; inadmissible states latch (fm_ctx_check). */
int fm_descent(fm_ctx *ctx, const fm_model *model, double *v, const double *b, double alpha,
               int iters, double *g, double *J_hist, void *stream);

/* Device-resident Steihaug truncated CG of the trust-region minimizer
 * (solver.py:77-113).  `state` is a device double[32]
 * holding the CG scalars: [4] radius, [5] rtol, [13] h scale sqrt(eps)(1+|x|),
 * [18] fixed FD step (0: h = scale / |d|) are set by the caller; [16] done,
 * [17] hit the boundary, [15] iterations are read back.  `part` / `ticket`:
 * device scratch of fm_cg_scratch_doubles() doubles / one zeroed unsigned.
 * fm_cg_init: z = 0, r = -g, d = r.  fm_cg_embed: out[free dof q] = x[q] +
 * sign * h * d[q] (x NULL: 0; use_h 0: h = 1), the full field of a
 * Hessian-vector product.  fm_cg_iterate: one CG iteration after the product
 * (Hd given, or gp / gm the gradients at x -/+ h d: Hd = (gp - gm) / (2 h)),
 * all decisions on the device; no-op once done. */
int fm_cg_scratch_doubles(void);
int fm_cg_init(int64_t n, const double *g, double *r, double *d, double *z, double *state,
               double *part, unsigned *ticket, void *stream);
int fm_cg_embed(fm_ctx *ctx, const double *x, const double *d, const double *state, int use_h,
                double sign, double *out, void *stream);
int fm_cg_iterate(int64_t n, const double *gp, const double *gm, double *Hd, double *z,
                  double *znew, double *r, double *d, double *state, double *part,
                  unsigned *ticket, void *stream);

/* x1-slab exchange of the multi-GPU split (one process per GPU).
 * NCCL is resolved at run time (the process's already-loaded libnccl.so.2
 * first).  fm_comm_unique_id: rank 0's 128-byte ncclUniqueId, to be
 * broadcast by the caller.  fm_slab_create: the communicator (current device)
 * and the device positions in g of the interface-plane dofs shared with the
 * left / right neighbour (n_plane each; NULL where there is no neighbour).
 * fm_slab_reduce (stream-ordered): g += the neighbours' partials at the plane
 * dofs and J (device double[3]) = the sum over ranks of every rank's J
 * partials in rank order; one pack kernel, one grouped NCCL launch (planes
 * both ways + J all-gather), one unpack kernel.  Either g or J may be NULL. */
typedef struct fm_slab fm_slab;
int fm_comm_unique_id(void *id_host);
int fm_slab_create(const void *id_host, int rank, int world, int64_t n_plane,
                   const int64_t *left_pos, const int64_t *right_pos, fm_slab **out);
int fm_slab_reduce(fm_slab *x, double *g, double *J, void *stream);
int fm_slab_destroy(fm_slab *x);

/* Sub-slab stack (new): a rank's slab held as K evaluation contexts on one
 * GPU (cfg5 at 2 GPUs: 805 M tetrahedra per rank exceed one context), their
 * gradients back to back in g.  For the n interface dofs shared by
 * consecutive sub-slabs (positions a[k], b[k] in g, device int64):
 * g[a[k]] = g[b[k]] = g[a[k]] + g[b[k]]; with J non-NULL, J (device
 * double[3]) = the K sub-slab partials jk (K x 3) summed in order.  No
 * reference counterpart (the reference is single-domain); the sums are the
 * element sums of gradients.py:124-149 split at the sub-slab planes. */
int fm_stack_reduce(int64_t n, const int64_t *a, const int64_t *b, double *g, const double *jk,
                    int K, double *J, void *stream);

/* Synchronises `stream`, returns the latched condition of the evaluations
 * since the last check and clears it: FM_OK or FM_INADMISSIBLE with
 * *index_host = offending dof (FD, gradients.py:77-81) or -1 (exact path). */
int fm_ctx_check(fm_ctx *ctx, void *stream, int64_t *index_host);

/* Model plugin on flat row batches (models.py:59-138).  F holds D*dim arrays
 * of n rows (entry (j,m) at offset (j*dim+m)*n).  W (n,) and/or P (same
 * layout as F) may be NULL; *nbad_host = rows with det <= 0 (NH dW/dF). */
int fm_density_rows(const fm_model *model, int64_t n, const double *F, double *W, double *P,
                    int64_t *nbad_host, void *stream);
/* batch_determinant / batch_cofactor (models.py:59-86); det, cof nullable. */
int fm_det_rows(int dim, int64_t n, const double *F, double *det, double *cof, void *stream);
/* evaluate_F (assembly.py:35-49): vals d x (rows, dim+1), dphi dim x (rows, dim+1)
 * -> F (d*dim, rows), numpy einsum summation order. */
int fm_eval_F(int dim, int d, int64_t rows, const double *vals, const double *dphi, double *F,
              void *stream);
/* linear_term (assembly.py:89-91): out[0] = a . b; out is device double[3]. */
int fm_dot(int64_t n, const double *a, const double *b, double *out, void *stream);
/* segment_sums (patches.py:80-83) as direct fixed-order per-segment sums. */
int fm_segment_sums(int64_t nseg, const double *vals, const int64_t *indx, double *out,
                    void *stream);

/* ------------------------------------------------------------------------ */
/* Hessian utilities (solver.py:344-398).                   */

/* hessian_sparsity (solver.py:344-357): boolean pattern of the free-dof
 * Hessian (node adjacency of the elements, d x d blocks, rows / columns =
 * positions in dofs_minim) as CSR with ascending columns.  indptr
 * (nfree_dofs + 1) may be NULL to query *nnz_host; indices (nnz) NULL skips
 * the column pass. */
int fm_hessian_pattern(int64_t nn, int64_t ne, int nv, int d, const int64_t *conn,
                       int64_t nfree_dofs, const int64_t *dofs_minim, int64_t *indptr,
                       int64_t *indices, int64_t *nnz_host, void *stream);
/* greedy_coloring (solver.py:360-376) contract: distance-2 colouring of a
 * symmetric pattern (columns sharing a row get distinct colours); parallel
 * rounds instead of the sequential greedy sweep, so the colours may differ. */
int fm_color_d2(int64_t n, const int64_t *indptr, const int64_t *indices, int32_t *colors,
                int32_t *ncolors_host, void *stream);
/* colored_fd_hessian (solver.py:379-398) steps: xp[cols of colour] += step on
 * the full field vp; H[rows, col] = (g_pert - g0)[rows] / step for the
 * pattern columns of that colour; out = (H + H^T) * 0.5 on the pattern. */
int fm_hess_perturb(int64_t nfree_dofs, const int64_t *dofs_minim, const int32_t *colors,
                    int color, double step, double *vp, void *stream);
int fm_hess_scatter(int64_t n, const int64_t *indptr, const int64_t *indices,
                    const int32_t *colors, int color, const double *g_pert, const double *g0,
                    double step, double *vals, void *stream);
int fm_hess_symmetrize(int64_t n, const int64_t *indptr, const int64_t *indices,
                       const double *vals, double *out, void *stream);

/* Arms two cudaEvent_t to be recorded around the next dominant kernel launch
 * of this context (tile kernel of fm_grad_exact / fm_grad_fd, element kernel
 * of fm_energy) on its stream; used by bench.py for the roofline timing. */
int fm_ctx_time_next(fm_ctx *ctx, void *ev_start, void *ev_stop);

/* Number of kernel launches issued by this context so far (bench evidence). */
int64_t fm_ctx_launches(const fm_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* FEMMIN_B200_H */
