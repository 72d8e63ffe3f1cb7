/*
 * dgmf.h -- C ABI of the B200-native matrix-free DG operator library.
 *
 * Drop-in boundary for the hot path of the reference package `dgins`
 * (arXiv 1607.01323 velocity-correction DG solver; reference tree
 * /root/reference/pkg/src/dgins).  Each entry point below replaces one
 * reference operator/solver function; the citation names the reference
 * signature it stands in for.  The Python shim paper_1607_01323_b200/
 * (operators.py, solvers.py) keeps the reference call signatures and
 * forwards here through ctypes.
 *
 * Conventions
 *  - All vector arguments are DEVICE pointers to fp64 data in element-major
 *    order: (component, cell, [z,] y, x), x fastest, cell id
 *    e = ix + nx*(iy + ny*iz) over the cells this context owns
 *    (the reference serialisation FieldVector.element_major, spaces.py:49-51).
 *  - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *    on that stream (host-side scalars are returned only by functions whose
 *    name says so).
 *  - Outputs are fully overwritten (no hidden accumulation) unless stated.
 *  - Return value: 0 on success, <0 on error; dg_last_error() gives text.
 *    DG_EINVAL maps to the reference's ValueError, DG_ECUDA/DG_ENCCL to
 *    RuntimeError in the shim.
 */
#ifndef DGMF_H
#define DGMF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_OK 0
#define DG_EINVAL -1
#define DG_ECUDA -2
#define DG_ENOTSUP -3

/* boundary kinds per tag; velocity semantics as in the reference
 * (operators.py:189-193: velocity-Dirichlet faces are pressure-Neumann,
 * velocity-Neumann faces are pressure-Dirichlet) */
#define DG_BC_NONE 0              /* periodic axis: no boundary faces        */
#define DG_BC_VELOCITY_DIRICHLET 1 /* reference DirichletBC                  */
#define DG_BC_VELOCITY_NEUMANN 2  /* reference NeumannBC                     */

typedef struct dg_ctx dg_ctx;

/* Mesh + discretisation description.  Replaces the reference's
 * build_box_mesh(...) (mesh.py:279-351) + DgSpace(mesh, k) (spaces.py:61-81)
 * + BoundarySpec.resolve (operators.py:97-131) for axis-aligned boxes. */
typedef struct {
  int dim;                    /* 2 or 3                                        */
  int k;                      /* polynomial degree 1..7 (n = k+1 GLL nodes)    */
  int n_q_over;               /* convective rule points; 0 -> floor(3k/2)+1    */
  int counts[3];              /* GLOBAL cells per axis (counts[2]=1 in 2D)     */
  const double *vertices[3];  /* HOST per-axis vertex coordinates, counts+1    */
  int periodic[3];            /* per axis                                      */
  int bc_kind[6];             /* per tag xmin,xmax,ymin,ymax,zmin,zmax          */
  int slab_begin, slab_end;   /* owned x-cells [begin,end); end<=0 -> all       */
} dg_mesh_desc;

/* ---- context ------------------------------------------------------------ */
int dg_ctx_create(const dg_mesh_desc *desc, dg_ctx **out);
int dg_ctx_destroy(dg_ctx *ctx);
const char *dg_last_error(void);
/* local cells / scalar dofs per component owned by this context */
int dg_ctx_sizes(const dg_ctx *ctx, int64_t *n_cells, int64_t *n_dofs);
/* copy tau_e (Eq. 18, geometry.py:90-108) of the owned cells to host */
int dg_ctx_tau(const dg_ctx *ctx, double *tau_e_host);

/* 1D tables on the host, computed in long double: S[q,i]=l_i(x_q),
 * D[q,i]=l_i'(x_q) on the n_q-point Gauss rule, GLL nodes, Gauss points and
 * weights, endpoint derivative rows.  Replaces gauss_rule/gll_nodes
 * (quadrature.py:48-95) and Basis1D (basis.py:61-84). */
int dg_basis_tables(int k, int n_q, double *S, double *D, double *nodes,
                    double *points, double *weights, double *left_deriv,
                    double *right_deriv);

/* ---- operators (replace operators.py functions) ------------------------- */
/* apply_pressure_laplace(space, p, bcs, tau_scale)  operators.py:187-238 */
int dg_laplace_vmult(dg_ctx *ctx, const double *src, double *dst,
                     double tau_scale, void *stream);
/* apply_pressure_laplace with HOST buffers (the numpy call form of the
 * reference): src_host -> device -> vmult -> dst_host, pipelined in
 * n_chunks z-chunks of whole x-y layers on three streams (H2D, kernel, D2H
 * overlap when the host buffers are pinned).  Whole-mesh contexts; results
 * identical to dg_laplace_vmult.  dst_host is complete once `stream` has
 * reached this call's end (e.g. after cudaStreamSynchronize). */
int dg_laplace_vmult_host(dg_ctx *ctx, const double *src_host, double *dst_host,
                          double tau_scale, int n_chunks, void *stream);
/* laplace_diagonal(space, bcs, tau_scale)  operators.py:717-730 */
int dg_laplace_diagonal(dg_ctx *ctx, double *diag, double tau_scale,
                        void *stream);
/* mass_apply / inverse_mass_apply(space, x)  operators.py:167-181,
 * kernels.py:95-113; ncomp components stored back to back */
int dg_mass(dg_ctx *ctx, const double *src, double *dst, int ncomp,
            void *stream);
int dg_inverse_mass(dg_ctx *ctx, const double *src, double *dst, int ncomp,
                    void *stream);
/* apply_viscous_helmholtz(space, u, gamma0_dt, nu, bcs)  operators.py:418-491;
 * src/dst hold dim components */
int dg_helmholtz_vmult(dg_ctx *ctx, const double *src, double *dst,
                       double gamma0_dt, double nu, void *stream);
/* apply_projection_operator(space, w, tau_d_e, tau_c_f)  operators.py:372-412.
 * tau_d: per owned cell (device, or NULL); tau_c: per face, device array of
 * dim*n_cells entries indexed [d*n_cells + e] = penalty of the face between
 * cell e and its +d neighbour (NULL -> no jump term). */
int dg_projection_vmult(dg_ctx *ctx, const double *src, double *dst,
                        const double *tau_d, const double *tau_c,
                        void *stream);
/* eval_convective_rhs(space, bcs, history, betas, ...)  operators.py:533-594
 * with homogeneous Dirichlet data and no body force (the C3 hot-path case;
 * dg_convective_rhs_ex below takes the data);
 * hist[j] -> dim-component velocity at history level j. dst overwritten. */
int dg_convective_rhs(dg_ctx *ctx, int n_hist, const double *const *hist,
                      const double *betas, double *dst, void *stream);
/* The full eval_convective_rhs: g_data[j*6 + side] = Dirichlet data g of
 * history level j at time times[j] on the over-integration face points
 * (layout of the boundary data below, dim components; NULL entries or a NULL
 * array = zero data); body = body force f(x, t_np1) at the over-integration
 * volume points, [comp][cell][n_q_over^dim] (NULL = none). */
int dg_convective_rhs_ex(dg_ctx *ctx, int n_hist, const double *const *hist,
                         const double *betas, const double *const *g_data,
                         const double *body, double *dst, void *stream);

/* ---- once-per-step right-hand sides (operators.py:241-366, 494-527,
 * 610-672) and the element-local PCG (solvers.py:201-256) --------------
 *
 * Boundary data: bnd[side] (side = 2*d + s: xmin, xmax, ymin, ymax, zmin,
 * zmax) is NULL (zero data) or a device array [ntan][ncomp][n_f] over the
 * boundary cells of that side, ntan = product of the two (one in 2D) other
 * cell counts with the tangential cell index (slow, fast) in decreasing axis
 * order (d=0: iz*ny+iy, d=1: iz*nx+ix, d=2: iy*nx+ix; 2D: iy or ix), and the
 * n_f = n^(dim-1) face Gauss points [slow][fast] in the same axis order.  The
 * caller evaluates the reference's boundary callables at those points. */

/* eval_divergence_rhs(space, u, bcs, scale, form)  operators.py:265-316;
 * form 0 standard, 1 weak (central flux, interior trace on boundaries),
 * 2 strong.  src: dim components; dst: scalar. */
int dg_divergence_rhs(dg_ctx *ctx, const double *src, double *dst, double scale,
                      int form, void *stream);
/* eval_pressure_gradient_rhs(space, p, bcs, scale, form)  operators.py:322-366;
 * form 0 standard, 1 weak.  src: scalar; dst: dim components. */
int dg_pressure_gradient_rhs(dg_ctx *ctx, const double *src, double *dst,
                             double scale, int form, void *stream);
/* compute_vorticity(space, u)  operators.py:610-618: element-local L2
 * projection of curl u; dst: 1 component in 2D, 3 in 3D (no aliasing). */
int dg_vorticity(dg_ctx *ctx, const double *src, double *dst, void *stream);
/* eval_pressure_neumann_rhs(space, bcs, history, vorticity_history, betas, nu,
 * t, body_force)  operators.py:621-672 on velocity-Dirichlet sides.
 * hist[j]: dim-component velocity, vort[j]: its vorticity (1 or 3 comps);
 * bnd[side]: dim components of dg/dt - f at the face points (or NULL). */
int dg_pressure_neumann_rhs(dg_ctx *ctx, int n_hist, const double *const *hist,
                            const double *const *vort, const double *betas,
                            double nu, const double *const *bnd, double *dst,
                            void *stream);
/* gp_dirichlet_rhs(space, bcs, t, tau_scale)  operators.py:241-259 on
 * velocity-Neumann sides; bnd[side]: 1 component (g_p). dst: scalar. */
int dg_gp_dirichlet_rhs(dg_ctx *ctx, const double *const *bnd, double tau_scale,
                        double *dst, void *stream);
/* viscous_rhs_bc(space, bcs, t, nu)  operators.py:494-527.  bnd[side]:
 * velocity-Dirichlet sides dim components (g); velocity-Neumann sides dim+1
 * components (h, g_p).  dst: dim components. */
int dg_viscous_rhs_bc(dg_ctx *ctx, const double *const *bnd, double nu,
                      double *dst, void *stream);
/* element_local_pcg(op_local, prec_local, b, rel_tol, max_iter, floor_factor)
 * solvers.py:201-256 with op_local = apply_projection_operator(space, ., tau_d,
 * None) and prec_local = inverse_mass_apply (the V3 projection).  b, x: dim
 * components (no aliasing); tau_d: per cell (device, NULL = 0); iters /
 * converged: per-cell int32 device arrays (may be NULL). */
int dg_element_local_pcg(dg_ctx *ctx, const double *b, double *x,
                         const double *tau_d, double rel_tol, int max_iter,
                         double floor_factor, int *iters, int *converged,
                         void *stream);

/* compute_penalty_parameters(space, u, dt, cfl, cfg)  operators.py:736-755:
 * tau_D per cell = zeta_d_star/cfl |u_mean| V^(1/dim) dt (tau_d NULL: skip);
 * tau_C per face = average of zeta_c_star/cfl |u_mean| dt of the two cells,
 * in the face layout of dg_projection_vmult (tau_c NULL: skip).  u: dim
 * components. */
int dg_penalty_parameters(dg_ctx *ctx, const double *u, double dt, double cfl,
                          double zeta_d_star, double zeta_c_star, double *tau_d,
                          double *tau_c, void *stream);

/* ---- vector kernels for the solvers (solvers.py) ------------------------ */
/* deterministic fixed-order dot product; result written to device *out */
int dg_dot(dg_ctx *ctx, const double *x, const double *y, int64_t n,
           double *out_dev, void *stream);
/* zero_mean_project_dual (solvers.py:187-198), in place on b (1 component);
 * zero_mean_project (solvers.py:179-184), in place */
int dg_zero_mean_dual(dg_ctx *ctx, double *b, void *stream);
int dg_zero_mean(dg_ctx *ctx, double *p, void *stream);

/* Fused PCG for the SIP Laplacian (solvers.py:30-73), preconditioner
 * Chebyshev(degree, range, lambda_max) over point Jacobi (solvers.py:93-129)
 * or plain Jacobi (degree 0), optional dual zero-mean projection of the
 * operator (pure-Neumann problems).  x: device, initial guess zero.
 * Residual history sqrt(r.z) per iteration written to hist_host
 * (max_iter+1 entries) if non-NULL.  Blocking: returns when done. */
typedef struct {
  double tau_scale;
  int project_dual;        /* op = zero_mean_project_dual o L                */
  int cheb_degree;         /* 0 -> Jacobi                                    */
  double cheb_range;       /* smoothing range (20)                           */
  double cheb_lambda_max;  /* safety * Lanczos estimate                      */
  double rel_tol, abs_tol;
  int max_iter;
} dg_pcg_params;
typedef struct {
  int iterations;
  double residual;
  int converged;
  int breakdown;
} dg_pcg_stats;
int dg_laplace_pcg(dg_ctx *ctx, const double *b, double *x,
                   const double *diag, const dg_pcg_params *prm,
                   dg_pcg_stats *stats, double *hist_host, void *stream);

/* PCG of the velocity solves (solvers.py:30-73 with prec = inverse_mass_apply,
 * operators.py:176-181): op 0 = viscous Helmholtz (gamma0_dt, nu; the
 * context's boundary kinds), op 1 = projection (tau_d per cell, tau_c in the
 * layout of dg_projection_vmult; either NULL to skip).  3D, 3 components.
 * x: initial guess in, solution out (reference x0 semantics; zeros = None).
 * Reference stopping rule sqrt(r.z) <= max(rel_tol sqrt(r0.z0), abs_tol),
 * breakdown flags, residual history as dg_laplace_pcg.  Blocking. */
int dg_vector_pcg(dg_ctx *ctx, int op, double gamma0_dt, double nu,
                  const double *tau_d, const double *tau_c, const double *b,
                  double *x, double rel_tol, double abs_tol, int max_iter,
                  dg_pcg_stats *stats, double *hist_host, void *stream);

/* One Chebyshev step (solvers.py:121-128) fused into the vmult epilogue:
 * rc -= L d_old ; d_new = a d_old + b rc/diag ; x += d_new.  The vector
 * update rounds like the reference's numpy expression (no FMA contraction). */
int dg_cheb_step(dg_ctx *ctx, const double *d_old, double *d_new, double *rc,
                 double *x, const double *diag, double a, double b,
                 double tau_scale, void *stream);

/* ---- geometric multigrid (multigrid.py:33-151, mesh.py:354-374) ---------
 * Levels are contexts of nested boxes (counts doubling per axis, same dim,
 * degree, periodicity and boundary kinds), coarse (0) to fine. */
typedef struct dg_mg dg_mg;
/* Transfer.prolong (multigrid.py:49-58): xf (+)= E xc (add != 0 accumulates);
 * Transfer.restrict (multigrid.py:60-69): xc = E^T xf */
int dg_mg_prolong(dg_ctx *coarse, dg_ctx *fine, const double *xc, double *xf,
                  int add, void *stream);
int dg_mg_restrict(dg_ctx *fine, dg_ctx *coarse, const double *xf, double *xc,
                   void *stream);
/* MultigridHierarchy (multigrid.py:76-128): per-level Jacobi diagonals
 * (device, caller-owned, kept alive) and Chebyshev lambda_max (the
 * reference's safety * Lanczos estimate, computed by the caller from its
 * seeded start vectors); smoother Chebyshev(degree, smoothing_range) over
 * Jacobi; coarsest level Chebyshev(coarse_iters, coarse_range). */
int dg_mg_create(dg_ctx *const *levels, int n_levels, const double *const *diag,
                 const double *lambda_max, int degree, double smoothing_range,
                 int coarse_iters, double coarse_range, double tau_scale,
                 dg_mg **out);
int dg_mg_destroy(dg_mg *mg);
/* MultigridHierarchy.vcycle (multigrid.py:133-151): x = V(b), finest level */
/* Run the V-cycle in single precision (bits = 32; the paper's multigrid is
 * fp32) or back in fp64 (bits = 64, the default and the
 * reference's arithmetic).  fp32: the same algorithm on float level vectors,
 * diagonals and dense coarse operator; input / output stay fp64, so the
 * outer CG (dg_laplace_pcg_mg) is unchanged.  3D hierarchies. */
int dg_mg_set_precision(dg_mg *mg, int bits);
int dg_mg_vcycle(dg_mg *mg, const double *b, double *x, void *stream);
/* dg_laplace_pcg with the V-cycle as preconditioner (prm->cheb_* unused);
 * ctx must be the hierarchy's finest level */
int dg_laplace_pcg_mg(dg_ctx *ctx, dg_mg *mg, const double *b, double *x,
                      const dg_pcg_params *prm, dg_pcg_stats *stats,
                      double *hist_host, void *stream);

/* ---- general-geometry 2D path (reference geometry.py, operators.py) -----
 * Quadrilateral meshes with iso-parametric (curved) mappings and arbitrary
 * conforming connectivity, the reference's own 2D setting.  The caller
 * computes the geometry at the quadrature points (geometry.py:29-87) and
 * the per-(cell, slot) links (spaces.py:140-163) and passes DEVICE arrays in
 * the element-major layouts below; the context keeps the pointers (not
 * owned) and copies the 1D tables.
 *   jxw  [e][q][q]        jit  [e][4][q][q] (J^-T entries 00 01 10 11)
 *   fsj  [e][4][q]        fnrm [e][4][2][q]  fjit [e][4][4][q]
 *   nbr  [e][4] int64 neighbour cell or -1, nslot / nflip [e][4] int32
 *   tau  [e]   Eq. 18 per cell (compute_tau_ip, geometry.py:90-108)
 * On interior faces both cells carry the minus side's sJxW and normal
 * (negated on the plus side) as the reference's gather/scatter does. */
typedef struct dg_g2 dg_g2;
typedef struct {
  int n, nq;            /* nodes per direction (k+1), Gauss points n_q */
  int64_t ncells;
  const double *jxw, *jit, *fsj, *fnrm, *fjit, *tau;   /* device */
  const int64_t *nbr;                                  /* device */
  const int *nslot, *nflip;                            /* device */
  const double *S, *D, *Si, *ld, *rd;                  /* host 1D tables */
} dg_g2_desc;
int dg_g2_create(const dg_g2_desc *desc, dg_g2 **out);
int dg_g2_destroy(dg_g2 *g);
/* op 0 mass (operators.py:167-173), 1 exact inverse mass (:176-181,
 * kernels.py:95-107), 2 SIP pressure Laplacian (:187-238) with kind[e][4]
 * (device int32: 0 interior, DG_BC_VELOCITY_DIRICHLET, DG_BC_VELOCITY_NEUMANN)
 * and tau_scale; ncomp fields of ncells*n*n values each (mass ops) */
int dg_g2_apply(dg_g2 *g, int op, double tau_scale, const int *kind,
                const double *src, double *dst, int ncomp, void *stream);
/* The remaining 2D operators on a general mesh: op 2 SIP Laplacian (tau_scale),
 * 3 viscous Helmholtz (:418-491; gamma0_dt, nu), 4 projection (:372-412;
 * tau_d [e] / tau_c [e][4] per (cell, slot), either NULL), 5 convective term
 * (:533-604; on a context built for the over-integration rule: n_hist levels,
 * beta, Dirichlet data gdata[j] [e][4][2][q] or NULL, body force at the
 * points [2][e][q][q] or NULL; src unused), 6 divergence a(q, u) (:265-316;
 * scale, form 0 standard / 1 weak / 2 strong), 7 pressure gradient b(v, p)
 * (:322-366; form 0 / 1), 8 vorticity moments (:610-618, before the inverse
 * mass), and the boundary-data right-hand sides with data sampled by the
 * caller at the face points (fdata, device): 10 pressure-Dirichlet data
 * (:241-259; g_p [e][4][q], tau_scale), 11 viscous boundary data (:494-527;
 * [e][4][3][q] = g0 g1 on velocity-Dirichlet sides, h0 h1 g_p on
 * velocity-Neumann sides; nu), 12 consistent pressure Neumann data
 * (:621-672; history velocity levels hist[j], vorticity levels vort[j],
 * beta, nu, fdata [e][4][2][q] = dg/dt - f or NULL).  Vector fields: 2
 * components of ncells*n*n values each. */
typedef struct {
  int op;
  double tau_scale;
  const int *kind;                 /* device [e][4] */
  double gamma0_dt, nu;
  const double *tau_d, *tau_c;     /* device */
  double scale;
  int form;
  int n_hist;
  const double *hist[4];           /* device */
  double beta[4];
  const double *gdata[4];          /* device */
  const double *body;              /* device */
  const double *vort[4];           /* device */
  const double *fdata;             /* device */
} dg_g2_params;
int dg_g2_operator(dg_g2 *g, const dg_g2_params *p, const double *src, double *dst,
                   void *stream);
/* multigrid transfer on a refined general mesh (multigrid.py:33-73):
 * prolong (1): out[fine] (+)= (E_dy x E_dx) in[parent[fine]] with
 * quadrant = 2 dy + dx; restrict (0): out[coarse] = sum over
 * children[coarse][4] (-1 = none) of the transposed embedding.  Device
 * int64 parent / children, int32 quadrant. */
int dg_g2_transfer(int k, int prolong, int64_t n_fine, const int64_t *parent,
                   const int *quadrant, int64_t n_coarse, const int64_t *children,
                   const double *in, double *out, int add, void *stream);
/* exact Jacobi diagonal (operators.py:675-730) */
int dg_g2_laplace_diagonal(dg_g2 *g, double tau_scale, const int *kind,
                           double *diag, void *stream);

/* ---- multi-GPU x-slabs (ghost layers) ----------------------------------- */
/* doubles in one ghost layer, ny*nz cells ordered by (iz, iy) -- the size of
 * every send/recv buffer below.  3D Q3-Q5 (the column kernel): owner-computed
 * face traces, per cell [z][y][value | x-derivative] at the facing end
 * (2 n^2 doubles: the face data of kernels.py:119-156); other degrees: whole
 * cells (n^dim doubles). */
int dg_halo_count(const dg_ctx *ctx, int64_t *count);
/* pack the first/last owned x-layer of src into caller-owned device buffers
 * send_lo / send_hi (either may be NULL): traces of the left end (value,
 * dL . line) for send_lo, of the right end (value, dR . line) for send_hi */
int dg_halo_pack(dg_ctx *ctx, const double *src, double *send_lo,
                 double *send_hi, void *stream);
/* attach caller-owned device buffers holding the neighbours' layers; they
 * are read by subsequent vmults on the sides that have a remote neighbour */
int dg_halo_attach(dg_ctx *ctx, const double *recv_lo, const double *recv_hi);
/* identifier of the kernel dg_laplace_vmult launches on this context,
 * "name<template args>" (bench / profile bookkeeping) */
int dg_laplace_kernel_name(dg_ctx *ctx, char *buf, int len);
/* part: 0 = all cells, 1 = cells not touching a ghost layer,
 *       2 = only cells touching a ghost layer (needs recv_* filled) */
int dg_laplace_vmult_part(dg_ctx *ctx, const double *src, double *dst,
                          double tau_scale, int part, void *stream);

/* x-slab vmult around the ghost exchange (traced-ghost contexts, 3D Q3-Q5):
 * phase 1: dst = L src over the whole slab with ZERO ghost traces (needs no
 * exchanged data: runs while the traces move); phase 2: dst += the terms
 * of the ghost traces (the x-face lifts on the first / last x-layer; src
 * unused).  The two phases equal dg_laplace_vmult_part(part 0) up to
 * rounding (the operator is linear in the ghost data). */
int dg_laplace_vmult_split(dg_ctx *ctx, const double *src, double *dst, double tau_scale,
                           int phase, void *stream);

/* ---- sharded (x-slab) PCG building blocks (parallel.SlabPCG) ------------
 * The reference pcg (solvers.py:30-73) on x-slab contexts: every call works
 * on this rank's slab; the caller all-reduces the partial sums between calls
 * (one all-reduce per CG sync point) and the updates read the REDUCED device
 * scalars scal[8]: [0] r.z, [1] p.Lp, [2] sum(Lp), [3] p.w, [4] r.z new.
 * out3 = partial [p.Lp, sum(Lp), p.w] (w = dual weights; deterministic). */
int dg_cg_dots(dg_ctx *ctx, const double *p, const double *Lp, double *out3,
               void *stream);
/* The CG step's operator application with its dot products in one pass
 * (solvers.py:56-60: Ap = op(p), pAp = p.Ap): Lp = L p and out3 as
 * dg_cg_dots.  3D Q4 meshes of >= 16k cells: one launch of the column
 * kernel, the sums formed in its y phase from a shared-memory copy of the
 * layer's p (p and Lp cross HBM once); otherwise dg_laplace_vmult followed
 * by dg_cg_dots.  Contexts without remote sides only (x-slab ranks use
 * dg_laplace_vmult_split + dg_cg_dots): DG_EINVAL otherwise. */
int dg_laplace_vmult_dots(dg_ctx *ctx, const double *p, double *Lp, double tau_scale,
                          double *out3, void *stream);
/* The same on an x-slab rank, in the two phases of dg_laplace_vmult_split
 * (traced-ghost 3D contexts): phase 1 = the whole slab on zero ghost traces
 * with its sums -> out3 (no dependence on the exchange); phase 2 = the
 * ghost-trace lifts, their share of p.Lp and sum(Lp) added to out3.  out3 is
 * this rank's partial triple after phase 2 (all-reduce it). */
int dg_laplace_vmult_split_dots(dg_ctx *ctx, const double *p, double *Lp, double tau_scale,
                                int phase, double *out3, void *stream);
/* alpha = scal[0] / pAp, pAp = p.Lp - (sum(Lp)/|Omega|) p.w (project_dual:
 * op = zero_mean_project_dual o L, solvers.py:187-198) or p.Lp; no update
 * when pAp <= 0 (breakdown, the caller stops).  x += alpha p ;
 * r -= alpha (Lp - c w) ; diag != NULL (Jacobi): z = r / diag and
 * out_rz = partial r.z (device).  Vector updates round like numpy. */
int dg_cg_update(dg_ctx *ctx, double *x, double *r, const double *p,
                 const double *Lp, const double *scal, int project_dual,
                 const double *diag, double *z, double *out_rz, void *stream);
/* p = z + (scal[4] / scal[0]) p ; then scal[0] = scal[4] */
int dg_cg_pupdate(dg_ctx *ctx, double *p, const double *z, double *scal,
                  void *stream);
/* Chebyshev (solvers.py:93-129) vector parts: init from x = 0
 * (d = (r/diag)/theta ; x = d ; rc = r) and one step after the caller's
 * L d_old (rc -= Ld ; d_new = a d_old + b rc/diag ; x += d_new) */
int dg_cheb_vec_init(dg_ctx *ctx, const double *r, const double *diag,
                     double *rc, double *d, double *x, double theta,
                     void *stream);
int dg_cheb_vec_step(dg_ctx *ctx, double *rc, const double *Ld,
                     const double *d_old, double *d_new, const double *diag,
                     double *x, double a, double b, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DGMF_H */
