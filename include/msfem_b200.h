/*
 * msfem_b200.h -- C ABI of the B200 hot path of
 *   J. Alexandersen, B. S. Lazarov, "Robust topology optimisation of microstructural
 *   details without length scale separation - using a spectral coarse basis
 *   preconditioner" (arxiv 1411.3923), cited below as PAPER.md <line>.
 *
 * The library solves, for n_rhs robust realisations (§4.4: "several
 * projections using different threshold values"), the SIMP plane-stress system
 *        K(xbar_eta) u_eta = f            (Eq. 4-5, lines 73 and 84)
 * on a structured nelx x nely Q4 grid with PCG preconditioned by the two-level
 * spectral-MsFEM V-cycle (§2.4, §2.4.2), and computes the robust
 * compliance sensitivities (Eq. 14-15, 17) and an optimality-criteria design update.
 *
 * Conventions (all arrays are dense, little-endian):
 *   node (ix,iy): id = ix*(nely+1) + iy ;  DOF = 2*node + {0:x, 1:y} ;  n_dof = 2*(nelx+1)*(nely+1)
 *   element (ex,ey): id = ex*nely + ey ;  n_el = nelx*nely
 *   design tile (tile_x,tile_y): id = tx*tile_y + ty ; element (ex,ey) <- tile (ex%tile_x, ey%tile_y)
 *   multi-RHS vectors: realisation-major, rhs k occupies [k*n_dof, (k+1)*n_dof)
 *   "device" = a CUDA device pointer on the context's device; "host" = host memory
 *   (pinned host memory recommended for the *_host entry points).
 *
 * Ownership: the caller owns every buffer it passes.  The context keeps pointers into the
 * caller-provided device workspace (msf_workspace_bytes / msf_setup_mesh) and must not
 * outlive it; msf_destroy frees only the small host-side context.  All entry points
 * enqueue work on the context's stream; entry points that return host scalars
 * synchronise that stream before returning.
 *
 * Errors: every entry point returns MSF_OK (0) or a negative MSF_ERR_* code; the message
 * is available from msf_last_error(ctx) (or msf_last_error(NULL) for errors raised before
 * a context exists).  There is no CPU fallback: without a usable sm_100 device every
 * compute entry point returns MSF_ERR_CUDA.
 */
#ifndef MSFEM_B200_H
#define MSFEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSF_OK 0
#define MSF_ERR_ARG (-1)     /* invalid argument / unsupported configuration            */
#define MSF_ERR_CUDA (-2)    /* CUDA runtime error (message carries cudaGetErrorString)  */
#define MSF_ERR_STATE (-3)   /* call order violated (e.g. pcg before assemble_coarse)    */
#define MSF_ERR_NOCONV (-4)  /* PCG reached max_it for at least one rhs (results valid)  */
#define MSF_ERR_FACTOR (-5)  /* non-positive pivot in a dense SPD factorisation          */
#define MSF_ERR_SPACE (-6)   /* workspace smaller than msf_workspace_bytes()             */

#define MSF_MAX_RHS 4
#define MSF_MAX_MODES 16

typedef struct msf_problem {
  int32_t nelx, nely;     /* fine elements along x / y (§2.4: fine mesh T^h)   */
  int32_t cx, cy;         /* fine elements per coarse cell; nelx%cx == nely%cy == 0 (T^H, l.114) */
  int32_t n_modes;        /* eigenpairs kept per agglomerate (cap), 1..MSF_MAX_MODES (l.132)      */
  int32_t tile_x, tile_y; /* periodic design tile (§4.1); nelx%tile_x == 0 ...  */
  int32_t n_rhs;          /* robust realisations, 1..MSF_MAX_RHS (§4.4)          */
  int32_t dilated;        /* realisation whose field builds the basis (§5.3)    */
  int32_t eig_max_iter;   /* max subspace iterations of the local eigensolver (0 -> 60)           */
  double nu;              /* Poisson ratio, plane stress                        */
  double E0, Emin, penal; /* modified SIMP, Eq. 5 (line 84)                               */
  double rmin;            /* density-filter cone radius in elements; < 1 -> identity (line 275)    */
  double beta;            /* Heaviside sharpness, Eq. 16 (line 263); <= 0 -> identity              */
  double eta[MSF_MAX_RHS];/* projection thresholds, one per realisation (line 291)                 */
  double lam_threshold;   /* lambda_Omega (line 132); <= 0 or >= 1e300 -> keep exactly n_modes   */
  double eig_tol;         /* Ritz residual tolerance (D^-1 norm, D-normalised vectors); 0 -> 1e-9 */
} msf_problem;

typedef struct msf_ctx msf_ctx;

/* ---- boundary entry points ----------------------------------------- */

/* Device workspace needed by msf_setup_mesh for this problem.  fixed_mask: host uint8
 * [n_dof], 1 = displacement prescribed zero (§2.1 line 57: Gamma_D).  Runs the
 * host-side plan only (agglomerate classes, §2.4.1); no device work. */
int msf_workspace_bytes(const msf_problem* p, const uint8_t* fixed_mask, size_t* bytes);

/* setup_mesh: builds the structured fine/coarse meshes, DOF maps, Dirichlet masks and the
 * agglomerate decomposition omega_i = union of coarse cells containing y_i (PAPER.md line
 * 118) with its periodicity classes (line 142).  fixed_mask, load: host [n_dof] (load is f
 * of Eq. 4).  workspace: device, >= msf_workspace_bytes(); stream: cudaStream_t or NULL. */
int msf_setup_mesh(const msf_problem* p, const uint8_t* fixed_mask, const double* load,
                   void* workspace, size_t workspace_bytes, void* stream, msf_ctx** out);

int msf_destroy(msf_ctx* ctx);
int msf_set_stream(msf_ctx* ctx, void* stream);
const char* msf_last_error(const msf_ctx* ctx);

/* filter_project: x_tile (device [tile_x*tile_y], design variables) -> density filter
 * (§4.3, periodic 3x3-block form line 275) -> Heaviside projection per
 * eta (Eq. 16) -> tiled physical field -> SIMP moduli (Eq. 5). */
int msf_filter_project(msf_ctx* ctx, const double* x_tile);

/* Direct physical input (no filter / projection): xbar_el device [n_el] for realisation
 * rhs.  Only allowed when the tile is the whole grid (no periodicity classes). */
int msf_set_physical(msf_ctx* ctx, int rhs, const double* xbar_el);

/* build_coarse_basis: per agglomerate class, the n_modes smallest eigenpairs of
 * K_omega psi = lambda diag(K_omega) psi (Eq. 9, §3.2) for the
 * realisation p->dilated (§5.3), filtered by lambda_Omega, multiplied by the bilinear
 * partition of unity chi_i (line 132).  Batched: one CTA per class. */
int msf_build_coarse_basis(msf_ctx* ctx);

/* assemble_coarse: K_c = R_c K(xbar_k) R_c^T per realisation (Eq. 10)
 * and its block-cyclic-reduction factorisation (the exact coarse solve of line 146). */
int msf_assemble_coarse(msf_ctx* ctx);

/* pcg_solve(n_rhs): PCG with the two-level V-cycle, all n_rhs
 * realisations batched, x0 = 0, stop when ||r||_2 <= tol ||f||_2 (reading R9).
 * u: device [n_rhs*n_dof] or NULL (solution kept inside the context); iters, compliance:
 * host [n_rhs] or NULL (compliance = f^T u, Eq. 6).  Returns MSF_ERR_NOCONV if any rhs
 * hit max_it. */
int msf_pcg_solve(msf_ctx* ctx, int n_rhs, double tol, int max_it, double* u,
                  int32_t* iters, double* compliance);

/* sensitivities: robust objective F = E[c] + kappa sqrt(Var[c]) and volume constraint
 * g = E[xbar^T v]/(volfrac e^T v) - 1 (Eq. 17) with gradients w.r.t. the tile
 * design variables (Eq. 14-15, chain rule line 267, tile summation line 236).
 * dF, dg: device [tile_x*tile_y]; F, g, compliance: host scalars / [n_rhs] (any may be NULL). */
int msf_sensitivities(msf_ctx* ctx, double kappa, double volfrac, double* dF, double* dg,
                      double* F, double* g, double* compliance);

/* oc_update: optimality-criteria update (reading R11) of x (device tile) into x_new
 * (device tile, may not alias x) with move limit `move`, bisection on the multiplier with
 * the constraint g evaluated exactly through filter + projections. */
int msf_oc_update(msf_ctx* ctx, const double* x, const double* dF, const double* dg,
                  double volfrac, double move, double* x_new);

/* One full design iteration (filter_project, build_coarse_basis, assemble_coarse,
 * pcg_solve, sensitivities, oc_update) on device buffers.  x, x_new: device tile. */
int msf_design_iteration(msf_ctx* ctx, const double* x, double* x_new, double tol, int max_it,
                         double kappa, double volfrac, double move, int32_t* iters,
                         double* compliance, double* F, double* g);

/* Same, from/to HOST buffers: x_host, x_new_host [tile]; the host->device copy of x and
 * the device->host copies of x_new and the scalars are part of the call. */
int msf_design_iteration_host(msf_ctx* ctx, const double* x_host, double* x_new_host,
                              double tol, int max_it, double kappa, double volfrac,
                              double move, int32_t* iters, double* compliance, double* F,
                              double* g);

/* ---- diagnostics (parity tests; same kernels as the path) ----------------------------- */

/* y = P K(xbar_rhs) P x (reading R2), x, y: device [n_dof]. */
int msf_matvec(msf_ctx* ctx, int rhs, const double* x, double* y);
/* z = M^{-1} r with the two-level V-cycle of realisation rhs; r, z: device [n_dof]. */
int msf_precond_apply(msf_ctx* ctx, int rhs, const double* r, double* z);
/* One symmetric Gauss-Seidel sweep (reading R7) on K z = r, z updated in place. */
int msf_sgs(msf_ctx* ctx, int rhs, const double* r, double* z);
/* msf_sgs with flags: bit 0 starts from z = 0 (z's input is ignored; the pre-smoothing form
 * of the V-cycle), bit 1 runs the sweep as the seven colour-phase launches of the strip
 * partition instead of the streaming kernel (the two are bitwise equal; parity tests).
 * Unknown flag bits: MSF_ERR_ARG. */
int msf_sgs_ex(msf_ctx* ctx, int rhs, const double* r, double* z, int flags);
/* c = K_c^{-1} b for realisation rhs; b, c: device [n_coarse_slots] (slot layout:
 * ((I*(ncy+1)+J)*n_modes + a), unused slots carry identity rows). */
int msf_coarse_solve(msf_ctx* ctx, int rhs, const double* b, double* c);
/* Copies phi_{I,J,a} (padded (2cx+1)x(2cy+1)-node box centred on coarse node (I,J),
 * layout [a][px*(2cy+1)+py][comp]) of every agglomerate into phi_host
 * [n_agg*n_modes*box_nodes*2], the kept mode counts into nkept_host [n_agg] and the
 * eigenvalues into lam_host [n_agg*n_modes] (any may be NULL). */
int msf_get_basis(msf_ctx* ctx, double* phi_host, int32_t* nkept_host, double* lam_host);
/* Copies the coarse block-tridiagonal K_c (diagonal blocks D_I, coupling blocks
 * U_I = K_c[I, I+1], each m x m row-major, m = (ncy+1)*n_modes) of realisation rhs. */
int msf_get_coarse_blocks(msf_ctx* ctx, int rhs, double* D_host, double* U_host);
/* Element moduli E_e (Eq. 5) of realisation rhs into device [n_el]; projected tile
 * into device [tile] (either may be NULL). */
int msf_get_physical(msf_ctx* ctx, int rhs, double* E_el, double* xbar_tile);
/* u of the last pcg_solve for realisations [0, n_rhs) into device [n_rhs * n_dof_local]
 * (n_dof_local = n_dof on one GPU; the strip layout of msf_dist_setup on a strip context). */
int msf_get_solution(msf_ctx* ctx, int n_rhs, double* u);
/* info[0..15]: n_dof, n_el, n_agg, n_classes, ncx, ncy, coarse block size m,
 * coarse slots, box_nodes, eig iterations used (max over classes), last PCG iteration
 * counts (4 entries), kernel launches of the last pcg_solve, workspace bytes. */
int msf_info(msf_ctx* ctx, int64_t* info);
/* Kernel launches enqueued by the library since the last reset (reset if reset != 0). */
int msf_launch_count(msf_ctx* ctx, int64_t* count, int reset);

/* Times the path's kernels in their PCG launch configuration (all n_rhs realisations
 * batched) with CUDA events on the context stream, `reps` launches each, after
 * assemble_coarse.  Clobbers the PCG work vectors.  ms[i]: average ms per launch;
 * bytes[i]: algorithmic HBM bytes per launch, for
 * i = 0 operator apply q = K p (+ p.q), 1 one Gauss-Seidel colour sweep, 2 restriction,
 * 3 coarse solve (all cyclic-reduction levels), 4 prolongation, 5 residual t = r - K z,
 * 6 full V-cycle, 7 one PCG iteration (graph), 8 PCG update fused with the zero-start colour-0
 * phase, 9 p update, 10 K_c assembly: Galerkin products + chain levels (a strip: its own
 * cells and chain), 11 K_c assembly: interface levels + top system, 12 coarse solve:
 * forward chain levels, 13 coarse solve: interface levels + top (+ back), 14 coarse solve:
 * back chain levels (10-14 on one GPU: the same split of the whole chain; a strip's 10-14
 * are its per-rank shares, without the exchanges).  ms and bytes hold 15 entries; the
 * factors are valid again when it returns. */
int msf_bench_kernels(msf_ctx* ctx, int reps, double* ms, double* bytes);

/* ---- strip partition over ranks (multi-GPU) -------------------------
 * The fine grid is cut into strips of whole coarse-cell columns, one per rank.  Rank r
 * owns the node columns of coarse columns [C0, C1) (the last rank also owns column nelx),
 * stores its strip plus a halo on each interior side -- 8 node columns when every strip is
 * at least 8 columns wide (the 7-column dependency halo of the streaming Gauss-Seidel sweep,
 * rounded up), else one column -- and one padding column on the left when needed so that its
 * first local column is even (the 4-colour Gauss-Seidel order of reading R7 is the global
 * one), and runs every fine-grid kernel on it.  The moduli of the whole grid and the spectral
 * basis are replicated.  K_c is distributed over the nested dissection of the coarse grid:
 * rank r computes the Galerkin products of its coarse cells [C0, C1) and factors the fronts
 * of its own box; the separators between the ranks' boxes (interface fronts) are summed by
 * one all-reduce and factored (and later solved) redundantly on every rank.  Per PCG
 * iteration on 8-column halos: 4 halo exchanges (q, the pre-smoothed z, the prolonged
 * iterate, the post-smoothed z) and sum all-reduces of p.Ap, ||r||^2, r.z and of the
 * interface fronts' right-hand sides; on one-column halos the sweeps run as colour phases with
 * a halo exchange after each (15 exchanges).  Results equal the single-GPU path up to the
 * summation order of the dot products and the elimination order of K_c (the interface
 * separators are eliminated last).
 *
 * Transports: MSF_TRANSPORT_NCCL, handle = host pointer to the 128-byte NCCL unique id
 * (msf_nccl_unique_id on rank 0, broadcast by the caller), one process per GPU; all the
 * ordinary entry points then work on the strip context (pcg_solve, sensitivities and
 * design_iteration communicate inside).  MSF_TRANSPORT_GROUP, handle = msf_group*: all
 * ranks of the group are contexts of this process on the current device sharing one
 * stream; the communicating steps are driven by msf_group_assemble_coarse /
 * msf_group_pcg_solve / msf_group_sensitivities (the per-rank msf_assemble_coarse /
 * msf_pcg_solve / msf_sensitivities return MSF_ERR_STATE); the replicated steps use the
 * ordinary per-context calls.
 * Vectors returned from a strip context (u of msf_pcg_solve) are
 * LOCAL: [n_rhs][ncols*(nely+1)][2] over global node columns [gox, gox+ncols).
 * msf_matvec / msf_precond_apply / msf_sgs / msf_coarse_solve / msf_get_coarse_blocks
 * return MSF_ERR_STATE on a strip context of more than one rank;
 * msf_bench_kernels times only the kernels without communication (ms[6] = ms[7] = -1). */
#define MSF_TRANSPORT_NCCL 1
#define MSF_TRANSPORT_GROUP 2
typedef struct msf_group msf_group;

/* bounds[8] = owned node columns [own0, own1), local columns [gox, gox+ncols), owned
 * element columns [e0, e1), owned coarse columns [C0, C1) (all global).  Host only. */
int msf_strip_bounds(const msf_problem* p, int rank, int nranks, int32_t* bounds);
int msf_dist_workspace_bytes(const msf_problem* p, const uint8_t* fixed_mask, int rank,
                             int nranks, size_t* bytes);
/* fixed_mask, load: host, GLOBAL [n_dof] (each rank keeps its strip). */
int msf_dist_setup(const msf_problem* p, const uint8_t* fixed_mask, const double* load,
                   int rank, int nranks, int transport, void* handle, void* workspace,
                   size_t workspace_bytes, void* stream, msf_ctx** out);
/* id: host [128]; loads libnccl at run time (MSF_ERR_CUDA if unavailable). */
int msf_nccl_unique_id(uint8_t* id);
int msf_group_create(int nranks, msf_group** out);
int msf_group_destroy(msf_group* g);
/* Distributed K_c assembly + factorisation of every rank of the group (after each rank's
 * msf_build_coarse_basis). */
int msf_group_assemble_coarse(msf_group* g);
/* Parity diagnostic of the distributed coarse solve: c = K_c^{-1} b for realisation rhs,
 * b and c device, GLOBAL [n_coarse_slots] (layout of msf_coarse_solve). */
int msf_group_coarse_solve(msf_group* g, int rhs, const double* b, double* c);
/* Parity diagnostic of the partitioned preconditioner: z = M^{-1} r (one V-cycle, reading
 * R8) for realisation rhs; r, z device, GLOBAL [n_dof] (z written on every node). */
int msf_group_precond_apply(msf_group* g, int rhs, const double* r, double* z);
/* iters, compliance: host [n_rhs] (identical on every rank) or NULL. */
int msf_group_pcg_solve(msf_group* g, int n_rhs, double tol, int max_it, int32_t* iters,
                        double* compliance);
/* dF, dg: device [tile] (rank 0's copy) or NULL; F, g, compliance as msf_sensitivities. */
int msf_group_sensitivities(msf_group* g, double kappa, double volfrac, double* dF, double* dg,
                            double* F, double* g_out, double* compliance);

#ifdef __cplusplus
}
#endif
#endif /* MSFEM_B200_H */
