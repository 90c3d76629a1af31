// Internal declarations of the B200 MsFEM-PCG library (not part of the C ABI).
// Design notes: DESIGN.md.  Paper citations: PAPER.md line numbers (arxiv 1411.3923).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/msfem_b200.h"

#define MSF_MAX_BLOCK_EIG 24   // subspace-iteration block size cap (n_modes + guard)

// Q4 plane-stress element matrix for unit modulus, passed by value so that the unrolled
// stencil loops read it from the kernel-parameter constant bank (Eq. 5: K0).
struct K0Mat {
  double v[64];
};

// Grid geometry passed by value to every kernel.
struct Dims {
  int nelx, nely;      // fine elements
  int nnx, nny;        // nodes per direction (nelx+1, nely+1)
  int nn, ne;          // node / element counts
  int tile_x, tile_y;  // design tile
  int nt;              // tile size
  int cx, cy;          // fine elements per coarse cell
  int ncx, ncy;        // coarse cells per direction
  int kmax;            // eigen-slots per agglomerate
  int bx, by;          // padded agglomerate box in nodes (2cx+1, 2cy+1)
  int box_nodes;       // bx*by
  int n_agg;           // (ncx+1)*(ncy+1)
  int mc;              // coarse block size (ncy+1)*kmax
  int nbc;             // coarse blocks (ncx+1)
  int R;               // realisations
  // strip partition (multi-GPU); single GPU: gox = 0, own = [0, nnx)
  int gox;             // global node column of local node column 0
  int own_lo, own_hi;  // owned local node columns [own_lo, own_hi)
  long long estride;   // elements between realisations in the moduli array
};

// Per-realisation PCG scalars living in device memory (reading R9).
struct PcgScalars {
  double rz;      // r.z of the current iterate
  double pq;      // p.Ap
  double rr;      // ||r||^2
  double fnorm2;  // ||f||^2
  double alpha, beta;
  double tol2;    // tol^2
  double comp;    // compliance f.u
  int iters;
  int active;     // 1 while iterating
  int max_it;
  int noconv;
};

// Per-class eigen-solve bookkeeping (device).
struct EigClass {
  int rep_agg;      // representative agglomerate index
  int bx0, by0;     // clipped box origin (global node coords)
  int nbx, nby;     // clipped box nodes per direction
  long long off;    // offset (doubles) of this class's work area
  int iters;        // subspace iterations used (written by the kernel)
  int nkept;        // kept modes (written by the kernel)
};

// Nested-dissection coarse solve (msf_nd.cu): one front per box of the recursive dissection
// of the coarse node grid.  S = the box's separator (or all nodes of a leaf box), B = the
// ring of nodes around the box; the front matrix F (n_f x n_f, n_f = (s_n + b_n) kmax,
// row-major, S first) holds after the factorisation -A^{-1}, B A^{-1}, A^{-1} B^T and the
// Schur complement.
struct NdFront {
  int s_n, b_n;       // nodes of S / B
  int node_off;       // nodes[node_off ..]: s_n S nodes then b_n B nodes (global coarse node ids)
  int ch0, ch1;       // children fronts (-1: none on this rank)
  int chmap_off;      // chmap[chmap_off + 2 j + q]: index of front node j in child q's B list (-1)
  int level;          // height among fronts of its kind (box / interface), leaves 0
  int vmap_off;       // vmap[vmap_off + j] (int4) for the n_f front variables
  int flags;          // bit 0: interface front (replicated); bits 1, 2: child 0 / 1 is one
  int vtop_off;       // interface fronts: offset of its variables in vtop (-1: box front)
  long long F_off;    // doubles, per realisation (n_f rows, even leading dimension)
  long long u_off;    // doubles (b_n kmax update vector), per realisation
};

struct NdPlan {
  struct List {       // task list in `lists`: fronts[n] then prefix sums of per-front counts
    int off = 0, n = 0, total = 0, total2 = 0, total3 = 0;
    int RB = 8;       // solve lists: rows per stage
    int NS = 1;       // ... stages per CTA (rows per CTA = RB NS)
  };
  struct Levels {     // a group of levels (this rank's box / the interface tree)
    std::vector<List> asmb, fwd, back;        // per level: assembly tiles, solve row blocks
    std::vector<std::vector<List>> panel;     // per level, per 64-pivot panel
    std::vector<int> fwd_smem, back_smem;     // per level: solve launch shared memory
  };
  std::vector<NdFront> fr;
  std::vector<int> nodes, chmap, lists, vmap, packmap;
  int root = -1, H = 0, TH = 0, n_top = 0;
  bool ok = true;
  long long F_total = 0, u_total = 0, scr_doubles = 0;
  long long top_F = 0;         // doubles of the interface fronts (start of each realisation)
  long long vtop_total = 0;    // interface fronts' right-hand-side entries per realisation
  int max_act = 0, max_nf = 0;
  Levels loc, top;
  List tpart;                  // interface fronts: the rank's partial assembly (mode 1)
  long long solve_bytes = 0;   // matrix bytes streamed per solve and realisation
};

// Device-side dot products awaiting the cross-rank all-reduce (strip partition): kernels
// that end in a reduction write their local sum to dsum[kind][rhs] instead of finalising the
// PCG scalars; k_finalize applies the same update to the all-reduced sums.
enum FinKind { FIN_PQ = 0, FIN_RR = 1, FIN_RZ = 2, FIN_F = 3, FIN_COMP = 4, FIN_KINDS = 5 };

struct msf_group;   // in-process rank group (msf_dist.cu)

// Strip partition of the fine grid over ranks: rank r owns the node
// columns of coarse columns [C0, C1) and keeps a one-column halo on each side (plus one
// padding column on the left when needed to keep the 4-colour parity of the global grid).
// Halo width (node columns per side) of a strip whose sweeps run as ONE streaming kernel: the
// 7 columns the seven colour phases reach into the neighbour, rounded up so that the first
// local column stays even.  Strips narrower than this keep the one-column halo and the
// colour-phase sweep (a halo exchange after every phase).
constexpr int MSF_STRIP_HALO = 8;

struct StripBounds {
  int halo;          // halo node columns per interior side: MSF_STRIP_HALO or 1
  int own0, own1;    // owned global node columns [own0, own1)
  int gox, ncols;    // local node columns = global [gox, gox + ncols)
  int e0, e1;        // owned global element columns
  int C0, C1;        // owned coarse columns
};
int strip_bounds(const Dims& d, int rank, int nranks, StripBounds& b, std::string& msg);
struct msf_ctx;
int dist_comm_create(msf_ctx* c, int transport, void* handle);
void dist_comm_destroy(msf_ctx* c);
int dist_allreduce(const std::vector<msf_ctx*>& cs, double* msf_ctx::*buf, size_t off,
                   size_t count);
int dist_halo(const std::vector<msf_ctx*>& cs, double* msf_ctx::*vec, int rhs0, int nr, int w = 1);
std::vector<msf_ctx*> group_ranks(msf_group* g);

struct msf_comm {
  int kind = 0;          // MSF_TRANSPORT_NCCL / MSF_TRANSPORT_GROUP
  void* nccl = nullptr;  // ncclComm_t
  msf_group* grp = nullptr;
};

struct msf_ctx {
  msf_problem p{};
  Dims d{};            // global grid (coarse space, filter, moduli, basis)
  Dims dl{};           // fine grid of this rank (== d on one GPU)
  int rank = 0, nranks = 1;
  int n_sm = 148;             // multiprocessors of the device (read at setup; grid sizing rules)
  StripBounds sb{};
  msf_comm* comm = nullptr;   // null: single GPU
  double* E_loc = nullptr;    // E + first local element column (stride dl.estride)
  double* dsum = nullptr;     // [FIN_KINDS][MSF_MAX_RHS] local sums (strip partition only)
  K0Mat K0{};
  cudaStream_t stream = nullptr;
  cudaStream_t cap_stream = nullptr;  // private stream used only to capture graphs
  std::string err;
  size_t ws_bytes = 0;
  char* ws = nullptr;

  // host plan
  std::vector<int> cls_of_agg;
  std::vector<EigClass> classes;
  int n_cls = 0;
  int mb = 0;  // eigensolver block size
  long long eig_work_doubles = 0;
  // nested-dissection coarse solve (msf_nd.cu)
  NdPlan nd;
  double* nd_F = nullptr;       // [R][F_total] fronts
  double* nd_u = nullptr;       // [R][u_total] update vectors of the forward sweep
  double* nd_Q = nullptr;       // sweep scratch: pivot blocks, row panels
  double* nd_Ar = nullptr;
  double* nd_Rp = nullptr;
  NdFront* nd_fr = nullptr;
  int* nd_nodes = nullptr;
  int* nd_chmap = nullptr;
  int* nd_lists = nullptr;
  int* nd_vmap = nullptr;       // int4 per front variable
  int* nd_pack = nullptr;       // int2 per interface-front variable (strip partition)
  double* nd_vtop = nullptr;    // [R][vtop_total] interface fronts' right-hand sides
  // strip partition: the agglomerate columns [cr_lo, cr_hi] this rank restricts onto (its
  // coarse cells' corners; the two ends are interface columns shared with the neighbours)
  int cr_lo = 0, cr_hi = 0;       // chain blocks
  int cell_lo = 0, cell_hi = 0;   // Galerkin coarse cell columns [cell_lo, cell_hi)
  std::vector<int> filt_dx, filt_dy;
  std::vector<double> filt_w;
  bool periodic = false;

  // device buffers (carved from the workspace)
  uint8_t* fixn = nullptr;      // per-node bitmask: bit0 x fixed, bit1 y fixed (this rank's strip;
                                // halo / padding columns = 3)
  uint8_t* fixg = nullptr;      // the same for the whole grid (local eigenproblems)
  uint8_t* fixs = nullptr;      // fixn in the streaming sweep's planar padded layout (msf_sgsw.cu)
  int fs_col = 0, fs_plane = 0;
  double* f = nullptr;          // load [2*nn]
  double* x_tile = nullptr;     // design [nt]
  double* xt_tile = nullptr;    // filtered [nt]
  double* xbar_tile = nullptr;  // projected [R*nt]
  double* E = nullptr;          // element moduli [R*ne]
  double* u = nullptr;          // solutions [R*2nn]
  double* r = nullptr;
  double* r2 = nullptr;         // second residual buffer (odd PCG iterations, one GPU)
  double* z = nullptr;
  double* pv = nullptr;
  double* q = nullptr;
  double* t = nullptr;
  double* tile_tmp = nullptr;   // [4*nt] scratch (sensitivities / OC)
  double* dc_el = nullptr;      // [ne] scratch
  double* dF = nullptr;         // [nt]
  double* dg = nullptr;         // [nt]
  double* x_new = nullptr;      // [nt] staging for the host entry point
  int* filt_dx_d = nullptr;
  int* filt_dy_d = nullptr;
  double* filt_w_d = nullptr;
  int n_filt = 0;
  double filt_wsum = 1.0;

  int* cls_of_agg_d = nullptr;
  EigClass* classes_d = nullptr;
  double* phi = nullptr;        // [n_cls][kmax][box_nodes][2]
  double* lam = nullptr;        // [n_cls][kmax]
  double* eig_work = nullptr;

  double* Kcell = nullptr;      // [R][ncells][(4k)^2]
  double* cb = nullptr;         // [R][nbc*mc] coarse rhs
  double* cx = nullptr;         // [R][nbc*mc] coarse solution
  // coarse-cell-class restriction / prolongation (msf_xfer.cu)
  int xf_G = 1, xf_ntasks = 0, xf_n_cls = 0;   // 16-column groups, CTA tasks, cell classes
  int xf_nch = 1;                              // pattern-column chunks per cell group
  void* xf_cls = nullptr;       // XferClass[]
  void* xf_tasks = nullptr;     // XferTask[]
  int* xf_cells = nullptr;      // this rank's cells sorted by class
  double* xf_part = nullptr;    // [R][ncx * ncy][16 G] restriction column sums per cell
  // Galerkin products by cell class (msf_xfer.cu): element matrices of every class
  // [class][cx * cy][packed upper triangle], GEMM tile tasks, packed column -> (p, q)
  double* gal_M = nullptr;
  int4* gal_tasks = nullptr;
  int2* gal_pq = nullptr;
  int gal_ntasks = 0;
  int* factor_status = nullptr; // [2 * MSF_MAX_RHS] nonzero on failed pivot
  bool apply_tma = true;        // operator apply / residual fed by TMA tiles (env MSF_APPLY_TMA=0: off)
  struct TmapSlot {             // cached TMA descriptor (CUtensorMap, 128 B) per base pointer
    const void* ptr;
    int kind;
    alignas(64) unsigned char bytes[128];
  };
  std::vector<TmapSlot> tmaps;
  double* apart = nullptr;      // [R][max_partials] operator p.Ap partials (one GPU)
  int apart_n = 0;              // partial count left by the last matvec (0: none pending)     // threads per agglomerate CTA (0: from the box size)    // m from which SPD block inverses use the blocked path

  PcgScalars* sc = nullptr;     // [R]
  double* partials = nullptr;   // [R][max_blocks]
  unsigned* counters = nullptr; // [R*8]
  int max_partials = 0;
  double* scal = nullptr;       // misc device scalars [64]

  PcgScalars* sc_host = nullptr;  // pinned mirror
  double* scal_host = nullptr;    // pinned [64]

  // state
  bool have_E = false, have_basis = false, have_coarse = false, have_solution = false;
  int last_iters[MSF_MAX_RHS] = {0, 0, 0, 0};
  long long launches = 0;
  long long pcg_launches = 0;
  int eig_iters_used = 0;

  cudaGraphExec_t iter_graph = nullptr;   // strip partition: one iteration for all realisations
  int iter_graph_R = -1;
  // one graph per contiguous active realisation range [rhs0, rhs0 + nr): converged
  // realisations drop out of the launch grids instead of exiting from every CTA
  // [parity]: the PCG residual alternates between r and r2 (the pre-smoothing writes the
  // updated residual out of place), so even and odd iterations are two graphs
  cudaGraphExec_t range_graph[2][MSF_MAX_RHS][MSF_MAX_RHS + 1] = {};
};

// ---------------------------------------------------------------- launch bookkeeping
#define MSF_LAUNCHED(ctx) ((ctx)->launches++)

// Kernel launch with programmatic dependent launch (msfk::pdl_wait / pdl_launch) when
// g_msf_pdl is set (env MSF_PDL=0 disables).  Only for kernels that call pdl_wait before
// reading anything a predecessor writes.
extern bool g_msf_pdl;
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_msf_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------- kernels (fem / pcg)
void launch_matvec(msf_ctx* c, int rhs0, int nr, const double* x, double* y, bool gated,
                   bool dot_pq);
void launch_residual(msf_ctx* c, int rhs0, int nr, const double* b, const double* x, double* y,
                     bool gated);
void launch_sgs(msf_ctx* c, int rhs0, int nr, const double* r, double* z, bool gated);
void launch_sgs_sweep(msf_ctx* c, int rhs0, int nr, const double* r, double* z, bool gated,
                      bool zero_start, int rz_mode, bool skip_f0);
// one colour phase of the sweep: 0 F0 from z = 0, 1 F0, 2 F1, 3 F2, 4 F3B3, 5 B2, 6 B1,
// 7 B0 (r.z -> beta when rz_mode != 0)
void launch_sgs_phase(msf_ctx* c, int rhs0, int nr, const double* r, double* z, bool gated,
                      int phase, int rz_mode);
// PCG scalar update from the all-reduced dsum[kind] (strip partition)
void launch_finalize(msf_ctx* c, int kind, int rhs0, int nr, bool gated, int rz_mode);
// fused u/r update + ||r||^2 + zero-start forward GS colour 0 (PCG iteration)
void launch_update_f0(msf_ctx* c, int rhs0, int nr);
void launch_mask_copy(msf_ctx* c, const double* x, double* y, int n2nn);
void launch_pcg_init(msf_ctx* c, int nr, double tol, int max_it);
// mode 0: p = z (init); 1: u += alpha p, p = z + beta p; 2: p = z + beta p; 3: u += alpha p
// (all realisations, after the last iteration)
void launch_pcg_p(msf_ctx* c, int rhs0, int nr, int mode);
// streaming symmetric Gauss-Seidel sweep (msf_sgsw.cu: the iterate in registers, one warp per band): z = SGS(z; r), zero_start: from z = 0;
// upd: r -= alpha q first (alpha from the operator's partials, ||r||^2 -> convergence);
// rz_mode != 0: r.z -> beta
// zin: the starting iterate (not read when zero_start; must differ from z: other CTAs read
// their halo of it while this one writes)
// upd: the updated residual goes to rout (r is read only)
void launch_sgs_stream(msf_ctx* c, int rhs0, int nr, const double* r, double* rout,
                       const double* zin, double* z, bool gated, bool zero_start, bool upd,
                       int rz_mode);
int sgs_warp_partials_needed(const Dims& d);
void sgs_fix_layout(const Dims& d, int& fs_col, int& fs_plane);
void sgs_fix_build(const Dims& d, const uint8_t* fixn, std::vector<uint8_t>& out);
void launch_compliance(msf_ctx* c, int nr);

// ---------------------------------------------------------------- filter / design
void launch_filter_project(msf_ctx* c, const double* x_tile);
void launch_set_physical(msf_ctx* c, int rhs, const double* xbar_el);
// compliance + element sensitivities of the owned elements summed per tile variable (dcT)
void launch_sens_local(msf_ctx* c);
// robust weights, chain rule, filter adjoint, volume (replicated; after the dcT all-reduce)
void launch_sens_global(msf_ctx* c, double kappa, double volfrac);
void launch_sensitivities(msf_ctx* c, double kappa, double volfrac);
void launch_oc(msf_ctx* c, const double* x, const double* dF, const double* dg, double volfrac,
               double move, double* x_new);

// ---------------------------------------------------------------- coarse space
void launch_build_basis(msf_ctx* c);
// K_c assembly (Galerkin cell products) + nested-dissection factorisation, one GPU
void launch_assemble_coarse(msf_ctx* c);
// restriction / prolongation by coarse-cell class (msf_xfer.cu)
int xfer_setup(msf_ctx* c, char*& cur);
size_t xfer_workspace_bytes(const Dims& d, const std::vector<int>& cls_of_agg, int C0, int C1);
void launch_restrict(msf_ctx* c, int rhs0, int nr, const double* t, bool gated);
// z = zin + R^T c (zin == z: in place)
void launch_prolong(msf_ctx* c, int rhs0, int nr, const double* zin, double* z, bool gated);
constexpr int MSF_BENCH_ENTRIES = 15;   // msf_bench_kernels

// nested dissection (msf_nd.cu)
bool nd_build_plan(const Dims& d, NdPlan& P, int rank, int nranks, const std::vector<int>& icol);
size_t nd_workspace_bytes(const Dims& d, const NdPlan& P);
cudaError_t nd_setup(msf_ctx* c, char*& cur);
void launch_nd_factor(msf_ctx* c);
void launch_nd_factor_local(msf_ctx* c);
void launch_nd_factor_top(msf_ctx* c);
void launch_nd_solve(msf_ctx* c, int rhs0, int nr, bool gated);
void launch_nd_solve_local_fwd(msf_ctx* c, int rhs0, int nr, bool gated);
void launch_nd_solve_top(msf_ctx* c, int rhs0, int nr, bool gated);
void launch_nd_solve_local_back(msf_ctx* c, int rhs0, int nr, bool gated);
// Galerkin cell products K_cell of this rank's cells; a block-tridiagonal copy D / U of K_c
// gathered from them (diagnostic read-out)
void launch_galerkin_cells(msf_ctx* c);
void launch_coarse_gather(msf_ctx* c, double* D, double* U, int nslot);

// ---------------------------------------------------------------- helpers
int msf_fail(msf_ctx* c, int code, const std::string& msg);
int msf_cuda_check(msf_ctx* c, cudaError_t e, const char* where);
K0Mat make_K0(double nu);
