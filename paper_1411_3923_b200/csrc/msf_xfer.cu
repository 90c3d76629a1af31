// Restriction c = R_c t and prolongation z += R_c^T c of the two-level preconditioner
// (§2.4.2 l.146; R_c^T = [phi_1 ... phi_N], phi_{i,a} = chi_i psi_a^{omega_i}, Eq. 9-10
// l.128-136), organised by COARSE-CELL CLASS.
//
// Inside coarse cell (CI, CJ) every fine node is covered by the cell's four corner agglomerates,
// so the transfer is a dense (P = nodes x 2) x (4 k) block per cell, Phi_cell.  The periodic
// microstructure (§2.4.1 l.142: identical local problems share their basis) makes the
// block the same for every cell whose four corners belong to the same agglomerate classes: a
// handful of cell classes cover the grid, and the transfer of the cells of one class is a
// real dense contraction (the realisations share the basis, so the three
// robust right-hand sides batch too):
//   * restriction  C[4k x cells] = Phi_cell^T [4k x P] . T [P x cells],
//   * prolongation Z[P x cells] += Phi_cell [P x 4k] . X^T [4k x cells],
// run on the fp64 tensor cores (mma.m8n8k4) one pattern column at a time: a CTA takes 64
// cells of a class, moves the column's values of its cells through shared memory in coalesced
// 16-byte pieces, and stages the column's Phi block (16 basis columns per pass) next to it.
// Every output element is one warp's fixed-order accumulation (deterministic).
//
// Nodes are owned half-open by cells (cell (CI, CJ): local columns [0, cx), rows [0, cy), the
// last cell column / row also owns the closing node line), so every node belongs to exactly one
// cell.  A strip processes its own cells [C0, C1): exactly its owned nodes.
// Restriction then adds, per agglomerate, the column sums of its (up to) four cells in a fixed
// order.
#include "msf_kern.cuh"

#include <algorithm>
#include <map>
#include <vector>

using namespace msfk;

namespace {

#ifndef MSF_XFER_XT
#define MSF_XFER_XT 256
#endif
#ifndef MSF_XFER_NCC
#define MSF_XFER_NCC 64
#endif
constexpr int XT = MSF_XFER_XT;    // threads per CTA: XT / 32 warps x CW cells
constexpr int NCC = MSF_XFER_NCC;  // cells per task
constexpr int CW = NCC / (XT / 32), NI = CW / 8;   // cells / 8-cell DMMA tiles per warp
static_assert(NI >= 1 && CW % 8 == 0, "each warp takes whole 8-cell DMMA tiles");
constexpr int XNJ = 16;    // Phi columns per pass (one column group)
constexpr int SPJ = 20;    // shared row stride of Phi chunks / coarse coefficients (conflict-free)
constexpr int GT = 64;     // Galerkin GEMM tile (rows x packed columns)
constexpr int GK = 32;     // Galerkin GEMM k-chunk (elements)
constexpr int GPAD = GT + 4;   // shared row stride of the GEMM panels (conflict-free fragments)

struct XferClass {   // device: one coarse-cell class
  int cls[4];        // agglomerate class of corner (di, dj) = (q >> 1, q & 1)
  int nx, ny;        // owned node columns / rows of the pattern
  int cell_off;      // first cell in the class-sorted cell list
  int pad;
};
struct XferTask {    // device: (class, cells [c0, c0 + nc) of the class list, nc <= NCC, column
  int k, c0, nc, ch;  // chunk ch of the pattern: columns [ch nx / nch, (ch + 1) nx / nch))
};
// Pattern-column chunks per cell group: a CTA walks its columns in sequence (two barriers per
// column, ~2 us each), so a whole 20-column pattern is a ~45 us pipeline however few cells there
// are; when the cell groups alone do not fill the device (3 CTAs resident per SM: small grids,
// the strips of a partition) the pattern is cut into chunks for more, shorter CTAs.  Chunks of
// at least 4 columns.  (With the device already full, chunks only repeat the per-CTA prologue:
// configs[4] on one GPU, 4 chunks: restriction 0.094 -> 0.084 ms but prolongation 0.143 -> 0.163.)
inline int xfer_nchunk(const Dims& d, size_t ngroups) {
  const int want = (int)((444 + ngroups - 1) / std::max<size_t>(ngroups, 1));
  return std::max(1, std::min(want, d.cx / 4));
}

// entries of one pattern column (2 ny, (node row, DOF)) padded to whole 8-row DMMA tiles, and
// the shared row stride of a column tile (stride = 4 or 12 mod 16 doubles: the fragment loads
// of 4 rows x 4 entries hit 16 distinct bank pairs)
__host__ __device__ __forceinline__ int col_pad(int ny) { return (2 * ny + 7) & ~7; }
__host__ __device__ __forceinline__ int tile_stride(int ny) {
  int s = col_pad(ny);
  while ((s & 15) != 4 && (s & 15) != 12) ++s;
  return s;
}

__device__ __forceinline__ uint32_t xs_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void xcp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(xs_u32(dst)), "l"(src) : "memory");
}
// D = A B + C on the fp64 tensor cores, m8n8k4 (lane = 4 g + t: A(g, t), B(t, g), C(g, 2t + {0,1}))
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Phi chunk of pattern column lx, column group g: SP[e][jj] = Phi_cell[(lx, e)][g*16 + jj],
// e < 2 ny (zero rows up to col_pad, zero columns beyond 4 k), by 8-byte cp.async (zero fill):
// the issuing thread does not wait for the L2 round trip
__device__ __forceinline__ void stage_phi_col(const Dims& d, const XferClass& C,
                                              const double* __restrict__ phi, int g, int lx,
                                              double* SP) {
  const int ne = 2 * C.ny, ep = col_pad(C.ny);
  const int jj = threadIdx.x & (XNJ - 1), j = g * XNJ + jj;   // fixed per thread (XT % 16 == 0)
  const bool vj = j < 4 * d.kmax;
  const int corner = vj ? j / d.kmax : 0, a = vj ? j - corner * d.kmax : 0;
  const int di = corner >> 1, dj = corner & 1;
  const double* colp = phi + ((size_t)C.cls[corner] * d.kmax + a) * d.box_nodes * 2 +
                       (size_t)(lx + d.cx * (1 - di)) * d.by * 2 + (size_t)d.cy * (1 - dj) * 2;
  for (int e = threadIdx.x >> 4; e < ep; e += XT / XNJ) {
    const bool v = vj && e < ne;
    // entry e = (ly, q): box node row cy (1 - dj) + ly, DOF q -> colp + 2 ly + q = colp + e
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(xs_u32(SP + e * SPJ + jj)),
                 "l"(v ? colp + e : phi), "r"(v ? 8 : 0)
                 : "memory");
  }
}

// column lx of the task's cells (ny nodes = 2 ny doubles each, 16-byte pieces) into tile rows:
// warp w moves the columns of cells w, w + 8, ..., lane ly the node row ly.  cbase[c]: the
// cell's first node (node (lx, ly) at cbase + lx nny + ly)
__device__ __forceinline__ void load_col_tile(const Dims& d, const XferClass& C,
                                              const long long* cbase, int nc,
                                              const double* __restrict__ v, int lx, double* Tt,
                                              int st) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane >= C.ny) return;
  for (int c = w; c < nc; c += XT / 32)
    xcp16(Tt + (size_t)c * st + 2 * lane, v + 2 * (cbase[c] + (long long)lx * d.nny + lane));
}

// part[rhs][cell][j] = sum over the cell's pattern entries e of Phi_cell[e][j] t(e):
// per pattern column, C[16 x 64 cells] += Phi_col^T [16 x 2ny] . T_col [2ny x 64 cells] on the
// fp64 tensor cores (mma.m8n8k4; warp w: columns 0..15 x cells CW w .. CW w + CW - 1).  One CTA
// per (task, realisation); the next column's tile and Phi block load while this one computes.
__global__ void __launch_bounds__(XT) k_restrict_cells(Dims d, const XferClass* __restrict__ cls,
                                                       const XferTask* __restrict__ tasks,
                                                       const int* __restrict__ cells,
                                                       const double* __restrict__ phi,
                                                       const double2* __restrict__ tall,
                                                       double* part, const PcgScalars* sc,
                                                       int rhs0, int gated, int G, int nch) {
  extern __shared__ __align__(16) double xsm[];
  __shared__ int cid[NCC];
  __shared__ long long cbase[NCC];
  pdl_launch();
  const XferTask T = tasks[blockIdx.x];
  const XferClass C = cls[T.k];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int st = tile_stride(C.ny), ep = col_pad(C.ny), ne = 2 * C.ny;
  // two buffers each: column tiles [NCC][st] at xsm, Phi blocks [ep][SPJ] after them
  double* const SP0 = xsm + (size_t)2 * NCC * st;
  auto Tt = [&](int b) { return xsm + (size_t)b * NCC * st; };
  auto SP = [&](int b) { return SP0 + (size_t)b * ep * SPJ; };
  for (int c = tid; c < NCC; c += XT) {
    const int cell = cells[C.cell_off + T.c0 + min(c, T.nc - 1)], CI = cell / d.ncy;
    cid[c] = cell;
    cbase[c] = (long long)(CI * d.cx - d.gox) * d.nny + (cell - CI * d.ncy) * d.cy;
  }
  // tile entries beyond 2 ny (never loaded) stay zero; rows of missing cells are ignored
  for (int k = tid; k < 2 * NCC * (st - ne); k += XT) {
    const int row = k / (st - ne);
    xsm[(size_t)row * st + ne + k % (st - ne)] = 0.0;
  }
  pdl_wait();
  const int rhs = rhs0 + blockIdx.y;
  if (gated && !sc[rhs].active) return;   // uniform
  __syncthreads();
  const double* t = reinterpret_cast<const double*>(tall + (size_t)rhs * d.nn);
  const int lx0 = T.ch * C.nx / nch, ncol = (T.ch + 1) * C.nx / nch - lx0;   // this task's columns
  // sub-step i = (column lc = i / G, column group g = i % G): the column tile is loaded once
  // (buffer lc & 1) and contracted with each group's Phi block (buffer i & 1) into that group's
  // accumulators, so t is read once however many basis columns there are
  const int GJ = G * XNJ, nsteps = G * ncol;
  auto stage = [&](int i) {
    const int lc = i / G, g = i - lc * G;
    stage_phi_col(d, C, phi, g, lx0 + lc, SP(i & 1));
    if (g == 0) load_col_tile(d, C, cbase, T.nc, t, lx0 + lc, Tt(lc & 1), st);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage(0);
  double acc[4][2][NI][2];   // [group]
#pragma unroll
  for (int k = 0; k < 16 * NI; ++k) (&acc[0][0][0][0])[k] = 0.0;
  for (int lc = 0; lc < ncol; ++lc) {
    const double* B = Tt(lc & 1);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (g < G) {
        const int i = lc * G + g;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();   // sub-step i's data visible; sub-step i - 1's compute done everywhere
        if (i + 1 < nsteps) stage(i + 1);
        const double* S = SP(i & 1);
        for (int k0 = 0; k0 < ep; k0 += 4) {
          double a[2], b[NI];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) a[mi] = S[(k0 + tq) * SPJ + mi * 8 + gq];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) b[ni] = B[(size_t)(CW * w + ni * 8 + gq) * st + k0 + tq];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma884(acc[g][mi][ni][0], acc[g][mi][ni][1], a[mi], b[ni]);
        }
      }
    }
  }
  // C(gq, 2 tq + h) of (g, mi, ni): column g*16 + mi*8 + gq, cell CW w + ni*8 + 2 tq + h
#pragma unroll
  for (int g = 0; g < 4; ++g)
    if (g < G) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = CW * w + ni * 8 + 2 * tq + h;
            if (c < T.nc)
              part[(((size_t)rhs * d.ncx * d.ncy + cid[c]) * nch + T.ch) * GJ + g * XNJ + mi * 8 + gq] = acc[g][mi][ni][h];
          }
    }
}

// t = zin + R_c^T x on the task's cells for realisation rhs0 + blockIdx.y (if active): per
// pattern column, Z_col[2ny x 64 cells] += Phi_col [2ny x 16] . X^T [16 x 64 cells] on the fp64
// tensor cores (warp w: all entries x cells CW w .. CW w + CW - 1), the column tile moved in and
// out with coalesced 16-byte pieces; the next column loads while this one computes.  More than
// 16 basis columns (G > 1): the groups add to the column tile one after the other.
__global__ void __launch_bounds__(XT) k_prolong_cells(Dims d, const XferClass* __restrict__ cls,
                                                      const XferTask* __restrict__ tasks,
                                                      const int* __restrict__ cells,
                                                      const double* __restrict__ phi,
                                                      const double* __restrict__ xall,
                                                      const double2* zin, double2* tout,
                                                      const PcgScalars* sc, int rhs0, int gated,
                                                      int G, int nch) {
  extern __shared__ __align__(16) double xsm[];
  __shared__ int cid[NCC];
  __shared__ long long cbase[NCC];
  pdl_launch();
  const XferTask T = tasks[blockIdx.x];
  const XferClass C = cls[T.k];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int st = tile_stride(C.ny), ep = col_pad(C.ny), ne = 2 * C.ny;
  // two buffers each: column tiles [NCC][st] at xsm, Phi blocks [ep][SPJ] after them
  double* const SP0 = xsm + (size_t)2 * NCC * st;
  auto Zt = [&](int b) { return xsm + (size_t)b * NCC * st; };
  auto SP = [&](int b) { return SP0 + (size_t)b * ep * SPJ; };
  double* X = SP0 + (size_t)2 * ep * SPJ;   // [G][NCC][SPJ]
  for (int c = tid; c < NCC; c += XT) {
    const int cell = cells[C.cell_off + T.c0 + min(c, T.nc - 1)], CI = cell / d.ncy;
    cid[c] = cell;
    cbase[c] = (long long)(CI * d.cx - d.gox) * d.nny + (cell - CI * d.ncy) * d.cy;
  }
  pdl_wait();
  const int rhs = rhs0 + blockIdx.y;
  if (gated && !sc[rhs].active) return;   // uniform
  __syncthreads();
  const size_t cstride = (size_t)d.nbc * d.mc;
  {
    // coefficient j = g*16 + jj of cell c: slot (agglomerate of its corner) * kmax + a; the
    // corner offset in slots is fixed per j, the cell's (CI, CJ) slot base per cell
    const int jj = tid & (XNJ - 1);
    for (int g = 0; g < G; ++g) {
      const int j = g * XNJ + jj;
      const bool vj = j < 4 * d.kmax;
      const int corner = vj ? j / d.kmax : 0, a = vj ? j - corner * d.kmax : 0;
      const int off = ((corner >> 1) * (d.ncy + 1) + (corner & 1)) * d.kmax + a;
      for (int c = tid >> 4; c < NCC; c += XT / XNJ) {
        const int cell = cid[c], CI = cell / d.ncy, CJ = cell - CI * d.ncy;
        X[((size_t)g * NCC + c) * SPJ + jj] =
            vj ? xall[(size_t)rhs * cstride + (CI * (d.ncy + 1) + CJ) * d.kmax + off] : 0.0;
      }
    }
  }
  const double* zi0 = reinterpret_cast<const double*>(zin + (size_t)rhs * d.nn);
  double* to = reinterpret_cast<double*>(tout + (size_t)rhs * d.nn);
  const int lx0 = T.ch * C.nx / nch, ncol = (T.ch + 1) * C.nx / nch - lx0;   // this task's columns
  // sub-step i = (column lc = i / G, column group g = i % G): the column tile is loaded once
  // (buffer lc & 1), every group's Phi block (buffer i & 1) adds its part, and the column is
  // stored once after the last group
  const int nsteps = G * ncol;
  auto stage = [&](int i) {
    const int lc = i / G, g = i - lc * G;
    stage_phi_col(d, C, phi, g, lx0 + lc, SP(i & 1));
    if (g == 0) load_col_tile(d, C, cbase, T.nc, zi0, lx0 + lc, Zt(lc & 1), st);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage(0);
  for (int i = 0; i < nsteps; ++i) {
    const int lc = i / G, g = i - lc * G, lx = lx0 + lc;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();   // sub-step i's data (and X) visible; sub-step i - 1's buffers free
    if (i + 1 < nsteps) stage(i + 1);
    const double* S = SP(i & 1);
    double* Z = Zt(lc & 1);
    const double* Xg = X + (size_t)g * NCC * SPJ;
    double acc[7][NI][2];   // up to 7 entry tiles (2 ny <= 56)
#pragma unroll
    for (int k = 0; k < 14 * NI; ++k) (&acc[0][0][0])[k] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < XNJ; k0 += 4) {
      double b[NI];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) b[ni] = Xg[(CW * w + ni * 8 + gq) * SPJ + k0 + tq];
#pragma unroll
      for (int mi = 0; mi < 7; ++mi) {
        if (mi * 8 < ep) {
          const double a = S[(mi * 8 + gq) * SPJ + k0 + tq];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a, b[ni]);
        }
      }
    }
    // C(gq, 2 tq + h) of (mi, ni): entry mi*8 + gq of cell CW w + ni*8 + 2 tq + h (the warp's own
    // cells: no other warp touches these tile rows between the groups)
#pragma unroll
    for (int mi = 0; mi < 7; ++mi) {
      const int e = mi * 8 + gq;
      if (mi * 8 < ep && e < ne) {
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) Z[(size_t)(CW * w + ni * 8 + 2 * tq + h) * st + e] += acc[mi][ni][h];
      }
    }
    if (g == G - 1) {
      __syncthreads();
      if (lane < C.ny)   // column back out, 16-byte pieces (warp w: cells w, w + 8, ...)
        for (int c = w; c < T.nc; c += XT / 32)
          *reinterpret_cast<double2*>(to + 2 * (cbase[c] + (long long)lx * d.nny + lane)) =
              *reinterpret_cast<const double2*>(Z + (size_t)c * st + 2 * lane);
    }
  }
}

// c[slot(I, J, a)] = sum over the (up to) four cells of agglomerate (I, J) in this rank's cell
// columns [C0, C1) of the column (corner of (I, J), a) of their partials, in a fixed order
__global__ void __launch_bounds__(256) k_restrict_aggs(Dims d, const double* __restrict__ part,
                                                       int GJ, int nch, int I0, int I1, int C0, int C1,
                                                       double* cball, const PcgScalars* sc,
                                                       int rhs0, int gated) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.y;
  if (gated && !sc[rhs].active) return;
  const int k = blockIdx.x * 256 + threadIdx.x;
  const int naggs = (I1 - I0 + 1) * (d.ncy + 1);
  if (k >= naggs * d.kmax) return;
  const int a = k % d.kmax, ag = k / d.kmax;
  const int I = I0 + ag / (d.ncy + 1), J = ag % (d.ncy + 1);
  double s = 0.0;
#pragma unroll
  for (int di = 0; di < 2; ++di) {
    const int CI = I - 1 + di;
    if (CI < C0 || CI >= C1) continue;
#pragma unroll
    for (int dj = 0; dj < 2; ++dj) {
      const int CJ = J - 1 + dj;
      if (CJ < 0 || CJ >= d.ncy) continue;
      const int corner = (1 - di) * 2 + (1 - dj);   // (I, J) = (CI + 1 - di, CJ + 1 - dj)
      const double* pc = part + ((size_t)rhs * d.ncx * d.ncy + CI * d.ncy + CJ) * nch * GJ + corner * d.kmax + a;
      for (int ch = 0; ch < nch; ++ch) s += pc[(size_t)ch * GJ];   // the cell's column chunks, in order
    }
  }
  cball[(size_t)rhs * d.nbc * d.mc + ((size_t)I * (d.ncy + 1) + J) * d.kmax + a] = s;
}

// ------------------------------------------------------------------ Galerkin cell products
// Kcell[rhs][cell][p][q] = sum_{e in cell} E_e Phi_e^T K0 Phi_e (Eq. 10, per coarse
// cell; p, q = corner * k + mode).  For the cells of one class Phi_e is the same, so
//     Kcell[rhs][cell] = sum_e E[rhs][cell, e] M_k[e],   M_k[e] = Phi_e^T K0 Phi_e,
// i.e. one GEMM per class, C[(cell, rhs) x pq] = A[(cell, rhs) x e] . B[e x pq], with B the
// class's element matrices (upper triangle p <= q, packed) -- on the fp64 tensor cores.

// M_k[e][s] for class k, element e = lex * cy + ley of the cell, packed column s = (p, q):
// V = K0 Phi_e, then M = Phi_e^T V (the arithmetic of the per-element products of round 1)
__global__ void __launch_bounds__(256) k_galerkin_M(Dims d, K0Mat K, const XferClass* __restrict__ cls,
                                                    const double* __restrict__ phi,
                                                    const int2* __restrict__ pq, int psp, double* M) {
  extern __shared__ double gsm[];
  const int k = blockIdx.y, e = blockIdx.x, P = 4 * d.kmax;
  const XferClass C = cls[k];
  const int lex = e / d.cy, ley = e - (e / d.cy) * d.cy;
  double* Ph = gsm;            // [8][P]
  double* V = gsm + 8 * P;     // [8][P]
  for (int t = threadIdx.x; t < 8 * P; t += blockDim.x) {
    const int i = t / P, p = t - (t / P) * P;
    const int b = i >> 1, comp = i & 1;
    const int lx = lex + ((b == 1 || b == 2) ? 1 : 0), ly = ley + ((b >= 2) ? 1 : 0);
    const int corner = p / d.kmax, a = p - corner * d.kmax;
    const int di = corner >> 1, dj = corner & 1;
    const int px = lx + d.cx * (1 - di), py = ly + d.cy * (1 - dj);
    Ph[t] = phi[(((size_t)C.cls[corner] * d.kmax + a) * d.box_nodes + px * d.by + py) * 2 + comp];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 8 * P; t += blockDim.x) {
    const int i = t / P, q = t - (t / P) * P;
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) v = fma(K.v[i * 8 + j], Ph[j * P + q], v);
    V[t] = v;
  }
  __syncthreads();
  double* Mk = M + ((size_t)k * d.cx * d.cy + e) * psp;
  for (int s = threadIdx.x; s < psp; s += blockDim.x) {
    const int2 c = pq[s];
    double t = 0.0;
    if (c.x >= 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) t = fma(Ph[i * P + c.x], V[i * P + c.y], t);
    }
    Mk[s] = t;
  }
}

// One 64 x 64 tile of C = A B for class k: rows r0 .. r0 + 63 = (class cell, realisation)
// pairs, packed columns q0 .. q0 + 63; k-chunks of 32 elements staged k-major in shared
// memory; DMMA m8n8k4, 8 warps as 2 x 4, each a 32 x 16 sub-tile.  C(p, q) goes to Kcell[p][q]
// and Kcell[q][p].
__global__ void __launch_bounds__(256) k_galerkin_gemm(Dims d, const XferClass* __restrict__ cls,
                                                       const int4* __restrict__ tasks,
                                                       const int* __restrict__ cells,
                                                       const double* __restrict__ Eall,
                                                       const double* __restrict__ M,
                                                       const int2* __restrict__ pq, int psp,
                                                       double* Kcell) {
  __shared__ __align__(16) double sA[GK][GPAD];   // A^T chunk: [element][row]
  __shared__ __align__(16) double sB[GK][GPAD];   // B chunk:   [element][column]
  __shared__ long long rbase[GT];                 // row -> E offset of its cell (realisation incl.)
  __shared__ int eoff[GK];
  const int4 T = tasks[blockIdx.x];
  const XferClass C = cls[T.x];
  const int R = d.R, nel = d.cx * d.cy, P = 4 * d.kmax;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t4 = lane & 3;
  const int m0 = (w >> 2) * 32, n0 = (w & 3) * 16;
  // rows of this tile: (class cell c, realisation r), row = c * R + r < T.w (= cells x R)
  for (int m = tid; m < GT; m += 256) {
    const int row = T.y + m, c = row / R, r = row - c * R;
    long long b = -1;
    if (row < T.w) {
      const int cell = cells[C.cell_off + c];
      const int CI = cell / d.ncy, CJ = cell - CI * d.ncy;
      b = (long long)r * d.ne + (long long)(CI * d.cx) * d.nely + CJ * d.cy;
    }
    rbase[m] = b;
  }
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) (&acc[0][0][0])[i] = 0.0;
  const double* Mk = M + (size_t)T.x * nel * psp + T.z;
  for (int e0 = 0; e0 < nel; e0 += GK) {
    __syncthreads();   // rbase ready / previous chunk consumed
    for (int kk = tid; kk < GK; kk += 256) {
      const int e = e0 + kk;
      eoff[kk] = e < nel ? (e / d.cy) * d.nely + (e - (e / d.cy) * d.cy) : -1;
    }
    __syncthreads();
    for (int t = tid; t < GK * GT; t += 256) {
      const int kk = t / GT, x = t - kk * GT;
      const long long rb = rbase[x];
      const int eo = eoff[kk];
      sA[kk][x] = (rb >= 0 && eo >= 0) ? __ldg(Eall + rb + eo) : 0.0;
      sB[kk][x] = eo >= 0 ? __ldg(Mk + (size_t)(e0 + kk) * psp + x) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k0 = 0; k0 < GK; k0 += 4) {
      double a[4], bq[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = sA[k0 + t4][m0 + mi * 8 + g];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bq[ni] = sB[k0 + t4][n0 + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], bq[ni]);
    }
  }
  // C(g, 2 t4 + h) of fragment (mi, ni): row m0 + mi*8 + g, packed column n0 + ni*8 + 2 t4 + h
  const size_t cs = (size_t)P * P;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int m = m0 + mi * 8 + g;
    if (rbase[m] < 0) continue;
    const int row = T.y + m, c = row / R, r = row - c * R;
    const int cell = cells[C.cell_off + c];
    double* Kc = Kcell + ((size_t)r * d.ncx * d.ncy + cell) * cs;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s = T.z + n0 + ni * 8 + 2 * t4 + h;
        if (s >= psp) continue;
        const int2 ij = pq[s];
        if (ij.x < 0) continue;
        Kc[(size_t)ij.x * P + ij.y] = acc[mi][ni][h];
        Kc[(size_t)ij.y * P + ij.x] = acc[mi][ni][h];
      }
  }
}

size_t restrict_smem(const Dims& d) {
  const int ny = d.cy + 1;
  return (2 * (size_t)NCC * tile_stride(ny) + 2 * (size_t)col_pad(ny) * SPJ) * sizeof(double);
}
size_t prolong_smem(const Dims& d) {
  const int ny = d.cy + 1, G = (4 * d.kmax + XNJ - 1) / XNJ;
  return (2 * (size_t)NCC * tile_stride(ny) + 2 * (size_t)col_pad(ny) * SPJ + (size_t)G * NCC * SPJ) * sizeof(double);
}

}  // namespace

namespace {
// Cell classes of the cells [C0, C1) x [0, ncy): key = the four corner agglomerate classes and
// whether the cell owns the closing node column / row; members in grid order.
void cell_classes(const Dims& d, const std::vector<int>& cls_of_agg, int C0, int C1,
                  std::vector<XferClass>& K, std::vector<std::vector<int>>& members) {
  std::map<std::vector<int>, int> key2k;
  K.clear();
  members.clear();
  for (int CI = C0; CI < C1; ++CI)
    for (int CJ = 0; CJ < d.ncy; ++CJ) {
      const int lastx = CI == d.ncx - 1, lasty = CJ == d.ncy - 1;
      std::vector<int> key(6);
      for (int q = 0; q < 4; ++q) key[q] = cls_of_agg[(CI + (q >> 1)) * (d.ncy + 1) + CJ + (q & 1)];
      key[4] = lastx;
      key[5] = lasty;
      auto it = key2k.find(key);
      int k;
      if (it == key2k.end()) {
        k = (int)K.size();
        key2k.emplace(key, k);
        XferClass X{};
        for (int q = 0; q < 4; ++q) X.cls[q] = key[q];
        X.nx = d.cx + lastx;
        X.ny = d.cy + lasty;
        K.push_back(X);
        members.emplace_back();
      } else {
        k = it->second;
      }
      members[k].push_back(CI * d.ncy + CJ);
    }
}

// Galerkin GEMM layout: packed upper-triangle column count (P = 4k) padded to whole 64-column
// tiles; row tiles of 64 (cell, realisation) pairs
int gal_psp(const Dims& d) {
  const int P = 4 * d.kmax, PS = P * (P + 1) / 2;
  return (PS + GT - 1) / GT * GT;
}
}  // namespace

// Host plan of the cell-class transfer and Galerkin products for this rank's cells [C0, C1)
// (all cells on one GPU).
int xfer_setup(msf_ctx* c, char*& cur) {
  const Dims& d = c->d;
  const int G = (4 * d.kmax + XNJ - 1) / XNJ;
  // entry tiles of a pattern column: 2 (cy + 1) <= 56
  if (G < 1 || G > 4 || 2 * (d.cy + 1) > 56 || prolong_smem(d) > 200 * 1024) return -1;
  std::vector<XferClass> K;
  std::vector<std::vector<int>> members;
  cell_classes(d, c->cls_of_agg, c->sb.C0, c->sb.C1, K, members);
  std::vector<int> cells;
  std::vector<XferTask> tasks;
  std::vector<int4> gtasks;   // Galerkin GEMM tiles: (class, first row, first column, -)
  const int R = d.R, psp = gal_psp(d);
  size_t ngroups = 0;
  for (const auto& m : members) ngroups += (m.size() + NCC - 1) / NCC;
  const int nch = xfer_nchunk(d, ngroups);
  for (size_t k = 0; k < K.size(); ++k) {
    K[k].cell_off = (int)cells.size();
    cells.insert(cells.end(), members[k].begin(), members[k].end());
    const int ncell = (int)members[k].size();
    for (int c0 = 0; c0 < ncell; c0 += NCC)
      for (int ch = 0; ch < nch; ++ch) tasks.push_back(XferTask{(int)k, c0, std::min(NCC, ncell - c0), ch});
    for (int r0 = 0; r0 < ncell * R; r0 += GT)
      for (int q0 = 0; q0 < psp; q0 += GT) gtasks.push_back(make_int4((int)k, r0, q0, ncell * R));
  }
  // packed upper triangle: column s -> (p, q), p <= q
  const int P = 4 * d.kmax;
  std::vector<int2> pq(psp, make_int2(-1, -1));
  for (int p = 0, s = 0; p < P; ++p)
    for (int q = p; q < P; ++q) pq[s++] = make_int2(p, q);
  auto take = [&](size_t bytes) {
    char* r = cur;
    cur += (bytes + 255) & ~(size_t)255;
    return (void*)r;
  };
  c->xf_G = G;
  c->xf_nch = nch;
  c->xf_ntasks = (int)tasks.size();
  c->xf_n_cls = (int)K.size();
  c->xf_cls = take(K.size() * sizeof(XferClass));
  c->xf_tasks = take(tasks.size() * sizeof(XferTask));
  c->xf_cells = (int*)take(cells.size() * 4);
  c->xf_part = (double*)take((size_t)d.R * d.ncx * d.ncy * nch * G * XNJ * 8);
  c->gal_ntasks = (int)gtasks.size();
  c->gal_tasks = (int4*)take(gtasks.size() * sizeof(int4));
  c->gal_pq = (int2*)take(pq.size() * sizeof(int2));
  c->gal_M = (double*)take(K.size() * (size_t)d.cx * d.cy * psp * 8);
  cudaFuncSetAttribute(k_prolong_cells, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prolong_smem(d));
  cudaFuncSetAttribute(k_restrict_cells, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)restrict_smem(d));
  cudaError_t e = cudaMemcpyAsync(c->xf_cls, K.data(), K.size() * sizeof(XferClass), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->xf_tasks, tasks.data(), tasks.size() * sizeof(XferTask), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->xf_cells, cells.data(), cells.size() * 4, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->gal_tasks, gtasks.data(), gtasks.size() * sizeof(int4), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->gal_pq, pq.data(), pq.size() * sizeof(int2), cudaMemcpyHostToDevice, c->stream);
  return e == cudaSuccess ? 0 : -2;
}

size_t xfer_workspace_bytes(const Dims& d, const std::vector<int>& cls_of_agg, int C0, int C1) {
  const int G = (4 * d.kmax + XNJ - 1) / XNJ;
  std::vector<XferClass> K;
  std::vector<std::vector<int>> members;
  cell_classes(d, cls_of_agg, C0, C1, K, members);
  size_t ntask = 0, ngt = 0, ngroups = 0;
  const int psp = gal_psp(d);
  for (const auto& m : members) ngroups += (m.size() + NCC - 1) / NCC;
  const int nch = xfer_nchunk(d, ngroups);
  for (const auto& m : members) {
    ntask += nch * ((m.size() + NCC - 1) / NCC);
    ngt += ((m.size() * d.R + GT - 1) / GT) * (psp / GT);
  }
  const size_t ncell = (size_t)d.ncx * d.ncy;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  return al(K.size() * sizeof(XferClass)) + al(ntask * sizeof(XferTask)) + al(ncell * 4) +
         al((size_t)d.R * ncell * nch * G * XNJ * 8) + al(ngt * sizeof(int4)) + al(psp * sizeof(int2)) +
         al(K.size() * (size_t)d.cx * d.cy * psp * 8);
}

void launch_prolong(msf_ctx* c, int rhs0, int nr, const double* zin, double* z, bool gated) {
  launch_k(k_prolong_cells, dim3(c->xf_ntasks, nr), dim3(XT), prolong_smem(c->d), c->stream, c->dl,
           (const XferClass*)c->xf_cls, (const XferTask*)c->xf_tasks, (const int*)c->xf_cells,
           (const double*)c->phi, (const double*)c->cx, (const double2*)zin, (double2*)z,
           (const PcgScalars*)c->sc, rhs0, gated ? 1 : 0, c->xf_G, c->xf_nch);
  MSF_LAUNCHED(c);
}

void launch_restrict(msf_ctx* c, int rhs0, int nr, const double* t, bool gated) {
  const Dims& d = c->dl;
  launch_k(k_restrict_cells, dim3(c->xf_ntasks, nr), dim3(XT), restrict_smem(c->d), c->stream, d,
           (const XferClass*)c->xf_cls, (const XferTask*)c->xf_tasks, (const int*)c->xf_cells,
           (const double*)c->phi, (const double2*)t, c->xf_part, (const PcgScalars*)c->sc, rhs0,
           gated ? 1 : 0, c->xf_G, c->xf_nch);
  MSF_LAUNCHED(c);
  const int naggs = (c->cr_hi - c->cr_lo + 1) * (d.ncy + 1);
  launch_k(k_restrict_aggs, dim3((naggs * d.kmax + 255) / 256, nr), dim3(256), 0, c->stream, d,
           (const double*)c->xf_part, c->xf_G * XNJ, c->xf_nch, c->cr_lo, c->cr_hi, c->sb.C0, c->sb.C1, c->cb,
           (const PcgScalars*)c->sc, rhs0, gated ? 1 : 0);
  MSF_LAUNCHED(c);
}

// Galerkin cell products Kcell = Phi_C^T (E K0) Phi_C of this rank's coarse cells (Eq. 10),
// all realisations: the class element matrices M_k, then one DMMA GEMM tile per task
void launch_galerkin_cells(msf_ctx* c) {
  const Dims& d = c->d;
  const int psp = gal_psp(d), P = 4 * d.kmax;
  k_galerkin_M<<<dim3(d.cx * d.cy, c->xf_n_cls), 256, 16 * P * sizeof(double), c->stream>>>(
      d, c->K0, (const XferClass*)c->xf_cls, (const double*)c->phi, (const int2*)c->gal_pq, psp,
      c->gal_M);
  MSF_LAUNCHED(c);
  k_galerkin_gemm<<<dim3(c->gal_ntasks), 256, 0, c->stream>>>(
      d, (const XferClass*)c->xf_cls, (const int4*)c->gal_tasks, (const int*)c->xf_cells,
      (const double*)c->E, (const double*)c->gal_M, (const int2*)c->gal_pq, psp, c->Kcell);
  MSF_LAUNCHED(c);
}
