// Coarse solve K_c x = c by nested dissection (Eq. 10, l.136: K_c = R_c K R_c^T is
// solved exactly in every application of the two-level preconditioner, §2.4.2 l.146).
//
// K_c couples the k eigen-slots of coarse node (I, J) with those of its 8 neighbours (the
// agglomerates of two nodes overlap iff the nodes share a coarse cell), so it is a 9-point
// block stencil on the (ncx+1) x (ncy+1) coarse node grid.  The grid is dissected
// recursively: a box of nodes is split by its middle column or
// row (the longer side) into two boxes and a separator line; boxes of at most ND_LEAF x
// ND_LEAF nodes are leaves.  Every box is a *front*: S = its separator (or all nodes of a
// leaf) is eliminated, B = the ring of nodes around the box (all eliminated later) is its
// boundary.  With F = [A B^T; B C] the front matrix over S u B (original entries of the rows
// of S plus the children's Schur complements, extend-added), the sweep operator applied to
// the pivots of S turns F into
//     F_SS = -A^{-1},  F_BS = B A^{-1},  F_SB = A^{-1} B^T,  F_BB = C - B A^{-1} B^T,
// i.e. the inverse pivot block, the elimination multipliers and the Schur complement handed
// to the parent, in one blocked, tensor-core algorithm.  The solve then is
//     forward (leaves to root):  v = [c_S; 0] + sum_children u_child,   u = v_B - F_BS v_S
//     back    (root to leaves):  x_S = -(F_SS v_S + F_SB x_B)
// with x_B read from the already solved ancestors.  Each level is one launch in each
// direction, one warp per matrix row; all realisations are batched (launch z).
//
// Compared with block cyclic reduction over coarse columns (dense m x m blocks, m = (ncy+1) k)
// the solve streams O(n log n) instead of O(n m) entries: configs[4] 0.33 GB instead of
// 2.74 GB per solve and realisation, configs[3] (k = 16) 2.4 GB instead of 22 GB.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <unordered_map>

#include "msf_internal.cuh"
#include "msf_kern.cuh"

using namespace msfk;

namespace {

constexpr int NB = 64;        // sweep panel / GEMM tile size

// largest i in [0, n) with P[i] <= x (P non-decreasing, P[0] = 0 <= x < P[n])
__device__ __forceinline__ int nd_find(const int* __restrict__ P, int n, int x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Original K_c entry (coarse node gp, slot a; node gq, slot b) summed over the coarse cells
// [clo, chi) x [0, ncy) common to both agglomerates (K_c = sum over cells of the Galerkin cell
// products, Eq. 10; cells = false: none); unused eigen-slots (a >= nkept) are identity rows
// (ident = false: left out).
__device__ __forceinline__ double kc_entry(const Dims& d, const double* __restrict__ Kc,
                                           const int* __restrict__ cls_of_agg,
                                           const EigClass* __restrict__ cls, int gp, int a, int gq,
                                           int b, int clo, int chi, bool cells, bool ident) {
  const int Y = d.ncy + 1, k = d.kmax, P = 4 * k;
  const int Ip = gp / Y, Jp = gp - (gp / Y) * Y, Iq = gq / Y, Jq = gq - (gq / Y) * Y;
  if (abs(Ip - Iq) > 1 || abs(Jp - Jq) > 1) return 0.0;
  const int nka = cls[cls_of_agg[gp]].nkept, nkb = cls[cls_of_agg[gq]].nkept;
  if (a >= nka || b >= nkb) return (ident && gp == gq && a == b) ? 1.0 : 0.0;
  if (!cells) return 0.0;
  double v = 0.0;
  const int CIlo = max(max(max(Ip, Iq) - 1, 0), clo), CIhi = min(min(Ip, Iq), chi - 1);
  const int CJlo = max(max(Jp, Jq) - 1, 0), CJhi = min(min(Jp, Jq), d.ncy - 1);
  for (int CI = CIlo; CI <= CIhi; ++CI)
    for (int CJ = CJlo; CJ <= CJhi; ++CJ) {
      const int pr = ((Ip - CI) * 2 + (Jp - CJ)) * k + a;
      const int pc = ((Iq - CI) * 2 + (Jq - CJ)) * k + b;
      v += Kc[((size_t)CI * d.ncy + CJ) * P * P + (size_t)pr * P + pc];
    }
  return v;
}

// ------------------------------------------------------------------ assembly of the fronts
// F = original entries of the rows / columns of S  +  extend-add of the children's F_BB.
// Tasks: 64 x 64 tiles of the fronts of one level (list: fronts[n], tile prefix[n + 1]).
// mode 0 (fronts of this rank's box): cell entries of the cells [clo, chi), identity rows of
//   the unused eigen-slots, every child;
// mode 1 (interface fronts, this rank's partial before the all-reduce): cell entries of the
//   rank's cells and the rank's own box root (a local child) only;
// mode 2 (interface fronts after the all-reduce, replicated): identity rows and the
//   interface children, ADDED to the all-reduced partial sum.
__global__ void __launch_bounds__(256) k_nd_assemble(Dims d, const NdFront* __restrict__ fr,
                                                     const int* __restrict__ nodes,
                                                     const int* __restrict__ chmap,
                                                     const int* __restrict__ list, int n,
                                                     const double* __restrict__ Kcell,
                                                     const int* __restrict__ cls_of_agg,
                                                     const EigClass* __restrict__ cls, double* Fall,
                                                     long long Fstride, int clo, int chi, int mode) {
  const int li = nd_find(list + n, n, blockIdx.x);
  const int f = list[li], t = blockIdx.x - list[n + li];
  const NdFront F = fr[f];
  const int k = d.kmax, nf = (F.s_n + F.b_n) * k, ld = nf + (nf & 1), nt = (nf + NB - 1) / NB;
  const int ti = t / nt, tj = t - (t / nt) * nt;
  const int rhs = blockIdx.y;
  const int ch[2] = {F.ch0, F.ch1};
  int cs[2] = {0, 0}, cld[2] = {0, 0};
  long long coff[2] = {0, 0};
#pragma unroll
  for (int c = 0; c < 2; ++c)
    if (ch[c] >= 0) {
      const NdFront C = fr[ch[c]];
      cs[c] = C.s_n * k;
      cld[c] = (C.s_n + C.b_n) * k;
      cld[c] += cld[c] & 1;
      coff[c] = C.F_off;
    }
  const double* Fr = Fall + (size_t)rhs * Fstride;
  double* A = Fall + (size_t)rhs * Fstride + F.F_off;
  const double* Kc = Kcell + (size_t)rhs * d.ncx * d.ncy * 16 * k * k;
  for (int e = threadIdx.x; e < NB * NB; e += 256) {
    const int i = ti * NB + (e >> 6), j = tj * NB + (e & 63);
    if (i >= nf || j >= nf) continue;
    const int pn = i / k, a = i - pn * k, qn = j / k, b = j - qn * k;
    double v = 0.0;
    if (pn < F.s_n || qn < F.s_n)
      v = kc_entry(d, Kc, cls_of_agg, cls, nodes[F.node_off + pn], a, nodes[F.node_off + qn], b, clo,
                   chi, mode != 2, mode != 1);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (ch[c] < 0) continue;
      const bool ctop = (F.flags >> (1 + c)) & 1;
      if ((mode == 1 && ctop) || (mode == 2 && !ctop)) continue;
      const int cp = chmap[F.chmap_off + 2 * pn + c], cq = chmap[F.chmap_off + 2 * qn + c];
      if (cp >= 0 && cq >= 0)
        v += Fr[coff[c] + (size_t)(cs[c] + cp * k + a) * cld[c] + cs[c] + cq * k + b];
    }
    if (mode == 2) A[(size_t)i * ld + j] += v;
    else A[(size_t)i * ld + j] = v;
  }
}

// ------------------------------------------------------------------ blocked sweep
// Panel pt of the pivots of S (rows / columns [p0, p0 + pb), p0 = 64 pt) of every front of
// one level with s > p0 (list: fronts[n], tile prefix[n + 1], tile^2 prefix[n + 1],
// n_f prefix[n + 1] for the scratch offsets).  Four launches per panel:
//   pivot:    L = chol(A_pp),  Q = -A_pp^{-1} = -L^{-T} L^{-1}            (one CTA per front)
//   rowpanel: Z = L^{-1} A[p, :],  Rp = L^{-T} Z = A_pp^{-1} A[p, :]      (tiles of 64 columns)
//   trailing: A[i, j] -= Z[:, i]^T Z[:, j]  (= A_ip A_pp^{-1} A_pj)      (DMMA, 64 x 64 tiles)
//   panels:   A[p, j] = Rp[:, j],  A[i, p] = Rp[:, i]^T,  A_pp = Q
// This is the block form of the sweep a_ij <- a_ij - a_ik a_kj / a_kk, a_ik <- a_ik / a_kk,
// a_kk <- -1 / a_kk (a_ip = a_pi, the front is symmetric), with every panel eliminated
// through the Cholesky factor of its pivot block: the Schur update is the symmetric Z^T Z and
// no explicit block inverse multiplies a panel.  (Multiplying by an explicit pivot-block
// inverse, Rp = A_pp^{-1} A[p, :] then A -= A[:, p] Rp, lost all accuracy on K_c of
// condition 3e12 -- E_min = 1e-9 binary cells -- relative residual 1.8e7 in a numpy model;
// this form gives 2.9e-6, as a scalar sweep or a full Cholesky solve do.)
struct PanelArgs {
  const int* list;   // fronts[n] | P_nt[n+1] | P_nt2[n+1] | P_nf[n+1]
  int n;
  int pt;
  double* Q;         // [R][n][64*64]  -A_pp^{-1}
  double* L;         // [R][n][64*64]  chol(A_pp)
  double* Z;         // [R][64 * P_nf[n]]  L^{-1} A[p, :]  (ld n_f)
  double* Rp;        // [R][64 * P_nf[n]]  A_pp^{-1} A[p, :]
  long long Qstride, Sstride;
};

// n_f, its (even) leading dimension in storage, s, and the panel's pivot range
__device__ __forceinline__ void front_dims(const NdFront& F, int k, int pt, int& nf, int& ld, int& s,
                                           int& p0, int& pb) {
  nf = (F.s_n + F.b_n) * k;
  ld = nf + (nf & 1);
  s = F.s_n * k;
  p0 = pt * NB;
  pb = min(NB, s - p0);
}

__global__ void __launch_bounds__(256) k_nd_pivot(Dims d, const NdFront* __restrict__ fr,
                                                  double* Fall, long long Fstride, PanelArgs pa,
                                                  int* status) {
  extern __shared__ double psm[];
  double (*a)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(psm);                  // A_pp -> L
  double (*x)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(psm + NB * (NB + 1));  // L^{-1}
  const int f = pa.list[blockIdx.x], rhs = blockIdx.y;
  const NdFront F = fr[f];
  int nf, ld, s, p0, pb;
  front_dims(F, d.kmax, pa.pt, nf, ld, s, p0, pb);
  const double* A = Fall + (size_t)rhs * Fstride + F.F_off;
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 256) {
    const int i = e >> 6, j = e & 63;
    a[i][j] = (i < pb && j < pb) ? A[(size_t)(p0 + i) * ld + p0 + j] : 0.0;
    x[i][j] = 0.0;
  }
  __syncthreads();
  // right-looking Cholesky, lower triangle
  for (int kk = 0; kk < pb; ++kk) {
    const double piv = a[kk][kk];
    if (!(piv > 0.0)) {
      if (tid == 0) atomicExch(status + rhs, 2);
    }
    const double dk = sqrt(fmax(piv, 1e-300));
    __syncthreads();
    for (int i = kk + 1 + tid; i < pb; i += 256) a[i][kk] /= dk;
    __syncthreads();
    if (tid == 0) a[kk][kk] = dk;
    const int m = pb - kk - 1;
    for (int e = tid; e < m * m; e += 256) {
      const int i = kk + 1 + e / m, j = kk + 1 + (e - (e / m) * m);
      if (j <= i) a[i][j] = fma(-a[i][kk], a[j][kk], a[i][j]);
    }
    __syncthreads();
  }
  // X = L^{-1}: column j by forward substitution (one thread per column)
  if (tid < pb) {
    const int j = tid;
    for (int i = j; i < pb; ++i) {
      double v = (i == j) ? 1.0 : 0.0;
      for (int l = j; l < i; ++l) v = fma(-a[i][l], x[l][j], v);
      x[i][j] = v / a[i][i];
    }
  }
  __syncthreads();
  double* Q = pa.Q + (size_t)rhs * pa.Qstride + (size_t)blockIdx.x * NB * NB;
  double* Lg = pa.L + (size_t)rhs * pa.Qstride + (size_t)blockIdx.x * NB * NB;
  for (int e = tid; e < NB * NB; e += 256) {
    const int i = e >> 6, j = e & 63;
    double q = 0.0;
    if (i < pb && j < pb)
      for (int l = max(i, j); l < pb; ++l) q = fma(x[l][i], x[l][j], q);   // (X^T X)_ij
    Q[e] = -q;
    Lg[e] = (j <= i) ? a[i][j] : 0.0;
  }
}

// Z = L^{-1} A[p, tile], Rp = L^{-T} Z: one thread per column (substitutions over the panel)
__global__ void __launch_bounds__(NB) k_nd_rowpanel(Dims d, const NdFront* __restrict__ fr,
                                                    const double* __restrict__ Fall,
                                                    long long Fstride, PanelArgs pa) {
  extern __shared__ double rsm[];
  double (*Ls)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(rsm);
  double (*zs)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(rsm + NB * (NB + 1));   // [row][col]
  const int* Pnt = pa.list + pa.n;
  const int* Pnf = pa.list + 3 * (pa.n + 1) - 1;
  const int li = nd_find(Pnt, pa.n, blockIdx.x);
  const int f = pa.list[li], tj = blockIdx.x - Pnt[li], rhs = blockIdx.y;
  const NdFront F = fr[f];
  int nf, ld, s, p0, pb;
  front_dims(F, d.kmax, pa.pt, nf, ld, s, p0, pb);
  const double* A = Fall + (size_t)rhs * Fstride + F.F_off;
  const double* Lg = pa.L + (size_t)rhs * pa.Qstride + (size_t)li * NB * NB;
  double* Z = pa.Z + (size_t)rhs * pa.Sstride + (size_t)NB * Pnf[li];
  double* Rp = pa.Rp + (size_t)rhs * pa.Sstride + (size_t)NB * Pnf[li];
  const int j0 = tj * NB, jw = min(NB, nf - j0);
  const int t = threadIdx.x;
  for (int i = 0; i < NB; ++i) {
    Ls[i][t] = Lg[i * NB + t];
    zs[i][t] = (i < pb && t < jw) ? A[(size_t)(p0 + i) * ld + j0 + t] : 0.0;
  }
  __syncthreads();
  if (t < jw) {
    for (int i = 0; i < pb; ++i) {             // forward: L z = a
      double v = zs[i][t];
      for (int l = 0; l < i; ++l) v = fma(-Ls[i][l], zs[l][t], v);
      zs[i][t] = v / Ls[i][i];
    }
    for (int i = 0; i < pb; ++i) Z[(size_t)i * nf + j0 + t] = zs[i][t];
    for (int i = pb - 1; i >= 0; --i) {        // back: L^T r = z
      double v = zs[i][t];
      for (int l = i + 1; l < pb; ++l) v = fma(-Ls[l][i], zs[l][t], v);
      zs[i][t] = v / Ls[i][i];
    }
    for (int i = 0; i < pb; ++i) Rp[(size_t)i * nf + j0 + t] = zs[i][t];
  }
}

// ---- DMMA (fp64 tensor core, mma.sync m8n8k4) 64 x 64 tile update
// C[0:mr, 0:nc] += alpha * sum_k A[k][0:mr]^T B[k][0:nc]; A, B k-major (row k contiguous).
// 8 warps as 2 (rows) x 4 (columns), each warp a 32 x 16 sub-tile = 4 x 2 DMMA fragments.
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64): lane = 4 g + t;  A(g, t), B(t, g),
// C(g, 2t + {0, 1}).  Shared rows padded to 68 doubles: conflict-free fragment loads.
constexpr int SPAD = NB + 4;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// stage K rows of 64 doubles (A and B panels) into shared memory, zero-padded to Kp (mult. of 4)
__device__ __forceinline__ void stage_kpanel(double* sX, const double* __restrict__ X, int ldx,
                                             int K, int Kp, int w) {
  for (int e = threadIdx.x; e < Kp * NB; e += blockDim.x) {
    const int kk = e >> 6, x = e & 63;
    sX[kk * SPAD + x] = (kk < K && x < w) ? X[(size_t)kk * ldx + x] : 0.0;
  }
}

__device__ __forceinline__ void dmma_tile_acc(const double* sA, const double* sB, int Kp,
                                              double (&acc)[4][2][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (w >> 2) * 32, n0 = (w & 3) * 16;
  for (int k0 = 0; k0 < Kp; k0 += 4) {
    double a[4], b[2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = sA[(k0 + t) * SPAD + m0 + mi * 8 + g];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) b[ni] = sB[(k0 + t) * SPAD + n0 + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
  }
}

__device__ __forceinline__ void dmma_tile_store(double* C, int ldc, int mr, int nc,
                                                const double (&acc)[4][2][2], double alpha,
                                                bool add) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (w >> 2) * 32, n0 = (w & 3) * 16;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int r = m0 + mi * 8 + g;
    if (r >= mr) continue;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int c = n0 + ni * 8 + 2 * t;
      double* p = C + (size_t)r * ldc + c;
      if (c + 1 < nc && !(ldc & 1)) {
        double2 o = add ? *reinterpret_cast<double2*>(p) : make_double2(0.0, 0.0);
        o.x = fma(alpha, acc[mi][ni][0], o.x);
        o.y = fma(alpha, acc[mi][ni][1], o.y);
        *reinterpret_cast<double2*>(p) = o;
      } else {
        if (c < nc) p[0] = fma(alpha, acc[mi][ni][0], add ? p[0] : 0.0);
        if (c + 1 < nc) p[1] = fma(alpha, acc[mi][ni][1], add ? p[1] : 0.0);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_nd_trailing(Dims d, const NdFront* __restrict__ fr,
                                                     double* Fall, long long Fstride, PanelArgs pa) {
  extern __shared__ double tsm[];
  double* sA = tsm;                 // [64][SPAD]
  double* sB = tsm + NB * SPAD;     // [64][SPAD]
  const int* Pnt2 = pa.list + 2 * pa.n + 1;
  const int* Pnf = pa.list + 3 * (pa.n + 1) - 1;
  const int li = nd_find(Pnt2, pa.n, blockIdx.x);
  const int f = pa.list[li], t = blockIdx.x - Pnt2[li], rhs = blockIdx.y;
  const NdFront F = fr[f];
  int nf, ld, s, p0, pb;
  front_dims(F, d.kmax, pa.pt, nf, ld, s, p0, pb);
  const int nt = (nf + NB - 1) / NB;
  const int ti = t / nt, tj = t - (t / nt) * nt;
  // (tiles of the pivot panel are updated too: their pivot rows / columns are rewritten by
  // k_nd_panels, their other rows / columns need the update)
  const double* Z = pa.Z + (size_t)rhs * pa.Sstride + (size_t)NB * Pnf[li];
  const int i0 = ti * NB, j0 = tj * NB;
  const int mr = min(NB, nf - i0), nc = min(NB, nf - j0);
  const int Kp = (pb + 3) & ~3;
  stage_kpanel(sA, Z + i0, nf, pb, Kp, mr);
  stage_kpanel(sB, Z + j0, nf, pb, Kp, nc);
  __syncthreads();
  double* A = Fall + (size_t)rhs * Fstride + F.F_off;
  double acc[4][2][2] = {};
  dmma_tile_acc(sA, sB, Kp, acc);
  dmma_tile_store(A + (size_t)i0 * ld + j0, ld, mr, nc, acc, -1.0, true);
}

__global__ void __launch_bounds__(256) k_nd_panels(Dims d, const NdFront* __restrict__ fr,
                                                   double* Fall, long long Fstride, PanelArgs pa) {
  __shared__ double tile[NB][NB + 1];
  const int* Pnt = pa.list + pa.n;
  const int* Pnf = pa.list + 3 * (pa.n + 1) - 1;
  const int li = nd_find(Pnt, pa.n, blockIdx.x);
  const int f = pa.list[li], tt = blockIdx.x - Pnt[li], rhs = blockIdx.y;
  const NdFront F = fr[f];
  int nf, ld, s, p0, pb;
  front_dims(F, d.kmax, pa.pt, nf, ld, s, p0, pb);
  double* A = Fall + (size_t)rhs * Fstride + F.F_off;
  const int t0 = tt * NB, tw = min(NB, nf - t0);
  const double* Q = pa.Q + (size_t)rhs * pa.Qstride + (size_t)li * NB * NB;
  const double* Rp = pa.Rp + (size_t)rhs * pa.Sstride + (size_t)NB * Pnf[li];
  // pivot rows of this column tile: Q inside the pivot block, Rp elsewhere
  for (int e = threadIdx.x; e < NB * NB; e += 256) {
    const int i = e >> 6, j = e & 63;
    if (i < pb && j < tw) {
      const int col = t0 + j;
      const double v = (col >= p0 && col < p0 + pb) ? Q[i * NB + (col - p0)] : Rp[(size_t)i * nf + col];
      tile[i][j] = v;
      A[(size_t)(p0 + i) * ld + col] = v;
    }
  }
  __syncthreads();
  // pivot columns (the transpose; the front stays symmetric)
  for (int e = threadIdx.x; e < NB * NB; e += 256) {
    const int j = e >> 6, i = e & 63;        // A[t0 + j, p0 + i] = A[p0 + i, t0 + j]
    if (i < pb && j < tw) A[(size_t)(t0 + j) * ld + p0 + i] = tile[i][j];
  }
}

// ------------------------------------------------------------------ solve
// One launch per level and direction.  A CTA owns RB rows of one front: one bulk copy per row
// (cp.async.bulk, completion counted in bytes on an mbarrier) stages them in shared memory,
// issued BEFORE the PDL wait -- the fronts are constant during PCG, so the matrix stream of a
// level overlaps the levels before it and a latency-bound top level finds its rows on chip.
// After the wait the CTA gathers the front's right-hand side through its vmap (global coarse
// index, children's update indices), then one warp per row forms the dot product from shared
// memory:
//   forward (FWD):  u[r] = v_B[r] - F[s + r, 0:s] . v_S          rows r < b
//   back:           x_S[r] = -F[r, 0:n_f] . [v_S; x_B]           rows r < s
// RB per level: whole leaf fronts per CTA at the bottom, 8 rows per CTA at the top, at most
// ND_STAGE bytes of rows per CTA.  Dependents are signalled once the CTA's row copies are
// issued (see k_nd_solve).
#ifndef MSF_ND_NSMAX
#define MSF_ND_NSMAX 4
#endif
#ifndef MSF_ND_NSDIV
#define MSF_ND_NSDIV 2
#endif
#ifndef MSF_ND_STAGE_KB
#define MSF_ND_STAGE_KB 32
#endif
constexpr int ND_STAGE = MSF_ND_STAGE_KB * 1024;       // staged rows per CTA ...
constexpr int ND_STAGE_MAX = 96 * 1024;                 // ... raised up to this for 8 rows of a long front

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <bool FWD, bool MULTI>
__global__ void __launch_bounds__(256) k_nd_solve(Dims d, const NdFront* __restrict__ fr,
                                                  const int4* __restrict__ vmap,
                                                  const int* __restrict__ list, int n, int RB, int NS_,
                                                  const double* __restrict__ Fall, long long Fstride,
                                                  double* uall, long long ustride,
                                                  const double* __restrict__ cball, double* cxall,
                                                  const double* __restrict__ vtall, long long vstride,
                                                  const PcgScalars* sc, int rhs0, int gated) {
  extern __shared__ __align__(16) double nsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(nsm);
  const int NS = MULTI ? NS_ : 1;   // one stage: the stage loop below folds away
  const int li = nd_find(list + n, n, blockIdx.x);
  // the CTA takes NS stages of RB rows: the right-hand side is gathered once for all of them
  // (long fronts: the gather is as long as a row)
  const int f = list[li], rb0 = (blockIdx.x - list[n + li]) * RB * NS;
  const int rhs = rhs0 + blockIdx.y;
  const NdFront F = fr[f];
  const int k = d.kmax, s = F.s_n * k, nf = (F.s_n + F.b_n) * k, ld = nf + (nf & 1);
  const int rows = FWD ? nf - s : s, len = FWD ? s : nf, lenp = len + (len & 1);
  const int nrow_all = min(rows, rb0 + RB * NS) - rb0;   // rows of this CTA
  const int nrow = min(nrow_all, RB);                      // ... of its first stage
  double* sv = nsm + 2;                    // [lenp] right-hand side
  double* vb = sv + lenp;                  // [RB NS] forward: children's updates of the rows
  double* sA = vb + ((RB * NS + 1) & ~1);  // [RB][lenp] staged rows (16-byte aligned)
  const double* A = Fall + (size_t)rhs * Fstride + F.F_off + (size_t)(FWD ? s : 0) * ld;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"((unsigned)(nrow * lenp * 8))
                 : "memory");
  }
  __syncthreads();
  if (wid == 0)
    for (int r = lane; r < nrow; r += 32)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sA + (size_t)r * lenp)),
          "l"(A + (size_t)(rb0 + r) * ld), "r"((unsigned)(lenp * 8)), "r"(smem_u32(bar))
          : "memory");
  // the next level may launch now: its CTAs stage their (constant) rows while this level
  // finishes (measured: 0.266 -> 0.226 ms per configs[4] solve at one realisation).  Signalled
  // at kernel entry instead, the cascade of early grids held SMs and cost 0.48 ms per V-cycle.
  pdl_launch();
  pdl_wait();
  const bool live = !(gated && !sc[rhs].active);
  const double* cb = cball + (size_t)rhs * d.nbc * d.mc;
  double* cx = cxall + (size_t)rhs * d.nbc * d.mc;
  double* u = uall + (size_t)rhs * ustride;
  const double* vt = vtall + (size_t)rhs * vstride;
  const int4* vm = vmap + F.vmap_off;
  if (live) {
    for (int c = threadIdx.x; c < lenp; c += 256) {
      double x = 0.0;
      if (c < len) {
        const int4 m = vm[c];
        if (c < s) {
          x = m.w >= 0 ? vt[m.w] : cb[m.x];
          if (m.y >= 0) x += u[m.y];
          if (m.z >= 0) x += u[m.z];
        } else {
          x = cx[m.x];
        }
      }
      sv[c] = x;
    }
    if (FWD)
      for (int r = threadIdx.x; r < nrow_all; r += 256) {
        const int4 m = vm[s + rb0 + r];
        double x = m.w >= 0 ? vt[m.w] : 0.0;
        if (m.y >= 0) x += u[m.y];
        if (m.z >= 0) x += u[m.z];
        vb[r] = x;
      }
  }
  __syncthreads();
  for (int j = 0, r0 = 0; r0 < nrow_all; ++j, r0 += RB) {
    const int nr = min(nrow_all - r0, RB);
    if (j > 0) {
      // next stage into the same buffer: every warp is done reading it (barrier), and the generic
      // reads are ordered before the async-proxy writes
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                     "r"((unsigned)(nr * lenp * 8))
                     : "memory");
      }
      __syncthreads();
      if (wid == 0)
        for (int r = lane; r < nr; r += 32)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sA + (size_t)r * lenp)),
              "l"(A + (size_t)(rb0 + r0 + r) * ld), "r"((unsigned)(lenp * 8)), "r"(smem_u32(bar))
              : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(smem_u32(bar)),
        "r"((unsigned)(j & 1))
        : "memory");
    if (!live) continue;
    for (int r = wid; r < nr; r += 8) {
      const double* Ar = sA + (size_t)r * lenp;
      double a0 = 0.0, a1 = 0.0;
      int c = lane;
      for (; c + 32 < len; c += 64) {
        a0 = fma(Ar[c], sv[c], a0);
        a1 = fma(Ar[c + 32], sv[c + 32], a1);
      }
      if (c < len) a0 = fma(Ar[c], sv[c], a0);
      const double t = warp_sum(a0 + a1);
      if (lane == 0) {
        if (FWD) u[F.u_off + rb0 + r0 + r] = vb[r0 + r] - t;
        else cx[vm[rb0 + r0 + r].x] = -t;
      }
    }
  }
}

// Interface fronts' partial right-hand sides of this rank, for the all-reduce (strip partition):
// vtop[i] = c[pm.x] (the rank's partial restriction, S variables) + u[pm.y] (its box root's
// update, when the box root is a child of the front)
__global__ void __launch_bounds__(256) k_nd_pack(const int2* __restrict__ pm, int n,
                                                 const double* __restrict__ cball, long long cstride,
                                                 const double* __restrict__ uall, long long ustride,
                                                 double* vtall, long long vstride, const PcgScalars* sc,
                                                 int rhs0, int gated) {
  pdl_wait();
  const int rhs = rhs0 + blockIdx.y;
  if (gated && !sc[rhs].active) return;
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i < n) {
    const int2 m = pm[i];
    double v = 0.0;
    if (m.x >= 0) v += cball[(size_t)rhs * cstride + m.x];
    if (m.y >= 0) v += uall[(size_t)rhs * ustride + m.y];
    vtall[(size_t)rhs * vstride + i] = v;
  }
  pdl_launch();
}

}  // namespace

// ================================================================== host: plan
namespace {

// Leaf boxes of at most leaf x leaf coarse nodes.  Larger leaves trade levels (launch latency)
// for factor bytes: 5 on large boxes (configs[4] solve: 0.216 ms with 5, 0.233 with 7 or 9);
// 9 on boxes of 1,024 .. 8,192 nodes with up to 4 modes, whose solve is all level latency
// (configs[1]: 0.072 -> 0.036 ms; a rank of 8 strips of configs[4]: 0.100 -> 0.094 ms).
constexpr int ND_LEAF = 5, ND_LEAF_SMALL = 9;
inline int nd_leaf(long long box_nodes, int k) {
  return (k <= 4 && box_nodes >= 1024 && box_nodes <= 8192) ? ND_LEAF_SMALL : ND_LEAF;
}

struct Builder {
  int X, Y, k;
  NdPlan& P;
  int rank;
  const std::vector<int>& icol;   // interface column of each rank > 0 (icol[r], r = 1..N-1)
  int leaf = ND_LEAF;             // leaf size of this rank's box (set before its dissection)

  // ring of the box [x0, x1) x [y0, y1) inside the grid
  std::vector<int> ring(int x0, int x1, int y0, int y1) const {
    std::vector<int> r;
    auto add = [&](int x, int y) {
      if (x >= 0 && x < X && y >= 0 && y < Y) r.push_back(x * Y + y);
    };
    for (int y = y0 - 1; y <= y1; ++y) add(x0 - 1, y);
    for (int y = y0 - 1; y <= y1; ++y) add(x1, y);
    for (int x = x0; x < x1; ++x) add(x, y0 - 1);
    for (int x = x0; x < x1; ++x) add(x, y1);
    return r;
  }

  int make(const std::vector<int>& S, const std::vector<int>& B, int c0, int c1, bool top) {
    NdFront F{};
    F.s_n = (int)S.size();
    F.b_n = (int)B.size();
    F.node_off = (int)P.nodes.size();
    F.ch0 = c0;
    F.ch1 = c1;
    F.chmap_off = (int)P.chmap.size();
    F.flags = (top ? 1 : 0) | (c0 >= 0 && (P.fr[c0].flags & 1) ? 2 : 0) | (c1 >= 0 && (P.fr[c1].flags & 1) ? 4 : 0);
    F.vtop_off = -1;
    P.nodes.insert(P.nodes.end(), S.begin(), S.end());
    P.nodes.insert(P.nodes.end(), B.begin(), B.end());
    // for every node of this front, its index in each child's boundary list (-1: none)
    const int chs[2] = {c0, c1};
    std::unordered_map<int, int> pos[2];
    for (int q = 0; q < 2; ++q) {
      if (chs[q] < 0) continue;
      const NdFront& C = P.fr[chs[q]];
      for (int j = 0; j < C.b_n; ++j) pos[q][P.nodes[C.node_off + C.s_n + j]] = j;
    }
    for (int j = 0; j < F.s_n + F.b_n; ++j) {
      const int g = P.nodes[F.node_off + j];
      for (int q = 0; q < 2; ++q) {
        int v = -1;
        if (chs[q] >= 0) {
          auto it = pos[q].find(g);
          if (it != pos[q].end()) v = it->second;
        }
        P.chmap.push_back(v);
      }
    }
    // every boundary node of a child is a node of this front (nested dissection invariant)
    for (int q = 0; q < 2; ++q)
      if (chs[q] >= 0) {
        int found = 0;
        for (int j = 0; j < F.s_n + F.b_n; ++j) found += P.chmap[F.chmap_off + 2 * j + q] >= 0;
        if (found != P.fr[chs[q]].b_n) P.ok = false;
      }
    // level: height among fronts of the same kind (box subtree / interface tree)
    int lv = 0;
    for (int q = 0; q < 2; ++q)
      if (chs[q] >= 0 && ((P.fr[chs[q]].flags & 1) == (top ? 1 : 0))) lv = std::max(lv, P.fr[chs[q]].level + 1);
    F.level = lv;
    P.fr.push_back(F);
    return (int)P.fr.size() - 1;
  }

  // nested dissection of this rank's box (local fronts)
  int rec(int x0, int x1, int y0, int y1) {
    const int w = x1 - x0, h = y1 - y0;
    if (w <= 0 || h <= 0) return -1;
    std::vector<int> S;
    int c0 = -1, c1 = -1;
    if (w <= leaf && h <= leaf) {
      for (int x = x0; x < x1; ++x)
        for (int y = y0; y < y1; ++y) S.push_back(x * Y + y);
    } else if (w >= h) {
      const int xm = x0 + w / 2;
      c0 = rec(x0, xm, y0, y1);
      c1 = rec(xm + 1, x1, y0, y1);
      for (int y = y0; y < y1; ++y) S.push_back(xm * Y + y);
    } else {
      const int ym = y0 + h / 2;
      c0 = rec(x0, x1, y0, ym);
      c1 = rec(x0, x1, ym + 1, y1);
      for (int x = x0; x < x1; ++x) S.push_back(x * Y + ym);
    }
    return make(S, ring(x0, x1, y0, y1), c0, c1, false);
  }

  // ranks [ra, rb) over the node columns [gx0, gx1): a single rank is its box (built only by
  // that rank); a group is split at the interface column of its middle rank, whose front is an
  // interface front (replicated on every rank)
  int group(int ra, int rb, int gx0, int gx1) {
    if (rb - ra == 1) {
      if (ra != rank) return -1;
      leaf = nd_leaf((long long)(gx1 - gx0) * Y, k);
      return rec(gx0, gx1, 0, Y);
    }
    const int rm = (ra + rb) / 2, xm = icol[rm];
    const int c0 = group(ra, rm, gx0, xm);
    const int c1 = group(rm, rb, xm + 1, gx1);
    std::vector<int> S;
    for (int y = 0; y < Y; ++y) S.push_back(xm * Y + y);
    return make(S, ring(gx0, gx1, 0, Y), c0, c1, true);
  }
};

// task list block: fronts[n] then prefix sums of each count function
template <typename... Fn>
NdPlan::List add_list(NdPlan& P, const std::vector<int>& fronts, Fn... cnt) {
  NdPlan::List L;
  L.off = (int)P.lists.size();
  L.n = (int)fronts.size();
  P.lists.insert(P.lists.end(), fronts.begin(), fronts.end());
  auto pref = [&](auto fn) {
    long long s = 0;
    P.lists.push_back(0);
    for (int f : fronts) {
      s += fn(P.fr[f]);
      P.lists.push_back((int)s);
    }
    return s;
  };
  long long tot[] = {pref(cnt)...};
  L.total = (int)tot[0];
  return L;
}

// the task lists of one group of levels (box subtree or interface tree)
void level_lists(NdPlan& P, int k, const std::vector<std::vector<int>>& lev, NdPlan::Levels& Lv) {
  const int H = (int)lev.size();
  Lv.asmb.resize(H);
  Lv.fwd.resize(H);
  Lv.back.resize(H);
  Lv.panel.resize(H);
  Lv.fwd_smem.assign(H, 0);
  Lv.back_smem.assign(H, 0);
  auto nt = [k](const NdFront& F) { return (long long)((F.s_n + F.b_n) * k + NB - 1) / NB; };
  // rows per solve CTA: the level's rows over about 4 CTAs per SM, a multiple of 8, at least 8,
  // at most the largest front's rows and ND_STAGE bytes of staged rows (very long rows, k = 16:
  // fewer rows than warps)
  auto pick = [&](const std::vector<int>& fl, bool fwd, int& lmax) {
    long long rows = 0;
    int rmax = 0;
    lmax = 0;
    for (int f : fl) {
      const NdFront& F = P.fr[f];
      const int r = (fwd ? F.b_n : F.s_n) * k;
      const int len = fwd ? F.s_n * k : (F.s_n + F.b_n) * k;
      rows += r;
      rmax = std::max(rmax, r);
      lmax = std::max(lmax, len + (len & 1));
    }
    const long long want = std::max<long long>(8, (rows / (148LL * 4) + 7) / 8 * 8);
    // (measured, configs[4] / configs[3] solve at one realisation: 96 KB stages 0.223 / 1.145 ms,
    // 48 KB 0.214 / 1.043, 32 KB 0.210 / 1.074 -- small stages keep more CTAs, i.e. more row
    // pipelines, per SM; but 8 rows, one per warp, are kept where they fit 96 KB)
    const long long stage = std::min<long long>(ND_STAGE_MAX, std::max<long long>(ND_STAGE, 64LL * std::max(1, lmax)));
    long long cap = stage / (8LL * std::max(1, lmax));
    if (cap < 8) {
      long long p = 1;
      while (p * 2 <= cap) p *= 2;
      return (int)p;
    }
    cap = cap / 8 * 8;
    return (int)std::min<long long>(std::min(want, cap), std::max(8, (rmax + 7) / 8 * 8));
  };
  auto smem = [](int lmax, int RB, int NS) {
    return (int)(8 * (2 + (long long)lmax + ((RB * NS + 1) & ~1) + (long long)RB * lmax));
  };
  // stages per CTA: a long front's right-hand-side gather (index map + values, ~32 B per entry)
  // is as long as a row, so CTAs of 8 rows spent a third of their time on it; up to 4 stages per
  // CTA where the level still leaves 3 CTAs per SM (short fronts: 1 stage, as before)
  auto stages = [&](const std::vector<int>& fl, bool fwd, int RB, int lmax) {
    if (lmax < 512) return 1;
    long long rows = 0;
    for (int f : fl) rows += (long long)(fwd ? P.fr[f].b_n : P.fr[f].s_n) * k;
    return (int)std::max<long long>(1, std::min<long long>(MSF_ND_NSMAX, rows / ((long long)RB * 148 * MSF_ND_NSDIV)));
  };
  for (int h = 0; h < H; ++h) {
    Lv.asmb[h] = add_list(P, lev[h], [&](const NdFront& F) { return nt(F) * nt(F); });
    std::vector<int> fw;
    for (int f : lev[h])
      if (P.fr[f].b_n > 0) fw.push_back(f);
    int lmax = 0;
    int RB = pick(fw, true, lmax);
    int NS = stages(fw, true, RB, lmax);
    Lv.fwd[h] = add_list(P, fw, [&](const NdFront& F) { return (long long)(F.b_n * k + RB * NS - 1) / (RB * NS); });
    Lv.fwd[h].RB = RB;
    Lv.fwd[h].NS = NS;
    Lv.fwd_smem[h] = smem(lmax, RB, NS);
    RB = pick(lev[h], false, lmax);
    NS = stages(lev[h], false, RB, lmax);
    Lv.back[h] = add_list(P, lev[h], [&](const NdFront& F) { return (long long)(F.s_n * k + RB * NS - 1) / (RB * NS); });
    Lv.back[h].RB = RB;
    Lv.back[h].NS = NS;
    Lv.back_smem[h] = smem(lmax, RB, NS);
    int smax = 0;
    for (int f : lev[h]) smax = std::max(smax, P.fr[f].s_n * k);
    for (int pt = 0; pt * NB < smax; ++pt) {
      std::vector<int> act;
      for (int f : lev[h])
        if (P.fr[f].s_n * k > pt * NB) act.push_back(f);
      NdPlan::List L = add_list(
          P, act, [&](const NdFront& F) { return nt(F); }, [&](const NdFront& F) { return nt(F) * nt(F); },
          [&](const NdFront& F) { return (long long)(F.s_n + F.b_n) * k; });
      L.total2 = P.lists[L.off + 2 * L.n + 1 + L.n];
      L.total3 = P.lists[L.off + 3 * L.n + 2 + L.n];
      Lv.panel[h].push_back(L);
      P.max_act = std::max(P.max_act, L.n);
      P.scr_doubles = std::max(P.scr_doubles, (long long)NB * L.total3);
    }
  }
}

}  // namespace

// Builds the nested-dissection plan of the coarse node grid for rank `rank` of `nranks`
// (DESIGN.md §8(e)): the interface columns icol[1..N-1] (the first coarse column of each rank
// > 0) are the separators of a bisection over the ranks (interface fronts, replicated); each
// rank dissects its own box between them (local fronts).  One GPU: one box, every node.
// Returns false on an internal inconsistency.
bool nd_build_plan(const Dims& d, NdPlan& P, int rank, int nranks, const std::vector<int>& icol) {
  P = NdPlan();
  const int X = d.ncx + 1, Y = d.ncy + 1, k = d.kmax;
  Builder b{X, Y, k, P, rank, icol};
  P.root = b.group(0, nranks, 0, X);
  if (!P.ok) return false;
  // storage: interface fronts first (identical layout on every rank: one all-reduce), then
  // the rank's box fronts; 256-byte aligned, even leading dimension
  long long Fo = 0, uo = 0, vo = 0;
  int H = 0, TH = 0;
  for (int pass = 0; pass < 2; ++pass) {
    for (NdFront& F : P.fr) {
      const bool top = F.flags & 1;
      if (top != (pass == 0)) continue;
      const long long nf = (long long)(F.s_n + F.b_n) * k, ld = nf + (nf & 1);
      F.F_off = Fo;
      F.u_off = uo;
      Fo += (nf * ld + 31) & ~31LL;
      uo += (long long)F.b_n * k;
      if (top) {
        F.vtop_off = (int)vo;
        vo += nf;
        TH = std::max(TH, F.level + 1);
        P.n_top++;
      } else {
        H = std::max(H, F.level + 1);
      }
    }
    if (pass == 0) P.top_F = Fo;
  }
  // every rank's realisation stride is the same (its box fronts padded to the largest box's),
  // so that the interface fronts of every realisation sit at the same offsets on all ranks
  // (the in-process group all-reduces them through one offset)
  long long locmax = Fo - P.top_F;
  for (int q = 0; q < nranks && nranks > 1; ++q) {
    if (q == rank) continue;
    NdPlan Q;
    Builder bq{X, Y, k, Q, q, icol};
    bq.group(0, nranks, 0, X);
    long long lf = 0;
    for (const NdFront& F : Q.fr)
      if (!(F.flags & 1)) {
        const long long nf = (long long)(F.s_n + F.b_n) * k, ld = nf + (nf & 1);
        lf += (nf * ld + 31) & ~31LL;
      }
    locmax = std::max(locmax, lf);
  }
  P.F_total = P.top_F + locmax;
  P.u_total = uo;
  P.vtop_total = vo;
  P.H = H;
  P.TH = TH;
  // vmap: for every front variable its global coarse index, the absolute indices of the
  // children's update entries that add into it (-1: none; interface fronts: interface
  // children only) and, for interface fronts, its index in vtop (-1: box front)
  P.vmap.clear();
  P.packmap.assign(2 * vo, -1);
  for (NdFront& F : P.fr) {
    F.vmap_off = (int)(P.vmap.size() / 4);
    const bool top = F.flags & 1;
    const int nn = F.s_n + F.b_n;
    for (int j = 0; j < nn; ++j)
      for (int a = 0; a < k; ++a) {
        int u[2] = {-1, -1};
        const int chs[2] = {F.ch0, F.ch1};
        for (int q = 0; q < 2; ++q) {
          const int cp = chs[q] >= 0 ? P.chmap[F.chmap_off + 2 * j + q] : -1;
          if (cp < 0) continue;
          const int ui = (int)(P.fr[chs[q]].u_off + (long long)cp * k + a);
          const bool ctop = P.fr[chs[q]].flags & 1;
          if (!top || ctop) u[q] = ui;
          else P.packmap[2 * (F.vtop_off + j * k + a) + 1] = ui;   // the box root's update
        }
        const int g = P.nodes[F.node_off + j] * k + a;
        if (top && j < F.s_n) P.packmap[2 * (F.vtop_off + j * k + a)] = g;
        P.vmap.insert(P.vmap.end(), {g, u[0], u[1], top ? F.vtop_off + j * k + a : -1});
      }
  }
  std::vector<std::vector<int>> lev(H), tlev(TH), tall;
  tall.resize(1);
  for (int f = 0; f < (int)P.fr.size(); ++f) {
    if (P.fr[f].flags & 1) {
      tlev[P.fr[f].level].push_back(f);
      tall[0].push_back(f);
    } else {
      lev[P.fr[f].level].push_back(f);
    }
  }
  P.max_act = 1;
  P.scr_doubles = NB;
  level_lists(P, k, lev, P.loc);
  level_lists(P, k, tlev, P.top);
  auto nt = [k](const NdFront& F) { return (long long)((F.s_n + F.b_n) * k + NB - 1) / NB; };
  P.tpart = add_list(P, tall[0], [&](const NdFront& F) { return nt(F) * nt(F); });
  P.max_nf = 0;
  for (const NdFront& F : P.fr) P.max_nf = std::max(P.max_nf, (F.s_n + F.b_n) * k);
  // bytes streamed per solve and realisation (forward B x S blocks, back S rows)
  P.solve_bytes = 0;
  for (const NdFront& F : P.fr) {
    const long long s = (long long)F.s_n * k, nf = (long long)(F.s_n + F.b_n) * k;
    P.solve_bytes += 8 * ((nf - s) * s + s * nf);
  }
  return true;
}

size_t nd_workspace_bytes(const Dims& d, const NdPlan& P) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t R = d.R;
  return al(R * P.F_total * 8) + al(R * P.u_total * 8) + al(2 * R * (size_t)P.max_act * NB * NB * 8) +
         2 * al(R * (size_t)P.scr_doubles * 8) + al(P.fr.size() * sizeof(NdFront)) +
         al(P.nodes.size() * 4) + al(P.chmap.size() * 4) + al(P.lists.size() * 4) + al(P.vmap.size() * 4) +
         al(P.packmap.size() * 4) + al(R * (size_t)std::max<long long>(1, P.vtop_total) * 8);
}

// carve + upload (called at setup)
cudaError_t nd_setup(msf_ctx* c, char*& cur) {
  auto take = [&](size_t bytes) {
    char* r = cur;
    cur += (bytes + 255) & ~(size_t)255;
    return (void*)r;
  };
  const NdPlan& P = c->nd;
  const size_t R = c->d.R;
  c->nd_F = (double*)take(R * P.F_total * 8);
  c->nd_u = (double*)take(R * P.u_total * 8);
  c->nd_Q = (double*)take(2 * R * (size_t)P.max_act * NB * NB * 8);   // Q, then L
  c->nd_Ar = (double*)take(R * (size_t)P.scr_doubles * 8);
  c->nd_Rp = (double*)take(R * (size_t)P.scr_doubles * 8);
  c->nd_fr = (NdFront*)take(P.fr.size() * sizeof(NdFront));
  c->nd_nodes = (int*)take(P.nodes.size() * 4);
  c->nd_chmap = (int*)take(P.chmap.size() * 4);
  c->nd_lists = (int*)take(P.lists.size() * 4);
  c->nd_vmap = (int*)take(P.vmap.size() * 4);
  c->nd_pack = (int*)take(P.packmap.size() * 4);
  c->nd_vtop = (double*)take(R * (size_t)std::max<long long>(1, P.vtop_total) * 8);
  cudaError_t e = cudaMemcpyAsync(c->nd_fr, P.fr.data(), P.fr.size() * sizeof(NdFront), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->nd_nodes, P.nodes.data(), P.nodes.size() * 4, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->nd_chmap, P.chmap.data(), P.chmap.size() * 4, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->nd_lists, P.lists.data(), P.lists.size() * 4, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->nd_vmap, P.vmap.data(), P.vmap.size() * 4, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess && !P.packmap.empty())
    e = cudaMemcpyAsync(c->nd_pack, P.packmap.data(), P.packmap.size() * 4, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->nd_u, 0, R * P.u_total * 8, c->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->nd_vtop, 0, R * (size_t)std::max<long long>(1, P.vtop_total) * 8, c->stream);
  return e;
}

namespace {

void factor_levels(msf_ctx* c, const NdPlan::Levels& Lv, int mode) {
  const NdPlan& P = c->nd;
  const Dims& d = c->d;
  const int R = d.R;
  static bool attrs = false;
  if (!attrs) {
    cudaFuncSetAttribute(k_nd_trailing, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB * SPAD * 8);
    cudaFuncSetAttribute(k_nd_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB * (NB + 1) * 8);
    cudaFuncSetAttribute(k_nd_rowpanel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB * (NB + 1) * 8);
    attrs = true;
  }
  const long long Fs = P.F_total;
  for (size_t h = 0; h < Lv.asmb.size(); ++h) {
    const NdPlan::List& A = Lv.asmb[h];
    if (A.total == 0) continue;
    k_nd_assemble<<<dim3(A.total, R), 256, 0, c->stream>>>(
        d, c->nd_fr, c->nd_nodes, c->nd_chmap, c->nd_lists + A.off, A.n, c->Kcell, c->cls_of_agg_d,
        c->classes_d, c->nd_F, Fs, c->cell_lo, c->cell_hi, mode);
    MSF_LAUNCHED(c);
    for (size_t pt = 0; pt < Lv.panel[h].size(); ++pt) {
      const NdPlan::List& L = Lv.panel[h][pt];
      PanelArgs pa{c->nd_lists + L.off, L.n, (int)pt, c->nd_Q, c->nd_Q + (size_t)R * P.max_act * NB * NB,
                   c->nd_Ar, c->nd_Rp, (long long)P.max_act * NB * NB, P.scr_doubles};
      k_nd_pivot<<<dim3(L.n, R), 256, 2 * NB * (NB + 1) * 8, c->stream>>>(d, c->nd_fr, c->nd_F, Fs, pa, c->factor_status);
      k_nd_rowpanel<<<dim3(L.total, R), NB, 2 * NB * (NB + 1) * 8, c->stream>>>(d, c->nd_fr, c->nd_F, Fs, pa);
      k_nd_trailing<<<dim3(L.total2, R), 256, 2 * NB * SPAD * 8, c->stream>>>(d, c->nd_fr, c->nd_F, Fs, pa);
      k_nd_panels<<<dim3(L.total, R), 256, 0, c->stream>>>(d, c->nd_fr, c->nd_F, Fs, pa);
      c->launches += 4;
    }
  }
}

void solve_levels(msf_ctx* c, const NdPlan::Levels& Lv, bool fwd, int rhs0, int nr, bool gated) {
  const NdPlan& P = c->nd;
  const Dims& d = c->d;
  static bool smem_set = false;
  if (!smem_set) {
    cudaFuncSetAttribute(k_nd_solve<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_nd_solve<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_nd_solve<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_nd_solve<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    smem_set = true;
  }
  const int H = (int)Lv.fwd.size();
  for (int i = 0; i < H; ++i) {
    const int h = fwd ? i : H - 1 - i;
    const NdPlan::List& L = fwd ? Lv.fwd[h] : Lv.back[h];
    if (L.total == 0) continue;
    const size_t smem = (size_t)(fwd ? Lv.fwd_smem[h] : Lv.back_smem[h]);
    auto kern = L.NS > 1 ? (fwd ? k_nd_solve<true, true> : k_nd_solve<false, true>)
                         : (fwd ? k_nd_solve<true, false> : k_nd_solve<false, false>);
    launch_k(kern, dim3(L.total, nr), dim3(256), smem, c->stream, d, (const NdFront*)c->nd_fr,
             (const int4*)c->nd_vmap, (const int*)(c->nd_lists + L.off), L.n, L.RB, L.NS, (const double*)c->nd_F,
             (long long)P.F_total, c->nd_u, (long long)P.u_total, (const double*)c->cb, c->cx,
             (const double*)c->nd_vtop, (long long)std::max<long long>(1, P.vtop_total),
             (const PcgScalars*)c->sc, rhs0, gated ? 1 : 0);
    MSF_LAUNCHED(c);
  }
}

}  // namespace

// K_c factorisation, box part: this rank's fronts level by level (leaves first), then its
// partial sums of the interface fronts (cell entries of its cells, its box root's Schur
// complement) -- all-reduced over the ranks before launch_nd_factor_top.  All realisations.
void launch_nd_factor_local(msf_ctx* c) {
  factor_levels(c, c->nd.loc, 0);
  const NdPlan::List& T = c->nd.tpart;
  if (T.total > 0) {
    k_nd_assemble<<<dim3(T.total, c->d.R), 256, 0, c->stream>>>(
        c->d, c->nd_fr, c->nd_nodes, c->nd_chmap, c->nd_lists + T.off, T.n, c->Kcell, c->cls_of_agg_d,
        c->classes_d, c->nd_F, c->nd.F_total, c->cell_lo, c->cell_hi, 1);
    MSF_LAUNCHED(c);
  }
}

// interface fronts (replicated): identity rows + interface children, then the sweep
void launch_nd_factor_top(msf_ctx* c) { factor_levels(c, c->nd.top, 2); }

void launch_nd_factor(msf_ctx* c) {
  launch_nd_factor_local(c);
  launch_nd_factor_top(c);
}

// Coarse solve phases for realisations [rhs0, rhs0 + nr): forward over the box fronts (+ the
// interface partial right-hand sides, all-reduced by the caller on a strip partition),
// forward + back over the interface fronts, back over the box fronts.  cb is read, cx written.
void launch_nd_solve_local_fwd(msf_ctx* c, int rhs0, int nr, bool gated) {
  solve_levels(c, c->nd.loc, true, rhs0, nr, gated);
  const long long n = c->nd.vtop_total;
  if (n > 0) {
    launch_k(k_nd_pack, dim3((unsigned)((n + 255) / 256), nr), dim3(256), 0, c->stream, (const int2*)c->nd_pack,
             (int)n, (const double*)c->cb, (long long)c->d.nbc * c->d.mc, (const double*)c->nd_u,
             (long long)c->nd.u_total, c->nd_vtop, (long long)n, (const PcgScalars*)c->sc, rhs0, gated ? 1 : 0);
    MSF_LAUNCHED(c);
  }
}

void launch_nd_solve_top(msf_ctx* c, int rhs0, int nr, bool gated) {
  solve_levels(c, c->nd.top, true, rhs0, nr, gated);
  solve_levels(c, c->nd.top, false, rhs0, nr, gated);
}

void launch_nd_solve_local_back(msf_ctx* c, int rhs0, int nr, bool gated) {
  solve_levels(c, c->nd.loc, false, rhs0, nr, gated);
}

void launch_nd_solve(msf_ctx* c, int rhs0, int nr, bool gated) {
  launch_nd_solve_local_fwd(c, rhs0, nr, gated);
  launch_nd_solve_top(c, rhs0, nr, gated);
  launch_nd_solve_local_back(c, rhs0, nr, gated);
}
