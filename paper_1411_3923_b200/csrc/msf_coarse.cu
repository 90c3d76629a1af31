// Coarse space of the two-level preconditioner (§2.4, Eq. 10, §2.4.2
// line 146):
//   * restriction c = R_c t and prolongation z += R_c^T c with R_c^T = [phi_1 ... phi_Nt],
//     phi_{i,a} = chi_i psi_a^{omega_i} stored per agglomerate class on a padded
//     (2cx+1)x(2cy+1)-node box (periodic classes share storage, §2.4.1);
//   * Galerkin K_c = R_c K R_c^T per realisation, assembled from per-coarse-cell dense
//     (4k x 4k) products Phi_C^T K_C Phi_C (the dense contraction of the path);
//   * K_c is block tridiagonal over coarse-node columns (block size m = (ncy+1) k);
//     exact coarse solve by block cyclic reduction: per level the odd blocks are
//     eliminated with explicit SPD inverses (batched sweep operator) and batched GEMMs,
//     so every level is parallel across blocks and realisations.
#include <array>
#include <map>
#include <cublas_v2.h>

#include "msf_kern.cuh"

#include <algorithm>
#include <cmath>

using namespace msfk;

namespace {

constexpr int NT = 256;

// ------------------------------------------------------------------ per-realisation restriction
// One CTA per (agglomerate, realisation): the cost follows the number of ACTIVE realisations
// (most PCG iterations run the slowest-converging realisation alone).  Agglomerates in
// class order (consecutive CTAs share the class basis in L2).
template <int KM, int NTR>
__global__ void __launch_bounds__(NTR) k_restrict1(Dims d, const double2* __restrict__ tall,
                                                  const double* __restrict__ phi,
                                                  const int* __restrict__ cls_of_agg,
                                                  const int* __restrict__ agg_by_cls,
                                                  double* cball, const PcgScalars* sc, int rhs0,
                                                  int gated) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.y;
  if (gated && !sc[rhs].active) return;
  __shared__ double red[NTR / 32][KM];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int agg = agg_by_cls[blockIdx.x];
  const int I = agg / (d.ncy + 1), J = agg - (agg / (d.ncy + 1)) * (d.ncy + 1);
  const double* ph = phi + (size_t)cls_of_agg[agg] * d.kmax * d.box_nodes * 2;
  const double2* t = tall + (size_t)rhs * d.nn;
  const int gx0 = I * d.cx - d.cx - d.gox, gy0 = J * d.cy - d.cy;
  // interior of the padded box (chi vanishes on its boundary ring), clipped to the strip
  const int ix_lo = max(1, -gx0), ix_hi = min(d.bx - 2, d.nnx - 1 - gx0);
  const int iy_lo = max(1, -gy0), iy_hi = min(d.by - 2, d.nny - 1 - gy0);
  const int w = iy_hi - iy_lo + 1, h = ix_hi - ix_lo + 1;
  double acc[KM];
#pragma unroll
  for (int a = 0; a < KM; ++a) acc[a] = 0.0;
  for (int k = tid; k < w * h; k += NTR) {
    const int px = ix_lo + k / w, py = iy_lo + (k - (k / w) * w);
    const double2 tv = t[(size_t)(gx0 + px) * d.nny + (gy0 + py)];
    const int bn = px * d.by + py;
#pragma unroll
    for (int a = 0; a < KM; ++a) {
      if (a < d.kmax) {
        const double2 pv = __ldg(reinterpret_cast<const double2*>(ph + ((size_t)a * d.box_nodes + bn) * 2));
        acc[a] = fma(pv.x, tv.x, fma(pv.y, tv.y, acc[a]));
      }
    }
  }
#pragma unroll
  for (int a = 0; a < KM; ++a) {
    if (a < d.kmax) {
      const double v = warp_sum(acc[a]);
      if (lane == 0) red[wid][a] = v;
    }
  }
  __syncthreads();
  if (tid < d.kmax) {
    double s2 = 0.0;
    for (int w2 = 0; w2 < NTR / 32; ++w2) s2 += red[w2][tid];
    cball[(size_t)rhs * d.nbc * d.mc + (size_t)agg * d.kmax + tid] = s2;
  }
}

// One WARP per (agglomerate, realisation): lanes stride the agglomerate's clipped box (y
// fastest, the position stepped incrementally), the KM sums are reduced by shuffles only (no
// shared memory, no block barrier), 8 agglomerates per CTA.  (One 256-thread CTA per
// agglomerate spent its time in CTA turnover and block reductions: ~4 loop passes per CTA.)
template <int KM>
__global__ void __launch_bounds__(256) k_restrict_warp(Dims d, const double2* __restrict__ tall,
                                                       const double* __restrict__ phi,
                                                       const int* __restrict__ cls_of_agg,
                                                       const int* __restrict__ agg_list, int n_agg,
                                                       double* cball, const PcgScalars* sc, int rhs0,
                                                       int gated) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.y;
  if (gated && !sc[rhs].active) return;
  const int lane = threadIdx.x & 31;
  const int slot = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (slot >= n_agg) return;
  const int agg = agg_list[slot];
  const int I = agg / (d.ncy + 1), J = agg - (agg / (d.ncy + 1)) * (d.ncy + 1);
  const double2* ph = reinterpret_cast<const double2*>(phi) + (size_t)cls_of_agg[agg] * d.kmax * d.box_nodes;
  const double2* t = tall + (size_t)rhs * d.nn;
  const int gx0 = I * d.cx - d.cx - d.gox, gy0 = J * d.cy - d.cy;
  // interior of the padded box (chi vanishes on its boundary ring), clipped to the strip
  const int ix_lo = max(1, -gx0), ix_hi = min(d.bx - 2, d.nnx - 1 - gx0);
  const int iy_lo = max(1, -gy0), iy_hi = min(d.by - 2, d.nny - 1 - gy0);
  const int w = iy_hi - iy_lo + 1, h = ix_hi - ix_lo + 1;
  double acc[KM];
#pragma unroll
  for (int a = 0; a < KM; ++a) acc[a] = 0.0;
  // position of element k = lane + 32 i of the w-by-h box, stepped without divisions
  int px = lane / w, py = lane - (lane / w) * w;
  const int step_x = 32 / w, step_y = 32 - (32 / w) * w;
  const int n = w * h;
#pragma unroll 4
  for (int k = lane; k < n; k += 32) {
    const int bx = ix_lo + px, by = iy_lo + py;
    const double2 tv = t[(size_t)(gx0 + bx) * d.nny + (gy0 + by)];
    const int bn = bx * d.by + by;
#pragma unroll
    for (int a = 0; a < KM; ++a) {
      if (a < d.kmax) {
        const double2 pv = __ldg(ph + (size_t)a * d.box_nodes + bn);
        acc[a] = fma(pv.x, tv.x, fma(pv.y, tv.y, acc[a]));
      }
    }
    px += step_x;
    py += step_y;
    if (py >= w) {
      py -= w;
      ++px;
    }
  }
#pragma unroll
  for (int a = 0; a < KM; ++a) {
    if (a < d.kmax) {
      double v = acc[a];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == a) cball[(size_t)rhs * d.nbc * d.mc + (size_t)agg * d.kmax + a] = v;
    }
  }
}

// One WARP per group of B agglomerates of the same class and the same clipped box (host:
// restrict_groups).  The members share the basis, so each lane loads phi_a(node) once and
// applies it to the B members' t at the same box position: the class-basis traffic through
// L2/L1, which bounds k_restrict_warp (64 B per node, mode and agglomerate against 16 B of
// t), falls by B.  Same per-agglomerate sums and summation order as k_restrict_warp.
#ifndef MSF_RB_MINB
#define MSF_RB_MINB 2
#endif
#ifndef MSF_RB_UNROLL
#define MSF_RB_UNROLL 1
#endif
constexpr int RB_UNROLL = MSF_RB_UNROLL;
template <int KM, int B>
__global__ void __launch_bounds__(256, MSF_RB_MINB) k_restrict_batch(Dims d, const double2* __restrict__ tall,
                                                        const double* __restrict__ phi,
                                                        const int* __restrict__ cls_of_agg,
                                                        const int* __restrict__ groups, int n_groups,
                                                        double* cball, const PcgScalars* sc, int rhs0,
                                                        int gated) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.y;
  if (gated && !sc[rhs].active) return;
  const int lane = threadIdx.x & 31;
  const int slot = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (slot >= n_groups) return;
  int agg[B];
#pragma unroll
  for (int b = 0; b < B; ++b) agg[b] = __ldg(groups + (size_t)slot * B + b);
  const int a0 = agg[0];
  const int I = a0 / (d.ncy + 1), J = a0 - (a0 / (d.ncy + 1)) * (d.ncy + 1);
  const double2* ph = reinterpret_cast<const double2*>(phi) + (size_t)cls_of_agg[a0] * d.kmax * d.box_nodes;
  const double2* t = tall + (size_t)rhs * d.nn;
  const int gx0 = I * d.cx - d.cx - d.gox, gy0 = J * d.cy - d.cy;
  const int ix_lo = max(1, -gx0), ix_hi = min(d.bx - 2, d.nnx - 1 - gx0);
  const int iy_lo = max(1, -gy0), iy_hi = min(d.by - 2, d.nny - 1 - gy0);
  const int w = iy_hi - iy_lo + 1, h = ix_hi - ix_lo + 1;
  long long toff[B];   // t offset of each member's box origin (padding slots repeat member 0)
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int ab = agg[b] >= 0 ? agg[b] : a0;
    const int Ib = ab / (d.ncy + 1), Jb = ab - (ab / (d.ncy + 1)) * (d.ncy + 1);
    toff[b] = (long long)(Ib * d.cx - d.cx - d.gox) * d.nny + (Jb * d.cy - d.cy);
  }
  double acc[B][KM];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int a = 0; a < KM; ++a) acc[b][a] = 0.0;
  int px = lane / w, py = lane - (lane / w) * w;
  const int step_x = 32 / w, step_y = 32 - (32 / w) * w;
  const int n = w * h;
#pragma unroll RB_UNROLL
  for (int k = lane; k < n; k += 32) {
    const int bx = ix_lo + px, by = iy_lo + py;
    const int bn = bx * d.by + by;
    double2 pv[KM];
#pragma unroll
    for (int a = 0; a < KM; ++a)
      pv[a] = a < d.kmax ? __ldg(ph + (size_t)a * d.box_nodes + bn) : make_double2(0.0, 0.0);
    const long long rel = (long long)bx * d.nny + by;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const double2 tv = t[toff[b] + rel];
#pragma unroll
      for (int a = 0; a < KM; ++a)
        if (a < d.kmax) acc[b][a] = fma(pv[a].x, tv.x, fma(pv[a].y, tv.y, acc[b][a]));
    }
    px += step_x;
    py += step_y;
    if (py >= w) {
      py -= w;
      ++px;
    }
  }
  double* cb = cball + (size_t)rhs * d.nbc * d.mc;
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int a = 0; a < KM; ++a) {
      if (a < d.kmax) {
        double v = acc[b][a];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == ((b * KM + a) & 31) && agg[b] >= 0) cb[(size_t)agg[b] * d.kmax + a] = v;
      }
    }
}

// ------------------------------------------------------------------ per-realisation prolongation
// z(n) += sum_{I,J,a} phi_{I,J,a}(n) x_c[slot(I,J,a)], one (node, realisation) per thread.
template <int KM>
__global__ void __launch_bounds__(NT) k_prolong1(Dims d, const double* __restrict__ phi,
                                                 const int* __restrict__ cls_of_agg,
                                                 const double* __restrict__ cxall, double2* zall,
                                                 const PcgScalars* sc, int rhs0, int gated) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.z;
  if (gated && !sc[rhs].active) return;
  const int iy = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ix = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (ix >= d.nnx || iy >= d.nny) return;
  const double* xc = cxall + (size_t)rhs * d.nbc * d.mc;
  const int gix = ix + d.gox;
  const int I0 = gix / d.cx, J0 = iy / d.cy;
  double sx = 0.0, sy = 0.0;
#pragma unroll
  for (int di = 0; di < 2; ++di) {
    const int I = I0 + di;
    const int px = gix - (I * d.cx - d.cx);
    if (I > d.ncx || px >= d.bx) continue;
#pragma unroll
    for (int dj = 0; dj < 2; ++dj) {
      const int J = J0 + dj;
      const int py = iy - (J * d.cy - d.cy);
      if (J > d.ncy || py >= d.by) continue;
      const int agg = I * (d.ncy + 1) + J;
      const double* ph = phi + (size_t)cls_of_agg[agg] * d.kmax * d.box_nodes * 2 + (size_t)(px * d.by + py) * 2;
#pragma unroll
      for (int a = 0; a < KM; ++a) {
        if (a < d.kmax) {
          const double2 pv = __ldg(reinterpret_cast<const double2*>(ph + (size_t)a * d.box_nodes * 2));
          const double cv = __ldg(xc + (size_t)agg * d.kmax + a);
          sx = fma(pv.x, cv, sx);
          sy = fma(pv.y, cv, sy);
        }
      }
    }
  }
  double2* z = zall + (size_t)rhs * d.nn + (size_t)ix * d.nny + iy;
  double2 zv = *z;
  zv.x += sx;
  zv.y += sy;
  *z = zv;
}

// Prolongation for NR > 1 active realisations, one node per thread for all of them: the
// realisations share the coarse basis, so phi is loaded once per (covering
// agglomerate, mode) and applied to each realisation's coefficients (k_prolong1 loads it
// once per realisation).  Per realisation the sum runs in k_prolong1's order: z is bitwise
// the same.
template <int KM, int NR>
__global__ void __launch_bounds__(NT) k_prolong_nr(Dims d, const double* __restrict__ phi,
                                                   const int* __restrict__ cls_of_agg,
                                                   const double* __restrict__ cxall, double2* zall,
                                                   const PcgScalars* sc, int rhs0, int gated) {
  pdl_launch();
  pdl_wait();
  bool act[NR];
  bool any = false;
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    act[k] = !gated || sc[rhs0 + k].active;
    any |= act[k];
  }
  if (!any) return;
  const int iy = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ix = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (ix >= d.nnx || iy >= d.nny) return;
  const size_t cstride = (size_t)d.nbc * d.mc;
  const double* xc = cxall + (size_t)rhs0 * cstride;
  const int gix = ix + d.gox;
  const int I0 = gix / d.cx, J0 = iy / d.cy;
  double sx[NR], sy[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) sx[k] = sy[k] = 0.0;
#pragma unroll
  for (int di = 0; di < 2; ++di) {
    const int I = I0 + di;
    const int px = gix - (I * d.cx - d.cx);
    if (I > d.ncx || px >= d.bx) continue;
#pragma unroll
    for (int dj = 0; dj < 2; ++dj) {
      const int J = J0 + dj;
      const int py = iy - (J * d.cy - d.cy);
      if (J > d.ncy || py >= d.by) continue;
      const int agg = I * (d.ncy + 1) + J;
      const double* ph = phi + (size_t)cls_of_agg[agg] * d.kmax * d.box_nodes * 2 + (size_t)(px * d.by + py) * 2;
#pragma unroll
      for (int a = 0; a < KM; ++a) {
        if (a < d.kmax) {
          const double2 pv = __ldg(reinterpret_cast<const double2*>(ph + (size_t)a * d.box_nodes * 2));
#pragma unroll
          for (int k = 0; k < NR; ++k) {
            const double cv = __ldg(xc + k * cstride + (size_t)agg * d.kmax + a);
            sx[k] = fma(pv.x, cv, sx[k]);
            sy[k] = fma(pv.y, cv, sy[k]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    if (!act[k]) continue;
    double2* z = zall + (size_t)(rhs0 + k) * d.nn + (size_t)ix * d.nny + iy;
    double2 zv = *z;
    zv.x += sx[k];
    zv.y += sy[k];
    *z = zv;
  }
}

// ------------------------------------------------------------------ Galerkin cell products
// Kcell[rhs][cell][p][q] = sum_{e in cell} E_e Phi_e[:,p]^T K0 Phi_e[:,q],  p,q in 0..4k-1,
// p = corner*k + a, corner = ci*2 + cj for coarse node (CI+ci, CJ+cj).  The (4k)x(4k) output
// is computed in CH x CH chunks (blockIdx.z = chunk pair) so the staged cell bases fit in
// shared memory for any mode count; with a single chunk Phi_p and Phi_q coincide.
__device__ __forceinline__ void stage_cell_cols(const Dims& d, const double* __restrict__ phi,
                                                const int* __restrict__ cls_of_agg, int CI, int CJ,
                                                int c0, int cw, int CH, double* S) {
  const int km = d.kmax, ncn_y = d.cy + 1, ncn = (d.cx + 1) * (d.cy + 1);
  for (int k = threadIdx.x; k < ncn * 2 * CH; k += NT) {
    const int j = k % CH, nc = k / CH;          // column j, node*2 + comp
    if (j >= cw) continue;
    const int comp = nc & 1, node = nc >> 1;
    const int lx = node / ncn_y, ly = node - (node / ncn_y) * ncn_y;
    const int p = c0 + j;
    const int corner = p / km, a = p - (p / km) * km;
    const int I = CI + (corner >> 1), J = CJ + (corner & 1);
    const int px = CI * d.cx + lx - (I * d.cx - d.cx), py = CJ * d.cy + ly - (J * d.cy - d.cy);
    const int agg = I * (d.ncy + 1) + J;
    S[k] = phi[(((size_t)cls_of_agg[agg] * d.kmax + a) * d.box_nodes + px * d.by + py) * 2 + comp];
  }
}

__global__ void __launch_bounds__(NT) k_cell_galerkin(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                      const double* __restrict__ phi,
                                                      const int* __restrict__ cls_of_agg,
                                                      double* Kcell, int CH, int cell0) {
  extern __shared__ double sm[];
  // all realisations in one CTA: V_e = K0 Phi_e and Phi_e^T V_e do not depend on the
  // realisation, only the scalar modulus E_e does (R accumulators per output entry)
  const int cell = cell0 + blockIdx.x;
  const int CI = cell / d.ncy, CJ = cell - (cell / d.ncy) * d.ncy;
  const int P = 4 * d.kmax;
  const int nch = (P + CH - 1) / CH;
  const int pc = blockIdx.z / nch, qc = blockIdx.z - pc * nch;
  const int p0 = pc * CH, q0 = qc * CH, pw = min(CH, P - p0), qw = min(CH, P - q0);
  const int ncn_y = d.cy + 1, ncn = (d.cx + 1) * (d.cy + 1);
  const bool single = nch == 1;
  double* PhiP = sm;                                       // [ncn][2][CH]
  double* PhiQ = single ? PhiP : PhiP + (size_t)ncn * 2 * CH;
  double* V = PhiQ + (size_t)ncn * 2 * CH;                 // [16][8][CH]
  double* Ech = V + 16 * 8 * CH;                           // [MSF_MAX_RHS][16]
  stage_cell_cols(d, phi, cls_of_agg, CI, CJ, p0, pw, CH, PhiP);
  if (!single) stage_cell_cols(d, phi, cls_of_agg, CI, CJ, q0, qw, CH, PhiQ);
  const int R = d.R;
  const int nel = d.cx * d.cy;
  const int nent = CH * CH;   // <= NT
  double acc[MSF_MAX_RHS] = {0.0, 0.0, 0.0, 0.0};
  __syncthreads();
  for (int e0 = 0; e0 < nel; e0 += 16) {
    const int ne = min(16, nel - e0);
    // V_e = K0 Phi_e[:, q-chunk] for the element chunk
    for (int k = threadIdx.x; k < ne * 8 * CH; k += NT) {
      const int q = k % CH, rest = k / CH;
      const int i = rest & 7, el = rest >> 3;
      if (q >= qw) continue;
      const int le = e0 + el;
      const int lex = le / d.cy, ley = le - (le / d.cy) * d.cy;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int b = j >> 1, comp = j & 1;
        const int nx = lex + ((b == 1 || b == 2) ? 1 : 0), ny = ley + ((b >= 2) ? 1 : 0);
        s = fma(K.v[i * 8 + j], PhiQ[((nx * ncn_y + ny) * 2 + comp) * CH + q], s);
      }
      V[(el * 8 + i) * CH + q] = s;
    }
    for (int k = threadIdx.x; k < ne * R; k += NT) {
      const int r = k / ne, el = k - r * ne;
      const int le = e0 + el;
      const int lex = le / d.cy, ley = le - (le / d.cy) * d.cy;
      Ech[r * 16 + el] = Eall[(size_t)r * d.ne + (size_t)(CI * d.cx + lex) * d.nely + CJ * d.cy + ley];
    }
    __syncthreads();
    const int ent = threadIdx.x;
    if (ent < nent) {
      const int p = ent / CH, q = ent - (ent / CH) * CH;
      if (p < pw && q < qw) {
        for (int el = 0; el < ne; ++el) {
          const int le = e0 + el;
          const int lex = le / d.cy, ley = le - (le / d.cy) * d.cy;
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int b = i >> 1, comp = i & 1;
            const int nx = lex + ((b == 1 || b == 2) ? 1 : 0), ny = ley + ((b >= 2) ? 1 : 0);
            t = fma(PhiP[((nx * ncn_y + ny) * 2 + comp) * CH + p], V[(el * 8 + i) * CH + q], t);
          }
#pragma unroll
          for (int r = 0; r < MSF_MAX_RHS; ++r)
            if (r < R) acc[r] = fma(Ech[r * 16 + el], t, acc[r]);
        }
      }
    }
    __syncthreads();
  }
  const int ent = threadIdx.x;
  if (ent < nent) {
    const int p = ent / CH, q = ent - (ent / CH) * CH;
    if (p < pw && q < qw)
#pragma unroll
      for (int r = 0; r < MSF_MAX_RHS; ++r)
        if (r < R) Kcell[((size_t)r * d.ncx * d.ncy + cell) * P * P + (size_t)(p0 + p) * P + (q0 + q)] = acc[r];
  }
}

// Galerkin products as one GEMM per cell (the same sum, re-associated): with K0 = L^T L
// (L = Lambda^1/2 Q^T over the 5 nonzero eigenpairs of the element matrix, host),
//   Kcell = sum_e E_e Phi_e^T K0 Phi_e = G^T G,   G = [sqrt(E_e) L Phi_e]_e   ((5 nel) x P),
// G built here (columns in chunks of CH staged like k_cell_galerkin), G^T G by cuBLAS strided
// batched DGEMM over the cells of a chunk.  (k_cell_galerkin: 3-5% of the FP64 peak on
// configs[3] / [4], 232 / 41 ms.)
struct LMat {
  double v[5 * 8];
};
__global__ void __launch_bounds__(NT) k_galerkin_G(Dims d, LMat L, const double* __restrict__ Eall,
                                                   const double* __restrict__ phi,
                                                   const int* __restrict__ cls_of_agg, int rhs,
                                                   int cell0, int CH, double* G) {
  extern __shared__ double gsm[];   // [ncn * 2][CH]
  const int cell = cell0 + blockIdx.x;
  const int CI = cell / d.ncy, CJ = cell - (cell / d.ncy) * d.ncy;
  const int P = 4 * d.kmax, p0 = blockIdx.z * CH, pw = min(CH, P - p0);
  const int ncn_y = d.cy + 1, nel = d.cx * d.cy;
  stage_cell_cols(d, phi, cls_of_agg, CI, CJ, p0, pw, CH, gsm);
  __syncthreads();
  double* Gc = G + (size_t)blockIdx.x * 5 * nel * P;
  const double* E = Eall + (size_t)rhs * d.ne;
  for (int k = threadIdx.x; k < nel * CH; k += NT) {
    const int el = k / CH, q = k - (k / CH) * CH;
    if (q >= pw) continue;
    const int lex = el / d.cy, ley = el - (el / d.cy) * d.cy;
    const double se = sqrt(E[(size_t)(CI * d.cx + lex) * d.nely + CJ * d.cy + ley]);
    double ph[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int b = i >> 1, comp = i & 1;
      const int nx = lex + ((b == 1 || b == 2) ? 1 : 0), ny = ley + ((b >= 2) ? 1 : 0);
      ph[i] = gsm[((nx * ncn_y + ny) * 2 + comp) * CH + q];
    }
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) t = fma(L.v[l * 8 + i], ph[i], t);
      Gc[((size_t)el * 5 + l) * P + p0 + q] = se * t;
    }
  }
}

// Gather the cell products into the block-tridiagonal K_c (D_I, U_I = K_c[I, I+1]) for
// the blocks D_I, I in [dlo, dlo + nD), and U_I, I in [ulo, ulo + nU), from the coarse cell
// columns [ulo, ulo + nU) (a strip: its own cells, so its chain's end blocks get partial
// sums); unused eigen-slots (a >= nkept) carry identity rows in D_I for I in [idlo, idhi]
// (each block's identity added by one rank).
__global__ void k_coarse_gather(Dims d, const double* __restrict__ Kcell,
                                const int* __restrict__ cls_of_agg,
                                const EigClass* __restrict__ cls, double* Dall, double* Uall,
                                int dlo, int nD, int ulo, int nU, int idlo, int idhi, int slot0,
                                int nslot) {
  const int km = d.kmax, P = 4 * km, m = d.mc;
  const size_t per = (size_t)m * m;
  const size_t total = (size_t)(nD + nU) * per;
  const int rhs = blockIdx.y;
  const double* Kc = Kcell + (size_t)rhs * d.ncx * d.ncy * P * P;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int isU = idx >= (size_t)nD * per;
    const size_t li = isU ? idx - (size_t)nD * per : idx;
    const int I = (int)(li / per) + (isU ? ulo : dlo);
    const int e = (int)(li - (size_t)(I - (isU ? ulo : dlo)) * per);
    const int row = e / m, col = e - (e / m) * m;
    const int J = row / km, a = row - (row / km) * km;
    const int Jp = col / km, b = col - (col / km) * km;
    double v = 0.0;
    const int Ir = I, Ic = isU ? I + 1 : I;
    const int nka = cls[cls_of_agg[Ir * (d.ncy + 1) + J]].nkept;
    const int nkb = cls[cls_of_agg[Ic * (d.ncy + 1) + Jp]].nkept;
    if (a >= nka || b >= nkb) {
      v = (!isU && row == col && I >= idlo && I <= idhi) ? 1.0 : 0.0;
    } else if (abs(J - Jp) <= 1) {
      const int CIlo = isU ? I : max(I - 1, ulo), CIhi = isU ? I : min(I, ulo + nU - 1);
      const int CJlo = max(max(J, Jp) - 1, 0), CJhi = min(min(J, Jp), d.ncy - 1);
      for (int CI = CIlo; CI <= CIhi; ++CI)
        for (int CJ = CJlo; CJ <= CJhi; ++CJ) {
          const int pr = ((Ir - CI) * 2 + (J - CJ)) * km + a;
          const int pc = ((Ic - CI) * 2 + (Jp - CJ)) * km + b;
          v += Kc[((size_t)CI * d.ncy + CJ) * P * P + (size_t)pr * P + pc];
        }
    }
    double* dst = (isU ? Uall : Dall) + ((size_t)rhs * nslot + (I - slot0)) * per;   // chain slots
    dst[e] = v;
  }
}

// Strip partition: this rank's share of the interface entries of the coarse vector
// (pack: comp = b of interface blocks a, b (its chain ends), 0 elsewhere) or the all-reduced
// interface rhs written back (unpack), realisations [rhs0, rhs0 + gridDim.y).
__global__ void k_iface_vec(Dims d, const int* __restrict__ iface, int nI, int a, int b,
                            double* cball, double* comp, int rhs0, int unpack) {
  const int rhs = rhs0 + blockIdx.y;
  const size_t n = (size_t)nI * d.mc;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx / d.mc), row = (int)(idx - (size_t)j * d.mc);
    double* cbp = cball + ((size_t)rhs * d.nbc + iface[j]) * d.mc + row;
    double* cp = comp + (size_t)rhs * n + idx;
    if (unpack) *cbp = *cp;
    else *cp = (j == a || j == b) ? *cbp : 0.0;
  }
}

// ------------------------------------------------------------------ dense batched kernels
// In-place inverse of SPD blocks by the sweep operator (all pivots), then negation:
// sweep(k): a_kk <- -1/a_kk, a_ik <- a_ik/a_kk, a_kj <- a_kj/a_kk, a_ij <- a_ij - a_ik a_kj/a_kk
__global__ void __launch_bounds__(1024) k_spd_inverse(double** mats, int m, int* status) {
  extern __shared__ double sm[];
  double* rowk = sm;           // [m]
  double* colk = sm + m;       // [m]
  double* A = mats[blockIdx.x];
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int k = 0; k < m; ++k) {
    for (int i = tid; i < m; i += nth) {
      rowk[i] = A[(size_t)k * m + i];
      colk[i] = A[(size_t)i * m + k];
    }
    __syncthreads();
    const double piv = rowk[k];
    if (!(piv > 0.0)) {
      if (tid == 0) atomicExch(status, 1);
    }
    const double ip = 1.0 / piv;
    for (size_t e = tid; e < (size_t)m * m; e += nth) {
      const int i = (int)(e / m), j = (int)(e - (e / m) * m);
      double v;
      if (i == k && j == k) v = -ip;
      else if (i == k) v = rowk[j] * ip;
      else if (j == k) v = colk[i] * ip;
      else v = A[e] - colk[i] * rowk[j] * ip;
      A[e] = v;
    }
    __syncthreads();
  }
  for (size_t e = tid; e < (size_t)m * m; e += nth) A[e] = -A[e];
}

// ------------------------------------------------------------------ blocked SPD inverse
// In-place inverse of a batch of SPD m x m matrices by block Gauss-Jordan with GB x GB
// pivot blocks (the blocked form of the sweep above, for large m where one CTA per matrix
// is O(m^3) on a single SM).  Pivot block p (rows/cols [p0, p0+pb)):
//   P = A_pp^-1 ;  R_j = P A_pj ;  A_ij -= A_ip R_j (i, j != p) ;  A_ip = -A_ip P ;
//   A_pj = R_j ;  A_pp = P.
// After all pivots A holds A^-1.  Pivots are checked > 0 (SPD).
constexpr int GB = 64;

// acc(4x4 per thread) += A[0:64, 0:K] (lda) * B[0:K, 0:64] (ldb) for a 64x64 output tile;
// rows >= M / cols >= N / k >= K are zero-padded.  256 threads: rows (tid/16)*4.., cols (tid%16)*4..
__device__ __forceinline__ void gemm_tile_acc(const double* __restrict__ A, int lda,
                                              const double* __restrict__ B, int ldb, int M, int N,
                                              int K, double (&acc)[4][4], double (*As)[33],
                                              double (*Bs)[65]) {
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int e = tid; e < 64 * 32; e += 256) {
      const int r = e >> 5, kk = e & 31;
      As[r][kk] = (r < M && k0 + kk < K) ? A[(size_t)r * lda + k0 + kk] : 0.0;
    }
    for (int e = tid; e < 32 * 64; e += 256) {
      const int kk = e >> 6, c = e & 63;
      Bs[kk][c] = (k0 + kk < K && c < N) ? B[(size_t)(k0 + kk) * ldb + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[tr * 4 + i][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tc * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
}

// C (ldc, M x N valid) = alpha * acc + beta * C
__device__ __forceinline__ void gemm_tile_store(double* C, int ldc, int M, int N,
                                                const double (&acc)[4][4], double alpha,
                                                double beta) {
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = tr * 4 + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = tc * 4 + j;
      if (c >= N) continue;
      double* p = C + (size_t)r * ldc + c;
      *p = alpha * acc[i][j] + (beta != 0.0 ? beta * *p : 0.0);
    }
  }
}

// P = A_pp^-1 by the scalar sweep in shared memory (pb <= GB)
__global__ void __launch_bounds__(256) k_binv_pivot(double** mats, int m, int p0, int pb,
                                                    double* Pbuf, int* status) {
  __shared__ double a[GB][GB + 1];
  __shared__ double rowk[GB], colk[GB];
  const double* A = mats[blockIdx.x];
  double* P = Pbuf + (size_t)blockIdx.x * GB * GB;
  const int tid = threadIdx.x;
  for (int e = tid; e < pb * pb; e += 256) {
    const int i = e / pb, j = e - (e / pb) * pb;
    a[i][j] = A[(size_t)(p0 + i) * m + p0 + j];
  }
  __syncthreads();
  for (int k = 0; k < pb; ++k) {
    for (int i = tid; i < pb; i += 256) {
      rowk[i] = a[k][i];
      colk[i] = a[i][k];
    }
    __syncthreads();
    const double piv = rowk[k];
    if (!(piv > 0.0) && tid == 0) atomicExch(status, 1);
    const double ip = 1.0 / piv;
    for (int e = tid; e < pb * pb; e += 256) {
      const int i = e / pb, j = e - (e / pb) * pb;
      double v;
      if (i == k && j == k) v = -ip;
      else if (i == k) v = rowk[j] * ip;
      else if (j == k) v = colk[i] * ip;
      else v = a[i][j] - colk[i] * rowk[j] * ip;
      a[i][j] = v;
    }
    __syncthreads();
  }
  for (int e = tid; e < pb * pb; e += 256) {
    const int i = e / pb, j = e - (e / pb) * pb;
    P[i * GB + j] = -a[i][j];
  }
}

// R[0:pb, j-tile] = P A[p rows, j-tile]   (Rbuf per matrix: GB x m, ld m)
__global__ void __launch_bounds__(256) k_binv_rowpanel(double** mats, int m, int p0, int pb,
                                                       const double* Pbuf, double* Rbuf) {
  __shared__ double As[64][33];
  __shared__ double Bs[32][65];
  const double* A = mats[blockIdx.y];
  const int j0 = blockIdx.x * 64;
  double acc[4][4] = {};
  gemm_tile_acc(Pbuf + (size_t)blockIdx.y * GB * GB, GB, A + (size_t)p0 * m + j0, m, pb,
                min(64, m - j0), pb, acc, As, Bs);
  gemm_tile_store(Rbuf + (size_t)blockIdx.y * GB * m + j0, m, pb, min(64, m - j0), acc, 1.0, 0.0);
}

// A[i-tile, j-tile] -= A[i-tile, p cols] R[:, j-tile]  for i-tile, j-tile != p
__global__ void __launch_bounds__(256) k_binv_trailing(double** mats, int m, int p0, int pb,
                                                       const double* Rbuf) {
  const int it = blockIdx.y, jt = blockIdx.x, pt = p0 / GB;
  if (it == pt || jt == pt) return;
  __shared__ double As[64][33];
  __shared__ double Bs[32][65];
  double* A = mats[blockIdx.z];
  const int i0 = it * 64, j0 = jt * 64;
  double acc[4][4] = {};
  gemm_tile_acc(A + (size_t)i0 * m + p0, m, Rbuf + (size_t)blockIdx.z * GB * m + j0, m,
                min(64, m - i0), min(64, m - j0), pb, acc, As, Bs);
  gemm_tile_store(A + (size_t)i0 * m + j0, m, min(64, m - i0), min(64, m - j0), acc, -1.0, 1.0);
}

// Cbuf[m][64] (per matrix) = A[:, p cols]: the pivot column panel, copied before a full-matrix
// trailing GEMM (cuBLAS path) modifies it
__global__ void __launch_bounds__(256) k_binv_colcopy(double** mats, int m, int p0, int pb, double* Cbuf) {
  const double* A = mats[blockIdx.y];
  double* Cp = Cbuf + (size_t)blockIdx.y * m * GB;
  for (int e = blockIdx.x * 256 + threadIdx.x; e < m * pb; e += gridDim.x * 256) {
    const int r = e / pb, cc = e - (e / pb) * pb;
    Cp[(size_t)r * GB + cc] = A[(size_t)r * m + p0 + cc];
  }
}

// y = 0: A[i-tile, p cols] = -A[i-tile, p cols] P (i-tile != p), A_pp = P (i-tile == p)
// y = 1: A[p rows, j-tile] = R[:, j-tile] (j-tile != p)
// (Cbuf non-null: the p columns are read from the copy Cbuf, the trailing GEMM having updated
// the whole matrix)
__global__ void __launch_bounds__(256) k_binv_panels(double** mats, int m, int p0, int pb,
                                                     const double* Pbuf, const double* Rbuf,
                                                     const double* Cbuf) {
  __shared__ double As[64][33];
  __shared__ double Bs[32][65];
  double* A = mats[blockIdx.z];
  const double* P = Pbuf + (size_t)blockIdx.z * GB * GB;
  const int t = blockIdx.x, pt = p0 / GB, t0 = t * 64, tn = min(64, m - t0);
  if (blockIdx.y == 0) {
    if (t == pt) {
      for (int e = threadIdx.x; e < pb * pb; e += 256) {
        const int i = e / pb, j = e - (e / pb) * pb;
        A[(size_t)(p0 + i) * m + p0 + j] = P[i * GB + j];
      }
      return;
    }
    double acc[4][4] = {};
    if (Cbuf) gemm_tile_acc(Cbuf + (size_t)blockIdx.z * m * GB + (size_t)t0 * GB, GB, P, GB, tn, pb, pb, acc, As, Bs);
    else gemm_tile_acc(A + (size_t)t0 * m + p0, m, P, GB, tn, pb, pb, acc, As, Bs);
    gemm_tile_store(A + (size_t)t0 * m + p0, m, tn, pb, acc, -1.0, 0.0);
  } else {
    if (t == pt) return;
    const double* R = Rbuf + (size_t)blockIdx.z * GB * m;
    for (int e = threadIdx.x; e < pb * tn; e += 256) {
      const int i = e / tn, j = e - (e / tn) * tn;
      A[(size_t)(p0 + i) * m + t0 + j] = R[(size_t)i * m + t0 + j];
    }
  }
}

// In-place inverse of a batch of SPD m x m matrices (m <= 158) by the sweep operator with the
// matrix resident in shared memory (one CTA per matrix, 32 row groups x 32 column lanes, no
// index division); each pivot step touches only shared memory.
__global__ void __launch_bounds__(1024) k_spd_inverse_smem(double** mats, int m, int* status) {
  extern __shared__ double smi[];
  double* S = smi;              // [m*m]
  double* rowk = S + m * m;     // [m]
  double* colk = rowk + m;      // [m]
  double* A = mats[blockIdx.x];
  const int tid = threadIdx.x, jl = tid & 31, ig = tid >> 5;
  for (int e = tid; e < m * m; e += 1024) S[e] = A[e];
  __syncthreads();
  for (int k = 0; k < m; ++k) {
    for (int i = tid; i < m; i += 1024) {
      rowk[i] = S[k * m + i];
      colk[i] = S[i * m + k];
    }
    __syncthreads();
    const double piv = rowk[k];
    if (!(piv > 0.0) && tid == 0) atomicExch(status, 1);
    const double ip = 1.0 / piv;
    for (int i = ig; i < m; i += 32) {
      const double ci = colk[i] * ip;
      double* Si = S + i * m;
      if (i == k) {
        for (int j = jl; j < m; j += 32) Si[j] = (j == k) ? -ip : rowk[j] * ip;
      } else {
        for (int j = jl; j < m; j += 32) Si[j] = (j == k) ? ci : fma(-ci, rowk[j], Si[j]);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < m * m; e += 1024) A[e] = -S[e];
}

// The same inverses by the blocked sweep (msfk::inverse_blocked, 8-pivot panels, 512 threads):
// 3 barriers per 8 pivots instead of 2 per pivot; m <= 160 with the matrix and the panel
// scratch in shared memory.
__global__ void __launch_bounds__(512) k_spd_inverse_smem_blk(double** mats, int m, int* status) {
  extern __shared__ double smi[];
  double* S = smi;              // [m*m]
  double* scr = S + m * m;      // [3 m IB + IB IB]
  double* A = mats[blockIdx.x];
  for (int e = threadIdx.x; e < m * m; e += 512) S[e] = A[e];
  __syncthreads();
  msfinv::inverse_blocked<512, 5>(S, m, scr, status, 1);
  for (int e = threadIdx.x; e < m * m; e += 512) A[e] = S[e];
}

__global__ void k_copy_blocks(double** src, double** dst, int m) {
  const double* s = src[blockIdx.y];
  double* t = dst[blockIdx.y];
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < (size_t)m * m;
       e += (size_t)gridDim.x * blockDim.x)
    t[e] = s[e];
}

// Batched C = alpha op(A) op(B) + beta C, m x m row-major blocks, 64x64 tiles.
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_gemm(double** As, double** Bs, double** Cs, int m,
                                              double alpha, double beta) {
  constexpr int BM = 64, BK = 16;
  __shared__ double sA[BK][BM + 1];
  __shared__ double sB[BK][BM + 1];
  const double* A = As[blockIdx.z];
  const double* B = Bs[blockIdx.z];
  double* C = Cs[blockIdx.z];
  const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BM;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < m; k0 += BK) {
    // tile loads mapped so that consecutive threads read consecutive addresses: along the
    // row index for a transposed operand, along k for a row-major one
    for (int e = threadIdx.x; e < BK * BM; e += 256) {
      int kk, rr;
      if (TA) { kk = e / BM; rr = e - kk * BM; } else { rr = e / BK; kk = e - rr * BK; }
      const int gr = row0 + rr, gk = k0 + kk;
      sA[kk][rr] = (gr < m && gk < m) ? (TA ? A[(size_t)gk * m + gr] : A[(size_t)gr * m + gk]) : 0.0;
    }
    for (int e = threadIdx.x; e < BK * BM; e += 256) {
      int kk, cc;
      if (TB) { cc = e / BK; kk = e - cc * BK; } else { kk = e / BM; cc = e - kk * BM; }
      const int gc = col0 + cc, gk = k0 + kk;
      sB[kk][cc] = (gc < m && gk < m) ? (TB ? B[(size_t)gc * m + gk] : B[(size_t)gk * m + gc]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = row0 + ty * 4 + i, cc = col0 + tx * 4 + j;
      if (r < m && cc < m) {
        const size_t o = (size_t)r * m + cc;
        C[o] = alpha * acc[i][j] + (beta == 0.0 ? 0.0 : beta * C[o]);
      }
    }
}

// ------------------------------------------------------------------ cyclic-reduction solve
// forward, survivors i (jobs [i, il, ir]): b_i -= Q_il b_il + P_ir b_ir
__global__ void __launch_bounds__(256) k_cr_forward(Dims d, const int* __restrict__ surv,
                                                    const int* __restrict__ slot, int nslot,
                                                    const double* __restrict__ Qall,
                                                    const double* __restrict__ Pall,
                                                    double* cball, const PcgScalars* sc,
                                                    int rhs0, int gated) {
  pdl_launch();
  const int rhs = rhs0 + blockIdx.z;
  extern __shared__ double sv[];  // [2][m]
  const int* job = surv + 3 * blockIdx.y;
  const int i = job[0], il = job[1], ir = job[2];
  const size_t per = (size_t)d.mc * d.mc;
  // matrices by storage slot (a strip stores its chain and the interface blocks only),
  // vectors by global block
  const int sl = il >= 0 ? slot[il] : 0, sr = ir >= 0 ? slot[ir] : 0;
  cr_forward_rows(d, i, il, ir, blockIdx.x * CR_ROWS, Qall + ((size_t)rhs * nslot + sl) * per,
                  Pall + ((size_t)rhs * nslot + sr) * per, cball + (size_t)rhs * d.nbc * d.mc,
                  sv, threadIdx.x, blockDim.x, gated ? &sc[rhs].active : nullptr);
}

// back, eliminated k (jobs [k, kl, kr]): x_k = Dinv_k b_k - P_k^T x_kl - Q_k^T x_kr
__global__ void __launch_bounds__(256) k_cr_back(Dims d, const int* __restrict__ elim,
                                                 const int* __restrict__ slot, int nslot,
                                                 const double* __restrict__ Dinv,
                                                 const double* __restrict__ PTall,
                                                 const double* __restrict__ QTall,
                                                 const double* __restrict__ cball, double* cxall,
                                                 const PcgScalars* sc, int rhs0, int gated) {
  pdl_launch();
  const int rhs = rhs0 + blockIdx.z;
  extern __shared__ double sv[];  // [3][m]
  const int* job = elim + 3 * blockIdx.y;
  const int k = job[0], kl = job[1], kr = job[2];
  const size_t per = (size_t)d.mc * d.mc;
  const size_t blk = ((size_t)rhs * nslot + slot[k]) * per;
  cr_back_rows(d, k, kl, kr, blockIdx.x * CR_ROWS, Dinv + blk, PTall + blk, QTall + blk,
               cball + (size_t)rhs * d.nbc * d.mc, cxall + (size_t)rhs * d.nbc * d.mc, sv,
               threadIdx.x, blockDim.x, gated ? &sc[rhs].active : nullptr);
}

// batched transpose dst = src^T for blocks given by src pointers; dst = dst_base + (src - src_base)
__global__ void k_transpose_blocks(double** src, const double* src_base, double* dst_base, int m) {
  __shared__ double tile[32][33];
  const double* S = src[blockIdx.z];
  double* D = dst_base + (S - src_base);
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int r = by + j, c = bx + threadIdx.x;
    if (r < m && c < m) tile[j][threadIdx.x] = S[(size_t)r * m + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int r = bx + j, c = by + threadIdx.x;
    if (r < m && c < m) D[(size_t)r * m + c] = tile[threadIdx.x][j];
  }
}

// ------------------------------------------------------------------ dense top system
// Top (T*m x T*m, block-major) from the diagonal / coupling blocks of the active blocks tb[]
// left after the truncated cyclic reduction.
__global__ void k_build_top(Dims d, const int* __restrict__ tb, int T, const double* __restrict__ Dall,
                            const double* __restrict__ Uall, double* Atop, const int* __restrict__ slot,
                            int nslot) {
  const int rhs = blockIdx.y, m = d.mc;
  const size_t mm = (size_t)m * m, per = (size_t)T * T * mm;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < per;
       e += (size_t)gridDim.x * blockDim.x) {
    const int blk = (int)(e / mm), w = (int)(e - (size_t)blk * mm);
    const int bi = blk / T, bj = blk - bi * T, rr = w / m, cc = w - (w / m) * m;
    double v = 0.0;
    const size_t base = (size_t)rhs * nslot;
    if (bi == bj) v = Dall[(base + slot[tb[bi]]) * mm + (size_t)rr * m + cc];
    else if (bj == bi + 1) v = Uall[(base + slot[tb[bi]]) * mm + (size_t)rr * m + cc];
    else if (bi == bj + 1) v = Uall[(base + slot[tb[bj]]) * mm + (size_t)cc * m + rr];
    Atop[(size_t)rhs * per + e] = v;
  }
}

// dst = scale * src^T (trans) or dst = scale * src, for pointer-table block batches
template <bool TRANS>
__global__ void k_copy_blocks_ex(double** src, double** dst, int m, double scale) {
  __shared__ double tile[32][33];
  const double* S = src[blockIdx.z];
  double* D = dst[blockIdx.z];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int r = by + j, c = bx + threadIdx.x;
    if (r < m && c < m) tile[j][threadIdx.x] = S[(size_t)r * m + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    if (TRANS) {
      const int r = bx + j, c = by + threadIdx.x;
      if (r < m && c < m) D[(size_t)r * m + c] = scale * tile[threadIdx.x][j];
    } else {
      const int r = by + j, c = bx + threadIdx.x;
      if (r < m && c < m) D[(size_t)r * m + c] = scale * tile[j][threadIdx.x];
    }
  }
}

// x_top = -A b_top  (A = -Top^{-1})
__global__ void __launch_bounds__(256) k_top_solve(Dims d, const int* __restrict__ tb, int T,
                                                   const double* __restrict__ Atop,
                                                   const double* __restrict__ cball, double* cxall,
                                                   const PcgScalars* sc, int rhs0, int gated) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.y;
  if (gated && !sc[rhs].active) return;
  extern __shared__ double sv[];   // [T*m]
  const size_t mm = (size_t)d.mc * d.mc;
  top_solve_rows(d, tb, T, Atop + (size_t)rhs * T * T * mm, cball + (size_t)rhs * d.nbc * d.mc,
                 cxall + (size_t)rhs * d.nbc * d.mc, blockIdx.x * CR_ROWS, sv, threadIdx.x,
                 blockDim.x);
}

}  // namespace

// ================================================================== host side
// Restriction groups for k_restrict_batch: the work list (grid order) split into groups of B
// agglomerates with the same class and the same clipped box, each group filled in grid order
// (members of a periodic class lie a period apart, so the group's boxes are close in memory).
// Returns the number of groups; groups (n x B, padded with -1).
int restrict_groups(const Dims& d, const std::vector<int>& work, const std::vector<int>& cls,
                    int B, std::vector<int>& groups) {
  groups.clear();
  std::map<std::array<int, 5>, int> open;   // key -> group being filled
  for (int a : work) {
    const int I = a / (d.ncy + 1), J = a % (d.ncy + 1);
    const int gx0 = I * d.cx - d.cx - d.gox, gy0 = J * d.cy - d.cy;
    const std::array<int, 5> key = {cls[a], std::max(1, -gx0), std::min(d.bx - 2, d.nnx - 1 - gx0),
                                    std::max(1, -gy0), std::min(d.by - 2, d.nny - 1 - gy0)};
    auto it = open.find(key);
    int gi;
    if (it == open.end()) {
      gi = (int)(groups.size() / B);
      groups.resize(groups.size() + B, -1);
    } else {
      gi = it->second;
    }
    int* g = groups.data() + (size_t)gi * B;
    int fill = 0;
    while (g[fill] >= 0) ++fill;
    g[fill] = a;
    if (fill + 1 == B)
      open.erase(key);
    else
      open[key] = gi;
  }
  return (int)(groups.size() / B);
}

void launch_restrict(msf_ctx* c, int rhs0, int nr, const double* t, bool gated) {
  // global coarse fields, this rank's node columns; a strip restricts the agglomerates of its
  // chain [cr_lo, cr_hi] (the chain's end blocks get the partial sums of its owned nodes)
  const Dims& d = c->dl;
#define MSF_RESTRICT(KM, NTR)                                                                   \
  launch_k(k_restrict1<KM, NTR>, dim3(c->n_restrict, nr), dim3(NTR), 0, c->stream, d,            \
           (const double2*)t, (const double*)c->phi, (const int*)c->cls_of_agg_d,                \
           (const int*)c->agg_by_cls_d, c->cb, (const PcgScalars*)c->sc, rhs0, gated ? 1 : 0)
#define MSF_RESTRICT_T(NTR)                     \
  do {                                          \
    if (d.kmax <= 4) MSF_RESTRICT(4, NTR);      \
    else if (d.kmax <= 8) MSF_RESTRICT(8, NTR); \
    else MSF_RESTRICT(16, NTR);                 \
  } while (0)
  // one warp per agglomerate when that gives >= 32 warps per SM (configs[4]: 320 -> 230 us per
  // launch); otherwise one CTA per agglomerate (configs[1] at one realisation, 2145 warps:
  // 15 vs 20 us)
  // same-class groups when they still give >= 1000 warps: configs[4] 224 -> 178 us at one
  // realisation (664 -> 495 at three), configs[1] at three realisations 37 -> 23 us; with
  // fewer warps (configs[1], one realisation: 537) the per-agglomerate CTAs below are faster
  // (15 vs 22 us)
  if (c->n_rgroups > 0 && ((long long)c->n_rgroups * nr >= 1000 || c->rgroup_force)) {
#define MSF_RESTRICT_B(KM, B)                                                                      \
  launch_k(k_restrict_batch<KM, B>, dim3((c->n_rgroups + 7) / 8, nr), dim3(256), 0, c->stream, d,   \
           (const double2*)t, (const double*)c->phi, (const int*)c->cls_of_agg_d,                     \
           (const int*)c->rgroups_d, c->n_rgroups, c->cb, (const PcgScalars*)c->sc, rhs0,            \
           gated ? 1 : 0)
    if (c->rgroup_B == 4) MSF_RESTRICT_B(4, 4);
    else MSF_RESTRICT_B(8, 2);
#undef MSF_RESTRICT_B
    MSF_LAUNCHED(c);
    return;
  }
  if (c->restrict_warp && (long long)c->n_restrict * nr >= 32LL * c->n_sm) {
#define MSF_RESTRICT_W(KM)                                                                         \
  launch_k(k_restrict_warp<KM>, dim3((c->n_restrict + 7) / 8, nr), dim3(256), 0, c->stream, d,        \
           (const double2*)t, (const double*)c->phi, (const int*)c->cls_of_agg_d,                     \
           (const int*)c->agg_by_cls_d, c->n_restrict, c->cb, (const PcgScalars*)c->sc, rhs0,         \
           gated ? 1 : 0)
    if (d.kmax <= 4) MSF_RESTRICT_W(4);
    else if (d.kmax <= 8) MSF_RESTRICT_W(8);
    else MSF_RESTRICT_W(16);
#undef MSF_RESTRICT_W
    MSF_LAUNCHED(c);
    return;
  }
  // threads per agglomerate CTA: 256 measured fastest (512 / 1024: 19 / 40 us vs 15 us at one
  // realisation on configs[1]; larger block reductions, fewer CTAs per SM)
  const int ntr = c->restrict_threads > 0 ? c->restrict_threads : 256;
  if (ntr >= 1024) MSF_RESTRICT_T(1024);
  else if (ntr >= 512) MSF_RESTRICT_T(512);
  else if (ntr >= 256) MSF_RESTRICT_T(256);
  else MSF_RESTRICT_T(128);
#undef MSF_RESTRICT_T
#undef MSF_RESTRICT
  MSF_LAUNCHED(c);
}

void launch_prolong(msf_ctx* c, int rhs0, int nr, double* z, bool gated) {
  const Dims& d = c->dl;   // every local node, halo included (identical increments on both ranks)
  dim3 g((d.nny + 31) / 32, (d.nnx + 7) / 8, 1);
  if (nr > 1 && nr <= 3 && d.kmax <= 8 && c->prolong_nr) {
#define MSF_PROLONG_NR(KM, NR)                                                                    \
  launch_k(k_prolong_nr<KM, NR>, g, dim3(NT), 0, c->stream, d, (const double*)c->phi,              \
           (const int*)c->cls_of_agg_d, (const double*)c->cx, (double2*)z, (const PcgScalars*)c->sc, \
           rhs0, gated ? 1 : 0)
    if (d.kmax <= 4) {
      if (nr == 2) MSF_PROLONG_NR(4, 2);
      else MSF_PROLONG_NR(4, 3);
    } else {
      if (nr == 2) MSF_PROLONG_NR(8, 2);
      else MSF_PROLONG_NR(8, 3);
    }
#undef MSF_PROLONG_NR
    MSF_LAUNCHED(c);
    return;
  }
#define MSF_PROLONG(KM)                                                                           \
  launch_k(k_prolong1<KM>, dim3(g.x, g.y, nr), dim3(NT), 0, c->stream, d, (const double*)c->phi,    \
           (const int*)c->cls_of_agg_d, (const double*)c->cx, (double2*)z, (const PcgScalars*)c->sc, \
           rhs0, gated ? 1 : 0)
  if (d.kmax <= 4) MSF_PROLONG(4);
  else if (d.kmax <= 8) MSF_PROLONG(8);
  else MSF_PROLONG(16);
#undef MSF_PROLONG
  MSF_LAUNCHED(c);
}

// Factor K0 = L^T L: Jacobi eigendecomposition of the 8 x 8 element matrix, the 5 eigenpairs
// above the rigid-body null space.  Returns false if the rank is not 5.
static bool factor_K0(const K0Mat& K, LMat& L) {
  double A[8][8], V[8][8];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      A[i][j] = K.v[i * 8 + j];
      V[i][j] = i == j ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < 8; ++i)
      for (int j = i + 1; j < 8; ++j) off += A[i][j] * A[i][j];
    if (off < 1e-30) break;
    for (int p = 0; p < 8; ++p)
      for (int q = p + 1; q < 8; ++q) {
        if (std::fabs(A[p][q]) < 1e-300) continue;
        const double th = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < 8; ++k) {
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = cs * akp - sn * akq;
          A[k][q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < 8; ++k) {
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = cs * apk - sn * aqk;
          A[q][k] = sn * apk + cs * aqk;
        }
        for (int k = 0; k < 8; ++k) {
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = cs * vkp - sn * vkq;
          V[k][q] = sn * vkp + cs * vkq;
        }
      }
  }
  double lmax = 0.0;
  for (int i = 0; i < 8; ++i) lmax = std::max(lmax, A[i][i]);
  int l = 0;
  for (int i = 0; i < 8; ++i) {
    if (A[i][i] <= 1e-12 * lmax) continue;
    if (l == 5) return false;
    const double sq = std::sqrt(A[i][i]);
    for (int k = 0; k < 8; ++k) L.v[l * 8 + k] = sq * V[k][i];
    ++l;
  }
  return l == 5;
}

static bool galerkin_gemm(msf_ctx* c) {
  const Dims& d = c->d;
  // large cell products only: configs[3] (256 elements x 64 columns) 0.78 -> 0.56 s assembly,
  // configs[4] (400 x 16) 122 -> 117 ms; at 256 x 16 (configs[1]) the per-cell kernel wins
  if (!c->cublas || !c->galerkin_gemm || !c->galerkin_G || d.cx * d.cy * 4 * d.kmax < 5000) return false;
  static thread_local LMat L;
  static thread_local double Lnu = -1.0;
  if (Lnu != c->p.nu) {
    if (!factor_K0(c->K0, L)) return false;
    Lnu = c->p.nu;
  }
  const int P = 4 * d.kmax, nel = d.cx * d.cy;
  const size_t per_cell = (size_t)5 * nel * P;
  const int CH = std::min(P, 16);
  const int nch = (P + CH - 1) / CH;
  const size_t smem = (size_t)(d.cx + 1) * (d.cy + 1) * 2 * CH * sizeof(double);
  cudaFuncSetAttribute(k_galerkin_G, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int c_lo = c->cell_lo * d.ncy, c_hi = c->cell_hi * d.ncy;
  const int chunk = (int)std::max<size_t>(1, c->galerkin_G_doubles / per_cell);
  for (int r = 0; r < d.R; ++r)
    for (int c0 = c_lo; c0 < c_hi; c0 += chunk) {
      const int nc = std::min(chunk, c_hi - c0);
      k_galerkin_G<<<dim3(nc, 1, nch), NT, smem, c->stream>>>(d, L, c->E, c->phi, c->cls_of_agg_d, r, c0, CH,
                                                             c->galerkin_G);
      MSF_LAUNCHED(c);
      // Kcell (P x P, symmetric) = G^T G; G row-major (5 nel) x P = column-major G^T (P x 5 nel)
      const double one = 1.0, zero = 0.0;
      double* Kc = c->Kcell + ((size_t)r * d.ncx * d.ncy + c0) * P * P;
      cublasDgemmStridedBatched((cublasHandle_t)c->cublas, CUBLAS_OP_N, CUBLAS_OP_T, P, P, 5 * nel, &one,
                                c->galerkin_G, P, (long long)per_cell, c->galerkin_G, P, (long long)per_cell,
                                &zero, Kc, P, (long long)P * P, nc);
    }
  return true;
}

// Galerkin cell products Kcell = Phi_C^T (E K0) Phi_C of this rank's coarse cells (Eq. 10)
void launch_galerkin_cells(msf_ctx* c) {
  const Dims& d = c->d;
  const int P = 4 * d.kmax;
  if (galerkin_gemm(c)) return;
  const size_t ncn2 = (size_t)(d.cx + 1) * (d.cy + 1) * 2;
  // largest column chunk whose staged bases fit in shared memory (<= 16 so CH^2 <= NT)
  int CH = std::min(P, 16);
  auto smem_for = [&](int ch) {
    const bool single = ch >= P;
    return ((single ? 1 : 2) * ncn2 * ch + 16 * 8 * (size_t)ch + 16 * MSF_MAX_RHS) * sizeof(double);
  };
  while (CH > 2 && smem_for(CH) > 220 * 1024) CH /= 2;
  const size_t smem = smem_for(CH);
  const int nch = (P + CH - 1) / CH;
  cudaFuncSetAttribute(k_cell_galerkin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // this rank's coarse cell columns (all of them on one GPU)
  k_cell_galerkin<<<dim3((c->cell_hi - c->cell_lo) * d.ncy, 1, nch * nch), NT, smem, c->stream>>>(
      d, c->K0, c->E, c->phi, c->cls_of_agg_d, c->Kcell, CH, c->cell_lo * d.ncy);
  MSF_LAUNCHED(c);
}

// Block-tridiagonal copies D_I, U_I of K_c (this rank's chain) gathered from the cell products
void launch_coarse_gather(msf_ctx* c, double* D, double* U, int nslot) {
  const Dims& d = c->d;
  const int nD = c->cr_hi - c->cr_lo + 1, nU = c->cell_hi - c->cell_lo;
  const size_t total = (size_t)(nD + nU) * d.mc * d.mc;
  int blocks = (int)std::min<size_t>((total + 255) / 256, 65535);
  k_coarse_gather<<<dim3(blocks, d.R), 256, 0, c->stream>>>(d, c->Kcell, c->cls_of_agg_d, c->classes_d, D, U,
                                                            c->cr_lo, nD, c->cell_lo, nU, c->id_lo, c->id_hi,
                                                            c->cr_lo, nslot);
  MSF_LAUNCHED(c);
}

void launch_coarse_galerkin(msf_ctx* c) {
  launch_galerkin_cells(c);
  launch_coarse_gather(c, c->Dc, c->Uc, c->nslot);
}

// In-place inverses of n SPD m x m matrices (device pointer table mats): the one-CTA sweep for
// small m, the blocked Gauss-Jordan above for m >= blocked_inv_min.
static void launch_spd_inverse(msf_ctx* c, double** mats, int n, int m) {
  if (m >= c->blocked_inv_min) {
    const int T = (m + GB - 1) / GB;
    for (int pt = 0; pt < T; ++pt) {
      const int p0 = pt * GB, pb = std::min(GB, m - p0);
      k_binv_pivot<<<n, 256, 0, c->stream>>>(mats, m, p0, pb, c->binv_P, c->factor_status);
      k_binv_rowpanel<<<dim3(T, n), 256, 0, c->stream>>>(mats, m, p0, pb, c->binv_P, c->binv_R);
      if (c->cublas && c->binv_Cp) {
        // trailing update A -= A[:, p] R as one batched GEMM over the whole matrix (the p row and
        // column panels are rewritten by k_binv_panels from R and the column copy):
        // column-major A^T -= R^T Cp^T
        k_binv_colcopy<<<dim3((m * pb + 255) / 256 < 64 ? (m * pb + 255) / 256 : 64, n), 256, 0, c->stream>>>(
            mats, m, p0, pb, c->binv_C);
        const double mone = -1.0, one = 1.0;
        cublasDgemmBatched((cublasHandle_t)c->cublas, CUBLAS_OP_N, CUBLAS_OP_N, m, m, pb, &mone,
                           (const double* const*)c->binv_Rp, m, (const double* const*)c->binv_Cp, GB, &one,
                           mats, m, n);
        k_binv_panels<<<dim3(T, 2, n), 256, 0, c->stream>>>(mats, m, p0, pb, c->binv_P, c->binv_R, c->binv_C);
        c->launches += 4;
      } else {
        k_binv_trailing<<<dim3(T, T, n), 256, 0, c->stream>>>(mats, m, p0, pb, c->binv_R);
        k_binv_panels<<<dim3(T, 2, n), 256, 0, c->stream>>>(mats, m, p0, pb, c->binv_P, c->binv_R, nullptr);
        c->launches += 4;
      }
    }
  } else if (c->inv_blocked_smem && m <= 160 &&
             (size_t)(m * m + 3 * m * msfinv::IB + msfinv::IB * msfinv::IB) * sizeof(double) <= 220 * 1024) {
    const size_t smem = (size_t)(m * m + 3 * m * msfinv::IB + msfinv::IB * msfinv::IB) * sizeof(double);
    cudaFuncSetAttribute(k_spd_inverse_smem_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_spd_inverse_smem_blk<<<n, 512, smem, c->stream>>>(mats, m, c->factor_status);
    MSF_LAUNCHED(c);
  } else if ((size_t)(m * m + 2 * m) * sizeof(double) <= 200 * 1024) {
    const size_t smem = (size_t)(m * m + 2 * m) * sizeof(double);
    cudaFuncSetAttribute(k_spd_inverse_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_spd_inverse_smem<<<n, 1024, smem, c->stream>>>(mats, m, c->factor_status);
    MSF_LAUNCHED(c);
  } else {
    k_spd_inverse<<<n, 1024, 2 * (size_t)m * sizeof(double), c->stream>>>(mats, m, c->factor_status);
    MSF_LAUNCHED(c);
  }
}

// Batched m x m products of the K_c factorisation, row-major C = alpha op(A) op(B) + beta C over
// device pointer tables.  cuBLAS batched DGEMM (a plain library GEMM, outside the PCG path;
// column-major: C^T = op(B)^T op(A)^T), or the hand-written k_gemm (MSF_CUBLAS=0).  configs[3]:
// the products were 67% of a 1.86 s assembly at about 23% of the FP64 peak.
template <bool TA, bool TB>
static void gemm_batched(msf_ctx* c, double** As, double** Bs, double** Cs, int m, double alpha,
                         double beta, int count) {
  if (count <= 0) return;
  if (c->cublas && m >= 64) {   // small blocks (configs[0]: m = 28) stay on k_gemm
    cublasDgemmBatched((cublasHandle_t)c->cublas, TB ? CUBLAS_OP_T : CUBLAS_OP_N,
                       TA ? CUBLAS_OP_T : CUBLAS_OP_N, m, m, m, &alpha, (const double* const*)Bs, m,
                       (const double* const*)As, m, &beta, Cs, m, count);
    return;
  }
  const dim3 gt((m + 63) / 64, (m + 63) / 64, count);
  k_gemm<TA, TB><<<gt, 256, 0, c->stream>>>(As, Bs, Cs, m, alpha, beta);
  MSF_LAUNCHED(c);
}

// factorisation of the reduction levels [l0, l1)
static void assemble_levels(msf_ctx* c, int l0, int l1) {
  const Dims& d = c->d;
  const int m = d.mc;
    for (int l = l0; l < l1; ++l) {
    const CrLevel& L = c->cr[l];
    k_copy_blocks<<<dim3(64, L.n_inv), 256, 0, c->stream>>>(L.invsrc, L.inv, m);
    MSF_LAUNCHED(c);
    launch_spd_inverse(c, L.inv, L.n_inv, m);
    gemm_batched<false, false>(c, L.pA, L.pB, L.pC, m, 1.0, 0.0, L.nP);
    gemm_batched<true, false>(c, L.qA, L.qB, L.qC, m, 1.0, 0.0, L.nQ);
    {
      const dim3 tg((m + 31) / 32, (m + 31) / 32, L.nP);
      k_transpose_blocks<<<tg, dim3(32, 8), 0, c->stream>>>(L.pC, c->Pc, c->PTc, m);
      MSF_LAUNCHED(c);
      if (L.nQ) {
        const dim3 tq((m + 31) / 32, (m + 31) / 32, L.nQ);
        k_transpose_blocks<<<tq, dim3(32, 8), 0, c->stream>>>(L.qC, c->Qc, c->QTc, m);
        MSF_LAUNCHED(c);
      }
    }
    gemm_batched<false, true>(c, L.dlA, L.dlB, L.dlC, m, -1.0, 1.0, L.nDl);
    gemm_batched<false, false>(c, L.drA, L.drB, L.drC, m, -1.0, 1.0, L.nDr);
    gemm_batched<false, false>(c, L.uA, L.uB, L.uC, m, -1.0, 0.0, L.nU);
  }
}

void launch_assemble_local(msf_ctx* c) {
  launch_coarse_galerkin(c);
  assemble_levels(c, 0, c->n_local);
}

void launch_iface_mat_pack(msf_ctx* c) {
  const size_t nI = c->iface.size(), mm = (size_t)c->d.mc * c->d.mc;
  cudaMemsetAsync(c->iface_mat, 0, (size_t)c->d.R * (2 * nI - 1) * mm * 8, c->stream);
  k_copy_blocks<<<dim3(64, 3 * c->d.R), 256, 0, c->stream>>>(c->ifm_pack, c->ifm_pack + 3 * c->d.R, c->d.mc);
  MSF_LAUNCHED(c);
}

void launch_iface_mat_unpack(msf_ctx* c) {
  const int n = (int)(2 * c->iface.size() - 1) * c->d.R;
  k_copy_blocks<<<dim3(64, n), 256, 0, c->stream>>>(c->ifm_unpack, c->ifm_unpack + n, c->d.mc);
  MSF_LAUNCHED(c);
}

void launch_assemble_coarse(msf_ctx* c) {
  if (c->use_nd) {
    launch_galerkin_cells(c);
    launch_nd_factor(c);
    return;
  }
  launch_assemble_local(c);
  launch_assemble_top(c);
}

void launch_assemble_top(msf_ctx* c) {
  assemble_levels(c, c->n_local, (int)c->cr.size());
  const Dims& d = c->d;
  const int m = d.mc;
    // dense inverse of the remaining top system by block Gauss-Jordan (block sweep operator):
  // pivot k: Pk = A_kk^-1, W_i = A_ik Pk, A_ij -= W_i A_kj, A_ik = W_i, A_ki = W_i^T,
  // A_kk = -Pk; after all pivots A = -Top^-1.
  const int T = c->top_T;
  {
    const size_t per = (size_t)T * T * m * m;
    const int blocks = (int)std::min<size_t>((per + 255) / 256, 65535);
    k_build_top<<<dim3(blocks, d.R), 256, 0, c->stream>>>(d, c->top_blocks_d, T, c->Dc, c->Uc, c->Atop,
                                                          c->slot_d, c->nslot);
    MSF_LAUNCHED(c);
  }
  const dim3 tg((m + 31) / 32, (m + 31) / 32);
  for (const TopStep& S : c->top_steps) {
    k_copy_blocks<<<dim3(64, S.nI), 256, 0, c->stream>>>(S.invsrc, S.inv, m);
    MSF_LAUNCHED(c);
    launch_spd_inverse(c, S.inv, S.nI, m);
    MSF_LAUNCHED(c);
    gemm_batched<false, false>(c, S.wA, S.wB, S.wC, m, 1.0, 0.0, S.nW);
    gemm_batched<false, false>(c, S.uA, S.uB, S.uC, m, -1.0, 1.0, S.nU);
    if (S.nC) {
      k_copy_blocks_ex<false><<<dim3(tg.x, tg.y, S.nC), dim3(32, 8), 0, c->stream>>>(S.cps, S.cpd, m, 1.0);
      MSF_LAUNCHED(c);
      k_copy_blocks_ex<true><<<dim3(tg.x, tg.y, S.nC), dim3(32, 8), 0, c->stream>>>(S.cps, S.tpd, m, 1.0);
      MSF_LAUNCHED(c);
    }
    k_copy_blocks_ex<false><<<dim3(tg.x, tg.y, S.nI), dim3(32, 8), 0, c->stream>>>(S.ngs, S.ngd, m, -1.0);
    MSF_LAUNCHED(c);
  }
}

// ---------------------------------------------------------------- coarse solve
static void cr_smem_attrs(msf_ctx* c) {
  const int m = c->d.mc;
  if (3 * (size_t)m * sizeof(double) > 48 * 1024 ||
      (size_t)c->top_T * m * sizeof(double) > 48 * 1024) {
    const int need = (int)(std::max<size_t>(3, c->top_T) * m * sizeof(double));
    cudaFuncSetAttribute(k_cr_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, need);
    cudaFuncSetAttribute(k_cr_back, cudaFuncAttributeMaxDynamicSharedMemorySize, need);
    cudaFuncSetAttribute(k_top_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, need);
  }
}

static void cr_forward_levels(msf_ctx* c, int l0, int l1, int rhs0, int nr, bool gated) {
  const Dims& d = c->d;
  const int m = d.mc;
  for (int l = l0; l < l1; ++l) {
    const CrLevel& L = c->cr[l];
    if (L.surv.empty()) continue;
    launch_k(k_cr_forward, dim3((m + CR_ROWS - 1) / CR_ROWS, (unsigned)L.surv.size(), nr), dim3(256),
             2 * m * sizeof(double), c->stream, d, (const int*)L.surv_d, (const int*)c->slot_d, c->nslot,
             (const double*)c->Qc,
             (const double*)c->Pc, c->cb, (const PcgScalars*)c->sc, rhs0, gated ? 1 : 0);
    MSF_LAUNCHED(c);
  }
}

static void cr_back_levels(msf_ctx* c, int l0, int l1, int rhs0, int nr, bool gated) {
  const Dims& d = c->d;
  const int m = d.mc;
  for (int l = l1 - 1; l >= l0; --l) {
    const CrLevel& L = c->cr[l];
    launch_k(k_cr_back, dim3((m + CR_ROWS - 1) / CR_ROWS, (unsigned)L.elim.size(), nr), dim3(256),
             3 * m * sizeof(double), c->stream, d, (const int*)L.elim_d, (const int*)c->slot_d, c->nslot,
             (const double*)c->Dinv,
             (const double*)c->PTc, (const double*)c->QTc, (const double*)c->cb, c->cx,
             (const PcgScalars*)c->sc, rhs0, gated ? 1 : 0);
    MSF_LAUNCHED(c);
  }
}

void launch_coarse_forward_local(msf_ctx* c, int rhs0, int nr, bool gated) {
  cr_smem_attrs(c);
  cr_forward_levels(c, 0, c->n_local, rhs0, nr, gated);
}

// interface levels (strips), the dense top system, interface back substitution
void launch_coarse_top(msf_ctx* c, int rhs0, int nr, bool gated) {
  cr_smem_attrs(c);
  const int nl = (int)c->cr.size();
  cr_forward_levels(c, c->n_local, nl, rhs0, nr, gated);
  {
    const int T = c->top_T, n = T * c->d.mc;
    launch_k(k_top_solve, dim3((n + CR_ROWS - 1) / CR_ROWS, nr), dim3(256), (size_t)n * sizeof(double),
             c->stream, c->d, (const int*)c->top_blocks_d, T, (const double*)c->Atop,
             (const double*)c->cb, c->cx, (const PcgScalars*)c->sc, rhs0, gated ? 1 : 0);
    MSF_LAUNCHED(c);
  }
  cr_back_levels(c, c->n_local, nl, rhs0, nr, gated);
}

void launch_coarse_back_local(msf_ctx* c, int rhs0, int nr, bool gated) {
  cr_back_levels(c, 0, c->n_local, rhs0, nr, gated);
}

void launch_iface_vec_pack(msf_ctx* c, int rhs0, int nr) {
  const int nI = (int)c->iface.size();
  const int blocks = std::max(1, std::min(c->n_sm, (nI * c->d.mc + 255) / 256));
  k_iface_vec<<<dim3(blocks, nr), 256, 0, c->stream>>>(c->d, c->iface_d, nI, c->rank, c->rank + 1, c->cb,
                                                       c->iface_vec, rhs0, 0);
  MSF_LAUNCHED(c);
}

void launch_iface_vec_unpack(msf_ctx* c, int rhs0, int nr) {
  const int nI = (int)c->iface.size();
  const int blocks = std::max(1, std::min(c->n_sm, (nI * c->d.mc + 255) / 256));
  k_iface_vec<<<dim3(blocks, nr), 256, 0, c->stream>>>(c->d, c->iface_d, nI, -1, -1, c->cb,
                                                       c->iface_vec, rhs0, 1);
  MSF_LAUNCHED(c);
}

// c <- K_c^{-1} c for realisations [rhs0, rhs0+nr) on one GPU: forward elimination over the
// levels, top system, back substitution in reverse level order.  (A strip context runs the
// same phases with the interface exchange between them, msf_capi.cu dist_vcycle.)
void launch_coarse_solve(msf_ctx* c, int rhs0, int nr, bool gated) {
  if (c->use_nd) {
    launch_nd_solve(c, rhs0, nr, gated);
    return;
  }
  launch_coarse_forward_local(c, rhs0, nr, gated);
  launch_coarse_top(c, rhs0, nr, gated);
  launch_coarse_back_local(c, rhs0, nr, gated);
}
