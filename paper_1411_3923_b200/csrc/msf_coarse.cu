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
// zout(n) = zin(n) + sum_{I,J,a} phi_{I,J,a}(n) x_c[slot(I,J,a)], one (node, realisation) per
// thread (zout == zin: in place).
template <int KM>
__global__ void __launch_bounds__(NT) k_prolong1(Dims d, const double* __restrict__ phi,
                                                 const int* __restrict__ cls_of_agg,
                                                 const double* __restrict__ cxall,
                                                 const double2* zin, double2* zall,
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
  const size_t n = (size_t)rhs * d.nn + (size_t)ix * d.nny + iy;
  double2 zv = zin[n];
  zv.x += sx;
  zv.y += sy;
  zall[n] = zv;
}

// Prolongation for NR > 1 active realisations, one node per thread for all of them: the
// realisations share the coarse basis, so phi is loaded once per (covering
// agglomerate, mode) and applied to each realisation's coefficients (k_prolong1 loads it
// once per realisation).  Per realisation the sum runs in k_prolong1's order: z is bitwise
// the same.
template <int KM, int NR>
__global__ void __launch_bounds__(NT) k_prolong_nr(Dims d, const double* __restrict__ phi,
                                                   const int* __restrict__ cls_of_agg,
                                                   const double* __restrict__ cxall,
                                                   const double2* zin, double2* zall,
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
    const size_t n = (size_t)(rhs0 + k) * d.nn + (size_t)ix * d.nny + iy;
    double2 zv = zin[n];
    zv.x += sx[k];
    zv.y += sy[k];
    zall[n] = zv;
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
  if (c->restrict_warp && ((long long)c->n_restrict * nr >= 32LL * c->n_sm || c->restrict_warp_force)) {
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

void launch_prolong(msf_ctx* c, int rhs0, int nr, const double* zin, double* z, bool gated) {
  const Dims& d = c->dl;   // every local node, halo included (identical increments on both ranks)
  dim3 g((d.nny + 31) / 32, (d.nnx + 7) / 8, 1);
  if (nr > 1 && nr <= 3 && d.kmax <= 8 && c->prolong_nr) {
#define MSF_PROLONG_NR(KM, NR)                                                                    \
  launch_k(k_prolong_nr<KM, NR>, g, dim3(NT), 0, c->stream, d, (const double*)c->phi,              \
           (const int*)c->cls_of_agg_d, (const double*)c->cx, (const double2*)zin, (double2*)z,         \
           (const PcgScalars*)c->sc,                                                              \
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
           (const int*)c->cls_of_agg_d, (const double*)c->cx, (const double2*)zin, (double2*)z,         \
           (const PcgScalars*)c->sc,                                                              \
           rhs0, gated ? 1 : 0)
  if (d.kmax <= 4) MSF_PROLONG(4);
  else if (d.kmax <= 8) MSF_PROLONG(8);
  else MSF_PROLONG(16);
#undef MSF_PROLONG
  MSF_LAUNCHED(c);
}

// Galerkin cell products Kcell = Phi_C^T (E K0) Phi_C of this rank's coarse cells (Eq. 10)
void launch_galerkin_cells(msf_ctx* c) {
  const Dims& d = c->d;
  const int P = 4 * d.kmax;
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
                                                            c->cr_lo, nD, c->cell_lo, nU, 0, d.ncx,
                                                            c->cr_lo, nslot);
  MSF_LAUNCHED(c);
}

// K_c assembly (Eq. 10) and its nested-dissection factorisation (msf_nd.cu), one GPU
void launch_assemble_coarse(msf_ctx* c) {
  launch_galerkin_cells(c);
  launch_nd_factor(c);
}
