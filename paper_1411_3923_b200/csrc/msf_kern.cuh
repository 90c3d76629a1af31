// Device-side building blocks of the B200 MsFEM-PCG path, shared by the kernels of
// msf_fem.cu, msf_sgsw.cu and msf_coarse.cu so that they execute the same arithmetic.  All functions are called by a whole CTA unless
// stated otherwise.
#pragma once

#include "msf_internal.cuh"
#include "msf_inverse.cuh"

namespace msfk {

// Programmatic dependent launch (PDL): kernels of the PCG iteration are launched with the
// programmatic-serialisation attribute (launch_k, msf_internal.cuh).  pdl_launch lets the
// next kernel's CTAs be scheduled once every CTA of this grid has started; pdl_wait blocks
// until the previous grid has completed and its writes are visible.  Every such kernel
// calls pdl_wait before touching data a predecessor writes (including the PCG scalars);
// only loads of data that is constant during PCG (moduli, coarse blocks) may precede it.
// Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Build switches of the Gauss-Seidel arithmetic (R7a): MSF_GS_RCP pivots by refined
// reciprocal; MSF_F0_DIAG zero-start phase without the (vanishing) stencil.
#ifndef MSF_GS_RCP
#define MSF_GS_RCP 1
#endif
#ifndef MSF_F0_DIAG
#define MSF_F0_DIAG 1
#endif

// ------------------------------------------------------------------ Q4 node stencil
// local index a of the centre node inside element (sx,sy) = (ix-1+sx, iy-1+sy)
__device__ __forceinline__ constexpr int a_of(int sx, int sy) {
  return (sx == 0 && sy == 0) ? 2 : (sx == 1 && sy == 0) ? 3 : (sx == 0 && sy == 1) ? 1 : 0;
}
__device__ __forceinline__ constexpr int DXB(int b) { return (b == 1 || b == 2) ? 1 : 0; }
__device__ __forceinline__ constexpr int DYB(int b) { return (b >= 2) ? 1 : 0; }

// make_K0's element matrix has 8 distinct entries: K0[i][j] = K0[0][K0_IDX(i, j)] (the index
// table of the closed form, msf_fem.cu make_K0).  The stencil loops read K0 through this table,
// so only K.v[0..7] are live (8 uniform register pairs instead of up to 64: sm_100 keeps the
// DFMA constant operands of a kernel parameter in uniform registers, and 64 of them spilled).
// The values are the same entries, so the arithmetic is bitwise unchanged.
__device__ __forceinline__ constexpr int K0_IDX(int i, int j) {
  return (i == 0)   ? j
         : (i == 1) ? (j == 0 ? 1 : j == 1 ? 0 : 9 - j)
         : (i == 2) ? (j == 0 ? 2 : j == 1 ? 7 : j == 2 ? 0 : j == 3 ? 5 : j == 4 ? 6 : j == 5 ? 3 : j == 6 ? 4 : 1)
         : (i == 3) ? (j == 0 ? 3 : j == 1 ? 6 : j == 2 ? 5 : j == 3 ? 0 : j == 4 ? 7 : j == 5 ? 2 : j == 6 ? 1 : 4)
         : (i == 4) ? (j < 4 ? j + 4 : j - 4)
         : (i == 5) ? (j == 0 ? 5 : j == 1 ? 4 : j == 2 ? 3 : j == 3 ? 2 : j == 4 ? 1 : j == 5 ? 0 : j == 6 ? 7 : 6)
         : (i == 6) ? (j == 0 ? 6 : j == 1 ? 3 : j == 2 ? 4 : j == 3 ? 1 : j == 4 ? 2 : j == 5 ? 7 : j == 6 ? 0 : 5)
                    : (j == 0 ? 7 : j == 1 ? 2 : j == 2 ? 1 : j == 3 ? 4 : j == 4 ? 3 : j == 5 ? 6 : j == 6 ? 5 : 0);
}
#define MSF_K0(K, i, j) ((K).v[K0_IDX((i), (j))])

// (K z)_node and the node's own 2x2 diagonal block from the 4 element moduli E[sx][sy]
// and the 3x3 neighbourhood z[i][j] = node (ix-1+i, iy-1+j)  (Eq. 4-5).
// SYM: the pivot block's lower row is taken from its upper one (make_K0: K0 is bitwise
// symmetric with equal diagonal entries, so this is bitwise the same result with 8 fewer
// FMAs; the choice only moves register allocation, see launch_sgs_phase).
// NZ: bit 3 i + j set = z[i][j] may be nonzero.  A term whose z is exactly +0 leaves its
// accumulator bitwise unchanged (acc + K * 0 = acc), so a caller that KNOWS a neighbour is still
// zero (the first forward phases of a sweep from z = 0) may drop its bit: same result, fewer FMAs.
template <bool SYM = true, int NZ = 0x1ff>
__device__ __forceinline__ void apply_node(const K0Mat& K, const double (&E)[2][2],
                                           const double2 (&z)[3][3], double& ox, double& oy,
                                           double& dxx, double& dxy, double& dyx, double& dyy) {
  ox = oy = dxx = dxy = dyx = dyy = 0.0;
#pragma unroll
  for (int sx = 0; sx < 2; ++sx)
#pragma unroll
    for (int sy = 0; sy < 2; ++sy) {
      const int a = a_of(sx, sy);
      double ax = 0.0, ay = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (!((NZ >> (3 * (sx + DXB(b)) + sy + DYB(b))) & 1)) continue;
        const double2 v = z[sx + DXB(b)][sy + DYB(b)];
        ax = fma(MSF_K0(K, 2 * a, 2 * b), v.x, ax);
        ax = fma(MSF_K0(K, 2 * a, 2 * b + 1), v.y, ax);
        ay = fma(MSF_K0(K, 2 * a + 1, 2 * b), v.x, ay);
        ay = fma(MSF_K0(K, 2 * a + 1, 2 * b + 1), v.y, ay);
      }
      const double e = E[sx][sy];
      ox = fma(e, ax, ox);
      oy = fma(e, ay, oy);
      dxx = fma(e, MSF_K0(K, 2 * a, 2 * a), dxx);
      dxy = fma(e, MSF_K0(K, 2 * a, 2 * a + 1), dxy);
      if (!SYM) {
        dyx = fma(e, MSF_K0(K, 2 * a + 1, 2 * a), dyx);
        dyy = fma(e, MSF_K0(K, 2 * a + 1, 2 * a + 1), dyy);
      }
    }
  if (SYM) {
    dyx = dxy;
    dyy = dxx;
  }
}

// The node's own 2x2 block of K from the 4 element moduli.  make_K0's element matrix is
// bitwise symmetric with one diagonal value, so the block is [dxx dxy; dxy dxx] and these
// are bitwise the dxx, dxy (= dyx), dyy of apply_node.
__device__ __forceinline__ void diag_node(const K0Mat& K, const double (&E)[2][2], double& dxx,
                                          double& dxy) {
  dxx = dxy = 0.0;
#pragma unroll
  for (int sx = 0; sx < 2; ++sx)
#pragma unroll
    for (int sy = 0; sy < 2; ++sy) {
      const int a = a_of(sx, sy);
      const double e = E[sx][sy];
      dxx = fma(e, MSF_K0(K, 2 * a, 2 * a), dxx);
      dxy = fma(e, MSF_K0(K, 2 * a, 2 * a + 1), dxy);
    }
}

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block reduction; result valid in every thread.  nthreads multiple of 32,
// sm >= nthreads/32 + 1 doubles.
__device__ __forceinline__ double block_sum_all(double v, double* sm, int tid, int nthreads) {
  v = warp_sum(v);
  if ((tid & 31) == 0) sm[tid >> 5] = v;
  __syncthreads();
  const int nw = nthreads >> 5;
  if (tid < 32) {
    double s = (tid < nw) ? sm[tid] : 0.0;
    s = warp_sum(s);
    if (tid == 0) sm[nw] = s;   // broadcast slot
  }
  __syncthreads();
  const double s = sm[nw];
  __syncthreads();
  return s;
}

// ------------------------------------------------------------------ cross-CTA reductions
// Every PCG reduction: block sums -> per-CTA partials -> the last CTA to arrive sums the
// partials in a fixed order (deterministic) and finalises the PCG scalar.
// Writes this block's partial, returns true in the last block to arrive.
__device__ __forceinline__ bool arrive_last(double v, double* partials, int slot, unsigned* counter,
                            unsigned total, int tid) {
  __shared__ unsigned s_ticket;
  if (tid == 0) {
    partials[slot] = v;
    __threadfence();
    s_ticket = atomicAdd(counter, 1u);
  }
  __syncthreads();
  return s_ticket == total - 1;
}

// In the last block: deterministic sum of partials[0..n).  Eight independent loads per
// thread are in flight at once (the last block is the serial tail of every PCG reduction).
__device__ __forceinline__ double reduce_partials(const double* partials, int n, double* sm, int tid,
                                  int nthreads) {
  double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int i = tid;
  for (; i + 7 * nthreads < n; i += 8 * nthreads) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] += __ldcg(partials + i + j * nthreads);
  }
  for (int j = 0; i < n; i += nthreads, ++j) s[j & 7] += __ldcg(partials + i);
  const double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  return block_sum_all(t, sm, tid, nthreads);
}

// PCG scalar update from a completed (global) dot product (reading R9)
__device__ __forceinline__ void fin_scalar(PcgScalars& S, int kind, double tot, int rz_mode) {
  switch (kind) {
    case FIN_PQ:
      S.pq = tot;
      S.alpha = S.rz / tot;
      break;
    case FIN_RR:
      S.rr = tot;
      S.iters += 1;
      if (tot <= S.tol2 * S.fnorm2) {
        S.active = 0;
      } else if (S.iters >= S.max_it) {
        S.active = 0;
        S.noconv = 1;
      }
      break;
    case FIN_RZ:
      S.beta = (rz_mode == 1) ? 0.0 : tot / S.rz;
      S.rz = tot;
      break;
    case FIN_F:
      S.fnorm2 = tot;
      S.rr = tot;
      S.active = (tot > 0.0 && !(tot <= S.tol2 * tot)) ? 1 : 0;
      break;
    default:
      S.comp = tot;
      break;
  }
}

// last block of a reduction: finalise in place (one GPU) or park the local sum for the
// cross-rank all-reduce (strip partition, dsum != null)
__device__ __forceinline__ void fin_or_park(PcgScalars* sc, double* dsum, int rhs, int kind,
                                            double tot, int rz_mode) {
  if (dsum)
    dsum[kind * MSF_MAX_RHS + rhs] = tot;
  else
    fin_scalar(sc[rhs], kind, tot, rz_mode);
}


// ------------------------------------------------------------------ Gauss-Seidel
// 1/x for the Gauss-Seidel pivots: the hardware approximation refined by two Newton steps
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = fma(y, fma(-x, y, 1.0), y);
  y = fma(y, fma(-x, y, 1.0), y);
  return y;
}

// One Gauss-Seidel node update (reading R7): the 2x2 block of the node is relaxed in place,
// x then y (FWD), y then x (BWD), or both (the F3B3 phase).  Eloc / zloc: the 4 element moduli
// and the 3x3 neighbourhood of the node (zloc[1][1] = its current value), rv its residual
// entry, fm its Dirichlet bits.  ZERO: z = 0 around the node, only the pivot block is needed.
// Shared by the colour-phase kernels and the streaming sweep (msf_sgsw.cu), so both execute
// the same arithmetic.  Per-thread.
template <bool FWD, bool BWD, bool ZERO, int NZ = 0x1ff>
__device__ __forceinline__ double2 gs_node(const K0Mat& K, const double (&Eloc)[2][2],
                                         const double2 (&zloc)[3][3], double2 rv, uint8_t fm) {
  double ox, oy, dxx, dxy, dyx, dyy;
  if (ZERO && MSF_F0_DIAG) {
    // z = 0 around the node: (K z) vanishes, only the pivot block is needed
    ox = oy = 0.0;
    diag_node(K, Eloc, dxx, dxy);
    dyx = dxy;
    dyy = dxx;
  } else {
    apply_node<true, NZ>(K, Eloc, zloc, ox, oy, dxx, dxy, dyx, dyy);
  }
  double2 zn = zloc[1][1];
  double rx = rv.x - ox, ry = rv.y - oy;
#if MSF_GS_RCP
  // reciprocal of the pivot (dyy == dxx bitwise, R7b): off the dependent chain, <= 2 ulp from
  // the quotient
  const double ixx = rcp_nr(dxx), iyy = ixx;
#define MSF_DIVX(a) ((a) * ixx)
#define MSF_DIVY(a) ((a) * iyy)
#else
#define MSF_DIVX(a) ((a) / dxx)
#define MSF_DIVY(a) ((a) / dyy)
#endif
  if (FWD) {
    if (!(fm & 1)) {
      const double dz = MSF_DIVX(rx);
      zn.x += dz;
      ry -= dyx * dz;
      rx -= dxx * dz;
    }
    if (!(fm & 2)) {
      const double dz = MSF_DIVY(ry);
      zn.y += dz;
      rx -= dxy * dz;
      ry -= dyy * dz;
    }
  }
  if (BWD) {
    if (!(fm & 2)) {
      const double dz = MSF_DIVY(ry);
      zn.y += dz;
      rx -= dxy * dz;
    }
    if (!(fm & 1)) zn.x += MSF_DIVX(rx);
#undef MSF_DIVX
#undef MSF_DIVY
  }
  return zn;
}

// One colour phase (reading R7) for node quad (qx, qy): updates the quad's node of
// `colour`.  FWD: x then y ; BWD: y then x ; both: the F3B3 phase.  ZERO: first forward
// phase from z = 0 (writes zeros to the quad's other nodes).  Returns r.z over the whole
// quad when RZ (after the final backward phase).  Per-thread.
template <bool FWD, bool BWD, bool ZERO, bool RZ, bool SYM = true>
__device__ __forceinline__ double sgs_quad(const Dims& d, const K0Mat& K, const double* __restrict__ E,
                                           const double2* __restrict__ r, double2* z,
                                           const uint8_t* __restrict__ fixn, int qx, int qy,
                                           int colour) {
  const int ix = 2 * qx + (colour & 1), iy = 2 * qy + (colour >> 1);
  double dot = 0.0;
  if (ZERO) {
#pragma unroll
    for (int dn = 0; dn < 4; ++dn) {
      const int gx = 2 * qx + (dn & 1), gy = 2 * qy + (dn >> 1);
      if (dn != colour && gx < d.nnx && gy < d.nny) z[(size_t)gx * d.nny + gy] = make_double2(0.0, 0.0);
    }
  }
  if (ix < d.nnx && iy < d.nny) {
    double Eloc[2][2];
    double2 zloc[3][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int ex = ix - 1 + a, ey = iy - 1 + b;
        Eloc[a][b] = (ex >= 0 && ex < d.nelx && ey >= 0 && ey < d.nely) ? __ldg(E + (size_t)ex * d.nely + ey) : 0.0;
      }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int gx = ix - 1 + a, gy = iy - 1 + b;
        zloc[a][b] = (!ZERO && gx >= 0 && gx < d.nnx && gy >= 0 && gy < d.nny)
                         ? z[(size_t)gx * d.nny + gy]
                         : make_double2(0.0, 0.0);
      }
    const size_t n = (size_t)ix * d.nny + iy;
    const double2 rv = r[n];
    const uint8_t fm = fixn[n];
    const double2 zn = gs_node<FWD, BWD, ZERO>(K, Eloc, zloc, rv, fm);
    z[n] = zn;
    if (RZ) dot = rv.x * zn.x + rv.y * zn.y;
  }
  if (RZ) {
#pragma unroll
    for (int dn = 0; dn < 4; ++dn) {
      const int gx = 2 * qx + (dn & 1), gy = 2 * qy + (dn >> 1);
      if (dn != colour && gx < d.nnx && gy < d.nny) {
        const size_t m = (size_t)gx * d.nny + gy;
        const double2 a = r[m], b = z[m];
        dot += a.x * b.x + a.y * b.y;
      }
    }
  }
  return dot;
}

// ------------------------------------------------------------------ restriction
// c[rhs][agg*kmax + a] = sum_n phi_{agg,a}(n) . t_rhs(n) for the realisations in act[].
template <int KM>
__device__ __forceinline__ void restrict_agg(const Dims& d, const double2* __restrict__ tall,
                                             const double* __restrict__ phi,
                                             const int* __restrict__ cls_of_agg, double* cball,
                                             int agg, const bool (&act)[MSF_MAX_RHS], int nthreads,
                                             int tid, double (*red)[MSF_MAX_RHS * KM]) {
  const int I = agg / (d.ncy + 1), J = agg - (agg / (d.ncy + 1)) * (d.ncy + 1);
  const double* ph = phi + (size_t)cls_of_agg[agg] * d.kmax * d.box_nodes * 2;
  // box origin in this rank's node columns (gox = 0 on one GPU); t vanishes on halo columns,
  // so a strip restricts exactly its owned nodes and the ranks' sums add up to R_c t
  const int gx0 = I * d.cx - d.cx - d.gox, gy0 = J * d.cy - d.cy;
  // interior of the padded box (chi vanishes on its boundary ring)
  const int ix_lo = max(1, -gx0), ix_hi = min(d.bx - 2, d.nnx - 1 - gx0);
  const int iy_lo = max(1, -gy0), iy_hi = min(d.by - 2, d.nny - 1 - gy0);
  const int w = iy_hi - iy_lo + 1, h = ix_hi - ix_lo + 1;
  double acc[MSF_MAX_RHS][KM];
#pragma unroll
  for (int r = 0; r < MSF_MAX_RHS; ++r)
#pragma unroll
    for (int a = 0; a < KM; ++a) acc[r][a] = 0.0;
  for (int k = tid; k < w * h; k += nthreads) {
    const int px = ix_lo + k / w, py = iy_lo + (k - (k / w) * w);
    const size_t n = (size_t)(gx0 + px) * d.nny + (gy0 + py);
    double2 tv[MSF_MAX_RHS];
#pragma unroll
    for (int r = 0; r < MSF_MAX_RHS; ++r) tv[r] = act[r] ? tall[(size_t)r * d.nn + n] : make_double2(0.0, 0.0);
    const int bn = px * d.by + py;
#pragma unroll
    for (int a = 0; a < KM; ++a) {
      if (a < d.kmax) {
        const double2 pv = *reinterpret_cast<const double2*>(ph + ((size_t)a * d.box_nodes + bn) * 2);
#pragma unroll
        for (int r = 0; r < MSF_MAX_RHS; ++r) acc[r][a] = fma(pv.x, tv[r].x, fma(pv.y, tv[r].y, acc[r][a]));
      }
    }
  }
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int r = 0; r < MSF_MAX_RHS; ++r)
#pragma unroll
    for (int a = 0; a < KM; ++a) {
      if (act[r] && a < d.kmax) {
        const double v = warp_sum(acc[r][a]);
        if (lane == 0) red[wid][r * KM + a] = v;
      }
    }
  __syncthreads();
  const int r = tid / KM, a = tid - (tid / KM) * KM;
  if (r < MSF_MAX_RHS && a < d.kmax && act[r]) {
    double s = 0.0;
    for (int w2 = 0; w2 < nthreads / 32; ++w2) s += red[w2][r * KM + a];
    cball[(size_t)r * d.nbc * d.mc + (size_t)agg * d.kmax + a] = s;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ prolongation
// z(n) += sum_{I,J,a} phi_{I,J,a}(n) x_c[slot(I,J,a)] for the realisations in act[].
// Per-thread (node ix, iy).  KM >= kmax: the mode loop is unrolled so that all basis and
// coarse-value loads of the node are in flight together (one memory latency per node).
template <int KM>
__device__ __forceinline__ void prolong_node(const Dims& d, const double* __restrict__ phi,
                                             const int* __restrict__ cls_of_agg,
                                             const double* __restrict__ cxall, double2* zall,
                                             int ix, int iy, const bool (&act)[MSF_MAX_RHS]) {
  double sx[MSF_MAX_RHS], sy[MSF_MAX_RHS];
#pragma unroll
  for (int r = 0; r < MSF_MAX_RHS; ++r) sx[r] = sy[r] = 0.0;
  const int gix = ix + d.gox;   // global node column (ix is local to this rank's strip)
  const int I0 = gix / d.cx, J0 = iy / d.cy;
#pragma unroll
  for (int di = 0; di < 2; ++di) {
    const int I = I0 + di;
    if (I > d.ncx) continue;
    const int px = gix - (I * d.cx - d.cx);
    if (px < 0 || px >= d.bx) continue;
#pragma unroll
    for (int dj = 0; dj < 2; ++dj) {
      const int J = J0 + dj;
      if (J > d.ncy) continue;
      const int py = iy - (J * d.cy - d.cy);
      if (py < 0 || py >= d.by) continue;
      const int agg = I * (d.ncy + 1) + J;
      const double* ph = phi + (size_t)cls_of_agg[agg] * d.kmax * d.box_nodes * 2;
      const int bn = px * d.by + py;
#pragma unroll
      for (int a = 0; a < KM; ++a) {
        if (a < d.kmax) {
          const double2 pv = __ldg(reinterpret_cast<const double2*>(ph + ((size_t)a * d.box_nodes + bn) * 2));
#pragma unroll
          for (int r = 0; r < MSF_MAX_RHS; ++r) {
            if (act[r]) {
              const double cv = cxall[(size_t)r * d.nbc * d.mc + (size_t)agg * d.kmax + a];
              sx[r] = fma(pv.x, cv, sx[r]);
              sy[r] = fma(pv.y, cv, sy[r]);
            }
          }
        }
      }
    }
  }
  const size_t n = (size_t)ix * d.nny + iy;
#pragma unroll
  for (int r = 0; r < MSF_MAX_RHS; ++r) {
    if (act[r]) {
      double2* z = zall + (size_t)r * d.nn;
      double2 zv = z[n];
      zv.x += sx[r];
      zv.y += sy[r];
      z[n] = zv;
    }
  }
}

}  // namespace msfk
