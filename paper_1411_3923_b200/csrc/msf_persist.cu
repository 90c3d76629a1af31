// Persistent cooperative PCG kernel: every PCG iteration of every realisation runs inside ONE
// launch (cooperative, one or more CTAs per SM, all resident), phases separated by
// grid-wide barriers.  The per-iteration work is the same as the single-purpose kernels
// (it calls the same msf_kern.cuh device functions):
//   A  q = K p, p.q                 (tiles)           -> alpha = rz / pq
//   B  u += alpha p, r -= alpha q, ||r||^2, and the zero-start first GS colour   -> convergence
//   C  Gauss-Seidel colours F1 F2 F3B3 B2 B1 B0 (pre-smoothing, reading R7/R8)
//   D  t = r - K z                  (tiles)
//   E  restriction c = R_c t        (agglomerates in class order)
//   F  coarse solve: cyclic-reduction forward levels, final block, back levels
//   G  prolongation z += R_c^T x_c  (nodes)
//   H  Gauss-Seidel colours F0 F1 F2 F3B3 B2 B1 B0 (post-smoothing), r.z in B0 -> beta
//   I  p = z + beta p
// Dot products: each CTA reduces its own items in a fixed order into one partial per
// realisation; after the barrier every CTA sums the partials in the same fixed order, so all
// CTAs take identical (deterministic) convergence decisions.  (§2.4.2 l.146; the
// PCG recurrence and stopping rule of reading R9.)
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "msf_kern.cuh"

namespace cg = cooperative_groups;
using namespace msfk;

namespace {

constexpr int PT = 256;             // threads per CTA (== TILE_THREADS)
#ifndef MSF_PERSIST_MINB
#define MSF_PERSIST_MINB 2
#endif
constexpr int PMINB = MSF_PERSIST_MINB;   // resident CTAs per SM the register budget targets
static_assert(PT == TILE_THREADS, "tile routine expects 256 threads");

struct CrLevelDev {
  int s;        // stride (0: final level)
  int nsurv;
  int nelim;
  const int* surv;   // [nsurv][3]: survivor, eliminated left / right neighbour (-1: none)
  const int* elim;   // [nelim][3]: eliminated block, surviving left / right neighbour
};

struct PersistArgs {
  Dims d;
  const double* E;
  const uint8_t* fixn;
  double2* u;
  double2* r;
  double2* z;
  double2* p;
  double2* q;
  double2* t;
  const double* phi;
  const int* cls_of_agg;
  const int* agg_by_cls;
  double* cb;
  double* cx;
  const double* Dinv;
  const double* Pc;
  const double* Qc;
  const double* PTc;
  const double* QTc;
  const CrLevelDev* levels;
  int nlev;
  const int* top_blocks;   // active blocks of the dense top system
  int topT;
  const double* Atop;      // [R][T*T][mc*mc], -Top^{-1}
  PcgScalars* sc;
  double* part;   // [3][MSF_MAX_RHS][gridDim.x]
  int nr;
  unsigned long long* prof;   // optional phase timeline (nullptr: off)
};

// Sum of part[slot][rhs][0..G) in fixed order, identical in every CTA.
__device__ __forceinline__ double grid_total(const double* part, int G, double* red, int tid) {
  double s = 0.0;
  for (int j = tid; j < G; j += PT) s += __ldcg(part + j);
  return block_sum_all(s, red, tid, PT);
}

template <int KM>
__global__ void __launch_bounds__(PT, PMINB) k_pcg_persistent(PersistArgs A, K0Mat K) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ double red[PT / 32 + 1];
  __shared__ double rred[PT / 32][MSF_MAX_RHS * KM];
  const Dims& d = A.d;
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int nr = A.nr;
  double* partA = A.part;
  double* partB = A.part + MSF_MAX_RHS * G;
  double* partH = A.part + 2 * MSF_MAX_RHS * G;

  // per-realisation state, identical in every CTA
  bool act[MSF_MAX_RHS];
  double rz[MSF_MAX_RHS], tol2[MSF_MAX_RHS], fn2[MSF_MAX_RHS], rr_last[MSF_MAX_RHS];
  int iters[MSF_MAX_RHS], maxit[MSF_MAX_RHS], noconv[MSF_MAX_RHS];
#pragma unroll
  for (int k = 0; k < MSF_MAX_RHS; ++k) {
    const bool in = k < nr;
    act[k] = in && A.sc[k].active;
    rz[k] = in ? A.sc[k].rz : 0.0;
    tol2[k] = in ? A.sc[k].tol2 : 0.0;
    fn2[k] = in ? A.sc[k].fnorm2 : 0.0;
    rr_last[k] = in ? A.sc[k].rr : 0.0;
    iters[k] = in ? A.sc[k].iters : 0;
    maxit[k] = in ? A.sc[k].max_it : 0;
    noconv[k] = in ? A.sc[k].noconv : 0;
  }
  const int nty = (d.nny + TY - 1) / TY, ntx = (d.nnx + TX - 1) / TX, ntiles = ntx * nty;
  const int nqy = (d.nny + 1) / 2, nqx = (d.nnx + 1) / 2;
  const int nqchunks = (nqx * nqy + PT - 1) / PT;
  const int nnchunks = (d.nn + PT - 1) / PT;
  const size_t vstride = (size_t)d.nn;
  TileSmem& S = *reinterpret_cast<TileSmem*>(dyn);
  double* sv = reinterpret_cast<double*>(dyn);

  // grid barrier; optional phase timeline (A.prof: %globaltimer after every barrier of the
  // first 32 iterations, written by CTA 0)
  int prof_it = 0, prof_ph = 0;
  auto gsync = [&]() {
    grid.sync( );
    if (A.prof && b == 0 && tid == 0 && prof_it < 32 && prof_ph < 64) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      A.prof[prof_it * 64 + prof_ph] = t;
    }
    ++prof_ph;
  };

  // one Gauss-Seidel colour phase over all quads of the active realisations
  auto gs_phase = [&](int colour, int kind) {
    for (int item = b; item < nqchunks * nr; item += G) {
      const int k = item / nqchunks, chunk = item - k * nqchunks;
      if (!act[k]) continue;
      const int qd = chunk * PT + tid;
      if (qd >= nqx * nqy) continue;
      const int qx = qd / nqy, qy = qd - (qd / nqy) * nqy;
      const double* E = A.E + (size_t)k * d.ne;
      const double2* r = A.r + k * vstride;
      double2* z = A.z + k * vstride;
      switch (kind) {
        case 0: sgs_quad<true, false, false, false>(d, K, E, r, z, A.fixn, qx, qy, colour); break;
        case 1: sgs_quad<true, true, false, false>(d, K, E, r, z, A.fixn, qx, qy, colour); break;
        default: sgs_quad<false, true, false, false>(d, K, E, r, z, A.fixn, qx, qy, colour); break;
      }
    }
    gsync();
  };

  for (;; ++prof_it) {
    prof_ph = 0;
    if (A.prof && b == 0 && tid == 0 && prof_it < 32) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      A.prof[prof_it * 64 + 63] = t;
    }
    bool any = false;
#pragma unroll
    for (int k = 0; k < MSF_MAX_RHS; ++k) any |= act[k];
    if (!any) break;

    // ---------------- A: q = K p, p.q
    {
      double dots[MSF_MAX_RHS] = {0.0, 0.0, 0.0, 0.0};
      for (int item = b; item < ntiles * nr; item += G) {
        const int k = item / ntiles, tile = item - k * ntiles;
        if (!act[k]) continue;
        const int tx = tile / nty, ty = tile - (tile / nty) * nty;
        const double dv = apply_tile<0>(d, K, A.E + (size_t)k * d.ne, A.p + k * vstride,
                                        A.q + k * vstride, nullptr, A.fixn, tx * TX, ty * TY, tid, S);
#pragma unroll
        for (int kk = 0; kk < MSF_MAX_RHS; ++kk)
          if (kk == k) dots[kk] += dv;
      }
#pragma unroll
      for (int k = 0; k < MSF_MAX_RHS; ++k) {
        if (!act[k]) continue;
        const double s = block_sum_all(dots[k], red, tid, PT);
        if (tid == 0) partA[k * G + b] = s;
      }
      __threadfence();
      gsync();
    }
    double alpha[MSF_MAX_RHS];
#pragma unroll
    for (int k = 0; k < MSF_MAX_RHS; ++k) {
      alpha[k] = 0.0;
      if (act[k]) alpha[k] = rz[k] / grid_total(partA + k * G, G, red, tid);
    }

    // ---------------- B: x/r update, ||r||^2, zero-start GS colour 0
    {
      double rrp[MSF_MAX_RHS] = {0.0, 0.0, 0.0, 0.0};
      for (int item = b; item < nqchunks * nr; item += G) {
        const int k = item / nqchunks, chunk = item - k * nqchunks;
        if (!act[k]) continue;
        const int qd = chunk * PT + tid;
        if (qd >= nqx * nqy) continue;
        const int qx = qd / nqy, qy = qd - (qd / nqy) * nqy;
        double2* u = A.u + k * vstride;
        double2* r = A.r + k * vstride;
        const double2* p = A.p + k * vstride;
        const double2* q = A.q + k * vstride;
        double s = 0.0;
#pragma unroll
        for (int dn = 0; dn < 4; ++dn) {
          const int gx = 2 * qx + (dn & 1), gy = 2 * qy + (dn >> 1);
          if (gx < d.nnx && gy < d.nny) {
            const size_t n = (size_t)gx * d.nny + gy;
            const double2 pv = p[n], qv = q[n];
            double2 uv = u[n], rv = r[n];
            uv.x = fma(alpha[k], pv.x, uv.x);
            uv.y = fma(alpha[k], pv.y, uv.y);
            rv.x = fma(-alpha[k], qv.x, rv.x);
            rv.y = fma(-alpha[k], qv.y, rv.y);
            u[n] = uv;
            r[n] = rv;
            s += rv.x * rv.x + rv.y * rv.y;
          }
        }
#pragma unroll
        for (int kk = 0; kk < MSF_MAX_RHS; ++kk)
          if (kk == k) rrp[kk] += s;
        sgs_quad<true, false, true, false>(d, K, A.E + (size_t)k * d.ne, r, A.z + k * vstride,
                                           A.fixn, qx, qy, 0);
      }
#pragma unroll
      for (int k = 0; k < MSF_MAX_RHS; ++k) {
        if (!act[k]) continue;
        const double s = block_sum_all(rrp[k], red, tid, PT);
        if (tid == 0) partB[k * G + b] = s;
      }
      __threadfence();
      gsync();
    }
#pragma unroll
    for (int k = 0; k < MSF_MAX_RHS; ++k) {
      if (!act[k]) continue;
      const double rr = grid_total(partB + k * G, G, red, tid);
      rr_last[k] = rr;
      iters[k] += 1;
      if (rr <= tol2[k] * fn2[k]) {
        act[k] = false;
      } else if (iters[k] >= maxit[k]) {
        act[k] = false;
        noconv[k] = 1;
      }
    }
    {
      bool any2 = false;
#pragma unroll
      for (int k = 0; k < MSF_MAX_RHS; ++k) any2 |= act[k];
      if (!any2) break;
    }

    // ---------------- C: pre-smoothing colours F1 F2 F3B3 B2 B1 B0
    gs_phase(1, 0);
    gs_phase(2, 0);
    gs_phase(3, 1);
    gs_phase(2, 2);
    gs_phase(1, 2);
    gs_phase(0, 2);

    // ---------------- D: t = r - K z
    for (int item = b; item < ntiles * nr; item += G) {
      const int k = item / ntiles, tile = item - k * ntiles;
      if (!act[k]) continue;
      const int tx = tile / nty, ty = tile - (tile / nty) * nty;
      apply_tile<1>(d, K, A.E + (size_t)k * d.ne, A.z + k * vstride, A.t + k * vstride,
                    A.r + k * vstride, A.fixn, tx * TX, ty * TY, tid, S);
    }
    gsync();

    // ---------------- E: restriction (all active realisations per agglomerate)
    for (int item = b; item < d.n_agg; item += G)
      restrict_agg<KM>(d, A.t, A.phi, A.cls_of_agg, A.cb, A.agg_by_cls[item], act, PT, tid, rred);
    gsync();

    // ---------------- F: coarse solve by cyclic reduction
    const int nrc = (d.mc + CR_ROWS - 1) / CR_ROWS;
    const size_t per = (size_t)d.mc * d.mc;
    for (int l = 0; l < A.nlev; ++l) {
      const CrLevelDev L = A.levels[l];
      if (L.s == 0) continue;
      for (int item = b; item < nrc * L.nsurv * nr; item += G) {
        const int k = item / (nrc * L.nsurv), rest = item - k * (nrc * L.nsurv);
        if (!act[k]) continue;
        const int si = rest / nrc, rc = rest - (rest / nrc) * nrc;
        const int i = L.surv[3 * si], il = L.surv[3 * si + 1], ir = L.surv[3 * si + 2];
        cr_forward_rows(d, i, il, ir, rc * CR_ROWS, A.Qc + ((size_t)k * d.nbc + max(il, 0)) * per,
                        A.Pc + ((size_t)k * d.nbc + max(ir, 0)) * per, A.cb + (size_t)k * d.nbc * d.mc,
                        sv, tid, PT);
      }
      gsync();
    }
    {
      const int n = A.topT * d.mc, nrt = (n + CR_ROWS - 1) / CR_ROWS;
      for (int item = b; item < nrt * nr; item += G) {
        const int k = item / nrt, rc = item - k * nrt;
        if (!act[k]) continue;
        top_solve_rows(d, A.top_blocks, A.topT, A.Atop + (size_t)k * A.topT * A.topT * per,
                       A.cb + (size_t)k * d.nbc * d.mc, A.cx + (size_t)k * d.nbc * d.mc,
                       rc * CR_ROWS, sv, tid, PT);
      }
      gsync();
    }
    for (int l = A.nlev - 1; l >= 0; --l) {
      const CrLevelDev L = A.levels[l];
      for (int item = b; item < nrc * L.nelim * nr; item += G) {
        const int k = item / (nrc * L.nelim), rest = item - k * (nrc * L.nelim);
        if (!act[k]) continue;
        const int ei = rest / nrc, rc = rest - (rest / nrc) * nrc;
        const int kb = L.elim[3 * ei], kl = L.elim[3 * ei + 1], kr = L.elim[3 * ei + 2];
        const size_t blk = ((size_t)k * d.nbc + kb) * per;
        cr_back_rows(d, kb, kl, kr, rc * CR_ROWS, A.Dinv + blk, A.PTc + blk, A.QTc + blk,
                     A.cb + (size_t)k * d.nbc * d.mc, A.cx + (size_t)k * d.nbc * d.mc, sv, tid, PT);
      }
      gsync();
    }

    // ---------------- G: prolongation
    for (int item = b; item < nnchunks; item += G) {
      const int n = item * PT + tid;
      if (n < d.nn) prolong_node<KM>(d, A.phi, A.cls_of_agg, A.cx, A.z, n / d.nny, n - (n / d.nny) * d.nny, act);
    }
    gsync();

    // ---------------- H: post-smoothing colours F0 F1 F2 F3B3 B2 B1, then B0 with r.z
    gs_phase(0, 0);
    gs_phase(1, 0);
    gs_phase(2, 0);
    gs_phase(3, 1);
    gs_phase(2, 2);
    gs_phase(1, 2);
    {
      double dots[MSF_MAX_RHS] = {0.0, 0.0, 0.0, 0.0};
      for (int item = b; item < nqchunks * nr; item += G) {
        const int k = item / nqchunks, chunk = item - k * nqchunks;
        if (!act[k]) continue;
        const int qd = chunk * PT + tid;
        if (qd >= nqx * nqy) continue;
        const int qx = qd / nqy, qy = qd - (qd / nqy) * nqy;
        const double v = sgs_quad<false, true, false, true>(d, K, A.E + (size_t)k * d.ne,
                                                            A.r + k * vstride, A.z + k * vstride,
                                                            A.fixn, qx, qy, 0);
#pragma unroll
        for (int kk = 0; kk < MSF_MAX_RHS; ++kk)
          if (kk == k) dots[kk] += v;
      }
#pragma unroll
      for (int k = 0; k < MSF_MAX_RHS; ++k) {
        if (!act[k]) continue;
        const double s = block_sum_all(dots[k], red, tid, PT);
        if (tid == 0) partH[k * G + b] = s;
      }
      __threadfence();
      gsync();
    }
    double beta[MSF_MAX_RHS];
#pragma unroll
    for (int k = 0; k < MSF_MAX_RHS; ++k) {
      beta[k] = 0.0;
      if (act[k]) {
        const double rzn = grid_total(partH + k * G, G, red, tid);
        beta[k] = rzn / rz[k];
        rz[k] = rzn;
      }
    }

    // ---------------- I: p = z + beta p
    for (int item = b; item < nnchunks * nr; item += G) {
      const int k = item / nnchunks, chunk = item - k * nnchunks;
      if (!act[k]) continue;
      const int n = chunk * PT + tid;
      if (n >= d.nn) continue;
      const double2 zv = A.z[k * vstride + n];
      double2 pv = A.p[k * vstride + n];
      pv.x = fma(beta[k], pv.x, zv.x);
      pv.y = fma(beta[k], pv.y, zv.y);
      A.p[k * vstride + n] = pv;
    }
    gsync();
  }
  if (b == 0 && tid == 0) {
    for (int k = 0; k < nr; ++k) {
      A.sc[k].active = 0;
      A.sc[k].iters = iters[k];
      A.sc[k].noconv = noconv[k];
      A.sc[k].rr = rr_last[k];
      A.sc[k].rz = rz[k];
    }
  }
}

// ------------------------------------------------------------------ coarse correction in one launch
// The coarse part of the V-cycle (restriction c = R_c t, cyclic-reduction forward levels, top
// solve, back levels, prolongation z += R_c^T x_c) as ONE cooperative launch with grid-wide
// barriers between the phases.  The phases are latency-bound (later reduction levels touch a
// few m x m blocks), so a 1.2 us barrier replaces a ~4 us kernel boundary per level.
struct CoarseArgs {
  Dims d;
  const double2* t;
  double2* z;
  const double* phi;
  const int* cls_of_agg;
  const int* agg_by_cls;
  int n_restrict;
  double* cb;
  double* cx;
  const double* Dinv;
  const double* Pc;
  const double* Qc;
  const double* PTc;
  const double* QTc;
  const CrLevelDev* levels;
  int nlev;
  const int* top_blocks;
  int topT;
  const double* Atop;
  const PcgScalars* sc;
  int rhs0, nr, gated;
};

template <int KM>
__global__ void __launch_bounds__(PT) k_coarse_coop(CoarseArgs A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sv[];
  __shared__ double rred[PT / 32][MSF_MAX_RHS * KM];
  const Dims& d = A.d;
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  bool act[MSF_MAX_RHS];
  bool any = false;
#pragma unroll
  for (int k = 0; k < MSF_MAX_RHS; ++k) {
    act[k] = k >= A.rhs0 && k < A.rhs0 + A.nr && (!A.gated || A.sc[k].active);
    any |= act[k];
  }
  if (!any) return;   // identical decision in every CTA: no barrier is reached
  // restriction
  for (int item = b; item < A.n_restrict; item += G)
    restrict_agg<KM>(d, A.t, A.phi, A.cls_of_agg, A.cb, A.agg_by_cls[item], act, PT, tid, rred);
  grid.sync();
  const int nrc = (d.mc + CR_ROWS - 1) / CR_ROWS;
  const size_t per = (size_t)d.mc * d.mc;
  const int k0 = A.rhs0, nk = A.nr;
  for (int l = 0; l < A.nlev; ++l) {
    const CrLevelDev L = A.levels[l];
    if (L.s == 0) continue;
    for (int item = b; item < nrc * L.nsurv * nk; item += G) {
      const int k = k0 + item / (nrc * L.nsurv), rest = item - (k - k0) * (nrc * L.nsurv);
      if (!act[k]) continue;
      const int si = rest / nrc, rc = rest - (rest / nrc) * nrc;
      const int i = L.surv[3 * si], il = L.surv[3 * si + 1], ir = L.surv[3 * si + 2];
      cr_forward_rows(d, i, il, ir, rc * CR_ROWS, A.Qc + ((size_t)k * d.nbc + max(il, 0)) * per,
                      A.Pc + ((size_t)k * d.nbc + max(ir, 0)) * per, A.cb + (size_t)k * d.nbc * d.mc,
                      sv, tid, PT);
    }
    grid.sync();
  }
  {
    const int n = A.topT * d.mc, nrt = (n + CR_ROWS - 1) / CR_ROWS;
    for (int item = b; item < nrt * nk; item += G) {
      const int k = k0 + item / nrt, rc = item - (k - k0) * nrt;
      if (!act[k]) continue;
      top_solve_rows(d, A.top_blocks, A.topT, A.Atop + (size_t)k * A.topT * A.topT * per,
                     A.cb + (size_t)k * d.nbc * d.mc, A.cx + (size_t)k * d.nbc * d.mc,
                     rc * CR_ROWS, sv, tid, PT);
    }
    grid.sync();
  }
  for (int l = A.nlev - 1; l >= 0; --l) {
    const CrLevelDev L = A.levels[l];
    for (int item = b; item < nrc * L.nelim * nk; item += G) {
      const int k = k0 + item / (nrc * L.nelim), rest = item - (k - k0) * (nrc * L.nelim);
      if (!act[k]) continue;
      const int ei = rest / nrc, rc = rest - (rest / nrc) * nrc;
      const int kb = L.elim[3 * ei], kl = L.elim[3 * ei + 1], kr = L.elim[3 * ei + 2];
      const size_t blk = ((size_t)k * d.nbc + kb) * per;
      cr_back_rows(d, kb, kl, kr, rc * CR_ROWS, A.Dinv + blk, A.PTc + blk, A.QTc + blk,
                   A.cb + (size_t)k * d.nbc * d.mc, A.cx + (size_t)k * d.nbc * d.mc, sv, tid, PT);
    }
    grid.sync();
  }
  // prolongation, one node per thread (all active realisations)
  const int nnchunks = (d.nn + PT - 1) / PT;
  for (int item = b; item < nnchunks; item += G) {
    const int n = item * PT + tid;
    if (n < d.nn) prolong_node<KM>(d, A.phi, A.cls_of_agg, A.cx, A.z, n / d.nny, n - (n / d.nny) * d.nny, act);
  }
}

template <int KM>
int launch_coarse_coop_km(msf_ctx* c, int rhs0, int nr, const double* t, double* z, bool gated) {
  const Dims& d = c->dl;
  const size_t smem = (size_t)std::max(3, c->top_T) * d.mc * sizeof(double);
  int& G = c->coop_grid;   // CTAs per launch (all resident), computed once per context
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_coarse_coop<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (G == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_coarse_coop<KM>, PT, smem);
    int cap = 4;
    if (const char* e = std::getenv("MSF_COARSE_COOP_CTAS")) cap = std::max(1, std::atoi(e));
    G = sms * std::max(1, std::min(per, cap));
  }
  CoarseArgs A;
  A.d = d;
  A.t = (const double2*)t;
  A.z = (double2*)z;
  A.phi = c->phi;
  A.cls_of_agg = c->cls_of_agg_d;
  A.agg_by_cls = c->agg_by_cls_d;
  A.n_restrict = c->n_restrict;
  A.cb = c->cb;
  A.cx = c->cx;
  A.Dinv = c->Dinv;
  A.Pc = c->Pc;
  A.Qc = c->Qc;
  A.PTc = c->PTc;
  A.QTc = c->QTc;
  A.levels = (const CrLevelDev*)c->cr_levels_d;
  A.nlev = (int)c->cr.size();
  A.top_blocks = c->top_blocks_d;
  A.topT = c->top_T;
  A.Atop = c->Atop;
  A.sc = c->sc;
  A.rhs0 = rhs0;
  A.nr = nr;
  A.gated = gated ? 1 : 0;
  void* args[] = {&A};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_coarse_coop<KM>, dim3(G), dim3(PT), args,
                                              smem, c->stream);
  MSF_LAUNCHED(c);
  return msf_cuda_check(c, e, "cudaLaunchCooperativeKernel(k_coarse_coop)");
}

template <int KM>
int launch_persistent_km(msf_ctx* c, int nr) {
  const Dims& d = c->d;
  const size_t smem = std::max(sizeof(TileSmem),
                               (size_t)std::max(3, c->top_T) * d.mc * sizeof(double));
  cudaFuncSetAttribute(k_pcg_persistent<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_persistent<KM>, PT, smem);
  if (oe != cudaSuccess || per < 1)
    return msf_fail(c, MSF_ERR_CUDA, std::string("persistent PCG kernel cannot be resident: ") +
                                         cudaGetErrorString(oe) + " (blocks/SM " +
                                         std::to_string(per) + ", smem " + std::to_string(smem) + ")");
  const int G = sms * std::min(per, PMINB);
  if ((size_t)G * 3 * MSF_MAX_RHS > (size_t)c->max_partials * d.R + MSF_PERSIST_PARTIALS)
    return msf_fail(c, MSF_ERR_ARG, "partials buffer too small for the persistent grid");
  PersistArgs A;
  A.d = d;
  A.E = c->E;
  A.fixn = c->fixn;
  A.u = (double2*)c->u;
  A.r = (double2*)c->r;
  A.z = (double2*)c->z;
  A.p = (double2*)c->pv;
  A.q = (double2*)c->q;
  A.t = (double2*)c->t;
  A.phi = c->phi;
  A.cls_of_agg = c->cls_of_agg_d;
  A.agg_by_cls = c->agg_by_cls_d;
  A.cb = c->cb;
  A.cx = c->cx;
  A.Dinv = c->Dinv;
  A.Pc = c->Pc;
  A.Qc = c->Qc;
  A.PTc = c->PTc;
  A.QTc = c->QTc;
  A.levels = (const CrLevelDev*)c->cr_levels_d;
  A.nlev = (int)c->cr.size();
  A.top_blocks = c->top_blocks_d;
  A.topT = c->top_T;
  A.Atop = c->Atop;
  A.sc = c->sc;
  A.part = c->partials;
  A.nr = nr;
  A.prof = (unsigned long long*)c->prof_d;
  K0Mat K = c->K0;
  void* args[] = {&A, &K};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_pcg_persistent<KM>, dim3(G), dim3(PT), args,
                                              smem, c->stream);
  MSF_LAUNCHED(c);
  return msf_cuda_check(c, e, "cudaLaunchCooperativeKernel(k_pcg_persistent)");
}

}  // namespace

// Device table of the cyclic-reduction levels for the persistent kernel.
size_t cr_levels_dev_bytes(int nlev) { return (size_t)nlev * sizeof(CrLevelDev); }

void fill_cr_levels_dev(const std::vector<CrLevel>& cr, void* host_buf) {
  CrLevelDev* h = (CrLevelDev*)host_buf;
  for (size_t l = 0; l < cr.size(); ++l) {
    h[l].s = cr[l].s;
    h[l].nsurv = (int)cr[l].surv.size();
    h[l].nelim = (int)cr[l].elim.size();
    h[l].surv = cr[l].surv_d;
    h[l].elim = cr[l].elim_d;
  }
}

int launch_coarse_coop(msf_ctx* c, int rhs0, int nr, const double* t, double* z, bool gated) {
  if (c->d.kmax <= 4) return launch_coarse_coop_km<4>(c, rhs0, nr, t, z, gated);
  if (c->d.kmax <= 8) return launch_coarse_coop_km<8>(c, rhs0, nr, t, z, gated);
  return launch_coarse_coop_km<16>(c, rhs0, nr, t, z, gated);
}

int launch_pcg_persistent(msf_ctx* c, int nr) {
  if (c->d.kmax <= 4) return launch_persistent_km<4>(c, nr);
  if (c->d.kmax <= 8) return launch_persistent_km<8>(c, nr);
  return launch_persistent_km<16>(c, nr);
}
