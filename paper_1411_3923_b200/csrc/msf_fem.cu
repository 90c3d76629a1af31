// Matrix-free Q4 stiffness operator, multicolour symmetric Gauss-Seidel phases and the PCG
// vector kernels of the B200 MsFEM path (the streaming sweep of msf_sgsw.cu runs the same
// Gauss-Seidel node arithmetic, msfk::gs_node).
//
//   * y = P K(xbar) P x  with  K = sum_e (Emin + xbar_e^p (E0-Emin)) K0   (Eq. 4-5,
//     lines 73/84; reading R2: Dirichlet DOFs eliminated).  Node-centric gather: each thread
//     owns one node, reads the 4 adjacent element moduli and the 3x3 nodal neighbourhood
//     from a shared-memory tile with a one-node halo (coalesced double2 loads along y).
//   * Gauss-Seidel in the 4-colour node order of reading R7 (PAPER.md line 146 does not fix
//     an order): nodes of one colour share no element, so a colour is one parallel sweep;
//     one symmetric sweep = 7 launches F0 F1 F2 F3B3 B2 B1 B0.
//   * PCG dot products: warp-shuffle + shared-memory block reduction, per-block partials,
//     the last block to finish reduces the partials in a fixed order (deterministic) and
//     updates the per-realisation scalars (alpha, beta, convergence) on the device.
#include <cuda.h>            // CUtensorMap (TMA descriptors)
#include <cudaTypedefs.h>    // PFN_cuTensorMapEncodeTiled

#include <cstring>
#include <cstdlib>
#include <string>

#include "msf_kern.cuh"

using namespace msfk;

namespace {

constexpr int NTHR = 256;   // threads per CTA of the operator and colour-phase kernels

// ------------------------------------------------------------------ sliding-window operator apply
// Thread per (node row iy, run of KX consecutive node columns): the 3x3 neighbourhood of x and
// the 2x2 element moduli slide along the columns in registers, so a node costs three
// coalesced double2 loads (its new column, rows iy-1..iy+1), two moduli and almost no index
// arithmetic.  (ncu, configs[4]: the one-node-per-thread form below is issue-bound, 67% of
// issue slots on address and bounds arithmetic for 13 loads per node, at 2.3 TB/s.)
template <int MODE, int KX>
__global__ void __launch_bounds__(NTHR) k_apply_sw(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                   const double2* __restrict__ xall,
                                                   double2* __restrict__ yall,
                                                   const double2* __restrict__ ball,
                                                   const uint8_t* __restrict__ fixn, PcgScalars* sc,
                                                   double* partials, unsigned* counters, int rhs0,
                                                   int gated, int dot, int max_partials,
                                                   double* dsum, double* apart) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.z;
  if (gated && !sc[rhs].active) return;
  __shared__ double red[NTHR / 32 + 1];
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int iy = blockIdx.x * blockDim.x + threadIdx.x;
  const int ix0 = (blockIdx.y * blockDim.y + threadIdx.y) * KX;
  const double* E = Eall + (size_t)rhs * d.estride;
  const double2* x = xall + (size_t)rhs * d.nn;
  double dv = 0.0;
  if (iy < d.nny && ix0 < d.nnx) {
    const bool ylo = iy >= 1, yhi = iy + 1 < d.nny;   // node rows iy-1, iy+1 exist
    const bool ehi = iy < d.nely;                      // element row iy exists (iy-1: ylo)
    const double2 zero = make_double2(0.0, 0.0);
    double2 w[3][3];  // node (ix-1+i, iy-1+j)
    double e[2][2];   // element (ix-1+i, iy-1+j)
    auto load_col = [&](int gx, double2 (&col)[3]) {
      if (gx >= 0 && gx < d.nnx) {
        const double2* p = x + (size_t)gx * d.nny + iy;
        col[0] = ylo ? __ldg(p - 1) : zero;
        col[1] = __ldg(p);
        col[2] = yhi ? __ldg(p + 1) : zero;
      } else {
        col[0] = col[1] = col[2] = zero;
      }
    };
    auto load_ecol = [&](int ex, double (&ec)[2]) {
      if (ex >= 0 && ex < d.nelx) {
        const double* p = E + (size_t)ex * d.nely + iy;
        ec[0] = ylo ? __ldg(p - 1) : 0.0;
        ec[1] = ehi ? __ldg(p) : 0.0;
      } else {
        ec[0] = ec[1] = 0.0;
      }
    };
    load_col(ix0 - 1, w[0]);
    load_col(ix0, w[1]);
    load_ecol(ix0 - 1, e[0]);
#pragma unroll
    for (int s = 0; s < KX; ++s) {
      const int ix = ix0 + s;
      load_col(ix + 1, w[2]);
      load_ecol(ix, e[1]);
      if (ix < d.nnx) {
        double ox, oy, dxx, dxy, dyx, dyy;
        apply_node(K, e, w, ox, oy, dxx, dxy, dyx, dyy);
        const size_t n = (size_t)ix * d.nny + iy;
        const uint8_t fm = fixn[n];
        double2 out;
        if (MODE == 1) {
          const double2 bb = ball[(size_t)rhs * d.nn + n];
          out = make_double2(bb.x - ox, bb.y - oy);
        } else {
          out = make_double2(ox, oy);
        }
        if (fm & 1) out.x = 0.0;
        if (fm & 2) out.y = 0.0;
        yall[(size_t)rhs * d.nn + n] = out;
        dv += w[1][1].x * out.x + w[1][1].y * out.y;
      }
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        w[0][j] = w[1][j];
        w[1][j] = w[2][j];
      }
      e[0][0] = e[1][0];
      e[0][1] = e[1][1];
    }
  }
  if (dot == 2) {
    // partial only (no fence / ticket): the consumer (k_update_f0) reduces the partials
    const double s = block_sum_all(dv, red, tid, NTHR);
    if (tid == 0) apart[(size_t)rhs * max_partials + blockIdx.y * gridDim.x + blockIdx.x] = s;
  } else if (dot) {
    const double s = block_sum_all(dv, red, tid, NTHR);
    const unsigned nblk = gridDim.x * gridDim.y;
    const int slot = blockIdx.y * gridDim.x + blockIdx.x;
    if (arrive_last(s, partials + (size_t)rhs * max_partials, slot, counters + rhs * 8, nblk, tid)) {
      const double tot = reduce_partials(partials + (size_t)rhs * max_partials, nblk, red, tid, NTHR);
      if (tid == 0) {
        fin_or_park(sc, dsum, rhs, FIN_PQ, tot, 0);
        counters[rhs * 8] = 0;
      }
    }
  }
}

// ------------------------------------------------------------------ TMA-fed operator apply
// Persistent CTAs stream halo'd tiles of x (10 x 128 node columns x rows, double2, from row
// y0-1) and of the moduli (9 x 128, from row y0-2: the start of a box's inner dimension must
// be 16-byte aligned) through a 3-stage shared-memory ring: one thread issues both
// cp.async.bulk.tensor loads of a stage (completion counted on an mbarrier in bytes) while
// the CTA computes the tile two stages back.  The tensor maps zero-fill outside the grid, so
// the stencil needs no bounds logic; in flight data lives in shared memory, not registers.
// Each thread slides along 4 node columns of one row (3 new double2 + 2 moduli per node from
// shared memory, conflict-free).  Tiles: 8 columns x 126 rows of outputs.
constexpr int TMA_TX = 8, TMA_TY = 126, TMA_STAGES = 3;
constexpr int TMA_XS = (TMA_TX + 2) * 256;   // doubles per stage: x tile [10][128] double2
constexpr int TMA_ES = (TMA_TX + 1) * 128;   //                    E tile [9][128]
constexpr int TMA_STAGE = TMA_XS + TMA_ES;
constexpr size_t TMA_SMEM = (size_t)TMA_STAGES * TMA_STAGE * sizeof(double) + 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(NTHR, 2) k_apply_tma(const __grid_constant__ CUtensorMap tmx,
                                                      const __grid_constant__ CUtensorMap tme, Dims d,
                                                      K0Mat K, const double2* __restrict__ ball,
                                                      double2* __restrict__ yall,
                                                      const uint8_t* __restrict__ fixn, PcgScalars* sc,
                                                      double* partials, unsigned* counters, int rhs0,
                                                      int nr, int gated, int dot, int max_partials,
                                                      double* dsum, double* apart) {
  // persistent grid: the dependent kernel is signalled after the tile loop (at entry its
  // early CTAs competed with the resident tiles: +2% per PCG iteration on configs[4])
  extern __shared__ __align__(128) unsigned char tsm_raw[];
  // stage ring 128-byte aligned by hand (static shared memory precedes the dynamic window)
  double* tsm = reinterpret_cast<double*>(tsm_raw + ((128u - (smem_u32(tsm_raw) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t full[TMA_STAGES];
  __shared__ double red[NTHR / 32 + 1];
  const int tid = threadIdx.x;
  const int ntx = (d.nnx + TMA_TX - 1) / TMA_TX, nty = (d.nny + TMA_TY - 1) / TMA_TY;
  const int per = ntx * nty, ntiles = per * nr;
  if (tid == 0) {
    for (int s = 0; s < TMA_STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();   // x (and the realisation flags) come from the preceding kernels
  // the CTA's tiles t = blockIdx.x + k gridDim.x (y fastest within a column strip, realisation
  // slowest); tiles of converged realisations are skipped identically by every thread
  auto active = [&](int t) { return !gated || sc[rhs0 + t / per].active; };
  auto next_tile = [&](int t) {
    for (t += gridDim.x; t < ntiles && !active(t); t += gridDim.x) {}
    return t;
  };
  int t_issue = blockIdx.x;
  if (t_issue < ntiles && !active(t_issue)) t_issue = next_tile(t_issue);
  int n_issued = 0;
  auto issue = [&]() {   // thread 0: next active tile into stage n_issued % STAGES
    if (t_issue >= ntiles) return;
    const int rr = t_issue / per, tl = t_issue - rr * per;
    const int tx = tl / nty, ty = tl - tx * nty;
    const int x0 = tx * TMA_TX, y0 = ty * TMA_TY;
    const int st = n_issued % TMA_STAGES;
    double* base = tsm + st * TMA_STAGE;
    mbar_expect_tx(&full[st], TMA_STAGE * sizeof(double));
    tma_load_3d(base, &tmx, 2 * (y0 - 1), x0 - 1, rhs0 + rr, &full[st]);
    tma_load_3d(base + TMA_XS, &tme, y0 - 2, x0 - 1, rhs0 + rr, &full[st]);
    ++n_issued;
    t_issue = next_tile(t_issue);
  };
  if (tid == 0)
    for (int s = 0; s < TMA_STAGES; ++s) issue();
  double dv[MSF_MAX_RHS] = {0.0, 0.0, 0.0, 0.0};
  const int r = tid & 127, lc0 = (tid >> 7) * 4;
  int t = blockIdx.x;
  if (t < ntiles && !active(t)) t = next_tile(t);
  for (int n_used = 0; t < ntiles; ++n_used, t = next_tile(t)) {
    const int st = n_used % TMA_STAGES;
    mbar_wait(&full[st], (uint32_t)(n_used / TMA_STAGES) & 1u);
    const int rr = t / per, tl = t - rr * per;
    const int tx = tl / nty, ty = tl - tx * nty;
    const int x0 = tx * TMA_TX, y0 = ty * TMA_TY;
    const int rhs = rhs0 + rr, iy = y0 + r;
    const double2* xs = reinterpret_cast<const double2*>(tsm + st * TMA_STAGE);   // [10][128]
    const double* es = tsm + st * TMA_STAGE + TMA_XS;                              // [9][128]
    if (r < TMA_TY && iy < d.nny) {
      // Dirichlet masks of the thread's 4 nodes, loaded before the stencil work (a global
      // load per node issued just before its store was the top stall)
      uint8_t fm4[4];
      double2 bb4[4];   // MODE 1: the right-hand side, likewise loaded up front
#pragma unroll
      for (int sx = 0; sx < 4; ++sx) {
        const int ix = x0 + lc0 + sx;
        const size_t n = (size_t)min(ix, d.nnx - 1) * d.nny + iy;
        fm4[sx] = ix < d.nnx ? fixn[n] : (uint8_t)0;
        if (MODE == 1) bb4[sx] = ball[(size_t)rhs * d.nn + n];
      }
      double2 w[3][3];   // node (ix-1+i, iy-1+j)    = x tile (lc+i, r+j)
      double e[2][2];    // element (ix-1+i, iy-1+j) = E tile (lc+i, r+j+1): the E box starts
                         // at row y0-2 (TMA needs a 16-byte aligned start of the inner dim)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) w[i][j] = xs[(lc0 + i) * 128 + r + j];
      e[0][0] = es[lc0 * 128 + r + 1];
      e[0][1] = es[lc0 * 128 + r + 2];
      double dsum_t = 0.0;
#pragma unroll
      for (int sx = 0; sx < 4; ++sx) {
        const int lc = lc0 + sx, ix = x0 + lc;
#pragma unroll
        for (int j = 0; j < 3; ++j) w[2][j] = xs[(lc + 2) * 128 + r + j];
        e[1][0] = es[(lc + 1) * 128 + r + 1];
        e[1][1] = es[(lc + 1) * 128 + r + 2];
        if (ix < d.nnx) {
          double ox, oy, dxx, dxy, dyx, dyy;
          apply_node(K, e, w, ox, oy, dxx, dxy, dyx, dyy);
          const size_t n = (size_t)ix * d.nny + iy;
          const uint8_t fm = fm4[sx];
          double2 out;
          if (MODE == 1) {
            out = make_double2(bb4[sx].x - ox, bb4[sx].y - oy);
          } else {
            out = make_double2(ox, oy);
          }
          if (fm & 1) out.x = 0.0;
          if (fm & 2) out.y = 0.0;
          yall[(size_t)rhs * d.nn + n] = out;
          dsum_t += w[1][1].x * out.x + w[1][1].y * out.y;
        }
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          w[0][j] = w[1][j];
          w[1][j] = w[2][j];
        }
        e[0][0] = e[1][0];
        e[0][1] = e[1][1];
      }
#pragma unroll
      for (int q = 0; q < MSF_MAX_RHS; ++q)
        if (q == rr) dv[q] += dsum_t;
    }
    __syncthreads();   // every thread is done with this stage
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue();
    }
  }
  pdl_launch();
  if (!dot) return;
#pragma unroll
  for (int q = 0; q < MSF_MAX_RHS; ++q) {
    if (q >= nr) break;
    const int rhs = rhs0 + q;
    if (gated && !sc[rhs].active) continue;   // uniform: no block of this realisation arrives
    const double sblk = block_sum_all(dv[q], red, tid, NTHR);
    if (dot == 2) {
      if (tid == 0) apart[(size_t)rhs * max_partials + blockIdx.x] = sblk;
    } else if (arrive_last(sblk, partials + (size_t)rhs * max_partials, blockIdx.x, counters + rhs * 8,
                           gridDim.x, tid)) {
      const double tot = reduce_partials(partials + (size_t)rhs * max_partials, gridDim.x, red, tid, NTHR);
      if (tid == 0) {
        fin_or_park(sc, dsum, rhs, FIN_PQ, tot, 0);
        counters[rhs * 8] = 0;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ direct-load operator apply
// One node per thread, neighbourhood and moduli loaded straight from global memory through
// L1 (the access pattern of the Gauss-Seidel colour kernel), no shared-memory staging or
// block barrier before the stencil.
template <int MODE>
__global__ void __launch_bounds__(NTHR) k_apply_direct(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                       const double2* __restrict__ xall,
                                                       double2* __restrict__ yall,
                                                       const double2* __restrict__ ball,
                                                       const uint8_t* __restrict__ fixn, PcgScalars* sc,
                                                       double* partials, unsigned* counters, int rhs0,
                                                       int gated, int dot, int max_partials,
                                                       double* dsum, double* apart) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.z;
  if (gated && !sc[rhs].active) return;
  __shared__ double red[NTHR / 32 + 1];
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int ix = blockIdx.y * blockDim.y + threadIdx.y;
  const int iy = blockIdx.x * blockDim.x + threadIdx.x;
  const double* E = Eall + (size_t)rhs * d.estride;
  const double2* x = xall + (size_t)rhs * d.nn;
  double dv = 0.0;
  if (ix < d.nnx && iy < d.nny) {
    double Eloc[2][2];
    double2 zloc[3][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int ex = ix - 1 + a, ey = iy - 1 + c;
        Eloc[a][c] = (ex >= 0 && ex < d.nelx && ey >= 0 && ey < d.nely) ? __ldg(E + (size_t)ex * d.nely + ey) : 0.0;
      }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int gx = ix - 1 + a, gy = iy - 1 + c;
        zloc[a][c] = (gx >= 0 && gx < d.nnx && gy >= 0 && gy < d.nny) ? __ldg(x + (size_t)gx * d.nny + gy)
                                                                      : make_double2(0.0, 0.0);
      }
    double ox, oy, dxx, dxy, dyx, dyy;
    apply_node(K, Eloc, zloc, ox, oy, dxx, dxy, dyx, dyy);
    const size_t n = (size_t)ix * d.nny + iy;
    const uint8_t fm = fixn[n];
    double2 out;
    if (MODE == 1) {
      const double2 bb = ball[(size_t)rhs * d.nn + n];
      out = make_double2(bb.x - ox, bb.y - oy);
    } else {
      out = make_double2(ox, oy);
    }
    if (fm & 1) out.x = 0.0;
    if (fm & 2) out.y = 0.0;
    yall[(size_t)rhs * d.nn + n] = out;
    dv = zloc[1][1].x * out.x + zloc[1][1].y * out.y;
  }
  if (dot == 2) {
    // partial only (no fence / ticket): the consumer (k_update_f0) reduces the partials
    const double s = block_sum_all(dv, red, tid, NTHR);
    if (tid == 0) apart[(size_t)rhs * max_partials + blockIdx.y * gridDim.x + blockIdx.x] = s;
  } else if (dot) {
    const double s = block_sum_all(dv, red, tid, NTHR);
    const unsigned nblk = gridDim.x * gridDim.y;
    const int slot = blockIdx.y * gridDim.x + blockIdx.x;
    if (arrive_last(s, partials + (size_t)rhs * max_partials, slot, counters + rhs * 8, nblk, tid)) {
      const double tot = reduce_partials(partials + (size_t)rhs * max_partials, nblk, red, tid, NTHR);
      if (tid == 0) {
        fin_or_park(sc, dsum, rhs, FIN_PQ, tot, 0);
        counters[rhs * 8] = 0;
      }
    }
  }
}

// ------------------------------------------------------------------ Gauss-Seidel colour phase
// Thread per node quad; see msfk::sgs_quad.  RZ: r.z of the final iterate -> beta (rz_mode 1:
// PCG init, beta = 0; 2: iteration).
template <bool FWD, bool BWD, bool ZERO, bool RZ>
__global__ void __launch_bounds__(NTHR) k_sgs_colour(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                     const double2* __restrict__ rall,
                                                     double2* zall,
                                                     const uint8_t* __restrict__ fixn,
                                                     PcgScalars* sc, double* partials,
                                                     unsigned* counters, int max_partials,
                                                     int rhs0, int gated, int colour,
                                                     int rz_mode, double* dsum) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.z;
  if (gated && !sc[rhs].active) return;
  __shared__ double red[NTHR / 32 + 1];
  const int qx = blockIdx.y * blockDim.y + threadIdx.y;
  const int qy = blockIdx.x * blockDim.x + threadIdx.x;
  const double dot = sgs_quad<FWD, BWD, ZERO, RZ>(d, K, Eall + (size_t)rhs * d.estride,
                                                  rall + (size_t)rhs * d.nn,
                                                  zall + (size_t)rhs * d.nn, fixn, qx, qy, colour);
  if (RZ) {
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const double sblk = block_sum_all(dot, red, tid, NTHR);
    const unsigned nblk = gridDim.x * gridDim.y;
    const int slot = blockIdx.y * gridDim.x + blockIdx.x;
    if (arrive_last(sblk, partials + (size_t)rhs * max_partials, slot, counters + rhs * 8, nblk,
                    tid)) {
      const double tot = reduce_partials(partials + (size_t)rhs * max_partials, nblk, red, tid,
                                         NTHR);
      if (tid == 0) {
        fin_or_park(sc, dsum, rhs, FIN_RZ, tot, rz_mode);
        counters[rhs * 8] = 0;
      }
    }
  }
}


// ------------------------------------------------------------------ PCG vector kernels
constexpr int VB = 256;  // threads per block of the vector kernels

__global__ void __launch_bounds__(VB) k_mask_copy(const double2* __restrict__ x, double2* y,
                                                  const uint8_t* __restrict__ fixn, int nn) {
  for (int i = blockIdx.x * VB + threadIdx.x; i < nn; i += gridDim.x * VB) {
    double2 v = x[i];
    const uint8_t fm = fixn[i];
    if (fm & 1) v.x = 0.0;
    if (fm & 2) v.y = 0.0;
    y[i] = v;
  }
}

// x = 0, r = P f, ||f||^2 -> scalars
__global__ void __launch_bounds__(VB) k_pcg_init(Dims d, const double2* __restrict__ f,
                                                 const uint8_t* __restrict__ fixn,
                                                 double2* uall, double2* rall, PcgScalars* sc,
                                                 double* partials, unsigned* counters,
                                                 int max_partials, double tol, int max_it,
                                                 double* dsum) {
  __shared__ double red[VB / 32 + 1];
  const int rhs = blockIdx.z;
  const int tid = threadIdx.x;
  double2* u = uall + (size_t)rhs * d.nn;
  double2* r = rall + (size_t)rhs * d.nn;
  double s = 0.0;
  for (int i = blockIdx.x * VB + tid; i < d.nn; i += gridDim.x * VB) {
    double2 v = f[i];
    const uint8_t fm = fixn[i];
    if (fm & 1) v.x = 0.0;
    if (fm & 2) v.y = 0.0;
    r[i] = v;
    u[i] = make_double2(0.0, 0.0);
    s += v.x * v.x + v.y * v.y;
  }
  s = block_sum_all(s, red, tid, VB);
  if (arrive_last(s, partials + (size_t)rhs * max_partials, blockIdx.x, counters + rhs * 8,
                  gridDim.x, tid)) {
    const double tot = reduce_partials(partials + (size_t)rhs * max_partials, gridDim.x, red,
                                       tid, VB);
    if (tid == 0) {
      PcgScalars& S = sc[rhs];
      S.tol2 = tol * tol;
      S.iters = 0;
      S.max_it = max_it;
      S.noconv = 0;
      S.rz = 0.0;
      S.alpha = S.beta = S.pq = 0.0;
      fin_or_park(sc, dsum, rhs, FIN_F, tot, 0);
      counters[rhs * 8] = 0;
    }
  }
}

// Fused PCG update + first pre-smoothing colour: thread per node quad, u += alpha p,
// r -= alpha q on the quad's 4 nodes, ||r||^2 (-> convergence, last block), then the
// zero-start forward Gauss-Seidel phase of colour 0 (msfk::sgs_quad<.., ZERO>) with the new r.
__global__ void __launch_bounds__(NTHR) k_update_f0(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                    double2* uall, double2* rall,
                                                    const double2* __restrict__ pall,
                                                    const double2* __restrict__ qall, double2* zall,
                                                    const uint8_t* __restrict__ fixn, PcgScalars* sc,
                                                    double* partials, unsigned* counters,
                                                    int max_partials, double* dsum, int rhs0,
                                                    const double* __restrict__ apart, int napart) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.z;
  if (!sc[rhs].active) return;
  __shared__ double red[NTHR / 32 + 1];
  const int qx = blockIdx.y * blockDim.y + threadIdx.y;
  const int qy = blockIdx.x * blockDim.x + threadIdx.x;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const size_t off = (size_t)rhs * d.nn;
#ifndef MSF_F0_PRELOAD
#define MSF_F0_PRELOAD 0
#endif
  // MSF_F0_PRELOAD 1: the quad's p and q are loaded before alpha is known (overlaps the
  // partial reduction); 0: alpha first (fewer live registers)
  double2 pv[4], qv[4];
  if (MSF_F0_PRELOAD) {
#pragma unroll
    for (int dn = 0; dn < 4; ++dn) {
      const int gx = 2 * qx + (dn & 1), gy = 2 * qy + (dn >> 1);
      if (gx < d.nnx && gy < d.nny) {
        const size_t n = off + (size_t)gx * d.nny + gy;
        pv[dn] = pall[n];
        qv[dn] = qall[n];
      }
    }
  }
  double alpha;
  if (napart > 0) {
    // p.Ap from the operator's per-CTA partials: every CTA sums them in the same fixed order
    // (identical alpha everywhere); CTA 0 records pq and alpha
    const double pq = reduce_partials(apart + (size_t)rhs * max_partials, napart, red, tid, NTHR);
    alpha = sc[rhs].rz / pq;
    if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
      sc[rhs].pq = pq;
      sc[rhs].alpha = alpha;
    }
  } else {
    alpha = sc[rhs].alpha;
  }
  double s = 0.0;
#pragma unroll
  for (int dn = 0; dn < 4; ++dn) {
    const int gx = 2 * qx + (dn & 1), gy = 2 * qy + (dn >> 1);
    if (gx < d.nnx && gy < d.nny) {
      const size_t n = off + (size_t)gx * d.nny + gy;
      const double2 p2 = MSF_F0_PRELOAD ? pv[dn] : pall[n];
      const double2 q2 = MSF_F0_PRELOAD ? qv[dn] : qall[n];
      double2 u2 = uall[n], r2 = rall[n];
      u2.x = fma(alpha, p2.x, u2.x);
      u2.y = fma(alpha, p2.y, u2.y);
      r2.x = fma(-alpha, q2.x, r2.x);
      r2.y = fma(-alpha, q2.y, r2.y);
      uall[n] = u2;
      rall[n] = r2;
      s += r2.x * r2.x + r2.y * r2.y;
    }
  }
  __syncthreads();   // red[] reused below
  sgs_quad<true, false, true, false>(d, K, Eall + (size_t)rhs * d.estride, rall + off, zall + off,
                                     fixn, qx, qy, 0);
  s = block_sum_all(s, red, tid, NTHR);
  const unsigned nblk = gridDim.x * gridDim.y;
  const int slot = blockIdx.y * gridDim.x + blockIdx.x;
  if (arrive_last(s, partials + (size_t)rhs * max_partials, slot, counters + rhs * 8, nblk, tid)) {
    const double tot = reduce_partials(partials + (size_t)rhs * max_partials, nblk, red, tid, NTHR);
    if (tid == 0) {
      fin_or_park(sc, dsum, rhs, FIN_RR, tot, 0);
      counters[rhs * 8] = 0;
    }
  }
}

// PCG scalar update from the all-reduced sums (strip partition): same arithmetic as the
// in-kernel finalisation of the single-GPU path.
__global__ void k_finalize(PcgScalars* sc, const double* __restrict__ dsum, int kind, int rhs0,
                           int nr, int gated, int rz_mode) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + threadIdx.x;
  if (threadIdx.x >= nr) return;
  if (gated && !sc[rhs].active) return;
  fin_scalar(sc[rhs], kind, dsum[kind * MSF_MAX_RHS + rhs], rz_mode);
}

// PCG direction update (reading R9).  mode 0: p = z (init); 1: u += alpha p, then
// p = z + beta p (the solution update of the iteration, deferred to here so that it reads
// the p it needs once); 2: p = z + beta p (strip partition: u was updated by k_update_f0);
// 3: u += alpha p for every realisation, ungated (after the last iteration: the iteration
// that converged skipped mode 1).
__global__ void __launch_bounds__(VB) k_pcg_p(Dims d, const double2* __restrict__ zall,
                                              double2* pall, double2* uall, const PcgScalars* sc,
                                              int mode, int rhs0) {
  pdl_launch();
  pdl_wait();
  const int rhs = rhs0 + blockIdx.z;
  if (mode != 3 && !sc[rhs].active) return;
  const double beta = mode == 0 ? 0.0 : sc[rhs].beta;
  const double alpha = sc[rhs].alpha;
  const double2* z = zall + (size_t)rhs * d.nn;
  double2* p = pall + (size_t)rhs * d.nn;
  double2* u = uall + (size_t)rhs * d.nn;
  for (int i = blockIdx.x * VB + threadIdx.x; i < d.nn; i += gridDim.x * VB) {
    double2 pv = mode == 0 ? make_double2(0.0, 0.0) : p[i];
    if (mode == 1 || mode == 3) {
      double2 uv = u[i];
      uv.x = fma(alpha, pv.x, uv.x);
      uv.y = fma(alpha, pv.y, uv.y);
      u[i] = uv;
    }
    if (mode != 3) {
      const double2 zv = z[i];
      pv.x = fma(beta, pv.x, zv.x);
      pv.y = fma(beta, pv.y, zv.y);
      p[i] = pv;
    }
  }
}

// compliance c = f.u (Eq. 6)
__global__ void __launch_bounds__(VB) k_compliance(Dims d, const double2* __restrict__ f,
                                                   const double2* __restrict__ uall,
                                                   PcgScalars* sc, double* partials,
                                                   unsigned* counters, int max_partials,
                                                   double* dsum) {
  __shared__ double red[VB / 32 + 1];
  const int rhs = blockIdx.z;
  const int tid = threadIdx.x;
  const double2* u = uall + (size_t)rhs * d.nn;
  double s = 0.0;
  for (int i = blockIdx.x * VB + tid; i < d.nn; i += gridDim.x * VB) {
    const double2 a = f[i], b = u[i];
    s += a.x * b.x + a.y * b.y;
  }
  s = block_sum_all(s, red, tid, VB);
  if (arrive_last(s, partials + (size_t)rhs * max_partials, blockIdx.x, counters + rhs * 8,
                  gridDim.x, tid)) {
    const double tot = reduce_partials(partials + (size_t)rhs * max_partials, gridDim.x, red,
                                       tid, VB);
    if (tid == 0) {
      fin_or_park(sc, dsum, rhs, FIN_COMP, tot, 0);
      counters[rhs * 8] = 0;
    }
  }
}

inline int vec_blocks(const Dims& d) {
  // about one node per thread: every thread's loads are in flight at once (a grid-stride loop
  // over a 592-CTA grid chains ~4 dependent round trips per thread at configs[1] size)
  int b = (d.nn + VB - 1) / VB;
  return b < 65535 ? b : 65535;
}

}  // namespace

// ================================================================== host launchers
K0Mat make_K0(double nu) {
  // Published closed form of the unit-modulus plane-stress Q4 element (K0 is
  // the bilinear form of PAPER.md Eq. 3a on one square element; node order
  // (0,0),(1,0),(1,1),(0,1)).  The oracle integrates the same matrix by quadrature.
  const double k[8] = {0.5 - nu / 6.0,           0.125 + nu / 8.0, -0.25 - nu / 12.0,
                       -0.125 + 3.0 * nu / 8.0,  -0.25 + nu / 12.0, -0.125 - nu / 8.0,
                       nu / 6.0,                 0.125 - 3.0 * nu / 8.0};
  static const int idx[8][8] = {{0, 1, 2, 3, 4, 5, 6, 7}, {1, 0, 7, 6, 5, 4, 3, 2},
                                {2, 7, 0, 5, 6, 3, 4, 1}, {3, 6, 5, 0, 7, 2, 1, 4},
                                {4, 5, 6, 7, 0, 1, 2, 3}, {5, 4, 3, 2, 1, 0, 7, 6},
                                {6, 3, 4, 1, 2, 7, 0, 5}, {7, 2, 1, 4, 3, 6, 5, 0}};
  K0Mat K;
  const double s = 1.0 / (1.0 - nu * nu);
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) K.v[i * 8 + j] = s * k[idx[i][j]];
  return K;
}

int apply_partials_needed(const Dims& d) {   // one partial per CTA of k_apply_direct's grid
  const int a = ((d.nny + 31) / 32) * ((d.nnx + 7) / 8);
  return a > 592 ? a : 592;
}

int sgs_colour_partials_needed(const Dims& d) {
  const int hx = (d.nnx + 1) / 2, hy = (d.nny + 1) / 2;
  return ((hy + 31) / 32) * ((hx + 7) / 8);
}

// Fine-grid launchers run on this rank's grid c->dl with the moduli c->E_loc (the whole grid
// on one GPU); reductions park their sums in c->dsum on a strip context.
// TMA descriptors of the operator apply: kind 0 = node vector x (dims 2 nny doubles, nnx
// columns, R realisations), kind 1 = moduli (nely, nelx, R); cached per base pointer.
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)f;
  }();
  return fn;
}

// Copies the descriptor out (the cache vector may reallocate on the next insertion).
static bool tmap_for(msf_ctx* c, const void* base, int kind, CUtensorMap* out) {
  for (const msf_ctx::TmapSlot& t : c->tmaps)
    if (t.ptr == base && t.kind == kind) {
      std::memcpy(out, t.bytes, sizeof(CUtensorMap));
      return true;
    }
  auto enc = tmap_encode();
  if (!enc) return false;
  const Dims& d = c->dl;
  msf_ctx::TmapSlot slot{};
  slot.ptr = base;
  slot.kind = kind;
  static_assert(sizeof(CUtensorMap) <= sizeof(slot.bytes), "tensor map size");
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(slot.bytes);
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r;
  if (kind == 0) {
    const cuuint64_t dims[3] = {(cuuint64_t)2 * d.nny, (cuuint64_t)d.nnx, (cuuint64_t)d.R};
    const cuuint64_t strides[2] = {(cuuint64_t)2 * d.nny * 8, (cuuint64_t)2 * d.nn * 8};
    const cuuint32_t box[3] = {256, TMA_TX + 2, 1};
    r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[3] = {(cuuint64_t)d.nely, (cuuint64_t)d.nelx, (cuuint64_t)d.R};
    const cuuint64_t strides[2] = {(cuuint64_t)d.nely * 8, (cuuint64_t)d.estride * 8};
    const cuuint32_t box[3] = {128, TMA_TX + 1, 1};
    r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return false;
  c->tmaps.push_back(slot);
  std::memcpy(out, slot.bytes, sizeof(CUtensorMap));
  return true;
}

template <int MODE>
static bool launch_apply_tma(msf_ctx* c, int rhs0, int nr, const double* x, double* y,
                             const double* bvec, bool gated, int dmode) {
  const Dims& d = c->dl;
  // 16-byte global strides / base alignment of the moduli map; a grid of at least one tile
  if (!c->apply_tma || (d.nely & 1) || (d.estride & 1) || d.nny < TMA_TY || d.nnx < TMA_TX)
    return false;
  CUtensorMap mx, me;
  if (!tmap_for(c, x, 0, &mx) || !tmap_for(c, c->E_loc, 1, &me)) return false;
  static bool attr = [] {
    cudaFuncSetAttribute(k_apply_tma<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TMA_SMEM);
    return true;
  }();
  (void)attr;
  const long long ntiles = (long long)((d.nnx + TMA_TX - 1) / TMA_TX) * ((d.nny + TMA_TY - 1) / TMA_TY) * nr;
  const int grid = (int)std::min<long long>(ntiles, 2LL * c->n_sm);
  launch_k(k_apply_tma<MODE>, dim3(grid), dim3(NTHR), TMA_SMEM, c->stream, mx, me, d, c->K0,
           (const double2*)bvec, (double2*)y, c->fixn, c->sc, c->partials, c->counters, rhs0, nr,
           gated ? 1 : 0, dmode, c->max_partials, c->dsum, c->apart);
  c->apart_n = dmode == 2 ? grid : 0;
  MSF_LAUNCHED(c);
  return true;
}

// Operator apply (MODE 0) / residual (MODE 1) on this rank's grid: the TMA-fed tile kernel
// when the grid allows it (even nely, >= one 8 x 126 tile), else the sliding-window apply /
// one-node-per-thread residual (odd nely or small grids, e.g. most test grids).
template <int MODE>
static void launch_apply(msf_ctx* c, int rhs0, int nr, const double* x, double* y,
                         const double* bvec, bool gated, bool dot) {
  const Dims& d = c->dl;
  // p.Ap on one GPU: partials only, reduced by the next kernel (the pre-smoothing); strips need
  // the all-reduce, so the last-block finalisation parks the local sum
  const int dmode = !dot ? 0 : c->comm ? 1 : 2;
  if (launch_apply_tma<MODE>(c, rhs0, nr, x, y, bvec, gated, dmode)) return;
  if (MODE == 0) {
    // columns per thread: the longest run that still gives >= 4 CTAs per SM (measured: the
    // residual form, which also streams b, is faster one node per thread)
    const int by = (d.nny + 31) / 32;
    int kx = 8;
    while (kx > 2 && (long long)by * ((d.nnx + 8 * kx - 1) / (8 * kx)) * nr < 4LL * c->n_sm) kx /= 2;
    const dim3 grid(by, (d.nnx + 8 * kx - 1) / (8 * kx), nr);
#define MSF_SW(KX)                                                                                  \
  launch_k(k_apply_sw<MODE, KX>, grid, dim3(32, 8), 0, c->stream, d, c->K0, (const double*)c->E_loc, \
           (const double2*)x, (double2*)y, (const double2*)bvec, c->fixn, c->sc, c->partials,        \
           c->counters, rhs0, gated ? 1 : 0, dmode, c->max_partials, c->dsum, c->apart)
    if (kx == 8) MSF_SW(8);
    else if (kx == 4) MSF_SW(4);
    else MSF_SW(2);
#undef MSF_SW
    c->apart_n = dmode == 2 ? (int)(grid.x * grid.y) : 0;
    MSF_LAUNCHED(c);
    return;
  }
  launch_k(k_apply_direct<MODE>, dim3((d.nny + 31) / 32, (d.nnx + 7) / 8, nr), dim3(32, 8), 0,
           c->stream, d, c->K0, (const double*)c->E_loc, (const double2*)x, (double2*)y,
           (const double2*)bvec, c->fixn, c->sc, c->partials, c->counters, rhs0, gated ? 1 : 0,
           dmode, c->max_partials, c->dsum, c->apart);
  c->apart_n = dmode == 2 ? ((d.nny + 31) / 32) * ((d.nnx + 7) / 8) : 0;
  MSF_LAUNCHED(c);
}

void launch_matvec(msf_ctx* c, int rhs0, int nr, const double* x, double* y, bool gated,
                   bool dot_pq) {
  launch_apply<0>(c, rhs0, nr, x, y, nullptr, gated, dot_pq);
}

void launch_residual(msf_ctx* c, int rhs0, int nr, const double* b, const double* x, double* y,
                     bool gated) {
  launch_apply<1>(c, rhs0, nr, x, y, b, gated, false);
}

void launch_sgs_phase(msf_ctx* c, int rhs0, int nr, const double* r, double* z, bool gated,
                      int phase, int rz_mode) {
  const Dims& d = c->dl;
  const int hx = (d.nnx + 1) / 2, hy = (d.nny + 1) / 2;
  dim3 blk(32, 8);
  dim3 grd((hy + 31) / 32, (hx + 7) / 8, nr);
  const int g = gated ? 1 : 0;
  // One-wave grids (configs[1] at one realisation: 585 CTAs) are spread at most 4 CTAs per
  // SM by an unused 46 KB dynamic shared-memory request (the 48-register kernel would take 5
  // per SM and leave SMs idle): configs[1] PCG 115.2 -> 114.3 ms.  MSF_SGS_CAP=0: off.
  static const bool cap_env = [] {
    const char* e = std::getenv("MSF_SGS_CAP");
    return !(e && std::string(e) == "0");
  }();
  const size_t smem = (cap_env && (long long)grd.x * grd.y * nr <= 4LL * c->n_sm) ? 46 * 1024 : 0;
#define MSF_SGS(F, B, Z, RZ, col)                                                               \
  launch_k(k_sgs_colour<F, B, Z, RZ>, grd, blk, smem, c->stream, d, c->K0, c->E_loc,           \
           (const double2*)r, (double2*)z, c->fixn, c->sc, c->partials, c->counters,            \
           c->max_partials, rhs0, g, (int)(col), rz_mode, c->dsum);                               \
  break
  switch (phase) {
    case 0: MSF_SGS(true, false, true, false, 0);
    case 1: MSF_SGS(true, false, false, false, 0);
    case 2: MSF_SGS(true, false, false, false, 1);
    case 3: MSF_SGS(true, false, false, false, 2);
    case 4: MSF_SGS(true, true, false, false, 3);
    case 5: MSF_SGS(false, true, false, false, 2);
    case 6: MSF_SGS(false, true, false, false, 1);
    default:
      if (rz_mode) {
        MSF_SGS(false, true, false, true, 0);
      } else {
        MSF_SGS(false, true, false, false, 0);
      }
  }
#undef MSF_SGS
  MSF_LAUNCHED(c);
}

// One symmetric GS sweep as 7 colour launches F0 F1 F2 F3B3 B2 B1 B0.  zero_start: z = 0 on
// entry (fused into F0); rz_mode != 0: r.z and beta fused into B0.
void launch_sgs_sweep(msf_ctx* c, int rhs0, int nr, const double* r, double* z, bool gated,
                      bool zero_start, int rz_mode, bool skip_f0) {
  if (zero_start)
    launch_sgs_phase(c, rhs0, nr, r, z, gated, 0, 0);
  else if (!skip_f0)
    launch_sgs_phase(c, rhs0, nr, r, z, gated, 1, 0);
  for (int ph = 2; ph <= 7; ++ph) launch_sgs_phase(c, rhs0, nr, r, z, gated, ph, rz_mode);
}

void launch_sgs(msf_ctx* c, int rhs0, int nr, const double* r, double* z, bool gated) {
  launch_sgs_sweep(c, rhs0, nr, r, z, gated, false, 0, false);
}

void launch_update_f0(msf_ctx* c, int rhs0, int nr) {
  const Dims& d = c->dl;
  const int hx = (d.nnx + 1) / 2, hy = (d.nny + 1) / 2;
  dim3 grd((hy + 31) / 32, (hx + 7) / 8, nr);
  // alpha from the operator's partials when the preceding matvec left them (one GPU)
  const int napart = c->apart_n;
  c->apart_n = 0;
  // one-wave grids (configs[1] at one realisation: 585 CTAs) spread at most 4 CTAs per SM:
  // an unused 46 KB dynamic shared-memory request caps the residency (MSF_F0_CAP=0: off)
  static const bool cap_env = [] {
    const char* e = std::getenv("MSF_F0_CAP");
    return !(e && std::string(e) == "0");
  }();
  const size_t cap = (cap_env && (long long)grd.x * grd.y * nr <= 4LL * c->n_sm) ? 46 * 1024 : 0;
  launch_k(k_update_f0, grd, dim3(32, 8), cap, c->stream,
           d, c->K0, c->E_loc, (double2*)c->u, (double2*)c->r, (const double2*)c->pv,
           (const double2*)c->q, (double2*)c->z, c->fixn, c->sc, c->partials, c->counters,
           c->max_partials, c->dsum, rhs0, (const double*)c->apart, napart);
  MSF_LAUNCHED(c);
}

void launch_finalize(msf_ctx* c, int kind, int rhs0, int nr, bool gated, int rz_mode) {
  launch_k(k_finalize, dim3(1), dim3(32), 0, c->stream, c->sc, (const double*)c->dsum, kind, rhs0,
           nr, gated ? 1 : 0, rz_mode);
  MSF_LAUNCHED(c);
}

void launch_mask_copy(msf_ctx* c, const double* x, double* y, int nn) {
  int b = (nn + VB - 1) / VB;
  b = b < 592 ? b : 592;
  k_mask_copy<<<b, VB, 0, c->stream>>>((const double2*)x, (double2*)y, c->fixn, nn);
  MSF_LAUNCHED(c);
}

void launch_pcg_init(msf_ctx* c, int nr, double tol, int max_it) {
  k_pcg_init<<<dim3(vec_blocks(c->dl), 1, nr), VB, 0, c->stream>>>(
      c->dl, (const double2*)c->f, c->fixn, (double2*)c->u, (double2*)c->r, c->sc, c->partials,
      c->counters, c->max_partials, tol, max_it, c->dsum);
  MSF_LAUNCHED(c);
}

void launch_pcg_p(msf_ctx* c, int rhs0, int nr, int mode) {
  launch_k(k_pcg_p, dim3(vec_blocks(c->dl), 1, nr), dim3(VB), 0, c->stream,
           c->dl, (const double2*)c->z, (double2*)c->pv, (double2*)c->u, (const PcgScalars*)c->sc,
           mode, rhs0);
  MSF_LAUNCHED(c);
}

void launch_compliance(msf_ctx* c, int nr) {
  k_compliance<<<dim3(vec_blocks(c->dl), 1, nr), VB, 0, c->stream>>>(
      c->dl, (const double2*)c->f, (const double2*)c->u, c->sc, c->partials, c->counters,
      c->max_partials, c->dsum);
  MSF_LAUNCHED(c);
}
