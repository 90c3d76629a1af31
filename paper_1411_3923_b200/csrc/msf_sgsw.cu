// Warp-synchronous streaming symmetric Gauss-Seidel sweep: the seven colour phases F0 F1 F2 F3B3
// B2 B1 B0 of one symmetric sweep (readings R7, R8; "single pre- and
// post-smoothing using symmetric Gauss-Seidel") with the iterate held in REGISTERS.
//
// The first streaming form (k_sgs_stream, earlier in round 2) kept a 20-column ring of z in shared memory and read the 3x3
// neighbourhood of every node update from it (10 LDS.128 per update; the shared-memory data
// pipe, 54% busy, was its most loaded unit, and the CTA barrier per step kept the four phase
// warps in lock step).  Here every WARP owns a band of 64 node rows (two per lane: rows
// Yb + 2 lane and Yb + 2 lane + 1; the 48 middle rows are the band's, 8 above and below are
// halo) and a run of node columns, and marches along x two columns per step.  Each lane holds
// its two rows of a 9-column window of z in registers.  At step s (even) the phases run one
// after the other on columns s, s-1, ..., s-6 (phase k on column s + 1 - k: the column
// parities are the colours'), so every phase finds its predecessor phase complete on the
// column to its right and its successor not yet started on the column to its left -- the
// dependency order of the colour-phase launches without any barrier.  Of the 3x3 neighbourhood
// six values are the lane's own registers; the row above (even rows) or below (odd rows) comes
// from the neighbouring lane by warp shuffle.  r and the moduli wait in a per-warp ring in
// shared memory (cp.async four columns ahead; thread-private slots except the moduli row of the
// lane below), z (or q) and the Dirichlet bits arrive in registers one step ahead.
//
// Halo rows / columns (7 each side, one per phase) are swept redundantly from the same inputs
// with the same arithmetic (msfk::gs_node), so the result is bitwise the colour-phase sweep's.
// Variants: ZERO (z = 0 on entry), UPD (r' = r - alpha q fused in front, r' to
// a second buffer, ||r'||^2 -> convergence), RZ (r.z of the result -> beta).
#include "msf_kern.cuh"

#include <algorithm>
#include <vector>

using namespace msfk;

namespace {

#ifndef MSF_SW_WARPS
#define MSF_SW_WARPS 8
#endif
#ifndef MSF_SW_PF
#define MSF_SW_PF 1
#endif
constexpr int SW_WARPS = MSF_SW_WARPS;   // resident warps per SM; ONE warp per CTA: the band / run indices, the loop
                                         // bounds and the shuffles are then provably warp-uniform for the compiler
constexpr int SW_PF = MSF_SW_PF;         // r / moduli copies run SW_PF steps (2 SW_PF columns) ahead
constexpr int SW_T = 32;
constexpr int SW_BAND = 48;           // band rows: warp rows [SW_LO, SW_LO + SW_BAND)
constexpr int SW_LO = 8;
constexpr int SW_NR = 10 + 2 * SW_PF;    // ring columns: 9 in the window + 2 SW_PF in flight (+1: even)
constexpr int SW_DEP = 7;             // phases per sweep = halo width

struct SwSlot {
  double2 r[2][32];   // [row parity][lane]
  double e[2][34];    // [row parity][lane + 1] (index 0: the row of "lane -1", zero)
};
struct SwRing {
  SwSlot s[SW_NR];
};
constexpr size_t SW_SMEM = sizeof(SwRing);

__device__ __forceinline__ uint32_t sw_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sw_cpa16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sw_u32(dst)), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void sw_cpa8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sw_u32(dst)), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void sw_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void sw_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ double2 shfl_up2(double2 v) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ double2 shfl_down2(double2 v) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}

// One colour phase on window column J (node column s + 1 - J), row parity P of every lane.
// sc / sm: ring slots of node column c = s + 1 - J and of c - 1.
// NZ: the neighbours that may be nonzero (apply_node; a sweep from z = 0 knows which colours
// are still untouched).
// nb0 / nb1 / nb2: the neighbouring lane's row (above for P = 0, below for P = 1) of node columns
// c - 1 / c / c + 1, shuffled by the caller (successive phases share them).
template <int J, int P, bool FWD, bool BWD, bool Z0, int NZ = 0x1ff>
__device__ __forceinline__ void sw_phase(const K0Mat& K, double2 (&W)[9][2], const SwRing& S, int sc,
                                         int sm, unsigned long long fw, int lane, double2 nb0,
                                         double2 nb1, double2 nb2) {
  double Eloc[2][2];
  double2 zloc[3][3];
  // moduli of elements (c-1 .. c, y-1 .. y): y-1 is the odd row of the lane below (P = 0)
  Eloc[0][0] = S.s[sm].e[1 - P][lane + P];
  Eloc[0][1] = S.s[sm].e[P][lane + 1];
  Eloc[1][0] = S.s[sc].e[1 - P][lane + P];
  Eloc[1][1] = S.s[sc].e[P][lane + 1];
  if (Z0) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) zloc[a][b] = make_double2(0.0, 0.0);
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int j = J + 1 - a;   // node column c - 1 + a
      const double2 nb = a == 0 ? nb0 : a == 1 ? nb1 : nb2;
      if (P == 0) {
        zloc[a][0] = nb;
        zloc[a][1] = W[j][0];
        zloc[a][2] = W[j][1];
      } else {
        zloc[a][0] = W[j][0];
        zloc[a][1] = W[j][1];
        zloc[a][2] = nb;
      }
    }
  }
  const double2 rv = S.s[sc].r[P][lane];
  const uint8_t fm = (uint8_t)((fw >> (4 * J + 2 * P)) & 3ull);
  W[J][P] = gs_node<FWD, BWD, Z0, NZ>(K, Eloc, zloc, rv, fm);
}

template <bool ZERO, bool UPD, bool RZ>
__global__ void __launch_bounds__(SW_T, SW_WARPS)
    k_sgs_warp(Dims d, K0Mat K, const double* __restrict__ Eall, const double2* __restrict__ rall,
               double2* routall, const double2* __restrict__ zinall, double2* zall,
               const double2* __restrict__ qall, const uint8_t* __restrict__ fixs, int fs_col,
               int fs_plane, PcgScalars* sc, double* partials, unsigned* counters, int max_partials,
               double* dsum, const double* __restrict__ apart, int napart, int rhs0, int gated,
               int rz_mode, int nyb, int nxb, int nextra) {
  extern __shared__ __align__(16) unsigned char sw_raw[];
  __shared__ double red[SW_T / 32 + 1];
  pdl_wait();
  const int rhs = rhs0 + blockIdx.y;
  if (gated && !sc[rhs].active) return;
  const int tid = threadIdx.x, lane = tid;
  SwRing& S = *reinterpret_cast<SwRing*>(sw_raw);

  double alpha = 0.0;
  if (UPD) {
    // p.Ap from the operator's per-CTA partials: every CTA sums them in the same fixed order
    if (napart > 0) {
      const double pq = reduce_partials(apart + (size_t)rhs * max_partials, napart, red, tid, SW_T);
      alpha = sc[rhs].rz / pq;
      if (tid == 0 && blockIdx.x == 0) {
        sc[rhs].pq = pq;
        sc[rhs].alpha = alpha;
      }
    } else {
      alpha = sc[rhs].alpha;
    }
  }

  double dot = 0.0;
  const int unit = blockIdx.x;   // (band, column run) of this warp
  {
    // bands [0, nextra) are cut into nxb + 1 column runs, the others into nxb (the grid fills the
    // resident warp slots of the device exactly); consecutive CTAs take neighbouring bands of the
    // same run, whose halo rows they share through L2
    int ib, ir;
    if (unit < nxb * nyb) {
      ir = unit / nyb;
      ib = unit - ir * nyb;
    } else {
      ir = nxb;
      ib = unit - nxb * nyb;
    }
    const int nxs = ib < nextra ? nxb + 1 : nxb;
    const int Y0 = ib * SW_BAND, Yb = Y0 - SW_LO;   // Yb even: lane row parity = node row parity
    // column runs over this rank's owned columns (one GPU: all of them)
    const int nown = d.own_hi - d.own_lo;
    const int X0 = d.own_lo + (int)((long long)ir * nown / nxs), X1 = d.own_lo + (int)((long long)(ir + 1) * nown / nxs);
    // wide-halo strip: the first / last run also writes the updated residual of the halo columns
    // it swept redundantly (r' = r - alpha q is exact there: q's halo was exchanged), so that the
    // residual's halo is valid for the next sweeps without an exchange of its own
    const bool lh = UPD && ir == 0 && d.own_lo > 0, rh = UPD && ir == nxs - 1 && d.own_hi < d.nnx;
    const double* E = Eall + (size_t)rhs * d.estride;
    const double2* r = rall + (size_t)rhs * d.nn;
    double2* rout = UPD ? routall + (size_t)rhs * d.nn : nullptr;
    double2* z = zall + (size_t)rhs * d.nn;
    const double2* zsrc = ZERO ? (UPD ? qall + (size_t)rhs * d.nn : nullptr) : zinall + (size_t)rhs * d.nn;

    // this lane's two rows
    const int gy0 = Yb + 2 * lane, gy1 = gy0 + 1;
    const bool vn0 = gy0 >= 0 && gy0 < d.nny, vn1 = gy1 >= 0 && gy1 < d.nny;
    const bool ve0 = gy0 >= 0 && gy0 < d.nely, ve1 = gy1 >= 0 && gy1 < d.nely;
    const int gn0 = vn0 ? gy0 : 0, gn1 = vn1 ? gy1 : 0, ge0 = ve0 ? gy0 : 0, ge1 = ve1 ? gy1 : 0;
    const bool band = lane >= SW_LO / 2 && lane < (SW_LO + SW_BAND) / 2;
    const uint8_t* fx = fixs + (Yb >> 1) + 4 + lane;   // + c fs_col + parity fs_plane

    // zero the ring once: the "lane -1" moduli entries are never written by the copies, and the
    // slots of the columns in front of the run are read (masked) before anything lands in them
    {
      double2* p = reinterpret_cast<double2*>(&S);
      for (int i = lane; i < (int)(sizeof(SwRing) / 16); i += 32) p[i] = make_double2(0.0, 0.0);
      __syncwarp();
    }

    // r and the moduli of node column c into ring slot sl (thread-private slots)
    auto issue = [&](int c, int sl) {
      // (32-bit node / element indices: msf_setup_mesh checks the grid size)
      const bool vc = c >= 0 && c < d.nnx;
      const int n = (vc ? c : 0) * d.nny;
      sw_cpa16(&S.s[sl].r[0][lane], r + (n + gn0), vc && vn0);
      sw_cpa16(&S.s[sl].r[1][lane], r + (n + gn1), vc && vn1);
      const bool vce = c >= 0 && c < d.nelx;
      const int m = (vce ? c : 0) * d.nely;
      sw_cpa8(&S.s[sl].e[0][lane + 1], E + (m + ge0), vce && ve0);
      sw_cpa8(&S.s[sl].e[1][lane + 1], E + (m + ge1), vce && ve1);
    };
    // z (or q) and the Dirichlet bits of node column c into registers
    // (the two mask bytes stay apart until they are used, one step later: combining them here
    // would wait for the loads)
    auto fetch = [&](int c, double2& a0, double2& a1, unsigned& f0, unsigned& f1) {
      const bool vc = c >= 0 && c < d.nnx;
      a0 = a1 = make_double2(0.0, 0.0);
      f0 = f1 = 3u;
      if (vc) {
        const int n = c * d.nny;
        if (!ZERO || UPD) {
          if (vn0) a0 = zsrc[n + gn0];
          if (vn1) a1 = zsrc[n + gn1];
        }
        const uint8_t* fc = fx + c * fs_col;
        f0 = fc[0];
        f1 = fc[fs_plane];
      }
    };

    // steps s = sb, sb + 2, ..., se: columns s, s + 1 enter; columns s - 7, s - 6 leave
    const int sb = (X0 - SW_DEP) & ~1;
    const int se0 = (X1 + SW_DEP) & ~1;   // smallest even s with s - 7 >= X1 - 1
    const int se = rh ? se0 + 8 : se0;    // ... the right halo's columns up to se0 + 1 leave too
    double2 W[9][2];
#pragma unroll
    for (int j = 0; j < 9; ++j) W[j][0] = W[j][1] = make_double2(0.0, 0.0);
    unsigned long long fw = ~0ull;   // Dirichlet bits of the window: column j, row p at 4 j + 2 p
#pragma unroll
    for (int i = 0; i < SW_PF; ++i) {
      issue(sb + 2 * i, 2 * i);
      issue(sb + 2 * i + 1, 2 * i + 1);
      sw_commit();
    }
    double2 pa0, pa1, pb0, pb1;   // columns s (a), s + 1 (b), one step ahead
    unsigned pfa0, pfa1, pfb0, pfb1;
    fetch(sb, pa0, pa1, pfa0, pfa1);
    fetch(sb + 1, pb0, pb1, pfb0, pfb1);
    int sl = 0;   // ring slot of column s (even)
    for (int s = sb; s <= se; s += 2) {
      sw_wait<SW_PF - 1>();   // columns s, s + 1 have landed (this lane's copies) ...
      __syncwarp();    // ... and the lane below's; every lane has finished step s - 2
      {
        const int s4 = sl + 2 * SW_PF >= SW_NR ? sl + 2 * SW_PF - SW_NR : sl + 2 * SW_PF;
        issue(s + 2 * SW_PF, s4);
        issue(s + 2 * SW_PF + 1, s4 + 1);
        sw_commit();
      }
      // the window moves two columns
#pragma unroll
      for (int j = 8; j >= 2; --j) {
        W[j][0] = W[j - 2][0];
        W[j][1] = W[j - 2][1];
      }
      fw = (fw << 8) | (unsigned long long)(pfb0 | (pfb1 << 2) | (pfa0 << 4) | (pfa1 << 6));
      if (ZERO) {
        W[0][0] = W[0][1] = W[1][0] = W[1][1] = make_double2(0.0, 0.0);
        if (UPD) {
          // r' = r - alpha q in the ring (this lane's slots)
          double2 v;
          v = S.s[sl].r[0][lane]; v.x = fma(-alpha, pa0.x, v.x); v.y = fma(-alpha, pa0.y, v.y); S.s[sl].r[0][lane] = v;
          v = S.s[sl].r[1][lane]; v.x = fma(-alpha, pa1.x, v.x); v.y = fma(-alpha, pa1.y, v.y); S.s[sl].r[1][lane] = v;
          v = S.s[sl + 1].r[0][lane]; v.x = fma(-alpha, pb0.x, v.x); v.y = fma(-alpha, pb0.y, v.y); S.s[sl + 1].r[0][lane] = v;
          v = S.s[sl + 1].r[1][lane]; v.x = fma(-alpha, pb1.x, v.x); v.y = fma(-alpha, pb1.y, v.y); S.s[sl + 1].r[1][lane] = v;
        }
      } else {
        W[1][0] = pa0;
        W[1][1] = pa1;
        W[0][0] = pb0;
        W[0][1] = pb1;
      }
      fetch(s + 2, pa0, pa1, pfa0, pfa1);
      fetch(s + 3, pb0, pb1, pfb0, pfb1);

      // ring slots of columns s - k
      int sk[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) sk[k] = sl - k < 0 ? sl - k + SW_NR : sl - k;
      // The neighbouring lanes' rows, shuffled once and shared by successive phases: U[j] = the
      // odd row of the lane below (window column j), D[j] = the even row of the lane above.  A
      // phase changes one row of one window column, which no later phase of the step needs from
      // the cache except where it is re-shuffled below (13 double2 shuffles per step, not 21).
      // From z = 0 the forward phases see only the colours already swept: F1 its horizontal
      // neighbours (colour 0), F2 the vertical (0) and diagonal (1) ones, F3 all but itself.
      constexpr int NZ_H = (1 << 1) | (1 << 7), NZ_V = (1 << 3) | (1 << 5);
      constexpr int NZ_D = (1 << 0) | (1 << 2) | (1 << 6) | (1 << 8), NZ_ALL = 0x1ff;
      const double2 zz = make_double2(0.0, 0.0);
      double2 U0 = zz, U1 = zz, U2 = zz, U3 = zz;
      if (!ZERO) {
        U0 = shfl_up2(W[0][1]);
        U1 = shfl_up2(W[1][1]);
        U2 = shfl_up2(W[2][1]);
        U3 = shfl_up2(W[3][1]);
      }
      sw_phase<1, 0, true, false, ZERO>(K, W, S, sk[0], sk[1], fw, lane, U2, U1, U0);    // F0   column s
      sw_phase<2, 0, true, false, false, ZERO ? NZ_H : NZ_ALL>(K, W, S, sk[1], sk[2], fw, lane, U3, U2, U1);          // F1   s - 1
      const double2 D2 = shfl_down2(W[2][0]), D3 = shfl_down2(W[3][0]), D4 = shfl_down2(W[4][0]);
      sw_phase<3, 1, true, false, false, ZERO ? (NZ_V | NZ_D) : NZ_ALL>(K, W, S, sk[2], sk[3], fw, lane, D4, D3, D2);  // F2   s - 2
      const double2 D5 = shfl_down2(W[5][0]);
      sw_phase<4, 1, true, true, false, ZERO ? (NZ_H | NZ_V | NZ_D) : NZ_ALL>(K, W, S, sk[3], sk[4], fw, lane, D5, D4, D3);   // F3B3 s - 3
      const double2 D6 = shfl_down2(W[6][0]);
      sw_phase<5, 1, false, true, false>(K, W, S, sk[4], sk[5], fw, lane, D6, D5, D4);   // B2   s - 4
      const double2 U5 = shfl_up2(W[5][1]), U6 = shfl_up2(W[6][1]), U7 = shfl_up2(W[7][1]);
      sw_phase<6, 0, false, true, false>(K, W, S, sk[5], sk[6], fw, lane, U7, U6, U5);   // B1   s - 5
      const double2 U8 = shfl_up2(W[8][1]);
      sw_phase<7, 0, false, true, false>(K, W, S, sk[6], sk[7], fw, lane, U8, U7, U6);   // B0   s - 6

      // columns s - 7 (window 8) and s - 6 (window 7) are final: band rows to global
      if (band) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int wc = s - 7 + q, j = 8 - q, ss = sk[7 - q];
          if (UPD && ((lh && wc >= sb && wc >= 0 && wc < X0) || (rh && wc >= X1 && wc <= se0 + 1 && wc < d.nnx))) {
            const int n = wc * d.nny;
            if (vn0) rout[n + gn0] = S.s[ss].r[0][lane];
            if (vn1) rout[n + gn1] = S.s[ss].r[1][lane];
          }
          if (wc >= X0 && wc < X1) {
            const int n = wc * d.nny;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
              if (p ? vn1 : vn0) {
                const int m = n + (p ? gn1 : gn0);
                const double2 zv = W[j][p];
                z[m] = zv;
                if (UPD || RZ) {
                  const double2 rv = S.s[ss].r[p][lane];
                  if (UPD) {
                    rout[m] = rv;
                    dot += rv.x * rv.x + rv.y * rv.y;
                  } else {
                    dot += rv.x * zv.x + rv.y * zv.y;
                  }
                }
              }
            }
          }
        }
      }
      sl = sl + 2 >= SW_NR ? sl + 2 - SW_NR : sl + 2;
    }
    sw_wait<0>();
  }
  pdl_launch();
  if (UPD || RZ) {
    const double sblk = block_sum_all(dot, red, tid, SW_T);
    const unsigned nblk = gridDim.x;
    if (arrive_last(sblk, partials + (size_t)rhs * max_partials, blockIdx.x, counters + rhs * 8, nblk, tid)) {
      const double tot = reduce_partials(partials + (size_t)rhs * max_partials, nblk, red, tid, SW_T);
      if (tid == 0) {
        fin_or_park(sc, dsum, rhs, UPD ? FIN_RR : FIN_RZ, tot, rz_mode);
        counters[rhs * 8] = 0;
      }
    }
  }
}

}  // namespace

// Dirichlet bits in the sweep's layout: per node column, two row-parity planes of fs_plane bytes;
// node row gy sits at plane gy & 1, byte (gy >> 1) + 4; rows outside the grid (down to -8, up
// past the last band's halo) hold 3.
void sgs_fix_layout(const Dims& d, int& fs_col, int& fs_plane) {
  fs_plane = ((d.nny + 1) / 2 + 4 + 64 + 8 + 15) & ~15;
  fs_col = 2 * fs_plane;
}

void sgs_fix_build(const Dims& d, const uint8_t* fixn, std::vector<uint8_t>& out) {
  int fc, fp;
  sgs_fix_layout(d, fc, fp);
  out.assign((size_t)d.nnx * fc, 3);
  for (int ix = 0; ix < d.nnx; ++ix)
    for (int iy = 0; iy < d.nny; ++iy)
      out[(size_t)ix * fc + (iy & 1) * fp + (iy >> 1) + 4] = fixn[(size_t)ix * d.nny + iy];
}

// z = SGS(zin; r) (zero_start: from z = 0) for realisations [rhs0, rhs0 + nr) of this rank's
// owned columns, out of place (neighbouring warps read their halo of zin while this one writes
// z).  upd: r -= alpha q first, the updated residual to rout (PCG iteration; ||r||^2 ->
// convergence).  rz_mode != 0: r.z of the result -> beta (1: PCG init, 2: iteration).
void launch_sgs_stream(msf_ctx* c, int rhs0, int nr, const double* r, double* rout, const double* zin,
                       double* z, bool gated, bool zero_start, bool upd, int rz_mode) {
  const Dims& d = c->dl;
  const int nyb = (d.nny + SW_BAND - 1) / SW_BAND;
  // one wave of SW_WARPS one-warp CTAs per SM; runs of at least 32 columns
  int units = std::max(nyb, (c->n_sm * SW_WARPS) / nr);
  units = std::min(units, nyb * std::max(1, (d.own_hi - d.own_lo) / 32));
  units = std::min(units, std::max(nyb, c->max_partials));   // one partial per CTA
  const int nxb = units / nyb, nextra = units - nxb * nyb;
  const int nblk = units;
  const dim3 grid(nblk, nr);
  int napart = 0;
  if (upd) {
    napart = c->apart_n;
    c->apart_n = 0;
  }
#define MSF_SW(ZR, UP, RZ)                                                                       \
  do {                                                                                           \
    static bool attr = [] {                                                                      \
      cudaFuncSetAttribute(k_sgs_warp<ZR, UP, RZ>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                           (int)SW_SMEM);                                                        \
      return true;                                                                               \
    }();                                                                                         \
    (void)attr;                                                                                  \
    launch_k(k_sgs_warp<ZR, UP, RZ>, grid, dim3(SW_T), SW_SMEM, c->stream, d, c->K0,             \
             (const double*)c->E_loc, (const double2*)r, (double2*)rout,                         \
             (const double2*)(zero_start ? z : zin), (double2*)z, (const double2*)c->q, c->fixs, \
             c->fs_col, c->fs_plane, c->sc, c->partials, c->counters, c->max_partials, c->dsum,  \
             (const double*)c->apart, napart, rhs0, gated ? 1 : 0, rz_mode, nyb, nxb, nextra);           \
  } while (0)
  if (zero_start) {
    if (upd) MSF_SW(true, true, false);
    else MSF_SW(true, false, false);
  } else {
    if (rz_mode) MSF_SW(false, false, true);
    else MSF_SW(false, false, false);
  }
#undef MSF_SW
  MSF_LAUNCHED(c);
}

int sgs_warp_partials_needed(const Dims& d) {
  return (d.nny + SW_BAND - 1) / SW_BAND + SW_WARPS * 192;
}
