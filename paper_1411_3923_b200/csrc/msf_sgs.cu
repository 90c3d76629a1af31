// Streaming symmetric Gauss-Seidel sweep: the seven colour phases F0 F1 F2 F3B3 B2 B1 B0 of
// one symmetric sweep (readings R7, R8; "single pre- and post-smoothing using
// symmetric Gauss-Seidel") in ONE kernel that reads r, z and the moduli once and writes z once.
//
// The colour-phase form (msf_fem.cu k_sgs_colour) streams the moduli and the whole of z seven
// times per sweep.  Here every CTA owns a band of 112 node rows (y, the contiguous direction)
// and a run of node columns, and marches along x with a ring of 20 columns in shared memory
// (z, r, moduli, Dirichlet bits; each split by row parity so that the stride-2 colour rows are
// conflict-free).  Phase k (1..7) works on column s - 2k at step s: the phases are skewed by two
// columns, so everything a phase reads was completed by its predecessor phase at an earlier
// step and not yet touched by its successor, and one barrier per step orders all seven phases.
// A band needs a 7-row / 7-column halo (one per phase) that neighbouring CTAs also compute;
// those redundant updates use the same inputs and arithmetic (msfk::gs_node), so the sweep is
// bitwise the one of the colour-phase kernels.  Columns arrive by cp.async five steps ahead.
//
// Variants: ZERO (pre-smoothing, z = 0 on entry), UPD (the PCG update r -= alpha q fused in
// front: q is staged in z's ring slot, the new r is written to a second buffer with
// ||r||^2 -> convergence), RZ (post-smoothing: r.z of the result -> beta).  Every output is
// out of place: neighbouring CTAs read their halo of the inputs while this one writes.
#include "msf_kern.cuh"

#include <algorithm>
#include <climits>

using namespace msfk;

namespace {

constexpr int SG_T = 128;    // threads: 4 phase-slot warps x 32 lanes, two colour rows per lane
constexpr int SG_H = 128;    // buffered node rows per column (band + 8-row halos)
constexpr int SG_HP = 64;    // ... per parity plane
constexpr int SG_IN = 112;   // band rows: buffer rows [SG_LO, SG_LO + SG_IN)
constexpr int SG_LO = 8;
constexpr int SG_NR = 20;    // ring columns
constexpr int SG_DEP = 7;    // phases per sweep = halo width
constexpr int SG_P = SG_NR - 15;   // prefetch distance (columns)

struct SgRing {
  double2 z[SG_NR][2][SG_HP];
  double2 r[SG_NR][2][SG_HP];
  double e[SG_NR][2][SG_HP];    // element (column c, row Yb + ly)
  uint8_t f[SG_NR][2][SG_HP];   // Dirichlet bits; 3 outside the grid
};
constexpr size_t SG_SMEM = sizeof(SgRing);

__device__ __forceinline__ uint32_t sg_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// cp.async with zero fill (src_bytes = 0: nothing is read, the destination is zeroed)
__device__ __forceinline__ void cpa16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sg_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cpa8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sg_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// The moduli and the 3x3 neighbourhood of the node at plane index k of row parity YP (buffer
// row ly = 2 k + YP) at ring slots (c-1, c, c+1).  With YP a template parameter the parity
// planes of rows ly-1 / ly / ly+1 are compile-time, so every load is a slot base plus an
// immediate offset (the row arithmetic per load was the largest integer cost of the sweep).
template <bool Z0, int YP>
__device__ __forceinline__ void sg_gather(const SgRing& S, int sm, int s0, int sp, int k,
                                          double (&Eloc)[2][2], double2 (&zloc)[3][3]) {
  constexpr int PM = 1 - YP, DM = YP - 1, DP = YP;   // row ly-1 / ly+1: plane 1-YP, k+DM / k+DP
  Eloc[0][0] = S.e[sm][PM][k + DM];
  Eloc[0][1] = S.e[sm][YP][k];
  Eloc[1][0] = S.e[s0][PM][k + DM];
  Eloc[1][1] = S.e[s0][YP][k];
  if (Z0) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) zloc[a][b] = make_double2(0.0, 0.0);
  } else {
    zloc[0][0] = S.z[sm][PM][k + DM];
    zloc[0][1] = S.z[sm][YP][k];
    zloc[0][2] = S.z[sm][PM][k + DP];
    zloc[1][0] = S.z[s0][PM][k + DM];
    zloc[1][1] = S.z[s0][YP][k];
    zloc[1][2] = S.z[s0][PM][k + DP];
    zloc[2][0] = S.z[sp][PM][k + DM];
    zloc[2][1] = S.z[sp][YP][k];
    zloc[2][2] = S.z[sp][PM][k + DP];
  }
}

// Two nodes (plane indices k0, k1 of row parity YP in one column) of phase (FWD, BWD, Z0) at
// ring slots (c-1, c, c+1), computed together so that their independent FMA chains
// interleave.  A node whose DOFs are both fixed (or outside the grid) comes back unchanged.
template <bool FWD, bool BWD, bool Z0, int YP>
__device__ __forceinline__ void sg_node2(const K0Mat& K, SgRing& S, int sm, int s0, int sp,
                                         int k0, int k1, bool v0, bool v1) {
  double E0[2][2], E1[2][2];
  double2 z0[3][3], z1[3][3];
  sg_gather<Z0, YP>(S, sm, s0, sp, k0, E0, z0);
  sg_gather<Z0, YP>(S, sm, s0, sp, k1, E1, z1);
  const double2 r0 = S.r[s0][YP][k0], r1 = S.r[s0][YP][k1];
  const uint8_t f0 = S.f[s0][YP][k0], f1 = S.f[s0][YP][k1];
#ifdef MSF_SGS_EXP_NOCOMPUTE   // A/B experiment: the sweep's data movement alone
  const double2 n0 = make_double2(z0[1][1].x + E0[0][0] + r0.x + f0, z0[0][0].y + z0[2][2].y + E0[1][1] + E1[0][1]);
  const double2 n1 = make_double2(z1[1][1].x + E1[0][0] + r1.x + f1, z1[0][0].y + z1[2][2].y + E1[1][1] + E0[1][0]);
#else
  const double2 n0 = gs_node<FWD, BWD, Z0>(K, E0, z0, r0, f0);
  const double2 n1 = gs_node<FWD, BWD, Z0>(K, E1, z1, r1, f1);
#endif
  if (v0) S.z[s0][YP][k0] = n0;
  if (v1) S.z[s0][YP][k1] = n1;
}

template <bool ZERO, bool UPD, bool RZ>
__global__ void __launch_bounds__(SG_T, 2)
    k_sgs_stream(Dims d, K0Mat K, const double* __restrict__ Eall, const double2* __restrict__ rall,
                 double2* routall, const double2* __restrict__ zinall, double2* zall,
                 const double2* __restrict__ qall, const uint8_t* __restrict__ fixs, int fs_col,
                 int fs_plane, PcgScalars* sc, double* partials, unsigned* counters,
                 int max_partials, double* dsum, const double* __restrict__ apart, int napart,
                 int rhs0, int gated, int rz_mode, int nxs) {
  extern __shared__ __align__(16) unsigned char sg_raw[];
  SgRing& S = *reinterpret_cast<SgRing*>(sg_raw);
  __shared__ double red[SG_T / 32 + 1];
  pdl_wait();
  const int rhs = rhs0 + blockIdx.z;
  if (gated && !sc[rhs].active) return;
  const int tid = threadIdx.x;
  const int Y0 = blockIdx.x * SG_IN, Yb = Y0 - SG_LO;   // Yb even: buffer row parity = node row parity
  const int X0 = (int)((long long)blockIdx.y * d.nnx / nxs);
  const int X1 = (int)((long long)(blockIdx.y + 1) * d.nnx / nxs);
  const double* E = Eall + (size_t)rhs * d.estride;
  const double2* r = rall + (size_t)rhs * d.nn;
  double2* rout = UPD ? routall + (size_t)rhs * d.nn : nullptr;
  double2* z = zall + (size_t)rhs * d.nn;
  const double2* zin = zinall + (size_t)rhs * d.nn;
  const double2* q = UPD ? qall + (size_t)rhs * d.nn : nullptr;

  double alpha = 0.0;
  if (UPD) {
    // p.Ap from the operator's per-CTA partials: every CTA sums them in the same fixed order
    // (identical alpha everywhere); CTA 0 records pq and alpha
    if (napart > 0) {
      const double pq = reduce_partials(apart + (size_t)rhs * max_partials, napart, red, tid, SG_T);
      alpha = sc[rhs].rz / pq;
      if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
        sc[rhs].pq = pq;
        sc[rhs].alpha = alpha;
      }
    } else {
      alpha = sc[rhs].alpha;
    }
  }

  const int cs = X0 - SG_DEP, c_last = X1 + SG_DEP - 1;   // buffered columns [cs, c_last]
  auto wrap = [](int x) { return x >= SG_NR ? x - SG_NR : (x < 0 ? x + SG_NR : x); };
  // ---- per-thread constants (the step loop only moves the column)
  // issue / transform / write-back row of this thread
  const int pl_t = tid & 1, k_t = tid >> 1, gy_t = Yb + tid;
  const bool vz_t = gy_t >= 0 && gy_t < d.nny, ve_t = gy_t >= 0 && gy_t < d.nely;
  const int gyc_t = vz_t ? gy_t : 0, gye_t = ve_t ? gy_t : 0;
  // node tasks: warp w runs phase 2w + 1 on even steps (F0 F2 B2 B0, even columns) and 2w + 2
  // on odd steps (F1 F3B3 B1, odd columns), colour rows lane and lane + 32 of the phase's row
  // parity; rows outside [1 + ph, 127 - ph) are computed from a valid row and not stored
  const int wp = tid >> 5, lane = tid & 31;
  // (even-step / odd-step values as named scalars: an array indexed by the step parity would
  // live in local memory)
  int ph0, ly00, ly10, slo0, shi0, ph1, ly01, ly11, slo1, shi1;
  bool vA0, vB0, vA1, vB1;
  auto task_consts = [&](int par, int& ph, int& ly0, int& ly1, bool& vA, bool& vB, int& slo, int& shi) {
    ph = 2 * wp + 1 + par;
    const int colour = (ph <= 4) ? ph - 1 : 7 - ph;
    const int lyA = 2 * lane + (colour >> 1), lyB = lyA + 64;
    vA = lyA >= 1 + ph;
    vB = lyB < SG_H - 1 - ph;
    ly0 = vA ? lyA : lyA + 2 * ((2 + ph - lyA) / 2);
    ly1 = vB ? lyB : lyB - 2 * ((lyB - (SG_H - 2 - ph)) / 2 + 1);
    // steps at which the phase's column s - 2 ph lies in [X0 - 7 + ph, X1 + 7 - ph) and the grid
    slo = max(X0 - SG_DEP + ph, 0) + 2 * ph;
    shi = ph <= 7 ? min(X1 + SG_DEP - ph, d.nnx) + 2 * ph : INT_MIN;
  };
  task_consts(0, ph0, ly00, ly10, vA0, vB0, slo0, shi0);
  task_consts(1, ph1, ly01, ly11, vA1, vB1, slo1, shi1);
  // column c into ring slot sl: z (or q), r, moduli, Dirichlet bits (this thread: row tid)
  auto issue = [&](int c, int sl) {
#ifdef MSF_SGS_EXP_NOLOAD   // A/B experiment: the sweep's arithmetic alone
    return;
#endif
    if (c > c_last) return;
    if (c < 0 || c >= d.nnx) {   // outside the grid: zero values, both DOFs fixed
      S.z[sl][pl_t][k_t] = make_double2(0.0, 0.0);
      S.r[sl][pl_t][k_t] = make_double2(0.0, 0.0);
      S.e[sl][pl_t][k_t] = 0.0;
      S.f[sl][pl_t][k_t] = 3;
      return;
    }
    const size_t n = (size_t)c * d.nny + gyc_t;
    if (!ZERO) cpa16(&S.z[sl][pl_t][k_t], zin + n, vz_t);
    else if (UPD) cpa16(&S.z[sl][pl_t][k_t], q + n, vz_t);
    cpa16(&S.r[sl][pl_t][k_t], r + n, vz_t);
    const bool ve = ve_t && c < d.nelx;
    cpa8(&S.e[sl][pl_t][k_t], E + (ve ? (size_t)c * d.nely + gye_t : 0), ve);
    if (tid < 16) {   // 2 planes x 64 bytes of the planar padded mask (setup: fixs)
      const int p2 = tid >> 3, ch = tid & 7;
      cpa8(&S.f[sl][p2][ch * 8], fixs + (size_t)c * fs_col + p2 * fs_plane + (Y0 >> 1) + ch * 8, true);
    }
  };

  for (int c = cs; c < cs + SG_P; ++c) {
    issue(c, c - cs);
    cpa_commit();
  }
  double dot = 0.0;
  int sl = 1;   // ring slot of column s (slot(c) = (c - cs) mod SG_NR)
  for (int s = cs + 1; s <= X1 + 14; ++s, sl = sl + 1 == SG_NR ? 0 : sl + 1) {
    cpa_wait<SG_P - 1>();   // column s - 1 has landed (this thread's copies) ...
    __syncthreads();        // ... for every thread; step s - 1 is complete everywhere
    issue(s - 1 + SG_P, wrap(sl - 1 + SG_P));   // into the slot of column s - 16, last read at step s - 1
    cpa_commit();
    if (ZERO && s - 1 <= c_last) {
      // column s - 1 becomes the sweep's input: z = 0 (UPD: r -= alpha q, q from z's slot)
      const int st = wrap(sl - 1);
      if (UPD) {
        double2 rv = S.r[st][pl_t][k_t];
        const double2 qv = S.z[st][pl_t][k_t];
        rv.x = fma(-alpha, qv.x, rv.x);
        rv.y = fma(-alpha, qv.y, rv.y);
        S.r[st][pl_t][k_t] = rv;
      }
      S.z[st][pl_t][k_t] = make_double2(0.0, 0.0);
    }
    {
      // column s - 15 is final (phase 7 ran on it at step s - 1): band rows to global
      const int wc = s - 15, i = tid;
      if (i < SG_IN && wc >= X0 && wc < X1 && Y0 + i < d.nny) {
        const int ly = SG_LO + i, sw = wrap(sl - 15);
        const size_t n = (size_t)wc * d.nny + (Y0 + i);
        const double2 zv = S.z[sw][ly & 1][ly >> 1];
        z[n] = zv;
        if (UPD) {
          const double2 rv = S.r[sw][ly & 1][ly >> 1];
          rout[n] = rv;
          dot += rv.x * rv.x + rv.y * rv.y;
        }
        if (RZ) {
          const double2 rv = S.r[sw][ly & 1][ly >> 1];
          dot += rv.x * zv.x + rv.y * zv.y;
        }
      }
    }
    {
      const bool odd = s & 1;
      const int ph = odd ? ph1 : ph0;
      if (s >= (odd ? slo1 : slo0) && s < (odd ? shi1 : shi0)) {
        const int s0 = wrap(sl - 2 * ph), sm = s0 == 0 ? SG_NR - 1 : s0 - 1, sp = s0 == SG_NR - 1 ? 0 : s0 + 1;
        const int ly0 = odd ? ly01 : ly00, ly1 = odd ? ly11 : ly10;
        const bool vA = odd ? vA1 : vA0, vB = odd ? vB1 : vB0;
        // colour rows: phases 1, 2, 6, 7 (colours 0, 1) even, phases 3, 4, 5 (colours 2, 3) odd
        const int k0 = ly0 >> 1, k1 = ly1 >> 1;
        switch (ph) {
          case 1: sg_node2<true, false, ZERO, 0>(K, S, sm, s0, sp, k0, k1, vA, vB); break;
          case 2: sg_node2<true, false, false, 0>(K, S, sm, s0, sp, k0, k1, vA, vB); break;
          case 3: sg_node2<true, false, false, 1>(K, S, sm, s0, sp, k0, k1, vA, vB); break;
          case 4: sg_node2<true, true, false, 1>(K, S, sm, s0, sp, k0, k1, vA, vB); break;
          case 5: sg_node2<false, true, false, 1>(K, S, sm, s0, sp, k0, k1, vA, vB); break;
          default: sg_node2<false, true, false, 0>(K, S, sm, s0, sp, k0, k1, vA, vB); break;
        }
      }
    }
  }
  cpa_wait<0>();
  pdl_launch();
  if (UPD || RZ) {
    const double sblk = block_sum_all(dot, red, tid, SG_T);
    const unsigned nblk = gridDim.x * gridDim.y;
    const int sb = blockIdx.y * gridDim.x + blockIdx.x;
    if (arrive_last(sblk, partials + (size_t)rhs * max_partials, sb, counters + rhs * 8, nblk, tid)) {
      const double tot = reduce_partials(partials + (size_t)rhs * max_partials, nblk, red, tid, SG_T);
      if (tid == 0) {
        fin_or_park(sc, dsum, rhs, UPD ? FIN_RR : FIN_RZ, tot, rz_mode);
        counters[rhs * 8] = 0;
      }
    }
  }
}

}  // namespace

// Dirichlet bits in the streaming sweep's layout: per node column, two parity planes of
// fs_plane bytes; node row gy sits at plane gy & 1, byte (gy >> 1) + 4; rows outside the grid
// (down to -8, up past the last band's halo) hold 3.
void sgs_fix_layout(const Dims& d, int& fs_col, int& fs_plane) {
  fs_plane = ((d.nny + 1) / 2 + 4 + SG_H / 2 + 8 + 15) & ~15;
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

size_t sgs_stream_smem() { return SG_SMEM; }

// z = SGS(zin; r) (zero_start: from z = 0) for realisations [rhs0, rhs0 + nr) of this rank's
// grid (out of place: neighbouring CTAs read their halo of zin while this one writes z).  upd: r -= alpha q first (PCG iteration; ||r||^2 -> convergence).  rz_mode != 0: r.z
// of the result -> beta (1: PCG init, 2: iteration).
void launch_sgs_stream(msf_ctx* c, int rhs0, int nr, const double* r, double* rout,
                       const double* zin, double* z, bool gated, bool zero_start, bool upd,
                       int rz_mode) {
  // (a wide-halo strip always takes it: k_sgs_stream sweeps all local columns)
  if ((c->sgs_warp || c->sb.halo > 1) && (long long)c->dl.nnx * c->fs_col < (1ll << 31)) {   // 32-bit indices there
    launch_sgs_warp(c, rhs0, nr, r, rout, zin, z, gated, zero_start, upd, rz_mode);
    return;
  }
  const Dims& d = c->dl;
  const int nyb = (d.nny + SG_IN - 1) / SG_IN;
  // one wave at 2 CTAs per SM; runs of at least 32 columns
  int nxs = std::max(1, (2 * c->n_sm) / (nyb * nr));
  nxs = std::min(nxs, std::max(1, d.nnx / 32));
  nxs = std::min(nxs, std::max(1, c->max_partials / nyb));   // one partial per CTA
  const dim3 grid(nyb, nxs, nr);
  int napart = 0;
  if (upd) {
    napart = c->apart_n;
    c->apart_n = 0;
  }
#define MSF_SG(ZR, UP, RZ)                                                                       \
  do {                                                                                           \
    static bool attr = [] {                                                                      \
      cudaFuncSetAttribute(k_sgs_stream<ZR, UP, RZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)SG_SMEM);                                                        \
      return true;                                                                               \
    }();                                                                                         \
    (void)attr;                                                                                  \
    launch_k(k_sgs_stream<ZR, UP, RZ>, grid, dim3(SG_T), SG_SMEM, c->stream, d, c->K0,           \
             (const double*)c->E_loc, (const double2*)r, (double2*)rout,                         \
             (const double2*)(zero_start ? z : zin),                                             \
             (double2*)z, (const double2*)c->q, c->fixs,                                         \
             c->fs_col, c->fs_plane, c->sc, c->partials, c->counters, c->max_partials, c->dsum,  \
             (const double*)c->apart, napart, rhs0, gated ? 1 : 0, rz_mode, nxs);               \
  } while (0)
  if (zero_start) {
    if (upd) MSF_SG(true, true, false);
    else MSF_SG(true, false, false);
  } else {
    if (rz_mode) MSF_SG(false, false, true);
    else MSF_SG(false, false, false);
  }
#undef MSF_SG
  MSF_LAUNCHED(c);
}

int sgs_stream_partials_needed(const Dims& d) { return (d.nny + SG_IN - 1) / SG_IN; }
