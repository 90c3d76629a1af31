// Matrix-free Q4 stiffness operator, multicolour symmetric Gauss-Seidel and the PCG vector
// kernels of the B200 MsFEM path.
//
//   * y = P K(xbar) P x  with  K = sum_e (Emin + xbar_e^p (E0-Emin)) K0   (Eq. 4-5,
//     lines 73/84; reading R2: Dirichlet DOFs eliminated).  Node-centric gather: each thread
//     owns one node, reads the 4 adjacent element moduli and the 3x3 nodal neighbourhood
//     from a shared-memory tile with a one-node halo (coalesced double2 loads along y).
//   * Gauss-Seidel in the 4-colour node order of reading R7 (PAPER.md line 146 does not fix
//     an order): nodes of one colour share no element, so a colour is one parallel sweep.
//   * PCG dot products: warp-shuffle + shared-memory block reduction, per-block partials,
//     the last block to finish reduces the partials in a fixed order (deterministic) and
//     updates the per-realisation scalars (alpha, beta, convergence) on the device.
#include "msf_internal.cuh"

namespace {

constexpr int TX = 8;    // nodes per tile along x (threadIdx.y)
constexpr int TY = 32;   // nodes per tile along y (threadIdx.x)
constexpr int NTHR = TX * TY;

// local index a of the centre node inside element (sx,sy) = (ix-1+sx, iy-1+sy)
__device__ __forceinline__ constexpr int a_of(int sx, int sy) {
  return (sx == 0 && sy == 0) ? 2 : (sx == 1 && sy == 0) ? 3 : (sx == 0 && sy == 1) ? 1 : 0;
}
__device__ __forceinline__ constexpr int DXB(int b) { return (b == 1 || b == 2) ? 1 : 0; }
__device__ __forceinline__ constexpr int DYB(int b) { return (b >= 2) ? 1 : 0; }

// (A z)_node and the node's own 2x2 diagonal block from the 4 element moduli E[sx][sy]
// and the 3x3 neighbourhood z[i][j] = node (ix-1+i, iy-1+j).
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
        const double2 v = z[sx + DXB(b)][sy + DYB(b)];
        ax = fma(K.v[(2 * a) * 8 + 2 * b], v.x, ax);
        ax = fma(K.v[(2 * a) * 8 + 2 * b + 1], v.y, ax);
        ay = fma(K.v[(2 * a + 1) * 8 + 2 * b], v.x, ay);
        ay = fma(K.v[(2 * a + 1) * 8 + 2 * b + 1], v.y, ay);
      }
      const double e = E[sx][sy];
      ox = fma(e, ax, ox);
      oy = fma(e, ay, oy);
      dxx = fma(e, K.v[(2 * a) * 8 + 2 * a], dxx);
      dxy = fma(e, K.v[(2 * a) * 8 + 2 * a + 1], dxy);
      dyx = fma(e, K.v[(2 * a + 1) * 8 + 2 * a], dyx);
      dyy = fma(e, K.v[(2 * a + 1) * 8 + 2 * a + 1], dyy);
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block reduction; result valid in thread 0.  nthreads multiple of 32.
__device__ double block_sum(double v, double* sm, int tid, int nthreads) {
  v = warp_sum(v);
  if ((tid & 31) == 0) sm[tid >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (tid < 32) {
    s = (tid < (nthreads >> 5)) ? sm[tid] : 0.0;
    s = warp_sum(s);
  }
  __syncthreads();
  return s;
}

// Writes this block's partial, returns true in the last block to arrive.
__device__ bool arrive_last(double v, double* partials, int slot, unsigned* counter,
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

// In the last block: deterministic sum of partials[0..n).
__device__ double reduce_partials(const double* partials, int n, double* sm, int tid,
                                  int nthreads) {
  double s = 0.0;
  for (int i = tid; i < n; i += nthreads) s += __ldcg(partials + i);
  return block_sum(s, sm, tid, nthreads);
}

// ------------------------------------------------------------------ operator apply
// MODE 0: y = P K P x ; MODE 1: y = b - P K P x.  dot: accumulate x.y (p.Ap) and set
// alpha = rz / pq in the last block.
template <int MODE>
__global__ void __launch_bounds__(NTHR) k_apply(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                const double2* __restrict__ xall,
                                                double2* __restrict__ yall,
                                                const double2* __restrict__ ball,
                                                const uint8_t* __restrict__ fixn, PcgScalars* sc,
                                                double* partials, unsigned* counters, int rhs0,
                                                int gated, int dot, int max_partials) {
  const int rhs = rhs0 + blockIdx.z;
  if (gated && !sc[rhs].active) return;
  const double* E = Eall + (size_t)rhs * d.ne;
  const double2* x = xall + (size_t)rhs * d.nn;
  double2* y = yall + (size_t)rhs * d.nn;
  __shared__ double2 xs[TX + 2][TY + 2];
  __shared__ double Es[TX + 1][TY + 1];
  __shared__ double red[NTHR / 32];
  const int ix0 = blockIdx.y * TX, iy0 = blockIdx.x * TY;
  const int tid = threadIdx.y * TY + threadIdx.x;
  for (int k = tid; k < (TX + 2) * (TY + 2); k += NTHR) {
    const int i = k / (TY + 2), j = k - i * (TY + 2);
    const int gx = ix0 - 1 + i, gy = iy0 - 1 + j;
    double2 v = make_double2(0.0, 0.0);
    if (gx >= 0 && gx < d.nnx && gy >= 0 && gy < d.nny) v = x[(size_t)gx * d.nny + gy];
    xs[i][j] = v;
  }
  for (int k = tid; k < (TX + 1) * (TY + 1); k += NTHR) {
    const int i = k / (TY + 1), j = k - i * (TY + 1);
    const int ex = ix0 - 1 + i, ey = iy0 - 1 + j;
    Es[i][j] = (ex >= 0 && ex < d.nelx && ey >= 0 && ey < d.nely) ? E[(size_t)ex * d.nely + ey]
                                                                  : 0.0;
  }
  __syncthreads();
  const int li = threadIdx.y, lj = threadIdx.x;
  const int ix = ix0 + li, iy = iy0 + lj;
  double dv = 0.0;
  if (ix < d.nnx && iy < d.nny) {
    double Eloc[2][2];
    double2 zloc[3][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) Eloc[a][b] = Es[li + a][lj + b];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) zloc[a][b] = xs[li + a][lj + b];
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
    y[n] = out;
    if (dot) dv = zloc[1][1].x * out.x + zloc[1][1].y * out.y;
  }
  if (dot) {
    const double s = block_sum(dv, red, tid, NTHR);
    const unsigned nblk = gridDim.x * gridDim.y;
    const int slot = blockIdx.y * gridDim.x + blockIdx.x;
    if (arrive_last(s, partials + (size_t)rhs * max_partials, slot, counters + rhs * 8, nblk,
                    tid)) {
      const double tot = reduce_partials(partials + (size_t)rhs * max_partials, nblk, red, tid,
                                         NTHR);
      if (tid == 0) {
        sc[rhs].pq = tot;
        sc[rhs].alpha = sc[rhs].rz / tot;
        counters[rhs * 8] = 0;
      }
    }
  }
}

// ------------------------------------------------------------------ Gauss-Seidel colour sweep
// One colour phase of the symmetric Gauss-Seidel sweep (reading R7).  Thread per node quad
// (2qx..2qx+1, 2qy..2qy+1) -- one node of every colour -- updating the quad's node of the
// phase colour.  FWD: x then y ; BWD: y then x ; FWD&&BWD: the F3B3 phase (forward colour 3
// immediately followed by backward colour 3 on the same nodes, nothing changes in between).
// ZERO: the first forward phase from z = 0 (writes the whole quad: replaces a memset).
// RZ: after the last backward phase, r.z over the whole quad -> per-rhs beta (deterministic
// last-block reduction); rz_mode 1 = PCG init (beta = 0), 2 = iteration.
template <bool FWD, bool BWD, bool ZERO, bool RZ>
__global__ void __launch_bounds__(NTHR) k_sgs_colour(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                     const double2* __restrict__ rall,
                                                     double2* zall,
                                                     const uint8_t* __restrict__ fixn,
                                                     PcgScalars* sc, double* partials,
                                                     unsigned* counters, int max_partials,
                                                     int rhs0, int gated, int colour,
                                                     int rz_mode) {
  const int rhs = rhs0 + blockIdx.z;
  if (gated && !sc[rhs].active) return;
  __shared__ double red[NTHR / 32];
  const int qx = blockIdx.y * blockDim.y + threadIdx.y;
  const int qy = blockIdx.x * blockDim.x + threadIdx.x;
  const int ix = 2 * qx + (colour & 1), iy = 2 * qy + (colour >> 1);
  const double* E = Eall + (size_t)rhs * d.ne;
  double2* z = zall + (size_t)rhs * d.nn;
  const double2* r = rall + (size_t)rhs * d.nn;
  double dot = 0.0;
  if (ZERO) {   // zero the quad's other nodes
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
        Eloc[a][b] = (ex >= 0 && ex < d.nelx && ey >= 0 && ey < d.nely)
                         ? __ldg(E + (size_t)ex * d.nely + ey)
                         : 0.0;
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
    double ox, oy, dxx, dxy, dyx, dyy;
    apply_node(K, Eloc, zloc, ox, oy, dxx, dxy, dyx, dyy);
    const size_t n = (size_t)ix * d.nny + iy;
    const double2 rv = r[n];
    const uint8_t fm = fixn[n];
    double2 zn = zloc[1][1];
    double rx = rv.x - ox, ry = rv.y - oy;
    if (FWD) {
      if (!(fm & 1)) {
        const double dz = rx / dxx;
        zn.x += dz;
        ry -= dyx * dz;
        rx -= dxx * dz;
      }
      if (!(fm & 2)) {
        const double dz = ry / dyy;
        zn.y += dz;
        rx -= dxy * dz;
        ry -= dyy * dz;
      }
    }
    if (BWD) {
      if (!(fm & 2)) {
        const double dz = ry / dyy;
        zn.y += dz;
        rx -= dxy * dz;
      }
      if (!(fm & 1)) zn.x += rx / dxx;
    }
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
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const double sblk = block_sum(dot, red, tid, NTHR);
    const unsigned nblk = gridDim.x * gridDim.y;
    const int slot = blockIdx.y * gridDim.x + blockIdx.x;
    if (arrive_last(sblk, partials + (size_t)rhs * max_partials, slot, counters + rhs * 8, nblk,
                    tid)) {
      const double tot = reduce_partials(partials + (size_t)rhs * max_partials, nblk, red, tid,
                                         NTHR);
      if (tid == 0) {
        PcgScalars& S = sc[rhs];
        S.beta = (rz_mode == 1) ? 0.0 : tot / S.rz;
        S.rz = tot;
        counters[rhs * 8] = 0;
      }
    }
  }
}

// ------------------------------------------------------------------ fused symmetric GS
// One symmetric Gauss-Seidel sweep (reading R7: colours 0,1,2,3 forward, 3,2,1,0 backward)
// in ONE kernel by temporal blocking: a CTA stages a 64x64-node region (50x50 core + 7-node
// halo) of z, r, the element moduli and the Dirichlet mask in shared memory and runs the 7
// colour phases F0 F1 F2 F3B3 B2 B1 B0 there (each phase invalidates one more halo ring,
// the core stays exact).  Each thread owns 4 node quads (one node of every colour per
// quad), so every thread works in every phase; r is staged in shared memory as well.
//   MODE 0 (pre-smoothing):  z = SGS(0; r), also writes t = r - K z on the core.
//   MODE 1 (post-smoothing): z = SGS(z; r), optionally fused r.z reduction -> beta.
constexpr int SG_H = 7;
#ifndef MSF_SG_R
#define MSF_SG_R 64
#endif
constexpr int SG_R = MSF_SG_R;           // region nodes per direction
constexpr int SG_C = SG_R - 2 * SG_H;    // core nodes per direction
constexpr int SG_Q = SG_R / 2;           // quads per direction
constexpr int SG_QPT = 2;                // quads per thread
constexpr int SG_NT = SG_Q * SG_Q / SG_QPT;
constexpr int SG_E = SG_R + 1;           // element region per direction (one extra ring)
constexpr int SG_MINB = SG_R <= 48 ? 2 : 1;

__host__ __device__ constexpr size_t sgs_smem_bytes() {
  return (size_t)4 * (SG_Q + 2) * (SG_Q + 2) * (16 + 16 + 1) +
         (size_t)4 * ((SG_E + 1) / 2) * ((SG_E + 1) / 2) * 8;
}

constexpr int SG_QP = SG_Q + 2;          // padded plane extent (one zero quad border)
constexpr int SG_PP = SG_QP * SG_QP;     // nodes per padded colour plane
constexpr int SG_EQ = (SG_E + 1) / 2;    // element plane extent
constexpr int SG_EP = SG_EQ * SG_EQ;     // elements per plane

// colour-planar shared-memory layout: node (lx,ly) lives in plane (lx&1) + 2(ly&1) at quad
// (lx>>1, ly>>1) (+1 border); within a colour phase all 9 neighbour and 4 element offsets
// are warp-uniform constants and a warp reads unit-stride addresses.
__device__ __forceinline__ int zq(int lx, int ly) {
  return ((lx & 1) + 2 * (ly & 1)) * SG_PP + ((lx >> 1) + 1) * SG_QP + ((ly >> 1) + 1);
}
__device__ __forceinline__ int eq(int i, int j) {
  return ((i & 1) + 2 * (j & 1)) * SG_EP + (i >> 1) * SG_EQ + (j >> 1);
}

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? bytes : 0;   // src-size 0 -> zero fill
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

template <int MODE>
__global__ void __launch_bounds__(SG_NT, SG_MINB) k_sgs_fused(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                        const double2* __restrict__ rall,
                                                        double2* zall, double2* tall,
                                                        const uint8_t* __restrict__ fixn,
                                                        PcgScalars* sc, double* partials,
                                                        unsigned* counters, int max_partials,
                                                        int rhs0, int gated, int rz_mode) {
  const int rhs = rhs0 + blockIdx.z;
  if (gated && !sc[rhs].active) return;
  extern __shared__ __align__(16) unsigned char sg_raw[];
  double2* zs = reinterpret_cast<double2*>(sg_raw);                           // 4 padded planes
  double2* rs = zs + 4 * SG_PP;                                               // 4 padded planes
  double* Es = reinterpret_cast<double*>(rs + 4 * SG_PP);                     // 4 planes
  uint8_t* fs = reinterpret_cast<uint8_t*>(Es + 4 * SG_EP);                   // 4 padded planes
  __shared__ double red[SG_NT / 32];
  const int gx0 = blockIdx.y * SG_C - SG_H, gy0 = blockIdx.x * SG_C - SG_H;
  const double* E = Eall + (size_t)rhs * d.ne;
  double2* z = zall + (size_t)rhs * d.nn;
  const double2* r = rall + (size_t)rhs * d.nn;
  const int tid = threadIdx.x;
  // zero the padded borders (never loaded): z and fix
  for (int k = tid; k < 4 * SG_PP; k += SG_NT) {
    const int w = k - (k / SG_PP) * SG_PP, a = w / SG_QP, b = w - (w / SG_QP) * SG_QP;
    if (a == 0 || a == SG_QP - 1 || b == 0 || b == SG_QP - 1) {
      zs[k] = make_double2(0.0, 0.0);
      fs[k] = 3;
    }
  }
  // ---- stage the region: every copy in flight at once (cp.async, zero fill outside)
  for (int k = tid; k < SG_R * SG_R; k += SG_NT) {
    const int lx = k / SG_R, ly = k - (k / SG_R) * SG_R;
    const int gx = gx0 + lx, gy = gy0 + ly;
    const bool in = gx >= 0 && gx < d.nnx && gy >= 0 && gy < d.nny;
    const size_t n = in ? (size_t)gx * d.nny + gy : 0;
    const int q = zq(lx, ly);
    cp_async(&rs[q], r + n, 16, in);
    if (MODE == 1) cp_async(&zs[q], z + n, 16, in);
  }
  for (int k = tid; k < SG_E * SG_E; k += SG_NT) {
    const int i = k / SG_E, j = k - (k / SG_E) * SG_E;
    const int ex = gx0 - 1 + i, ey = gy0 - 1 + j;
    const bool in = ex >= 0 && ex < d.nelx && ey >= 0 && ey < d.nely;
    cp_async(&Es[eq(i, j)], E + (in ? (size_t)ex * d.nely + ey : 0), 8, in);
  }
  asm volatile("cp.async.commit_group;\n" ::);
  {
    uint8_t fv[SG_R * SG_R / SG_NT];
#pragma unroll
    for (int it = 0; it < SG_R * SG_R / SG_NT; ++it) {
      const int k = tid + it * SG_NT;
      const int lx = k / SG_R, ly = k - (k / SG_R) * SG_R;
      const int gx = gx0 + lx, gy = gy0 + ly;
      const bool in = gx >= 0 && gx < d.nnx && gy >= 0 && gy < d.nny;
      fv[it] = in ? __ldg(fixn + (size_t)gx * d.nny + gy) : (uint8_t)3;
    }
#pragma unroll
    for (int it = 0; it < SG_R * SG_R / SG_NT; ++it) {
      const int k = tid + it * SG_NT;
      const int lx = k / SG_R, ly = k - (k / SG_R) * SG_R;
      fs[zq(lx, ly)] = fv[it];
      if (MODE == 0) zs[zq(lx, ly)] = make_double2(0.0, 0.0);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  const int px = gx0 & 1, py = gy0 & 1;  // parity of the region origin
#pragma unroll 1
  for (int ph = 0; ph < 7; ++ph) {
    const int col = ph <= 3 ? ph : 6 - ph;
    const bool fwd = ph <= 3, bwd = ph >= 3;
    const int dx = (col & 1) ^ px, dy = (col >> 1) ^ py;   // local parity of the colour
    // warp-uniform offsets of the 3x3 neighbours and the 4 elements, relative to the quad
    int zo[3][3], eo[2][2];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int sx = dx - 1 + a, sy = dy - 1 + b;   // in [-1, 2]
        zo[a][b] = ((sx & 1) + 2 * (sy & 1)) * SG_PP + (sx >> 1) * SG_QP + (sy >> 1);
      }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int sx = dx + a, sy = dy + b;           // in [0, 2]
        eo[a][b] = ((sx & 1) + 2 * (sy & 1)) * SG_EP + (sx >> 1) * SG_EQ + (sy >> 1);
      }
    const int self = (dx + 2 * dy) * SG_PP;
#pragma unroll 1
    for (int s = 0; s < SG_QPT; ++s) {
      const int qd = tid + s * SG_NT, qx = qd / SG_Q, qy = qd - (qd / SG_Q) * SG_Q;
      const int zb = (qx + 1) * SG_QP + (qy + 1);
      const int eb = qx * SG_EQ + qy;
      const uint8_t fm = fs[self + zb];
      double Eloc[2][2];
      double2 zloc[3][3];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) Eloc[a][b] = Es[eb + eo[a][b]];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) zloc[a][b] = zs[zb + zo[a][b]];
      double ox, oy, dxx, dxy, dyx, dyy;
      apply_node(K, Eloc, zloc, ox, oy, dxx, dxy, dyx, dyy);
      const double2 rv = rs[self + zb];
      double2 zn = zloc[1][1];
      double rx = rv.x - ox, ry = rv.y - oy;
      if (fwd) {
        if (!(fm & 1)) {
          const double dz = rx / dxx;
          zn.x += dz;
          ry -= dyx * dz;
          rx -= dxx * dz;
        }
        if (!(fm & 2)) {
          const double dz = ry / dyy;
          zn.y += dz;
          rx -= dxy * dz;
          ry -= dyy * dz;
        }
      }
      if (bwd) {
        if (!(fm & 2)) {
          const double dz = ry / dyy;
          zn.y += dz;
          rx -= dxy * dz;
        }
        if (!(fm & 1)) zn.x += rx / dxx;
      }
      zs[self + zb] = zn;
    }
    __syncthreads();
  }
  // ---- write the core; MODE 0: residual t = r - K z; MODE 1: r.z partial
  double dot = 0.0;
#pragma unroll 1
  for (int k = tid; k < SG_C * SG_C; k += SG_NT) {
    const int cx = k / SG_C, cy = k - (k / SG_C) * SG_C;
    const int lx = SG_H + cx, ly = SG_H + cy;
    const int gx = gx0 + lx, gy = gy0 + ly;
    if (gx >= d.nnx || gy >= d.nny) continue;
    const size_t n = (size_t)gx * d.nny + gy;
    const double2 zn = zs[zq(lx, ly)];
    const double2 rv = rs[zq(lx, ly)];
    z[n] = zn;
    if (MODE == 0) {
      double Eloc[2][2];
      double2 zloc[3][3];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) Eloc[a][b] = Es[eq(lx + a, ly + b)];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) zloc[a][b] = zs[zq(lx - 1 + a, ly - 1 + b)];
      double ox, oy, dxx, dxy, dyx, dyy;
      apply_node(K, Eloc, zloc, ox, oy, dxx, dxy, dyx, dyy);
      const uint8_t fm = fs[zq(lx, ly)];
      double2 tv = make_double2(rv.x - ox, rv.y - oy);
      if (fm & 1) tv.x = 0.0;
      if (fm & 2) tv.y = 0.0;
      tall[(size_t)rhs * d.nn + n] = tv;
    } else {
      dot += rv.x * zn.x + rv.y * zn.y;
    }
  }
  if (MODE == 1 && rz_mode) {
    const double sblk = block_sum(dot, red, tid, SG_NT);
    const unsigned nblk = gridDim.x * gridDim.y;
    const int slot = blockIdx.y * gridDim.x + blockIdx.x;
    if (arrive_last(sblk, partials + (size_t)rhs * max_partials, slot, counters + rhs * 8, nblk,
                    tid)) {
      const double tot = reduce_partials(partials + (size_t)rhs * max_partials, nblk, red, tid,
                                         SG_NT);
      if (tid == 0) {
        PcgScalars& S = sc[rhs];
        S.beta = (rz_mode == 1) ? 0.0 : tot / S.rz;
        S.rz = tot;
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
                                                 int max_partials, double tol, int max_it) {
  __shared__ double red[VB / 32];
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
  s = block_sum(s, red, tid, VB);
  if (arrive_last(s, partials + (size_t)rhs * max_partials, blockIdx.x, counters + rhs * 8,
                  gridDim.x, tid)) {
    const double tot = reduce_partials(partials + (size_t)rhs * max_partials, gridDim.x, red,
                                       tid, VB);
    if (tid == 0) {
      PcgScalars& S = sc[rhs];
      S.fnorm2 = tot;
      S.rr = tot;
      S.tol2 = tol * tol;
      S.iters = 0;
      S.max_it = max_it;
      S.noconv = 0;
      S.rz = 0.0;
      S.alpha = S.beta = S.pq = 0.0;
      S.active = (tot > 0.0 && !(tot <= S.tol2 * tot)) ? 1 : 0;
      counters[rhs * 8] = 0;
    }
  }
}

// u += alpha p ; r -= alpha q ; rr = ||r||^2 ; iteration bookkeeping (reading R9)
__global__ void __launch_bounds__(VB) k_pcg_update_xr(Dims d, double2* uall, double2* rall,
                                                      const double2* __restrict__ pall,
                                                      const double2* __restrict__ qall,
                                                      PcgScalars* sc, double* partials,
                                                      unsigned* counters, int max_partials) {
  __shared__ double red[VB / 32];
  const int rhs = blockIdx.z;
  if (!sc[rhs].active) return;
  const int tid = threadIdx.x;
  const double alpha = sc[rhs].alpha;
  double2* u = uall + (size_t)rhs * d.nn;
  double2* r = rall + (size_t)rhs * d.nn;
  const double2* p = pall + (size_t)rhs * d.nn;
  const double2* q = qall + (size_t)rhs * d.nn;
  double s = 0.0;
  for (int i = blockIdx.x * VB + tid; i < d.nn; i += gridDim.x * VB) {
    const double2 pv = p[i], qv = q[i];
    double2 uv = u[i], rv = r[i];
    uv.x = fma(alpha, pv.x, uv.x);
    uv.y = fma(alpha, pv.y, uv.y);
    rv.x = fma(-alpha, qv.x, rv.x);
    rv.y = fma(-alpha, qv.y, rv.y);
    u[i] = uv;
    r[i] = rv;
    s += rv.x * rv.x + rv.y * rv.y;
  }
  s = block_sum(s, red, tid, VB);
  if (arrive_last(s, partials + (size_t)rhs * max_partials, blockIdx.x, counters + rhs * 8,
                  gridDim.x, tid)) {
    const double tot = reduce_partials(partials + (size_t)rhs * max_partials, gridDim.x, red,
                                       tid, VB);
    if (tid == 0) {
      PcgScalars& S = sc[rhs];
      S.rr = tot;
      S.iters += 1;
      if (tot <= S.tol2 * S.fnorm2) {
        S.active = 0;
      } else if (S.iters >= S.max_it) {
        S.active = 0;
        S.noconv = 1;
      }
      counters[rhs * 8] = 0;
    }
  }
}

// rz_new = r.z ; beta = rz_new / rz (or rz = r.z at init)
__global__ void __launch_bounds__(VB) k_pcg_rz(Dims d, const double2* __restrict__ rall,
                                               const double2* __restrict__ zall, PcgScalars* sc,
                                               double* partials, unsigned* counters,
                                               int max_partials, int init) {
  __shared__ double red[VB / 32];
  const int rhs = blockIdx.z;
  if (!sc[rhs].active) return;
  const int tid = threadIdx.x;
  const double2* r = rall + (size_t)rhs * d.nn;
  const double2* z = zall + (size_t)rhs * d.nn;
  double s = 0.0;
  for (int i = blockIdx.x * VB + tid; i < d.nn; i += gridDim.x * VB) {
    const double2 a = r[i], b = z[i];
    s += a.x * b.x + a.y * b.y;
  }
  s = block_sum(s, red, tid, VB);
  if (arrive_last(s, partials + (size_t)rhs * max_partials, blockIdx.x, counters + rhs * 8,
                  gridDim.x, tid)) {
    const double tot = reduce_partials(partials + (size_t)rhs * max_partials, gridDim.x, red,
                                       tid, VB);
    if (tid == 0) {
      PcgScalars& S = sc[rhs];
      if (init) {
        S.beta = 0.0;
      } else {
        S.beta = tot / S.rz;
      }
      S.rz = tot;
      counters[rhs * 8] = 0;
    }
  }
}

// p = z + beta p  (p = z at init)
__global__ void __launch_bounds__(VB) k_pcg_p(Dims d, const double2* __restrict__ zall,
                                              double2* pall, const PcgScalars* sc, int init) {
  const int rhs = blockIdx.z;
  if (!sc[rhs].active) return;
  const double beta = init ? 0.0 : sc[rhs].beta;
  const double2* z = zall + (size_t)rhs * d.nn;
  double2* p = pall + (size_t)rhs * d.nn;
  for (int i = blockIdx.x * VB + threadIdx.x; i < d.nn; i += gridDim.x * VB) {
    const double2 zv = z[i];
    double2 pv = init ? make_double2(0.0, 0.0) : p[i];
    pv.x = fma(beta, pv.x, zv.x);
    pv.y = fma(beta, pv.y, zv.y);
    p[i] = pv;
  }
}

// compliance c = f.u (Eq. 6)
__global__ void __launch_bounds__(VB) k_compliance(Dims d, const double2* __restrict__ f,
                                                   const double2* __restrict__ uall,
                                                   PcgScalars* sc, double* partials,
                                                   unsigned* counters, int max_partials) {
  __shared__ double red[VB / 32];
  const int rhs = blockIdx.z;
  const int tid = threadIdx.x;
  const double2* u = uall + (size_t)rhs * d.nn;
  double s = 0.0;
  for (int i = blockIdx.x * VB + tid; i < d.nn; i += gridDim.x * VB) {
    const double2 a = f[i], b = u[i];
    s += a.x * b.x + a.y * b.y;
  }
  s = block_sum(s, red, tid, VB);
  if (arrive_last(s, partials + (size_t)rhs * max_partials, blockIdx.x, counters + rhs * 8,
                  gridDim.x, tid)) {
    const double tot = reduce_partials(partials + (size_t)rhs * max_partials, gridDim.x, red,
                                       tid, VB);
    if (tid == 0) {
      sc[rhs].comp = tot;
      counters[rhs * 8] = 0;
    }
  }
}

inline int vec_blocks(const Dims& d) {
  int b = (d.nn + VB - 1) / VB;
  return b < 592 ? b : 592;  // 148 SMs x 4
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

static dim3 apply_grid(const Dims& d, int nr) {
  return dim3((d.nny + TY - 1) / TY, (d.nnx + TX - 1) / TX, nr);
}

int apply_partials_needed(const Dims& d) {
  dim3 g = apply_grid(d, 1);
  int a = (int)(g.x * g.y);
  return a > 592 ? a : 592;
}

void launch_matvec(msf_ctx* c, int rhs0, int nr, const double* x, double* y, bool gated,
                   bool dot_pq) {
  k_apply<0><<<apply_grid(c->d, nr), dim3(TY, TX), 0, c->stream>>>(
      c->d, c->K0, c->E, (const double2*)x, (double2*)y, nullptr, c->fixn, c->sc, c->partials,
      c->counters, rhs0, gated ? 1 : 0, dot_pq ? 1 : 0, c->max_partials);
  MSF_LAUNCHED(c);
}

void launch_residual(msf_ctx* c, int rhs0, int nr, const double* b, const double* x, double* y,
                     bool gated) {
  k_apply<1><<<apply_grid(c->d, nr), dim3(TY, TX), 0, c->stream>>>(
      c->d, c->K0, c->E, (const double2*)x, (double2*)y, (const double2*)b, c->fixn, c->sc,
      c->partials, c->counters, rhs0, gated ? 1 : 0, 0, c->max_partials);
  MSF_LAUNCHED(c);
}

// One symmetric GS sweep as 7 colour launches F0 F1 F2 F3B3 B2 B1 B0.  zero_start: z = 0 on
// entry (fused into F0); rz_mode != 0: r.z and beta fused into B0.
void launch_sgs_sweep(msf_ctx* c, int rhs0, int nr, const double* r, double* z, bool gated,
                      bool zero_start, int rz_mode) {
  const Dims& d = c->d;
  const int hx = (d.nnx + 1) / 2, hy = (d.nny + 1) / 2;
  dim3 blk(32, 8);
  dim3 grd((hy + 31) / 32, (hx + 7) / 8, nr);
  const int g = gated ? 1 : 0;
#define MSF_SGS(F, B, Z, RZ, col)                                                              \
  k_sgs_colour<F, B, Z, RZ><<<grd, blk, 0, c->stream>>>(d, c->K0, c->E, (const double2*)r,      \
                                                        (double2*)z, c->fixn, c->sc,           \
                                                        c->partials, c->counters,              \
                                                        c->max_partials, rhs0, g, col, rz_mode); \
  MSF_LAUNCHED(c)
  if (zero_start) {
    MSF_SGS(true, false, true, false, 0);
  } else {
    MSF_SGS(true, false, false, false, 0);
  }
  MSF_SGS(true, false, false, false, 1);
  MSF_SGS(true, false, false, false, 2);
  MSF_SGS(true, true, false, false, 3);
  MSF_SGS(false, true, false, false, 2);
  MSF_SGS(false, true, false, false, 1);
  if (rz_mode) {
    MSF_SGS(false, true, false, true, 0);
  } else {
    MSF_SGS(false, true, false, false, 0);
  }
#undef MSF_SGS
}

int sgs_colour_partials_needed(const Dims& d) {
  const int hx = (d.nnx + 1) / 2, hy = (d.nny + 1) / 2;
  return ((hy + 31) / 32) * ((hx + 7) / 8);
}

void launch_sgs(msf_ctx* c, int rhs0, int nr, const double* r, double* z, bool gated) {
  launch_sgs_sweep(c, rhs0, nr, r, z, gated, false, 0);
}

void launch_sgs_fused(msf_ctx* c, int rhs0, int nr, const double* r, double* z, double* t,
                      int mode, bool gated, int rz_mode) {
  const Dims& d = c->d;
  dim3 grd((d.nny + SG_C - 1) / SG_C, (d.nnx + SG_C - 1) / SG_C, nr);
  const size_t smem = sgs_smem_bytes();
  if (mode == 0) {
    cudaFuncSetAttribute(k_sgs_fused<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sgs_fused<0><<<grd, SG_NT, smem, c->stream>>>(d, c->K0, c->E, (const double2*)r, (double2*)z,
                                                    (double2*)t, c->fixn, c->sc, c->partials,
                                                    c->counters, c->max_partials, rhs0,
                                                    gated ? 1 : 0, 0);
  } else {
    cudaFuncSetAttribute(k_sgs_fused<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sgs_fused<1><<<grd, SG_NT, smem, c->stream>>>(d, c->K0, c->E, (const double2*)r, (double2*)z,
                                                    (double2*)t, c->fixn, c->sc, c->partials,
                                                    c->counters, c->max_partials, rhs0,
                                                    gated ? 1 : 0, rz_mode);
  }
  MSF_LAUNCHED(c);
}

int sgs_partials_needed(const Dims& d) {
  return ((d.nny + SG_C - 1) / SG_C) * ((d.nnx + SG_C - 1) / SG_C);
}

void launch_mask_copy(msf_ctx* c, const double* x, double* y, int nn) {
  int b = (nn + VB - 1) / VB;
  b = b < 592 ? b : 592;
  k_mask_copy<<<b, VB, 0, c->stream>>>((const double2*)x, (double2*)y, c->fixn, nn);
  MSF_LAUNCHED(c);
}

void launch_pcg_init(msf_ctx* c, int nr, double tol, int max_it) {
  k_pcg_init<<<dim3(vec_blocks(c->d), 1, nr), VB, 0, c->stream>>>(
      c->d, (const double2*)c->f, c->fixn, (double2*)c->u, (double2*)c->r, c->sc, c->partials,
      c->counters, c->max_partials, tol, max_it);
  MSF_LAUNCHED(c);
}

void launch_pcg_update_xr(msf_ctx* c, int nr) {
  k_pcg_update_xr<<<dim3(vec_blocks(c->d), 1, nr), VB, 0, c->stream>>>(
      c->d, (double2*)c->u, (double2*)c->r, (const double2*)c->pv, (const double2*)c->q, c->sc,
      c->partials, c->counters, c->max_partials);
  MSF_LAUNCHED(c);
}

void launch_pcg_rz(msf_ctx* c, int nr, bool init) {
  k_pcg_rz<<<dim3(vec_blocks(c->d), 1, nr), VB, 0, c->stream>>>(
      c->d, (const double2*)c->r, (const double2*)c->z, c->sc, c->partials, c->counters,
      c->max_partials, init ? 1 : 0);
  MSF_LAUNCHED(c);
}

void launch_pcg_p(msf_ctx* c, int nr, bool init) {
  k_pcg_p<<<dim3(vec_blocks(c->d), 1, nr), VB, 0, c->stream>>>(
      c->d, (const double2*)c->z, (double2*)c->pv, c->sc, init ? 1 : 0);
  MSF_LAUNCHED(c);
}

void launch_compliance(msf_ctx* c, int nr) {
  k_compliance<<<dim3(vec_blocks(c->d), 1, nr), VB, 0, c->stream>>>(
      c->d, (const double2*)c->f, (const double2*)c->u, c->sc, c->partials, c->counters,
      c->max_partials);
  MSF_LAUNCHED(c);
}
