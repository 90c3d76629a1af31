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
template <bool BACKWARD>
__global__ void __launch_bounds__(NTHR) k_sgs_colour(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                     const double2* __restrict__ rall,
                                                     double2* zall,
                                                     const uint8_t* __restrict__ fixn,
                                                     const PcgScalars* sc, int rhs0, int gated,
                                                     int colour) {
  const int rhs = rhs0 + blockIdx.z;
  if (gated && !sc[rhs].active) return;
  const int ix = 2 * (blockIdx.y * blockDim.y + threadIdx.y) + (colour & 1);
  const int iy = 2 * (blockIdx.x * blockDim.x + threadIdx.x) + (colour >> 1);
  if (ix >= d.nnx || iy >= d.nny) return;
  const double* E = Eall + (size_t)rhs * d.ne;
  double2* z = zall + (size_t)rhs * d.nn;
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
      zloc[a][b] = (gx >= 0 && gx < d.nnx && gy >= 0 && gy < d.nny)
                       ? z[(size_t)gx * d.nny + gy]
                       : make_double2(0.0, 0.0);
    }
  double ox, oy, dxx, dxy, dyx, dyy;
  apply_node(K, Eloc, zloc, ox, oy, dxx, dxy, dyx, dyy);
  const size_t n = (size_t)ix * d.nny + iy;
  const double2 rr = rall[(size_t)rhs * d.nn + n];
  const uint8_t fm = fixn[n];
  double2 zn = zloc[1][1];
  double rx = rr.x - ox, ry = rr.y - oy;
  if (!BACKWARD) {
    if (!(fm & 1)) {
      const double dz = rx / dxx;
      zn.x += dz;
      ry -= dyx * dz;
    }
    if (!(fm & 2)) zn.y += ry / dyy;
  } else {
    if (!(fm & 2)) {
      const double dz = ry / dyy;
      zn.y += dz;
      rx -= dxy * dz;
    }
    if (!(fm & 1)) zn.x += rx / dxx;
  }
  z[n] = zn;
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

void launch_sgs(msf_ctx* c, int rhs0, int nr, const double* r, double* z, bool gated) {
  const Dims& d = c->d;
  const int hx = (d.nnx + 1) / 2, hy = (d.nny + 1) / 2;
  dim3 blk(32, 8);
  dim3 grd((hy + 31) / 32, (hx + 7) / 8, nr);
  for (int col = 0; col < 4; ++col) {
    k_sgs_colour<false><<<grd, blk, 0, c->stream>>>(d, c->K0, c->E, (const double2*)r,
                                                    (double2*)z, c->fixn, c->sc, rhs0,
                                                    gated ? 1 : 0, col);
    MSF_LAUNCHED(c);
  }
  for (int col = 3; col >= 0; --col) {
    k_sgs_colour<true><<<grd, blk, 0, c->stream>>>(d, c->K0, c->E, (const double2*)r,
                                                   (double2*)z, c->fixn, c->sc, rhs0,
                                                   gated ? 1 : 0, col);
    MSF_LAUNCHED(c);
  }
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
