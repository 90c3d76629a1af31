// Design-side kernels: periodic density filter + Heaviside projection (§4.3,
// Eq. 16, periodic 3x3-block filter line 275 -> toroidal filter, reading R3/R4),
// SIMP moduli (Eq. 5), adjoint sensitivities of the robust objective (Eq. 14-15, 17,
// chain rule line 267, tile summation line 236) and the optimality-criteria update
// (reading R11).
#include "msf_internal.cuh"

namespace {

constexpr int FB = 256;

__device__ __forceinline__ int wrap(int i, int n) {
  int r = i % n;
  return r < 0 ? r + n : r;
}

__device__ __forceinline__ double heaviside(double xt, double beta, double eta) {
  if (beta <= 0.0) return xt;
  const double num = tanh(beta * eta) + tanh(beta * (xt - eta));
  const double den = tanh(beta * eta) + tanh(beta * (1.0 - eta));
  return num / den;
}

__device__ __forceinline__ double heaviside_d(double xt, double beta, double eta) {
  if (beta <= 0.0) return 1.0;
  const double den = tanh(beta * eta) + tanh(beta * (1.0 - eta));
  const double th = tanh(beta * (xt - eta));
  return beta * (1.0 - th * th) / den;
}

__device__ __forceinline__ double tile_filter(const double* x, int t, int tx, int ty,
                                              const int* fdx, const int* fdy,
                                              const double* fw, int nf, double wsum) {
  const int i = t / ty, j = t - (t / ty) * ty;
  double acc = 0.0;
  for (int k = 0; k < nf; ++k) acc += fw[k] * x[wrap(i + fdx[k], tx) * ty + wrap(j + fdy[k], ty)];
  return acc / wsum;
}

__device__ __forceinline__ double tile_filter_adj(const double* g, int t, int tx, int ty,
                                                  const int* fdx, const int* fdy,
                                                  const double* fw, int nf, double wsum) {
  const int i = t / ty, j = t - (t / ty) * ty;
  double acc = 0.0;
  for (int k = 0; k < nf; ++k) acc += fw[k] * g[wrap(i - fdx[k], tx) * ty + wrap(j - fdy[k], ty)];
  return acc / wsum;
}

struct FiltArgs {
  const int* dx;
  const int* dy;
  const double* w;
  int n;
  double wsum;
};

struct ProjArgs {
  double beta;
  double eta[MSF_MAX_RHS];
  int R;
};

// filtered tile + one projected tile per realisation
__global__ void k_filter_project(Dims d, const double* __restrict__ x, double* xt,
                                 double* xbar, FiltArgs fa, ProjArgs pa) {
  for (int t = blockIdx.x * FB + threadIdx.x; t < d.nt; t += gridDim.x * FB) {
    const double v = tile_filter(x, t, d.tile_x, d.tile_y, fa.dx, fa.dy, fa.w, fa.n, fa.wsum);
    xt[t] = v;
    for (int k = 0; k < pa.R; ++k) xbar[(size_t)k * d.nt + t] = heaviside(v, pa.beta, pa.eta[k]);
  }
}

// E[k][e] = Emin + xbar_k(tile(e))^p (E0 - Emin)   (Eq. 5)
__global__ void k_moduli(Dims d, const double* __restrict__ xbar, double* Eall, double E0,
                         double Emin, double penal) {
  const int k = blockIdx.z;
  const double* xb = xbar + (size_t)k * d.nt;
  double* E = Eall + (size_t)k * d.ne;
  for (int ex = blockIdx.y; ex < d.nelx; ex += gridDim.y) {
    const int tx = ex % d.tile_x;
    for (int ey = blockIdx.x * FB + threadIdx.x; ey < d.nely; ey += gridDim.x * FB) {
      const double v = xb[tx * d.tile_y + ey % d.tile_y];
      E[(size_t)ex * d.nely + ey] = Emin + pow(v, penal) * (E0 - Emin);
    }
  }
}

__global__ void k_set_physical(Dims d, const double* __restrict__ xb_el, double* E, double E0,
                               double Emin, double penal) {
  for (int e = blockIdx.x * FB + threadIdx.x; e < d.ne; e += gridDim.x * FB)
    E[e] = Emin + pow(xb_el[e], penal) * (E0 - Emin);
}

// dc/dxbar_e = -p xbar^{p-1} (E0-Emin) u_e^T K0 u_e  (Eq. 14-15) for the element
// columns [ex0, ex1) (global); u holds the node columns from gox on (this rank's strip)
__global__ void k_dc_element(Dims d, K0Mat K, const double2* __restrict__ u,
                             const double* __restrict__ xbar, double* dc, double E0, double Emin,
                             double penal, int ex0, int ex1, int gox) {
  for (int ex = ex0 + blockIdx.y; ex < ex1; ex += gridDim.y) {
    const int tx = ex % d.tile_x;
    for (int ey = blockIdx.x * FB + threadIdx.x; ey < d.nely; ey += gridDim.x * FB) {
      const size_t n0 = (size_t)(ex - gox) * d.nny + ey;
      const double2 a = u[n0], b = u[n0 + d.nny], c = u[n0 + d.nny + 1], e = u[n0 + 1];
      const double ue[8] = {a.x, a.y, b.x, b.y, c.x, c.y, e.x, e.y};
      double en = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) s = fma(K.v[i * 8 + j], ue[j], s);
        en = fma(ue[i], s, en);
      }
      const double xv = xbar[tx * d.tile_y + ey % d.tile_y];
      dc[(size_t)ex * d.nely + ey] = -penal * pow(xv, penal - 1.0) * (E0 - Emin) * en;
    }
  }
}

// tile-variable sum over all controlled elements, fixed (element-id) order
__global__ void k_tile_sum(Dims d, const double* __restrict__ el, double* out) {
  const int cxn = d.nelx / d.tile_x, cyn = d.nely / d.tile_y;
  for (int t = blockIdx.x * FB + threadIdx.x; t < d.nt; t += gridDim.x * FB) {
    const int i = t / d.tile_y, j = t - (t / d.tile_y) * d.tile_y;
    double s = 0.0;
    for (int a = 0; a < cxn; ++a) {
      const size_t base = (size_t)(a * d.tile_x + i) * d.nely + j;
      for (int b = 0; b < cyn; ++b) s += el[base + (size_t)b * d.tile_y];
    }
    out[t] = s;
  }
}

// robust weights (Eq. 17, reading R10): scal[0]=F, [1]=mean, [2]=var, [8+k]=w_k
__global__ void k_robust_weights(const PcgScalars* sc, int R, double kappa, double* scal) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mean = 0.0;
  for (int k = 0; k < R; ++k) mean += sc[k].comp;
  mean /= R;
  double var = 0.0;
  for (int k = 0; k < R; ++k) var += (sc[k].comp - mean) * (sc[k].comp - mean);
  var /= R;
  for (int k = 0; k < R; ++k) {
    double w = 1.0 / R;
    if (var > 0.0) w += kappa * (sc[k].comp - mean) / (R * sqrt(var));
    scal[8 + k] = w;
    scal[16 + k] = sc[k].comp;
  }
  scal[0] = mean + kappa * sqrt(var);
  scal[1] = mean;
  scal[2] = var;
}

// g1 = sum_k w_k H'_k dcT_k ; g2 = sum_k H'_k count / (m n_el vf)
__global__ void k_chain_pre(Dims d, const double* __restrict__ xt, const double* __restrict__ dcT,
                            const double* scal, double* g1, double* g2, ProjArgs pa,
                            double volfrac) {
  const double count = (double)(d.nelx / d.tile_x) * (double)(d.nely / d.tile_y);
  const double scale = 1.0 / ((double)pa.R * (double)d.ne * volfrac);
  for (int t = blockIdx.x * FB + threadIdx.x; t < d.nt; t += gridDim.x * FB) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < pa.R; ++k) {
      const double h = heaviside_d(xt[t], pa.beta, pa.eta[k]);
      a += scal[8 + k] * (h * dcT[(size_t)k * d.nt + t]);
      b += h * count * scale;
    }
    g1[t] = a;
    g2[t] = b;
  }
}

__global__ void k_filter_adjoint2(Dims d, const double* __restrict__ g1,
                                  const double* __restrict__ g2, double* o1, double* o2,
                                  FiltArgs fa) {
  for (int t = blockIdx.x * FB + threadIdx.x; t < d.nt; t += gridDim.x * FB) {
    o1[t] = tile_filter_adj(g1, t, d.tile_x, d.tile_y, fa.dx, fa.dy, fa.w, fa.n, fa.wsum);
    o2[t] = tile_filter_adj(g2, t, d.tile_x, d.tile_y, fa.dx, fa.dy, fa.w, fa.n, fa.wsum);
  }
}

__device__ double block_sum_1024(double v, double* sm) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((tid & 31) == 0) sm[tid >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (tid < 32) {
    s = (tid < (int)(blockDim.x >> 5)) ? sm[tid] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (tid == 0) sm[32] = s;
  }
  __syncthreads();
  s = sm[32];
  __syncthreads();
  return s;
}

// volume constraint of the current projected tiles: scal[3] = g (Eq. 17)
__global__ void k_volume(Dims d, const double* __restrict__ xbar, double* scal, int R,
                         double volfrac) {
  __shared__ double sm[33];
  const double count = (double)(d.nelx / d.tile_x) * (double)(d.nely / d.tile_y);
  double s = 0.0;
  for (int t = threadIdx.x; t < d.nt; t += blockDim.x)
    for (int k = 0; k < R; ++k) s += xbar[(size_t)k * d.nt + t];
  s = block_sum_1024(s, sm);
  if (threadIdx.x == 0) scal[3] = s * count / ((double)R * (double)d.ne * volfrac) - 1.0;
}

// OC update with bisection (reading R11); one CTA, tile-sized work per bisection step
__global__ void __launch_bounds__(1024) k_oc(Dims d, const double* __restrict__ x,
                                             const double* __restrict__ dF,
                                             const double* __restrict__ dg, double* xnew,
                                             FiltArgs fa, ProjArgs pa, double volfrac,
                                             double move) {
  __shared__ double sm[33];
  const double count = (double)(d.nelx / d.tile_x) * (double)(d.nely / d.tile_y);
  double l1 = 0.0, l2 = 1e9;
  while ((l2 - l1) / (l1 + l2) > 1e-3) {
    const double lmid = 0.5 * (l1 + l2);
    for (int t = threadIdx.x; t < d.nt; t += blockDim.x) {
      const double ratio = fmax(0.0, -dF[t]) / fmax(dg[t], 1e-30);
      const double lo = fmax(0.0, x[t] - move), hi = fmin(1.0, x[t] + move);
      xnew[t] = fmin(hi, fmax(lo, x[t] * sqrt(ratio / lmid)));
    }
    __syncthreads();
    double s = 0.0;
    for (int t = threadIdx.x; t < d.nt; t += blockDim.x) {
      const double v = tile_filter(xnew, t, d.tile_x, d.tile_y, fa.dx, fa.dy, fa.w, fa.n, fa.wsum);
      for (int k = 0; k < pa.R; ++k) s += heaviside(v, pa.beta, pa.eta[k]);
    }
    s = block_sum_1024(s, sm);
    const double g = s * count / ((double)pa.R * (double)d.ne * volfrac) - 1.0;
    if (g > 0.0)
      l1 = lmid;
    else
      l2 = lmid;
    __syncthreads();
  }
}

FiltArgs filt_args(msf_ctx* c) {
  return FiltArgs{c->filt_dx_d, c->filt_dy_d, c->filt_w_d, c->n_filt, c->filt_wsum};
}
ProjArgs proj_args(msf_ctx* c) {
  ProjArgs pa{};
  pa.beta = c->p.beta;
  pa.R = c->d.R;
  for (int k = 0; k < MSF_MAX_RHS; ++k) pa.eta[k] = c->p.eta[k];
  return pa;
}
inline int tblocks(int n) {
  int b = (n + FB - 1) / FB;
  return b < 1184 ? (b > 0 ? b : 1) : 1184;
}

}  // namespace

void launch_filter_project(msf_ctx* c, const double* x_tile) {
  const Dims& d = c->d;
  k_filter_project<<<tblocks(d.nt), FB, 0, c->stream>>>(d, x_tile, c->xt_tile, c->xbar_tile,
                                                        filt_args(c), proj_args(c));
  MSF_LAUNCHED(c);
  dim3 g((d.nely + FB - 1) / FB, d.nelx < 4096 ? d.nelx : 4096, d.R);
  k_moduli<<<g, FB, 0, c->stream>>>(d, c->xbar_tile, c->E, c->p.E0, c->p.Emin, c->p.penal);
  MSF_LAUNCHED(c);
}

void launch_set_physical(msf_ctx* c, int rhs, const double* xb_el) {
  const Dims& d = c->d;
  k_set_physical<<<tblocks(d.ne), FB, 0, c->stream>>>(d, xb_el, c->E + (size_t)rhs * d.ne,
                                                       c->p.E0, c->p.Emin, c->p.penal);
  MSF_LAUNCHED(c);
}

void launch_sens_local(msf_ctx* c) {
  const Dims& d = c->d;
  launch_compliance(c, d.R);
  double* dcT = c->tile_tmp;                 // [R*nt] (R <= 4 slots of tile_tmp)
  const int ncol = c->sb.e1 - c->sb.e0;
  if (c->comm) cudaMemsetAsync(c->dc_el, 0, (size_t)d.ne * sizeof(double), c->stream);
  for (int k = 0; k < d.R; ++k) {
    dim3 g((d.nely + FB - 1) / FB, ncol < 4096 ? ncol : 4096, 1);
    k_dc_element<<<g, FB, 0, c->stream>>>(d, c->K0,
                                          (const double2*)(c->u + (size_t)k * 2 * c->dl.nn),
                                          c->xbar_tile + (size_t)k * d.nt, c->dc_el, c->p.E0,
                                          c->p.Emin, c->p.penal, c->sb.e0, c->sb.e1, c->dl.gox);
    MSF_LAUNCHED(c);
    k_tile_sum<<<tblocks(d.nt), FB, 0, c->stream>>>(d, c->dc_el, dcT + (size_t)k * d.nt);
    MSF_LAUNCHED(c);
  }
}

void launch_sensitivities(msf_ctx* c, double kappa, double volfrac) {
  launch_sens_local(c);
  launch_sens_global(c, kappa, volfrac);
}

void launch_sens_global(msf_ctx* c, double kappa, double volfrac) {
  const Dims& d = c->d;
  double* dcT = c->tile_tmp;
  k_robust_weights<<<1, 32, 0, c->stream>>>(c->sc, d.R, kappa, c->scal);
  MSF_LAUNCHED(c);
  // g1 -> dc_el[0:nt], g2 -> dc_el[nt:2nt] (scratch, ne >= 2 nt not assumed: use x_new/dg)
  double* g1 = c->dc_el;
  double* g2 = c->dc_el + d.nt;
  k_chain_pre<<<tblocks(d.nt), FB, 0, c->stream>>>(d, c->xt_tile, dcT, c->scal, g1, g2,
                                                   proj_args(c), volfrac);
  MSF_LAUNCHED(c);
  k_filter_adjoint2<<<tblocks(d.nt), FB, 0, c->stream>>>(d, g1, g2, c->dF, c->dg, filt_args(c));
  MSF_LAUNCHED(c);
  k_volume<<<1, 1024, 0, c->stream>>>(d, c->xbar_tile, c->scal, d.R, volfrac);
  MSF_LAUNCHED(c);
}

void launch_oc(msf_ctx* c, const double* x, const double* dF, const double* dg, double volfrac,
               double move, double* x_new) {
  k_oc<<<1, 1024, 0, c->stream>>>(c->d, x, dF, dg, x_new, filt_args(c), proj_args(c), volfrac,
                                  move);
  MSF_LAUNCHED(c);
}
