// Spectral MsFEM coarse basis (§2.4, Eq. 9, §3.2).
//
// For every agglomerate class (§2.4.1: periodic designs have few unique
// agglomerates) one CTA computes the n_modes smallest eigenpairs of
//        K_omega psi = lambda diag(K_omega) psi
// where K_omega is the Neumann stiffness of the elements of omega_i with the physical
// Dirichlet DOFs of the full problem removed (line 130), by shift-invert block subspace
// iteration with Rayleigh-Ritz:
//   A = K_omega - sigma D (SPD, sigma < 0) is block tridiagonal over the node columns of
//   the box; it is factorised once by block Thomas with explicit SPD block inverses
//   (sweep operator in shared memory); each iteration solves A Y = D X, forms the
//   projected pencil (Y^T K Y, Y^T D Y), solves it with Cholesky + cyclic Jacobi in one
//   warp, and updates X = Y C.  Converged when every kept Ritz pair has
//   ||K x - theta D x||_{D^-1} <= eig_tol (x D-normalised).
// The basis phi_{i,a} = chi_i psi_a (bilinear partition of unity, reading R6) is written on
// the padded (2cx+1)x(2cy+1)-node box of the class.
#include "msf_internal.cuh"

namespace {

constexpr int NT = 256;

struct EigArgs {
  double sigma;
  double tol;
  double lam_thr;
  int maxit;
  int mb;
  int mlmax;   // max block size (smem sizing)
};

__device__ __forceinline__ int local_a(int dx, int dy) {
  return (dx == 0) ? (dy == 0 ? 0 : 3) : (dy == 0 ? 1 : 2);
}

// Entry of the (unshifted, Neumann) box stiffness between DOF (lx,ly,c) and (lx2,ly2,c2).
__device__ double box_K(const Dims& d, const K0Mat& K, const double* __restrict__ E,
                        const EigClass& C, int lx, int ly, int c, int lx2, int ly2, int c2) {
  if (abs(lx - lx2) > 1 || abs(ly - ly2) > 1) return 0.0;
  double v = 0.0;
  const int ex_lo = max(max(lx, lx2) - 1, 0), ex_hi = min(min(lx, lx2), C.nbx - 2);
  const int ey_lo = max(max(ly, ly2) - 1, 0), ey_hi = min(min(ly, ly2), C.nby - 2);
  for (int ex = ex_lo; ex <= ex_hi; ++ex)
    for (int ey = ey_lo; ey <= ey_hi; ++ey) {
      const int a = local_a(lx - ex, ly - ey), b = local_a(lx2 - ex, ly2 - ey);
      const double Ee = E[(size_t)(C.bx0 + ex) * d.nely + (C.by0 + ey)];
      v = fma(Ee, K.v[(2 * a + c) * 8 + 2 * b + c2], v);
    }
  return v;
}

__device__ __forceinline__ bool dof_fixed(const Dims& d, const uint8_t* __restrict__ fixn,
                                          const EigClass& C, int lx, int ly, int c) {
  return (fixn[(size_t)(C.bx0 + lx) * d.nny + (C.by0 + ly)] >> c) & 1;
}

// S (ml x ml) = A block (rows node column Ir, cols node column Ic) of A = K - sigma D with
// identity rows/cols on fixed DOFs.
__device__ void assemble_block(const Dims& d, const K0Mat& K, const double* __restrict__ E,
                               const uint8_t* __restrict__ fixn, const EigClass& C, int Ir,
                               int Ic, double sigma, double* S, int ml) {
  for (int e = threadIdx.x; e < ml * ml; e += NT) {
    const int r = e / ml, cc = e - (e / ml) * ml;
    const int ly = r >> 1, c = r & 1, ly2 = cc >> 1, c2 = cc & 1;
    double v;
    const bool fr = dof_fixed(d, fixn, C, Ir, ly, c), fc = dof_fixed(d, fixn, C, Ic, ly2, c2);
    if (fr || fc) {
      v = (Ir == Ic && r == cc) ? 1.0 : 0.0;
    } else {
      v = box_K(d, K, E, C, Ir, ly, c, Ic, ly2, c2);
      if (Ir == Ic && r == cc) v -= sigma * v;   // D = diag(K)
    }
    S[e] = v;
  }
}

// in-place SPD inverse of S (m x m, shared memory) by the sweep operator
__device__ void cta_inverse(double* S, int m, double* rowk, double* colk, int* status) {
  for (int k = 0; k < m; ++k) {
    for (int i = threadIdx.x; i < m; i += NT) {
      rowk[i] = S[k * m + i];
      colk[i] = S[i * m + k];
    }
    __syncthreads();
    const double piv = rowk[k];
    if (!(piv > 0.0) && threadIdx.x == 0) atomicExch(status, 2);
    const double ip = 1.0 / piv;
    for (int e = threadIdx.x; e < m * m; e += NT) {
      const int i = e / m, j = e - (e / m) * m;
      double v;
      if (i == k && j == k) v = -ip;
      else if (i == k) v = rowk[j] * ip;
      else if (j == k) v = colk[i] * ip;
      else v = S[e] - colk[i] * rowk[j] * ip;
      S[e] = v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * m; e += NT) S[e] = -S[e];
  __syncthreads();
}

__device__ __forceinline__ double hash_uniform(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return (double)(x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// Small generalised symmetric eigenproblem G c = theta H c (mb <= 24), executed by warp 0.
// Outputs theta ascending and Cm (columns = H-orthonormal eigenvectors).  Work: L, M, V.
__device__ void small_gen_eig(double* G, double* H, int mb, double* theta, double* Cm,
                              double* L, double* M, double* V, int* status) {
  const int lane = threadIdx.x & 31;
  // Cholesky H = L L^T
  for (int i = lane; i < mb * mb; i += 32) L[i] = 0.0;
  __syncwarp();
  for (int j = 0; j < mb; ++j) {
    if (lane == 0) {
      double s = H[j * mb + j];
      for (int k = 0; k < j; ++k) s -= L[j * mb + k] * L[j * mb + k];
      if (!(s > 0.0)) {
        atomicExch(status, 3);
        s = 1e-300;
      }
      L[j * mb + j] = sqrt(s);
    }
    __syncwarp();
    for (int i = j + 1 + lane; i < mb; i += 32) {
      double s = H[i * mb + j];
      for (int k = 0; k < j; ++k) s -= L[i * mb + k] * L[j * mb + k];
      L[i * mb + j] = s / L[j * mb + j];
    }
    __syncwarp();
  }
  // Z = L^{-1} G  (column c per lane) -> stored in V
  if (lane < mb) {
    const int c = lane;
    for (int i = 0; i < mb; ++i) {
      double s = G[i * mb + c];
      for (int k = 0; k < i; ++k) s -= L[i * mb + k] * V[k * mb + c];
      V[i * mb + c] = s / L[i * mb + i];
    }
  }
  __syncwarp();
  // M^T = L^{-1} Z^T : column c of Z^T is row c of Z
  if (lane < mb) {
    const int c = lane;
    for (int i = 0; i < mb; ++i) {
      double s = V[c * mb + i];
      for (int k = 0; k < i; ++k) s -= L[i * mb + k] * M[c * mb + k];
      M[c * mb + i] = s / L[i * mb + i];   // M[c][i] = (L^{-1} Z^T)[i][c]
    }
  }
  __syncwarp();
  // symmetrise, V = I
  for (int e = lane; e < mb * mb; e += 32) {
    const int i = e / mb, j = e - (e / mb) * mb;
    if (i < j) {
      const double a = 0.5 * (M[i * mb + j] + M[j * mb + i]);
      M[i * mb + j] = a;
      M[j * mb + i] = a;
    }
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncwarp();
  // cyclic Jacobi
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = lane; e < mb * mb; e += 32) {
      const int i = e / mb, j = e - (e / mb) * mb;
      const double v = M[e] * M[e];
      tot += v;
      if (i != j) off += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < mb - 1; ++p)
      for (int q = p + 1; q < mb; ++q) {
        const double apq = M[p * mb + q];
        if (apq == 0.0) continue;
        const double app = M[p * mb + p], aqq = M[q * mb + q];
        const double tau = (aqq - app) / (2.0 * apq);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        __syncwarp();
        if (lane < mb) {
          const int k = lane;
          const double a = M[k * mb + p], b = M[k * mb + q];
          M[k * mb + p] = c * a - s * b;
          M[k * mb + q] = s * a + c * b;
          const double va = V[k * mb + p], vb = V[k * mb + q];
          V[k * mb + p] = c * va - s * vb;
          V[k * mb + q] = s * va + c * vb;
        }
        __syncwarp();
        if (lane < mb) {
          const int k = lane;
          const double a = M[p * mb + k], b = M[q * mb + k];
          M[p * mb + k] = c * a - s * b;
          M[q * mb + k] = s * a + c * b;
        }
        __syncwarp();
        if (lane == 0) {
          M[p * mb + q] = 0.0;
          M[q * mb + p] = 0.0;
        }
        __syncwarp();
      }
  }
  // sort ascending (lane 0), theta and permutation into G (as scratch ints in doubles)
  if (lane == 0) {
    for (int i = 0; i < mb; ++i) {
      theta[i] = M[i * mb + i];
      G[i] = (double)i;
    }
    for (int i = 0; i < mb; ++i) {
      int best = i;
      for (int j = i + 1; j < mb; ++j)
        if (theta[j] < theta[best]) best = j;
      const double tv = theta[i];
      theta[i] = theta[best];
      theta[best] = tv;
      const double pv = G[i];
      G[i] = G[best];
      G[best] = pv;
    }
  }
  __syncwarp();
  // Cm = L^{-T} V(:, perm)
  if (lane < mb) {
    const int c = lane;
    const int src = (int)G[c];
    for (int i = mb - 1; i >= 0; --i) {
      double s = V[i * mb + src];
      for (int k = i + 1; k < mb; ++k) s -= L[k * mb + i] * Cm[k * mb + c];
      Cm[i * mb + c] = s / L[i * mb + i];
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(NT) k_eigen(Dims d, K0Mat K, const double* __restrict__ E,
                                              const uint8_t* __restrict__ fixn,
                                              EigClass* classes, double* work, double* phi,
                                              double* lam, EigArgs ea, int* status) {
  extern __shared__ double sm[];
  EigClass C = classes[blockIdx.x];
  const int ml = 2 * C.nby, nbl = C.nbx, n = nbl * ml;
  const int mb = ea.mb;
  const int sz = ml * max(ml, mb);
  double* S = sm;                 // [sz]
  double* T = S + sz;             // [sz]
  double* G = T + sz;             // [mb*mb]
  double* H = G + mb * mb;
  double* Cm = H + mb * mb;
  double* Lw = Cm + mb * mb;
  double* Mw = Lw + mb * mb;
  double* Vw = Mw + mb * mb;
  double* theta = Vw + mb * mb;   // [mb]
  double* rowk = theta + 32;      // [ml]
  double* colk = rowk + ea.mlmax; // [ml]
  double* red = colk + ea.mlmax;  // [NT/32 * 32]
  __shared__ int s_stop;

  double* Sinv = work + C.off;
  double* W = Sinv + (size_t)nbl * ml * ml;
  double* X = W + (size_t)nbl * ml * ml;
  double* Y = X + (size_t)n * mb;
  double* KY = Y + (size_t)n * mb;
  double* Dv = KY + (size_t)n * mb;

  // ---------------- factorisation A = K - sigma D by block Thomas
  for (int I = 0; I < nbl; ++I) {
    assemble_block(d, K, E, fixn, C, I, I, ea.sigma, S, ml);
    if (I > 0) {
      assemble_block(d, K, E, fixn, C, I - 1, I, ea.sigma, T, ml);   // U_{I-1}
      __syncthreads();
      const double* Sp = Sinv + (size_t)(I - 1) * ml * ml;
      double* WI = W + (size_t)I * ml * ml;
      for (int e = threadIdx.x; e < ml * ml; e += NT) {
        const int r = e / ml, cc = e - (e / ml) * ml;
        double s = 0.0;
        for (int k = 0; k < ml; ++k) s = fma(Sp[r * ml + k], T[k * ml + cc], s);
        WI[e] = s;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < ml * ml; e += NT) {
        const int r = e / ml, cc = e - (e / ml) * ml;
        double s = 0.0;
        for (int k = 0; k < ml; ++k) s = fma(T[k * ml + r], WI[k * ml + cc], s);
        S[e] -= s;
      }
    }
    __syncthreads();
    cta_inverse(S, ml, rowk, colk, status);
    double* SI = Sinv + (size_t)I * ml * ml;
    for (int e = threadIdx.x; e < ml * ml; e += NT) SI[e] = S[e];
    __syncthreads();
  }
  // ---------------- D = diag(K) on free DOFs, random start
  for (int i = threadIdx.x; i < n; i += NT) {
    const int lx = i / ml, rr = i - (i / ml) * ml, ly = rr >> 1, c = rr & 1;
    Dv[i] = dof_fixed(d, fixn, C, lx, ly, c) ? 0.0 : box_K(d, K, E, C, lx, ly, c, lx, ly, c);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * mb; e += NT) {
    const int i = e / mb;
    X[e] = (Dv[i] > 0.0) ? hash_uniform((unsigned long long)e * 2654435761ull + 17ull) : 0.0;
  }
  __syncthreads();

  int it = 0;
  for (; it < ea.maxit; ++it) {
    // Y = D X
    for (int e = threadIdx.x; e < n * mb; e += NT) Y[e] = Dv[e / mb] * X[e];
    __syncthreads();
    // forward: Y_I -= W_I^T Y_{I-1}
    for (int I = 1; I < nbl; ++I) {
      const double* WI = W + (size_t)I * ml * ml;
      const double* Yp = Y + (size_t)(I - 1) * ml * mb;
      double* Yc = Y + (size_t)I * ml * mb;
      for (int e = threadIdx.x; e < ml * mb; e += NT) {
        const int r = e / mb, j = e - (e / mb) * mb;
        double s = 0.0;
        for (int k = 0; k < ml; ++k) s = fma(WI[k * ml + r], Yp[k * mb + j], s);
        Yc[e] -= s;
      }
      __syncthreads();
    }
    // Y_I = Sinv_I Y_I
    for (int I = 0; I < nbl; ++I) {
      double* Yc = Y + (size_t)I * ml * mb;
      for (int e = threadIdx.x; e < ml * mb; e += NT) T[e] = Yc[e];
      __syncthreads();
      const double* SI = Sinv + (size_t)I * ml * ml;
      for (int e = threadIdx.x; e < ml * mb; e += NT) {
        const int r = e / mb, j = e - (e / mb) * mb;
        double s = 0.0;
        for (int k = 0; k < ml; ++k) s = fma(SI[r * ml + k], T[k * mb + j], s);
        Yc[e] = s;
      }
      __syncthreads();
    }
    // back: Y_I -= W_{I+1} Y_{I+1}
    for (int I = nbl - 2; I >= 0; --I) {
      const double* WI = W + (size_t)(I + 1) * ml * ml;
      const double* Yn = Y + (size_t)(I + 1) * ml * mb;
      double* Yc = Y + (size_t)I * ml * mb;
      for (int e = threadIdx.x; e < ml * mb; e += NT) {
        const int r = e / mb, j = e - (e / mb) * mb;
        double s = 0.0;
        for (int k = 0; k < ml; ++k) s = fma(WI[r * ml + k], Yn[k * mb + j], s);
        Yc[e] -= s;
      }
      __syncthreads();
    }
    // KY = K Y (unshifted Neumann box stiffness, fixed rows -> 0)
    for (int e = threadIdx.x; e < n * mb; e += NT) {
      const int i = e / mb, j = e - (e / mb) * mb;
      double s = 0.0;
      if (Dv[i] > 0.0) {
        const int lx = i / ml, rr = i - (i / ml) * ml, ly = rr >> 1, c = rr & 1;
        for (int lx2 = max(lx - 1, 0); lx2 <= min(lx + 1, nbl - 1); ++lx2)
          for (int ly2 = max(ly - 1, 0); ly2 <= min(ly + 1, C.nby - 1); ++ly2)
            for (int c2 = 0; c2 < 2; ++c2) {
              const int i2 = lx2 * ml + 2 * ly2 + c2;
              if (Dv[i2] > 0.0)
                s = fma(box_K(d, K, E, C, lx, ly, c, lx2, ly2, c2), Y[(size_t)i2 * mb + j], s);
            }
      }
      KY[e] = s;
    }
    __syncthreads();
    // G = Y^T KY, H = Y^T D Y
    for (int e = threadIdx.x; e < 2 * mb * mb; e += NT) {
      const int which = e / (mb * mb), ee = e - which * mb * mb;
      const int a = ee / mb, b = ee - (ee / mb) * mb;
      double s = 0.0;
      if (which == 0)
        for (int i = 0; i < n; ++i) s = fma(Y[(size_t)i * mb + a], KY[(size_t)i * mb + b], s);
      else
        for (int i = 0; i < n; ++i) s = fma(Y[(size_t)i * mb + a] * Dv[i], Y[(size_t)i * mb + b], s);
      (which == 0 ? G : H)[ee] = s;
    }
    __syncthreads();
    if (threadIdx.x < 32) small_gen_eig(G, H, mb, theta, Cm, Lw, Mw, Vw, status);
    __syncthreads();
    // X = Y Cm ; then KX = KY Cm into Y
    for (int e = threadIdx.x; e < n * mb; e += NT) {
      const int i = e / mb, j = e - (e / mb) * mb;
      double s = 0.0;
      for (int l = 0; l < mb; ++l) s = fma(Y[(size_t)i * mb + l], Cm[l * mb + j], s);
      X[e] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * mb; e += NT) {
      const int i = e / mb, j = e - (e / mb) * mb;
      double s = 0.0;
      for (int l = 0; l < mb; ++l) s = fma(KY[(size_t)i * mb + l], Cm[l * mb + j], s);
      Y[e] = s;
    }
    __syncthreads();
    // residuals of the kept pairs
    const int kk = min(d.kmax, mb);
    for (int j = 0; j < kk; ++j) {
      double s = 0.0;
      for (int i = threadIdx.x; i < n; i += NT) {
        if (Dv[i] > 0.0) {
          const double rv = Y[(size_t)i * mb + j] - theta[j] * Dv[i] * X[(size_t)i * mb + j];
          s += rv * rv / Dv[i];
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((threadIdx.x & 31) == 0) red[j * (NT / 32) + (threadIdx.x >> 5)] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double mx = 0.0;
      for (int j = 0; j < kk; ++j) {
        double s = 0.0;
        for (int w = 0; w < NT / 32; ++w) s += red[j * (NT / 32) + w];
        mx = fmax(mx, s);
      }
      s_stop = (sqrt(mx) <= ea.tol) ? 1 : 0;
    }
    __syncthreads();
    if (s_stop) {
      ++it;
      break;
    }
  }
  // ---------------- write phi = chi psi on the padded box, eigenvalues, kept count
  int nk = min(d.kmax, mb);
  if (ea.lam_thr > 0.0 && ea.lam_thr < 1e300) {
    int cnt = 0;
    while (cnt < nk && theta[cnt] < ea.lam_thr) ++cnt;
    nk = cnt;
  }
  const int I = C.rep_agg / (d.ncy + 1), J = C.rep_agg - (C.rep_agg / (d.ncy + 1)) * (d.ncy + 1);
  const int gx0 = I * d.cx - d.cx, gy0 = J * d.cy - d.cy;
  double* ph = phi + (size_t)blockIdx.x * d.kmax * d.box_nodes * 2;
  for (int e = threadIdx.x; e < d.kmax * d.box_nodes * 2; e += NT) {
    const int a = e / (d.box_nodes * 2), rest = e - a * d.box_nodes * 2;
    const int bn = rest >> 1, c = rest & 1;
    const int px = bn / d.by, py = bn - (bn / d.by) * d.by;
    const int lx = gx0 + px - C.bx0, ly = gy0 + py - C.by0;
    double v = 0.0;
    if (a < nk && lx >= 0 && lx < C.nbx && ly >= 0 && ly < C.nby) {
      const int i = lx * ml + 2 * ly + c;
      const double chi = fmax(0.0, 1.0 - fabs((double)(px - d.cx)) / d.cx) *
                         fmax(0.0, 1.0 - fabs((double)(py - d.cy)) / d.cy);
      v = chi * X[(size_t)i * mb + a];
    }
    ph[e] = v;
  }
  for (int a = threadIdx.x; a < d.kmax; a += NT)
    lam[(size_t)blockIdx.x * d.kmax + a] = (a < mb) ? theta[a] : 0.0;
  if (threadIdx.x == 0) {
    classes[blockIdx.x].iters = it;
    classes[blockIdx.x].nkept = nk;
  }
}

}  // namespace

size_t eig_smem_bytes(int mlmax, int mb) {
  const int sz = mlmax * (mlmax > mb ? mlmax : mb);
  return (size_t)(2 * sz + 6 * mb * mb + 32 + 2 * mlmax + MSF_MAX_BLOCK_EIG * (NT / 32)) *
         sizeof(double);
}

void launch_build_basis(msf_ctx* c) {
  const Dims& d = c->d;
  EigArgs ea;
  ea.sigma = -1e-3;
  ea.tol = c->p.eig_tol > 0.0 ? c->p.eig_tol : 1e-9;
  ea.lam_thr = c->p.lam_threshold;
  ea.maxit = c->p.eig_max_iter > 0 ? c->p.eig_max_iter : 60;
  ea.mb = c->mb;
  ea.mlmax = 2 * d.by;
  const size_t smem = eig_smem_bytes(ea.mlmax, ea.mb);
  cudaFuncSetAttribute(k_eigen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_eigen<<<c->n_cls, NT, smem, c->stream>>>(d, c->K0,
                                              c->E + (size_t)c->p.dilated * d.ne, c->fixg,
                                              c->classes_d, c->eig_work, c->phi, c->lam, ea,
                                              c->factor_status + MSF_MAX_RHS);
  MSF_LAUNCHED(c);
}
