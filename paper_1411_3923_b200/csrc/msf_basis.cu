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
#include <algorithm>

#include "msf_internal.cuh"
#include "msf_inverse.cuh"

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

// in-place SPD inverse of S (m x m, shared memory) by the sweep operator.  Threads are laid
// out as NT/32 row groups x 32 column lanes, so no index division in the m sweep steps.
__device__ void cta_inverse(double* S, int m, double* rowk, double* colk, int* status) {
  const int jl = threadIdx.x & 31, ig = threadIdx.x >> 5;
  constexpr int RG = NT / 32;
  for (int k = 0; k < m; ++k) {
    for (int i = threadIdx.x; i < m; i += NT) {
      rowk[i] = S[k * m + i];
      colk[i] = S[i * m + k];
    }
    __syncthreads();
    const double piv = rowk[k];
    if (!(piv > 0.0) && threadIdx.x == 0) atomicExch(status, 2);
    const double ip = 1.0 / piv;
    for (int i = ig; i < m; i += RG) {
      const double ci = colk[i] * ip;
      double* Si = S + i * m;
      if (i == k) {
        for (int j = jl; j < m; j += 32) Si[j] = (j == k) ? -ip : rowk[j] * ip;
      } else {
        for (int j = jl; j < m; j += 32) Si[j] = (j == k) ? ci : fma(-ci, rowk[j], Si[j]);
      }
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

// Thread-block cluster per class: EIG_CL CTAs share the per-iteration work of one class
// (8x the threads of a single CTA on these latency-bound loops); phases are separated by
// cluster barriers (release / acquire: global writes of one CTA are visible to the others).
#ifndef MSF_EIG_CL
#define MSF_EIG_CL 8
#endif
constexpr int EIG_CL = MSF_EIG_CL;   // <= 8: the workspace holds 8 x 16 residual partials per class

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// s = sum_k A[k*sa] B[k*sb], 4 independent accumulators
__device__ __forceinline__ double dot4(const double* A, int sa, const double* B, int sb, int n) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = 0;
  for (; k + 3 < n; k += 4) {
    s0 = fma(A[(size_t)k * sa], B[(size_t)k * sb], s0);
    s1 = fma(A[(size_t)(k + 1) * sa], B[(size_t)(k + 1) * sb], s1);
    s2 = fma(A[(size_t)(k + 2) * sa], B[(size_t)(k + 2) * sb], s2);
    s3 = fma(A[(size_t)(k + 3) * sa], B[(size_t)(k + 3) * sb], s3);
  }
  for (; k < n; ++k) s0 = fma(A[(size_t)k * sa], B[(size_t)k * sb], s0);
  return (s0 + s1) + (s2 + s3);
}

// C[0:m,0:m] (ld m) = beta C + alpha A B, A element (r, k) at A[r*ar + k*ak], B (k, c) at
// B[k*m + c], all in shared memory; 4x4 outputs per thread (0.5 shared loads per FMA).
__device__ void smem_gemm44(const double* A, int ar, int ak, const double* B, double* C, int m,
                            double alpha, double beta, double* C2 = nullptr) {
  const int nt = (m + 3) / 4;
  for (int tile = threadIdx.x; tile < nt * nt; tile += NT) {
    const int r0 = (tile / nt) * 4, c0 = (tile - (tile / nt) * nt) * 4;
    double acc[4][4] = {};
    for (int k = 0; k < m; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = (r0 + i < m) ? A[(r0 + i) * ar + k * ak] : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = (c0 + j < m) ? B[k * m + c0 + j] : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (r0 + i < m && c0 + j < m) {
          const int e = (r0 + i) * m + c0 + j;
          const double v = (beta != 0.0 ? beta * C[e] : 0.0) + alpha * acc[i][j];
          C[e] = v;
          if (C2) C2[e] = v;
        }
  }
}

// All diagonal blocks D_I of A = K - sigma D and coupling blocks U_{I-1} of every class in
// parallel (blockIdx.x = class * 2 * nbl_max + 2 I + {0: D_I -> Sinv slot I, 1: U_{I-1} -> W
// slot I}); the sequential block-Thomas kernel then only multiplies and inverts.
__global__ void __launch_bounds__(NT) k_eigen_blocks(Dims d, K0Mat K, const double* __restrict__ E,
                                                     const uint8_t* __restrict__ fixn,
                                                     const EigClass* __restrict__ classes,
                                                     double* work, EigArgs ea, int nbl_max) {
  const int cls = blockIdx.x / (2 * nbl_max), rest = blockIdx.x - cls * 2 * nbl_max;
  const int I = rest >> 1, which = rest & 1;
  const EigClass C = classes[cls];
  const int ml = 2 * C.nby, nbl = C.nbx;
  if (I >= nbl || (which == 1 && I == 0)) return;
  double* Sinv = work + C.off;
  double* W = Sinv + (size_t)nbl * ml * ml;
  if (which == 0)
    assemble_block(d, K, E, fixn, C, I, I, ea.sigma, Sinv + (size_t)I * ml * ml, ml);
  else
    assemble_block(d, K, E, fixn, C, I - 1, I, ea.sigma, W + (size_t)I * ml * ml, ml);
}

__global__ void __launch_bounds__(NT) k_eigen_factor(Dims d, K0Mat K, const double* __restrict__ E,
                                              const uint8_t* __restrict__ fixn,
                                              EigClass* classes, double* work, double* phi,
                                              double* lam, EigArgs ea, int* status) {
  extern __shared__ double sm[];
  // one CTA per class: A = K - sigma D by block Thomas in shared memory
  const int cls = blockIdx.x;
  EigClass C = classes[cls];
  const int ml = 2 * C.nby, nbl = C.nbx, n = nbl * ml;
  const int mb = ea.mb;
  const int sz = ml * max(ml, mb);
  double* S = sm;                 // [sz]
  double* T = S + sz;             // [sz]
  double* Pv = T + sz;            // [sz] previous block inverse
  double* Wv = Pv + sz;           // [sz] current W block
  double* rowk = Wv + sz;         // [ml]
  double* colk = rowk + ea.mlmax; // [ml]

  double* Sinv = work + C.off;
  double* W = Sinv + (size_t)nbl * ml * ml;

  {
    for (int I = 0; I < nbl; ++I) {
      // D_I and U_{I-1} were assembled by k_eigen_blocks into the Sinv / W slots of I
      const double* DI = Sinv + (size_t)I * ml * ml;
      for (int e = threadIdx.x; e < ml * ml; e += NT) S[e] = DI[e];
      if (I > 0) {
        const double* UI = W + (size_t)I * ml * ml;
        for (int e = threadIdx.x; e < ml * ml; e += NT) T[e] = UI[e];
        __syncthreads();
        double* WI = W + (size_t)I * ml * ml;
        smem_gemm44(Pv, ml, 1, T, Wv, ml, 1.0, 0.0, WI);              // W_I = Sinv_{I-1} U_{I-1}
        __syncthreads();
        smem_gemm44(T, 1, ml, Wv, S, ml, -1.0, 1.0);                 // S -= U^T W
      }
      __syncthreads();
      // T and Wv are dead here (W_I is in global memory): scratch of the blocked inverse
      if (ml <= 96) msfinv::inverse_blocked<NT, 3>(S, ml, T, status);
      else cta_inverse(S, ml, rowk, colk, status);
      double* SI = Sinv + (size_t)I * ml * ml;
      for (int e = threadIdx.x; e < ml * ml; e += NT) {
        SI[e] = S[e];
        Pv[e] = S[e];
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(NT) k_eigen(Dims d, K0Mat K, const double* __restrict__ E,
                                              const uint8_t* __restrict__ fixn,
                                              EigClass* classes, double* work, double* phi,
                                              double* lam, EigArgs ea, int* status) {
  extern __shared__ double sm[];
  const int cls = blockIdx.x / EIG_CL, rank = blockIdx.x - cls * EIG_CL;
  const int t0 = rank * NT + threadIdx.x, tstride = EIG_CL * NT;   // cluster-wide thread index
  EigClass C = classes[cls];
  const int ml = 2 * C.nby, nbl = C.nbx, n = nbl * ml;
  const int mb = ea.mb;
  double* G = sm;                 // [mb*mb]
  double* H = G + mb * mb;
  double* Cm = H + mb * mb;
  double* Lw = Cm + mb * mb;
  double* Mw = Lw + mb * mb;
  double* Vw = Mw + mb * mb;
  double* theta = Vw + mb * mb;   // [mb]

  double* Sinv = work + C.off;
  double* W = Sinv + (size_t)nbl * ml * ml;
  double* X = W + (size_t)nbl * ml * ml;
  double* Y = X + (size_t)n * mb;
  double* KY = Y + (size_t)n * mb;
  double* Dv = KY + (size_t)n * mb;
  double* gG = Dv + n;                 // [mb*mb] cluster-shared scratch (global)
  double* gH = gG + mb * mb;           // [mb*mb]
  double* gC = gH + mb * mb;           // [mb*mb] Ritz coefficients
  double* gT = gC + mb * mb;           // [32]   Ritz values
  double* gR = gT + 32;                // [EIG_CL * 16] residual partials

  // ---------------- D = diag(K) on free DOFs, random start
  for (int i = t0; i < n; i += tstride) {
    const int lx = i / ml, rr = i - (i / ml) * ml, ly = rr >> 1, c = rr & 1;
    Dv[i] = dof_fixed(d, fixn, C, lx, ly, c) ? 0.0 : box_K(d, K, E, C, lx, ly, c, lx, ly, c);
  }
  cl_sync();
  for (int e = t0; e < n * mb; e += tstride) {
    const int i = e / mb;
    X[e] = (Dv[i] > 0.0) ? hash_uniform((unsigned long long)e * 2654435761ull + 17ull) : 0.0;
  }
  cl_sync();

  // Three n x mb buffers rotate through an iteration: B0 = X, B1 = D X -> forward-eliminated
  // right-hand side -> K Y, B2 = block-diagonal solve -> Y -> K X.
  double* B0 = X;
  double* B1 = Y;
  double* B2 = KY;
  const int nby = C.nby;
  const int lane = threadIdx.x & 31;
  const int gwarp = rank * (NT / 32) + (threadIdx.x >> 5), nwarps = EIG_CL * (NT / 32);
  int it = 0;
  for (; it < ea.maxit; ++it) {
    for (int e = t0; e < n * mb; e += tstride) B1[e] = Dv[e / mb] * B0[e];
    cl_sync();
    // forward: B1_I -= W_I^T B1_{I-1}  (sequential over the node columns)
    for (int I = 1; I < nbl; ++I) {
      const double* WI = W + (size_t)I * ml * ml;
      const double* Yp = B1 + (size_t)(I - 1) * ml * mb;
      double* Yc = B1 + (size_t)I * ml * mb;
      // two lanes per output (halves of the inner product), combined by a shuffle
      for (int e2 = t0; e2 < 2 * ml * mb + (tstride - (2 * ml * mb) % tstride) % tstride; e2 += tstride) {
        const int e = e2 >> 1, h = e2 & 1;
        double v = 0.0;
        if (e < ml * mb) {
          const int r = e / mb, j = e - (e / mb) * mb;
          const int k0 = h ? ml / 2 : 0, k1 = h ? ml : ml / 2;
          v = dot4(WI + (size_t)k0 * ml + r, ml, Yp + (size_t)k0 * mb + j, mb, k1 - k0);
        }
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (e < ml * mb && h == 0) Yc[e] -= v;
      }
      cl_sync();
    }
    // B2_I = Sinv_I B1_I for all node columns at once (independent blocks)
    for (int e = t0; e < n * mb; e += tstride) {
      const int i = e / mb, j = e - (e / mb) * mb;
      const int I = i / ml, r = i - I * ml;
      B2[e] = dot4(Sinv + (size_t)I * ml * ml + (size_t)r * ml, 1, B1 + (size_t)I * ml * mb + j, mb, ml);
    }
    cl_sync();
    // back: B2_I -= W_{I+1} B2_{I+1}
    for (int I = nbl - 2; I >= 0; --I) {
      const double* WI = W + (size_t)(I + 1) * ml * ml;
      const double* Yn = B2 + (size_t)(I + 1) * ml * mb;
      double* Yc = B2 + (size_t)I * ml * mb;
      for (int e2 = t0; e2 < 2 * ml * mb + (tstride - (2 * ml * mb) % tstride) % tstride; e2 += tstride) {
        const int e = e2 >> 1, h = e2 & 1;
        double v = 0.0;
        if (e < ml * mb) {
          const int r = e / mb, j = e - (e / mb) * mb;
          const int k0 = h ? ml / 2 : 0, k1 = h ? ml : ml / 2;
          v = dot4(WI + (size_t)r * ml + k0, 1, Yn + (size_t)k0 * mb + j, mb, k1 - k0);
        }
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (e < ml * mb && h == 0) Yc[e] -= v;
      }
      cl_sync();
    }
    // B1 = K B2: unshifted Neumann box stiffness element by element, fixed rows -> 0
    for (int e = t0; e < (n / 2) * mb; e += tstride) {
      const int node = e / mb, j = e - (e / mb) * mb;
      const int lx = node / nby, ly = node - (node / nby) * nby;
      double ox = 0.0, oy = 0.0;
#pragma unroll
      for (int sx = 0; sx < 2; ++sx)
#pragma unroll
        for (int sy = 0; sy < 2; ++sy) {
          const int ex = lx - 1 + sx, ey = ly - 1 + sy;
          if (ex < 0 || ex > nbl - 2 || ey < 0 || ey > nby - 2) continue;
          const double Ee = E[(size_t)(C.bx0 + ex) * d.nely + (C.by0 + ey)];
          const int a = local_a(lx - ex, ly - ey);
          double ax = 0.0, ay = 0.0;
#pragma unroll
          for (int bnode = 0; bnode < 4; ++bnode) {
            const int nx = ex + ((bnode == 1 || bnode == 2) ? 1 : 0), ny = ey + (bnode >= 2 ? 1 : 0);
            const size_t i2 = (size_t)nx * ml + 2 * ny;
            const double yx = B2[i2 * mb + j], yy = B2[(i2 + 1) * mb + j];
            ax = fma(K.v[(2 * a) * 8 + 2 * bnode], yx, fma(K.v[(2 * a) * 8 + 2 * bnode + 1], yy, ax));
            ay = fma(K.v[(2 * a + 1) * 8 + 2 * bnode], yx, fma(K.v[(2 * a + 1) * 8 + 2 * bnode + 1], yy, ay));
          }
          ox = fma(Ee, ax, ox);
          oy = fma(Ee, ay, oy);
        }
      const size_t i0 = (size_t)lx * ml + 2 * ly;
      B1[i0 * mb + j] = Dv[i0] > 0.0 ? ox : 0.0;
      B1[(i0 + 1) * mb + j] = Dv[i0 + 1] > 0.0 ? oy : 0.0;
    }
    cl_sync();
    // G = Y^T K Y, H = Y^T D Y (symmetric: upper triangles), one warp of the cluster per
    // entry, lanes over the DOFs (fixed order within the warp)
    {
      const int ntri = mb * (mb + 1) / 2;
      for (int t = gwarp; t < 2 * ntri; t += nwarps) {
        const int which = t / ntri;
        int tt = t - which * ntri, a2 = 0;
        while (tt >= mb - a2) {
          tt -= mb - a2;
          ++a2;
        }
        const int b2 = a2 + tt;
        double s = 0.0;
        if (which == 0)
          for (int i = lane; i < n; i += 32) s = fma(B2[(size_t)i * mb + a2], B1[(size_t)i * mb + b2], s);
        else
          for (int i = lane; i < n; i += 32) s = fma(B2[(size_t)i * mb + a2] * Dv[i], B2[(size_t)i * mb + b2], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          double* Mt = which == 0 ? gG : gH;
          Mt[a2 * mb + b2] = s;
          Mt[b2 * mb + a2] = s;
        }
      }
    }
    cl_sync();
    if (rank == 0) {
      for (int e = threadIdx.x; e < mb * mb; e += NT) {
        G[e] = __ldcg(gG + e);
        H[e] = __ldcg(gH + e);
      }
      __syncthreads();
      if (threadIdx.x < 32) small_gen_eig(G, H, mb, theta, Cm, Lw, Mw, Vw, status);
      __syncthreads();
      for (int e = threadIdx.x; e < mb * mb; e += NT) gC[e] = Cm[e];
      for (int e = threadIdx.x; e < mb; e += NT) gT[e] = theta[e];
    }
    cl_sync();
    // X = Y Cm ; then K X = (K Y) Cm into B2
    for (int e = t0; e < n * mb; e += tstride) {
      const int i = e / mb, j = e - (e / mb) * mb;
      B0[e] = dot4(B2 + (size_t)i * mb, 1, gC + j, mb, mb);
    }
    cl_sync();
    for (int e = t0; e < n * mb; e += tstride) {
      const int i = e / mb, j = e - (e / mb) * mb;
      B2[e] = dot4(B1 + (size_t)i * mb, 1, gC + j, mb, mb);
    }
    cl_sync();
    // residuals of the kept pairs: one warp of the cluster per pair, lanes over the DOFs
    const int kk = min(d.kmax, mb);
    for (int j = gwarp; j < kk; j += nwarps) {
      const double th = __ldcg(gT + j);
      double s = 0.0;
      for (int i = lane; i < n; i += 32) {
        if (Dv[i] > 0.0) {
          const double rv = B2[(size_t)i * mb + j] - th * Dv[i] * B0[(size_t)i * mb + j];
          s += rv * rv / Dv[i];
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) gR[j] = s;
    }
    cl_sync();
    double mx = 0.0;
    for (int j = 0; j < kk; ++j) mx = fmax(mx, __ldcg(gR + j));
    const bool stop = sqrt(mx) <= ea.tol;   // identical in every CTA of the cluster
    cl_sync();                               // gR / gC / gT are rewritten next iteration
    if (stop) {
      ++it;
      break;
    }
  }
  for (int e = threadIdx.x; e < mb; e += NT) theta[e] = __ldcg(gT + e);
  __syncthreads();
  // ---------------- write phi = chi psi on the padded box, eigenvalues, kept count
  int nk = min(d.kmax, mb);
  if (ea.lam_thr > 0.0 && ea.lam_thr < 1e300) {
    int cnt = 0;
    while (cnt < nk && theta[cnt] < ea.lam_thr) ++cnt;
    nk = cnt;
  }
  const int I = C.rep_agg / (d.ncy + 1), J = C.rep_agg - (C.rep_agg / (d.ncy + 1)) * (d.ncy + 1);
  const int gx0 = I * d.cx - d.cx, gy0 = J * d.cy - d.cy;
  double* ph = phi + (size_t)cls * d.kmax * d.box_nodes * 2;
  for (int e = t0; e < d.kmax * d.box_nodes * 2; e += tstride) {
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
  if (rank == 0) {
    for (int a = threadIdx.x; a < d.kmax; a += NT)
      lam[(size_t)cls * d.kmax + a] = (a < mb) ? theta[a] : 0.0;
    if (threadIdx.x == 0) {
      classes[cls].iters = it;
      classes[cls].nkept = nk;
    }
  }
}

}  // namespace

size_t eig_smem_bytes(int mlmax, int mb) {   // factorisation kernel
  const int sz = mlmax * (mlmax > mb ? mlmax : mb);
  return (size_t)(4 * sz + 2 * mlmax) * sizeof(double);
}
static size_t eig_iter_smem_bytes(int mb) { return (size_t)(6 * mb * mb + 32) * sizeof(double); }

void launch_build_basis(msf_ctx* c) {
  const Dims& d = c->d;
  EigArgs ea;
  ea.sigma = -1e-3;
  ea.tol = c->p.eig_tol > 0.0 ? c->p.eig_tol : 1e-9;
  ea.lam_thr = c->p.lam_threshold;
  ea.maxit = c->p.eig_max_iter > 0 ? c->p.eig_max_iter : 60;
  ea.mb = c->mb;
  ea.mlmax = 2 * d.by;
  int nbl_max = 1;
  for (const EigClass& C : c->classes) nbl_max = std::max(nbl_max, C.nbx);
  k_eigen_blocks<<<c->n_cls * 2 * nbl_max, NT, 0, c->stream>>>(
      d, c->K0, c->E + (size_t)c->p.dilated * d.ne, c->fixg, c->classes_d, c->eig_work, ea, nbl_max);
  MSF_LAUNCHED(c);
  const size_t smem_f = eig_smem_bytes(ea.mlmax, ea.mb);
  cudaFuncSetAttribute(k_eigen_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f);
  k_eigen_factor<<<c->n_cls, NT, smem_f, c->stream>>>(d, c->K0,
                                                     c->E + (size_t)c->p.dilated * d.ne, c->fixg,
                                                     c->classes_d, c->eig_work, c->phi, c->lam, ea,
                                                     c->factor_status + MSF_MAX_RHS);
  MSF_LAUNCHED(c);
  const size_t smem = eig_iter_smem_bytes(ea.mb);
  // one thread-block cluster of EIG_CL CTAs per class
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c->n_cls * EIG_CL);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = EIG_CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_eigen, d, c->K0, (const double*)(c->E + (size_t)c->p.dilated * d.ne),
                     (const uint8_t*)c->fixg, c->classes_d, c->eig_work, c->phi, c->lam, ea,
                     c->factor_status + MSF_MAX_RHS);
  MSF_LAUNCHED(c);
}
