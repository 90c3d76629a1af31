// Blocked SPD inverse in shared memory by the block sweep operator (msf_basis.cu local
// eigenproblem factorisation, msf_coarse.cu cyclic-reduction pivots).
#pragma once

namespace msfinv {

// In-place inverse of the SPD m x m matrix S (shared memory) by the BLOCK sweep operator, pivot
// blocks K of IB = 8: with P = A_KK^-1,
//   A_ij -= A_iK P A_Kj,  A_iK <- A_iK P,  A_Kj <- P A_Kj,  A_KK <- -P   (i, j outside K),
// which equals sweeping the pivots of K one by one; after all blocks the matrix holds -A^-1,
// negated at the end, so S = A^-1 on return.  A non-positive pivot sets *status = code.  3 block barriers per 8 pivots instead of 2 per pivot (the per-pivot sweep was 75% of
// k_eigen_factor in ncu, configs[1]).  Scratch: scr >= 3 m IB + IB IB doubles.
constexpr int IB = 8;
template <int NTH, int NU>   // NTH threads (32-lane row groups); columns m <= 32 NU
__device__ void inverse_blocked(double* S, int m, double* scr, int* status, int code = 2) {
  const int tid = threadIdx.x, jl = tid & 31, ig = tid >> 5;
  constexpr int RG = NTH / 32;
  constexpr int NT = NTH;
  double* rowK = scr;              // [IB][m]  A_Kj (original)
  double* Y = rowK + IB * m;       // [m][IB]  A_iK P
  double* Z = Y + IB * m;          // [IB][m]  P A_Kj
  double* Pb = Z + IB * m;         // [IB][IB] -P after the warp sweep
  for (int k0 = 0; k0 < m; k0 += IB) {
    const int bk = min(IB, m - k0);
    for (int e = tid; e < bk * m; e += NT) {
      const int b = e / m, j = e - b * m;
      rowK[b * m + j] = S[(k0 + b) * m + j];
    }
    __syncthreads();
    if (ig == 0) {
      // warp 0: sweep of the bk x bk pivot block -> Pb = -A_KK^-1
      for (int e = jl; e < bk * bk; e += 32) Pb[e] = rowK[(e / bk) * m + k0 + e % bk];
      __syncwarp();
      for (int k = 0; k < bk; ++k) {
        const double piv = Pb[k * bk + k];
        if (!(piv > 0.0) && jl == 0) atomicExch(status, code);
        const double ip = 1.0 / piv;
        double nv[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int e = jl + 32 * q;
          if (e < bk * bk) {
            const int i = e / bk, j = e - (e / bk) * bk;
            const double aij = Pb[e], aik = Pb[i * bk + k], akj = Pb[k * bk + j];
            nv[q] = (i == k) ? ((j == k) ? -ip : akj * ip) : ((j == k) ? aik * ip : fma(-aik * ip, akj, aij));
          }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (jl + 32 * q < bk * bk) Pb[jl + 32 * q] = nv[q];
        __syncwarp();
      }
    }
    __syncthreads();
    // Y = A_iK P, Z = P A_Kj  (P = -Pb)
    for (int e = tid; e < m * bk; e += NT) {
      const int i = e / bk, b = e - (e / bk) * bk;
      double y = 0.0;
      for (int c = 0; c < bk; ++c) y = fma(S[i * m + k0 + c], -Pb[c * bk + b], y);
      Y[i * IB + b] = y;
    }
    for (int e = tid; e < bk * m; e += NT) {
      const int b = e / m, j = e - b * m;
      double z = 0.0;
      for (int c = 0; c < bk; ++c) z = fma(-Pb[b * bk + c], rowK[c * m + j], z);
      Z[b * m + j] = z;
    }
    __syncthreads();
    // S update; the thread's columns j = jl + 32 u keep their A_Kj in registers
    double rk[NU][IB];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int j = jl + 32 * u;
#pragma unroll
      for (int b = 0; b < IB; ++b) rk[u][b] = (j < m && b < bk) ? rowK[b * m + j] : 0.0;
    }
    for (int i = ig; i < m; i += RG) {
      const bool iK = i >= k0 && i < k0 + bk;
      double yi[IB];
#pragma unroll
      for (int b = 0; b < IB; ++b) yi[b] = b < bk ? Y[i * IB + b] : 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const int j = jl + 32 * u;
        if (j >= m) continue;
        const bool jK = j >= k0 && j < k0 + bk;
        double v;
        if (iK && jK) v = Pb[(i - k0) * bk + (j - k0)];
        else if (iK) v = Z[(i - k0) * m + j];
        else if (jK) v = Y[i * IB + (j - k0)];
        else {
          v = S[i * m + j];
#pragma unroll
          for (int b = 0; b < IB; ++b) v = fma(-yi[b], rk[u][b], v);
        }
        S[i * m + j] = v;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < m * m; e += NT) S[e] = -S[e];
  __syncthreads();
}

}  // namespace msfinv
