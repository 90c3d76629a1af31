// Coarse space of the two-level preconditioner (§2.4, Eq. 10, §2.4.2
// line 146):
//   * phi_{i,a} = chi_i psi_a^{omega_i} is stored per agglomerate class on a padded
//     (2cx+1)x(2cy+1)-node box (periodic classes share storage, §2.4.1);
//     restriction / prolongation: msf_xfer.cu;
//   * Galerkin K_c = R_c K R_c^T per realisation, assembled from per-coarse-cell dense
//     (4k x 4k) products Phi_C^T K_C Phi_C (the dense contraction of the path);
//   * the exact coarse solve factors K_c over a nested dissection of the coarse node grid
//     (msf_nd.cu); k_coarse_gather reads out its block-tridiagonal form (diagnostics).
#include <array>
#include <map>

#include "msf_kern.cuh"

#include <algorithm>
#include <cmath>

using namespace msfk;

namespace {

constexpr int NT = 256;

// ------------------------------------------------------------------ Galerkin cell products
// Kcell[rhs][cell][p][q] = sum_{e in cell} E_e Phi_e[:,p]^T K0 Phi_e[:,q],  p,q in 0..4k-1,
// p = corner*k + a, corner = ci*2 + cj for coarse node (CI+ci, CJ+cj).  The (4k)x(4k) output
// is computed in CH x CH chunks (blockIdx.z = chunk pair) so the staged cell bases fit in
// shared memory for any mode count; with a single chunk Phi_p and Phi_q coincide.
__device__ __forceinline__ void stage_cell_cols(const Dims& d, const double* __restrict__ phi,
                                                const int* __restrict__ cls_of_agg, int CI, int CJ,
                                                int c0, int cw, int CH, double* S) {
  const int km = d.kmax, ncn_y = d.cy + 1, ncn = (d.cx + 1) * (d.cy + 1);
  for (int k = threadIdx.x; k < ncn * 2 * CH; k += NT) {
    const int j = k % CH, nc = k / CH;          // column j, node*2 + comp
    if (j >= cw) continue;
    const int comp = nc & 1, node = nc >> 1;
    const int lx = node / ncn_y, ly = node - (node / ncn_y) * ncn_y;
    const int p = c0 + j;
    const int corner = p / km, a = p - (p / km) * km;
    const int I = CI + (corner >> 1), J = CJ + (corner & 1);
    const int px = CI * d.cx + lx - (I * d.cx - d.cx), py = CJ * d.cy + ly - (J * d.cy - d.cy);
    const int agg = I * (d.ncy + 1) + J;
    S[k] = phi[(((size_t)cls_of_agg[agg] * d.kmax + a) * d.box_nodes + px * d.by + py) * 2 + comp];
  }
}

__global__ void __launch_bounds__(NT) k_cell_galerkin(Dims d, K0Mat K, const double* __restrict__ Eall,
                                                      const double* __restrict__ phi,
                                                      const int* __restrict__ cls_of_agg,
                                                      double* Kcell, int CH, int cell0) {
  extern __shared__ double sm[];
  // all realisations in one CTA: V_e = K0 Phi_e and Phi_e^T V_e do not depend on the
  // realisation, only the scalar modulus E_e does (R accumulators per output entry)
  const int cell = cell0 + blockIdx.x;
  const int CI = cell / d.ncy, CJ = cell - (cell / d.ncy) * d.ncy;
  const int P = 4 * d.kmax;
  const int nch = (P + CH - 1) / CH;
  const int pc = blockIdx.z / nch, qc = blockIdx.z - pc * nch;
  const int p0 = pc * CH, q0 = qc * CH, pw = min(CH, P - p0), qw = min(CH, P - q0);
  const int ncn_y = d.cy + 1, ncn = (d.cx + 1) * (d.cy + 1);
  const bool single = nch == 1;
  double* PhiP = sm;                                       // [ncn][2][CH]
  double* PhiQ = single ? PhiP : PhiP + (size_t)ncn * 2 * CH;
  double* V = PhiQ + (size_t)ncn * 2 * CH;                 // [16][8][CH]
  double* Ech = V + 16 * 8 * CH;                           // [MSF_MAX_RHS][16]
  stage_cell_cols(d, phi, cls_of_agg, CI, CJ, p0, pw, CH, PhiP);
  if (!single) stage_cell_cols(d, phi, cls_of_agg, CI, CJ, q0, qw, CH, PhiQ);
  const int R = d.R;
  const int nel = d.cx * d.cy;
  const int nent = CH * CH;   // <= NT
  double acc[MSF_MAX_RHS] = {0.0, 0.0, 0.0, 0.0};
  __syncthreads();
  for (int e0 = 0; e0 < nel; e0 += 16) {
    const int ne = min(16, nel - e0);
    // V_e = K0 Phi_e[:, q-chunk] for the element chunk
    for (int k = threadIdx.x; k < ne * 8 * CH; k += NT) {
      const int q = k % CH, rest = k / CH;
      const int i = rest & 7, el = rest >> 3;
      if (q >= qw) continue;
      const int le = e0 + el;
      const int lex = le / d.cy, ley = le - (le / d.cy) * d.cy;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int b = j >> 1, comp = j & 1;
        const int nx = lex + ((b == 1 || b == 2) ? 1 : 0), ny = ley + ((b >= 2) ? 1 : 0);
        s = fma(K.v[i * 8 + j], PhiQ[((nx * ncn_y + ny) * 2 + comp) * CH + q], s);
      }
      V[(el * 8 + i) * CH + q] = s;
    }
    for (int k = threadIdx.x; k < ne * R; k += NT) {
      const int r = k / ne, el = k - r * ne;
      const int le = e0 + el;
      const int lex = le / d.cy, ley = le - (le / d.cy) * d.cy;
      Ech[r * 16 + el] = Eall[(size_t)r * d.ne + (size_t)(CI * d.cx + lex) * d.nely + CJ * d.cy + ley];
    }
    __syncthreads();
    const int ent = threadIdx.x;
    if (ent < nent) {
      const int p = ent / CH, q = ent - (ent / CH) * CH;
      if (p < pw && q < qw) {
        for (int el = 0; el < ne; ++el) {
          const int le = e0 + el;
          const int lex = le / d.cy, ley = le - (le / d.cy) * d.cy;
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int b = i >> 1, comp = i & 1;
            const int nx = lex + ((b == 1 || b == 2) ? 1 : 0), ny = ley + ((b >= 2) ? 1 : 0);
            t = fma(PhiP[((nx * ncn_y + ny) * 2 + comp) * CH + p], V[(el * 8 + i) * CH + q], t);
          }
#pragma unroll
          for (int r = 0; r < MSF_MAX_RHS; ++r)
            if (r < R) acc[r] = fma(Ech[r * 16 + el], t, acc[r]);
        }
      }
    }
    __syncthreads();
  }
  const int ent = threadIdx.x;
  if (ent < nent) {
    const int p = ent / CH, q = ent - (ent / CH) * CH;
    if (p < pw && q < qw)
#pragma unroll
      for (int r = 0; r < MSF_MAX_RHS; ++r)
        if (r < R) Kcell[((size_t)r * d.ncx * d.ncy + cell) * P * P + (size_t)(p0 + p) * P + (q0 + q)] = acc[r];
  }
}

// Gather the cell products into the block-tridiagonal K_c (D_I, U_I = K_c[I, I+1]) for
// the blocks D_I, I in [dlo, dlo + nD), and U_I, I in [ulo, ulo + nU), from the coarse cell
// columns [ulo, ulo + nU) (a strip: its own cells, so its chain's end blocks get partial
// sums); unused eigen-slots (a >= nkept) carry identity rows in D_I for I in [idlo, idhi]
// (each block's identity added by one rank).
__global__ void k_coarse_gather(Dims d, const double* __restrict__ Kcell,
                                const int* __restrict__ cls_of_agg,
                                const EigClass* __restrict__ cls, double* Dall, double* Uall,
                                int dlo, int nD, int ulo, int nU, int idlo, int idhi, int slot0,
                                int nslot) {
  const int km = d.kmax, P = 4 * km, m = d.mc;
  const size_t per = (size_t)m * m;
  const size_t total = (size_t)(nD + nU) * per;
  const int rhs = blockIdx.y;
  const double* Kc = Kcell + (size_t)rhs * d.ncx * d.ncy * P * P;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int isU = idx >= (size_t)nD * per;
    const size_t li = isU ? idx - (size_t)nD * per : idx;
    const int I = (int)(li / per) + (isU ? ulo : dlo);
    const int e = (int)(li - (size_t)(I - (isU ? ulo : dlo)) * per);
    const int row = e / m, col = e - (e / m) * m;
    const int J = row / km, a = row - (row / km) * km;
    const int Jp = col / km, b = col - (col / km) * km;
    double v = 0.0;
    const int Ir = I, Ic = isU ? I + 1 : I;
    const int nka = cls[cls_of_agg[Ir * (d.ncy + 1) + J]].nkept;
    const int nkb = cls[cls_of_agg[Ic * (d.ncy + 1) + Jp]].nkept;
    if (a >= nka || b >= nkb) {
      v = (!isU && row == col && I >= idlo && I <= idhi) ? 1.0 : 0.0;
    } else if (abs(J - Jp) <= 1) {
      const int CIlo = isU ? I : max(I - 1, ulo), CIhi = isU ? I : min(I, ulo + nU - 1);
      const int CJlo = max(max(J, Jp) - 1, 0), CJhi = min(min(J, Jp), d.ncy - 1);
      for (int CI = CIlo; CI <= CIhi; ++CI)
        for (int CJ = CJlo; CJ <= CJhi; ++CJ) {
          const int pr = ((Ir - CI) * 2 + (J - CJ)) * km + a;
          const int pc = ((Ic - CI) * 2 + (Jp - CJ)) * km + b;
          v += Kc[((size_t)CI * d.ncy + CJ) * P * P + (size_t)pr * P + pc];
        }
    }
    double* dst = (isU ? Uall : Dall) + ((size_t)rhs * nslot + (I - slot0)) * per;   // chain slots
    dst[e] = v;
  }
}

}  // namespace

// Galerkin cell products Kcell = Phi_C^T (E K0) Phi_C of this rank's coarse cells (Eq. 10)
void launch_galerkin_cells(msf_ctx* c) {
  const Dims& d = c->d;
  const int P = 4 * d.kmax;
  const size_t ncn2 = (size_t)(d.cx + 1) * (d.cy + 1) * 2;
  // largest column chunk whose staged bases fit in shared memory (<= 16 so CH^2 <= NT)
  int CH = std::min(P, 16);
  auto smem_for = [&](int ch) {
    const bool single = ch >= P;
    return ((single ? 1 : 2) * ncn2 * ch + 16 * 8 * (size_t)ch + 16 * MSF_MAX_RHS) * sizeof(double);
  };
  while (CH > 2 && smem_for(CH) > 220 * 1024) CH /= 2;
  const size_t smem = smem_for(CH);
  const int nch = (P + CH - 1) / CH;
  cudaFuncSetAttribute(k_cell_galerkin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // this rank's coarse cell columns (all of them on one GPU)
  k_cell_galerkin<<<dim3((c->cell_hi - c->cell_lo) * d.ncy, 1, nch * nch), NT, smem, c->stream>>>(
      d, c->K0, c->E, c->phi, c->cls_of_agg_d, c->Kcell, CH, c->cell_lo * d.ncy);
  MSF_LAUNCHED(c);
}

// Block-tridiagonal copies D_I, U_I of K_c (this rank's chain) gathered from the cell products
void launch_coarse_gather(msf_ctx* c, double* D, double* U, int nslot) {
  const Dims& d = c->d;
  const int nD = c->cr_hi - c->cr_lo + 1, nU = c->cell_hi - c->cell_lo;
  const size_t total = (size_t)(nD + nU) * d.mc * d.mc;
  int blocks = (int)std::min<size_t>((total + 255) / 256, 65535);
  k_coarse_gather<<<dim3(blocks, d.R), 256, 0, c->stream>>>(d, c->Kcell, c->cls_of_agg_d, c->classes_d, D, U,
                                                            c->cr_lo, nD, c->cell_lo, nU, 0, d.ncx,
                                                            c->cr_lo, nslot);
  MSF_LAUNCHED(c);
}

// K_c assembly (Eq. 10) and its nested-dissection factorisation (msf_nd.cu), one GPU
void launch_assemble_coarse(msf_ctx* c) {
  launch_galerkin_cells(c);
  launch_nd_factor(c);
}
