// Coarse space of the two-level preconditioner (§2.4, Eq. 10, §2.4.2
// line 146):
//   * phi_{i,a} = chi_i psi_a^{omega_i} is stored per agglomerate class on a padded
//     (2cx+1)x(2cy+1)-node box (periodic classes share storage, §2.4.1);
//     restriction / prolongation: msf_xfer.cu;
//   * Galerkin K_c = R_c K R_c^T per realisation, from per-coarse-cell dense (4k x 4k)
//     products Phi_C^T K_C Phi_C: one DMMA GEMM per coarse-cell class (msf_xfer.cu);
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
