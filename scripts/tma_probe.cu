// Standalone check of the TMA tile-load mechanics used by k_apply_tma (msf_fem.cu): a 3D
// FP64 tensor map (dims 2*nny x nnx x R, box 256 x 10 x 1, negative start coordinates,
// zero fill), one cp.async.bulk.tensor into shared memory completed on an mbarrier, the
// tile compared with the host copy.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -o scripts/tma_probe scripts/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map0, const __grid_constant__ CUtensorMap map1, double* out,
                      int c0, int c1, int c2, int mode, int which, uint32_t bytes) {
  const CUtensorMap& map = which ? map1 : map0;
  extern __shared__ __align__(128) unsigned char raw[];
  double* tile = reinterpret_cast<double*>(raw + ((128u - (smem_u32(raw) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes)
                 : "memory");
    if (mode == 0)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              smem_u32(tile)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              smem_u32(tile)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar))
          : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(
          smem_u32(&bar)),
      "r"(0)
      : "memory");
  for (int i = threadIdx.x; i < 2560; i += blockDim.x) out[i] = tile[i];
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;   // 0: node-vector map, 1: moduli map
  const int nely = 130, nelx = 160, R = 3, nny = nely + 1, nnx = nelx + 1;
  const size_t nx = (size_t)2 * nny * nnx * R, ne = (size_t)nely * nelx * R;
  std::vector<double> hx(nx), he(ne);
  for (size_t i = 0; i < nx; ++i) hx[i] = (double)i;
  for (size_t i = 0; i < ne; ++i) he[i] = 0.5 + (double)i;
  double *dx, *de, *o;
  cudaMalloc(&dx, nx * 8);
  cudaMalloc(&de, ne * 8);
  cudaMalloc(&o, 2560 * 8);
  cudaMemcpy(dx, hx.data(), nx * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(de, he.data(), ne * 8, cudaMemcpyHostToDevice);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
  CUtensorMap mx, me;
  const cuuint32_t es[3] = {1, 1, 1};
  {
    const cuuint64_t dims[3] = {(cuuint64_t)2 * nny, (cuuint64_t)nnx, (cuuint64_t)R};
    const cuuint64_t strides[2] = {(cuuint64_t)2 * nny * 8, (cuuint64_t)2 * nny * nnx * 8};
    const cuuint32_t box[3] = {256, 10, 1};
    printf("encode x %d\n", (int)enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dx, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {
    const cuuint64_t dims[3] = {(cuuint64_t)nely, (cuuint64_t)nelx, (cuuint64_t)R};
    const cuuint64_t strides[2] = {(cuuint64_t)nely * 8, (cuuint64_t)nely * nelx * 8};
    const cuuint32_t box[3] = {128, 9, 1};
    printf("encode e %d\n", (int)enc(&me, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, de, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2560 * 8 + 128);
  const int c0 = which ? -1 : -2, c1 = 3, c2 = 1;
  const uint32_t bytes = which ? 128 * 9 * 8 : 256 * 10 * 8;
  for (int order = 0; order < 2; ++order) {
    // order 0: map under test as the first parameter; 1: as the second
    const CUtensorMap& test = which ? me : mx;
    if (order == 0) probe<<<1, 128, 2560 * 8 + 128>>>(test, test, o, c0, c1, c2, 0, 0, bytes);
    else probe<<<1, 128, 2560 * 8 + 128>>>(mx, test, o, c0, c1, c2, 0, 1, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    printf("which %d order %d kernel: %s\n", which, order, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
