// FP64 pipe probe (B200): dependent-DFMA latency, and DFMA throughput per SM as a function of
// independent chains per thread (ILP) and warps per SM.  nvcc -arch=sm_100a -O3 dfma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double* out, int iters, long long* cyc) {
  double a[ILP];
  const double b = 1.0000001, c = 1e-9;
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, c);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int ILP>
void run(int warps, double* out, long long* cyc) {
  const int iters = 2000;
  k<ILP><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<ILP><<<148, warps * 32>>>(out, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double n = (double)iters * 8 * ILP;   // DFMA per thread
  printf("ILP %2d warps/SM %2d: %.2f cyc per dependent step, %.1f DFMA/clk/SM, %.2f TFLOP/s\n", ILP, warps,
         (double)h / (iters * 8), n * warps * 32 / (double)h, 2 * n * warps * 32 * 148 / (ms * 1e-3) * 1e-12);
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 16, 32}) {
    run<1>(w, out, cyc); run<2>(w, out, cyc); run<4>(w, out, cyc); run<8>(w, out, cyc); run<16>(w, out, cyc);
  }
  return 0;
}
