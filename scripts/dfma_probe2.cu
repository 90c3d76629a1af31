// FP64 operand-bandwidth probe (B200): DFMA throughput with 3 distinct register operands vs a
// uniform (kernel-parameter) multiplier.  8 warps/SM, 8 chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
struct P { double v[8]; };
template <int MODE>
__global__ void k(double* out, const double* in, int iters, long long* cyc, P kp) {
  double a[8], x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; x[i] = in[threadIdx.x + i]; y[i] = in[threadIdx.x + 8 + i]; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0) a[i] = fma(x[i], y[(i + u) & 7], a[i]);        // R, R, R (all distinct)
        if (MODE == 1) a[i] = fma(x[(i + u) & 7], kp.v[u], a[i]);     // R, UR/const, R
        if (MODE == 2) a[i] = fma(x[u], y[u], a[i]);                  // R, R (shared by the 8 chains: .reuse), R
      }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int MODE>
void run(int warps, double* out, double* in, long long* cyc) {
  const int iters = 2000;
  P kp; for (int i = 0; i < 8; ++i) kp.v[i] = 1.0 + 1e-9 * i;
  k<MODE><<<148, warps * 32>>>(out, in, iters, cyc, kp);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("mode %d warps/SM %2d: %.1f DFMA/clk/SM\n", MODE, warps, (double)iters * 64 * warps * 32 / (double)h);
}
int main() {
  double *out, *in; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&in, 4096 * 8); cudaMemset(in, 0, 4096 * 8); cudaMalloc(&cyc, 8);
  for (int w : {4, 8, 16}) { run<0>(w, out, in, cyc); run<1>(w, out, in, cyc); run<2>(w, out, in, cyc); }
  return 0;
}
