// FP64 + integer mix probe (B200): DFMA (uniform multiplier) interleaved 1:1 with IMAD / MOV-like work.
#include <cstdio>
#include <cuda_runtime.h>
struct P { double v[8]; };
template <int MODE>
__global__ void k(double* out, const double* in, int iters, long long* cyc, P kp, int m) {
  double a[8], x[8];
  int n[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; x[i] = in[threadIdx.x + i]; n[i] = threadIdx.x * i + m; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a[i] = fma(x[(i + u) & 7], kp.v[u], a[i]);
        if (MODE == 1) n[i] = n[i] * m + u;                       // IMAD
        if (MODE == 2) n[i] = __shfl_up_sync(0xffffffffu, n[i], 1);   // SHFL
        if (MODE == 3) { n[i] = n[i] * m + u; n[(i + 1) & 7] ^= n[i]; }   // IMAD + LOP3
      }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + n[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int MODE>
void run(int warps, double* out, double* in, long long* cyc) {
  const int iters = 2000;
  P kp; for (int i = 0; i < 8; ++i) kp.v[i] = 1.0 + 1e-9 * i;
  k<MODE><<<148, warps * 32>>>(out, in, iters, cyc, kp, 3);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("mode %d warps/SM %2d: %.1f DFMA/clk/SM\n", MODE, warps, (double)iters * 64 * warps * 32 / (double)h);
}
int main() {
  double *out, *in; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&in, 4096 * 8); cudaMemset(in, 0, 4096 * 8); cudaMalloc(&cyc, 8);
  for (int w : {4, 8, 16}) { run<0>(w, out, in, cyc); run<1>(w, out, in, cyc); run<2>(w, out, in, cyc); run<3>(w, out, in, cyc); }
  return 0;
}
