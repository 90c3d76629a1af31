// Microbenchmark: cost of cooperative_groups grid.sync() on the B200 for the persistent
// PCG design.  Prints us per sync for several CTA counts.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int n, double* out) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < n; ++i) { acc += threadIdx.x * 1e-9; g.sync(); }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}
int main() {
  int dev = 0, sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out; cudaMalloc(&out, 8);
  for (int threads : {256, 512}) for (int per : {1, 2, 4}) {
    int maxb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k, threads, 0);
    if (per > maxb) continue;
    int blocks = sms * per, n = 2000;
    void* args[] = {&n, &out};
    cudaLaunchCooperativeKernel((void*)k, blocks, threads, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k, blocks, threads, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("threads %d blocks %d: %.3f us per grid.sync (err %s)\n", threads, blocks, ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
  }
  // plain dependent launches for comparison
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int one = 1; 
  cudaEventRecord(a);
  for (int i = 0; i < 2000; ++i) { void* args[] = {&one, &out}; cudaLaunchCooperativeKernel((void*)k, sms, 256, args, 0, 0); }
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("back-to-back cooperative launches: %.3f us each\n", ms * 1e3 / 2000);
  return 0;
}
