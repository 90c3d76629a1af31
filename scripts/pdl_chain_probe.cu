// Latency floor of a PCG iteration's launch chain: a CUDA graph of N (default 34) dependent
// kernels launched with programmatic dependent launch (griddepcontrol.launch_dependents /
// wait), each a grid of `blocks` CTAs doing no work, replayed many times.  Prints us per
// graph and per kernel, with and without the PDL attribute.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/pdl_chain_probe scripts/pdl_chain_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__global__ void k_empty(int* sink) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0 && sink[0] == 12345) sink[1] = 1;
}

static float run(int nk, int blocks, bool pdl, int reps) {
  int* sink;
  cudaMalloc(&sink, 8);
  cudaMemset(sink, 0, 8);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < nk; ++i) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_empty, sink);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphExec_t ge;
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / reps;
}

int main(int argc, char** argv) {
  const int nk = argc > 1 ? atoi(argv[1]) : 34;
  for (int blocks : {148, 592, 2048}) {
    const float a = run(nk, blocks, true, 500), b = run(nk, blocks, false, 500);
    printf("%d kernels x %d CTAs: PDL %.1f us/graph (%.2f us/kernel), plain %.1f us/graph (%.2f us/kernel)\n",
           nk, blocks, a, a / nk, b, b / nk);
  }
  return 0;
}
