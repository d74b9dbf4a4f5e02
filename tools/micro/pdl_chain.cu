// Floor of a dependent launch chain on this GPU: N kernels captured in one
// CUDA graph, each waiting (griddepcontrol.wait) for its predecessor, with
// and without programmatic dependent launch; grids of 1 and 444 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_chain pdl_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(float* buf, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] += 1.f;
}

static float run(int nk, int grid, bool pdl, float* buf) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < nk; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_step, buf, grid * 128);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 20; ++w) cudaGraphLaunch(ge, s);
  const int reps = 200;
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, s);
    for (int w = 0; w < reps; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return best / reps * 1e3f;  // us per graph
}

int main() {
  float* buf;
  cudaMalloc(&buf, 444 * 128 * sizeof(float));
  for (int grid : {1, 444})
    for (int nk : {1, 2, 10})
      for (int pdl : {0, 1})
        printf("grid %3d  kernels %2d  pdl %d : %6.2f us per graph replay\n", grid, nk, pdl, run(nk, grid, pdl, buf));
  return 0;
}
