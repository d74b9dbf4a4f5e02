// Host<->device bandwidth of SM-driven copies through mapped pinned memory
// (zero-copy loads / stores over PCIe) versus the copy engines
// (cudaMemcpyAsync), for one 1080p fp32 frame.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zerocopy zerocopy.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_copy(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t bytes = 8294400, n = bytes / 16;
  float *h_in, *h_out, *d_a, *d_b;
  cudaHostAlloc(&h_in, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&h_out, bytes, cudaHostAllocDefault);
  cudaMalloc(&d_a, bytes);
  cudaMalloc(&d_b, bytes);
  for (size_t i = 0; i < bytes / 4; ++i) h_in[i] = (float)i;
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 20;
  auto bw = [&](const char* name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a, s1);
    cudaStreamWaitEvent(s2, a, 0);
    for (int r = 0; r < reps; ++r) fn();
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s2);
    cudaStreamWaitEvent(s1, e, 0);
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-34s %7.1f us per frame  %6.1f GB/s\n", name, ms * 1e3f / reps, bytes / (ms * 1e-3 / reps) / 1e9);
  };
  for (int grid : {148, 296, 592, 1184}) {
    char nm[64];
    snprintf(nm, sizeof nm, "kernel H2D (grid %d x 256)", grid);
    bw(nm, [&] { k_copy<<<grid, 256, 0, s1>>>((const float4*)h_in, (float4*)d_a, n); });
  }
  for (int grid : {148, 592}) {
    char nm[64];
    snprintf(nm, sizeof nm, "kernel D2H (grid %d x 256)", grid);
    bw(nm, [&] { k_copy<<<grid, 256, 0, s1>>>((const float4*)d_b, (float4*)h_out, n); });
  }
  bw("memcpy H2D", [&] { cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1); });
  bw("memcpy D2H", [&] { cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s1); });
  bw("kernel H2D + memcpy D2H (2 streams)", [&] {
    k_copy<<<592, 256, 0, s1>>>((const float4*)h_in, (float4*)d_a, n);
    cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
  });
  bw("memcpy H2D + memcpy D2H (2 streams)", [&] {
    cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
  });
  bw("kernel H2D + kernel D2H (2 streams)", [&] {
    k_copy<<<592, 256, 0, s1>>>((const float4*)h_in, (float4*)d_a, n);
    k_copy<<<148, 256, 0, s2>>>((const float4*)d_b, (float4*)h_out, n);
  });
  // correctness of the zero-copy path
  k_copy<<<592, 256, 0, s1>>>((const float4*)h_in, (float4*)d_a, n);
  cudaMemcpy(h_out, d_a, bytes, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < bytes / 4; ++i) bad += h_out[i] != (float)i;
  printf("zero-copy H2D mismatches: %zu, last error: %s\n", bad, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
