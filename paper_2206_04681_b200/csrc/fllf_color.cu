// Colour handling and the variance-driven gain map of the pixel-by-pixel
// enhancement (Sec. IV: "The degree of
// enhancement is determined according to the variance of the pixels in a
// local window; the low variance is a small enhancement" and "LLF is applied
// to the Y channel of the YUV color space, and the other components are
// kept").  Readings R13-R16: BT.601 full-range YCbCr, population
// variance over a (2r+1)^2 reflect-101 window, m_p = m_lo + (m_hi - m_lo)
// min(1, v_p / v_ref), uniform sigma_r.
//
// All three kernels are HBM-bound elementwise / small-stencil passes:
//  k_rgb_to_yuv / k_yuv_to_rgb -- one pixel per thread, coalesced rows.
//  k_gain_map -- 32x64 output tile per CTA; the (32+2r) x (64+2r) input
//                window is staged in shared memory, horizontal window sums of
//                y and y^2 are formed once per staged row, then vertical sums;
//                sums in fp64 (E[y^2] - E[y]^2 cancels; B200 has full-rate
//                fp64 at half the fp32 rate, and this pass is memory-bound).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fllf_internal.h"

namespace fllf {
namespace {

// R13: BT.601 luma weights, chroma zero-centred (JFIF scaling)
constexpr float KR = 0.299f, KG = 0.587f, KB = 0.114f;
constexpr float CB_SCALE = 1.772f, CR_SCALE = 1.402f;

__global__ void k_rgb_to_yuv(ColorParams P) {
  const long long n = (long long)P.H * P.W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / P.W), x = (int)(i - (long long)y * P.W);
    const long long o = (long long)y * P.pitch + x;
    const float r = P.src[0][o], g = P.src[1][o], b = P.src[2][o];
    const float Y = fmaf(KR, r, fmaf(KG, g, KB * b));
    P.dst[0][o] = Y;
    P.dst[1][o] = (b - Y) * (1.f / CB_SCALE);
    P.dst[2][o] = (r - Y) * (1.f / CR_SCALE);
  }
}

__global__ void k_yuv_to_rgb(ColorParams P) {
  const long long n = (long long)P.H * P.W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / P.W), x = (int)(i - (long long)y * P.W);
    const long long o = (long long)y * P.pitch + x;
    const float Y = P.src[0][o], cb = P.src[1][o], cr = P.src[2][o];
    const float r = fmaf(CR_SCALE, cr, Y);
    const float b = fmaf(CB_SCALE, cb, Y);
    // G from Y = KR r + KG g + KB b
    const float g = (Y - KR * r - KB * b) * (1.f / KG);
    P.dst[0][o] = r;
    P.dst[1][o] = g;
    P.dst[2][o] = b;
  }
}

// reflect-101 folded with period 2(n-1): any index, any number of bounces
__device__ __forceinline__ int refl_fold(int i, int n) {
  if (n == 1) return 0;
  const int p = 2 * (n - 1);
  int r = i % p;
  if (r < 0) r += p;
  return r < n ? r : p - r;
}

constexpr int GT_H = 32, GT_W = 64;

__global__ void __launch_bounds__(256) k_gain_map(GainParams P) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int r = P.radius;
  const int SW = GT_W + 2 * r, SH = GT_H + 2 * r;
  float* tile = reinterpret_cast<float*>(sm);                      // SH x SW, y - shift
  double* h1 = reinterpret_cast<double*>(sm + ((SH * SW * 4 + 15) & ~15));  // SH x GT_W
  double* h2 = h1 + SH * GT_W;
  const int y0 = blockIdx.y * GT_H, x0 = blockIdx.x * GT_W;
  // shift by one sample of the tile: variance is shift-invariant, the sums stay small
  const float shift = __ldg(P.y + (long long)min(y0, P.H - 1) * P.y_pitch + min(x0, P.W - 1));
  for (int t = threadIdx.x; t < SH * SW; t += blockDim.x) {
    const int ty = t / SW, tx = t - ty * SW;
    const int gy = refl_fold(y0 - r + ty, P.H), gx = refl_fold(x0 - r + tx, P.W);
    tile[t] = __ldg(P.y + (long long)gy * P.y_pitch + gx) - shift;
  }
  __syncthreads();
  // horizontal window sums for every staged row, the GT_W output columns
  for (int t = threadIdx.x; t < SH * GT_W; t += blockDim.x) {
    const int ty = t / GT_W, tx = t - ty * GT_W;
    const float* row = tile + ty * SW + tx;
    double s1 = 0.0, s2 = 0.0;
    for (int d = 0; d <= 2 * r; ++d) {
      const double v = row[d];
      s1 += v;
      s2 = fma(v, v, s2);
    }
    h1[t] = s1;
    h2[t] = s2;
  }
  __syncthreads();
  const double inv_n = 1.0 / ((2.0 * r + 1.0) * (2.0 * r + 1.0));
  for (int t = threadIdx.x; t < GT_H * GT_W; t += blockDim.x) {
    const int ty = t / GT_W, tx = t - ty * GT_W;
    const int gy = y0 + ty, gx = x0 + tx;
    if (gy >= P.H || gx >= P.W) continue;
    double s1 = 0.0, s2 = 0.0;
    for (int d = 0; d <= 2 * r; ++d) {
      s1 += h1[(ty + d) * GT_W + tx];
      s2 += h2[(ty + d) * GT_W + tx];
    }
    const double mean = s1 * inv_n;
    const double var = fmax(s2 * inv_n - mean * mean, 0.0);
    const double g = P.m_lo + (P.m_hi - P.m_lo) * fmin(1.0, var * P.inv_vref);
    P.m[(long long)gy * P.m_pitch + gx] = (float)g;
  }
}

__global__ void k_fill(float* p, long long pitch, int H, int W, float v) {
  const long long n = (long long)H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / W), x = (int)(i - (long long)y * W);
    p[(long long)y * pitch + x] = v;
  }
}

int grid_for(long long n) {
  long long g = (n + 255) / 256;
  return (int)(g < 148LL * 16 ? (g < 1 ? 1 : g) : 148LL * 16);
}

}  // namespace

cudaError_t launch_rgb_to_yuv(const ColorParams& p, cudaStream_t s) {
  k_rgb_to_yuv<<<grid_for((long long)p.H * p.W), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_yuv_to_rgb(const ColorParams& p, cudaStream_t s) {
  k_yuv_to_rgb<<<grid_for((long long)p.H * p.W), 256, 0, s>>>(p);
  return cudaGetLastError();
}

size_t gain_map_smem(int radius) {
  const int SW = GT_W + 2 * radius, SH = GT_H + 2 * radius;
  return (size_t)((SH * SW * 4 + 15) & ~15) + 2 * sizeof(double) * SH * GT_W;
}

cudaError_t launch_gain_map(const GainParams& p, cudaStream_t s) {
  const size_t smem = gain_map_smem(p.radius);
  cudaError_t e = cudaFuncSetAttribute(k_gain_map, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((p.W + GT_W - 1) / GT_W, (p.H + GT_H - 1) / GT_H);
  k_gain_map<<<grid, 256, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fill(float* ptr, long long pitch, int H, int W, float v, cudaStream_t s) {
  k_fill<<<grid_for((long long)H * W), 256, 0, s>>>(ptr, pitch, H, W, v);
  return cudaGetLastError();
}

}  // namespace fllf
