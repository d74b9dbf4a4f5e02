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
//                window is staged in shared memory; vertical window sums of y
//                and y^2 as sliding runs per staged column, then horizontal
//                sliding runs per output row; sums in fp64 (E[y^2] - E[y]^2
//                cancels).
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
constexpr int GRUN = 8;  // outputs per sliding-window run

// smem row stride (in doubles) of the vertical-sum planes: odd, so that the
// 32 lanes of a warp reading one column of 32 different rows hit 32 banks
__host__ __device__ constexpr int gain_vstride(int r) { return (GT_W + 2 * r) | 1; }

// Window sums as sliding runs: a thread forms one full (2r+1)-tap sum and then
// advances it by one add and one subtract per output.  The window is staged
// once as fp64 (y - shift; warps on rows, lanes on columns: no index
// division); vertical pass first (per staged column, two runs of 16 output
// rows, lanes on consecutive columns), then the horizontal pass on the column
// sums (per output row, runs of GRUN columns, lanes on consecutive rows of an
// odd-stride plane: conflict-free); the gain values go through shared memory
// to a coalesced store.  Interior tiles skip the reflect-101 index arithmetic.
__global__ void __launch_bounds__(256) k_gain_map(GainParams P) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int r = P.radius;
  const int SW = GT_W + 2 * r, SH = GT_H + 2 * r, VS = gain_vstride(r);
  double* tile = reinterpret_cast<double*>(sm);  // SH x SW, y - shift
  double* v1 = tile + SH * SW;                   // GT_H x VS
  double* v2 = v1 + GT_H * VS;
  float* gout = reinterpret_cast<float*>(tile);  // GT_H x (GT_W + 1), reuses the window after the vertical pass
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int y0 = blockIdx.y * GT_H, x0 = blockIdx.x * GT_W;
  // shift by one sample of the tile: variance is shift-invariant, the sums stay small
  const float shift = __ldg(P.y + (long long)min(y0, P.H - 1) * P.y_pitch + min(x0, P.W - 1));
  const bool interior = y0 - r >= 0 && y0 + GT_H + r <= P.H && x0 - r >= 0 && x0 + GT_W + r <= P.W;
  if (interior) {
    // SW <= 128: at most four 32-column passes per row, unrolled
    const float* src = P.y + (long long)(y0 - r + warp) * P.y_pitch + (x0 - r) + lane;
    const long long step = 8 * P.y_pitch;
    double* dst = tile + warp * SW + lane;
    for (int ty = warp; ty < SH; ty += 8, src += step, dst += 8 * SW) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (lane + 32 * u < SW) dst[32 * u] = (double)(__ldg(src + 32 * u) - shift);
    }
  } else {
    for (int ty = warp; ty < SH; ty += 8) {
      const float* src = P.y + (long long)refl_fold(y0 - r + ty, P.H) * P.y_pitch;
      for (int tx = lane; tx < SW; tx += 32)
        tile[ty * SW + tx] = (double)(__ldg(src + refl_fold(x0 - r + tx, P.W)) - shift);
    }
  }
  __syncthreads();
  // vertical: per staged column, two runs of GT_H / 2 output rows
  constexpr int VR = GT_H / 2;
  for (int t = threadIdx.x; t < 2 * SW; t += blockDim.x) {
    const int col = t < SW ? t : t - SW, r0 = t < SW ? 0 : VR;
    const double* c = tile + r0 * SW + col;
    double s1 = 0.0, s2 = 0.0;
    for (int d = 0; d <= 2 * r; ++d) {
      const double v = c[d * SW];
      s1 += v;
      s2 = fma(v, v, s2);
    }
    v1[r0 * VS + col] = s1;
    v2[r0 * VS + col] = s2;
#pragma unroll 4
    for (int q = 1; q < VR; ++q) {
      const double vin = c[(q + 2 * r) * SW], vout = c[(q - 1) * SW];
      s1 += vin - vout;
      s2 += fma(vin, vin, -vout * vout);
      v1[(r0 + q) * VS + col] = s1;
      v2[(r0 + q) * VS + col] = s2;
    }
  }
  __syncthreads();
  // horizontal: per output row, runs of GRUN output columns (lanes = rows)
  const double inv_n = 1.0 / ((2.0 * r + 1.0) * (2.0 * r + 1.0));
  const float mlo = (float)P.m_lo, dm = (float)(P.m_hi - P.m_lo), ivr = (float)P.inv_vref;
  {
    const int row = threadIdx.x % GT_H, c0 = (threadIdx.x / GT_H) * GRUN;  // 256 = GT_H x GT_W / GRUN
    const double* a1 = v1 + row * VS + c0;
    const double* a2 = v2 + row * VS + c0;
    double s1 = 0.0, s2 = 0.0;
    for (int d = 0; d <= 2 * r; ++d) {
      s1 += a1[d];
      s2 += a2[d];
    }
#pragma unroll
    for (int q = 0; q < GRUN; ++q) {
      if (q > 0) {
        s1 += a1[q + 2 * r] - a1[q - 1];
        s2 += a2[q + 2 * r] - a2[q - 1];
      }
      const double mean = s1 * inv_n;
      const float var = (float)fma(s2, inv_n, -mean * mean);  // fp64 where it cancels, fp32 after
      gout[row * (GT_W + 1) + c0 + q] = fmaf(dm, fminf(1.f, fmaxf(var, 0.f) * ivr), mlo);
    }
  }
  __syncthreads();
  for (int ty = warp; ty < GT_H; ty += 8) {
    const int gy = y0 + ty;
    if (gy >= P.H) break;
    for (int tx = lane; tx < GT_W; tx += 32)
      if (x0 + tx < P.W) P.m[(long long)gy * P.m_pitch + x0 + tx] = gout[ty * (GT_W + 1) + tx];
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
  return sizeof(double) * ((size_t)SH * SW + 2 * (size_t)GT_H * gain_vstride(radius));
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
