// Device helpers shared by the pyramid kernels (fllf_kernels.cu) and the
// fused materialise-once kernels (fllf_fused.cu): packed fp32x2 math, warp
// shuffles, border index rules, phasors, debug-bounds stores.  Included
// inside `namespace fllf { namespace {` of each translation unit (internal
// linkage, no ODR coupling between the two).
#pragma once
constexpr unsigned FULL = 0xffffffffu;

// Debug-bounds builds (`build --variant dbg -DFLLF_DEBUG_BOUNDS`; compute-
// sanitizer is closed on this GPU pool): every global store of the pyramid
// kernels is checked against the range the host declared for the launch
// (the plan workspace, or the caller's output) and traps on a miss.
#ifdef FLLF_DEBUG_BOUNDS
#define FLLF_DBG_STORE(P, ptr, nbytes)                                                                       \
  do {                                                                                                      \
    const char* p_ = reinterpret_cast<const char*>(ptr);                                                   \
    if (p_ < (P).dbg_lo || p_ + (nbytes) > (P).dbg_hi) {                                                    \
      printf("fllf bounds: line %d block (%d,%d,%d) thread %d\n", __LINE__, blockIdx.x, blockIdx.y,        \
             blockIdx.z, threadIdx.x);                                                                      \
      __trap();                                                                                             \
    }                                                                                                       \
  } while (0)
#else
#define FLLF_DBG_STORE(P, ptr, nbytes) ((void)0)
#endif
// [1,4,6,4,1]/16
constexpr float W0 = 0.375f, W1 = 0.25f, W2 = 0.0625f;
constexpr float TWO_PI = 6.28318530717958647692f;

// ------------------------------------------------------------- helpers
__device__ __forceinline__ float2 bc(float w) { return make_float2(w, w); }
__device__ __forceinline__ float2 pfma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 pmul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 padd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 pneg(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 lo2(float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(float4 v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float4 cat4(float2 a, float2 b) { return make_float4(a.x, a.y, b.x, b.y); }

__device__ __forceinline__ float2 shfl_up2(float2 v) {
  return make_float2(__shfl_up_sync(FULL, v.x, 1), __shfl_up_sync(FULL, v.y, 1));
}
__device__ __forceinline__ float2 shfl_down2(float2 v) {
  return make_float2(__shfl_down_sync(FULL, v.x, 1), __shfl_down_sync(FULL, v.y, 1));
}

// Reflect-101 (reading R2) for indices within one bounce; clamps beyond (those
// lanes only feed halo values that are never stored).
__device__ __forceinline__ int refl101(int i, int n) {
  i = i < 0 ? -i : i;
  i = i >= n ? 2 * (n - 1) - i : i;
  return min(max(i, 0), n - 1);
}

// Coarse index used by the polyphase up-sampling at fine size nf (coarse
// C = ceil(nf/2)), equivalent to reflect-101 on the zero-inserted fine grid:
// x_{-1} := x_1; x_C := x_{C-1} if nf is even, x_{C-2} if nf is odd.
__device__ __forceinline__ int upmap(int c, int C, int nf) {
  if (c < 0) c = -c;
  if (c >= C) c = (c == C) ? ((nf & 1) ? C - 2 : C - 1) : C - 1;
  return min(c, C - 1);
}

// theta = w_1 * val = 2 pi * frac(val / T): range-reduced in turns first.
__device__ __forceinline__ void sincos_turns(float val, float invT, float* s, float* c) {
  float u = val * invT;
  u -= rintf(u);
  __sincosf(TWO_PI * u, s, c);
}

// e^{i n theta}: n * frac(val/T) reduced again to [-1/2, 1/2] turns.
__device__ __forceinline__ void sincos_turns_n(float val, float invT, int n, float* s, float* c) {
  float u = val * invT;
  u -= rintf(u);
  u *= (float)n;
  u -= rintf(u);
  __sincosf(TWO_PI * u, s, c);
}

// complex products for unit phasors.  (s, c) layout = (Im, Re).
__device__ __forceinline__ float2 cmul_sc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.y, a.y * b.x), fmaf(a.y, b.y, -a.x * b.x));
}
// (c, s) layout = (Re, Im).
__device__ __forceinline__ float2 cmul_cs(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// global store of a float2 (the address came through inline PTX, so say "global")
__device__ __forceinline__ void stg2(float2* q, float2 v) {
  asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(q), "f"(v.x), "f"(v.y) : "memory");
}
// base + off (float2 elements, 32-bit unsigned offset) as one IMAD.WIDE.U32
__device__ __forceinline__ float2* wide_off(float2* base, unsigned off) {
  float2* r;
  asm("mad.wide.u32 %0, %1, 8, %2;" : "=l"(r) : "r"(off), "l"(base));
  return r;
}
__device__ __forceinline__ float2 ldg2(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ldg4(const float2* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// One vertical step over a row pair (even row 2o, odd row 2o+1) for one
// packed value: Pv holds output o-1 missing its last tap, Av output o.
// After the step the roles swap (new P = Av, new A = Pv):
//   Av += w0 ve + w1 vo ;  Pv = w2 ve + w1 vo.
__device__ __forceinline__ void vstep(float2& Pv, float2& Av, float2 ve, float2 vo) {
  Av = pfma(bc(W1), vo, pfma(bc(W0), ve, Av));
  Pv = pfma(bc(W1), vo, pmul(bc(W2), ve));
}

// Same step with fixed names: P = pending output o-1 (missing its last tap),
// A = output o.  After the pair: P <- A + w0 ve + w1 vo (output o, missing its
// last tap), A <- w2 ve + w1 vo (output o+1).
__device__ __forceinline__ void vstep_fixed(float2& Pv, float2& Av, float2 ve, float2 vo) {
  Pv = pfma(bc(W1), vo, pfma(bc(W0), ve, Av));
  Av = pfma(bc(W1), vo, pmul(bc(W2), ve));
}

// Horizontal 5-tap + decimation of a finished complex row value held as
// (a, b) = (fine col 2x, 2x+1), each (Im, Re):
//   h(x) = w2 f(2x-2) + w1 f(2x-1) + w0 f(2x) + w1 f(2x+1) + w2 f(2x+2)
// The left neighbour's two taps travel as one partial sum
// u(x-1) = w2 f(2x-2) + w1 f(2x-1): two shuffles per value instead of three.
__device__ __forceinline__ float2 hfilt_c(float2 a, float2 b) {
  const float2 u = pfma(bc(W1), b, pmul(bc(W2), a));
  const float2 pu = shfl_up2(u), na = shfl_down2(a);
  return pfma(bc(W0), a, pfma(bc(W1), b, pfma(bc(W2), na, pu)));
}
__device__ __forceinline__ float hfilt_r(float a, float b) {
  const float pu = __shfl_up_sync(FULL, fmaf(W1, b, W2 * a), 1);
  const float na = __shfl_down_sync(FULL, a, 1);
  return fmaf(W0, a, fmaf(W1, b, fmaf(W2, na, pu)));
}

// ------------------------------------------------------------ host helpers
// cudaLaunchKernelEx with optional programmatic stream serialization (PDL).
template <typename Kern, typename... Args>
cudaError_t launch_ex(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, const Args&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Per-device state: cudaFuncSetAttribute applies to the device current at the
// call, and SM counts differ between devices, so both are kept per ordinal.
constexpr int kMaxDevices = 64;
struct DeviceFlags {
  std::atomic<int> v[kMaxDevices] = {};
};
inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return dev >= 0 && dev < kMaxDevices ? dev : 0;
}
inline int sm_count() {
  static std::atomic<int> n[kMaxDevices] = {};
  const int dev = current_device();
  int v = n[dev].load(std::memory_order_relaxed);
  if (v <= 0) {
    v = 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    n[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}
// Opt a kernel into `smem` bytes of dynamic shared memory (> 48 KB) on the
// current device, once per device.
template <typename Kern>
cudaError_t smem_opt_in(Kern kern, int smem, DeviceFlags& done) {
  const int dev = current_device();
  if (done.v[dev].load(std::memory_order_relaxed)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) done.v[dev].store(1, std::memory_order_relaxed);
  return e;
}
