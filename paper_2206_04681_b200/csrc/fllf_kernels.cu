// Fourier LLF hot-path kernels for sm_100a (B200).
//
// Two kernel families:
//
//  k_build  -- one 2x reduce step of Eq. 1 for a chunk of
//              channels: the real G_l[I] and the complex Gaussian Fourier
//              pyramids Z_{l,k} = G_l[cos w_k I] + i G_l[sin w_k I].
//              At level 0 the channels cos/sin(w_k I) are generated on the
//              fly from I (one sincos per pixel + a Chebyshev recurrence in k)
//              and fed straight into the blur: level-0 Fourier planes are
//              never written (north star).
//              Layout: lane owns fine columns (2x, 2x+1) -> coarse column x;
//              the warp streams down a strip of rows doing the VERTICAL
//              5-tap first (two rolling accumulators per channel in
//              registers, one pass over each input row, rows prefetched two
//              pairs ahead), then the HORIZONTAL 5-tap on the finished row
//              with warp shuffles.  Lanes 0 and 31 only supply halo columns
//              (30 outputs per warp).  Complex values are float2 (Im, Re) and
//              all filtering is packed fp32x2 math (FFMA2 / FADD2 / FMUL2).
//
//  k_apply  -- Eq. 14 fused with the collapse of Eq. 4
//              (P:138-141), coarse to fine.  For level l it computes
//                D_l = up(D_{l+1}) + sum_k a_k Im(e^{-i w_k g} (Z_{l,k} - up Z_{l+1,k}))
//              (D_l = O_l - G_l; D_lmax = 0) and at level 0
//                O = I + up(D_1) - sum_k a_k Im(e^{-i w_k I} up Z_{1,k})
//              (the same-level level-0 term vanishes).  All K orders
//              are accumulated in registers; e^{i w_k g} comes from one
//              sincos(w_1 g) and a Chebyshev recurrence.
//              Layout: thread owns a 2x4 block of fine pixels (one coarse row,
//              two coarse columns); per order it reads the three coarse rows
//              it needs (next order prefetched), coarse neighbours come from
//              warp shuffles.  Small levels split the K orders over the 4
//              warps of a CTA (KSPLIT) and reduce through shared memory.
//
// No tensor cores: this is a stencil + elementwise path (no contraction).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fllf_internal.h"

namespace fllf {
namespace {

constexpr unsigned FULL = 0xffffffffu;
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

// complex products for unit phasors.  (s, c) layout = (Im, Re).
__device__ __forceinline__ float2 cmul_sc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.y, a.y * b.x), fmaf(a.y, b.y, -a.x * b.x));
}
// (c, s) layout = (Re, Im).
__device__ __forceinline__ float2 cmul_cs(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// z^n by binary powering (n >= 0, warp-uniform); identity is (0,1) / (1,0).
__device__ __forceinline__ float2 cpow_sc(float2 z, int n) {
  float2 r = make_float2(0.f, 1.f);
  while (n) {
    if (n & 1) r = cmul_sc(r, z);
    z = cmul_sc(z, z);
    n >>= 1;
  }
  return r;
}
__device__ __forceinline__ float2 cpow_cs(float2 z, int n) {
  float2 r = make_float2(1.f, 0.f);
  while (n) {
    if (n & 1) r = cmul_cs(r, z);
    z = cmul_cs(z, z);
    n >>= 1;
  }
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

// Horizontal 5-tap + decimation of a finished complex row value held as
// (a, b) = (fine col 2x, 2x+1), each (Im, Re):
//   h(x) = w2 f(2x-2) + w1 f(2x-1) + w0 f(2x) + w1 f(2x+1) + w2 f(2x+2)
__device__ __forceinline__ float2 hfilt_c(float2 a, float2 b) {
  const float2 pa = shfl_up2(a), pb = shfl_up2(b), na = shfl_down2(a);
  return pfma(bc(W0), a, pfma(bc(W1), padd(pb, b), pmul(bc(W2), padd(pa, na))));
}
__device__ __forceinline__ float hfilt_r(float a, float b) {
  const float pa = __shfl_up_sync(FULL, a, 1);
  const float pb = __shfl_up_sync(FULL, b, 1);
  const float na = __shfl_down_sync(FULL, a, 1);
  return fmaf(W2, pa + na, fmaf(W1, pb + b, W0 * a));
}

// ----------------------------------------------------------------- build
// NC complex channels per chunk, NR real channels (1: G; 2: sigma/m maps).
template <int NC, int NR, bool FROM_IMAGE>
__global__ void __launch_bounds__(128) k_build(const BuildParams P) {
  constexpr int NCX = NC > 0 ? NC : 1;
  constexpr int NCL = FROM_IMAGE ? 1 : NCX;  // complex values loaded per row
  const int lane = threadIdx.x & 31;
  const int cb = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (cb * 30 >= P.Wc) return;
  const int o0 = blockIdx.y * P.rows_per_strip;
  if (o0 >= P.Hc) return;
  const int R = min(P.rows_per_strip, P.Hc - o0);  // output rows of this strip
  const int chunk = blockIdx.z % P.nchunks;
  const int frame = blockIdx.z / P.nchunks;
  const int x = cb * 30 + lane - 1;
  const bool store_lane = lane >= 1 && lane <= 30 && x < P.Wc;
  const int c0 = 2 * x;
  const bool inside = (c0 >= 0) && (c0 + 1 < P.Wf);
  const int rc0 = refl101(c0, P.Wf), rc1 = refl101(c0 + 1, P.Wf);
  const int k0 = chunk * NC;
  const int nc = NC > 0 ? min(NC, P.KL - k0) : 0;
  const bool do_real = (chunk == 0);

  // ---- real planes: sources / destinations
  const float* rsrc[NR];
  float* rdst[NR];
  long long rpitch;
  bool raligned;
  if (FROM_IMAGE) {
    rsrc[0] = P.img.p + frame * P.img.fstride;
    if (NR > 1) rsrc[NR - 1] = P.img2.p + frame * P.img2.fstride;
    rpitch = P.img.pitch;
    raligned = ((reinterpret_cast<uintptr_t>(P.img.p) & 7) == 0) && ((P.img.pitch & 1) == 0) &&
               (NR < 2 || (((reinterpret_cast<uintptr_t>(P.img2.p) & 7) == 0) && P.img2.pitch == P.img.pitch));
  } else {
    if (P.maps) {
      rsrc[0] = P.src.MS;
      if (NR > 1) rsrc[NR - 1] = P.src.MM;
    } else {
      rsrc[0] = P.src.G + frame * P.src.fstride_r;
    }
    rpitch = P.src.pitch;
    raligned = true;
  }
  if (P.maps) {
    rdst[0] = P.dst.MS;
    if (NR > 1) rdst[NR - 1] = P.dst.MM;
  } else {
    rdst[0] = P.dst.G + frame * P.dst.fstride_r;
  }
  const bool rvec = inside && raligned;

  const float2* zsrc = nullptr;
  float2* zdst = nullptr;
  if (NC > 0) {
    if (!FROM_IMAGE) zsrc = P.src.Z + frame * P.src.fstride_z + (long long)k0 * P.src.kstride_z;
    zdst = P.dst.Z + frame * P.dst.fstride_z + (long long)k0 * P.dst.kstride_z;
  }
  const int g0 = P.kbase + k0;  // global order of this chunk's first channel

  struct Row {
    float2 r[NR];
    float4 c[NCL];
  };
  struct Pair {
    Row e, o;
  };
  auto load_row = [&](int row, Row& d) {
    const int rr = refl101(row, P.Hf);
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const float* rp = rsrc[i] + (long long)rr * rpitch;
      d.r[i] = rvec ? ldg2(rp + c0) : make_float2(__ldg(rp + rc0), __ldg(rp + rc1));
    }
    if (!FROM_IMAGE && NC > 0) {
#pragma unroll
      for (int i = 0; i < NCX; ++i) {
        if (i < nc) {
          const float2* zp = zsrc + (long long)i * P.src.kstride_z + (long long)rr * P.src.pitch;
          if (inside) {
            d.c[i] = ldg4(zp + c0);
          } else {
            d.c[i] = cat4(__ldg(zp + rc0), __ldg(zp + rc1));
          }
        }
      }
    }
  };
  // pair p holds rows 2(o0+p-1), 2(o0+p-1)+1 (p = 0: the two halo rows above)
  auto load_pair = [&](int p, Pair& d) {
    const int r0 = 2 * (o0 + p - 1);
    load_row(r0, d.e);
    load_row(r0 + 1, d.o);
  };

  // two role-swapping accumulators per channel (see vstep)
  float4 S0c[NCX] = {}, S1c[NCX] = {};
  float2 S0r[NR] = {}, S1r[NR] = {};

  // Process one row pair with roles (Pc/Pr = pending output, Ac/Ar = current).
  // emit >= 0: finish output row `emit` with the even row and store it.
  // only_emit: the final row (no accumulator update).
  auto proc = [&](const Pair& d, float4 (&Pc)[NCX], float4 (&Ac)[NCX], float2 (&Pr)[NR],
                  float2 (&Ar)[NR], int emit, bool only_emit) {
    if (do_real) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        if (emit >= 0) {
          const float2 e = pfma(bc(W2), d.e.r[i], Pr[i]);
          const float h = hfilt_r(e.x, e.y);
          if (store_lane) rdst[i][(long long)emit * P.dst.pitch + x] = h;
        }
        if (!only_emit) vstep(Pr[i], Ar[i], d.e.r[i], d.o.r[i]);
      }
    }
    if (NC == 0) return;
    auto chan = [&](int i, float4 ve, float4 vo) {
      if (emit >= 0) {
        const float2 ea = pfma(bc(W2), lo2(ve), lo2(Pc[i]));
        const float2 eb = pfma(bc(W2), hi2(ve), hi2(Pc[i]));
        const float2 h = hfilt_c(ea, eb);
        if (store_lane) zdst[(long long)i * P.dst.kstride_z + (long long)emit * P.dst.pitch + x] = h;
      }
      if (!only_emit) {
        float2 pa = lo2(Pc[i]), pb = hi2(Pc[i]), aa = lo2(Ac[i]), ab = hi2(Ac[i]);
        vstep(pa, aa, lo2(ve), lo2(vo));
        vstep(pb, ab, hi2(ve), hi2(vo));
        Pc[i] = cat4(pa, pb);
        Ac[i] = cat4(aa, ab);
      }
    };
    if (FROM_IMAGE) {
      // e^{i k w_1 I} for the 4 pixels (even/odd row x col a/b), (s, c) layout
      float2 z1[4], zc[4], zp[4], tc[4];
      const float I4[4] = {d.e.r[0].x, d.e.r[0].y, d.o.r[0].x, d.o.r[0].y};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float s, c;
        sincos_turns(I4[q], P.invT, &s, &c);
        z1[q] = make_float2(s, c);
        tc[q] = bc(2.f * c);
        if (g0 == 1) {
          zp[q] = make_float2(0.f, 1.f);
          zc[q] = z1[q];
        } else {
          zp[q] = cpow_sc(z1[q], g0 - 1);
          zc[q] = cmul_sc(zp[q], z1[q]);
        }
      }
#pragma unroll
      for (int i = 0; i < NCX; ++i) {
        if (i < nc) {
          chan(i, cat4(zc[0], zc[1]), cat4(zc[2], zc[3]));
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 zn = pfma(tc[q], zc[q], pneg(zp[q]));
            zp[q] = zc[q];
            zc[q] = zn;
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < NCX; ++i)
        if (i < nc) chan(i, d.e.c[i], d.o.c[i]);
    }
  };

  Pair BA, BB;
  load_pair(0, BA);
  load_pair(1, BB);
  proc(BA, S1c, S0c, S1r, S0r, -1, false);  // p = 0: halo rows
  load_pair(2, BA);
  proc(BB, S0c, S1c, S0r, S1r, -1, false);  // p = 1: first pair, nothing to emit
  load_pair(3, BB);
  int p = 2;
#pragma unroll 1
  for (; p + 1 <= R; p += 2) {
    proc(BA, S1c, S0c, S1r, S0r, o0 + p - 2, false);
    load_pair(p + 2, BA);
    proc(BB, S0c, S1c, S0r, S1r, o0 + p - 1, false);
    load_pair(p + 3, BB);
  }
  if (p <= R) {
    proc(BA, S1c, S0c, S1r, S0r, o0 + p - 2, false);
    proc(BB, S0c, S1c, S0r, S1r, o0 + R - 1, true);  // final row = even row of pair R+1
  } else {
    proc(BA, S1c, S0c, S1r, S0r, o0 + R - 1, true);
  }
}

// ----------------------------------------------------------------- apply
template <bool LEVEL0, bool HAS_D, bool MAPS, int KSPLIT>
__global__ void __launch_bounds__(128) k_apply(const ApplyParams P) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int jb = KSPLIT == 1 ? blockIdx.x * 4 + warp : blockIdx.x;
  if (jb * 60 >= P.Wc) return;       // warp- (KSPLIT=1) or block-uniform (KSPLIT>1)
  const int j = jb * 30 + lane - 1;  // coarse columns 2j, 2j+1 -> fine columns 4j..4j+3
  const int r = blockIdx.y;          // coarse row -> fine rows 2r, 2r+1
  const int frame = blockIdx.z;
  const bool act = lane >= 1 && lane <= 30 && 4 * j < P.Wf;
  const bool row1 = 2 * r + 1 < P.Hf;
  const int yf[2] = {2 * r, row1 ? 2 * r + 1 : 2 * r};
  const int xf0 = 4 * j;
  const bool fvec_ok = xf0 >= 0 && xf0 + 3 < P.Wf;
  int xf[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) xf[q] = min(max(xf0 + q, 0), P.Wf - 1);

  // coarse rows r-1, r, r+1 and columns 2j, 2j+1 (polyphase border rule)
  const int cr[3] = {upmap(r - 1, P.Hc, P.Hf), r, upmap(r + 1, P.Hc, P.Hf)};
  const bool cvec = (2 * j >= 0) && (2 * j + 1 < P.Wc);
  const int cc0 = upmap(2 * j, P.Wc, P.Wf), cc1 = upmap(2 * j + 1, P.Wc, P.Wf);

  int k_lo = 0, k_hi = P.KL;
  if (KSPLIT > 1) {
    const int per = (P.KL + KSPLIT - 1) / KSPLIT;
    k_lo = min(warp * per, P.KL);
    k_hi = min(k_lo + per, P.KL);
  }

  // ---- up(D_{l+1}) coarse rows: issue early (used after the order loop)
  float dq[3][2];
  if (HAS_D && (KSPLIT == 1 || warp == 0)) {
    const float* dc = P.coarse.D + frame * P.coarse.fstride_r;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const float* rp = dc + (long long)cr[t] * P.coarse.pitch;
      if (cvec) {
        const float2 q = ldg2(rp + 2 * j);
        dq[t][0] = q.x; dq[t][1] = q.y;
      } else {
        dq[t][0] = __ldg(rp + cc0); dq[t][1] = __ldg(rp + cc1);
      }
    }
  }

  // ---- per fine pixel p = 4*t + q (t: fine row 2r+t, q: fine col 4j+q): g
  float g[8];
  {
    const float* base;
    long long pitch;
    bool al;
    if (LEVEL0) {
      base = P.img.p + frame * P.img.fstride;
      pitch = P.img.pitch;
      al = ((reinterpret_cast<uintptr_t>(P.img.p) & 15) == 0) && ((P.img.pitch & 3) == 0);
    } else {
      base = P.fine.G + frame * P.fine.fstride_r;
      pitch = P.fine.pitch;
      al = true;
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const float* rp = base + (long long)yf[t] * pitch;
      if (fvec_ok && al) {
        const float4 v = ldg4(rp + xf0);
        g[4 * t + 0] = v.x; g[4 * t + 1] = v.y; g[4 * t + 2] = v.z; g[4 * t + 3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) g[4 * t + q] = __ldg(rp + xf[q]);
      }
    }
  }

  // Chebyshev state per pixel, (c, s) layout: z = e^{i k w_1 g}, zp = e^{i (k-1) w_1 g}
  float2 z[8], zp[8], tc[8], acc[8];
  const int g0 = P.kbase + k_lo;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    float s, c;
    sincos_turns(g[p], P.invT, &s, &c);
    const float2 z1 = make_float2(c, s);
    tc[p] = bc(2.f * c);
    if (g0 == 1) {
      zp[p] = make_float2(1.f, 0.f);
      z[p] = z1;
    } else {
      zp[p] = cpow_cs(z1, g0 - 1);
      z[p] = cmul_cs(zp[p], z1);
    }
    acc[p] = make_float2(0.f, 0.f);
  }

  // MAPS: a_k(p) = m sigma^3 c0 k exp(-k^2 hq sigma^2) (Sec. III-B; Eq. 9-11),
  // carried as mA = a_k, mR = exp(-(2k+1) beta), mQ = exp(-2 beta)
  float mA[8], mR[8], mQ[8];
  if (MAPS) {
    const float* sptr;
    const float* mptr;
    long long mp;
    if (LEVEL0) {
      sptr = P.smap.p; mptr = P.mmap.p; mp = P.smap.pitch;
    } else {
      sptr = P.fine.MS; mptr = P.fine.MM; mp = P.fine.pitch;
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long off = (long long)yf[t] * mp + xf[q];
        const float sg = __ldg(sptr + off), m = __ldg(mptr + off);
        const float beta = P.hq * sg * sg;
        const int p = 4 * t + q;
        mA[p] = m * sg * sg * sg * P.c0 * (float)g0 * __expf(-(float)g0 * (float)g0 * beta);
        mR[p] = __expf(-(float)(2 * g0 + 1) * beta);
        mQ[p] = __expf(-2.f * beta);
      }
    }
  }

  const float2* zc_base = P.coarse.Z + frame * P.coarse.fstride_z;
  const float2* zf_base = LEVEL0 ? nullptr : P.fine.Z + frame * P.fine.fstride_z;

  struct KData {
    float4 q[3];  // coarse rows r-1, r, r+1 at coarse cols (2j, 2j+1)
    float4 f[4];  // fine Z_{l,k}: rows 2r, 2r+1 x cols (4j, 4j+1), (4j+2, 4j+3)
  };
  auto loadk = [&](int k, KData& d) {
    const float2* zc = zc_base + (long long)k * P.coarse.kstride_z;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const float2* rp = zc + (long long)cr[t] * P.coarse.pitch;
      d.q[t] = cvec ? ldg4(rp + 2 * j) : cat4(__ldg(rp + cc0), __ldg(rp + cc1));
    }
    if (!LEVEL0) {
      const float2* zf = zf_base + (long long)k * P.fine.kstride_z;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const float2* rp = zf + (long long)yf[t] * P.fine.pitch;
        if (fvec_ok) {
          d.f[2 * t] = ldg4(rp + xf0);
          d.f[2 * t + 1] = ldg4(rp + xf0 + 2);
        } else {
          d.f[2 * t] = cat4(__ldg(rp + xf[0]), __ldg(rp + xf[1]));
          d.f[2 * t + 1] = cat4(__ldg(rp + xf[2]), __ldg(rp + xf[3]));
        }
      }
    }
  };

  auto compute = [&](const KData& d, int k) {
    // horizontal polyphase up-sampling of the 3 coarse rows (unscaled):
    //   even fine col 2c: x_{c-1} + 6 x_c + x_{c+1} (/8); odd 2c+1: x_c + x_{c+1} (/2)
    float2 h[3][4];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const float2 x0 = lo2(d.q[t]), x1 = hi2(d.q[t]);
      const float2 L = shfl_up2(x1), Rn = shfl_down2(x0);
      h[t][0] = pfma(bc(6.f), x0, padd(L, x1));
      h[t][1] = padd(x0, x1);
      h[t][2] = pfma(bc(6.f), x1, padd(x0, Rn));
      h[t][3] = padd(x1, Rn);
    }
    float2 waa, w1, w2, w3;
    if (MAPS) {
      waa = bc(1.f); w1 = bc(-1.f / 64.f); w2 = bc(-1.f / 16.f); w3 = bc(-1.f / 4.f);
    } else {
      waa = P.wk[k][0]; w1 = P.wk[k][1]; w2 = P.wk[k][2]; w3 = P.wk[k][3];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // vertical: even fine row (h[-1] + 6 h[0] + h[+1]) (/8); odd (h[0] + h[+1]) (/2)
      const float2 re = pfma(bc(6.f), h[1][q], padd(h[0][q], h[2][q]));
      const float2 ro = padd(h[1][q], h[2][q]);
      const float2 we = (q & 1) ? w2 : w1;  // even row: ee 1/64, eo 1/16
      const float2 wo = (q & 1) ? w3 : w2;  // odd row:  oe 1/16, oo 1/4
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int p = 4 * t + q;
        const float2 raw = t == 0 ? re : ro;
        const float2 w = t == 0 ? we : wo;
        float2 V;  // (Im, Re) of a_k (Z_l - up Z_{l+1}) at this pixel
        float2 zf = make_float2(0.f, 0.f);
        if (!LEVEL0) {
          const float4 fv = d.f[2 * t + (q >> 1)];
          zf = (q & 1) ? hi2(fv) : lo2(fv);
        }
        if (MAPS) {
          V = pmul(bc(mA[p]), LEVEL0 ? pmul(w, raw) : pfma(w, raw, zf));
        } else {
          V = LEVEL0 ? pmul(w, raw) : pfma(w, raw, pmul(waa, zf));
        }
        // acc += (c V.im, s V.re); result = acc.x - acc.y = a Im(e^{-i k w g} (...))
        acc[p] = pfma(z[p], V, acc[p]);
        const float2 zn = pfma(tc[p], z[p], pneg(zp[p]));
        zp[p] = z[p];
        z[p] = zn;
        if (MAPS) {
          // a_{k+1} = a_k (k+1)/k exp(-(2k+1) beta)
          const float kk = (float)(P.kbase + k);
          mA[p] *= mR[p] * ((kk + 1.f) / kk);
          mR[p] *= mQ[p];
        }
      }
    }
  };

  {
    KData A, B;
    int k = k_lo;
    if (k < k_hi) loadk(k, A);
#pragma unroll 1
    while (k < k_hi) {
      if (k + 1 < k_hi) loadk(k + 1, B);
      compute(A, k);
      if (k + 1 >= k_hi) break;
      if (k + 2 < k_hi) loadk(k + 2, A);
      compute(B, k + 1);
      k += 2;
    }
  }

  float res[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) res[p] = acc[p].x - acc[p].y;

  if (KSPLIT > 1) {
    __shared__ float red[KSPLIT > 1 ? KSPLIT - 1 : 1][8][32];
    if (warp > 0) {
#pragma unroll
      for (int p = 0; p < 8; ++p) red[warp - 1][p][lane] = res[p];
    }
    __syncthreads();
    if (warp > 0) return;
#pragma unroll
    for (int w = 0; w < KSPLIT - 1; ++w)
#pragma unroll
      for (int p = 0; p < 8; ++p) res[p] += red[w][p][lane];
  }

  // --- collapse: + up(D_{l+1})
  if (HAS_D) {
    float hd[3][4];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const float x0 = dq[t][0], x1 = dq[t][1];
      const float L = __shfl_up_sync(FULL, x1, 1);
      const float Rn = __shfl_down_sync(FULL, x0, 1);
      hd[t][0] = fmaf(6.f, x0, L + x1) * 0.125f;
      hd[t][1] = (x0 + x1) * 0.5f;
      hd[t][2] = fmaf(6.f, x1, x0 + Rn) * 0.125f;
      hd[t][3] = (x1 + Rn) * 0.5f;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      res[q] += 0.125f * fmaf(6.f, hd[1][q], hd[0][q] + hd[2][q]);
      res[4 + q] += 0.5f * (hd[1][q] + hd[2][q]);
    }
  }
  if (LEVEL0 && P.include_base) {
#pragma unroll
    for (int p = 0; p < 8; ++p) res[p] += g[p];
  }

  if (!act) return;
  float* op;
  long long opitch;
  bool oal;
  if (LEVEL0) {
    op = P.out + frame * P.out_fstride;
    opitch = P.out_pitch;
    oal = ((reinterpret_cast<uintptr_t>(P.out) & 15) == 0) && ((P.out_pitch & 3) == 0);
  } else {
    op = P.fine.D + frame * P.fine.fstride_r;
    opitch = P.fine.pitch;
    oal = true;
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    if (t == 1 && !row1) break;
    float* rp = op + (long long)(2 * r + t) * opitch;
    if (fvec_ok && oal) {
      *reinterpret_cast<float4*>(rp + xf0) = make_float4(res[4 * t], res[4 * t + 1], res[4 * t + 2], res[4 * t + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (xf0 + q < P.Wf) rp[xf0 + q] = res[4 * t + q];
    }
  }
}

// Rows per warp strip: long strips amortise the 3 halo rows; shorter strips
// when the grid would not fill the GPU.
int pick_rows(int Hc, int blocks_x, int z) {
  int R = 16;
  while (R > 2 && (long long)blocks_x * ((Hc + R - 1) / R) * z < 148LL * 4) R >>= 1;
  return R;
}

}  // namespace

cudaError_t launch_build(const BuildParams& p0, int level_src, int batch, cudaStream_t s) {
  BuildParams p = p0;
  const int warps_x = (p.Wc + 29) / 30;
  const int bx = (warps_x + 3) / 4;
  if (p.maps) {
    p.nchunks = 1;
    p.rows_per_strip = pick_rows(p.Hc, bx, 1);
    dim3 grid(bx, (p.Hc + p.rows_per_strip - 1) / p.rows_per_strip, 1);
    if (level_src == 0)
      k_build<0, 2, true><<<grid, 128, 0, s>>>(p);
    else
      k_build<0, 2, false><<<grid, 128, 0, s>>>(p);
    return cudaGetLastError();
  }
  if (level_src == 0) {
    if (p.KL <= 4) {
      p.nchunks = 1;
      p.rows_per_strip = pick_rows(p.Hc, bx, batch);
      dim3 grid(bx, (p.Hc + p.rows_per_strip - 1) / p.rows_per_strip, batch);
      k_build<4, 1, true><<<grid, 128, 0, s>>>(p);
    } else {
      constexpr int NC = 8;
      p.nchunks = (p.KL + NC - 1) / NC;
      p.rows_per_strip = pick_rows(p.Hc, bx, batch * p.nchunks);
      dim3 grid(bx, (p.Hc + p.rows_per_strip - 1) / p.rows_per_strip, batch * p.nchunks);
      k_build<NC, 1, true><<<grid, 128, 0, s>>>(p);
    }
  } else {
    constexpr int NC = 2;
    p.nchunks = (p.KL + NC - 1) / NC;
    p.rows_per_strip = pick_rows(p.Hc, bx, batch * p.nchunks);
    dim3 grid(bx, (p.Hc + p.rows_per_strip - 1) / p.rows_per_strip, batch * p.nchunks);
    k_build<NC, 1, false><<<grid, 128, 0, s>>>(p);
  }
  return cudaGetLastError();
}

template <bool L0, bool HD, bool MP>
static void launch_apply_t(const ApplyParams& p, int batch, cudaStream_t s) {
  const int pairs = (p.Wc + 1) / 2;
  const int warps_x = (pairs + 29) / 30;
  const long long ctas1 = (long long)((warps_x + 3) / 4) * p.Hc * batch;
  if (ctas1 >= 2 * 148 || p.KL < 4) {
    dim3 grid((warps_x + 3) / 4, p.Hc, batch);
    k_apply<L0, HD, MP, 1><<<grid, 128, 0, s>>>(p);
  } else {
    dim3 grid(warps_x, p.Hc, batch);
    k_apply<L0, HD, MP, 4><<<grid, 128, 0, s>>>(p);
  }
}

cudaError_t launch_apply(const ApplyParams& p, int level_fine, bool has_d, bool maps, int batch,
                         cudaStream_t s) {
#define FLLF_APPLY(L0, HD, MP) launch_apply_t<L0, HD, MP>(p, batch, s)
  if (level_fine == 0) {
    if (maps) {
      if (has_d) FLLF_APPLY(true, true, true); else FLLF_APPLY(true, false, true);
    } else {
      if (has_d) FLLF_APPLY(true, true, false); else FLLF_APPLY(true, false, false);
    }
  } else {
    if (maps) {
      if (has_d) FLLF_APPLY(false, true, true); else FLLF_APPLY(false, false, true);
    } else {
      if (has_d) FLLF_APPLY(false, true, false); else FLLF_APPLY(false, false, false);
    }
  }
#undef FLLF_APPLY
  return cudaGetLastError();
}

}  // namespace fllf
