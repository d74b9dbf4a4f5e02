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
//              5-tap first (rolling accumulators in registers, one pass over
//              each input row), then the HORIZONTAL 5-tap on the finished
//              half-height row with warp shuffles.  Lanes 0 and 31 only
//              supply halo columns (30 outputs per warp).
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
//              two coarse columns); the three coarse rows it needs are read
//              per order, coarse neighbours come from warp shuffles.
//
// No tensor cores: this is a stencil + elementwise path (no contraction).
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "fllf_internal.h"

namespace fllf {
namespace {

constexpr unsigned FULL = 0xffffffffu;
// [1,4,6,4,1]/16
constexpr float W0 = 0.375f, W1 = 0.25f, W2 = 0.0625f;
constexpr float TWO_PI = 6.28318530717958647692f;

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

// e^{i n theta} with theta = 2 pi u, u = frac(I/T): returned as (sin, cos).
__device__ __forceinline__ float2 cis_turns(float u_frac, int n) {
  float v = u_frac * (float)n;
  v -= rintf(v);
  float s, c;
  __sincosf(TWO_PI * v, &s, &c);
  return make_float2(s, c);
}

__device__ __forceinline__ float frac_turns(float val, float invT) {
  float u = val * invT;
  return u - rintf(u);
}

__device__ __forceinline__ float2 ldg2(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ldg4(const float2* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

__device__ __forceinline__ float4 f4fma(float w, float4 v, float4 a) {
  return make_float4(fmaf(w, v.x, a.x), fmaf(w, v.y, a.y), fmaf(w, v.z, a.z), fmaf(w, v.w, a.w));
}
__device__ __forceinline__ float4 f4mul(float w, float4 v) {
  return make_float4(w * v.x, w * v.y, w * v.z, w * v.w);
}
__device__ __forceinline__ float2 f2fma(float w, float2 v, float2 a) {
  return make_float2(fmaf(w, v.x, a.x), fmaf(w, v.y, a.y));
}
__device__ __forceinline__ float2 f2mul(float w, float2 v) { return make_float2(w * v.x, w * v.y); }

// Horizontal 5-tap + decimation of a vertically filtered row held as the
// pair (a, b) = (fine col 2x, 2x+1) per lane:
//   h(x) = w2 f(2x-2) + w1 f(2x-1) + w0 f(2x) + w1 f(2x+1) + w2 f(2x+2)
__device__ __forceinline__ float hfilt(float a, float b) {
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
  const int lane = threadIdx.x & 31;
  const int cb = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (cb * 30 >= P.Wc) return;
  const int o0 = blockIdx.y * P.rows_per_strip;
  if (o0 >= P.Hc) return;
  const int oend = min(o0 + P.rows_per_strip, P.Hc);
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

  // rolling vertical accumulators: P = output o-1 (missing its last tap),
  // A = output o, B = output o+1
  float4 Pc[NCX] = {}, Ac[NCX] = {}, Bc[NCX] = {};
  float2 Pr[NR] = {}, Ar[NR] = {}, Br[NR] = {};

  // phase: 0 = first halo row, 1 = second halo row, 2 = even row 2o,
  //        3 = odd row 2o+1, 4 = final row.  emit = output row to store or -1.
  auto consume_c = [&](int i, float4 v, int phase, int emit) {
    if (phase == 0) {
      Ac[i] = f4mul(W2, v);
    } else if (phase == 1) {
      Ac[i] = f4fma(W1, v, Ac[i]);
    } else if (phase == 2 || phase == 4) {
      if (emit >= 0) {
        const float4 e = f4fma(W2, v, Pc[i]);
        const float him = hfilt(e.x, e.z);
        const float hre = hfilt(e.y, e.w);
        if (store_lane)
          zdst[(long long)i * P.dst.kstride_z + (long long)emit * P.dst.pitch + x] = make_float2(him, hre);
      }
      if (phase == 2) {
        Ac[i] = f4fma(W0, v, Ac[i]);
        Bc[i] = f4mul(W2, v);
      }
    } else {
      Ac[i] = f4fma(W1, v, Ac[i]);
      Bc[i] = f4fma(W1, v, Bc[i]);
      Pc[i] = Ac[i];
      Ac[i] = Bc[i];
    }
  };
  auto consume_r = [&](int i, float2 v, int phase, int emit) {
    if (phase == 0) {
      Ar[i] = f2mul(W2, v);
    } else if (phase == 1) {
      Ar[i] = f2fma(W1, v, Ar[i]);
    } else if (phase == 2 || phase == 4) {
      if (emit >= 0) {
        const float2 e = f2fma(W2, v, Pr[i]);
        const float h = hfilt(e.x, e.y);
        if (store_lane) rdst[i][(long long)emit * P.dst.pitch + x] = h;
      }
      if (phase == 2) {
        Ar[i] = f2fma(W0, v, Ar[i]);
        Br[i] = f2mul(W2, v);
      }
    } else {
      Ar[i] = f2fma(W1, v, Ar[i]);
      Br[i] = f2fma(W1, v, Br[i]);
      Pr[i] = Ar[i];
      Ar[i] = Br[i];
    }
  };

  auto row = [&](int r, int phase, int emit) {
    const int rr = refl101(r, P.Hf);
    float2 rv[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const float* rp = rsrc[i] + (long long)rr * rpitch;
      rv[i] = rvec ? ldg2(rp + c0) : make_float2(__ldg(rp + rc0), __ldg(rp + rc1));
    }
    if (do_real) {
#pragma unroll
      for (int i = 0; i < NR; ++i) consume_r(i, rv[i], phase, emit);
    }
    if (NC > 0) {
      if (FROM_IMAGE) {
        // cos/sin(w_k I) for the two fine columns, orders g0 .. g0+nc-1
        const float ua = frac_turns(rv[0].x, P.invT), ub = frac_turns(rv[0].y, P.invT);
        const float2 z1a = cis_turns(ua, 1), z1b = cis_turns(ub, 1);
        float2 pa, pb, ca, cb2;
        if (g0 == 1) {
          pa = make_float2(0.f, 1.f);
          pb = pa;
          ca = z1a;
          cb2 = z1b;
        } else {
          pa = cis_turns(ua, g0 - 1);
          pb = cis_turns(ub, g0 - 1);
          ca = cis_turns(ua, g0);
          cb2 = cis_turns(ub, g0);
        }
        const float ta = 2.f * z1a.y, tb = 2.f * z1b.y;
#pragma unroll
        for (int i = 0; i < NCX; ++i) {
          if (i < nc) {
            consume_c(i, make_float4(ca.x, ca.y, cb2.x, cb2.y), phase, emit);
            const float2 na = make_float2(fmaf(ta, ca.x, -pa.x), fmaf(ta, ca.y, -pa.y));
            const float2 nb = make_float2(fmaf(tb, cb2.x, -pb.x), fmaf(tb, cb2.y, -pb.y));
            pa = ca;
            pb = cb2;
            ca = na;
            cb2 = nb;
          }
        }
      } else {
        float4 cv[NCX];
#pragma unroll
        for (int i = 0; i < NCX; ++i) {
          if (i < nc) {
            const float2* zp = zsrc + (long long)i * P.src.kstride_z + (long long)rr * P.src.pitch;
            if (inside) {
              cv[i] = ldg4(zp + c0);
            } else {
              const float2 u = __ldg(zp + rc0), w = __ldg(zp + rc1);
              cv[i] = make_float4(u.x, u.y, w.x, w.y);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < NCX; ++i)
          if (i < nc) consume_c(i, cv[i], phase, emit);
      }
    }
  };

  row(2 * o0 - 2, 0, -1);
  row(2 * o0 - 1, 1, -1);
  row(2 * o0, 2, -1);
  row(2 * o0 + 1, 3, -1);
  for (int o = o0 + 1; o < oend; ++o) {
    row(2 * o, 2, o - 1);
    row(2 * o + 1, 3, -1);
  }
  row(2 * oend, 4, oend - 1);
}

// ----------------------------------------------------------------- apply
// Horizontal polyphase up-sampling of one coarse row pair (x0, x1) =
// (coarse 2j, 2j+1) into fine columns 4j..4j+3, scaled by 8:
//   even fine col 2c: x_{c-1} + 6 x_c + x_{c+1};  odd 2c+1: 4 (x_c + x_{c+1})
template <typename T>
struct Up4 {
  T v[4];
};

__device__ __forceinline__ float2 add2(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }

__device__ __forceinline__ Up4<float2> hup_c(float2 x0, float2 x1) {
  float2 L, R;
  L.x = __shfl_up_sync(FULL, x1.x, 1);
  L.y = __shfl_up_sync(FULL, x1.y, 1);
  R.x = __shfl_down_sync(FULL, x0.x, 1);
  R.y = __shfl_down_sync(FULL, x0.y, 1);
  Up4<float2> h;
  h.v[0] = f2fma(6.f, x0, add2(L, x1));
  h.v[1] = f2mul(4.f, add2(x0, x1));
  h.v[2] = f2fma(6.f, x1, add2(x0, R));
  h.v[3] = f2mul(4.f, add2(x1, R));
  return h;
}

__device__ __forceinline__ Up4<float> hup_r(float x0, float x1) {
  const float L = __shfl_up_sync(FULL, x1, 1);
  const float R = __shfl_down_sync(FULL, x0, 1);
  Up4<float> h;
  h.v[0] = fmaf(6.f, x0, L + x1);
  h.v[1] = 4.f * (x0 + x1);
  h.v[2] = fmaf(6.f, x1, x0 + R);
  h.v[3] = 4.f * (x1 + R);
  return h;
}

template <bool LEVEL0, bool HAS_D, bool MAPS>
__global__ void __launch_bounds__(128) k_apply(const ApplyParams P) {
  const int lane = threadIdx.x & 31;
  const int jb = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (jb * 60 >= P.Wc) return;
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

  // ---- per fine pixel: g (LEVEL0: I), recurrence state, accumulator
  float g[8];
  if (LEVEL0) {
    const float* ip = P.img.p + frame * P.img.fstride;
    const bool al = ((reinterpret_cast<uintptr_t>(P.img.p) & 15) == 0) && ((P.img.pitch & 3) == 0);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const float* rp = ip + (long long)yf[t] * P.img.pitch;
      if (fvec_ok && al) {
        const float4 v = ldg4(rp + xf0);
        g[4 * t + 0] = v.x; g[4 * t + 1] = v.y; g[4 * t + 2] = v.z; g[4 * t + 3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) g[4 * t + q] = __ldg(rp + xf[q]);
      }
    }
  } else {
    const float* gp = P.fine.G + frame * P.fine.fstride_r;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const float* rp = gp + (long long)yf[t] * P.fine.pitch;
      if (fvec_ok) {
        const float4 v = ldg4(rp + xf0);
        g[4 * t + 0] = v.x; g[4 * t + 1] = v.y; g[4 * t + 2] = v.z; g[4 * t + 3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) g[4 * t + q] = __ldg(rp + xf[q]);
      }
    }
  }

  float sk[8], ck[8], sp[8], cp[8], tc[8], acc[8];
  const int g0 = P.kbase;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const float u = frac_turns(g[p], P.invT);
    const float2 z1 = cis_turns(u, 1);
    tc[p] = 2.f * z1.y;
    if (g0 == 1) {
      sp[p] = 0.f; cp[p] = 1.f; sk[p] = z1.x; ck[p] = z1.y;
    } else {
      const float2 zp = cis_turns(u, g0 - 1), zc = cis_turns(u, g0);
      sp[p] = zp.x; cp[p] = zp.y; sk[p] = zc.x; ck[p] = zc.y;
    }
    acc[p] = 0.f;
  }

  // MAPS: a_k(p) = m sigma^3 c0 k exp(-k^2 hq sigma^2)  (Sec. III-B, Eq. 9-11)
  float mA[8], mE[8], mR[8], mQ[8];
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
        const float s = __ldg(sptr + off), m = __ldg(mptr + off);
        const float beta = P.hq * s * s;
        const int p = 4 * t + q;
        mA[p] = m * s * s * s * P.c0;
        mE[p] = __expf(-(float)g0 * (float)g0 * beta);
        mR[p] = __expf(-(float)(2 * g0 + 1) * beta);
        mQ[p] = __expf(-2.f * beta);
      }
    }
  }

  const float2* zc_base = P.coarse.Z + frame * P.coarse.fstride_z;
  const float2* zf_base = LEVEL0 ? nullptr : P.fine.Z + frame * P.fine.fstride_z;

#pragma unroll 1
  for (int k = 0; k < P.KL; ++k) {
    // --- up(Z_{l+1,k}) at the 8 fine pixels (scaled by 64)
    const float2* zc = zc_base + (long long)k * P.coarse.kstride_z;
    Up4<float2> h[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const float2* rp = zc + (long long)cr[t] * P.coarse.pitch;
      float2 x0, x1;
      if (cvec) {
        const float4 q = ldg4(rp + 2 * j);
        x0 = make_float2(q.x, q.y);
        x1 = make_float2(q.z, q.w);
      } else {
        x0 = __ldg(rp + cc0);
        x1 = __ldg(rp + cc1);
      }
      h[t] = hup_c(x0, x1);
    }
    float2 V[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // even fine row: (h[-1] + 6 h[0] + h[+1]) / 64 ; odd: 4 (h[0] + h[+1]) / 64
      const float2 e = f2fma(6.f, h[1].v[q], add2(h[0].v[q], h[2].v[q]));
      const float2 o = f2mul(4.f, add2(h[1].v[q], h[2].v[q]));
      V[q] = f2mul(-1.f / 64.f, e);
      V[4 + q] = f2mul(-1.f / 64.f, o);
    }
    if (!LEVEL0) {
      // + Z_{l,k} at the fine pixels
      const float2* zf = zf_base + (long long)k * P.fine.kstride_z;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const float2* rp = zf + (long long)yf[t] * P.fine.pitch;
        if (fvec_ok) {
          const float4 a = ldg4(rp + xf0), b = ldg4(rp + xf0 + 2);
          V[4 * t + 0] = add2(V[4 * t + 0], make_float2(a.x, a.y));
          V[4 * t + 1] = add2(V[4 * t + 1], make_float2(a.z, a.w));
          V[4 * t + 2] = add2(V[4 * t + 2], make_float2(b.x, b.y));
          V[4 * t + 3] = add2(V[4 * t + 3], make_float2(b.z, b.w));
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) V[4 * t + q] = add2(V[4 * t + q], __ldg(rp + xf[q]));
        }
      }
    }
    // --- product-sum: acc += a_k Im(e^{-i w_k g} V) = a_k (cos V.im - sin V.re)
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      float a;
      if (MAPS) {
        a = mA[p] * (float)(g0 + k) * mE[p];
        mE[p] *= mR[p];
        mR[p] *= mQ[p];
      } else {
        a = P.a[k];
      }
      acc[p] = fmaf(a, fmaf(ck[p], V[p].x, -sk[p] * V[p].y), acc[p]);
      const float ns = fmaf(tc[p], sk[p], -sp[p]);
      const float nc = fmaf(tc[p], ck[p], -cp[p]);
      sp[p] = sk[p]; cp[p] = ck[p];
      sk[p] = ns; ck[p] = nc;
    }
  }

  // --- collapse: + up(D_{l+1})
  if (HAS_D) {
    const float* dc = P.coarse.D + frame * P.coarse.fstride_r;
    Up4<float> h[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const float* rp = dc + (long long)cr[t] * P.coarse.pitch;
      float x0, x1;
      if (cvec) {
        const float2 q = ldg2(rp + 2 * j);
        x0 = q.x; x1 = q.y;
      } else {
        x0 = __ldg(rp + cc0); x1 = __ldg(rp + cc1);
      }
      h[t] = hup_r(x0, x1);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      acc[q] += (1.f / 64.f) * fmaf(6.f, h[1].v[q], h[0].v[q] + h[2].v[q]);
      acc[4 + q] += (4.f / 64.f) * (h[1].v[q] + h[2].v[q]);
    }
  }
  if (LEVEL0 && P.include_base) {
#pragma unroll
    for (int p = 0; p < 8; ++p) acc[p] += g[p];
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
      *reinterpret_cast<float4*>(rp + xf0) = make_float4(acc[4 * t], acc[4 * t + 1], acc[4 * t + 2], acc[4 * t + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (xf0 + q < P.Wf) rp[xf0 + q] = acc[4 * t + q];
    }
  }
}

int pick_rows(int Hc, int blocks_x, int z) {
  int R = 16;
  while (R > 4 && (long long)blocks_x * ((Hc + R - 1) / R) * z < 148LL * 8) R >>= 1;
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
    constexpr int NC = 4;
    p.nchunks = (p.KL + NC - 1) / NC;
    p.rows_per_strip = pick_rows(p.Hc, bx, batch * p.nchunks);
    dim3 grid(bx, (p.Hc + p.rows_per_strip - 1) / p.rows_per_strip, batch * p.nchunks);
    k_build<NC, 1, true><<<grid, 128, 0, s>>>(p);
  } else {
    constexpr int NC = 2;
    p.nchunks = (p.KL + NC - 1) / NC;
    p.rows_per_strip = pick_rows(p.Hc, bx, batch * p.nchunks);
    dim3 grid(bx, (p.Hc + p.rows_per_strip - 1) / p.rows_per_strip, batch * p.nchunks);
    k_build<NC, 1, false><<<grid, 128, 0, s>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_apply(const ApplyParams& p, int level_fine, bool has_d, bool maps, int batch,
                         cudaStream_t s) {
  const int pairs = (p.Wc + 1) / 2;
  const int warps_x = (pairs + 29) / 30;
  dim3 grid((warps_x + 3) / 4, p.Hc, batch);
#define FLLF_APPLY(L0, HD, MP) k_apply<L0, HD, MP><<<grid, 128, 0, s>>>(p)
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
