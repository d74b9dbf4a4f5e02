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
//              Layout: CTA = 4 warps = 4 coarse rows x 30 coarse column
//              pairs; thread owns a 2x4 block of fine pixels.  Per order k the
//              CTA's 6 coarse rows (and 8 fine rows for l >= 1) of Z are staged
//              into shared memory by TMA bulk copies (cp.async.bulk + mbarrier,
//              4-stage ring, issued by one thread) -- the Z planes carry halo
//              columns so every copy is a whole aligned row segment; threads
//              read their values with LDS.128 and coarse neighbours come from
//              warp shuffles.
//
// No tensor cores: this is a stencil + elementwise path (no contraction).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>
#include <algorithm>
#include <atomic>

#include "fllf_internal.h"
#include "fllf_ptx.h"

namespace fllf {
namespace {

#include "fllf_dev.h"  // device helpers shared with fllf_fused.cu


// ----------------------------------------------------------------- build
// One warp = 30 coarse output columns x a strip of R output rows, for NC
// complex channels (orders kbase + k0 .. + NC-1, exactly NC: the launcher
// picks NC dividing the local order count) and NR real channels (1: G_l[I];
// 2: the sigma / m maps).  EDGE = false: all 64 fine columns of the warp lie
// inside the row, no index mapping; EDGE = true: reflect-101 per column.
template <int NC, int NR, bool FROM_IMAGE, bool EDGE, bool ZFIRST>
struct BuildWarp {
  static constexpr int NCX = NC > 0 ? NC : 1;
  static constexpr int NCL = FROM_IMAGE ? 1 : NCX;  // complex values loaded per row

  struct Row {
    float2 r[NR];
    float2 c[NCL][2];
  };
  struct Pair {
    Row e, o;
  };

  const BuildParams& P;
  int o0, x, c0, rc0, rc1, g0;
  bool store_lane, halo_l, halo_r, do_real;
  int hoff_r;  // offset (float2) from column x to the right halo column Wc
  const float* rsrc[NR];
  float* rdst[NR];
  long long rpitch;
  const float2* zsrc;
  float2* zdst;
  // two accumulators per channel and column half (see vstep_fixed)
  float2 Pc[NCX][2], Ac[NCX][2];
  float2 Pr[NR], Ar[NR];

  __device__ __forceinline__ BuildWarp(const BuildParams& P_, int cb, int o0_, int chunk, int frame) : P(P_), o0(o0_) {
    const int lane = threadIdx.x & 31;
    x = cb * 30 + lane - 1;
    store_lane = lane >= 1 && lane <= 30 && x < P.Wc;
    c0 = 2 * x;
    rc0 = EDGE ? refl101(c0, P.Wf) : c0;
    rc1 = EDGE ? refl101(c0 + 1, P.Wf) : c0 + 1;
    const int k0 = chunk * NC;
    g0 = P.kbase + k0;  // global order of this chunk's first channel
    do_real = (chunk == 0);
    // halo columns of the destination Z planes (see ZHALO): col -1 := x_1,
    // col Wc := x_{Wc-1} (Wf even) or x_{Wc-2} (Wf odd)
    // (both can hold for one lane when Wc = 3)
    // (only edge warps can hold them: interior warps start at fine column >= 58
    // and end before the last fine column, so the stores compile out there)
    halo_l = EDGE && store_lane && x == 1;
    halo_r = EDGE && store_lane && x == ((P.Wf & 1) ? P.Wc - 2 : P.Wc - 1);
    hoff_r = P.Wc - x;
    if (FROM_IMAGE) {
      rsrc[0] = P.img.p + frame * P.img.fstride;
      if (NR > 1) rsrc[NR - 1] = P.img2.p + frame * P.img2.fstride;
      rpitch = P.img.pitch;
    } else {
      if (P.maps) {
        rsrc[0] = P.src.MS + frame * P.ms_stride_src;
        if (NR > 1) rsrc[NR - 1] = P.src.MM + frame * P.ms_stride_src;
      } else {
        rsrc[0] = P.src.G + frame * P.src.fstride_r;
      }
      rpitch = P.src.pitch;
    }
    if (P.maps) {
      rdst[0] = P.dst.MS + frame * P.ms_stride_dst;
      if (NR > 1) rdst[NR - 1] = P.dst.MM + frame * P.ms_stride_dst;
    } else {
      rdst[0] = P.dst.G + frame * P.dst.fstride_r;
    }
    zsrc = nullptr;
    zdst = nullptr;
    if (NC > 0) {
      if (!FROM_IMAGE) zsrc = P.src.Z + frame * P.src.fstride_z + (long long)k0 * P.src.kstride_z;
      zdst = P.dst.Z + frame * P.dst.fstride_z + (long long)k0 * P.dst.kstride_z;
    }
#pragma unroll
    for (int i = 0; i < NCX; ++i) Pc[i][0] = Pc[i][1] = Ac[i][0] = Ac[i][1] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < NR; ++i) Pr[i] = Ar[i] = make_float2(0.f, 0.f);
  }

  __device__ __forceinline__ void load_row(int row, Row& d) const {
    const int rr = min(max(refl101(row, P.Hf), P.fr_lo), P.fr_hi);
    // real rows only for the warps that filter them (chunk 0; every map-build warp)
    if (do_real || FROM_IMAGE || NC == 0) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const float* rp = rsrc[i] + (long long)rr * rpitch;
        d.r[i] = EDGE ? make_float2(__ldg(rp + rc0), __ldg(rp + rc1)) : ldg2(rp + c0);
      }
    }
    if (!FROM_IMAGE && NC > 0) {
      const float2* q = zsrc + (long long)rr * P.src.zpitch;
      const long long ks = P.src.kstride_z;
#pragma unroll
      for (int i = 0; i < NCX; ++i, q += ks) {
        if (EDGE) {
          d.c[i][0] = __ldg(q + rc0);
          d.c[i][1] = __ldg(q + rc1);
        } else {
          const float4 v = ldg4(q + c0);
          d.c[i][0] = lo2(v);
          d.c[i][1] = hi2(v);
        }
      }
    }
  }
  // pair p holds rows 2(o0+p-1), 2(o0+p-1)+1 (p = 0: the two halo rows above)
  __device__ __forceinline__ void load_pair(int p, Pair& d) const {
    const int r0 = 2 * (o0 + p - 1);
    load_row(r0, d.e);
    load_row(r0 + 1, d.o);
  }

  // One channel over a row pair.
  template <bool EMIT, bool ONLY>
  __device__ __forceinline__ void chan(float2 (&Pv)[2], float2 (&Av)[2], float2 ea_, float2 eb_, float2 oa,
                                       float2 ob, float2* q) {
    if (EMIT) {
      const float2 ea = pfma(bc(W2), ea_, Pv[0]);
      const float2 eb = pfma(bc(W2), eb_, Pv[1]);
      const float2 h = hfilt_c(ea, eb);
      if (store_lane) {
        FLLF_DBG_STORE(P, q, 8);
        q[0] = h;
      }
      if (halo_l) {
        FLLF_DBG_STORE(P, q - 2, 8);
        q[-2] = h;  // x == 1: column -1
      }
      if (halo_r) {
        FLLF_DBG_STORE(P, q + hoff_r, 8);
        q[hoff_r] = h;
      }
    }
    if (!ONLY) {
      vstep_fixed(Pv[0], Av[0], ea_, oa);
      vstep_fixed(Pv[1], Av[1], eb_, ob);
    }
  }

  // One row pair.  EMIT: finish output row `emit` with the even row and
  // store it; ONLY: the final row (no accumulator update).
  template <bool EMIT, bool ONLY>
  __device__ __forceinline__ void proc(const Pair& d, int emit) {
    if (do_real) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        if (EMIT) {
          const float2 e = pfma(bc(W2), d.e.r[i], Pr[i]);
          const float h = hfilt_r(e.x, e.y);
          if (store_lane) {
            FLLF_DBG_STORE(P, rdst[i] + (long long)emit * P.dst.pitch + x, 4);
            rdst[i][(long long)emit * P.dst.pitch + x] = h;
          }
        }
        if (!ONLY) vstep_fixed(Pr[i], Ar[i], d.e.r[i], d.o.r[i]);
      }
    }
    if (NC == 0) return;
    // store pointer of channel 0 at (emit, x); channels advance by kstride
    float2* q = zdst + ((long long)emit * P.dst.zpitch + x);
    const long long ks = P.dst.kstride_z;
    if (FROM_IMAGE) {
      // e^{i k w_1 I} for the 4 pixels (even/odd row x col a/b), (s, c) layout
      float2 zc[4], zp[4];
      float tc[4];
      const float I4[4] = {d.e.r[0].x, d.e.r[0].y, d.o.r[0].x, d.o.r[0].y};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float sn, cs;
        sincos_turns(I4[u], P.invT, &sn, &cs);
        const float2 z1 = make_float2(sn, cs);
        tc[u] = 2.f * cs;
        if (ZFIRST) {
          zp[u] = make_float2(0.f, 1.f);
          zc[u] = z1;
        } else {
          // chunk start: e^{i g0 theta} directly (range-reduced in turns),
          // e^{i (g0-1) theta} = e^{i g0 theta} e^{-i theta}
          float sg, cg;
          sincos_turns_n(I4[u], P.invT, g0, &sg, &cg);
          zc[u] = make_float2(sg, cg);
          zp[u] = make_float2(fmaf(sg, cs, -cg * sn), fmaf(cg, cs, sg * sn));
        }
      }
#pragma unroll
      for (int i = 0; i < NCX; ++i) {
        chan<EMIT, ONLY>(Pc[i], Ac[i], zc[0], zc[1], zc[2], zc[3], q);
        q += ks;
        if (i + 1 < NCX) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 zn = pfma(bc(-1.f), zp[u], pmul(bc(tc[u]), zc[u]));
            zp[u] = zc[u];
            zc[u] = zn;
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < NCX; ++i)
      {
        chan<EMIT, ONLY>(Pc[i], Ac[i], d.e.c[i][0], d.e.c[i][1], d.o.c[i][0], d.o.c[i][1], q);
        q += ks;
      }
    }
  }

  // Stream the strip: pairs 0 (halo rows) .. R and the final row (even row of
  // pair R+1).  ROTATE: one pair per iteration with a two-buffer rotation
  // (small loop body; the rotation copies only the prefetched row data, cheap
  // at level 0).  Otherwise two pairs per iteration with static buffers.
  template <bool ROTATE>
  __device__ __forceinline__ void run(int R) {
    if (ROTATE) {
      Pair cur, nxt;
      load_pair(0, cur);
      load_pair(1, nxt);
      proc<false, false>(cur, 0);  // p = 0: halo rows
      cur = nxt;
      load_pair(2, nxt);
      proc<false, false>(cur, 0);  // p = 1: first pair, nothing to emit
      cur = nxt;
      load_pair(3, nxt);
#pragma unroll 1
      for (int p = 2; p <= R; ++p) {
        proc<true, false>(cur, o0 + p - 2);
        cur = nxt;
        load_pair(p + 2, nxt);
      }
      proc<true, true>(cur, o0 + R - 1);
    } else {
      Pair BA, BB;
      load_pair(0, BA);
      load_pair(1, BB);
      proc<false, false>(BA, 0);
      load_pair(2, BA);
      proc<false, false>(BB, 0);
      load_pair(3, BB);
      int p = 2;
#pragma unroll 1
      for (; p + 1 <= R; p += 2) {
        proc<true, false>(BA, o0 + p - 2);
        load_pair(p + 2, BA);
        proc<true, false>(BB, o0 + p - 1);
        load_pair(p + 3, BB);
      }
      if (p <= R) {
        proc<true, false>(BA, o0 + p - 2);
        proc<true, true>(BB, o0 + R - 1);
      } else {
        proc<true, true>(BA, o0 + R - 1);
      }
    }
  }

  // Three row pairs in flight (prefetch distance 3 instead of 2): for levels
  // >= 1, whose warps are latency-bound on their row loads (L2 round trips
  // longer than two pairs of compute).  Pair p lives in buffer p % 3.
  __device__ __forceinline__ void run3(int R) {
    Pair B0, B1, B2;
    load_pair(0, B0);
    load_pair(1, B1);
    load_pair(2, B2);
    proc<false, false>(B0, 0);  // p = 0: halo rows
    load_pair(3, B0);
    proc<false, false>(B1, 0);  // p = 1: nothing to emit
    if (R >= 3) load_pair(4, B1);
    int p = 2;
#pragma unroll 1
    for (; p + 2 <= R; p += 3) {
      proc<true, false>(B2, o0 + p - 2);
      if (p + 3 <= R + 1) load_pair(p + 3, B2);
      proc<true, false>(B0, o0 + p - 1);
      if (p + 4 <= R + 1) load_pair(p + 4, B0);
      proc<true, false>(B1, o0 + p);
      if (p + 5 <= R + 1) load_pair(p + 5, B1);
    }
    // pairs p .. R+1 remain (1..3); the last one holds only the final row
    const int rem = R + 2 - p;
    if (rem == 1) {
      proc<true, true>(B2, o0 + R - 1);
    } else if (rem == 2) {
      proc<true, false>(B2, o0 + p - 2);
      proc<true, true>(B0, o0 + R - 1);
    } else {
      proc<true, false>(B2, o0 + p - 2);
      proc<true, false>(B0, o0 + p - 1);
      proc<true, true>(B1, o0 + R - 1);
    }
  }

  // Strips of exactly 2 output rows (tiny levels): every input row is loaded
  // up front, one memory round trip.
  __device__ __forceinline__ void run2() {
    Pair B0, B1, B2, B3;
    load_pair(0, B0);
    load_pair(1, B1);
    load_pair(2, B2);
    load_pair(3, B3);
    proc<false, false>(B0, 0);
    proc<false, false>(B1, 0);
    proc<true, false>(B2, o0);
    proc<true, true>(B3, o0 + 1);
  }
};

template <int NC, int NR, bool FROM_IMAGE, bool SMALL, bool DEEP = false>
__global__ void __launch_bounds__(32) k_build(const BuildParams P) {
  pdl_wait();     // the previous level's planes are complete
  pdl_trigger();  // let the next kernel get scheduled
  const int cb = blockIdx.x;  // one warp per CTA: all control flow is blockIdx-uniform
  if (cb * 30 >= P.Wc) return;
  const int o0 = P.o_begin + blockIdx.y * P.rows_per_strip;
  if (o0 >= P.o_end) return;
  const int R = min(P.rows_per_strip, P.o_end - o0);
  // level 0: chunk-major (CTAs are dispatched in blockIdx order, so resident
  // warps mostly run the same code variant -- instruction-cache locality);
  // above: frame-major (L2 locality of the shared G plane)
  const int nframes = gridDim.z / P.nchunks;
  const int chunk = FROM_IMAGE ? blockIdx.z / nframes : blockIdx.z % P.nchunks;
  const int frame = FROM_IMAGE ? blockIdx.z % nframes : blockIdx.z / P.nchunks;
  // are all 64 fine columns of this warp inside the row (and, for the
  // caller's image, 8-byte aligned)?
  bool interior = (60 * cb - 2 >= 0) && (60 * cb + 61 < P.Wf);
  if (FROM_IMAGE)
    interior = interior && ((reinterpret_cast<uintptr_t>(P.img.p) & 7) == 0) && ((P.img.pitch & 1) == 0) &&
               (NR < 2 || (((reinterpret_cast<uintptr_t>(P.img2.p) & 7) == 0) && P.img2.pitch == P.img.pitch));
  // chunks starting at order 1 need no chunk-start phasor (level 0 only)
  const bool zfirst = !FROM_IMAGE || (P.kbase + chunk * NC == 1);
  if (interior) {
    if (zfirst) {
      BuildWarp<NC, NR, FROM_IMAGE, false, true> w(P, cb, o0, chunk, frame);
      if (SMALL && R == 2) w.run2(); else if (DEEP && R >= 2) w.run3(R); else w.template run<FROM_IMAGE>(R);
    } else {
      BuildWarp<NC, NR, FROM_IMAGE, false, false> w(P, cb, o0, chunk, frame);
      if (SMALL && R == 2) w.run2(); else if (DEEP && R >= 2) w.run3(R); else w.template run<FROM_IMAGE>(R);
    }
  } else {
    if (zfirst) {
      BuildWarp<NC, NR, FROM_IMAGE, true, true> w(P, cb, o0, chunk, frame);
      if (SMALL && R == 2) w.run2(); else if (DEEP && R >= 2) w.run3(R); else w.template run<FROM_IMAGE>(R);
    } else {
      BuildWarp<NC, NR, FROM_IMAGE, true, false> w(P, cb, o0, chunk, frame);
      if (SMALL && R == 2) w.run2(); else if (DEEP && R >= 2) w.run3(R); else w.template run<FROM_IMAGE>(R);
    }
  }
}

// --------------------------------------------------------------- build0 v2
// Level-0 build (steps a2 + a3 from the image): same warp geometry as k_build
// (lane = fine columns 2x, 2x+1 -> coarse column x; 30 outputs per warp;
// vertical 5-tap first over row pairs, horizontal on the finished row with
// warp shuffles), restructured for issue efficiency:
//  * integer binomial weights [1,4,6,4,1] in both passes, the (1/16)^2 folded
//    into the phasor amplitude (complex channels) or one multiply at emit (G);
//  * the order recurrence z_{k+1} = 2 cos(theta) z_k - z_{k-1} is ONE packed
//    FFMA2 per pixel (negated addend);
//  * up to 8 orders per warp (amortises the per-pixel sincos + chunk-start
//    phasor); I rows prefetched PD pairs ahead;
//  * 32-bit in-frame offsets; halo-column stores only in edge warps.
#ifndef FLLF_B0_PIPE
#define FLLF_B0_PIPE 1
#endif
// two-chunk order interleaving (odd / even orders, no chunk-start sincos):
// measured 1-3 % slower at config 5 (1.24-1.27 vs 1.22-1.23 ms), off; A/B knob
#ifndef FLLF_B0_INTERLEAVE
#define FLLF_B0_INTERLEAVE 0
#endif
template <int NC, bool EDGE>
struct Build0Warp {
  const BuildParams& P;
  int o0, x, c0, rc0, rc1;
  bool store_lane, halo_l, halo_r, do_real, zfirst;
  int g0;
  // inter: two chunks over orders 1 .. 2 NC interleaved -- chunk 0 the odd
  // orders, chunk 1 the even ones, each a step-2 recurrence in 2 theta whose
  // start phasors come from the one sincos of theta (no chunk-start sincos)
  bool inter, odd;
  int kst;  // planes between consecutive orders of this chunk
  const float* isrc;
  long long ipitch;
  float* gdst;
  float2* zdst;  // channel 0 of this chunk, frame base
  float2 Pc[NC][2], Ac[NC][2];
  float2 Pr, Ar;

  __device__ __forceinline__ Build0Warp(const BuildParams& P_, int cb, int o0_, int chunk, int frame)
      : P(P_), o0(o0_) {
    const int lane = threadIdx.x & 31;
    x = cb * 30 + lane - 1;
    store_lane = lane >= 1 && lane <= 30 && x < P.Wc;
    c0 = 2 * x;
    rc0 = EDGE ? refl101(c0, P.Wf) : c0;
    rc1 = EDGE ? refl101(c0 + 1, P.Wf) : c0 + 1;
    inter = FLLF_B0_INTERLEAVE && P.kbase == 1 && P.nchunks == 2;
    odd = chunk == 0;
    kst = inter ? 2 : 1;
    g0 = P.kbase + chunk * NC;
    zfirst = g0 == 1;  // chunks starting at order 1 need no chunk-start phasor
    do_real = chunk == 0;
    halo_l = EDGE && store_lane && x == 1;
    halo_r = EDGE && store_lane && x == ((P.Wf & 1) ? P.Wc - 2 : P.Wc - 1);
    isrc = P.img.p + frame * P.img.fstride;
    ipitch = P.img.pitch;
    gdst = P.dst.G + frame * P.dst.fstride_r;
    zdst = P.dst.Z + frame * P.dst.fstride_z + (long long)(inter ? chunk : chunk * NC) * P.dst.kstride_z;
#pragma unroll
    for (int i = 0; i < NC; ++i) Pc[i][0] = Pc[i][1] = Ac[i][0] = Ac[i][1] = make_float2(0.f, 0.f);
    Pr = Ar = make_float2(0.f, 0.f);
  }

  struct Pair {
    float2 e, o;  // even / odd fine row, (col a, col b)
  };
  // I rows are staged through a per-warp shared-memory ring with cp.async:
  // PD row pairs in flight without holding them in registers.
#ifndef FLLF_B0_PD
#define FLLF_B0_PD 8
#endif
  static constexpr int PD = FLLF_B0_PD;
  float2 (*ring)[2][32];
  // issue the copies of pair p (rows 2(o0+p-1), +1; p = 0: the two halo rows above)
  // rows_in: no row of this strip's reads (incl. the prefetch overrun) needs
  // reflection -> the row pointer just advances by two rows per pair
  bool rows_in;
  const float* rowp;  // this lane's column in fine row 2(o0+p-1) of the next pair to issue
  __device__ __forceinline__ void issue_pair(int p) {
    const int lane = threadIdx.x & 31;
    float2* d0 = &ring[p % PD][0][lane];
    float2* d1 = &ring[p % PD][1][lane];
    if (rows_in) {
      if (EDGE) {
        cp_async4(&d0->x, rowp + rc0);
        cp_async4(&d0->y, rowp + rc1);
        cp_async4(&d1->x, rowp + ipitch + rc0);
        cp_async4(&d1->y, rowp + ipitch + rc1);
      } else {
        cp_async8(d0, rowp + c0);
        cp_async8(d1, rowp + ipitch + c0);
      }
      rowp += 2 * ipitch;
    } else {
      const int r0 = 2 * (o0 + p - 1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float* rp = isrc + (long long)min(max(refl101(r0 + h, P.Hf), P.fr_lo), P.fr_hi) * ipitch;
        float2* d = h ? d1 : d0;
        if (EDGE) {
          cp_async4(&d->x, rp + rc0);
          cp_async4(&d->y, rp + rc1);
        } else {
          cp_async8(d, rp + c0);
        }
      }
    }
    cp_async_commit();
  }
  __device__ __forceinline__ Pair read_pair(int p) const {
    const int lane = threadIdx.x & 31;
    Pair d;
    d.e = ring[p % PD][0][lane];
    d.o = ring[p % PD][1][lane];
    return d;
  }

  // horizontal [1,4,6,4,1] + decimation of a finished row (complex), a = col 2x, b = 2x+1
  // (shuffling a partial sum of the left neighbour's taps, as hfilt_c does,
  // saves 2 of 6 shuffles but measured 5 % slower here: the shuffles wait for
  // the FFMA2 that forms it)
  __device__ __forceinline__ static float2 hsum_c(float2 a, float2 b) {
    const float2 La = shfl_up2(a), Lb = shfl_up2(b), Ra = shfl_down2(a);
    return pfma(bc(6.f), a, pfma(bc(4.f), padd(b, Lb), padd(La, Ra)));
  }

  template <bool EMIT, bool ONLY>
  __device__ __forceinline__ void proc(const Pair& d, int emit) {
    if (do_real) {
      // G channel, packed over the two columns
      if (EMIT) {
        const float2 e = padd(Pr, d.e);
        const float a = e.x, b = e.y;
        const float La = __shfl_up_sync(FULL, a, 1), Lb = __shfl_up_sync(FULL, b, 1);
        const float Ra = __shfl_down_sync(FULL, a, 1);
        const float h = fmaf(6.f, a, fmaf(4.f, b + Lb, La + Ra)) * (1.f / 256.f);
        if (store_lane) {
          FLLF_DBG_STORE(P, gdst + emit * P.dst.pitch + x, 4);
          gdst[emit * P.dst.pitch + x] = h;
        }
      }
      if (!ONLY) {
        Pr = pfma(bc(6.f), d.e, pfma(bc(4.f), d.o, Ar));
        Ar = pfma(bc(4.f), d.o, d.e);
      }
    }
    // phasors of the 4 pixels (even/odd row x col a/b), (Im, Re) = (sin, cos),
    // amplitude 1/256 (the binomial normalisation of both passes)
    const float I4[4] = {d.e.x, d.e.y, d.o.x, d.o.y};
    float2 zc[4], zp[4];
    float tc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float sn, cs;
      sincos_turns(I4[u], P.invT, &sn, &cs);
      tc[u] = 2.f * cs;
      if (inter) {  // step 2 theta: z_{k+2} = 2 cos(2 theta) z_k - z_{k-2}
        const float c2 = fmaf(cs, cs, -sn * sn), s2 = 2.f * sn * cs;
        tc[u] = 2.f * c2;
        if (odd) {  // z_1, z_{-1}
          zc[u] = make_float2(sn * (1.f / 256.f), cs * (1.f / 256.f));
          zp[u] = make_float2(-sn * (1.f / 256.f), cs * (1.f / 256.f));
        } else {  // z_2, z_0
          zc[u] = make_float2(s2 * (1.f / 256.f), c2 * (1.f / 256.f));
          zp[u] = make_float2(0.f, 1.f / 256.f);
        }
      } else if (zfirst) {
        zp[u] = make_float2(0.f, 1.f / 256.f);
        zc[u] = make_float2(sn * (1.f / 256.f), cs * (1.f / 256.f));
      } else {
        float sg, cg;
        sincos_turns_n(I4[u], P.invT, g0, &sg, &cg);
        sg *= 1.f / 256.f;
        cg *= 1.f / 256.f;
        zc[u] = make_float2(sg, cg);
        zp[u] = make_float2(fmaf(sg, cs, -cg * sn), fmaf(cg, cs, sg * sn));  // e^{i (g0-1) theta}
      }
    }
    const int off0 = emit * P.dst.zpitch + x;  // in-frame float2 offset of (emit, x), channel 0
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      if (EMIT) {
        const float2 ea = padd(Pc[i][0], zc[0]);
        const float2 eb = padd(Pc[i][1], zc[1]);
        const float2 h = hsum_c(ea, eb);
        float2* q = wide_off(zdst, (unsigned)(off0 + i * kst * (int)P.dst.kstride_z));
        if (store_lane) {
          FLLF_DBG_STORE(P, q, 8);
          stg2(q, h);
        }
        if (EDGE) {
          if (halo_l) {
            FLLF_DBG_STORE(P, q - 2, 8);
            q[-2] = h;  // x == 1: column -1
          }
          if (halo_r) {
            FLLF_DBG_STORE(P, q + (P.Wc - x), 8);
            q[P.Wc - x] = h;
          }
        }
      }
      if (!ONLY) {
        Pc[i][0] = pfma(bc(6.f), zc[0], pfma(bc(4.f), zc[2], Ac[i][0]));
        Pc[i][1] = pfma(bc(6.f), zc[1], pfma(bc(4.f), zc[3], Ac[i][1]));
        Ac[i][0] = pfma(bc(4.f), zc[2], zc[0]);
        Ac[i][1] = pfma(bc(4.f), zc[3], zc[1]);
      }
      if (i + 1 < NC) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2 zn = pfma(bc(tc[u]), zc[u], pneg(zp[u]));
          zp[u] = zc[u];
          zc[u] = zn;
        }
      }
    }
  }

  // Stream the strip: pairs 0 (halo rows) .. R and the final row (even row of
  // pair R+1), PD pairs in flight through the shared-memory ring.
  __device__ __forceinline__ void run(int R) {
    // pairs 0 .. R+1 are read: rows 2(o0-1) .. 2(o0+R)+1 (no copies past the
    // strip: empty commit groups keep the wait counts uniform)
    rows_in = o0 >= 1 && 2 * (o0 - 1) >= P.fr_lo && 2 * (o0 + R) + 1 <= P.fr_hi;
    rowp = isrc + (long long)(2 * (o0 - 1)) * ipitch;
#pragma unroll
    for (int q = 0; q < PD; ++q) {
      if (q <= R + 1) issue_pair(q);
      else cp_async_commit();
    }
    cp_async_wait<PD - 1>();
    proc<false, false>(read_pair(0), 0);
    if (PD <= R + 1) issue_pair(PD); else cp_async_commit();
    cp_async_wait<PD - 1>();
    proc<false, false>(read_pair(1), 0);
    if (PD + 1 <= R + 1) issue_pair(PD + 1); else cp_async_commit();
#if FLLF_B0_PIPE
    // pair p+1 is read from the ring before pair p is processed (the wait is
    // a compiler fence: this keeps the shared-memory load latency off the
    // start of every pair)
    cp_async_wait<PD - 1>();
    Pair d = read_pair(2);
#pragma unroll 1
    for (int p = 2; p <= R; ++p) {
      if (p + PD <= R + 1) issue_pair(p + PD); else cp_async_commit();
      cp_async_wait<PD - 1>();
      const Pair nd = read_pair(p + 1);
      proc<true, false>(d, o0 + p - 2);
      d = nd;
    }
    proc<true, true>(d, o0 + R - 1);
#else
#pragma unroll 1
    for (int p = 2; p <= R; ++p) {
      cp_async_wait<PD - 1>();
      const Pair d = read_pair(p);
      if (p + PD <= R + 1) issue_pair(p + PD); else cp_async_commit();
      proc<true, false>(d, o0 + p - 2);
    }
    cp_async_wait<PD - 1>();
    proc<true, true>(read_pair(R + 1), o0 + R - 1);
#endif
    cp_async_wait<0>();
  }
};

template <int NC>
#ifndef FLLF_B0_MINB
#define FLLF_B0_MINB 16
#endif
__global__ void __launch_bounds__(32, FLLF_B0_MINB) k_build0(const BuildParams P) {
  pdl_trigger();
  const int cb = blockIdx.x;
  if (cb * 30 >= P.Wc) return;
  const int o0 = P.o_begin + blockIdx.y * P.rows_per_strip;
  if (o0 >= P.o_end) return;
  const int R = min(P.rows_per_strip, P.o_end - o0);
  const int nframes = gridDim.z / P.nchunks;
  const int chunk = blockIdx.z / nframes;
  const int frame = blockIdx.z % nframes;
  bool interior = (60 * cb - 2 >= 0) && (60 * cb + 61 < P.Wf);
  interior = interior && ((reinterpret_cast<uintptr_t>(P.img.p) & 7) == 0) && ((P.img.pitch & 1) == 0);
  __shared__ __align__(16) float2 ring[Build0Warp<NC, false>::PD][2][32];
  if (interior) {
    Build0Warp<NC, false> w(P, cb, o0, chunk, frame);
    w.ring = ring;
    w.run(R);
  } else {
    Build0Warp<NC, true> w(P, cb, o0, chunk, frame);
    w.ring = ring;
    w.run(R);
  }
}

// ----------------------------------------------------------------- apply
// TMA ring depth: enough stages in flight to cover the L2/HBM round trip
// (level 0 stages are 3 KB, level >= 1 stages 11 KB)
template <bool LEVEL0>
__host__ __device__ constexpr int apply_stages() {
  return LEVEL0 ? 16 : 6;
}
constexpr int CROW_BYTES = 64 * 8;   // 32 lanes x 2 coarse complex values
constexpr int FROW_BYTES = 128 * 8;  // 32 lanes x 4 fine complex values

template <bool LEVEL0>
__host__ __device__ constexpr int apply_stage_bytes() {
  return 6 * CROW_BYTES + (LEVEL0 ? 0 : 8 * FROW_BYTES);
}

// Persistent, warp-specialised: a CTA loops over tiles (4 coarse rows x 30
// coarse column pairs of one frame); warps 0..3 compute (one coarse row each),
// warp 4 is the TMA producer that streams (tile, order) stages through the
// shared-memory ring ahead of the consumers -- across tile boundaries, so the
// start-up latency of a tile is hidden behind the previous one.
struct ApplyTile {
  int jb, r0, frame;
};
__device__ __forceinline__ ApplyTile apply_tile(int t, const ApplyParams& P) {
  const int nx = (P.Wf + 119) / 120, ny = (P.r_end - P.r_begin + 3) / 4;
  ApplyTile T;
  T.jb = t % nx;
  t /= nx;
  T.r0 = P.r_begin + (t % ny) * 4;
  T.frame = t / ny;
  return T;
}

// Tile sequence t = blockIdx.x, blockIdx.x + gridDim.x, ... decomposed
// incrementally (no divisions per tile).
struct TileIter {
  int nx, ny, dj, dr, df;
  ApplyTile T;
  __device__ __forceinline__ TileIter(const ApplyParams& P) {
    nx = (P.Wf + 119) / 120;
    ny = (P.r_end - P.r_begin + 3) / 4;
    rb0 = P.r_begin;
    const int q = gridDim.x / nx;
    dj = gridDim.x - q * nx;
    dr = q % ny;
    df = q / ny;
    T = apply_tile(blockIdx.x, P);
    T.r0 = (T.r0 - rb0) >> 2;  // row block index while iterating
  }
  int rb0;
  __device__ __forceinline__ ApplyTile tile() const {
    ApplyTile u = T;
    u.r0 = rb0 + u.r0 * 4;
    return u;
  }
  __device__ __forceinline__ void next() {
    T.jb += dj;
    int c = T.jb >= nx;
    T.jb -= c ? nx : 0;
    T.r0 += dr + c;
    c = T.r0 >= ny;
    T.r0 -= c ? ny : 0;
    T.frame += df + c;
  }
};

template <bool LEVEL0, bool HAS_D, bool MAPS>
__global__ void __launch_bounds__(160, MAPS ? 2 : 3) k_apply(const ApplyParams P, const int ntiles) {
  constexpr int S = apply_stages<LEVEL0>();
  constexpr int STAGE = apply_stage_bytes<LEVEL0>();
  constexpr int FOFF = 6 * CROW_BYTES;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t empty[S];

  // PDL: the Z / G planes of the build pass are complete once the first apply
  // of the sequence has waited; only D_{l+1} (previous apply) needs a wait,
  // taken right before it is first read.
  if (P.wait_first) pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int KL = P.KL;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 4) {
    // ---- producer: one lane issues, per (tile, order k), 6 coarse row
    // segments of Z_{l+1,k} (coarse cols 2j0 .. 2j0+63, j0 = 30 jb - 1) and,
    // for l >= 1, 8 fine row segments of Z_{l,k} (fine cols 4j0 .. 4j0+127)
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const ApplyTile T = apply_tile(t, P);
        const float2* zc0 = P.coarse.Z + T.frame * P.coarse.fstride_z + (60 * T.jb - 2);
        const float2* zf0 = LEVEL0 ? nullptr : P.fine.Z + T.frame * P.fine.fstride_z + (120 * T.jb - 4);
        for (int k = 0; k < KL; ++k, ++it) {
          const int s = it % S;
          if (it >= S) mbar_wait_parity(&empty[s], ((it / S) - 1) & 1);
          unsigned char* st = smem + s * STAGE;
          mbar_arrive_expect_tx(&full[s], STAGE);
          const float2* zc = zc0 + (long long)k * P.coarse.kstride_z;
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const int cr = upmap(T.r0 - 1 + q, P.Hc, P.Hf);
            tma_load_1d(st + q * CROW_BYTES, zc + (long long)cr * P.coarse.zpitch, CROW_BYTES, &full[s]);
          }
          if (!LEVEL0) {
            const float2* zf = zf0 + (long long)k * P.fine.kstride_z;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int fr = min(2 * T.r0 + q, P.Hf - 1);
              tma_load_1d(st + FOFF + q * FROW_BYTES, zf + (long long)fr * P.fine.zpitch, FROW_BYTES, &full[s]);
            }
          }
        }
      }
    }
    return;
  }

  // ---- consumers
  const bool img_al = ((reinterpret_cast<uintptr_t>(P.img.p) & 15) == 0) && ((P.img.pitch & 3) == 0);
  const bool out_al = ((reinterpret_cast<uintptr_t>(P.out) & 15) == 0) && ((P.out_pitch & 3) == 0);
  // g = I (level 0) or G_l at the thread's 2x4 fine pixels of tile T
  auto load_g = [&](const ApplyTile& T, float (&g)[8]) {
    const int r = min(T.r0 + warp, P.Hc - 1);
    const int j = T.jb * 30 + lane - 1;
    const int xf0 = 4 * j;
    const bool fvec_ok = xf0 >= 0 && xf0 + 3 < P.Wf;
    const float* base;
    long long pitch;
    bool al;
    if (LEVEL0) {
      base = P.img.p + T.frame * P.img.fstride;
      pitch = P.img.pitch;
      al = img_al;
    } else {
      base = P.fine.G + T.frame * P.fine.fstride_r;
      pitch = P.fine.pitch;
      al = true;
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const float* rp = base + (long long)min(2 * r + t, P.Hf - 1) * pitch;
      if (fvec_ok && al) {
        const float4 v = ldg4(rp + xf0);
        g[4 * t + 0] = v.x; g[4 * t + 1] = v.y; g[4 * t + 2] = v.z; g[4 * t + 3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) g[4 * t + q] = __ldg(rp + min(max(xf0 + q, 0), P.Wf - 1));
      }
    }
  };
  // coarse D_{l+1} at rows r-1..r+1, columns 2j, 2j+1 (polyphase border rule)
  auto load_d = [&](const ApplyTile& T, float (&dq)[3][2]) {
    const int r = T.r0 + warp;
    const int j = T.jb * 30 + lane - 1;
    const int cr[3] = {upmap(r - 1, P.Hc, P.Hf), min(r, P.Hc - 1), upmap(r + 1, P.Hc, P.Hf)};
    const bool cvec = (2 * j >= 0) && (2 * j + 1 < P.Wc);
    const int cc0 = upmap(2 * j, P.Wc, P.Wf), cc1 = upmap(2 * j + 1, P.Wc, P.Wf);
    const float* dc = P.coarse.D + T.frame * P.coarse.fstride_r;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const float* rp = dc + (long long)cr[t] * P.coarse.pitch;
      if (cvec) {
        const float2 q = ldg2(rp + 2 * j);
        dq[t][0] = q.x;
        dq[t][1] = q.y;
      } else {
        dq[t][0] = __ldg(rp + cc0);
        dq[t][1] = __ldg(rp + cc1);
      }
    }
  };

  bool waited = P.wait_first != 0;  // D_{l+1} is readable once the PDL wait returned
  int it = 0;
#pragma unroll 1
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const ApplyTile T = apply_tile(t, P);
    const int r = T.r0 + warp;
    const int j = T.jb * 30 + lane - 1;  // coarse columns 2j, 2j+1 -> fine columns 4j..4j+3
    const bool act = r < P.Hc && lane >= 1 && lane <= 30 && 4 * j < P.Wf;
    float g[8];
    load_g(T, g);
    float dq[3][2];
    if (HAS_D && waited) load_d(T, dq);

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
      const int xf0 = 4 * j;
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const long long off = (long long)min(2 * r + tt, P.Hf - 1) * mp + min(max(xf0 + q, 0), P.Wf - 1);
          const float sg = __ldg(sptr + off), m = __ldg(mptr + off);
          const float beta = P.hq * sg * sg;
          const int p = 4 * tt + q;
          const float kb = (float)P.kbase;
          // a_k = m sigma^3 c0 k exp(-k^2 beta), carried with R = exp(-(2k+1) beta), Q = exp(-2 beta)
          mA[p] = m * sg * sg * sg * P.c0 * kb * __expf(-kb * kb * beta);
          mR[p] = __expf(-(2.f * kb + 1.f) * beta);
          mQ[p] = __expf(-2.f * beta);
        }
      }
    }
    // Chebyshev state per pixel, (c, s) layout: z = e^{i k w_1 g}, zp = e^{i (k-1) w_1 g}
    float2 z[8], zp[8], acc[8];
    float tc[8];
    const int g0 = P.kbase;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      float sn, cs;
      sincos_turns(g[p], P.invT, &sn, &cs);
      const float2 z1 = make_float2(cs, sn);
      tc[p] = 2.f * cs;
      if (g0 == 1) {
        zp[p] = make_float2(1.f, 0.f);
        z[p] = z1;
      } else {
        float sg, cg;
        sincos_turns_n(g[p], P.invT, g0, &sg, &cg);
        z[p] = make_float2(cg, sg);
        zp[p] = make_float2(fmaf(cg, cs, sg * sn), fmaf(sg, cs, -cg * sn));
      }
      acc[p] = make_float2(0.f, 0.f);
    }

    // ---- order loop (unrolled by 2 so the recurrence state rotates without moves)
#pragma unroll 2
    for (int k = 0; k < KL; ++k, ++it) {
      const int s = it % S;
      mbar_wait_parity(&full[s], (it / S) & 1);
      const unsigned char* st = smem + s * STAGE;
      float2 h[3][4];
#pragma unroll
      for (int tt = 0; tt < 3; ++tt) {
        const float4 qv = *reinterpret_cast<const float4*>(st + (warp + tt) * CROW_BYTES + lane * 16);
        const float2 x0 = lo2(qv), x1 = hi2(qv);
        const float2 L = shfl_up2(x1), Rn = shfl_down2(x0);
        // horizontal polyphase (unscaled): even fine col x_{c-1} + 6 x_c + x_{c+1} (/8), odd x_c + x_{c+1} (/2)
        h[tt][0] = pfma(bc(6.f), x0, padd(L, x1));
        h[tt][1] = padd(x0, x1);
        h[tt][2] = pfma(bc(6.f), x1, padd(x0, Rn));
        h[tt][3] = padd(x1, Rn);
      }
      float4 fz[4];
      if (!LEVEL0) {
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          const unsigned char* fr = st + FOFF + (2 * warp + tt) * FROW_BYTES + lane * 32;
          fz[2 * tt] = *reinterpret_cast<const float4*>(fr);
          fz[2 * tt + 1] = *reinterpret_cast<const float4*>(fr + 16);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // this warp has read slot s
      float2 waa, w1, w2, w3;
      if (MAPS) {
        waa = bc(1.f); w1 = bc(-1.f / 64.f); w2 = bc(-1.f / 16.f); w3 = bc(-1.f / 4.f);
      } else {
        waa = P.wk[k][0]; w1 = P.wk[k][1]; w2 = P.wk[k][2]; w3 = P.wk[k][3];
      }
      const float kk = (float)(P.kbase + k);
      const float kratio = (kk + 1.f) / kk;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // vertical: even fine row (h[-1] + 6 h[0] + h[+1]) (/8); odd (h[0] + h[+1]) (/2)
        const float2 re = pfma(bc(6.f), h[1][q], padd(h[0][q], h[2][q]));
        const float2 ro = padd(h[1][q], h[2][q]);
        const float2 we = (q & 1) ? w2 : w1;  // even row: ee 1/64, eo 1/16
        const float2 wo = (q & 1) ? w3 : w2;  // odd row:  oe 1/16, oo 1/4
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          const int p = 4 * tt + q;
          const float2 raw = tt == 0 ? re : ro;
          const float2 w = tt == 0 ? we : wo;
          float2 V;  // (Im, Re) of a_k (Z_l - up Z_{l+1}) at this pixel
          float2 zf = make_float2(0.f, 0.f);
          if (!LEVEL0) {
            const float4 fv = fz[2 * tt + (q >> 1)];
            zf = (q & 1) ? hi2(fv) : lo2(fv);
          }
          if (MAPS) {
            V = pmul(bc(mA[p]), LEVEL0 ? pmul(w, raw) : pfma(w, raw, zf));
          } else {
            V = LEVEL0 ? pmul(w, raw) : pfma(w, raw, pmul(waa, zf));
          }
          // acc += (c V.im, s V.re); result = acc.x - acc.y = a_k Im(e^{-i k w_1 g} (...))
          acc[p] = pfma(z[p], V, acc[p]);
          const float2 zn = pfma(bc(-1.f), zp[p], pmul(bc(tc[p]), z[p]));
          zp[p] = z[p];
          z[p] = zn;
          if (MAPS) {
            mA[p] *= mR[p] * kratio;
            mR[p] *= mQ[p];
          }
        }
      }
    }

    float res[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) res[p] = acc[p].x - acc[p].y;

    // --- collapse: + up(D_{l+1}) (written by the previous apply grid)
    if (HAS_D) {
      if (!waited) {
        pdl_wait();
        waited = true;
        load_d(T, dq);
      }
      float hd[3][4];
#pragma unroll
      for (int tt = 0; tt < 3; ++tt) {
        const float x0 = dq[tt][0], x1 = dq[tt][1];
        const float L = __shfl_up_sync(FULL, x1, 1);
        const float Rn = __shfl_down_sync(FULL, x0, 1);
        hd[tt][0] = fmaf(6.f, x0, L + x1) * 0.125f;
        hd[tt][1] = (x0 + x1) * 0.5f;
        hd[tt][2] = fmaf(6.f, x1, x0 + Rn) * 0.125f;
        hd[tt][3] = (x1 + Rn) * 0.5f;
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

    if (act) {
      const int xf0 = 4 * j;
      const bool fvec_ok = xf0 + 3 < P.Wf;
      float* op;
      long long opitch;
      bool oal;
      if (LEVEL0) {
        op = P.out + T.frame * P.out_fstride;
        opitch = P.out_pitch;
        oal = out_al;
      } else {
        op = P.fine.D + T.frame * P.fine.fstride_r;
        opitch = P.fine.pitch;
        oal = true;
      }
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        if (2 * r + tt >= P.Hf) break;
        float* rp = op + (long long)(2 * r + tt) * opitch;
        if (fvec_ok && oal) {
          FLLF_DBG_STORE(P, rp + xf0, 16);
          *reinterpret_cast<float4*>(rp + xf0) =
              make_float4(res[4 * tt], res[4 * tt + 1], res[4 * tt + 2], res[4 * tt + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (xf0 + q < P.Wf) {
              FLLF_DBG_STORE(P, rp + xf0 + q, 4);
              rp[xf0 + q] = res[4 * tt + q];
            }
        }
      }
    }
  }
}

// --------------------------------------------------------- apply (Clenshaw)
// Uniform coefficients (SCALAR / COEFFS).  Same tiles and warp roles as
// k_apply, but the producer streams the orders in DESCENDING k and the
// consumers evaluate the order sum with Clenshaw's recurrence instead of
// carrying the phasors e^{i k theta} forward: with c_k = (c_cos, c_sin) the
// per-order coefficient pair of a pixel,
//   b_k = c_k + 2 cos(theta) b_{k+1} - b_{k+2},   b_{k1+1} = b_{k1+2} = 0,
//   sum_{k=k0}^{k1} (c_cos,k cos k theta + c_sin,k sin k theta)
//     = b_{k0} . (cos k0 theta, sin k0 theta) - b_{k0+1} . (cos (k0-1) theta, sin (k0-1) theta)
// (cos k theta and sin k theta both satisfy phi_{k+1} = 2 cos theta phi_k - phi_{k-1}).
// Per pixel and order that is two packed FFMA2 (one with a negated addend) at
// level 0, three at l >= 1 (same-level Z term), instead of the phasor update
// plus accumulate.  The up-sampling is done vertically first: per coarse
// column the even fine row takes (x_{r-1} + 6 x_r + x_{r+1}), the odd one
// (x_r + x_{r+1}); the horizontal polyphase step then needs only the two
// neighbour columns of those two values (4 complex shuffles per order).
// The polyphase scales 1/64, 1/16, 1/4 and the sign pattern of
// Im(e^{-i k theta} V) = cos k theta V_im - sin k theta V_re are folded into
// P.cw (see ApplyParams).
//
// Tile header (double-buffered, staged by the producer like the order stages):
// the 8 fine rows of g (I at level 0, G_l above; 120 fine columns from 120 jb)
// and the 6 coarse rows of D_{l+1} (68 columns from 60 jb - 4, 16-byte
// aligned; the up-sampling border rule is applied when the consumers index it).
constexpr int HDR_G_ROW = 480;
constexpr int HDR_D_ROW = 272;
constexpr int HDR_D_OFF = 8 * HDR_G_ROW;
constexpr int HDR_BYTES = 5504;  // 8*480 + 6*272 = 5472, rounded to 128
static_assert(HDR_D_OFF + 6 * HDR_D_ROW <= HDR_BYTES, "tile header layout");
// MAPS mode: the header also carries the 8 fine rows of the sigma_r and m maps
// (their Gaussian pyramids at l >= 1, reading R7)
constexpr int HDR_S_OFF = HDR_BYTES;
constexpr int HDR_M_OFF = HDR_S_OFF + 8 * HDR_G_ROW;
template <bool MAPS>
__host__ __device__ constexpr int hdr_bytes() {
  return MAPS ? HDR_M_OFF + 8 * HDR_G_ROW : HDR_BYTES;  // 13184 = 103 x 128
}

// Orders per ring stage (level 0: two, which halves the barrier and index
// bookkeeping per order) and ring depth.
template <bool LEVEL0>
__host__ __device__ constexpr int apply_cl_ops() {
  return LEVEL0 ? 2 : 1;
}
// resident CTAs per SM (launch bounds).  A fourth level-0 CTA (96 registers,
// a few spilled, 6 stages) measured slower on B200 (config 2 apply0 20.8 ->
// 22.0 us), so 3.
#ifndef FLLF_APPLY0_CTAS
#define FLLF_APPLY0_CTAS 3
#endif
#ifndef FLLF_MAPS1_CTAS
#define FLLF_MAPS1_CTAS 3
#endif
template <bool LEVEL0, bool MAPS = false>
__host__ __device__ constexpr int apply_cl_ctas() {
  return LEVEL0 ? FLLF_APPLY0_CTAS : (MAPS ? FLLF_MAPS1_CTAS : 3);
}
// level-0 order loop unrolled over two ring stages (4 orders): the Clenshaw
// accumulator roles then repeat without register moves (61.8 instead of
// 66.5 instructions per order and warp)
#ifndef FLLF_A0_UNROLL
#define FLLF_A0_UNROLL 2
#endif
constexpr int kApply0Unroll = FLLF_A0_UNROLL;
#ifndef FLLF_A1_UNROLL
#define FLLF_A1_UNROLL 1
#endif
constexpr int kApply1Unroll = FLLF_A1_UNROLL;  // levels >= 1 (A/B knob)
// K-specialised level-0 order loop software-pipelined across ring stages (A/B knob)
#ifndef FLLF_APPLY_PIPE
#define FLLF_APPLY_PIPE 1
#endif
constexpr bool kApplyPipe = FLLF_APPLY_PIPE != 0;
#ifndef FLLF_APPLY_PIPE_MAPS
#define FLLF_APPLY_PIPE_MAPS 0
#endif
constexpr bool kApplyPipeMaps = FLLF_APPLY_PIPE_MAPS != 0;
// KT > 0 (level 0): a whole tile's orders in a ring of K/2 stages when that
// is 6..8 (the ring then restarts at the same stage every tile)
template <bool LEVEL0, bool MAPS = false, int KT = 0>
__host__ __device__ constexpr int apply_cl_stages() {
  return (LEVEL0 && KT == 12) ? 6
                              : (LEVEL0 ? (FLLF_APPLY0_CTAS >= 4 ? 6 : 8) : (MAPS ? (FLLF_MAPS1_CTAS <= 2 ? 6 : 4) : 5));
}
template <bool LEVEL0, bool MAPS = false, int KT = 0>
__host__ __device__ constexpr int apply_cl_smem() {
  return apply_cl_stages<LEVEL0, MAPS, KT>() * apply_cl_ops<LEVEL0>() * apply_stage_bytes<LEVEL0>() + 2 * hdr_bytes<MAPS>();
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// KT > 0: the plan's order count as a compile-time constant (level 0, SCALAR /
// COEFFS, K = 8 or 16): the order loop unrolls completely, every coefficient
// pair is an immediate constant-bank operand and the ring stages of a tile
// are compile-time offsets from the tile's first stage (a tile uses K/2 of the
// 8 stages, so it never wraps inside a tile).
template <bool LEVEL0, bool HAS_D, bool MAPS, int KT = 0>
__global__ void __launch_bounds__(160, apply_cl_ctas<LEVEL0, MAPS>()) k_apply_cl(const __grid_constant__ ApplyParams P, const int ntiles) {
  constexpr int S = apply_cl_stages<LEVEL0, MAPS, KT>();
  constexpr int HB = hdr_bytes<MAPS>();
  constexpr int OPS = apply_cl_ops<LEVEL0>();
  constexpr int OBYTES = apply_stage_bytes<LEVEL0>();  // one order
  constexpr int STAGE = OPS * OBYTES;
  constexpr int FOFF = 6 * CROW_BYTES;
  constexpr int HOFF = S * STAGE;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t empty[S];
  __shared__ __align__(8) uint64_t gfull[2], dfull[2], hempty[2], mfull[2];

  if (P.wait_first) pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int KL = KT > 0 ? KT : P.KL;
  // g rows by TMA: internal planes always; the caller's image when its rows
  // are 16-byte aligned and W is a multiple of 4 (copies never leave a row)
  const bool tma_g = !LEVEL0 || (((reinterpret_cast<uintptr_t>(P.img.p) & 15) == 0) &&
                                 ((P.img.pitch & 3) == 0) && ((P.Wf & 3) == 0));

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      mbar_init(&gfull[b], 1);
      mbar_init(&dfull[b], 1);
      mbar_init(&mfull[b], 1);
      mbar_init(&hempty[b], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 4) {
    // ---- producer (whole warp, uniform control flow; one elected lane
    // issues).  Per tile: g rows, the order stages k = KL-1 .. 0 (6 coarse row
    // segments of Z_{l+1,k} + 8 fine row segments of Z_{l,k}), then the D rows
    // (after the PDL wait: D_{l+1} is the previous grid's output).
    int s = 0;
    uint32_t ph = 0;
    int n = 0, nt = 0;
    bool waited = P.wait_first != 0;
    TileIter it(P);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt, it.next()) {
      const ApplyTile T = it.tile();
      const int hb = nt & 1;
      unsigned char* hdr = smem + HOFF + hb * HB;
      if (nt >= 2) mbar_wait_parity(&hempty[hb], ((nt >> 1) & 1) ^ 1u);
      // interior tiles: the 8 fine g rows / 6 coarse D rows are contiguous -> one tensor copy each
      // (only when the consumers take g from the header: tma_g; else they load it themselves)
      const bool tmg = tma_g && P.use_tm_g && 2 * T.r0 + 7 <= min(P.Hf - 1, P.fr_hi);
      if (tmg) {
        if (elect_one()) {
          mbar_arrive_expect_tx(&gfull[hb], 8 * HDR_G_ROW);
          tma_load_3d(hdr, &P.tm_g, 120 * T.jb, 2 * T.r0 - P.fr_lo, T.frame * P.gz, &gfull[hb]);
        }
        __syncwarp();
      } else if (tma_g) {
        const float* gb;
        long long gp;
        int wlim;
        if (LEVEL0) {
          gb = P.img.p + T.frame * P.gz * P.img.fstride;
          gp = P.img.pitch;
          wlim = P.Wf;
        } else {
          gb = P.fine.G + T.frame * P.gz * P.fine.fstride_r;
          gp = P.fine.pitch;
          wlim = P.fine.pitch;
        }
        const uint32_t gbytes = (uint32_t)min(HDR_G_ROW, (wlim - 120 * T.jb) * 4);
        if (elect_one()) {
          mbar_arrive_expect_tx(&gfull[hb], 8 * gbytes);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            tma_load_1d(hdr + q * HDR_G_ROW, gb + (long long)min(2 * T.r0 + q, P.fr_hi) * gp + 120 * T.jb, gbytes,
                        &gfull[hb]);
        }
        __syncwarp();
      }
      if (MAPS) {  // sigma_r / m rows (full frame; 16-byte aligned rows, checked by the host)
        const float* sb;
        const float* mb;
        long long mp;
        int wlim;
        if (LEVEL0) {
          sb = P.smap.p + T.frame * P.smap.fstride;
          mb = P.mmap.p + T.frame * P.mmap.fstride;
          mp = P.smap.pitch;
          wlim = P.Wf;
        } else {
          sb = P.fine.MS + T.frame * P.ms_fstride;
          mb = P.fine.MM + T.frame * P.ms_fstride;
          mp = P.fine.pitch;
          wlim = P.fine.pitch;
        }
        const uint32_t mbytes = (uint32_t)min(HDR_G_ROW, (wlim - 120 * T.jb) * 4);
        if (elect_one()) {
          mbar_arrive_expect_tx(&mfull[hb], 16 * mbytes);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const long long ro = (long long)min(2 * T.r0 + q, P.Hf - 1) * mp + 120 * T.jb;
            tma_load_1d(hdr + HDR_S_OFF + q * HDR_G_ROW, sb + ro, mbytes, &mfull[hb]);
            tma_load_1d(hdr + HDR_M_OFF + q * HDR_G_ROW, mb + ro, mbytes, &mfull[hb]);
          }
        }
        __syncwarp();
      }
      const int zfr = T.frame * P.zz;
      const float2* zc0 = P.coarse.Z + zfr * P.coarse.fstride_z + (60 * T.jb - 2);
      int crow[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) crow[q] = min(max(upmap(T.r0 - 1 + q, P.Hc, P.Hf), P.cr_lo), P.cr_hi);
      const float2* zf0 = LEVEL0 ? nullptr : P.fine.Z + zfr * P.fine.fstride_z + (120 * T.jb - 4);
      // interior tiles: the 6 coarse (8 fine) rows are contiguous -> one tensor copy per order
      const bool tmc = P.use_tm && T.r0 >= 1 && T.r0 - 1 >= P.cr_lo && T.r0 + 4 <= min(P.Hc - 1, P.cr_hi);
      const bool tmf = !LEVEL0 && P.use_tm && 2 * T.r0 + 7 <= min(P.Hf - 1, P.fr_hi);
      const int xc = 2 * (ZHALO + 60 * T.jb - 2), xf = 2 * (ZHALO + 120 * T.jb - 4);  // float columns
#pragma unroll 1
      for (int i = KL - 1; i >= 0; i -= OPS) {
        if (n >= S) mbar_wait_parity(&empty[s], ph ^ 1u);
        unsigned char* st = smem + s * STAGE;
        const int no = min(OPS, i + 1);  // orders in this stage: i, i-1, ...
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[s], no * OBYTES);
#pragma unroll
          for (int h = 0; h < OPS; ++h) {
            if (h < no) {
              unsigned char* so = st + h * OBYTES;
              if (tmc) {
                tma_load_3d(so, &P.tm_coarse, xc, T.r0 - 1 - P.cr_lo, zfr * KL + i - h, &full[s]);
              } else {
                const float2* zc = zc0 + (long long)(i - h) * P.coarse.kstride_z;
#pragma unroll
                for (int q = 0; q < 6; ++q)
                  tma_load_1d(so + q * CROW_BYTES, zc + (long long)crow[q] * P.coarse.zpitch, CROW_BYTES, &full[s]);
              }
              if (!LEVEL0) {
                if (tmf) {
                  tma_load_3d(so + FOFF, &P.tm_fine, xf, 2 * T.r0 - P.fr_lo, zfr * KL + i - h, &full[s]);
                } else {
                  const float2* zf = zf0 + (long long)(i - h) * P.fine.kstride_z;
#pragma unroll
                  for (int q = 0; q < 8; ++q)
                    tma_load_1d(so + FOFF + q * FROW_BYTES,
                                zf + (long long)min(2 * T.r0 + q, P.fr_hi) * P.fine.zpitch, FROW_BYTES, &full[s]);
                }
              }
            }
          }
        }
        __syncwarp();
        ++n;
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
      if (HAS_D) {
        if (!waited) {
          pdl_wait();
          waited = true;
        }
        const float* db = P.coarse.D + T.frame * P.coarse.fstride_r + (60 * T.jb - 4);
        if (elect_one()) {
          mbar_arrive_expect_tx(&dfull[hb], 6 * HDR_D_ROW);
          if (P.use_tm_d && tmc) {
            tma_load_3d(hdr + HDR_D_OFF, &P.tm_d, 60 * T.jb - 4, T.r0 - 1 - P.cr_lo, T.frame, &dfull[hb]);
          } else {
#pragma unroll
            for (int q = 0; q < 6; ++q)
              tma_load_1d(hdr + HDR_D_OFF + q * HDR_D_ROW, db + (long long)crow[q] * P.coarse.pitch, HDR_D_ROW,
                          &dfull[hb]);
          }
        }
        __syncwarp();
      }
    }
    return;
  }

  // ---- consumers
  const bool out_al = ((reinterpret_cast<uintptr_t>(P.out) & 15) == 0) && ((P.out_pitch & 3) == 0);
  const unsigned char* rowc = smem + warp * CROW_BYTES + lane * 16;              // coarse row r-1 of this warp
  const unsigned char* rowf = smem + FOFF + 2 * warp * FROW_BYTES + lane * 32;  // fine row 2r
  const int lg = min(max(lane - 1, 0), 29);  // header g column block of this lane (halo lanes: any)
  int s = 0;
  uint32_t ph = 0;
  int nt = 0;
  TileIter it(P);
#pragma unroll 1
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt, it.next()) {
    const ApplyTile T = it.tile();
    const int hb = nt & 1;
    const uint32_t hph = (nt >> 1) & 1;
    const unsigned char* hdr = smem + HOFF + hb * HB;
    const int r = T.r0 + warp;
    const int j = T.jb * 30 + lane - 1;  // coarse columns 2j, 2j+1 -> fine columns 4j..4j+3
    const bool act = r < P.r_end && lane >= 1 && lane <= 30 && 4 * j < P.Wf;
    float g[8];
    if (tma_g) {
      mbar_wait_parity(&gfull[hb], hph);
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        const float4 v = *reinterpret_cast<const float4*>(hdr + (2 * warp + tt) * HDR_G_ROW + lg * 16);
        g[4 * tt + 0] = v.x; g[4 * tt + 1] = v.y; g[4 * tt + 2] = v.z; g[4 * tt + 3] = v.w;
      }
    } else {  // caller image not TMA-compatible: direct loads (level 0 only)
      const int rr = min(r, P.Hc - 1);
      const int xf0 = 4 * j;
      const float* base = P.img.p + T.frame * P.gz * P.img.fstride;
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        const float* rp = base + (long long)min(2 * rr + tt, P.fr_hi) * P.img.pitch;
#pragma unroll
        for (int q = 0; q < 4; ++q) g[4 * tt + q] = __ldg(rp + min(max(xf0 + q, 0), P.Wf - 1));
      }
    }
    float tc[8], sn[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      float c;
      sincos_turns(g[p], P.invT, &sn[p], &c);
      tc[p] = 2.f * c;
    }
    // MAPS (Sec. III-B): a_k(p) = m sigma^3 c0 k exp(-k^2 hq sigma^2).  Per
    // pixel and order ONE exp2 of  k^2 Bm[p] + Lm[p] + log2 k  with
    // Bm = -hq log2(e) sigma^2 and Lm = log2(sigma^3 c0) (+ log2 of the
    // polyphase up-sampling scale at level 0); the factor m multiplies the
    // finished order sum (it is linear in the a_k).  Bm / Lm packed over the
    // pixel pairs (2q, 2q+1); (k^2, log2 k) per order in P.cw[i][0].
    float2 Bm[4], Lm[4];
    if (MAPS) {
      mbar_wait_parity(&mfull[hb], hph);
      const float lc0 = __log2f(P.c0);
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        const float4 sv = *reinterpret_cast<const float4*>(hdr + HDR_S_OFF + (2 * warp + tt) * HDR_G_ROW + lg * 16);
        const float sg[4] = {sv.x, sv.y, sv.z, sv.w};
        float bq[4], lq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bq[q] = -P.hq * 1.4426950408889634f * (sg[q] * sg[q]);
          // level 0: the scale 1/64, 1/16 (even row) and 1/16, 1/4 (odd row) of
          // pixel (even, odd) column, as P.cw[i][0..2] carries it for SCALAR
          const float ls = LEVEL0 ? (tt == 0 ? ((q & 1) ? -4.f : -6.f) : ((q & 1) ? -2.f : -4.f)) : 0.f;
          lq[q] = fmaf(3.f, __log2f(sg[q]), lc0 + ls);
        }
        Bm[2 * tt] = make_float2(bq[0], bq[1]);
        Bm[2 * tt + 1] = make_float2(bq[2], bq[3]);
        Lm[2 * tt] = make_float2(lq[0], lq[1]);
        Lm[2 * tt + 1] = make_float2(lq[2], lq[3]);
      }
    }
    float2 b1[8], b2[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) b1[p] = b2[p] = make_float2(0.f, 0.f);

    // one order from stage slot `so` (order-local base): bn holds b_{k+2} on
    // entry and b_k on exit, bp = b_{k+1}
    // one order's stage data in registers: coarse rows r-1, r, r+1 (and the
    // fine Z rows for levels >= 1)
    struct OrderIn {
      float4 x0, x1, x2;
      float4 fz[LEVEL0 ? 1 : 4];
    };
    auto load_order = [&](const unsigned char* so) {
      OrderIn d;
      d.x0 = *reinterpret_cast<const float4*>(so);
      d.x1 = *reinterpret_cast<const float4*>(so + CROW_BYTES);
      d.x2 = *reinterpret_cast<const float4*>(so + 2 * CROW_BYTES);
      if (!LEVEL0) {
        const unsigned char* sf = so + (rowf - rowc);
        d.fz[0] = *reinterpret_cast<const float4*>(sf);
        d.fz[1] = *reinterpret_cast<const float4*>(sf + 16);
        d.fz[2] = *reinterpret_cast<const float4*>(sf + FROW_BYTES);
        d.fz[3] = *reinterpret_cast<const float4*>(sf + FROW_BYTES + 16);
      }
      return d;
    };
    auto order_in = [&](int i, const OrderIn& d, float2 (&bn)[8], const float2 (&bp)[8]) {
      const float4 x0 = d.x0, x1 = d.x1, x2 = d.x2;
      const float4* fz = d.fz;
      // vertical: even fine row (x_{r-1} + 6 x_r + x_{r+1}), odd (x_r + x_{r+1}); columns a = 2j, b = 2j+1
      const float2 vea = pfma(bc(6.f), lo2(x1), padd(lo2(x0), lo2(x2)));
      const float2 veb = pfma(bc(6.f), hi2(x1), padd(hi2(x0), hi2(x2)));
      const float2 voa = padd(lo2(x1), lo2(x2));
      const float2 vob = padd(hi2(x1), hi2(x2));
      const float2 Le = shfl_up2(veb), Lo = shfl_up2(vob), Re = shfl_down2(vea), Ro = shfl_down2(voa);
      // horizontal: fine col 4j (x_{c-1} + 6 x_c + x_{c+1}), 4j+1 (x_c + x_{c+1}), ...
      float2 raw[8];
      raw[0] = pfma(bc(6.f), vea, padd(Le, veb));
      raw[1] = padd(vea, veb);
      raw[2] = pfma(bc(6.f), veb, padd(vea, Re));
      raw[3] = padd(veb, Re);
      raw[4] = pfma(bc(6.f), voa, padd(Lo, vob));
      raw[5] = padd(voa, vob);
      raw[6] = pfma(bc(6.f), vob, padd(voa, Ro));
      raw[7] = padd(vob, Ro);
      if constexpr (MAPS) {
        // sign convention of the MAPS recurrence: the cosine component carries
        // -b (c_cos = -a Im(.) becomes +a Im(.)), undone at the end; then
        // c = a_k(p)/m * (s raw - fine Z) in both components
        const float2 mk = P.cw[i][0];  // (k^2, log2 k)
        float2 ea[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 arg = pfma(bc(mk.x), Bm[q], padd(Lm[q], bc(mk.y)));
          ea[q] = make_float2(ex2_approx(arg.x), ex2_approx(arg.y));
        }
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const float e = (p & 1) ? ea[p >> 1].y : ea[p >> 1].x;
          float2 d = raw[p];
          if (!LEVEL0) {
            const float sc = (p < 4) ? ((p & 1) ? 1.f / 16.f : 1.f / 64.f) : ((p & 1) ? 0.25f : 1.f / 16.f);
            const float4 fv = fz[(p >> 2) * 2 + ((p & 3) >> 1)];
            d = pfma(bc(sc), raw[p], pneg((p & 1) ? hi2(fv) : lo2(fv)));
          }
          bn[p] = pfma(bc(tc[p]), bp[p], pfma(d, bc(e), pneg(bn[p])));
        }
      } else {
        const float2 w64 = P.cw[i][0], w16 = P.cw[i][1], w4 = P.cw[i][2];
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const float2 w = (p < 4) ? ((p & 1) ? w16 : w64) : ((p & 1) ? w4 : w16);
          float2 c = pfma(raw[p], w, pneg(bn[p]));
          if (!LEVEL0) {
            const float4 fv = fz[(p >> 2) * 2 + ((p & 3) >> 1)];
            c = pfma((p & 1) ? hi2(fv) : lo2(fv), P.cw[i][3], c);
          }
          bn[p] = pfma(bc(tc[p]), bp[p], c);
        }
      }
    };
    auto order = [&](int i, const unsigned char* so, float2 (&bn)[8], const float2 (&bp)[8]) {
      order_in(i, load_order(so), bn, bp);
    };
    auto stage_wait = [&]() -> const unsigned char* {
      mbar_wait_parity(&full[s], ph);
      return rowc + s * STAGE;
    };
    auto stage_release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) {
        s = 0;
        ph ^= 1u;
      }
    };

    int i = KL - 1;
    constexpr bool kFull = KT > 0 && OPS == 2 && (KT % 2) == 0 && (S % (KT / 2)) == 0;
    if constexpr (kFull && kApplyPipe && (!MAPS || kApplyPipeMaps)) {  // (MAPS: 20-24 bytes of spills)
      // software-pipelined: the next stage's wait and shared-memory loads are
      // issued before the current stage's second order is evaluated (the
      // barrier wait is a compiler fence, so without this every stage starts
      // with an exposed LDS + shuffle latency)
      const unsigned char* rs = rowc + s * STAGE;
      const uint32_t fb = smem_u32(&full[s]), eb = smem_u32(&empty[s]);
      mbar_wait_u32(fb, ph);
      OrderIn oa = load_order(rs), ob = load_order(rs + OBYTES);
#pragma unroll
      for (int jst = 0; jst < KT / 2; ++jst) {
        order_in(KT - 1 - 2 * jst, oa, b2, b1);
        if (jst + 1 < KT / 2) {
          mbar_wait_u32(fb + (jst + 1) * 8, ph);
          oa = load_order(rs + (jst + 1) * STAGE);
        }
        order_in(KT - 2 - 2 * jst, ob, b1, b2);
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(eb + jst * 8);
        if (jst + 1 < KT / 2) ob = load_order(rs + (jst + 1) * STAGE + OBYTES);
      }
      s += KT / 2;
      if (s == S) {
        s = 0;
        ph ^= 1u;
      }
      i = -1;
    } else if constexpr (kFull) {
      const unsigned char* rs = rowc + s * STAGE;
      const uint32_t fb = smem_u32(&full[s]), eb = smem_u32(&empty[s]);
#pragma unroll
      for (int jst = 0; jst < KT / 2; ++jst) {
        mbar_wait_u32(fb + jst * 8, ph);
        const unsigned char* so = rs + jst * STAGE;
        order(KT - 1 - 2 * jst, so, b2, b1);
        order(KT - 2 - 2 * jst, so + OBYTES, b1, b2);
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(eb + jst * 8);
      }
      s += KT / 2;
      if (s == S) {
        s = 0;
        ph ^= 1u;
      }
      i = -1;
    } else if constexpr (KT > 0 && OPS == 1 && (KT % S) == 0 && (KT % 2) == 0) {
      // levels >= 1 with the order count at compile time (MAPS, K = 12): a
      // tile consumes KT / S whole turns of the ring, so every tile starts
      // at stage 0 and the loop unrolls with compile-time stage offsets and
      // barrier addresses (one parity flip per turn)
      const uint32_t fb = smem_u32(&full[0]), eb = smem_u32(&empty[0]);
#pragma unroll
      for (int jj = 0; jj < KT; ++jj) {
        const int st = jj % S;
        mbar_wait_u32(fb + st * 8, ph ^ (uint32_t)((jj / S) & 1));
        if (jj & 1) order(KT - 1 - jj, rowc + st * STAGE, b1, b2);
        else order(KT - 1 - jj, rowc + st * STAGE, b2, b1);
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(eb + st * 8);
      }
      if ((KT / S) & 1) ph ^= 1u;
      i = -1;
    } else if (OPS == 2) {
      constexpr int UNR = MAPS ? 1 : kApply0Unroll;  // MAPS: unrolling measured slower
#pragma unroll UNR
      for (; i >= 1; i -= 2) {
        const unsigned char* so = stage_wait();
        order(i, so, b2, b1);
        order(i - 1, so + OBYTES, b1, b2);
        stage_release();
      }
    } else {
#pragma unroll kApply1Unroll
      for (; i >= 1; i -= 2) {
        order(i, stage_wait(), b2, b1);
        stage_release();
        order(i - 1, stage_wait(), b1, b2);
        stage_release();
      }
    }
    if (i == 0) {  // odd order count: the last b_k landed in b2
      order(0, stage_wait(), b2, b1);
      stage_release();
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const float2 tmp = b1[p];
        b1[p] = b2[p];
        b2[p] = tmp;
      }
    }
    // b1 = b_{k0}, b2 = b_{k0+1}
    if constexpr (MAPS) {  // back to the common sign convention
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        b1[p].x = -b1[p].x;
        b2[p].x = -b2[p].x;
      }
    }
    float res[8];
    if (P.kbase == 1) {
#pragma unroll
      for (int p = 0; p < 8; ++p) res[p] = fmaf(b1[p].x, 0.5f * tc[p], fmaf(b1[p].y, sn[p], -b2[p].x));
    } else {
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        float sk, ck;
        sincos_turns_n(g[p], P.invT, P.kbase, &sk, &ck);
        const float c1 = 0.5f * tc[p], s1 = sn[p];
        const float cm = fmaf(ck, c1, sk * s1), sm = fmaf(sk, c1, -ck * s1);  // e^{i (k0-1) theta}
        res[p] = fmaf(b1[p].x, ck, fmaf(b1[p].y, sk, -fmaf(b2[p].x, cm, b2[p].y * sm)));
      }
    }
    if constexpr (MAPS) {  // the factor m of a_k (header rows, still held)
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        const float4 mv = *reinterpret_cast<const float4*>(hdr + HDR_M_OFF + (2 * warp + tt) * HDR_G_ROW + lg * 16);
        res[4 * tt + 0] *= mv.x;
        res[4 * tt + 1] *= mv.y;
        res[4 * tt + 2] *= mv.z;
        res[4 * tt + 3] *= mv.w;
      }
    }

    // --- collapse: + up(D_{l+1}) from the tile header
    if (HAS_D) {
      float dq[3][2];
      mbar_wait_parity(&dfull[hb], hph);
      const int c0 = 60 * T.jb - 4;
      int cc0 = 2 * lane + 2, cc1 = 2 * lane + 3;  // interior column tiles: no border mapping
      if (T.jb == 0 || T.jb == it.nx - 1) {
        cc0 = upmap(2 * j, P.Wc, P.Wf) - c0;
        cc1 = upmap(2 * j + 1, P.Wc, P.Wf) - c0;
      }
      const float* dh = reinterpret_cast<const float*>(hdr + HDR_D_OFF + warp * HDR_D_ROW);
#pragma unroll
      for (int tt = 0; tt < 3; ++tt) {
        dq[tt][0] = dh[tt * (HDR_D_ROW / 4) + cc0];
        dq[tt][1] = dh[tt * (HDR_D_ROW / 4) + cc1];
      }
      float hd[3][4];
#pragma unroll
      for (int tt = 0; tt < 3; ++tt) {
        const float x0 = dq[tt][0], x1 = dq[tt][1];
        const float L = __shfl_up_sync(FULL, x1, 1);
        const float Rn = __shfl_down_sync(FULL, x0, 1);
        hd[tt][0] = fmaf(6.f, x0, L + x1) * 0.125f;
        hd[tt][1] = (x0 + x1) * 0.5f;
        hd[tt][2] = fmaf(6.f, x1, x0 + Rn) * 0.125f;
        hd[tt][3] = (x1 + Rn) * 0.5f;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        res[q] += 0.125f * fmaf(6.f, hd[1][q], hd[0][q] + hd[2][q]);
        res[4 + q] += 0.5f * (hd[1][q] + hd[2][q]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&hempty[hb]);  // this warp is done with the tile header
    if (LEVEL0 && P.include_base) {
#pragma unroll
      for (int p = 0; p < 8; ++p) res[p] += g[p];
    }

    if (act) {
      const int xf0 = 4 * j;
      const bool fvec_ok = xf0 + 3 < P.Wf;
      float* op;
      long long opitch;
      bool oal;
      if (LEVEL0) {
        op = P.out + T.frame * P.out_fstride;
        opitch = P.out_pitch;
        oal = out_al;
      } else {
        op = P.fine.D + T.frame * P.fine.fstride_r;
        opitch = P.fine.pitch;
        oal = true;
      }
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        if (2 * r + tt >= P.Hf) break;
        float* rp = op + (long long)(2 * r + tt) * opitch;
        if (LEVEL0 && P.accumulate) {
          // fused combine (order sharding): add this partial output into the
          // destination -- local, or a peer GPU's buffer mapped through CUDA
          // IPC, the adds then travel over NVLink -- with hardware atomics
          if (fvec_ok && oal) {
            FLLF_DBG_STORE(P, rp + xf0, 16);
            atomicAdd(reinterpret_cast<float4*>(rp + xf0),
                      make_float4(res[4 * tt], res[4 * tt + 1], res[4 * tt + 2], res[4 * tt + 3]));
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (xf0 + q < P.Wf) {
                FLLF_DBG_STORE(P, rp + xf0 + q, 4);
                atomicAdd(rp + xf0 + q, res[4 * tt + q]);
              }
          }
        } else if (fvec_ok && oal) {
          FLLF_DBG_STORE(P, rp + xf0, 16);
          *reinterpret_cast<float4*>(rp + xf0) =
              make_float4(res[4 * tt], res[4 * tt + 1], res[4 * tt + 2], res[4 * tt + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (xf0 + q < P.Wf) {
              FLLF_DBG_STORE(P, rp + xf0 + q, 4);
              rp[xf0 + q] = res[4 * tt + q];
            }
        }
      }
    }
  }
}


// Rows per warp strip: long strips amortise the 3 halo rows; shorter strips
// only when the grid would leave SMs without warps.
int pick_rows(int Hc, int blocks_x, int z) {
  static const long long target = [] {
    const char* e = std::getenv("FLLF_BL_WARPS");
    return e ? std::atoll(e) : 148LL * 8;
  }();
  static const int rmax = [] {
    const char* e = std::getenv("FLLF_BL_RMAX");
    return e ? std::atoi(e) : 16;
  }();
  int R = rmax;
  while (R > 2 && (long long)blocks_x * ((Hc + R - 1) / R) * z < target) R >>= 1;
  return R;
}

}  // namespace

template <int NC, bool FROM_IMAGE>
static cudaError_t launch_build_nc(BuildParams p, int batch, cudaStream_t s, bool pdl) {
  const int bx = (p.Wc + 29) / 30;  // one warp (CTA) per 30 coarse columns
  p.nchunks = p.KL / NC;
  const int nrows = p.o_end - p.o_begin;
  p.rows_per_strip = pick_rows(nrows, bx, batch * p.nchunks);
  dim3 grid(bx, (nrows + p.rows_per_strip - 1) / p.rows_per_strip, batch * p.nchunks);
  if (p.rows_per_strip == 2) return launch_ex(k_build<NC, 1, FROM_IMAGE, true>, grid, dim3(32), 0, s, pdl, p);
  static const int depth = [] {  // FLLF_BUILD_DEPTH: row pairs in flight per warp (2 or 3)
    const char* e = std::getenv("FLLF_BUILD_DEPTH");
    return e ? std::atoi(e) : 3;  // 3 measured best on B200
  }();
  if (!FROM_IMAGE && depth >= 3) return launch_ex(k_build<NC, 1, FROM_IMAGE, false, true>, grid, dim3(32), 0, s, pdl, p);
  return launch_ex(k_build<NC, 1, FROM_IMAGE, false>, grid, dim3(32), 0, s, pdl, p);
}

template <int NC>
static cudaError_t launch_build0_nc(BuildParams p, int batch, cudaStream_t s, bool pdl) {
  const int bx = (p.Wc + 29) / 30;
  p.nchunks = p.KL / NC;
  // strips of >= 4 output rows (the run loop needs R >= 2; halo rows 3/(2R))
  int R = 16;
  { const char* e = std::getenv("FLLF_B0_WARPS"); const long long tw = e ? std::atoll(e) : 148LL * 8;
    while (R > 4 && (long long)bx * ((p.o_end - p.o_begin + R - 1) / R) * batch * p.nchunks < tw) R >>= 1; }
  if (R > p.o_end - p.o_begin) R = std::max(p.o_end - p.o_begin, 2);
  p.rows_per_strip = R;
  dim3 grid(bx, (p.o_end - p.o_begin + R - 1) / R, batch * p.nchunks);
  return launch_ex(k_build0<NC>, grid, dim3(32), 0, s, pdl, p);
}

// largest channel chunk (<= cap) dividing the local order count
static int chunk_for(int KL, int cap) {
  for (int c = cap; c > 1; --c)
    if (KL % c == 0) return c;
  return 1;
}

cudaError_t launch_build(const BuildParams& p0, int level_src, int batch, cudaStream_t s, bool pdl) {
  BuildParams p = p0;
  if (p.maps) {
    const int bx = (p.Wc + 29) / 30;
    p.nchunks = 1;
    p.rows_per_strip = pick_rows(p.o_end - p.o_begin, bx, batch);
    dim3 grid(bx, (p.o_end - p.o_begin + p.rows_per_strip - 1) / p.rows_per_strip, batch);  // z: map pairs
    if (level_src == 0) return launch_ex(k_build<0, 2, true, false>, grid, dim3(32), 0, s, pdl, p);
    return launch_ex(k_build<0, 2, false, false>, grid, dim3(32), 0, s, pdl, p);
  }
  if (level_src == 0) {
    static const int cap = [] {
      const char* e = std::getenv("FLLF_BUILD0V2_CHUNK");
      const int v = e ? std::atoi(e) : 8;
      return v >= 1 && v <= 8 ? v : 8;
    }();
    switch (chunk_for(p.KL, cap)) {
      case 8: return launch_build0_nc<8>(p, batch, s, pdl);
      case 7: return launch_build0_nc<7>(p, batch, s, pdl);
      case 6: return launch_build0_nc<6>(p, batch, s, pdl);
      case 5: return launch_build0_nc<5>(p, batch, s, pdl);
      case 4: return launch_build0_nc<4>(p, batch, s, pdl);
      case 3: return launch_build0_nc<3>(p, batch, s, pdl);
      case 2: return launch_build0_nc<2>(p, batch, s, pdl);
      default: return launch_build0_nc<1>(p, batch, s, pdl);
    }
  }
  static const int cap1 = [] {
    const char* e = std::getenv("FLLF_BUILD_CHUNK");
    const int v = e ? std::atoi(e) : 2;  // measured best on B200
    return v >= 1 && v <= 4 ? v : 2;
  }();
  switch (chunk_for(p.KL, cap1)) {
    case 4: return launch_build_nc<4, false>(p, batch, s, pdl);
    case 3: return launch_build_nc<3, false>(p, batch, s, pdl);
    case 2: return launch_build_nc<2, false>(p, batch, s, pdl);
    default: return launch_build_nc<1, false>(p, batch, s, pdl);
  }
}


template <bool L0, bool HD, bool MP>
static cudaError_t launch_apply_t(const ApplyParams& p, int batch, cudaStream_t s, bool pdl) {
  const int ntiles = ((p.Wf + 119) / 120) * ((p.r_end - p.r_begin + 3) / 4) * batch;
  const int per_sm = MP ? 2 : 3;  // resident CTAs per SM (launch bounds)
  dim3 grid(std::min(ntiles, sm_count() * per_sm));
  const int smem = apply_stages<L0>() * apply_stage_bytes<L0>();
  static DeviceFlags attr_set;  // > 48 KB of dynamic shared memory needs an opt-in, per device
  cudaError_t e = smem_opt_in(k_apply<L0, HD, MP>, smem, attr_set);
  if (e != cudaSuccess) return e;
  return launch_ex(k_apply<L0, HD, MP>, grid, dim3(160), smem, s, pdl, p, ntiles);
}

template <bool L0, bool HD, bool MP, int KT = 0>
static cudaError_t launch_apply_cl_k(const ApplyParams& p, int batch, cudaStream_t s, bool pdl) {
  const int ntiles = ((p.Wf + 119) / 120) * ((p.r_end - p.r_begin + 3) / 4) * batch;
  dim3 grid(std::min(ntiles, sm_count() * apply_cl_ctas<L0, MP>()));
  const int smem = apply_cl_smem<L0, MP, KT>();
  static DeviceFlags attr_set;
  cudaError_t e = smem_opt_in(k_apply_cl<L0, HD, MP, KT>, smem, attr_set);
  if (e != cudaSuccess) return e;
  return launch_ex(k_apply_cl<L0, HD, MP, KT>, grid, dim3(160), smem, s, pdl, p, ntiles);
}

template <bool L0, bool HD, bool MP>
static cudaError_t launch_apply_cl_t(const ApplyParams& p, int batch, cudaStream_t s, bool pdl) {
  static const bool generic = [] {  // FLLF_APPLY0_GENERIC=1: no order-count specialisation (A/B)
    const char* e = std::getenv("FLLF_APPLY0_GENERIC");
    return e && e[0] == '1';
  }();
  if constexpr (L0 && !MP) {
    if (!generic && p.KL == 16) return launch_apply_cl_k<L0, HD, MP, 16>(p, batch, s, pdl);
    if (!generic && p.KL == 8) return launch_apply_cl_k<L0, HD, MP, 8>(p, batch, s, pdl);
  }
  if constexpr (MP) {  // BASELINE configs[3]: K = 12 (level 0 and levels >= 1)
    if (!generic && p.KL == 12) return launch_apply_cl_k<L0, HD, MP, 12>(p, batch, s, pdl);
  }
  return launch_apply_cl_k<L0, HD, MP>(p, batch, s, pdl);
}

cudaError_t launch_apply(const ApplyParams& p, int level_fine, bool has_d, bool maps, int batch,
                         cudaStream_t s, bool pdl) {
  // MAPS through the Clenshaw kernel when the level-0 maps can be staged by
  // bulk copies (16-byte aligned rows, W a multiple of 4); else the forward kernel
  const bool maps_cl = maps && (((reinterpret_cast<uintptr_t>(p.smap.p) | reinterpret_cast<uintptr_t>(p.mmap.p)) & 15) == 0) &&
                       ((p.smap.pitch & 3) == 0) && ((p.mmap.pitch & 3) == 0) && (p.smap.pitch == p.mmap.pitch) &&
                       ((p.img.W & 3) == 0);
  static const bool maps_v1 = [] {
    const char* e = std::getenv("FLLF_MAPS_V1");
    return e && e[0] == '1';
  }();
  if (!maps || (maps_cl && !maps_v1)) {
#define FLLF_CL(L0, HD) return maps ? launch_apply_cl_t<L0, HD, true>(p, batch, s, pdl) : launch_apply_cl_t<L0, HD, false>(p, batch, s, pdl)
    if (level_fine == 0) {
      if (has_d) FLLF_CL(true, true);
      FLLF_CL(true, false);
    }
    if (has_d) FLLF_CL(false, true);
    FLLF_CL(false, false);
#undef FLLF_CL
  }
#define FLLF_APPLY(L0, HD, MP) return launch_apply_t<L0, HD, MP>(p, batch, s, pdl)
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
}

}  // namespace fllf
