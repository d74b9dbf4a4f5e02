// Design F ("materialise once") kernels for sm_100a: the level-l order sum of
// Eq. 14 fused into the build step l -> l+1 of Eq. 1,
// plus the collapse of Eq. 4 over the real D planes.
//
// Design AB (fllf_kernels.cu) builds every pyramid first and then, coarse to
// fine, re-reads Z_l and Z_{l+1} in the apply pass: each level >= 1 plane is
// written once and read twice.  The paper's cost model is "the computing cost
// of 2K+1 pyramids"; design F meets it by consuming Z_l while it
// is streamed for the build:
//
//   k_fuse, level l >= 1 (one launch per level, fine to coarse):
//     reads  G_l, Z_{l,k}                      (as k_build)
//     writes G_{l+1}, Z_{l+1,k}                (as k_build)
//     writes S_l = sum_k a_k Im(e^{-i k w_1 g} (Z_{l,k} - up Z_{l+1,k})),  g = G_l,
//            into the D_l plane
//   k_collapse, l = l_max-2 .. 1:  D_l += up(D_{l+1})   (D_{l_max-1} = S_{l_max-1})
//   then the level-0 apply of design AB reads D_1 (k_apply_cl<LEVEL0>).
//
// D_l = O_l - G_l is the collapse from level l of the output pyramid minus
// G_l; S_l is its level-l increment, so the two designs
// compute the same D planes (exact algebra, different rounding order only).
//
// k_fuse layout.  CTA = one strip (R coarse rows x 28 coarse columns of one
// frame) with one warp per NC orders (NC = 1 for K <= 16: 16 warps, plus a
// 17th warp that builds only the real channel G_l -> G_{l+1} and stages the
// g values of the order sums, FUSE_GWARP; with NC = 2 warp 0 does that on
// top of its orders).  Warp w
// owns the NC orders [w NC, (w+1) NC) of the plan's order range; lane L holds
// coarse column x = 28 cb + L - 2 and fine columns 2x, 2x+1 (reflect-101 per
// lane at the frame borders).  It streams fine row pairs P_j = (2j, 2j+1),
// j = o0-2 .. o0+R+1, through its own shared-memory ring (cp.async, PD pairs
// ahead; the G warp stages G_l): the VERTICAL 5-tap with two rolling
// accumulators per order and column, then the HORIZONTAL 5-tap on the
// finished coarse row from warp shuffles (k_build's arithmetic, so G_{l+1}
// and Z_{l+1} are bit-identical to design AB).  Lanes 1..30 hold valid coarse
// values; with the reflected fine columns / rows those obey the up-sampling
// border rule (column -1 = x_1, column C = x_{C-1} or x_{C-2}), so the coarse
// rows o0-1, o0+R and lanes 1, 30 are the up-sampling halo.  The last three
// coarse rows stay in registers, and so do the Z_l values of the last three
// pairs; once coarse row i+1 is finished the warp forms, for the 4 fine
// pixels of pair P_i per lane, the Clenshaw coefficient pair of its order
//     c_k = a_k (Im V_k, -Re V_k),   V_k = Z_{l,k} - up(Z_{l+1,k}),
// and writes it to the shared array C[pair][k][row][col].  Every 3 pairs (one
// iteration of the stream loop, unrolled by 3 for the register rotation) the
// CTA meets at a named barrier and evaluates the batch's order sums
//     S = sum_k a_k Im(e^{-i k theta} V_k),   theta = w_1 g,
// one pixel per thread, Clenshaw's recurrence over ALL the plan's orders (one
// sincos per pixel, no cross-warp reduction), stores S into D_l and meets at
// the barrier again before C is overwritten.
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

#include "fllf_dev.h"

constexpr int FUSE_COLS = 28;  // owned coarse columns per warp (lanes 2..29)
constexpr int FUSE_BAR = 1;    // named barrier id of the batch hand-over

// warps per CTA (one per NC-order chunk), bounded so that the CTA fits one
// SM's register file at 128 registers per thread (16 warps = 4 per SMSP)
constexpr int FUSE_MAX_WARPS = 16;
// order-sum batch: NB = 3 fine row pairs (384 pixels), the steps of one
// iteration of the stream loop (unrolled by 3 for the register rotation), so
// the order sums sit at one place in the loop
constexpr int FUSE_NB = 3;
__host__ __device__ inline int fuse_nb(int) { return FUSE_NB; }

__device__ __forceinline__ void bar_sync_id(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// shared-memory accesses through 32-bit shared addresses
__device__ __forceinline__ void cpa16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds1(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void sts2(uint32_t a, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}

// Order-sum hand-over buffers: 1 = one buffer and two CTA barriers per batch
// (default); 2 = double-buffered C / Gb with mbarriers (warps run one batch
// apart: a warp streams batch b while the order sums of batch b-1 wait only
// for the last warp's coefficients of b-1).  Measured at config 5: level 1
// 1.44-1.51 ms with 2 vs 1.38-1.41 ms with 1, so the
// barrier coupling is not what limits this kernel; kept for A/B.
#ifndef FLLF_FUSE_NBUF
#define FLLF_FUSE_NBUF 1
#endif
constexpr int FUSE_NBUF = FLLF_FUSE_NBUF;
// G_l (the real channel: G_{l+1} and the g of the order sums) built by a
// 17th warp instead of by warp 0 on top of its order: warp 0 no longer sets
// the pace of the CTA's batch barriers (one order per warp only; A/B knob)
#ifndef FLLF_FUSE_GWARP
#define FLLF_FUSE_GWARP 1
#endif
constexpr bool FUSE_GWARP = FLLF_FUSE_GWARP != 0;
// read each ring pair into registers one step ahead (the cp.async wait is a
// compiler fence); K = 16 only, where it fits 128 registers once the
// coefficient pairs come from the kernel parameters.  Off: measured 10 %
// slower at config 5 level 1 (1.51-1.53 vs 1.38-1.39 ms); A/B knob.
// Order sums of an even compile-time order count (KT) from k = 1 as two
// interleaved half-length Clenshaw chains in 2 theta (even / odd orders)
// instead of one chain in theta: same instruction count, half the dependent
// latency of the phase the whole CTA waits for between its batch barriers.
// Measured at config 5 (4 interleaved A/B pairs): level 1 1.41-1.46 ms with
// it vs 1.39-1.43 ms without, so off; kept for A/B.
#ifndef FLLF_FUSE_SPLIT
#define FLLF_FUSE_SPLIT 0
#endif

#ifndef FLLF_FUSE_PIPE
#define FLLF_FUSE_PIPE 0
#endif

// Stream-loop iterations (of FUSE_NB = 3 pairs) per order-sum batch with one
// order per warp and one hand-over buffer: 2 = batches of 6 pairs (768
// pixels, two passes of the CTA's threads) between half as many CTA barrier
// pairs, C twice as large (96 KB at K = 16).  Measured at config 5: no gain
// in the step (4.33-4.38 vs 4.31-4.35 ms), so 1.
#ifndef FLLF_FUSE_NBI
#define FLLF_FUSE_NBI 1
#endif

// Shared-memory layout of one CTA (bytes), NB = fuse_nb(warps):
//   C    [NBUF][NB pairs][KL orders][2 fine rows][64 fine columns] float2   (NBUF x NB x 1024 KL)
//   Gb   [NBUF][NB pairs][2 fine rows][64 fine columns] float                 (NBUF x NB x 512)
//   GW = 0: ring of warp 0:  DEPTH slots x (G 512 + Z 1024 NC)
//           ring of warp w:  DEPTH slots x Z 1024 NC
//   GW = 1: ring of order warp w (0 .. KL/NC - 1): DEPTH slots x Z 1024 NC,
//           then the G warp's (warp KL/NC): DEPTH slots x G 512
template <int NC, int PD>
struct FuseLayout {
  static constexpr int NBUF = NC == 1 ? FUSE_NBUF : 1;  // (two orders per warp: K > 16, shared memory)
  static constexpr int NBI = (NC == 1 && NBUF == 1) ? FLLF_FUSE_NBI : 1;
  static constexpr int NB = FUSE_NB * NBI;  // fine row pairs per order-sum batch
  static constexpr bool GW = FUSE_GWARP && NC == 1;      // G_l built by a warp of its own
  static constexpr int DEPTH = PD + 1;
  static constexpr int ZSLOT = NC * 1024;  // NC orders x 2 rows x 32 lanes x float4
  static constexpr int G0SLOT = 512 + ZSLOT;
  __host__ __device__ static int c_buf(int KL) { return NB * KL * 1024; }
  __host__ __device__ static int g_buf(int KL) { return NB * 512; }
  __host__ __device__ static int g_off(int KL) { return NBUF * c_buf(KL); }
  __host__ __device__ static int ring_off(int KL, int w) {
    if (GW) return g_off(KL) + NBUF * g_buf(KL) + w * DEPTH * ZSLOT;  // (w = KL/NC: the G warp)
    return g_off(KL) + NBUF * g_buf(KL) + (w == 0 ? 0 : DEPTH * G0SLOT + (w - 1) * DEPTH * ZSLOT);
  }
  __host__ __device__ static int smem(int KL) { return ring_off(KL, KL / NC) + (GW ? DEPTH * 512 : 0); }
  __host__ __device__ static int warps(int KL) { return KL / NC + (GW ? 1 : 0); }
};

// ---- one warp: NC orders of the strip (DO_G: warp 0 also builds G;
// ROWS_IN: no fine row of the strip needs reflection)
template <int NC, int PD, bool EDGE, bool DO_G, bool ROWS_IN, int KT, bool HAS_Z = true>
struct FuseWarp {
  using L = FuseLayout<NC, PD>;
  static constexpr int DEPTH = L::DEPTH;
  static constexpr int SLOT = (DO_G ? 512 : 0) + (HAS_Z ? L::ZSLOT : 0);
  static constexpr int NZ = HAS_Z ? NC : 0;  // complex orders of this warp (0: the G warp)
  static constexpr int ZOFF = DO_G ? 512 : 0;
  // the plan's order count (compile time for KT > 0)
  __device__ __forceinline__ int kl() const { return KT > 0 ? KT : P.KL; }

  const FuseParams& P;
  int o0, R, lane, warp, nw, nb;
  int x, rc0, rc1, Hf;
  bool store_lane, halo_l, halo_r;
  long long zks, gpitch, zpitch;
  const float* gsrc;    // G_l: next row pair (ROWS_IN) or the frame base
  const float2* zsrc;   // Z_l, first order of the chunk: next row pair (ROWS_IN) or the frame base
  float* gout;          // G_{l+1} at (o0 - 1, x): advanced one coarse row per emit
  float2* zout;         // Z_{l+1} at (o0 - 1, x), first order of the chunk
  uint32_t ring;        // this warp's ring (shared address)
  uint32_t si, sr;      // ring slot offsets: next issue, next read
  uint32_t crow;        // C[0][il0][0][2 lane] (shared address)
  uint32_t gbrow;       // Gb[0][0][2 lane]
  int jn;               // fine row pair of the next issue (reflected path)
  // PIPE: each ring pair is read one step ahead (K = 16, one order per warp:
  // the other instantiations spill).  This warp's Clenshaw coefficient pairs
  // (ApplyParams::cw) are then read from the kernel parameters at each use
  // instead of being held in registers.
  // (With the G warp of its own, GW, the order warps have the registers to
  // keep the pairs.)
  static constexpr bool PIPE = FLLF_FUSE_PIPE && KT == 16 && NC == 1;
  static constexpr bool CW_PARAM = PIPE && !L::GW;
  int il0_;
  float2 cwk_[CW_PARAM ? 1 : NC][4];
  __device__ __forceinline__ float2 cwk(int i, int u) const { return CW_PARAM ? P.cw[il0_ + i][u] : cwk_[i][u]; }
  int cb_;
  uint32_t sbase_;
  float* dbase;         // D_l of the frame
  uint32_t bars;        // mbarriers (NBUF = 2): full[0], full[1], empty[0], empty[1]
  uint32_t cbo, gbo;    // C / Gb offsets of the buffer being written
  float2 Pc[NC][2], Ac[NC][2];
  float2 Pr, Ar;

  __device__ __forceinline__ FuseWarp(const FuseParams& P_, int cb, int o0_, int R_, int frame, int nw_,
                                      int warp_, uint32_t smem, uint32_t bars_)
      : P(P_), o0(o0_), R(R_), warp(warp_), nw(nw_), bars(bars_) {
    lane = threadIdx.x & 31;
    nb = fuse_nb(nw);
    Hf = P.Hf;
    x = FUSE_COLS * cb + lane - 2;
    const int c0 = 2 * x;
    rc0 = EDGE ? refl101(c0, P.Wf) : c0;
    rc1 = EDGE ? refl101(c0 + 1, P.Wf) : c0 + 1;
    store_lane = lane >= 2 && lane <= 29 && x < P.Wc;
    halo_l = EDGE && store_lane && x == 1;
    halo_r = EDGE && store_lane && x == ((P.Wf & 1) ? P.Wc - 2 : P.Wc - 1);
    const int il0 = warp * NC;
    il0_ = il0;
    zks = P.src.kstride_z;
    gpitch = P.src.pitch;
    zpitch = P.src.zpitch;
    const long long r0 = ROWS_IN ? 2LL * (o0 - 2) : 0;
    gsrc = P.src.G + frame * P.src.fstride_r + r0 * gpitch + (EDGE ? 0 : c0);
    zsrc = P.src.Z + frame * P.src.fstride_z + (long long)il0 * zks + r0 * zpitch + (EDGE ? 0 : c0);
    gout = P.dst.G + frame * P.dst.fstride_r + (long long)(o0 - 1) * P.dst.pitch + x;
    zout = P.dst.Z + frame * P.dst.fstride_z + (long long)il0 * P.dst.kstride_z + (long long)(o0 - 1) * P.dst.zpitch + x;
    ring = smem + L::ring_off(kl(), warp);
    si = sr = 0;
    crow = smem + il0 * 1024 + lane * 16;
    gbrow = smem + L::g_off(kl()) + lane * 8;
    jn = o0 - 2;
#pragma unroll
    for (int i = 0; i < NZ; ++i) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (!CW_PARAM && HAS_Z) cwk_[i][u] = P.cw[il0 + i][u];
      Pc[i][0] = Pc[i][1] = Ac[i][0] = Ac[i][1] = make_float2(0.f, 0.f);
    }
    Pr = Ar = make_float2(0.f, 0.f);
    cb_ = cb;
    sbase_ = smem;
    dbase = P.src.D + frame * P.src.fstride_r;
    cbo = gbo = 0;
  }

  // copies of the next pair (fine rows 2 jn, 2 jn + 1) into the next ring slot
  __device__ __forceinline__ void issue() {
    const uint32_t sl = ring + si;
    si = si + SLOT == DEPTH * SLOT ? 0 : si + SLOT;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float* gp;
      const float2* zp;
      if (ROWS_IN) {
        gp = gsrc + r * gpitch;
        zp = zsrc + r * zpitch;
      } else {
        const int rr = refl101(2 * jn + r, Hf);
        gp = gsrc + rr * gpitch;
        zp = zsrc + rr * zpitch;
      }
      if (DO_G) {
        const uint32_t gd = sl + r * 256 + lane * 8;
        if (EDGE) {
          cpa4(gd, gp + rc0);
          cpa4(gd + 4, gp + rc1);
        } else {
          cpa8(gd, gp);
        }
      }
#pragma unroll
      for (int i = 0; i < NZ; ++i) {
        const uint32_t zd = sl + ZOFF + (i * 2 + r) * 512 + lane * 16;
        const float2* q = zp + i * zks;
        if (EDGE) {
          cpa8(zd, q + rc0);
          cpa8(zd + 8, q + rc1);
        } else {
          cpa16(zd, q);
        }
      }
    }
    if (ROWS_IN) {
      gsrc += 2 * gpitch;
      zsrc += 2 * zpitch;
    } else {
      ++jn;
    }
  }

  struct Pair {
    float2 ge, go;
    float4 ze[NC], zo[NC];
  };
  Pair nxt;  // FLLF_FUSE_PIPE: the next pair, read from the ring one step ahead
  __device__ __forceinline__ void read(Pair& d) {
    const uint32_t sl = ring + sr;
    sr = sr + SLOT == DEPTH * SLOT ? 0 : sr + SLOT;
    if (DO_G) {
      d.ge = lds2(sl + lane * 8);
      d.go = lds2(sl + 256 + lane * 8);
    }
#pragma unroll
    for (int i = 0; i < NZ; ++i) {
      d.ze[i] = lds4(sl + ZOFF + (i * 2) * 512 + lane * 16);
      d.zo[i] = lds4(sl + ZOFF + (i * 2 + 1) * 512 + lane * 16);
    }
  }

  // finish the next coarse row from the even row of the current pair
  // (k_build's arithmetic); OWN: store it
  template <bool OWN>
  __device__ __forceinline__ void emit(const Pair& d, float2 (&h)[NC]) {
#pragma unroll
    for (int i = 0; i < NZ; ++i) {
      const float2 ea = pfma(bc(W2), lo2(d.ze[i]), Pc[i][0]);
      const float2 eb = pfma(bc(W2), hi2(d.ze[i]), Pc[i][1]);
      h[i] = hfilt_c(ea, eb);
      if (OWN) {
        float2* q = zout + i * P.dst.kstride_z;
        if (store_lane) {
          FLLF_DBG_STORE(P, q, 8);
          stg2(q, h[i]);
        }
        if (EDGE && halo_l) {
          FLLF_DBG_STORE(P, q - 2, 8);
          q[-2] = h[i];  // x == 1: column -1
        }
        if (EDGE && halo_r) {
          FLLF_DBG_STORE(P, q + (P.Wc - x), 8);
          q[P.Wc - x] = h[i];
        }
      }
    }
    if (DO_G) {
      const float2 e = pfma(bc(W2), d.ge, Pr);
      const float hg = hfilt_r(e.x, e.y);
      if (OWN && store_lane) {
        FLLF_DBG_STORE(P, gout, 4);
        *gout = hg;
      }
      gout += P.dst.pitch;
    }
    zout += P.dst.zpitch;
  }
  __device__ __forceinline__ void vstep(const Pair& d) {
#pragma unroll
    for (int i = 0; i < NZ; ++i) {
      vstep_fixed(Pc[i][0], Ac[i][0], lo2(d.ze[i]), lo2(d.zo[i]));
      vstep_fixed(Pc[i][1], Ac[i][1], hi2(d.ze[i]), hi2(d.zo[i]));
    }
    if (DO_G) vstep_fixed(Pr, Ar, d.ge, d.go);
  }

  // c_k = a_k (Im V_k, -Re V_k) with V_k = Z_{l,k} - up(Z_{l+1,k}) at the 4
  // fine pixels of own pair n, from the coarse rows i-1, i, i+1 (Cm, C0, Cp)
  // and the pair's Z_l values (ze, zo); at the end of a batch of NB pairs (or
  // of the strip) the CTA evaluates the batch's order sums
  __device__ __forceinline__ void coef(const float2 (&Cm)[NC], const float2 (&C0)[NC], const float2 (&Cp)[NC],
                                       const float4 (&ze)[NC], const float4 (&zo)[NC], const float4& gg, int n,
                                       int& q) {
    const uint32_t cb = crow + cbo + q * (kl() * 1024);
#pragma unroll
    for (int i = 0; i < NZ; ++i) {
      // vertical up-sampling (unscaled): even fine row x_{i-1} + 6 x_i + x_{i+1}, odd x_i + x_{i+1}
      const float2 ve = pfma(bc(6.f), C0[i], padd(Cm[i], Cp[i]));
      const float2 vo = padd(C0[i], Cp[i]);
      const float2 veL = shfl_up2(ve), veR = shfl_down2(ve), voL = shfl_up2(vo), voR = shfl_down2(vo);
      // horizontal + polyphase scales and a_k with the sign pattern (cwk)
      const float2 c0 = pfma(pfma(bc(6.f), ve, padd(veL, veR)), cwk(i, 0), pmul(lo2(ze[i]), cwk(i, 3)));
      const float2 c1 = pfma(padd(ve, veR), cwk(i, 1), pmul(hi2(ze[i]), cwk(i, 3)));
      const float2 c2 = pfma(pfma(bc(6.f), vo, padd(voL, voR)), cwk(i, 1), pmul(lo2(zo[i]), cwk(i, 3)));
      const float2 c3 = pfma(padd(vo, voR), cwk(i, 2), pmul(hi2(zo[i]), cwk(i, 3)));
      sts4(cb + i * 1024, cat4(c0, c1));
      sts4(cb + i * 1024 + 512, cat4(c2, c3));
    }
    if (DO_G) {  // g of the pair for the order sums
      const uint32_t gb = gbrow + gbo + q * 512;
      sts2(gb, lo2(gg));
      sts2(gb + 256, hi2(gg));
    }
    ++q;
  }

  // Order sums (Eq. 14) of the batch of cnt fine row pairs just completed
  // (own pairs n0 .. n0+cnt-1): per pixel p = tid + j * 32 nw (pair q = p/128,
  // row r, fine column f)
  //   S = sum_k a_k Im(e^{-i k theta} V_k) = sum_k (c_cos,k cos k theta + c_sin,k sin k theta),
  // theta = w_1 g, from the coefficient pairs c_k in C and g in Gb, by
  // Clenshaw's recurrence (descending k: b_k = c_k + 2 cos theta b_{k+1} - b_{k+2};
  // see k_apply_cl), stored into D_l.  Between two CTA barriers: C / Gb are
  // complete before, consumed after.
  // Batch bt (own pairs 3 bt ..) in buffer bt % NBUF.  NBUF = 2: wait until
  // every warp has written its coefficients (full), release the buffer
  // after reading it (empty); the pixel slots rotate by 4 warps per batch so
  // the idle quarter (384 pixels, 512 threads) moves around.  NBUF = 1: two
  // CTA barriers.
  __device__ __forceinline__ void order_sum(int bt, int cnt) {
    const int n0 = L::NB * bt;
    const int ub = L::NBUF == 2 ? (bt & 1) : 0;
    if (L::NBUF == 2) mbar_wait_u32(bars + 8 * ub, (bt >> 1) & 1);
    else bar_sync_id(FUSE_BAR, blockDim.x);
    if (!(P.exp & 1)) {
      const int KL = kl();
      const uint32_t cbase = sbase_ + ub * L::c_buf(KL);
      const int goff = L::g_off(KL) + ub * L::g_buf(KL);
      const int row0 = 2 * (o0 + n0);
      const int slot = L::NBUF == 2 ? (warp + 4 * bt) % (blockDim.x / 32) : warp;
#pragma unroll 1
      for (int p = slot * 32 + lane; p < cnt * 128; p += blockDim.x) {
        const int q = p >> 7, r = (p >> 6) & 1, f = p & 63;
        const float g = lds1(sbase_ + goff + ((q * 2 + r) * 64 + f) * 4);
        float sn, c1;
        sincos_turns(g, P.invT, &sn, &c1);
        const float2 tc = bc(2.f * c1);
        float2 b1 = make_float2(0.f, 0.f), b2 = b1;
        uint32_t a = cbase + ((q * KL + KL - 1) * 2 + r) * 512 + f * 8;
        float res;
#if FLLF_FUSE_SPLIT
        if (KT > 0 && (KT & 1) == 0 && P.kbase == 1) {
          // two independent half-length chains in phi = 2 theta (half the
          // dependent latency between the batch barriers):
          //   even k = 2j, j = 1..KT/2:  b_1 cos phi - b_2 + b_1' sin phi
          //   odd  k = 2j+1 = j phi + theta, j = 0..KT/2-1: Clenshaw with
          //   F_j = cos(j phi + theta), F_{-1} = F_0 = cos theta (sin: -G_{-1} = G_0),
          //   sum = (b_0 - b_1) cos theta + (b_0' + b_1') sin theta
          const float c2 = fmaf(c1, c1, -sn * sn), s2 = 2.f * sn * c1;
          const float2 tc2 = bc(2.f * c2);
          float2 e1 = make_float2(0.f, 0.f), e2 = e1, q1 = e1, q2 = e1;
#pragma unroll
          for (int t = 0; t < KT / 2; ++t) {
            const float2 ce = lds2(a - (2 * t) * 1024), co = lds2(a - (2 * t + 1) * 1024);
            const float2 ne = pfma(tc2, e1, padd(ce, pneg(e2)));
            const float2 no = pfma(tc2, q1, padd(co, pneg(q2)));
            e2 = e1;
            e1 = ne;
            q2 = q1;
            q1 = no;
          }
          res = fmaf(e1.x, c2, fmaf(e1.y, s2, -e2.x)) + fmaf(q1.x - q2.x, c1, (q1.y + q2.y) * sn);
        } else
#endif
        {
        int k = KL;
#pragma unroll(KT > 0 ? 8 : 1)
        for (; k >= 4; k -= 4, a -= 4096) {
          const float2 c3 = lds2(a), c2 = lds2(a - 1024), c1v = lds2(a - 2048), c0 = lds2(a - 3072);
          b2 = pfma(tc, b1, padd(c3, pneg(b2)));
          b1 = pfma(tc, b2, padd(c2, pneg(b1)));
          b2 = pfma(tc, b1, padd(c1v, pneg(b2)));
          b1 = pfma(tc, b2, padd(c0, pneg(b1)));
        }
#pragma unroll 1
        for (; k > 0; --k, a -= 1024) {
          const float2 nb2 = pfma(tc, b1, padd(lds2(a), pneg(b2)));
          b2 = b1;
          b1 = nb2;
        }
        // b1 = b_{k0}, b2 = b_{k0+1}
        if (P.kbase == 1) {
          res = fmaf(b1.x, c1, fmaf(b1.y, sn, -b2.x));
        } else {
          float sk, ck;
          sincos_turns_n(g, P.invT, P.kbase, &sk, &ck);
          const float cm = fmaf(ck, c1, sk * sn), sm = fmaf(sk, c1, -ck * sn);  // e^{i (k0-1) theta}
          res = fmaf(b1.x, ck, fmaf(b1.y, sk, -fmaf(b2.x, cm, b2.y * sm)));
        }
        }
        const int row = row0 + 2 * q + r;
        const int col = 2 * (FUSE_COLS * cb_ - 2) + f;  // lanes 2..29 own f in [4, 60)
        if (f >= 4 && f < 60 && col < P.Wf && row < Hf) {
          float* sp = dbase + (long long)row * gpitch + col;
          FLLF_DBG_STORE(P, sp, 4);
          *sp = res;
        }
      }
    }
    if (L::NBUF == 2) mbar_arrive_u32(bars + 16 + 8 * ub);
    else bar_sync_id(FUSE_BAR, blockDim.x);
  }

  // NBUF = 2: before the first coefficients of batch bt, wait until the order
  // sums of batch bt-2 (same buffer) have read it; after the last, publish.
  __device__ __forceinline__ void begin_batch(int bt) {
    if (L::NBUF != 2) return;
    const int ub = bt & 1;
    if (bt >= 2) mbar_wait_u32(bars + 16 + 8 * ub, ((bt >> 1) - 1) & 1);
    cbo = ub * L::c_buf(kl());
    gbo = ub * L::g_buf(kl());
  }
  __device__ __forceinline__ void end_batch(int bt) {
    if (L::NBUF == 2) mbar_arrive_u32(bars + 8 * (bt & 1));
  }

  // One step t (pair P_{o0-2+t}): Wm, W0 = coarse rows j-3, j-2; Wn <- row
  // j-1 (emitted); De/Do/Dg <- this pair's Z_l (and G_l); Dm2 = pair j-2's.
  template <bool EMIT, bool OWN, bool VSTEP, bool VC>
  __device__ __forceinline__ void step(int t, int np, int& q, float2 (&Wm)[NC], float2 (&W0)[NC],
                                       float2 (&Wn)[NC], float4 (&De)[NC], float4 (&Do)[NC], float4 (&Dg),
                                       const float4 (&Dm2e)[NC], const float4 (&Dm2o)[NC], const float4& Dm2g) {
    if (t + PD < np) issue();
    cp_async_commit();
    Pair d;
    if (PIPE) {  // pair t was read one step ahead; read pair t+1 now
      d = nxt;
      cp_async_wait<PD - 1>();
      if (t + 1 < np) read(nxt);
    } else {
      cp_async_wait<PD>();
      read(d);
    }
    if (EMIT) emit<OWN>(d, Wn);
    if (VSTEP) vstep(d);
    if (VC) {
      if (P.exp & 2) {
        ++q;
      } else {
        coef(Wm, W0, Wn, Dm2e, Dm2o, Dm2g, t - 4, q);
      }
    }
#pragma unroll
    for (int i = 0; i < NZ; ++i) {
      De[i] = d.ze[i];
      Do[i] = d.zo[i];
    }
    if (DO_G) Dg = cat4(d.ge, d.go);
  }

  // Stream pairs P_{o0-2} .. P_{o0+R+1} (t = 0 .. R+3):
  //   t = 0, 1: accumulate; t = 2: emit the halo row o0-1; t = 3: emit row o0;
  //   t = 4 .. R+2: emit row o0-3+t, coefficients of own pair t-4;
  //   t = R+3: emit the halo row o0+R, coefficients of the last own pair.
  // The coarse window (rows j-3, j-2, j-1) and the delay line (pairs j-2,
  // j-1, j) rotate with period 3 by renaming: phase t % 3 uses
  //   0: (CB, CC -> CA; A <- pair, B = pair j-2)
  //   1: (CC, CA -> CB; B <- pair, C = pair j-2)
  //   2: (CA, CB -> CC; C <- pair, A = pair j-2)
  __device__ __forceinline__ void run() {
    const int np = R + 4;
#pragma unroll
    for (int i = 0; i < PD; ++i) {
      if (i < np) issue();
      cp_async_commit();
    }
    if (PIPE) {
      cp_async_wait<PD - 1>();
      read(nxt);
    }
    float2 CA[NC], CB[NC], CC[NC];
    float4 ZAe[NC], ZAo[NC], ZBe[NC], ZBo[NC], ZCe[NC], ZCo[NC];
    float4 GA = make_float4(0.f, 0.f, 0.f, 0.f), GB = GA, GC = GA;
#pragma unroll
    for (int i = 0; i < NZ; ++i) {
      CA[i] = CB[i] = CC[i] = make_float2(0.f, 0.f);
      ZAe[i] = ZAo[i] = ZBe[i] = ZBo[i] = ZCe[i] = ZCo[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    int q = 0;
#define FUSE_PH0 q, CB, CC, CA, ZAe, ZAo, GA, ZBe, ZBo, GB
#define FUSE_PH1 q, CC, CA, CB, ZBe, ZBo, GB, ZCe, ZCo, GC
#define FUSE_PH2 q, CA, CB, CC, ZCe, ZCo, GC, ZAe, ZAo, GA
    step<false, false, true, false>(0, np, FUSE_PH0);
    step<false, false, true, false>(1, np, FUSE_PH1);
    step<true, false, true, false>(2, np, FUSE_PH2);
    step<true, true, true, false>(3, np, FUSE_PH0);
    int t = 4, bt = 0, it = 0;
#pragma unroll 1
    for (; t + 2 <= R + 2; t += 3) {  // own pairs t-4 .. t-2; NBI iterations per batch bt
      if (it == 0) {
        q = 0;
        begin_batch(bt);
      }
      step<true, true, true, true>(t, np, FUSE_PH1);
      step<true, true, true, true>(t + 1, np, FUSE_PH2);
      step<true, true, true, true>(t + 2, np, FUSE_PH0);
      if (++it == L::NBI) {
        end_batch(bt);
        // NBUF = 2: the order sums run one batch behind the coefficients
        if (L::NBUF == 2) {
          if (bt > 0) order_sum(bt - 1, L::NB);
        } else {
          order_sum(bt, L::NB);
        }
        ++bt;
        it = 0;
      }
    }
    // 0..2 steady steps remain (phase 1 first), then the last step t = R+3:
    // the last (partial) batch, after the it iterations already in it
    const int rem = R + 3 - t;
    if (it == 0) {
      q = 0;
      begin_batch(bt);
    }
    if (rem == 0) {
      step<true, false, false, true>(t, np, FUSE_PH1);
    } else if (rem == 1) {
      step<true, true, true, true>(t, np, FUSE_PH1);
      step<true, false, false, true>(t + 1, np, FUSE_PH2);
    } else {
      step<true, true, true, true>(t, np, FUSE_PH1);
      step<true, true, true, true>(t + 1, np, FUSE_PH2);
      step<true, false, false, true>(t + 2, np, FUSE_PH0);
    }
    end_batch(bt);
    if (L::NBUF == 2 && bt > 0) order_sum(bt - 1, L::NB);
    order_sum(bt, FUSE_NB * it + rem + 1);
#undef FUSE_PH0
#undef FUSE_PH1
#undef FUSE_PH2
    cp_async_wait<0>();
  }
};

template <int NC, int PD, bool EDGE, bool ROWS_IN, int KT>
__device__ __forceinline__ void fuse_run(const FuseParams& P, int cb, int o0, int R, int frame, int nw, int warp,
                                         uint32_t sbase, uint32_t bars) {
  if (FuseLayout<NC, PD>::GW) {
    if (warp == nw) {  // the G warp
      FuseWarp<NC, PD, EDGE, true, ROWS_IN, KT, false> w(P, cb, o0, R, frame, nw, warp, sbase, bars);
      w.run();
    } else {
      FuseWarp<NC, PD, EDGE, false, ROWS_IN, KT> w(P, cb, o0, R, frame, nw, warp, sbase, bars);
      w.run();
    }
  } else if (warp == 0 && !(P.exp & 4)) {  // (exp bit 4, timing only: no warp builds G)
    FuseWarp<NC, PD, EDGE, true, ROWS_IN, KT> w(P, cb, o0, R, frame, nw, warp, sbase, bars);
    w.run();
  } else {
    FuseWarp<NC, PD, EDGE, false, ROWS_IN, KT> w(P, cb, o0, R, frame, nw, warp, sbase, bars);
    w.run();
  }
}

// KT > 0: the plan's order count at compile time (16 or 8; the order sums'
// Clenshaw loop unrolls completely, the layout offsets fold)
template <int NC, int PD, int KT = 0>
__global__ void __launch_bounds__((FUSE_MAX_WARPS + (FuseLayout<NC, PD>::GW ? 1 : 0)) * 32, 1)
    k_fuse(const __grid_constant__ FuseParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[4];  // NBUF = 2: full[2], empty[2] of the order-sum buffers
  if (FuseLayout<NC, PD>::NBUF == 2) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) mbar_init(&bar[i], blockDim.x);
    }
    __syncthreads();
  }
  pdl_wait();     // level l (G_l, Z_l) is complete
  pdl_trigger();  // let the next level's kernel get scheduled
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bars = smem_u32(bar);
  const int cb = blockIdx.x;
  const int o0 = blockIdx.y * P.rows_per_strip;
  const int R = min(P.rows_per_strip, P.Hc - o0);
  const int frame = blockIdx.z;
  const int nw = (KT > 0 ? KT : P.KL) / NC;
  const int warp = threadIdx.x >> 5;
  // all 64 fine columns of the warp inside the row: no per-lane reflection
  const bool interior = cb >= 1 && 2 * FUSE_COLS * cb + 60 <= P.Wf;
  // pairs o0-2 .. o0+R+1 inside the frame: no row reflection
  const bool rows_in = o0 >= 2 && 2 * (o0 + R + 1) + 1 < P.Hf;
  if (interior) {
    if (rows_in) fuse_run<NC, PD, false, true, KT>(P, cb, o0, R, frame, nw, warp, sbase, bars);
    else fuse_run<NC, PD, false, false, KT>(P, cb, o0, R, frame, nw, warp, sbase, bars);
  } else {
    if (rows_in) fuse_run<NC, PD, true, true, KT>(P, cb, o0, R, frame, nw, warp, sbase, bars);
    else fuse_run<NC, PD, true, false, KT>(P, cb, o0, R, frame, nw, warp, sbase, bars);
  }
}

// D_l += up(D_{l+1}) (polyphase up-sampling with the border rule of upmap):
// one thread per 2 x 2 coarse pixels = a 4 x 4 block of fine pixels (16
// coarse loads for 4 coarse pixels, four independent 16-byte read-modify-
// writes of the fine rows).  Same arithmetic per fine pixel as one thread
// per coarse pixel: vertical (x_{r-1} + 6 x_r + x_{r+1}) / 8 | (x_r + x_{r+1}) / 2,
// then the same horizontally.
__global__ void __launch_bounds__(128) k_collapse(const CollapseParams P) {
  pdl_wait();  // D_{l+1} is complete
  pdl_trigger();
  const int x0 = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int r0 = 2 * blockIdx.y;
  if (x0 >= P.Wc) return;
  const float* dc = P.coarse + blockIdx.z * P.cfstride;
  float* df = P.fine + blockIdx.z * P.ffstride;
  int xs[4], rs[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    xs[j] = upmap(x0 - 1 + j, P.Wc, P.Wf);
    rs[j] = upmap(r0 - 1 + j, P.Hc, P.Hf);
  }
  float d[4][4];  // [coarse row r0-1+i][coarse column x0-1+j]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) d[i][j] = __ldg(dc + (long long)rs[i] * P.cpitch + xs[j]);
  // vertical: fine rows 2 r0 + t, t = 0..3 (coarse rows r0, r0 + 1; even / odd)
  float v[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[0][j] = fmaf(6.f, d[1][j], d[0][j] + d[2][j]) * 0.125f;
    v[1][j] = (d[1][j] + d[2][j]) * 0.5f;
    v[2][j] = fmaf(6.f, d[2][j], d[1][j] + d[3][j]) * 0.125f;
    v[3][j] = (d[2][j] + d[3][j]) * 0.5f;
  }
  const bool vec = ((reinterpret_cast<uintptr_t>(df) & 15) == 0) && ((P.fpitch & 3) == 0) && 2 * x0 + 3 < P.Wf;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int row = 2 * r0 + t;
    if (row >= P.Hf) break;
    const float o0 = fmaf(6.f, v[t][1], v[t][0] + v[t][2]) * 0.125f;
    const float o1 = (v[t][1] + v[t][2]) * 0.5f;
    const float o2 = fmaf(6.f, v[t][2], v[t][1] + v[t][3]) * 0.125f;
    const float o3 = (v[t][2] + v[t][3]) * 0.5f;
    float* fp = df + (long long)row * P.fpitch + 2 * x0;
    if (vec) {
      FLLF_DBG_STORE(P, fp, 16);
      float4 q = *reinterpret_cast<float4*>(fp);
      q.x += o0;
      q.y += o1;
      q.z += o2;
      q.w += o3;
      *reinterpret_cast<float4*>(fp) = q;
    } else {
      const float o[4] = {o0, o1, o2, o3};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (2 * x0 + u < P.Wf) {
          FLLF_DBG_STORE(P, fp + u, 4);
          fp[u] += o[u];
        }
    }
  }
}

constexpr int kFuseSmemMax = 227 * 1024 - 64;  // (static shared: the kernel's mbarriers)
// ring depth (pairs ahead): 4 with one order per warp, 2 with two (shared memory)
#ifndef FLLF_FUSE_PD1
#define FLLF_FUSE_PD1 6
#endif
template <int NC>
constexpr int fuse_pd() {
  return NC == 1 ? FLLF_FUSE_PD1 : 2;
}

template <int NC>
cudaError_t launch_fuse_nc(const FuseParams& p0, int batch, cudaStream_t s, bool pdl) {
  constexpr int PD = fuse_pd<NC>();
  FuseParams p = p0;
  const int bx = (p.Wc + FUSE_COLS - 1) / FUSE_COLS;
  // strip height: long strips amortise the 8 halo fine rows (pairs o0-2,
  // o0-1, o0+R, o0+R+1); shorter ones only while the grid would leave SMs idle
  static const int rmax = [] {
    const char* e = std::getenv("FLLF_FUSE_RMAX");
    const int v = e ? std::atoi(e) : 64;
    return v >= 1 ? v : 64;
  }();
  static const int target_ctas = [] {
    const char* e = std::getenv("FLLF_FUSE_CTAS");
    const int v = e ? std::atoi(e) : 148 * 4;
    return v >= 1 ? v : 148 * 4;
  }();
  int R = std::min(rmax, p.Hc);
  while (R > 4 && (long long)bx * ((p.Hc + R - 1) / R) * batch < target_ctas) R = (R + 1) / 2;
  p.rows_per_strip = R;
  static const int exp = [] {  // A/B experiments (timing only): 1 = no order sums, 2 = no coefficients, 4 = no G warp
    const char* e = std::getenv("FLLF_FUSE_EXP");
    return e ? std::atoi(e) : 0;
  }();
  p.exp = exp;
  const int smem = FuseLayout<NC, PD>::smem(p.KL);
  dim3 grid(bx, (p.Hc + R - 1) / R, batch);
  const dim3 block(32 * FuseLayout<NC, PD>::warps(p.KL));
  static DeviceFlags attr0, attr8, attr16;
  cudaError_t e;
  if (NC == 1 && p.KL == 16) {
    if ((e = smem_opt_in(k_fuse<NC, PD, 16>, kFuseSmemMax, attr16)) != cudaSuccess) return e;
    return launch_ex(k_fuse<NC, PD, 16>, grid, block, smem, s, pdl, p);
  }
  if (NC == 1 && p.KL == 8) {
    if ((e = smem_opt_in(k_fuse<NC, PD, 8>, kFuseSmemMax, attr8)) != cudaSuccess) return e;
    return launch_ex(k_fuse<NC, PD, 8>, grid, block, smem, s, pdl, p);
  }
  if ((e = smem_opt_in(k_fuse<NC, PD>, kFuseSmemMax, attr0)) != cudaSuccess) return e;
  return launch_ex(k_fuse<NC, PD>, grid, block, smem, s, pdl, p);
}

}  // namespace

int fuse_orders_per_warp(int KL) {
  if (KL <= FUSE_MAX_WARPS && FuseLayout<1, fuse_pd<1>()>::smem(KL) <= kFuseSmemMax) return 1;
  if (KL % 2 == 0 && KL / 2 <= FUSE_MAX_WARPS && FuseLayout<2, fuse_pd<2>()>::smem(KL) <= kFuseSmemMax) return 2;
  return 0;
}

cudaError_t launch_fuse(const FuseParams& p, int batch, cudaStream_t s, bool pdl) {
  switch (fuse_orders_per_warp(p.KL)) {
    case 2: return launch_fuse_nc<2>(p, batch, s, pdl);
    case 1: return launch_fuse_nc<1>(p, batch, s, pdl);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_collapse(const CollapseParams& p, int batch, cudaStream_t s, bool pdl) {
  dim3 grid(((p.Wc + 1) / 2 + 127) / 128, (p.Hc + 1) / 2, batch);
  return launch_ex(k_collapse, grid, dim3(128), 0, s, pdl, p);
}

}  // namespace fllf
