// Internal structures shared by the host code (fllf_host.cpp) and the kernels
// (fllf_kernels.cu).  Not part of the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fllf.h"

namespace fllf {

// Z planes carry ZHALO float2 columns left of column 0 and ZPAD columns of
// padding right of column W-1.  Column -1 holds x_1 and column W holds
// x_{W-1} or x_{W-2} (the up-sampling border rule for the finer level's width
// parity), written by the producing k_build; the apply kernel then stages
// whole, 16-byte-aligned row segments with TMA bulk copies and never maps a
// column index.
constexpr int ZHALO = 4;
constexpr int ZPAD = 128;

// One stored pyramid level l >= 1 (all frames).  Real planes (G, D, map
// pyramids) have `pitch` floats per row; complex planes Z_{l,k} have `zpitch`
// float2 per row, each float2 = (S~, C~) = (Im, Re) of Z = C~ + i S~.
struct DevLevel {
  int H, W;
  int pitch;           // floats per row of the real planes
  int zpitch;          // float2 per row of the complex planes (incl. halo + pad)
  float* G;            // G_l[I]
  float* D;            // D_l = O_l - G_l (collapse from level l of the output pyramid)
  float2* Z;           // Z_{l,k} column 0 of row 0, local orders k = 0..KL-1
  float* MS;           // G_l[sigma_r map]   (MAPS mode, shared by frames)
  float* MM;           // G_l[m map]
  long long fstride_r; // floats per frame for real planes  (H*pitch)
  long long kstride_z; // float2 per k plane                  (H*zpitch)
  long long fstride_z; // float2 per frame                    (KL*H*zpitch)
};

// A caller-owned full-resolution real plane (level 0).
struct DevImage {
  const float* p;
  int H, W;
  long long pitch;     // floats per row
  long long fstride;   // floats per frame
};

struct BuildParams {
  DevImage img;        // build0: the image (level 0); map build at level 0: sigma map
  DevImage img2;       // map build at level 0: m map
  DevLevel src;        // level l (l >= 1) source
  DevLevel dst;        // level l+1 destination
  int Hf, Wf, Hc, Wc;  // fine (l) and coarse (l+1) dims
  int KL;              // local number of orders
  int kbase;           // global order of local channel 0 (k_begin, 1-based)
  int nchunks;         // complex channel chunks per frame
  int rows_per_strip;  // coarse rows per warp
  int maps;            // 1: build the (sigma, m) map pyramids instead of G/Z
  // maps: floats between the map-pyramid slots of consecutive map pairs
  // (blockIdx.z = map index; fllf_apply_maps), at the source / destination level
  long long ms_stride_src, ms_stride_dst;
  float invT;          // 1/T
  // Row bands (NEXT-1; full frame: o_begin = 0, o_end = Hc, fr_lo = 0,
  // fr_hi = Hf-1).  Rows are GLOBAL level indices everywhere (the plane
  // pointers are offset so that a global row addresses the band's rows);
  // outputs are the coarse rows [o_begin, o_end); fine-row reads are clamped
  // to the allocated rows [fr_lo, fr_hi] (band + halo), which only ever
  // changes rows that feed no stored output.
  int o_begin, o_end;
  int fr_lo, fr_hi;
  const char* dbg_lo;  // FLLF_DEBUG_BOUNDS builds: every global store must land in [dbg_lo, dbg_hi)
  const char* dbg_hi;
};

struct ApplyParams {
  // TMA tensor maps (3-D: float columns x rows x (frame, order) planes) of the
  // coarse level's Z planes (box 128 floats x 6 rows) and the fine level's
  // (box 256 x 8): one tensor copy per order stage for interior tiles
  // (k_apply_cl); use_tm = 0 -> per-row bulk copies only.  Every map covers
  // only the rows its level stores (row-band plans: al .. ah; the image: the
  // rows the band reads), so its row coordinate is the global row minus
  // cr_lo (coarse level: tm_coarse, tm_d) or fr_lo (fine level / image:
  // tm_fine, tm_g) -- no map addresses memory outside its allocation.
  CUtensorMap tm_coarse;
  CUtensorMap tm_fine;
  CUtensorMap tm_g;    // g rows of the tile header: I (level 0) or G_l, box 120 floats x 8 rows
  CUtensorMap tm_d;    // D_{l+1} rows of the tile header, box 68 floats x 6 rows
  int use_tm;
  int use_tm_g, use_tm_d;
  DevImage img;        // level-0 input image I (LEVEL0 kernels)
  float* out;          // level-0 output O (LEVEL0 kernels)
  long long out_pitch; // floats
  long long out_fstride;
  DevImage smap, mmap; // MAPS at level 0: user maps (fstride 0)
  DevLevel fine;       // level l (for l >= 1)
  DevLevel coarse;     // level l+1
  int Hf, Wf, Hc, Wc;
  int KL, kbase;
  int include_base;
  int wait_first;      // PDL: wait for the preceding grid before any global read
  float invT;          // 1/T
  float c0;            // MAPS: 2 omega_1 sqrt(2 pi) / T
  float hq;            // MAPS: omega_1^2 / 2
  float a[FLLF_MAX_K]; // uniform a_k (SCALAR/COEFFS), local order index
  // uniform weights per local order k as broadcast pairs for packed math:
  // [0] = (a, a), [1] = -(a/64) (even row, even col), [2] = -(a/16) (mixed),
  // [3] = -(a/4) (odd row, odd col): the polyphase up-sampling scales folded
  // into a_k
  float2 wk[FLLF_MAX_K][4];
  // Clenshaw form (k_apply_cl): per local order k the coefficient pairs that
  // turn an up-sampled (Im, Re) value into (c_cos, c_sin) of the trig series
  // sum_k (c_cos cos k theta + c_sin sin k theta):
  // [0] = (-a/64, a/64) even row, even col; [1] = (-a/16, a/16) mixed;
  // [2] = (-a/4, a/4) odd row, odd col; [3] = (a, -a) same-level Z (l >= 1).
  // MAPS: [0] = (k^2, log2 k) of the global order k (a_k is per pixel).
  float2 cw[FLLF_MAX_K][4];
  // Row bands (see BuildParams): tiles cover the coarse rows [r_begin, r_end);
  // coarse-plane (Z_{l+1}, D_{l+1}) reads are clamped to [cr_lo, cr_hi],
  // fine-plane reads (Z_l, G_l or I) to [fr_lo, fr_hi]; tensor-map copies are
  // used only for boxes inside those ranges.
  int r_begin, r_end;
  int cr_lo, cr_hi, fr_lo, fr_hi;
  int accumulate;      // level 0: atomically add the output into out (fllf_apply_accumulate)
  // Frame index of a tile (T.frame) for the G / image planes (gz) and the Z
  // planes (zz): 1 = per frame; 0 = shared -- MAPS over a batch of map pairs
  // (fllf_apply_maps), where T.frame is the pair and only D, the map planes
  // (ms_fstride floats apart at the fine level; smap / mmap .fstride at level
  // 0) and the output differ between tiles of different pairs.
  int gz, zz;
  long long ms_fstride;
  const char* dbg_lo;  // FLLF_DEBUG_BOUNDS builds: every global store must land in [dbg_lo, dbg_hi)
  const char* dbg_hi;
};

// Materialise-once design F (fllf_fused.cu).  One
// launch per level l >= 1 builds level l+1 from level l (G_{l+1}, Z_{l+1}, as
// k_build) AND evaluates the level-l order sum
//   S_l = sum_k a_k Im(e^{-i w_k g} (Z_{l,k} - up Z_{l+1,k})),  g = G_l,
// from the same staged rows, storing S_l into the D_l plane; every Z plane
// is then written once and read once.
struct FuseParams {
  DevLevel src;        // level l: G_l, Z_l read; S_l written to src.D
  DevLevel dst;        // level l+1: G_{l+1}, Z_{l+1} written
  int Hf, Wf, Hc, Wc;  // dims of levels l and l+1
  int KL, kbase;       // local orders, global order of local order 0
  int rows_per_strip;  // coarse rows per CTA
  int exp;             // A/B experiments (FLLF_FUSE_EXP; 0 in production)
  float invT;          // 1/T
  // Clenshaw coefficient pairs per local order, as ApplyParams::cw
  float2 cw[FLLF_MAX_K][4];
  const char* dbg_lo;  // FLLF_DEBUG_BOUNDS builds: every global store must land in [dbg_lo, dbg_hi)
  const char* dbg_hi;
};

// Collapse step of design F: fine += up(coarse) on the D planes of two
// consecutive levels (D_l = S_l + up(D_{l+1}); Eq. 4).
struct CollapseParams {
  const float* coarse;  // D_{l+1}
  long long cpitch, cfstride;
  float* fine;          // D_l (in place)
  long long fpitch, ffstride;
  int Hf, Wf, Hc, Wc;
  const char* dbg_lo;
  const char* dbg_hi;
};

// Colour conversion (fllf_color.cu): three planes in, three planes out, all
// with the same row pitch (floats).
struct ColorParams {
  const float* src[3];
  float* dst[3];
  int H, W;
  long long pitch;
};

// Variance-driven gain map (fllf_color.cu).
struct GainParams {
  const float* y;
  long long y_pitch;
  float* m;
  long long m_pitch;
  int H, W, radius;
  double m_lo, m_hi, inv_vref;
};

cudaError_t launch_rgb_to_yuv(const ColorParams& p, cudaStream_t s);
cudaError_t launch_yuv_to_rgb(const ColorParams& p, cudaStream_t s);
cudaError_t launch_gain_map(const GainParams& p, cudaStream_t s);
cudaError_t launch_fill(float* ptr, long long pitch, int H, int W, float v, cudaStream_t s);

// Naive LLF ground truth (fllf_naive.cu), one launch per level.
struct NaiveParams {
  const float* img;     // level-0 image
  long long img_pitch;  // floats
  const float* G[FLLF_MAX_LEVELS];  // G_l[I] planes (l >= 1)
  long long gpitch[FLLF_MAX_LEVELS];
  int Hs[FLLF_MAX_LEVELS + 1], Ws[FLLF_MAX_LEVELS + 1];
  float* L[FLLF_MAX_LEVELS];        // output coefficient planes L_l[O]
  long long lpitch[FLLF_MAX_LEVELS];
  int level;            // l of this launch
  int mode;             // 0: exact Gaussian remap; 1: truncated series r_K
  int K;
  double m, inv2s2;     // exact remap: m, 1/(2 sigma_r^2)
  double a[FLLF_MAX_K], omega[FLLF_MAX_K];  // series remap
};
cudaError_t launch_naive_level(const NaiveParams& p, cudaStream_t s);
cudaError_t launch_collapse_up(float* fine, long long fpitch, const float* coarse, long long cpitch, int Hf, int Wf,
                               int Hc, int Wc, cudaStream_t s);

// Kernel launchers (fllf_kernels.cu).  Return cudaGetLastError() after launch.
// pdl: launch with programmatic stream serialization (the kernel may start
// while its predecessor is still running; it synchronises with griddepcontrol)
cudaError_t launch_build(const BuildParams& p, int level_src, int batch, cudaStream_t s, bool pdl);
cudaError_t launch_apply(const ApplyParams& p, int level_fine, bool has_d, bool maps, int batch,
                         cudaStream_t s, bool pdl);

// Design F (fllf_fused.cu).  fuse_orders_per_warp: the order chunk per warp
// for KL local orders (0: no supported split, the caller keeps design AB).
int fuse_orders_per_warp(int KL);
cudaError_t launch_fuse(const FuseParams& p, int batch, cudaStream_t s, bool pdl);
cudaError_t launch_collapse(const CollapseParams& p, int batch, cudaStream_t s, bool pdl);

}  // namespace fllf
