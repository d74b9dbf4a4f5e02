/*
 * libfllf -- B200-native Fourier local Laplacian filtering (C ABI).
 *
 * Implements the data-parallel hot path of "Gaussian Fourier Pyramid for
 * Local Laplacian Filter" (Sumiya, Otsuka, Maeda, Fukushima, arXiv 2206.04681).
 * Citations "P:n" are lines of the paper's text, given with the
 * section / equation they fall in.
 *
 * What is computed:
 *   omega_k = 2 pi k / T,  alpha_k = sigma_r sqrt(2 pi)/T exp(-(omega_k sigma_r)^2/2),
 *   alpha~_k = 2 sigma_r^2 alpha_k omega_k,  a_k = m alpha~_k     (Eq. 9-11)
 *   G_l = Gaussian pyramid of I (Eq. 1),
 *   Z_{l,k} = C~_{l,k} + i S~_{l,k} = G_l[cos w_k I] + i G_l[sin w_k I]
 *   L_l[O] = L_l[I] + sum_k a_k ( cos(w_k g) L_l[S~_k] - sin(w_k g) L_l[C~_k] ),
 *            g = G_l[I] pointwise, l < l_max;  L_lmax[O] = G_lmax[I]    (Eq. 14)
 *   O = collapse(L[O])                                                   (Eq. 4,  P:138-141)
 * with the enhancing remap sign r(i,g) = i + m (i-g) exp(-(i-g)^2/(2 sigma_r^2))
 * (reading R1).  Borders are reflect-101, sizes halve with ceil, the
 * up-sampling kernel is 2x the 5-tap binomial per axis (readings R2, R3, R5).
 *
 * Conventions for every entry point:
 *   - Images are fp32, row-major: pixel (x, y) of frame f lives at
 *     (char*)base + f*H*pitch_bytes + y*pitch_bytes + 4*x.  pitch_bytes = 0
 *     means W*4.  pitch_bytes must be >= W*4 and a multiple of 4.
 *   - Pointers prefixed d_ are DEVICE pointers on the plan's device; h_ are
 *     HOST pointers (pinned memory makes the copies asynchronous).
 *   - All work is enqueued asynchronously on the caller's stream `s`
 *     (a cudaStream_t; NULL = legacy default stream).  The caller keeps every
 *     buffer alive until that stream work has completed.
 *   - A plan owns all device workspace (the pyramids); it is bound to one
 *     device, is not thread-safe, and may be used by one stream at a time.
 *     Distinct plans may run concurrently on distinct streams.
 *   - No C++ exception crosses this boundary.  On failure the status code is
 *     returned and fllf_last_error_message() (thread-local) holds the detail;
 *     CUDA failures return FLLF_ERR_CUDA.
 *   - There is no CPU fallback: without a CUDA device every compute entry
 *     point returns FLLF_ERR_CUDA.
 */
#ifndef FLLF_H_
#define FLLF_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FLLF_API __attribute__((visibility("default")))
#else
#define FLLF_API
#endif

#define FLLF_MAX_K 32      /* maximum Fourier order K (2K+1 pyramids)          */
#define FLLF_MAX_LEVELS 16 /* maximum pyramid levels                            */

typedef struct fllf_plan_s* fllf_plan; /* opaque; owns the device workspace */

typedef enum {
  FLLF_OK = 0,
  FLLF_ERR_INVALID_ARGUMENT = 1, /* H,W<1; levels<2; K<1 or >FLLF_MAX_K; T<=0; sigma_r<=0;
                                    non-finite value; bad order range; batch<1         */
  FLLF_ERR_TOO_MANY_LEVELS = 2,  /* a dimension of the coarsest level would be < 3, or
                                    levels > FLLF_MAX_LEVELS                            */
  FLLF_ERR_OUT_OF_MEMORY = 3,    /* workspace allocation failed                         */
  FLLF_ERR_CUDA = 4,             /* a CUDA runtime call or kernel launch failed         */
  FLLF_ERR_NOT_BUILT = 5,        /* fllf_apply before fllf_build_fourier_pyramids       */
  FLLF_ERR_BAD_POINTER = 6,      /* NULL pointer, pitch < W*4 or not a multiple of 4    */
} fllf_status;

typedef enum {
  FLLF_SCALAR = 0, /* a_k = m alpha~_k from the plan's (sigma_r, m)   (Eq. 11)     */
  FLLF_COEFFS = 1, /* caller-given a_k, k = k_begin..k_end-1: any remap whose detail term
                      is odd in (i-g) with period T ("change the function by
                      switching only the coefficient")                                  */
  FLLF_MAPS = 2    /* per-pixel sigma_r(p), m(p) (Sec. III-B); at level l
                      the maps' Gaussian pyramids are used (reading R7)                 */
} fllf_apply_mode;

/* Full plan description (fllf_plan_create fills the defaults shown). */
typedef struct {
  int H, W;         /* frame size (pixels)                                             */
  int levels;       /* pyramid levels incl. the residual, >= 2 (l_max = levels-1) */
  int K;            /* Fourier order, 1..FLLF_MAX_K                                      */
  double T;         /* period of the expansion (Eq. 9)                        */
  double sigma_r;   /* remap range scale (Eq. 6)                                  */
  double m;         /* remap gain (Eq. 6; m > 0 enhances)                         */
  int batch;        /* frames per call, >= 1 (default 1); frames are contiguous          */
  int k_begin;      /* order range [k_begin, k_end), 1 <= k_begin < k_end <= K+1;        */
  int k_end;        /*   0,0 = all orders (default).  Order sharding across GPUs.        */
  int include_base; /* 1 (default): output = full O.  0: output = the partial collapse of
                       the range's Fourier terms only (no L[I], top level 0); summing the
                       partials of a partition of 1..K and adding I gives O (Eq. 4 is
                       linear).                                                           */
  int device;       /* CUDA device ordinal; -1 (default) = the current device            */
  int row_begin;    /* row band [row_begin, row_end) of the frame this plan computes      */
  int row_end;      /*   (NEXT-1, multi-GPU row split); 0,0 = the whole frame (default).
                       Both multiples of 2^(levels-1) (row_end may be H); batch must be
                       1.  Rows are global: d_img / d_out point at row row_begin, and
                       d_img must also hold the 2 rows above and below the band
                       (where they exist).  The pyramids are stored for the band plus
                       2 halo rows per side per level; the halo rows of the levels >= 1
                       are the neighbour bands' rows, exchanged by the caller between the
                       per-level calls (fllf_build_level / fllf_apply_level /
                       fllf_plan_band_plane).  SCALAR / COEFFS only.                    */
} fllf_plan_desc;

/* Per-apply arguments; NULL means FLLF_SCALAR. */
typedef struct {
  int mode;                /* fllf_apply_mode                                            */
  const double* a_k;       /* COEFFS: HOST array of (k_end - k_begin) values              */
  const float* d_sigma_r;  /* MAPS: DEVICE full-resolution sigma_r map (> 0), H x W      */
  const float* d_m;        /* MAPS: DEVICE full-resolution m map, H x W                  */
  size_t map_pitch_bytes;  /* MAPS: pitch of both maps (0 = W*4); maps are shared by all
                              frames of a batch                                           */
} fllf_apply_args;

/* Create a plan for H x W frames: validates the arguments (see fllf_status),
 * computes the level sizes (ceil-halving), allocates the pyramid workspace on
 * the device and converts the fp64 coefficients to fp32. */
FLLF_API fllf_status fllf_plan_create(int H, int W, int levels, int K, double T, double sigma_r,
                             double m, fllf_plan* out);
FLLF_API fllf_status fllf_plan_create_ex(const fllf_plan_desc* d, fllf_plan* out);

/* Destroy a plan and free its workspace.  NULL-safe; synchronises the device. */
FLLF_API fllf_status fllf_destroy(fllf_plan p);

/* Build the 2K+1 pyramids of P:262 for levels 1..l_max from d_img (batch
 * frames): G_l[I] and Z_{l,k} for the plan's order range.  Level 0 of the
 * Fourier pyramids is never stored: cos/sin(omega_k I) are formed on the fly
 * inside the first blur-and-decimate (north star; P:250 shows level 0 needs
 * only the up-sampled level-1 terms). */
FLLF_API fllf_status fllf_build_fourier_pyramids(fllf_plan p, const float* d_img, size_t pitch_bytes,
                                        void* s);

/* Product-sum + collapse (Eq. 14 + Eq. 4) from the pyramids of the most recent
 * build on this plan; writes O (or the partial output, include_base = 0) to
 * d_out.  `a` = NULL selects FLLF_SCALAR.  May be called many times per build
 * with different coefficients or maps.  Reads d_img of
 * that build again (level 0 needs I): the caller keeps it alive and unchanged. */
FLLF_API fllf_status fllf_apply(fllf_plan p, const fllf_apply_args* a, float* d_out,
                       size_t out_pitch_bytes, void* s);

/* n applies in MAPS mode (Sec. III-B: the pyramids do not depend on
 * the maps, "build once, apply many") with the map pairs (sigma_r_j, m_j),
 * j = 0..n-1, stacked at map_stride_bytes (0: H * map_pitch_bytes; a multiple
 * of 16) in d_sigma_r / d_m (each map H x W fp32, map_pitch_bytes per row,
 * 0 = W * 4; 16-byte aligned rows as fllf_apply(MAPS) needs for its TMA path),
 * outputs stacked at out_stride_bytes (0: one output = batch x H rows of
 * out_pitch_bytes) in d_out.  Output j equals fllf_apply(MAPS) with pair j,
 * bit for bit; the Gaussian pyramids of all n map pairs are built first, one
 * launch per level for all pairs (the plan keeps n pyramid slots), then the
 * applies run pair by pair.  Full-frame plans; FLLF_ERR_NOT_BUILT before a
 * build, FLLF_ERR_INVALID_ARGUMENT for n < 1, strides below one map / output
 * or row-band plans. */
FLLF_API fllf_status fllf_apply_maps(fllf_plan p, int n, const float* d_sigma_r, const float* d_m,
                                     size_t map_pitch_bytes, size_t map_stride_bytes, float* d_out,
                                     size_t out_pitch_bytes, size_t out_stride_bytes, void* s);

/* As fllf_apply (SCALAR / COEFFS, full-frame plans), but the level-0 result is
 * ADDED to d_out with hardware atomics instead of stored: the combine step of
 * order sharding (linearity of Eq. 4) fused into the apply's
 * epilogue.  d_out may be another GPU's buffer mapped through CUDA IPC
 * (fllf_ipc_open): every rank adds its partial output straight into the
 * owner's frame over NVLink, no separate reduce.  The caller zeroes d_out once
 * before the first partial and orders all partials before reading it; the
 * summation order is not fixed (fp32 atomics: results agree to rounding).
 * MAPS or row-band plans: FLLF_ERR_INVALID_ARGUMENT. */
FLLF_API fllf_status fllf_apply_accumulate(fllf_plan p, const fllf_apply_args* a, float* d_out,
                                           size_t out_pitch_bytes, void* s);

/* CUDA IPC plumbing for fllf_apply_accumulate across processes (host logic,
 * no kernels): fllf_ipc_alloc allocates `bytes` of device memory on the
 * current device and writes its FLLF_IPC_HANDLE_BYTES-byte IPC handle to
 * handle_out; fllf_ipc_open maps a handle from another process into this one
 * (peer access enabled lazily); fllf_ipc_close / fllf_ipc_free undo them.
 * Errors: FLLF_ERR_BAD_POINTER (NULL / 0 bytes), FLLF_ERR_OUT_OF_MEMORY,
 * FLLF_ERR_CUDA (the runtime refused, e.g. a handle from this same process). */
#define FLLF_IPC_HANDLE_BYTES 64
FLLF_API fllf_status fllf_ipc_alloc(size_t bytes, void** d_ptr, void* handle_out);
FLLF_API fllf_status fllf_ipc_free(void* d_ptr);
FLLF_API fllf_status fllf_ipc_open(const void* handle, void** d_ptr);
FLLF_API fllf_status fllf_ipc_close(void* d_ptr);

/* build + apply(SCALAR) in one call (the common one-shot filter).  Full-frame
 * plans with levels >= 3 run the materialise-once design F (DESIGN.md "Design
 * F"): each level-l >= 1 build step also evaluates the level-l order sum of
 * Eq. 14 from the rows it streams, so every pyramid plane of levels >= 1 is
 * written once and read once (the "2K+1 pyramids" cost of P:262-263); the
 * collapse (Eq. 4) follows over the real D planes, then the level-0 apply.
 * The result equals build + apply up to fp32 rounding order; the pyramids
 * (fllf_read_pyramid) are identical and a later fllf_apply on the plan works
 * as after fllf_build_fourier_pyramids.  FLLF_NO_FUSE=1 in the environment
 * (or an order count with no supported split) keeps the two-pass design AB.
 * The launch sequence is captured once into a CUDA graph (per plan,
 * input/output buffer pair and profiling flag) and replayed on `s`;
 * FLLF_NO_GRAPH=1 in the environment or fllf_plan_set_graphs(p, 0) launches
 * the kernels directly.  Row-band plans: FLLF_ERR_INVALID_ARGUMENT (use the
 * per-level calls). */
FLLF_API fllf_status fllf_filter(fllf_plan p, const float* d_img, size_t in_pitch_bytes, float* d_out,
                        size_t out_pitch_bytes, void* s);

/* End-to-end from HOST memory: copies the batch h_img -> device staging,
 * build, apply(SCALAR), copies the result -> h_out (dense W*4 pitch both).
 * Asynchronous on `s` (pinned host memory); synchronise `s` before reading h_out. */
FLLF_API fllf_status fllf_filter_host(fllf_plan p, const float* h_img, float* h_out, void* s);

/* Streaming end-to-end from HOST memory: nframes successive batches (each the
 * plan's B frames of H*W floats, dense W*4 pitch), batch i read from
 * h_in + i*in_stride_bytes and written to h_out + i*out_stride_bytes (a
 * stride of 0 reuses one buffer).  Three-stage pipeline on two internal copy
 * streams and `s`: the H2D copy of batch i+1 and the D2H copy of batch i-1
 * overlap the filter of batch i (double-buffered device staging owned by the
 * plan).  Asynchronous: `s` completes after the last result has reached the
 * host; work queued on `s` before the call is ordered before the first copy.
 * Host memory must be pinned for the copies to overlap.  Not for row-band
 * plans or inside a stream capture (FLLF_ERR_INVALID_ARGUMENT). */
FLLF_API fllf_status fllf_filter_host_frames(fllf_plan p, const float* h_in, size_t in_stride_bytes, float* h_out,
                                             size_t out_stride_bytes, int nframes, void* s);

/* Bench tooling: with a device buffer set, fllf_filter_host_frames writes it
 * (cudaMemsetAsync on `s`, inside the pipeline) before each batch's filter,
 * evicting the previous batch's data from L2.  bytes = 0 disables. */
FLLF_API fllf_status fllf_plan_set_l2_flush(fllf_plan p, void* d_buf, size_t bytes);

/* Host helper: omega_k and a_k = m alpha~_k for k = 1..K in fp64 (Eq. 9-11). */
FLLF_API fllf_status fllf_coefficients(int K, double T, double sigma_r, double m, double* omega_out,
                              double* a_out);

/* Host helper, Eq. 12: the period T minimising
 *   E_K(T) = erfc(pi sigma_r (2K+1) / T) + erfc((T - R) / sigma_r)
 * over T in [R, R + 12 sigma_r] (dense grid + golden-section refinement to
 * 1e-6); R is the number of tones (256 for 8-bit).  Reading R11: the
 * paper's sigma is sigma_r.  sigma_r = 30, K = 10 gives 405.5 (paper: 405.9,
 * P:296). */
FLLF_API fllf_status fllf_optimal_period(int K, double sigma_r, double R, double* T_out);

/* ---- Colour + variance-driven gain (Sec. IV, P:373-377:
 * "The degree of enhancement is determined according to the variance of the
 * pixels in a local window; the low variance is a small enhancement" and
 * "LLF is applied to the Y channel of the YUV color space, and the other
 * components are kept"; Sec. III-B, per-pixel m_p).  Readings
 * (R13-R16): YUV = BT.601 full-range YCbCr with zero-centred
 * chroma; local variance = population variance over the (2r+1)^2 window,
 * reflect-101 borders; m_p = m_lo + (m_hi - m_lo) min(1, v_p / v_ref);
 * sigma_r uniform (the plan's).
 *
 * Planar colour images: plane c of a 3-plane image lives at
 * (char*)base + c*H*pitch_bytes; rows as for grayscale images. */
#define FLLF_MAX_GAIN_RADIUS 32

typedef struct {
  int radius;      /* window half-size r, 0 <= r <= FLLF_MAX_GAIN_RADIUS          */
  double m_lo;     /* gain at zero variance (flat regions)                         */
  double m_hi;     /* gain at v_p >= v_ref                                         */
  double v_ref;    /* variance at which the gain saturates, > 0                    */
} fllf_gain_desc;

/* d_rgb -> d_yuv (3 planes each, device, same pitch; may not alias).
 * INVALID_ARGUMENT: H, W < 1.  BAD_POINTER: NULL or bad pitch. */
FLLF_API fllf_status fllf_rgb_to_yuv(const float* d_rgb, float* d_yuv, int H, int W, size_t pitch_bytes,
                                     void* s);
/* Inverse of fllf_rgb_to_yuv. */
FLLF_API fllf_status fllf_yuv_to_rgb(const float* d_yuv, float* d_rgb, int H, int W, size_t pitch_bytes,
                                     void* s);
/* Gain map m_p from the local variance of d_y (H x W, device) into d_m.
 * INVALID_ARGUMENT: bad sizes, radius out of range, v_ref <= 0, non-finite. */
FLLF_API fllf_status fllf_gain_map(const float* d_y, size_t y_pitch_bytes, int H, int W,
                                   const fllf_gain_desc* g, float* d_m, size_t m_pitch_bytes, void* s);
/* The Fig. 5 pipeline on a plan with batch 1: RGB -> YUV, build the pyramids
 * of Y, gain map, apply(FLLF_MAPS) with sigma_r = the plan's and m = the gain
 * map, U and V kept, YUV -> RGB into d_rgb_out.  Workspace for the YUV
 * planes and maps is owned by the plan (allocated on first use).  d_rgb and
 * d_rgb_out may not alias.  INVALID_ARGUMENT: plan batch != 1 or a bad
 * gain description. */
FLLF_API fllf_status fllf_enhance_rgb(fllf_plan p, const float* d_rgb, float* d_rgb_out, size_t pitch_bytes,
                                      const fllf_gain_desc* g, void* s);

/* ---- Naive LLF ground truth (Sec. II-C steps 1-5,
 * P:143-149, Eq. 13; the reference of the accuracy study, Fig. 4,
 * P:328-338).  For every level l < l_max and pixel q: g = G_l[I]_q, the image
 * is remapped around g and the Laplacian coefficient L_l[r(I, g)]_q is taken;
 * L_lmax = G_lmax[I]; O = collapse (Eq. 4).  remap_mode 0: the exact Gaussian
 * remap r(i,g) = i + m (i-g) exp(-(i-g)^2 / 2 sigma_r^2) with the plan's
 * sigma_r, m (reading R1); 1: the truncated series r_K(i,g) = i + sum_k a_k
 * sin(w_k (i-g)) with the plan's K, T (Fourier LLF with K terms is exactly the
 * naive LLF of r_K).  Only the pixels each coefficient depends on are
 * remapped (O(4^l) per coefficient, fp64); a brute-force tool, not a hot
 * path.  Needs a batch-1 plan with the full order range and include_base,
 * levels <= FLLF_NAIVE_MAX_LEVELS (TOO_MANY_LEVELS otherwise).  Rebuilds the
 * plan's pyramids from d_img (like fllf_build_fourier_pyramids) and uses its
 * level scratch planes.  d_out: H x W fp32, caller-owned. */
#define FLLF_NAIVE_MAX_LEVELS 5
FLLF_API fllf_status fllf_naive_llf(fllf_plan p, const float* d_img, size_t pitch_bytes, int remap_mode,
                                    float* d_out, size_t out_pitch_bytes, void* s);

/* ---- Per-level execution for row bands (NEXT-1; north star: "Large frames
 * can instead be split into row bands with halo exchange").  The level
 * recursions of Eq. 1 (build, fine to coarse) and Eq. 14 + Eq. 4 (apply,
 * coarse to fine) only couple neighbouring rows through the 5-tap stencil
 * (2 rows) and the up-sampling (1 row), so a band needs, per level, 2 halo
 * rows of G_l and Z_l (after the build of level l) and of D_l (after the apply
 * of level l) from its neighbours.
 *   fllf_build_level(p, d_img, pitch, l, s): build step l -> l+1 (l = 0..levels-2).
 *   fllf_apply_level(p, a, d_out, pitch, l, s): apply level l (call l = levels-2
 *     down to 0; SCALAR / COEFFS).
 *   fllf_plan_band_plane(p, l, kind, ...): the device layout of the stored
 *     rows of level l (kind 0 = G_l, 1 = Z_l complex planes incl. halo columns,
 *     2 = D_l): pointer to the first stored row `first_row` (global index),
 *     `rows` stored rows, row pitch, `planes` planes (orders x frames for Z) and
 *     the plane stride.  Rows [first_row, first_row + rows) minus the band's own
 *     rows are the halo rows the caller fills. */
FLLF_API fllf_status fllf_build_level(fllf_plan p, const float* d_img, size_t pitch_bytes, int level, void* s);
FLLF_API fllf_status fllf_apply_level(fllf_plan p, const fllf_apply_args* a, float* d_out, size_t out_pitch_bytes,
                                      int level, void* s);
FLLF_API fllf_status fllf_plan_band_plane(fllf_plan p, int level, int kind, void** d_ptr, size_t* pitch_bytes,
                                          int* first_row, int* rows, int* planes, size_t* plane_stride_bytes);

/* Introspection (tests, tooling). */
/* The plan's effective description: defaults resolved (k_begin/k_end of the
 * full range, row_end = H without a band, device = the plan's ordinal). */
FLLF_API fllf_status fllf_plan_get_desc(fllf_plan p, fllf_plan_desc* out);
FLLF_API fllf_status fllf_plan_level_dims(fllf_plan p, int level, int* H, int* W);
FLLF_API fllf_status fllf_workspace_bytes(fllf_plan p, size_t* bytes);
/* Copy one built pyramid plane (levels 1..l_max) of one frame to d_dst:
 * channel 0 = G_l[I] (H_l x W_l floats); channel c = 1..(k_end-k_begin) =
 * Z_{l, k_begin+c-1} as interleaved (S~, C~) float pairs (H_l x 2W_l floats). */
FLLF_API fllf_status fllf_read_pyramid(fllf_plan p, int frame, int level, int channel, float* d_dst,
                              size_t dst_pitch_bytes, void* s);

/* Kernels launched by the most recent build / apply / filter call of this plan. */
FLLF_API int fllf_plan_last_launch_count(fllf_plan p);

/* Per-kernel timing (bench tooling).  With profiling enabled every kernel
 * launch is bracketed by two CUDA events recorded on the launch stream.  The
 * record list restarts at each build (and at an apply that follows an apply).
 * fllf_plan_kernel_times synchronises those events and returns, per launch in
 * order: kind (FLLF_K_*), pyramid level (the fine level of the step) and the
 * duration in milliseconds; *count = number of records (<= capacity). */
enum {
  FLLF_K_BUILD0 = 0,   /* level-0 build (image -> G_1, Z_1)                                  */
  FLLF_K_BUILD = 1,    /* build step l -> l+1, l >= 1                                        */
  FLLF_K_MAPBUILD = 2, /* sigma_r / m map pyramids (MAPS)                                    */
  FLLF_K_APPLY = 3,    /* apply level l >= 1 (design AB)                                     */
  FLLF_K_APPLY0 = 4,   /* apply level 0 (+ collapse into the output)                         */
  FLLF_K_FUSE = 5,     /* design F: build step l -> l+1 fused with the level-l order sum      */
  FLLF_K_COLLAPSE = 6  /* design F: D_l += up(D_{l+1})                                        */
};
FLLF_API fllf_status fllf_plan_set_profiling(fllf_plan p, int enable);
/* Which design fllf_filter runs:
 *   FLLF_DESIGN_AUTO (default): design F on the pyramid levels l >= 1 whose
 *     pixel count over the batch is >= 4 MP (FLLF_FUSE_MIN_MP in the
 *     environment overrides), design AB on the coarser ones;
 *   FLLF_DESIGN_AB: build + apply everywhere;
 *   FLLF_DESIGN_F: design F on every level it supports.
 * Results agree to fp32 rounding.  INVALID_ARGUMENT for other values. */
enum { FLLF_DESIGN_AUTO = 0, FLLF_DESIGN_AB = 1, FLLF_DESIGN_F = 2 };
FLLF_API fllf_status fllf_plan_set_design(fllf_plan p, int design);
/* Finer control of the same choice: design F on levels 1 .. n (n >= 1; n is
 * clamped to l_max-1), design AB above; n = 0 restores FLLF_DESIGN_AUTO.
 * INVALID_ARGUMENT for n < 0. */
FLLF_API fllf_status fllf_plan_set_fused_levels(fllf_plan p, int n);
FLLF_API fllf_status fllf_plan_set_graphs(fllf_plan p, int enable);
FLLF_API fllf_status fllf_plan_kernel_times(fllf_plan p, int capacity, int* kind, int* level,
                                            float* ms, int* count);

FLLF_API const char* fllf_status_string(fllf_status st);
FLLF_API const char* fllf_last_error_message(void);

#ifdef __cplusplus
}
#endif
#endif /* FLLF_H_ */
