// Naive local Laplacian filtering on the GPU: the ground
// truth of the paper's accuracy study (Fig. 4: "the ground truth is
// naive LLF"), Sec. II-C steps 1-5:
//   for every level l < l_max and pixel q of level l: g = G_l[I]_q, remap the
//   image around g, I~ = r(I, g), and take the Laplacian coefficient
//   L_l[I~]_q = G_l[I~]_q - up(G_{l+1}[I~])_q  (Eq. 13);
//   L_lmax[O] = G_lmax[I]; O = collapse(L[O])  (Eq. 4).
// The remap is the exact Gaussian one (reading R1) or the truncated series
// r_K(i, g) = i + sum_k a_k sin(w_k (i - g)) (Fourier LLF with K terms is the
// naive LLF of r_K, an exact identity used as a GPU pin).
//
// One CTA per (l, q).  Only the pixels the coefficient depends on are
// remapped: per axis the index sets S_{l+1} (the up-sampling taps of q),
// S_l = {q} u {refl(2c + i)}, ..., S_0 are built in shared memory (sorted,
// reflect-101 at each level's own size, exactly as the global pyramid reads
// them), the remapped window V_0 = r(I[S_0 x S_0], g) is filtered level by
// level (horizontal then vertical 5-tap, fp64), and the coefficient is read
// off V_l and V_{l+1}.  O(4^l) work per coefficient instead of O(N): a
// brute-force tool (levels <= FLLF_NAIVE_MAX_LEVELS), not a hot path.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fllf_internal.h"

namespace fllf {
namespace {

constexpr int MAXL = 96;  // max set size per axis and level (l <= 3: |S_0| <= 93)
// per-level bound of |S_0| (|S_{l+1}| <= 3, |S_j| <= 2 |S_{j+1}| + 3): the V / Hb row stride
__host__ __device__ constexpr int naive_ld(int l) { return l == 0 ? 9 : l == 1 ? 21 : l == 2 ? 45 : 93; }
constexpr int NLV = FLLF_NAIVE_MAX_LEVELS;

__device__ __forceinline__ int refl101_any(int i, int n) {
  if (n == 1) return 0;
  const int p = 2 * (n - 1);
  int r = i % p;
  if (r < 0) r += p;
  return r < n ? r : p - r;
}

// polyphase up-sampling border rule (reading R2/R5): coarse index for the tap
// c of a fine size nf (coarse C = ceil(nf/2)): x_{-1} := x_1, x_C := x_{C-1}
// (nf even) or x_{C-2} (nf odd)
__device__ __forceinline__ int upmap_n(int c, int C, int nf) {
  if (c < 0) c = -c;
  if (c >= C) c = (c == C) ? ((nf & 1) ? C - 2 : C - 1) : C - 1;
  return c < 0 ? 0 : (c > C - 1 ? C - 1 : c);
}

struct AxisSets {
  int len[NLV + 1];
  int idx[NLV + 1][MAXL];           // sorted level indices
  unsigned char tap[NLV][MAXL][5];  // position in S_j of refl_j(2 S_{j+1}[a] + i - 2)
  int upc[3];                       // positions in S_{l+1} of the up taps of q
  double upw[3];
  int nup;
  int qpos;                         // position of q in S_l
};

__device__ int find_pos(const int* list, int n, int v) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (list[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// insert v into the sorted unique list (n <= MAXL)
__device__ void insert_sorted(int* list, int& n, int v) {
  int i = n;
  for (int k = 0; k < n; ++k) {
    if (list[k] == v) return;
    if (list[k] > v) { i = k; break; }
  }
  for (int k = n; k > i; --k) list[k] = list[k - 1];
  list[i] = v;
  ++n;
}

// Build the per-axis sets for coordinate q at level l; dims[j] = size of the axis at level j.
__device__ void build_axis(AxisSets& A, int l, int q, const int* dims) {
  const int nf = dims[l], C = dims[l + 1];
  const int c = q >> 1;
  int taps[3];
  double w[3];
  if ((q & 1) == 0) {
    taps[0] = upmap_n(c - 1, C, nf); w[0] = 0.125;
    taps[1] = upmap_n(c, C, nf);     w[1] = 0.75;
    taps[2] = upmap_n(c + 1, C, nf); w[2] = 0.125;
    A.nup = 3;
  } else {
    taps[0] = upmap_n(c, C, nf);     w[0] = 0.5;
    taps[1] = upmap_n(c + 1, C, nf); w[1] = 0.5;
    A.nup = 2;
  }
  A.len[l + 1] = 0;
  for (int t = 0; t < A.nup; ++t) insert_sorted(A.idx[l + 1], A.len[l + 1], taps[t]);
  for (int t = 0; t < A.nup; ++t) {
    A.upc[t] = find_pos(A.idx[l + 1], A.len[l + 1], taps[t]);
    A.upw[t] = w[t];
  }
  for (int j = l; j >= 0; --j) {
    A.len[j] = 0;
    if (j == l) insert_sorted(A.idx[j], A.len[j], q);
    for (int a = 0; a < A.len[j + 1]; ++a)
      for (int i = -2; i <= 2; ++i) insert_sorted(A.idx[j], A.len[j], refl101_any(2 * A.idx[j + 1][a] + i, dims[j]));
    for (int a = 0; a < A.len[j + 1]; ++a)
      for (int i = -2; i <= 2; ++i)
        A.tap[j][a][i + 2] = (unsigned char)find_pos(A.idx[j], A.len[j], refl101_any(2 * A.idx[j + 1][a] + i, dims[j]));
  }
  A.qpos = find_pos(A.idx[l], A.len[l], q);
}

__device__ __forceinline__ double remap(const NaiveParams& P, double i, double g) {
  const double d = i - g;
  if (P.mode == 0) return i + P.m * d * exp(-d * d * P.inv2s2);
  double s = 0.0;
  for (int k = 0; k < P.K; ++k) s += P.a[k] * sin(P.omega[k] * d);
  return i + s;
}

__device__ __forceinline__ double bw(int i) { return i == 2 ? 0.375 : (i == 1 || i == 3) ? 0.25 : 0.0625; }

__global__ void __launch_bounds__(128) k_naive(const NaiveParams P) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ AxisSets ax[2];  // 0 = rows, 1 = cols
  const int l = P.level;
  const int LD = naive_ld(l);
  double* V = reinterpret_cast<double*>(sm);
  double* Hb = V + LD * LD;
  const int qy = blockIdx.y, qx = blockIdx.x;
  if (threadIdx.x == 0) build_axis(ax[0], l, qy, P.Hs);
  if (threadIdx.x == 32) build_axis(ax[1], l, qx, P.Ws);
  __syncthreads();
  // g = G_l[I]_q
  const double g = (l == 0) ? (double)__ldg(P.img + (long long)qy * P.img_pitch + qx)
                            : (double)__ldg(P.G[l] + (long long)qy * P.gpitch[l] + qx);
  // V_0 = r(I[S_0 x S_0], g)
  const int R0 = ax[0].len[0], C0 = ax[1].len[0];
  for (int t = threadIdx.x; t < R0 * C0; t += blockDim.x) {
    const int a = t / C0, b = t - a * C0;
    const double v = (double)__ldg(P.img + (long long)ax[0].idx[0][a] * P.img_pitch + ax[1].idx[0][b]);
    V[a * LD + b] = remap(P, v, g);
  }
  __syncthreads();
  double Gl = 0.0;
  for (int j = 0; j <= l; ++j) {
    const int Rj = ax[0].len[j], Cn = ax[1].len[j + 1], Rn = ax[0].len[j + 1];
    if (j == l && threadIdx.x == 0) Gl = V[ax[0].qpos * LD + ax[1].qpos];
    // horizontal: Hb[a][b] = sum_i w_i V[a][tapC[j][b][i]]
    for (int t = threadIdx.x; t < Rj * Cn; t += blockDim.x) {
      const int a = t / Cn, b = t - a * Cn;
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 5; ++i) s += bw(i) * V[a * LD + ax[1].tap[j][b][i]];
      Hb[a * LD + b] = s;
    }
    __syncthreads();
    // vertical: V[a][b] = sum_i w_i Hb[tapR[j][a][i]][b]   (level j+1 values)
    for (int t = threadIdx.x; t < Rn * Cn; t += blockDim.x) {
      const int a = t / Cn, b = t - a * Cn;
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 5; ++i) s += bw(i) * Hb[ax[0].tap[j][a][i] * LD + b];
      V[a * LD + b] = s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double up = 0.0;
    for (int u = 0; u < ax[0].nup; ++u)
      for (int v = 0; v < ax[1].nup; ++v) up += ax[0].upw[u] * ax[1].upw[v] * V[ax[0].upc[u] * LD + ax[1].upc[v]];
    P.L[l][(long long)qy * P.lpitch[l] + qx] = (float)(Gl - up);
  }
}

// O_l = L_l + up(O_{l+1}) in place on the fine plane (collapse, Eq. 4)
__global__ void k_collapse_up(float* fine, long long fpitch, const float* coarse, long long cpitch, int Hf, int Wf,
                              int Hc, int Wc) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= Wf || y >= Hf) return;
  auto taps = [](int t, int C, int nf, int* c, float* w) -> int {
    const int h = t >> 1;
    if ((t & 1) == 0) {
      c[0] = upmap_n(h - 1, C, nf); w[0] = 0.125f;
      c[1] = upmap_n(h, C, nf);     w[1] = 0.75f;
      c[2] = upmap_n(h + 1, C, nf); w[2] = 0.125f;
      return 3;
    }
    c[0] = upmap_n(h, C, nf);     w[0] = 0.5f;
    c[1] = upmap_n(h + 1, C, nf); w[1] = 0.5f;
    return 2;
  };
  int cr[3], cc[3];
  float wr[3], wc[3];
  const int nr = taps(y, Hc, Hf, cr, wr), nc = taps(x, Wc, Wf, cc, wc);
  float s = 0.f;
  for (int u = 0; u < nr; ++u)
    for (int v = 0; v < nc; ++v) s += wr[u] * wc[v] * coarse[(long long)cr[u] * cpitch + cc[v]];
  fine[(long long)y * fpitch + x] += s;
}

}  // namespace

cudaError_t launch_naive_level(const NaiveParams& p, cudaStream_t s) {
  const size_t smem = 2 * sizeof(double) * naive_ld(p.level) * naive_ld(p.level);
  cudaError_t e = cudaFuncSetAttribute(k_naive, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(2 * sizeof(double) * MAXL * MAXL));
  if (e != cudaSuccess) return e;
  dim3 grid(p.Ws[p.level], p.Hs[p.level]);
  k_naive<<<grid, 128, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_collapse_up(float* fine, long long fpitch, const float* coarse, long long cpitch, int Hf, int Wf,
                               int Hc, int Wc, cudaStream_t s) {
  dim3 grid((Wf + 127) / 128, Hf);
  k_collapse_up<<<grid, 128, 0, s>>>(fine, fpitch, coarse, cpitch, Hf, Wf, Hc, Wc);
  return cudaGetLastError();
}

}  // namespace fllf
