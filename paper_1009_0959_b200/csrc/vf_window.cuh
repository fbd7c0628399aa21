// vf_window.cuh -- the per-window kernel: one thread = one output pixel, all
// n(n-1)/2 pairs of its window evaluated in registers (SURVEY.md 8(a) rows
// a1-a8 fused in one launch).
//
//   a1  stage the block's tile + halo (uint8 HWC -> fp32 in smem) with
//       replicate clamping against the GLOBAL image rows (stripes), Fig. 1 /
//       S:78;
//   a2  per-pixel precompute once per staged pixel: (r, g, b, |x|^2) and, for
//       the angular criterion, (|x|, 1/|x|);
//   a3  exp/log: window statistic S1 = sum_{i<j} |x_i - x_j|_1 and the scale
//       c_E = n^(1+kappa/3) / (2 S1) (= 1/h_W, Eq. 8) or c_L = (1-1/e)(n-1)/S1;
//   a4  pair geometry; a5 criterion (libm or minimax Horner, Tables 1-4);
//   a6  symmetric accumulation R_i += D, R_j += D (each pair computed once);
//   a7  argmin, strict '<' in increasing k (lowest index on ties);
//   a8  store the output sample (+ optional index / aggregates).
#pragma once
#include <cstdint>

#include "vf_device.cuh"

namespace vf {

constexpr int TX = 32;   // output tile width  (one warp per tile row)
constexpr int TY = 8;    // output tile height (8 warps per block)

struct Launch {
  const uint8_t* in;   // global row band_row0 of image 0
  uint8_t* out;        // output row out_row0 of image 0
  uint8_t* idx;        // nullable
  float* agg;          // nullable
  long long in_stride, out_stride;   // bytes between images (in / out)
  int H, W;            // global image size
  int band_row0, band_rows;
  int out_row0, out_rows;
  float kscale;        // exp: n^(1+kappa/3)/2 ; log: (1-1/e)(n-1)
};

template <int WIN, int CRIT, int VAR>
__global__ void __launch_bounds__(TX * TY) vf_window_kernel(const Launch L) {
  constexpr int R = WIN / 2;
  constexpr int N = WIN * WIN;
  constexpr int SW = TX + 2 * R;
  constexpr int SH = TY + 2 * R;
  __shared__ float4 s_px[SH * SW];                        // r, g, b, |x|^2
  __shared__ float2 s_nm[CRIT == ANGULAR ? SH * SW : 1];  // |x|, 1/|x|

  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX;
  const int y0 = L.out_row0 + blockIdx.y * TY;           // global row of tile row 0
  const uint8_t* __restrict__ in = L.in + (long long)b * L.in_stride;

  // ---- a1 + a2: stage tile + halo ------------------------------------------
  const int tid = threadIdx.y * TX + threadIdx.x;
  for (int p = tid; p < SH * SW; p += TX * TY) {
    const int sy = p / SW, sx = p - sy * SW;
    const int gy = clampi(y0 + sy - R, 0, L.H - 1) - L.band_row0;
    const int gx = clampi(x0 + sx - R, 0, L.W - 1);
    const uint8_t* q = in + ((long long)gy * L.W + gx) * 3;
    const float r = q[0], g = q[1], bl = q[2];
    const float nn = fmaf(r, r, fmaf(g, g, bl * bl));    // exact integer < 2^18
    s_px[p] = make_float4(r, g, bl, nn);
    if (CRIT == ANGULAR) {
      const float nrm = sqrtf(nn);
      s_nm[p] = make_float2(nrm, nn > 0.0f ? 1.0f / nrm : 0.0f);
    }
  }
  __syncthreads();

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int ox = x0 + tx, oy = y0 + ty;
  if (ox >= L.W || oy >= L.out_row0 + L.out_rows) return;

  float xr[N], xg[N], xb[N], xn[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const float4 v = s_px[(ty + k / WIN) * SW + tx + k % WIN];
    xr[k] = v.x; xg[k] = v.y; xb[k] = v.z; xn[k] = CRIT == ANGULAR ? v.w : 0.0f;
  }
  float Ra[N];
#pragma unroll
  for (int k = 0; k < N; ++k) Ra[k] = 0.0f;

  if (CRIT == ANGULAR) {
    float xm[N], xi[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const float2 v = s_nm[(ty + k / WIN) * SW + tx + k % WIN];
      xm[k] = v.x; xi[k] = v.y;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = i + 1; j < N; ++j) {
        const float d = angular_pair<VAR>(xr[i], xg[i], xb[i], xn[i], xm[i], xi[i],
                                          xr[j], xg[j], xb[j], xn[j], xm[j], xi[j]);
        Ra[i] += d;
        Ra[j] += d;
      }
    }
    if (VAR != EXACT) {
      // zero-vector fix-up: every pair touching a zero vector
      // contributed the ARCSIN row's a0 instead of 0.
      int zc = 0;
#pragma unroll
      for (int k = 0; k < N; ++k) zc += (xn[k] == 0.0f);
      if (zc) {
        const float corr = (float)zc * coef::ASIN().a0;
#pragma unroll
        for (int k = 0; k < N; ++k) Ra[k] = (xn[k] == 0.0f) ? 0.0f : Ra[k] - corr;
      }
    }
  } else {
    // ---- a3: window statistic S1 ------------------------------------------
    constexpr bool KEEP = (N <= 9);
    float d1k[KEEP ? N * (N - 1) / 2 : 1];
    float S1 = 0.0f;
#pragma unroll
    for (int i = 0, p = 0; i < N; ++i) {
#pragma unroll
      for (int j = i + 1; j < N; ++j, ++p) {
        // (written as max - min so that, for 5x5, the compiler does not keep
        // all 300 distances live until pass 2: recomputing is cheaper than spilling)
        const float d = KEEP ? l1(xr[i], xg[i], xb[i], xr[j], xg[j], xb[j])
                             : l1_maxmin(xr[i], xg[i], xb[i], xr[j], xg[j], xb[j]);
        if (KEEP) d1k[p] = d;
        S1 += d;                                          // exact: S1 < 2^18
      }
    }
    if (S1 > 0.0f) {                                      // flat window: all D = 0
      const float sc = L.kscale / S1;                     // c_E or c_L
#pragma unroll
      for (int i = 0, p = 0; i < N; ++i) {
#pragma unroll
        for (int j = i + 1; j < N; ++j, ++p) {
          const float d = KEEP ? d1k[p] : l1(xr[i], xg[i], xb[i], xr[j], xg[j], xb[j]);
          const float v = CRIT == EXPC ? exp_crit<VAR>(sc * d) : log_crit<VAR>(sc * d);
          Ra[i] += v;
          Ra[j] += v;
        }
      }
    }
  }

  // ---- a7: argmin, lowest index on ties ---------------------------------------
  int best = 0;
  float bv = Ra[0];
#pragma unroll
  for (int k = 1; k < N; ++k) {
    if (Ra[k] < bv) { bv = Ra[k]; best = k; }
  }
  // ---- a8: store -----------------------------------------------------------------
  float orr = xr[0], og = xg[0], ob = xb[0];
#pragma unroll
  for (int k = 1; k < N; ++k) {
    if (best == k) { orr = xr[k]; og = xg[k]; ob = xb[k]; }
  }
  const long long po = (long long)(oy - L.out_row0) * L.W + ox;
  uint8_t* o = L.out + (long long)b * L.out_stride + po * 3;
  o[0] = (uint8_t)orr; o[1] = (uint8_t)og; o[2] = (uint8_t)ob;
  const long long npix_img = (long long)L.out_rows * L.W;
  if (L.idx) L.idx[b * npix_img + po] = (uint8_t)best;
  if (L.agg) {
    float* a = L.agg + (b * npix_img + po) * N;
#pragma unroll
    for (int k = 0; k < N; ++k) a[k] = Ra[k];
  }
}

}  // namespace vf
