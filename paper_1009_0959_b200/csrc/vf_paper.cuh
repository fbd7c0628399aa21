// vf_paper.cuh -- the paper's other two filters on the same window engine
// (SURVEY.md 8(f2)-(f3)), one thread per output pixel:
//
//   AMNF (Eq. 8): y = sum_i x_i w_i / sum_j w_j,
//        w_i = h_i^-3 K((x_C - x_i)/h_i), h_i = n^(-kappa/3) sum_j |x_i - x_j|_1;
//        AMNFE K = exp(-|.|_1), AMNFG K = exp(-0.5 |.|_2^2); exp by libm expf
//        (exact), Table 3 rational or Table 2 p=4 (minimax), cutoff T = 10
//        (P:163); output rounded half away from zero and clamped.
//        Degenerate (all samples equal, h_i = 0) -> x_C.
//   EVMF (Eq. 9): x_C unless P_C > beta_C, then the L2 vector
//        median; P_i = |x_i - xbar|_2 / sum_j |x_j - xbar|_2,
//        beta_C = ENT(P_C) / sum_j ENT(P_j), ENT = z ln z (libm logf, exact)
//        or Table 4 rational with cutoff T = 0.05; degenerate rules of
//        S:344.
//
// Geometry is exact in integers (packed RGB0 words): L1 distances by one
// VABSDIFF4, dot products / squared norms by one IDP.4A.
#pragma once
#include <cstdint>

#include "vf_window.cuh"

namespace vf {

enum { AMNFE = 3, AMNFG = 4, EVMF = 5 };

__device__ __forceinline__ float u2f_exact(uint32_t v) {   // exact for v < 2^23
  return __uint_as_float(v + F2P23_BITS) - F2P23;
}

// EXP for the AMNF weights: exact libm expf or the paper's approximants with
// the P:163 cutoff (z > 10 -> 0; unreachable here, z <= n^(kappa/3), kept for
// fidelity to the paper's evaluator).
template <int VAR>
__device__ __forceinline__ float amnf_exp(float z) {
  if (VAR == EXACT) return expf(-z);
  const float e = VAR == MINIMAX ? horner4(coef::EXP_N(), z) * rcp_approx(horner4(coef::EXP_Q(), z))
                                 : horner4(coef::EXP_P4(), z);
  return z > 10.0f ? 0.0f : e;
}

// ENT(z) = z ln z for EVMF: exact libm logf (ENT(0) = 0) or Table 4 with the
// P:232 cutoff (z < 0.05 -> 0).
template <int VAR>
__device__ __forceinline__ float evmf_ent(float z) {
  if (VAR == EXACT) return z > 0.0f ? z * logf(z) : 0.0f;
  const float e = horner4(coef::ENT_N(), z) * rcp_approx(horner4(coef::ENT_Q(), z));
  return z < 0.05f ? 0.0f : e;
}

template <int WIN>
__device__ __forceinline__ void stage_packed(const Launch& L, const uint8_t* in, int x0, int y0, uint32_t* s_pk,
                                             int SW, int SH) {
  constexpr int R = WIN / 2;
  for (int row = threadIdx.y; row < SH; row += TY) {
    const int gy = clampi(y0 - R + row, L.band_row0, L.band_row0 + L.band_rows - 1) - L.band_row0;   // see pixel_ptr
    VF_CHECK(gy >= 0 && gy < L.band_rows);
    const uint8_t* rp = in + (long long)gy * L.W * 3;
    for (int col = threadIdx.x; col < SW; col += TX) {
      const uint8_t* q = rp + clampi(x0 - R + col, 0, L.W - 1) * 3;
      s_pk[row * SW + col] = pack_rgb(q[0], q[1], q[2]);
    }
  }
}

__device__ __forceinline__ void store_pixel(const Launch& L, int b, int ox, int oy, uint32_t o, int idx) {
  VF_CHECK(oy >= L.out_row0 && oy < L.out_row0 + L.out_rows && ox >= 0 && ox < L.W);
  const long long po = (long long)(oy - L.out_row0) * L.W + ox;
  uint8_t* op = L.out + (long long)b * L.out_stride + po * 3;
  op[0] = (uint8_t)(o & 0xff); op[1] = (uint8_t)((o >> 8) & 0xff); op[2] = (uint8_t)((o >> 16) & 0xff);
  const long long npix_img = (long long)L.out_rows * L.W;
  if (L.idx) L.idx[b * npix_img + po] = (uint8_t)idx;
}

// ---- AMNF --------------------------------------------------------------------------
template <int WIN, int GAUSS, int VAR>
__global__ void __launch_bounds__(TX * TY) vf_amnf_kernel(const Launch L) {
  constexpr int R = WIN / 2;
  constexpr int N = WIN * WIN;
  constexpr int C = (N - 1) / 2;
  constexpr int SW = TX + 2 * R;
  constexpr int SH = TY + 2 * R;
  __shared__ uint32_t s_pk[SH * SW];
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX;
  const int y0 = L.out_row0 + blockIdx.y * TY;
  stage_packed<WIN>(L, L.in + (long long)b * L.in_stride, x0, y0, s_pk, SW, SH);
  __syncthreads();
  const int ox = x0 + threadIdx.x, oy = y0 + threadIdx.y;
  if (ox >= L.W || oy >= L.out_row0 + L.out_rows) return;

  uint32_t w[N];
#pragma unroll
  for (int k = 0; k < N; ++k) w[k] = s_pk[(threadIdx.y + k / WIN) * SW + threadIdx.x + k % WIN];
  // h_i = n^(-kappa/3) * sum_j |x_i - x_j|_1   (integer row sums, exact)
  uint32_t rs[N];
#pragma unroll
  for (int k = 0; k < N; ++k) rs[k] = 0u;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i + 1; j < N; ++j) {
      const uint32_t d = sad4(w[i], w[j], 0u);
      rs[i] += d;
      rs[j] += d;
    }
  float v[3] = {0.0f, 0.0f, 0.0f};
  uint32_t o = w[C];
  if (rs[C] != 0u) {            // rs_i = 0 for one i <=> all samples equal (degenerate)
    float sw = 0.0f, s0 = 0.0f, s1 = 0.0f, s2 = 0.0f;
    const uint32_t nnC = __dp4a(w[C], w[C], 0u);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const float rh = rcp_approx(L.kscale * u2f_exact(rs[i]));   // 1 / h_i (kscale = n^(-kappa/3))
      float z;
      if (GAUSS) {
        const uint32_t d2 = nnC + __dp4a(w[i], w[i], 0u) - 2u * __dp4a(w[C], w[i], 0u);   // |x_C - x_i|_2^2
        z = 0.5f * u2f_exact(d2) * rh * rh;
      } else {
        z = u2f_exact(sad4(w[C], w[i], 0u)) * rh;                                       // |x_C - x_i|_1 / h_i
      }
      const float wt = amnf_exp<VAR>(z) * (rh * rh * rh);                               // h_i^-3 K
      sw += wt;
      s0 = fmaf(u2f_exact(w[i] & 0xffu), wt, s0);
      s1 = fmaf(u2f_exact((w[i] >> 8) & 0xffu), wt, s1);
      s2 = fmaf(u2f_exact(w[i] >> 16), wt, s2);
    }
    if (!(sw > 0.0f)) {               // all weights cut off: impossible here, guarded
      v[0] = (float)(w[C] & 0xffu); v[1] = (float)((w[C] >> 8) & 0xffu); v[2] = (float)(w[C] >> 16);
    } else {
      const float isw = 1.0f / sw;
      v[0] = s0 * isw; v[1] = s1 * isw; v[2] = s2 * isw;
      o = 0u;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float r = fminf(fmaxf(floorf(v[c] + 0.5f), 0.0f), 255.0f);   // half away from zero (v >= 0)
        o |= (uint32_t)r << (8 * c);
      }
    }
  }
  if (rs[C] == 0u) {
    v[0] = (float)(w[C] & 0xffu); v[1] = (float)((w[C] >> 8) & 0xffu); v[2] = (float)(w[C] >> 16);
  }
  store_pixel(L, b, ox, oy, o, C);
  if (L.agg) {
    const long long po = (long long)(oy - L.out_row0) * L.W + ox;
    float* a = L.agg + ((long long)b * L.out_rows * L.W + po) * N;
    a[0] = v[0]; a[1] = v[1]; a[2] = v[2];
#pragma unroll
    for (int k = 3; k < N; ++k) a[k] = 0.0f;
  }
}

// ---- EVMF --------------------------------------------------------------------------
template <int WIN, int VAR>
__global__ void __launch_bounds__(TX * TY) vf_evmf_kernel(const Launch L) {
  constexpr int R = WIN / 2;
  constexpr int N = WIN * WIN;
  constexpr int C = (N - 1) / 2;
  constexpr int SW = TX + 2 * R;
  constexpr int SH = TY + 2 * R;
  __shared__ uint32_t s_pk[SH * SW];
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX;
  const int y0 = L.out_row0 + blockIdx.y * TY;
  stage_packed<WIN>(L, L.in + (long long)b * L.in_stride, x0, y0, s_pk, SW, SH);
  __syncthreads();
  const int ox = x0 + threadIdx.x, oy = y0 + threadIdx.y;
  if (ox >= L.W || oy >= L.out_row0 + L.out_rows) return;

  uint32_t w[N];
#pragma unroll
  for (int k = 0; k < N; ++k) w[k] = s_pk[(threadIdx.y + k / WIN) * SW + threadIdx.x + k % WIN];
  // window mean (exact integer sums, one rounding each)
  uint32_t sr = 0u, sg = 0u, sb = 0u;
#pragma unroll
  for (int k = 0; k < N; ++k) { sr += w[k] & 0xffu; sg += (w[k] >> 8) & 0xffu; sb += w[k] >> 16; }
  const float invn = 1.0f / (float)N;
  const float mr = u2f_exact(sr) * invn, mg = u2f_exact(sg) * invn, mb = u2f_exact(sb) * invn;
  float dev[N];
  float S = 0.0f;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const float dr = u2f_exact(w[k] & 0xffu) - mr, dg = u2f_exact((w[k] >> 8) & 0xffu) - mg,
                db = u2f_exact(w[k] >> 16) - mb;
    dev[k] = sqrtf(fmaf(dr, dr, fmaf(dg, dg, db * db)));
    S += dev[k];
  }
  bool fire = false;
  float PC = 0.0f, beta = 0.0f;
  if (S > 0.0f) {                                           // else identity
    const float iS = 1.0f / S;
    float se = 0.0f, eC = 0.0f;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const float e = evmf_ent<VAR>(dev[k] * iS);
      se += e;
      if (k == C) eC = e;
    }
    PC = dev[C] * iS;
    beta = se == 0.0f ? 0.0f : eC / se;
    fire = PC > beta;
  }
  float Ra[N];
  const bool need_R = fire || L.agg;
  int sel = C;
  if (need_R) {
    uint32_t nn[N];
#pragma unroll
    for (int k = 0; k < N; ++k) { nn[k] = __dp4a(w[k], w[k], 0u); Ra[k] = -0.0f; }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i + 1; j < N; ++j) {
        const uint32_t d2 = nn[i] + nn[j] - 2u * __dp4a(w[i], w[j], 0u);   // exact |x_i - x_j|_2^2
        float d;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(u2f_exact(d2)));
        Ra[i] += d;
        Ra[j] += d;
      }
    if (fire) {
      float bv = Ra[0];
      sel = 0;
#pragma unroll
      for (int k = 1; k < N; ++k)
        if (Ra[k] < bv) { bv = Ra[k]; sel = k; }
    }
  }
  uint32_t o = w[0];
#pragma unroll
  for (int k = 1; k < N; ++k) o = (sel == k) ? w[k] : o;
  store_pixel(L, b, ox, oy, o, sel | (fire ? 0x80 : 0));   // bit 7: the switch fired
  if (L.agg) {
    const long long po = (long long)(oy - L.out_row0) * L.W + ox;
    float* a = L.agg + ((long long)b * L.out_rows * L.W + po) * N;
#pragma unroll
    for (int k = 0; k < N; ++k) a[k] = Ra[k];
  }
}

}  // namespace vf
