// vf_stats.cuh -- per-image fidelity statistics of two output images
// (MAE, MSE, NCD of PAPER.md P:286-293; CIELAB via sRGB/D65).
#pragma once
#include <cstdint>

namespace vf {

// sRGB decoding table (IEC 61966-2-1), filled once per block in shared memory.
__device__ __forceinline__ float srgb_to_linear_f(int c) {
  const float v = c / 255.0f;
  return v <= 0.04045f ? v / 12.92f : powf((v + 0.055f) / 1.055f, 2.4f);
}

// t^(1/3) for t in (0.0088, 1.1] (the CIELAB cube-root branch: positive
// normal arguments only, so none of cbrtf's special cases): MUFU.LG2 and
// MUFU.EX2 give ~4e-7 relative, one Newton step y += (t/y^2 - y)/3 brings it
// to ~1 ulp.
__device__ __forceinline__ float cbrt_pos(float t) {
  float l, y, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(t));
  const float e = l * (1.0f / 3.0f);
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(e));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y * y));
  return fmaf(fmaf(t, r, -y), 1.0f / 3.0f, y);
}

__device__ __forceinline__ float lab_f(float t) {
  constexpr float d = 6.0f / 29.0f;
  return t > d * d * d ? cbrt_pos(t) : t * (1.0f / (3.0f * d * d)) + 4.0f / 29.0f;
}

// CIELAB of one pixel (sRGB, BT.709 primaries, D65), fp32 per pixel (the sums
// are accumulated in double).  pk = packed RGB (r | g << 8 | b << 16).
__device__ __forceinline__ void rgb_to_lab(uint32_t pk, const float* lin, float& L, float& A, float& B) {
  const float r = lin[pk & 0xff], g = lin[(pk >> 8) & 0xff], b = lin[(pk >> 16) & 0xff];
  const float X = 0.4124564f * r + 0.3575761f * g + 0.1804375f * b;
  const float Y = 0.2126729f * r + 0.7151522f * g + 0.0721750f * b;
  const float Z = 0.0193339f * r + 0.1191920f * g + 0.9503041f * b;
  const float fx = lab_f(X * (1.0f / 0.95047f)), fy = lab_f(Y), fz = lab_f(Z * (1.0f / 1.08883f));
  L = 116.0f * fy - 16.0f;
  A = 500.0f * (fx - fy);
  B = 200.0f * (fy - fz);
}

// Packed RGB of pixel p of an HWC uint8 image: the aligned 32-bit word(s)
// holding its 3 bytes (one funnel shift), instead of three byte loads.  The
// words are aligned in absolute address, so they never leave the aligned
// words that hold the image's bytes.
__device__ __forceinline__ uint32_t load_px(const uint8_t* img, long long p) {
  const uintptr_t o = reinterpret_cast<uintptr_t>(img) + (uintptr_t)(p * 3);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(o & ~(uintptr_t)3);
  const int sh = (int)(o & 3) * 8;
  const uint32_t w0 = __ldg(w);
  const uint32_t w1 = sh > 8 ? __ldg(w + 1) : 0u;   // bytes 4.. only needed when the pixel crosses the word
  return __funnelshift_r(w0, w1, sh) & 0x00ffffffu;
}

// Fixed-point scale of the floating-point sums (columns 3, 4): each block's
// double partial sum is rounded to a multiple of 2^-24 and added as an
// integer, so the per-image totals do not depend on the order in which blocks
// finish (bit-reproducible, unlike double atomics).  Range: |sum| < 2^39
// (5.5e11, i.e. > 2.6e9 pixels of the largest Lab norm ~207); resolution
// 6e-8 per block.
constexpr double STATS_FIX = 16777216.0;   // 2^24

// Per-image statistics of NB outputs b_k against one reference a, in ONE pass
// over a (each reference pixel is read once and its CIELAB computed at most
// once).  grid (blocks, B), 256 threads.  acc[NB][B][8] (uint64, zeroed before
// launch): {count a != b, sum |a-b|, sum (a-b)^2, fix(sum |a_Lab - b_Lab|),
// fix(sum |a_Lab|), max |a-b|, 0, 0}; vf_stats_finalize converts to double.
// Per thread: exact integer sums and fp32 partial sums of the Lab norms,
// flushed into double every 32 pixels; block reduction in a fixed order.
struct StatsArgs {
  const uint8_t* b[8];
};

template <int NB>
__global__ void __launch_bounds__(256) vf_stats_multi_kernel(const uint8_t* __restrict__ a, const StatsArgs bs,
                                                             long long npix, int B,
                                                             unsigned long long* __restrict__ acc,
                                                             int want_ref_norm) {
  const int img = blockIdx.y;
  const uint8_t* pa = a + (long long)img * npix * 3;
  __shared__ float lin[256];
  lin[threadIdx.x] = srgb_to_linear_f(threadIdx.x);
  __syncthreads();
  unsigned long long ndiff[NB], l1[NB], l2[NB];
  uint32_t mx[NB];
  double s3[NB];
  float f3[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) { ndiff[k] = 0; l1[k] = 0; l2[k] = 0; mx[k] = 0; s3[k] = 0.0; f3[k] = 0.0f; }
  double s4 = 0.0;
  float f4 = 0.0f;
  int cnt = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
       p += (long long)gridDim.x * blockDim.x) {
    const uint32_t u = load_px(pa, p);
    float L1 = 0.0f, A1 = 0.0f, B1 = 0.0f;
    bool have_a = false;
    if (want_ref_norm) {
      rgb_to_lab(u, lin, L1, A1, B1);
      have_a = true;
      f4 += sqrtf(L1 * L1 + A1 * A1 + B1 * B1);
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const uint32_t v = load_px(bs.b[k] + (long long)img * npix * 3, p);
      if (u != v) {
        const uint32_t ad = __vabsdiffu4(u, v);             // |a - b| per channel
        const uint32_t d0 = ad & 0xff, d1 = (ad >> 8) & 0xff, d2 = (ad >> 16) & 0xff;
        ndiff[k] += 1;
        l1[k] += d0 + d1 + d2;
        l2[k] += d0 * d0 + d1 * d1 + d2 * d2;
        mx[k] = max(mx[k], max(d0, max(d1, d2)));
        if (!have_a) {
          rgb_to_lab(u, lin, L1, A1, B1);
          have_a = true;
        }
        float L2, A2, B2;
        rgb_to_lab(v, lin, L2, A2, B2);
        f3[k] += sqrtf((L1 - L2) * (L1 - L2) + (A1 - A2) * (A1 - A2) + (B1 - B2) * (B1 - B2));
      }
    }
    if (++cnt == 32) {
#pragma unroll
      for (int k = 0; k < NB; ++k) { s3[k] += f3[k]; f3[k] = 0.0f; }
      s4 += f4;
      f4 = 0.0f;
      cnt = 0;
    }
  }
  s4 += f4;
  __shared__ double red[8][6 * NB + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k <= NB; ++k) {
    double s[6];
    if (k < NB) {
      s3[k] += f3[k];
      s[0] = (double)ndiff[k]; s[1] = (double)l1[k]; s[2] = (double)l2[k]; s[3] = s3[k]; s[4] = 0.0;
      s[5] = (double)mx[k];
    } else {
      s[0] = s4;
    }
    const int nv = k < NB ? 6 : 1;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      if (c >= nv || c == 4) continue;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, s[c], o);
        s[c] = (c == 5) ? fmax(s[c], t) : s[c] + t;
      }
      if (lane == 0) red[warp][k * 6 + c] = s[c];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 6 * NB + 1; i += blockDim.x) {
    const int k = i / 6, c = i % 6;
    if (k < NB && c == 4) continue;
    double t = red[0][i];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = (c == 5 && k < NB) ? fmax(t, red[w][i]) : t + red[w][i];
    if (k == NB) {                                           // reference norm: column 4 of every output
      if (!want_ref_norm) continue;
      const unsigned long long q = (unsigned long long)llrint(t * STATS_FIX);
      for (int j = 0; j < NB; ++j) atomicAdd(&acc[((long long)j * B + img) * 8 + 4], q);
    } else if (c == 5) {
      atomicMax(&acc[((long long)k * B + img) * 8 + 5], (unsigned long long)t);
    } else {
      const unsigned long long q = c == 3 ? (unsigned long long)llrint(t * STATS_FIX) : (unsigned long long)t;
      atomicAdd(&acc[((long long)k * B + img) * 8 + c], q);   // integer: order-independent
    }
  }
}

// acc (uint64 sums, fixed point for columns 3 and 4) -> double, in place.
__global__ void vf_stats_finalize(unsigned long long* acc, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long q = acc[i];
  const int c = (int)(i % 8);
  const double v = (c == 3 || c == 4) ? (double)q / STATS_FIX : (double)q;
  reinterpret_cast<double*>(acc)[i] = v;
}

}  // namespace vf
