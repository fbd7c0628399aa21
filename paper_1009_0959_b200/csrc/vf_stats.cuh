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

// grid (blocks, B), 256 threads; stats[B][8] must be zeroed before launch.
// Per thread: exact integer sums (count, L1, L2^2, max) and fp32 partial sums
// of the Lab norms flushed into double every 32 pixels; one atomic per block
// and statistic.
// want_ref_norm = 0: skip sum |a_Lab| (stats[.][4] stays 0), a's Lab only where a != b.
__global__ void __launch_bounds__(256) vf_stats_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                                       long long npix, double* __restrict__ stats, int want_ref_norm) {
  const int img = blockIdx.y;
  const uint8_t* pa = a + (long long)img * npix * 3;
  const uint8_t* pb = b + (long long)img * npix * 3;
  __shared__ float lin[256];
  if (threadIdx.x < 256) lin[threadIdx.x] = srgb_to_linear_f(threadIdx.x);
  __syncthreads();
  unsigned long long ndiff = 0, l1 = 0, l2 = 0;
  uint32_t mx = 0;
  double s3 = 0.0, s4 = 0.0;
  float f3 = 0.0f, f4 = 0.0f;
  int cnt = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
       p += (long long)gridDim.x * blockDim.x) {
    const uint32_t u = load_px(pa, p), v = load_px(pb, p);
    const uint32_t ad = __vabsdiffu4(u, v);                 // |a - b| per channel
    const uint32_t d0 = ad & 0xff, d1 = (ad >> 8) & 0xff, d2 = (ad >> 16) & 0xff;
    ndiff += (u != v);
    l1 += d0 + d1 + d2;
    l2 += d0 * d0 + d1 * d1 + d2 * d2;
    mx = max(mx, max(d0, max(d1, d2)));
    float L1, A1, B1;
    if (want_ref_norm) {
      rgb_to_lab(u, lin, L1, A1, B1);
      f4 += sqrtf(L1 * L1 + A1 * A1 + B1 * B1);
    }
    if (u != v) {
      if (!want_ref_norm) rgb_to_lab(u, lin, L1, A1, B1);
      float L2, A2, B2;
      rgb_to_lab(v, lin, L2, A2, B2);
      f3 += sqrtf((L1 - L2) * (L1 - L2) + (A1 - A2) * (A1 - A2) + (B1 - B2) * (B1 - B2));
    }
    if (++cnt == 32) {
      s3 += f3; s4 += f4; f3 = 0.0f; f4 = 0.0f; cnt = 0;
    }
  }
  s3 += f3;
  s4 += f4;
  double s[6] = {(double)ndiff, (double)l1, (double)l2, s3, s4, (double)mx};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, s[k], o);
      s[k] = (k == 5) ? fmax(s[k], t) : s[k] + t;
    }
  }
  __shared__ double red[8][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int k = 0; k < 6; ++k) red[warp][k] = s[k];
  __syncthreads();
  if (threadIdx.x < 6) {
    const int k = threadIdx.x;
    double t = red[0][k];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = (k == 5) ? fmax(t, red[w][k]) : t + red[w][k];
    if (k == 5) {
      // non-negative doubles order like their bit patterns
      atomicMax((unsigned long long*)&stats[img * 8 + 5], (unsigned long long)__double_as_longlong(t));
    } else {
      atomicAdd(&stats[img * 8 + k], t);
    }
  }
}

}  // namespace vf
