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

__device__ __forceinline__ float lab_f(float t) {
  const float d = 6.0f / 29.0f;
  return t > d * d * d ? cbrtf(t) : t / (3.0f * d * d) + 4.0f / 29.0f;
}

// CIELAB of one pixel (sRGB, BT.709 primaries, D65), fp32 per pixel (the sums
// are accumulated in double).
__device__ __forceinline__ void rgb_to_lab(const uint8_t* p, const float* lin, float& L, float& A, float& B) {
  const float r = lin[p[0]], g = lin[p[1]], b = lin[p[2]];
  const float X = 0.4124564f * r + 0.3575761f * g + 0.1804375f * b;
  const float Y = 0.2126729f * r + 0.7151522f * g + 0.0721750f * b;
  const float Z = 0.0193339f * r + 0.1191920f * g + 0.9503041f * b;
  const float fx = lab_f(X / 0.95047f), fy = lab_f(Y), fz = lab_f(Z / 1.08883f);
  L = 116.0f * fy - 16.0f;
  A = 500.0f * (fx - fy);
  B = 200.0f * (fy - fz);
}

// grid (blocks, B), 256 threads; stats[B][8] must be zeroed before launch.
__global__ void __launch_bounds__(256) vf_stats_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                                       long long npix, double* __restrict__ stats) {
  const int img = blockIdx.y;
  const uint8_t* pa = a + (long long)img * npix * 3;
  const uint8_t* pb = b + (long long)img * npix * 3;
  __shared__ float lin[256];
  if (threadIdx.x < 256) lin[threadIdx.x] = srgb_to_linear_f(threadIdx.x);
  __syncthreads();
  double s[6] = {0, 0, 0, 0, 0, 0};
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
       p += (long long)gridDim.x * blockDim.x) {
    const uint8_t* u = pa + p * 3;
    const uint8_t* v = pb + p * 3;
    int d0 = (int)u[0] - v[0], d1 = (int)u[1] - v[1], d2 = (int)u[2] - v[2];
    s[0] += (d0 | d1 | d2) ? 1.0 : 0.0;
    s[1] += abs(d0) + abs(d1) + abs(d2);
    s[2] += d0 * d0 + d1 * d1 + d2 * d2;
    float L1, A1, B1;
    rgb_to_lab(u, lin, L1, A1, B1);
    s[4] += sqrtf(L1 * L1 + A1 * A1 + B1 * B1);
    if (d0 | d1 | d2) {
      float L2, A2, B2;
      rgb_to_lab(v, lin, L2, A2, B2);
      s[3] += sqrtf((L1 - L2) * (L1 - L2) + (A1 - A2) * (A1 - A2) + (B1 - B2) * (B1 - B2));
    }
    s[5] = fmax(s[5], (double)max(abs(d0), max(abs(d1), abs(d2))));
  }
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
