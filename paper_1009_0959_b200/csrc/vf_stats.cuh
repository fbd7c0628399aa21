// vf_stats.cuh -- per-image fidelity statistics of two output images
// (MAE, MSE, NCD of PAPER.md P:286-293; CIELAB via sRGB/D65).
#pragma once
#include <cstdint>

namespace vf {

__device__ __forceinline__ double srgb_to_linear(double c) {
  c = c / 255.0;
  return c <= 0.04045 ? c / 12.92 : pow((c + 0.055) / 1.055, 2.4);
}

__device__ __forceinline__ double lab_f(double t) {
  const double d = 6.0 / 29.0;
  return t > d * d * d ? cbrt(t) : t / (3.0 * d * d) + 4.0 / 29.0;
}

__device__ __forceinline__ void rgb_to_lab(const uint8_t* p, double& L, double& A, double& B) {
  const double r = srgb_to_linear(p[0]), g = srgb_to_linear(p[1]), b = srgb_to_linear(p[2]);
  // linear sRGB (BT.709 primaries) -> XYZ, D65
  const double X = 0.4124564 * r + 0.3575761 * g + 0.1804375 * b;
  const double Y = 0.2126729 * r + 0.7151522 * g + 0.0721750 * b;
  const double Z = 0.0193339 * r + 0.1191920 * g + 0.9503041 * b;
  const double fx = lab_f(X / 0.95047), fy = lab_f(Y / 1.0), fz = lab_f(Z / 1.08883);
  L = 116.0 * fy - 16.0;
  A = 500.0 * (fx - fy);
  B = 200.0 * (fy - fz);
}

// grid (blocks, B), 256 threads; stats[B][8] must be zeroed before launch.
__global__ void __launch_bounds__(256) vf_stats_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                                       long long npix, double* __restrict__ stats) {
  const int img = blockIdx.y;
  const uint8_t* pa = a + (long long)img * npix * 3;
  const uint8_t* pb = b + (long long)img * npix * 3;
  double s[6] = {0, 0, 0, 0, 0, 0};
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
       p += (long long)gridDim.x * blockDim.x) {
    const uint8_t* u = pa + p * 3;
    const uint8_t* v = pb + p * 3;
    int d0 = (int)u[0] - v[0], d1 = (int)u[1] - v[1], d2 = (int)u[2] - v[2];
    s[0] += (d0 | d1 | d2) ? 1.0 : 0.0;
    s[1] += abs(d0) + abs(d1) + abs(d2);
    s[2] += d0 * d0 + d1 * d1 + d2 * d2;
    double L1, A1, B1, L2, A2, B2;
    rgb_to_lab(u, L1, A1, B1);
    rgb_to_lab(v, L2, A2, B2);
    s[3] += sqrt((L1 - L2) * (L1 - L2) + (A1 - A2) * (A1 - A2) + (B1 - B2) * (B1 - B2));
    s[4] += sqrt(L1 * L1 + A1 * A1 + B1 * B1);
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
