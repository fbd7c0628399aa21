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
// normal arguments only, so none of cbrtf's special cases): 2^(log2(t) / 3)
// by MUFU.LG2 and MUFU.EX2, ~2e-7 relative -- the statistics pass is a
// reporting tool (NCD agrees with the float64 oracle to < 2e-6 relative,
// tests/test_gpu_parity.py); VF_STATS_CBRT_NEWTON=1 adds one division-free
// Newton step for the inverse cube root (~1e-7; measured 5.5 vs 3.7 ms for
// the C4 step's three passes).
#ifndef VF_STATS_CBRT_NEWTON
#define VF_STATS_CBRT_NEWTON 0
#endif
__device__ __forceinline__ float cbrt_pos(float t) {
  float l, z;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(t));
#if VF_STATS_CBRT_NEWTON
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(l * (-1.0f / 3.0f)));
  const float tz3 = t * (z * z) * z;
  z = z * fmaf(tz3, -1.0f / 3.0f, 4.0f / 3.0f);
  return t * z * z;
#else
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(l * (1.0f / 3.0f)));   // ~2e-7 relative
  return z;
#endif
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
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

// PX = 4: four consecutive pixels = three aligned 32-bit words (needs
// npix % 4 == 0 and 4-byte aligned image bases); PX = 1: one pixel (load_px).
template <int PX>
__device__ __forceinline__ void load_chunk(const uint8_t* img, long long ch, uint32_t (&px)[PX]) {
  if constexpr (PX == 4) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(img) + ch * 3;
    const uint32_t w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2);
    px[0] = w0 & 0x00ffffffu;
    px[1] = __byte_perm(w0, w1, 0x0543) & 0x00ffffffu;
    px[2] = __byte_perm(w1, w2, 0x0432) & 0x00ffffffu;
    px[3] = w2 >> 8;
  } else {
    px[0] = load_px(img, ch);
  }
}

template <int NB, int PX>
__global__ void __launch_bounds__(256) vf_stats_multi_kernel(const uint8_t* __restrict__ a, const StatsArgs bs,
                                                             long long npix, int B,
                                                             unsigned long long* __restrict__ acc,
                                                             int want_ref_norm) {
  const int img = blockIdx.y;
  const long long ioff = (long long)img * npix * 3;
  const uint8_t* pa = a + ioff;
  __shared__ float lin[256];
  lin[threadIdx.x] = srgb_to_linear_f(threadIdx.x);
  __syncthreads();
  // per thread: exact integer sums (u32: the grid keeps <= 4096 pixels per
  // thread, so sum (a-b)^2 < 8e8), byte-wise running max, fp32 Lab-distance
  // partial sums flushed into double every 8 chunks
  uint32_t ndiff[NB], l1[NB], l2[NB], mxv[NB];
  double s3[NB];
  float f3[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) { ndiff[k] = 0; l1[k] = 0; l2[k] = 0; mxv[k] = 0; s3[k] = 0.0; f3[k] = 0.0f; }
  double s4 = 0.0;
  float f4 = 0.0f;
  int cnt = 0;
  const long long nch = npix / PX;
  // warp-uniform trip count (the warp votes below need every lane): lanes past
  // the end compare the last chunk with itself (no difference, no sums)
  const int lane = threadIdx.x & 31;
  for (long long ch0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); ch0 < nch;
       ch0 += (long long)gridDim.x * blockDim.x) {
    const bool live = ch0 + lane < nch;
    const long long ch = live ? ch0 + lane : nch - 1;
    uint32_t u[PX];
    load_chunk<PX>(pa, ch, u);
    float La[PX], Aa[PX], Ba[PX];
    if (want_ref_norm) {
#pragma unroll
      for (int p = 0; p < PX; ++p) {
        rgb_to_lab(u[p], lin, La[p], Aa[p], Ba[p]);
        f4 += live ? sqrt_approx(La[p] * La[p] + Aa[p] * Aa[p] + Ba[p] * Ba[p]) : 0.0f;
      }
    }
    // exact integer statistics, branch free; dm: the (output, pixel) slots that differ
    uint32_t v[NB][PX];
    uint32_t dm = 0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      load_chunk<PX>(bs.b[k] + ioff, ch, v[k]);
#pragma unroll
      for (int p = 0; p < PX; ++p) {
        if (!live) v[k][p] = u[p];
        const uint32_t ad = __vabsdiffu4(u[p], v[k][p]);       // |a - b| per channel (byte 3 = 0)
        const bool d = u[p] != v[k][p];
        ndiff[k] += d;
        dm |= (d ? 1u : 0u) << (k * PX + p);
        l1[k] = __dp4a(ad, 0x01010101u, l1[k]);
        l2[k] = __dp4a(ad, ad, l2[k]);
        mxv[k] = __vmaxu4(mxv[k], ad);
      }
    }
    // CIELAB distances of the differing slots (filter outputs differ from the
    // reference in few pixels): one slot per lane per pass, so a warp runs
    // max-over-lanes passes instead of one divergent branch per slot
    while (__any_sync(0xffffffffu, dm != 0)) {
      if (dm) {
        const int bit = __ffs(dm) - 1;
        dm &= dm - 1;
        const int k = bit / PX, p = bit % PX;
        uint32_t uu = u[0], vv = v[0][0];
        float L1 = La[0], A1 = Aa[0], B1 = Ba[0];
#pragma unroll
        for (int q = 1; q < PX; ++q)
          if (p == q) { uu = u[q]; L1 = La[q]; A1 = Aa[q]; B1 = Ba[q]; }
#pragma unroll
        for (int kk = 0; kk < NB; ++kk)
#pragma unroll
          for (int q = 0; q < PX; ++q)
            if (bit == kk * PX + q) vv = v[kk][q];
        if (!want_ref_norm) rgb_to_lab(uu, lin, L1, A1, B1);
        float L2, A2, B2;
        rgb_to_lab(vv, lin, L2, A2, B2);
        const float dl = L1 - L2, da = A1 - A2, db = B1 - B2;
        const float dist = sqrt_approx(dl * dl + da * da + db * db);
#pragma unroll
        for (int kk = 0; kk < NB; ++kk) f3[kk] += (k == kk) ? dist : 0.0f;
      }
    }
    if (++cnt == 8) {
#pragma unroll
      for (int k = 0; k < NB; ++k) { s3[k] += f3[k]; f3[k] = 0.0f; }
      s4 += f4;
      f4 = 0.0f;
      cnt = 0;
    }
  }
  s4 += f4;
  __shared__ double red[8][6 * NB + 1];
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k <= NB; ++k) {
    double s[6];
    if (k < NB) {
      s3[k] += f3[k];
      const uint32_t m = mxv[k];
      const uint32_t mx = max(m & 0xffu, max((m >> 8) & 0xffu, (m >> 16) & 0xffu));
      s[0] = (double)ndiff[k]; s[1] = (double)l1[k]; s[2] = (double)l2[k]; s[3] = s3[k]; s[4] = 0.0;
      s[5] = (double)mx;
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
