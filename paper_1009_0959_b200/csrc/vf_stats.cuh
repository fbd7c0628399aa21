// vf_stats.cuh -- per-image fidelity statistics of two output images
// (MAE, MSE, NCD of PAPER.md P:286-293; CIELAB via sRGB/D65).
#pragma once
#include <cstdint>

namespace vf {

// sRGB decoding (IEC 61966-2-1) is a 256-entry table: computed once per
// device on the host in double precision (vf_api.cu, srgb_table) and copied
// into shared memory by each block that needs it (one load per thread).
__device__ __forceinline__ void load_srgb_table(float* lin_s, const float* __restrict__ tab, int tid, int nthreads) {
  for (int i = tid; i < 256; i += nthreads) lin_s[i] = __ldg(tab + i);
}

// t^(1/3) for t in (0.0088, 1.1] (the CIELAB cube-root branch: positive
// normal arguments only, so none of cbrtf's special cases): 2^(log2(t) / 3)
// by MUFU.LG2 and MUFU.EX2, ~2e-7 relative -- the statistics are a reporting
// tool (NCD agrees with the float64 oracle to < 2e-6 relative,
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
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(__fmul_rn(l, -1.0f / 3.0f)));
  const float tz3 = __fmul_rn(__fmul_rn(t, __fmul_rn(z, z)), z);
  z = __fmul_rn(z, fmaf(tz3, -1.0f / 3.0f, 4.0f / 3.0f));
  return __fmul_rn(__fmul_rn(t, z), z);
#else
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(__fmul_rn(l, 1.0f / 3.0f)));   // ~2e-7 relative
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
  return t > d * d * d ? cbrt_pos(t) : fmaf(t, 1.0f / (3.0f * d * d), 4.0f / 29.0f);
}

// CIELAB of one pixel (sRGB, BT.709 primaries, D65), fp32 per pixel.  pk =
// packed RGB (r | g << 8 | b << 16).  Every rounding is spelled out (fmaf /
// __fmul_rn / __fsub_rn, never contracted differently by the compiler), so a
// pixel's CIELAB -- and its fixed-point contributions below -- are the same
// bits in every instantiation that evaluates it.
__device__ __forceinline__ void rgb_to_lab(uint32_t pk, const float* lin, float& L, float& A, float& B) {
  const float r = lin[pk & 0xff], g = lin[(pk >> 8) & 0xff], b = lin[(pk >> 16) & 0xff];
  const float X = fmaf(0.1804375f, b, fmaf(0.3575761f, g, __fmul_rn(0.4124564f, r)));
  const float Y = fmaf(0.0721750f, b, fmaf(0.7151522f, g, __fmul_rn(0.2126729f, r)));
  const float Z = fmaf(0.9503041f, b, fmaf(0.1191920f, g, __fmul_rn(0.0193339f, r)));
  const float fx = lab_f(__fmul_rn(X, 1.0f / 0.95047f)), fy = lab_f(Y), fz = lab_f(__fmul_rn(Z, 1.0f / 1.08883f));
  L = fmaf(116.0f, fy, -16.0f);
  A = __fmul_rn(500.0f, __fsub_rn(fx, fy));
  B = __fmul_rn(200.0f, __fsub_rn(fy, fz));
}
__device__ __forceinline__ float norm3(float a, float b, float c) {
  return sqrt_approx(fmaf(a, a, fmaf(b, b, __fmul_rn(c, c))));
}
// |x_Lab|_2 and |x_Lab - y_Lab|_2 (NCD's denominator and numerator terms)
__device__ __forceinline__ float lab_norm(uint32_t pk, const float* lin) {
  float L, A, B;
  rgb_to_lab(pk, lin, L, A, B);
  return norm3(L, A, B);
}
__device__ __forceinline__ float lab_dist(float L1, float A1, float B1, uint32_t pk2, const float* lin) {
  float L2, A2, B2;
  rgb_to_lab(pk2, lin, L2, A2, B2);
  return norm3(__fsub_rn(L1, L2), __fsub_rn(A1, A2), __fsub_rn(B1, B2));
}

// Fixed point of the floating-point sums (columns 3, 4): every pixel's fp32
// value is rounded to a multiple of 2^-23 (a 32-bit integer: |Lab| <= 207 and
// Lab distances <= 300 stay below 512) and the per-image totals are integer
// sums (64-bit atomics), so they do not depend on the order in which threads,
// warps and blocks finish, nor on how the outputs are grouped into passes.
constexpr double STATS_FIX = 8388608.0;   // 2^23
__device__ __forceinline__ uint32_t stats_fix(float v) { return __float2uint_rn(__fmul_rn(v, 8388608.0f)); }

// Warp sum of 32-bit values as a 64-bit integer (two REDUX.SUM over the 16-bit
// halves; exact).  mask: the lanes taking part (all must call it).
__device__ __forceinline__ unsigned long long warp_sum_u32(uint32_t mask, uint32_t v) {
  const uint32_t hi = __reduce_add_sync(mask, v >> 16), lo = __reduce_add_sync(mask, v & 0xffffu);
  return ((unsigned long long)hi << 16) + lo;
}
__device__ __forceinline__ uint32_t max_byte3(uint32_t ad) {
  return max(ad & 0xffu, max((ad >> 8) & 0xffu, (ad >> 16) & 0xffu));
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

// Per-image statistics of NB outputs b_k against one reference a, in ONE pass
// over a (each reference pixel is read once and its CIELAB computed at most
// once).  grid (blocks, B), 256 threads.  acc[row[k]][B][8] (uint64, zeroed
// before launch): {count a != b, sum |a-b|, sum (a-b)^2, fix(sum |a_Lab -
// b_Lab|), fix(sum |a_Lab|), max |a-b|, 0, 0}; vf_stats_finalize converts to
// double.  Per thread: 32-bit integer sums (the grid keeps <= 4096 pixels per
// thread, so sum (a-b)^2 < 8e8) and 64-bit sums of the per-pixel fixed-point
// Lab values; per warp one reduction and one atomic per value.
struct StatsArgs {
  const uint8_t* b[8];
  int row[8];     // acc row of output k (vf_image_stats_multi: k; plans: the comparison index)
  const float* lin;   // the device's sRGB decoding table (256 floats)
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

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
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
  load_srgb_table(lin, bs.lin, threadIdx.x, blockDim.x);
  __syncthreads();
  uint32_t ndiff[NB], l1[NB], l2[NB], mxv[NB];
  unsigned long long s3[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) { ndiff[k] = 0; l1[k] = 0; l2[k] = 0; mxv[k] = 0; s3[k] = 0ull; }
  unsigned long long s4 = 0ull;
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
        s4 += live ? stats_fix(norm3(La[p], Aa[p], Ba[p])) : 0u;
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
        const uint32_t dist = stats_fix(lab_dist(L1, A1, B1, vv, lin));
#pragma unroll
        for (int kk = 0; kk < NB; ++kk) s3[kk] += (k == kk) ? dist : 0u;
      }
    }
  }
  // per warp: one reduction and one atomic per value (integers: order-independent)
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    unsigned long long* row = acc + ((long long)bs.row[k] * B + img) * 8;
    const unsigned long long c0 = warp_sum_u32(0xffffffffu, ndiff[k]);
    const unsigned long long c1 = warp_sum_u32(0xffffffffu, l1[k]);
    const unsigned long long c2 = warp_sum_u64(l2[k]);
    const unsigned long long c3 = warp_sum_u64(s3[k]);
    const uint32_t c5 = __reduce_max_sync(0xffffffffu, max_byte3(mxv[k]));
    if (lane == 0 && c0 != 0) {
      atomicAdd(&row[0], c0);
      atomicAdd(&row[1], c1);
      atomicAdd(&row[2], c2);
      atomicAdd(&row[3], c3);
      atomicMax(&row[5], (unsigned long long)c5);
    }
  }
  if (want_ref_norm) {                                       // reference norm: column 4 of every output
    const unsigned long long c4 = warp_sum_u64(s4);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < NB; ++k) atomicAdd(&acc[((long long)bs.row[k] * B + img) * 8 + 4], c4);
  }
}

// acc (uint64 sums, fixed point for columns 3 and 4) -> double, in place.
static __global__ void vf_stats_finalize(unsigned long long* acc, long long n) {   // (static: one per TU)
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long q = acc[i];
  const int c = (int)(i % 8);
  const double v = (c == 3 || c == 4) ? (double)q / STATS_FIX : (double)q;
  reinterpret_cast<double*>(acc)[i] = v;
}

}  // namespace vf
