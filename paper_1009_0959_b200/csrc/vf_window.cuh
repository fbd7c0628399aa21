// vf_window.cuh -- per-window kernels: one thread = one output pixel, all
// n(n-1)/2 pairs of its window evaluated in registers (SURVEY.md 8(a) rows
// a1-a8 fused in one launch).
//
//   a1  stage the block's tile + halo (uint8 HWC -> smem) with replicate
//       clamping against the GLOBAL image rows (stripes), Fig. 1 / S:78;
//   a2  per-pixel precompute once per staged pixel: packed RGB0 (exp/log), or
//       (r, g, b, |x|^2) and (|x|, 1/|x|) (angular);
//   a3  exp/log: window statistic S1 = sum_{i<j} |x_i - x_j|_1 (integer, one
//       VABSDIFF4 per pair) and the scale c_E = n^(1+kappa/3) / (2 S1)
//       (= 1/h_W, Eq. 8) or c_L = (1-1/e)(n-1)/S1;
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
// exp/log kernel: output rows per thread (3x3, large launches: 2 -- shares
// staging and, for the exact variants, 15 of 36 distances; small launches and
// 5x5: 1)

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

// Pointer to the input pixel of global (clamped) coordinates (gy, gx).
__device__ __forceinline__ const uint8_t* pixel_ptr(const Launch& L, const uint8_t* in, int gy, int gx) {
  // Replicate padding clamps to the GLOBAL rows [0, H); the band holds
  // every clamped row a valid output reads (checked by vf_filter_rows), and
  // rows a tile stages beyond the stripe's last output row are clamped into
  // the band too (they feed no stored output).  band = [band_row0,
  // band_row0 + band_rows) is inside [0, H), so one clamp does both.
  gy = clampi(gy, L.band_row0, L.band_row0 + L.band_rows - 1) - L.band_row0;
  gx = clampi(gx, 0, L.W - 1);
  VF_CHECK(gy >= 0 && gy < L.band_rows);
  return in + ((long long)gy * L.W + gx) * 3;
}

// a7 + a8: argmin (lowest index on ties) and store.  The selected sample is
// tracked directly (one FSETP + FSEL + SEL per candidate); its index is only
// formed when the caller asked for it.
template <int N>
__device__ __forceinline__ void store_result(const Launch& L, int b, int ox, int oy, const float (&Ra)[N], uint32_t o) {
  VF_CHECK(oy >= L.out_row0 && oy < L.out_row0 + L.out_rows && ox >= 0 && ox < L.W);
  const long long po = (long long)(oy - L.out_row0) * L.W + ox;
  uint8_t* op = L.out + (long long)b * L.out_stride + po * 3;
  op[0] = (uint8_t)(o & 0xff); op[1] = (uint8_t)((o >> 8) & 0xff); op[2] = (uint8_t)((o >> 16) & 0xff);
  const long long npix_img = (long long)L.out_rows * L.W;
  if (L.idx) {
    int best = 0;
    float bv = Ra[0];
#pragma unroll
    for (int k = 1; k < N; ++k)
      if (Ra[k] < bv) { bv = Ra[k]; best = k; }
    L.idx[b * npix_img + po] = (uint8_t)best;
  }
  if (L.agg) {
    float* a = L.agg + (b * npix_img + po) * N;
#pragma unroll
    for (int k = 0; k < N; ++k) a[k] = Ra[k];
  }
}

template <int N>
__device__ __forceinline__ void argmin_store(const Launch& L, int b, int ox, int oy, const float (&Ra)[N],
                                             const uint32_t (&pk)[N]) {
  float bv = Ra[0];
  uint32_t o = pk[0];
#pragma unroll
  for (int k = 1; k < N; ++k) {
    const bool lt = Ra[k] < bv;   // strict: the lowest index wins exact ties
    bv = lt ? Ra[k] : bv;
    o = lt ? pk[k] : o;
  }
  store_result<N>(L, b, ox, oy, Ra, o);
}

// ============================================================================
// exp / log criteria (readings R2, R3): everything derives from the integer L1
// distances, so a sample is one packed RGB0 word and the L1 distance of a pair
// is one VABSDIFF4.  Pass 1 forms S1 exactly in integers; pass 2 recomputes
// each distance already biased into a float (2^23 + d1) and turns it into the
// scaled argument with one FFMA.
// ============================================================================
// One exp/log window with kept biased distances (3x3).  SHIFTED: the kept
// values hold the previous (one row higher) window's pairs; pairs of rows
// 0..1 of this window are pairs of rows 1..2 of the previous one.
template <int WIN, int CRIT, int VAR, bool SHIFTED>
__device__ __forceinline__ void el_window(const Launch& L, int b, int ox, int oy, const uint32_t* w,
                                          uint32_t (&keep)[WIN * WIN * (WIN * WIN - 1) / 2]) {
  constexpr int N = WIN * WIN;
  constexpr int NPR = N * (N - 1) / 2;
  if (SHIFTED) {
    // pairs of rows 1..WIN-1 of the previous window move to rows 0..WIN-2
    static_for<NPR>([&](auto pc) {
      constexpr int p = decltype(pc)::value;
      constexpr int i = pair_i<N>(p), j = pair_j<N>(p);
      if constexpr (j < N - WIN) keep[p] = keep[pair_index<N>(i + WIN, j + WIN)];   // source index > p: not yet overwritten
    });
  }
  // a3: S1 = sum - NPR * 0x4B000000 (mod 2^32; exact integer)
  uint32_t acc[3] = {0u, 0u, 0u};
  static_for<NPR>([&](auto pc) {
    constexpr int p = decltype(pc)::value;
    constexpr int i = pair_i<N>(p), j = pair_j<N>(p);
    if constexpr (!SHIFTED || j >= N - WIN) keep[p] = sad4(w[i], w[j], F2P23_BITS);
    acc[p % 3] += keep[p];
  });
  const uint32_t S1 = (acc[0] + acc[1]) + acc[2] - (uint32_t)(NPR * F2P23_BITS);
  float Ra[N];
#pragma unroll
  for (int k = 0; k < N; ++k) Ra[k] = (S1 != 0u) ? -0.0f : 0.0f;   // -0 + v == v: first add folds
  if (S1 != 0u) {                                                   // flat window: all D = 0 (R18)
    const float sc = L.kscale * rcp_approx((float)S1);              // c_E = 1/h_W, or c_L
    const float bias = -sc * F2P23;                                 // exact
    static_for<NPR>([&](auto pc) {
      constexpr int p = decltype(pc)::value;
      const float zu = fmaf(sc, __uint_as_float(keep[p]), bias);   // c * d1, one rounding
      crit_accumulate<CRIT, VAR, (VAR == EXACT && WIN >= VF_EXACT_CALL_MINWIN)>(zu, Ra[pair_i<N>(p)], Ra[pair_j<N>(p)]);
    });
  }
  uint32_t ww[N];
#pragma unroll
  for (int k = 0; k < N; ++k) ww[k] = w[k];
  argmin_store<N>(L, b, ox, oy, Ra, ww);
}

// a3 for a thread's column strip of OPT vertically adjacent windows (rows
// 0..OPT+WIN-2 of samples w[row * WIN + col]): S1 of window o is the sum of
// the intra-row pair sums T[r] of its rows and the cross-row sums C[r][dr] of
// its row pairs, so the row pairs two windows share are summed once (3x3 with
// 4 windows per thread: 99 instead of 144 VABSDIFF4).
template <int WIN, int OPT>
struct StripS1 {
  static constexpr int LR = OPT + WIN - 1;
  uint32_t T[LR];
  uint32_t C[LR][WIN - 1];   // C[r][dr - 1]: pairs (row r, row r + dr)
  __device__ __forceinline__ void build(const uint32_t* w) {
#pragma unroll
    for (int r = 0; r < LR; ++r) {
      uint32_t t = 0u;
#pragma unroll
      for (int a = 0; a < WIN; ++a)
#pragma unroll
        for (int c = a + 1; c < WIN; ++c) t = sad4(w[r * WIN + a], w[r * WIN + c], t);
      T[r] = t;
#pragma unroll
      for (int dr = 1; dr < WIN; ++dr) {
        uint32_t x = 0u;
        if (r + dr < LR) {
#pragma unroll
          for (int a = 0; a < WIN; ++a)
#pragma unroll
            for (int c = 0; c < WIN; ++c) x = sad4(w[r * WIN + a], w[(r + dr) * WIN + c], x);
        }
        C[r][dr - 1] = x;
      }
    }
  }
  __device__ __forceinline__ uint32_t window(int o) const {   // o compile-time after unrolling
    uint32_t s = 0u;
#pragma unroll
    for (int r = 0; r < WIN; ++r) {
      s += T[o + r];
#pragma unroll
      for (int dr = 1; dr < WIN - r; ++dr) s += C[o + r][dr - 1];
    }
    return s;
  }
};

// One exp/log window recomputing the distances in pass 2, given S1.  A flat
// window (S1 = 0, all samples equal) runs the same code with scale 0: every
// pair then gets the same value D(0), all aggregates tie and the lowest index
// (= the common sample) wins; the reported aggregates are 0 (reading R18).
template <int WIN, int CRIT, int VAR>
__device__ __forceinline__ void el_window_s1(const Launch& L, int b, int ox, int oy, const uint32_t* w, uint32_t S1) {
  constexpr int N = WIN * WIN;
  const float sc = (S1 != 0u) ? L.kscale * rcp_approx((float)S1) : 0.0f;   // c_E = 1/h_W, or c_L
  const float bias = -sc * F2P23;                                         // exact
  float Ra[N];
#pragma unroll
  for (int k = 0; k < N; ++k) Ra[k] = -0.0f;   // -0 + v == v: the first add folds away
  if constexpr (VAR == EXACT && WIN >= VF_EXACT_ROLL_MINWIN) {
    // Rolled form (knob): N is odd, so the pairs {k, (k + d) mod N},
    // d = 1 .. (N - 1) / 2, k = 0 .. N - 1, are every unordered pair once.  One
    // loop iteration per d with the second sample and its partial aggregate in
    // registers that rotate by one position per iteration: N inlined libm
    // calls of code instead of N (N - 1) / 2.
    uint32_t wb[N];
    float Rb[N];
#pragma unroll
    for (int k = 0; k < N; ++k) { wb[k] = w[k]; Rb[k] = -0.0f; }
#pragma unroll 1
    for (int d = 1; d <= (N - 1) / 2; ++d) {
      const uint32_t w0 = wb[0];
      const float r0 = Rb[0];
#pragma unroll
      for (int k = 0; k + 1 < N; ++k) { wb[k] = wb[k + 1]; Rb[k] = Rb[k + 1]; }
      wb[N - 1] = w0;                                                    // wb[k] = w[(k + d) mod N]
      Rb[N - 1] = r0;                                                    // Rb[k]: partial aggregate of that sample
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const float fb = __uint_as_float(sad4(w[k], wb[k], F2P23_BITS));   // 2^23 + d1
        const float zu = fmaf(sc, fb, bias);                               // c * d1, one rounding
        crit_accumulate<CRIT, VAR>(zu, Ra[k], Rb[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) Ra[(k + (N - 1) / 2) % N] = __fadd_rn(Ra[(k + (N - 1) / 2) % N], Rb[k]);
  } else if constexpr (VAR == EXACT) {
    static_for<N * (N - 1) / 2>([&](auto pc) {
      constexpr int i = pair_i<N>(decltype(pc)::value), j = pair_j<N>(decltype(pc)::value);
      const float fb = __uint_as_float(sad4(w[i], w[j], F2P23_BITS));   // 2^23 + d1
      const float zu = fmaf(sc, fb, bias);                               // c * d1, one rounding
      crit_accumulate<CRIT, VAR, (WIN >= VF_EXACT_CALL_MINWIN)>(zu, Ra[i], Ra[j]);
    });
  } else {
    // polynomial variants: pairs 2q and 2q + 1 together in packed FP32
    // (FFMA2), one Horner chain issue for both, scalar accumulation (packed
    // aggregates were measured slower)
    const f32x2 sc2 = pack2(sc, sc), bias2 = pack2(bias, bias);
    static_for<N * (N - 1) / 4>([&](auto qc) {
      constexpr int p0 = 2 * decltype(qc)::value, p1 = p0 + 1;
      constexpr int i0 = pair_i<N>(p0), j0 = pair_j<N>(p0), i1 = pair_i<N>(p1), j1 = pair_j<N>(p1);
      const f32x2 fb2 = pack2(__uint_as_float(sad4(w[i0], w[j0], F2P23_BITS)),
                              __uint_as_float(sad4(w[i1], w[j1], F2P23_BITS)));   // 2^23 + d1, two pairs
      crit_accumulate2<CRIT, VAR>(fma2(sc2, fb2, bias2), Ra[i0], Ra[j0], Ra[i1], Ra[j1]);
    });
  }
  float bv = Ra[0];
  uint32_t o = w[0];
#pragma unroll
  for (int k = 1; k < N; ++k) {
    const bool lt = Ra[k] < bv;
    bv = lt ? Ra[k] : bv;
    o = lt ? w[k] : o;
  }
  if (L.agg && S1 == 0u) {
#pragma unroll
    for (int k = 0; k < N; ++k) Ra[k] = 0.0f;
  }
  store_result<N>(L, b, ox, oy, Ra, o);
}

// a1 + a2: stage the block's SH x SW pixel region (global origin (gx0, gy0),
// replicate-clamped against the image / band) as packed RGB0 words.
// Interior regions (no clamping needed) are read as whole 32-bit words, one
// warp per row (lane l loads word l of the row's byte range; the first and
// last word may extend up to 3 bytes beyond the range but never beyond the
// aligned words that hold its bytes), then repacked from shared memory with
// one funnel shift per pixel.  Regions touching a border take the clamped
// byte path.
template <int SW, int SH>
struct StageSmem {
  static constexpr int RWW = (SW * 3 + 3 + 3) / 4 + 1;   // raw words per row (+1: the funnel shift's high word)
  uint32_t pk[SH * SW];
  uint32_t raw[SH * RWW];
};

template <int SW, int SH, int NTH_X, int NTH_Y>
__device__ __forceinline__ void stage_packed(const Launch& L, const uint8_t* __restrict__ in, int gx0, int gy0,
                                             StageSmem<SW, SH>& sm) {
  constexpr int RWW = StageSmem<SW, SH>::RWW;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const bool inner = gx0 >= 0 && gx0 + SW <= L.W && gy0 >= L.band_row0 && gy0 + SH <= L.band_row0 + L.band_rows;
  if (inner) {
    const uint8_t* row0 = in + ((long long)(gy0 - L.band_row0) * L.W + gx0) * 3;
    const long long rstride = (long long)L.W * 3;
    for (int r = ty; r < SH; r += NTH_Y) {
      const uintptr_t ra = (uintptr_t)(row0 + r * rstride);
      const uint32_t* wp = (const uint32_t*)(ra & ~(uintptr_t)3);
      const int nw = (int)(((ra & 3) + SW * 3 + 3) >> 2);   // words holding the row's bytes
      for (int k = tx; k < nw; k += NTH_X) sm.raw[r * RWW + k] = __ldg(wp + k);
    }
    __syncthreads();
    const int tid = ty * NTH_X + tx;
    for (int p = tid; p < SH * SW; p += NTH_X * NTH_Y) {
      const int r = p / SW, c = p - r * SW;
      const int o = (int)((uintptr_t)(row0 + r * rstride) & 3) + 3 * c;
      VF_CHECK((o >> 2) + 1 < RWW);
      const uint32_t w0 = sm.raw[r * RWW + (o >> 2)], w1 = sm.raw[r * RWW + (o >> 2) + 1];
      sm.pk[p] = __funnelshift_r(w0, w1, (o & 3) * 8) & 0x00ffffffu;
    }
  } else {
    for (int row = ty; row < SH; row += NTH_Y) {
      const int gy = clampi(gy0 + row, L.band_row0, L.band_row0 + L.band_rows - 1) - L.band_row0;   // see pixel_ptr
      VF_CHECK(gy >= 0 && gy < L.band_rows);
      const uint8_t* rp = in + (long long)gy * L.W * 3;
      for (int col = tx; col < SW; col += NTH_X) {
        const uint8_t* q = rp + clampi(gx0 + col, 0, L.W - 1) * 3;
        sm.pk[row * SW + col] = pack_rgb(q[0], q[1], q[2]);
      }
    }
  }
  __syncthreads();
}

// a2-a8 for one staged tile: thread (tx, ty) reads its (OPT + w - 1) x w
// samples (packed RGB0, region row-major with row length TX + w - 1) and
// produces outputs (x0 + tx, y0 + OPT ty + o), o < OPT.
template <int WIN, int CRIT, int VAR, int OPT>
__device__ __forceinline__ void el_compute_tile(const Launch& L, int b, int x0, int y0, const uint32_t* s_pk) {
  constexpr int N = WIN * WIN;
  constexpr int SW = TX + WIN - 1;
  constexpr int LR = OPT + WIN - 1;            // sample rows a thread reads
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int ox = x0 + tx;
  const int oyb = y0 + OPT * ty;
  if (ox >= L.W || oyb >= L.out_row0 + L.out_rows) return;

  uint32_t pk[LR * WIN];
#pragma unroll
  for (int k = 0; k < LR * WIN; ++k) pk[k] = s_pk[(OPT * ty + k / WIN) * SW + tx + k % WIN];

  const int rows_here = min(OPT, L.out_row0 + L.out_rows - oyb);   // >= 1
  if (N <= 9 && VAR == EXACT) {
    // 3x3 exact: the biased L1 distances 2^23 + d1 of a window's 36 pairs are
    // computed once (one VABSDIFF4 each) and kept in registers for both passes;
    // the 15 pairs two vertically adjacent windows share are computed once per
    // thread (measured: -10% time for the libm variants, no gain for the
    // minimax ones, whose occupancy it lowers).
    uint32_t keep[N * (N - 1) / 2];
    el_window<WIN, CRIT, VAR, false>(L, b, ox, oyb, pk, keep);
#pragma unroll
    for (int o = 1; o < OPT; ++o)
      if (o < rows_here) el_window<WIN, CRIT, VAR, true>(L, b, ox, oyb + o, pk + o * WIN, keep);
  } else {
    StripS1<WIN, OPT> s1;
    s1.build(pk);
#pragma unroll
    for (int o = 0; o < OPT; ++o)
      if (o < rows_here) el_window_s1<WIN, CRIT, VAR>(L, b, ox, oyb + o, pk + o * WIN, s1.window(o));
  }
}

// NTY = warps per block (block 32 x NTY threads, output tile 32 x NTY*OPT).
template <int WIN, int CRIT, int VAR, int OPT, int NTY = TY>
__global__ void __launch_bounds__(TX * NTY) vf_el_kernel(const Launch L) {
  constexpr int R = WIN / 2;
  constexpr int TYE = NTY * OPT;               // output tile height
  constexpr int SW = TX + 2 * R;
  constexpr int SH = TYE + 2 * R;
  __shared__ StageSmem<SW, SH> sm;

  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX;
  const int y0 = L.out_row0 + blockIdx.y * TYE;
  const uint8_t* __restrict__ in = L.in + (long long)b * L.in_stride;
  stage_packed<SW, SH, TX, NTY>(L, in, x0 - R, y0 - R, sm);

  el_compute_tile<WIN, CRIT, VAR, OPT>(L, b, x0, y0, sm.pk);
}

// ============================================================================
// angular criterion, per-window (VF_ALGO_WINDOW).  See vf_shared.cuh for the
// cross-window pair-sharing kernel used by default.
// ============================================================================
template <int WIN, int VAR>
__global__ void __launch_bounds__(TX * TY) vf_angular_window_kernel(const Launch L) {
  constexpr int R = WIN / 2;
  constexpr int N = WIN * WIN;
  constexpr int SW = TX + 2 * R;
  constexpr int SH = TY + 2 * R;
  __shared__ float4 s_px[SH * SW];                        // r, g, b, |x|^2
  __shared__ float2 s_nm[SH * SW];                        // |x|, 1/|x|
  __shared__ uint32_t s_pk[SH * SW];                      // packed RGB0 (output)

  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX;
  const int y0 = L.out_row0 + blockIdx.y * TY;
  const uint8_t* __restrict__ in = L.in + (long long)b * L.in_stride;
  const int tid = threadIdx.y * TX + threadIdx.x;
  for (int p = tid; p < SH * SW; p += TX * TY) {
    const int sy = p / SW, sx = p - sy * SW;
    const uint8_t* q = pixel_ptr(L, in, y0 + sy - R, x0 + sx - R);
    const float r = q[0], g = q[1], bl = q[2];
    const float nn = fmaf(r, r, fmaf(g, g, bl * bl));    // exact integer < 2^18
    s_px[p] = make_float4(r, g, bl, nn);
    const float nrm = sqrtf(nn);
    s_nm[p] = make_float2(nrm, nn > 0.0f ? 1.0f / nrm : 0.0f);
    s_pk[p] = pack_rgb(q[0], q[1], q[2]);
  }
  __syncthreads();

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int ox = x0 + tx, oy = y0 + ty;
  if (ox >= L.W || oy >= L.out_row0 + L.out_rows) return;

  float xr[N], xg[N], xb[N], xn[N], xm[N], xi[N];
  uint32_t pk[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const int a = (ty + k / WIN) * SW + tx + k % WIN;
    const float4 v = s_px[a];
    xr[k] = v.x; xg[k] = v.y; xb[k] = v.z; xn[k] = v.w;
    const float2 u = s_nm[a];
    xm[k] = u.x; xi[k] = u.y;
  }
  float Ra[N];
#pragma unroll
  for (int k = 0; k < N; ++k) Ra[k] = -0.0f;              // -0 + v == v: the first add folds away
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = i + 1; j < N; ++j) {
      const float d = angular_pair<VAR>(xr[i], xg[i], xb[i], xn[i], xm[i], xi[i],
                                        xr[j], xg[j], xb[j], xn[j], xm[j], xi[j]);
      Ra[i] = __fadd_rn(Ra[i], d);   // never contracted with d's last product
      Ra[j] = __fadd_rn(Ra[j], d);
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
#pragma unroll
  for (int k = 0; k < N; ++k) pk[k] = s_pk[(ty + k / WIN) * SW + tx + k % WIN];
  argmin_store<N>(L, b, ox, oy, Ra, pk);
}

}  // namespace vf
