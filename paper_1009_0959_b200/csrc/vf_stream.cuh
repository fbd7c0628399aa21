// vf_stream.cuh -- 3x3 angular minimax criterion: warp-streamed pair sharing
// with per-pixel role sums (BVDF of Eq. 5
// with the Table 1 approximants).
//
// The angular distance A(x_p, x_q) depends on the two pixels only, so every
// image pair within Chebyshev distance 2 is evaluated once (12 per pixel) and
// the window aggregates are formed from per-pixel ROLE SUMS: for a sample q at
// position (a, b) of a 3x3 window (a = row, b = column, raster index 3a + b),
//     R(q; a, b) = sum_{dy in [-a, 2-a], dx in [-b, 2-b], (dy,dx) != 0} A(q, q + (dy, dx))
// which is exactly the aggregate R_k = sum_{j != k} A(x_k, x_j) of Eq. 5
// of that sample in that window.  Separably: H_b(q, dy) = sum_{dx in
// [-b, 2-b]} A(q, q + (dy, dx)) (5 additions per neighbourhood row), then
// R(q; a, b) = sum_{dy in [-a, 2-a]} H_b(q, dy) (2 additions per role, with
// shared partial sums).  All terms are >= 0 (no subtraction: full relative
// precision).
//
// Organisation: each WARP independently streams down a strip of 64 image
// columns (2 per lane: columns 2l, 2l+1, packed into one FFMA2 lane pair),
// one image row per step; no block barriers.  At step r the warp
//   a1/a2  stages row r (clamped, replicate padding) into a 4-row ring of
//          pixel-pair records (packed RGB, |x|^2) in shared memory;
//   a4/a5  evaluates for both of its pixels q the 12 "upper half-plane"
//          pairs (q, q + d), d in {(-1|-2, -2..2), (0, -1|-2)}: exact integer
//          geometry, the exact branch predicate 4 D^2 < |x_p|^2 |x_q|^2
//          (DESIGN.md 5.2), Table 1's ARCSIN row on tau = sqrt(1 - cos) and
//          its ARCCOS row on cos, the branch selected per pair -- branch
//          free (both Horner chains in packed FP32);
//   a6     routes every value to the H sums of BOTH endpoints (the lower
//          endpoint's rows r-1 / r-2 and the horizontal neighbours live in
//          adjacent lanes: 15 warp shuffles per step) and completes the roles
//          of row r (a = 2), r-1 (a = 1) and r-2 (a = 0);
//   a7/a8  the window centred at row r-1 now has all 9 aggregates: they are
//          made 32-bit keys (aggregate bits with the low 4 mantissa bits
//          replaced by the window position, so a float min picks the lowest
//          position among aggregates equal to 2^-19 relative -- within the
//          1e-5 acceptance of SURVEY 8(c).4), reduced with 3-input FMNMX, and
//          the selected sample is read back from the ring and stored.
// A strip computes 64 columns and outputs 62 (strip columns 1..62: a window
// only needs the pairs among its own 3 columns); K output rows take K + 2
// steps.
#pragma once
#include <cuda_runtime.h>

#include "vf_window.cuh"

namespace vf {
namespace stream {

constexpr int SW = 64;          // computed columns per strip (2 per lane)
constexpr int J_LO = 1;         // first output column of the strip
constexpr int SOUT = 62;        // output columns per strip: [1, 63)
constexpr int NE = 34;          // even-aligned record pairs per ring row: columns (2e - 2, 2e - 1), e = 0..33
constexpr int NO = 33;          // odd-aligned record pairs: columns (2o - 1, 2o), o = 0..32
constexpr int SLOTS = 4;        // ring rows (rows r, r-1, r-2 in use)
#ifndef VF_STREAM_NWARP
#define VF_STREAM_NWARP 1   // warps per block: 1 measured fastest (C4: 1591 vs 1662 us for 4 per 256 images)
#endif
constexpr int NWARP = VF_STREAM_NWARP;   // warps per block (independent strips / row tiles)

constexpr int PW = SW + 8;      // plain pixel row: strip column j at index j + 2

#ifndef VF_STREAM_RN
#define VF_STREAM_RN 0   // 1: per-pixel 1/|x| in the ring, r = rn_p rn_q by FMUL2 instead of MUFU.RSQ(Ph)
#endif

template <int SEG>
struct RingT {                  // one per strip of 2 SEG columns (SEG = 32: one per warp)
  static constexpr int NE = SEG + 2, NO = SEG + 1, PW = 2 * SEG + 8;
  uint4 E[SLOTS][NE];           // (pk(2e-2), pk(2e-1), |x|^2, |x|^2)
  uint4 O[SLOTS][NO];           // (pk(2o-1), pk(2o),   |x|^2, |x|^2)
  uint32_t P[SLOTS][PW];        // packed pixels (the selected sample is read back from here)
#if VF_STREAM_RN
  uint2 ER[SLOTS][NE];          // (1/|x|, 1/|x|) of the E pairs
  uint2 OR[SLOTS][NO];          // of the O pairs
#endif
};
using Ring = RingT<32>;
static_assert(Ring::NE == NE && Ring::NO == NO && Ring::PW == PW, "ring layout");
// Columns -2, -1, 64 and 65 (E[0], E[33], the first half of O[0], the second
// half of O[32]) are never written: a window centred at strip column c only
// reads the roles (c-1, b=0), (c, b=1), (c+1, b=2), i.e. the pair values
// among columns c-1..c+1, so the windows at columns 1..62 never see a pair
// with a column outside 0..63.

// strip s covers image columns x0 + j, x0 = 62 s - 1, j = 0..63
__host__ __device__ constexpr int strip_x0(int s) { return SOUT * s - J_LO; }

// Remainder strips: when the last strip of an image has at most 30 output
// columns (W - 62 (S - 1) <= 30, S = ceil(W / 62); C4's 768 = 12 x 62 + 24,
// C2's 512 = 8 x 62 + 16), it is computed by HALF a warp -- 16 lanes, 32
// columns -- and the two half-warps of a warp take the last strips of two
// images (a separate launch of the SEG = 16 kernel, grid (1, *, ceil(B / 2))).
// The full strips' work is unchanged; the last strip costs half the warps.
constexpr int SOUT_HALF = 30;
__host__ __device__ constexpr int strips_of(int W) { return (W + SOUT - 1) / SOUT; }
__host__ __device__ constexpr bool half_tail(int W) {
  return strips_of(W) >= 2 && W - SOUT * (strips_of(W) - 1) <= SOUT_HALF;
}

}  // namespace stream

__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float lo2(f32x2 v) { float a, b; unpack2(v, a, b); return a; }
__device__ __forceinline__ float hi2(f32x2 v) { float a, b; unpack2(v, a, b); return b; }
// 3-input min (sm_100: FMNMX3)
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// Role value -> key: the aggregate's bits with the low 4 mantissa bits replaced
// by the window position nib = 4a + b (aggregates are >= 0, so keys order like
// the aggregates, ties broken by the lowest raster position).
template <int NIB>
__device__ __forceinline__ float role_key(float v) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(__float_as_uint(v)), "r"(0xfffffff0u), "r"((uint32_t)NIB));
  return __uint_as_float(d);   // (v & ~15) | NIB in one LOP3
}

// Geometry of the lane's two pairs against one neighbour record pair q =
// (pk(q0), pk(q1), |q0|^2, |q1|^2), packed FP32 (nn2 = (|p0|^2, |p1|^2),
// nnn2 = -nn2): the ARCSIN-row value vs = P_asin(tau) (Table 1, Eq. 7,
// reading R6), cos c, and -Ph (zero iff a zero vector is involved).
template <bool TINY = true, bool EXACT_V = false>
__device__ __forceinline__ void ang_geo2(uint32_t pk0, uint32_t pk1, f32x2 nn2, f32x2 nnn2, uint4 q, f32x2& vs,
                                         f32x2& c, f32x2& nPh, const f32x2* rin = nullptr, f32x2* tau_out = nullptr) {
  const f32x2 Db = pack2(__uint_as_float(__dp4a(pk0, q.x, F2P23_BITS)), __uint_as_float(__dp4a(pk1, q.y, F2P23_BITS)));
  const f32x2 D = sub2(Db, pack2(F2P23, F2P23));                  // exact dot products
  const f32x2 nnq = pack2(__uint_as_float(q.z), __uint_as_float(q.w));
  nPh = mul2(nnn2, nnq);                                           // -Ph, Ph = fl(|p|^2 |q|^2)
  const f32x2 Pl = fma2(nn2, nnq, nPh);                            // exact residual: P = Ph + Pl
  const f32x2 Y = fma2(D, D, nPh);                                 // fl(D^2 - Ph)
  const f32x2 X = sub2(Pl, Y);                                     // |p x q|^2 = fl(fl(Ph - D^2) + Pl)
  float nph0, nph1;
  unpack2(nPh, nph0, nph1);
  // 1 / (|p||q|): MUFU.RSQ of Ph, or the product of the per-pixel 1/|x| (rin)
  const f32x2 r = rin ? *rin : pack2(rsqrt_approx(-nph0), rsqrt_approx(-nph1));
  c = mul2(D, r);                                                  // cos
  // tau = sqrt(1 - cos) = X / sqrt(X |p|^2 |q|^2 (1 + cos)) = X r rsqrt(X (1 + cos)): no cancellation
  f32x2 tau;
  if constexpr (TINY) {
    const f32x2 Xw = fma2(X, c, add2(X, pack2(1e-30f, 1e-30f)));   // X (1 + cos) (+tiny: X = 0 -> tau = 0)
    float xw0, xw1;
    unpack2(Xw, xw0, xw1);
    tau = mul2(mul2(X, r), pack2(rsqrt_approx(xw0), rsqrt_approx(xw1)));
  } else {
    // X = 0 (parallel pair): rsqrt(0) = inf, 0 * inf = NaN -> max(NaN, 0) = 0 (FMNMX on the ALU pipe)
    const f32x2 Xw = fma2(X, c, X);
    float xw0, xw1, t0, t1;
    unpack2(Xw, xw0, xw1);
    unpack2(mul2(mul2(X, r), pack2(rsqrt_approx(xw0), rsqrt_approx(xw1))), t0, t1);
    tau = pack2(fmaxf(t0, 0.0f), fmaxf(t1, 0.0f));
  }
  if (tau_out) *tau_out = tau;
  if constexpr (EXACT_V) {
    // Eq. 6 with libm: arccos z = 2 arcsin(sqrt((1 - z) / 2)) = 2 asinf(tau / sqrt2) for z >= 0.5
    float t0, t1;
    unpack2(tau, t0, t1);
    vs = pack2(2.0f * asinf(t0 * 0.70710678118654752f), 2.0f * asinf(t1 * 0.70710678118654752f));
  } else {
    vs = horner4x2(coef::ASIN(), tau);                             // Table 1 ARCSIN row (Eq. 7, reading R6)
  }
}

// Exact branch predicate (reading R5) of the two pairs: cos < 0.5 <=> 4 D^2 <
// |p|^2 |q|^2 <=> fl(D^2 - Ph/4) < Pl/4 (DESIGN.md 5.2's fl(4 D^2 - Ph) < Pl,
// scaled by the exact factor 1/4; the sign of fl(t - Pl/4) is that of t - Pl/4).
__device__ __forceinline__ void acos_branch_exact2(uint32_t pk0, uint32_t pk1, f32x2 nn2, f32x2 nnn2, uint4 q,
                                                   bool& a0, bool& a1) {
  const f32x2 Db = pack2(__uint_as_float(__dp4a(pk0, q.x, F2P23_BITS)), __uint_as_float(__dp4a(pk1, q.y, F2P23_BITS)));
  const f32x2 D = sub2(Db, pack2(F2P23, F2P23));
  const f32x2 nnq = pack2(__uint_as_float(q.z), __uint_as_float(q.w));
  const f32x2 nPh = mul2(nnn2, nnq);
  const f32x2 Pl = fma2(nn2, nnq, nPh);
  const f32x2 t = fma2(D, D, mul2(nPh, pack2(0.25f, 0.25f)));
  const f32x2 u = fma2(Pl, pack2(-0.25f, -0.25f), t);
  a0 = lo2(u) < 0.0f;
  a1 = hi2(u) < 0.0f;
}

// cos within this distance of 0.5 is decided exactly (cos = D rsqrt(Ph) is
// within ~4 ulp = 5e-7 of the true cosine).
constexpr float ACOS_AMBIG = 1.0f / 65536.0f;

#ifndef VF_STREAM_ACOS
#define VF_STREAM_ACOS 3   // ARCCOS-branch strategy (tuning knob), see ang_mm_row (3: C4 256 images 1.447 -> 1.437 ms)
#endif
#ifndef VF_STREAM_UNROLL
#define VF_STREAM_UNROLL 1   // row-loop unrolling (tuning knob)
#endif
#ifndef VF_STREAM_TINY
#define VF_STREAM_TINY 0   // X = 0 guard: 1 = X + 1e-30 (FADD2), 0 = max(tau, 0) (FMNMX, ALU pipe)
#endif

// Table 1 values (reading R5: ARCCOS row on cos for cos < 0.5, else ARCSIN row
// on tau) of the lane's two pairs for n neighbour record pairs q[i].
// VF_STREAM_ACOS 0: both rows for every pair, exact predicate inline, no
// votes; 1: per offset, the ARCCOS row (~1% of pairs) only when some lane of
// the warp may need it (one vote); 2: the same with the geometry of all n
// offsets computed first (independent chains, more registers); 3 (default,
// measured fastest in round 2: 1.437 vs 1.447 ms per 256 C4 images): both
// rows for every pair, the branch decided on cos.  With 1, 2 and 3, pairs
// within ACOS_AMBIG of cos = 0.5 set `amb`: the caller then re-decides the
// whole row exactly (ang_mm_row_exact), so the outputs are those of 0.
// ZG: zero vector -> 0.
template <bool ZG, int N, bool EXACT_V = false>
__device__ __forceinline__ void ang_mm_row(uint32_t pk0, uint32_t pk1, f32x2 nn2, f32x2 nnn2, const uint4 (&q)[N],
                                           f32x2 (&v)[N], bool& amb, const f32x2* rr = nullptr) {
  if constexpr (EXACT_V) {
    // exact variant (libm): the exact predicate for every pair; acosf (the ~1%
    // of pairs with cos < 0.5) only in lanes that need it, the ARCSIN side by
    // Eq. 6 with asinf.  Zero vectors need no fix-up: tau = 0 and cos < 0.5
    // is false, so the value is 2 asinf(0) = 0.
#pragma unroll
    for (int i = 0; i < N; ++i) {
      f32x2 vs, c, nPh;
      ang_geo2<false, true>(pk0, pk1, nn2, nnn2, q[i], vs, c, nPh);
      bool e0, e1;
      acos_branch_exact2(pk0, pk1, nn2, nnn2, q[i], e0, e1);
      float s0, s1;
      unpack2(vs, s0, s1);
      if (__any_sync(0xffffffffu, e0 || e1)) {
        if (e0) s0 = acosf(lo2(c));
        if (e1) s1 = acosf(hi2(c));
      }
      v[i] = pack2(s0, s1);
    }
    return;
  }
  auto finish = [&](int i, f32x2 c, f32x2 nPh) {
    float c0, c1;
    unpack2(c, c0, c1);
    amb |= fabsf(c0 - 0.5f) <= ACOS_AMBIG || fabsf(c1 - 0.5f) <= ACOS_AMBIG;
    if (__any_sync(0xffffffffu, fminf(c0, c1) < 0.5f - ACOS_AMBIG)) {
      float a0, a1, v0, v1;
      unpack2(horner4x2(coef::ACOS(), c), a0, a1);                       // Table 1 ARCCOS row
      unpack2(v[i], v0, v1);
      v[i] = pack2(c0 < 0.5f - ACOS_AMBIG ? a0 : v0, c1 < 0.5f - ACOS_AMBIG ? a1 : v1);
    }
    if (ZG) {
      float n0, n1, v0, v1;
      unpack2(nPh, n0, n1);
      unpack2(v[i], v0, v1);
      v[i] = pack2(n0 == 0.0f ? 0.0f : v0, n1 == 0.0f ? 0.0f : v1);
    }
  };
  if constexpr (VF_STREAM_ACOS == 2) {
    f32x2 c[N], nPh[N];
#pragma unroll
    for (int i = 0; i < N; ++i) ang_geo2(pk0, pk1, nn2, nnn2, q[i], v[i], c[i], nPh[i]);
#pragma unroll
    for (int i = 0; i < N; ++i) finish(i, c[i], nPh[i]);
  } else if constexpr (VF_STREAM_ACOS == 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      f32x2 c, nPh;
      ang_geo2(pk0, pk1, nn2, nnn2, q[i], v[i], c, nPh);
      finish(i, c, nPh);
    }
  } else if constexpr (VF_STREAM_ACOS == 3) {
    // both rows for every pair (no votes), the branch decided on cos with the
    // row-level exact fallback for |cos - 0.5| <= ACOS_AMBIG (FSETPs on the ALU
    // pipe instead of the FMA-pipe exact predicate)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      f32x2 vs, c, nPh;
      ang_geo2<false>(pk0, pk1, nn2, nnn2, q[i], vs, c, nPh);
      float c0, c1, a0, a1, s0, s1;
      unpack2(c, c0, c1);
      unpack2(horner4x2(coef::ACOS(), c), a0, a1);
      unpack2(vs, s0, s1);
      // |cos - 0.5| <= ACOS_AMBIG as one unsigned range test on the float bits
      // (cos >= 0 for these integer vectors, and NaN/garbage only in unused pairs)
      constexpr uint32_t LO = 0x3EFFFE00u;   // bits of 0.5 - 2^-16 = 0.4999847
      constexpr uint32_t SPAN = 0x3F000100u - LO;   // up to 0.5 + 2^-16 = 0.5000153
      amb |= (__float_as_uint(c0) - LO <= SPAN) | (__float_as_uint(c1) - LO <= SPAN);
      s0 = c0 < 0.5f ? a0 : s0;
      s1 = c1 < 0.5f ? a1 : s1;
      if (ZG) {
        float n0, n1;
        unpack2(nPh, n0, n1);
        s0 = n0 == 0.0f ? 0.0f : s0;
        s1 = n1 == 0.0f ? 0.0f : s1;
      }
      v[i] = pack2(s0, s1);
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      f32x2 vs, c, nPh;
      ang_geo2<VF_STREAM_TINY>(pk0, pk1, nn2, nnn2, q[i], vs, c, nPh, rr ? &rr[i] : nullptr);
      bool e0, e1;
      acos_branch_exact2(pk0, pk1, nn2, nnn2, q[i], e0, e1);
      float a0, a1, s0, s1;
      unpack2(horner4x2(coef::ACOS(), c), a0, a1);
      unpack2(vs, s0, s1);
      s0 = e0 ? a0 : s0;
      s1 = e1 ? a1 : s1;
      if (ZG) {
        float n0, n1;
        unpack2(nPh, n0, n1);
        s0 = n0 == 0.0f ? 0.0f : s0;
        s1 = n1 == 0.0f ? 0.0f : s1;
      }
      v[i] = pack2(s0, s1);
    }
  }
}

// The same values with the exact integer branch predicate for every pair
// (rare: only rows holding a pair with cos within ACOS_AMBIG of 0.5).
template <int N>
__device__ __forceinline__ void ang_mm_row_exact(uint32_t pk0, uint32_t pk1, f32x2 nn2, f32x2 nnn2,
                                                 const uint4 (&q)[N], f32x2 (&v)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    f32x2 vs, c, nPh;
    ang_geo2(pk0, pk1, nn2, nnn2, q[i], vs, c, nPh);
    bool e0, e1;
    acos_branch_exact2(pk0, pk1, nn2, nnn2, q[i], e0, e1);
    float a0, a1, s0, s1, n0, n1;
    unpack2(horner4x2(coef::ACOS(), c), a0, a1);
    unpack2(vs, s0, s1);
    unpack2(nPh, n0, n1);
    s0 = e0 ? a0 : s0;
    s1 = e1 ? a1 : s1;
    v[i] = pack2(n0 == 0.0f ? 0.0f : s0, n1 == 0.0f ? 0.0f : s1);
  }
}

// Both variants of the lane's two pairs for n neighbour record pairs from ONE
// geometry evaluation (plan-level fusion of BVDF exact and minimax): vm =
// Table 1 values (minimax, zero vectors -> 0), ve = libm values (Eq. 6).
template <int N>
__device__ __forceinline__ void ang_both_row(uint32_t pk0, uint32_t pk1, f32x2 nn2, f32x2 nnn2, const uint4 (&q)[N],
                                             f32x2 (&vm)[N], f32x2 (&ve)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    f32x2 vs, c, nPh, tau;
    ang_geo2<false, false>(pk0, pk1, nn2, nnn2, q[i], vs, c, nPh, nullptr, &tau);
    bool e0, e1;
    acos_branch_exact2(pk0, pk1, nn2, nnn2, q[i], e0, e1);
    float a0, a1, s0, s1, n0, n1, c0, c1, t0, t1;
    unpack2(horner4x2(coef::ACOS(), c), a0, a1);
    unpack2(vs, s0, s1);
    unpack2(nPh, n0, n1);
    unpack2(c, c0, c1);
    unpack2(tau, t0, t1);
    s0 = e0 ? a0 : s0;
    s1 = e1 ? a1 : s1;
    vm[i] = pack2(n0 == 0.0f ? 0.0f : s0, n1 == 0.0f ? 0.0f : s1);
    float x0 = 2.0f * asinf(t0 * 0.70710678118654752f), x1 = 2.0f * asinf(t1 * 0.70710678118654752f);
    if (__any_sync(0xffffffffu, e0 || e1)) {
      if (e0) x0 = acosf(c0);
      if (e1) x1 = acosf(c1);
    }
    ve[i] = pack2(x0, x1);
  }
}

// H sums of one neighbourhood row (values a(dx), dx = -2..2; a(0) = 0 for the
// pixel's own row): H_b = sum_{dx in [-b, 2-b]} a(dx), b = 0, 1, 2.  Packed
// over the lane's two pixels where both rows are register pairs.
__device__ __forceinline__ void hrow2(f32x2 am2, f32x2 am1, f32x2 a0, f32x2 ap1, f32x2 ap2, f32x2 (&H)[3]) {
  const f32x2 m = add2(a0, ap1);
  const f32x2 n = add2(am1, a0);
  H[0] = add2(m, ap2);
  H[1] = add2(m, am1);
  H[2] = add2(n, am2);
}
__device__ __forceinline__ void hrow(float am2, float am1, float a0, float ap1, float ap2, float (&H)[3]) {
  const float m = a0 + ap1;
  const float n = am1 + a0;
  H[0] = m + ap2;
  H[1] = m + am1;
  H[2] = n + am2;
}
__device__ __forceinline__ void hrow0(float am2, float am1, float ap1, float ap2, float (&H)[3]) {
  H[0] = ap1 + ap2;
  H[1] = am1 + ap1;
  H[2] = am2 + am1;
}

// nn = |x|^2 (exact integer < 2^18) as float, from the packed pixel.
__device__ __forceinline__ float nn_of(uint32_t pk) {
  return __uint_as_float(__dp4a(pk, pk, F2P23_BITS)) - F2P23;
}

// The lane's two pixels of a row: columns c0, c1 (clamped, replicate padding)
// are x_lo or x_lo + 1 with x_lo = clamp(x, 0, W - 2), loaded as three aligned
// words (the third only if it starts inside the input allocation).
struct PairLoad {
  int x_lo;          // first column of the loaded pair
  bool hi0, hi1;     // pixel k = column x_lo + 1
};

// Raw words of the lane's pair in a row (issued one step ahead: software
// prefetch of the next row, so the load latency hides behind a step's work).
struct PairWords {
  uint32_t w0, w1, w2;
  int sh;
};
__device__ __forceinline__ PairWords ld_pair_words(const uint8_t* row, const PairLoad& pl, const uint8_t* in_end) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(row) + 3 * pl.x_lo;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
  PairWords r;
  r.w0 = __ldg(w);
  r.w1 = __ldg(w + 1);
  // (an aligned word holding a byte of the allocation never leaves it)
  r.w2 = reinterpret_cast<const uint8_t*>(w + 2) < in_end ? __ldg(w + 2) : 0u;
  r.sh = (int)(a & 3) * 8;
  return r;
}
__device__ __forceinline__ void unpack_pair(const PairWords& r, const PairLoad& pl, uint32_t& p0, uint32_t& p1) {
  const uint32_t lo = __funnelshift_r(r.w0, r.w1, r.sh);        // bytes 3 x_lo .. + 3
  const uint32_t hi = __funnelshift_r(r.w1, r.w2, r.sh);        // bytes 3 x_lo + 4 .. + 7
  const uint32_t q0 = lo & 0x00ffffffu;
  const uint32_t q1 = __byte_perm(lo, hi, 0x0543) & 0x00ffffffu;
  p0 = pl.hi0 ? q1 : q0;
  p1 = pl.hi1 ? q1 : q0;
}

// SEG = 32: grid (S or S - 1, ceil(out_rows / (K NWARP)), B), block 32 NWARP;
// dynamic smem NWARP * sizeof(Ring).  Warp w of block (sx, sy) streams strip
// sx of image z over output rows [out_row0 + (sy NWARP + w) K, + K).
// SEG = 16 (half_tail(W)): grid (1, *, ceil(B / 2)); half-warp h of warp w
// streams the LAST strip of image 2 z + h (a ghost copy of image B - 1 that
// stores nothing when 2 z + h = B).  nimg = B.  Requires W >= 2.
#ifndef VF_STREAM_MINB
#define VF_STREAM_MINB (20 / VF_STREAM_NWARP)   // resident blocks per SM: 20 warps per SM, <= 102 registers
#endif
// NV = 2 (VAR = MINIMAX): both variants from one geometry evaluation per pair
// (plan-level fusion of BVDF minimax and exact): L writes the minimax output,
// L2 the exact one; NV = 1: the variant VAR into L (L2 unused).
#ifndef VF_STREAM_MINB2
#define VF_STREAM_MINB2 16   // the fused (NV = 2) kernel: 16 warps per SM, <= 128 registers (3.60 -> 3.51 ms per 256 images; 12: 3.82, 20: 3.60, 24: 3.80)
#endif
template <int SEG>
__device__ __forceinline__ float shup(float v, int d) { return __shfl_up_sync(0xffffffffu, v, d, SEG); }
template <int SEG>
__device__ __forceinline__ float shdn(float v, int d) { return __shfl_down_sync(0xffffffffu, v, d, SEG); }
template <int SEG>
__device__ __forceinline__ uint32_t shdn(uint32_t v, int d) { return __shfl_down_sync(0xffffffffu, v, d, SEG); }

template <int VAR, int NV = 1, int SEG = 32>
__global__ void __launch_bounds__(32 * stream::NWARP, NV == 2 ? VF_STREAM_MINB2 : VF_STREAM_MINB)
    vf_angular_stream_kernel(const Launch L, int K, const Launch L2, int nimg) {
  using namespace stream;
  static_assert(VAR == MINIMAX || VAR == EXACT, "streamed kernel: angular minimax or exact");
  static_assert(NV == 1 || (NV == 2 && VAR == MINIMAX), "fused: minimax + exact");
  static_assert(SEG == 32 || SEG == 16, "full or half-warp strips");
  constexpr int SOUTS = 2 * SEG - 2;                            // output columns of the strip
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, l = threadIdx.x & (SEG - 1), seg = (threadIdx.x & 31) / SEG;
  RingT<SEG>& R = reinterpret_cast<RingT<SEG>*>(smem_raw)[warp * (32 / SEG) + seg];
  int b = SEG == 32 ? (int)blockIdx.z : 2 * (int)blockIdx.z + seg;
  const bool ghost = b >= nimg;                                 // half-warp past the last image
  if (ghost) b = nimg - 1;
  const int x0 = SEG == 32 ? strip_x0(blockIdx.x) : strip_x0(strips_of(L.W) - 1);
  const int ty0 = L.out_row0 + (blockIdx.y * NWARP + warp) * K;
  const int ty1 = min(ty0 + K, L.out_row0 + L.out_rows);
  if (ty0 >= ty1) return;                                       // warp-uniform
  const int W = L.W;
  const uint8_t* __restrict__ in = L.in + (long long)b * L.in_stride;
  const uint8_t* in_end = L.in + (long long)(nimg - 1) * L.in_stride + (long long)L.band_rows * W * 3;
  const int xa = x0 + 2 * l;                                    // image column of the lane's first pixel
  PairLoad pl;
  pl.x_lo = clampi(xa, 0, W - 2);
  pl.hi0 = clampi(xa, 0, W - 1) != pl.x_lo;
  pl.hi1 = clampi(xa + 1, 0, W - 1) != pl.x_lo;
  // output columns: strip j = 2l + k, valid for j in [1, 2 SEG - 2] inside the image
  const bool ov0 = !ghost && 2 * l >= J_LO && 2 * l < J_LO + SOUTS && xa < W;
  const bool ov1 = !ghost && 2 * l + 1 >= J_LO && 2 * l + 1 < J_LO + SOUTS && xa + 1 < W;
  const int rowb = W * 3;

  // carried partial role sums (packed over the lane's two pixels):
  // U = H(-1) + H(0) and Z = H(0) of the previous row's pixels (-> role a = 1
  // and the partial W), Wp = H(0) + H(+1) of the row before (-> role a = 0)
  f32x2 U[NV][3], Z[NV][3], Wp[NV][3];
#pragma unroll
  for (int t = 0; t < NV; ++t)
#pragma unroll
    for (int i = 0; i < 3; ++i) U[t][i] = Z[t][i] = Wp[t][i] = 0ull;
  uint32_t zhist = 0;                                           // zero-vector flags of the last 3 staged rows

  auto row_ptr = [&](int r) {
    const int br = clampi(r, L.band_row0, L.band_row0 + L.band_rows - 1) - L.band_row0;
    VF_CHECK(br >= 0 && br < L.band_rows);
    return in + (long long)br * rowb;
  };
  PairWords nxt = ld_pair_words(row_ptr(ty0 - 1), pl, in_end);
  constexpr int kUnroll = VF_STREAM_UNROLL;
#pragma unroll (kUnroll)
  for (int r = ty0 - 1; r <= ty1; ++r) {
    const int slot = r & (SLOTS - 1);
    // ---- a1/a2: stage row r (loaded one step ahead), prefetch row r + 1 -------
    const PairWords cur = nxt;
    nxt = ld_pair_words(row_ptr(r + 1), pl, in_end);
    uint32_t pk0, pk1;
    unpack_pair(cur, pl, pk0, pk1);
    // |x|^2 of the two pixels created as one register pair (the packed pair
    // operands below then need no moves); exact integers < 2^18
    const f32x2 nnb = pack2(__uint_as_float(__dp4a(pk0, pk0, F2P23_BITS)), __uint_as_float(__dp4a(pk1, pk1, F2P23_BITS)));
    const f32x2 nn2 = sub2(nnb, pack2(F2P23, F2P23));
    const f32x2 nnn2 = sub2(pack2(F2P23, F2P23), nnb);
    const float nn0 = lo2(nn2), nn1 = hi2(nn2);
    const uint32_t pk2 = shdn<SEG>(pk0, 1);  // column 2l + 2 (last lane: unused)
    const float nn2n = shdn<SEG>(nn0, 1);
    R.E[slot][l + 1] = make_uint4(pk0, pk1, __float_as_uint(nn0), __float_as_uint(nn1));
    R.O[slot][l + 1] = make_uint4(pk1, pk2, __float_as_uint(nn1), __float_as_uint(nn2n));
    if (l == 0) R.O[slot][0] = make_uint4(0u, pk0, 0u, __float_as_uint(nn0));   // column 0 as an O-pair's second pixel
#if VF_STREAM_RN
    const float rn0 = rsqrt_approx(nn0), rn1 = rsqrt_approx(nn1);
    const f32x2 rn2 = pack2(rn0, rn1);
    const float rn2n = shdn<SEG>(rn0, 1);
    R.ER[slot][l + 1] = make_uint2(__float_as_uint(rn0), __float_as_uint(rn1));
    R.OR[slot][l + 1] = make_uint2(__float_as_uint(rn1), __float_as_uint(rn2n));
#endif
    *reinterpret_cast<uint2*>(&R.P[slot][2 * l + 2]) = make_uint2(pk0, pk1);
    zhist = ((zhist << 1) | (__any_sync(0xffffffffu, nn0 == 0.0f || nn1 == 0.0f) ? 1u : 0u)) & 7u;
    __syncwarp();

    const int s1 = (r - 1) & (SLOTS - 1), s2 = (r - 2) & (SLOTS - 1);
    auto nbr = [&](int sl, int dx) -> uint4 {
      // neighbour pair (columns 2l + dx, 2l + 1 + dx)
      return (dx & 1) ? R.O[sl][l + ((dx - 1) >> 1) + 1] : R.E[sl][l + (dx >> 1) + 1];
    };
    // ---- a4/a5 + a6, one neighbourhood row at a time ---------------------------
    // v[dxi]: the lane's pair values with offset (dy, dx = dxi - 2)
    auto eval_row = [&](int sl, auto& vv) {
      constexpr int N = sizeof(vv[0]) / sizeof(vv[0][0]);
      uint4 q[N];
#pragma unroll
      for (int dxi = 0; dxi < N; ++dxi) q[dxi] = nbr(sl, dxi - 2);
      if constexpr (NV == 2) {
        ang_both_row<N>(pk0, pk1, nn2, nnn2, q, vv[0], vv[1]);
      } else {
        auto& v = vv[0];
        bool amb = false;
#if VF_STREAM_RN
        f32x2 rr[N];
#pragma unroll
        for (int dxi = 0; dxi < N; ++dxi) {
          const int dx = dxi - 2;
          const uint2 t = (dx & 1) ? R.OR[sl][l + ((dx - 1) >> 1) + 1] : R.ER[sl][l + (dx >> 1) + 1];
          rr[dxi] = mul2(rn2, pack2(__uint_as_float(t.x), __uint_as_float(t.y)));
        }
        const f32x2* rrp = rr;
#else
        const f32x2* rrp = nullptr;
#endif
        if constexpr (VAR == EXACT) ang_mm_row<false, N, true>(pk0, pk1, nn2, nnn2, q, v, amb);
        else if (zhist == 0u) ang_mm_row<false, N>(pk0, pk1, nn2, nnn2, q, v, amb, rrp);
        else ang_mm_row<true, N>(pk0, pk1, nn2, nnn2, q, v, amb, rrp);
        if (VAR != EXACT && VF_STREAM_ACOS != 0 && __any_sync(0xffffffffu, amb)) {
          // rare: re-load the records (keeping q live across the row would cost registers)
          uint4 q2[N];
#pragma unroll
          for (int dxi = 0; dxi < N; ++dxi) q2[dxi] = nbr(sl, dxi - 2);
          ang_mm_row_exact<N>(pk0, pk1, nn2, nnn2, q2, v);
        }
      }
    };
    // rows r - d (d = 2, then 1): the partner pixels' H(+d) from values of row r
    // pixels with offset (-d, dx), partly from the adjacent lanes
    auto partner_rows = [&](const f32x2 (&v)[5], float (&H0)[3], float (&H1)[3]) {
      const float p_p2_0 = shup<SEG>(lo2(v[4]), 1);   // lane l-1: q0, offset (-d, +2)
      const float p_p1_1 = shup<SEG>(hi2(v[3]), 1);   // lane l-1: q1, offset (-d, +1)
      const float p_p2_1 = shup<SEG>(hi2(v[4]), 1);   // lane l-1: q1, offset (-d, +2)
      const float n_m2_0 = shdn<SEG>(lo2(v[0]), 1); // lane l+1: q0, offset (-d, -2)
      const float n_m1_0 = shdn<SEG>(lo2(v[1]), 1); // lane l+1: q0, offset (-d, -1)
      const float n_m2_1 = shdn<SEG>(hi2(v[0]), 1); // lane l+1: q1, offset (-d, -2)
      hrow(p_p2_0, p_p1_1, lo2(v[2]), hi2(v[1]), n_m2_0, H0);          // pixel (r - d, 2l)
      hrow(p_p2_1, lo2(v[3]), hi2(v[2]), n_m1_0, n_m2_1, H1);          // pixel (r - d, 2l + 1)
    };
    f32x2 Hm2[NV][3], Hm1[NV][3], H0[NV][3];
    f32x2 R0[NV][3], R1[NV][3], R2[NV][3];   // roles a = 0 (row r - 2), 1 (row r - 1), 2 (row r), b = 0..2
    {
      f32x2 v[NV][5];
      eval_row(s2, v);                                          // dy = -2
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        hrow2(v[t][0], v[t][1], v[t][2], v[t][3], v[t][4], Hm2[t]);
        float Ha[3], Hb[3];
        partner_rows(v[t], Ha, Hb);
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) R0[t][bb] = add2(Wp[t][bb], pack2(Ha[bb], Hb[bb]));
      }
    }
    {
      f32x2 v[NV][5];
      eval_row(s1, v);                                          // dy = -1
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        hrow2(v[t][0], v[t][1], v[t][2], v[t][3], v[t][4], Hm1[t]);
        float Ha[3], Hb[3];
        partner_rows(v[t], Ha, Hb);
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          const f32x2 Hp1 = pack2(Ha[bb], Hb[bb]);
          R1[t][bb] = add2(U[t][bb], Hp1);
          Wp[t][bb] = add2(Z[t][bb], Hp1);
        }
      }
    }
    {
      f32x2 v[NV][2];
      eval_row(slot, v);                                        // dy = 0, dx = -2, -1
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        // right values from (q1, lane l+1)
        const float n_m1_0 = shdn<SEG>(lo2(v[t][1]), 1);
        const float n_m2_0 = shdn<SEG>(lo2(v[t][0]), 1);
        const float n_m2_1 = shdn<SEG>(hi2(v[t][0]), 1);
        float Ha[3], Hb[3];
        hrow0(lo2(v[t][0]), lo2(v[t][1]), hi2(v[t][1]), n_m2_0, Ha);
        hrow0(hi2(v[t][0]), hi2(v[t][1]), n_m1_0, n_m2_1, Hb);
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          H0[t][bb] = pack2(Ha[bb], Hb[bb]);
          U[t][bb] = add2(Hm1[t][bb], H0[t][bb]);
          Z[t][bb] = H0[t][bb];
          R2[t][bb] = add2(U[t][bb], Hm2[t][bb]);
        }
      }
    }

    // ---- a7/a8: the window centred at row r - 1 --------------------------------
    const int gy = r - 1;
#pragma unroll
    for (int t = 0; t < NV; ++t) {
    const Launch& Lt = t == 0 ? L : L2;
    if (gy >= ty0) {
      // keys: window 2l uses (lane l-1: q1, b = 0), (q0, b = 1), (q1, b = 2);
      // window 2l + 1 uses (q0, b = 0), (q1, b = 1), (lane l+1: q0, b = 2)
      const float k00 = shup<SEG>(role_key<0>(hi2(R0[t][0])), 1);
      const float k10 = shup<SEG>(role_key<4>(hi2(R1[t][0])), 1);
      const float k20 = shup<SEG>(role_key<8>(hi2(R2[t][0])), 1);
      const float m02 = shdn<SEG>(role_key<2>(lo2(R0[t][2])), 1);
      const float m12 = shdn<SEG>(role_key<6>(lo2(R1[t][2])), 1);
      const float m22 = shdn<SEG>(role_key<10>(lo2(R2[t][2])), 1);
      const float kw0 = fmin3(fmin3(k00, role_key<1>(lo2(R0[t][1])), role_key<2>(hi2(R0[t][2]))),
                              fmin3(k10, role_key<5>(lo2(R1[t][1])), role_key<6>(hi2(R1[t][2]))),
                              fmin3(k20, role_key<9>(lo2(R2[t][1])), role_key<10>(hi2(R2[t][2]))));
      const float kw1 = fmin3(fmin3(role_key<0>(lo2(R0[t][0])), role_key<1>(hi2(R0[t][1])), m02),
                              fmin3(role_key<4>(lo2(R1[t][0])), role_key<5>(hi2(R1[t][1])), m12),
                              fmin3(role_key<8>(lo2(R2[t][0])), role_key<9>(hi2(R2[t][1])), m22));
      const uint32_t nib0 = __float_as_uint(kw0) & 15u, nib1 = __float_as_uint(kw1) & 15u;
      // selected samples: row r - 2 + a, strip column (2l + k) - 1 + b
      const uint32_t* prow0 = R.P[(r - 2) & (SLOTS - 1)];
      const uint32_t* prow1 = R.P[(r - 1) & (SLOTS - 1)];
      const uint32_t* prow2 = R.P[slot];
      auto pick = [&](uint32_t nib, int k) -> uint32_t {
        const uint32_t a = nib >> 2;
        const uint32_t* pr = a == 0 ? prow0 : (a == 1 ? prow1 : prow2);
        VF_CHECK(a <= 2 && (nib & 3u) <= 2);
        return pr[2 * l + k + 1 + (int)(nib & 3u)];
      };
      const uint32_t o0 = pick(nib0, 0), o1 = pick(nib1, 1);
      // a8: 6 bytes per lane, predicated stores (no divergence)
      VF_CHECK(!(ov0 || ov1) || (gy >= L.out_row0 && gy < L.out_row0 + L.out_rows && xa + (ov0 ? 0 : 1) >= 0 &&
                                  xa + (ov1 ? 1 : 0) < W));
      uint8_t* op = Lt.out + (long long)b * Lt.out_stride + ((long long)(gy - L.out_row0) * W + xa) * 3;
      if (((uintptr_t)op & 1u) == 0) {                          // warp-uniform: U16, U8 U8, U16
        if (ov0) *reinterpret_cast<uint16_t*>(op) = (uint16_t)o0;
        if (ov0) op[2] = (uint8_t)(o0 >> 16);
        if (ov1) op[3] = (uint8_t)o1;
        if (ov1) *reinterpret_cast<uint16_t*>(op + 4) = (uint16_t)(o1 >> 8);
      } else {                                                  // U8, U16, U16, U8
        if (ov0) op[0] = (uint8_t)o0;
        if (ov0) *reinterpret_cast<uint16_t*>(op + 1) = (uint16_t)(o0 >> 8);
        if (ov1) *reinterpret_cast<uint16_t*>(op + 3) = (uint16_t)o1;
        if (ov1) op[5] = (uint8_t)(o1 >> 16);
      }
      if (Lt.idx || Lt.agg) {
        // parity runs only: the index (raster 3a + b) and the exact aggregates
        const float f00 = shup<SEG>(hi2(R0[t][0]), 1), f10 = shup<SEG>(hi2(R1[t][0]), 1),
                    f20 = shup<SEG>(hi2(R2[t][0]), 1);
        const float g02 = shdn<SEG>(lo2(R0[t][2]), 1), g12 = shdn<SEG>(lo2(R1[t][2]), 1),
                    g22 = shdn<SEG>(lo2(R2[t][2]), 1);
        const long long npix_img = (long long)L.out_rows * W;
        const long long po = (long long)(gy - L.out_row0) * W + xa;
        if (ov0) {
          if (Lt.idx) Lt.idx[b * npix_img + po] = (uint8_t)(3 * (nib0 >> 2) + (nib0 & 3u));
          if (Lt.agg) {
            float* ag = Lt.agg + (b * npix_img + po) * 9;
            ag[0] = f00; ag[1] = lo2(R0[t][1]); ag[2] = hi2(R0[t][2]);
            ag[3] = f10; ag[4] = lo2(R1[t][1]); ag[5] = hi2(R1[t][2]);
            ag[6] = f20; ag[7] = lo2(R2[t][1]); ag[8] = hi2(R2[t][2]);
          }
        }
        if (ov1) {
          if (Lt.idx) Lt.idx[b * npix_img + po + 1] = (uint8_t)(3 * (nib1 >> 2) + (nib1 & 3u));
          if (Lt.agg) {
            float* ag = Lt.agg + (b * npix_img + po + 1) * 9;
            ag[0] = lo2(R0[t][0]); ag[1] = hi2(R0[t][1]); ag[2] = g02;
            ag[3] = lo2(R1[t][0]); ag[4] = hi2(R1[t][1]); ag[5] = g12;
            ag[6] = lo2(R2[t][0]); ag[7] = hi2(R2[t][1]); ag[8] = g22;
          }
        }
      }
    }
    }
    __syncwarp();   // ring slot (r + 1) & 3 = (r - 3) & 3 is no longer read
  }
}

#ifndef VF_ANGULAR_MM_TU
// defined in vf_stream.cu, whose compile flags (tuning knobs) fix the ring layout
// half = true: the SEG = 16 remainder-strip kernel
const void* stream_kernel_fn_mm(bool half = false);
const void* stream_kernel_fn_ex(bool half = false);
const void* stream_kernel_fn_both(bool half = false);
size_t stream_smem_bytes(bool half = false);
#endif

// rows per warp: long tiles (less vertical halo: K + 2 steps for K rows) when
// the launch has enough strips to fill the GPU, shorter ones for small images
inline int stream_rows_per_warp(long long strips_total_times_rows) {
  const long long target_warps = 148LL * 32 * 2;   // two waves of 32 warps per SM
  int K = 64;
  while (K > 8 && strips_total_times_rows / K < target_warps) K >>= 1;
  return K;
}

#ifdef VF_ANGULAR_MM_TU
// launch geometry, defined with the kernel (vf_stream.cu) so the tuning knobs
// of that translation unit fix it
// tail = false: the full strips (all of them, or all but the last when
// split_tail); tail = true: the half-warp launch of the last strips
inline dim3 stream_grid_impl(const Launch& L, int B, int K, bool split_tail, bool tail) {
  using namespace stream;
  const unsigned gy = (L.out_rows + K * NWARP - 1) / (K * NWARP);
  if (tail) return dim3(1, gy, (B + 1) / 2);
  return dim3(strips_of(L.W) - (split_tail ? 1 : 0), gy, B);
}
#else
dim3 stream_grid(const Launch& L, int B, int K, bool split_tail = false, bool tail = false);
int stream_block_threads();
#endif

}  // namespace vf
