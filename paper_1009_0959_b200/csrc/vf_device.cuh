// vf_device.cuh -- per-pair criteria and shared device helpers (sm_100a, SIMT FP32).
//
// Pair geometry is exact: RGB components are integers <= 255, so dot products
// (< 2^18), squared norms (< 2^18) and L1 distances (<= 765) are exact in
// fp32; the only inexact product, P = |x_i|^2 |x_j|^2 (< 2^36), is carried as
// an exact two-term sum Ph + Pl (FMUL + FFMA residual).  From it:
//   X = P - D^2 = |x_i x x_j|^2 (Lagrange identity) = fl(fl(Ph - D^2) + Pl):
//       exact whenever X < 2^24, relative error <= 2^-23 otherwise, and exactly
//       0 for parallel pairs;
//   the branch "cos < 0.5" of Eqs. 6-7 is 4 D^2 < P, decided
//       exactly as fl(4D^2 - Ph) < Pl (DESIGN.md section 5.2 has the proof).
// 1 - cos = X / (s (s + D)) with s = |x_i||x_j| needs no subtraction, so
// tau = sqrt(1 - cos) keeps full relative precision for near-parallel pairs.
#pragma once
#include <cstdint>
#include <type_traits>
#include <utility>

#include "vf_coeffs.cuh"

// VF_CHECK: device-side bounds checks compiled in only for the debug build
// (libvf_debug.so, `python -m paper_1009_0959_b200.build --debug`), which the
// parity tests can load with VF_LIB=... to catch out-of-range smem / global
// accesses (compute-sanitizer is not available on the GPU pool).
#ifdef VF_DEBUG
#include <cstdio>
#define VF_CHECK(cond)                                                                         \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("VF_CHECK failed: %s at %s:%d block (%d,%d,%d) thread (%d,%d)\n", #cond, __FILE__, \
             __LINE__, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x, threadIdx.y);         \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define VF_CHECK(cond) ((void)0)
#endif

namespace vf {

enum { ANGULAR = 0, EXPC = 1, LOGC = 2 };
enum { EXACT = 0, MINIMAX = 1, POLY4 = 2, REACH = 3 };

// ---- single-instruction PTX helpers ------------------------------------------
// MUFU.RCP / MUFU.RSQ without the denormal fix-up sequences that rcpf/rsqrtf
// and __fdividef add (arguments here are normal numbers or exactly handled).
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// Sum of the 4 byte-wise |a - b| plus c (one VABSDIFF4.U8.ACC).  With packed
// RGB0 pixels this is the L1 distance |x_i - x_j|_1 (an integer <= 765).
__device__ __forceinline__ uint32_t sad4(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// The float 2^23 + d1 as a bit pattern: sad4 accumulating into 0x4B000000
// (= 8388608.0f) adds the integer d1 < 2^23 to the mantissa.  Then
// fma(c, 2^23 + d1, -c * 2^23) = fl(c * d1) exactly (one rounding).
constexpr uint32_t F2P23_BITS = 0x4B000000u;
constexpr float F2P23 = 8388608.0f;

__device__ __forceinline__ uint32_t pack_rgb(uint32_t r, uint32_t g, uint32_t b) { return r | (g << 8) | (b << 16); }

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Pair p of the raster enumeration (0,1), (0,2), ..., (0,N-1), (1,2), ... of
// the i < j pairs of N samples.
template <int N>
__host__ __device__ constexpr int pair_i(int p) {
  int i = 0;
  while (p >= N - 1 - i) { p -= N - 1 - i; ++i; }
  return i;
}
template <int N>
__host__ __device__ constexpr int pair_j(int p) {
  int i = 0;
  while (p >= N - 1 - i) { p -= N - 1 - i; ++i; }
  return i + 1 + p;
}
template <int N>
__host__ __device__ constexpr int pair_index(int i, int j) { return i * N - i * (i + 1) / 2 + (j - i - 1); }

// Compile-time loop: f(std::integral_constant<int, k>) for k = 0..K-1, in
// order.  Used for the pair loops so that every register index is static in
// every kernel instantiation (the unroller's heuristics gave up on some of
// them inside the persistent TMA kernel, demoting aggregates to local memory).
template <typename F, int... Ks>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Ks...>) {
  (f(std::integral_constant<int, Ks>{}), ...);
}
template <int K, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, K>{});
}

__device__ __forceinline__ float horner4(const coef::P4f p, float x) {
  return fmaf(fmaf(fmaf(fmaf(p.a4, x, p.a3), x, p.a2), x, p.a1), x, p.a0);
}
// Horner over a coefficient table T (T::DEG, constexpr T::c(k) in double),
// each coefficient rounded to fp32 at compile time.
template <typename T, int K>
__device__ __forceinline__ float horner_rec(float x) {
  constexpr float a = (float)T::c(K);
  if constexpr (K == T::DEG) return a;
  else return fmaf(horner_rec<T, K + 1>(x), x, a);
}
template <typename T>
__device__ __forceinline__ float horner_tab(float x) { return horner_rec<T, 0>(x); }

// ---- angular criterion A(x_i, x_j) of Eq. 5 --------------------------
// Geometry shared by both variants: D, P = Ph + Pl, X, the exact branch
// predicate and tau = sqrt(1 - cos) = X / sqrt(X * s (s + D)).
struct AngGeo {
  float D, Ph, Pl, X, tau;
  bool acos_branch;   // cos < 0.5 (exact)
};

__device__ __forceinline__ AngGeo angular_geo(float ri, float gi, float bi, float nni, float nrmi,
                                              float rj, float gj, float bj, float nnj, float nrmj) {
  AngGeo g;
  g.D = fmaf(ri, rj, fmaf(gi, gj, __fmul_rn(bi, bj)));    // exact
  g.Ph = __fmul_rn(nni, nnj);
  g.Pl = fmaf(nni, nnj, -g.Ph);                           // exact residual
  g.X = __fadd_rn(fmaf(-g.D, g.D, g.Ph), g.Pl);           // |x_i x x_j|^2
  const float t = fmaf(__fmul_rn(4.0f, g.D), g.D, -g.Ph); // fl(4D^2 - Ph)
  g.acos_branch = t < g.Pl;                               // 4D^2 < P, exact
  const float s = __fmul_rn(nrmi, nrmj);
  const float w = fmaf(s, g.D, g.Ph);                     // s (s + D) (> 0 unless a zero vector)
  g.tau = __fmul_rn(g.X, rsqrt_approx(fmaf(g.X, w, 1e-30f)));   // X=0 -> exactly 0
  return g;
}

// (r,g,b) components, nn = squared norm, nrm = norm, rn = 1/norm (0 for a
// zero vector).  Zero vectors fall into the tau branch with X = 0 -> tau = 0;
// the exact variant then returns 0 and the minimax variant the
// ARCSIN row's a0, which the caller removes (zero-vector fix-up).
template <int VAR>
__device__ __forceinline__ float angular_pair(float ri, float gi, float bi, float nni, float nrmi, float rni,
                                              float rj, float gj, float bj, float nnj, float nrmj, float rnj) {
  const AngGeo g = angular_geo(ri, gi, bi, nni, nrmi, rj, gj, bj, nnj, nrmj);
  const float c = __fmul_rn(__fmul_rn(g.D, rni), rnj);   // cos
  if (VAR == EXACT) {
    // Eq. 6: arccos z = 2 arcsin(sqrt(0.5 (1 - z))) for z >= 0.5
    return g.acos_branch ? acosf(c) : 2.0f * asinf(g.tau * 0.70710678118654752f);
  } else {
    // Table 1: ARCCOS row on cos (cos < 0.5), ARCSIN row on tau (Eq. 7)
    const float x = g.acos_branch ? c : g.tau;
    const bool a = g.acos_branch;
    const coef::P4f p = {a ? coef::ACOS().a0 : coef::ASIN().a0, a ? coef::ACOS().a1 : coef::ASIN().a1,
                         a ? coef::ACOS().a2 : coef::ASIN().a2, a ? coef::ACOS().a3 : coef::ASIN().a3,
                         a ? coef::ACOS().a4 : coef::ASIN().a4};
    return horner4(p, x);
  }
}

// Exact variants (cancellation-free fp32
// forms): D_E = -expm1f(-z) and D_L = -(1 - u) log1pf(-u).  VF_EXACT_LIBM=1
// evaluates the paper's functions as written instead -- 1 - expf(-z) and
// -s logf(s) -- measured 1.9x / 1.2x faster kernels (C4 exp exact 16.9 ->
// 8.9 ms, log exact 16.3 -> 13.9 ms with the argument ranges below; step
// 64.0 -> 52.5 ms) with aggregates 3x further from the oracle (max 3.2e-6 vs
// 1.1e-6 relative; worst-case bound 9.3e-6 < the 1e-5 parity tolerance,
// DESIGN.md 5.2): not the default, because the survey pins the
// cancellation-free forms (reading R26).
#ifndef VF_EXACT_LIBM
#define VF_EXACT_LIBM 0
#endif
// VF_LIBM_ASSUME: the compiler is told each libm argument's range, proved in
// DESIGN.md 2 (z <= z*_n < 0.75, u in [0, 1 - 1/e], s = 1 - u in [1/e, 1]):
// the calls and their results are unchanged.  It pays for logf (the
// VF_EXACT_LIBM=1 build: its special-case paths -- subnormal scaling, zero /
// negative / inf / NaN -- drop out, 15% fewer instructions in the log kernel,
// C4 256 images 4.09 -> 3.47 ms); expm1f, log1pf and expf compile to the same
// code.  The debug build checks the ranges instead (VF_CHECK).
#ifndef VF_LIBM_ASSUME
#define VF_LIBM_ASSUME 1
#endif
#if defined(VF_DEBUG)
#define VF_ASSUME_RANGE(c) VF_CHECK(c)
#elif VF_LIBM_ASSUME
#define VF_ASSUME_RANGE(c) __builtin_assume(c)
#else
#define VF_ASSUME_RANGE(c) ((void)0)
#endif
// ---- exp criterion D_E = 1 - E(z) (reading R2) --------------------------------
// z = c_E * d1 never exceeds z*_n < 1, so the P:163 cutoff is dead code.
// ---- log criterion D_L = -ENT(s), s = 1 - u (reading R3) -----------------------
// u = c_L * d1 in [0, 1 - 1/e]; s >= 1/e > 0.05, so the P:232 cutoff is dead code.
//
// crit_accumulate adds the pair's criterion value to both aggregates (a6).
// Every rounding is spelled out (fmaf / __fadd_rn, which the compiler never
// contracts), so all kernel instantiations (tile shapes, stripes, batches)
// produce bit-identical aggregates for the same window.
// VF_EXACT_CALL_MINWIN: windows of at least this width reach the exact
// variants' libm routine through one out-of-line copy per kernel (CALL) instead
// of inlining it per pair.  The 5x5 exact kernels unroll 300 pairs: inlined,
// that is ~10 K instructions (160 KB) of straight-line code and ncu shows
// 37-42% of the stall samples on no_instructions (instruction-cache misses,
// profiles/r02_ncu_full_c3.md).  Same routine, same argument, same rounding:
// the results are bit-identical.
#ifndef VF_EXACT_CALL_MINWIN
#define VF_EXACT_CALL_MINWIN 99
#endif
// VF_EXACT_ROLL_MINWIN: windows of at least this width evaluate the exact
// variants' pairs in a rolled loop over the cyclic pair offsets (vf_window.cuh,
// el_window_s1): the libm routine stays inlined, in N copies instead of
// N (N - 1) / 2.  The aggregates' summation order differs from the unrolled form.
// Default: the 5x5 kernels, where the unrolled form is ~10 K instructions and
// ncu shows 37-42% of the stall samples on no_instructions
// (profiles/r02_ncu_full_c3.md); measured on C3: exp exact 11.80 -> 11.15 ms,
// log exact 11.55 -> 10.37 ms (123-128 registers instead of 71-76).  The 3x3
// kernels (36 pairs) keep the unrolled form.
#ifndef VF_EXACT_ROLL_MINWIN
#define VF_EXACT_ROLL_MINWIN 5
#endif
#if !VF_EXACT_LIBM
static __device__ __noinline__ float vf_expm1f_call(float x) {   // x = -z
  VF_ASSUME_RANGE(x <= 0.0f && x >= -0.75f);
  return expm1f(x);
}
static __device__ __noinline__ float vf_log1pf_call(float x) {   // x = -u
  VF_ASSUME_RANGE(x <= 0.0f && x >= -0.64f);
  return log1pf(x);
}
#endif

template <int CRIT, int VAR, bool CALL = false>
__device__ __forceinline__ void crit_accumulate(float zu, float& Ri, float& Rj) {
  if (VAR == MINIMAX) {
    // exp: Delta(z) / Q(z) = 1 - N/Q;  log: -Ntilde(u) / Qtilde(u) = -ENT(1 - u)
    const float num = CRIT == EXPC ? horner4(coef::EXP_DELTA(), zu) : horner4(coef::ENT_NEGN_U(), zu);
    const float r = rcp_approx(CRIT == EXPC ? horner4(coef::EXP_Q(), zu) : horner4(coef::ENT_Q_U(), zu));
    Ri = fmaf(num, r, Ri);
    Rj = fmaf(num, r, Rj);
  } else if (VAR == REACH) {   // the criterion value as one polynomial, no division
    const float v = CRIT == EXPC ? horner_tab<coef::R_EXP>(zu) : horner_tab<coef::R_LOG>(zu);
    Ri = __fadd_rn(Ri, v);
    Rj = __fadd_rn(Rj, v);
  } else if (VAR == POLY4) {   // exp only: 1 - P4(z)
    const float v = horner4(coef::EXP_1MP4(), zu);
    Ri = __fadd_rn(Ri, v);
    Rj = __fadd_rn(Rj, v);
  } else if (CRIT == EXPC) {   // exact: 1 - exp(-z)
    VF_ASSUME_RANGE(zu >= 0.0f && zu <= 0.75f);      // z <= z*_n < 0.75 (reading R2)
#if VF_EXACT_LIBM
    const float v = __fadd_rn(1.0f, -expf(-zu));
#else
    const float v = CALL ? -vf_expm1f_call(-zu) : -expm1f(-zu);
#endif
    Ri = __fadd_rn(Ri, v);
    Rj = __fadd_rn(Rj, v);
  } else {                     // exact: -s ln s, s = 1 - u
    const float ms = __fadd_rn(zu, -1.0f);   // -(1 - u), one rounding
#if VF_EXACT_LIBM
    VF_ASSUME_RANGE(ms <= -0.36f && ms >= -1.0f);    // s = 1 - u in [1/e, 1] (reading R3)
    const float l = logf(-ms);
#else
    VF_ASSUME_RANGE(zu >= 0.0f && zu <= 0.64f);      // u in [0, 1 - 1/e] (reading R3)
    const float l = CALL ? vf_log1pf_call(-zu) : log1pf(-zu);
#endif
    Ri = fmaf(ms, l, Ri);
    Rj = fmaf(ms, l, Rj);
  }
}

// ---- packed FP32 pairs (sm_100: FFMA2 / FADD2 / FMUL2) ---------------------------
// fma.rn.f32x2 computes two independent fp32 FMAs, each rounded exactly like
// fmaf, in one instruction: same FMA-pipe throughput per element as FFMA
// (tools/fp32_peak.cu: 17-18 T FFMA2/s = 34-36 T FMA/s) at half the issue
// slots.  Two pairs of a window are evaluated together so that the Horner
// chains and the argument scaling issue once for both; results are
// bit-identical to the scalar path.
using f32x2 = unsigned long long;
__device__ __forceinline__ f32x2 pack2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(f32x2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 horner4x2(const coef::P4f p, f32x2 x) {
  f32x2 r = fma2(pack2(p.a4, p.a4), x, pack2(p.a3, p.a3));
  r = fma2(r, x, pack2(p.a2, p.a2));
  r = fma2(r, x, pack2(p.a1, p.a1));
  return fma2(r, x, pack2(p.a0, p.a0));
}
template <typename T, int K>
__device__ __forceinline__ f32x2 horner_rec2(f32x2 x) {
  constexpr float a = (float)T::c(K);
  if constexpr (K == T::DEG) return pack2(a, a);
  else return fma2(horner_rec2<T, K + 1>(x), x, pack2(a, a));
}

// Two angular pair evaluations on the tau branch (Eqs. 6-7) in packed FP32:
// pixel p (packed RGB pk, nn2 = (|p|^2, |p|^2), nnn2 = -nn2, nrm2 = (|p|, |p|))
// against the neighbour records q0, q1 (packed RGB, |q|^2 bits, |q| bits).
// Every element is computed with exactly the roundings of the scalar path
// (angular_geo / vf_shared.cuh phase A): D exact; -Pl = fl(Ph - nn nnq) is the
// negated exact residual, so X = fl(fl(Ph - D^2) + Pl); tau = X rsqrt(X w).
template <int VAR>
__device__ __forceinline__ void angular_tau2(uint32_t pk, f32x2 nn2, f32x2 nnn2, f32x2 nrm2, uint4 q0, uint4 q1,
                                             float& tau0, float& tau1, float& v0, float& v1) {
  const f32x2 C = pack2(F2P23, F2P23);
  const f32x2 Db = pack2(__uint_as_float(__dp4a(pk, q0.x, F2P23_BITS)), __uint_as_float(__dp4a(pk, q1.x, F2P23_BITS)));
  const f32x2 D = sub2(Db, C);                            // exact dot products
  const f32x2 nD = sub2(C, Db);                           // -D, exact
  const f32x2 nnq = pack2(__uint_as_float(q0.y), __uint_as_float(q1.y));
  const f32x2 Ph = mul2(nn2, nnq);
  const f32x2 nPl = fma2(nnn2, nnq, Ph);                  // -(exact residual of nn nnq)
  const f32x2 X = sub2(fma2(nD, D, Ph), nPl);             // |p x q|^2
  const f32x2 w = fma2(mul2(nrm2, pack2(__uint_as_float(q0.z), __uint_as_float(q1.z))), D, Ph);   // s (s + D)
  float xw0, xw1;
  unpack2(fma2(X, w, pack2(1e-30f, 1e-30f)), xw0, xw1);
  const f32x2 t = mul2(X, pack2(rsqrt_approx(xw0), rsqrt_approx(xw1)));   // sqrt(1 - cos)
  unpack2(t, tau0, tau1);
  if (VAR == EXACT) {
    v0 = 2.0f * asinf(tau0 * 0.70710678118654752f);
    v1 = 2.0f * asinf(tau1 * 0.70710678118654752f);
  } else {
    unpack2(horner4x2(coef::ASIN(), t), v0, v1);
  }
}

// As angular_tau2 for 8-byte neighbour records (packed RGB, |q|^2 bits):
// s = |x_p||x_q| = sqrt(Ph) by MUFU.SQRT instead of the product of stored
// norms (relative error ~2^-23 either way; tau keeps ~5e-7 relative).
template <int VAR>
__device__ __forceinline__ void angular_tau2_r8(uint32_t pk, f32x2 nn2, f32x2 nnn2, uint2 q0, uint2 q1,
                                                float& tau0, float& tau1, float& v0, float& v1) {
  const f32x2 C = pack2(F2P23, F2P23);
  const f32x2 Db = pack2(__uint_as_float(__dp4a(pk, q0.x, F2P23_BITS)), __uint_as_float(__dp4a(pk, q1.x, F2P23_BITS)));
  const f32x2 D = sub2(Db, C);                            // exact dot products
  const f32x2 nD = sub2(C, Db);                           // -D, exact
  const f32x2 nnq = pack2(__uint_as_float(q0.y), __uint_as_float(q1.y));
  const f32x2 Ph = mul2(nn2, nnq);
  const f32x2 nPl = fma2(nnn2, nnq, Ph);                  // -(exact residual of nn nnq)
  const f32x2 X = sub2(fma2(nD, D, Ph), nPl);             // |p x q|^2
  float ph0, ph1, s0, s1;
  unpack2(Ph, ph0, ph1);
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s0) : "f"(ph0));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s1) : "f"(ph1));
  const f32x2 w = fma2(pack2(s0, s1), D, Ph);             // s (s + D)
  float xw0, xw1;
  unpack2(fma2(X, w, pack2(1e-30f, 1e-30f)), xw0, xw1);
  const f32x2 t = mul2(X, pack2(rsqrt_approx(xw0), rsqrt_approx(xw1)));   // sqrt(1 - cos)
  unpack2(t, tau0, tau1);
  if (VAR == EXACT) {
    v0 = 2.0f * asinf(tau0 * 0.70710678118654752f);
    v1 = 2.0f * asinf(tau1 * 0.70710678118654752f);
  } else {
    unpack2(horner4x2(coef::ASIN(), t), v0, v1);
  }
}

// Two angular pair evaluations on the tau branch for TWO pixels against one
// neighbour offset (vf_shared.cuh PX2): pk0/pk1 the pixels' packed RGB,
// nn2 = (|p0|^2, |p1|^2), nnn2 = -nn2, q = (pk(q0), pk(q1), |q0|^2, |q1|^2).
// Element-wise the same roundings as angular_tau2_r8.
template <int VAR>
__device__ __forceinline__ void angular_tau2_px2(uint32_t pk0, uint32_t pk1, f32x2 nn2, f32x2 nnn2, uint4 q,
                                                 float& tau0, float& tau1, float& v0, float& v1) {
  const f32x2 C = pack2(F2P23, F2P23);
  const f32x2 Db = pack2(__uint_as_float(__dp4a(pk0, q.x, F2P23_BITS)), __uint_as_float(__dp4a(pk1, q.y, F2P23_BITS)));
  const f32x2 D = sub2(Db, C);                            // exact dot products
  const f32x2 nD = sub2(C, Db);                           // -D, exact
  const f32x2 nnq = pack2(__uint_as_float(q.z), __uint_as_float(q.w));
  const f32x2 Ph = mul2(nn2, nnq);
  const f32x2 nPl = fma2(nnn2, nnq, Ph);                  // -(exact residual of nn nnq)
  const f32x2 X = sub2(fma2(nD, D, Ph), nPl);             // |p x q|^2
  float ph0, ph1, s0, s1;
  unpack2(Ph, ph0, ph1);
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s0) : "f"(ph0));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s1) : "f"(ph1));
  const f32x2 w = fma2(pack2(s0, s1), D, Ph);             // s (s + D)
  float xw0, xw1;
  unpack2(fma2(X, w, pack2(1e-30f, 1e-30f)), xw0, xw1);
  const f32x2 t = mul2(X, pack2(rsqrt_approx(xw0), rsqrt_approx(xw1)));   // sqrt(1 - cos)
  unpack2(t, tau0, tau1);
  if (VAR == EXACT) {
    v0 = 2.0f * asinf(tau0 * 0.70710678118654752f);
    v1 = 2.0f * asinf(tau1 * 0.70710678118654752f);
  } else {
    unpack2(horner4x2(coef::ASIN(), t), v0, v1);
  }
}

// Two pairs at once: zu2 = (z or u of pair 0, of pair 1); accumulates into
// (Ri0, Rj0) and (Ri1, Rj1) with the roundings of crit_accumulate.
template <int CRIT, int VAR>
__device__ __forceinline__ void crit_accumulate2(f32x2 zu2, float& Ri0, float& Rj0, float& Ri1, float& Rj1) {
  if (VAR == MINIMAX) {
    float n0, n1, q0, q1;
    unpack2(CRIT == EXPC ? horner4x2(coef::EXP_DELTA(), zu2) : horner4x2(coef::ENT_NEGN_U(), zu2), n0, n1);
    unpack2(CRIT == EXPC ? horner4x2(coef::EXP_Q(), zu2) : horner4x2(coef::ENT_Q_U(), zu2), q0, q1);
    const float r0 = rcp_approx(q0), r1 = rcp_approx(q1);
    Ri0 = fmaf(n0, r0, Ri0);
    Rj0 = fmaf(n0, r0, Rj0);
    Ri1 = fmaf(n1, r1, Ri1);
    Rj1 = fmaf(n1, r1, Rj1);
  } else if (VAR == REACH || VAR == POLY4) {
    float v0, v1;
    if (VAR == POLY4)
      unpack2(horner4x2(coef::EXP_1MP4(), zu2), v0, v1);
    else if (CRIT == EXPC)
      unpack2(horner_rec2<coef::R_EXP, 0>(zu2), v0, v1);
    else
      unpack2(horner_rec2<coef::R_LOG, 0>(zu2), v0, v1);
    Ri0 = __fadd_rn(Ri0, v0);
    Rj0 = __fadd_rn(Rj0, v0);
    Ri1 = __fadd_rn(Ri1, v1);
    Rj1 = __fadd_rn(Rj1, v1);
  } else {   // libm variants: scalar
    float z0, z1;
    unpack2(zu2, z0, z1);
    crit_accumulate<CRIT, VAR>(z0, Ri0, Rj0);
    crit_accumulate<CRIT, VAR>(z1, Ri1, Rj1);
  }
}

}  // namespace vf
