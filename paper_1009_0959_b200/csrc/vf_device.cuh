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
//       exactly as fl(4D^2 - Ph) < Pl (see DESIGN.md section 5.2 for the proof).
// 1 - cos = X / (s (s + D)) with s = |x_i||x_j| needs no subtraction, so
// tau = sqrt(1 - cos) keeps full relative precision for near-parallel pairs.
#pragma once
#include <cstdint>

#include "vf_coeffs.cuh"

namespace vf {

enum { ANGULAR = 0, EXPC = 1, LOGC = 2 };
enum { EXACT = 0, MINIMAX = 1, POLY4 = 2 };

__device__ __forceinline__ float horner4(const coef::P4f p, float x) {
  return fmaf(fmaf(fmaf(fmaf(p.a4, x, p.a3), x, p.a2), x, p.a1), x, p.a0);
}

// Angular criterion A(x_i, x_j) of Eq. 5 for one pair.
// (r,g,b) components, nn = squared norm, nrm = norm, rn = 1/norm (0 for a
// zero vector).  Zero vectors fall into the tau branch with X = 0 -> tau = 0;
// the exact variant then returns 0 and the minimax variant the
// ARCSIN row's a0, which the window code removes (zero-vector fix-up).
template <int VAR>
__device__ __forceinline__ float angular_pair(float ri, float gi, float bi, float nni, float nrmi, float rni,
                                              float rj, float gj, float bj, float nnj, float nrmj, float rnj) {
  const float D = fmaf(ri, rj, fmaf(gi, gj, __fmul_rn(bi, bj)));  // exact
  const float Ph = __fmul_rn(nni, nnj);
  const float Pl = fmaf(nni, nnj, -Ph);                           // exact residual
  const float X = __fadd_rn(fmaf(-D, D, Ph), Pl);                 // |x_i x x_j|^2
  const float t = fmaf(__fmul_rn(4.0f, D), D, -Ph);               // fl(4D^2 - Ph)
  const bool acos_branch = t < Pl;                                // cos < 0.5, exact
  const float s = __fmul_rn(nrmi, nrmj);
  const float w = fmaf(s, D, Ph);                                 // s (s + D)
  const float tau = __fmul_rn(X, rsqrtf(fmaxf(__fmul_rn(X, w), 1e-30f)));  // sqrt(1 - cos)
  const float c = __fmul_rn(__fmul_rn(D, rni), rnj);              // cos
  if (VAR == EXACT) {
    // Eq. 6: arccos z = 2 arcsin(sqrt(0.5 (1 - z))) for z >= 0.5
    return acos_branch ? acosf(c) : 2.0f * asinf(tau * 0.70710678118654752f);
  } else {
    // Table 1: ARCCOS row on cos (cos < 0.5), ARCSIN row on tau (Eq. 7)
    const float x = acos_branch ? c : tau;
    const coef::P4f p = {acos_branch ? coef::ACOS().a0 : coef::ASIN().a0, acos_branch ? coef::ACOS().a1 : coef::ASIN().a1,
                         acos_branch ? coef::ACOS().a2 : coef::ASIN().a2, acos_branch ? coef::ACOS().a3 : coef::ASIN().a3,
                         acos_branch ? coef::ACOS().a4 : coef::ASIN().a4};
    return horner4(p, x);
  }
}

// Exp criterion D_E = 1 - E(z) (reading R2), z = c_E * d1 (never above
// z*_n < 1, so the P:163 cutoff is dead code and omitted).
template <int VAR>
__device__ __forceinline__ float exp_crit(float z) {
  if (VAR == EXACT) return -expm1f(-z);
  if (VAR == MINIMAX) return __fdividef(horner4(coef::EXP_DELTA(), z), horner4(coef::EXP_Q(), z));
  return horner4(coef::EXP_1MP4(), z);
}

// Log criterion D_L = -ENT(s), s = 1 - u, u = c_L * d1 in [0, 1 - 1/e]
// (reading R3; s >= 1/e > 0.05, so the P:232 cutoff is dead code).
template <int VAR>
__device__ __forceinline__ float log_crit(float u) {
  if (VAR == EXACT) return -(1.0f - u) * log1pf(-u);
  return __fdividef(horner4(coef::ENT_NEGN_U(), u), horner4(coef::ENT_Q_U(), u));
}

__device__ __forceinline__ float l1(float ri, float gi, float bi, float rj, float gj, float bj) {
  return fabsf(ri - rj) + fabsf(gi - gj) + fabsf(bi - bj);   // exact integer
}

__device__ __forceinline__ float l1_maxmin(float ri, float gi, float bi, float rj, float gj, float bj) {
  return ((fmaxf(ri, rj) - fminf(ri, rj)) + (fmaxf(gi, gj) - fminf(gi, gj))) + (fmaxf(bi, bj) - fminf(bi, bj));
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

}  // namespace vf
