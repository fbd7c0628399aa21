// vf_coeffs.cuh -- the paper's minimax coefficients (Tables 1-4) and
// the fp32 evaluation forms the kernels use.
//
// The decimal literals are the paper's printed strings.  The derived sets are
// computed here in constexpr double arithmetic and rounded to fp32 once:
//   * Table 3 exp rational used as 1 - N/Q = (Q - N)/Q = Delta(z)/Q(z) with
//     Delta = Q - N coefficientwise: no cancellation (all Delta_k > 0), so the
//     criterion D_E = 1 - E(z) keeps full relative precision near z = 0.
//   * Table 2 p = 4 used as 1 - P4(z) with coefficients (1 - a0, -a1, ...).
//   * Table 4 ENT rational re-expanded in u = 1 - s (the kernels form
//     u = c_L * d1 exactly-scaled and never s itself), so that D_L = -N/Q
//     near s = 1 keeps its relative precision:
//       Ntilde_m = (-1)^m sum_{k>=m} C(k,m) N_k,  likewise Qtilde.
// Nothing here is shared with the CPU oracle (oracle/vf_oracle.c), which
// evaluates the printed tables directly in double.
#pragma once

namespace vf {
namespace coef {

// ---- Table 1 -----------------------------------------------
constexpr double T1_ASIN[5] = {2.097797e-05, 1.412840, 1.429881e-02, 6.704361e-02, 6.909677e-02};
constexpr double T1_ACOS[5] = {1.570786, -9.990285e-01, -1.429899e-02, -9.481335e-02, -1.381942e-01};
// ---- Table 2, p = 4 -------------------------------------------------
constexpr double T2_P4[5] = {9.666313e-01, -7.620584e-01, 2.145386e-01, -2.509526e-02, 1.032877e-03};
// ---- Table 3 -------------------------------------------------
constexpr double T3_N[5] = {3.206619e-02, -1.195191e-02, 1.756974e-03, -1.199261e-04, 3.182685e-06};
constexpr double T3_Q[5] = {3.206627e-02, 2.011147e-02, 5.853684e-03, 9.780143e-04, 1.251598e-04};
// ---- Table 4 -------------------------------------------------
constexpr double T4_N[5] = {-1.519742e-04, -6.835769e-02, -8.856923e-01, -5.369609e-01, 1.491165};
constexpr double T4_Q[5] = {1.532270e-02, 3.987796e-01, 1.461793, 6.827004e-01, -4.469776e-02};

__host__ __device__ constexpr double binom(int k, int m) {
  double r = 1.0;
  for (int i = 1; i <= m; ++i) r = r * (double)(k - m + i) / (double)i;
  return r;
}
// coefficient m of p(1 - u) in powers of u, p given in powers of s
__host__ __device__ constexpr double reexpand(const double* a, int m) {
  double r = 0.0;
  for (int k = m; k < 5; ++k) r += binom(k, m) * a[k];
  return (m % 2) ? -r : r;
}

// fp32 coefficient sets, a[0] + a[1] x + ... + a[4] x^4
struct P4f { float a0, a1, a2, a3, a4; };

__host__ __device__ constexpr P4f ACOS() { return P4f{(float)T1_ACOS[0], (float)T1_ACOS[1], (float)T1_ACOS[2], (float)T1_ACOS[3], (float)T1_ACOS[4]}; }
__host__ __device__ constexpr P4f ASIN() { return P4f{(float)T1_ASIN[0], (float)T1_ASIN[1], (float)T1_ASIN[2], (float)T1_ASIN[3], (float)T1_ASIN[4]}; }
// exp rational as Delta/Q
__host__ __device__ constexpr P4f EXP_DELTA() { return P4f{(float)(T3_Q[0] - T3_N[0]), (float)(T3_Q[1] - T3_N[1]), (float)(T3_Q[2] - T3_N[2]),
                           (float)(T3_Q[3] - T3_N[3]), (float)(T3_Q[4] - T3_N[4])}; }
__host__ __device__ constexpr P4f EXP_Q() { return P4f{(float)T3_Q[0], (float)T3_Q[1], (float)T3_Q[2], (float)T3_Q[3], (float)T3_Q[4]}; }
// exp polynomial p=4 as 1 - P4
__host__ __device__ constexpr P4f EXP_1MP4() { return P4f{(float)(1.0 - T2_P4[0]), (float)(-T2_P4[1]), (float)(-T2_P4[2]), (float)(-T2_P4[3]),
                          (float)(-T2_P4[4])}; }
// ENT rational in u = 1 - s; the numerator carries the minus sign of D_L = -ENT
__host__ __device__ constexpr P4f ENT_NEGN_U() { return P4f{(float)(-reexpand(T4_N, 0)), (float)(-reexpand(T4_N, 1)), (float)(-reexpand(T4_N, 2)),
                            (float)(-reexpand(T4_N, 3)), (float)(-reexpand(T4_N, 4))}; }
__host__ __device__ constexpr P4f ENT_Q_U() { return P4f{(float)reexpand(T4_Q, 0), (float)reexpand(T4_Q, 1), (float)reexpand(T4_Q, 2),
                         (float)reexpand(T4_Q, 3), (float)reexpand(T4_Q, 4)}; }

// Direct (unshifted) forms for the AMNF / EVMF filters, whose arguments are
// not near the cancellation points: Table 3 numerator, Table 2 p = 4, Table 4.
__host__ __device__ constexpr P4f EXP_N() { return P4f{(float)T3_N[0], (float)T3_N[1], (float)T3_N[2], (float)T3_N[3], (float)T3_N[4]}; }
__host__ __device__ constexpr P4f EXP_P4() { return P4f{(float)T2_P4[0], (float)T2_P4[1], (float)T2_P4[2], (float)T2_P4[3], (float)T2_P4[4]}; }
__host__ __device__ constexpr P4f ENT_N() { return P4f{(float)T4_N[0], (float)T4_N[1], (float)T4_N[2], (float)T4_N[3], (float)T4_N[4]}; }
__host__ __device__ constexpr P4f ENT_Q() { return P4f{(float)T4_Q[0], (float)T4_Q[1], (float)T4_Q[2], (float)T4_Q[3], (float)T4_Q[4]}; }

// ---- minimax polynomials re-derived (Remez exchange)
// for the criterion values on the arguments they can reach:
//   D_E(z) = 1 - exp(-z) on [0, z*_25 = 0.7421166], degree 5, eps 7.86e-8
//   D_L(u) = -(1 - u) ln(1 - u) on [0, 1 - 1/e], degree 7, eps 2.95e-7
// (the decimal strings of tests/golden/remez_reach.txt; no division, and
// every coefficient beyond a0 is O(1), so fp32 Horner keeps its precision)
struct R_EXP {
  static constexpr int DEG = 5;
  __host__ __device__ static constexpr double c(int k) {
    constexpr double t[6] = {7.8607071043670362e-08, 0.99999223556347028, -0.49987553301909632,
                             0.16593299907325132, -0.039686762479510071, 0.0057878343103810199};
    return t[k];
  }
};
struct R_LOG {
  static constexpr int DEG = 7;
  __host__ __device__ static constexpr double c(int k) {
    constexpr double t[8] = {2.951515920989309e-07, 0.99994488204903353, -0.49831625626187054,
                             -0.18607535607515613, 0.02447556559350492, -0.36382847261870294,
                             0.43713641586762925, -0.32653163848077049};
    return t[k];
  }
};

constexpr double KAPPA = 0.33;
constexpr double ONE_MINUS_INV_E = 0.63212055882855767840;  // 1 - e^-1 (reading R3)

}  // namespace coef
}  // namespace vf
