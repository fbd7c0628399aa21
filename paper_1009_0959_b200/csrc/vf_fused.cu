// vf_fused.cu -- plan-level fusion of the exp/log filters of one input
// (vf_plan_create): the exp and log criteria of readings R2/R3 both derive
// from the same integer L1 distances d1_ij and the same window statistic
// S1 = sum_{i<j} d1_ij (Eq. 8), so one kernel stages each tile once,
// forms S1 once per window (StripS1) and then runs every requested
// criterion x variant's pass 2, argmin and store (a5-a8) per window.  Each
// filter's output is bit-identical to its own kernel's (the same
// el_window_s1 arithmetic, every rounding spelled out).
#include "vf_window.cuh"

namespace vf {

struct ElFused {
  Launch L[8];     // one per filter: the same input / geometry, own out and kscale
  int code[8];     // 4 * criterion + variant (EXPC / LOGC x EXACT / MINIMAX / POLY4 / REACH)
  int n;
};

template <int WIN, int CRIT, int VAR, int OPT>
__device__ __forceinline__ void el_windows(const Launch& L, int b, int ox, int oyb, const uint32_t* pk,
                                           const StripS1<WIN, OPT>& s1, int rows_here) {
#pragma unroll
  for (int o = 0; o < OPT; ++o)
    if (o < rows_here) el_window_s1<WIN, CRIT, VAR>(L, b, ox, oyb + o, pk + o * WIN, s1.window(o));
}

// grid / block as vf_el_kernel<WIN, *, *, OPT, NTY> (the geometry of F.L[0]).
template <int WIN, int OPT, int NTY>
__global__ void __launch_bounds__(TX * NTY) vf_el_fused_kernel(const ElFused F) {
  constexpr int R = WIN / 2;
  constexpr int TYE = NTY * OPT;
  constexpr int SW = TX + 2 * R;
  constexpr int SH = TYE + 2 * R;
  constexpr int LR = OPT + WIN - 1;
  __shared__ StageSmem<SW, SH> sm;
  const Launch& L0 = F.L[0];
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX;
  const int y0 = L0.out_row0 + blockIdx.y * TYE;
  const uint8_t* __restrict__ in = L0.in + (long long)b * L0.in_stride;
  stage_packed<SW, SH, TX, NTY>(L0, in, x0 - R, y0 - R, sm);

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int ox = x0 + tx;
  const int oyb = y0 + OPT * ty;
  if (ox >= L0.W || oyb >= L0.out_row0 + L0.out_rows) return;
  uint32_t pk[LR * WIN];
#pragma unroll
  for (int k = 0; k < LR * WIN; ++k) pk[k] = sm.pk[(OPT * ty + k / WIN) * SW + tx + k % WIN];
  const int rows_here = min(OPT, L0.out_row0 + L0.out_rows - oyb);
  StripS1<WIN, OPT> s1;                                   // a3 once for every filter
  s1.build(pk);
  for (int f = 0; f < F.n; ++f) {                         // block-uniform dispatch
    switch (F.code[f]) {
      case 4 * EXPC + EXACT: el_windows<WIN, EXPC, EXACT, OPT>(F.L[f], b, ox, oyb, pk, s1, rows_here); break;
      case 4 * EXPC + MINIMAX: el_windows<WIN, EXPC, MINIMAX, OPT>(F.L[f], b, ox, oyb, pk, s1, rows_here); break;
      case 4 * EXPC + POLY4: el_windows<WIN, EXPC, POLY4, OPT>(F.L[f], b, ox, oyb, pk, s1, rows_here); break;
      case 4 * EXPC + REACH: el_windows<WIN, EXPC, REACH, OPT>(F.L[f], b, ox, oyb, pk, s1, rows_here); break;
      case 4 * LOGC + EXACT: el_windows<WIN, LOGC, EXACT, OPT>(F.L[f], b, ox, oyb, pk, s1, rows_here); break;
      case 4 * LOGC + MINIMAX: el_windows<WIN, LOGC, MINIMAX, OPT>(F.L[f], b, ox, oyb, pk, s1, rows_here); break;
      case 4 * LOGC + REACH: el_windows<WIN, LOGC, REACH, OPT>(F.L[f], b, ox, oyb, pk, s1, rows_here); break;
      default: break;
    }
  }
}

// The bench's set -- exp exact, exp minimax, exp poly4, log exact, log
// minimax -- in PAIR-MAJOR order: each pair's biased distance 2^23 + d1 is
// formed once (one VABSDIFF4), scaled once for exp (z) and once for log (u),
// and accumulated into all five filters' aggregates (45 registers).  Per
// filter the pairs are visited in the same order with the same arithmetic as
// its own kernel (el_window / el_window_s1), so every output is bit-identical.
// F.code must be {EXP_EX, EXP_MM, EXP_P4, LOG_EX, LOG_MM} in this order.
template <int WIN>
__device__ __forceinline__ void el_window5(const ElFused& F, int b, int ox, int oy, const uint32_t* w, uint32_t S1) {
  constexpr int N = WIN * WIN;
  constexpr int NPR = N * (N - 1) / 2;
  const float rs = (S1 != 0u) ? rcp_approx((float)S1) : 0.0f;
  const float scE = (S1 != 0u) ? F.L[0].kscale * rs : 0.0f;
  const float scL = (S1 != 0u) ? F.L[3].kscale * rs : 0.0f;
  const float bE = -scE * F2P23, bL = -scL * F2P23;
  float A[5][N];
#pragma unroll
  for (int f = 0; f < 5; ++f)
#pragma unroll
    for (int k = 0; k < N; ++k) A[f][k] = -0.0f;
  const f32x2 scE2 = pack2(scE, scE), bE2 = pack2(bE, bE), scL2 = pack2(scL, scL), bL2 = pack2(bL, bL);
  static_for<NPR / 2>([&](auto qc) {
    constexpr int p0 = 2 * decltype(qc)::value, p1 = p0 + 1;
    constexpr int i0 = pair_i<N>(p0), j0 = pair_j<N>(p0), i1 = pair_i<N>(p1), j1 = pair_j<N>(p1);
    const float fb0 = __uint_as_float(sad4(w[i0], w[j0], F2P23_BITS));
    const float fb1 = __uint_as_float(sad4(w[i1], w[j1], F2P23_BITS));
    const f32x2 fb2 = pack2(fb0, fb1);
    const f32x2 z2 = fma2(scE2, fb2, bE2), u2 = fma2(scL2, fb2, bL2);
    float z0, z1, u0, u1;
    unpack2(z2, z0, z1);
    unpack2(u2, u0, u1);
    crit_accumulate<EXPC, EXACT>(z0, A[0][i0], A[0][j0]);
    crit_accumulate<EXPC, EXACT>(z1, A[0][i1], A[0][j1]);
    crit_accumulate2<EXPC, MINIMAX>(z2, A[1][i0], A[1][j0], A[1][i1], A[1][j1]);
    crit_accumulate2<EXPC, POLY4>(z2, A[2][i0], A[2][j0], A[2][i1], A[2][j1]);
    crit_accumulate<LOGC, EXACT>(u0, A[3][i0], A[3][j0]);
    crit_accumulate<LOGC, EXACT>(u1, A[3][i1], A[3][j1]);
    crit_accumulate2<LOGC, MINIMAX>(u2, A[4][i0], A[4][j0], A[4][i1], A[4][j1]);
  });
  static_assert(NPR % 2 == 0, "pairs in packed twos");
#pragma unroll
  for (int f = 0; f < 5; ++f) {
    float bv = A[f][0];
    uint32_t o = w[0];
#pragma unroll
    for (int k = 1; k < N; ++k) {
      const bool lt = A[f][k] < bv;
      bv = lt ? A[f][k] : bv;
      o = lt ? w[k] : o;
    }
    if (F.L[f].agg && S1 == 0u) {
#pragma unroll
      for (int k = 0; k < N; ++k) A[f][k] = 0.0f;
    }
    store_result<N>(F.L[f], b, ox, oy, A[f], o);
  }
}

#ifndef VF_FUSED5_MINB
#define VF_FUSED5_MINB 3   // <= 85 registers (80, 24 B of spills): step 64.7 vs 65.0 ms (1: 107 registers)
#endif
template <int WIN, int OPT, int NTY>
__global__ void __launch_bounds__(TX * NTY, VF_FUSED5_MINB) vf_el_fused5_kernel(const ElFused F) {
  constexpr int R = WIN / 2;
  constexpr int TYE = NTY * OPT;
  constexpr int SW = TX + 2 * R;
  constexpr int SH = TYE + 2 * R;
  constexpr int LR = OPT + WIN - 1;
  __shared__ StageSmem<SW, SH> sm;
  const Launch& L0 = F.L[0];
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX;
  const int y0 = L0.out_row0 + blockIdx.y * TYE;
  const uint8_t* __restrict__ in = L0.in + (long long)b * L0.in_stride;
  stage_packed<SW, SH, TX, NTY>(L0, in, x0 - R, y0 - R, sm);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int ox = x0 + tx;
  const int oyb = y0 + OPT * ty;
  if (ox >= L0.W || oyb >= L0.out_row0 + L0.out_rows) return;
  uint32_t pk[LR * WIN];
#pragma unroll
  for (int k = 0; k < LR * WIN; ++k) pk[k] = sm.pk[(OPT * ty + k / WIN) * SW + tx + k % WIN];
  const int rows_here = min(OPT, L0.out_row0 + L0.out_rows - oyb);
  StripS1<WIN, OPT> s1;
  s1.build(pk);
#pragma unroll
  for (int o = 0; o < OPT; ++o)
    if (o < rows_here) el_window5<WIN>(F, b, ox, oyb + o, pk + o * WIN, s1.window(o));
}

#ifndef VF_FUSED5_OPT
#define VF_FUSED5_OPT 2   // measured: OPT 2 65.0 ms, 1 65.5 ms step (8 warps); 4 warps 67.0
#endif
#ifndef VF_FUSED5_NTY
#define VF_FUSED5_NTY 8
#endif
// the pair-major kernel for the canonical 5-filter set (3x3, large launches)
const void* el_fused5_kernel(int* opt, int* nty) {
  *opt = VF_FUSED5_OPT;
  *nty = VF_FUSED5_NTY;
  return (const void*)vf_el_fused5_kernel<3, VF_FUSED5_OPT, VF_FUSED5_NTY>;
}

#ifndef VF_FUSED_OPT3
#define VF_FUSED_OPT3 2     // 3x3: output rows per thread (tuning knob)
#endif
#ifndef VF_FUSED_NTY3
#define VF_FUSED_NTY3 8     // 3x3: warps per block
#endif

// Kernel and launch shape of the fused exp/log node for a window size (large
// launches; small ones use one row per thread so more blocks fill the GPU).
const void* el_fused_kernel(int window, bool big, int* opt, int* nty) {
  if (window == 3 && big) {
    *opt = VF_FUSED_OPT3;
    *nty = VF_FUSED_NTY3;
    return (const void*)vf_el_fused_kernel<3, VF_FUSED_OPT3, VF_FUSED_NTY3>;
  }
#ifndef VF_FUSED_SMALL_NTY
#define VF_FUSED_SMALL_NTY 8
#endif
  *opt = 1;
  *nty = VF_FUSED_SMALL_NTY;
  return window == 3 ? (const void*)vf_el_fused_kernel<3, 1, VF_FUSED_SMALL_NTY>
                     : (const void*)vf_el_fused_kernel<5, 1, VF_FUSED_SMALL_NTY>;
}

}  // namespace vf
