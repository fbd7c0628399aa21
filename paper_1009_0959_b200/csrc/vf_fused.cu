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
