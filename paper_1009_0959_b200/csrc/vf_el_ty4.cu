// vf_el_ty4.cu -- the 3x3 exp/log kernels of the non-libm variants (minimax,
// poly4, reach) in 4-warp blocks, the configuration vf_api.cu launches for
// large 3x3 launches.  They live in their own translation unit so that they
// can be compiled with their own ptxas setting (build.py SOURCE_FLAGS:
// --register-usage-level=2, measured ~1% faster for these kernels and up to
// 17% slower for the libm ones).
#include "vf_window.cuh"

namespace vf {

template <int OPT>
static const void* el_kernel_ty4_opt(int crit, int var) {
  if (crit == EXPC) {
    if (var == MINIMAX) return (const void*)vf_el_kernel<3, EXPC, MINIMAX, OPT, 4>;
    if (var == REACH) return (const void*)vf_el_kernel<3, EXPC, REACH, OPT, 4>;
    if (var == POLY4) return (const void*)vf_el_kernel<3, EXPC, POLY4, OPT, 4>;
    return nullptr;
  }
  if (var == REACH) return (const void*)vf_el_kernel<3, LOGC, REACH, OPT, 4>;
  if (var == MINIMAX) return (const void*)vf_el_kernel<3, LOGC, MINIMAX, OPT, 4>;
  return nullptr;
}

// 3x3, 4-warp blocks, opt = 2 or 4 output rows per thread; nullptr for the
// exact variants (not compiled in this configuration).
const void* el_kernel_ty4(int opt, int crit, int var) {
  return opt == 4 ? el_kernel_ty4_opt<4>(crit, var) : el_kernel_ty4_opt<2>(crit, var);
}

}  // namespace vf
