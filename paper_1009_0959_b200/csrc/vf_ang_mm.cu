// vf_ang_mm.cu -- the angular minimax kernels (pair-sharing 3x3/5x5 and
// role-sum kernels, every launch configuration) in their own translation unit,
// compiled with their own ptxas setting (build.py SOURCE_FLAGS:
// --register-usage-level=2).  vf_api.cu is compiled with
// VF_ANGULAR_MM_EXTERN and fetches them through these two functions.
#define VF_ANGULAR_MM_TU   // no kernel-selection helpers here (they would instantiate the exact kernels too)
#include "vf_role.cuh"
#include "vf_shared.cuh"

namespace vf {

template <int WIN>
static const void* shared_mm_w(int cfg) {
  switch (cfg) {
    case 1: return (const void*)vf_angular_shared_kernel<WIN, MINIMAX, 1>;
    case 2: return (const void*)vf_angular_shared_kernel<WIN, MINIMAX, 2>;
    case 3: return (const void*)vf_angular_shared_kernel<WIN, MINIMAX, 3>;
    default: return (const void*)vf_angular_shared_kernel<WIN, MINIMAX, 4>;
  }
}

template <int WIN>
static const void* role_mm_w(int cfg) {
  switch (cfg) {
    case 1: return (const void*)vf_angular_role_kernel<WIN, MINIMAX, shared::cfg_nt(1), shared::cfg_ppt(1)>;
    case 2: return (const void*)vf_angular_role_kernel<WIN, MINIMAX, shared::cfg_nt(2), shared::cfg_ppt(2)>;
    case 3: return (const void*)vf_angular_role_kernel<WIN, MINIMAX, shared::cfg_nt(3), shared::cfg_ppt(3)>;
    default: return (const void*)vf_angular_role_kernel<WIN, MINIMAX, shared::cfg_nt(4), shared::cfg_ppt(4)>;
  }
}

const void* shared_kernel_fn_mm(int window, int cfg) { return window == 3 ? shared_mm_w<3>(cfg) : shared_mm_w<5>(cfg); }
const void* role_kernel_fn_mm(int window, int cfg) { return window == 3 ? role_mm_w<3>(cfg) : role_mm_w<5>(cfg); }

}  // namespace vf
