// vf_stream.cu -- the warp-streamed 3x3 angular kernels (vf_stream.cuh)
// in its own translation unit, so its ptxas settings and tuning knobs
// (VF_STREAM_MINB, VF_STREAM_ACOS) are independent of the other kernels.
#define VF_ANGULAR_MM_TU   // no kernel-selection helpers here
#include "vf_stream.cuh"

namespace vf {

const void* stream_kernel_fn_mm() { return (const void*)vf_angular_stream_kernel<MINIMAX>; }
const void* stream_kernel_fn_ex() { return (const void*)vf_angular_stream_kernel<EXACT>; }
const void* stream_kernel_fn_both() { return (const void*)vf_angular_stream_kernel<MINIMAX, 2>; }
size_t stream_smem_bytes() { return sizeof(stream::Ring) * stream::NWARP; }
dim3 stream_grid(const Launch& L, int B, int K) { return stream_grid_impl(L, B, K); }
int stream_block_threads() { return 32 * stream::NWARP; }

}  // namespace vf
