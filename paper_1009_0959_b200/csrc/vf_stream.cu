// vf_stream.cu -- the warp-streamed 3x3 angular kernels (vf_stream.cuh)
// in its own translation unit, so its ptxas settings and tuning knobs
// (VF_STREAM_MINB, VF_STREAM_ACOS) are independent of the other kernels.
#define VF_ANGULAR_MM_TU   // no kernel-selection helpers here
#include "vf_stream.cuh"

namespace vf {

const void* stream_kernel_fn_mm(bool half) {
  return half ? (const void*)vf_angular_stream_kernel<MINIMAX, 1, 16> : (const void*)vf_angular_stream_kernel<MINIMAX>;
}
const void* stream_kernel_fn_ex(bool half) {
  return half ? (const void*)vf_angular_stream_kernel<EXACT, 1, 16> : (const void*)vf_angular_stream_kernel<EXACT>;
}
const void* stream_kernel_fn_both(bool half) {
  return half ? (const void*)vf_angular_stream_kernel<MINIMAX, 2, 16> : (const void*)vf_angular_stream_kernel<MINIMAX, 2>;
}
size_t stream_smem_bytes(bool half) {
  return (half ? 2 * sizeof(stream::RingT<16>) : sizeof(stream::Ring)) * stream::NWARP;
}
dim3 stream_grid(const Launch& L, int B, int K, bool split_tail, bool tail) {
  return stream_grid_impl(L, B, K, split_tail, tail);
}
int stream_block_threads() { return 32 * stream::NWARP; }

}  // namespace vf
