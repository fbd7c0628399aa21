// vf_api.cu -- C ABI of libvf.so (declared in include/vf.h): argument
// validation, kernel dispatch, error reporting.  Host code only launches;
// every step of the filter runs in the kernels of vf_window.cuh /
// vf_shared.cuh.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/vf.h"
#include "vf_shared.cuh"
#include "vf_stats.cuh"
#include "vf_window.cuh"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, const char* a = "", long long v = 0) {
  std::snprintf(g_err, sizeof(g_err), fmt, a, v);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  std::snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
  return VF_ECUDA;
}

bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}

using vf::Launch;
typedef void (*KernelFn)(const Launch);

template <int WIN>
KernelFn window_kernel(int crit, int var) {
  using namespace vf;
  if (crit == ANGULAR) return var == EXACT ? vf_angular_window_kernel<WIN, EXACT> : vf_angular_window_kernel<WIN, MINIMAX>;
  if (crit == EXPC) {
    if (var == EXACT) return vf_el_kernel<WIN, EXPC, EXACT>;
    if (var == MINIMAX) return vf_el_kernel<WIN, EXPC, MINIMAX>;
    return vf_el_kernel<WIN, EXPC, POLY4>;
  }
  return var == EXACT ? vf_el_kernel<WIN, LOGC, EXACT> : vf_el_kernel<WIN, LOGC, MINIMAX>;
}

int validate(int B, int H, int W, int window, int crit, int var) {
  if (window < 3 || window % 2 == 0) return fail(VF_EINVAL, "window must be odd and >= 3%s (got %lld)", "", window);
  if (B < 1) return fail(VF_EINVAL, "batch must be >= 1%s (got %lld)", "", B);
  if (H < 1 || W < 1) return fail(VF_EINVAL, "image size must be positive%s", "");
  if (window > H || window > W) return fail(VF_EINVAL, "window larger than the image (S:64)%s", "");
  if (crit < 0 || crit > 2) return fail(VF_EINVAL, "criterion out of range%s (%lld)", "", crit);
  if (var < 0 || var > 2) return fail(VF_EINVAL, "variant out of range%s (%lld)", "", var);
  if (var == VF_MINIMAX_POLY4 && crit != VF_EXP) return fail(VF_EINVAL, "VF_MINIMAX_POLY4 is only defined for VF_EXP%s", "");
  if (window > 5) return fail(VF_EUNSUPPORTED, "window %s%lld is valid but not compiled (3 and 5 are)", "", window);
  return VF_OK;
}

float kscale(int crit, int window) {
  const double n = (double)window * window;
  if (crit == VF_EXP) return (float)(std::pow(n, 1.0 + vf::coef::KAPPA / 3.0) / 2.0);  // c_E * S1
  if (crit == VF_LOG) return (float)(vf::coef::ONE_MINUS_INV_E * (n - 1.0));          // c_L * S1
  return 0.0f;
}

int launch(const uint8_t* in, long long in_stride, int band_row0, int band_rows, int B, int H, int W,
           int out_row0, int out_rows, int window, int crit, int var, int algo, uint8_t* out,
           long long out_stride, uint8_t* index, float* agg, cudaStream_t st) {
  Launch L;
  L.in = in; L.out = out; L.idx = index; L.agg = agg;
  L.in_stride = in_stride; L.out_stride = out_stride;
  L.H = H; L.W = W; L.band_row0 = band_row0; L.band_rows = band_rows;
  L.out_row0 = out_row0; L.out_rows = out_rows;
  L.kscale = kscale(crit, window);

  if (crit == VF_ANGULAR && algo != VF_ALGO_WINDOW) {
    const int rc = vf::launch_shared(L, B, window, var, st);
    if (rc != -100) {   // -100: shared kernel not applicable, fall through
      if (rc != 0) return cuda_fail((cudaError_t)rc, "vf_shared_kernel launch");
      return VF_OK;
    }
  }
  KernelFn k = window == 3 ? window_kernel<3>(crit, var) : window_kernel<5>(crit, var);
  dim3 grid((W + vf::TX - 1) / vf::TX, (out_rows + vf::TY - 1) / vf::TY, B);
  dim3 block(vf::TX, vf::TY);
  if (grid.y > 65535 || grid.z > 65535) return fail(VF_EINVAL, "grid too large%s", "");
  k<<<grid, block, 0, st>>>(L);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "vf_window_kernel launch");
  return VF_OK;
}

}  // namespace

extern "C" {

int vf_filter_batch_algo(const uint8_t* imgs, int B, int H, int W, int window, int criterion, int variant,
                         int algo, uint8_t* outs, uint8_t* index, float* aggregates, void* stream) {
  g_err[0] = 0;
  int rc = validate(B, H, W, window, criterion, variant);
  if (rc) return rc;
  if (!imgs || !outs) return fail(VF_EINVAL, "NULL image or output pointer%s", "");
  if (algo < 0 || algo > 2) return fail(VF_EINVAL, "algo out of range%s", "");
  const size_t bytes = (size_t)B * H * W * 3;
  if (overlap(imgs, bytes, outs, bytes)) return fail(VF_EINVAL, "input and output overlap%s", "");
  const long long stride = (long long)H * W * 3;
  return launch(imgs, stride, 0, H, B, H, W, 0, H, window, criterion, variant, algo, outs, stride, index,
                aggregates, (cudaStream_t)stream);
}

int vf_filter_batch(const uint8_t* imgs, int B, int H, int W, int window, int criterion, int variant,
                    uint8_t* outs, uint8_t* index, float* aggregates, void* stream) {
  return vf_filter_batch_algo(imgs, B, H, W, window, criterion, variant, VF_ALGO_AUTO, outs, index, aggregates,
                              stream);
}

int vf_filter(const uint8_t* img, int H, int W, int window, int criterion, int variant, uint8_t* out,
              uint8_t* index, float* aggregates, void* stream) {
  return vf_filter_batch_algo(img, 1, H, W, window, criterion, variant, VF_ALGO_AUTO, out, index, aggregates,
                              stream);
}

int vf_filter_rows(const uint8_t* band, int band_row0, int band_rows, int H, int W, int out_row0, int out_rows,
                   int window, int criterion, int variant, uint8_t* out, uint8_t* index, float* aggregates,
                   void* stream) {
  g_err[0] = 0;
  int rc = validate(1, H, W, window, criterion, variant);
  if (rc) return rc;
  if (!band || !out) return fail(VF_EINVAL, "NULL band or output pointer%s", "");
  if (out_rows < 1 || out_row0 < 0 || out_row0 + out_rows > H)
    return fail(VF_EINVAL, "output rows outside the image%s", "");
  const int r = window / 2;
  const int need_lo = out_row0 - r < 0 ? 0 : out_row0 - r;
  const int need_hi = out_row0 + out_rows + r > H ? H : out_row0 + out_rows + r;
  if (band_rows < 1 || band_row0 < 0 || band_row0 > need_lo || band_row0 + band_rows < need_hi ||
      band_row0 + band_rows > H)
    return fail(VF_EINVAL, "row band does not cover the rows the stripe reads%s", "");
  if (overlap(band, (size_t)band_rows * W * 3, out, (size_t)out_rows * W * 3))
    return fail(VF_EINVAL, "input and output overlap%s", "");
  return launch(band, 0, band_row0, band_rows, 1, H, W, out_row0, out_rows, window, criterion, variant,
                VF_ALGO_AUTO, out, 0, index, aggregates, (cudaStream_t)stream);
}

size_t vf_host_workspace_bytes(int B, int H, int W) {
  if (B < 1 || H < 1 || W < 1) return 0;
  const size_t img = (size_t)B * H * W * 3;
  return 2 * ((img + 255) / 256 * 256);
}

int vf_filter_host(const uint8_t* h_imgs, int B, int H, int W, int window, int criterion, int variant,
                   uint8_t* h_outs, void* d_workspace, size_t workspace_bytes, void* stream) {
  g_err[0] = 0;
  int rc = validate(B, H, W, window, criterion, variant);
  if (rc) return rc;
  if (!h_imgs || !h_outs || !d_workspace) return fail(VF_EINVAL, "NULL pointer%s", "");
  const size_t need = vf_host_workspace_bytes(B, H, W);
  if (workspace_bytes < need) return fail(VF_EINVAL, "workspace too small (need %s%lld bytes)", "", (long long)need);
  const size_t img = (size_t)B * H * W * 3;
  uint8_t* d_in = (uint8_t*)d_workspace;
  uint8_t* d_out = d_in + (img + 255) / 256 * 256;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(d_in, h_imgs, img, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
  const long long stride = (long long)H * W * 3;
  rc = launch(d_in, stride, 0, H, B, H, W, 0, H, window, criterion, variant, VF_ALGO_AUTO, d_out, stride, nullptr,
              nullptr, st);
  if (rc) return rc;
  e = cudaMemcpyAsync(h_outs, d_out, img, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
  return VF_OK;
}

int vf_image_stats(const uint8_t* a, const uint8_t* b, int B, int H, int W, double* stats, void* stream) {
  g_err[0] = 0;
  if (!a || !b || !stats) return fail(VF_EINVAL, "NULL pointer%s", "");
  if (B < 1 || H < 1 || W < 1) return fail(VF_EINVAL, "bad size%s", "");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(stats, 0, sizeof(double) * 8 * (size_t)B, st);
  if (e != cudaSuccess) return cuda_fail(e, "stats memset");
  const long long npix = (long long)H * W;
  int blocks = (int)((npix + 255) / 256);
  if (blocks > 148 * 4) blocks = 148 * 4;
  vf::vf_stats_kernel<<<dim3(blocks, B), 256, 0, st>>>(a, b, npix, stats);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "vf_stats_kernel launch");
  return VF_OK;
}

const char* vf_status_string(int status) {
  switch (status) {
    case VF_OK: return "VF_OK";
    case VF_EINVAL: return "VF_EINVAL: invalid argument";
    case VF_EUNSUPPORTED: return "VF_EUNSUPPORTED: valid but not compiled";
    case VF_ECUDA: return "VF_ECUDA: CUDA error";
    default: return "unknown vf_status";
  }
}

const char* vf_last_error(void) { return g_err; }

int vf_version(void) { return 100; }

}  // extern "C"
