// vf_api.cu -- C ABI of libvf.so (declared in include/vf.h): argument
// validation, kernel selection, launches, the plan executor (an instantiated
// CUDA graph of parallel filter kernels) and error reporting.  Host code only
// launches; every step of the filter runs in the kernels of vf_window.cuh /
// vf_shared.cuh.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#define VF_ANGULAR_MM_EXTERN   // angular minimax kernels: vf_ang_mm.cu
#include "../../include/vf.h"
#include "vf_paper.cuh"
#include "vf_role.cuh"
#include "vf_shared.cuh"
#include "vf_stats.cuh"
#include "vf_stream.cuh"
#include "vf_tma.cuh"
#include "vf_window.cuh"

namespace vf {
// vf_el_ty4.cu (its own translation unit and ptxas setting)
const void* el_kernel_ty4(int opt, int crit, int var);
// vf_fused.cu: the fused exp/log node of a plan
struct ElFused {
  Launch L[8];
  int code[8];
  int n;
};
const void* el_fused_kernel(int window, bool big, int* opt, int* nty);
const void* el_fused5_kernel(int* opt, int* nty);
}  // namespace vf

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* msg, long long v = 0) {
  std::snprintf(g_err, sizeof(g_err), msg, v);
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

// One kernel launch, fully described (function, geometry, parameters), so that
// it can be launched on a stream or added to a graph as a kernel node.
struct KernelDesc {
  const void* fn;
  dim3 grid, block;
  size_t smem;   // dynamic shared memory bytes
  Launch L;
  bool tma = false;          // vf_el_tma_kernel: (map, L, tiles_x, tiles_y, ntiles)
  alignas(64) CUtensorMap map;
  int tiles_x = 0, tiles_y = 0, ntiles = 0;
  int stream_k = 0;          // vf_angular_stream_kernel: (L, K, L2, nimg)
  int stream_b = 0;          //   nimg = the batch size
  Launch L2;                 // the fused kernel's second output (exact); = L otherwise
  // optional second launch with the same parameters (the streamed kernels'
  // half-warp remainder strips, vf_stream.cuh); independent of the first
  const void* fn_tail = nullptr;
  dim3 grid_tail;
  size_t smem_tail = 0;
  void* args[5];
  void** params() {
    if (stream_k) { args[0] = &L; args[1] = &stream_k; args[2] = &L2; args[3] = &stream_b; return args; }
    if (!tma) { args[0] = &L; return args; }
    args[0] = &map; args[1] = &L; args[2] = &tiles_x; args[3] = &tiles_y; args[4] = &ntiles;
    return args;
  }
};

// cuTensorMapEncodeTiled from the driver (no -lcuda link: runtime entry point).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}

// Resident blocks per SM x SMs of the current device for a kernel (cached).
int persistent_blocks(const void* fn, int threads, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : cache)
    if (e.first.first == fn && e.first.second == dev) return e.second;
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1) per_sm = 1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) sms = 1;
  cache.push_back({{fn, dev}, per_sm * sms});
  return per_sm * sms;
}

// One-time per-process kernel attribute setup (thread-safe).
// Kernel attributes (> 48 KB dynamic shared memory) are per device: set once
// for each device the process launches on (thread-safe).
cudaError_t ensure_attributes() {
  static std::mutex mu;
  static std::vector<int> done;   // devices already set up
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  for (int d : done)
    if (d == dev) return cudaSuccess;
  e = vf::shared_set_attributes();
  if (e == cudaSuccess) e = vf::role_set_attributes();
  if (e == cudaSuccess) done.push_back(dev);
  return e;
}

template <int WIN, int OPT>
const void* el_kernel(int crit, int var) {
  using namespace vf;
  if (crit == EXPC) {
    if (var == EXACT) return (const void*)vf_el_kernel<WIN, EXPC, EXACT, OPT>;
    if (var == MINIMAX) return (const void*)vf_el_kernel<WIN, EXPC, MINIMAX, OPT>;
    if (var == REACH) return (const void*)vf_el_kernel<WIN, EXPC, REACH, OPT>;
    return (const void*)vf_el_kernel<WIN, EXPC, POLY4, OPT>;
  }
  if (var == REACH) return (const void*)vf_el_kernel<WIN, LOGC, REACH, OPT>;
  return var == EXACT ? (const void*)vf_el_kernel<WIN, LOGC, EXACT, OPT> : (const void*)vf_el_kernel<WIN, LOGC, MINIMAX, OPT>;
}

template <int WIN, int OPT>
const void* el_tma_kernel(int crit, int var) {
  using namespace vf;
  if (crit == EXPC) {
    if (var == EXACT) return (const void*)vf_el_tma_kernel<WIN, EXPC, EXACT, OPT>;
    if (var == MINIMAX) return (const void*)vf_el_tma_kernel<WIN, EXPC, MINIMAX, OPT>;
    if (var == REACH) return (const void*)vf_el_tma_kernel<WIN, EXPC, REACH, OPT>;
    return (const void*)vf_el_tma_kernel<WIN, EXPC, POLY4, OPT>;
  }
  if (var == REACH) return (const void*)vf_el_tma_kernel<WIN, LOGC, REACH, OPT>;
  return var == EXACT ? (const void*)vf_el_tma_kernel<WIN, LOGC, EXACT, OPT>
                      : (const void*)vf_el_tma_kernel<WIN, LOGC, MINIMAX, OPT>;
}

template <int WIN>
const void* window_kernel(int crit, int var) {
  using namespace vf;
  if (crit == AMNFE)
    return var == EXACT ? (const void*)vf_amnf_kernel<WIN, 0, EXACT>
                        : (var == MINIMAX ? (const void*)vf_amnf_kernel<WIN, 0, MINIMAX>
                                          : (const void*)vf_amnf_kernel<WIN, 0, POLY4>);
  if (crit == AMNFG)
    return var == EXACT ? (const void*)vf_amnf_kernel<WIN, 1, EXACT>
                        : (var == MINIMAX ? (const void*)vf_amnf_kernel<WIN, 1, MINIMAX>
                                          : (const void*)vf_amnf_kernel<WIN, 1, POLY4>);
  if (crit == EVMF) return var == EXACT ? (const void*)vf_evmf_kernel<WIN, EXACT> : (const void*)vf_evmf_kernel<WIN, MINIMAX>;
  if (crit == ANGULAR)
    return var == EXACT ? (const void*)vf_angular_window_kernel<WIN, EXACT>
                        : (const void*)vf_angular_window_kernel<WIN, MINIMAX>;
  return nullptr;   // exp/log: el_kernel
}

int validate(int B, int H, int W, int window, int crit, int var) {
  if (window < 3 || window % 2 == 0) return fail(VF_EINVAL, "window must be odd and >= 3 (got %lld)", window);
  if (B < 1) return fail(VF_EINVAL, "batch must be >= 1 (got %lld)", B);
  if (H < 1 || W < 1) return fail(VF_EINVAL, "image size must be positive");
  if (window > H || window > W) return fail(VF_EINVAL, "window larger than the image (S:64)");
  if (crit < 0 || crit > 5) return fail(VF_EINVAL, "criterion out of range (%lld)", crit);
  if (var < 0 || var > 3) return fail(VF_EINVAL, "variant out of range (%lld)", var);
  if (var == VF_MINIMAX_POLY4 && crit != VF_EXP && crit != VF_AMNFE && crit != VF_AMNFG)
    return fail(VF_EINVAL, "VF_MINIMAX_POLY4 is only defined for the EXP-based filters");
  if (var == VF_MINIMAX_REACH && crit != VF_EXP && crit != VF_LOG)
    return fail(VF_EINVAL, "VF_MINIMAX_REACH is only defined for the exp and log criteria");
  if (window > 5) return fail(VF_EUNSUPPORTED, "window %lld is valid but not compiled (3 and 5 are)", window);
  return VF_OK;
}

float kscale(int crit, int window) {
  const double n = (double)window * window;
  if (crit == VF_EXP) return (float)(std::pow(n, 1.0 + vf::coef::KAPPA / 3.0) / 2.0);  // c_E * S1
  if (crit == VF_LOG) return (float)(vf::coef::ONE_MINUS_INV_E * (n - 1.0));          // c_L * S1
  if (crit == VF_AMNFE || crit == VF_AMNFG) return (float)std::pow(n, -vf::coef::KAPPA / 3.0);  // h_i / row sum
  return 0.0f;
}

int describe(KernelDesc* kd, const uint8_t* in, long long in_stride, int band_row0, int band_rows, int B, int H, int W,
             int out_row0, int out_rows, int window, int crit, int var, int algo, uint8_t* out, long long out_stride,
             uint8_t* index, float* agg) {
  Launch& L = kd->L;
  L.in = in; L.out = out; L.idx = index; L.agg = agg;
  L.in_stride = in_stride; L.out_stride = out_stride;
  L.H = H; L.W = W; L.band_row0 = band_row0; L.band_rows = band_rows;
  L.out_row0 = out_row0; L.out_rows = out_rows;
  L.kscale = kscale(crit, window);
  const int tile = (algo >> 2) & 3;   // 0 = by size; 1..3 = forced rows per thread (tuning / tests)
  const bool no_tma = (algo & VF_ALGO_NO_TMA) != 0;
  const bool want_stream = (algo & VF_ALGO_STREAM) != 0;
  algo &= 3;
  // 3x3 angular (minimax and exact): the warp-streamed role-sum kernel
  // (vf_stream.cuh) is the default for large launches; VF_ANG3_STREAM=0
  // (both variants) or VF_ANG3_STREAM_EXACT=0 (exact only) fall back to the
  // block pair-sharing kernel, VF_ANG3_STREAM=1 forces the streamed one at any
  // size (tests) (C4 256 images: exact 2471 vs 2674 us, minimax 1467 vs 1849 us)
  static const bool env_no_stream = [] { const char* e = std::getenv("VF_ANG3_STREAM"); return e && e[0] == '0'; }();
  static const bool env_no_stream_ex = [] { const char* e = std::getenv("VF_ANG3_STREAM_EXACT"); return e && e[0] == '0'; }();
  // Small launches (less than one wave of 64-row warps, e.g. one 512x512
  // image) keep the block kernel: a warp-streamed strip needs long columns
  // of work (C2: stream exact 35 us vs 15 us)
  const long long strips = (W + vf::stream::SOUT - 1) / vf::stream::SOUT;
  static const bool env_force_stream = [] { const char* e = std::getenv("VF_ANG3_STREAM"); return e && e[0] == '1'; }();
  // (the minimax streamed kernel is also the faster one for small launches:
  // C2 11.4 vs 12.5 us; VF_ANG3_SMALL_SHARED=1 restores the block kernel there)
  static const bool env_small_shared = [] { const char* e = std::getenv("VF_ANG3_SMALL_SHARED"); return e && e[0] == '1'; }();
  const bool stream_big = env_force_stream || strips * out_rows * (long long)B >= 148LL * 20 * 64;
  if (crit == VF_ANGULAR && window == 3 && (var == VF_MINIMAX || var == VF_EXACT) &&
      (want_stream || (algo == VF_ALGO_AUTO && (stream_big || (var == VF_MINIMAX && !env_small_shared)) &&
                       !env_no_stream && !(var == VF_EXACT && env_no_stream_ex)))) {
    static const int k_env = [] { const char* e = std::getenv("VF_STREAM_K"); return e ? std::atoi(e) : 0; }();
    const int K = (k_env >= 2 && k_env <= 1024) ? k_env : vf::stream_rows_per_warp(strips * out_rows * (long long)B);
    // the last strip of each image on half a warp when it has <= 30 output
    // columns (vf_stream.cuh; C4 3x3 minimax 1.50 -> 1.45 ms per 256 images);
    // VF_STREAM_HALF=0 keeps full-warp strips everywhere
    static const bool env_no_half = [] { const char* e = std::getenv("VF_STREAM_HALF"); return e && e[0] == '0'; }();
    const bool split = !env_no_half && B >= 2 && vf::stream::half_tail(W);
    kd->fn = var == VF_EXACT ? vf::stream_kernel_fn_ex() : vf::stream_kernel_fn_mm();
    kd->grid = vf::stream_grid(L, B, K, split, false);
    kd->block = dim3(vf::stream_block_threads());
    kd->smem = vf::stream_smem_bytes();
    kd->stream_k = K;
    kd->stream_b = B;
    kd->L2 = L;
    if (split) {
      kd->fn_tail = var == VF_EXACT ? vf::stream_kernel_fn_ex(true) : vf::stream_kernel_fn_mm(true);
      kd->grid_tail = vf::stream_grid(L, B, K, true, true);
      kd->smem_tail = vf::stream_smem_bytes(true);
    }
    if (kd->grid.y > 65535 || kd->grid.z > 65535) return fail(VF_EINVAL, "grid too large");
    return VF_OK;
  }
  if (crit == VF_ANGULAR && algo != VF_ALGO_WINDOW) {
    // launch configuration (vf_shared.cuh: 1..3 = 256 threads x 1..3 region
    // pixels, 4 = 384 threads x 2 in a 32 x 24 region): 4 measured fastest
    // for the 3x3 sharing kernel (40 registers, 48 warps per SM: C2 -7%, C4
    // -1.5% vs 256 x 3) and for the 5x5 role-sum kernel (C3 -15%;
    // tools/tune_tiles.sh).  VF_SHARED_PPT=1..4 or the algo tile bits (1..3)
    // override, for tuning and tests.
    static const int ppt_env = [] { const char* e = std::getenv("VF_SHARED_PPT"); return e ? std::atoi(e) : 0; }();
    int ppt = (ppt_env >= 1 && ppt_env <= 4) ? ppt_env : 4;
    if (tile) ppt = tile;
    // per-pixel role sums (vf_role.cuh): the 5x5 default (C3 -33% vs the
    // per-window accumulation); at 3x3 only on request (VF_ALGO_ROLE): there
    // the 36-pair accumulation is cheaper than the extra barriers and row
    // sums (C4 angular minimax 151 vs 133 us)
    if (algo == VF_ALGO_ROLE || (window == 5 && algo != VF_ALGO_SHARED)) {
      kd->fn = vf::role_kernel_fn(window, var, ppt);
      kd->grid = vf::shared_grid(L, B, window, ppt);
      kd->block = dim3(vf::shared::cfg_nt(ppt));
      kd->smem = vf::role_smem_bytes(window, ppt);
      const cudaError_t e = ensure_attributes();
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
      return VF_OK;
    }
    kd->fn = vf::shared_kernel_fn(window, var, ppt);
    kd->grid = vf::shared_grid(L, B, window, ppt);
    kd->block = dim3(vf::shared::cfg_nt(ppt));
    kd->smem = vf::shared_smem_bytes(window, ppt);
    const cudaError_t e = ensure_attributes();
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  } else {
    int th = vf::TY;
    if (crit == VF_EXP || crit == VF_LOG) {
      // 3x3: several output rows per thread for large launches (staging and
      // the S1 row sums are shared by the stacked windows; the libm variants
      // 2, the others 4 -- below), 1 for small ones (more blocks); 5x5: 1.
      // VF_EL_OPT=1|2|4 or the algo tile bits (1, 2, 3 -> 1, 2, 4) override.
      // Large 3x3 launches of the non-libm variants: 4 rows per thread in
      // 4-warp blocks (32 x 16 outputs; C4: poly4 94.5 -> 92.6 us, exp reach
      // 101.9 -> 98.6 us, exp/log minimax 125.7 -> 124.4 us vs 8-warp blocks
      // with 4 / 2 rows); VF_EL_TY=8 restores the 8-warp blocks.
      const long long npix = (long long)B * out_rows * W;
      const bool big3 = window == 3 && npix >= (1LL << 21);
      // (the libm variants too: 4 rows in 8-warp blocks -- C4 256 images
      // exp + log exact 8.57 ms with 2 rows, 8.53 ms with 4; with the
      // VF_EXACT_LIBM=1 build 2.30 -> 2.24 and 4.11 -> 4.09 ms)
      int opt = big3 ? 4 : 1;
      int nty = (big3 && var != VF_EXACT) ? 4 : vf::TY;
      static const int opt_env = [] { const char* e = std::getenv("VF_EL_OPT"); return e ? std::atoi(e) : 0; }();
      if (window == 3 && (opt_env == 1 || opt_env == 2 || opt_env == 4)) opt = opt_env;
      if (window == 3 && tile) opt = tile == 3 ? 4 : tile;
      kd->fn = window == 3 ? (opt == 4 ? el_kernel<3, 4>(crit, var)
                                       : (opt == 2 ? el_kernel<3, 2>(crit, var) : el_kernel<3, 1>(crit, var)))
                           : el_kernel<5, 1>(crit, var);
      // persistent TMA-staged kernel when the rows are 16-byte aligned
      static const bool env_no_tma = [] { const char* e = std::getenv("VF_NO_TMA"); return e && e[0] == '1'; }();
      const unsigned long long row_bytes = (unsigned long long)W * 3;
      PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
      // (measured on C3/C4: with the scalar pair loop it was a few % faster for
      // the 3x3 polynomial variants; since the packed-FP32 pair loop the
      // plain-load kernel with 2 rows per thread is faster everywhere -- C4
      // exp minimax 131 vs 143 us -- because the persistent loop costs
      // registers and occupancy.  It stays available, bit-identical, through
      // the algo tile bits or VF_FORCE_TMA=1, and is tested that way.)
      const bool tma_pays = false;
      static const bool env_force_tma = [] { const char* e = std::getenv("VF_FORCE_TMA"); return e && e[0] == '1'; }();
      if ((tma_pays || env_force_tma || tile) && !no_tma && !env_no_tma && enc && row_bytes % 16 == 0 && ((uintptr_t)in % 16) == 0 &&
          (B == 1 || in_stride % 16 == 0) && row_bytes < (1ULL << 32)) {
        const int tye = vf::TY * opt;
        const cuuint64_t dims[3] = {row_bytes, (cuuint64_t)band_rows, (cuuint64_t)B};
        const cuuint64_t strides[2] = {row_bytes, (cuuint64_t)(B == 1 ? row_bytes * band_rows : in_stride)};
        const cuuint32_t box[3] = {(cuuint32_t)vf::tma::BOXW, (cuuint32_t)(tye + 2 * (window / 2)), 1u};
        const cuuint32_t estr[3] = {1u, 1u, 1u};
        CUresult cr = enc(&kd->map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)in, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr == CUDA_SUCCESS) {
          kd->tma = true;
          kd->fn = window == 3 ? (opt == 4 ? el_tma_kernel<3, 4>(crit, var)
                                           : (opt == 2 ? el_tma_kernel<3, 2>(crit, var) : el_tma_kernel<3, 1>(crit, var)))
                               : el_tma_kernel<5, 1>(crit, var);
          kd->tiles_x = (W + vf::TX - 1) / vf::TX;
          kd->tiles_y = (out_rows + tye - 1) / tye;
          const long long nt = (long long)B * kd->tiles_x * kd->tiles_y;
          if (nt > (1LL << 30)) return fail(VF_EINVAL, "too many tiles (%lld)", nt);
          kd->ntiles = (int)nt;
          const int cap = persistent_blocks(kd->fn, vf::TX * vf::TY, 0);
          kd->grid = dim3(kd->ntiles < cap ? kd->ntiles : cap);
          kd->block = dim3(vf::TX, vf::TY);
          kd->smem = 0;
          return VF_OK;
        }
      }
      th = vf::TY * opt;
      static const int ty_env = [] { const char* e = std::getenv("VF_EL_TY"); return e ? std::atoi(e) : 0; }();
      if (window == 3 && (ty_env == 4 || ty_env == vf::TY)) nty = ty_env;
      if (window == 3 && nty == 4 && opt >= 2 && var != VF_EXACT) {
        kd->fn = vf::el_kernel_ty4(opt, crit, var);
        if (!kd->fn) return fail(VF_EINVAL, "no 4-warp kernel for this variant");
        th = 4 * opt;
        kd->grid = dim3((W + vf::TX - 1) / vf::TX, (out_rows + th - 1) / th, B);
        kd->block = dim3(vf::TX, 4);
        kd->smem = 0;
        if (kd->grid.y > 65535 || kd->grid.z > 65535)
          return fail(VF_EINVAL, "grid too large (%lld blocks in y or z)",
                      (long long)(kd->grid.y > kd->grid.z ? kd->grid.y : kd->grid.z));
        return VF_OK;
      }
    } else {
      kd->fn = window == 3 ? window_kernel<3>(crit, var) : window_kernel<5>(crit, var);
    }
    kd->grid = dim3((W + vf::TX - 1) / vf::TX, (out_rows + th - 1) / th, B);
    kd->block = dim3(vf::TX, vf::TY);
    kd->smem = 0;
  }
  if (kd->grid.y > 65535 || kd->grid.z > 65535)
    return fail(VF_EINVAL, "grid too large (%lld blocks in y or z)",
                (long long)(kd->grid.y > kd->grid.z ? kd->grid.y : kd->grid.z));
  return VF_OK;
}

int launch_desc(KernelDesc& kd, cudaStream_t st) {
  cudaError_t e = cudaLaunchKernel(kd.fn, kd.grid, kd.block, kd.params(), kd.smem, st);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  if (kd.fn_tail) {
    e = cudaLaunchKernel(kd.fn_tail, kd.grid_tail, kd.block, kd.params(), kd.smem_tail, st);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch (remainder strips)");
  }
  return VF_OK;
}

// The kernel node(s) of a description (the remainder-strip launch as a second,
// independent node), each depending on deps[0..ndeps); returns the count.
int add_kernel_nodes(cudaGraph_t g, KernelDesc& kd, const cudaGraphNode_t* deps, int ndeps, cudaGraphNode_t* nodes,
                     const char* what) {
  cudaKernelNodeParams kp = {};
  kp.func = (void*)kd.fn;
  kp.gridDim = kd.grid;
  kp.blockDim = kd.block;
  kp.sharedMemBytes = (unsigned)kd.smem;
  kp.kernelParams = kd.params();
  cudaError_t e = cudaGraphAddKernelNode(&nodes[0], g, deps, ndeps, &kp);
  if (e != cudaSuccess) return -cuda_fail(e, what);
  if (!kd.fn_tail) return 1;
  kp.func = (void*)kd.fn_tail;
  kp.gridDim = kd.grid_tail;
  kp.sharedMemBytes = (unsigned)kd.smem_tail;
  e = cudaGraphAddKernelNode(&nodes[1], g, deps, ndeps, &kp);
  if (e != cudaSuccess) return -cuda_fail(e, what);
  return 2;
}

// The sRGB decoding table (IEC 61966-2-1: c/255 linearised), computed in
// double on the host and rounded to float once, in device memory of every
// device that runs statistics (allocated on first use, kept for the
// process).  Every statistics pass (standalone or a plan's node) reads the same
// table, so their per-pixel CIELAB values are the same bits.
const float* srgb_table(int* rc) {
  static std::mutex mu;
  static float* tabs[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev < 0 || dev >= 64) { *rc = cuda_fail(e == cudaSuccess ? cudaErrorInvalidDevice : e, "cudaGetDevice"); return nullptr; }
  std::lock_guard<std::mutex> lk(mu);
  if (!tabs[dev]) {
    float h[256];
    for (int c = 0; c < 256; ++c) {
      const double v = c / 255.0;
      h[c] = (float)(v <= 0.04045 ? v / 12.92 : std::pow((v + 0.055) / 1.055, 2.4));
    }
    float* d = nullptr;
    e = cudaMalloc(&d, sizeof(h));
    if (e == cudaSuccess) e = cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { if (d) cudaFree(d); *rc = cuda_fail(e, "sRGB table"); return nullptr; }
    tabs[dev] = d;
  }
  *rc = VF_OK;
  return tabs[dev];
}

// The statistics pass (vf_stats_multi_kernel) for a reference a and nb <= 8
// outputs: kernel, grid and the PX = 4 decision, shared by
// vf_image_stats_multi and the plans' statistics nodes.
template <int PX>
const void* stats_fn(int nb) {
  switch (nb) {
    case 1: return (const void*)vf::vf_stats_multi_kernel<1, PX>;
    case 2: return (const void*)vf::vf_stats_multi_kernel<2, PX>;
    case 3: return (const void*)vf::vf_stats_multi_kernel<3, PX>;
    case 4: return (const void*)vf::vf_stats_multi_kernel<4, PX>;
    case 5: return (const void*)vf::vf_stats_multi_kernel<5, PX>;
    case 6: return (const void*)vf::vf_stats_multi_kernel<6, PX>;
    case 7: return (const void*)vf::vf_stats_multi_kernel<7, PX>;
    default: return (const void*)vf::vf_stats_multi_kernel<8, PX>;
  }
}
struct StatsLaunch {
  const void* fn;
  dim3 grid;
  // kernel arguments (a, args, npix, B, acc, want_ref_norm)
  const uint8_t* a;
  vf::StatsArgs args;
  long long npix;
  int B;
  unsigned long long* acc;
  int ref;
  void* params[6];
  void** kparams() {
    params[0] = &a; params[1] = &args; params[2] = &npix; params[3] = &B; params[4] = &acc; params[5] = &ref;
    return params;
  }
};
int stats_launch(StatsLaunch* sl, const uint8_t* a, const uint8_t* const* bs, const int* rows, int nb, int B,
                 long long npix, unsigned long long* acc, int want_ref_norm) {
  // four pixels (three aligned words) per iteration when the images allow it
  bool px4 = npix % 4 == 0 && ((uintptr_t)a % 4) == 0;
  for (int k = 0; k < nb; ++k) px4 = px4 && ((uintptr_t)bs[k] % 4) == 0;
  const long long units = px4 ? npix / 4 : npix;
  // ~8 blocks per SM over the batch, and at most 4096 pixels per thread (the
  // per-thread integer sums are 32-bit)
  long long blocks = (units + 255) / 256;
  long long per_image = (148 * 8 + B - 1) / B;
  const long long min_blocks = (npix + 256LL * 4096 - 1) / (256LL * 4096);
  if (per_image < min_blocks) per_image = min_blocks;
  if (blocks > per_image) blocks = per_image;
  if (blocks > 2147483647LL) return fail(VF_EINVAL, "image too large (%lld pixels)", npix);
  if (B > 65535) return fail(VF_EINVAL, "too many images for the statistics grid (%lld)", B);
  int trc = VF_OK;
  const float* tab = srgb_table(&trc);
  if (!tab) return trc;
  sl->fn = px4 ? stats_fn<4>(nb) : stats_fn<1>(nb);
  sl->grid = dim3((unsigned)blocks, B);
  sl->a = a;
  sl->args = vf::StatsArgs{};
  for (int k = 0; k < nb; ++k) { sl->args.b[k] = bs[k]; sl->args.row[k] = rows[k]; }
  sl->args.lin = tab;
  sl->npix = npix;
  sl->B = B;
  sl->acc = acc;
  sl->ref = want_ref_norm;
  return VF_OK;
}

int launch(const uint8_t* in, long long in_stride, int band_row0, int band_rows, int B, int H, int W, int out_row0,
           int out_rows, int window, int crit, int var, int algo, uint8_t* out, long long out_stride, uint8_t* index,
           float* agg, cudaStream_t st) {
  KernelDesc kd;
  int rc = describe(&kd, in, in_stride, band_row0, band_rows, B, H, W, out_row0, out_rows, window, crit, var, algo,
                    out, out_stride, index, agg);
  if (rc) return rc;
  return launch_desc(kd, st);
}

}  // namespace

// ---- plan: an instantiated CUDA graph ---------------------------------------------
struct vf_plan_s {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int nkernels = 0;
};

// NVTX range over one C-ABI call (header-only NVTX v3: a no-op unless a
// profiler injects itself, e.g. ncu --nvtx / nsys), so host-side timelines
// show which entry point issued which kernels.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

extern "C" {

int vf_filter_batch_algo(const uint8_t* imgs, int B, int H, int W, int window, int criterion, int variant, int algo,
                         uint8_t* outs, uint8_t* index, float* aggregates, void* stream) {
  NvtxRange nvtx_("vf_filter_batch_algo");
  g_err[0] = 0;
  int rc = validate(B, H, W, window, criterion, variant);
  if (rc) return rc;
  if (!imgs || !outs) return fail(VF_EINVAL, "NULL image or output pointer");
  if (algo < 0 || algo > 63) return fail(VF_EINVAL, "algo out of range (%lld)", algo);
  const size_t bytes = (size_t)B * H * W * 3;
  if (overlap(imgs, bytes, outs, bytes)) return fail(VF_EINVAL, "input and output overlap");
  const long long stride = (long long)H * W * 3;
  return launch(imgs, stride, 0, H, B, H, W, 0, H, window, criterion, variant, algo, outs, stride, index, aggregates,
                (cudaStream_t)stream);
}

int vf_filter_batch(const uint8_t* imgs, int B, int H, int W, int window, int criterion, int variant, uint8_t* outs,
                    uint8_t* index, float* aggregates, void* stream) {
  return vf_filter_batch_algo(imgs, B, H, W, window, criterion, variant, VF_ALGO_AUTO, outs, index, aggregates,
                              stream);
}

int vf_filter(const uint8_t* img, int H, int W, int window, int criterion, int variant, uint8_t* out, uint8_t* index,
              float* aggregates, void* stream) {
  return vf_filter_batch_algo(img, 1, H, W, window, criterion, variant, VF_ALGO_AUTO, out, index, aggregates,
                              stream);
}

int vf_filter_rows(const uint8_t* band, int band_row0, int band_rows, int H, int W, int out_row0, int out_rows,
                   int window, int criterion, int variant, uint8_t* out, uint8_t* index, float* aggregates,
                   void* stream) {
  NvtxRange nvtx_("vf_filter_rows");
  g_err[0] = 0;
  int rc = validate(1, H, W, window, criterion, variant);
  if (rc) return rc;
  if (!band || !out) return fail(VF_EINVAL, "NULL band or output pointer");
  if (out_rows < 1 || out_row0 < 0 || out_row0 + out_rows > H) return fail(VF_EINVAL, "output rows outside the image");
  const int r = window / 2;
  const int need_lo = out_row0 - r < 0 ? 0 : out_row0 - r;
  const int need_hi = out_row0 + out_rows + r > H ? H : out_row0 + out_rows + r;
  if (band_rows < 1 || band_row0 < 0 || band_row0 > need_lo || band_row0 + band_rows < need_hi ||
      band_row0 + band_rows > H)
    return fail(VF_EINVAL, "row band does not cover the rows the stripe reads");
  if (overlap(band, (size_t)band_rows * W * 3, out, (size_t)out_rows * W * 3))
    return fail(VF_EINVAL, "input and output overlap");
  return launch(band, 0, band_row0, band_rows, 1, H, W, out_row0, out_rows, window, criterion, variant, VF_ALGO_AUTO,
                out, 0, index, aggregates, (cudaStream_t)stream);
}

size_t vf_host_workspace_bytes(int B, int H, int W) {
  if (B < 1 || H < 1 || W < 1) return 0;
  const size_t img = (size_t)B * H * W * 3;
  return 2 * ((img + 255) / 256 * 256);
}

int vf_filter_host(const uint8_t* h_imgs, int B, int H, int W, int window, int criterion, int variant, uint8_t* h_outs,
                   void* d_workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("vf_filter_host");
  g_err[0] = 0;
  int rc = validate(B, H, W, window, criterion, variant);
  if (rc) return rc;
  if (!h_imgs || !h_outs || !d_workspace) return fail(VF_EINVAL, "NULL pointer");
  const size_t need = vf_host_workspace_bytes(B, H, W);
  if (workspace_bytes < need) return fail(VF_EINVAL, "workspace too small (need %lld bytes)", (long long)need);
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

int vf_kernel_info(int B, int H, int W, int window, int criterion, int variant, int algo, char* name, int name_cap,
                   long long* launch) {
  g_err[0] = 0;
  int rc = validate(B, H, W, window, criterion, variant);
  if (rc) return rc;
  if (algo < 0 || algo > 63) return fail(VF_EINVAL, "algo out of range (%lld)", algo);
  // a dummy, 16-byte aligned input address: describe() only inspects alignment
  const uint8_t* fake = reinterpret_cast<const uint8_t*>(uintptr_t(1) << 20);
  const long long stride = (long long)H * W * 3;
  KernelDesc kd;
  rc = describe(&kd, fake, stride, 0, H, B, H, W, 0, H, window, criterion, variant, algo, (uint8_t*)fake + 1,
                stride, nullptr, nullptr);
  if (rc) return rc;
  if (name && name_cap > 0) {
    const char* nm = nullptr;
    cudaError_t e = cudaFuncGetName(&nm, kd.fn);
    if (e != cudaSuccess || !nm) return cuda_fail(e == cudaSuccess ? cudaErrorInvalidDeviceFunction : e, "cudaFuncGetName");
    std::snprintf(name, (size_t)name_cap, "%s", nm);
  }
  if (launch) {
    launch[0] = kd.grid.x; launch[1] = kd.grid.y; launch[2] = kd.grid.z;
    launch[3] = kd.block.x; launch[4] = kd.block.y; launch[5] = kd.block.z;
    launch[6] = (long long)kd.smem;
  }
  return VF_OK;
}

int vf_plan_create(vf_plan* plan, int B, int H, int W, int window, int n, const int* criteria, const int* variants,
                   const uint8_t* d_in, uint8_t* const* d_outs, const uint8_t* h_in, uint8_t* const* h_outs) {
  return vf_plan_create_ex(plan, B, H, W, window, n, criteria, variants, d_in, d_outs, h_in, h_outs, nullptr,
                           nullptr);
}

int vf_plan_create_ex(vf_plan* plan, int B, int H, int W, int window, int n, const int* criteria, const int* variants,
                      const uint8_t* d_in, uint8_t* const* d_outs, const uint8_t* h_in, uint8_t* const* h_outs,
                      const int* refs, double* d_stats) {
  NvtxRange nvtx_("vf_plan_create_ex");
  g_err[0] = 0;
  if (!plan) return fail(VF_EINVAL, "NULL plan pointer");
  *plan = nullptr;
  if (n < 1 || n > 64) return fail(VF_EINVAL, "number of filters must be in [1, 64] (got %lld)", n);
  if (!criteria || !variants || !d_in || !d_outs) return fail(VF_EINVAL, "NULL argument");
  const size_t bytes = (size_t)B * H * W * 3;
  for (int i = 0; i < n; ++i) {
    int rc = validate(B, H, W, window, criteria[i], variants[i]);
    if (rc) return rc;
    if (!d_outs[i]) return fail(VF_EINVAL, "NULL output %lld", i);
    if (overlap(d_in, bytes, d_outs[i], bytes)) return fail(VF_EINVAL, "input and output %lld overlap", i);
    for (int j = 0; j < i; ++j)
      if (overlap(d_outs[j], bytes, d_outs[i], bytes)) return fail(VF_EINVAL, "outputs %lld overlap", i);
    if (h_outs && !h_outs[i]) return fail(VF_EINVAL, "NULL host output %lld", i);
  }
  // fidelity comparisons: filter i against filter refs[i] (row cmp_of[i] of d_stats)
  int cmp_of[64], ncmp = 0;
  for (int i = 0; i < n; ++i) {
    cmp_of[i] = -1;
    if (!refs || refs[i] == -1) continue;
    if (refs[i] < 0 || refs[i] >= n || refs[i] == i)
      return fail(VF_EINVAL, "refs[%lld] must be -1 or another filter's index", i);
    cmp_of[i] = ncmp++;
  }
  if (ncmp > 0 && !d_stats) return fail(VF_EINVAL, "NULL statistics buffer");
  if (ncmp > 0 && B > 65535) return fail(VF_EINVAL, "too many images for the statistics grid (%lld)", B);
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(d_stats);
  const size_t nstat = (size_t)8 * B * ncmp;
  if (ncmp > 0 && overlap((const uint8_t*)d_stats, nstat * 8, d_in, bytes))
    return fail(VF_EINVAL, "statistics buffer overlaps the input");
  for (int i = 0; i < n && ncmp > 0; ++i)
    if (overlap((const uint8_t*)d_stats, nstat * 8, d_outs[i], bytes))
      return fail(VF_EINVAL, "statistics buffer overlaps output %lld", i);

  vf_plan_s* p = new (std::nothrow) vf_plan_s();
  if (!p) return fail(VF_ECUDA, "out of host memory");
  cudaError_t e = cudaGraphCreate(&p->graph, 0);
  if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaGraphCreate"); }
  auto bail = [&](int rc) { cudaGraphDestroy(p->graph); delete p; return rc; };
  // roots: the H2D copy of the input and the zeroing of the statistics accumulators
  cudaGraphNode_t roots[2];
  int nroots = 0;
  if (h_in) {
    e = cudaGraphAddMemcpyNode1D(&roots[nroots], p->graph, nullptr, 0, (void*)d_in, h_in, bytes,
                                 cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaGraphAddMemcpyNode1D (H2D)"));
    ++nroots;
  }
  if (ncmp > 0) {
    cudaMemsetParams mp = {};
    mp.dst = d_stats;
    mp.value = 0;
    mp.elementSize = 4;
    mp.width = nstat * 2;
    mp.height = 1;
    mp.pitch = nstat * 8;
    e = cudaGraphAddMemsetNode(&roots[nroots], p->graph, nullptr, 0, &mp);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaGraphAddMemsetNode (statistics)"));
    ++nroots;
  }
  std::vector<cudaGraphNode_t> prod[64];   // the kernel node(s) writing filter i
  std::vector<cudaGraphNode_t> stat_nodes; // nodes adding to the statistics accumulators
  auto add_d2h = [&](const cudaGraphNode_t* kn, int nk, int i) -> int {
    if (!h_outs) return VF_OK;
    cudaGraphNode_t d2h;
    cudaError_t e2 = cudaGraphAddMemcpyNode1D(&d2h, p->graph, kn, nk, h_outs[i], d_outs[i], bytes,
                                              cudaMemcpyDeviceToHost);
    return e2 == cudaSuccess ? VF_OK : cuda_fail(e2, "cudaGraphAddMemcpyNode1D (D2H)");
  };
  const long long stride = (long long)H * W * 3;
  // Plan-level fusion: the exp/log filters share d1 and S1 (readings R2/R3),
  // so two or more of them become ONE kernel node that stages each tile and
  // forms S1 once (vf_fused.cu; outputs bit-identical to the single-filter
  // kernels).  VF_PLAN_FUSE=0 keeps one node per filter.
  static const bool env_no_fuse = [] { const char* e = std::getenv("VF_PLAN_FUSE"); return e && e[0] == '0'; }();
  static const bool env_force_fuse = [] { const char* e = std::getenv("VF_PLAN_FUSE"); return e && e[0] == '2'; }();
  bool fused[64] = {};
  {
    int idx[8], m = 0;
    for (int i = 0; i < n && m < 8; ++i)
      if (criteria[i] == VF_EXP || criteria[i] == VF_LOG) idx[m++] = i;
    // (small inputs keep one node per filter: the graph's concurrency then
    // matters more than the shared staging -- C2: 70 vs 60 us)
    const bool fuse_big = env_force_fuse || (long long)B * H * W >= (1LL << 21);
    if (m >= 2 && !env_no_fuse && window <= 5 && fuse_big) {
      vf::ElFused F = {};
      F.n = m;
      for (int k = 0; k < m; ++k) {
        KernelDesc kd;
        int rc = describe(&kd, d_in, stride, 0, H, B, H, W, 0, H, window, criteria[idx[k]], variants[idx[k]],
                          VF_ALGO_AUTO | VF_ALGO_NO_TMA, d_outs[idx[k]], stride, nullptr, nullptr);
        if (rc) return bail(rc);
        F.L[k] = kd.L;
        F.code[k] = 4 * (criteria[idx[k]] == VF_EXP ? vf::EXPC : vf::LOGC) + variants[idx[k]];
        fused[idx[k]] = true;
      }
      int opt = 1, nty = vf::TY;
      const bool big = window == 3 && (long long)B * H * W >= (1LL << 21);
      cudaKernelNodeParams kp = {};
      kp.func = (void*)vf::el_fused_kernel(window, big, &opt, &nty);
      // the canonical 5-filter set (exp exact / minimax / poly4, log exact /
      // minimax): the pair-major kernel, filters reordered to its layout
      static const bool env_no_pm = [] { const char* e = std::getenv("VF_FUSED5"); return e && e[0] == '0'; }();
      const int canon[5] = {4 * vf::EXPC + vf::EXACT, 4 * vf::EXPC + vf::MINIMAX, 4 * vf::EXPC + vf::POLY4,
                            4 * vf::LOGC + vf::EXACT, 4 * vf::LOGC + vf::MINIMAX};
      if (window == 3 && big && m == 5 && !env_no_pm) {
        vf::ElFused G = {};
        bool ok = true;
        for (int c = 0; c < 5 && ok; ++c) {
          int hit = -1;
          for (int k = 0; k < 5; ++k)
            if (F.code[k] == canon[c]) hit = k;
          if (hit < 0) ok = false;
          else { G.L[c] = F.L[hit]; G.code[c] = canon[c]; }
        }
        if (ok) {
          G.n = 5;
          F = G;
          kp.func = (void*)vf::el_fused5_kernel(&opt, &nty);
        }
      }
      kp.gridDim = dim3((W + vf::TX - 1) / vf::TX, (H + nty * opt - 1) / (nty * opt), B);
      kp.blockDim = dim3(vf::TX, nty);
      kp.sharedMemBytes = 0;
      void* args[1] = {&F};
      kp.kernelParams = args;
      if (kp.gridDim.y > 65535 || kp.gridDim.z > 65535) return bail(fail(VF_EINVAL, "grid too large"));
      cudaGraphNode_t kn;
      e = cudaGraphAddKernelNode(&kn, p->graph, roots, nroots, &kp);
      if (e != cudaSuccess) return bail(cuda_fail(e, "cudaGraphAddKernelNode (fused)"));
      ++p->nkernels;
      for (int k = 0; k < m; ++k) {
        prod[idx[k]].push_back(kn);
        int rc = add_d2h(&kn, 1, idx[k]);
        if (rc) return bail(rc);
      }
    }
  }
  // Plan-level fusion of BVDF minimax and exact (3x3, streamed kernels): one
  // geometry evaluation per pair feeds both variants (vf_stream.cuh, NV = 2).
  // VF_PLAN_FUSE=0 keeps one node per filter.
  {
    int im = -1, ie = -1;
    for (int i = 0; i < n; ++i) {
      if (criteria[i] != VF_ANGULAR || fused[i]) continue;
      if (variants[i] == VF_MINIMAX && im < 0) im = i;
      if (variants[i] == VF_EXACT && ie < 0) ie = i;
    }
    if (im >= 0 && ie >= 0 && window == 3 && !env_no_fuse) {
      KernelDesc km, ke;
      int rc = describe(&km, d_in, stride, 0, H, B, H, W, 0, H, window, VF_ANGULAR, VF_MINIMAX, VF_ALGO_AUTO,
                        d_outs[im], stride, nullptr, nullptr);
      if (rc) return bail(rc);
      rc = describe(&ke, d_in, stride, 0, H, B, H, W, 0, H, window, VF_ANGULAR, VF_EXACT, VF_ALGO_AUTO, d_outs[ie],
                    stride, nullptr, nullptr);
      if (rc) return bail(rc);
      if (km.stream_k && ke.stream_k) {               // both streamed (large launches)
        km.fn = vf::stream_kernel_fn_both();
        if (km.fn_tail) km.fn_tail = vf::stream_kernel_fn_both(true);
        km.L2 = ke.L;
        const int slot[2] = {im, ie};
        cudaGraphNode_t kn[2];
        const int nk = add_kernel_nodes(p->graph, km, roots, nroots, kn, "cudaGraphAddKernelNode (fused angular)");
        if (nk < 0) return bail(-nk);
        p->nkernels += nk;
        fused[im] = fused[ie] = true;
        for (int k = 0; k < 2; ++k) {
          prod[slot[k]].assign(kn, kn + nk);
          rc = add_d2h(kn, nk, slot[k]);
          if (rc) return bail(rc);
        }
      }
    }
  }
  for (int i = 0; i < n; ++i) {
    if (fused[i]) continue;
    KernelDesc kd;
    int rc = describe(&kd, d_in, stride, 0, H, B, H, W, 0, H, window, criteria[i], variants[i], VF_ALGO_AUTO,
                      d_outs[i], stride, nullptr, nullptr);
    if (rc) return bail(rc);
    cudaGraphNode_t kn[2];
    const int nk = add_kernel_nodes(p->graph, kd, roots, nroots, kn, "cudaGraphAddKernelNode");
    if (nk < 0) return bail(-nk);
    p->nkernels += nk;
    prod[i].assign(kn, kn + nk);
    rc = add_d2h(kn, nk, i);
    if (rc) return bail(rc);
  }
  // the fidelity comparisons: one statistics pass per reference (<= 8 outputs
  // each: the reference is read and its CIELAB evaluated once), a graph node
  // after the nodes writing its inputs (so it can overlap other filters'
  // nodes)
  for (int r = 0; r < n && ncmp > 0; ++r) {
    int outs_i[64], no = 0;
    for (int i = 0; i < n; ++i)
      if (cmp_of[i] >= 0 && refs[i] == r) outs_i[no++] = i;
    for (int c0 = 0; c0 < no; c0 += 8) {
      const int nb = no - c0 < 8 ? no - c0 : 8;
      const uint8_t* bs[8];
      int rows[8];
      std::vector<cudaGraphNode_t> deps(prod[r]);
      for (int k = 0; k < nb; ++k) {
        bs[k] = d_outs[outs_i[c0 + k]];
        rows[k] = cmp_of[outs_i[c0 + k]];
        deps.insert(deps.end(), prod[outs_i[c0 + k]].begin(), prod[outs_i[c0 + k]].end());
      }
      deps.insert(deps.end(), roots, roots + nroots);
      std::sort(deps.begin(), deps.end());
      deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
      StatsLaunch sl;
      int rc = stats_launch(&sl, d_outs[r], bs, rows, nb, B, (long long)H * W, acc, 1);
      if (rc) return bail(rc);
      cudaKernelNodeParams kp = {};
      kp.func = (void*)sl.fn;
      kp.gridDim = sl.grid;
      kp.blockDim = dim3(256);
      kp.sharedMemBytes = 0;
      kp.kernelParams = sl.kparams();
      cudaGraphNode_t sn;
      e = cudaGraphAddKernelNode(&sn, p->graph, deps.data(), deps.size(), &kp);
      if (e != cudaSuccess) return bail(cuda_fail(e, "cudaGraphAddKernelNode (statistics)"));
      stat_nodes.push_back(sn);
      ++p->nkernels;
    }
  }
  if (ncmp > 0) {                                   // fixed point -> double, in place
    unsigned long long* accp = acc;
    long long nst = (long long)nstat;
    void* fargs[2] = {&accp, &nst};
    cudaKernelNodeParams kp = {};
    kp.func = (void*)vf::vf_stats_finalize;
    kp.gridDim = dim3((unsigned)((nstat + 255) / 256));
    kp.blockDim = dim3(256);
    kp.kernelParams = fargs;
    cudaGraphNode_t fn;
    e = cudaGraphAddKernelNode(&fn, p->graph, stat_nodes.data(), stat_nodes.size(), &kp);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaGraphAddKernelNode (statistics finalize)"));
    ++p->nkernels;
  }
  e = cudaGraphInstantiate(&p->exec, p->graph, 0);
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaGraphInstantiate"));
  *plan = p;
  return VF_OK;
}

int vf_plan_launch(vf_plan plan, void* stream) {
  NvtxRange nvtx_("vf_plan_launch");
  g_err[0] = 0;
  if (!plan || !plan->exec) return fail(VF_EINVAL, "invalid plan");
  cudaError_t e = cudaGraphLaunch(plan->exec, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
  return VF_OK;
}

int vf_plan_kernels(vf_plan plan) {
  g_err[0] = 0;
  if (!plan || !plan->exec) return fail(VF_EINVAL, "invalid plan");
  return plan->nkernels;
}

int vf_plan_destroy(vf_plan plan) {
  g_err[0] = 0;
  if (!plan) return VF_OK;
  if (plan->exec) cudaGraphExecDestroy(plan->exec);
  if (plan->graph) cudaGraphDestroy(plan->graph);
  delete plan;
  return VF_OK;
}

int vf_image_stats(const uint8_t* a, const uint8_t* b, int B, int H, int W, double* stats, void* stream) {
  return vf_image_stats_ex(a, b, B, H, W, stats, 0, stream);
}

int vf_image_stats_ex(const uint8_t* a, const uint8_t* b, int B, int H, int W, double* stats, int flags,
                      void* stream) {
  NvtxRange nvtx_("vf_image_stats_ex");
  return vf_image_stats_multi(a, &b, 1, B, H, W, stats, flags, stream);
}

int vf_image_stats_multi(const uint8_t* a, const uint8_t* const* bs, int nb, int B, int H, int W, double* stats,
                         int flags, void* stream) {
  NvtxRange nvtx_("vf_image_stats_multi");
  g_err[0] = 0;
  if (!a || !bs || !stats) return fail(VF_EINVAL, "NULL pointer");
  if (nb < 1 || nb > 8) return fail(VF_EINVAL, "number of compared outputs must be in [1, 8] (got %lld)", nb);
  for (int k = 0; k < nb; ++k)
    if (!bs[k]) return fail(VF_EINVAL, "NULL output %lld", k);
  if (flags & ~VF_STATS_NO_REF_NORM) return fail(VF_EINVAL, "unknown stats flags (%lld)", flags);
  if (B < 1 || H < 1 || W < 1) return fail(VF_EINVAL, "bad size");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t nstat = (size_t)8 * B * nb;
  cudaError_t e = cudaMemsetAsync(stats, 0, sizeof(double) * nstat, st);
  if (e != cudaSuccess) return cuda_fail(e, "stats memset");
  const long long npix = (long long)H * W;
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(stats);
  const int rows[8] = {0, 1, 2, 3, 4, 5, 6, 7};
  StatsLaunch sl;
  int rc = stats_launch(&sl, a, bs, rows, nb, B, npix, acc, (flags & VF_STATS_NO_REF_NORM) ? 0 : 1);
  if (rc) return rc;
  e = cudaLaunchKernel(sl.fn, sl.grid, dim3(256), sl.kparams(), 0, st);
  if (e != cudaSuccess) return cuda_fail(e, "vf_stats_multi_kernel launch");
  vf::vf_stats_finalize<<<(unsigned)((nstat + 255) / 256), 256, 0, st>>>(acc, (long long)nstat);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "vf_stats_finalize launch");
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

int vf_version(void) { return 105; }

}  // extern "C"
