// vf_tma.cuh -- persistent exp/log kernel fed by TMA (SURVEY.md 8(a) rows
// a1-a8, the B200 staging path).
//
// The input batch is described to the Tensor Memory Accelerator as a 3-D
// uint8 tensor [B][rows][3W] (bytes).  Each block loops over output tiles
// (static stride gridDim.x); once a tile's bytes are repacked, one elected
// thread issues the TMA copy of the NEXT tile's (SH x 3 SW)-byte halo region
// into the freed stage while the block computes the current one, so staging
// costs the SMs no load instructions and its latency is hidden behind the
// pair arithmetic.  Completion is signalled on an mbarrier (expect_tx bytes).
//
// Rows/columns outside the tensor are zero-filled by the TMA unit; replicate
// padding is applied in the repack: border tiles clamp each pixel's
// row/column into the valid part of the box.  A pixel's 3 bytes start at byte
// shift + 3c of its box row; one funnel shift extracts them as a packed RGB0
// word.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "vf_window.cuh"

namespace vf {
namespace tma {

// Box width in bytes.  The TMA unit requires the innermost box coordinate to
// be a multiple of 16 bytes (measured: other offsets fault with an illegal
// instruction), so a tile's box starts at floor16(3 gx0) and its pixels sit
// at byte shift + 3c, shift = 3 gx0 mod 16 < 16: 16 + 3 (32 + 2r) <= 128.
constexpr int BOXW = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 3-D tile load global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}

// Packed RGB0 word of the pixel whose 3 bytes start at byte `o` of a
// word-aligned shared-memory row.
__device__ __forceinline__ uint32_t pixel_at(const uint32_t* row, int o) {
  return __funnelshift_r(row[o >> 2], row[(o >> 2) + 1], (o & 3) * 8) & 0x00ffffffu;
}

template <int SH>
struct Smem {
  alignas(128) uint8_t raw[SH * BOXW];   // TMA stage (refilled while the previous tile computes)
  alignas(8) uint64_t bar;
};

}  // namespace tma

// Persistent exp/log kernel: tiles of TX x (TY * OPT) outputs, tile t ->
// (image, tile row, tile column) in raster order.  Per tile: wait for the
// TMA stage, repack it into RGB0 words (replicate clamping folded into the
// source index), barrier, let the leader start the next tile's TMA into the
// freed stage, compute (el_compute_tile, shared with the plain-load kernel),
// barrier.
// Resident blocks per SM the register allocation is held to (the persistent
// loop otherwise keeps loop-invariant values in registers at the cost of
// occupancy): 5 (<= 48 registers) for the 3x3 polynomial variants with 1-2
// rows per thread, 4 with 4 rows, 3 (<= 80) for the libm variants and 5x5.
#ifndef VF_TMA_MINB_OPT4
#define VF_TMA_MINB_OPT4 4   // tuning knob (tools/dev experiments)
#endif
template <int WIN, int VAR, int OPT>
constexpr int el_tma_min_blocks() { return (WIN == 3 && VAR != EXACT) ? (OPT <= 2 ? 5 : VF_TMA_MINB_OPT4) : 3; }

template <int WIN, int CRIT, int VAR, int OPT>
__global__ void __launch_bounds__(TX * TY, el_tma_min_blocks<WIN, VAR, OPT>()) vf_el_tma_kernel(const __grid_constant__ CUtensorMap map, const Launch L,
                                                             int tiles_x, int tiles_y, int ntiles) {
  using namespace tma;
  constexpr int R = WIN / 2;
  constexpr int TYE = TY * OPT;                // output tile height
  constexpr int SW = TX + 2 * R;               // staged columns
  constexpr int SH = TYE + 2 * R;              // staged rows
  constexpr int RWD = BOXW / 4;                // words per staged row
  constexpr uint32_t BYTES = SH * BOXW;
  static_assert(15 + 3 * SW + 1 <= BOXW, "box too narrow");
  __shared__ Smem<SH> sm;
  __shared__ uint32_t s_pk[SH * SW];

  const int tid = threadIdx.y * TX + threadIdx.x;
  const bool leader = tid == 0;
  const int per_img = tiles_x * tiles_y;
  const int out_row0 = L.out_row0, band_row0 = L.band_row0, band_rows = L.band_rows, W = L.W;
  // leader only: TMA of tile t's halo region (no lambda: capturing the Launch
  // parameter by reference would copy it to local memory)
#define VF_TMA_ISSUE(t_)                                                                                     \
  do {                                                                                                      \
    const int b_ = (t_) / per_img, rem_ = (t_) - b_ * per_img;                                              \
    const int tyi_ = rem_ / tiles_x, txi_ = rem_ - tyi_ * tiles_x;                                          \
    mbar_expect_tx(&sm.bar, BYTES);                                                                         \
    load_3d(sm.raw, &map, &sm.bar, (3 * (txi_ * TX - R)) & ~15, out_row0 + tyi_ * TYE - R - band_row0, b_); \
  } while (0)
  if (leader) {
    prefetch_map(&map);
    mbar_init(&sm.bar, 1);
    fence_mbar_init();
    if ((int)blockIdx.x < ntiles) VF_TMA_ISSUE((int)blockIdx.x);
  }
  __syncthreads();

  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int b = t / per_img, rem = t - b * per_img;
    const int tyi = rem / tiles_x, txi = rem - tyi * tiles_x;
    const int x0 = txi * TX;
    const int y0 = out_row0 + tyi * TYE;
    const int gx0 = x0 - R;                       // global column of box pixel 0
    const int gyb = y0 - R - band_row0;           // band row of box row 0
    const bool border = gx0 < 0 || gx0 + SW > W || gyb < 0 || gyb + SH > band_rows;
    const int shift = (3 * gx0) & 15;             // byte of box pixel 0 within the 16-aligned box

    mbar_wait(&sm.bar, (uint32_t)it & 1u);
    const uint32_t* raw = reinterpret_cast<const uint32_t*>(sm.raw);
    if (!border) {
      for (int p = tid; p < SH * SW; p += TX * TY) {
        const int r = p / SW, c = p - r * SW;
        s_pk[p] = pixel_at(raw + r * RWD, shift + 3 * c);
      }
    } else {   // replicate padding: clamp into the image / band, then into the box
      for (int p = tid; p < SH * SW; p += TX * TY) {
        const int r = p / SW, c = p - r * SW;
        const int rs = clampi(clampi(gyb + r, 0, band_rows - 1) - gyb, 0, SH - 1);
        const int cs = clampi(clampi(gx0 + c, 0, W - 1) - gx0, 0, SW - 1);
        s_pk[p] = pixel_at(raw + rs * RWD, shift + 3 * cs);
      }
    }
    __syncthreads();                              // stage consumed, s_pk ready
    if (leader && t + (int)gridDim.x < ntiles) VF_TMA_ISSUE(t + (int)gridDim.x);   // overlaps the compute below
    el_compute_tile<WIN, CRIT, VAR, OPT>(L, b, x0, y0, s_pk);
    __syncthreads();                              // s_pk free for the next tile
  }
#undef VF_TMA_ISSUE
}

}  // namespace vf
