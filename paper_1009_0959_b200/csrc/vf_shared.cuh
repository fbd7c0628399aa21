// vf_shared.cuh -- angular criterion with cross-window pair sharing
// (SURVEY.md 8(f1)).
//
// The angular distance A(x_p, x_q) of Eq. 5 depends only on the two pixels,
// not on the window, so each image pair within Chebyshev distance 2r = w - 1
// is evaluated ONCE per block and read by every window that contains it:
// 12 (3x3) or 40 (5x5) evaluations per pixel instead of 36 or 300.  The
// aggregates R_i = sum_{j != i} A(x_i, x_j) are then formed per window from the
// stored pair values, exactly as in Eq. 5, so results agree with the
// per-window kernel and the oracle within the parity tolerance.
//
// Block = 256 threads over a 32 x PH region P of input pixels (PH = 8 PPT,
// PPT = 1..3 pixels per thread); the output tile is the interior
// (32-2r) x (PH-2r).
//   stage   P (uint8 HWC, replicate-clamped) -> smem: packed RGB0, |x|^2, |x|
//   phase A for every pair offset delta in the half plane (dy > 0, or dy = 0
//           and dx > 0), |dy|,|dx| <= 2r, and every p in P:
//           M[delta][p] = A(x_p, x_{p+delta}) (minimax: Table 1 ARCSIN row in
//           tau; exact: Eq. 6 with libm asinf).  Pairs that may have cos < 0.5
//           (a conservative test on tau, ~1% of pairs) are flagged
//           and re-evaluated exactly afterwards (exact 4D^2 < P predicate,
//           ARCCOS row / acosf).  Zero vectors are fixed by a
//           block-uniform slow path in the (rare) blocks that contain one.
//   phase C for each output window and each pair i < j of it:
//           v = M[o_j - o_i][c + o_i];  R_i += v;  R_j += v
//   then argmin (lowest index on ties) and store.
// For 5x5 the 40 offsets are processed in 4 groups of 10 so M fits in 30 KB.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>
#include <utility>

#include "vf_window.cuh"

#ifndef SHARED_REC8
#define SHARED_REC8 1        // 8-byte neighbour records (packed RGB0, |x|^2): half the phase-A smem wavefronts, s = sqrt(Ph) by MUFU
#endif
#ifndef SHARED_PX2
#define SHARED_PX2 1         // 3x3, CFG 4: phase A packs a thread's two pixels (not two offsets) per FFMA2 chain
#endif
#ifndef SHARED_ZLAYOUT
#define SHARED_ZLAYOUT 1     // 3x3, 384 x 2 configuration: region rows r and r + 12 interleaved in the pair maps
#endif
#ifndef SHARED_MINB_CFG4
#define SHARED_MINB_CFG4 4   // 384-thread blocks: <= 40 registers, 48 warps per SM (tuning knob)
#endif

namespace vf {

namespace shared {

constexpr int PW = 32;              // region width  (= warp width)
constexpr int PAD = 5 * PW;         // reads past the region stay in bounds
constexpr int NTHR = 256;
// Launch configurations (CFG): 1..3 = 256 threads with CFG region pixels each
// (region 32 x 8 CFG); 4 = 384 threads with 2 pixels each (region 32 x 24).
__host__ __device__ constexpr int cfg_nt(int cfg) { return cfg == 4 ? 384 : 256; }
__host__ __device__ constexpr int cfg_ppt(int cfg) { return cfg == 4 ? 2 : cfg; }
// PPT = region pixels per thread (1..3): region 32 x 8 PPT.  Large images use
// PPT = 3 (least halo overhead), small ones fewer so more blocks fill the GPU.
__host__ __device__ constexpr int region_np(int cfg) { return cfg_nt(cfg) * cfg_ppt(cfg); }
__host__ __device__ constexpr int region_h(int cfg) { return region_np(cfg) / PW; }

__host__ __device__ constexpr int n_delta(int r) { return 4 * r * (2 * r + 1); }
// offset index d -> (dy, dx): d < 2r: (0, d+1); else dy = 1 + (d-2r)/(4r+1), dx = -2r + (d-2r)%(4r+1)
__host__ __device__ constexpr int delta_dy(int r, int d) { return d < 2 * r ? 0 : 1 + (d - 2 * r) / (4 * r + 1); }
__host__ __device__ constexpr int delta_dx(int r, int d) { return d < 2 * r ? d + 1 : -2 * r + (d - 2 * r) % (4 * r + 1); }
__host__ __device__ constexpr int delta_index(int r, int dy, int dx) {
  return dy == 0 ? dx - 1 : 2 * r + (dy - 1) * (4 * r + 1) + (dx + 2 * r);
}

}  // namespace shared

// Pair-map layout.  Default: M[d][p], p = row * 32 + col.  ZL (3x3, CFG 4:
// 384 threads, region rows 0..23, thread tid owns rows tid/32 and tid/32 + 12):
// M[d][2 (p mod 384) + p / 384], i.e. rows r and r + 12 are interleaved, so a
// thread stores its two pixels' values with one STS.64 and reads the values of
// its two output windows (rows ty and ty + 12) with one LDS.64.
// Measured (C4): exact 175.5 -> 171.5 us, minimax 120.8 -> 125.0 us, so the
// interleaved layout is used for the exact variant only.
template <int WIN, int CFG, int VAR>
struct MapLayout {
  static constexpr bool ZL = SHARED_ZLAYOUT && WIN == 3 && CFG == 4 && VAR == EXACT;
  __device__ __forceinline__ static int idx(int p) { return ZL ? ((p % 384) << 1) + p / 384 : p; }
};

// Per-block shared-memory state of the pair-sharing kernel.
// Pixel records.  Default: px[m] per region pixel m.  PX2 (3x3, CFG 4, whose
// threads own pixels p and p + 384): px[j] = (pk(j), pk(j + 384), |x_j|^2,
// |x_{j+384}|^2) for j < 384 + PAD (zero past the region), so one LDS.128 of
// px[p + off] gives the neighbours of BOTH of a thread's pixels for offset
// off as ready register pairs, and one FFMA2 chain evaluates the two pairs.
template <int GD, int CFG>
struct SharedSmem {
  static constexpr int QCAP = 64;                   // rare-pair queue entries per warp
  static constexpr bool PX2 = SHARED_PX2 && CFG == 4 && GD == 12;   // GD 12 <=> 3x3
#if SHARED_REC8
  using Rec = typename std::conditional<PX2, uint4, uint2>::type;   // (packed RGB0, |x|^2 bits): one LDS.64 per neighbour
#else
  using Rec = uint4;   // (packed RGB0, |x|^2 bits, |x| bits, 0): one LDS.128 per neighbour
#endif
  Rec px[(PX2 ? 384 : shared::region_np(CFG)) + shared::PAD];
  float M[GD][shared::region_np(CFG)];
  uint32_t queue[shared::cfg_nt(CFG) / 32][QCAP];   // flagged pairs of one warp: p | dl << 16
  int off[40];                                      // region offset of pair offset d (d < n_delta(r) <= 40)
};

// (packed RGB0, |x|^2 bits) of region pixel m (m < region + PAD: zero past it).
template <int GD, int CFG>
__device__ __forceinline__ uint2 rec_get(const SharedSmem<GD, CFG>& sm, int m) {
  if constexpr (SharedSmem<GD, CFG>::PX2) {
    const uint4 r = sm.px[m < 384 ? m : m - 384];
    return m < 384 ? make_uint2(r.x, r.z) : make_uint2(r.y, r.w);
  } else {
    const auto r = sm.px[m];
    return make_uint2(r.x, r.y);
  }
}

// Exact re-evaluation of a flagged pair (p, p + off) of offset slot dl: the
// exact branch predicate 4D^2 < P; if the pair is on the
// arccos branch (cos < 0.5), its map entry is replaced by the ARCCOS row /
// acosf of cos = D / (|x_p||x_q|).  Zero vectors never get here (tau = 0 is
// never flagged) and are handled by the block-uniform path anyway.
template <int VAR, int WIN, int GD, int CFG>
__device__ __forceinline__ void angular_fix(SharedSmem<GD, CFG>& sm, int p, int dl, int d) {
  const uint2 pv = rec_get(sm, p), qv = rec_get(sm, p + sm.off[d]);
  const float D = __uint_as_float(__dp4a(pv.x, qv.x, F2P23_BITS)) - F2P23;   // exact dot
  const float nna = __uint_as_float(pv.y), nnb = __uint_as_float(qv.y);
  const float Ph = __fmul_rn(nna, nnb);
  const float Pl = fmaf(nna, nnb, -Ph);                     // exact residual
  const float t = fmaf(__fmul_rn(4.0f, D), D, -Ph);         // fl(4D^2 - Ph)
  if (t < Pl) {                                             // 4D^2 < P, exact
    const float c = D * rsqrt_approx(Ph);                   // cos = D / sqrt(|x_p|^2 |x_q|^2)
    sm.M[dl][MapLayout<WIN, CFG, VAR>::idx(p)] = (VAR == EXACT) ? acosf(c) : horner4(coef::ACOS(), c);
  }
}

// One group of GD offsets: phase A (pair maps) + rare fix-ups + phase C.
// G is a template parameter so that every register index stays static.
template <int WIN, int VAR, int GD, int OPT, int CFG, int G>
__device__ __forceinline__ void shared_group(SharedSmem<GD, CFG>& sm, const uint32_t (&my_pk)[shared::cfg_ppt(CFG)],
                                             const float (&my_nn)[shared::cfg_ppt(CFG)],
                                             const float (&my_nrm)[shared::cfg_ppt(CFG)],
                                             float (&Ra)[OPT][WIN * WIN], int tid, bool blk_zero) {
  using namespace shared;
  constexpr int PPT = cfg_ppt(CFG);
  constexpr int NT = cfg_nt(CFG);
  constexpr int NW = NT / 32;
  constexpr int PH = region_h(CFG);
  constexpr int R = WIN / 2;
  constexpr int N = WIN * WIN;
  constexpr int TW = PW - 2 * R;
  constexpr int TH = PH - 2 * R;
  constexpr int QCAP = SharedSmem<GD, CFG>::QCAP;
  const int tx = tid & 31, ty = tid >> 5;
  if (G > 0) __syncthreads();   // previous phase C done with M (G = 0: the staging barrier)
  // ---- phase A: pair maps for offsets [G*GD, G*GD + GD) ------------------------------
  uint32_t flags[PPT];                                      // bit dl: pair (p_k, p_k + delta) flagged
#pragma unroll
  for (int k = 0; k < PPT; ++k) flags[k] = 0u;
  using ML = MapLayout<WIN, CFG, VAR>;
  if constexpr (SharedSmem<GD, CFG>::PX2) {
    // one offset per step, the thread's two pixels in packed FP32
    const f32x2 nn2 = pack2(my_nn[0], my_nn[1]), nnn2 = pack2(-my_nn[0], -my_nn[1]);
#pragma unroll
    for (int dl = 0; dl < GD; ++dl) {
      const int d = G * GD + dl;
      const int j = tid + delta_dy(R, d) * PW + delta_dx(R, d);
      VF_CHECK(j >= 0 && j < 384 + PAD);
      float tau0, tau1, v0, v1;
      angular_tau2_px2<VAR>(my_pk[0], my_pk[1], nn2, nnn2, sm.px[j], tau0, tau1, v0, v1);
      if (tau0 > 0.70641626f) flags[0] |= 1u << dl;           // (1/sqrt2) (1 - 2^-10), see below
      if (tau1 > 0.70641626f) flags[1] |= 1u << dl;
      if constexpr (ML::ZL) {
        *reinterpret_cast<float2*>(&sm.M[dl][2 * tid]) = make_float2(v0, v1);
      } else {
        sm.M[dl][tid] = v0;
        sm.M[dl][tid + NT] = v1;
      }
    }
  } else {
  // two offsets per step in packed FP32 (FFMA2 / FADD2 / FMUL2, GD is even)
#pragma unroll
  for (int dl = 0; dl < GD; dl += 2) {
    const int d0 = G * GD + dl, d1 = d0 + 1;
    float va[PPT][2];
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int p = tid + NT * k;
      const f32x2 nn2 = pack2(my_nn[k], my_nn[k]), nnn2 = pack2(-my_nn[k], -my_nn[k]);
      const int q0 = p + delta_dy(R, d0) * PW + delta_dx(R, d0);   // in bounds (PAD); garbage if outside P
      const int q1 = p + delta_dy(R, d1) * PW + delta_dx(R, d1);
      VF_CHECK(q0 >= 0 && q0 < region_np(CFG) + PAD && q1 >= 0 && q1 < region_np(CFG) + PAD);
      float tau0, tau1;
#if SHARED_REC8
      angular_tau2_r8<VAR>(my_pk[k], nn2, nnn2, sm.px[q0], sm.px[q1], tau0, tau1, va[k][0], va[k][1]);
#else
      const f32x2 nrm2 = pack2(my_nrm[k], my_nrm[k]);
      angular_tau2<VAR>(my_pk[k], nn2, nnn2, nrm2, sm.px[q0], sm.px[q1], tau0, tau1, va[k][0], va[k][1]);
#endif
      // cos < 0.5 <=> tau > 1/sqrt2: flag a superset (margin 2^-10 >> the
      // ~5e-7 relative error of tau) for the exact decision below.  Offsets
      // reaching below the region read the zero padding: tau = 0, never flagged.
      if (tau0 > 0.70641626f) flags[k] |= 1u << dl;           // (1/sqrt2) (1 - 2^-10)
      if (tau1 > 0.70641626f) flags[k] |= 1u << (dl + 1);
    }
    if constexpr (ML::ZL) {
      *reinterpret_cast<float2*>(&sm.M[dl][2 * tid]) = make_float2(va[0][0], va[1][0]);
      *reinterpret_cast<float2*>(&sm.M[dl + 1][2 * tid]) = make_float2(va[0][1], va[1][1]);
    } else {
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        sm.M[dl][tid + NT * k] = va[k][0];
        sm.M[dl + 1][tid + NT * k] = va[k][1];
      }
    }
  }
  }
  // ---- rare pairs: exact branch decision, warp-cooperative ---------------------------
  // The flagged pairs of the warp (~1% of its pairs, spread over a few lanes)
  // are compacted into a per-warp queue and re-evaluated one per lane, so the
  // warp pays ~one fix-up pass instead of one per flagged pair of its busiest
  // lane.  Entries beyond QCAP (adversarial images) fall back to per-lane loops.
  {
    const int lane = tx;
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) cnt += __popc(flags[k]);
    if (__any_sync(0xffffffffu, cnt != 0)) {
      int incl = cnt;                                         // inclusive warp scan of cnt
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      int pos = incl - cnt;
      uint32_t* q = sm.queue[ty];
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const uint32_t p = tid + NT * k;
        while (flags[k] && pos < QCAP) {
          const uint32_t dl = __ffs(flags[k]) - 1;
          flags[k] &= flags[k] - 1;
          q[pos++] = p | (dl << 16);
        }
      }
      __syncwarp();
      const int nq = total < QCAP ? total : QCAP;
      for (int e = lane; e < nq; e += 32) {
        const uint32_t en = q[e];
        angular_fix<VAR, WIN>(sm, (int)(en & 0xffffu), (int)(en >> 16), G * GD + (int)(en >> 16));
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) {                         // overflow only
        while (flags[k]) {
          const int dl = __ffs(flags[k]) - 1;
          flags[k] &= flags[k] - 1;
          angular_fix<VAR, WIN>(sm, tid + NT * k, dl, G * GD + dl);
        }
      }
      __syncwarp();                                           // queue reusable by the next group
    }
  }
  // zero vectors: block-uniform slow path, only in blocks that hold
  // a black pixel.  Every pair touching a zero pixel is set to 0, including
  // the entries other threads wrote with the zero pixel on the q side.
  if (blk_zero) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      if (my_nn[k] == 0.0f) {
        const int p = tid + NT * k;
#pragma unroll
        for (int dl = 0; dl < GD; ++dl) {
          const int d = G * GD + dl;
          const int off = delta_dy(R, d) * PW + delta_dx(R, d);
          sm.M[dl][ML::idx(p)] = 0.0f;
          if (p - off >= 0) sm.M[dl][ML::idx(p - off)] = 0.0f;
        }
      }
    }
  }
  __syncthreads();
  // ---- phase C: accumulate the window aggregates ------------------------------------
  // Two outputs per thread (rows ty and ty + NW): their aggregates R_i are one
  // packed pair and each pair value pair (v_row0, v_row1) is added with one
  // FADD2 (per-element rounding = __fadd_rn, same order: bit-identical to the
  // scalar loop).  Warps whose second row is past the tile accumulate a copy
  // of the first window and discard it (warp-uniform, no divergence).
  if constexpr (ML::ZL) {
    // rows ty and ty + 12 of the maps are adjacent: one LDS.64 per pair feeds
    // both windows of warps 0..9; warps 10, 11 (second row past the 22-row
    // tile) read their one window's values one by one
    static_assert(OPT == 2 && NW == 12 && TH == 22 && GD == 12, "ZL layout: 3x3, CFG 4");
    if (tx < TW) {
      const int base = ty * PW + tx;                          // P index of window sample (0,0), row ty
      if (ty + NW < TH) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
#pragma unroll
          for (int j = i + 1; j < N; ++j) {
            const int d = delta_index(R, j / WIN - i / WIN, j % WIN - i % WIN);
            const int q = base + (i / WIN) * PW + (i % WIN);  // row <= 11
            VF_CHECK(q < 384);
            const float2 v = *reinterpret_cast<const float2*>(&sm.M[d][2 * q]);
            Ra[0][i] += v.x;
            Ra[0][j] += v.x;
            Ra[1][i] += v.y;
            Ra[1][j] += v.y;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) {
#pragma unroll
          for (int j = i + 1; j < N; ++j) {
            const int d = delta_index(R, j / WIN - i / WIN, j % WIN - i % WIN);
            const float v = sm.M[d][ML::idx(base + (i / WIN) * PW + (i % WIN))];
            Ra[0][i] += v;
            Ra[0][j] += v;
          }
        }
      }
    }
  } else {
  // Rows past the output tile (TH not a multiple of 8) are skipped warp-
  // uniformly; the aggregates start at -0 inside the branch so that the first
  // addition of each folds away.
#pragma unroll
  for (int k = 0; k < OPT; ++k) {
    const int oy = ty + NW * k;
    if ((TH % NW == 0 || oy < TH) && tx < TW) {
      const int base = oy * PW + tx;                          // P index of window sample (0,0)
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = i + 1; j < N; ++j) {
          const int d = delta_index(R, j / WIN - i / WIN, j % WIN - i % WIN);
          if (d / GD == G) {
            VF_CHECK(base + (i / WIN) * PW + (i % WIN) < region_np(CFG));
            const float v = sm.M[d - G * GD][base + (i / WIN) * PW + (i % WIN)];
            Ra[k][i] += v;
            Ra[k][j] += v;
          }
        }
      }
    }
  }
  }
}

template <int WIN, int VAR, int GD, int OPT, int CFG, int... Gs>
__device__ __forceinline__ void shared_groups(std::integer_sequence<int, Gs...>, SharedSmem<GD, CFG>& sm,
                                              const uint32_t (&my_pk)[shared::cfg_ppt(CFG)],
                                              const float (&my_nn)[shared::cfg_ppt(CFG)],
                                              const float (&my_nrm)[shared::cfg_ppt(CFG)], float (&Ra)[OPT][WIN * WIN],
                                              int tid, bool blk_zero) {
  (shared_group<WIN, VAR, GD, OPT, CFG, Gs>(sm, my_pk, my_nn, my_nrm, Ra, tid, blk_zero), ...);
}

// Resident blocks per SM the register allocation is held to.
__host__ __device__ constexpr int shared_min_blocks(int win, int cfg) {
  return win == 5 ? 2 : (cfg == 4 ? SHARED_MINB_CFG4 : 4);
}

template <int WIN, int VAR, int CFG>
__global__ void __launch_bounds__(shared::cfg_nt(CFG), shared_min_blocks(WIN, CFG)) vf_angular_shared_kernel(const Launch L) {
  using namespace shared;
  constexpr int NT = cfg_nt(CFG);
  constexpr int NW = NT / 32;
  constexpr int PPT = cfg_ppt(CFG);
  constexpr int PH = region_h(CFG);
  constexpr int NP = region_np(CFG);
  constexpr int R = WIN / 2;
  constexpr int N = WIN * WIN;
  constexpr int TW = PW - 2 * R;            // output tile width
  constexpr int TH = PH - 2 * R;            // output tile height
  constexpr int ND = n_delta(R);            // 12 or 40
  constexpr int GD = (WIN == 3) ? 12 : 10;  // offsets per group
  constexpr int NG = ND / GD;
  constexpr int OPT = (TH + NW - 1) / NW;   // outputs per thread (rows ty, ty + NW, ...)
  static_assert(ND % GD == 0, "groups must tile the offsets");
  extern __shared__ __align__(16) unsigned char smem_raw[];   // sizeof(SharedSmem<GD, CFG>), dynamic (> 48 KB)
  SharedSmem<GD, CFG>& sm = *reinterpret_cast<SharedSmem<GD, CFG>*>(smem_raw);

  const int b = blockIdx.z;
  const int ox0 = blockIdx.x * TW;                        // output tile origin (global)
  const int oy0 = L.out_row0 + blockIdx.y * TH;
  const uint8_t* __restrict__ in = L.in + (long long)b * L.in_stride;
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;

  // ---- stage P ----------------------------------------------------------------
  uint32_t my_pk[PPT];
  float my_nn[PPT], my_nrm[PPT];
  bool has_zero = false;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int p = tid + NT * k;
    const int py = p >> 5, px = p & 31;
    const uint8_t* q = pixel_ptr(L, in, oy0 - R + py, ox0 - R + px);
    const uint32_t r = q[0], g = q[1], bl = q[2];
    const float nn = (float)(r * r + g * g + bl * bl);          // exact
    float nrm;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(nrm) : "f"(nn));   // MUFU.SQRT, ~1 ulp
    my_pk[k] = pack_rgb(r, g, bl);
    my_nn[k] = nn;
    my_nrm[k] = nrm;
    has_zero |= (nn == 0.0f);
    if constexpr (!SharedSmem<GD, CFG>::PX2) {
#if SHARED_REC8
      sm.px[p] = make_uint2(my_pk[k], __float_as_uint(nn));
#else
      sm.px[p] = make_uint4(my_pk[k], __float_as_uint(nn), __float_as_uint(nrm), 0u);
#endif
    }
  }
  if constexpr (SharedSmem<GD, CFG>::PX2) {
    static_assert(PPT == 2 && NT == 384 && PAD <= 384, "PX2: 384 threads x 2 pixels");
    sm.px[tid] = make_uint4(my_pk[0], my_pk[1], __float_as_uint(my_nn[0]), __float_as_uint(my_nn[1]));
    if (tid < PAD) sm.px[384 + tid] = make_uint4(my_pk[1], 0u, __float_as_uint(my_nn[1]), 0u);   // rows 12.., zero pad
  } else {
#if SHARED_REC8
    if (tid < PAD) sm.px[NP + tid] = make_uint2(0u, 0u);
#else
    if (tid < PAD) sm.px[NP + tid] = make_uint4(0u, 0u, 0u, 0u);
#endif
  }
  if (tid < ND) sm.off[tid] = delta_dy(R, tid) * PW + delta_dx(R, tid);
  const bool blk_zero = __syncthreads_or(has_zero) != 0;       // staging barrier

  float Ra[OPT][N];
#pragma unroll
  for (int k = 0; k < OPT; ++k)
#pragma unroll
    for (int i = 0; i < N; ++i) Ra[k][i] = -0.0f;
  shared_groups<WIN, VAR, GD, OPT, CFG>(std::make_integer_sequence<int, NG>{}, sm, my_pk, my_nn, my_nrm, Ra, tid,
                                        blk_zero);

  // ---- argmin + store ------------------------------------------------------------------
#pragma unroll
  for (int k = 0; k < OPT; ++k) {
    const int oy = ty + NW * k;
    const int gy = oy0 + oy, gx = ox0 + tx;
    if ((TH % NW == 0 || oy < TH) && tx < TW && gx < L.W && gy < L.out_row0 + L.out_rows) {
      // argmin over the window (lowest index on ties), tracking the region
      // offset of the selected sample, then one load of its packed RGB
      const int base = oy * PW + tx;
      float bv = Ra[k][0];
      int so = 0;
#pragma unroll
      for (int i = 1; i < N; ++i) {
        const bool lt = Ra[k][i] < bv;
        bv = lt ? Ra[k][i] : bv;
        so = lt ? (i / WIN) * PW + (i % WIN) : so;
      }
      store_result<N>(L, b, gx, gy, Ra[k], rec_get(sm, base + so).x);
    }
  }
}

// Kernel + grid of the pair-sharing kernel for a launch (see vf_api.cu);
// cfg = launch configuration (shared::cfg_nt / cfg_ppt).
// VF_ANGULAR_MM_EXTERN (vf_api.cu): the minimax kernels are instantiated in
// their own translation unit (vf_ang_mm.cu, own ptxas setting) and fetched
// from there; only the exact ones are instantiated here.
#ifndef VF_ANGULAR_MM_TU   // kernel selection: vf_api.cu only (vf_ang_mm.cu instantiates the minimax kernels itself)
#ifdef VF_ANGULAR_MM_EXTERN
const void* shared_kernel_fn_mm(int window, int cfg);
#endif
template <int WIN, int CFG>
inline const void* shared_kernel_fn_t(int var) {
#ifdef VF_ANGULAR_MM_EXTERN
  if (var != EXACT) return shared_kernel_fn_mm(WIN, CFG);
  return (const void*)vf_angular_shared_kernel<WIN, EXACT, CFG>;
#else
  return var == EXACT ? (const void*)vf_angular_shared_kernel<WIN, EXACT, CFG>
                      : (const void*)vf_angular_shared_kernel<WIN, MINIMAX, CFG>;
#endif
}

template <int WIN>
inline const void* shared_kernel_fn_w(int var, int cfg) {
  switch (cfg) {
    case 1: return shared_kernel_fn_t<WIN, 1>(var);
    case 2: return shared_kernel_fn_t<WIN, 2>(var);
    case 3: return shared_kernel_fn_t<WIN, 3>(var);
    default: return shared_kernel_fn_t<WIN, 4>(var);
  }
}
inline const void* shared_kernel_fn(int window, int var, int cfg) {
  return window == 3 ? shared_kernel_fn_w<3>(var, cfg) : shared_kernel_fn_w<5>(var, cfg);
}

template <int WIN>
inline size_t shared_smem_bytes_w(int cfg) {
  constexpr int GD = (WIN == 3) ? 12 : 10;
  switch (cfg) {
    case 1: return sizeof(SharedSmem<GD, 1>);
    case 2: return sizeof(SharedSmem<GD, 2>);
    case 3: return sizeof(SharedSmem<GD, 3>);
    default: return sizeof(SharedSmem<GD, 4>);
  }
}
inline size_t shared_smem_bytes(int window, int cfg) {
  return window == 3 ? shared_smem_bytes_w<3>(cfg) : shared_smem_bytes_w<5>(cfg);
}

// Opt the kernels in to > 48 KB of dynamic shared memory (once per process).
inline cudaError_t shared_set_attributes() {
  const int ws[2] = {3, 5};
  for (int w : ws)
    for (int cfg = 1; cfg <= 4; ++cfg)
      for (int v = 0; v < 2; ++v) {
        cudaError_t e = cudaFuncSetAttribute(shared_kernel_fn(w, v, cfg), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)shared_smem_bytes(w, cfg));
        if (e != cudaSuccess) return e;
      }
  return cudaSuccess;
}

inline dim3 shared_grid(const Launch& L, int B, int window, int cfg) {
  using namespace shared;
  const int R = window / 2;
  const int TW = PW - 2 * R, TH = region_h(cfg) - 2 * R;
  return dim3((L.W + TW - 1) / TW, (L.out_rows + TH - 1) / TH, B);
}

#endif  // VF_ANGULAR_MM_TU

}  // namespace vf
