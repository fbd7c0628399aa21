// vf_role.cuh -- angular criterion, 5x5 windows: cross-window pair sharing
// with per-pixel ROLE SUMS instead of per-window pair
// accumulation.
//
// In a window with top-left t, sample i sits at q = t + (a, b) and its
// aggregate is (Eq. 5)
//     R_i = sum over (dy, dx) in [-a, 4-a] x [-b, 4-b], (dy, dx) != 0, of A(q, q + (dy, dx)),
// which depends only on the pixel q and its role (a, b) in the window.  So
// every pixel of the block's region computes its 25 role sums once, from the
// 80 pair values of its 9x9 neighbourhood, and every output window reads its
// 25 aggregates with one load each -- 25 loads instead of 300 loads and 600
// additions per window (the per-window accumulation of vf_shared.cuh).
//
// Per pixel and neighbourhood row dy, the five row sums
//     H_b(dy) = sum_{dx=-b}^{4-b} A(q, q + (dy, dx)),  b = 0..4,
// are formed without subtractions (14 additions: all terms are >= 0, so the
// sums keep full relative precision), and R_(a,b) += H_b(dy) for every a with
// -a <= dy <= 4-a.
//
// The pair maps are built one neighbourhood row at a time (group g = the
// offsets with dy = g: 4 for g = 0, 9 for g = 1..4), exactly as in
// vf_shared.cuh (phase A: tau-branch value of Table 1 / Eq. 6, superset flag
// of the cos < 0.5 pairs re-decided exactly by a warp-cooperative pass,
// block-uniform zero-vector rule S:342); phase B then adds the rows +g and -g
// of every pixel's neighbourhood (row -g is the map of offset (g, -dx) read at
// the neighbour) into its role sums.  After the last group the role sums
// replace the maps in shared memory and the outputs take their argmin.
#pragma once
#include <cuda_runtime.h>

#include <utility>

#include "vf_shared.cuh"

namespace vf {

namespace role {
constexpr int PW = shared::PW;          // region width (32)
constexpr int PRE = 5 * PW;             // map padding before the region: reverse reads reach 2r rows + 2r px back
constexpr int POST = 5 * PW;            // and after it
// group g = the offsets (g, dx): dx = 1..2r for g = 0, dx = -2r..2r for g = 1..2r
__host__ __device__ constexpr int nslots(int r, int g) { return g == 0 ? 2 * r : 4 * r + 1; }
__host__ __device__ constexpr int slot_dx(int r, int g, int s) { return g == 0 ? s + 1 : s - 2 * r; }
}  // namespace role

// Block of NT threads (256 or 384) over a 32 x (NT PPT / 32) region, PPT
// region pixels per thread; window side WIN (3 or 5).
template <int WIN, int NT, int PPT>
struct RoleSmem {
  static constexpr int N = WIN * WIN;
  static constexpr int NSM = 2 * WIN - 1;   // maps of one group (4r + 1)
  static constexpr int NP = NT * PPT;
  static constexpr int MS = role::PRE + NP + role::POST;   // map stride (floats)
  static constexpr int QCAP = 64;
  struct Maps {
    uint4 px[NP + shared::PAD];   // (packed RGB0, |x|^2 bits, |x| bits, 0)
    float M[NSM][MS];             // pair maps of one neighbourhood row g
  };
  union U {
    Maps a;
    float S[N][NP];               // role sums, after the last group
  } u;
  uint32_t pk[NP];                // packed RGB of the region (output store)
  uint32_t queue[NT / 32][QCAP];
};

// Exact re-decision of a flagged pair (p, p + (g, dx)) of slot s: as
// angular_fix in vf_shared.cuh, on this kernel's map layout.
template <int VAR, int WIN, int NT, int PPT>
__device__ __forceinline__ void role_fix(RoleSmem<WIN, NT, PPT>& sm, int p, int s, int off) {
  const uint4 pv = sm.u.a.px[p], qv = sm.u.a.px[p + off];
  const float D = __uint_as_float(__dp4a(pv.x, qv.x, F2P23_BITS)) - F2P23;   // exact dot
  const float nna = __uint_as_float(pv.y), nnb = __uint_as_float(qv.y);
  const float Ph = __fmul_rn(nna, nnb);
  const float Pl = fmaf(nna, nnb, -Ph);
  const float t = fmaf(__fmul_rn(4.0f, D), D, -Ph);         // fl(4D^2 - Ph)
  if (t < Pl) {                                             // 4D^2 < P: cos < 0.5, exact
    const float c = D * rcp_approx(__fmul_rn(__uint_as_float(pv.z), __uint_as_float(qv.z)));
    sm.u.a.M[s][role::PRE + p] = (VAR == EXACT) ? acosf(c) : horner4(coef::ACOS(), c);
  }
}

// H_b = sum_{dx=-b}^{2-b} v[2 + dx], b = 0..2, without subtractions.
__device__ __forceinline__ void row_sums(const float (&v)[5], float (&H)[3]) {
  const float e = v[2] + v[3];
  H[0] = e + v[4];
  H[1] = e + v[1];
  H[2] = (v[0] + v[1]) + v[2];
}
// H_b = sum_{dx=-b}^{4-b} v[4 + dx], b = 0..4, without subtractions.
__device__ __forceinline__ void row_sums(const float (&v)[9], float (&H)[5]) {
  const float e = v[4] + v[5];
  const float c = e + v[6];
  H[0] = c + (v[7] + v[8]);
  H[1] = c + (v[3] + v[7]);
  H[2] = c + (v[2] + v[3]);
  const float a12 = v[1] + v[2];
  H[3] = a12 + (v[3] + e);
  H[4] = (v[0] + a12) + (v[3] + v[4]);
}

template <int WIN, int VAR, int NT, int PPT, int G>
__device__ __forceinline__ void role_group(RoleSmem<WIN, NT, PPT>& sm, const uint32_t (&my_pk)[PPT],
                                           const float (&my_nn)[PPT], const float (&my_nrm)[PPT],
                                           float (&Rs)[PPT][WIN * WIN], int tid, bool blk_zero) {
  using namespace role;
  constexpr int R = WIN / 2;
  constexpr int NS = nslots(R, G);
  constexpr int QCAP = RoleSmem<WIN, NT, PPT>::QCAP;
  [[maybe_unused]] constexpr int NPL = RoleSmem<WIN, NT, PPT>::NP;   // (VF_CHECK)
  const int lane = tid & 31, warp = tid >> 5;
  if (G > 0) __syncthreads();   // previous phase B done with the maps (G = 0: the staging barrier)
  // ---- phase A: maps of the offsets (G, dx) ----------------------------------------
  uint32_t flags[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) flags[k] = 0u;
  // slots in pairs in packed FP32 (FFMA2 / FADD2 / FMUL2), an odd last slot scalar
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int p = tid + NT * k;
    const f32x2 nn2 = pack2(my_nn[k], my_nn[k]), nnn2 = pack2(-my_nn[k], -my_nn[k]);
    const f32x2 nrm2 = pack2(my_nrm[k], my_nrm[k]);
#pragma unroll
    for (int s = 0; s + 1 < NS; s += 2) {
      const int q0 = p + G * PW + slot_dx(R, G, s), q1 = p + G * PW + slot_dx(R, G, s + 1);
      VF_CHECK(q0 >= 0 && q0 < NPL + shared::PAD && q1 >= 0 && q1 < NPL + shared::PAD);
      float tau0, tau1, v0, v1;
      angular_tau2<VAR>(my_pk[k], nn2, nnn2, nrm2, sm.u.a.px[q0], sm.u.a.px[q1], tau0, tau1, v0, v1);
      sm.u.a.M[s][PRE + p] = v0;
      sm.u.a.M[s + 1][PRE + p] = v1;
      if (tau0 > 0.70641626f) flags[k] |= 1u << s;          // possible cos < 0.5 (see vf_shared.cuh)
      if (tau1 > 0.70641626f) flags[k] |= 1u << (s + 1);
    }
    if (NS % 2) {
      constexpr int s = NS - 1;
      const int off = G * PW + slot_dx(R, G, s);
      VF_CHECK(p + off >= 0 && p + off < NPL + shared::PAD);
      const uint4 qv = sm.u.a.px[p + off];
      const float D = __uint_as_float(__dp4a(my_pk[k], qv.x, F2P23_BITS)) - F2P23;   // exact dot
      const float nnq = __uint_as_float(qv.y);
      const float Ph = __fmul_rn(my_nn[k], nnq);
      const float Pl = fmaf(my_nn[k], nnq, -Ph);
      const float X = __fadd_rn(fmaf(-D, D, Ph), Pl);         // |x_p x x_q|^2
      const float w = fmaf(__fmul_rn(my_nrm[k], __uint_as_float(qv.z)), D, Ph);   // s (s + D)
      const float tau = __fmul_rn(X, rsqrt_approx(fmaf(X, w, 1e-30f)));          // sqrt(1 - cos)
      const float v = (VAR == EXACT) ? 2.0f * asinf(tau * 0.70710678118654752f) : horner4(coef::ASIN(), tau);
      sm.u.a.M[s][PRE + p] = v;
      if (tau > 0.70641626f) flags[k] |= 1u << s;
    }
  }
  // ---- flagged pairs, warp-cooperative (as in vf_shared.cuh) --------------------------
  {
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) cnt += __popc(flags[k]);
    if (__any_sync(0xffffffffu, cnt != 0)) {
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      int pos = incl - cnt;
      uint32_t* q = sm.queue[warp];
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const uint32_t p = tid + NT * k;
        while (flags[k] && pos < QCAP) {
          const uint32_t s = __ffs(flags[k]) - 1;
          flags[k] &= flags[k] - 1;
          q[pos++] = p | (s << 16);
        }
      }
      __syncwarp();
      const int nq = total < QCAP ? total : QCAP;
      for (int e = lane; e < nq; e += 32) {
        const uint32_t en = q[e];
        const int s = (int)(en >> 16);
        role_fix<VAR>(sm, (int)(en & 0xffffu), s, G * PW + slot_dx(R, G, s));
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        while (flags[k]) {
          const int s = __ffs(flags[k]) - 1;
          flags[k] &= flags[k] - 1;
          role_fix<VAR>(sm, tid + NT * k, s, G * PW + slot_dx(R, G, s));
        }
      }
      __syncwarp();
    }
  }
  // ---- zero vectors: block-uniform slow path -----------------------------------
  if (blk_zero) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      if (my_nn[k] == 0.0f) {
        const int p = tid + NT * k;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const int off = G * PW + slot_dx(R, G, s);
          sm.u.a.M[s][PRE + p] = 0.0f;
          if (p - off >= 0) sm.u.a.M[s][PRE + p - off] = 0.0f;
        }
      }
    }
  }
  __syncthreads();
  // ---- phase B: rows +G and -G of every pixel's neighbourhood into its role sums -----
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int q = PRE + tid + NT * k;
    constexpr int D2 = 2 * R;                 // 2r: neighbourhood half-width
    float vf[2 * D2 + 1], H[WIN];
    if (G == 0) {   // row 0: (0, dx) for dx > 0 from the maps, dx < 0 from the neighbour's map
#pragma unroll
      for (int dx = 1; dx <= D2; ++dx) {
        vf[D2 + dx] = sm.u.a.M[dx - 1][q];
        vf[D2 - dx] = sm.u.a.M[dx - 1][q - dx];
      }
      vf[D2] = -0.0f;   // the sample itself (-0 + x == x: folds away)
    } else {
#pragma unroll
      for (int dx = -D2; dx <= D2; ++dx) vf[D2 + dx] = sm.u.a.M[dx + D2][q];
    }
    row_sums(vf, H);
#pragma unroll
    for (int b = 0; b < WIN; ++b)
#pragma unroll
      for (int a = 0; a < WIN; ++a)
        if (-a <= G && G <= D2 - a) Rs[k][a * WIN + b] += H[b];
    if (G > 0) {    // row -G: A(q, q + (-G, dx)) = map of offset (G, -dx) at q + (-G, dx)
      float vr[2 * D2 + 1];
#pragma unroll
      for (int dx = -D2; dx <= D2; ++dx) vr[D2 + dx] = sm.u.a.M[D2 - dx][q - G * PW + dx];
      row_sums(vr, H);
#pragma unroll
      for (int b = 0; b < WIN; ++b)
#pragma unroll
        for (int a = 0; a < WIN; ++a)
          if (-a <= -G && -G <= D2 - a) Rs[k][a * WIN + b] += H[b];
    }
  }
}

template <int WIN, int VAR, int NT, int PPT, int... Gs>
__device__ __forceinline__ void role_groups(std::integer_sequence<int, Gs...>, RoleSmem<WIN, NT, PPT>& sm,
                                            const uint32_t (&my_pk)[PPT], const float (&my_nn)[PPT],
                                            const float (&my_nrm)[PPT], float (&Rs)[PPT][WIN * WIN], int tid,
                                            bool blk_zero) {
  (role_group<WIN, VAR, NT, PPT, Gs>(sm, my_pk, my_nn, my_nrm, Rs, tid, blk_zero), ...);
}

// Resident blocks per SM the register allocation is held to: 5x5: 2 (<= 80
// registers at 384 threads); 3x3 (384 threads): 4 (<= 40).
__host__ __device__ constexpr int role_min_blocks(int win, int nt) { return win == 5 ? 2 : (nt == 384 ? 4 : 4); }

template <int WIN, int VAR, int NT, int PPT>
__global__ void __launch_bounds__(NT, role_min_blocks(WIN, NT)) vf_angular_role_kernel(const Launch L) {
  using namespace role;
  constexpr int R = WIN / 2, N = WIN * WIN;
  constexpr int NW = NT / 32;               // warps = region rows per pixel slab
  constexpr int NP = RoleSmem<WIN, NT, PPT>::NP;
  constexpr int PH = NP / PW;               // region height
  constexpr int TW = PW - 2 * R;            // output tile width (30 / 28)
  constexpr int TH = PH - 2 * R;            // output tile height
  constexpr int OPT = (TH + NW - 1) / NW;   // outputs per thread (rows ty, ty + NW, ...)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RoleSmem<WIN, NT, PPT>& sm = *reinterpret_cast<RoleSmem<WIN, NT, PPT>*>(smem_raw);

  const int b = blockIdx.z;
  const int ox0 = blockIdx.x * TW;
  const int oy0 = L.out_row0 + blockIdx.y * TH;
  const uint8_t* __restrict__ in = L.in + (long long)b * L.in_stride;
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;

  // ---- stage the region --------------------------------------------------------------
  uint32_t my_pk[PPT];
  float my_nn[PPT], my_nrm[PPT];
  bool has_zero = false;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int p = tid + NT * k;
    const uint8_t* q = pixel_ptr(L, in, oy0 - R + (p >> 5), ox0 - R + (p & 31));
    const uint32_t r = q[0], g = q[1], bl = q[2];
    const float nn = (float)(r * r + g * g + bl * bl);          // exact
    float nrm;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(nrm) : "f"(nn));
    my_pk[k] = pack_rgb(r, g, bl);
    my_nn[k] = nn;
    my_nrm[k] = nrm;
    has_zero |= (nn == 0.0f);
    sm.u.a.px[p] = make_uint4(my_pk[k], __float_as_uint(nn), __float_as_uint(nrm), 0u);
    sm.pk[p] = my_pk[k];
  }
  if (tid < shared::PAD) sm.u.a.px[NP + tid] = make_uint4(0u, 0u, 0u, 0u);
  const bool blk_zero = __syncthreads_or(has_zero) != 0;

  float Rs[PPT][N];
#pragma unroll
  for (int k = 0; k < PPT; ++k)
#pragma unroll
    for (int i = 0; i < N; ++i) Rs[k][i] = -0.0f;   // -0 + v == v: the first add folds away
  role_groups<WIN, VAR, NT, PPT>(std::make_integer_sequence<int, 2 * R + 1>{}, sm, my_pk, my_nn, my_nrm, Rs, tid,
                                 blk_zero);

  // ---- role sums replace the maps ------------------------------------------------------
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PPT; ++k)
#pragma unroll
    for (int i = 0; i < N; ++i) sm.u.S[i][tid + NT * k] = Rs[k][i];
  __syncthreads();

  // ---- outputs: 25 aggregates per window, argmin, store ---------------------------------
#pragma unroll
  for (int k = 0; k < OPT; ++k) {
    const int oy = ty + NW * k;
    const int gy = oy0 + oy, gx = ox0 + tx;
    if ((TH % NW == 0 || oy < TH) && tx < TW && gx < L.W && gy < L.out_row0 + L.out_rows) {
      const int t = oy * PW + tx;                             // region index of window sample (0, 0)
      float Ra[N];
#pragma unroll
      for (int i = 0; i < N; ++i) Ra[i] = sm.u.S[i][t + (i / WIN) * PW + (i % WIN)];
      float bv = Ra[0];
      int so = 0;
#pragma unroll
      for (int i = 1; i < N; ++i) {
        const bool lt = Ra[i] < bv;
        bv = lt ? Ra[i] : bv;
        so = lt ? (i / WIN) * PW + (i % WIN) : so;
      }
      store_result<N>(L, b, gx, gy, Ra, sm.pk[t + so]);
    }
  }
}

// Launch configurations (as shared::cfg_nt / cfg_ppt): cfg 1..3 = 256
// threads with 1..3 pixels each; cfg 4 (default) = 384 threads with 2 pixels
// each: the same 32 x 24 region as cfg 3 with two thirds of the role
// accumulators per thread, so more warps fit per SM (5x5: 24 instead of 16).
#ifndef VF_ANGULAR_MM_TU   // kernel selection: vf_api.cu only (vf_ang_mm.cu instantiates the minimax kernels itself)
#ifdef VF_ANGULAR_MM_EXTERN
const void* role_kernel_fn_mm(int window, int cfg);
#endif
template <int WIN, int CFG>
inline const void* role_kernel_fn_t(int var) {
  constexpr int NT = shared::cfg_nt(CFG), PPT = shared::cfg_ppt(CFG);
#ifdef VF_ANGULAR_MM_EXTERN
  if (var != EXACT) return role_kernel_fn_mm(WIN, CFG);   // vf_ang_mm.cu
  return (const void*)vf_angular_role_kernel<WIN, EXACT, NT, PPT>;
#else
  return var == EXACT ? (const void*)vf_angular_role_kernel<WIN, EXACT, NT, PPT>
                      : (const void*)vf_angular_role_kernel<WIN, MINIMAX, NT, PPT>;
#endif
}
template <int WIN>
inline const void* role_kernel_fn_w(int var, int cfg) {
  switch (cfg) {
    case 1: return role_kernel_fn_t<WIN, 1>(var);
    case 2: return role_kernel_fn_t<WIN, 2>(var);
    case 3: return role_kernel_fn_t<WIN, 3>(var);
    default: return role_kernel_fn_t<WIN, 4>(var);
  }
}
inline const void* role_kernel_fn(int window, int var, int cfg) {
  return window == 3 ? role_kernel_fn_w<3>(var, cfg) : role_kernel_fn_w<5>(var, cfg);
}
template <int WIN>
inline size_t role_smem_bytes_w(int cfg) {
  switch (cfg) {
    case 1: return sizeof(RoleSmem<WIN, 256, 1>);
    case 2: return sizeof(RoleSmem<WIN, 256, 2>);
    case 3: return sizeof(RoleSmem<WIN, 256, 3>);
    default: return sizeof(RoleSmem<WIN, 384, 2>);
  }
}
inline size_t role_smem_bytes(int window, int cfg) {
  return window == 3 ? role_smem_bytes_w<3>(cfg) : role_smem_bytes_w<5>(cfg);
}
inline cudaError_t role_set_attributes() {
  const int ws[2] = {3, 5};
  for (int w : ws)
    for (int cfg = 1; cfg <= 4; ++cfg)
      for (int v = 0; v < 2; ++v) {
        cudaError_t e = cudaFuncSetAttribute(role_kernel_fn(w, v, cfg), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)role_smem_bytes(w, cfg));
        if (e != cudaSuccess) return e;
      }
  return cudaSuccess;
}

#endif  // VF_ANGULAR_MM_TU

}  // namespace vf
