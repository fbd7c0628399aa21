/*
 * vf.h -- C ABI of libvf.so: B200 (sm_100a) order-statistics vector filters
 * with exact and minimax elementary functions.
 *
 * Paper: Celebi, Kingravi, Lukac, Celiker, "Cost-Effective Implementation of
 * Order-Statistics Based Vector Filters Using Minimax Approximations",
 * arXiv 1009.0959 (/root/reference/PAPER.md, cited P:<line>).
 *
 * OPERATION (every vf_filter* entry point)
 *   For every output pixel (y, x) take the w x w window W(y, x) of the input
 *   (w = `window`, n = w*w samples re-indexed in raster order k = dy*w + dx,
 *   Fig. 1; replicate (clamp) padding at the image border),
 *   compute the pairwise criterion D(i, j) for all i < j, the aggregates
 *   R_i = sum_{j != i} D(i, j) and output x_{k*}, k* = argmin_i R_i
 *   (Eq. 5), the lowest index winning bit-equal aggregates.
 *   Criteria (readings R2-R5):
 *     VF_ANGULAR  D = angle between x_i and x_j (Eq. 5); exact = libm
 *                 arccos / Eq. 6 identity; minimax = Table 1 composite
 *                 (ARCCOS row for cos < 0.5, ARCSIN row in tau = sqrt(1-cos)
 *                 otherwise; Eqs. 6-7).  Zero vectors give 0.
 *     VF_EXP      D = 1 - exp(-z), z = |x_i-x_j|_1 / h_W, h_W the window mean
 *                 of Eq. 8's bandwidth h_i (kappa = 0.33);
 *                 minimax = Table 3 rational (VF_MINIMAX) or Table 2
 *                 p = 4 polynomial (VF_MINIMAX_POLY4).
 *     VF_LOG      D = -ENT(s), ENT(s) = s ln s, s = 1 - (1 - 1/e) q,
 *                 q = (n-1) |x_i-x_j|_1 / sum_{k<l} |x_k-x_l|_1;
 *                 minimax = Table 4 rational.
 *     VF_MINIMAX_REACH (VF_EXP, VF_LOG only): the criterion
 *                 value itself as one minimax polynomial re-derived by the
 *                 Remez exchange on the arguments the criterion can
 *                 reach (z <= z*_25, u = 1 - s <= 1 - 1/e):
 *                 degree 5 for D_E (eps 7.86e-8), 7 for D_L (eps 2.95e-7),
 *                 coefficients tests/golden/remez_reach.txt.
 *   VF_EXACT evaluates the functions with fp32 libm: acosf / asinf (Eq. 6),
 *   and the cancellation-free -expm1f(-z) and -(1-u) log1pf(-u) (SURVEY
 *   8(a) a5); the libvf_paperlibm.so build (VF_EXACT_LIBM=1) uses the
 *   paper's 1 - expf(-z) and -s logf(s) instead (reading R26).
 *   Arithmetic: fp32 on the device, with exact integer geometry (dot
 *   products, squared norms, L1 distances and the cos < 0.5 branch decision
 *   are exact); aggregates agree with the double-precision oracle within
 *   1e-5 relative (tests/test_gpu_parity.py).
 *
 * LAYOUT
 *   Images are uint8 RGB, HWC, row-major, row stride 3*W bytes, batches
 *   dense [B][H][W][3].  `index` (nullable) is uint8 [..][H][W] holding k*.
 *   `aggregates` (nullable) is float [..][H][W][n] holding R_0..R_{n-1}.
 *
 * OWNERSHIP / EXECUTION
 *   All buffers are owned by the caller.  Unless stated otherwise they are
 *   DEVICE pointers (e.g. from PyTorch's caching allocator).  The library never
 *   allocates, frees or synchronises; every call enqueues work on `stream`
 *   (a cudaStream_t passed as void*, NULL = legacy default stream) and
 *   returns immediately.  The library is stateless and thread-safe; the
 *   only per-thread state is the text of the last error.
 *
 * ERRORS
 *   Every entry point returns a vf_status.  VF_EINVAL: invalid argument
 *   (window even or < 3, H or W < 1, window > min(H, W), B < 1, NULL
 *   img/out, input and output ranges overlap, criterion/variant out of range,
 *   VF_MINIMAX_POLY4 with a criterion other than VF_EXP/VF_AMNFE/VF_AMNFG,
 *   VF_MINIMAX_REACH with one other than VF_EXP/VF_LOG, a row band that does
 *   not cover the rows the output stripe reads).  VF_EUNSUPPORTED: an odd
 *   window >= 7 (valid, not compiled).  VF_ECUDA: a CUDA launch/copy error
 *   (details from vf_last_error()).  No exception crosses the ABI.  On error
 *   nothing has been enqueued.
 */
#ifndef VF_H_
#define VF_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define VF_API __attribute__((visibility("default")))
#else
#define VF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* criterion: the pairwise ordering criteria of the order-statistics filter
 * (0-2), or one of the paper's other two filters (3-5):
 *   VF_AMNFE / VF_AMNFG  AMNF of Eq. 8 with the exponential /
 *                        Gaussian kernel: a weighted average, output rounded
 *                        half away from zero; exp exact (expf) or the
 *                        Table 3 rational (VF_MINIMAX) / Table 2 p=4
 *                        (VF_MINIMAX_POLY4), cutoff T = 10;
 *                        `aggregates` [..][n]: the 3 unrounded output channels
 *                        then zeros; `index`: the centre index.
 *   VF_EVMF              EVMF of Eq. 9: L2 vector median when
 *                        P_C > beta_C, else the centre; ENT exact (logf) or
 *                        Table 4 with cutoff T = 0.05; `aggregates`:
 *                        the median's sums R_i = sum_j |x_i - x_j|_2; `index`:
 *                        selected sample, bit 7 set iff the switch fired. */
typedef enum { VF_ANGULAR = 0, VF_EXP = 1, VF_LOG = 2, VF_AMNFE = 3, VF_AMNFG = 4, VF_EVMF = 5 } vf_criterion;
typedef enum { VF_EXACT = 0, VF_MINIMAX = 1, VF_MINIMAX_POLY4 = 2, VF_MINIMAX_REACH = 3 } vf_variant;
typedef enum { VF_OK = 0, VF_EINVAL = -1, VF_EUNSUPPORTED = -2, VF_ECUDA = -3 } vf_status;

/* Kernel selection for the angular criterion (both variants are window
 * independent, so pairs may be shared between overlapping windows,
 * SURVEY.md 8(f1)).  VF_ALGO_AUTO picks the fastest; results are identical
 * within the parity tolerance either way.  VF_ALGO_NO_TMA (or-ed in) keeps the
 * exp/log criteria on the plain-load kernel instead of the persistent
 * TMA-staged one (which needs 16-byte aligned rows: 3W % 16 == 0, a 16-byte
 * aligned base and batch stride); the two give bit-identical results. */
typedef enum {
  VF_ALGO_AUTO = 0,     /* fastest measured choice                                              */
  VF_ALGO_WINDOW = 1,   /* angular: one thread per window, all n(n-1)/2 pairs                    */
  VF_ALGO_SHARED = 2,   /* angular: pairs shared across windows, per-window accumulation         */
  VF_ALGO_ROLE = 3,     /* angular 5x5: pairs shared, per-pixel role sums (the 5x5 default)      */
  VF_ALGO_NO_TMA = 16,
  VF_ALGO_STREAM = 32   /* angular 3x3 minimax: warp-streamed pair sharing + role sums (the 3x3
                           minimax default under VF_ALGO_AUTO; or-ed in, it forces that kernel) */
} vf_algo;

/* One image.  img, out: device [H][W][3]; index: device [H][W] or NULL;
 * aggregates: device [H][W][n] or NULL. */
VF_API int vf_filter(const uint8_t *img, int H, int W, int window, int criterion, int variant,
              uint8_t *out, uint8_t *index, float *aggregates, void *stream);

/* Dense batch of B images of equal size: imgs, outs device [B][H][W][3];
 * index [B][H][W]; aggregates [B][H][W][n]. */
VF_API int vf_filter_batch(const uint8_t *imgs, int B, int H, int W, int window, int criterion,
                    int variant, uint8_t *outs, uint8_t *index, float *aggregates, void *stream);

/* Row stripe of one H x W image (the spatial partitioner's call).
 * band: device pointer to global rows [band_row0, band_row0 + band_rows)
 * (stride 3W).  Writes global output rows [out_row0, out_row0 + out_rows)
 * to out (device [out_rows][W][3]; index [out_rows][W]; aggregates
 * [out_rows][W][n]).  Border clamping uses the GLOBAL image rows [0, H); the
 * band must contain every clamped row the stripe reads, i.e.
 * band_row0 <= max(out_row0 - w/2, 0) and
 * band_row0 + band_rows >= min(out_row0 + out_rows + w/2, H). */
VF_API int vf_filter_rows(const uint8_t *band, int band_row0, int band_rows, int H, int W,
                   int out_row0, int out_rows, int window, int criterion, int variant,
                   uint8_t *out, uint8_t *index, float *aggregates, void *stream);

/* As vf_filter_batch with an explicit kernel choice: algo = a vf_algo value,
 * optionally | (t << 2) with t in 1..3 forcing the tile height (pixel rows
 * per thread) instead of the size-based choice: t pixels per thread of the
 * angular sharing kernel's region, output rows per thread of the 3x3 exp/log
 * kernel (t = 1, 2, 3 -> 1, 2, 4 rows).  Results are identical within the parity tolerance for every
 * choice (tested); the knob exists for tuning and tests. */
VF_API int vf_filter_batch_algo(const uint8_t *imgs, int B, int H, int W, int window, int criterion,
                         int variant, int algo, uint8_t *outs, uint8_t *index,
                         float *aggregates, void *stream);

/* End-to-end call with HOST buffers: h_imgs and h_outs are host [B][H][W][3]
 * (pinned memory gives asynchronous copies); d_workspace is a caller-owned
 * device buffer of at least vf_host_workspace_bytes(B, H, W) bytes.  Enqueues
 * H2D copy -> filter -> D2H copy on `stream`; the caller synchronises the
 * stream before reading h_outs. */
VF_API size_t vf_host_workspace_bytes(int B, int H, int W);
VF_API int vf_filter_host(const uint8_t *h_imgs, int B, int H, int W, int window, int criterion,
                   int variant, uint8_t *h_outs, void *d_workspace, size_t workspace_bytes,
                   void *stream);

/* Introspection: the kernel the library would launch for vf_filter_batch_algo
 * with these arguments (no device work).  name: its (mangled) function name,
 * written as a NUL-terminated string of at most name_cap bytes (nullable);
 * launch: nullable long long[7] = {grid x, y, z, block x, y, z, dynamic smem
 * bytes}.  Used to match profiler records to (criterion, variant).  Errors as
 * vf_filter_batch_algo's argument checks; VF_ECUDA if the name is unavailable. */
VF_API int vf_kernel_info(int B, int H, int W, int window, int criterion, int variant, int algo, char *name,
                          int name_cap, long long *launch);

/* PLAN (executor): n filters of the same input, built once as an
 * instantiated CUDA graph whose n kernel nodes are independent (they run
 * concurrently, so small images fill the GPU), optionally preceded by an H2D
 * copy node (h_in != NULL: host [B][H][W][3] -> d_in) and followed by n D2H
 * copy nodes (h_outs != NULL: d_outs[i] -> h_outs[i]).  All pointers are fixed
 * at creation (device buffers d_in, d_outs[i] of [B][H][W][3]; host buffers
 * should be pinned) and must stay valid while the plan is used.
 * vf_plan_launch enqueues the whole graph on `stream`.  criteria[i],
 * variants[i] as in vf_filter; n in [1, 64]. */
typedef struct vf_plan_s *vf_plan;
VF_API int vf_plan_create(vf_plan *plan, int B, int H, int W, int window, int n, const int *criteria,
                          const int *variants, const uint8_t *d_in, uint8_t *const *d_outs,
                          const uint8_t *h_in, uint8_t *const *h_outs);
/* As vf_plan_create, plus the paper's fidelity measures of approximate vs exact
 * filters (the bench's per-step statistics) computed by the plan:
 * refs (host int[n], nullable): refs[i] = j compares filter i's output with
 * filter j's (its reference, j != i), -1 = no comparison.  The comparisons
 * are numbered k = 0, 1, ... in increasing i; d_stats (device double
 * [ncmp][B][8], non-NULL when any refs[i] >= 0, not overlapping the images)
 * receives, at every launch, row [k][b] exactly as vf_image_stats_multi(
 * d_outs[refs[i]], {d_outs[i]}) would write it for image b -- bit-identical:
 * both sum the same per-pixel fixed-point values.  The graph zeroes d_stats,
 * runs one statistics node per reference (its comparisons, <= 8 per node: the
 * reference is read and its CIELAB evaluated once) after the kernel nodes
 * writing its inputs -- so it overlaps the other filters' nodes -- and a
 * finalize node.  (Measured: computing the comparisons inside the fused
 * filter kernels' epilogues is slower -- the exp/log node is issue-bound --
 * DESIGN.md 5.3.5.)
 * Errors: VF_EINVAL as vf_plan_create, for refs[i] outside [-1, n) or == i,
 * or a NULL / overlapping d_stats.  (ABI 105.) */
VF_API int vf_plan_create_ex(vf_plan *plan, int B, int H, int W, int window, int n, const int *criteria,
                             const int *variants, const uint8_t *d_in, uint8_t *const *d_outs,
                             const uint8_t *h_in, uint8_t *const *h_outs, const int *refs, double *d_stats);
VF_API int vf_plan_launch(vf_plan plan, void *stream);
/* Number of kernel nodes of a plan (>= 1; VF_EINVAL for an invalid plan).  Plans
 * of at least 2^21 pixels fuse their exp/log filters into one node (they share
 * the L1 distances and S1, readings R2/R3) and their 3x3 angular exact and
 * minimax filters into one node (one pair-geometry evaluation for both
 * variants); outputs are bit-identical to the single-filter kernels; the
 * environment variable VF_PLAN_FUSE=0 disables fusion.  A large plan of the 7
 * paper filters has 3 kernel nodes (the angular node's remainder strips are a
 * second node); with statistics (vf_plan_create_ex) the count includes the
 * statistics nodes and the finalize node (the paper grouping: 3 + 3 + 1). */
VF_API int vf_plan_kernels(vf_plan plan);
VF_API int vf_plan_destroy(vf_plan plan);

/* Per-image fidelity statistics of two device image batches a, b
 * ([B][H][W][3]); stats: device double [B][8] =
 *   {pixels with a != b, sum |a-b| (all channels), sum (a-b)^2,
 *    sum |a_Lab - b_Lab|_2, sum |a_Lab|_2, max |a-b|, 0, 0}
 * (MAE/MSE/NCD of P:286-293; CIELAB via sRGB/D65, evaluated in fp32 per
 * pixel and summed exactly in 2^-23 fixed point).  Overwrites stats. */
VF_API int vf_image_stats(const uint8_t *a, const uint8_t *b, int B, int H, int W, double *stats,
                   void *stream);
/* As vf_image_stats; flags = VF_STATS_NO_REF_NORM (1) skips the reference
 * norm sum stats[.][4] (written as 0): it depends on `a` only, so a caller
 * comparing several outputs with one reference computes it once.  Then a's
 * CIELAB is only evaluated where a != b.  Other flags: VF_EINVAL. */
#define VF_STATS_NO_REF_NORM 1
VF_API int vf_image_stats_ex(const uint8_t *a, const uint8_t *b, int B, int H, int W, double *stats, int flags,
                             void *stream);

/* ONE pass over the reference a comparing it with nb outputs bs[0..nb-1]
 * (host array of nb device pointers, each [B][H][W][3]; 1 <= nb <= 8):
 * stats = device double [nb][B][8], row [k][i] exactly as vf_image_stats(a, bs[k])
 * would write it for image i (column 4, the reference norm, is computed once
 * and written into every row unless flags = VF_STATS_NO_REF_NORM).  Each
 * reference pixel is read once and its CIELAB evaluated at most once, so
 * comparing the 7 filters of a step against one reference costs one pass
 * instead of 7.  Deterministic: every pixel's fp32 CIELAB norm / distance is
 * rounded to 2^-23 fixed point and the sums are integers (64-bit atomics), so
 * results are bit-identical run to run and across kernels (vf_image_stats /
 * _ex call this with nb = 1; plans with statistics produce the same bits).
 * The first statistics call (or plan with statistics) on a device allocates
 * and fills a 1 KB sRGB decoding table there (cudaMalloc + cudaMemcpy, kept
 * for the process), so that first call must not be inside a stream capture.
 * Errors: VF_EINVAL for NULL pointers, nb outside [1, 8], bad sizes or
 * unknown flags; VF_ECUDA if the table cannot be created. */
VF_API int vf_image_stats_multi(const uint8_t *a, const uint8_t *const *bs, int nb, int B, int H, int W,
                                double *stats, int flags, void *stream);

VF_API const char *vf_status_string(int status);
/* Text of the last error on the calling thread ("" if none). */
VF_API const char *vf_last_error(void);
/* ABI version (major*100 + minor): 105 (102: vf_image_stats_ex; 103: vf_image_stats_multi,
 * deterministic statistics, vf_kernel_info; 104: vf_plan_kernels, fused exp/log plan nodes;
 * 105: vf_plan_create_ex (plan statistics), per-pixel fixed-point statistics sums). */
VF_API int vf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VF_H_ */
