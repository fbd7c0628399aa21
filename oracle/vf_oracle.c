/*
 * vf_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * order-statistics vector filters of Celebi, Kingravi, Lukac, Celiker,
 * "Cost-Effective Implementation of Order-Statistics Based Vector Filters
 * Using Minimax Approximations" (arXiv 1009.0959, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1009_0959_b200/) never imports, links or calls it,
 * and it shares no code, header, table or constant generator with the CUDA
 * path: every coefficient below is the paper's printed decimal string.
 *
 * Arithmetic: IEEE double for all real-valued quantities, int64 for all
 * geometry (dot products, squared norms, L1 distances), glibc libm for the
 * exact elementary functions.  Compiled with -O2 -ffp-contract=off (no
 * fast-math, no FMA contraction).
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n,
 * "R<k>" = the reading numbered k in DESIGN.md section 2.
 *
 * Parity status of every exported function is listed in DESIGN.md section 4
 * (all are pinned by tests in tests/test_oracle_*.py; none is "parity
 * unpinned").
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_API __attribute__((visibility("default")))

enum { CRIT_ANGULAR = 0, CRIT_EXP = 1, CRIT_LOG = 2 };
enum { VAR_EXACT = 0, VAR_MINIMAX = 1, VAR_MINIMAX_POLY4 = 2, VAR_MINIMAX_REACH = 3 };

/* ---- Table 1: fourth degree minimax polynomials ------------ */
/* ARCSIN row: fitted to g(tau) = 2 arcsin(tau/sqrt 2) on
 * [0, 1/sqrt 2] (Eq. 7; reading R6/R7).                          */
static const double T1_ARCSIN[5] = {2.097797e-05, 1.412840, 1.429881e-02,
                                    6.704361e-02, 6.909677e-02};
/* ARCCOS row: arccos(z) on [0, 0.5].                                 */
static const double T1_ARCCOS[5] = {1.570786, -9.990285e-01, -1.429899e-02,
                                    -9.481335e-02, -1.381942e-01};
/* ---- Table 2: minimax polynomials for exp(-z) on [0, 10] --- */
static const double T2_P2[3] = {8.214528e-01, -3.186948e-01, 2.544088e-02};
static const double T2_P3[4] = {9.174126e-01, -5.631179e-01, 1.015041e-01,
                                -5.519183e-03};
static const double T2_P4[5] = {9.666313e-01, -7.620584e-01, 2.145386e-01,
                                -2.509526e-02, 1.032877e-03};
/* ---- Table 3: 4/4 minimax rational for exp(-z) on [0, 10] - */
static const double T3_NUM[5] = {3.206619e-02, -1.195191e-02, 1.756974e-03,
                                 -1.199261e-04, 3.182685e-06};
static const double T3_DEN[5] = {3.206627e-02, 2.011147e-02, 5.853684e-03,
                                 9.780143e-04, 1.251598e-04};
/* ---- Table 4: 4/4 minimax rational for z ln z on [0.05, 1] - */
static const double T4_NUM[5] = {-1.519742e-04, -6.835769e-02, -8.856923e-01,
                                 -5.369609e-01, 1.491165};
static const double T4_DEN[5] = {1.532270e-02, 3.987796e-01, 1.461793,
                                 6.827004e-01, -4.469776e-02};

/* ---- Re-derived minimax polynomials on the reachable arguments --------- *
 * (VAR_MINIMAX_REACH.)  Computed by the Remez exchange of
 * P:70 (oracle/minimax.py, tools/remez_reach.py -> tests/golden/
 * remez_reach.txt, which these decimal strings repeat) for the criterion
 * values themselves on the intervals the triangle-inequality bounds allow
 * (DESIGN.md section 2):
 *   D_E(z) = 1 - exp(-z) on [0, z*_25 = 0.7421166...], degree 5, eps 7.86e-8
 *   D_L(u) = -(1 - u) ln(1 - u) on [0, 1 - 1/e], degree 7, eps 2.95e-7
 * (u = 1 - s, s the ENT argument of reading R3).                            */
static const double R_EXP[6] = {7.8607071043670362e-08, 0.99999223556347028, -0.49987553301909632,
                                0.16593299907325132, -0.039686762479510071, 0.0057878343103810199};
static const double R_LOG[8] = {2.951515920989309e-07, 0.99994488204903353, -0.49831625626187054,
                                -0.18607535607515613, 0.02447556559350492, -0.36382847261870294,
                                0.43713641586762925, -0.32653163848077049};

static const double T_EXP = 10.0;  /* EXP cutoff                     */
static const double T_ENT = 0.05;  /* ENT cutoff                     */
static const double KAPPA = 0.33;  /* kernel-width scaling factor    */

/* Horner-scheme evaluation a_0 + a_1 z + ... + a_deg z^deg. */
static double horner(const double *a, int deg, double z)
{
    double r = a[deg];
    for (int k = deg - 1; k >= 0; --k)
        r = r * z + a[k];
    return r;
}

/* ---- scalar elementary functions and their approximants ----------------- */

/* Composite minimax arccos of Eqs. 6-7 in the cosine z:
 * z < 0.5 -> ARCCOS polynomial; z >= 0.5 -> ARCSIN-row polynomial in
 * tau = sqrt(1 - z) ("for z >= 0.5"; reading R5).                      */
static double arccos_mm(double z)
{
    if (z < 0.5)
        return horner(T1_ARCCOS, 4, z);
    return horner(T1_ARCSIN, 4, sqrt(1.0 - z));
}

/* EXP approximants with the P:163 cutoff: 0 outside [0, T].                 */
static double exp_mm_rational(double z)
{
    if (z > T_EXP || z < 0.0)
        return 0.0;
    return horner(T3_NUM, 4, z) / horner(T3_DEN, 4, z);
}

static double exp_mm_poly(double z, int p)
{
    if (z > T_EXP || z < 0.0)
        return 0.0;
    if (p == 2) return horner(T2_P2, 2, z);
    if (p == 3) return horner(T2_P3, 3, z);
    return horner(T2_P4, 4, z);
}

/* ENT(z) = z ln z (natural log, reading R10), exact with ENT(0) = 0.        */
static double ent_exact(double z)
{
    return z > 0.0 ? z * log(z) : 0.0;
}

/* ENT approximant with the P:232 cutoff: 0 for arguments below T.           */
static double ent_mm(double z)
{
    if (z < T_ENT)
        return 0.0;
    return horner(T4_NUM, 4, z) / horner(T4_DEN, 4, z);
}

/* ---- pairwise criteria -------------------------------------------------- */

/* Angular criterion A(x_i, x_j) of Eq. 5.
 * c = x_i.x_j / (|x_i|_2 |x_j|_2).  For c < 0.5 (decided exactly in
 * integers: 4 D^2 < |x_i|^2 |x_j|^2) arccos is evaluated directly; for
 * c >= 0.5 Eq. 6 is used, arccos c = 2 arcsin(sqrt(0.5 (1 - c))),
 * where 1 - c = X / (s (s + D)) with X = |x_i|^2|x_j|^2 - D^2 = |x_i x x_j|^2
 * (Lagrange identity, exact in int64) and s = |x_i||x_j| -- the same value
 * without cancellation.  The minimax variant uses Table 1: ARCCOS row on c,
 * ARCSIN row on tau = sqrt(1 - c) (Eq. 7).  Zero-norm vectors give 0 (S:342,
 * reading R4).                                                              */
static double pair_angular(const int64_t *a, const int64_t *b, int var)
{
    int64_t nna = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
    int64_t nnb = b[0] * b[0] + b[1] * b[1] + b[2] * b[2];
    if (nna == 0 || nnb == 0)
        return 0.0;
    int64_t D = a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
    int64_t P = nna * nnb;          /* <= 195075^2 < 2^36          */
    int64_t X = P - D * D;          /* >= 0 by Cauchy-Schwarz      */
    double s = sqrt((double)P);     /* exact integer < 2^53 -> one rounding */
    if (4 * D * D < P) {            /* c < 0.5                      */
        double c = (double)D / s;
        return var == VAR_EXACT ? acos(c) : horner(T1_ARCCOS, 4, c);
    }
    double one_minus_c = (double)X / (s * (s + (double)D));
    if (var == VAR_EXACT)
        return 2.0 * asin(sqrt(0.5 * one_minus_c));          /* Eq. 6 */
    return horner(T1_ARCSIN, 4, sqrt(one_minus_c));          /* Eq. 7 */
}

/* ---- one window ---------------------------------------------------------- */

#define NMAX 49   /* windows up to 7x7 */

/* Pairwise criterion matrix Dm (n x n, symmetric, zero diagonal) of one
 * window of n samples (uint8 RGB, raster order of Fig. 1).
 *
 * Exp criterion (reading R2): Eq. 8's bandwidths
 *   h_i = n^(-kappa/3) sum_j |x_i - x_j|_1           (kappa P:161)
 * their window mean h_W = (1/n) sum_i h_i, and the AMNFE kernel
 * K = exp(-|.|_1) applied to z_ij = |x_i - x_j|_1 / h_W:
 *   D_E(i,j) = 1 - exp(-z_ij)       exact
 *   D_E(i,j) = 1 - E(z_ij)          E = Table 3 rational (or Table 2 p=4),
 *                                   0 for z > T = 10.
 * Log criterion (reading R3): q_ij = (n-1) |x_i - x_j|_1 / sum_{k<l} |x_k - x_l|_1,
 *   s_ij = 1 - (1 - 1/e) q_ij,  D_L(i,j) = -ENT(s_ij),
 *   ENT exact = s ln s, ENT minimax = Table 4 rational (0 below T = 0.05,
 *   P:232).
 * Flat window (all L1 distances zero): every D = 0 (reading R18).            */
static void window_matrix(const uint8_t *smp, int n, int crit, int var, double *Dm)
{
    int64_t x[NMAX][3];
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k)
            x[i][k] = smp[3 * i + k];
    for (int i = 0; i < n * n; ++i)
        Dm[i] = 0.0;

    if (crit == CRIT_ANGULAR) {
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) {
                double d = pair_angular(x[i], x[j], var);
                Dm[i * n + j] = d;
                Dm[j * n + i] = d;
            }
        return;
    }

    int64_t d1[NMAX][NMAX];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            int64_t s = 0;
            for (int k = 0; k < 3; ++k)
                s += x[i][k] > x[j][k] ? x[i][k] - x[j][k] : x[j][k] - x[i][k];
            d1[i][j] = s;
        }

    if (crit == CRIT_EXP) {
        double nk = pow((double)n, -KAPPA / 3.0);
        double hsum = 0.0;
        for (int i = 0; i < n; ++i) {
            int64_t row = 0;
            for (int j = 0; j < n; ++j)
                row += d1[i][j];
            double h_i = nk * (double)row;                     /* Eq. 8 */
            hsum += h_i;
        }
        double h_W = hsum / (double)n;
        if (h_W == 0.0)
            return;                                            /* flat window */
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) {
                double z = (double)d1[i][j] / h_W;
                double d;
                if (var == VAR_EXACT)
                    d = 1.0 - exp(-z);
                else if (var == VAR_MINIMAX)
                    d = 1.0 - exp_mm_rational(z);
                else if (var == VAR_MINIMAX_POLY4)
                    d = 1.0 - exp_mm_poly(z, 4);
                else
                    d = horner(R_EXP, 5, z);                   /* f4: D_E itself */
                Dm[i * n + j] = d;
                Dm[j * n + i] = d;
            }
        return;
    }

    /* CRIT_LOG */
    int64_t S1 = 0;
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j)
            S1 += d1[i][j];
    if (S1 == 0)
        return;                                                /* flat window */
    const double a = 1.0 - exp(-1.0);
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            double q = (double)(n - 1) * (double)d1[i][j] / (double)S1;
            double s = 1.0 - a * q;
            double d = var == VAR_EXACT ? -ent_exact(s)
                     : var == VAR_MINIMAX ? -ent_mm(s)
                     : horner(R_LOG, 7, a * q);                /* f4: D_L(u), u = 1 - s */
            Dm[i * n + j] = d;
            Dm[j * n + i] = d;
        }
}

/* Aggregates R_i = sum_{j != i} D(i,j) and the argmin of Eq. 5, the
 * lowest raster index winning exact ties (reading R3b).  The j = i
 * term of Eq. 5 is excluded (reading R17).                                  */
static int window_eval(const uint8_t *smp, int n, int crit, int var, double *R, double *Dm_out)
{
    double Dm[NMAX * NMAX];
    window_matrix(smp, n, crit, var, Dm);
    int best = 0;
    for (int i = 0; i < n; ++i) {
        double r = 0.0;
        for (int j = 0; j < n; ++j)
            if (j != i)
                r += Dm[i * n + j];
        R[i] = r;
        if (r < R[best])
            best = i;
    }
    if (Dm_out)
        memcpy(Dm_out, Dm, sizeof(double) * (size_t)n * (size_t)n);
    return best;
}

/* Window W(y,x) of side w, raster re-indexed (Fig. 1), replicate
 * padding at the borders (reading R2b).                               */
static void gather_window(const uint8_t *img, int H, int W, int w, int y, int x, uint8_t *smp)
{
    int r = w / 2, k = 0;
    for (int dy = 0; dy < w; ++dy) {
        int yy = y + dy - r;
        yy = yy < 0 ? 0 : (yy > H - 1 ? H - 1 : yy);
        for (int dx = 0; dx < w; ++dx) {
            int xx = x + dx - r;
            xx = xx < 0 ? 0 : (xx > W - 1 ? W - 1 : xx);
            const uint8_t *p = img + ((size_t)yy * (size_t)W + (size_t)xx) * 3;
            smp[3 * k + 0] = p[0];
            smp[3 * k + 1] = p[1];
            smp[3 * k + 2] = p[2];
            ++k;
        }
    }
}

static int check_args(int H, int W, int window, int crit, int var)
{
    if (H < 1 || W < 1) return -1;
    if (window < 3 || window % 2 == 0 || window * window > NMAX) return -1;
    if (window > H || window > W) return -1;
    if (crit < 0 || crit > 2) return -1;
    if (var < 0 || var > 3) return -1;
    if (var == VAR_MINIMAX_POLY4 && crit != CRIT_EXP) return -1;
    if (var == VAR_MINIMAX_REACH && crit == CRIT_ANGULAR) return -1;
    return 0;
}

/* ======================= exported entry points ========================= */

/* Full image: out (H*W*3), optional index (H*W, 0..n-1), optional
 * aggregates (H*W*n doubles, [y][x][k]).  Returns 0, or -1 on bad args.    */
ORACLE_API int oracle_filter(const uint8_t *img, int H, int W, int window, int crit, int var,
                             uint8_t *out, uint8_t *index, double *agg, int nthreads)
{
    if (check_args(H, W, window, crit, var) != 0 || !img || !out)
        return -1;
    int n = window * window;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int y = 0; y < H; ++y) {
        uint8_t smp[NMAX * 3];
        double R[NMAX];
        for (int x = 0; x < W; ++x) {
            gather_window(img, H, W, window, y, x, smp);
            int k = window_eval(smp, n, crit, var, R, NULL);
            size_t p = (size_t)y * (size_t)W + (size_t)x;
            out[3 * p + 0] = smp[3 * k + 0];
            out[3 * p + 1] = smp[3 * k + 1];
            out[3 * p + 2] = smp[3 * k + 2];
            if (index)
                index[p] = (uint8_t)k;
            if (agg)
                memcpy(agg + p * (size_t)n, R, sizeof(double) * (size_t)n);
        }
    }
    (void)nthreads;
    return 0;
}

/* Sampled pixels (ys[i], xs[i]) of a full image; outputs are per sample.   */
ORACLE_API int oracle_filter_pixels(const uint8_t *img, int H, int W, int window, int crit, int var,
                                    const int32_t *ys, const int32_t *xs, int64_t npix,
                                    uint8_t *out, uint8_t *index, double *agg, int nthreads)
{
    if (check_args(H, W, window, crit, var) != 0 || !img || !out)
        return -1;
    int n = window * window;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
    for (int64_t i = 0; i < npix; ++i) {
        uint8_t smp[NMAX * 3];
        double R[NMAX];
        int y = ys[i], x = xs[i];
        if (y < 0 || y >= H || x < 0 || x >= W)
            continue;
        gather_window(img, H, W, window, y, x, smp);
        int k = window_eval(smp, n, crit, var, R, NULL);
        out[3 * i + 0] = smp[3 * k + 0];
        out[3 * i + 1] = smp[3 * k + 1];
        out[3 * i + 2] = smp[3 * k + 2];
        if (index)
            index[i] = (uint8_t)k;
        if (agg)
            memcpy(agg + i * (size_t)n, R, sizeof(double) * (size_t)n);
    }
    (void)nthreads;
    return 0;
}

/* One window given as n raw samples: aggregates R (n), optional full
 * criterion matrix Dm (n*n).  Returns k* (lowest-index argmin) or -1.       */
ORACLE_API int oracle_window(const uint8_t *samples, int n, int crit, int var, double *R, double *Dm)
{
    if (n < 2 || n > NMAX || crit < 0 || crit > 2 || var < 0 || var > 3)
        return -1;
    if ((var == VAR_MINIMAX_POLY4 && crit != CRIT_EXP) || (var == VAR_MINIMAX_REACH && crit == CRIT_ANGULAR))
        return -1;
    return window_eval(samples, n, crit, var, R, Dm);
}

ORACLE_API int oracle_gather_window(const uint8_t *img, int H, int W, int window, int y, int x,
                                    uint8_t *samples)
{
    if (H < 1 || W < 1 || window < 1 || window % 2 == 0 || window * window > NMAX)
        return -1;
    gather_window(img, H, W, window, y, x, samples);
    return 0;
}

/* Angular criterion of one pair (x, y each 3 uint8).                      */
ORACLE_API double oracle_pair_angular(const uint8_t *a, const uint8_t *b, int var)
{
    int64_t x[3] = {a[0], a[1], a[2]}, y[3] = {b[0], b[1], b[2]};
    return pair_angular(x, y, var);
}

/* Scalar functions on arrays, for certification against the paper's
 * epsilons (Tables 1-4) and the SPEC examples.                             */
enum {
    FN_ARCCOS_EXACT = 0,  /* acos(z)                                      */
    FN_ARCCOS_MM = 1,     /* composite of Eqs. 6-7 in z                   */
    FN_P_ARCCOS = 2,      /* Table 1 ARCCOS polynomial                    */
    FN_P_ARCSIN = 3,      /* Table 1 ARCSIN polynomial (in tau)           */
    FN_EXP_EXACT = 4,     /* exp(-z)                                      */
    FN_EXP_RATIONAL = 5,  /* Table 3 with cutoff                          */
    FN_EXP_POLY2 = 6,     /* Table 2 p=2 with cutoff                      */
    FN_EXP_POLY3 = 7,
    FN_EXP_POLY4 = 8,
    FN_ENT_EXACT = 9,     /* z ln z                                       */
    FN_ENT_MM = 10,       /* Table 4 with cutoff                          */
    FN_EXP_REACH = 11,    /* f4: D_E(z) polynomial (no cutoff)            */
    FN_LOG_REACH = 12,    /* f4: D_L(u) polynomial                        */
};

ORACLE_API int oracle_eval(int fn, const double *z, int64_t n, double *out)
{
    for (int64_t i = 0; i < n; ++i) {
        double v = z[i], r;
        switch (fn) {
        case FN_ARCCOS_EXACT: r = acos(v); break;
        case FN_ARCCOS_MM: r = arccos_mm(v); break;
        case FN_P_ARCCOS: r = horner(T1_ARCCOS, 4, v); break;
        case FN_P_ARCSIN: r = horner(T1_ARCSIN, 4, v); break;
        case FN_EXP_EXACT: r = exp(-v); break;
        case FN_EXP_RATIONAL: r = exp_mm_rational(v); break;
        case FN_EXP_POLY2: r = exp_mm_poly(v, 2); break;
        case FN_EXP_POLY3: r = exp_mm_poly(v, 3); break;
        case FN_EXP_POLY4: r = exp_mm_poly(v, 4); break;
        case FN_ENT_EXACT: r = ent_exact(v); break;
        case FN_ENT_MM: r = ent_mm(v); break;
        case FN_EXP_REACH: r = horner(R_EXP, 5, v); break;
        case FN_LOG_REACH: r = horner(R_LOG, 7, v); break;
        default: return -1;
        }
        out[i] = r;
    }
    return 0;
}

/* The oracle's coefficient tables, for comparison with tests/golden/.     */
ORACLE_API int oracle_coeffs(int table, double *out)
{
    const double *t; int m;
    switch (table) {
    case 0: t = T1_ARCSIN; m = 5; break;
    case 1: t = T1_ARCCOS; m = 5; break;
    case 2: t = T2_P2; m = 3; break;
    case 3: t = T2_P3; m = 4; break;
    case 4: t = T2_P4; m = 5; break;
    case 5: t = T3_NUM; m = 5; break;
    case 6: t = T3_DEN; m = 5; break;
    case 7: t = T4_NUM; m = 5; break;
    case 8: t = T4_DEN; m = 5; break;
    case 9: out[0] = T_EXP; out[1] = T_ENT; out[2] = KAPPA; return 3;
    case 10: t = R_EXP; m = 6; break;
    case 11: t = R_LOG; m = 8; break;
    default: return -1;
    }
    memcpy(out, t, sizeof(double) * (size_t)m);
    return m;
}

/* ======================= the paper's AMNF and EVMF filters ================ *
 * SURVEY.md 8(f2)-(f3).  Same window engine (Fig. 1, replicate border).      */

enum { FILT_AMNFE = 3, FILT_AMNFG = 4, FILT_EVMF = 5 };

/* AMNF, Eq. 8:
 *   y = sum_i x_i w_i / sum_j w_j,  w_i = h_i^-3 K((x_C - x_i) / h_i),
 *   h_i = n^(-kappa/3) sum_j |x_i - x_j|_1,  kappa = 0.33,
 *   AMNFE: K(x) = exp(-|x|_1)  ->  K = exp(-|x_C - x_i|_1 / h_i)
 *   AMNFG: K(x) = exp(-0.5 |x|_2^2) -> K = exp(-0.5 |x_C - x_i|_2^2 / h_i^2)
 * exp evaluated exactly (libm) or by Table 3 (VAR_MINIMAX) / Table 2 p = 4
 * (VAR_MINIMAX_POLY4), both with the P:163 cutoff.  Output rounded to nearest,
 * half away from zero, clamped to [0, 255].  Degenerate
 * windows (some h_i = 0, i.e. all samples equal, or sum w = 0) return x_C
 * (S:343).  aux (n + 3 doubles): v[3] unrounded output, w_i / sum w.        */
static int amnf_window(const uint8_t *smp, int n, int gauss, int var, uint8_t *out, double *aux)
{
    int C = (n - 1) / 2;
    int64_t x[NMAX][3];
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k)
            x[i][k] = smp[3 * i + k];
    double nk = pow((double)n, -KAPPA / 3.0);
    double h[NMAX], w[NMAX];
    int degenerate = 0;
    for (int i = 0; i < n; ++i) {
        int64_t row = 0;
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < 3; ++k)
                row += x[i][k] > x[j][k] ? x[i][k] - x[j][k] : x[j][k] - x[i][k];
        h[i] = nk * (double)row;                                   /* Eq. 8 */
        if (h[i] == 0.0)
            degenerate = 1;
    }
    double sw = 0.0;
    if (!degenerate) {
        for (int i = 0; i < n; ++i) {
            int64_t l1 = 0, l2 = 0;
            for (int k = 0; k < 3; ++k) {
                int64_t d = x[C][k] - x[i][k];
                l1 += d < 0 ? -d : d;
                l2 += d * d;
            }
            double z = gauss ? 0.5 * (double)l2 / (h[i] * h[i]) : (double)l1 / h[i];
            double K;
            if (var == VAR_EXACT)
                K = exp(-z);
            else if (var == VAR_MINIMAX)
                K = exp_mm_rational(z);
            else
                K = exp_mm_poly(z, 4);
            w[i] = K / (h[i] * h[i] * h[i]);                       /* h_i^-3 K */
            sw += w[i];
        }
        if (sw == 0.0)
            degenerate = 1;
    }
    if (degenerate) {
        for (int k = 0; k < 3; ++k) {
            out[k] = (uint8_t)x[C][k];
            if (aux) aux[k] = (double)x[C][k];
        }
        if (aux)
            for (int i = 0; i < n; ++i) aux[3 + i] = (i == C);
        return 0;
    }
    for (int k = 0; k < 3; ++k) {
        double v = 0.0;
        for (int i = 0; i < n; ++i)
            v += (double)x[i][k] * w[i];
        v /= sw;
        if (aux) aux[k] = v;
        double r = floor(v + 0.5);                                 /* v >= 0: half away from zero */
        out[k] = (uint8_t)(r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r));
    }
    if (aux)
        for (int i = 0; i < n; ++i) aux[3 + i] = w[i] / sw;
    return 0;
}

/* EVMF, Eq. 9:
 *   y = argmin_i sum_j |x_i - x_j|_2 (vector median) if P_C > beta_C, else x_C;
 *   P_i = |x_i - xbar|_2 / sum_j |x_j - xbar|_2,  xbar = window mean,
 *   beta_i = -P_i log P_i / (-sum_j P_j log P_j) = ENT(P_i) / sum_j ENT(P_j),
 *   ENT exact = z ln z (natural log, R10), minimax = Table 4 with the P:232
 *   cutoff (0 below 0.05).  Degenerate: sum_j |x_j - xbar| = 0 ->
 *   identity; sum_j ENT(P_j) = 0 -> beta_C = 0.  Ties of the median: lowest
 *   index.  Returns the selected index (C when the switch does not
 *   fire).  aux (n + 3 doubles): R_i (VMF aggregates), P_C, beta_C, fired.   */
static int evmf_window(const uint8_t *smp, int n, int var, uint8_t *out, double *aux)
{
    int C = (n - 1) / 2;
    int64_t x[NMAX][3];
    double mean[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            x[i][k] = smp[3 * i + k];
            mean[k] += (double)x[i][k];
        }
    for (int k = 0; k < 3; ++k)
        mean[k] /= (double)n;
    double dev[NMAX], S = 0.0;
    for (int i = 0; i < n; ++i) {
        double s2 = 0.0;
        for (int k = 0; k < 3; ++k)
            s2 += ((double)x[i][k] - mean[k]) * ((double)x[i][k] - mean[k]);
        dev[i] = sqrt(s2);
        S += dev[i];
    }
    double R[NMAX];
    for (int i = 0; i < n; ++i) {
        double r = 0.0;
        for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            int64_t d2 = 0;
            for (int k = 0; k < 3; ++k)
                d2 += (x[i][k] - x[j][k]) * (x[i][k] - x[j][k]);
            r += sqrt((double)d2);
        }
        R[i] = r;
    }
    double PC = 0.0, betaC = 0.0;
    int fired = 0;
    if (S > 0.0) {
        double sent = 0.0, entC = 0.0;
        for (int i = 0; i < n; ++i) {
            double P = dev[i] / S;
            double e = var == VAR_EXACT ? ent_exact(P) : ent_mm(P);
            sent += e;
            if (i == C) { entC = e; PC = P; }
        }
        betaC = sent == 0.0 ? 0.0 : entC / sent;
        fired = PC > betaC;
    }
    int sel = C;
    if (fired) {
        sel = 0;
        for (int i = 1; i < n; ++i)
            if (R[i] < R[sel]) sel = i;
    }
    for (int k = 0; k < 3; ++k)
        out[k] = (uint8_t)x[sel][k];
    if (aux) {
        for (int i = 0; i < n; ++i) aux[i] = R[i];
        aux[n] = PC;
        aux[n + 1] = betaC;
        aux[n + 2] = fired;
    }
    return sel;
}

static int paper_window(const uint8_t *smp, int n, int filt, int var, uint8_t *out, double *aux)
{
    if (filt == FILT_EVMF)
        return evmf_window(smp, n, var, out, aux);
    return amnf_window(smp, n, filt == FILT_AMNFG, var, out, aux);
}

static int check_paper_args(int n, int filt, int var)
{
    if (n < 2 || n > NMAX) return -1;
    if (filt < FILT_AMNFE || filt > FILT_EVMF) return -1;
    if (var < 0 || var > 2) return -1;
    if (var == VAR_MINIMAX_POLY4 && filt == FILT_EVMF) return -1;
    return 0;
}

/* One window of n raw samples.  Returns the selected index (EVMF) or 0
 * (AMNF), or -1 on bad args.  out: 3 bytes; aux: n + 3 doubles or NULL.    */
ORACLE_API int oracle_paper_window(const uint8_t *samples, int n, int filt, int var, uint8_t *out, double *aux)
{
    if (check_paper_args(n, filt, var) != 0)
        return -1;
    return paper_window(samples, n, filt, var, out, aux);
}

/* Full image (or sampled pixels when ys/xs != NULL): out (npix*3), optional
 * index (npix, EVMF selection), optional aux (npix*(n+3)).                 */
ORACLE_API int oracle_paper_filter(const uint8_t *img, int H, int W, int window, int filt, int var,
                                   const int32_t *ys, const int32_t *xs, int64_t npix,
                                   uint8_t *out, uint8_t *index, double *aux, int nthreads)
{
    if (H < 1 || W < 1 || window < 3 || window % 2 == 0 || window > H || window > W || !img || !out)
        return -1;
    int n = window * window;
    if (check_paper_args(n, filt, var) != 0)
        return -1;
    int64_t total = ys ? npix : (int64_t)H * W;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 256)
#endif
    for (int64_t i = 0; i < total; ++i) {
        uint8_t smp[NMAX * 3];
        int y = ys ? ys[i] : (int)(i / W), x = xs ? xs[i] : (int)(i % W);
        if (y < 0 || y >= H || x < 0 || x >= W)
            continue;
        gather_window(img, H, W, window, y, x, smp);
        int k = paper_window(smp, n, filt, var, out + 3 * i, aux ? aux + i * (size_t)(n + 3) : NULL);
        if (index)
            index[i] = (uint8_t)k;
    }
    (void)nthreads;
    return 0;
}

ORACLE_API int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
