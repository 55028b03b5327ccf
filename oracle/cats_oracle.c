/*
 * cats_oracle.c -- plain, slow, obviously-correct CPU oracle for the CATS hot path
 * (arXiv 2404.08763). TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library. It shares no source, header, table or helper with the
 * CUDA library under paper_2404_08763_b200/csrc/, and it never includes a CUDA header.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared cats_oracle.c -o libcats_oracle.so -lm
 * (no -ffast-math, no FMA contraction: every sum is a chain of correctly rounded
 * fp64 additions in ascending index order). That serial build is the checker.
 * A second build of the SAME source with -fopenmp (libcats_oracle_omp.so) is used only to time
 * the CPU baseline on all host cores: the `omp parallel for` pragmas below split independent
 * iterations (neurons j for u / v / x1, output columns c for y) across threads and change no
 * summation order, so both builds return identical bits (tests/test_oracle_pins.py checks it).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 *
 * Conventions:
 *   - weights are passed NEURON-MAJOR [m][d]: Wg[j*d+i] is the paper's W_gate[i][j]
 *     (P:196 defines W_gate, W_up in R^{d x m}; W_down in R^{m x d}, so W_down is
 *     already [m][d] and neuron j is its row j; for W_gate/W_up neuron j is column j,
 *     P:204 "the columns of W_up and the rows of W_down are the experts").
 *   - input dtype 0 = IEEE fp32, 1 = bfloat16 (upper 16 bits of an fp32); both widen
 *     exactly to double.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_F32 0
#define ORACLE_BF16 1

/* Exact widening of one stored element to double. */
static double widen(const void *base, uint64_t i, int dtype) {
    if (dtype == ORACLE_F32) {
        return (double)((const float *)base)[i];
    } else {
        uint32_t bits = ((uint32_t)((const uint16_t *)base)[i]) << 16;
        float f;
        memcpy(&f, &bits, sizeof f);
        return (double)f;
    }
}

/* Eq. 2: SiLU(u) = u * sigmoid(u) = u / (1 + e^{-u}).
 * Evaluated in the numerically stable two-branch form: for u < 0,
 * u / (1 + e^{-u}) = u * e^{u} / (1 + e^{u}), which avoids e^{-u} overflow. */
double oracle_silu(double u) {
    if (u >= 0.0) {
        return u / (1.0 + exp(-u));
    } else {
        double e = exp(u);
        return u * e / (1.0 + e);
    }
}

/* Eq. 4: CATS_t keeps x_j iff |x_j| >= t ("≥": ties kept, reading G1).
 * Writes keep[j] in {0,1}. */
void oracle_cats_mask(const double *v, int64_t m, double t, uint8_t *keep) {
    for (int64_t j = 0; j < m; ++j) keep[j] = (fabs(v[j]) >= t) ? 1 : 0;
}

/* The gated MLP with the CATS activation, one token at a time.
 *
 *   Eq. 1:  Gated-MLP(x) = (SiLU(x W_gate) * (x W_up)) W_down
 *   Eq. 5:  CATS_t(SiLU(x W_gate)) replaces SiLU(x W_gate)
 *   Custom GPU Kernel "MLP using CATS":
 *       v <- SiLU(x W_gate); Mask <- |v| >= t; x1 <- (x W_up[Mask]) * v[Mask];
 *       y <- x1 W_down[Mask]
 *
 * mode 0 (ORACLE_SPARSE): the algorithm above literally -- loop only over kept
 *         neurons j in ascending order; y_c = sum_{j kept} x1_j * Wd[j][c].
 * mode 1 (ORACLE_MASKED): App. D eq. for y: y = (v' * (x W'_up)) W'_down,
 *         v' = v with masked entries set to 0, summing over ALL j (zeros included).
 * mode 2 (ORACLE_DENSE):  Eq. 1 with no threshold (every neuron kept).
 *
 * keep_in (nullable, [b][m]): if given, these keep decisions are used instead of
 *         |v| >= t (used by the y-parity rule of DESIGN.md, reading R9).
 * Outputs: y_out [b][d] (fp64), v_out [b][m] (nullable), keep_out [b][m] (nullable).
 * Sums run in ascending index order in fp64. Returns 0, or -1 on bad arguments.
 */
int oracle_mlp(int64_t d, int64_t m, int64_t b, int dtype,
               const void *x, const void *Wg, const void *Wu, const void *Wd,
               double t, int mode, const uint8_t *keep_in,
               double *y_out, double *v_out, uint8_t *keep_out) {
    if (d <= 0 || m <= 0 || b <= 0 || (dtype != ORACLE_F32 && dtype != ORACLE_BF16)) return -1;
    if (mode < 0 || mode > 2) return -1;
    double *xs = (double *)malloc(sizeof(double) * (size_t)d);
    double *v = (double *)malloc(sizeof(double) * (size_t)m);
    uint8_t *keep = (uint8_t *)malloc((size_t)m);
    double *x1 = (double *)malloc(sizeof(double) * (size_t)m);
    if (!xs || !v || !keep || !x1) { free(xs); free(v); free(keep); free(x1); return -1; }

    for (int64_t bt = 0; bt < b; ++bt) {
        for (int64_t i = 0; i < d; ++i) xs[i] = widen(x, (uint64_t)(bt * d + i), dtype);

        /* v <- SiLU(x W_gate) */
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < m; ++j) {
            double u = 0.0;
            for (int64_t i = 0; i < d; ++i) u += xs[i] * widen(Wg, (uint64_t)(j * d + i), dtype);
            v[j] = oracle_silu(u);
        }
        /* Mask <- 1 if |v| >= t else 0 */
        if (keep_in) {
            for (int64_t j = 0; j < m; ++j) keep[j] = keep_in[bt * m + j] ? 1 : 0;
        } else if (mode == 2) {
            for (int64_t j = 0; j < m; ++j) keep[j] = 1;
        } else {
            oracle_cats_mask(v, m, t, keep);
        }
        /* x1 <- (x W_up[Mask]) * v[Mask] */
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < m; ++j) {
            if (mode == 0 && !keep[j]) { x1[j] = 0.0; continue; }
            double up = 0.0;
            for (int64_t i = 0; i < d; ++i) up += xs[i] * widen(Wu, (uint64_t)(j * d + i), dtype);
            double vj = keep[j] ? v[j] : 0.0; /* v' of P:702 */
            x1[j] = vj * up;
        }
        /* y <- x1 W_down[Mask]; each y_c is the ascending-j sum */
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < d; ++c) {
            double acc = 0.0;
            for (int64_t j = 0; j < m; ++j) {
                if (mode == 0 && !keep[j]) continue;
                acc += x1[j] * widen(Wd, (uint64_t)(j * d + c), dtype);
            }
            y_out[bt * d + c] = acc;
        }
        if (v_out) for (int64_t j = 0; j < m; ++j) v_out[bt * m + j] = v[j];
        if (keep_out) for (int64_t j = 0; j < m; ++j) keep_out[bt * m + j] = keep[j];
    }
    free(xs); free(v); free(keep); free(x1);
    return 0;
}

/* App. B: CATS applied to the hidden vector before the attention projections,
 * CATS_t(x) (Eq. 4, applied to x itself: no SiLU), followed by the projection
 * y = CATS_t(x) W, W stored input-major [d_in][d_out] (row i = the weights input i feeds).
 * Per token: keep_i = |x_i| >= t (ties kept, G1); y_n = sum over kept i, ascending, of x_i W[i][n].
 * fp64 accumulation of the exactly widened inputs. keep_out [b][d_in] may be NULL. */
int oracle_xsparse_gemv(int64_t d_in, int64_t d_out, int64_t b, int dtype, const void *x, const void *W,
                        double t, double *y_out, uint8_t *keep_out) {
    if (d_in <= 0 || d_out <= 0 || b <= 0 || (dtype != ORACLE_F32 && dtype != ORACLE_BF16)) return -1;
    for (int64_t bt = 0; bt < b; ++bt) {
        for (int64_t n = 0; n < d_out; ++n) y_out[bt * d_out + n] = 0.0;
        for (int64_t i = 0; i < d_in; ++i) {
            const double xi = widen(x, (uint64_t)(bt * d_in + i), dtype);
            const int keep = fabs(xi) >= t;
            if (keep_out) keep_out[bt * d_in + i] = (uint8_t)keep;
            if (!keep) continue;
            for (int64_t n = 0; n < d_out; ++n) y_out[bt * d_out + n] += xi * widen(W, (uint64_t)(i * d_out + n), dtype);
        }
    }
    return 0;
}

/* Eq. 3 rank: t = min{t' : F(t') >= k}, F the empirical CDF of N
 * magnitudes. F(a_(r)) = r/N >= k  <=>  r >= k N, so the answer is the r-th smallest
 * magnitude with r = ceil(k N), computed exactly on the binary value of the double k
 * (reading G5): k = M * 2^(e-53) with integer M < 2^53, so k N = M N / 2^(53-e).
 * Returns r (0 when k == 0). Caller guarantees 0 <= k < 1. */
uint64_t oracle_rank(double k, uint64_t n) {
    if (!(k > 0.0)) return 0;
    int e;
    double fr = frexp(k, &e);                 /* k = fr * 2^e, fr in [0.5, 1) */
    uint64_t M = (uint64_t)ldexp(fr, 53);      /* exact: fr has <= 53 significant bits */
    int sh = 53 - e;                           /* k = M / 2^sh, sh >= 53 since e <= 0 */
    unsigned __int128 prod = (unsigned __int128)M * (unsigned __int128)n;
    if (sh >= 128) return prod ? 1 : 0;        /* unreachable for normal doubles and n < 2^64 */
    unsigned __int128 q = prod >> sh;
    unsigned __int128 rem = prod - (q << sh);
    if (rem) q += 1;
    return (uint64_t)q;
}

static int cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* Eq. 3 by sorting (tiny / medium inputs): a_i = |acts_i| widened to double (so -0
 * becomes +0, reading G18), sort ascending, t = a_(r) (1-indexed), t = 0 if r = 0
 * (k = 0, reading G4; "augmented with 0"). Also returns
 * count_lt = #{a < t}, count_le = #{a <= t}. Returns -2 if any value is NaN/Inf
 * (reading G17), -1 on bad arguments. */
int oracle_calibrate_sort(const void *acts, uint64_t n, int dtype, double k,
                          double *t_out, uint64_t *r_out, uint64_t *count_lt, uint64_t *count_le) {
    if (n == 0 || !(k >= 0.0 && k < 1.0)) return -1;
    double *a = (double *)malloc(sizeof(double) * (size_t)n);
    if (!a) return -1;
    for (uint64_t i = 0; i < n; ++i) {
        double w = widen(acts, i, dtype);
        if (!isfinite(w)) { free(a); return -2; }
        a[i] = fabs(w);
    }
    qsort(a, (size_t)n, sizeof(double), cmp_double);
    uint64_t r = oracle_rank(k, n);
    double t = (r == 0) ? 0.0 : a[r - 1];
    uint64_t lt = 0, le = 0;
    for (uint64_t i = 0; i < n; ++i) { lt += (a[i] < t); le += (a[i] <= t); }
    *t_out = t; *r_out = r; *count_lt = lt; *count_le = le;
    free(a);
    return 0;
}

/* Full-scale bf16 variant of the same definition. A multiset of bf16 values is fully
 * described by the multiplicity of each of the 2^16 bit patterns, so the oracle first
 * counts patterns (oracle_bf16_count, may be called on consecutive chunks), then
 * orders the DISTINCT magnitudes |value| (as doubles, sorted with qsort) and walks
 * them with their multiplicities to the r-th smallest. Same answer as sorting the
 * whole multiset; memory O(2^16) instead of O(N). */
void oracle_bf16_count(const uint16_t *acts, uint64_t n, uint64_t *counts /*[65536]*/) {
    for (uint64_t i = 0; i < n; ++i) counts[acts[i]] += 1;
}

typedef struct { double mag; uint64_t cnt; } mag_count_t;
static int cmp_mag(const void *a, const void *b) {
    double x = ((const mag_count_t *)a)->mag, y = ((const mag_count_t *)b)->mag;
    return (x > y) - (x < y);
}

int oracle_calibrate_bf16_counts(const uint64_t *counts /*[65536]*/, double k,
                                 double *t_out, uint64_t *r_out, uint64_t *count_lt, uint64_t *count_le,
                                 uint64_t *n_out) {
    if (!(k >= 0.0 && k < 1.0)) return -1;
    mag_count_t *mc = (mag_count_t *)malloc(sizeof(mag_count_t) * 65536);
    if (!mc) return -1;
    uint64_t n = 0;
    int nonfinite = 0, nd = 0;
    for (uint32_t p = 0; p < 65536; ++p) {
        if (!counts[p]) continue;
        uint16_t bits = (uint16_t)p;
        double w = widen(&bits, 0, ORACLE_BF16);
        if (!isfinite(w)) { nonfinite = 1; continue; }
        mc[nd].mag = fabs(w); mc[nd].cnt = counts[p]; ++nd;
        n += counts[p];
    }
    if (nonfinite) { free(mc); return -2; }
    if (n == 0) { free(mc); return -1; }
    qsort(mc, (size_t)nd, sizeof(mag_count_t), cmp_mag);
    uint64_t r = oracle_rank(k, n);
    double t = 0.0;
    if (r > 0) {
        uint64_t seen = 0;
        for (int i = 0; i < nd; ++i) {
            seen += mc[i].cnt;
            if (seen >= r) { t = mc[i].mag; break; }
        }
    }
    uint64_t lt = 0, le = 0;
    for (int i = 0; i < nd; ++i) {
        if (mc[i].mag < t) lt += mc[i].cnt;
        if (mc[i].mag <= t) le += mc[i].cnt;
    }
    *t_out = t; *r_out = r; *count_lt = lt; *count_le = le; *n_out = n;
    free(mc);
    return 0;
}
