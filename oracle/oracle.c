/*
 * oracle.c -- float64 CPU oracle for the Approx-BP / MS-BP hot path of
 * arXiv 2406.16282 ("Reducing Fine-Tuning Memory Overhead by Approximate and
 * Memory-Sharing Backpropagation").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2406_16282_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * Plain, slow, obviously-correct definitions, written in the paper's order and
 * notation.  All arithmetic is IEEE binary64; inputs arrive already converted
 * exactly to double by the Python wrapper (oracle/__init__.py).  OpenMP is used
 * only to split independent rows / element ranges across threads; it changes
 * no result (every output element or row is computed by exactly one thread in
 * a fixed sequential order).
 *
 * Citations: P:L<n> = /root/reference/PAPER.md line n (section / equation /
 * algorithm given beside it); S:L<n> = SPEC.md line n.
 *
 * Parity status: every function below is pinned by tests/test_oracle_pins.py
 * (mpmath, torch float64 autograd, finite differences, closed forms, the
 * paper's printed constants).  No function is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORACLE_GELU = 0, ORACLE_SILU = 1 };

/* ------------------------------------------------------------------------ */
/* Step-function constants.                                                  */
/*                                                                           */
/* Eq. 14 (k=2) and its explicit k=2 form (App. E):     */
/*   h~(x) = a1 ReLU(x-c1) + a2 ReLU(x-c2) + (1-a1-a2) ReLU(x-c3).           */
/* Published full-precision solutions:                                       */
/*   GELU: a* = [-0.04922261145617846, 1.0979632065417297]    */
/*         c* = [-3.1858810036855245, -0.001178821281161997,                 */
/*                3.190832613414926]    */
/*   SiLU: a* = [-0.04060357190528599, 1.080925428529668]    */
/*         c* = [-6.3050461001646445, -0.0008684942046214787,                */
/*                6.325815242089708]    */
/* The derivative of h~ is the 4-segment step function (Prop. 4.1): */
/*   dh~(x) = 0 for x<c1, a1 on (c1,c2), a1+a2 on (c2,c3), 1 for x>c3.       */
/* At a kink the lower segment applies (strict '>').          */
/* ------------------------------------------------------------------------ */
static const double GELU_A[2] = {-0.04922261145617846, 1.0979632065417297};
static const double GELU_C[3] = {-3.1858810036855245, -0.001178821281161997, 3.190832613414926};
static const double SILU_A[2] = {-0.04060357190528599, 1.080925428529668};
static const double SILU_C[3] = {-6.3050461001646445, -0.0008684942046214787, 6.325815242089708};

/* Returns 0 on success, -1 for an unknown kind.  c = thresholds (3),
 * s = levels (4) = cumulative ReLU weights: s0 = 0, s1 = a1, s2 = a1 + a2,
 * s3 = a1 + a2 + (1 - a1 - a2) = 1 exactly (the weights sum to one, Eq. 14). */
int oracle_step_table(int kind, double c[3], double s[4], double a[2])
{
    const double *A, *C;
    if (kind == ORACLE_GELU) { A = GELU_A; C = GELU_C; }
    else if (kind == ORACLE_SILU) { A = SILU_A; C = SILU_C; }
    else return -1;
    for (int i = 0; i < 3; ++i) c[i] = C[i];
    a[0] = A[0];
    a[1] = A[1];
    s[0] = 0.0;
    s[1] = A[0];
    s[2] = A[0] + A[1];
    s[3] = 1.0;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Exact primitives (the forward is unchanged).                      */
/* GELU(x) = x/2 (1 + erf(x/sqrt2)).  Evaluated as        */
/* x/2 * erfc(-x/sqrt2), the same function, because 1 + erf(z) = erfc(-z)   */
/* and the erfc form does not cancel for x << 0.                             */
/* SiLU(x) = x / (1 + e^{-x}); for x < 0 the algebraically */
/* equal x e^{x} / (1 + e^{x}) keeps e^{-x} from overflowing.                 */
/* ------------------------------------------------------------------------ */
double oracle_gelu(double x)
{
    return 0.5 * x * erfc(-x / sqrt(2.0));
}

double oracle_silu(double x)
{
    if (x >= 0.0) return x / (1.0 + exp(-x));
    double e = exp(x);
    return x * e / (1.0 + e);
}

/* Exact derivatives, reference-only (gradient-gap diagnostic).
 * GELU'(x) = Phi(x) + x phi(x); SiLU'(x) = s + x s (1 - s) with
 * s = sigmoid(x) (App. G eq. silu_dsilu). */
double oracle_gelu_deriv(double x)
{
    const double PI = 3.14159265358979323846;
    double Phi = 0.5 * erfc(-x / sqrt(2.0));
    double phi = exp(-0.5 * x * x) / sqrt(2.0 * PI);
    return Phi + x * phi;
}

double oracle_silu_deriv(double x)
{
    double s = (x >= 0.0) ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
    return s + x * s * (1.0 - s);
}

/* h~(x) itself, Eq. 14 / P:L1017, reference-only (pins the levels by finite
 * differences and the limiting behaviour of Prop. 4.1). */
double oracle_combo_eval(int kind, double x)
{
    double c[3], s[4], a[2];
    if (oracle_step_table(kind, c, s, a) != 0) return NAN;
    double r1 = x - c[0] > 0.0 ? x - c[0] : 0.0;
    double r2 = x - c[1] > 0.0 ? x - c[1] : 0.0;
    double r3 = x - c[2] > 0.0 ? x - c[2] : 0.0;
    return a[0] * r1 + a[1] * r2 + (1.0 - a[0] - a[1]) * r3;
}

/* ------------------------------------------------------------------------ */
/* ReGELU2 / ReSiLU2 forward: y = h(x) exactly, and the 2-bit   */
/* segment index code = #{i : x > c_i}, packed four per byte, */
/* element j in byte j>>2 at bits 2*(j&3) (LSB first), the   */
/* unused trailing bits of the last byte zero.                      */
/* NaN compares false, so NaN -> code 0.                            */
/* codes must hold (n + 3) / 4 bytes.                                        */
/* ------------------------------------------------------------------------ */
int oracle_act_fwd(int kind, const double *x, int64_t n, double *y, uint8_t *codes, int nthreads)
{
    double c[3], s[4], a[2];
    if (oracle_step_table(kind, c, s, a) != 0) return -1;
    int64_t nbytes = (n + 3) / 4;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t b = 0; b < nbytes; ++b) {
        unsigned byte = 0;
        for (int k = 0; k < 4; ++k) {
            int64_t j = 4 * b + k;
            if (j >= n) break;
            double xj = x[j];
            y[j] = (kind == ORACLE_GELU) ? oracle_gelu(xj) : oracle_silu(xj);
            unsigned code = (unsigned)(xj > c[0]) + (unsigned)(xj > c[1]) + (unsigned)(xj > c[2]);
            byte |= code << (2 * k);
        }
        codes[b] = (uint8_t)byte;
    }
    return 0;
}

/* Unpack the 2-bit code of element j (inverse of the packing above). */
static unsigned code_at(const uint8_t *codes, int64_t j)
{
    return (codes[j >> 2] >> (2 * (j & 3))) & 3u;
}

/* ------------------------------------------------------------------------ */
/* ReGELU2 / ReSiLU2 backward: dx = dh~(x) * dy = s[code] * dy (P:L371,      */
/* P:L1081).  Value mode: fp64 product with fp64 levels.             */
/* ------------------------------------------------------------------------ */
int oracle_act_bwd(int kind, const uint8_t *codes, const double *dy, int64_t n, double *dx, int nthreads)
{
    double c[3], s[4], a[2];
    if (oracle_step_table(kind, c, s, a) != 0) return -1;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t j = 0; j < n; ++j)
        dx[j] = s[code_at(codes, j)] * dy[j];
    return 0;
}

/* Contract mode (reading R5): the kernel multiplies in fp32 by the
 * fp32-rounded level.  Here: level rounded to binary32 (C cast, round to
 * nearest even), product of two binary32 values formed EXACTLY in binary64
 * (24 + 24 significand bits <= 53), returned unrounded.  The wrapper then
 * rounds to binary32 and to the storage type, both round-to-nearest-even. */
int oracle_act_bwd_contract_exact(int kind, const uint8_t *codes, const double *dy, int64_t n, double *prod, int nthreads)
{
    double c[3], s[4], a[2];
    if (oracle_step_table(kind, c, s, a) != 0) return -1;
    double s32[4];
    for (int i = 0; i < 4; ++i) s32[i] = (double)(float)s[i];
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t j = 0; j < n; ++j)
        prod[j] = s32[code_at(codes, j)] * dy[j];
    return 0;
}

/* ------------------------------------------------------------------------ */
/* MS-LN (Alg. 2, App. F; Alg. 1).                 */
/*   H = I - p^{-1} 1 1^T, p = cols.                        */
/*   sigma = sqrt(p^{-1} z^T H z + eps)   (biased, two-pass)        */
/*   y     = sigma^{-1} H z                          */
/* Saved: y and sigma; we return rstd = 1/sigma (reading R9).      */
/* ------------------------------------------------------------------------ */
int oracle_msln_fwd(const double *x, int64_t rows, int64_t cols, double eps, double *y, double *rstd, int nthreads)
{
    if (cols <= 0) return -1;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < rows; ++r) {
        const double *xr = x + r * cols;
        double *yr = y + r * cols;
        double mean = 0.0;
        for (int64_t i = 0; i < cols; ++i) mean += xr[i];
        mean /= (double)cols;                          /* (1/p) 1^T z           */
        double var = 0.0;
        for (int64_t i = 0; i < cols; ++i) {
            double h = xr[i] - mean;                   /* (H z)_i               */
            var += h * h;                              /* z^T H z (H idempotent) */
        }
        var /= (double)cols;
        double sigma = sqrt(var + eps);
        for (int64_t i = 0; i < cols; ++i) yr[i] = (xr[i] - mean) / sigma;
        rstd[r] = 1.0 / sigma;
    }
    return 0;
}

/* Backward, Alg. 2:
 *   dz = sigma^{-1} (H - p^{-1} y y^T) dy
 *      = rstd * (dy - mean(dy) - y * (y^T dy)/p).
 * Uses only (y, rstd, dy): the input z is never read (memory sharing). */
int oracle_msln_bwd(const double *dy, const double *y, const double *rstd, int64_t rows, int64_t cols, double *dx, int nthreads)
{
    if (cols <= 0) return -1;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < rows; ++r) {
        const double *gr = dy + r * cols, *yr = y + r * cols;
        double *dr = dx + r * cols;
        double m1 = 0.0, m2 = 0.0;
        for (int64_t i = 0; i < cols; ++i) {
            m1 += gr[i];                               /* 1^T dy                */
            m2 += yr[i] * gr[i];                       /* y^T dy                */
        }
        m1 /= (double)cols;
        m2 /= (double)cols;
        for (int64_t i = 0; i < cols; ++i)
            dr[i] = rstd[r] * (gr[i] - m1 - yr[i] * m2);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* MS-RMSNorm (Alg. 3, App. F):                                */
/*   sigma = sqrt(p^{-1} z^T z + eps)                       */
/*   y     = sigma^{-1} z                       */
/*   dz    = sigma^{-1} (I - p^{-1} y y^T) dy                       */
/* ------------------------------------------------------------------------ */
int oracle_msrms_fwd(const double *x, int64_t rows, int64_t cols, double eps, double *y, double *rstd, int nthreads)
{
    if (cols <= 0) return -1;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < rows; ++r) {
        const double *xr = x + r * cols;
        double *yr = y + r * cols;
        double ms = 0.0;
        for (int64_t i = 0; i < cols; ++i) ms += xr[i] * xr[i];
        ms /= (double)cols;
        double sigma = sqrt(ms + eps);
        for (int64_t i = 0; i < cols; ++i) yr[i] = xr[i] / sigma;
        rstd[r] = 1.0 / sigma;
    }
    return 0;
}

int oracle_msrms_bwd(const double *dy, const double *y, const double *rstd, int64_t rows, int64_t cols, double *dx, int nthreads)
{
    if (cols <= 0) return -1;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < rows; ++r) {
        const double *gr = dy + r * cols, *yr = y + r * cols;
        double *dr = dx + r * cols;
        double m2 = 0.0;
        for (int64_t i = 0; i < cols; ++i) m2 += yr[i] * gr[i];
        m2 /= (double)cols;
        for (int64_t i = 0; i < cols; ++i)
            dr[i] = rstd[r] * (gr[i] - yr[i] * m2);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* ReSwiGLU2: LLaMA's SwiGLU gate            */
/*   h = SiLU(g) * u  with SiLU replaced by ReSiLU2:           */
/* forward exact, backward through the step derivative:                      */
/*   a = SiLU(g), h = a u, code = #{i : g > c_i}  (SiLU table)       */
/*   du = dh a,   dg = dh u s[code]                                           */
/* ------------------------------------------------------------------------ */
int oracle_reswiglu2_fwd(const double *g, const double *u, int64_t n, double *h, double *a, uint8_t *codes,
                         int nthreads)
{
    int rc = oracle_act_fwd(ORACLE_SILU, g, n, a, codes, nthreads);
    if (rc != 0) return rc;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t j = 0; j < n; ++j) h[j] = a[j] * u[j];
    return 0;
}

int oracle_reswiglu2_bwd(const double *dh, const double *u, const double *a, const uint8_t *codes, int64_t n,
                         double *dg, double *du, int nthreads)
{
    double c[3], s[4], w[2];
    if (oracle_step_table(ORACLE_SILU, c, s, w) != 0) return -1;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t j = 0; j < n; ++j) {
        du[j] = dh[j] * a[j];
        dg[j] = dh[j] * u[j] * s[code_at(codes, j)];
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* k-bit step activations: Eq. 14 with 2^k - 1 ReLUs  */
/* (P:L353-362); derivative = 2^k-segment step (Prop. 4.1).          */
/* code = #{i : x > c_i}; packed k bits per element, element j at bits       */
/* k*j .. k*j+k-1 of the LSB-first bit stream, trailing bits zero. */
/* k = 1..4 ("k is the required bit number"; k bits per element,   */
/* P:L371; "a larger k ... is also feasible").  For k = 3 a code    */
/* straddles a byte boundary whenever k*j mod 8 > 5, so codes are written   */
/* and read one bit at a time: bit b of code j is stream bit k*j + b.       */
/* ------------------------------------------------------------------------ */
int oracle_stepact_fwd(int kind, int k, const double *c, const double *x, int64_t n, double *y, uint8_t *codes)
{
    if (k < 1 || k > 4) return -1;
    int nt = (1 << k) - 1;
    int64_t nbytes = (n * k + 7) / 8;
    for (int64_t b = 0; b < nbytes; ++b) codes[b] = 0;
    for (int64_t j = 0; j < n; ++j) {
        y[j] = (kind == ORACLE_GELU) ? oracle_gelu(x[j]) : oracle_silu(x[j]);
        unsigned code = 0;
        for (int i = 0; i < nt; ++i) code += (unsigned)(x[j] > c[i]);
        for (int b = 0; b < k; ++b) {
            int64_t bit = (int64_t)k * j + b;
            codes[bit / 8] |= (uint8_t)(((code >> b) & 1u) << (bit % 8));
        }
    }
    return 0;
}

int oracle_stepact_bwd(int k, const double *s, const uint8_t *codes, const double *dy, int64_t n, double *dx)
{
    if (k < 1 || k > 4) return -1;
    for (int64_t j = 0; j < n; ++j) {
        unsigned code = 0;
        for (int b = 0; b < k; ++b) {
            int64_t bit = (int64_t)k * j + b;
            code |= (unsigned)((codes[bit / 8] >> (bit % 8)) & 1u) << b;
        }
        dx[j] = s[code] * dy[j];
    }
    return 0;
}

/* ReGELU2-d (App. I): the derivative-L2 fit of GELU. */
static const double GELUD_A[2] = {0.32465931184406527, 0.34812875668739607};
static const double GELUD_C[3] = {-0.4535743722857079, -0.0010587205574873046, 0.4487575313884231};

int oracle_regelu2d_table(double c[3], double s[4])
{
    for (int i = 0; i < 3; ++i) c[i] = GELUD_C[i];
    s[0] = 0.0;
    s[1] = GELUD_A[0];
    s[2] = GELUD_A[0] + GELUD_A[1];
    s[3] = 1.0;
    return 0;
}

/* Number of OpenMP threads a parallel region would use (for reporting). */
int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
