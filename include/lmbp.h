/*
 * lmbp.h -- C ABI of the B200 (sm_100a) hot path of Approx-BP and
 * Memory-Sharing BP (arXiv 2406.16282, "Reducing Fine-Tuning Memory Overhead
 * by Approximate and Memory-Sharing Backpropagation").
 *
 * Citations: P:L<n> = reference PAPER.md line n (section / equation /
 * algorithm beside it); S:L<n> = reference SPEC.md line n.  DESIGN.md lists
 * every reading (R1..) of the paper that these contracts rely on.
 *
 * ---------------------------------------------------------------------------
 * Conventions shared by every entry point
 * ---------------------------------------------------------------------------
 * Memory.  Every tensor pointer is a DEVICE pointer on the current CUDA
 *   device.  The caller owns all memory; the library never allocates, frees
 *   or synchronises.  Tensors are contiguous row-major [rows, cols]
 *   (row stride = cols elements).  All work is enqueued on `stream`
 *   (a cudaStream_t passed as void*; NULL = the legacy default stream).
 * Types.  x / y / dy / dx share `dtype` (LMBP_F32 / LMBP_BF16 / LMBP_F16);
 *   arithmetic is binary32; conversions round to nearest even; no
 *   flush-to-zero of stored values.  `rstd` is always binary32.
 * Packed codes (activation kernels).  n = rows * cols elements are processed
 *   as one flat sequence; element j's 2-bit segment code is stored in byte
 *   j >> 2 at bits 2*(j & 3) (LSB first); the buffer holds
 *   exactly lmbp_codes_bytes(n) = ceil(n / 4) bytes and the unused high bits of
 *   the last byte are written as 0.
 * Alignment.  The vector (TMA) path needs 16-byte aligned tensor and `codes`
 *   pointers.  Anything else runs a scalar path with bitwise-identical
 *   activation results; misalignment is never an error.
 * Aliasing.  Exact aliasing y == x (forward) or dx == dy (backward) is
 *   allowed: every element / row is read before it is written.  Partial
 *   overlap is undefined.
 * Errors.  Arguments are validated synchronously and a status is returned:
 *   rows < 0, cols <= 0 or rows*cols overflowing int64 -> LMBP_ERR_SHAPE;
 *   a NULL tensor pointer with rows > 0 -> LMBP_ERR_NULLPTR; unknown dtype ->
 *   LMBP_ERR_DTYPE; eps not finite or <= 0 -> LMBP_ERR_EPS; a failed launch
 *   (cudaGetLastError) -> LMBP_ERR_CUDA.  rows == 0 is a no-op returning
 *   LMBP_OK.  Faults during asynchronous execution surface at the caller's
 *   next synchronisation, as usual in CUDA.  Nothing is printed, no C++
 *   exception crosses the ABI.
 * Launch.  Kernels are launched with programmatic stream serialization
 *   (programmatic dependent launch): following another kernel on `stream`,
 *   a launch may start its prologue before that kernel finishes, and waits
 *   for its completion (griddepcontrol.wait) before touching any tensor, so
 *   stream order is preserved for every caller-visible byte.  Stream capture
 *   records the launches as programmatic graph edges.  Each kernel signals
 *   launch_dependents at entry, so a caller's OWN kernel launched with the
 *   PDL attribute right after one of ours may start early and must call
 *   cudaGridDependencySynchronize() before reading our outputs (as PDL
 *   requires of any dependent); plain launches are unaffected.  The
 *   environment variable LMBP_PDL=0, read once per process, launches ours
 *   plainly.
 * State.  No global mutable state (constants only): reentrant across host
 *   threads, streams and devices.  Deterministic: no atomics, fixed
 *   reduction order, so results are bitwise identical run to run.
 */
#ifndef LMBP_H_
#define LMBP_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LMBP_API __attribute__((visibility("default")))
#else
#define LMBP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { LMBP_F32 = 0, LMBP_BF16 = 1, LMBP_F16 = 2 } lmbp_dtype;

typedef enum {
  LMBP_OK = 0,
  LMBP_ERR_NULLPTR = 1,
  LMBP_ERR_SHAPE = 2,
  LMBP_ERR_DTYPE = 3,
  LMBP_ERR_EPS = 4,
  LMBP_ERR_CUDA = 5,
  LMBP_ERR_KIND = 6,
  LMBP_ERR_TABLE = 7,
  LMBP_ERR_ARG = 8
} lmbp_status;

typedef enum { LMBP_GELU = 0, LMBP_SILU = 1 } lmbp_act_kind;

/* ceil(n / 4): bytes of packed 2-bit codes for n elements.
 * Returns 0 for n <= 0. */
LMBP_API size_t lmbp_codes_bytes(int64_t n);

/* Static, NUL-terminated description of a status code. */
LMBP_API const char *lmbp_status_string(int status);

/* Library version string, e.g. "lmbp 0.1.0 sm_100a". */
LMBP_API const char *lmbp_version(void);

/* Host-side copy of the binary32 step table the kernels use for `kind`
 * (LMBP_GELU / LMBP_SILU): thresholds[3] and levels[4].  thresholds[i] is the
 * largest binary32 value <= c_i (round toward -inf, reading R2), so
 * that for every fp32/bf16/fp16 input `x > thresholds[i]` <=> `x > c_i`
 * exactly; levels = RN32(0, a1, a1 + a2, 1) (reading R5).  c, a from
 * P:L1062-1063 (GELU) and P:L1139-1140 (SiLU).  No device access.
 * Returns LMBP_ERR_NULLPTR / LMBP_ERR_KIND on bad arguments. */
LMBP_API int lmbp_step_table(int kind, float *thresholds, float *levels);

/* ---------------------------------------------------------------------------
 * ReGELU2 / ReSiLU2 (Sec. 4.2; App. E)
 * ---------------------------------------------------------------------------
 * Forward ("keeps the same primitive function"):
 *   y[j]  = GELU(x[j]) = x/2 (1 + erf(x/sqrt2))
 *        or SiLU(x[j]) = x / (1 + e^{-x})
 *   code[j] = #{i : x[j] > c_i}, c = the published thresholds (P:L1063 /
 *        P:L1140); strict '>' so a kink takes the lower segment;
 *        NaN -> code 0.  The code is taken from x as stored in
 *        `dtype` (reading R3).
 *   Only `codes` (ceil(n/4) bytes) needs to be kept for backward.
 *   x: [rows, cols] input; y: [rows, cols] output (may equal x);
 *   codes: lmbp_codes_bytes(rows*cols) bytes, written in full.
 * Backward (Prop. 4.1; the derivative of Eq. 14 is the 4-segment
 *   step function with levels s = (0, a1, a1 + a2, 1)):
 *   dx[j] = dy[j] * s[code[j]], computed as RN_dtype(RN32(dy * RN32(s)))
 *   (reading R5; for bf16/fp16 this equals one rounding of the exact product).
 *   dy: [rows, cols]; codes: as written by the matching *_fwd; dx: [rows,
 *   cols] output (may equal dy). */
LMBP_API int regelu2_fwd(const void *x, void *y, uint8_t *codes, int64_t rows, int64_t cols,
                int dtype, void *stream);
LMBP_API int regelu2_bwd(const void *dy, const uint8_t *codes, void *dx, int64_t rows, int64_t cols,
                int dtype, void *stream);
LMBP_API int resilu2_fwd(const void *x, void *y, uint8_t *codes, int64_t rows, int64_t cols,
                int dtype, void *stream);
LMBP_API int resilu2_bwd(const void *dy, const uint8_t *codes, void *dx, int64_t rows, int64_t cols,
                int dtype, void *stream);

/* ---------------------------------------------------------------------------
 * MS-LN (Alg. 1; Alg. 2, App. F)
 * ---------------------------------------------------------------------------
 * The affine (alpha, beta) is merged into the next linear layer,
 * so the layer is parameter-free and its output y is the next linear layer's
 * saved input (Prop. 5.1).  Per row of p = cols elements:
 * Forward:  mu = (1/p) sum x;  var = (1/p) sum (x - mu)^2   (biased)
 *           rstd = 1 / sqrt(var + eps);  y = (x - mu) * rstd
 *           x: [rows, cols]; y: [rows, cols] output (may equal x);
 *           rstd: [rows] binary32 output (the paper saves sigma = 1/rstd,
 *           P:L1246; reading R9).  eps: finite, > 0 (1e-6 or 1e-8).
 * Backward: dx = rstd * (dy - mean(dy) - y * mean(dy * y))   (Alg. 2)
 *           from (dy, y, rstd) only -- x is never read.
 *           dy, y: [rows, cols]; rstd: [rows]; dx: [rows, cols] output (may
 *           equal dy).
 * ------------------------------------------------------------------------- */
LMBP_API int msln_fwd(const void *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps,
             int dtype, void *stream);
LMBP_API int msln_bwd(const void *dy, const void *y, const float *rstd, void *dx, int64_t rows,
             int64_t cols, int dtype, void *stream);

/* ---------------------------------------------------------------------------
 * MS-RMSNorm (Alg. 3, App. F): as MS-LN with H = I, beta = 0.
 * Forward:  rstd = 1 / sqrt((1/p) sum x^2 + eps);  y = x * rstd
 * Backward: dx = rstd * (dy - y * mean(dy * y))
 * Arguments as msln_*.
 * ------------------------------------------------------------------------- */
LMBP_API int msrms_fwd(const void *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps,
              int dtype, void *stream);
LMBP_API int msrms_bwd(const void *dy, const void *y, const float *rstd, void *dx, int64_t rows,
              int64_t cols, int dtype, void *stream);

/* ---------------------------------------------------------------------------
 * Mixed-precision MS-LN / MS-RMSNorm: fp32 residual stream, 16-bit output.
 * Under AMP the paper's norms run in fp32 while the linears run in 16 bits
 * (Fig. 5 / 6 captions).  Sharing y with the next linear
 * (Prop. 5.1 condition 3) needs y in that linear's input dtype, so:
 * Forward:  x: fp32 [rows, cols]; y: [rows, cols] in `dtype` (LMBP_BF16 or
 *           LMBP_F16), y = RN_dtype((x - mu) rstd) (RMS: x rstd), statistics
 *           in fp32 exactly as msln_fwd / msrms_fwd; rstd: fp32 [rows].
 * Backward: dy, y: [rows, cols] in `dtype`; rstd: fp32 [rows]; dx: fp32
 *           [rows, cols] output: rstd (dy - mean dy - y mean(dy y)) (RMS
 *           without mean dy), not rounded to 16 bits.
 * dtype LMBP_F32 (or unknown) -> LMBP_ERR_DTYPE (use msln_* / msrms_*).  No
 * aliasing between the fp32 and 16-bit tensors.  Other arguments, errors and
 * alignment rules as msln_* (misaligned or cols % 8 != 0: a scalar path).
 * ------------------------------------------------------------------------- */
LMBP_API int msln_fwd_mixed(const float *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps,
                            int dtype, void *stream);
LMBP_API int msln_bwd_mixed(const void *dy, const void *y, const float *rstd, float *dx, int64_t rows,
                            int64_t cols, int dtype, void *stream);
LMBP_API int msrms_fwd_mixed(const float *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps,
                             int dtype, void *stream);
LMBP_API int msrms_bwd_mixed(const void *dy, const void *y, const float *rstd, float *dx, int64_t rows,
                             int64_t cols, int dtype, void *stream);

/* ---------------------------------------------------------------------------
 * ReSwiGLU2: fused LLaMA gate h = SiLU(gate) * up with ReSiLU2's backward
 * (SwiGLU; ReSiLU2).  Semantics are
 * exactly those of the unfused composition resilu2_fwd -> elementwise mul
 * (and its reverse), with one HBM pass instead of three:
 * Forward:  a = RN_dtype(SiLU(gate))        -- saved (the mul's operand)
 *           h = RN_dtype(RN32(a * up))       -- output
 *           codes of gate as resilu2_fwd     -- saved (2 bits / element)
 *           gate, up: [rows, cols]; h, a: [rows, cols] outputs;
 *           codes: lmbp_codes_bytes(rows*cols) bytes.
 *           Activation memory kept for backward: a, up and codes (2b + 1/4
 *           bytes per element) instead of gate, up and SiLU(gate) (3b).
 * Backward: dup   = RN_dtype(RN32(dh * a))
 *           dgate = RN_dtype(RN32(RN_dtype(RN32(dh * up)) * RN32(s[code])))
 *           dh, up, a: [rows, cols]; codes as written by reswiglu2_fwd;
 *           dgate, dup: [rows, cols] outputs.
 * Vector path: all tensor and codes pointers 16-byte aligned, else a scalar
 * path with bitwise-identical results.  Any output may exactly alias any
 * input of the same shape.  Errors as above.
 * ------------------------------------------------------------------------- */
LMBP_API int reswiglu2_fwd(const void *gate, const void *up, void *h, void *a, uint8_t *codes, int64_t rows,
                           int64_t cols, int dtype, void *stream);
LMBP_API int reswiglu2_bwd(const void *dh, const void *up, const void *a, const uint8_t *codes, void *dgate,
                           void *dup, int64_t rows, int64_t cols, int dtype, void *stream);

/* ---------------------------------------------------------------------------
 * Table-driven k-bit step activations: Eq. 14 with
 * 2^k - 1 ReLUs, whose derivative is a 2^k-segment step function
 * needing k bits per element (Prop. 4.1); "a larger k ... is also
 * feasible".  k = 2 with the published tables reproduces
 * regelu2_* / resilu2_* bitwise; other tables give e.g. ReGELU2-d (App. I,
 * P:L1333-1351).
 * Forward:  y = GELU(x) or SiLU(x) (act = LMBP_GELU / LMBP_SILU, unchanged
 *           primitive); code = #{i : x > thresholds[i]}, i < 2^k - 1.
 *           thresholds: HOST pointer to 2^k - 1 finite, strictly increasing
 *           binary64 values; the library compares x > RD32(threshold), exact
 *           for every fp32/bf16/fp16 x (reading R2).
 * Backward: dx = RN_dtype(RN32(dy * RN32(levels[code])));
 *           levels: HOST pointer to 2^k finite binary64 values.
 * codes: lmbp_codes_bytes_k(rows*cols, k) = ceil(n k / 8) bytes; element j
 *        at bits k*j .. k*j+k-1 of the LSB-first bit stream;
 *        trailing bits of the last byte written as 0.  For k = 3 a code
 *        may straddle two bytes (every 8 elements from a multiple of 8 fill
 *        exactly 3 bytes).
 * k must be 1, 2, 3 or 4 (else LMBP_ERR_TABLE, as for a malformed table).
 * Layout, alignment (any; 16-byte aligned tensors take the vector path with
 * identical results), aliasing and the other errors as above.
 * ------------------------------------------------------------------------- */
LMBP_API size_t lmbp_codes_bytes_k(int64_t n, int k);
LMBP_API int stepact_fwd(int act, int k, const double *thresholds, const void *x, void *y, uint8_t *codes,
                         int64_t rows, int64_t cols, int dtype, void *stream);
LMBP_API int stepact_bwd(int k, const double *levels, const void *dy, const uint8_t *codes, void *dx,
                         int64_t rows, int64_t cols, int dtype, void *stream);

/* ---------------------------------------------------------------------------
 * Offline coefficient fitter: the step tables above are
 * the minimisers of App. E's objective (Eq. 15, P:L1009-1065 GELU,
 * P:L1086-1142 SiLU)
 *     J(a, c) = int_A^B (h(x) - h~_{a,c}(x))^2 dx,
 *     h~_{a,c}(x) = sum_{i<m} a_i ReLU(x - c_i) + (1 - sum a) ReLU(x - c_m)
 * (Eq. 14, m = 2^k - 1 ReLUs), or of App. I's derivative
 * objective (Eq. 17: h', h~' in place of h, h~), found by
 * simulated annealing from many initialisations.
 *
 * theta: binary64 (a_1 .. a_{m-1}, c_1 .. c_m), P = 2m - 1 values; for k = 2
 *   exactly the paper's five scalars (a1, a2, c1, c2, c3).
 * act: LMBP_GELU / LMBP_SILU.  objective: LMBP_FIT_H (Eq. 15) or LMBP_FIT_DH
 *   (Eq. 17).  k: 1..4.  eps: the tail tolerance that fixes [A, B]
 *   (lmbp_fit_bounds; the paper uses 1e-8).
 * Arithmetic: binary64 throughout; the integral is a composite 16-point
 *   Gauss-Legendre rule on panels of length <= 2 between the sorted kinks
 *   (on intervals of >= 12 panels the theta-independent outer pieces come
 *   from per-block prefix tables plus one partial panel each).
 * Errors: act / objective unknown -> LMBP_ERR_KIND; k outside 1..4 or
 *   n < 0 -> LMBP_ERR_SHAPE; eps not in (0, 1) -> LMBP_ERR_EPS (also for
 *   lmbp_fit_anneal_vp when [A, B] spans more than 64 panels of length 2,
 *   e.g. SiLU with eps < ~2.5e-14: its tables cannot hold them); NULL pointer
 *   with work to do -> LMBP_ERR_NULLPTR; bad annealing schedule (chains < 1,
 *   iters < 0, t0 / t1 / step0 / step1 not finite and > 0) -> LMBP_ERR_ARG;
 *   launch failure -> LMBP_ERR_CUDA.  Deterministic for a given seed.
 * ------------------------------------------------------------------------- */
typedef enum { LMBP_FIT_H = 0, LMBP_FIT_DH = 1 } lmbp_fit_objective_kind;

/* Host only: the truncated interval [A, B] of App. E for tail tolerance eps:
 * GELU B = -A = sqrt(-2 ln eps); SiLU B = -A = -2 ln(eps / 2)
 * (P:L1121).  A, B: HOST pointers. */
LMBP_API int lmbp_fit_bounds(int act, double eps, double *A, double *B);

/* J for n parameter vectors: theta DEVICE [n, P] row-major, J DEVICE [n].
 * A J that is NaN (non-finite theta) is returned as +inf. */
LMBP_API int lmbp_fit_objective(int act, int objective, int k, double eps, const double *theta, double *J,
                                int64_t n, void *stream);

/* Simulated annealing, one chain per GPU thread.  Chain i starts from init
 * (DEVICE [P], shared by every chain; NULL = a random start per chain:
 * weights around 1/m, thresholds uniform in [A/2, B/2]), then for `iters`
 * steps perturbs one coordinate j (cyclically) by sigma_j N(0, 1) and
 * accepts with probability min(1, exp(-(J' - J) / (T J))) (Metropolis at a
 * temperature relative to the current J), T falling
 * geometrically from t0 to t1.  sigma_j adapts per coordinate (x1.25 on
 * accept, x0.92 on reject) within [step1, 4 step0] x (1 for weights,
 * (B - A)/8 for thresholds), starting at step0 x that scale.
 * Random numbers: a counter-based generator of
 * (seed, chain, step), so results do not depend on the launch shape.
 * Outputs (DEVICE, caller-owned): chain_theta [chains, P] and chain_J [chains]
 * = each chain's best point, canonical (ReLUs sorted by threshold), and its
 * J; best [P + 1] = the best chain's theta followed by its J (ties -> lowest
 * chain index). */
LMBP_API int lmbp_fit_anneal(int act, int objective, int k, double eps, const double *init, int64_t chains,
                             int64_t iters, uint64_t seed, double t0, double t1, double step0, double step1,
                             double *chain_theta, double *chain_J, double *best, void *stream);

/* Variable-projection annealing: the same chains, but only the m thresholds
 * anneal; for each proposal the weights are the exact least-squares optimum
 * under sum w = 1 (Eq. 14's objective is quadratic in w for fixed c: a small
 * (m+1)-dimensional linear solve), so the search space is m-dimensional and
 * the weight directions' bad conditioning drops out (needed for k >= 3).
 * init: as above (only its thresholds are used).  Steps scale with
 * (B - A)/8.  Outputs as lmbp_fit_anneal, chain J re-evaluated by the direct
 * quadrature.  When [A, B] spans more than 64 panels (eps below ~1e-27 for
 * SiLU) every chain reports J = +inf (use lmbp_fit_anneal). */
LMBP_API int lmbp_fit_anneal_vp(int act, int objective, int k, double eps, const double *init, int64_t chains,
                                int64_t iters, uint64_t seed, double t0, double t1, double step0, double step1,
                                double *chain_theta, double *chain_J, double *best, void *stream);

/* Local refinement of n starting points (e.g. every annealing chain's best):
 * Levenberg-Marquardt on J with a central-difference gradient and Hessian
 * (steps 1e-4 x (1 for weights, (B - A)/8 for thresholds)), Cholesky solve
 * of (H + lambda diag H) d = -g, at most `iters` accepted steps; a step is
 * taken only if J decreases, so J_out <= J(theta) for every row.
 * theta DEVICE [n, P] (may alias theta_out); theta_out DEVICE [n, P]
 * (canonical form), J_out DEVICE [n]; best DEVICE [P + 1] or NULL (as in
 * lmbp_fit_anneal).  iters < 0 -> LMBP_ERR_ARG; n < 0 -> LMBP_ERR_SHAPE. */
LMBP_API int lmbp_fit_refine(int act, int objective, int k, double eps, const double *theta, int64_t n,
                             int64_t iters, double *theta_out, double *J_out, double *best, void *stream);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* LMBP_H_ */
