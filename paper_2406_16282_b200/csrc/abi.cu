// abi.cu -- the extern "C" boundary declared in include/lmbp.h.
// Synchronous argument validation, dtype dispatch, status codes.  No
// allocation, no synchronisation, nothing printed, no exceptions escape.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "../../include/lmbp.h"
#include "common.cuh"
#include "kernels.h"

namespace lmbp {

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  return n;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char *v = std::getenv("LMBP_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

static int check_shape(int64_t rows, int64_t cols) {
  if (rows < 0 || cols <= 0) return LMBP_ERR_SHAPE;
  if (rows > 0 && cols > INT64_MAX / rows) return LMBP_ERR_SHAPE;
  return LMBP_OK;
}

static int check_dtype(int dtype) {
  return (dtype == LMBP_F32 || dtype == LMBP_BF16 || dtype == LMBP_F16) ? LMBP_OK : LMBP_ERR_DTYPE;
}

static int status_of(cudaError_t e) { return e == cudaSuccess ? LMBP_OK : LMBP_ERR_CUDA; }

static int act_fwd_entry(int kind, const void *x, void *y, uint8_t *codes, int64_t rows, int64_t cols, int dtype,
                         void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = check_dtype(dtype)) != LMBP_OK) return st;
  if (rows == 0) return LMBP_OK;
  if (!x || !y || !codes) return LMBP_ERR_NULLPTR;
  return status_of(act_fwd(kind, dtype, x, y, codes, rows * cols, static_cast<cudaStream_t>(stream)));
}

static int act_bwd_entry(int kind, const void *dy, const uint8_t *codes, void *dx, int64_t rows, int64_t cols,
                         int dtype, void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = check_dtype(dtype)) != LMBP_OK) return st;
  if (rows == 0) return LMBP_OK;
  if (!dy || !dx || !codes) return LMBP_ERR_NULLPTR;
  return status_of(act_bwd(kind, dtype, dy, codes, dx, rows * cols, static_cast<cudaStream_t>(stream)));
}

static int norm_fwd_entry(int kind, const void *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps,
                          int dtype, void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = check_dtype(dtype)) != LMBP_OK) return st;
  if (!(eps > 0.0f) || !std::isfinite(eps)) return LMBP_ERR_EPS;
  if (rows == 0) return LMBP_OK;
  if (!x || !y || !rstd) return LMBP_ERR_NULLPTR;
  return status_of(norm_fwd(kind, dtype, x, y, rstd, rows, cols, eps, static_cast<cudaStream_t>(stream)));
}

static int mixed_dtype(int dtype) { return (dtype == LMBP_BF16 || dtype == LMBP_F16) ? LMBP_OK : LMBP_ERR_DTYPE; }

static int norm_fwd_mixed_entry(int kind, const float *x, void *y, float *rstd, int64_t rows, int64_t cols,
                                float eps, int dtype, void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = mixed_dtype(dtype)) != LMBP_OK) return st;
  if (!(eps > 0.0f) || !std::isfinite(eps)) return LMBP_ERR_EPS;
  if (rows == 0) return LMBP_OK;
  if (!x || !y || !rstd) return LMBP_ERR_NULLPTR;
  return status_of(norm_fwd_mixed(kind, dtype, x, y, rstd, rows, cols, eps, static_cast<cudaStream_t>(stream)));
}

static int norm_bwd_mixed_entry(int kind, const void *dy, const void *y, const float *rstd, float *dx, int64_t rows,
                                int64_t cols, int dtype, void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = mixed_dtype(dtype)) != LMBP_OK) return st;
  if (rows == 0) return LMBP_OK;
  if (!dy || !y || !rstd || !dx) return LMBP_ERR_NULLPTR;
  return status_of(norm_bwd_mixed(kind, dtype, dy, y, rstd, dx, rows, cols, static_cast<cudaStream_t>(stream)));
}

static int norm_bwd_entry(int kind, const void *dy, const void *y, const float *rstd, void *dx, int64_t rows,
                          int64_t cols, int dtype, void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = check_dtype(dtype)) != LMBP_OK) return st;
  if (rows == 0) return LMBP_OK;
  if (!dy || !y || !rstd || !dx) return LMBP_ERR_NULLPTR;
  return status_of(norm_bwd(kind, dtype, dy, y, rstd, dx, rows, cols, static_cast<cudaStream_t>(stream)));
}

static int swiglu_fwd_entry(const void *g, const void *u, void *h, void *a, uint8_t *codes, int64_t rows,
                            int64_t cols, int dtype, void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = check_dtype(dtype)) != LMBP_OK) return st;
  if (rows == 0) return LMBP_OK;
  if (!g || !u || !h || !a || !codes) return LMBP_ERR_NULLPTR;
  return status_of(swiglu_fwd(dtype, g, u, h, a, codes, rows * cols, static_cast<cudaStream_t>(stream)));
}

static int swiglu_bwd_entry(const void *dh, const void *u, const void *a, const uint8_t *codes, void *dg, void *du,
                            int64_t rows, int64_t cols, int dtype, void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = check_dtype(dtype)) != LMBP_OK) return st;
  if (rows == 0) return LMBP_OK;
  if (!dh || !u || !a || !codes || !dg || !du) return LMBP_ERR_NULLPTR;
  return status_of(swiglu_bwd(dtype, dh, u, a, codes, dg, du, rows * cols, static_cast<cudaStream_t>(stream)));
}

static bool k_ok(int k) { return k >= 1 && k <= 4; }

// Round a binary64 threshold toward -inf into binary32 (reading R2).
static float rd32(double c) {
  float f = (float)c;
  if ((double)f > c) f = std::nextafter(f, -INFINITY);
  return f;
}

static int stepact_fwd_entry(int act, int k, const double *thr, const void *x, void *y, uint8_t *codes,
                             int64_t rows, int64_t cols, int dtype, void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = check_dtype(dtype)) != LMBP_OK) return st;
  if (act != LMBP_GELU && act != LMBP_SILU) return LMBP_ERR_KIND;
  if (!k_ok(k)) return LMBP_ERR_TABLE;
  if (!thr) return LMBP_ERR_NULLPTR;
  StepTable t{};
  t.k = k;
  for (int i = 0; i < (1 << k) - 1; ++i) {
    if (!std::isfinite(thr[i]) || (i > 0 && !(thr[i] > thr[i - 1]))) return LMBP_ERR_TABLE;
    t.thr[i] = rd32(thr[i]);
    // RD_T(RD32(c)) == RD_T(c): every value of T is a binary32 value.
    uint16_t h = 0;
    if (dtype == LMBP_BF16) h = __bfloat16_as_ushort(__float2bfloat16_rd(t.thr[i]));
    else if (dtype == LMBP_F16) h = __half_as_ushort(__float2half_rd(t.thr[i]));
    t.thr2[i] = (uint32_t)h | ((uint32_t)h << 16);
  }
  if (rows == 0) return LMBP_OK;
  if (!x || !y || !codes) return LMBP_ERR_NULLPTR;
  return status_of(stepact_fwd(act, dtype, t, x, y, codes, rows * cols, static_cast<cudaStream_t>(stream)));
}

static int stepact_bwd_entry(int k, const double *lvl, const void *dy, const uint8_t *codes, void *dx, int64_t rows,
                             int64_t cols, int dtype, void *stream) {
  int st = check_shape(rows, cols);
  if (st != LMBP_OK) return st;
  if ((st = check_dtype(dtype)) != LMBP_OK) return st;
  if (!k_ok(k)) return LMBP_ERR_TABLE;
  if (!lvl) return LMBP_ERR_NULLPTR;
  StepTable t{};
  t.k = k;
  for (int i = 0; i < (1 << k); ++i) {
    if (!std::isfinite(lvl[i])) return LMBP_ERR_TABLE;
    t.lvl[i] = (float)lvl[i];
  }
  if (rows == 0) return LMBP_OK;
  if (!dy || !dx || !codes) return LMBP_ERR_NULLPTR;
  return status_of(stepact_bwd(dtype, t, dy, codes, dx, rows * cols, static_cast<cudaStream_t>(stream)));
}

static bool fit_bounds(int act, double eps, double *A, double *B) {
  if (!(eps > 0.0 && eps < 1.0)) return false;
  const double b = act == kActGelu ? std::sqrt(-2.0 * std::log(eps)) : -2.0 * std::log(eps / 2.0);
  *A = -b;
  *B = b;
  return true;
}

static int fit_spec(int act, int objective, int k, double eps, FitSpec *s) {
  if (act != LMBP_GELU && act != LMBP_SILU) return LMBP_ERR_KIND;
  if (objective != LMBP_FIT_H && objective != LMBP_FIT_DH) return LMBP_ERR_KIND;
  if (k < 1 || k > 4) return LMBP_ERR_SHAPE;
  if (!fit_bounds(act, eps, &s->A, &s->B)) return LMBP_ERR_EPS;
  s->act = act == LMBP_GELU ? kActGelu : kActSilu;
  s->obj = objective;
  s->panel = 2.0;
  return LMBP_OK;
}

static bool pos_finite(double v) { return std::isfinite(v) && v > 0.0; }

}  // namespace lmbp

extern "C" {

size_t lmbp_codes_bytes(int64_t n) { return n <= 0 ? 0 : (size_t)((n + 3) / 4); }

size_t lmbp_codes_bytes_k(int64_t n, int k) {
  if (n <= 0 || !lmbp::k_ok(k)) return 0;
  return (size_t)((n * k + 7) / 8);
}

const char *lmbp_status_string(int status) {
  switch (status) {
    case LMBP_OK: return "LMBP_OK";
    case LMBP_ERR_NULLPTR: return "LMBP_ERR_NULLPTR: a required pointer is NULL";
    case LMBP_ERR_SHAPE: return "LMBP_ERR_SHAPE: rows < 0, cols <= 0 or rows*cols overflows int64";
    case LMBP_ERR_DTYPE: return "LMBP_ERR_DTYPE: dtype is not LMBP_F32, LMBP_BF16 or LMBP_F16";
    case LMBP_ERR_EPS: return "LMBP_ERR_EPS: eps must be finite and > 0";
    case LMBP_ERR_CUDA: return "LMBP_ERR_CUDA: kernel launch failed (cudaGetLastError)";
    case LMBP_ERR_KIND: return "LMBP_ERR_KIND: unknown activation kind";
    case LMBP_ERR_TABLE: return "LMBP_ERR_TABLE: k not in {1, 2, 4}, or thresholds not finite and strictly increasing, or levels not finite";
    case LMBP_ERR_ARG: return "LMBP_ERR_ARG: invalid annealing schedule (chains < 1, iters < 0, or t0/t1/step0/step1 not finite and > 0)";
    default: return "LMBP: unknown status";
  }
}

const char *lmbp_version(void) { return "lmbp 0.1.0 sm_100a"; }

int lmbp_step_table(int kind, float *thresholds, float *levels) {
  if (!thresholds || !levels) return LMBP_ERR_NULLPTR;
  const uint32_t *t, *l;
  if (kind == LMBP_GELU) {
    t = lmbp::kGELU_THR_F32;
    l = lmbp::kGELU_LVL_F32;
  } else if (kind == LMBP_SILU) {
    t = lmbp::kSILU_THR_F32;
    l = lmbp::kSILU_LVL_F32;
  } else {
    return LMBP_ERR_KIND;
  }
  std::memcpy(thresholds, t, 3 * sizeof(float));
  std::memcpy(levels, l, 4 * sizeof(float));
  return LMBP_OK;
}

int regelu2_fwd(const void *x, void *y, uint8_t *codes, int64_t rows, int64_t cols, int dtype, void *stream) {
  return lmbp::act_fwd_entry(lmbp::kActGelu, x, y, codes, rows, cols, dtype, stream);
}
int regelu2_bwd(const void *dy, const uint8_t *codes, void *dx, int64_t rows, int64_t cols, int dtype, void *stream) {
  return lmbp::act_bwd_entry(lmbp::kActGelu, dy, codes, dx, rows, cols, dtype, stream);
}
int resilu2_fwd(const void *x, void *y, uint8_t *codes, int64_t rows, int64_t cols, int dtype, void *stream) {
  return lmbp::act_fwd_entry(lmbp::kActSilu, x, y, codes, rows, cols, dtype, stream);
}
int resilu2_bwd(const void *dy, const uint8_t *codes, void *dx, int64_t rows, int64_t cols, int dtype, void *stream) {
  return lmbp::act_bwd_entry(lmbp::kActSilu, dy, codes, dx, rows, cols, dtype, stream);
}
int msln_fwd(const void *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps, int dtype, void *stream) {
  return lmbp::norm_fwd_entry(lmbp::kNormLN, x, y, rstd, rows, cols, eps, dtype, stream);
}
int msln_bwd(const void *dy, const void *y, const float *rstd, void *dx, int64_t rows, int64_t cols, int dtype,
             void *stream) {
  return lmbp::norm_bwd_entry(lmbp::kNormLN, dy, y, rstd, dx, rows, cols, dtype, stream);
}
int msrms_fwd(const void *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps, int dtype, void *stream) {
  return lmbp::norm_fwd_entry(lmbp::kNormRMS, x, y, rstd, rows, cols, eps, dtype, stream);
}
int msrms_bwd(const void *dy, const void *y, const float *rstd, void *dx, int64_t rows, int64_t cols, int dtype,
              void *stream) {
  return lmbp::norm_bwd_entry(lmbp::kNormRMS, dy, y, rstd, dx, rows, cols, dtype, stream);
}

int msln_fwd_mixed(const float *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps, int dtype,
                   void *stream) {
  return lmbp::norm_fwd_mixed_entry(lmbp::kNormLN, x, y, rstd, rows, cols, eps, dtype, stream);
}
int msln_bwd_mixed(const void *dy, const void *y, const float *rstd, float *dx, int64_t rows, int64_t cols, int dtype,
                   void *stream) {
  return lmbp::norm_bwd_mixed_entry(lmbp::kNormLN, dy, y, rstd, dx, rows, cols, dtype, stream);
}
int msrms_fwd_mixed(const float *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps, int dtype,
                    void *stream) {
  return lmbp::norm_fwd_mixed_entry(lmbp::kNormRMS, x, y, rstd, rows, cols, eps, dtype, stream);
}
int msrms_bwd_mixed(const void *dy, const void *y, const float *rstd, float *dx, int64_t rows, int64_t cols,
                    int dtype, void *stream) {
  return lmbp::norm_bwd_mixed_entry(lmbp::kNormRMS, dy, y, rstd, dx, rows, cols, dtype, stream);
}

int reswiglu2_fwd(const void *gate, const void *up, void *h, void *a, uint8_t *codes, int64_t rows, int64_t cols,
                  int dtype, void *stream) {
  return lmbp::swiglu_fwd_entry(gate, up, h, a, codes, rows, cols, dtype, stream);
}
int reswiglu2_bwd(const void *dh, const void *up, const void *a, const uint8_t *codes, void *dgate, void *dup,
                  int64_t rows, int64_t cols, int dtype, void *stream) {
  return lmbp::swiglu_bwd_entry(dh, up, a, codes, dgate, dup, rows, cols, dtype, stream);
}

int stepact_fwd(int act, int k, const double *thresholds, const void *x, void *y, uint8_t *codes, int64_t rows,
                int64_t cols, int dtype, void *stream) {
  return lmbp::stepact_fwd_entry(act, k, thresholds, x, y, codes, rows, cols, dtype, stream);
}
int stepact_bwd(int k, const double *levels, const void *dy, const uint8_t *codes, void *dx, int64_t rows,
                int64_t cols, int dtype, void *stream) {
  return lmbp::stepact_bwd_entry(k, levels, dy, codes, dx, rows, cols, dtype, stream);
}

int lmbp_fit_bounds(int act, double eps, double *A, double *B) {
  if (act != LMBP_GELU && act != LMBP_SILU) return LMBP_ERR_KIND;
  if (!A || !B) return LMBP_ERR_NULLPTR;
  return lmbp::fit_bounds(act == LMBP_GELU ? lmbp::kActGelu : lmbp::kActSilu, eps, A, B) ? LMBP_OK : LMBP_ERR_EPS;
}

int lmbp_fit_objective(int act, int objective, int k, double eps, const double *theta, double *J, int64_t n,
                       void *stream) {
  lmbp::FitSpec s{};
  int st = lmbp::fit_spec(act, objective, k, eps, &s);
  if (st != LMBP_OK) return st;
  if (n < 0) return LMBP_ERR_SHAPE;
  if (n == 0) return LMBP_OK;
  if (!theta || !J) return LMBP_ERR_NULLPTR;
  return lmbp::status_of(lmbp::fit_objective(s, k, theta, J, n, static_cast<cudaStream_t>(stream)));
}

static int fit_anneal_entry(bool vp, int act, int objective, int k, double eps, const double *init, int64_t chains,
                            int64_t iters, uint64_t seed, double t0, double t1, double step0, double step1,
                            double *chain_theta, double *chain_J, double *best, void *stream) {
  lmbp::FitSpec s{};
  int st = lmbp::fit_spec(act, objective, k, eps, &s);
  if (st != LMBP_OK) return st;
  if (chains < 1 || iters < 0 || !lmbp::pos_finite(t0) || !lmbp::pos_finite(t1) || !lmbp::pos_finite(step0) ||
      !lmbp::pos_finite(step1))
    return LMBP_ERR_ARG;
  if (!chain_theta || !chain_J || !best) return LMBP_ERR_NULLPTR;
  // the projected anneal integrates the weights' normal equations from
  // per-CTA tables of ceil((B - A) / panel) cells; a tail tolerance so small
  // that [A, B] needs more cells than the tables hold cannot be served
  if (vp && std::ceil((s.B - s.A) / s.panel) > lmbp::kFitMaxCells) return LMBP_ERR_EPS;
  lmbp::AnnealCfg a{chains, iters, seed, t0, t1, step0, step1};
  const cudaStream_t cs = static_cast<cudaStream_t>(stream);
  return lmbp::status_of(vp ? lmbp::fit_anneal_vp(s, k, a, init, chain_theta, chain_J, best, cs)
                            : lmbp::fit_anneal(s, k, a, init, chain_theta, chain_J, best, cs));
}

int lmbp_fit_anneal(int act, int objective, int k, double eps, const double *init, int64_t chains, int64_t iters,
                    uint64_t seed, double t0, double t1, double step0, double step1, double *chain_theta,
                    double *chain_J, double *best, void *stream) {
  return fit_anneal_entry(false, act, objective, k, eps, init, chains, iters, seed, t0, t1, step0, step1,
                          chain_theta, chain_J, best, stream);
}

int lmbp_fit_anneal_vp(int act, int objective, int k, double eps, const double *init, int64_t chains, int64_t iters,
                       uint64_t seed, double t0, double t1, double step0, double step1, double *chain_theta,
                       double *chain_J, double *best, void *stream) {
  return fit_anneal_entry(true, act, objective, k, eps, init, chains, iters, seed, t0, t1, step0, step1,
                          chain_theta, chain_J, best, stream);
}

int lmbp_fit_refine(int act, int objective, int k, double eps, const double *theta, int64_t n, int64_t iters,
                    double *theta_out, double *J_out, double *best, void *stream) {
  lmbp::FitSpec s{};
  int st = lmbp::fit_spec(act, objective, k, eps, &s);
  if (st != LMBP_OK) return st;
  if (n < 0) return LMBP_ERR_SHAPE;
  if (iters < 0) return LMBP_ERR_ARG;
  if (n == 0) return LMBP_OK;
  if (!theta || !theta_out || !J_out) return LMBP_ERR_NULLPTR;
  return lmbp::status_of(lmbp::fit_refine(s, k, theta, n, iters, theta_out, J_out, best,
                                          static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
