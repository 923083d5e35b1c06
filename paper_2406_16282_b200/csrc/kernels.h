// kernels.h -- internal launch entry points behind the C ABI (abi.cu).
// Arguments are already validated; every function enqueues on `s` and returns
// cudaGetLastError().
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace lmbp {

enum { kActGelu = 0, kActSilu = 1 };
enum { kNormLN = 0, kNormRMS = 1 };

cudaError_t act_fwd(int kind, int dtype, const void *x, void *y, uint8_t *codes, int64_t n, cudaStream_t s);
cudaError_t act_bwd(int kind, int dtype, const void *dy, const uint8_t *codes, void *dx, int64_t n,
                    cudaStream_t s);
cudaError_t norm_fwd(int kind, int dtype, const void *x, void *y, float *rstd, int64_t rows, int64_t cols,
                     float eps, cudaStream_t s);
cudaError_t norm_bwd(int kind, int dtype, const void *dy, const void *y, const float *rstd, void *dx,
                     int64_t rows, int64_t cols, cudaStream_t s);
// fp32 residual stream, 16-bit y / dy (norm_mixed.cu); dtype: 1 bf16, 2 fp16
cudaError_t norm_fwd_mixed(int kind, int dtype, const float *x, void *y, float *rstd, int64_t rows, int64_t cols,
                           float eps, cudaStream_t s);
cudaError_t norm_bwd_mixed(int kind, int dtype, const void *dy, const void *y, const float *rstd, float *dx,
                           int64_t rows, int64_t cols, cudaStream_t s);
// the same on norm.cu's row pipeline; cudaErrorNotSupported when the row does not fit it
cudaError_t norm_bwd_mixed_rows(int kind, int dtype, const void *dy, const void *y, const float *rstd, float *dx,
                                int64_t rows, int64_t cols, cudaStream_t s);

struct StepTable;  // common.cuh
cudaError_t stepact_fwd(int act, int dtype, const StepTable &t, const void *x, void *y, uint8_t *codes, int64_t n,
                        cudaStream_t s);
cudaError_t stepact_bwd(int dtype, const StepTable &t, const void *dy, const uint8_t *codes, void *dx, int64_t n,
                        cudaStream_t s);

cudaError_t swiglu_fwd(int dtype, const void *g, const void *u, void *h, void *a, uint8_t *codes, int64_t n,
                       cudaStream_t s);
cudaError_t swiglu_bwd(int dtype, const void *dh, const void *u, const void *a, const uint8_t *codes, void *dg,
                       void *du, int64_t n, cudaStream_t s);

// Coefficient fitter (fit.cu).
struct FitSpec {
  int act;       // kActGelu / kActSilu
  int obj;       // 0: int (h - h~)^2 (Eq. 15), 1: int (h' - h~')^2 (Eq. 17)
  double A, B;   // truncated interval (App. E tail bounds)
  double panel;  // longest Gauss-Legendre panel
};
// Cells of the per-CTA prefix tables (panel grid over [A, B]); the
// variable-projection anneal needs them, so it refuses a wider interval.
constexpr int kFitMaxCells = 64;
struct AnnealCfg {
  int64_t chains, iters;
  uint64_t seed;
  double t0, t1, step0, step1;
};
cudaError_t fit_objective(const FitSpec &s, int k, const double *theta, double *J, int64_t n, cudaStream_t st);
cudaError_t fit_anneal(const FitSpec &s, int k, const AnnealCfg &a, const double *init, double *chain_theta,
                       double *chain_J, double *best, cudaStream_t st);
cudaError_t fit_anneal_vp(const FitSpec &s, int k, const AnnealCfg &a, const double *init, double *chain_theta,
                          double *chain_J, double *best, cudaStream_t st);
cudaError_t fit_refine(const FitSpec &s, int k, const double *in, int64_t n, int64_t iters, double *out,
                       double *Jout, double *best, cudaStream_t st);

}  // namespace lmbp
