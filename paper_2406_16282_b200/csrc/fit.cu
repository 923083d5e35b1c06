// fit.cu -- the offline coefficient fitter on the GPU.
//
// App. E (P:L1009-1065 GELU, P:L1086-1142 SiLU) obtains ReGELU2 / ReSiLU2's
// constants by minimising
//     J(a, c) = int_A^B (h(x) - h~_{a,c}(x))^2 dx                     (Eq. 15)
// over the 2^k - 1 ReLUs of Eq. 14, h~ = sum_i w_i ReLU(x - c_i),
// w = (a_1 .. a_{m-1}, 1 - sum a), after truncating the tails to [A, B]
// (P:L1045), with simulated annealing restarted from many
// initialisations ("searching multiple times with different
// initialization").  App. I does the same for the derivatives
// (Eq. 17), giving ReGELU2-d.
//
// B200 design: the restarts are the parallelism.  One thread runs one
// annealing chain; thousands of chains run at once and a final kernel takes
// the best.  Each objective evaluation is a fixed composite Gauss-Legendre
// rule in binary64 (B200 has full-rate-ish FP64 pipes): [A, B] is split at the
// sorted kinks c_i -- on each piece h~ is one affine function (h~' one
// constant), so the integrand is analytic there -- and every piece into
// panels of at most `panel` length with 16 nodes each.  For SiLU the nearest
// singularities of the integrand are at +-i pi, so a 2-long panel's 16-point
// rule errs by ~1e-26 relative; GELU is entire.  The objective is ALU (FP64)
// bound; nothing is read from memory but the parameters.
//
// The oracle (oracle/fit.py) evaluates the same integral with QUADPACK; the
// two share nothing.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace lmbp {

namespace {

static_assert(kGLN == 16, "the constant tables below list 8 node pairs");
__constant__ unsigned long long cGLX[8] = {kGLX[0], kGLX[1], kGLX[2], kGLX[3], kGLX[4], kGLX[5], kGLX[6], kGLX[7]};
__constant__ unsigned long long cGLW[8] = {kGLW[0], kGLW[1], kGLW[2], kGLW[3], kGLW[4], kGLW[5], kGLW[6], kGLW[7]};
__device__ __forceinline__ double gl_x(int i) { return __longlong_as_double((long long)cGLX[i]); }
__device__ __forceinline__ double gl_w(int i) { return __longlong_as_double((long long)cGLW[i]); }

// h and h' in binary64.
__device__ __forceinline__ double h_fn(int act, double x) {
  if (act == kActGelu) return 0.5 * x * erfc(-x * 0.70710678118654752440);
  const double e = exp(-fabs(x));            // SiLU, stable in both tails
  return x >= 0.0 ? x / (1.0 + e) : x * e / (1.0 + e);
}

__device__ __forceinline__ double dh_fn(int act, double x) {
  if (act == kActGelu)
    return 0.5 * erfc(-x * 0.70710678118654752440) + x * exp(-0.5 * x * x) * 0.39894228040143267794;
  const double e = exp(-fabs(x));
  const double r = 1.0 / (1.0 + e);
  const double s = x >= 0.0 ? r : e * r;     // sigma(x)
  const double sc = x >= 0.0 ? e * r : r;    // 1 - sigma(x), no cancellation
  return s + x * s * sc;
}

// int_l^r f(x) dx, f = (h - alpha x - beta)^2 (obj 0) or (h' - alpha)^2 (obj 1).
__device__ double integrate_piece(const FitSpec &s, double l, double r, double alpha, double beta) {
  if (!(r > l)) return 0.0;
  const int np = max(1, (int)ceil((r - l) / s.panel));
  const double half = 0.5 * (r - l) / np;
  double acc = 0.0;
  for (int p = 0; p < np; ++p) {
    const double mid = l + (2 * p + 1) * half;
    double pa = 0.0;
#pragma unroll
    for (int i = 0; i < kGLN / 2; ++i) {
      const double dx = half * gl_x(i);
      const double x0 = mid - dx, x1 = mid + dx;
      double f0, f1;
      if (s.obj == 0) {
        f0 = h_fn(s.act, x0) - fma(alpha, x0, beta);
        f1 = h_fn(s.act, x1) - fma(alpha, x1, beta);
      } else {
        f0 = dh_fn(s.act, x0) - alpha;
        f1 = dh_fn(s.act, x1) - alpha;
      }
      pa = fma(gl_w(i), fma(f0, f0, f1 * f1), pa);
    }
    acc += pa;
  }
  return acc * half;
}

// Sort the ReLUs by threshold (weights travel with them); fully unrolled so
// the arrays stay in registers.
template <int M>
__device__ __forceinline__ void sort_pairs(double (&w)[M], double (&c)[M]) {
#pragma unroll
  for (int i = 0; i < M - 1; ++i) {
#pragma unroll
    for (int j = 0; j < M - 1 - i; ++j) {
      const bool sw = c[j + 1] < c[j];
      const double cj = c[j], wj = w[j];
      c[j] = sw ? c[j + 1] : cj;
      c[j + 1] = sw ? cj : c[j + 1];
      w[j] = sw ? w[j + 1] : wj;
      w[j + 1] = sw ? wj : w[j + 1];
    }
  }
}

// theta = (a_1 .. a_{M-1}, c_1 .. c_M) -> (w[M], c[M]), w_M = 1 - sum a.
template <int M>
__device__ __forceinline__ void unpack_theta(const double *th, double (&w)[M], double (&c)[M]) {
  double sa = 0.0;
#pragma unroll
  for (int i = 0; i < M - 1; ++i) {
    w[i] = th[i];
    sa += th[i];
  }
  w[M - 1] = 1.0 - sa;
#pragma unroll
  for (int i = 0; i < M; ++i) c[i] = th[M - 1 + i];
}

// J(theta).  Pieces between consecutive sorted kinks, clipped to [A, B]: on
// piece j, h~(x) = alpha_j x + beta_j with alpha_j = sum_{i<j} w_i,
// beta_j = -sum_{i<j} w_i c_i (ReLUs with c <= A are active from A on; those
// with c >= B never switch on inside [A, B]).
template <int M>
__device__ double objective_t(const FitSpec &s, const double *th) {
  double w[M], c[M];
  unpack_theta<M>(th, w, c);
  sort_pairs<M>(w, c);
  double J = 0.0, alpha = 0.0, beta = 0.0;
#pragma unroll
  for (int j = 0; j <= M; ++j) {
    const double l = j == 0 ? s.A : fmin(fmax(c[j - 1], s.A), s.B);
    const double r = j == M ? s.B : fmin(fmax(c[j], s.A), s.B);
    J += integrate_piece(s, l, r, alpha, beta);
    if (j < M) {
      alpha += w[j];
      beta = fma(-w[j], c[j], beta);
    }
  }
  return isnan(J) ? INFINITY : J;
}

// Canonical form: ReLUs sorted by threshold, theta = (w_1 .. w_{M-1}, c_1 .. c_M)
// of the sorted pairs (the same function h~, Eq. 14 is symmetric in the pairs
// once the weights sum to 1).
template <int M>
__device__ void canonical(const double *th, double *out) {
  double w[M], c[M];
  unpack_theta<M>(th, w, c);
  sort_pairs<M>(w, c);
#pragma unroll
  for (int i = 0; i < M - 1; ++i) out[i] = w[i];
#pragma unroll
  for (int i = 0; i < M; ++i) out[M - 1 + i] = c[i];
}

template <int M>
__global__ void __launch_bounds__(128) fit_objective_k(FitSpec s, const double *theta, double *J, int64_t n) {
  constexpr int P = 2 * M - 1;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double th[P];
#pragma unroll
  for (int i = 0; i < P; ++i) th[i] = theta[t * P + i];
  J[t] = objective_t<M>(s, th);
}

// Counter-based random numbers (splitmix64 finaliser over (seed, chain,
// counter)): every chain's stream is reproducible and independent of the
// launch shape.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u01(uint64_t seed, uint64_t chain, uint64_t ctr) {
  const uint64_t z = mix64(seed ^ mix64(chain * 0xD1B54A32D192ED03ull + ctr));
  return ((double)(z >> 11) + 0.5) * 0x1p-53;  // (0, 1)
}
__device__ __forceinline__ double gauss(uint64_t seed, uint64_t chain, uint64_t ctr) {
  const double u1 = u01(seed, chain, 2 * ctr), u2 = u01(seed, chain, 2 * ctr + 1);
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// One annealing chain per thread.  Proposal: one coordinate per step
// (cyclic), Gaussian with scale step(t) * (1 for weights, (B - A)/8 for
// thresholds); Metropolis acceptance at temperature T(t); T and step decay
// geometrically from (t0, step0) to (t1, step1).  Writes the chain's best
// point (canonical form) and its J.
template <int M>
__global__ void __launch_bounds__(128) fit_anneal_k(FitSpec s, AnnealCfg a, const double *init, double *chain_theta,
                                                     double *chain_J) {
  constexpr int P = 2 * M - 1;
  const int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= a.chains) return;
  const double cscale = (s.B - s.A) * 0.125;
  double th[P], best[P];
  uint64_t ctr = 0;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    if (init) {
      th[i] = init[i];
    } else if (i < M - 1) {
      th[i] = (1.0 + 3.0 * (2.0 * u01(a.seed, ch, ctr++) - 1.0)) / M;  // around equal weights
    } else {
      th[i] = s.A * 0.5 + (s.B - s.A) * 0.5 * u01(a.seed, ch, ctr++);
    }
    best[i] = th[i];
  }
  ctr = 1ull << 40;  // proposals draw from a separate counter range
  double J = objective_t<M>(s, th);
  double bestJ = J;
  const double lt = log(a.t1 / a.t0), ls = log(a.step1 / a.step0);
  for (int64_t it = 0; it < a.iters; ++it) {
    const double frac = a.iters > 1 ? (double)it / (double)(a.iters - 1) : 1.0;
    const double T = a.t0 * exp(lt * frac);
    const double step = a.step0 * exp(ls * frac);
    const int j = (int)(it % P);
    const double d = step * (j < M - 1 ? 1.0 : cscale) * gauss(a.seed, ch, ctr);
    const double u = u01(a.seed, ch, (1ull << 62) + ctr);
    ctr += 1;
    double prop[P];
#pragma unroll
    for (int i = 0; i < P; ++i) prop[i] = th[i] + (i == j ? d : 0.0);
    const double Jp = objective_t<M>(s, prop);
    if (Jp <= J || u < exp((J - Jp) / T)) {
#pragma unroll
      for (int i = 0; i < P; ++i) th[i] = prop[i];
      J = Jp;
      if (J < bestJ) {
        bestJ = J;
#pragma unroll
        for (int i = 0; i < P; ++i) best[i] = th[i];
      }
    }
  }
  double out[P];
  canonical<M>(best, out);
#pragma unroll
  for (int i = 0; i < P; ++i) chain_theta[ch * P + i] = out[i];
  chain_J[ch] = bestJ;
}

// best = (theta of the chain with the smallest J, J); ties -> lowest chain
// index, so the result does not depend on scheduling.
__global__ void __launch_bounds__(1024) fit_best_k(const double *chain_theta, const double *chain_J, int64_t chains,
                                                    int P, double *best) {
  __shared__ double sj[1024];
  __shared__ int64_t si[1024];
  double bj = INFINITY;
  int64_t bi = -1;
  for (int64_t c = threadIdx.x; c < chains; c += blockDim.x) {
    const double v = chain_J[c];
    if (v < bj) {  // strided scan in increasing c: first minimum kept
      bj = v;
      bi = c;
    }
  }
  sj[threadIdx.x] = bj;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v = sj[threadIdx.x + o];
      const int64_t i = si[threadIdx.x + o];
      if (i >= 0 && (si[threadIdx.x] < 0 || v < sj[threadIdx.x] || (v == sj[threadIdx.x] && i < si[threadIdx.x]))) {
        sj[threadIdx.x] = v;
        si[threadIdx.x] = i;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int64_t i = si[0] < 0 ? 0 : si[0];
    for (int p = 0; p < P; ++p) best[p] = chain_theta[i * P + p];
    best[P] = chain_J[i];
  }
}

template <int M>
cudaError_t objective_m(const FitSpec &s, const double *theta, double *J, int64_t n, cudaStream_t st) {
  const int64_t blocks = (n + 127) / 128;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  fit_objective_k<M><<<(int)blocks, 128, 0, st>>>(s, theta, J, n);
  return cudaGetLastError();
}

template <int M>
cudaError_t anneal_m(const FitSpec &s, const AnnealCfg &a, const double *init, double *chain_theta, double *chain_J,
                     double *best, cudaStream_t st) {
  const int64_t blocks = (a.chains + 127) / 128;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  fit_anneal_k<M><<<(int)blocks, 128, 0, st>>>(s, a, init, chain_theta, chain_J);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  fit_best_k<<<1, 1024, 0, st>>>(chain_theta, chain_J, a.chains, 2 * M - 1, best);
  return cudaGetLastError();
}

}  // namespace

cudaError_t fit_objective(const FitSpec &s, int k, const double *theta, double *J, int64_t n, cudaStream_t st) {
  switch (k) {
    case 1: return objective_m<1>(s, theta, J, n, st);
    case 2: return objective_m<3>(s, theta, J, n, st);
    case 3: return objective_m<7>(s, theta, J, n, st);
    default: return objective_m<15>(s, theta, J, n, st);
  }
}

cudaError_t fit_anneal(const FitSpec &s, int k, const AnnealCfg &a, const double *init, double *chain_theta,
                       double *chain_J, double *best, cudaStream_t st) {
  switch (k) {
    case 1: return anneal_m<1>(s, a, init, chain_theta, chain_J, best, st);
    case 2: return anneal_m<3>(s, a, init, chain_theta, chain_J, best, st);
    case 3: return anneal_m<7>(s, a, init, chain_theta, chain_J, best, st);
    default: return anneal_m<15>(s, a, init, chain_theta, chain_J, best, st);
  }
}

}  // namespace lmbp
