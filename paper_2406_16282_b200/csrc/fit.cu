// fit.cu -- the offline coefficient fitter on the GPU.
//
// App. E (P:L1009-1065 GELU, P:L1086-1142 SiLU) obtains ReGELU2 / ReSiLU2's
// constants by minimising
//     J(a, c) = int_A^B (h(x) - h~_{a,c}(x))^2 dx                     (Eq. 15)
// over the 2^k - 1 ReLUs of Eq. 14, h~ = sum_i w_i ReLU(x - c_i),
// w = (a_1 .. a_{m-1}, 1 - sum a), after truncating the tails to [A, B]
// (P:L1044), with simulated annealing restarted from many
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
// Kernels: fit_objective_k (batched J), fit_anneal_k (all 2m - 1 parameters
// annealed), fit_anneal_vp_k (thresholds annealed, weights by the
// constrained least-squares solve -- variable projection), fit_refine_k
// (Levenberg-Marquardt from each chain's best), fit_best_k (deterministic
// arg-min).  Per-CTA shared-memory tables of the theta-independent integrals
// (tails; moments for the projection) replace most panels on long intervals.
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
template <int ACT>
__device__ __forceinline__ double h_fn(double x) {
  if constexpr (ACT == kActGelu) {
    return 0.5 * x * erfc(-x * 0.70710678118654752440);
  } else {
    const double e = exp(-fabs(x));            // SiLU, stable in both tails
    return x >= 0.0 ? x / (1.0 + e) : x * e / (1.0 + e);
  }
}

template <int ACT>
__device__ __forceinline__ double dh_fn(double x) {
  if constexpr (ACT == kActGelu) {
    return 0.5 * erfc(-x * 0.70710678118654752440) + x * exp(-0.5 * x * x) * 0.39894228040143267794;
  } else {
    const double e = exp(-fabs(x));
    const double r = 1.0 / (1.0 + e);
    const double s = x >= 0.0 ? r : e * r;     // sigma(x)
    const double sc = x >= 0.0 ? e * r : r;    // 1 - sigma(x), no cancellation
    return s + x * s * sc;
  }
}

// int_l^r f(x) dx, f = (h - alpha x - beta)^2 (OBJ 0) or (h' - alpha)^2 (OBJ 1).
// One out-of-line specialisation per (activation, objective): a launch only
// ever runs one of them, so the instruction cache holds one small body.
template <int ACT, int OBJ>
__device__ __noinline__ double integrate_piece_t(double l, double r, double alpha, double beta, double panel) {
  if (!(r > l)) return 0.0;
  const int np = max(1, (int)ceil((r - l) / panel));
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
      if constexpr (OBJ == 0) {
        f0 = h_fn<ACT>(x0) - fma(alpha, x0, beta);
        f1 = h_fn<ACT>(x1) - fma(alpha, x1, beta);
      } else {
        f0 = dh_fn<ACT>(x0) - alpha;
        f1 = dh_fn<ACT>(x1) - alpha;
      }
      pa = fma(gl_w(i), fma(f0, f0, f1 * f1), pa);
    }
    acc += pa;
  }
  return acc * half;
}

__device__ __forceinline__ double integrate_piece(const FitSpec &s, double l, double r, double alpha, double beta) {
  if (s.act == kActGelu)
    return s.obj == 0 ? integrate_piece_t<kActGelu, 0>(l, r, alpha, beta, s.panel)
                      : integrate_piece_t<kActGelu, 1>(l, r, alpha, beta, s.panel);
  return s.obj == 0 ? integrate_piece_t<kActSilu, 0>(l, r, alpha, beta, s.panel)
                    : integrate_piece_t<kActSilu, 1>(l, r, alpha, beta, s.panel);
}

// Tail tables.  Left of the lowest kink h~ = 0 and right of the highest
// h~ = x + beta (all ReLUs on, weights summing to 1), so the two outer pieces
// depend on theta only through their inner end point (and beta): with
//   L(t)  = int_A^t g0,  R0(t) = int_t^B g1^2,  R1(t) = int_t^B g1
// (obj 0: g0 = h^2, g1 = h - x; obj 1: g0 = h'^2, g1 = h' - 1) the outer
// pieces are L(c_min) and R0 - 2 beta R1 + beta^2 (B - c_max) (obj 1: R0).
// Each CTA tabulates L, R0, R1 at the panel grid x_i = A + i panel once
// (16-point Gauss-Legendre per cell, prefix sums), and an evaluation adds one
// partial-cell panel per tail -- for SiLU (B - A = 76) that replaces ~35 of
// ~41 panels per objective.
constexpr int kMaxCells = kFitMaxCells;
constexpr int kMinCells = 12;
struct FitTables {
  int n;                                       // cells; 0 = no table (too many cells)
  double L[kMaxCells + 1], R0[kMaxCells + 1], R1[kMaxCells + 1];
};

// Integrals of g0, g1^2, g1 over [l, r] with one 16-point panel.
template <int ACT, int OBJ>
__device__ __noinline__ void cell_t(double l, double r, double *i0, double *i1, double *i2) {
  const double mid = 0.5 * (l + r), half = 0.5 * (r - l);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int i = 0; i < kGLN / 2; ++i) {
    const double dx = half * gl_x(i);
    const double x0 = mid - dx, x1 = mid + dx;
    double g0, g1, e0, e1;
    if constexpr (OBJ == 0) {
      g0 = h_fn<ACT>(x0);
      g1 = h_fn<ACT>(x1);
      e0 = g0 - x0;
      e1 = g1 - x1;
    } else {
      g0 = dh_fn<ACT>(x0);
      g1 = dh_fn<ACT>(x1);
      e0 = g0 - 1.0;
      e1 = g1 - 1.0;
    }
    const double w = gl_w(i);
    a0 = fma(w, fma(g0, g0, g1 * g1), a0);
    a1 = fma(w, fma(e0, e0, e1 * e1), a1);
    a2 = fma(w, e0 + e1, a2);
  }
  *i0 = a0 * half;
  *i1 = a1 * half;
  *i2 = a2 * half;
}

__device__ __forceinline__ void cell(const FitSpec &s, double l, double r, double *i0, double *i1, double *i2) {
  if (s.act == kActGelu) {
    if (s.obj == 0) cell_t<kActGelu, 0>(l, r, i0, i1, i2);
    else cell_t<kActGelu, 1>(l, r, i0, i1, i2);
  } else {
    if (s.obj == 0) cell_t<kActSilu, 0>(l, r, i0, i1, i2);
    else cell_t<kActSilu, 1>(l, r, i0, i1, i2);
  }
}

__device__ __forceinline__ double grid_x(const FitSpec &s, const FitTables &T, int i) {
  return i >= T.n ? s.B : s.A + i * s.panel;
}

// Every thread of the block must call this (it synchronises the block).
__device__ const FitTables *build_tables(const FitSpec &s, FitTables &T) {
  const int n = (int)ceil((s.B - s.A) / s.panel);
  // Short intervals (GELU: 7 cells) gain nothing from the tables.
  if (threadIdx.x == 0) T.n = (n >= kMinCells && n <= kMaxCells) ? n : 0;
  __syncthreads();
  if (T.n == 0) return nullptr;
  for (int i = threadIdx.x; i < n; i += blockDim.x)   // cell integrals, stored at i + 1
    cell(s, grid_x(s, T, i), grid_x(s, T, i + 1), &T.L[i + 1], &T.R0[i], &T.R1[i]);
  __syncthreads();
  if (threadIdx.x == 0) {                            // prefix / suffix sums, fixed order
    T.L[0] = 0.0;
    for (int i = 1; i <= n; ++i) T.L[i] += T.L[i - 1];
    T.R0[n] = T.R1[n] = 0.0;
    for (int i = n - 1; i >= 0; --i) {
      T.R0[i] += T.R0[i + 1];
      T.R1[i] += T.R1[i + 1];
    }
  }
  __syncthreads();
  return &T;
}

// L(t) and (R0(t), R1(t)) for t in [A, B].
__device__ __forceinline__ double tail_left(const FitSpec &s, const FitTables &T, double t) {
  const int i = min(T.n - 1, max(0, (int)floor((t - s.A) / s.panel)));
  double p0, p1, p2;
  cell(s, grid_x(s, T, i), t, &p0, &p1, &p2);
  return T.L[i] + p0;
}
__device__ __forceinline__ void tail_right(const FitSpec &s, const FitTables &T, double t, double *r0, double *r1) {
  const int i = min(T.n - 1, max(0, (int)floor((t - s.A) / s.panel)));
  double p0, p1, p2;
  cell(s, t, grid_x(s, T, i + 1), &p0, &p1, &p2);
  *r0 = T.R0[i + 1] + p1;
  *r1 = T.R1[i + 1] + p2;
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
__device__ double objective_t(const FitSpec &s, const double *th, const FitTables *T) {
  double w[M], c[M];
  unpack_theta<M>(th, w, c);
  sort_pairs<M>(w, c);
  double J = 0.0, alpha = 0.0, beta = 0.0;
#pragma unroll 1
  for (int j = 0; j <= M; ++j) {
    const double l = j == 0 ? s.A : fmin(fmax(c[j - 1], s.A), s.B);
    const double r = j == M ? s.B : fmin(fmax(c[j], s.A), s.B);
    if (T && j == 0) {
      J += tail_left(s, *T, r);
    } else if (T && j == M) {
      double r0, r1;
      tail_right(s, *T, l, &r0, &r1);
      J += s.obj == 0 ? fma(beta, fma(beta, s.B - l, -2.0 * r1), r0) : r0;
    } else {
      J += integrate_piece(s, l, r, alpha, beta);
    }
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
  __shared__ FitTables tabs;
  const FitTables *T = build_tables(s, tabs);
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double th[P];
#pragma unroll
  for (int i = 0; i < P; ++i) th[i] = theta[t * P + i];
  J[t] = objective_t<M>(s, th, T);
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

// One annealing chain per thread.  Proposal: one coordinate j per step
// (cyclic), theta_j += sigma_j N(0, 1).  Acceptance: Metropolis at a
// temperature relative to the current objective, P = exp(-(J' - J) / (T J)),
// T falling geometrically from t0 to t1.  The objective's curvature differs
// by ~1e5 between coordinates (an outer threshold barely moves J, a weight
// does), so each coordinate keeps its own step: sigma_j grows by 1.25 on an
// accepted move and shrinks by 0.92 on a rejected one (equilibrium acceptance
// ~27 %), within [step1, 4 step0] x (1 for weights, (B - A)/8 for thresholds).
// Writes the chain's best point (canonical form) and its J.
template <int M>
__global__ void __launch_bounds__(128) fit_anneal_k(FitSpec s, AnnealCfg a, const double *init, double *chain_theta,
                                                     double *chain_J) {
  constexpr int P = 2 * M - 1;
  __shared__ FitTables tabs;
  const FitTables *T = build_tables(s, tabs);
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
  double sig[P];
#pragma unroll
  for (int i = 0; i < P; ++i) sig[i] = a.step0 * (i < M - 1 ? 1.0 : cscale);
  double J = objective_t<M>(s, th, T);
  double bestJ = J;
  const double lt = log(a.t1 / a.t0);
  for (int64_t it = 0; it < a.iters; ++it) {
    const double frac = a.iters > 1 ? (double)it / (double)(a.iters - 1) : 1.0;
    const double temp = a.t0 * exp(lt * frac);
    const int j = (int)(it % P);
    const double g = gauss(a.seed, ch, ctr);
    const double u = u01(a.seed, ch, (1ull << 62) + ctr);
    ctr += 1;
    double prop[P], sj = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      prop[i] = th[i] + (i == j ? sig[i] * g : 0.0);
      sj = i == j ? sig[i] : sj;
    }
    const double Jp = objective_t<M>(s, prop, T);
    const bool acc = Jp <= J || u < exp((J - Jp) / (temp * J));
    const double sc = j < M - 1 ? 1.0 : cscale;
    sj = fmin(fmax(sj * (acc ? 1.25 : 0.92), a.step1 * sc), 4.0 * a.step0 * sc);
#pragma unroll
    for (int i = 0; i < P; ++i) sig[i] = i == j ? sj : sig[i];
    if (acc) {
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

// Local refinement (Levenberg-Marquardt on J): SA settles slowly into the
// bottom of SiLU's long, curved valley (the objective's curvature spans ~1e5
// across coordinates and its valley is diagonal in (a, c)), so every chain's
// best point is finished by damped Newton steps.  Gradient and Hessian by
// central differences (2 P^2 evaluations per step) with steps 1e-4 x (1 for
// weights, (B - A)/8 for thresholds); solve (H + lambda diag H) d = -g by
// Cholesky; accept if J falls (lambda / 10), else lambda x 10; stop after
// `iters` steps or when 12 damping increases in a row find no decrease.
// Out-of-line objective for the refinement kernel: it is called 2 P^2 times
// per step, and inlining it into the Hessian loops made ptxas take hours.
template <int M>
__device__ __noinline__ double objective_call(const FitSpec &s, const double *th, const FitTables *T) {
  return objective_t<M>(s, th, T);
}

// ---------------------------------------------------------------------------
// Variable projection.  For fixed thresholds c the objective is a quadratic
// in the weights w under the linear constraint sum w = 1 (Eq. 14), so the
// optimal weights are a small linear solve:
//   J(w) = H0 - 2 b.w + w.G w,  G_ij = int r_i r_j,  b_i = int g r_i,
//   G w = b - lambda 1,  1.w = 1   =>   J*(c) = H0 - b.w - lambda,
// with r_i = ReLU(x - c_i), g = h (Eq. 15), or r_i = [x > c_i], g = h'
// (Eq. 17), all over [A, B].  Annealing then moves only the m thresholds:
// the search space halves and the ill-conditioned weight directions (an
// outer ReLU's weight is ~-0.04) disappear from it, which is what lets
// k >= 3 fits converge.  G has closed forms; b needs int_t^B h and
// int_t^B x h (obj 0; obj 1: b_i = h(B) - h(c_i) exactly), tabulated per CTA
// on the panel grid like the tail tables, plus one partial panel per kink.
// J* carries the cancellation H0 - ... (H0 ~ 1.8e4 for SiLU vs J ~ 0.04: ~1e-11
// relative), fine for the search; the reported J is re-evaluated directly.
// ---------------------------------------------------------------------------
struct VpTables {
  int n;                                        // cells; 0 = interval too long for the table
  double M0[kMaxCells + 1], M1[kMaxCells + 1];  // int_{x_i}^B h, int_{x_i}^B x h (obj 0)
  double H0;                                    // int_A^B h^2 (obj 0) or h'^2 (obj 1)
};

// int g, int x g, int g^2 over [l, r] (g = h for obj 0, h' for obj 1), one panel.
template <int ACT, int OBJ>
__device__ __noinline__ void vp_cell_t(double l, double r, double *m0, double *m1, double *gg) {
  const double mid = 0.5 * (l + r), half = 0.5 * (r - l);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int i = 0; i < kGLN / 2; ++i) {
    const double dx = half * gl_x(i);
    const double x0 = mid - dx, x1 = mid + dx;
    const double g0 = OBJ == 0 ? h_fn<ACT>(x0) : dh_fn<ACT>(x0);
    const double g1 = OBJ == 0 ? h_fn<ACT>(x1) : dh_fn<ACT>(x1);
    const double w = gl_w(i);
    a0 = fma(w, g0 + g1, a0);
    a1 = fma(w, fma(x0, g0, x1 * g1), a1);
    a2 = fma(w, fma(g0, g0, g1 * g1), a2);
  }
  *m0 = a0 * half;
  *m1 = a1 * half;
  *gg = a2 * half;
}

__device__ __forceinline__ void vp_cell(const FitSpec &s, double l, double r, double *m0, double *m1, double *gg) {
  if (s.act == kActGelu) {
    if (s.obj == 0) vp_cell_t<kActGelu, 0>(l, r, m0, m1, gg);
    else vp_cell_t<kActGelu, 1>(l, r, m0, m1, gg);
  } else {
    if (s.obj == 0) vp_cell_t<kActSilu, 0>(l, r, m0, m1, gg);
    else vp_cell_t<kActSilu, 1>(l, r, m0, m1, gg);
  }
}

__device__ __forceinline__ double vp_grid_x(const FitSpec &s, int n, int i) { return i >= n ? s.B : s.A + i * s.panel; }

// Every thread of the block must call this (it synchronises the block).
__device__ const VpTables *build_vp_tables(const FitSpec &s, VpTables &V, double *scratch /* >= kMaxCells */) {
  const int n = (int)ceil((s.B - s.A) / s.panel);
  if (threadIdx.x == 0) V.n = n <= kMaxCells ? n : 0;
  __syncthreads();
  if (V.n == 0) return nullptr;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    vp_cell(s, vp_grid_x(s, n, i), vp_grid_x(s, n, i + 1), &V.M0[i], &V.M1[i], &scratch[i]);
  __syncthreads();
  if (threadIdx.x == 0) {  // suffix sums and the total, fixed order
    V.M0[n] = V.M1[n] = 0.0;
    double h0 = 0.0;
    for (int i = n - 1; i >= 0; --i) {
      V.M0[i] += V.M0[i + 1];
      V.M1[i] += V.M1[i + 1];
      h0 += scratch[i];
    }
    V.H0 = h0;
  }
  __syncthreads();
  return &V;
}

// (int_t^B h, int_t^B x h) for t in [A, B].
__device__ __forceinline__ void vp_moments(const FitSpec &s, const VpTables &V, double t, double *m0, double *m1) {
  const int i = min(V.n - 1, max(0, (int)floor((t - s.A) / s.panel)));
  double p0, p1, p2;
  vp_cell(s, t, vp_grid_x(s, V.n, i + 1), &p0, &p1, &p2);
  *m0 = V.M0[i + 1] + p0;
  *m1 = V.M1[i + 1] + p1;
}

__device__ __forceinline__ double h_any(int act, double x) {
  return act == kActGelu ? h_fn<kActGelu>(x) : h_fn<kActSilu>(x);
}

// J*(c) and the optimal weights w (sum w = 1).  +inf if the normal equations
// are singular (e.g. several kinks beyond B).
template <int M>
__device__ double vp_objective(const FitSpec &s, const VpTables &V, const double *c, double *w) {
  double cc[M], b[M], G[M * M];
  for (int i = 0; i < M; ++i) {
    cc[i] = fmin(fmax(c[i], s.A), s.B);
    if (s.obj == 0) {
      double m0, m1;
      vp_moments(s, V, cc[i], &m0, &m1);
      b[i] = fma(-c[i], m0, m1);                    // int_{cc}^B h (x - c)
    } else {
      b[i] = h_any(s.act, s.B) - h_any(s.act, cc[i]);  // int_{cc}^B h'
    }
  }
  for (int i = 0; i < M; ++i) {
    for (int j = 0; j <= i; ++j) {
      const double m = fmax(cc[i], cc[j]);
      double g;
      if (s.obj == 0) {  // int_m^B (x - c_i)(x - c_j), u = x - c_i
        const double u0 = m - c[i], u1 = s.B - c[i], d = c[i] - c[j];
        g = (u1 * u1 * u1 - u0 * u0 * u0) / 3.0 + d * (u1 * u1 - u0 * u0) * 0.5;
      } else {
        g = s.B - m;
      }
      G[i * M + j] = G[j * M + i] = g;
    }
  }
  // Cholesky with a relative ridge, two right-hand sides (b and 1).
  double L[M * M];
  for (int i = 0; i < M; ++i) {
    for (int j = 0; j <= i; ++j) {
      double v = G[i * M + j] + (i == j ? 1e-13 * (fabs(G[i * M + i]) + 1.0) : 0.0);
      for (int q = 0; q < j; ++q) v -= L[i * M + q] * L[j * M + q];
      if (i == j) {
        if (!(v > 0.0)) return INFINITY;
        L[i * M + i] = sqrt(v);
      } else {
        L[i * M + j] = v / L[j * M + j];
      }
    }
  }
  double y[M], z[M];
  for (int i = 0; i < M; ++i) {
    double vy = b[i], vz = 1.0;
    for (int q = 0; q < i; ++q) {
      vy -= L[i * M + q] * y[q];
      vz -= L[i * M + q] * z[q];
    }
    y[i] = vy / L[i * M + i];
    z[i] = vz / L[i * M + i];
  }
  for (int i = M - 1; i >= 0; --i) {
    double vy = y[i], vz = z[i];
    for (int q = i + 1; q < M; ++q) {
      vy -= L[q * M + i] * y[q];
      vz -= L[q * M + i] * z[q];
    }
    y[i] = vy / L[i * M + i];
    z[i] = vz / L[i * M + i];
  }
  double sy = 0.0, sz = 0.0;
  for (int i = 0; i < M; ++i) {
    sy += y[i];
    sz += z[i];
  }
  const double lam = (sy - 1.0) / sz;
  double bw = 0.0;
  for (int i = 0; i < M; ++i) {
    w[i] = y[i] - lam * z[i];
    bw += b[i] * w[i];
  }
  const double J = V.H0 - bw - lam;
  return isfinite(J) ? fmax(J, 0.0) : INFINITY;
}

template <int M>
__device__ __noinline__ double vp_call(const FitSpec &s, const VpTables &V, const double *c, double *w) {
  return vp_objective<M>(s, V, c, w);
}

// Annealing over the thresholds only, weights by variable projection.  Same
// proposal / acceptance / step adaptation as fit_anneal_k; the chain's best
// (w*, c) is written in canonical form with its J re-evaluated by the direct
// quadrature (objective_t).  Intervals too long for the table: J = +inf.
template <int M>
__global__ void __launch_bounds__(128) fit_anneal_vp_k(FitSpec s, AnnealCfg a, const double *init,
                                                        double *chain_theta, double *chain_J) {
  constexpr int P = 2 * M - 1;
  __shared__ VpTables vt;
  __shared__ double scratch[kMaxCells];
  const VpTables *V = build_vp_tables(s, vt, scratch);
  const int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= a.chains) return;
  if (!V) {
    for (int i = 0; i < P; ++i) chain_theta[ch * P + i] = 0.0;
    chain_J[ch] = INFINITY;
    return;
  }
  const double cscale = (s.B - s.A) * 0.125;
  double c[M], w[M], bc[M], bw[M], sig[M], pc[M], pw[M];
  uint64_t ctr = 0;
  for (int i = 0; i < M; ++i) {
    c[i] = init ? init[M - 1 + i] : s.A * 0.5 + (s.B - s.A) * 0.5 * u01(a.seed, ch, ctr++);
    sig[i] = a.step0 * cscale;
  }
  double J = vp_call<M>(s, *V, c, w);
  double bestJ = J;
  for (int i = 0; i < M; ++i) {
    bc[i] = c[i];
    bw[i] = w[i];
  }
  ctr = 1ull << 40;
  const double lt = log(a.t1 / a.t0);
  for (int64_t it = 0; it < a.iters; ++it) {
    const double frac = a.iters > 1 ? (double)it / (double)(a.iters - 1) : 1.0;
    const double temp = a.t0 * exp(lt * frac);
    const int j = (int)(it % M);
    const double g = gauss(a.seed, ch, ctr);
    const double u = u01(a.seed, ch, (1ull << 62) + ctr);
    ctr += 1;
    for (int i = 0; i < M; ++i) pc[i] = c[i] + (i == j ? sig[i] * g : 0.0);
    const double Jp = vp_call<M>(s, *V, pc, pw);
    const bool acc = Jp <= J || u < exp((J - Jp) / (temp * J));
    sig[j] = fmin(fmax(sig[j] * (acc ? 1.25 : 0.92), a.step1 * cscale), 4.0 * a.step0 * cscale);
    if (acc) {
      J = Jp;
      for (int i = 0; i < M; ++i) {
        c[i] = pc[i];
        w[i] = pw[i];
      }
      if (J < bestJ) {
        bestJ = J;
        for (int i = 0; i < M; ++i) {
          bc[i] = c[i];
          bw[i] = w[i];
        }
      }
    }
  }
  double th[P], out[P];
  for (int i = 0; i < M - 1; ++i) th[i] = bw[i];
  for (int i = 0; i < M; ++i) th[M - 1 + i] = bc[i];
  canonical<M>(th, out);
  for (int i = 0; i < P; ++i) chain_theta[ch * P + i] = out[i];
  chain_J[ch] = objective_call<M>(s, out, nullptr);
}

template <int P>
__device__ bool cholesky_solve(const double *H, const double *g, double lam, double *d) {
  double L[P * P];
  for (int i = 0; i < P; ++i) {
    for (int j = 0; j <= i; ++j) {
      double v = H[i * P + j] + (i == j ? lam * fabs(H[i * P + i]) + 1e-300 : 0.0);
      for (int q = 0; q < j; ++q) v -= L[i * P + q] * L[j * P + q];
      if (i == j) {
        if (!(v > 0.0)) return false;
        L[i * P + i] = sqrt(v);
      } else {
        L[i * P + j] = v / L[j * P + j];
      }
    }
  }
  double y[P];
  for (int i = 0; i < P; ++i) {
    double v = -g[i];
    for (int q = 0; q < i; ++q) v -= L[i * P + q] * y[q];
    y[i] = v / L[i * P + i];
  }
  for (int i = P - 1; i >= 0; --i) {
    double v = y[i];
    for (int q = i + 1; q < P; ++q) v -= L[q * P + i] * d[q];
    d[i] = v / L[i * P + i];
  }
  return true;
}

template <int M>
__global__ void __launch_bounds__(128) fit_refine_k(FitSpec s, const double *in, int64_t n, int64_t iters,
                                                     double *out, double *Jout) {
  constexpr int P = 2 * M - 1;
  __shared__ FitTables tabs;
  const FitTables *T = build_tables(s, tabs);
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double cscale = (s.B - s.A) * 0.125;
  double th[P], h[P], g[P], H[P * P], tp[P], d[P];
  for (int i = 0; i < P; ++i) {
    th[i] = in[t * P + i];
    h[i] = 1e-4 * (i < M - 1 ? 1.0 : cscale);
  }
  double J = objective_call<M>(s, th, T);
  double lam = 1e-3;
  for (int64_t it = 0; it < iters && isfinite(J); ++it) {
    for (int i = 0; i < P; ++i) tp[i] = th[i];
    for (int i = 0; i < P; ++i) {
      tp[i] = th[i] + h[i];
      const double jp = objective_call<M>(s, tp, T);
      tp[i] = th[i] - h[i];
      const double jm = objective_call<M>(s, tp, T);
      tp[i] = th[i];
      g[i] = (jp - jm) / (2.0 * h[i]);
      H[i * P + i] = (jp - 2.0 * J + jm) / (h[i] * h[i]);
    }
    for (int i = 0; i < P; ++i) {
      for (int j = 0; j < i; ++j) {
        double acc = 0.0;
        for (int q = 0; q < 4; ++q) {
          const double si = (q & 1) ? -1.0 : 1.0, sj = (q & 2) ? -1.0 : 1.0;
          tp[i] = th[i] + si * h[i];
          tp[j] = th[j] + sj * h[j];
          acc += si * sj * objective_call<M>(s, tp, T);
        }
        tp[i] = th[i];
        tp[j] = th[j];
        H[i * P + j] = H[j * P + i] = acc / (4.0 * h[i] * h[j]);
      }
    }
    bool moved = false;
    for (int tries = 0; tries < 12 && !moved; ++tries, lam *= 10.0) {
      if (!cholesky_solve<P>(H, g, lam, d)) continue;
      for (int i = 0; i < P; ++i) tp[i] = th[i] + d[i];
      const double Jn = objective_call<M>(s, tp, T);
      if (Jn < J) {
        for (int i = 0; i < P; ++i) th[i] = tp[i];
        J = Jn;
        moved = true;
        lam = fmax(lam * 0.01, 1e-12);  // / 10 after the loop's x 10
      }
    }
    if (!moved) break;
  }
  double o[P];
  canonical<M>(th, o);
  for (int i = 0; i < P; ++i) out[t * P + i] = o[i];
  Jout[t] = J;
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

template <int M>
cudaError_t anneal_vp_m(const FitSpec &s, const AnnealCfg &a, const double *init, double *chain_theta,
                        double *chain_J, double *best, cudaStream_t st) {
  const int64_t blocks = (a.chains + 127) / 128;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  fit_anneal_vp_k<M><<<(int)blocks, 128, 0, st>>>(s, a, init, chain_theta, chain_J);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  fit_best_k<<<1, 1024, 0, st>>>(chain_theta, chain_J, a.chains, 2 * M - 1, best);
  return cudaGetLastError();
}

template <int M>
cudaError_t refine_m(const FitSpec &s, const double *in, int64_t n, int64_t iters, double *out, double *Jout,
                     double *best, cudaStream_t st) {
  const int64_t blocks = (n + 127) / 128;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  fit_refine_k<M><<<(int)blocks, 128, 0, st>>>(s, in, n, iters, out, Jout);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !best) return e;
  fit_best_k<<<1, 1024, 0, st>>>(out, Jout, n, 2 * M - 1, best);
  return cudaGetLastError();
}

}  // namespace

cudaError_t fit_anneal_vp(const FitSpec &s, int k, const AnnealCfg &a, const double *init, double *chain_theta,
                          double *chain_J, double *best, cudaStream_t st) {
  switch (k) {
    case 1: return anneal_vp_m<1>(s, a, init, chain_theta, chain_J, best, st);
    case 2: return anneal_vp_m<3>(s, a, init, chain_theta, chain_J, best, st);
    case 3: return anneal_vp_m<7>(s, a, init, chain_theta, chain_J, best, st);
    default: return anneal_vp_m<15>(s, a, init, chain_theta, chain_J, best, st);
  }
}

cudaError_t fit_refine(const FitSpec &s, int k, const double *in, int64_t n, int64_t iters, double *out,
                       double *Jout, double *best, cudaStream_t st) {
  switch (k) {
    case 1: return refine_m<1>(s, in, n, iters, out, Jout, best, st);
    case 2: return refine_m<3>(s, in, n, iters, out, Jout, best, st);
    case 3: return refine_m<7>(s, in, n, iters, out, Jout, best, st);
    default: return refine_m<15>(s, in, n, iters, out, Jout, best, st);
  }
}

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
