// bgk_besselk.cu -- batch K_nu(x) for sm_100a (the "K1" kernel of SURVEY.md 2.2).
//
// Replaces kernels.refined_log_bessel / fixed_window_log_pair / temme_series_log
// (kernels.py:212-302) over device arrays.  Same discretisation as the
// reference -- nodes t_m = t0 + m h, trapezoid weights 1/2 at both ends, strict
// x < threshold routing, Temme + log-space recurrence below it -- so results
// agree with the reference to ~1e-13 relative (tests/test_parity_besselk.py).
//
// Integral path, per element (x, nu), a = |nu|:
//   anchor node m_a near the log-integrand peak: 0 if a^2 <= x (g decreasing,
//   kernels.py:148-151), else round(asinh(a/x)/h) (fp32 is plenty -- the anchor
//   only sets the scale of the sum; any node near the peak gives the same value
//   to rounding).
//   With E = e^{a h} and q = e^{-2 a t_a}, node m_a +- j contributes
//       2 cosh(a t_k) e^{-x c_k} / (e^{a t_a} e^{-x c_a}) = (E^{+-j} + q E^{-+j}) e^{-x (c_k - c_a)}
//   so every node costs one table exp plus three multiplies -- no per-node
//   log_cosh (the reference's 73% hot spot).  c_k = cosh(t_k) is a
//   per-CTA shared-memory table.  Both directions are walked in the same loop
//   iteration (two independent exp chains for ILP) until the term falls below
//   e^{-50} of the anchor, which includes every node the reference's e^{-46}
//   break keeps.
//       ln K = a t_a - ln2 - x c_a + ln(h * acc)
//
// Series elements (x < thr, 0.08% of the BK config) are rare but ~10x the work
// of an integral element; a lane that takes them stalls its whole warp.  Each
// CTA therefore defers them into a shared-memory queue and runs the queue
// compacted after the integral pass.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bgk_device.cuh"
#include "bgk_internal.h"

namespace bgk {

constexpr int kBkThreads = 256;
constexpr int kBkPerThread = 4;
constexpr int kBkChunk = kBkThreads * kBkPerThread;

struct BkArgs {
  const double *x;
  const double *nu;
  double *log_k;
  double *k;
  uint8_t *path;
  long long n;
  double t0, t1, h, thr, eps;
  long long cap;
  int bins;
  int route;
  int table_ok;  // 1: c table fits in shared memory and t0 >= 0 -> fast path allowed
};

// Fast fixed-window quadrature (see file header).  Requires t0 >= 0 and
// a * max(t1, t0) <= 600 so that E^j never overflows.
__device__ __forceinline__ double fixed_window_fast(double x, double a, const BkArgs &A,
                                                    const double *__restrict__ ctab,
                                                    const double *__restrict__ tab) {
  const int bins = A.bins;
  int m;
  if (a * a <= x) {
    m = 0;
  } else {
    float ts = asinhf((float)a / (float)x);
    float fm = rintf((ts - (float)A.t0) * (float)(1.0 / A.h));
    fm = fminf(fmaxf(fm, 0.0f), (float)bins);
    m = (int)fm;
  }
  const double ta = A.t0 + (double)m * A.h;
  const double ca = ctab[m];
  const double E = exp_tab(a * A.h, tab);
  const double Ei = exp_tab(-a * A.h, tab);
  const double two_at = 2.0 * a * ta;
  const double q = (two_at < 700.0) ? exp_tab(-two_at, tab) : 0.0;
  const double anchor = 1.0 + q;
  const double tiny = 1.9287498479639178e-22 * anchor;  // e^-50 of the anchor term
  const double mx = -x;
  double acc = ((m == 0 || m == bins) ? 0.5 : 1.0) * anchor;

  double pu = 1.0, qu = 1.0, pd = 1.0, qd = 1.0;
  bool up = m < bins, dn = m > 0;
  int j = 1;
  while (up || dn) {
    if (up) {
      pu *= E;
      qu *= Ei;
      const int k = m + j;
      double s = fma(q, qu, pu);
      double y = fmax(mx * (ctab[k] - ca), -700.0);
      double term = s * exp_tab(y, tab);
      if (term < tiny) {
        up = false;
      } else {
        acc = fma((k == bins) ? 0.5 : 1.0, term, acc);
        up = k < bins;
      }
    }
    if (dn) {
      pd *= Ei;
      qd *= E;
      const int k = m - j;
      double s = fma(q, qd, pd);
      double y = fmax(mx * (ctab[k] - ca), -700.0);
      double term = s * exp_tab(y, tab);
      if (term < tiny) {
        dn = false;
      } else {
        acc = fma((k == 0) ? 0.5 : 1.0, term, acc);
        dn = k > 0;
      }
    }
    ++j;
  }
  return (a * ta - kLn2) - x * ca + log(A.h * acc);
}

__device__ __forceinline__ void bk_store(const BkArgs &A, long long i, double lk, uint8_t path,
                                         const double *tab) {
  A.log_k[i] = lk;
  if (A.k) A.k[i] = exp_full(lk, tab);
  if (A.path) A.path[i] = path;
}

__global__ void __launch_bounds__(kBkThreads) besselk_kernel(BkArgs A) {
  extern __shared__ double smem[];
  double *tab = smem;       // 64
  double *ctab = smem + 64;  // bins + 1 (only when table_ok)
  __shared__ int q_count;
  __shared__ int q_idx[kBkChunk];

  load_exp_tab(tab);
  if (A.table_ok)
    for (int k = threadIdx.x; k <= A.bins; k += blockDim.x) ctab[k] = cosh(A.t0 + (double)k * A.h);
  if (threadIdx.x == 0) q_count = 0;
  __syncthreads();

  const long long base = (long long)blockIdx.x * kBkChunk;
  const double tmax = fmax(fabs(A.t0), fabs(A.t1));
#pragma unroll 1
  for (int s = 0; s < kBkPerThread; ++s) {
    const int off = s * kBkThreads + threadIdx.x;
    const long long i = base + off;
    if (i >= A.n) break;
    const double x = A.x[i];
    const double nu = A.nu[i];
    const bool series = (A.route == 1) || (A.route == 0 && x < A.thr);
    if (series) {
      q_idx[atomicAdd(&q_count, 1)] = off;
      continue;
    }
    const double a = fabs(nu);
    double lk;
    if (A.table_ok && a * tmax <= 600.0)
      lk = fixed_window_fast(x, a, A, ctab, tab);
    else
      lk = fixed_window_log_ref(x, nu, A.t0, A.t1, A.bins);
    bk_store(A, i, lk, 1, tab);
  }
  __syncthreads();
  // Deferred series elements, compacted across the CTA.
  const int nq = q_count;
  for (int s = threadIdx.x; s < nq; s += blockDim.x) {
    const long long i = base + q_idx[s];
    const double x = A.x[i];
    const TemmeConst T = temme_const(A.nu[i]);
    const double lk = temme_series_log_c(x, T, A.eps, A.cap);
    bk_store(A, i, lk, 0, tab);
  }
}

__global__ void temme_sums_kernel(const double *x, const double *mu, long long n, double eps,
                                  long long cap, double *s0, double *s1, int64_t *terms) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // temme_sums takes mu directly (kernels.py:230); build the mu-only constants.
  TemmeConst T;
  T.mu = mu[i];
  T.m_steps = 0;
  T.gam1 = gamma1(T.mu);
  T.g1m = tgamma(1.0 - T.mu);
  T.g1p = tgamma(1.0 + T.mu);
  T.gam2 = 0.5 * (1.0 / T.g1m + 1.0 / T.g1p);
  T.fact = (fabs(T.mu) < 1e-10) ? 1.0 : T.mu * kPi / sin(T.mu * kPi);
  double a, b;
  long long t = temme_sums_c(x[i], T, eps, cap, a, b);
  s0[i] = a;
  s1[i] = b;
  if (terms) terms[i] = t;
}

// kernels.py:52-72
__global__ void log_integrand_kernel(const double *t, const double *x, const double *nu,
                                     long long n, int order, double *out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double ti = t[i], xi = x[i], ni = nu[i];
  double r;
  if (order == 0) {
    r = log_cosh(ni * ti) - xi * cosh(ti);
  } else if (order == 1) {
    r = ni * tanh(ni * ti) - xi * sinh(ti);
  } else {
    double z = fabs(ni * ti);
    double sech = (z < 350.0) ? 1.0 / cosh(z) : 0.0;
    r = ni * ni * sech * sech - xi * cosh(ti);
  }
  out[i] = r;
}

}  // namespace bgk

// ---------------------------------------------------------------------------------
// launchers (called from bgk_capi.cpp)
// ---------------------------------------------------------------------------------
int bgk_launch_besselk(const double *x, const double *nu, int64_t n, const bgk_config *cfg,
                       int route, double *log_k, double *k, uint8_t *path, cudaStream_t stream) {
  if (n == 0) return 0;
  bgk::BkArgs A;
  A.x = x;
  A.nu = nu;
  A.log_k = log_k;
  A.k = k;
  A.path = path;
  A.n = n;
  A.t0 = cfg->t_lower;
  A.t1 = cfg->t_upper;
  A.h = (cfg->t_upper - cfg->t_lower) / (double)cfg->bins;
  A.thr = cfg->small_x_threshold;
  A.eps = cfg->eps_machine;
  A.cap = cfg->series_cap;
  A.bins = (int)cfg->bins;
  A.route = route;
  const int64_t kMaxTable = 16383;  // 128 KB of shared memory
  A.table_ok = (cfg->t_lower >= 0.0 && cfg->bins <= kMaxTable) ? 1 : 0;
  size_t smem = sizeof(double) * (64 + (A.table_ok ? (size_t)cfg->bins + 1 : 0));
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(bgk::besselk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * (64 + kMaxTable + 1)));
    attr_set = true;
  }
  long long grid = (n + bgk::kBkChunk - 1) / bgk::kBkChunk;
  bgk::besselk_kernel<<<(unsigned)grid, bgk::kBkThreads, smem, stream>>>(A);
  bgk_note_launch();
  return bgk_check_launch("besselk_kernel");
}

int bgk_launch_temme_sums(const double *x, const double *mu, int64_t n, const bgk_config *cfg,
                          double *s0, double *s1, int64_t *terms, cudaStream_t stream) {
  if (n == 0) return 0;
  long long grid = (n + 255) / 256;
  bgk::temme_sums_kernel<<<(unsigned)grid, 256, 0, stream>>>(x, mu, n, cfg->eps_machine,
                                                             cfg->series_cap, s0, s1, terms);
  bgk_note_launch();
  return bgk_check_launch("temme_sums_kernel");
}

int bgk_launch_log_integrand(const double *t, const double *x, const double *nu, int64_t n,
                             int order, double *out, cudaStream_t stream) {
  if (n == 0) return 0;
  long long grid = (n + 255) / 256;
  bgk::log_integrand_kernel<<<(unsigned)grid, 256, 0, stream>>>(t, x, nu, n, order, out);
  bgk_note_launch();
  return bgk_check_launch("log_integrand_kernel");
}
