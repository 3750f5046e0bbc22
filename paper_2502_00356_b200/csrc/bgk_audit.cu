// bgk_audit.cu -- GPU accuracy audit: the reference's
// dynamic-window oracle (oracle.py:47-160, Takekawa's FINDRANGE / FINDZERO with
// Newton + bisection, then the fine-grid window_lse of kernels.py:154-209) and
// the production / pure-integral decompositions, emitted as base-10 logs with
// the reference's double-double assembly (kernels.py:97-109, 332-335).
//
// One CTA per (nu, x) point.  Thread 0 finds the window (a serial root finder,
// ~1e4 FP64 ops); the CTA then sums the 2^16-bin trapezoid: each thread takes a
// contiguous run of nodes with Kahan summation, partials are combined in thread
// order (deterministic).  Node exponents use the reference's hyperbolic
// identities (node_exponent_ref) and the result is rebased onto the canonical
// anchor exactly as window_lse does.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bgk_device.cuh"
#include "bgk_internal.h"

namespace bgk {

constexpr int kAuditThreads = 128;
constexpr double kLnEps = -36.04365338911715;  // log(2^-52), oracle.py:26
constexpr double kInvLn10Hi = 0.4342944819032518, kInvLn10Lo = 1.098319650216765e-17;

// kernels.py:52-72
__device__ __forceinline__ double g0f(double t, double x, double nu) {
  return log_cosh(nu * t) - x * cosh(t);
}
__device__ __forceinline__ double g1f(double t, double x, double nu) {
  return nu * tanh(nu * t) - x * sinh(t);
}
__device__ __forceinline__ double g2f(double t, double x, double nu) {
  const double z = fabs(nu * t);
  const double sech = (z < 350.0) ? 1.0 / cosh(z) : 0.0;
  return nu * nu * sech * sech - x * cosh(t);
}

// the three functions the window search roots (selected by `which`)
struct Fn {
  double x, nu, target, shift;
  int which;  // 0: g'(t)  1: g(t) - target  2: g(shift + s) - target
  __device__ double f(double t) const {
    if (which == 0) return g1f(t, x, nu);
    if (which == 1) return g0f(t, x, nu) - target;
    return g0f(shift + t, x, nu) - target;
  }
  __device__ double df(double t) const {
    if (which == 0) return g2f(t, x, nu);
    if (which == 1) return g1f(t, x, nu);
    return g1f(shift + t, x, nu);
  }
};

// oracle.py:47-56: smallest m in [-40, 64] with f(2^m) < 0 -> (2^(m-1), 2^m)
__device__ bool find_range(const Fn &F, double &lo, double &hi) {
  for (int m = -40; m <= 64; ++m) {
    const double t = ldexp(1.0, m);
    if (F.f(t) < 0.0) {
      lo = ldexp(1.0, m - 1);
      hi = t;
      return true;
    }
  }
  return false;
}

__device__ __forceinline__ double copysign1(double v) { return copysign(1.0, v); }

// oracle.py:59-89: bisection, switching to Newton when the step stays inside.
__device__ bool find_zero(const Fn &F, double lo, double hi, double tol, double &root) {
  double flo = F.f(lo);
  if (flo == 0.0) { root = lo; return true; }
  const double fhi = F.f(hi);
  if (fhi == 0.0) { root = hi; return true; }
  if (copysign1(flo) == copysign1(fhi)) return false;
  for (int it = 0; it < 200; ++it) {
    if (hi - lo <= tol) { root = 0.5 * (lo + hi); return true; }
    const double mid = 0.5 * (lo + hi);
    double step_to = mid;
    const double d = F.df(mid);
    if (d != 0.0) {
      const double newton = mid - F.f(mid) / d;
      if (lo < newton && newton < hi) step_to = newton;
    }
    const double fm = F.f(step_to);
    if (fm == 0.0) { root = step_to; return true; }
    if (copysign1(fm) == copysign1(flo)) { lo = step_to; flo = fm; } else { hi = step_to; }
  }
  return false;
}

// oracle.py:92-125 integration_window; returns false on ConvergenceError.
__device__ bool integration_window(double x, double nu, double tol, double &t0, double &t1,
                                   double &t_max) {
  Fn F{x, nu, 0.0, 0.0, 0};
  if (nu * nu <= x) {
    t_max = 0.0;
  } else {
    double lo, hi;
    if (!find_range(F, lo, hi) || !find_zero(F, lo, hi, tol, t_max)) return false;
  }
  const double target = g0f(t_max, x, nu) + kLnEps;
  Fn D{x, nu, target, 0.0, 1};
  if (D.f(0.0) >= 0.0) {
    t0 = 0.0;
  } else if (!find_zero(D, 0.0, t_max, tol, t0)) {
    return false;
  }
  Fn S{x, nu, target, t_max, 2};
  double lo, hi;
  if (!find_range(S, lo, hi)) return false;
  return find_zero(D, t_max + lo, t_max + hi, tol, t1);
}

// kernels.py:97-109: (shift + ln_sum) / ln 10 with one final rounding
__device__ __forceinline__ void two_prod(double a, double b, double &p, double &e) {
  p = __dmul_rn(a, b);
  e = fma(a, b, -p);  // exact product error (the reference uses Dekker's split)
}
__device__ __forceinline__ double assemble_log10(double shift, double ln_sum) {
  double p1, e1, p2, e2;
  two_prod(shift, kInvLn10Hi, p1, e1);
  two_prod(ln_sum, kInvLn10Hi, p2, e2);
  const double lo = shift * kInvLn10Lo + ln_sum * kInvLn10Lo + e1 + e2;
  const double s = p1 + p2;
  const double bb = s - p1;
  const double e = (p1 - (s - bb)) + (p2 - bb);
  return s + (e + lo);
}

struct AuditArgs {
  const double *nus, *xs;
  long long nnu, nx;
  double t0, t1, thr, eps, tol;
  long long bins, cap;
  int method;  // 0 refined, 1 pure integral (fixed window), 2 dynamic-window oracle
  int base10;   // 1: base-10 log (double-double assembly), 0: natural log shift + ln_sum
  double *out;  // nnu x nx, row-major, log K (NaN where the oracle fails)
};

// CTA-parallel window_lse (kernels.py:154-209): nodes with dg > -46 from the
// anchor m_star (the reference's walk stops at the first such node on each side;
// g is unimodal so the sets agree), Kahan per thread, ordered combine, rebase.
__device__ void window_lse_cta(double x, double nu, double t0, double t1, long long bins,
                               long long m_star, double *red, double &shift, double &ln_sum) {
  const double h = (t1 - t0) / (double)bins;
  const double anu = fabs(nu);
  const double t_star = t0 + (double)m_star * h;
  const double z_star = anu * t_star;
  const double lc_star = log_cosh(z_star);
  const double ch_star = (z_star < 25.0) ? cosh(z_star) : INFINITY;
  const double ss = sinh(t_star), cs = cosh(t_star);
  const long long n = bins + 1;
  const long long per = (n + blockDim.x - 1) / blockDim.x;
  const long long k0 = threadIdx.x * per;
  const long long k1 = min(n, k0 + per);
  double acc = 0.0, comp = 0.0;
  for (long long m = k0; m < k1; ++m) {
    double term;
    if (m == m_star) {
      term = (0 < m_star && m_star < bins) ? 1.0 : 0.5;
    } else {
      const double dt = (m > m_star) ? (double)(m - m_star) * h : -((double)(m_star - m) * h);
      const double dg = node_exponent_ref(anu, x, dt, z_star, lc_star, ch_star, ss, cs);
      if (dg <= -46.0) continue;
      term = ((m == 0 || m == bins) ? 0.5 : 1.0) * exp(dg);
    }
    const double y = term - comp;
    const double ta = acc + y;
    comp = (ta - acc) - y;
    acc = ta;
  }
  red[2 * threadIdx.x] = acc;
  red[2 * threadIdx.x + 1] = comp;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const double y = (red[2 * t] - red[2 * t + 1]) - c;
      const double ta = a + y;
      c = (ta - a) - y;
      a = ta;
    }
    const double t_hat = (anu * anu <= x) ? 0.0 : asinh(anu / x);
    const double z_hat = anu * t_hat;
    shift = log_cosh(z_hat) - x * cosh(t_hat);
    const double dt_sh = t_star - t_hat;
    const double da_sh =
        (z_star >= 30.0 && z_hat >= 30.0) ? anu * dt_sh : lc_star - log_cosh(z_hat);
    const double sh = sinh(0.5 * dt_sh);
    const double db_sh = 2.0 * x * (sinh(t_hat) * cosh(0.5 * dt_sh) + cosh(t_hat) * sh) * sh;
    ln_sum = (da_sh - db_sh) + log(h * a);
  }
}

__global__ void __launch_bounds__(kAuditThreads) audit_kernel(const __grid_constant__ AuditArgs A) {
  __shared__ double red[2 * kAuditThreads];
  __shared__ double s_win[3];
  __shared__ long long s_mstar;
  __shared__ int s_mode;  // 0 series, 1 window, 2 failed
  const long long pt = blockIdx.x;
  const long long i = pt / A.nx, j = pt % A.nx;
  const double nu = A.nus[i], x = A.xs[j];
  if (threadIdx.x == 0) {
    const bool series = (A.method != 1) && x < A.thr;
    s_mode = series ? 0 : 1;
    if (!series) {
      double t0 = A.t0, t1 = A.t1, t_max = 0.0;
      long long ms;
      if (A.method == 2) {
        if (!(x > 0.0) || !integration_window(x, nu, A.tol, t0, t1, t_max)) s_mode = 2;
        const double h = (t1 - t0) / (double)A.bins;
        ms = (long long)rint((t_max - t0) / h);  // oracle.py:131 round()
        ms = ms < 0 ? 0 : (ms > A.bins ? A.bins : ms);
      } else {  // grid argmax, kernels.py:112-123
        const double h = (t1 - t0) / (double)A.bins;
        double best = -INFINITY;
        ms = 0;
        for (long long m = 0; m <= A.bins; ++m) {
          const double g = g0f(t0 + (double)m * h, x, nu);
          if (g > best) { best = g; ms = m; }
        }
      }
      s_win[0] = t0;
      s_win[1] = t1;
      s_win[2] = t_max;
      s_mstar = ms;
    }
  }
  __syncthreads();
  const int mode = s_mode;
  if (mode == 2) {
    if (threadIdx.x == 0) A.out[pt] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  if (mode == 0) {
    if (threadIdx.x == 0) {  // kernels.py:312-314 / oracle.py:157-159
      const TemmeConst T = temme_const(nu);
      const double ln_k = temme_series_log_c(x, T, A.eps, A.cap);
      A.out[pt] = A.base10 ? ln_k * kInvLn10Hi + ln_k * kInvLn10Lo : ln_k;
    }
    return;
  }
  double shift = 0.0, ln_sum = 0.0;
  window_lse_cta(x, nu, s_win[0], s_win[1], A.bins, s_mstar, red, shift, ln_sum);
  if (threadIdx.x == 0) A.out[pt] = A.base10 ? assemble_log10(shift, ln_sum) : shift + ln_sum;
}

}  // namespace bgk

extern "C" int bgk_log_grid(const double *nus, int64_t nnu, const double *xs, int64_t nx,
                            const bgk_config *cfg, int method, int64_t bins, int base10,
                            double *out, void *stream) {
  if (!cfg || nnu < 0 || nx < 0 || method < 0 || method > 2 || bins < 1 ||
      (nnu * nx > 0 && (!nus || !xs || !out))) {
    bgk_set_error("bgk_log_grid: bad arguments");
    return BGK_ERR_INVALID;
  }
  if (nnu * nx == 0) return BGK_OK;
  if (nnu * nx > 0x7fffffffLL) {
    bgk_set_error("bgk_log_grid: grid too large for one launch");
    return BGK_ERR_UNSUPPORTED;
  }
  bgk::AuditArgs A;
  A.nus = nus;
  A.xs = xs;
  A.nnu = nnu;
  A.nx = nx;
  A.t0 = cfg->t_lower;
  A.t1 = cfg->t_upper;
  A.thr = cfg->small_x_threshold;
  A.eps = cfg->eps_machine;
  A.cap = cfg->series_cap;
  A.tol = 1e-12;  // oracle.py:92 default
  A.bins = (method == 2) ? bins : cfg->bins;
  A.method = method;
  A.base10 = base10 ? 1 : 0;
  A.out = out;
  bgk::audit_kernel<<<(unsigned)(nnu * nx), bgk::kAuditThreads, 0, (cudaStream_t)stream>>>(A);
  bgk_note_launch();
  return bgk_check_launch("audit_kernel");
}
