// bgk_device.cuh -- device math shared by the BesselK and Matern kernels (sm_100a).
//
// Everything here is FP64.  The hot loops are bound by the FP64 pipe (64 lanes
// per SM per clock on B200), so exponentials and logs are table-driven
// (128-entry tables in shared memory, 7-11 FP64 ops) instead of libdevice exp /
// log (15-29 ops + range checks); rarely-hit paths (Temme series, out-of-range
// parameters) keep libdevice for robustness.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "bgk_tables.cuh"

namespace bgk {

constexpr double kLn2 = 0.6931471805599453;  // kernels.py:16
constexpr double kPi = 3.141592653589793;

// ---------------------------------------------------------------------------------
// 128-entry table exp / log.  Coefficients live in __constant__ memory so DFMA
// takes them as constant-bank operands (no per-iteration register moves).
// ---------------------------------------------------------------------------------
__device__ __constant__ double kExpK[8] = {
    0x1.71547652b82fep+7,   // 0: 128/ln2
    0x1.62e42fefa39efp-8,   // 1: ln2/128 (hi)
    0x1.abc9e3b39803fp-63,  // 2: ln2/128 (lo)
    1.0 / 24.0,             // 3
    1.0 / 6.0,              // 4
    1.0 / 120.0,            // 5
    0x1.8p52,               // 6: round-to-int magic
    0.0};
__device__ __constant__ double kLogK[8] = {
    0.2, -1.0 / 6.0, -0.25, 1.0 / 3.0, -0.5,
    0x1.62e4200000000p-1,   // 5: ln2 hi (21 bits: e * hi is exact)
    0x1.fdf473de6af28p-22,  // 6: ln2 lo
    0.0};

// Copy the 128-entry exp table and the log tables into shared memory.  The exp
// table is stored "scale-compensated": entry j is 2^(j/128) with j << 13
// subtracted from its high word.  Adding n << 13 (n = 128 q + j) to that high
// word then yields 2^(j/128) 2^q, because n << 13 == (q << 20) + (j << 13)
// mod 2^32: one integer op (LEA) instead of shift + mask + add.  Read entries
// only through exp2_scaled().
__device__ __forceinline__ void load_tables128(double *exp128, double *invc, double *logc) {
  for (int j = threadIdx.x; j < 128; j += blockDim.x) {
    const double v = kExp2Tab128[j];
    exp128[j] = __hiloint2double(__double2hiint(v) - (j << 13), __double2loint(v));
    invc[j] = kInvC128[j];
    logc[j] = kLogC128[j];
  }
}

// 2^(n/128) from the scale-compensated table (load_tables128); exact for
// n/128 in the normal range.
__device__ __forceinline__ double exp2_scaled(const double *__restrict__ t128, int n) {
  const double tv = t128[n & 127];
  return __hiloint2double(__double2hiint(tv) + (n << 13), __double2loint(tv));
}

// e^y for a quadrature node, y in (-707, 700): 128-entry table, degree-4
// polynomial on |r| <= ln2/256 (truncation 1.2e-15) and a one-constant
// reduction (error |y| * 1.2e-16, harmless because the term is e^y).
// 7 FP64 ops + LDS + 4 integer ops.
__device__ __forceinline__ double exp_node(double y, const double *__restrict__ t128) {
  const double t = fma(y, kExpK[0], kExpK[6]);
  const double nd = t - kExpK[6];
  const int n = __double2loint(t);
  const double r = fma(nd, -kExpK[1], y);
  double p = fma(r, kExpK[3], kExpK[4]);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return exp2_scaled(t128, n) * p;
}

// e^y to ~2 ulp for |y| < 700 (two-constant reduction, degree 5).
__device__ __forceinline__ double exp_acc(double y, const double *__restrict__ t128) {
  const double t = fma(y, kExpK[0], kExpK[6]);
  const double nd = t - kExpK[6];
  const int n = __double2loint(t);
  double r = fma(nd, -kExpK[1], y);
  r = fma(nd, -kExpK[2], r);
  double p = fma(r, kExpK[5], kExpK[3]);
  p = fma(p, r, kExpK[4]);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return exp2_scaled(t128, n) * p;
}

// (e^z, e^-z) for |z| < 700 with one argument reduction: e^{+-r} = even +- odd
// (degree 6 / 5 in r, |r| <= ln2/256, truncation < 1e-21), scaled by 2^{+-n/128}.
// 15 FP64 ops for both (two exp_acc: 22).
__device__ __forceinline__ void exp_pair(double z, const double *__restrict__ t128, double &ep,
                                         double &em) {
  const double t = fma(z, kExpK[0], kExpK[6]);
  const double nd = t - kExpK[6];
  const int n = __double2loint(t);
  double r = fma(nd, -kExpK[1], z);
  r = fma(nd, -kExpK[2], r);
  const double r2 = r * r;
  double ev = fma(r2, 1.0 / 720.0, 1.0 / 24.0);
  ev = fma(ev, r2, 0.5);
  ev = fma(ev, r2, 1.0);
  double od = fma(r2, 1.0 / 120.0, 1.0 / 6.0);
  od = fma(od, r2, 1.0);
  od *= r;
  ep = exp2_scaled(t128, n) * (ev + od);
  em = exp2_scaled(t128, -n) * (ev - od);
}

// log(x) for positive, normal, finite x: x = 2^e m, m in [1,2), table point
// c_j = 1 + (j+1/2)/128, f = m/c_j - 1 (|f| <= 1/256), log1p(f) to degree 6.
// ~11 FP64 ops, <= 1 ulp-ish.
__device__ __forceinline__ double log_fast(double x, const double *__restrict__ invc,
                                           const double *__restrict__ logc) {
  const int hi = __double2hiint(x);
  const int e = (hi >> 20) - 1023;
  const int j = (hi >> 13) & 127;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(x));
  const double f = fma(m, invc[j], -1.0);
  double q = fma(f, kLogK[1], kLogK[0]);
  q = fma(q, f, kLogK[2]);
  q = fma(q, f, kLogK[3]);
  q = fma(q, f, kLogK[4]);
  const double l1p = fma(q, f * f, f);
  const double ed = (double)e;
  return fma(ed, kLogK[5], logc[j]) + fma(ed, kLogK[6], l1p);
}

// kernels.py:43-49
__device__ __forceinline__ double log_cosh(double z) {
  z = fabs(z);
  if (z < 25.0) return log(cosh(z));
  return z - kLn2 + log1p(exp(-2.0 * z));
}

// ---------------------------------------------------------------------------------
// Temme small-argument series (kernels.py:219-293).  Same formulas and stop rule
// as the reference; libdevice tgamma/sin/sinh/cosh/exp/log (<= 2 ulp).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double gamma1(double mu) {  // kernels.py:219-227
  const double G[12] = {
      0.57721566490153286061,   -0.042002635034095235529, -0.042197734555544336748,
      0.0072189432466630995424, -0.00021524167411495097282, -2.0134854780788238656e-05,
      1.1330272319816958824e-06, 6.1160951044814158179e-09, -1.1812745704870201446e-09,
      7.782263439905071254e-12,  5.100370287454475979e-13,  -5.3481225394230179824e-15};
  double acc = 0.0, mu2 = mu * mu, p = 1.0;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    acc += G[i] * p;
    p *= mu2;
  }
  return -acc;
}

// The nu-only part of temme_sums (kernels.py:240-245, 251-252).
struct TemmeConst {
  double mu, gam1, gam2, fact, g1p, g1m;
  int m_steps;
};

__device__ __forceinline__ TemmeConst temme_const(double nu) {
  TemmeConst T;
  T.m_steps = (int)floor(nu + 0.5);  // kernels.py:281
  T.mu = nu - (double)T.m_steps;
  T.gam1 = gamma1(T.mu);
  T.g1m = tgamma(1.0 - T.mu);
  T.g1p = tgamma(1.0 + T.mu);
  T.gam2 = 0.5 * (1.0 / T.g1m + 1.0 / T.g1p);
  T.fact = (fabs(T.mu) < 1e-10) ? 1.0 : T.mu * kPi / sin(T.mu * kPi);
  return T;
}

// kernels.py:230-270 with the nu-only constants supplied.  Returns terms.
__device__ __forceinline__ long long temme_sums_c(double x, const TemmeConst &T, double eps,
                                                  long long cap, double &s0o, double &s1o) {
  const double mu = T.mu;
  double d = log(2.0 / x);
  double sigma = mu * d;
  double sh = (sigma == 0.0) ? 1.0 : sinh(sigma) / sigma;
  double f = T.fact * (cosh(sigma) * T.gam1 + T.gam2 * sh * d);
  double p = 0.5 * exp(sigma) * T.g1p;
  double q = 0.5 * exp(-sigma) * T.g1m;
  double c = 1.0, s0 = f, s1 = p, x2_4 = 0.25 * x * x;
  long long terms = 1;
  for (long long k = 1; k < cap + 1; ++k) {
    double kd = (double)k;
    f = (kd * f + p + q) / (kd * kd - mu * mu);
    p /= (kd - mu);
    q /= (kd + mu);
    c *= x2_4 / kd;
    double del0 = c * f;
    double del1 = c * (p - kd * f);
    s0 += del0;
    s1 += del1;
    terms = k + 1;
    if (fabs(del0) < eps * fabs(s0) && fabs(del1) < eps * fabs(s1)) break;
  }
  s0o = s0;
  s1o = s1;
  return terms;
}

// kernels.py:273-293: ln K_nu(x) via Temme + log-space forward recurrence.
__device__ __forceinline__ double temme_series_log_c(double x, const TemmeConst &T, double eps,
                                                     long long cap) {
  double s0, s1;
  temme_sums_c(x, T, eps, cap, s0, s1);
  double l_prev = log(s0);
  if (T.m_steps == 0) return l_prev;
  double l_cur = kLn2 - log(x) + log(s1);
  // The reference's log-space step l' = l + log(2 eta / x + e^{l_prev - l}) is
  // the linear forward recurrence K' = (2 eta / x) K + K_prev (stable: K grows
  // with the order) taken in logs.  Run it linearly from K_prev = 1 (scale
  // e^{l_prev}) -- one FMA per step instead of a log and an exp -- rescaling
  // when K grows large, and take one log at the end.  Same values to a few ulp
  // of ln K.
  // Overflow-safe bounds: one step grows K by at most (eta 2/x + 1) <= 2^311
  // for x >= 2^-300 and fewer than 1000 steps, so rescaling above 2^400 keeps
  // every intermediate finite; outside those bounds, the log-space loop.
  if (T.m_steps > 1 && T.m_steps < 1000 && x >= 0x1p-300) {
    const double inv2x = 2.0 / x;
    double kp = 1.0, kc = exp(l_cur - l_prev), off = l_prev;
    if (kc <= 0x1p400) {
      for (int k = 1; k < T.m_steps; ++k) {
        const double kn = fma(T.mu + (double)k, inv2x * kc, kp);
        kp = kc;
        kc = kn;
        if (kc > 0x1p400) {  // rescale by an exact power of two (rare)
          kp *= 0x1p-400;
          kc *= 0x1p-400;
          off += 400.0 * kLn2;
        }
      }
      return off + log(kc);
    }
  }
  for (int k = 1; k < T.m_steps; ++k) {
    double eta = T.mu + (double)k;
    double l_next = l_cur + log(2.0 * eta / x + exp(l_prev - l_cur));
    l_prev = l_cur;
    l_cur = l_next;
  }
  return l_cur;
}

// ---------------------------------------------------------------------------------
// Reference-faithful fixed-window quadrature (kernels.py:112-216): grid argmax,
// hyperbolic-identity node exponents, walk with the -46 break, Kahan, rebase.
// Used only where the fast kernels' preconditions fail (t_lower < 0, nu*t so
// large that e^(nu t) overflows, very large bin counts).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double node_exponent_ref(double anu, double x, double dt,
                                                    double z_star, double lc_star,
                                                    double ch_star, double ss, double cs) {
  double z_m = z_star + anu * dt;
  double da;
  if (z_m >= 30.0 && z_star >= 30.0)
    da = anu * dt;
  else if (z_m < 25.0 && z_star < 25.0)
    da = log(cosh(z_m) / ch_star);
  else
    da = log_cosh(z_m) - lc_star;
  double sh = sinh(0.5 * dt);
  double ch = cosh(0.5 * dt);
  double db = 2.0 * x * (ss * ch + cs * sh) * sh;
  return da - db;
}

__device__ __noinline__ static double fixed_window_log_ref(double x, double nu, double t0, double t1, long long bins) {
  const double h = (t1 - t0) / (double)bins;
  // grid_peak_index, kernels.py:112-123
  double best = -INFINITY;
  long long m_star = 0;
  for (long long m = 0; m < bins + 1; ++m) {
    double t = t0 + (double)m * h;
    double g = log_cosh(nu * t) - x * cosh(t);
    if (g > best) {
      best = g;
      m_star = m;
    }
  }
  // window_lse, kernels.py:154-209
  double anu = fabs(nu);
  double t_star = t0 + (double)m_star * h;
  double z_star = anu * t_star;
  double lc_star = log_cosh(z_star);
  double ch_star = (z_star < 25.0) ? cosh(z_star) : INFINITY;
  double ss = sinh(t_star), cs = cosh(t_star);
  double acc = (0 < m_star && m_star < bins) ? 1.0 : 0.5;
  double comp = 0.0;
  for (int direction = 0; direction < 2; ++direction) {
    double sign = (direction == 0) ? 1.0 : -1.0;
    long long span = (direction == 0) ? (bins - m_star) : m_star;
    for (long long k = 1; k < span + 1; ++k) {
      double dt = sign * ((double)k * h);
      double dg = node_exponent_ref(anu, x, dt, z_star, lc_star, ch_star, ss, cs);
      if (dg <= -46.0) break;
      long long m = m_star + ((direction == 0) ? k : -k);
      double w = (m == 0 || m == bins) ? 0.5 : 1.0;
      double y = w * exp(dg) - comp;
      double t_acc = acc + y;
      comp = (t_acc - acc) - y;
      acc = t_acc;
    }
  }
  double t_hat = (anu * anu <= x) ? 0.0 : asinh(anu / x);
  double z_hat = anu * t_hat;
  double shift = log_cosh(z_hat) - x * cosh(t_hat);
  double dt_sh = t_star - t_hat;
  double da_sh = (z_star >= 30.0 && z_hat >= 30.0) ? anu * dt_sh : lc_star - log_cosh(z_hat);
  double sh = sinh(0.5 * dt_sh);
  double db_sh = 2.0 * x * (sinh(t_hat) * cosh(0.5 * dt_sh) + cosh(t_hat) * sh) * sh;
  return shift + ((da_sh - db_sh) + log(h * acc));
}

}  // namespace bgk
