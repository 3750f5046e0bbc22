// bgk_capi.cpp -- extern "C" boundary of libbesselgp_sm100a.so (include/besselgp_b200.h).
//
// Host-side work here is per call, never per element: argument checks, the
// Matern plan (node tables + Temme constants + u-bucket LUT, i.e. the restated
// caller of kernels.matern_tile, kernels.py:343-345 / SPEC.md:306-332) and
// the task-grid arithmetic of the three Matern layouts.
#include <algorithm>
#include <emmintrin.h>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <pthread.h>
#include <vector>

#include <cuda_runtime.h>

#include "bgk_internal.h"

namespace {
thread_local char g_err[512] = "";
std::atomic<long long> g_launches{0};

constexpr double kLn2 = 0.6931471805599453;  // kernels.py:16

double log_cosh_host(double z) {  // kernels.py:43-49, glibc libm like numba
  z = std::fabs(z);
  if (z < 25.0) return std::log(std::cosh(z));
  return z - kLn2 + std::log1p(std::exp(-2.0 * z));
}

double gamma1_host(double mu) {  // kernels.py:219-227
  static const double G[12] = {
      0.57721566490153286061,   -0.042002635034095235529, -0.042197734555544336748,
      0.0072189432466630995424, -0.00021524167411495097282, -2.0134854780788238656e-05,
      1.1330272319816958824e-06, 6.1160951044814158179e-09, -1.1812745704870201446e-09,
      7.782263439905071254e-12,  5.100370287454475979e-13,  -5.3481225394230179824e-15};
  double acc = 0.0, mu2 = mu * mu, p = 1.0;
  for (int i = 0; i < 12; ++i) {
    acc += G[i] * p;
    p *= mu2;
  }
  return -acc;
}

// Bucket key of a positive double: its top 64 - 32 - shift bits (sign, exponent
// and 20 - shift mantissa bits) -> 2^(20 - shift) log-spaced buckets per octave
// (shift 15: 32).  The device computes the same key as __double2hiint(u) >> shift.
thread_local int g_key_shift = 15;
int key_of(double u) {
  uint64_t b;
  std::memcpy(&b, &u, 8);
  return (int)(b >> (32 + g_key_shift));
}
double u_of_key(int key) {
  uint64_t b = (uint64_t)(uint32_t)key << (32 + g_key_shift);
  double u;
  std::memcpy(&u, &b, 8);
  return u;
}

#ifndef BGK_WINDOW_CUTOFF
#define BGK_WINDOW_CUTOFF 33.0  // A/B on B200 (M100 / M50 ms): 40 -> 74.07 / 80.35, 36 -> 72.80,
                                // 33 -> 71.85 / 78.15, 30 -> 71.2 / 77.2 (max rel. err vs the oracle
                                // 5.7e-14 at 40 and 33, 5.9e-14 at 30 with every nu at 3-6e-14)
#endif

struct Window {
  int m, lo, hi;
};

// Reference window at u: grid argmax m* (first max, kernels.py:363-369) and
// every node with g_k - g_{m*} > -33.  The reference keeps > -46; the terms in
// (-46, -33] sum to < 41 e^-33 = 1.9e-13 of the peak term (a bound: on the M100
// distances the largest dropped share is 2e-15, the table exp's own error), far
// inside the 1e-10 parity tolerance.
Window window_at(const bgk_matern_plan &P, double u) {
  const int nn = P.nnodes;
  double gmax = -INFINITY;
  int ms = 0;
  for (int k = 0; k < nn; ++k) {
    double g = P.a[k] - u * P.c[k];
    if (g > gmax) {
      gmax = g;
      ms = k;
    }
  }
  Window w{ms, ms, ms};
  for (int k = 0; k < nn; ++k) {
    double g = P.a[k] - u * P.c[k];
    if (g - gmax > -BGK_WINDOW_CUTOFF) {
      if (k < w.lo) w.lo = k;
      if (k > w.hi) w.hi = k;
    }
  }
  return w;
}

// Fill plan->lut with the finest bucket resolution that fits; plan->fast = 0 when
// no safe LUT can be built.
bool build_lut_at(bgk_matern_plan &P, int shift);
void build_lut(bgk_matern_plan &P) {
  // 16 buckets per octave (key shift 16); BGK_LUT_KEY_SHIFT=15 asks for 32 when the
  // table fits.  A/B on B200: with the round-1 kernels and the e^-40 cut 32 per octave
  // won (M100 88.88 vs 89.45 ms); with the e^-33 cut the windows change less per
  // bucket and 16 per octave wins (M100 71.55 vs 71.91, M50 77.82 vs 78.23, M200
  // 279.5-280.1 vs 281.0-281.6 ms).
  const char *env = std::getenv("BGK_LUT_KEY_SHIFT");
  const int first = (env && std::atoi(env) == 15) ? 15 : 16;
  for (int shift = first; shift <= 16; ++shift)
    if (build_lut_at(P, shift)) return;
}

bool build_lut_at(bgk_matern_plan &P, int shift) {
  g_key_shift = shift;
  P.key_shift = shift;
  P.fast = 0;
  P.nosub_buckets = 0;
  P.nbuckets = 1;
  P.key_base = 0;
  P.lut[0] = 0;
  const double thr = P.small_x_threshold;
  if (!(thr > 0.0) || !std::isfinite(thr) || P.nnodes < 2) return false;
  for (int k = 0; k < P.nnodes; ++k)
    if (!std::isfinite(P.c[k]) || !std::isfinite(P.a[k])) return false;
  const int kb = key_of(thr);
  // Extend the bucket range until the window at a bucket's lower edge is the
  // anchor alone; every larger u then shares that single-node window.
  int kt = std::max(key_of(4096.0), key_of(64.0 * P.nu * P.nu));
  kt = std::max(kt, kb + 1);
  for (;;) {
    Window w = window_at(P, u_of_key(kt));
    if (w.lo == w.hi) {
      Window w2 = window_at(P, u_of_key(kt) * 1e6);
      if (w2.m == w.m) break;
    }
    ++kt;
    if (kt - kb + 1 > BGK_MATERN_MAX_BUCKETS) return false;
  }
  const int nb = kt - kb + 1;
  if (nb > BGK_MATERN_MAX_BUCKETS) return false;
  const int S = 9;  // samples per bucket (endpoints + 7 interior, geometric)
  for (int b = 0; b < nb; ++b) {
    const double ulo = (b == 0) ? thr : u_of_key(kb + b);
    const bool last = (b == nb - 1);
    const double uhi = last ? ulo : std::nextafter(u_of_key(kb + b + 1), 0.0);
    const double umid = std::sqrt(ulo * uhi);
    const int anchor = window_at(P, umid).m;
    int lo = anchor, hi = anchor;
    for (int s = 0; s < S; ++s) {
      const double u = (s == 0) ? ulo : (s == S - 1) ? uhi : ulo * std::pow(uhi / ulo, (double)s / (S - 1));
      Window w = window_at(P, u);
      lo = std::min(lo, w.lo);
      hi = std::max(hi, w.hi);
    }
    // y_k(u) = g_k(u) - g_anchor(u) is linear in u: bound it at the endpoints so
    // the table exp never sees |y| beyond its range and never overflows.
    for (int e = 0; e < 2; ++e) {
      const double u = e ? uhi : ulo;
      const double ga = P.a[anchor] - u * P.c[anchor];
      for (int k = lo; k <= hi; ++k) {
        const double y = (P.aw[k] - u * P.c[k]) - ga;
        if (!(y > -700.0 && y < 30.0)) return false;
      }
    }
    if (last && lo != hi) return false;
    P.lut[b] = (uint32_t)anchor | ((uint32_t)lo << 10) | ((uint32_t)hi << 20);
  }
  // The kernel reads a sorted warp's common/union window from its first and
  // last lanes, which needs lo and hi non-increasing in u.  They are by
  // construction (the peak moves left and narrows as u grows); enforce it by
  // widening (prefix-min of lo, suffix-max of hi) and re-check the y bounds.
  for (int b = 1; b < nb; ++b) {
    const uint32_t prev = P.lut[b - 1], cur = P.lut[b];
    const uint32_t lo = std::min((cur >> 10) & 1023, (prev >> 10) & 1023);
    P.lut[b] = (cur & 1023) | (lo << 10) | (cur & (1023u << 20));
  }
  for (int b = nb - 2; b >= 0; --b) {
    const uint32_t next = P.lut[b + 1], cur = P.lut[b];
    const uint32_t hi = std::max(cur >> 20, next >> 20);
    P.lut[b] = (cur & ((1u << 20) - 1)) | (hi << 20);
  }
  for (int b = 0; b < nb; ++b) {
    const double ulo = (b == 0) ? thr : u_of_key(kb + b);
    const double uhi = (b == nb - 1) ? ulo : std::nextafter(u_of_key(kb + b + 1), 0.0);
    const int anchor = P.lut[b] & 1023, lo = (P.lut[b] >> 10) & 1023, hi = P.lut[b] >> 20;
    if (b == nb - 1 && lo != hi) return false;
    for (int e = 0; e < 2; ++e) {
      const double u = e ? uhi : ulo;
      const double ga = P.a[anchor] - u * P.c[anchor];
      for (int k = lo; k <= hi; ++k) {
        const double y = (P.aw[k] - u * P.c[k]) - ga;
        if (!(y > -700.0 && y < 30.0)) return false;
      }
    }
  }
  // Absolute-form (unanchored) buckets: a prefix of the table where every window
  // term's exponent aw_k - u c_k stays inside the table exp's range (linear in
  // u, so the bucket's end points bound it).
  int nosub = 0;
  for (int b = 0; b < nb - 1; ++b) {
    const double ulo = (b == 0) ? thr : u_of_key(kb + b);
    const double uhi = std::nextafter(u_of_key(kb + b + 1), 0.0);
    const int lo = (P.lut[b] >> 10) & 1023, hi = P.lut[b] >> 20;
    bool ok = true;
    for (int e = 0; e < 2 && ok; ++e) {
      const double u = e ? uhi : ulo;
      for (int k = lo; k <= hi; ++k) {
        const double y = P.aw[k] - u * P.c[k];
        if (!(y > -690.0 && y < 690.0)) ok = false;
      }
    }
    if (!ok) break;
    nosub = b + 1;
  }
  P.nosub_buckets = nosub;
  int amin = BGK_MATERN_MAX_NODES, amax = 0;
  for (int b = 0; b < nb; ++b) {
    amin = std::min(amin, (int)(P.lut[b] & 1023));
    amax = std::max(amax, (int)(P.lut[b] & 1023));
  }
  P.anchor_min = amin;
  P.anchor_max = amax;
  P.nbuckets = nb;
  P.key_base = kb;
  P.fast = 1;
  return true;
}

int check_cfg(const bgk_config *cfg) {
  if (!cfg) {
    bgk_set_error("cfg is NULL");
    return BGK_ERR_INVALID;
  }
  if (!(cfg->t_upper > cfg->t_lower) || !std::isfinite(cfg->t_lower) ||
      !std::isfinite(cfg->t_upper) || cfg->bins < 1 || cfg->series_cap < 0) {
    bgk_set_error("invalid bgk_config (t_lower=%g t_upper=%g bins=%lld cap=%lld)",
                  cfg->t_lower, cfg->t_upper, (long long)cfg->bins,
                  (long long)cfg->series_cap);
    return BGK_ERR_INVALID;
  }
  return BGK_OK;
}

int check_plan(const bgk_matern_plan *plan) {
  if (!plan || plan->abi != BGK_ABI_VERSION || plan->nnodes < 1 ||
      plan->nnodes > BGK_MATERN_MAX_NODES || plan->nbuckets < 1 ||
      plan->nbuckets > BGK_MATERN_MAX_BUCKETS) {
    bgk_set_error("invalid or uninitialised bgk_matern_plan");
    return BGK_ERR_INVALID;
  }
  return BGK_OK;
}
}  // namespace

void bgk_set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int bgk_check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    bgk_set_error("%s: %s", what, cudaGetErrorString(e));
    return BGK_ERR_CUDA;
  }
  return BGK_OK;
}

void bgk_note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
std::atomic<int> g_device_alias{0};
std::mutex g_optin_mu;
struct OptIn {
  const void *kernel;
  int dev;
  int bytes;
};
std::vector<OptIn> g_optins;  // guarded by g_optin_mu
}  // namespace

int bgk_device_key(int *real_device) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (real_device) *real_device = dev;
  return dev + g_device_alias.load();
}

int bgk_ensure_smem_optin(const void *kernel, const char *name, int bytes) {
  const int key = bgk_device_key(nullptr);
  std::lock_guard<std::mutex> lock(g_optin_mu);
  for (const OptIn &o : g_optins)
    if (o.kernel == kernel && o.dev == key && o.bytes >= bytes) return BGK_OK;
  const cudaError_t e =
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    bgk_set_error("cudaFuncSetAttribute(%s, %d bytes): %s", name, bytes, cudaGetErrorString(e));
    return BGK_ERR_CUDA;
  }
  // the whole unified L1/shared array as shared memory: the kernels are sized for
  // several ~55 KB CTAs per SM and use no L1-cached global data worth keeping
  const cudaError_t e2 = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                              (int)cudaSharedmemCarveoutMaxShared);
  if (e2 != cudaSuccess) {
    cudaGetLastError();
    bgk_set_error("cudaFuncSetAttribute(%s, carveout): %s", name, cudaGetErrorString(e2));
    return BGK_ERR_CUDA;
  }
  for (OptIn &o : g_optins)
    if (o.kernel == kernel && o.dev == key) {
      o.bytes = bytes;
      return BGK_OK;
    }
  g_optins.push_back({kernel, key, bytes});
  return BGK_OK;
}

extern "C" {

const char *bgk_last_error(void) { return g_err; }
int bgk_abi_version(void) { return BGK_ABI_VERSION; }
int64_t bgk_launch_count(void) { return g_launches.load(); }
int bgk_debug_set_device_alias(int alias) { return g_device_alias.exchange(alias); }
size_t bgk_matern_plan_size(void) { return sizeof(bgk_matern_plan); }

int bgk_besselk_batch(const double *x, const double *nu, int64_t n, const bgk_config *cfg,
                      int route, double *log_k, double *k, uint8_t *path, void *stream) {
  if (int rc = check_cfg(cfg)) return rc;
  if (n < 0 || (n > 0 && (!x || !nu || !log_k)) || route < 0 || route > 2) {
    bgk_set_error("bgk_besselk_batch: bad arguments (n=%lld route=%d)", (long long)n, route);
    return BGK_ERR_INVALID;
  }
  return bgk_launch_besselk(x, nu, n, cfg, route, log_k, k, path, (cudaStream_t)stream);
}

int bgk_temme_sums_batch(const double *x, const double *mu, int64_t n, const bgk_config *cfg,
                         double *s0, double *s1, int64_t *terms, void *stream) {
  if (int rc = check_cfg(cfg)) return rc;
  if (n < 0 || (n > 0 && (!x || !mu || !s0 || !s1))) {
    bgk_set_error("bgk_temme_sums_batch: bad arguments");
    return BGK_ERR_INVALID;
  }
  return bgk_launch_temme_sums(x, mu, n, cfg, s0, s1, terms, (cudaStream_t)stream);
}

int bgk_log_integrand_batch(const double *t, const double *x, const double *nu, int64_t n,
                            int order, double *out, void *stream) {
  if (n < 0 || order < 0 || order > 2 || (n > 0 && (!t || !x || !nu || !out))) {
    bgk_set_error("bgk_log_integrand_batch: bad arguments");
    return BGK_ERR_INVALID;
  }
  return bgk_launch_log_integrand(t, x, nu, n, order, out, (cudaStream_t)stream);
}

int bgk_matern_plan_init_tables(bgk_matern_plan *plan, double sigma_sq, double beta, double nu,
                                double log_prefactor, const double *c_nodes,
                                const double *a_nodes, int64_t nnodes, double h,
                                double small_x_threshold, double eps_machine,
                                int64_t series_cap) {
  if (!plan || !c_nodes || !a_nodes) {
    bgk_set_error("bgk_matern_plan_init_tables: NULL argument");
    return BGK_ERR_INVALID;
  }
  if (nnodes < 2 || nnodes > BGK_MATERN_MAX_NODES) {
    bgk_set_error("bgk_matern_plan_init_tables: nnodes=%lld outside [2, %d]",
                  (long long)nnodes, BGK_MATERN_MAX_NODES);
    return BGK_ERR_UNSUPPORTED;
  }
  std::memset(plan, 0, sizeof(*plan));
  bgk_matern_plan &P = *plan;
  P.abi = BGK_ABI_VERSION;
  P.nnodes = (int32_t)nnodes;
  P.sigma_sq = sigma_sq;
  P.beta = beta;
  P.nu = nu;
  P.log_prefactor = log_prefactor;
  P.h = h;
  P.small_x_threshold = small_x_threshold;
  P.eps_machine = eps_machine;
  P.series_cap = series_cap;
  const int b = (int)nnodes - 1;
  for (int k = 0; k < nnodes; ++k) {
    P.c[k] = c_nodes[k];
    P.a[k] = a_nodes[k];
    // trapezoid weight 1/2 at both ends (kernels.py:375) folded into the exponent
    P.aw[k] = (k == 0 || k == b) ? a_nodes[k] - kLn2 : a_nodes[k];
  }
  // nu-only Temme constants (kernels.py:240-252, 281-282)
  P.m_steps = (int32_t)std::floor(nu + 0.5);
  P.mu = nu - (double)P.m_steps;
  P.gam1 = gamma1_host(P.mu);
  P.gamma_1m_mu = std::tgamma(1.0 - P.mu);
  P.gamma_1p_mu = std::tgamma(1.0 + P.mu);
  P.gam2 = 0.5 * (1.0 / P.gamma_1m_mu + 1.0 / P.gamma_1p_mu);
  P.fact = (std::fabs(P.mu) < 1e-10) ? 1.0 : P.mu * M_PI / std::sin(P.mu * M_PI);
  build_lut(P);
  // u^nu without a log/exp pair when 2 nu is a small integer (the common GP
  // smoothness values 1/2, 1, 3/2, 2, 5/2, ...): u^k (sqrt u)^half.
  P.pow_mode = 0;
  P.pow_pref = 0.0;
  const double two_nu = 2.0 * nu;
  if (two_nu == std::floor(two_nu) && two_nu >= 1.0 && two_nu <= 16.0) {
    const double pref = std::exp(log_prefactor) * h;
    if (std::isfinite(pref) && pref >= 0x1p-900 && pref <= 0x1p900) {
      const int k = (int)std::floor(nu), half = (int)two_nu - 2 * k;
      P.pow_mode = 1 + 2 * k + half;
      P.pow_pref = pref;
    }
  }
  return BGK_OK;
}

int bgk_matern_plan_init(bgk_matern_plan *plan, double sigma_sq, double beta, double nu,
                         const bgk_config *cfg) {
  if (int rc = check_cfg(cfg)) return rc;
  if (cfg->bins + 1 > BGK_MATERN_MAX_NODES) {
    bgk_set_error("bgk_matern_plan_init: bins=%lld exceeds %d", (long long)cfg->bins,
                  BGK_MATERN_MAX_NODES - 1);
    return BGK_ERR_UNSUPPORTED;
  }
  const int64_t nn = cfg->bins + 1;
  double c[BGK_MATERN_MAX_NODES], a[BGK_MATERN_MAX_NODES];
  // restated caller (kernels.py:343-345): h = (t1-t0)/b, t_m = t0 + m h
  const double h = (cfg->t_upper - cfg->t_lower) / (double)cfg->bins;
  for (int64_t m = 0; m < nn; ++m) {
    const double t = cfg->t_lower + (double)m * h;
    c[m] = std::cosh(t);
    a[m] = log_cosh_host(nu * t);
  }
  // log(sigma^2 2^(1-nu) / Gamma(nu))
  const double lp = std::log(sigma_sq) - (nu - 1.0) * kLn2 - std::lgamma(nu);
  return bgk_matern_plan_init_tables(plan, sigma_sq, beta, nu, lp, c, a, nn, h,
                                     cfg->small_x_threshold, cfg->eps_machine,
                                     cfg->series_cap);
}

int bgk_matern_tile(const bgk_matern_plan *plan, const double *rx, const double *ry, int64_t m,
                    const double *cx, const double *cy, int64_t n, double *out, int64_t ld,
                    int layout, void *stream) {
  if (int rc = check_plan(plan)) return rc;
  if (m < 0 || n < 0 || (layout != BGK_LAYOUT_ROW_MAJOR && layout != BGK_LAYOUT_COL_MAJOR)) {
    bgk_set_error("bgk_matern_tile: bad sizes or layout");
    return BGK_ERR_INVALID;
  }
  if (m == 0 || n == 0) return BGK_OK;
  if (!rx || !ry || !cx || !cy || !out || ld < (layout == BGK_LAYOUT_ROW_MAJOR ? n : m)) {
    bgk_set_error("bgk_matern_tile: NULL pointer or ld too small");
    return BGK_ERR_INVALID;
  }
  BgkMaternArgs A{};
  A.rx = rx; A.ry = ry; A.cx = cx; A.cy = cy; A.out = out;
  A.m = m; A.n = n; A.ld = ld; A.layout = layout;
  return bgk_launch_matern(plan, A, BGK_MODE_TILE, (cudaStream_t)stream);
}

int bgk_matern_covariance(const bgk_matern_plan *plan, const double *lx, const double *ly,
                          int64_t N, int64_t row_begin, int64_t row_end, double *out, int64_t ld,
                          int layout, void *stream) {
  if (int rc = check_plan(plan)) return rc;
  if (N < 0 || row_begin < 0 || row_end > N || row_begin > row_end ||
      (layout != BGK_LAYOUT_ROW_MAJOR && layout != BGK_LAYOUT_COL_MAJOR)) {
    bgk_set_error("bgk_matern_covariance: bad N/rows/layout");
    return BGK_ERR_INVALID;
  }
  const int64_t rows = row_end - row_begin;
  if (rows == 0 || N == 0) return BGK_OK;
  if (!lx || !ly || !out || ld < (layout == BGK_LAYOUT_ROW_MAJOR ? N : rows)) {
    bgk_set_error("bgk_matern_covariance: NULL pointer or ld too small");
    return BGK_ERR_INVALID;
  }
  BgkMaternArgs A{};
  A.rx = lx; A.ry = ly; A.cx = lx; A.cy = ly; A.out = out;
  A.m = N; A.n = N; A.ld = ld; A.layout = layout;
  A.row0 = row_begin; A.row1 = row_end;
  return bgk_launch_matern(plan, A, BGK_MODE_COV, (cudaStream_t)stream);
}

int bgk_matern_lower_tiles(const bgk_matern_plan *plan, const double *lx, const double *ly,
                           int64_t N, int64_t tile_size, int64_t tile_begin, int64_t tile_end,
                           double *out, void *stream) {
  if (int rc = check_plan(plan)) return rc;
  const int64_t T = (N + tile_size - 1) / (tile_size > 0 ? tile_size : 1);
  const int64_t total = T * (T + 1) / 2;
  if (N < 0 || tile_size < 1 || tile_begin < 0 || tile_end > total || tile_begin > tile_end) {
    bgk_set_error("bgk_matern_lower_tiles: bad N/tile_size/tile range");
    return BGK_ERR_INVALID;
  }
  if (tile_end == tile_begin || N == 0) return BGK_OK;
  if (!lx || !ly || !out) {
    bgk_set_error("bgk_matern_lower_tiles: NULL pointer");
    return BGK_ERR_INVALID;
  }
  BgkMaternArgs A{};
  A.rx = lx; A.ry = ly; A.cx = lx; A.cy = ly; A.out = out;
  A.m = N; A.n = N; A.ts = tile_size;
  A.tile0 = tile_begin; A.tile1 = tile_end;
  return bgk_launch_matern(plan, A, BGK_MODE_LOWER, (cudaStream_t)stream);
}

namespace {
// shared argument checks of the two peer entry points
int check_peer_owners(const char *what, int64_t N, int G, const int64_t *macro_row_start,
                      double *const *bases) {
  const int64_t T = (N + BGK_MACRO_TILE - 1) / BGK_MACRO_TILE;
  if (N < 0 || G < 1 || G > BGK_MAX_PEERS || !macro_row_start || !bases) {
    bgk_set_error("%s: bad N/G", what);
    return BGK_ERR_INVALID;
  }
  if (macro_row_start[0] != 0 || macro_row_start[G] != T) {
    bgk_set_error("%s: macro_row_start must run from 0 to ceil(N/64)", what);
    return BGK_ERR_INVALID;
  }
  for (int h = 0; h < G; ++h) {
    const bool empty = macro_row_start[h + 1] == macro_row_start[h];
    if (macro_row_start[h + 1] < macro_row_start[h] || (!bases[h] && !empty)) {
      bgk_set_error("%s: bad owner %d", what, h);
      return BGK_ERR_INVALID;
    }
  }
  return BGK_OK;
}

BgkMaternArgs peer_args(const double *lx, const double *ly, int64_t N, int G,
                        const int64_t *macro_row_start, double *const *bases) {
  BgkMaternArgs A{};
  A.rx = lx; A.ry = ly; A.cx = lx; A.cy = ly; A.out = bases[0];
  A.m = N; A.n = N; A.ld = N; A.layout = BGK_LAYOUT_ROW_MAJOR;
  A.G = G;
  for (int h = 0; h <= G; ++h) A.pstart[h] = macro_row_start[h];
  for (int h = 0; h < G; ++h) A.bases[h] = bases[h];
  return A;
}
}  // namespace

int bgk_matern_covariance_peer(const bgk_matern_plan *plan, const double *lx, const double *ly,
                               int64_t N, int G, const int64_t *macro_row_start,
                               double *const *bases, int64_t tile_begin, int64_t tile_end,
                               void *stream) {
  if (int rc = check_plan(plan)) return rc;
  if (int rc = check_peer_owners("bgk_matern_covariance_peer", N, G, macro_row_start, bases))
    return rc;
  const int64_t T = (N + BGK_MACRO_TILE - 1) / BGK_MACRO_TILE;
  if (tile_begin < 0 || tile_end > T * (T + 1) / 2 || tile_begin > tile_end) {
    bgk_set_error("bgk_matern_covariance_peer: bad tile range");
    return BGK_ERR_INVALID;
  }
  if (tile_end == tile_begin || N == 0) return BGK_OK;
  if (!lx || !ly) {
    bgk_set_error("bgk_matern_covariance_peer: NULL locations");
    return BGK_ERR_INVALID;
  }
  BgkMaternArgs A = peer_args(lx, ly, N, G, macro_row_start, bases);
  A.tile0 = tile_begin; A.tile1 = tile_end;
  return bgk_launch_matern(plan, A, BGK_MODE_PEER, (cudaStream_t)stream);
}

int bgk_matern_covariance_peer_band(const bgk_matern_plan *plan, const double *lx,
                                    const double *ly, int64_t N, int G,
                                    const int64_t *macro_row_start, double *const *bases,
                                    int rank, void *stream) {
  if (int rc = check_plan(plan)) return rc;
  if (int rc = check_peer_owners("bgk_matern_covariance_peer_band", N, G, macro_row_start, bases))
    return rc;
  if (rank < 0 || rank >= G) {
    bgk_set_error("bgk_matern_covariance_peer_band: rank %d outside [0, %d)", rank, G);
    return BGK_ERR_INVALID;
  }
  const int64_t T = (N + BGK_MACRO_TILE - 1) / BGK_MACRO_TILE;
  const int64_t p0 = macro_row_start[rank], p1 = macro_row_start[rank + 1];
  if (p1 == p0 || N == 0) return BGK_OK;
  if (!lx || !ly) {
    bgk_set_error("bgk_matern_covariance_peer_band: NULL locations");
    return BGK_ERR_INVALID;
  }
  BgkMaternArgs A = peer_args(lx, ly, N, G, macro_row_start, bases);
  A.band = 1;
  A.bT = T;
  A.bW = T / 2 + 1;  // d = 0 .. floor(T/2); for odd T that is (T - 1)/2 + 1
  A.brow0 = p0;
  A.tile0 = p0; A.tile1 = p1;
  return bgk_launch_matern(plan, A, BGK_MODE_PEER, (cudaStream_t)stream);
}

int bgk_ipc_export(const void *ptr, void *handle, uint64_t *offset) {
  if (!ptr || !handle || !offset) {
    bgk_set_error("bgk_ipc_export: NULL argument");
    return BGK_ERR_INVALID;
  }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(ptr));
  if (e != cudaSuccess) {
    bgk_set_error("cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    return BGK_ERR_CUDA;
  }
  // offset of ptr inside its allocation (cuMemGetAddressRange via the runtime's
  // driver entry point, so the library needs no -lcuda)
  typedef int (*GetRange)(unsigned long long *, size_t *, unsigned long long);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || !fn) {
      bgk_set_error("cuMemGetAddressRange unavailable");
      return BGK_ERR_CUDA;
    }
    get_range = (GetRange)fn;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0) {
    bgk_set_error("cuMemGetAddressRange failed");
    return BGK_ERR_CUDA;
  }
  static_assert(sizeof(h) == BGK_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  *offset = (uint64_t)((uintptr_t)ptr - base);
  return BGK_OK;
}

int bgk_ipc_open(const void *handle, uint64_t offset, void **ptr) {
  if (!handle || !ptr) {
    bgk_set_error("bgk_ipc_open: NULL argument");
    return BGK_ERR_INVALID;
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void *base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    bgk_set_error("cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    return BGK_ERR_CUDA;
  }
  *ptr = (char *)base + offset;
  return BGK_OK;
}

int bgk_ipc_close(void *ptr, uint64_t offset) {
  cudaError_t e = cudaIpcCloseMemHandle((char *)ptr - offset);
  if (e != cudaSuccess) {
    bgk_set_error("cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return BGK_ERR_CUDA;
  }
  return BGK_OK;
}

int bgk_can_access_peer(int peer_device, int *can_access) {
  int dev = 0;
  if (!can_access) {
    bgk_set_error("bgk_can_access_peer: NULL result pointer");
    return BGK_ERR_INVALID;
  }
  cudaGetDevice(&dev);
  if (peer_device == dev) {
    *can_access = 1;
    return BGK_OK;
  }
  const cudaError_t e = cudaDeviceCanAccessPeer(can_access, dev, peer_device);
  if (e != cudaSuccess) {
    cudaGetLastError();
    bgk_set_error("cudaDeviceCanAccessPeer(%d, %d): %s", dev, peer_device, cudaGetErrorString(e));
    return BGK_ERR_CUDA;
  }
  return BGK_OK;
}

int bgk_enable_peer_access(int peer_device) {
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return BGK_OK;
  }
  if (e != cudaSuccess) {
    bgk_set_error("cudaDeviceEnablePeerAccess(%d): %s", peer_device, cudaGetErrorString(e));
    return BGK_ERR_CUDA;
  }
  return BGK_OK;
}

}  // extern "C"

namespace {
// A persistent host thread pool for the host-side helpers (staging copies, matrix
// mirror): they run many times per call (per chunk / per row block), and spawning
// and joining threads each time costs tens of microseconds per thread.  One job
// at a time; the calling thread takes part.
class HostPool {
 public:
  template <class F>
  void run(int n, F &&f) {
    if (n <= 1) {
      if (n == 1) f(0);
      return;
    }
    std::lock_guard<std::mutex> one_job(job_mu_);
    grow(n - 1);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = [&f](int i) { f(i); };
      njobs_ = n;
      next_.store(0);
      remaining_ = n;
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return remaining_ == 0; });
    job_ = nullptr;
  }

 private:
  void grow(int want) {
    while ((int)workers_.size() < want) workers_.emplace_back([this] { loop(); });
  }
  void drain() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= njobs_) return;
      job_(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--remaining_ == 0) done_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
      }
      drain();
    }
  }
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> workers_;
  std::function<void(int)> job_;
  int njobs_ = 0, remaining_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
};

// never destroyed (workers outlive main's statics); a forked child starts with a
// fresh pool, since the parent's worker threads do not exist there
HostPool *g_host_pool = nullptr;
std::once_flag g_host_pool_once;

template <class F>
void host_parallel_for(int n, F &&f) {
  std::call_once(g_host_pool_once, [] {
    g_host_pool = new HostPool();
    pthread_atfork(nullptr, nullptr, [] { g_host_pool = new HostPool(); });
  });
  g_host_pool->run(n, std::forward<F>(f));
}
}  // namespace

int bgk_memcpy2d_d2h(void *dst, int64_t dpitch, const void *src, int64_t spitch,
                     int64_t width_bytes, int64_t rows, void *stream) {
  if (rows < 0 || width_bytes < 0 || width_bytes > dpitch || width_bytes > spitch ||
      (rows > 0 && width_bytes > 0 && (!dst || !src))) {
    bgk_set_error("bgk_memcpy2d_d2h: bad arguments");
    return BGK_ERR_INVALID;
  }
  if (rows == 0 || width_bytes == 0) return BGK_OK;
  const cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch,
                                          (size_t)width_bytes, (size_t)rows,
                                          cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    bgk_set_error("cudaMemcpy2DAsync: %s", cudaGetErrorString(e));
    return BGK_ERR_CUDA;
  }
  return BGK_OK;
}

int bgk_host_mirror_lower(double *out, int64_t ld, int64_t r0, int64_t r1, int nthreads) {
  return bgk_host_mirror_block(out, ld, r0, r1, 0, r0, nthreads);
}

int bgk_host_mirror_block(double *out, int64_t ld, int64_t r0, int64_t r1, int64_t c0,
                          int64_t c1, int nthreads) {
  if (r0 < 0 || r1 < r0 || c0 < 0 || c1 < c0 || ld < r1 || ld < c1 ||
      (r1 > r0 && c1 > c0 && !out) || (c0 < r1 && r0 < c1 && c1 > c0 && r1 > r0)) {
    bgk_set_error("bgk_host_mirror_block: bad arguments (ranges must not overlap)");
    return BGK_ERR_INVALID;
  }
  if (r1 == r0 || c1 == c0) return BGK_OK;
  constexpr int64_t B = 64;
  const int64_t nq = (c1 - c0 + B - 1) / B;  // destination row tiles (source column tiles)
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads < 1 ? 1 : nthreads, nq));
  auto work = [&](int t) {
    alignas(64) double tile[B][B];
    // static interleave over destination row tiles: disjoint writes per thread
    for (int64_t qt = t; qt < nq; qt += nt) {
      const int64_t j0 = c0 + qt * B, nj = std::min(B, c1 - j0);
      for (int64_t i0 = r0; i0 < r1; i0 += B) {
        const int64_t ni = std::min(B, r1 - i0);
        for (int64_t i = 0; i < ni; ++i)
          std::memcpy(tile[i], out + (i0 + i) * ld + j0, (size_t)nj * sizeof(double));
        for (int64_t j = 0; j < nj; ++j) {
          double *dst = out + (j0 + j) * ld + i0;
          if (ni == B && ((uintptr_t)dst & 15) == 0) {
            // non-temporal stores: the destination lines are written whole, so
            // skip the read-for-ownership (a third of the mirror's DRAM traffic)
            for (int64_t i = 0; i < B; i += 2)
              _mm_stream_pd(dst + i, _mm_set_pd(tile[i + 1][j], tile[i][j]));
          } else {
            for (int64_t i = 0; i < ni; ++i) dst[i] = tile[i][j];
          }
        }
      }
    }
    _mm_sfence();
  };
  if (nt == 1) {
    work(0);
    return BGK_OK;
  }
  host_parallel_for(nt, work);
  return BGK_OK;
}

int bgk_host_copy(void *dst, const void *src, int64_t bytes, int nthreads) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) {
    bgk_set_error("bgk_host_copy: bad arguments");
    return BGK_ERR_INVALID;
  }
  if (bytes == 0) return BGK_OK;
  char *d = static_cast<char *>(dst);
  const char *s = static_cast<const char *>(src);
  // per-thread ranges of whole 4 KB pages; each range streams 16-byte NT stores
  // once the destination is 16-byte aligned
  const int64_t page = 4096;
  const int64_t pages = (bytes + page - 1) / page;
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads < 1 ? 1 : nthreads,
                                                             pages / 16 + 1));
  auto work = [&](int t) {
    const int64_t a = std::min(bytes, (pages * t / nt) * page);
    const int64_t b = std::min(bytes, (pages * (t + 1) / nt) * page);
    int64_t i = a;
    while (i < b && ((uintptr_t)(d + i) & 15)) { d[i] = s[i]; ++i; }
    for (; i + 64 <= b; i += 64) {
      const __m128i v0 = _mm_loadu_si128((const __m128i *)(s + i));
      const __m128i v1 = _mm_loadu_si128((const __m128i *)(s + i + 16));
      const __m128i v2 = _mm_loadu_si128((const __m128i *)(s + i + 32));
      const __m128i v3 = _mm_loadu_si128((const __m128i *)(s + i + 48));
      _mm_stream_si128((__m128i *)(d + i), v0);
      _mm_stream_si128((__m128i *)(d + i + 16), v1);
      _mm_stream_si128((__m128i *)(d + i + 32), v2);
      _mm_stream_si128((__m128i *)(d + i + 48), v3);
    }
    for (; i < b; ++i) d[i] = s[i];
    _mm_sfence();
  };
  if (nt == 1) {
    work(0);
    return BGK_OK;
  }
  host_parallel_for(nt, work);
  return BGK_OK;
}
