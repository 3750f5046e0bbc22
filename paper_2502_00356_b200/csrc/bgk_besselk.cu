// bgk_besselk.cu -- batch K_nu(x) for sm_100a (the "K1" kernel of SURVEY.md 2.2).
//
// Replaces kernels.refined_log_bessel / fixed_window_log_pair / temme_series_log
// (kernels.py:212-302) over device arrays.  Same discretisation as the
// reference -- nodes t_m = t0 + m h, trapezoid weights 1/2 at both ends, strict
// x < threshold routing, Temme + log-space recurrence below it -- so results
// agree with the reference to ~1e-13 (tests/test_parity_besselk.py).
//
// Integral path, per element (x, nu), a = |nu|:
//   anchor node m_a near the log-integrand peak: 0 if a^2 <= x (g decreasing,
//   kernels.py:148-151), else round(asinh(a/x)/h) (fp32 is plenty -- the anchor
//   only sets the scale of the sum; any node near the peak gives the same value
//   to rounding).
//   With E = e^{a h} and q = e^{-2 a t_a}, node m_a +- j contributes
//       2 cosh(a t_k) e^{-x c_k} / (e^{a t_a} e^{-x c_a}) = (E^{+-j} + q E^{-+j}) e^{-x (c_k - c_a)}
//   so every node costs one table exp (7 FP64 ops) plus a handful of FP64 ops --
//   no per-node log_cosh (the reference's 73% hot spot).
//   c_k = cosh(t_k) is a per-CTA shared-memory table.  Both directions are
//   walked in one loop (two independent exp chains) until the term falls below
//   e^-50 of the anchor, which includes every node the reference's e^-46
//   break keeps.       ln K = a t_a - ln2 - x c_a + ln(h acc)
//
// Divergence: walk lengths vary 1..40 over random (x, nu).  Each CTA stages its
// 1024 elements in shared memory and counting-sorts them by a predicted walk
// length (a host-built table over (log x, nu) cells), so a warp's 32 lanes walk
// about the same number of nodes; Temme elements (x < thr) form their own
// bucket.  Results go back through shared memory for coalesced stores.
// Every value is a pure function of (x, nu, cfg): bitwise independent of batch
// composition.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "bgk_device.cuh"
#include "bgk_internal.h"

namespace bgk {

constexpr int kBkThreads = 256;
constexpr int kBkPerThread = 4;
constexpr int kBkChunk = kBkThreads * kBkPerThread;
constexpr int kXCells = 64;   // x cells: 4 per octave from 2^-6
constexpr int kNuCells = 48;  // nu cells: width 1/2, last one open-ended
constexpr int kXKeyBase = (1023 - 6) << 2;
constexpr int kMaxPred = 63;  // predicted walk steps, clamped
constexpr int kBuckets = kMaxPred + 2;  // + series bucket

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
  const uint8_t *pred;  // device: predicted max(up, down) walk steps per (x, nu) cell
};

__host__ __device__ inline int x_cell(double x) {
  uint64_t b;
#ifdef __CUDA_ARCH__
  b = (uint64_t)__double_as_longlong(x);
#else
  std::memcpy(&b, &x, 8);
#endif
  const int key = (int)(b >> 50) - kXKeyBase;  // exponent + top 2 mantissa bits
  return key < 0 ? 0 : (key >= kXCells ? kXCells - 1 : key);
}
__host__ __device__ inline int nu_cell(double a) {
  const double c = a * 2.0;
  return c >= (double)(kNuCells - 1) ? kNuCells - 1 : (int)c;
}

// Anchor node for the fast path (host and device agree; fp32 asinh).
__host__ __device__ inline int anchor_node(double x, double a, double t0, double h, int bins) {
  if (a * a <= x) return 0;
  const float ts = asinhf((float)a / (float)x);
  float fm = rintf((ts - (float)t0) * (float)(1.0 / h));
  fm = fminf(fmaxf(fm, 0.0f), (float)bins);
  return (int)fm;
}

// Fast fixed-window quadrature (see file header).  Requires t0 >= 0 and
// a * max(|t0|, |t1|) <= 600 so that E^j never overflows.
__device__ __forceinline__ double fixed_window_fast(double x, double a, const BkArgs &A,
                                                    const double *__restrict__ ctab,
                                                    const double *__restrict__ t128,
                                                    const double *__restrict__ invc,
                                                    const double *__restrict__ logc) {
  const int bins = A.bins;
  const int m = anchor_node(x, a, A.t0, A.h, bins);
  const double ta = A.t0 + (double)m * A.h;
  const double ca = ctab[m];
  const double E = exp_acc(a * A.h, t128);
  const double Ei = exp_acc(-a * A.h, t128);
  const double two_at = 2.0 * a * ta;
  const double q = (two_at < 700.0) ? exp_acc(-two_at, t128) : 0.0;
  const double anchor = 1.0 + q;
  const double tiny = 1.9287498479639178e-22 * anchor;  // e^-50 of the anchor term
  const double mx = -x, xca = x * ca;
  double acc = ((m == 0 || m == bins) ? 0.5 : 1.0) * anchor;

  double pu = 1.0, qu = 1.0, pd = 1.0, qd = 1.0;
  bool up = m < bins, dn = m > 0;
  int j = 1;
  while (up || dn) {
    if (up) {
      pu *= E;
      qu *= Ei;
      const int k = m + j;
      const double s = fma(q, qu, pu);
      const double y = fmax(fma(mx, ctab[k], xca), -700.0);
      const double term = s * exp_node(y, t128);
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
      const double s = fma(q, qd, pd);
      const double y = fmax(fma(mx, ctab[k], xca), -700.0);
      const double term = s * exp_node(y, t128);
      if (term < tiny) {
        dn = false;
      } else {
        acc = fma((k == 0) ? 0.5 : 1.0, term, acc);
        dn = k > 0;
      }
    }
    ++j;
  }
  return (a * ta - kLn2) - xca + log_fast(A.h * acc, invc, logc);
}

__global__ void __launch_bounds__(kBkThreads, 4) besselk_kernel(const __grid_constant__ BkArgs A) {
  extern __shared__ double smem[];
  __shared__ double s_exp[128], s_invc[128], s_logc[128];
  __shared__ double sx[kBkChunk], snu[kBkChunk];
  __shared__ uint16_t perm[kBkChunk];
  __shared__ uint8_t spath[kBkChunk];
  __shared__ int hist[kBuckets + 1];
  __shared__ uint8_t spred[kXCells * kNuCells];
  __shared__ int s_next;
  double *ctab = smem;  // bins + 1 (only when table_ok)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  load_tables128(s_exp, s_invc, s_logc);
  if (A.table_ok)
    for (int k = tid; k <= A.bins; k += kBkThreads) ctab[k] = cosh(A.t0 + (double)k * A.h);
  for (int b = tid; b <= kBuckets; b += kBkThreads) hist[b] = 0;
  if (A.table_ok) {
    const uint32_t *src = reinterpret_cast<const uint32_t *>(A.pred);
    uint32_t *dst = reinterpret_cast<uint32_t *>(spred);
    for (int c = tid; c < kXCells * kNuCells / 4; c += kBkThreads) dst[c] = __ldg(src + c);
  }
  if (tid == 0) s_next = 0;

  const long long base = (long long)blockIdx.x * kBkChunk;
  const int cnt = (int)min((long long)kBkChunk, A.n - base);
  // coalesced staging of this CTA's elements
  for (int e = tid; e < cnt; e += kBkThreads) {
    sx[e] = A.x[base + e];
    snu[e] = A.nu[base + e];
  }
  __syncthreads();

  const double tmax = fmax(fabs(A.t0), fabs(A.t1));
  auto bucket_of = [&](double x, double nu) -> int {
    const bool series = (A.route == 1) || (A.route == 0 && x < A.thr);
    if (series) return 0;
    const double a = fabs(nu);
    if (!(A.table_ok && a * tmax <= 600.0)) return kBuckets - 1;  // general path: last
    // longest predicted walks first (they are pulled first in the compute phase)
    return kMaxPred - min((int)spred[x_cell(x) * kNuCells + nu_cell(a)], kMaxPred - 1);
  };
  for (int e = tid; e < cnt; e += kBkThreads) atomicAdd(&hist[bucket_of(sx[e], snu[e])], 1);
  __syncthreads();
  if (warp == 0) {  // exclusive scan over kBuckets (<= 65) bins, 3 per lane
    int v[3], local = 0;
    for (int t = 0; t < 3; ++t) {
      const int b = lane * 3 + t;
      v[t] = b < kBuckets ? hist[b] : 0;
      local += v[t];
    }
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
      const int w = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += w;
    }
    int run = incl - local;
    for (int t = 0; t < 3; ++t) {
      const int b = lane * 3 + t;
      if (b < kBuckets) hist[b] = run;
      run += v[t];
    }
  }
  __syncthreads();
  for (int e = tid; e < cnt; e += kBkThreads)
    perm[atomicAdd(&hist[bucket_of(sx[e], snu[e])], 1)] = (uint16_t)e;
  __syncthreads();

  // compute in sorted order: warps pull 32-element groups from a shared counter,
  // longest predicted walks first
  const int ngroups = (cnt + 31) >> 5;
  for (;;) {
    int g = lane == 0 ? atomicAdd(&s_next, 1) : 0;
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g >= ngroups) break;
    const int p = g * 32 + lane;
    if (p >= cnt) continue;
    const int e = perm[p];
    const double x = sx[e], nu = snu[e];
    const bool series = (A.route == 1) || (A.route == 0 && x < A.thr);
    double lk;
    if (series) {
      const TemmeConst T = temme_const(nu);
      lk = temme_series_log_c(x, T, A.eps, A.cap);
    } else {
      const double a = fabs(nu);
      if (A.table_ok && a * tmax <= 600.0)
        lk = fixed_window_fast(x, a, A, ctab, s_exp, s_invc, s_logc);
      else
        lk = fixed_window_log_ref(x, nu, A.t0, A.t1, A.bins);
    }
    sx[e] = lk;
    if (A.k) snu[e] = (fabs(lk) < 700.0) ? exp_acc(lk, s_exp) : exp(lk);
    spath[e] = series ? 0 : 1;
  }
  __syncthreads();
  for (int e = tid; e < cnt; e += kBkThreads) {
    A.log_k[base + e] = sx[e];
    if (A.k) A.k[base + e] = snu[e];
    if (A.path) A.path[base + e] = spath[e];
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

// ---------------------------------------------------------------------------------
// host: the walk-length prediction table, cached per (t0, t1, bins)
// ---------------------------------------------------------------------------------

// Host emulation of fixed_window_fast's walk length max(up, down) (libm exp).
static int walk_steps_host(double x, double a, double t0, double h, int bins, const double *c) {
  const int m = anchor_node(x, a, t0, h, bins);
  const double ta = t0 + m * h, ca = c[m];
  const double E = std::exp(a * h), Ei = std::exp(-a * h);
  const double q = (2 * a * ta < 700) ? std::exp(-2 * a * ta) : 0.0;
  const double tiny = 1.9287498479639178e-22 * (1 + q);
  int up = 0, dn = 0;
  double p = 1, qq = 1;
  for (int j = 1; m + j <= bins; ++j) {
    p *= E;
    qq *= Ei;
    ++up;
    if ((q * qq + p) * std::exp(std::fmax(-x * (c[m + j] - ca), -700.0)) < tiny) break;
  }
  p = 1;
  qq = 1;
  for (int j = 1; m - j >= 0; ++j) {
    p *= Ei;
    qq *= E;
    ++dn;
    if ((q * qq + p) * std::exp(std::fmax(-x * (c[m - j] - ca), -700.0)) < tiny) break;
  }
  return up > dn ? up : dn;
}

static void build_pred_table(double t0, double t1, int bins, uint8_t *pred) {
  std::vector<double> c(bins + 1);
  const double h = (t1 - t0) / bins;
  for (int k = 0; k <= bins; ++k) c[k] = std::cosh(t0 + k * h);
  for (int xi = 0; xi < kXCells; ++xi) {
    // cell xi covers [2^(e) * (1 + f/4), 2^e * (1 + (f+1)/4)) with e, f from the key
    const int key = xi + kXKeyBase;
    const double lo = std::ldexp(1.0 + (key & 3) / 4.0, (key >> 2) - 1023);
    const double hi = std::ldexp(1.0 + ((key & 3) + 1) / 4.0, (key >> 2) - 1023);
    for (int ni = 0; ni < kNuCells; ++ni) {
      const double nlo = ni * 0.5;
      const double nhi = (ni == kNuCells - 1) ? nlo + 8.0 : nlo + 0.5;
      int best = 0;
      for (int sx = 0; sx <= 2; ++sx)
        for (int sn = 0; sn <= 2; ++sn) {
          const double xv = lo + (hi - lo) * sx / 2.0 * 0.999;
          const double nv = nlo + (nhi - nlo) * sn / 2.0 * 0.999;
          const int w = walk_steps_host(xv, nv, t0, h, bins, c.data());
          best = w > best ? w : best;
        }
      pred[xi * kNuCells + ni] = (uint8_t)(best > kMaxPred ? kMaxPred : best);
    }
  }
}

}  // namespace bgk

// ---------------------------------------------------------------------------------
// launchers (called from bgk_capi.cpp)
// ---------------------------------------------------------------------------------
// Device copies of the walk-length prediction table, one per (t0, t1, bins), built
// on the host and uploaded once (3 KB each); kept for the life of the process.
struct PredEntry {
  double t0, t1;
  long long bins;
  uint8_t *dev;
};

int bgk_launch_besselk(const double *x, const double *nu, int64_t n, const bgk_config *cfg,
                       int route, double *log_k, double *k, uint8_t *path, cudaStream_t stream) {
  if (n == 0) return 0;
  static std::mutex mu;
  static std::vector<PredEntry> cache;
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
  A.pred = nullptr;
  if (A.table_ok) {
    std::lock_guard<std::mutex> lock(mu);
    for (const PredEntry &e : cache)
      if (e.t0 == cfg->t_lower && e.t1 == cfg->t_upper && e.bins == cfg->bins) A.pred = e.dev;
    if (!A.pred) {
      std::vector<uint8_t> host(bgk::kXCells * bgk::kNuCells);
      bgk::build_pred_table(cfg->t_lower, cfg->t_upper, (int)cfg->bins, host.data());
      uint8_t *dev = nullptr;
      cudaError_t err = cudaMalloc(&dev, host.size());
      if (err == cudaSuccess) err = cudaMemcpy(dev, host.data(), host.size(), cudaMemcpyHostToDevice);
      if (err != cudaSuccess) {
        bgk_set_error("besselk prediction table upload: %s", cudaGetErrorString(err));
        return BGK_ERR_CUDA;
      }
      cache.push_back({cfg->t_lower, cfg->t_upper, cfg->bins, dev});
      A.pred = dev;
    }
  }
  size_t smem = sizeof(double) * (A.table_ok ? (size_t)cfg->bins + 1 : 0);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(bgk::besselk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * (kMaxTable + 1)));
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
