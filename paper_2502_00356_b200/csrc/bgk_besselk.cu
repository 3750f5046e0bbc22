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
//   c_k = cosh(t_k) is a per-CTA shared-memory table.
//       ln K = a t_a - ln2 - x c_a + ln(h acc)
//
// Node window: a host-built table over (log x, nu) cells gives, relative to the
// anchor, how far up and down the terms stay above e^-34 of the anchor term
// (maximised over a 17 x 17 sample of the cell, edges included; the extra e^-1
// below the e^-33 cut covers the variation between samples: every node with a
// term above e^-33 of the grid max lies inside, checked on a denser
// sample by tests/test_bk_window_table.py); each lane sums its window
// [m - D, m + U] as one ascending sequence.  The reference's
// walk also keeps terms in (e^-46, e^-33]: together < 41 e^-33 = 1.9e-13 of the
// sum as a bound (max |d ln K| vs the oracle is 5.7e-14 with the cut at 40 or 33).  Elements outside the table's range use the
// full grid [0, bins].
//
// Divergence: window sizes vary 1..40 over random (x, nu).  Each CTA stages its
// 1024 elements in shared memory and counting-sorts them by predicted window
// size, so a warp's 32 lanes sum about the same number of nodes; Temme elements
// (x < thr) form their own bucket.  Results go back through shared memory for
// coalesced stores.
// Every value is a pure function of (x, nu, cfg): bitwise independent of batch
// composition.
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "bgk_device.cuh"
#include "bgk_internal.h"

namespace bgk {

#ifndef BGK_BK_THREADS
#define BGK_BK_THREADS 256  // A/B on B200: 128 threads x 8 (7 CTAs/SM) 1.68 ms, 128 x 16 2.00 ms, 256 x 8 1.54 ms
#endif
#ifndef BGK_BK_PER_THREAD
#define BGK_BK_PER_THREAD 8
#endif
#ifndef BGK_BK_MINBLOCKS
#define BGK_BK_MINBLOCKS 4
#endif
constexpr int kBkThreads = BGK_BK_THREADS;
constexpr int kBkPerThread = BGK_BK_PER_THREAD;
constexpr int kBkChunk = kBkThreads * kBkPerThread;
constexpr int kBkChunkBytes = kBkChunk * (8 + 8 + 4 + 2 + 1 + 1);  // + 1: keeps cw 16-B aligned
constexpr int bk_chunk_bytes(int per) { return kBkThreads * per * (8 + 8 + 4 + 2 + 1 + 1); }
#ifndef BGK_BK_XBITS
#define BGK_BK_XBITS 2  // window table: 2^XBITS x cells per octave
#endif
#ifndef BGK_BK_NODE_I2F
#define BGK_BK_NODE_I2F 0  // A/B on B200: 1 -> 1.521 vs 0 -> 1.511 ms (the Matern loop gains, this one not)
#endif
#ifndef BGK_BK_NODE_IMM
#define BGK_BK_NODE_IMM 1  // 1/24 (20-bit mantissa) and the magic as immediates: 1.503 -> 1.499 ms (BK 64 Mi)
#endif
#ifndef BGK_BK_FOLD
#define BGK_BK_FOLD 1  // cosh(a t) running products folded into the node exponent (12 FP64 ops per node)
#endif
#ifndef BGK_BK_NODE_UNROLL
#define BGK_BK_NODE_UNROLL 2
#endif
constexpr int kBkNodeUnroll = BGK_BK_NODE_UNROLL;
#ifndef BGK_BK_DYN_TAIL
#define BGK_BK_DYN_TAIL 4  // groups per warp pulled dynamically at the end of the compute phase
                          // (A/B on B200: 1 -> 1.556, 2 -> 1.534, 4 -> 1.512, 8 -> 1.542 ms)
#endif
#ifndef BGK_BK_MARGIN
#define BGK_BK_MARGIN 0  // nodes added to each side of the sampled window extents (A/B on
                         // B200: 0 -> 1.606 ms, 1 -> 1.661 ms; max|d ln K| unchanged, 5.7e-14)
#endif
#ifndef BGK_BK_WSAMP
#define BGK_BK_WSAMP 16  // window table: (WSAMP+1)^2 samples per cell, edges included
#endif
#ifndef BGK_BK_WCUT
#define BGK_BK_WCUT 34.0  // window table: keep nodes within e^-WCUT of the anchor term (the
                          // cut is e^-33 of the max; the extra 1 covers the variation between
                          // samples: tests/test_bk_window_table.py).  A/B on B200 (BK 64 Mi):
                          // 41 -> 1.499, 34 -> 1.483 ms, max |d ln K| 5.7e-14 both
#endif
#ifndef BGK_BK_NUSTEP
#define BGK_BK_NUSTEP 2  // window table: nu cells per unit of nu
#endif
constexpr int kXBits = BGK_BK_XBITS;
constexpr int kXCells = 16 << kXBits;             // x cells: 16 octaves from 2^-6
constexpr int kNuStep = BGK_BK_NUSTEP;
constexpr int kNuCells = 24 * kNuStep;            // nu cells of width 1/kNuStep, last open-ended
constexpr int kXKeyBase = (1023 - 6) << kXBits;
constexpr int kMaxPred = 63;  // predicted window size (sort key), clamped
// buckets: 0 series | 2 pb - 1 + (anchor not 0), pb = 1 (widest) .. kMaxPred - 1 |
// kBuckets - 1 reference path.  Elements whose anchor is node 0 (a^2 <= x) sort
// next to each other so whole warps skip the two anchor-shift exps.
constexpr int kBuckets = 2 * kMaxPred + 2;

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
  const uint32_t *win;  // device: per (x, nu) cell, U | D << 16 (window above / below anchor)
  const double2 *cwg;   // device: {cosh t_k, weight exponent adjust}, k = 0..bins (host libm cosh)
  float t0f, hinvf, binsf;  // anchor_node_fast's fp32 constants
};

// Unclamped x-cell key: exponent + top kXBits mantissa bits, relative to 2^-6.
__host__ __device__ inline int x_cell_key(double x) {
  uint64_t b;
#ifdef __CUDA_ARCH__
  b = (uint64_t)__double_as_longlong(x);
#else
  std::memcpy(&b, &x, 8);
#endif
  return (int)(b >> (52 - kXBits)) - kXKeyBase;
}
__host__ __device__ inline int x_cell(double x) {
  uint64_t b;
#ifdef __CUDA_ARCH__
  b = (uint64_t)__double_as_longlong(x);
#else
  std::memcpy(&b, &x, 8);
#endif
  const int key = (int)(b >> (52 - kXBits)) - kXKeyBase;  // exponent + top mantissa bits
  return key < 0 ? 0 : (key >= kXCells ? kXCells - 1 : key);
}
__host__ __device__ inline int nu_cell(double a) {
  const double c = a * (double)kNuStep;
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

// Device anchor: asinh(a/x) = ln(z + sqrt(z^2 + 1)) with fast fp32 intrinsics
// (~10 instructions instead of libdevice asinhf's ~80).  It can differ from the
// host's anchor_node only where t*/h sits within ~1e-5 of a half-integer; the
// window then shifts by one node (dropping an edge term of relative size
// <~ e^-30 on 1e-5 of elements at worst), and the anchor itself only
// sets the scale of the sum (rounding-level effect).
// (t0f = (float)t0, hinvf = (float)(1.0 / h), binsf = (float)bins: precomputed on
// the host, read from the parameter bank -- no live registers / spills)
__device__ __forceinline__ int anchor_node_fast(double x, double a, float t0f, float hinvf,
                                                float binsf) {
  if (a * a <= x) return 0;
  const float z = __fdividef((float)a, (float)x);
  const float ts = __logf(z + sqrtf(fmaf(z, z, 1.0f)));
  float fm = rintf((ts - t0f) * hinvf);
  fm = fminf(fmaxf(fm, 0.0f), binsf);
  return (int)fm;
}

// The fast path's window word for an integral-route element (0: not on the fast
// path -> reference port): the host-built table's U | D << 16 for cells proven
// underflow-free, the full grid for x outside the table when every exponent stays
// >= -600, else 0.  Shared by the kernel's classify pass and the window
// introspection exports (bgk_besselk_windows{,_host}).
__host__ __device__ inline uint32_t bk_window_word(double x, double a, int table_ok,
                                                   double tmax, double cmax, int bins,
                                                   const uint32_t *win) {
  uint32_t w = 0;
  if (table_ok && a * tmax <= 600.0) {  // E^{+-j} cannot overflow
    const int key = x_cell_key(x);
    if (key >= 0 && key < kXCells && a * (double)kNuStep < (double)(kNuCells - 1)) {
#ifdef __CUDA_ARCH__
      w = __ldg(win + key * kNuCells + nu_cell(a));
#else
      w = win[key * kNuCells + nu_cell(a)];
#endif
      if (w == 0xffffffffu) w = 0;  // cell not proven underflow-free: reference path
    } else if (x * cmax <= 600.0) {
      w = (uint32_t)bins | ((uint32_t)bins << 16);  // full grid, exponents >= -600
    }
  }
  return w;
}

__device__ __forceinline__ int ld_u16_volatile(const uint16_t *p) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}


// Fast fixed-window quadrature (see file header).  Requires t0 >= 0 and an
// element inside the window table (its window keeps every exponent above
// -600, checked when the table is built).  Called by ALL 32 lanes of a warp:
// lane i sums nodes lo_i .. lo_i + n_i - 1 in ascending order.  The warp runs
// min_i n_i nodes unmasked, then masks the ragged tail; inactive lanes
// (n = 0) compute throw-away values.  Per node: s_k = E^{k-m} + q E^{m-k} from
// two running products, e^{y_k} = T p (table exp), acc += (s_k T) p -- 14 FP64
// ops.  The value depends only on the lane's own (x, nu).
__device__ __forceinline__ double fixed_window_fast(bool active, double x, double a, uint32_t w,
                                                    const BkArgs &A,
                                                    const double2 *__restrict__ cw,
                                                    const double *__restrict__ t128,
                                                    const double *__restrict__ invc,
                                                    const double *__restrict__ logc) {
  const int bins = A.bins;
  const int m = active ? anchor_node_fast(x, a, A.t0f, A.hinvf, A.binsf) : 0;
  const int U = min((int)(w & 0xffff), bins - m), D = min((int)(w >> 16), m);
  const int lo = m - D, n = active ? U + D + 1 : 0;
  const int nmax = __reduce_max_sync(0xffffffffu, n);
  const int nmin = min(__reduce_min_sync(0xffffffffu, active ? n : 0x7fffffff), nmax);
  const double ta = A.t0 + (double)m * A.h;
  const double ca = cw[m].x;
  const double tlo = A.t0 + (double)lo * A.h;
#if BGK_BK_FOLD
  // 2 cosh(a t_k) e^{-x c_k} / (e^{a t_a} e^{-x c_a}) = e^{y'_k} (1 + R_k) with
  //   y'_k = -x c_k + [x c_a + a (t_k - t_a)]   (the bracket z_k: z += a h per node)
  //   R_k  = e^{-2 a t_k}                       (R *= e^{-2 a h} per node)
  // so the E^{+-j} running products fold into the exponent: 12 FP64 ops per node
  // (13 with two products and their sum) and one exp per element fewer.
  const double mx = -x, xca = x * ca, ah = a * A.h;
  double z = fma(a, tlo - ta, xca);
  double R = 1.0, Ei2 = 1.0;
  if (!(A.t0 == 0.0 && __all_sync(0xffffffffu, m == 0))) {  // (else t_lo = t_a = 0, R = 1)
    const double qa = 2.0 * a * tlo;
    R = (qa < 700.0) ? exp_acc(-qa, t128) : 0.0;
  }
  Ei2 = exp_acc(-2.0 * ah, t128);
  const double2 *row = cw + lo;
  double acc = 0.0;
  // one node: T u = e^{y'} (1 + R); the caller accumulates acc = fma(T, u, acc)
  auto node = [&](double2 c, double &T, double &u) {
    const double y = fma(mx, c.x, z);
    z += ah;
    const double tt = fma(y, kExpK[0], kExpK[6]);
    const int nn = __double2loint(tt);
#if BGK_BK_NODE_I2F
    const double nd = __int2double_rn(nn);
#elif BGK_BK_NODE_IMM
    const double nd = tt - 0x1.8p52;
#else
    const double nd = tt - kExpK[6];
#endif
    const double r = fma(nd, -kExpK[1], y);
#if BGK_BK_NODE_IMM
    double q = fma(r, 0x1.55555p-5, kExpK[4]);
#else
    double q = fma(r, kExpK[3], kExpK[4]);
#endif
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    const double p = fma(q, r, 1.0);
    u = fma(p, R, p);
    R *= Ei2;
    const double tv = t128[nn & 127];
    T = __hiloint2double(__double2hiint(tv) + (nn << 13) + __double2loint(c.y), __double2loint(tv));
  };
  int j = 0;
#pragma unroll(kBkNodeUnroll)
  for (; j < nmin; ++j) {
    double T, u;
    node(row[j], T, u);
    acc = fma(T, u, acc);
  }
  for (; j < nmax; ++j) {
    double T, u;
    node(row[min(j, bins - lo)], T, u);
    const double t = fma(T, u, acc);  // the same arithmetic as the unmasked loop
    acc = (j < n) ? t : acc;
  }
#else
  double E, Ei;
  exp_pair(a * A.h, t128, E, Ei);
  // E^{lo - m} and q E^{m - lo}.  With the anchor at node 0 of a grid starting at
  // t0 = 0 both are exactly 1 (lo = m = 0: exp of +-0); warps whose lanes all have
  // m = 0 (sorted together by the classify pass) skip the two exps.
  double P = 1.0, Qs = 1.0;
  if (!(A.t0 == 0.0 && __all_sync(0xffffffffu, m == 0))) {
    P = exp_acc(-a * (ta - tlo), t128);
    const double qa = a * (ta + tlo);
    Qs = (qa < 700.0) ? exp_acc(-qa, t128) : 0.0;
  }
  const double mx = -x, xca = x * ca;
  const double2 *row = cw + lo;
  double acc = 0.0;
  // cw[k] = {c_k, weight}: the trapezoid weight 1/2 at k = 0 and k = bins is an
  // exponent-field adjustment (-1 << 20, in the low word of .y) added to the
  // table value's high word -- an exact halving, no FP64 op per node.
  auto node = [&](double2 c) {
    const double y = fma(mx, c.x, xca);
    const double s = P + Qs;
    P *= E;
    Qs *= Ei;
    const double tt = fma(y, kExpK[0], kExpK[6]);
    const int nn = __double2loint(tt);
#if BGK_BK_NODE_I2F
    const double nd = __int2double_rn(nn);  // conversion pipe, exact (= tt - magic)
#else
#if BGK_BK_NODE_IMM
    const double nd = tt - 0x1.8p52;  // (the magic as a DADD immediate)
#else
    const double nd = tt - kExpK[6];
#endif
#endif
    const double r = fma(nd, -kExpK[1], y);
#if BGK_BK_NODE_IMM
    // 1/24 rounded to a 20-bit mantissa (a DFMA immediate; |r| <= ln2/256: the change
    // is < 1e-18 of the term), so this step reads one vector register, not two
    double q = fma(r, 0x1.55555p-5, kExpK[4]);
#else
    double q = fma(r, kExpK[3], kExpK[4]);
#endif
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    const double p = fma(q, r, 1.0);
    const double tv = t128[nn & 127];
    const double T = __hiloint2double(__double2hiint(tv) + (nn << 13) + __double2loint(c.y),
                                      __double2loint(tv));
    return s * T * p;  // (s T) p: T scaling is exact
  };
  int j = 0;
#pragma unroll(kBkNodeUnroll)
  for (; j < nmin; ++j) acc += node(row[j]);
  for (; j < nmax; ++j) {
    const double t = node(row[min(j, bins - lo)]);
    if (j < n) acc += t;
  }
#endif
  return (a * ta - kLn2) - xca + log_fast(A.h * acc, invc, logc);
}

// The Temme path (x < threshold: 0.08% of the BK elements) out of line, so its
// long chain does not take registers from the fast path's loop.
__device__ __noinline__ double bk_series_log(double x, double nu, double eps, long long cap) {
  // a non-finite order would saturate the recurrence's step count (floor(inf + 0.5)
  // -> INT_MAX steps): NaN at once instead (the validated API rejects it anyway)
  if (!(fabs(nu) <= 1.7976931348623157e308)) return __longlong_as_double(0x7ff8000000000000LL);
  const TemmeConst T = temme_const(nu);
  return temme_series_log_c(x, T, eps, cap);
}

// PER elements per thread (chunk = 256 PER): kBkPerThread, or fewer when that fills the
// last wave of CTAs better (bgk_launch_besselk).
template <int PER>
__global__ void __launch_bounds__(kBkThreads, BGK_BK_MINBLOCKS) besselk_kernel(const __grid_constant__ BkArgs A) {
  constexpr int kBkPerThread = PER, kBkChunk = kBkThreads * PER, kBkChunkBytes = bk_chunk_bytes(PER);
  extern __shared__ __align__(16) unsigned char bk_smem[];
  __shared__ double s_exp[128], s_invc[128], s_logc[128];
  __shared__ int hist[kBuckets + 1];
  __shared__ int s_next;
  __shared__ uint16_t s_eidx[kBkThreads];
  // dynamic: the chunk at fixed offsets (no pointer registers), then
  // {cosh t_k, ln w_k} (bins + 1, only when table_ok)
  const int ncw = A.table_ok ? A.bins + 1 : 0;
  double *sx = reinterpret_cast<double *>(bk_smem);
  double *snu = sx + kBkChunk;
  uint32_t *sw = reinterpret_cast<uint32_t *>(snu + kBkChunk);  // window word per element
  uint16_t *perm = reinterpret_cast<uint16_t *>(sw + kBkChunk);
  uint8_t *spath = reinterpret_cast<uint8_t *>(perm + kBkChunk);  // bucket, then path
  double2 *cw = reinterpret_cast<double2 *>(bk_smem + kBkChunkBytes);

  const int tid = threadIdx.x, lane = tid & 31;
  load_tables128(s_exp, s_invc, s_logc);
  for (int k = tid; k < ncw; k += kBkThreads) cw[k] = __ldg(A.cwg + k);
  for (int b = tid; b <= kBuckets; b += kBkThreads) hist[b] = 0;
  if (tid == 0) s_next = 0;

  const long long base = (long long)blockIdx.x * kBkChunk;
  const int cnt = (int)min((long long)kBkChunk, A.n - base);
  // coalesced staging of this CTA's elements (all loads in flight at once)
#pragma unroll
  for (int i = 0; i < kBkPerThread; ++i) {
    const int e = i * kBkThreads + tid;
    if (e < cnt) {
      sx[e] = __ldcs(A.x + base + e);
      snu[e] = __ldcs(A.nu + base + e);
    }
  }
  __syncthreads();

  const double tmax = fmax(fabs(A.t0), fabs(A.t1));
  const double cmax = ncw ? cw[A.bins].x : 0.0;  // cosh(t1): t0 >= 0 on the table path
  // classify once: bucket (widest predicted windows first; series 0, general
  // path last) and the element's window word (0: not on the fast path).
  // Fixed trip count so the window-table loads of all 8 elements overlap.
#pragma unroll
  for (int i = 0; i < kBkPerThread; ++i) {
    const int e = i * kBkThreads + tid;
    if (e >= cnt) break;
    const double x = sx[e], a = fabs(snu[e]);
    const bool series = (A.route == 1) || (A.route == 0 && x < A.thr);
    int b = kBuckets - 1;
    uint32_t w = 0;
    if (series) {
      b = 0;
    } else {
      w = bk_window_word(x, a, A.table_ok, tmax, cmax, A.bins, A.win);
      if (w) {
        const int nw = (int)(w & 0xffff) + (int)(w >> 16) + 1;
        b = 2 * (kMaxPred - min(nw, kMaxPred - 1)) - (a * a <= x ? 1 : 0);
      }
    }
    sw[e] = w;
    spath[e] = (uint8_t)b;
    atomicAdd(&hist[b], 1);
  }
  __syncthreads();
  static_assert(kBuckets <= 128, "scan: 4 buckets per lane");
  if (tid < 32) {  // exclusive scan over kBuckets (<= 128) bins, 4 per lane
    int v[4], local = 0;
    for (int t = 0; t < 4; ++t) {
      const int b = lane * 4 + t;
      v[t] = b < kBuckets ? hist[b] : 0;
      local += v[t];
    }
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
      const int w = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += w;
    }
    int run = incl - local;
    for (int t = 0; t < 4; ++t) {
      const int b = lane * 4 + t;
      if (b < kBuckets) hist[b] = run;
      run += v[t];
    }
  }
  __syncthreads();
  for (int e = tid; e < cnt; e += kBkThreads) perm[atomicAdd(&hist[spath[e]], 1)] = (uint16_t)e;
  __syncthreads();

  // compute in sorted order (widest predicted windows first): warp w takes
  // groups w, w + 8, ... statically, and the last ~2 groups per warp are pulled
  // from a shared counter so warps that met the slow Temme / reference-path
  // elements (first and last groups) do not hold the CTA back.  Every lane of
  // the warp enters the fast sum (lanes without a fast-path element sum
  // nothing) so it runs branch-free.
  const int ngroups = (cnt + 31) >> 5;
  constexpr int kWarps = kBkThreads / 32;
  const int nstatic = max(0, (ngroups - BGK_BK_DYN_TAIL * kWarps) / kWarps);
  const int warp = tid >> 5;
  for (int round = 0;; ++round) {
    int g;
    if (round < nstatic) {
      g = round * kWarps + warp;
    } else {
      g = lane == 0 ? nstatic * kWarps + atomicAdd(&s_next, 1) : 0;
      g = __shfl_sync(0xffffffffu, g, 0);
    }
    if (g >= ngroups) break;
    const int p = g * 32 + lane;
    const bool valid = p < cnt;
    const int e0 = valid ? perm[p] : 0;
    s_eidx[tid] = (uint16_t)e0;  // re-read for the result stores (not spilled)
    const int e = e0;
    const double x = valid ? sx[e] : 1.0, nu = valid ? snu[e] : 0.0;
    const uint32_t w = valid ? sw[e] : 0u;
    const bool series = (A.route == 1) || (A.route == 0 && x < A.thr);
    const double a = fabs(nu);
    const bool fast = valid && w != 0u;
    double lk = fixed_window_fast(fast, x, a, w, A, cw, s_exp, s_invc, s_logc);
    if (!valid) continue;
    if (series) {
      lk = bk_series_log(x, nu, A.eps, A.cap);
    } else if (!fast) {
      lk = fixed_window_log_ref(x, nu, A.t0, A.t1, A.bins);
    }
    const int er = ld_u16_volatile(&s_eidx[tid]);
    sx[er] = lk;
    if (A.k) snu[er] = (fabs(lk) < 700.0) ? exp_acc(lk, s_exp) : exp(lk);
    spath[er] = series ? 0 : 1;
  }
  __syncthreads();
  // coalesced streaming stores, fixed trip count (all of a thread's stores in flight)
#pragma unroll
  for (int i = 0; i < kBkPerThread; ++i) {
    const int e = i * kBkThreads + tid;
    if (e < cnt) {
      __stcs(A.log_k + base + e, sx[e]);
      if (A.k) __stcs(A.k + base + e, snu[e]);
      if (A.path) A.path[base + e] = spath[e];
    }
  }
}

// One (x, nu) on one warp: the batch kernel's per-element path without the chunk
// staging and the sort (the scalar drop-in API, besselk.py:94-165).  The same
// device routines on the same inputs -- fixed_window_fast is warp-collective, lane
// 0 active -- so the value is bitwise the batch kernel's.  x and nu arrive as
// kernel parameters; log K and then the call's sequence number are written to a
// page-locked, device-mapped host slot that the host polls.
__global__ void __launch_bounds__(32) besselk_scalar_kernel(const __grid_constant__ BkArgs A,
                                                            double x, double nu, double *slot,
                                                            unsigned long long seq) {
  extern __shared__ __align__(16) unsigned char bk_smem[];
  __shared__ double s_exp[128], s_invc[128], s_logc[128];
  double2 *cw = reinterpret_cast<double2 *>(bk_smem);
  const int lane = threadIdx.x;
  const int ncw = A.table_ok ? A.bins + 1 : 0;
  load_tables128(s_exp, s_invc, s_logc);
  for (int k = lane; k < ncw; k += 32) cw[k] = __ldg(A.cwg + k);
  __syncwarp();
  const double a = fabs(nu);
  const bool series = (A.route == 1) || (A.route == 0 && x < A.thr);
  uint32_t w = 0;
  if (!series) {
    const double tmax = fmax(fabs(A.t0), fabs(A.t1));
    const double cmax = ncw ? cw[A.bins].x : 0.0;
    w = bk_window_word(x, a, A.table_ok, tmax, cmax, A.bins, A.win);
  }
  const bool fast = lane == 0 && w != 0u;
  double lk = fixed_window_fast(fast, x, a, w, A, cw, s_exp, s_invc, s_logc);
  if (lane == 0) {
    if (series) {
      lk = bk_series_log(x, nu, A.eps, A.cap);
    } else if (!fast) {
      lk = fixed_window_log_ref(x, nu, A.t0, A.t1, A.bins);
    }
    volatile double *v = slot;
    v[0] = lk;
    __threadfence_system();  // the value is visible to the host before the sequence number
    reinterpret_cast<volatile unsigned long long *>(slot)[1] = seq;
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

// Host emulation of the reference-style walk from the fast path's anchor: how
// many nodes above (up) and below (down) the anchor have a term >= e^-WCUT of it.
// (The reference keeps terms down to e^-46 of its grid max; the ones in between
// are < 4e-18 of the sum each, far below an ulp.)
static void walk_extent_host(double x, double a, double t0, double h, int bins, const double *c,
                             int &up, int &dn) {
  const int m = anchor_node(x, a, t0, h, bins);
  const double ta = t0 + m * h, ca = c[m];
  const double E = std::exp(a * h), Ei = std::exp(-a * h);
  const double q = (2 * a * ta < 700) ? std::exp(-2 * a * ta) : 0.0;
  const double tiny = std::exp(-BGK_BK_WCUT) * (1 + q);
  up = dn = 0;
  double p = 1, qq = 1;
  for (int j = 1; m + j <= bins; ++j) {
    p *= E;
    qq *= Ei;
    if ((q * qq + p) * std::exp(std::fmax(-x * (c[m + j] - ca), -700.0)) < tiny) break;
    up = j;
  }
  p = 1;
  qq = 1;
  for (int j = 1; m - j >= 0; ++j) {
    p *= Ei;
    qq *= E;
    if ((q * qq + p) * std::exp(std::fmax(-x * (c[m - j] - ca), -700.0)) < tiny) break;
    dn = j;
  }
}

// Per (x, nu) cell: U | D << 16, the largest up / down extents over a
// (WSAMP + 1)^2 sample of the cell, edges included (plus BGK_BK_MARGIN nodes).
static void build_window_table(double t0, double t1, int bins, uint32_t *win) {
  std::vector<double> c(bins + 1);
  const double h = (t1 - t0) / bins;
  for (int k = 0; k <= bins; ++k) c[k] = std::cosh(t0 + k * h);
  for (int xi = 0; xi < kXCells; ++xi) {
    const int key = xi + kXKeyBase;
    const int sub = 1 << kXBits;
    const double lo = std::ldexp(1.0 + (double)(key & (sub - 1)) / sub, (key >> kXBits) - 1023);
    const double hi = std::ldexp(1.0 + (double)((key & (sub - 1)) + 1) / sub, (key >> kXBits) - 1023);
    for (int ni = 0; ni < kNuCells; ++ni) {
      const double nlo = ni / (double)kNuStep;
      const double nhi = nlo + 1.0 / kNuStep;
      int U = 0, D = 0;
      for (int sx = 0; sx <= BGK_BK_WSAMP; ++sx)
        for (int sn = 0; sn <= BGK_BK_WSAMP; ++sn) {
          const double xv = sx == BGK_BK_WSAMP ? std::nextafter(hi, 0.0)
                                               : lo + (hi - lo) * sx / (double)BGK_BK_WSAMP;
          const double nv = sn == BGK_BK_WSAMP ? std::nextafter(nhi, 0.0)
                                               : nlo + (nhi - nlo) * sn / (double)BGK_BK_WSAMP;
          int up, dn;
          walk_extent_host(xv, nv, t0, h, bins, c.data(), up, dn);
          U = std::max(U, up);
          D = std::max(D, dn);
        }
      U = std::min(U + BGK_BK_MARGIN, bins);
      D = std::min(D + BGK_BK_MARGIN, bins);
      // The fast path evaluates e^{x (c_a - c_k)} over the window without a
      // clamp: keep the cell only if every exponent stays far inside the table
      // exp's range on a dense sample of the cell (else: reference path).
      bool safe = true;
      for (int sx = 0; sx <= 8 && safe; ++sx)
        for (int sn = 0; sn <= 8 && safe; ++sn) {
          const double xv = lo + (hi - lo) * sx / 8.0 * 0.9999;
          const double nv = nlo + (nhi - nlo) * sn / 8.0 * 0.9999;
          const int m = anchor_node(xv, nv, t0, h, bins);
          for (int k = std::max(0, m - D); k <= std::min(bins, m + U); ++k)
            if (!(xv * (c[m] - c[k]) > -500.0)) safe = false;
        }
      win[xi * kNuCells + ni] = safe ? ((uint32_t)U | ((uint32_t)D << 16)) : 0xffffffffu;
    }
  }
}

}  // namespace bgk

// ---------------------------------------------------------------------------------
// launchers (called from bgk_capi.cpp)
// ---------------------------------------------------------------------------------
// Device copies of the node-window table, one per (device, t0, t1, bins), built
// on the host and uploaded once per device (12 KB each); kept for the life of the
// process.  The key is bgk_device_key(): a pointer uploaded on one device is never
// handed to a launch on another.
struct PredEntry {
  int device_key;
  double t0, t1;
  long long bins;
  uint32_t *dev;  // window table, then the {cosh t_k, ln w_k} node table
  double2 *cw;
};

namespace {
constexpr int64_t kMaxTable = 8191;  // 128 KB of shared memory ({c, ln w} pairs)

void bk_fill_args(bgk::BkArgs &A, const double *x, const double *nu, int64_t n,
                  const bgk_config *cfg, int route, double *log_k, double *k, uint8_t *path) {
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
  A.t0f = (float)A.t0;
  A.hinvf = (float)(1.0 / A.h);
  A.binsf = (float)A.bins;
  A.table_ok = (cfg->t_lower >= 0.0 && cfg->bins <= kMaxTable) ? 1 : 0;
  A.win = nullptr;
  A.cwg = nullptr;
}

// Host image of the tables: the window table (padded to 16 B), then the node table
// {cosh t_k, weight exponent adjust} exactly as the reference's caller builds it:
// t_k = t0 + k h, cosh via the host libm (what numba calls).
size_t bk_host_tables(const bgk_config *cfg, std::vector<uint32_t> &host) {
  const size_t nwin = (size_t)bgk::kXCells * bgk::kNuCells;
  const size_t nwin_pad = (nwin + 3) & ~(size_t)3;  // 16-byte aligned node table
  const int bins = (int)cfg->bins;
  host.assign(nwin_pad + 4 * (size_t)(bins + 1), 0u);
  bgk::build_window_table(cfg->t_lower, cfg->t_upper, bins, host.data());
  const double h = (cfg->t_upper - cfg->t_lower) / (double)bins;
  double *cwh = reinterpret_cast<double *>(host.data() + nwin_pad);
  for (int k = 0; k <= bins; ++k) {
    cwh[2 * k] = std::cosh(cfg->t_lower + (double)k * h);
    // weight 1/2 at the ends as an exponent adjustment (see fixed_window_fast)
    const uint64_t wbits = (k == 0 || k == bins) ? (uint64_t)(uint32_t)(-(1 << 20)) : 0u;
    std::memcpy(&cwh[2 * k + 1], &wbits, 8);
  }
  return nwin_pad;
}

// Device copies of the tables, one per (device, t0, t1, bins), uploaded once per
// device (12 KB + the node table); kept for the life of the process.
int bk_device_tables(const bgk_config *cfg, bgk::BkArgs &A) {
  static std::mutex mu;
  static std::vector<PredEntry> cache;
  if (!A.table_ok) return BGK_OK;
  const int dev_key = bgk_device_key(nullptr);
  std::lock_guard<std::mutex> lock(mu);
  for (const PredEntry &e : cache)
    if (e.device_key == dev_key && e.t0 == cfg->t_lower && e.t1 == cfg->t_upper &&
        e.bins == cfg->bins) {
      A.win = e.dev;
      A.cwg = e.cw;
      return BGK_OK;
    }
  std::vector<uint32_t> host;
  const size_t nwin_pad = bk_host_tables(cfg, host);
  uint32_t *dev = nullptr;
  const size_t bytes = host.size() * sizeof(uint32_t);
  cudaError_t err = cudaMalloc(&dev, bytes);
  if (err == cudaSuccess) err = cudaMemcpy(dev, host.data(), bytes, cudaMemcpyHostToDevice);
  if (err != cudaSuccess) {
    cudaGetLastError();
    bgk_set_error("besselk prediction table upload: %s", cudaGetErrorString(err));
    return BGK_ERR_CUDA;
  }
  double2 *cwd = reinterpret_cast<double2 *>(dev + nwin_pad);
  cache.push_back({dev_key, cfg->t_lower, cfg->t_upper, cfg->bins, dev, cwd});
  A.win = dev;
  A.cwg = cwd;
  return BGK_OK;
}

// The window an element is summed over, as the kernel decides it (anchor: the host
// fp32 asinhf on the CPU, the kernel's fast fp32 anchor on the device).
__host__ __device__ inline void bk_window_of(double x, double nu, const bgk::BkArgs &A,
                                             double cmax, bool device_anchor, int32_t &m,
                                             int32_t &lo, int32_t &hi) {
  m = lo = hi = -1;
  const double a = fabs(nu);
  const bool series = (A.route == 1) || (A.route == 0 && x < A.thr);
  if (series) return;
  const double tmax = fmax(fabs(A.t0), fabs(A.t1));
  const uint32_t w = bgk::bk_window_word(x, a, A.table_ok, tmax, cmax, A.bins, A.win);
  if (!w) return;
#ifdef __CUDA_ARCH__
  const int mm = device_anchor ? bgk::anchor_node_fast(x, a, A.t0f, A.hinvf, A.binsf)
                               : bgk::anchor_node(x, a, A.t0, A.h, A.bins);
#else
  (void)device_anchor;
  const int mm = bgk::anchor_node(x, a, A.t0, A.h, A.bins);
#endif
  const int U = min((int)(w & 0xffff), A.bins - mm), D = min((int)(w >> 16), mm);
  m = mm;
  lo = mm - D;
  hi = mm + U;
}

__global__ void bk_windows_kernel(const bgk::BkArgs A, int32_t *m, int32_t *lo, int32_t *hi) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  const double cmax = A.table_ok ? A.cwg[A.bins].x : 0.0;
  int32_t a, b, c;
  bk_window_of(A.x[i], A.nu[i], A, cmax, true, a, b, c);
  m[i] = a;
  lo[i] = b;
  hi[i] = c;
}
}  // namespace

extern "C" int bgk_besselk_windows_host(const double *x, const double *nu, int64_t n,
                                        const bgk_config *cfg, int32_t *m, int32_t *lo,
                                        int32_t *hi) {
  if (!cfg || n < 0 || (n > 0 && (!x || !nu || !m || !lo || !hi)) || cfg->bins < 1 ||
      !(cfg->t_upper > cfg->t_lower)) {
    bgk_set_error("bgk_besselk_windows_host: bad arguments");
    return BGK_ERR_INVALID;
  }
  bgk::BkArgs A;
  bk_fill_args(A, x, nu, n, cfg, 0, nullptr, nullptr, nullptr);
  std::vector<uint32_t> host;
  double cmax = 0.0;
  if (A.table_ok) {
    const size_t nwin_pad = bk_host_tables(cfg, host);
    A.win = host.data();
    cmax = reinterpret_cast<const double *>(host.data() + nwin_pad)[2 * cfg->bins];
  }
  for (int64_t i = 0; i < n; ++i) bk_window_of(x[i], nu[i], A, cmax, false, m[i], lo[i], hi[i]);
  return BGK_OK;
}

extern "C" int bgk_besselk_windows(const double *x, const double *nu, int64_t n,
                                   const bgk_config *cfg, int32_t *m, int32_t *lo, int32_t *hi,
                                   void *stream) {
  if (!cfg || n < 0 || (n > 0 && (!x || !nu || !m || !lo || !hi)) || cfg->bins < 1 ||
      !(cfg->t_upper > cfg->t_lower)) {
    bgk_set_error("bgk_besselk_windows: bad arguments");
    return BGK_ERR_INVALID;
  }
  if (n == 0) return BGK_OK;
  bgk::BkArgs A;
  bk_fill_args(A, x, nu, n, cfg, 0, nullptr, nullptr, nullptr);
  if (int rc = bk_device_tables(cfg, A)) return rc;
  bk_windows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(A, m, lo, hi);
  bgk_note_launch();
  return bgk_check_launch("bk_windows_kernel");
}

// One (x, nu): besselk_scalar_kernel on one warp, the inputs as kernel parameters,
// the result through a per-(thread, device) page-locked, device-mapped host slot
// [log K, sequence number] that the host polls -- no copies and no stream
// synchronisation on the fast path (the scalar drop-in API, besselk.py:94-165).
// Bitwise the batch result.  The poll falls back to cudaStreamQuery every 4096 spins,
// so a launch or kernel fault is reported instead of spinning forever.
extern "C" int bgk_besselk_scalar(double x, double nu, const bgk_config *cfg, int route,
                                  double *log_k, void *stream) {
  if (!cfg || !log_k || route < 0 || route > 2 || cfg->bins < 1 ||
      !(cfg->t_upper > cfg->t_lower)) {
    bgk_set_error("bgk_besselk_scalar: bad arguments");
    return BGK_ERR_INVALID;
  }
  struct Slot {
    int key;
    double *host;  // [log_k, seq]
    double *dev;   // the same memory, device view
    unsigned long long seq;
  };
  thread_local std::vector<Slot> slots;
  const int key = bgk_device_key(nullptr);
  Slot *sl = nullptr;
  for (Slot &e : slots)
    if (e.key == key) sl = &e;
  if (!sl) {
    Slot e{key, nullptr, nullptr, 0};
    cudaError_t err = cudaHostAlloc((void **)&e.host, 4 * sizeof(double), cudaHostAllocMapped);
    if (err == cudaSuccess) err = cudaHostGetDevicePointer((void **)&e.dev, e.host, 0);
    if (err != cudaSuccess) {
      cudaGetLastError();
      bgk_set_error("bgk_besselk_scalar: mapped host slot: %s", cudaGetErrorString(err));
      return BGK_ERR_CUDA;
    }
    reinterpret_cast<volatile unsigned long long *>(e.host)[1] = 0;
    slots.push_back(e);
    sl = &slots.back();
  }
  bgk::BkArgs A;
  bk_fill_args(A, nullptr, nullptr, 1, cfg, route, nullptr, nullptr, nullptr);
  if (int rc = bk_device_tables(cfg, A)) return rc;
  const size_t smem = A.table_ok ? sizeof(double2) * ((size_t)cfg->bins + 1) : 0;
  if (int rc = bgk_ensure_smem_optin((const void *)bgk::besselk_scalar_kernel,
                                     "besselk_scalar_kernel",
                                     (int)(sizeof(double2) * (kMaxTable + 1))))
    return rc;
  const unsigned long long seq = ++sl->seq;
  bgk::besselk_scalar_kernel<<<1, 32, smem, (cudaStream_t)stream>>>(A, x, nu, sl->dev, seq);
  bgk_note_launch();
  if (int rc = bgk_check_launch("besselk_scalar_kernel")) return rc;
  volatile unsigned long long *flag = reinterpret_cast<volatile unsigned long long *>(sl->host) + 1;
  for (unsigned spins = 1; *flag != seq; ++spins) {
    if ((spins & 4095) == 0) {
      const cudaError_t q = cudaStreamQuery((cudaStream_t)stream);
      if (q == cudaSuccess && *flag == seq) break;
      if (q != cudaSuccess && q != cudaErrorNotReady) {
        bgk_set_error("bgk_besselk_scalar: %s", cudaGetErrorString(q));
        return BGK_ERR_CUDA;
      }
      if (q == cudaSuccess && *flag != seq) {
        bgk_set_error("bgk_besselk_scalar: kernel finished without a result");
        return BGK_ERR_CUDA;
      }
    }
  }
  *log_k = reinterpret_cast<volatile double *>(sl->host)[0];
  return BGK_OK;
}

int bgk_launch_besselk(const double *x, const double *nu, int64_t n, const bgk_config *cfg,
                       int route, double *log_k, double *k, uint8_t *path, cudaStream_t stream) {
  if (n == 0) return 0;
  bgk::BkArgs A;
  bk_fill_args(A, x, nu, n, cfg, route, log_k, k, path);
  if (int rc = bk_device_tables(cfg, A)) return rc;
  // Elements per thread: 8 (2048 per CTA), or -- for batches of at most two waves of
  // CTAs over the SMs x resident CTAs slots -- fewer when that evens out the last wave:
  // cost ~ waves x chunk, ties to the larger chunk (1M elements: 586 CTAs of 1792 in
  // one wave instead of 512 of 2048 on 592 slots, A/B on B200 40 -> 37 us).  Larger
  // batches keep 2048: their CTAs finish at staggered times, so the waves do not
  // quantise, and smaller chunks only add per-CTA set-up (64 Mi: 1.48 -> 1.58 ms).
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long slots = (long long)nsm * BGK_BK_MINBLOCKS;
  int per = bgk::kBkPerThread;
  long long best = LLONG_MAX;
  const int pmin = n <= 2 * slots * bgk::kBkChunk ? bgk::kBkPerThread - 3 : bgk::kBkPerThread;
  for (int p = bgk::kBkPerThread; p >= pmin && p >= 1; --p) {
    const long long ctas = (n + (long long)bgk::kBkThreads * p - 1) / ((long long)bgk::kBkThreads * p);
    const long long cost = (ctas + slots - 1) / slots * p;
    if (cost < best) {
      best = cost;
      per = p;
    }
  }
#ifdef BGK_BK_FORCE_PER  // A/B builds only (BK 1M on B200: the choice above, 7 -> 38 us; 6 / 4 / 3 / 2 -> 40 / 42 / 45 / 48 us)
  per = BGK_BK_FORCE_PER;
#endif
  const long long grid = (n + (long long)bgk::kBkThreads * per - 1) / ((long long)bgk::kBkThreads * per);
  const size_t table_bytes = sizeof(double2) * (A.table_ok ? (size_t)cfg->bins + 1 : 0);
  switch (per - bgk::kBkPerThread) {
#define BGK_BK_LAUNCH(D)                                                                          \
  case D: {                                                                                       \
    constexpr int P = bgk::kBkPerThread + (D);                                                   \
    const void *fn = (const void *)bgk::besselk_kernel<P>;                                        \
    /* opt in once per device for the largest table (so every bins <= kMaxTable fits) */          \
    if (int rc = bgk_ensure_smem_optin(fn, "besselk_kernel",                                      \
                                       (int)(sizeof(double2) * (kMaxTable + 1) + bgk::bk_chunk_bytes(P)))) \
      return rc;                                                                                  \
    bgk::besselk_kernel<P><<<(unsigned)grid, bgk::kBkThreads, table_bytes + bgk::bk_chunk_bytes(P), stream>>>(A); \
    break;                                                                                        \
  }
    BGK_BK_LAUNCH(0)
    BGK_BK_LAUNCH(-1)
    BGK_BK_LAUNCH(-2)
    BGK_BK_LAUNCH(-3)
#ifdef BGK_BK_FORCE_PER
    BGK_BK_LAUNCH(-4)
    BGK_BK_LAUNCH(-5)
    BGK_BK_LAUNCH(-6)
#endif
#undef BGK_BK_LAUNCH
    default:
      bgk_set_error("besselk launch: no kernel for %d elements per thread", per);
      return BGK_ERR_UNSUPPORTED;
  }
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
