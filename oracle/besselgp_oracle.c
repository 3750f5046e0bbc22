/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the BesselK / Matern hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It is never linked into, called by or
 * used as a fallback for the product (paper_2502_00356_b200/).
 *
 * What it is: a scalar C restatement of the reference's numba kernels
 * (/root/reference/pkg/src/besselgp/kernels.py) plus the restated Matern
 * caller that the reference only specifies.  Each function
 * cites the reference line range it follows.  It is compiled with
 * -ffp-contract=off and no fast-math against glibc libm, which is what the
 * numba JIT emits for kernels.py (LLVM IR with no fma / contract flags; exp and
 * log as llvm intrinsics lowered to libm, cosh/sinh/asinh/log1p as direct libm
 * calls -- SURVEY.md Appendix A.6).  The one known divergence: numba's
 * math.gamma is CPython's Lanczos routine, this file uses glibc tgamma; that
 * only touches the Temme (x < 0.1) branch, at the ulp level.
 *
 * Pinning: tests/test_oracle_golden.py checks this file against golden vectors
 * produced by importing the reference itself (tests/golden/make_golden.py).
 *
 * Threaded drivers (pthreads) exist for the CPU baseline: the reference's own
 * idiom is a ThreadPoolExecutor over independent chunks / tiles of nogil
 * kernels (oracle.py:211-213).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EPS_MACHINE (2.220446049250313e-16) /* kernels.py:15, 2**-52 */
#define LN2 0.6931471805599453              /* kernels.py:16 */

/* kernels.py:27-40 -- odd Taylor coefficients of 1/Gamma(1+z). */
static const double G1_ODD[12] = {
    0.57721566490153286061,
    -0.042002635034095235529,
    -0.042197734555544336748,
    0.0072189432466630995424,
    -0.00021524167411495097282,
    -2.0134854780788238656e-05,
    1.1330272319816958824e-06,
    6.1160951044814158179e-09,
    -1.1812745704870201446e-09,
    7.782263439905071254e-12,
    5.100370287454475979e-13,
    -5.3481225394230179824e-15,
};

/* kernels.py:43-49 */
double orc_log_cosh(double z) {
  z = fabs(z);
  if (z < 25.0) return log(cosh(z));
  return z - LN2 + log1p(exp(-2.0 * z));
}

/* kernels.py:52-55 */
double orc_log_integrand(double t, double x, double nu) {
  return orc_log_cosh(nu * t) - x * cosh(t);
}

/* kernels.py:58-61 */
double orc_log_integrand_d1(double t, double x, double nu) {
  return nu * tanh(nu * t) - x * sinh(t);
}

/* kernels.py:64-72 */
double orc_log_integrand_d2(double t, double x, double nu) {
  double z = fabs(nu * t);
  double sech = (z < 350.0) ? 1.0 / cosh(z) : 0.0;
  return nu * nu * sech * sech - x * cosh(t);
}

/* kernels.py:112-123 -- first maximum wins (strict >). */
int64_t orc_grid_peak_index(double x, double nu, double t0, double t1, int64_t bins) {
  double h = (t1 - t0) / (double)bins;
  double best = -INFINITY;
  int64_t m_star = 0;
  for (int64_t m = 0; m < bins + 1; ++m) {
    double g = orc_log_integrand(t0 + (double)m * h, x, nu);
    if (g > best) {
      best = g;
      m_star = m;
    }
  }
  return m_star;
}

/* kernels.py:126-139 */
static inline double node_exponent(double anu, double x, double dt, double t_star, double z_star,
                                   double lc_star, double ch_star, double ss, double cs) {
  (void)t_star;
  double z_m = z_star + anu * dt;
  double da;
  if (z_m >= 30.0 && z_star >= 30.0) {
    da = anu * dt;
  } else if (z_m < 25.0 && z_star < 25.0) {
    da = log(cosh(z_m) / ch_star);
  } else {
    da = orc_log_cosh(z_m) - lc_star;
  }
  double sh = sinh(0.5 * dt);
  double ch = cosh(0.5 * dt);
  double db = 2.0 * x * (ss * ch + cs * sh) * sh;
  return da - db;
}

/* kernels.py:142-151 */
double orc_canonical_anchor_t(double x, double nu) {
  double anu = fabs(nu);
  if (anu * anu <= x) return 0.0;
  return asinh(anu / x);
}

/* kernels.py:154-209 -- walk outward from m_star, break at dg <= -46, Kahan,
 * then rebase onto the canonical anchor.  Returns shift, writes ln_sum. */
double orc_window_lse(double x, double nu, double t0, double t1, int64_t bins, int64_t m_star,
                      double *ln_sum_out) {
  double h = (t1 - t0) / (double)bins;
  double anu = fabs(nu);
  double t_star = t0 + (double)m_star * h;
  double z_star = anu * t_star;
  double lc_star = orc_log_cosh(z_star);
  double ch_star = (z_star < 25.0) ? cosh(z_star) : INFINITY;
  double ss = sinh(t_star);
  double cs = cosh(t_star);

  double acc = (0 < m_star && m_star < bins) ? 1.0 : 0.5;
  double comp = 0.0;
  for (int direction = 0; direction < 2; ++direction) {
    double sign = (direction == 0) ? 1.0 : -1.0;
    int64_t span = (direction == 0) ? (bins - m_star) : m_star;
    for (int64_t k = 1; k < span + 1; ++k) {
      double dt = sign * ((double)k * h);
      double dg = node_exponent(anu, x, dt, t_star, z_star, lc_star, ch_star, ss, cs);
      if (dg <= -46.0) break;
      int64_t m = m_star + ((direction == 0) ? k : -k);
      double w = (m == 0 || m == bins) ? 0.5 : 1.0;
      double y = w * exp(dg) - comp;
      double t_acc = acc + y;
      comp = (t_acc - acc) - y;
      acc = t_acc;
    }
  }

  double t_hat = orc_canonical_anchor_t(x, nu);
  double z_hat = anu * t_hat;
  double shift = orc_log_cosh(z_hat) - x * cosh(t_hat);
  double dt_sh = t_star - t_hat;
  double da_sh;
  if (z_star >= 30.0 && z_hat >= 30.0) {
    da_sh = anu * dt_sh;
  } else {
    da_sh = lc_star - orc_log_cosh(z_hat);
  }
  double sh = sinh(0.5 * dt_sh);
  double db_sh = 2.0 * x * (sinh(t_hat) * cosh(0.5 * dt_sh) + cosh(t_hat) * sh) * sh;
  double dg_sh = da_sh - db_sh;
  *ln_sum_out = dg_sh + log(h * acc);
  return shift;
}

/* kernels.py:212-216 */
double orc_fixed_window_log_pair(double x, double nu, double t0, double t1, int64_t bins,
                                 double *ln_sum_out) {
  int64_t m_star = orc_grid_peak_index(x, nu, t0, t1, bins);
  return orc_window_lse(x, nu, t0, t1, bins, m_star, ln_sum_out);
}

/* kernels.py:219-227 */
static double gamma1(double mu) {
  double acc = 0.0;
  double mu2 = mu * mu;
  double p = 1.0;
  for (int i = 0; i < 12; ++i) {
    acc += G1_ODD[i] * p;
    p *= mu2;
  }
  return -acc;
}

/* kernels.py:230-270 -- returns terms; writes (s0, s1). */
int64_t orc_temme_sums(double x, double mu, double eps, int64_t series_cap, double *s0_out,
                       double *s1_out) {
  double d = log(2.0 / x);
  double sigma = mu * d;
  double gam1 = gamma1(mu);
  double gam2 = 0.5 * (1.0 / tgamma(1.0 - mu) + 1.0 / tgamma(1.0 + mu));
  double fact = (fabs(mu) < 1e-10) ? 1.0 : mu * M_PI / sin(mu * M_PI);
  double sh = (sigma == 0.0) ? 1.0 : sinh(sigma) / sigma;
  double f = fact * (cosh(sigma) * gam1 + gam2 * sh * d);
  double p = 0.5 * exp(sigma) * tgamma(1.0 + mu);
  double q = 0.5 * exp(-sigma) * tgamma(1.0 - mu);
  double c = 1.0;
  double s0 = f;
  double s1 = p;
  double x2_4 = 0.25 * x * x;
  int64_t terms = 1;
  for (int64_t k = 1; k < series_cap + 1; ++k) {
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
  *s0_out = s0;
  *s1_out = s1;
  return terms;
}

/* kernels.py:273-293 */
double orc_temme_series_log(double x, double nu, double eps, int64_t series_cap) {
  int64_t m_steps = (int64_t)floor(nu + 0.5);
  double mu = nu - (double)m_steps;
  double s0, s1;
  orc_temme_sums(x, mu, eps, series_cap, &s0, &s1);
  double l_prev = log(s0);
  if (m_steps == 0) return l_prev;
  double l_cur = LN2 - log(x) + log(s1);
  for (int64_t k = 1; k < m_steps; ++k) {
    double eta = mu + (double)k;
    double l_next = l_cur + log(2.0 * eta / x + exp(l_prev - l_cur));
    l_prev = l_cur;
    l_cur = l_next;
  }
  return l_cur;
}

/* kernels.py:296-302 */
double orc_refined_log_bessel(double x, double nu, double t0, double t1, int64_t bins,
                              double thr, double eps, int64_t series_cap) {
  if (x < thr) return orc_temme_series_log(x, nu, eps, series_cap);
  double ln_sum;
  double shift = orc_fixed_window_log_pair(x, nu, t0, t1, bins, &ln_sum);
  return shift + ln_sum;
}

/* kernels.py:338-381 -- one tile, out is row-major m x n with leading dim ld. */
void orc_matern_tile(double *out, int64_t ld, const double *rx, const double *ry, int64_t m,
                     const double *cx, const double *cy, int64_t n, double sigma_sq, double beta,
                     double nu, double log_prefactor, const double *c_nodes,
                     const double *a_nodes, int64_t nnodes, double h, double thr, double eps,
                     int64_t series_cap) {
  int64_t b = nnodes - 1;
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double dx = rx[i] - cx[j];
      double dy = ry[i] - cy[j];
      double r = sqrt(dx * dx + dy * dy);
      if (r == 0.0) {
        out[i * ld + j] = sigma_sq;
        continue;
      }
      double u = r / beta;
      double ln_k;
      if (u < thr) {
        ln_k = orc_temme_series_log(u, nu, eps, series_cap);
      } else {
        double g_max = -INFINITY;
        int64_t m_star = 0;
        for (int64_t k = 0; k < b + 1; ++k) {
          double g = a_nodes[k] - u * c_nodes[k];
          if (g > g_max) {
            g_max = g;
            m_star = k;
          }
        }
        double acc = 0.0, comp = 0.0;
        for (int64_t k = 0; k < b + 1; ++k) {
          double dg = (a_nodes[k] - a_nodes[m_star]) - u * (c_nodes[k] - c_nodes[m_star]);
          if (dg > -46.0) {
            double w = (k == 0 || k == b) ? 0.5 : 1.0;
            double y = w * exp(dg) - comp;
            double t_acc = acc + y;
            comp = (t_acc - acc) - y;
            acc = t_acc;
          }
        }
        ln_k = g_max + log(h * acc);
      }
      out[i * ld + j] = exp(log_prefactor + nu * log(u) + ln_k);
    }
  }
}

/* ---- restated Matern caller (kernels.py:343-345) ------------------- */

/* Node tables exactly as the restated caller builds them: h=(t1-t0)/b,
 * c_m = cosh(t0 + m h), a_m = log_cosh(nu (t0 + m h)). */
void orc_matern_tables(double nu, double t0, double t1, int64_t bins, double *c_nodes,
                       double *a_nodes, double *h_out) {
  double h = (t1 - t0) / (double)bins;
  for (int64_t m = 0; m < bins + 1; ++m) {
    double t = t0 + (double)m * h;
    c_nodes[m] = cosh(t);
    a_nodes[m] = orc_log_cosh(nu * t);
  }
  *h_out = h;
}

/* log(sigma^2 2^(1-nu) / Gamma(nu)) -- the Matern log-prefactor. */
double orc_matern_log_prefactor(double sigma_sq, double nu) {
  return log(sigma_sq) - (nu - 1.0) * LN2 - lgamma(nu);
}

/* ---- threaded drivers (CPU baseline) ------------------------------------------------ */

typedef struct {
  const double *x, *nu;
  double *out;
  int64_t n;
  double t0, t1, thr, eps;
  int64_t bins, cap;
  int64_t chunk;
  int64_t next; /* shared work cursor */
  pthread_mutex_t lock;
} bk_job;

static void *bk_worker(void *arg) {
  bk_job *J = (bk_job *)arg;
  for (;;) {
    pthread_mutex_lock(&J->lock);
    int64_t s = J->next;
    J->next += J->chunk;
    pthread_mutex_unlock(&J->lock);
    if (s >= J->n) break;
    int64_t e = s + J->chunk < J->n ? s + J->chunk : J->n;
    for (int64_t i = s; i < e; ++i)
      J->out[i] = orc_refined_log_bessel(J->x[i], J->nu[i], J->t0, J->t1, J->bins, J->thr,
                                         J->eps, J->cap);
  }
  return NULL;
}

/* ln K for a batch on `threads` workers pulling chunks (the reference's
 * ThreadPoolExecutor-over-chunks idiom, oracle.py:211-213). */
void orc_refined_log_bessel_batch(const double *x, const double *nu, int64_t n, double t0,
                                  double t1, int64_t bins, double thr, double eps,
                                  int64_t series_cap, double *out, int threads) {
  bk_job J;
  J.x = x;
  J.nu = nu;
  J.out = out;
  J.n = n;
  J.t0 = t0;
  J.t1 = t1;
  J.thr = thr;
  J.eps = eps;
  J.bins = bins;
  J.cap = series_cap;
  J.chunk = n / 256 > 0 ? n / 256 : 1;
  J.next = 0;
  pthread_mutex_init(&J.lock, NULL);
  if (threads < 1) threads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, bk_worker, &J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&J.lock);
}

typedef struct {
  const double *lx, *ly;
  int64_t N, ts, T;
  int64_t row0, row1; /* rows of the full matrix to produce, [row0,row1) */
  double *out;        /* row-major (row1-row0) x N, leading dim ld */
  int64_t ld;
  int mirror;
  double sigma_sq, beta, nu, lp, h, thr, eps;
  const double *c, *a;
  int64_t nnodes, cap;
  int64_t next, ntiles;
  pthread_mutex_t lock;
} cov_job;

static void *cov_worker(void *arg) {
  cov_job *J = (cov_job *)arg;
  double *tile = (double *)malloc(sizeof(double) * (size_t)(J->ts * J->ts));
  int64_t p0 = J->row0 / J->ts;
  for (;;) {
    pthread_mutex_lock(&J->lock);
    int64_t l = J->next++;
    pthread_mutex_unlock(&J->lock);
    if (l >= J->ntiles) break;
    /* tiles enumerated row-major over (p, q); with mirror only q <= p */
    int64_t p, q;
    if (J->mirror) {
      /* l indexes lower tiles of the full matrix */
      p = (int64_t)((sqrt(8.0 * (double)l + 1.0) - 1.0) / 2.0);
      while ((p + 1) * (p + 2) / 2 <= l) ++p;
      while (p * (p + 1) / 2 > l) --p;
      q = l - p * (p + 1) / 2;
    } else {
      int64_t prow = (J->row1 - J->row0 + J->ts - 1) / J->ts;
      (void)prow;
      p = p0 + l / J->T;
      q = l % J->T;
    }
    int64_t r0 = p * J->ts, c0 = q * J->ts;
    int64_t m = (r0 + J->ts <= J->N) ? J->ts : J->N - r0;
    int64_t n = (c0 + J->ts <= J->N) ? J->ts : J->N - c0;
    /* restrict rows to [row0,row1) for the non-mirrored row-block mode */
    int64_t rs = r0 < J->row0 ? J->row0 : r0;
    int64_t re = r0 + m > J->row1 ? J->row1 : r0 + m;
    if (re <= rs) continue;
    orc_matern_tile(tile, n, J->lx + rs, J->ly + rs, re - rs, J->lx + c0, J->ly + c0, n,
                    J->sigma_sq, J->beta, J->nu, J->lp, J->c, J->a, J->nnodes, J->h, J->thr,
                    J->eps, J->cap);
    for (int64_t i = rs; i < re; ++i)
      memcpy(J->out + (i - J->row0) * J->ld + c0, tile + (i - rs) * n, sizeof(double) * n);
    if (J->mirror && p != q) {
      for (int64_t i = 0; i < re - rs; ++i)
        for (int64_t j = 0; j < n; ++j) J->out[(c0 + j) * J->ld + rs + i] = tile[i * n + j];
    }
  }
  free(tile);
  return NULL;
}

/* Restated generate_covariance: lower tiles computed with
 * matern_tile and mirrored, tiles handed to `threads` workers.  mirror=1
 * produces the full N x N matrix (row0=0,row1=N).  mirror=0 produces the row
 * block [row0,row1) by computing every tile of those rows directly (used to
 * time a bounded sample of the big configs). */
static void generate_covariance_impl(const double *lx, const double *ly, int64_t N,
                                     double sigma_sq, double beta, double nu, double t0,
                                     double t1, int64_t bins, double thr, double eps,
                                     int64_t series_cap, int64_t tile_size, int64_t row0,
                                     int64_t row1, int mirror, double *out, int64_t ld,
                                     int threads, int64_t l0, int64_t l1);

void orc_generate_covariance(const double *lx, const double *ly, int64_t N, double sigma_sq,
                             double beta, double nu, double t0, double t1, int64_t bins,
                             double thr, double eps, int64_t series_cap, int64_t tile_size,
                             int64_t row0, int64_t row1, int mirror, double *out, int64_t ld,
                             int threads) {
  generate_covariance_impl(lx, ly, N, sigma_sq, beta, nu, t0, t1, bins, thr, eps, series_cap,
                           tile_size, row0, row1, mirror, out, ld, threads, 0, -1);
}

/* The full-matrix job (lower tiles + mirror) restricted to lower-tile indices
 * [l0, l1): K calls over a partition of [0, T(T+1)/2) produce the whole matrix,
 * so bench.py can spread one generate_covariance over K timed steps. */
void orc_generate_covariance_tiles(const double *lx, const double *ly, int64_t N,
                                   double sigma_sq, double beta, double nu, double t0, double t1,
                                   int64_t bins, double thr, double eps, int64_t series_cap,
                                   int64_t tile_size, int64_t l0, int64_t l1, double *out,
                                   int64_t ld, int threads) {
  generate_covariance_impl(lx, ly, N, sigma_sq, beta, nu, t0, t1, bins, thr, eps, series_cap,
                           tile_size, 0, N, 1, out, ld, threads, l0, l1);
}

/* First touch of a host buffer with `threads` threads (page faults outside a timed
 * region). */
typedef struct {
  double *p;
  int64_t n;
  int t, nt;
} touch_job;
static void *touch_worker(void *arg) {
  touch_job *J = (touch_job *)arg;
  int64_t a = J->n * J->t / J->nt, b = J->n * (J->t + 1) / J->nt;
  memset(J->p + a, 0, sizeof(double) * (size_t)(b - a));
  return NULL;
}
void orc_touch(double *p, int64_t n, int threads) {
  if (threads < 1) threads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
  touch_job *jobs = (touch_job *)malloc(sizeof(touch_job) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t].p = p; jobs[t].n = n; jobs[t].t = t; jobs[t].nt = threads;
    pthread_create(&th[t], NULL, touch_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(jobs);
  free(th);
}

static void generate_covariance_impl(const double *lx, const double *ly, int64_t N,
                                     double sigma_sq, double beta, double nu, double t0,
                                     double t1, int64_t bins, double thr, double eps,
                                     int64_t series_cap, int64_t tile_size, int64_t row0,
                                     int64_t row1, int mirror, double *out, int64_t ld,
                                     int threads, int64_t l0, int64_t l1) {
  cov_job J;
  double *c = (double *)malloc(sizeof(double) * (size_t)(bins + 1));
  double *a = (double *)malloc(sizeof(double) * (size_t)(bins + 1));
  orc_matern_tables(nu, t0, t1, bins, c, a, &J.h);
  J.lx = lx;
  J.ly = ly;
  J.N = N;
  J.ts = tile_size;
  J.T = (N + tile_size - 1) / tile_size;
  J.row0 = mirror ? 0 : row0;
  J.row1 = mirror ? N : row1;
  J.out = out;
  J.ld = ld;
  J.mirror = mirror;
  J.sigma_sq = sigma_sq;
  J.beta = beta;
  J.nu = nu;
  J.lp = orc_matern_log_prefactor(sigma_sq, nu);
  J.thr = thr;
  J.eps = eps;
  J.c = c;
  J.a = a;
  J.nnodes = bins + 1;
  J.cap = series_cap;
  J.next = 0;
  if (mirror) {
    J.ntiles = J.T * (J.T + 1) / 2;
    if (l1 >= 0 && l1 < J.ntiles) J.ntiles = l1;
    J.next = l0 > 0 ? l0 : 0;
  } else {
    int64_t p0 = J.row0 / tile_size, p1 = (J.row1 + tile_size - 1) / tile_size;
    J.ntiles = (p1 - p0) * J.T;
  }
  pthread_mutex_init(&J.lock, NULL);
  if (threads < 1) threads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, cov_worker, &J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&J.lock);
  free(c);
  free(a);
}
