/*
 * besselgp_b200.h -- C ABI of libbesselgp_sm100a.so, the B200 (sm_100a) build of
 * the BesselK / Matern-covariance hot path of arXiv 2502.00356.
 *
 * Drop-in boundary.  The reference has no native code: its "operator layer" is
 * the set of numba kernels in /root/reference/pkg/src/besselgp/kernels.py that
 * take flat scalars plus caller-allocated arrays.  Each entry point below
 * replaces one of them (file:line cited) over device arrays, and the Python
 * package paper_2502_00356_b200 binds them with ctypes exactly where the
 * reference's besselk.py calls kernels.* (see INTEGRATION.md).
 *
 * Conventions:
 *   - every array argument is a DEVICE pointer (cudaMalloc / torch CUDA tensor);
 *     the caller owns all memory, the library never allocates;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *     every call is asynchronous and stream-ordered, re-entrant, and keeps no
 *     mutable global state (per-call tables travel as kernel parameters);
 *   - return 0 (BGK_OK) or a negative BGK_ERR_* code; bgk_last_error() gives a
 *     thread-local message.  Domain validation with the reference's exact
 *     messages lives in the Python layer (besselk.py:28-29, 43-51, 65-69);
 *     like the numba kernels, these entry points never raise on values --
 *     garbage in gives NaN/inf out;
 *   - results are pure functions of each element's inputs: bitwise
 *     independent of batch size, tiling, launch geometry and shard count.
 */
#ifndef BESSELGP_B200_H
#define BESSELGP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BGK_ABI_VERSION 4

#define BGK_OK 0
#define BGK_ERR_INVALID (-1)     /* bad argument (null pointer, bad size, bad enum) */
#define BGK_ERR_CUDA (-2)        /* a CUDA runtime error (launch / config) */
#define BGK_ERR_UNSUPPORTED (-3) /* configuration outside what the kernels support */

/* QuadratureConfig (besselk.py:32-41): fixed window [t_lower, t_upper], bins
 * trapezoid intervals, series below small_x_threshold, Temme cap / epsilon. */
typedef struct bgk_config {
  double t_lower;
  double t_upper;
  int64_t bins;
  double small_x_threshold;
  int64_t series_cap;
  double eps_machine;
} bgk_config;

/* Routing for bgk_besselk_batch. */
#define BGK_ROUTE_HYBRID 0   /* refined_log_bessel (kernels.py:296-302): x < thr -> series */
#define BGK_ROUTE_SERIES 1   /* temme_series_log (kernels.py:273-293) for every element   */
#define BGK_ROUTE_INTEGRAL 2 /* fixed_window_log_pair (kernels.py:212-216), no guard      */

/* path[] codes (PathTaken, besselk.py:23-25) */
#define BGK_PATH_SERIES 0
#define BGK_PATH_INTEGRAL 1

/* Matern output layouts */
#define BGK_LAYOUT_ROW_MAJOR 0 /* element (i,j) at out[i*ld + j] (numpy C order) */
#define BGK_LAYOUT_COL_MAJOR 1 /* element (i,j) at out[i + j*ld] (SPEC.md:283 tiles) */

/* ln K_nu(x) over n elements.
 * Replaces kernels.refined_log_bessel (kernels.py:297) / temme_series_log
 * (kernels.py:274) / fixed_window_log_pair (kernels.py:213) as called by
 * besselk.bessel_k (besselk.py:158-165), bessel_k_series (:104-110),
 * fixed_window_log_bessel_k (:134-146).
 *   log_k  required, ln K
 *   k      optional (NULL), exp(ln K) with overflow -> +inf (besselk.py:80-84)
 *   path   optional (NULL), BGK_PATH_* per element                       */
int bgk_besselk_batch(const double *x, const double *nu, int64_t n, const bgk_config *cfg,
                      int route, double *log_k, double *k, uint8_t *path, void *stream);

/* Temme starting sums (s0, s1, terms) with K_mu = s0, K_{mu+1} = (2/x) s1.
 * Replaces kernels.temme_sums (kernels.py:230-270) as called by
 * besselk.temme_pair (besselk.py:94-101).  terms may be NULL. */
/* One (x, nu): ln K into *log_k (a HOST pointer), synchronously on `stream`.  One
 * one-warp kernel launch with x and nu as kernel parameters; the result and a
 * sequence number come back through a per-thread, per-device mapped page-locked
 * slot that the host polls (no memcpy, no stream sync; a fault is still reported
 * through periodic cudaStreamQuery).  Same bits as bgk_besselk_batch.  Backs the
 * scalar drop-in API (besselk.py:94-165). */
int bgk_besselk_scalar(double x, double nu, const bgk_config *cfg, int route, double *log_k,
                       void *stream);

/* Introspection of the fast integral path's node windows (tests: the window table
 * must cover every node the reference keeps).  Per element: m = the anchor node
 * the kernel uses, [lo, hi] = the nodes it sums; m = -1 when the element does
 * not take the fast windowed path (series, reference path).  The _host variant
 * runs on the CPU with the host anchor (fp32 asinhf); the device variant runs
 * the kernel's own classify + fast fp32 anchor on device pointers. */
int bgk_besselk_windows_host(const double *x, const double *nu, int64_t n,
                             const bgk_config *cfg, int32_t *m, int32_t *lo, int32_t *hi);
int bgk_besselk_windows(const double *x, const double *nu, int64_t n, const bgk_config *cfg,
                        int32_t *m, int32_t *lo, int32_t *hi, void *stream);

int bgk_temme_sums_batch(const double *x, const double *mu, int64_t n, const bgk_config *cfg,
                         double *s0, double *s1, int64_t *terms, void *stream);

/* g(t) = log cosh(nu t) - x cosh t (order 0), g' (order 1), g'' (order 2).
 * Replaces kernels.log_integrand / _d1 / _d2 (kernels.py:52-72). */
int bgk_log_integrand_batch(const double *t, const double *x, const double *nu, int64_t n,
                            int order, double *out, void *stream);

/* ---- Matern covariance ------------------------------------------------------------ */

#define BGK_MATERN_MAX_NODES 1024
#define BGK_MATERN_MAX_BUCKETS 1024

/* Per-call plan: the restated caller's per-nu work (kernels.py:343-345,
 * SPEC.md:306-332) hoisted out of the entry loop -- node tables
 * c_m = cosh(t_m), a_m = log_cosh(nu t_m), the Matern log-prefactor, the
 * nu-only Temme constants and the u-bucket -> (anchor node, node window)
 * lookup table the kernel uses instead of a 41-node argmax scan.
 * Caller-allocated POD (sizeof == bgk_matern_plan_size()); fill it with one of
 * the bgk_matern_plan_init* calls; it is passed to kernels by value. */
typedef struct bgk_matern_plan {
  int32_t abi;      /* BGK_ABI_VERSION */
  int32_t nnodes;   /* bins + 1 */
  int32_t nbuckets; /* entries of lut[] */
  int32_t key_base; /* u-bucket key of lut[0]: the double's bits >> (32 + key_shift) */
  int32_t fast;     /* 1: lut path; 0: general argmax-scan path */
  int32_t m_steps;  /* Temme: floor(nu + 0.5) */
  int32_t anchor_min, anchor_max; /* range of anchor nodes used by lut[] */
  int32_t key_shift;     /* 15: 32 buckets per octave, 16: 16 per octave */
  int32_t nosub_buckets; /* lut[0, nosub_buckets): every window term e^(aw_k - u c_k) has
                            |exponent| < 690, so the kernel may sum it unanchored */
  int32_t pow_mode;      /* 0: u^nu as exp(nu ln u); else 2 nu = 2k + half is a small integer:
                            pow_mode = 1 + 2k + half, u^nu = u^k (sqrt u)^half */
  int32_t pad_;
  double pow_pref;       /* exp(log_prefactor) h, normal (pow_mode != 0 only) */
  double sigma_sq, beta, nu, log_prefactor, h, small_x_threshold, eps_machine;
  int64_t series_cap;
  double mu, gam1, gam2, fact, gamma_1p_mu, gamma_1m_mu; /* Temme, nu-only */
  double c[BGK_MATERN_MAX_NODES];  /* cosh(t_m)                          */
  double a[BGK_MATERN_MAX_NODES];  /* log_cosh(nu t_m)                   */
  double aw[BGK_MATERN_MAX_NODES]; /* a_m + log(trapezoid weight w_m)    */
  uint32_t lut[BGK_MATERN_MAX_BUCKETS]; /* anchor | lo << 10 | hi << 20 */
} bgk_matern_plan;

size_t bgk_matern_plan_size(void);

/* Plan from Matern parameters + QuadratureConfig (the SPEC covariance API):
 * tables built like the restated caller, log_prefactor =
 * log(sigma_sq) - (nu - 1) ln2 - lgamma(nu). */
int bgk_matern_plan_init(bgk_matern_plan *plan, double sigma_sq, double beta, double nu,
                         const bgk_config *cfg);

/* Plan from explicit tables, i.e. the exact argument list of
 * kernels.matern_tile (kernels.py:339-340): sigma_sq, beta, nu,
 * log_prefactor, c_nodes, a_nodes (nnodes each), h, threshold, eps, cap. */
int bgk_matern_plan_init_tables(bgk_matern_plan *plan, double sigma_sq, double beta, double nu,
                                double log_prefactor, const double *c_nodes,
                                const double *a_nodes, int64_t nnodes, double h,
                                double small_x_threshold, double eps_machine,
                                int64_t series_cap);

/* One tile: out(i,j) = Matern(|(rx_i,ry_i) - (cx_j,cy_j)|) for i < m, j < n.
 * Replaces kernels.matern_tile (kernels.py:339-381); layout BGK_LAYOUT_*. */
int bgk_matern_tile(const bgk_matern_plan *plan, const double *rx, const double *ry, int64_t m,
                    const double *cx, const double *cy, int64_t n, double *out, int64_t ld,
                    int layout, void *stream);

/* Rows [row_begin, row_end) of the full N x N covariance matrix of the
 * locations (lx, ly), i.e. one row-block shard of SPEC generate_covariance
 * (SPEC.md:324-332).  Row row_begin is stored first: element (i, j) of the
 * full matrix lands at out[(i-row_begin)*ld + j] (ROW_MAJOR) or
 * out[(i-row_begin) + j*ld] (COL_MAJOR, i.e. the column block).  Inside the
 * diagonal block [row_begin,row_end)^2 each entry pair (i,j)/(j,i) is
 * computed once and stored twice; entries are symmetric bitwise anyway. */
int bgk_matern_covariance(const bgk_matern_plan *plan, const double *lx, const double *ly,
                          int64_t N, int64_t row_begin, int64_t row_end, double *out, int64_t ld,
                          int layout, void *stream);

/* Packed lower-triangle tiles (the M200 layout): tile (p, q), q <= p, of size
 * ts x ts has linear index l = p(p+1)/2 + q and is stored column-major at
 * out + (l - tile_begin) * ts * ts; diagonal tiles are stored complete; entries
 * of edge tiles beyond N are left untouched.  Produces l in
 * [tile_begin, tile_end) -- the area-balanced shard of one GPU. */
int bgk_matern_lower_tiles(const bgk_matern_plan *plan, const double *lx, const double *ly,
                           int64_t N, int64_t tile_size, int64_t tile_begin, int64_t tile_end,
                           double *out, void *stream);

/* ---- accuracy audit (oracle.py, kernels.py:306-335) ------------------- */

#define BGK_AUDIT_REFINED 0       /* refined_log10_grid (kernels.py:306-318)       */
#define BGK_AUDIT_PURE_INTEGRAL 1 /* pure_integral_log10_grid (kernels.py:321-329) */
#define BGK_AUDIT_ORACLE 2        /* dynamic-window oracle (oracle.py:92-160)      */

/* log K over the nnu x nx (nu, x) grid (row-major out[i*nx + j]), one CTA per
 * point, reference-faithful arithmetic: window search by FINDRANGE / FINDZERO
 * (Newton + bisection, tol 1e-12) for the oracle with `bins` intervals
 * (cfg->bins for the other methods), the series below cfg->small_x_threshold
 * (not for PURE_INTEGRAL).  base10: 1 -> double-double base-10 assembly
 * (kernels.py:97-109), 0 -> natural log.  Failed window searches give NaN. */
int bgk_log_grid(const double *nus, int64_t nnu, const double *xs, int64_t nx,
                 const bgk_config *cfg, int method, int64_t bins, int base10, double *out,
                 void *stream);

/* ---- location preprocessing --------------------------------------- */

/* normalize_locations: out = clip((c - min) / max(extent_x, extent_y), 0, 1) per
 * axis; `bounds` is 4 x uint64 of device scratch (order-mapped min x, min y,
 * max x, max y).  Bitwise equal to the host definition. */
int bgk_normalize_locations(const double *x, const double *y, int64_t n, unsigned long long *bounds,
                            double *out_x, double *out_y, void *stream);

/* Morton keys for morton_order: q = floor(c (2^bits - 1)) per axis, bits
 * interleaved with x in the low bit.  Sort the keys stably for the permutation. */
int bgk_morton_keys(const double *x, const double *y, int64_t n, int bits_per_axis,
                    uint64_t *keys, void *stream);

/* ---- multi-GPU: fused compute + NVLink peer stores ---------------------------------- */

#define BGK_MACRO_TILE 64
#define BGK_MAX_PEERS 32
#define BGK_IPC_HANDLE_BYTES 64

/* Full N x N matrix over G owners (one GPU each).  Lower 64x64 macro tiles
 * l in [tile_begin, tile_end) of the WHOLE matrix (l = p(p+1)/2 + q, q <= p,
 * T = ceil(N/64) macro rows) are each computed once: tile (p, q) is stored at its
 * row owner and, for p != q, its transpose at its column owner.  Owner h holds
 * macro rows [macro_row_start[h], macro_row_start[h+1]) -- matrix rows
 * [64 start[h], min(N, 64 start[h+1])) -- row-major with ld = N at bases[h], a
 * local pointer or a peer pointer mapped with bgk_ipc_open (NVLink P2P stores).
 * macro_row_start[0] = 0, macro_row_start[G] = T, non-decreasing.  Equal ranges
 * of [0, T(T+1)/2) over the ranks are equal work: every rank computes N^2/(2G)
 * entries instead of the (1/G - 1/(2G^2)) N^2 of the no-communication row blocks.
 * The matrix is complete once every rank's launch has finished (barrier). */
int bgk_matern_covariance_peer(const bgk_matern_plan *plan, const double *lx, const double *ly,
                               int64_t N, int G, const int64_t *macro_row_start,
                               double *const *bases, int64_t tile_begin, int64_t tile_end,
                               void *stream);

/* The same matrix with an owner-computes assignment ("cyclic half band"): owner
 * `rank` computes, for each of its macro rows p, the tiles (p, q) with
 * q = p - d (mod T), d = 0 .. floor(T/2) (d = T/2, T even, only for p < T/2).
 * Every unordered tile pair is computed exactly once across the ranks and the
 * work is balanced for equal row blocks, as with bgk_matern_covariance_peer, but
 * every direct store lands in the rank's own block: only the mirrors cross
 * NVLink, half the peer traffic of the lower-triangle ranges.  Upper tiles
 * (q > p) are computed directly; entries are pure functions of the location
 * pair, so the matrix is bitwise the same. */
int bgk_matern_covariance_peer_band(const bgk_matern_plan *plan, const double *lx,
                                    const double *ly, int64_t N, int G,
                                    const int64_t *macro_row_start, double *const *bases,
                                    int rank, void *stream);

/* CUDA IPC for one-process-per-GPU peer mapping.  export: handle (64 bytes) of the
 * allocation holding ptr and ptr's offset in it.  open: map a peer's allocation on
 * the current device and return base + offset.  close: unmap (pass the pointer
 * open returned and the same offset). */
int bgk_ipc_export(const void *ptr, void *handle, uint64_t *offset);
int bgk_ipc_open(const void *handle, uint64_t offset, void **ptr);
int bgk_ipc_close(void *ptr, uint64_t offset);
/* *can_access = cudaDeviceCanAccessPeer(current device, peer) (1 for the same device):
 * checked before any peer mapping. */
int bgk_can_access_peer(int peer_device, int *can_access);
/* cudaDeviceEnablePeerAccess(peer) on the current device; already-enabled is OK. */
int bgk_enable_peer_access(int peer_device);

/* ---- misc ------------------------------------------------------------------------- */
const char *bgk_last_error(void);
int bgk_abi_version(void);
/* FP64-pipe peak probe: `blocks` x 256 threads, each running 8 independent DFMA
 * chains of 16*iters steps; *dfma_per_launch receives the DFMA count (one
 * FP64-pipe op each).  Time it with events on `stream` to get the measured FP64
 * roofline denominator.  `scratch` must hold blocks*256 doubles. */
int bgk_fp64_probe(double *scratch, int64_t blocks, int iters, void *stream,
                   double *dfma_per_launch);

/* ---- host-side helpers of the host-buffer covariance path ----------------------------
 * The full N x N matrix into a host array moves only the lower triangle over PCIe
 * (rows [b0, b1) x cols [0, b1) per row block) and mirrors it on the host. */

/* Async strided device -> host copy (cudaMemcpy2DAsync): `rows` rows of
 * `width_bytes` bytes from src (pitch spitch bytes) to dst (pitch dpitch bytes);
 * dst should be page-locked for the copy to be asynchronous and at full speed. */
int bgk_memcpy2d_d2h(void *dst, int64_t dpitch, const void *src, int64_t spitch,
                     int64_t width_bytes, int64_t rows, void *stream);

/* Host mirror of a row block of a symmetric row-major matrix (leading dimension
 * ld, in doubles): out[j*ld + i] = out[i*ld + j] for i in [r0, r1), j in [0, r0),
 * i.e. rows [0, r0) x cols [r0, r1) from the lower block, with `nthreads` host
 * threads (64 x 64 tiles through a thread-local buffer: contiguous reads and
 * writes).  Host memory only; no CUDA. */
int bgk_host_mirror_lower(double *out, int64_t ld, int64_t r0, int64_t r1, int nthreads);

/* General form: out[j*ld + i] = out[i*ld + j] for i in [r0, r1), j in [c0, c1)
 * (the two index ranges must not overlap); bgk_host_mirror_lower is c0 = 0,
 * c1 = r0. */
int bgk_host_mirror_block(double *out, int64_t ld, int64_t r0, int64_t r1, int64_t c0,
                          int64_t c1, int nthreads);

/* Host memcpy with `nthreads` threads and non-temporal stores (no read-for-ownership
 * of the destination): the pageable -> page-locked staging copy of host-array
 * BesselK batches.  Host memory only; no CUDA. */
int bgk_host_copy(void *dst, const void *src, int64_t bytes, int nthreads);

/* Test hook for the Matern kernel's branch-free sqrt: fast[i] = the kernel's
 * sqrt_rn_fast(x[i]) where it claims its range (NaN elsewhere), ref[i] =
 * __dsqrt_rn(x[i]).  Device pointers. */
int bgk_sqrt_rn_check(const double *x, int64_t n, double *fast, double *ref, void *stream);

/* Launch geometry of the Matern kernel for this plan on the current device (test /
 * profiling hook): resident CTAs per SM, dynamic + static shared bytes per CTA,
 * registers per thread.  Sets the kernel's shared-memory opt-in like a launch. */
int bgk_matern_kernel_info(const bgk_matern_plan *plan, int *ctas_per_sm, int *smem_bytes,
                           int *regs);

/* Profiling hook: per-barrier work / wait cycles of the Matern kernel's task loop
 * summed over all warps since the last reset (12 values: work, wait for the
 * barriers after classify, in the scan, after the scan, after the scatter, after
 * the compute phase, after the stores).  Only libraries built with
 * -DBGK_MATERN_PROFILE=1 (tools/matern_phases.py); else BGK_ERR_UNSUPPORTED. */
int bgk_matern_phase_profile(double *out12, int reset);

/* Number of kernel launches issued by this library since load (for bench.py's
 * gpu_launches accounting). */
int64_t bgk_launch_count(void);

/* Test hook for the per-device caches (shared-memory opt-ins, uploaded BesselK
 * tables, task counters): they are keyed by (current device + alias).  Setting a
 * new alias makes the next launches see a device the library has not configured
 * yet, so a one-GPU box exercises the cache-miss path a second GPU would take.
 * Returns the previous alias.  Not for production use. */
int bgk_debug_set_device_alias(int alias);

#ifdef __cplusplus
}
#endif

#endif /* BESSELGP_B200_H */
