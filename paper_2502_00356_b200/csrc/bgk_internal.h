// bgk_internal.h -- declarations shared between the CUDA launchers and the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/besselgp_b200.h"

// error/launch bookkeeping (bgk_capi.cpp)
void bgk_set_error(const char *fmt, ...);
int bgk_check_launch(const char *what);
void bgk_note_launch();

// Per-device state.  Shared-memory opt-ins, uploaded tables and task counters are
// per CUDA device: every cache is keyed by bgk_device_key() (the current device,
// plus a test-only alias offset set by bgk_debug_set_device_alias so a one-GPU
// box can exercise the cache-miss path), and the opt-in is re-checked per device.
int bgk_device_key(int *real_device);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) once per (kernel, device,
// size), under a mutex, return code checked.  0 or BGK_ERR_CUDA.
int bgk_ensure_smem_optin(const void *kernel, const char *name, int bytes);

// launchers
int bgk_launch_besselk(const double *x, const double *nu, int64_t n, const bgk_config *cfg,
                       int route, double *log_k, double *k, uint8_t *path, cudaStream_t stream);
int bgk_launch_temme_sums(const double *x, const double *mu, int64_t n, const bgk_config *cfg,
                          double *s0, double *s1, int64_t *terms, cudaStream_t stream);
int bgk_launch_log_integrand(const double *t, const double *x, const double *nu, int64_t n,
                             int order, double *out, cudaStream_t stream);

// Matern launch descriptor (one of three task decoders)
enum BgkMaternMode { BGK_MODE_TILE = 0, BGK_MODE_COV = 1, BGK_MODE_LOWER = 2, BGK_MODE_PEER = 3 };

#define BGK_MAX_PEERS 32

struct BgkMaternArgs {
  const double *rx, *ry;  // row locations (COV/LOWER: all N locations)
  const double *cx, *cy;  // column locations
  double *out;
  long long m, n;         // TILE: rows/cols; COV/LOWER: N, N
  long long ld;           // TILE/COV leading dimension
  int layout;             // BGK_LAYOUT_*
  long long row0, row1;   // COV shard
  long long ts;           // LOWER storage tile size
  long long tile0, tile1; // LOWER tile range
  long long ntasks;
  unsigned long long *task_counter;  // persistent variant only (BGK_MATERN_PERSISTENT)
  double inv_beta;        // 1 / beta, computed once on the host (bgk_launch_matern)
  double lp_h;            // log_prefactor + ln h (absolute-form epilogue)
  // COV decode helpers (filled by bgk_launch_matern)
  long long nTr, nL, nR, nD;
  // LOWER decode helpers (filled by bgk_launch_matern)
  long long sub, subc;    // sub-tiles per storage tile: rows, cols
  // PEER: G row-block owners; owner h holds macro rows [pstart[h], pstart[h+1])
  // (rows [64 pstart[h], min(N, 64 pstart[h+1]))) at bases[h], row-major, ld = N.
  int G;
  int band;               // 0: tiles [tile0, tile1) of the lower triangle; 1: cyclic half
                          // band of macro rows [tile0, tile1) (= brow0 ..), bW tiles per row
  long long brow0, bW, bT;
  long long pstart[BGK_MAX_PEERS + 1];
  double *bases[BGK_MAX_PEERS];
};

int bgk_launch_matern(const bgk_matern_plan *plan, BgkMaternArgs &args, int mode,
                      cudaStream_t stream);
