// bgk_locations.cu -- location preprocessing on the device:
// SPEC normalize_locations and the Morton keys of
// morton_order.  Same arithmetic as the host definitions in
// covariance.py (correctly rounded subtract / divide, floor of c (2^bits - 1)),
// so device and host results are bitwise equal.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bgk_internal.h"

namespace bgk {

// order-preserving map of a double onto uint64 (for atomicMin / atomicMax)
__device__ __forceinline__ unsigned long long ord(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord(unsigned long long o) {
  const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double((long long)b);
}

// bounds[0..3] = ord(min x), ord(min y), ord(max x), ord(max y); caller pre-fills
// {~0, ~0, 0, 0}.
__global__ void bounds_kernel(const double *x, const double *y, long long n,
                              unsigned long long *bounds) {
  unsigned long long mnx = ~0ull, mny = ~0ull, mxx = 0, mxy = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long ox = ord(x[i]), oy = ord(y[i]);
    mnx = ox < mnx ? ox : mnx;
    mny = oy < mny ? oy : mny;
    mxx = ox > mxx ? ox : mxx;
    mxy = oy > mxy ? oy : mxy;
  }
  for (int o = 16; o; o >>= 1) {
    mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(bounds + 0, mnx);
    atomicMin(bounds + 1, mny);
    atomicMax(bounds + 2, mxx);
    atomicMax(bounds + 3, mxy);
  }
}

// (c - min) / ell with ell = max(extent_x, extent_y), clipped to [0, 1].
__global__ void normalize_kernel(const double *x, const double *y, long long n,
                                 const unsigned long long *bounds, double *ox, double *oy) {
  const double mnx = unord(bounds[0]), mny = unord(bounds[1]);
  const double ell = fmax(__dsub_rn(unord(bounds[2]), mnx), __dsub_rn(unord(bounds[3]), mny));
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    ox[i] = fmin(fmax(__ddiv_rn(__dsub_rn(x[i], mnx), ell), 0.0), 1.0);
    oy[i] = fmin(fmax(__ddiv_rn(__dsub_rn(y[i], mny), ell), 0.0), 1.0);
  }
}

__device__ __forceinline__ unsigned long long part1by1(unsigned long long v) {
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// key = interleave(q_x, q_y) with x in the low bit, q = floor(c (2^bits - 1)).
__global__ void morton_kernel(const double *x, const double *y, long long n, double scale,
                              unsigned long long *keys) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long qx = (unsigned long long)floor(__dmul_rn(x[i], scale));
    const unsigned long long qy = (unsigned long long)floor(__dmul_rn(y[i], scale));
    keys[i] = part1by1(qx) | (part1by1(qy) << 1);
  }
}

}  // namespace bgk

extern "C" int bgk_normalize_locations(const double *x, const double *y, int64_t n,
                                       unsigned long long *bounds, double *out_x, double *out_y,
                                       void *stream) {
  if (n <= 0 || !x || !y || !bounds || !out_x || !out_y) {
    bgk_set_error("bgk_normalize_locations: bad arguments");
    return BGK_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned long long init[4] = {~0ull, ~0ull, 0ull, 0ull};
  cudaError_t e = cudaMemcpyAsync(bounds, init, sizeof(init), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) {
    bgk_set_error("bgk_normalize_locations: %s", cudaGetErrorString(e));
    return BGK_ERR_CUDA;
  }
  const int grid = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
  bgk::bounds_kernel<<<grid, 256, 0, s>>>(x, y, n, bounds);
  bgk_note_launch();
  bgk::normalize_kernel<<<grid, 256, 0, s>>>(x, y, n, bounds, out_x, out_y);
  bgk_note_launch();
  return bgk_check_launch("normalize_kernel");
}

extern "C" int bgk_morton_keys(const double *x, const double *y, int64_t n, int bits_per_axis,
                               uint64_t *keys, void *stream) {
  if (n < 0 || bits_per_axis < 1 || bits_per_axis > 31 || (n > 0 && (!x || !y || !keys))) {
    bgk_set_error("bgk_morton_keys: bad arguments");
    return BGK_ERR_INVALID;
  }
  if (n == 0) return BGK_OK;
  const double scale = (double)((1u << bits_per_axis) - 1u);
  const int grid = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
  bgk::morton_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      x, y, n, scale, reinterpret_cast<unsigned long long *>(keys));
  bgk_note_launch();
  return bgk_check_launch("morton_kernel");
}
