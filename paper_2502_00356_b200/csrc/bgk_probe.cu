// bgk_probe.cu -- FP64-pipe peak probe (the roofline denominator bench.py reports;
// MEASURED_PEAKS.json carries no FP64 figure).  Each thread runs 8 independent
// DFMA chains, so the pipe -- not latency -- bounds it; one DFMA = one FP64-pipe op.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bgk_internal.h"

namespace bgk {
__global__ void __launch_bounds__(256) fp64_probe_kernel(double *out, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.6789) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keep the work alive
}
}  // namespace bgk

extern "C" int bgk_fp64_probe(double *scratch, int64_t blocks, int iters, void *stream,
                              double *dfma_per_launch) {
  if (blocks < 1 || iters < 1 || !scratch) return BGK_ERR_INVALID;
  bgk::fp64_probe_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(scratch, iters, 0.5);
  bgk_note_launch();
  if (dfma_per_launch) *dfma_per_launch = (double)blocks * 256.0 * (double)iters * 16.0 * 8.0;
  return bgk_check_launch("fp64_probe_kernel");
}
