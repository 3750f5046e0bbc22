// pipe_probe.cu -- FP64-pipe microbenchmarks on one GPU (not product code): how the
// DFMA issue rate depends on operand sources, instruction mix and occupancy.  Each
// thread runs 6 independent chains; per step every chain does one DFMA plus the
// listed extra work (all results feed the chains, so nothing is dead code).
//   P1 fma(a, c, c')                 constant operands (the roofline probe)
//   P3 fma(a, b, d)                  three register operands, b and d vary per step
//   M1 P3 + 1 integer op             (IMAD / LOP3)
//   M2 P3 + 1 LDS.64 (table gather, 16 copies, conflict-free)
//   M3 P3 + 1 I2F.F64
//   M4 the node-loop mix per 8 DFMA: 1 I2F, 1 LDS.64, 4 integer
// Occupancy: 16 warps/SMSP (8 CTAs x 256 / SM) or 8 warps/SMSP (4 CTAs, as the
// Matern kernel).  Latency: a single dependent chain.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ab/pipe_probe tools/pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kC = 6;  // independent chains per thread (fits 64 registers)
template <int P>
__global__ void __launch_bounds__(256, 4) probe(double *out, int iters, double s0, double s1) {
  __shared__ __align__(16) double tab[64 * 16];
  for (int i = threadIdx.x; i < 64 * 16; i += 256) tab[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double a[kC], b[kC], d[kC];
  int n[kC];
  for (int i = 0; i < kC; ++i) {
    a[i] = threadIdx.x + i;
    b[i] = s0 + i * 1e-9 + threadIdx.x * 1e-12;
    d[i] = s1 + i * 1e-9 + threadIdx.x * 1e-13;
    n[i] = threadIdx.x * 7 + i;
  }
  const unsigned lb = (threadIdx.x & 15) << 3;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        if (P == 1) a[c] = fma(a[c], 0.999999, 1e-7);
        if (P == 2) a[c] = fma(a[c], b[c], 1e-7);          // 2 register operands
        if (P >= 3 && P != 4) a[c] = fma(a[c], b[c], d[c]);  // 3 register operands
        if (P == 4) a[c] = fma(a[c], b[0], d[0]);           // 3, two shared (reuse cache)
        if (P == 11) n[c] = n[c] * 3 + 1;
        if (P == 12) {
          const unsigned off = ((unsigned)n[c] & 63u) * 128u + lb;
          const int2 v = *reinterpret_cast<const int2 *>(reinterpret_cast<const char *>(tab) + off);
          n[c] += v.x;
        }
        if (P == 13) a[c] += 0.0 * __int2double_rn(n[c]);  // (DADD folded? keep: FMA)
        if (P == 14 && (u & 7) == 0) {
          const double nd = __int2double_rn(n[c]);
          const unsigned off = ((unsigned)n[c] & 63u) * 128u + lb;
          const int2 v = *reinterpret_cast<const int2 *>(reinterpret_cast<const char *>(tab) + off);
          n[c] = (n[c] ^ v.y) + (v.x << 3) + 1;
          a[c] = fma(nd, 1e-30, a[c]);
        }
        if (P == 5 && c == 0) a[0] = fma(a[0], b[0], d[0]);
      }
    }
  }
  double s = 0;
  for (int i = 0; i < kC; ++i) s += a[i] + n[i] + b[i] + d[i];
  if (s == 12345.6789) out[threadIdx.x] = s;
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double hz = clk * 1e3;
  double *out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto launch) {
    launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 3 * 1e-3;
  };
  const int it = 2000;
  for (int occ : {4}) {
    const int grid = nsm * occ;
    const double dfma = (double)grid * 256 * it * 8 * kC;  // DFMA per launch
    auto rate = [&](double t, double extra) { return (dfma * extra) / t / hz / nsm; };
    double t;
    printf("-- %d CTAs x 256 threads per SM (%d warps per SMSP)\n", occ, occ * 2);
    t = run([&] { probe<1><<<grid, 256>>>(out, it, 0.999999, 1e-7); });
    printf("P1 fma(a, const, const)        %.2f DFMA lane-ops/clk/SM\n", rate(t, 1.0));
    t = run([&] { probe<2><<<grid, 256>>>(out, it, 0.999999, 1e-7); });
    printf("P2 fma(a, b, const)            %.2f\n", rate(t, 1.0));
    t = run([&] { probe<3><<<grid, 256>>>(out, it, 0.999999, 1e-7); });
    printf("P3 fma(a, b, d) registers      %.2f\n", rate(t, 1.0));
    t = run([&] { probe<4><<<grid, 256>>>(out, it, 0.999999, 1e-7); });
    printf("P4 fma(a, b0, d0) shared b, d  %.2f\n", rate(t, 1.0));
    t = run([&] { probe<11><<<grid, 256>>>(out, it, 0.999999, 1e-7); });
    printf("M1 P3 + 1 IMAD per DFMA        %.2f\n", rate(t, 1.0));
    t = run([&] { probe<12><<<grid, 256>>>(out, it, 0.999999, 1e-7); });
    printf("M2 P3 + LDS.64 + 3 int / DFMA  %.2f\n", rate(t, 1.0));
    t = run([&] { probe<14><<<grid, 256>>>(out, it, 0.999999, 1e-7); });
    printf("M4 per 8 DFMA: I2F LDS 4 int   %.2f (+1 DFMA per 8 counted)\n", rate(t, 9.0 / 8.0));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
