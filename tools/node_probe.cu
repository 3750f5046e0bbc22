// node_probe.cu -- microbenchmark of the Matern node-loop body variants on one GPU
// (not product code).  Each thread sums R passes over a 41-node window for two u
// values (the ILP-2 pair-group loop), reading the node table and the replicated
// 64 x 16 exp table from shared memory exactly like bgk_matern.cu's nodes_run2.
//   V1  current: y = fma(-u, c, aw); tt = fma(y, 64/ln2, magic); nd = I2F(lo tt);
//       r = fma(nd, -ln2/64, y); poly4(r); acc = fma(T, p, acc)       (8 FP64 + 1 cvt)
//   V2  prescaled tables: z = fma(-u, c', aw') = y 64/ln2; n = F2I.rn(z); nd = I2F(n);
//       r' = z - nd (exact); poly4'(r'); acc                            (7 FP64 + 2 cvt)
//   V3  V1 with a degree-3 polynomial                                     (7 FP64 + 1 cvt)
//   V4  V2 with tt = z + magic (DADD) instead of F2I                      (8 FP64 + 1 cvt)
//   DF  8 independent DFMA chains (the FP64 peak), I2 / F2: conversion-only loops.
// Prints lane-node-evaluations per second, per-SM per-clock rates.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ab/node_probe tools/node_probe.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

constexpr int kThreads = 256, kNodes = 41;
__constant__ double kC[12];
__constant__ double2 kTab[kNodes + 3];  // V5: the node table in constant memory (uniform index)

__device__ __forceinline__ double tab_exp(const double *g, unsigned lb, int n) {
  const unsigned off = (((unsigned)n & 63u) * 128u) + lb;
  const int2 v = *reinterpret_cast<const int2 *>(reinterpret_cast<const char *>(g) + off);
  return __hiloint2double(v.y + (n << 14), v.x);
}

template <int V>
__device__ __forceinline__ double node(double nu_, double2 t, const double *g, unsigned lb) {
  if (V == 1 || V == 3 || V == 5) {
    const double y = fma(nu_, t.x, t.y);
    const double tt = fma(y, kC[0], kC[3]);
    const int n = __double2loint(tt);
    const double nd = __int2double_rn(n);
    const double r = fma(nd, -kC[1], y);
    double q;
    if (V == 1) {
      q = fma(r, kC[8], kC[7]);
      q = fma(q, r, kC[6]);
    } else {
      q = fma(r, kC[7], kC[6]);
    }
    q = fma(q, r, kC[5]);
    const double p = fma(q, r, kC[4]);
    return tab_exp(g, lb, n) * p;  // (the caller's fma folds this)
  } else {
    const double z = fma(nu_, t.x, t.y);
    int n;
    double nd;
    if (V == 2) {
      n = __double2int_rn(z);
      nd = __int2double_rn(n);
    } else {
      const double tt = z + kC[3];
      n = __double2loint(tt);
      nd = __int2double_rn(n);
    }
    const double r = z - nd;
    double q = fma(r, kC[8], kC[7]);
    q = fma(q, r, kC[6]);
    q = fma(q, r, kC[5]);
    const double p = fma(q, r, kC[4]);
    return tab_exp(g, lb, n) * p;
  }
}

template <int V, int E, int K>
__global__ void __launch_bounds__(kThreads, 4) loop_kernel(const double2 *tab_g, double *out, int reps,
                                                          double u0base) {
  __shared__ __align__(16) double g[64 * 16];
  __shared__ __align__(16) double2 tab[kNodes + 3];
  for (int i = threadIdx.x; i < 64 * 16; i += kThreads) {
    const int j = i / 16;
    const double v = exp2(j / 64.0);
    g[i] = __hiloint2double(__double2hiint(v) - (j << 14), __double2loint(v));
  }
  for (int i = threadIdx.x; i < kNodes; i += kThreads) tab[i] = tab_g[i];
  __syncthreads();
  const unsigned lb = (threadIdx.x & 15) << 3;
  double nu[E], a[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    nu[e] = -(u0base + 1e-4 * threadIdx.x + 0.01 * e);
    a[e] = 0.0;
  }
#pragma unroll 1
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int k = 0; k + K - 1 < kNodes - 1; k += K) {
      double2 t[K];
#pragma unroll
      for (int q = 0; q < K; ++q) t[q] = V == 5 ? kTab[k + q] : tab[k + q];
#pragma unroll
      for (int q = 0; q < K; ++q)
#pragma unroll
        for (int e = 0; e < E; ++e) a[e] += node<V>(nu[e], t[q], g, lb);
    }
  }
  double s = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) s += a[e];
  if (s == 1234.5) out[threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = s;
}

__global__ void __launch_bounds__(256) dfma_kernel(double *out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
#pragma unroll 1
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c] = fma(a[c], 0.999999, 1e-7);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.6789) out[threadIdx.x] = s;
}

// conversions: 8 independent chains int -> double -> int (I2F.F64 + F2I.F64 per step)
__global__ void __launch_bounds__(256) cvt_kernel(double *out, int iters) {
  int a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
#pragma unroll 1
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c] = __double2int_rn(__int2double_rn(a[c]) * 1.0000001);
  int s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234567) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double hz = clk * 1e3;
  double hc[12] = {64 / 0.6931471805599453, 0.6931471805599453 / 64, 0, 0x1.8p52,
                   0x1.0000000000000p+0, 0x1.fffffffffb135p-1, 0x1.0000000005bedp-1,
                   0x1.55557e54f8e10p-3, 0x1.55553a001e26ap-5, 0, 0, 0};
  double2 ht[kNodes], hs[kNodes];
  for (int k = 0; k < kNodes; ++k) {
    const double t = k * 0.225, c = cosh(t), a = log(cosh(1.5 * t)) + (k == 0 || k == 40 ? -log(2.0) : 0);
    ht[k] = make_double2(c, a);
    hs[k] = make_double2(c * hc[0], a * hc[0]);
  }
  double2 *dt, *ds;
  double *out;
  cudaMalloc(&dt, sizeof(ht));
  cudaMalloc(&ds, sizeof(hs));
  cudaMalloc(&out, 1 << 20);
  cudaMemcpy(dt, ht, sizeof(ht), cudaMemcpyHostToDevice);
  cudaMemcpy(ds, hs, sizeof(hs), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(kTab, ht, sizeof(ht));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = nsm * 4, reps = 200;
  auto time_it = [&](auto launch) {
    launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5 * 1e-3;
  };
  struct Var { int v, e, k; const char *name; };
  const Var vars[] = {{1, 2, 2, "V1 E2 K2 (current loop)"}, {2, 2, 2, "V2 E2 K2 scaled F2I"},
                      {3, 2, 2, "V3 E2 K2 deg3"},          {4, 2, 2, "V4 E2 K2 scaled magic"},
                      {1, 1, 4, "V1 E1 K4"},               {1, 4, 1, "V1 E4 K1"},
                      {1, 2, 4, "V1 E2 K4"},               {1, 4, 2, "V1 E4 K2"},
                      {5, 2, 2, "V5 E2 K2 table in cmem"},  {5, 4, 2, "V5 E4 K2 table in cmem"}};
  for (const Var &V : vars) {
    double c2[12];
    for (int i = 0; i < 12; ++i) c2[i] = hc[i];
    if (V.v == 2 || V.v == 4) {
      const double s = 0.6931471805599453 / 64;
      c2[5] *= s; c2[6] *= s * s; c2[7] *= s * s * s; c2[8] *= s * s * s * s;
    }
    if (V.v == 3) { c2[7] = 0x1.5555555555555p-3; }
    cudaMemcpyToSymbol(kC, c2, sizeof(c2));
    const double2 *tb = (V.v == 2 || V.v == 4) ? ds : dt;
    const int steps = (kNodes - 1) / V.k * V.k;
    const double node_entries = (double)grid * kThreads * reps * V.e * steps;
    double s = time_it([&] {
#define L(v_, e_, k_) if (V.v == v_ && V.e == e_ && V.k == k_) loop_kernel<v_, e_, k_><<<grid, kThreads>>>(tb, out, reps, 1.0);
      L(1, 2, 2) L(2, 2, 2) L(3, 2, 2) L(4, 2, 2) L(1, 1, 4) L(1, 4, 1) L(1, 2, 4) L(1, 4, 2)
      L(5, 2, 2) L(5, 4, 2)
#undef L
    });
    printf("%-28s %.3f ms  %.2f G node-entries/s  %.2f node-entries/clk/SM\n", V.name, s * 1e3,
           node_entries / s * 1e-9, node_entries / s / hz / nsm);
  }
  {
    const int it = 2000;
    double s = time_it([&] { dfma_kernel<<<grid * 2, 256>>>(out, it); });
    const double ops = (double)grid * 2 * 256 * it * 128;
    printf("%-28s %.2f DFMA lane-ops/clk/SM\n", "DFMA peak", ops / s / hz / nsm);
    s = time_it([&] { cvt_kernel<<<grid * 2, 256>>>(out, it / 4); });
    const double cv = (double)grid * 2 * 256 * (it / 4) * 128;
    printf("%-28s %.2f (I2F + DMUL + F2I) lane-steps/clk/SM\n", "cvt chain", cv / s / hz / nsm);
  }
  cudaError_t err = cudaGetLastError();
  printf("sm clock attr %.0f MHz, %d SMs, err %s\n", hz * 1e-6, nsm, cudaGetErrorString(err));
  return 0;
}
