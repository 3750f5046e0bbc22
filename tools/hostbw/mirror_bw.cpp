// Host-side probe: memory bandwidth of a threaded blocked mirror (out[j][i] = out[i][j]
// for the strict lower triangle of a row-major N x N double matrix), and of a plain
// threaded memcpy, on the GPU box's host.  usage: mirror_bw N threads
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <sys/mman.h>

int main(int argc, char **argv) {
  const long N = argc > 1 ? atol(argv[1]) : 32768;
  const int T = argc > 2 ? atoi(argv[2]) : 16;
  const size_t bytes = (size_t)N * N * 8;
  double *a = (double *)aligned_alloc(4096, bytes);
  double *b = (double *)aligned_alloc(4096, bytes);
  // touch
  std::vector<std::thread> th;
  auto par = [&](auto f) { th.clear(); for (int t = 0; t < T; ++t) th.emplace_back(f, t); for (auto &x : th) x.join(); };
  par([&](int t) { for (long i = t; i < N; i += T) { for (long j = 0; j < N; ++j) a[i * N + j] = i + 1e-6 * j; memset(b + i * N, 0, N * 8); } });
  auto now = [] { return std::chrono::steady_clock::now(); };
  // memcpy bandwidth
  auto t0 = now();
  par([&](int t) { size_t chunk = bytes / T; memcpy((char *)b + t * chunk, (char *)a + t * chunk, chunk); });
  double dt = std::chrono::duration<double>(now() - t0).count();
  printf("memcpy %.2f GB in %.3f s: %.1f GB/s copied\n", bytes / 1e9, dt, bytes / 1e9 / dt);
  // blocked mirror: tiles (p, q), q < p, of 64 x 64; tile rows dealt round-robin
  const int B = 64;
  const long TB = (N + B - 1) / B;
  t0 = now();
  par([&](int t) {
    for (long p = t; p < TB; p += T)
      for (long q = 0; q < p; ++q) {
        alignas(64) double tile[64][64];
        const long ni = std::min(N, (p + 1) * B) - p * B;
        for (long i = 0; i < ni; ++i) memcpy(tile[i], a + (p * B + i) * N + q * B, B * 8);
        for (long j = 0; j < B; ++j) {
          double *dst = a + (q * B + j) * N + p * B;
          for (long i = 0; i < ni; ++i) dst[i] = tile[i][j];
        }
      }
  });
  dt = std::chrono::duration<double>(now() - t0).count();
  double moved = (double)N * (N - 1) / 2 * 8;
  printf("mirror N=%ld threads=%d: %.2f GB mirrored in %.3f s: %.1f GB/s (of mirrored data)\n", N, T, moved / 1e9, dt, moved / 1e9 / dt);
  // check
  long bad = 0;
  for (long i = 1; i < N; i += 997) for (long j = 0; j < i; j += 13) bad += a[j * N + i] != a[i * N + j];
  printf("check bad=%ld\n", bad);
  return 0;
}
