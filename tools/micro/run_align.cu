// Microbenchmark: does sector alignment of the destination runs matter for a radix-style
// scatter? 19.86M (key, value) pairs, 4096-item tiles, 512 streams, runs of R items; stream
// s starts at element s*per + skew (per a multiple of 8: skew 0 -> every run of 8 is one full
// 32-byte sector; skew 4 -> every run straddles two sectors).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_runs(const unsigned* __restrict__ ki, const unsigned* __restrict__ vi, unsigned* ko, unsigned* vo,
                       unsigned n, int R, int D, unsigned per, unsigned skew) {
  const unsigned t = blockIdx.x, tb = t * 4096u;
  const int runs_per_tile = 4096 / R;
  for (int k = threadIdx.x; k < 4096; k += blockDim.x) {
    const unsigned e = tb + k;
    if (e >= n) break;
    const int r = k / R;
    const int s = (r + (int)t * 7) % D;
    const unsigned runs_before = (unsigned)t * (unsigned)(runs_per_tile / D > 0 ? runs_per_tile / D : 1) + (unsigned)(r / D);
    const unsigned pos = (unsigned)s * per + skew + (runs_before * (unsigned)R + (unsigned)(k % R)) % (per - 8);
    ko[pos] = ki[e];
    vo[pos] = vi[e];
  }
}
int main() {
  const unsigned n = 19855651u;
  unsigned *ki, *vi, *ko, *vo;
  cudaMalloc(&ki, n * 4ull); cudaMalloc(&vi, n * 4ull); cudaMalloc(&ko, n * 4ull + 64 * 1024 * 1024); cudaMalloc(&vo, n * 4ull + 64 * 1024 * 1024);
  cudaMemset(ki, 1, n * 4ull); cudaMemset(vi, 2, n * 4ull);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto time = [&](auto f) { for (int i = 0; i < 3; ++i) f(); cudaEventRecord(a); for (int i = 0; i < 10; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms / 10 * 1e3; };
  const unsigned tiles = (n + 4095) / 4096;
  const int D = 512;
  for (int R : {4, 8, 16, 32}) for (unsigned skew : {0u, 2u, 4u}) {
    const unsigned per = ((n + D - 1) / D + 64 + 7) / 8 * 8;
    float t = time([&] { k_runs<<<tiles, 256>>>(ki, vi, ko, vo, n, R, D, per, skew); });
    printf("streams %4d run %4d skew %u %8.1f us  %6.2f TB/s\n", D, R, skew, t, 16.0 * n / t / 1e6);
  }
  return 0;
}
