// Microbenchmark: how fast can B200 move 8-byte (key, value) items into D destination
// streams with runs of R items? (models one radix scatter pass of 19.86M pairs)
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
__global__ void k_copy(const unsigned* __restrict__ ki, const unsigned* __restrict__ vi, unsigned* ko, unsigned* vo, unsigned n) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) { ko[i] = ki[i]; vo[i] = vi[i]; }
}
// tile of 4096 items; item e of tile t belongs to run r = e / R (runs of R items); run r of
// tile t goes to stream s = r % D at position base[s] + (t * (4096/R/D) + r / D) * R + e % R
__global__ void k_runs(const unsigned* __restrict__ ki, const unsigned* __restrict__ vi, unsigned* ko, unsigned* vo,
                       unsigned n, int R, int D, unsigned per_stream) {
  const unsigned t = blockIdx.x, tb = t * 4096u;
  const int runs_per_tile = 4096 / R;
  for (int k = threadIdx.x; k < 4096; k += blockDim.x) {
    const unsigned e = tb + k;
    if (e >= n) break;
    const int r = k / R;
    // stream of this run: spread runs over streams with a per-tile rotation
    const int s = (r + (int)t * 7) % D;
    const unsigned runs_before = (unsigned)t * (unsigned)(runs_per_tile / D > 0 ? runs_per_tile / D : 1) + (unsigned)(r / D);
    const unsigned pos = (unsigned)s * per_stream + (runs_before * (unsigned)R + (unsigned)(k % R)) % per_stream;
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
  float c = time([&] { k_copy<<<148 * 8, 256>>>(ki, vi, ko, vo, n); });
  printf("copy               %8.1f us  %6.2f TB/s\n", c, 16.0 * n / c / 1e6);
  const unsigned tiles = (n + 4095) / 4096;
  for (int D : {16, 512}) for (int R : {4, 8, 16, 32, 128, 512}) {
    if (4096 / R < 1) continue;
    const unsigned per = (n + D - 1) / D;
    float t = time([&] { k_runs<<<tiles, 256>>>(ki, vi, ko, vo, n, R, D, per); });
    printf("streams %4d run %4d %8.1f us  %6.2f TB/s\n", D, R, t, 16.0 * n / t / 1e6);
  }
  return 0;
}
