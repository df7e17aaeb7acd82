// Microbenchmark: global-load latency (pointer chase) and batched-load time
// on the B200 box, to calibrate the search kernel's staging phase.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

__global__ void chase(const int* next, int steps, long long* out, int* sink) {
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = next[p];
  long long t1 = clock64();
  out[0] = (t1 - t0) / steps;
  sink[0] = p;
}

__global__ void batched(const double4* items, int n, long long* out, float* sink) {
  long long t0 = clock64();
  float acc = 0;
  double4 r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int idx = (blockIdx.x * 2048 + k * 256 + threadIdx.x) % n;
    r[k] = items[idx];
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) acc += (float)(r[k].x + r[k].w);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 1234.5f) sink[0] = acc;
}

int main() {
  const int n = 1 << 20;  // 4 MB of ints
  std::vector<int> h(n);
  // random cyclic permutation with stride to defeat prefetch
  for (int i = 0; i < n; ++i) h[i] = (int)((i * 2654435761u + 12345) % n) & ~31;
  int* d; long long* o; int* s; double4* items; float* fs;
  cudaMalloc(&d, n * 4); cudaMalloc(&o, 8 * 1024); cudaMalloc(&s, 4); cudaMalloc(&items, 100000 * 32); cudaMalloc(&fs, 4);
  cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemset(items, 0, 100000 * 32);
  for (int rep = 0; rep < 3; ++rep) {
    chase<<<1, 1>>>(d, 20000, o, s);
    long long c; cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
    printf("chase (4 MB, L2-resident after rep 0): %lld cycles/load\n", c);
  }
  chase<<<1, 1>>>(d, 200, o, s);
  for (int rep = 0; rep < 3; ++rep) {
    batched<<<144, 256>>>(items, 100000, o, fs);
    std::vector<long long> c(144); cudaMemcpy(c.data(), o, 8 * 144, cudaMemcpyDeviceToHost);
    long long mx = 0, sum = 0; for (auto x : c) { mx = x > mx ? x : mx; sum += x; }
    printf("batched 8 x double4 per thread, 144 CTAs: avg %lld max %lld cycles\n", sum / 144, mx);
  }
  return 0;
}
