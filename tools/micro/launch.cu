// Microbenchmark: cost of a kernel boundary inside a CUDA graph (empty and
// tiny kernels, 148..1200 CTAs), and of a cooperative grid barrier.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void empty_k(int* p) { if (p && threadIdx.x == 1023) p[0] = 1; }
__global__ void touch_k(double* p, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0000001 + 1.0;
}
__global__ void coop_k(double* p, int n, int iters) {
  cg::grid_group g = cg::this_grid();
  for (int it = 0; it < iters; ++it) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = p[i] * 1.0000001 + 1.0;
    g.sync();
  }
}

int main() {
  cudaStream_t st; cudaStreamCreate(&st);
  double* p; cudaMalloc(&p, 1 << 24); cudaMemset(p, 0, 1 << 24);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int variant = 0; variant < 3; ++variant) {
    cudaGraph_t g; cudaGraphExec_t ex;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < 50; ++k) {
      if (variant == 0) empty_k<<<148, 256, 0, st>>>(nullptr);
      else if (variant == 1) touch_k<<<400, 256, 0, st>>>(p, 100000);
      else touch_k<<<1200, 256, 0, st>>>(p, 300000);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ex, g, 0);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ex, st);
    cudaEventRecord(a, st);
    for (int r = 0; r < 20; ++r) cudaGraphLaunch(ex, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("graph of 50 kernels (variant %d): %.2f us per kernel\n", variant, ms * 1000 / (20 * 50));
  }
  int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, coop_k, 256, 0);
  int n = 100000, iters = 50;
  void* args[] = {&p, &n, &iters};
  for (int w = 0; w < 2; ++w) cudaLaunchCooperativeKernel((void*)coop_k, 148, 256, args, 0, st);
  cudaEventRecord(a, st);
  for (int r = 0; r < 10; ++r) cudaLaunchCooperativeKernel((void*)coop_k, 148, 256, args, 0, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("cooperative kernel, 148 CTAs: %.2f us per grid.sync step (touch 100k + sync)\n", ms * 1000 / (10 * iters));
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
