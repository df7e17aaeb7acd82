// Microbenchmark: per-warp cycles of the k_search core-scan loop over items
// staged in shared memory (SoA), for several warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_1711_07999_b200/csrc tools/micro/scan.cu -o tools/micro/scan
#include <cstdio>
#include <cuda_runtime.h>

#include "wt_kernels.cuh"

using namespace wt;

__global__ void k_scan(int nitems, int spans, long long* cyc, int* sink) {
  __shared__ double sx[4][320], sy[4][320], sz[4][320];
  __shared__ int si[4][320];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = lane; e < 320; e += 32) {
    sx[warp][e] = 0.001 * e;
    sy[warp][e] = 0.002 * e;
    sz[warp][e] = 1.0 + 0.0001 * e;
    si[warp][e] = e;
  }
  __syncwarp();
  const BoxItems it{sx[warp], sy[warp], sz[warp], si[warp]};
  const double px = 0.01 * lane, py = 0.02, pz = 1.01;
  double bx = INFINITY;
  int bi = -1;
  long long t0 = clock64();
  for (int sp = 0; sp < spans; ++sp) {
    const int e0 = (lane + 7 * sp) % 256, e1 = e0 + nitems / spans;
    scan_items_smem(it, e0, e1, px, py, pz, 1e9, bx, bi);
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 4 + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = bi;
}

__global__ void k_fp64chain(long long* cyc, double* sink) {
  double a = threadIdx.x * 1e-3, b = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) {
    a = __dadd_rn(a, b);
    b = __dmul_rn(b, 1.0000001);
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + (threadIdx.x >> 5)] = (t1 - t0) / 256;
  sink[threadIdx.x] = a + b;
}

int main() {
  long long* dc;
  int* sink;
  double* dsink;
  cudaMalloc(&dc, sizeof(long long) * 4096);
  cudaMalloc(&sink, sizeof(int) * 65536);
  cudaMalloc(&dsink, sizeof(double) * 4096);
  long long c[4096];
  for (int warps_per_cta : {1, 4})
    for (int ctas : {1, 148, 444}) {
      k_scan<<<ctas, 32 * warps_per_cta>>>(30, 5, dc, sink);
      k_scan<<<ctas, 32 * warps_per_cta>>>(30, 5, dc, sink);
      cudaMemcpy(c, dc, sizeof(long long) * ctas * 4, cudaMemcpyDeviceToHost);
      long long mx = 0, sum = 0;
      int n = 0;
      for (int b = 0; b < ctas; ++b)
        for (int w = 0; w < warps_per_cta; ++w) {
          mx = c[b * 4 + w] > mx ? c[b * 4 + w] : mx;
          sum += c[b * 4 + w];
          ++n;
        }
      printf("scan 30 items / 5 spans: %d CTAs x %d warps: mean %lld max %lld cycles\n", ctas, warps_per_cta,
             sum / n, mx);
    }
  for (int warps : {1, 4, 16, 32}) {
    k_fp64chain<<<1, 32 * warps>>>(dc, dsink);
    cudaMemcpy(c, dc, sizeof(long long) * warps, cudaMemcpyDeviceToHost);
    printf("dependent dadd+dmul pair per step, %d warps on one SM: %lld cycles\n", warps, c[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
