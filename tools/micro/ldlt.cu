// Microbenchmark: cycles of warp_ldlt_solve<N> (one warp, matrix in shared
// memory), first call (cold instruction cache) and repeated calls.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false --expt-relaxed-constexpr \
//        -I include -I paper_1711_07999_b200/csrc tools/micro/ldlt.cu -o tools/micro/ldlt
#include <cstdio>
#include <cuda_runtime.h>

#include "wt_kernels.cuh"

using namespace wt;

template <int N, bool PAIRS = false>
__global__ void k_ldlt(int L, long long* cyc, double* out) {
  __shared__ double A[32 * 33], b[32], x[32];
  __shared__ double scol[6][32];
  const int lane = threadIdx.x;
  for (int r = 0; r < 4; ++r) {
    for (int i = 0; i < L; ++i) A[i * (L + 1) + lane % (L + 1)] = 0.0;
    __syncwarp();
    if (lane < L) {
      for (int j = 0; j < L; ++j) A[lane * (L + 1) + j] = 1.0 / (1.0 + lane + j) + (lane == j ? L : 0.0);
      b[lane] = 1.0 + lane;
    }
    __syncwarp();
    const long long t0 = clock64();
    const int ok = PAIRS ? warp_ldlt_solve2<N>(L, L + 1, A, b, x, scol) : warp_ldlt_solve<N>(L, L + 1, A, b, x, scol);
    __syncwarp();
    const long long t1 = clock64();
    if (lane == 0) cyc[r] = t1 - t0;
    if (ok && lane < L) out[lane] = x[lane];
  }
}

template <int N, bool PAIRS = false>
void run(int L) {
  long long* dc;
  double* dout;
  cudaMalloc(&dc, sizeof(long long) * 4);
  cudaMalloc(&dout, sizeof(double) * 32);
  long long c[4];
  for (int rep = 0; rep < 2; ++rep) {
    k_ldlt<N, PAIRS><<<1, 32>>>(L, dc, dout);
    cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    double xo[32];
    cudaMemcpy(xo, dout, sizeof(xo), cudaMemcpyDeviceToHost);
    printf("N=%d L=%d %s launch %d: cycles %lld %lld %lld %lld  x0 %.17g x%d %.17g\n", N, L, PAIRS ? "pairs" : "single",
           rep, c[0], c[1], c[2], c[3], xo[0], L - 1, xo[L - 1]);
  }
  cudaFree(dc);
  cudaFree(dout);
}

// block_ldlt_solve (the CTA-wide form): 256 threads, one barrier per pivot
__global__ void k_bldlt(int L, long long* cyc, double* out) {
  __shared__ double A[32 * 33], b[32], x[32];
  __shared__ unsigned short ea[600], eb[600];
  const int NT = L * (L + 1) / 2;
  for (int e = threadIdx.x; e < NT; e += blockDim.x) {
    int r = 0, rem = e;
    while (rem >= L - r) { rem -= L - r; ++r; }
    ea[e] = r;
    eb[e] = r + rem;
  }
  for (int r = 0; r < 4; ++r) {
    for (int e = threadIdx.x; e < L * (L + 1); e += blockDim.x) {
      const int i = e / (L + 1), j = e % (L + 1);
      A[e] = j < L ? 1.0 / (1.0 + i + j) + (i == j ? L : 0.0) : 0.0;
    }
    if (threadIdx.x < L) b[threadIdx.x] = 1.0 + threadIdx.x;
    __syncthreads();
    const long long t0 = clock64();
    const int ok = block_ldlt_solve(L, L + 1, A, b, x, ea, eb, NT);
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[r] = t1 - t0;
    if (ok && threadIdx.x < L) out[threadIdx.x] = x[threadIdx.x];
  }
}

void run_block(int L) {
  long long* dc;
  double* dout;
  cudaMalloc(&dc, sizeof(long long) * 4);
  cudaMalloc(&dout, sizeof(double) * 32);
  long long c[4];
  for (int rep = 0; rep < 2; ++rep) {
    k_bldlt<<<1, 256>>>(L, dc, dout);
    cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("block L=%d launch %d: cycles %lld %lld %lld %lld\n", L, rep, c[0], c[1], c[2], c[3]);
  }
  cudaFree(dc);
  cudaFree(dout);
}

// dependent-chain latencies (one warp): DFMA, double SHFL, __drcp_rn
__global__ void k_lat(long long* cyc, double* out) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.999;
  long long t0 = clock64();
  for (int i = 0; i < 64; ++i) a = __fma_rn(a, b, 1e-3);
  long long t1 = clock64();
  for (int i = 0; i < 64; ++i) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31);
  long long t2 = clock64();
  for (int i = 0; i < 64; ++i) a = __drcp_rn(a);
  long long t3 = clock64();
  for (int i = 0; i < 64; ++i) a = __dmul_rn(a, 0.999) + 1e-3;
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 64;
    cyc[1] = (t2 - t1) / 64;
    cyc[2] = (t3 - t2) / 64;
    cyc[3] = (t4 - t3) / 64;
  }
  out[threadIdx.x] = a;
}

int main() {
  {
    long long* dc;
    double* dout;
    cudaMalloc(&dc, sizeof(long long) * 4);
    cudaMalloc(&dout, sizeof(double) * 32);
    long long c[4];
    for (int rep = 0; rep < 2; ++rep) {
      k_lat<<<1, 32>>>(dc, dout);
      cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    }
    printf("latency cycles: dfma %lld shfl.f64 %lld drcp_rn %lld dmul+dadd %lld\n", c[0], c[1], c[2], c[3]);
  }
  run<8>(6);
  run<8, true>(6);
  run<20>(20);
  run<20, true>(20);
  run<20, true>(19);
  run<20>(19);
  run<32>(27);
  run<32, true>(27);
  run_block(20);
  run_block(27);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
