// Microbenchmark of the pose kernel's serial tail pieces on one CTA:
// warp_ldlt_solve / block_ldlt_solve on a 20x20 SPD system, fp64 reciprocal
// and sincos latency, and fk_run on a 20-link chain. Prints cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_1711_07999_b200/csrc tools/micro/tail.cu -o tools/micro/tail
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

#include "wt_kernels.cuh"

using namespace wt;

// instrumented copy of warp_ldlt_solve: per-pivot cycle stamps
__device__ int warp_ldlt_timed(int L, int lda, double* A, const double* b, double* x, long long* tk) {
  const int lane = threadIdx.x & 31;
  const bool row = lane < L;
  double bi = row ? b[lane] : 0.0;
  for (int k = 0; k < L; ++k) {
    long long c0 = clock64();
    const double dk = A[k * lda + k];
    if (!(dk > 0.0)) return 0;
    const double inv = __drcp_rn(dk);
    const double zk = __shfl_sync(0xffffffffu, bi, k);
    const bool act = row && lane > k;
    const double lik = act ? A[lane * lda + k] * inv : 0.0;
    long long c1 = clock64();
#pragma unroll
    for (int h = 0; h < 32; h += 16) {
      if (k + 1 >= h + 16 || h >= L) continue;
      double cj[16], ri[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int j = h + t;
        cj[t] = A[j * lda + k];
        ri[t] = A[lane * lda + j];
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int j = h + t;
        if (act && j > k && j <= lane) A[lane * lda + j] = ri[t] - lik * cj[t];
      }
    }
    long long c2 = clock64();
    if (act) bi -= lik * zk;
    __syncwarp();
    if (act) A[lane * lda + k] = lik;
    __syncwarp();
    long long c3 = clock64();
    if (lane == 0 && k < 8) { tk[3 * k] = c1 - c0; tk[3 * k + 1] = c2 - c1; tk[3 * k + 2] = c3 - c2; }
  }
  return 1;
}

__global__ void k_timed(int L, const double* Ain, const double* bin, double* x, long long* tk) {
  __shared__ double A[33 * 33];
  __shared__ double b[32];
  const int lda = L | 1;
  for (int e = threadIdx.x; e < L * L; e += blockDim.x) A[(e / L) * lda + e % L] = Ain[e];
  for (int k = threadIdx.x; k < L; k += blockDim.x) b[k] = bin[k];
  __syncthreads();
  if (threadIdx.x < 32) warp_ldlt_timed(L, lda, A, b, x, tk);
}

__global__ void k_solve(int L, const double* Ain, const double* bin, double* x, long long* cyc, int variant) {
  __shared__ double A[33 * 33];
  __shared__ double b[32];
  __shared__ unsigned short ea[600], eb[600];
  const int lda = L | 1;
  for (int e = threadIdx.x; e < L * L; e += blockDim.x) A[(e / L) * lda + e % L] = Ain[e];
  for (int k = threadIdx.x; k < L; k += blockDim.x) b[k] = bin[k];
  const int NT = L * (L + 1) / 2;
  for (int e = threadIdx.x; e < NT; e += blockDim.x) {
    int r = 0, rem = e;
    while (rem >= L - r) {
      rem -= L - r;
      ++r;
    }
    ea[e] = r;
    eb[e] = r + rem;
  }
  __syncthreads();
  long long t0 = clock64();
  int ok = 0;
  if (variant == 0) {
    if (threadIdx.x < 32) ok = warp_ldlt_solve<20>(L, lda, A, b, x);
  } else {
    ok = block_ldlt_solve(L, lda, A, b, x, ea, eb, NT);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0, cyc[1] = ok;
}

__global__ void k_ops(double v, int n, long long* cyc, double* sink) {
  __shared__ double sm[64];
  sm[threadIdx.x] = v + threadIdx.x;
  __syncthreads();
  double r = v;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) r = __drcp_rn(r + 1.0);
  asm volatile("" : "+d"(r));
  long long t1 = clock64();
  double s = r, c;
  for (int i = 0; i < n; ++i) {
    sincos(s, &s, &c);
    s += c;
  }
  asm volatile("" : "+d"(s));
  long long t2 = clock64();
  double d = s;
  for (int i = 0; i < n; ++i) d = 1.0 / (d + 1.0);
  asm volatile("" : "+d"(d));
  long long t3 = clock64();
  double f = d;
  for (int i = 0; i < n; ++i) f = fma(f, 1.0000001, 0.5);
  asm volatile("" : "+d"(f));
  long long t4 = clock64();
  int idx = static_cast<int>(f) & 31;
  double g = 0;
  for (int i = 0; i < n; ++i) {
    g += sm[idx];
    idx = (static_cast<int>(g) + i) & 31;
  }
  asm volatile("" : "+d"(g));
  long long t5 = clock64();
  double h = g;
  for (int i = 0; i < n; ++i) h = __shfl_sync(0xffffffffu, h, (i + 1) & 31) + 1.0;
  asm volatile("" : "+d"(h));
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / n;
    cyc[1] = (t2 - t1) / n;
    cyc[2] = (t3 - t2) / n;
    cyc[3] = (t4 - t3) / n;
    cyc[4] = (t5 - t4) / n;
    cyc[5] = (t6 - t5) / n;
  }
  sink[threadIdx.x] = r + s + d + f + g + h;
}

__global__ void k_fkbench(DevModel m, DevState s, const double* theta, long long* cyc) {
  __shared__ FkTables t;
  fk_stage(m, t);
  __syncthreads();
  long long t0 = clock64();
  fk_run(m, s, theta, t);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  const int L = 20;
  std::vector<double> A(L * L), b(L);
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < L; ++j) A[i * L + j] = (i == j ? L + 1.0 : 0.0) + 1.0 / (1 + i + j);
  for (int i = 0; i < L; ++i) b[i] = i - 3.0;
  double *dA, *db, *dx, *sink;
  long long* dc;
  cudaMalloc(&dA, sizeof(double) * L * L);
  cudaMalloc(&db, sizeof(double) * L);
  cudaMalloc(&dx, sizeof(double) * 64);
  cudaMalloc(&sink, sizeof(double) * 256);
  cudaMalloc(&dc, sizeof(long long) * 8);
  cudaMemcpy(dA, A.data(), sizeof(double) * L * L, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), sizeof(double) * L, cudaMemcpyHostToDevice);
  long long c[8];
  for (int variant = 0; variant < 2; ++variant)
    for (int rep = 0; rep < 3; ++rep) {
      k_solve<<<1, 256>>>(L, dA, db, dx, dc, variant);
      cudaMemcpy(c, dc, sizeof(long long) * 2, cudaMemcpyDeviceToHost);
      std::vector<double> x(L);
      cudaMemcpy(x.data(), dx, sizeof(double) * L, cudaMemcpyDeviceToHost);
      double res = 0;
      for (int i = 0; i < L; ++i) {
        double r = -b[i];
        for (int j = 0; j < L; ++j) r += A[i * L + j] * x[j];
        res = fmax(res, fabs(r));
      }
      printf("%s solve L=%d: %lld cycles ok=%lld residual %.2e\n", variant ? "block" : "warp", L, c[0], c[1], res);
    }
  long long* dt;
  cudaMalloc(&dt, sizeof(long long) * 32);
  k_timed<<<1, 32>>>(L, dA, db, dx, dt);
  long long tk[24];
  cudaMemcpy(tk, dt, sizeof(long long) * 24, cudaMemcpyDeviceToHost);
  for (int k = 0; k < 8; ++k) printf("pivot %d: head %lld update %lld tail %lld\n", k, tk[3 * k], tk[3 * k + 1], tk[3 * k + 2]);
  k_ops<<<1, 32>>>(0.3, 64, dc, sink);
  cudaMemcpy(c, dc, sizeof(long long) * 6, cudaMemcpyDeviceToHost);
  printf("dependent-chain latency (cycles/op): drcp_rn %lld, sincos+add %lld, div %lld, dfma %lld, lds.64+dadd+cvt %lld, shfl.64+dadd %lld\n",
         c[0], c[1], c[2], c[3], c[4], c[5]);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
