// wt_exact.cu -- the geometry kernels whose rounding decides association:
// forward kinematics / link offsets (k_fk and the pose-solve tail,
// skeleton.cpp:56-108), skinning and vertex normals (skinmesh.cpp:60-139).
// This unit is compiled with -fmad=false: every product and sum rounds
// separately, in the reference's operation order, so given the same link
// offsets the posed vertices and fp64 normals are bitwise the reference's
// (device sin/cos of theta/2 may still differ from libm by an ulp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "wt_kernels.cuh"

namespace wt {

// wt_render.cu
void raster_launch(cudaStream_t st, int T, const double* vpos, const int* tri, double fx, double fy, double cx,
                   double cy, int W, int H, unsigned long long* zbits, int* owner);

// nseq: sequences of a batch (gridDim.y), see seq_state in wt_kernels.cuh
void launch_skin(cudaStream_t st, int grid, int nseq, int L, const DevModel& m, const DevState& s,
                 const double4* phi) {
  // a batch of 16+ sequences: several vertices per thread, so the grid is a
  // few waves of longer-lived CTAs instead of thousands of short ones
  // (C5: 110 -> 95 us per launch)
  const int vpt = std::max(1, std::min(4, nseq / 16));
  const int g = (grid + vpt - 1) / vpt;
  launch_pdl(nseq > 1 ? k_skin<true> : k_skin<false>, dim3(g, nseq), dim3(kVThreads), sizeof(double) * 8 * L, st,
             m, s, phi);
}

void launch_normals(cudaStream_t st, int grid, int nseq, const DevModel& m, const DevState& s, const DevIntr& in,
                    int do_bucket, int zero_acc, int compute) {
  // a batch of 16+ sequences: up to 8 vertices per thread (C5: 366 -> 311 us)
  const int vpt = std::max(1, std::min(8, nseq / 8));
  const int g = (grid + vpt - 1) / vpt;
  launch_pdl(nseq > 1 ? k_normals<true> : k_normals<false>, dim3(g, nseq), dim3(kVThreads), 0, st, m, s, in,
             do_bucket, zero_acc, compute);
}

void launch_fk(cudaStream_t st, int nseq, const DevModel& m, const DevState& s) {
  launch_pdl(nseq > 1 ? k_fk<true> : k_fk<false>, dim3(1, nseq), dim3(128), 0, st, m, s);
}

void launch_pose_solve(cudaStream_t st, int nseq, int L, const DevModel& m, const DevState& s, const PoseArgs& a) {
  launch_pdl(nseq > 1 ? k_pose_solve<true> : k_pose_solve<false>, dim3(1, nseq), dim3(256), pose_solve_smem_bytes(L), st, m, s, a);
}

}  // namespace wt

// ---- reconstruction error (metrics.cpp:110-142) -------------------------------------
// Exact: the visible set uses the bitwise normals / projection / z-buffer of
// the reference, and each visible vertex's distance is the square root of the
// minimum of the exact ((dx^2 + dy^2) + dz^2) over every valid observed point
// (a brute-force scan, tiled through shared memory).

namespace wt {

static __global__ void k_pack_pv(int V, const double4* pv, double* v3) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const double4 v = pv[i];
  v3[3 * i] = v.x;
  v3[3 * i + 1] = v.y;
  v3[3 * i + 2] = v.z;
}

static __global__ void k_recon_visible(DevModel m, const double4* pv, DevIntr in, const unsigned long long* zbits,
                                       const int* owner, int* vis_list, int* n_vis) {
  constexpr double kZTolerance = 1e-3;  // self-occlusion margin, metrics.cpp:115
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool vis = false;
  if (i < m.V) {
    const double4 v = pv[i];
    double nx, ny, nz;
    if (vertex_normal(m, pv, i, v, nx, ny, nz) && !(nx * v.x + ny * v.y + nz * v.z > 0.0) && v.z > 0.0) {
      const double ru = round(in.fx * v.x / v.z + in.cx), rv = round(in.fy * v.y / v.z + in.cy);
      if (ru >= 0.0 && rv >= 0.0 && ru < in.W && rv < in.H) {
        const size_t px = static_cast<size_t>(rv) * in.W + static_cast<size_t>(ru);
        // owner 0x7F7F7F7F: no triangle reached the pixel (raster.tri < 0)
        vis = owner[px] != 0x7F7F7F7F && !(v.z > __longlong_as_double(static_cast<long long>(zbits[px])) + kZTolerance);
      }
    }
  }
  const unsigned mk = __ballot_sync(0xffffffffu, vis);
  if (!mk) return;
  int base = 0;
  const int lane = threadIdx.x & 31;
  if (lane == __ffs(mk) - 1) base = atomicAdd(n_vis, __popc(mk));
  base = __shfl_sync(0xffffffffu, base, __ffs(mk) - 1);
  if (vis) vis_list[base + __popc(mk & ((1u << lane) - 1u))] = i;
}

static __global__ void k_recon_points(int P, const uint8_t* valid, const double* pts, double* ox, double* oy,
                                      double* oz, int* n_obs) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = p < P && valid[p];
  const unsigned mk = __ballot_sync(0xffffffffu, ok);
  if (!mk) return;
  int base = 0;
  const int lane = threadIdx.x & 31;
  if (lane == __ffs(mk) - 1) base = atomicAdd(n_obs, __popc(mk));
  base = __shfl_sync(0xffffffffu, base, __ffs(mk) - 1);
  if (ok) {
    const int k = base + __popc(mk & ((1u << lane) - 1u));
    ox[k] = pts[3 * p];
    oy[k] = pts[3 * p + 1];
    oz[k] = pts[3 * p + 2];
  }
}

constexpr int kNnTile = 1024;

static __global__ void __launch_bounds__(256) k_recon_nn(const int* vis_list, const int* n_vis, const double4* pv,
                                                         const double* ox, const double* oy, const double* oz,
                                                         const int* n_obs, double* dist) {
  __shared__ double tx[kNnTile], ty[kNnTile], tz[kNnTile];
  const int nvis = *n_vis, nobs = *n_obs;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = s < nvis;
  const int vi = act ? vis_list[s] : 0;
  double4 v = make_double4(0, 0, 0, 0);
  if (act) v = pv[vi];
  if (blockIdx.x * blockDim.x >= nvis) return;  // CTA-uniform
  double best = INFINITY;
  for (int t0 = 0; t0 < nobs; t0 += kNnTile) {
    const int n = min(kNnTile, nobs - t0);
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      tx[k] = ox[t0 + k];
      ty[k] = oy[t0 + k];
      tz[k] = oz[t0 + k];
    }
    __syncthreads();
    if (act) {
#pragma unroll 4
      for (int k = 0; k < n; ++k) {
        // (p - v).squaredNorm(), metrics.cpp:138
        const double dx = tx[k] - v.x, dy = ty[k] - v.y, dz = tz[k] - v.z;
        best = fmin(best, (dx * dx + dy * dy) + dz * dz);
      }
    }
  }
  if (act) dist[vi] = nobs > 0 ? sqrt(best) : 0.0;
}

void recon_launch(cudaStream_t st, const DevModel& m, const DevState& s, const DevIntr& in, int T, const int* tri,
                  double* v3, unsigned long long* zbits, int* owner, const uint8_t* pvalid, const double* pts,
                  double* ox, double* oy, double* oz, int* vis_list, int* counters, double* dist) {
  const int V = m.V, P = in.W * in.H;
  k_pack_pv<<<(V + 255) / 256, 256, 0, st>>>(V, s.pv, v3);
  raster_launch(st, T, v3, tri, in.fx, in.fy, in.cx, in.cy, in.W, in.H, zbits, owner);
  cudaMemsetAsync(counters, 0, 2 * sizeof(int), st);
  cudaMemsetAsync(dist, 0xFF, sizeof(double) * V, st);  // NaN: not visible
  k_recon_visible<<<(V + 255) / 256, 256, 0, st>>>(m, s.pv, in, zbits, owner, vis_list, counters);
  k_recon_points<<<(P + 255) / 256, 256, 0, st>>>(P, pvalid, pts, ox, oy, oz, counters + 1);
  k_recon_nn<<<(V + 255) / 256, 256, 0, st>>>(vis_list, counters, s.pv, ox, oy, oz, counters + 1, dist);
}

}  // namespace wt
