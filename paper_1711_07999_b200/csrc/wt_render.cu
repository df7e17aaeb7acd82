// wt_render.cu -- GPU synthetic depth renderer (synthesize_frame,
// proj/src/synth.cpp:139-270): fp64 dual-quaternion skinning, z-buffer
// rasterisation with 1/z interpolation, the stateless splitmix64 noise model
// and joint visibility. Compiled with -fmad=false so every product/sum is
// rounded exactly like the reference's unfused C++ (same operation order),
// which makes noiseless renders agree with the CPU reference pixel for pixel
// up to transcendental last-bit differences in FK.
//
// Ties in the z-buffer resolve like the reference's strict `z <` test in
// triangle order: pass 1 takes the minimum depth per pixel (positive doubles
// order like their bit patterns), pass 2 the lowest triangle index at that
// depth.
#include <cstdint>

#include "wt_dq.cuh"

namespace wt {

// skin() in fp64 (skinmesh.cpp:60-77,112-121) with double weights.
__global__ void k_skin64(int V, int L, const double* offsets, const double* v0, const double* phi,
                         const double* wgt, const int* wlink, const int* wcount, double* out) {
  extern __shared__ double s_off[];
  for (int k = threadIdx.x; k < 8 * L; k += blockDim.x) s_off[k] = offsets[k];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const double rest[3] = {v0[3 * i] + phi[3 * i], v0[3 * i + 1] + phi[3 * i + 1],
                          v0[3 * i + 2] + phi[3 * i + 2]};
  const int cnt = wcount[i];
  DQ sum;
  for (int c = 0; c < 4; ++c) sum.r[c] = sum.d[c] = 0.0;
  bool ok = false;
  if (cnt > 0) {
    const double* pivot = s_off + 8 * wlink[4 * i];
    for (int s = 0; s < cnt; ++s) {
      const double* h = s_off + 8 * wlink[4 * i + s];
      const double dot = pivot[0] * h[0] + pivot[1] * h[1] + pivot[2] * h[2] + pivot[3] * h[3];
      const double sign = dot < 0.0 ? -1.0 : 1.0;
      const double k = sign * wgt[4 * i + s];
      for (int c = 0; c < 4; ++c) {
        sum.r[c] = sum.r[c] + h[c] * k;
        sum.d[c] = sum.d[c] + h[4 + c] * k;
      }
    }
    const double n = sqrt(sum.r[0] * sum.r[0] + sum.r[1] * sum.r[1] + sum.r[2] * sum.r[2] +
                          sum.r[3] * sum.r[3]);
    ok = n > 1e-12;
  }
  double p[3] = {rest[0], rest[1], rest[2]};
  if (ok) dq_transform_point(dq_normalize(sum), rest, p);
  out[3 * i] = p[0];
  out[3 * i + 1] = p[1];
  out[3 * i + 2] = p[2];
}

struct RasterTri {
  bool ok;
  double ua, va, ub, vb, uc, vc, inv_area, iza, izb, izc;
  int u0, u1, v0, v1;
};

__device__ __forceinline__ RasterTri setup_tri(const double* v, const int* tri, int t, double fx,
                                               double fy, double cx, double cy, int W, int H) {
  RasterTri r;
  r.ok = false;
  const double* a = v + 3 * tri[3 * t];
  const double* b = v + 3 * tri[3 * t + 1];
  const double* c = v + 3 * tri[3 * t + 2];
  constexpr double kNear = 1e-6;
  if (a[2] <= kNear || b[2] <= kNear || c[2] <= kNear) return r;
  r.ua = fx * a[0] / a[2] + cx;
  r.va = fy * a[1] / a[2] + cy;
  r.ub = fx * b[0] / b[2] + cx;
  r.vb = fy * b[1] / b[2] + cy;
  r.uc = fx * c[0] / c[2] + cx;
  r.vc = fy * c[1] / c[2] + cy;
  const double area2 = (r.ub - r.ua) * (r.vc - r.va) - (r.vb - r.va) * (r.uc - r.ua);
  if (fabs(area2) < 1e-12) return r;
  r.inv_area = 1.0 / area2;
  r.u0 = max(0, static_cast<int>(ceil(fmin(r.ua, fmin(r.ub, r.uc)))));
  r.u1 = min(W - 1, static_cast<int>(floor(fmax(r.ua, fmax(r.ub, r.uc)))));
  r.v0 = max(0, static_cast<int>(ceil(fmin(r.va, fmin(r.vb, r.vc)))));
  r.v1 = min(H - 1, static_cast<int>(floor(fmax(r.va, fmax(r.vb, r.vc)))));
  r.iza = 1.0 / a[2];
  r.izb = 1.0 / b[2];
  r.izc = 1.0 / c[2];
  r.ok = true;
  return r;
}

__device__ __forceinline__ bool tri_depth(const RasterTri& r, int px, int py, double* z) {
  const double pu = px, pv = py;
  const double la = ((r.ub - pu) * (r.vc - pv) - (r.vb - pv) * (r.uc - pu)) * r.inv_area;
  const double lb = ((r.uc - pu) * (r.va - pv) - (r.vc - pv) * (r.ua - pu)) * r.inv_area;
  const double lc = 1.0 - la - lb;
  if (la < -1e-12 || lb < -1e-12 || lc < -1e-12) return false;
  const double inv_z = la * r.iza + lb * r.izb + lc * r.izc;
  if (inv_z <= 0.0) return false;
  *z = 1.0 / inv_z;
  return true;
}

__global__ void k_raster(int T, const double* v, const int* tri, double fx, double fy, double cx,
                         double cy, int W, int H, int pass, unsigned long long* zbits, int* owner) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const RasterTri r = setup_tri(v, tri, t, fx, fy, cx, cy, W, H);
  if (!r.ok) return;
  for (int py = r.v0; py <= r.v1; ++py)
    for (int px = r.u0; px <= r.u1; ++px) {
      double z;
      if (!tri_depth(r, px, py, &z)) continue;
      const size_t pi = static_cast<size_t>(py) * W + px;
      const unsigned long long zb = static_cast<unsigned long long>(__double_as_longlong(z));
      if (pass == 0) atomicMin(zbits + pi, zb);
      else if (zbits[pi] == zb) atomicMin(owner + pi, t);
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ double uniform01(uint64_t h) {
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

// synth.cpp:195-209,237-254
__global__ void k_noise(int P, const unsigned long long* zbits, int* owner, double sigma,
                        double dropout, double quant, uint64_t base, float* depth) {
  const int pi = blockIdx.x * blockDim.x + threadIdx.x;
  if (pi >= P) return;
  float out = 0.0f;
  if (owner[pi] == 0x7F7F7F7F) {
    owner[pi] = -1;  // no triangle reached this pixel
  } else {
    double z = __longlong_as_double(static_cast<long long>(zbits[pi]));
    bool keep = true;
    const uint64_t upi = static_cast<uint64_t>(pi);
    if (dropout > 0.0 && uniform01(splitmix64(base ^ (upi * 3 + 1))) < dropout) keep = false;
    if (keep) {
      if (sigma > 0.0) {
        const double u1 = 1.0 - uniform01(splitmix64(base ^ (upi * 3 + 2)));
        const double u2 = uniform01(splitmix64(base ^ (upi * 3 + 3)));
        z += sigma * (sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2));
      }
      if (quant > 0.0) z = round(z / quant) * quant;  // std::round: half away from zero
      if (z > 0.0) out = static_cast<float>(z);
    }
  }
  depth[pi] = out;
}

// Joint visibility (synth.cpp:256-268): a link is visible when a vertex it
// dominates belongs to a z-buffer winning triangle.
__global__ void k_visibility(int P, const int* owner, const int* tri, const int* dom,
                             uint8_t* vis) {
  const int pi = blockIdx.x * blockDim.x + threadIdx.x;
  if (pi >= P) return;
  const int t = owner[pi];
  if (t < 0) return;
  for (int c = 0; c < 3; ++c) {
    const int link = dom[tri[3 * t + c]];
    if (link >= 0) vis[link] = 1;
  }
}

// rasterize (synth.cpp:139-191) of fp64 vertices [V*3]: depth bits and the
// winning triangle per pixel (0x7F7F7F7F where no triangle reached it).
void raster_launch(cudaStream_t st, int T, const double* vpos, const int* tri, double fx, double fy, double cx,
                   double cy, int W, int H, unsigned long long* zbits, int* owner) {
  const int P = W * H;
  cudaMemsetAsync(zbits, 0xFF, sizeof(unsigned long long) * P, st);
  cudaMemsetAsync(owner, 0x7F, sizeof(int) * P, st);
  k_raster<<<(T + 127) / 128, 128, 0, st>>>(T, vpos, tri, fx, fy, cx, cy, W, H, 0, zbits, owner);
  k_raster<<<(T + 127) / 128, 128, 0, st>>>(T, vpos, tri, fx, fy, cx, cy, W, H, 1, zbits, owner);
}

void render_launch(cudaStream_t st, int V, int L, int T, const double* offsets, const double* v0,
                   const double* phi, const double* wgt, const int* wlink, const int* wcount,
                   const int* tri, const int* dom, double fx, double fy, double cx, double cy,
                   int W, int H, double sigma, double dropout, double quant, uint64_t base,
                   double* vpos, unsigned long long* zbits, int* owner, float* depth,
                   uint8_t* vis) {
  const int P = W * H;
  k_skin64<<<(V + 255) / 256, 256, sizeof(double) * 8 * L, st>>>(V, L, offsets, v0, phi, wgt,
                                                                  wlink, wcount, vpos);
  cudaMemsetAsync(zbits, 0xFF, sizeof(unsigned long long) * P, st);
  cudaMemsetAsync(owner, 0x7F, sizeof(int) * P, st);
  k_raster<<<(T + 127) / 128, 128, 0, st>>>(T, vpos, tri, fx, fy, cx, cy, W, H, 0, zbits, owner);
  k_raster<<<(T + 127) / 128, 128, 0, st>>>(T, vpos, tri, fx, fy, cx, cy, W, H, 1, zbits, owner);
  // pixels no triangle reached keep owner = 0x7F7F7F7F; k_noise maps them to -1
  k_noise<<<(P + 255) / 256, 256, 0, st>>>(P, zbits, owner, sigma, dropout, quant, base, depth);
  cudaMemsetAsync(vis, 0, L, st);
  k_visibility<<<(P + 255) / 256, 256, 0, st>>>(P, owner, tri, dom, vis);
}

}  // namespace wt
