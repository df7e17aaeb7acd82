// wt_model.cu -- model preprocessing on the device: Catmull-Clark subdivision
// with skin weights (subdivide, skinmesh.cpp:249-511), SkinnedMesh::finalize
// (triangulation + vertex->triangle CSR, skinmesh.cpp:13-58) and the exact
// k-nearest-neighbour lists (build_neighbors, skinmesh.cpp:145-247).
//
// Compiled with -fmad=false: every sum and product rounds separately and in
// the reference's order, so the output mesh is bitwise the reference's.
// Topology that the reference builds with hash maps in first-appearance
// order is rebuilt here with stable radix sorts (cub) over half-edges, which
// reproduces the same numbering: edges are numbered by their first
// half-edge in (face, side) order, each vertex's edge and face lists are
// ascending, exactly the push_back orders of catmull_clark_once.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "wt_gpu.h"

namespace {

struct Fail {
  int code;
  std::string msg;
};

#define WM_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) throw Fail{WT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

// A device array that frees itself.
template <class T>
struct DArr {
  T* p = nullptr;
  size_t n = 0;
  DArr() = default;
  explicit DArr(size_t count) { resize(count); }
  DArr(const DArr&) = delete;
  DArr& operator=(const DArr&) = delete;
  DArr(DArr&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DArr& operator=(DArr&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    return *this;
  }
  ~DArr() {
    if (p) cudaFree(p);
  }
  void resize(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    const cudaError_t e = cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1));
    if (e != cudaSuccess) throw Fail{WT_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e)};
  }
  void upload(const T* h, size_t count) {
    resize(count);
    if (count) WM_CUDA(cudaMemcpy(p, h, sizeof(T) * count, cudaMemcpyHostToDevice));
  }
  void download(T* h, size_t count) const {
    if (count && h) WM_CUDA(cudaMemcpy(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost));
  }
};

int blocks(long long n, int t = 256) { return static_cast<int>(std::max(1LL, (n + t - 1) / t)); }

void check_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Fail{WT_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

// exclusive scan of n ints (out[n] = total)
void exclusive_scan(const int* in, int* out, int n) {
  size_t tmp = 0;
  WM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n + 1));
  DArr<unsigned char> t(tmp);
  WM_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n + 1));
}

// stable sort of (key, value) pairs by key
template <class K>
void sort_pairs(const K* kin, K* kout, const int* vin, int* vout, int n, int end_bit) {
  size_t tmp = 0;
  WM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, end_bit));
  DArr<unsigned char> t(tmp);
  WM_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kin, kout, vin, vout, n, 0, end_bit));
}

int bits_for(long long n) {
  int b = 1;
  while ((1LL << b) <= n) ++b;
  return b;
}

}  // namespace

// The working mesh of the subdivision: positions, phi, dense skin weights
// (V x L, the reference's sparse WeightMap with absent links as 0 -- adding
// 0.0 never changes a sum), polygons as CSR.
struct wt_mesh {
  int device = 0;
  int V = 0, L = 0, F = 0, NI = 0;  // vertices, links, polygons, polygon items
  DArr<double> pos, phi, W;        // [3V], [3V], [V*L]
  DArr<int> foff, fitems;          // [F+1], [NI]
  bool weights_dense = true;       // false: weight rows passed through (iterations == 0)
  DArr<int> wcount, wlink;         // final rows [V], [4V]
  DArr<double> wval;               // [4V]
  int T = 0;
  DArr<int> tri, vtri_off, vtri_items;  // finalize
  int K = 0;
  DArr<int> nbr;                        // [V*K] build_neighbors
};

namespace wt_model {

// ---- Catmull-Clark, one level (catmull_clark_once, skinmesh.cpp:298-470) ----

__global__ void k_halfedges(int F, const int* foff, const int* items, int* face_of, int* side_of,
                            unsigned long long* key) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const int o = foff[f], n = foff[f + 1] - o;
  for (int s = 0; s < n; ++s) {
    const int a = items[o + s], b = items[o + (s + 1) % n];
    face_of[o + s] = f;
    side_of[o + s] = s;
    const unsigned lo = static_cast<unsigned>(min(a, b)), hi = static_cast<unsigned>(max(a, b));
    key[o + s] = (static_cast<unsigned long long>(lo) << 32) | hi;
  }
}

// group heads of the sorted keys; the first half-edge of each group (stable
// sort: the smallest h) marks its edge; more than two half-edges -> error
__global__ void k_edge_heads(int H, const unsigned long long* sk, const int* sh, int* is_first, int* err) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= H) return;
  const bool head = j == 0 || sk[j] != sk[j - 1];
  if (head) {
    is_first[sh[j]] = 1;
    if (j + 2 < H && sk[j + 2] == sk[j]) atomicExch(err, 1);  // a third face on this edge
  }
}

__global__ void k_edges(int H, const unsigned long long* sk, const int* sh, const int* eid_first, const int* face_of,
                        int* face_edge, int* ea, int* eb, int* ef0, int* ef1, int* nfe) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= H) return;
  const bool head = j == 0 || sk[j] != sk[j - 1];
  const int j0 = head ? j : j - 1;  // groups hold at most two half-edges
  const int e = eid_first[sh[j0]];
  face_edge[sh[j]] = e;
  if (head) {
    const bool two = j + 1 < H && sk[j + 1] == sk[j];
    ea[e] = static_cast<int>(sk[j] >> 32);
    eb[e] = static_cast<int>(sk[j] & 0xFFFFFFFFull);
    ef0[e] = face_of[sh[j]];
    ef1[e] = two ? face_of[sh[j + 1]] : -1;
    nfe[e] = two ? 2 : 1;
  }
}

// face points: p += pos[v] * c over the polygon, c = 1 / n (skinmesh.cpp:339-353)
__global__ void k_face_points(int F, int L, const int* foff, const int* items, const double* pos,
                              const double* phi, const double* W, double* opos, double* ophi, double* oW,
                              int face_base) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const int o = foff[f], n = foff[f + 1] - o;
  const double c = 1.0 / static_cast<double>(n);
  double p[3] = {0, 0, 0}, ph[3] = {0, 0, 0};
  for (int s = 0; s < n; ++s) {
    const int v = items[o + s];
    for (int d = 0; d < 3; ++d) {
      p[d] += pos[3 * v + d] * c;
      ph[d] += phi[3 * v + d] * c;
    }
  }
  const size_t out = static_cast<size_t>(face_base) + f;
  for (int d = 0; d < 3; ++d) {
    opos[3 * out + d] = p[d];
    ophi[3 * out + d] = ph[d];
  }
  for (int l = 0; l < L; ++l) {
    double w = 0.0;
    for (int s = 0; s < n; ++s) w += c * W[static_cast<size_t>(items[o + s]) * L + l];
    oW[out * L + l] = w;
  }
}

// edge points (skinmesh.cpp:355-383)
__global__ void k_edge_points(int NE, int L, const int* ea, const int* eb, const int* ef0, const int* ef1,
                              const int* nfe, const double* pos, const double* phi, const double* W, double* opos,
                              double* ophi, double* oW, int edge_base, int face_base) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= NE) return;
  const int a = ea[e], b = eb[e];
  const size_t out = static_cast<size_t>(edge_base) + e;
  if (nfe[e] == 2) {
    const size_t f0 = static_cast<size_t>(face_base) + ef0[e], f1 = static_cast<size_t>(face_base) + ef1[e];
    for (int d = 0; d < 3; ++d) {
      opos[3 * out + d] = (((pos[3 * a + d] + pos[3 * b + d]) + opos[3 * f0 + d]) + opos[3 * f1 + d]) * 0.25;
      ophi[3 * out + d] = (((phi[3 * a + d] + phi[3 * b + d]) + ophi[3 * f0 + d]) + ophi[3 * f1 + d]) * 0.25;
    }
    for (int l = 0; l < L; ++l)
      oW[out * L + l] = ((0.25 * W[static_cast<size_t>(a) * L + l] + 0.25 * W[static_cast<size_t>(b) * L + l]) +
                         0.25 * oW[f0 * L + l]) +
                        0.25 * oW[f1 * L + l];
  } else {
    for (int d = 0; d < 3; ++d) {
      opos[3 * out + d] = (pos[3 * a + d] + pos[3 * b + d]) * 0.5;
      ophi[3 * out + d] = (phi[3 * a + d] + phi[3 * b + d]) * 0.5;
    }
    for (int l = 0; l < L; ++l)
      oW[out * L + l] = 0.5 * W[static_cast<size_t>(a) * L + l] + 0.5 * W[static_cast<size_t>(b) * L + l];
  }
}

// (vertex, edge) pairs in edge order: ea[e], eb[e]
__global__ void k_vertex_edge_pairs(int NE, const int* ea, const int* eb, int* pv, int* pe) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= NE) return;
  pv[2 * e] = ea[e];
  pe[2 * e] = e;
  pv[2 * e + 1] = eb[e];
  pe[2 * e + 1] = e;
}

__global__ void k_count(int n, const int* keys, int* counts) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) atomicAdd(&counts[keys[j]], 1);
}

// original vertices (skinmesh.cpp:385-456): interior (F + 2R + (n-3)P)/n,
// boundary crease (m1 + 6P + m2)/8, isolated kept
__global__ void k_vertex_points(int V, int L, const int* ve_off, const int* ve, const int* vf_off, const int* vf,
                                const int* ea, const int* eb, const int* nfe, const double* pos, const double* phi,
                                const double* W, double* opos, double* ophi, double* oW, int face_base) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int e0 = ve_off[i], e1 = ve_off[i + 1];
  const int f0 = vf_off[i], f1 = vf_off[i + 1];
  bool boundary = false;
  for (int k = e0; k < e1; ++k) boundary = boundary || nfe[ve[k]] < 2;
  const size_t Li = static_cast<size_t>(i) * L;
  if (e0 == e1) {  // isolated vertex
    for (int d = 0; d < 3; ++d) {
      opos[3 * i + d] = pos[3 * i + d];
      ophi[3 * i + d] = phi[3 * i + d];
    }
    for (int l = 0; l < L; ++l) oW[Li + l] = W[Li + l];
    return;
  }
  if (boundary) {
    double p[3] = {0, 0, 0}, ph[3] = {0, 0, 0};
    for (int l = 0; l < L; ++l) oW[Li + l] = 0.0;
    for (int k = e0; k < e1; ++k) {
      const int e = ve[k];
      if (nfe[e] >= 2) continue;
      const int other = ea[e] == i ? eb[e] : ea[e];
      for (int d = 0; d < 3; ++d) {
        p[d] += (pos[3 * i + d] + pos[3 * other + d]) * 0.5;
        ph[d] += (phi[3 * i + d] + phi[3 * other + d]) * 0.5;
      }
      for (int l = 0; l < L; ++l) {
        oW[Li + l] += (0.5 / 8.0) * W[Li + l];
        oW[Li + l] += (0.5 / 8.0) * W[static_cast<size_t>(other) * L + l];
      }
    }
    for (int d = 0; d < 3; ++d) {
      opos[3 * i + d] = p[d] / 8.0 + pos[3 * i + d] * (6.0 / 8.0);
      ophi[3 * i + d] = ph[d] / 8.0 + phi[3 * i + d] * (6.0 / 8.0);
    }
    for (int l = 0; l < L; ++l) oW[Li + l] += (6.0 / 8.0) * W[Li + l];
    return;
  }
  const double n = static_cast<double>(e1 - e0);
  const double nf = static_cast<double>(f1 - f0);
  double fa[3] = {0, 0, 0}, fph[3] = {0, 0, 0}, ra[3] = {0, 0, 0}, rph[3] = {0, 0, 0};
  for (int k = f0; k < f1; ++k) {
    const size_t fp = static_cast<size_t>(face_base) + vf[k];
    for (int d = 0; d < 3; ++d) {
      fa[d] += opos[3 * fp + d];
      fph[d] += ophi[3 * fp + d];
    }
  }
  for (int k = e0; k < e1; ++k) {
    const int e = ve[k];
    for (int d = 0; d < 3; ++d) {
      ra[d] += (pos[3 * ea[e] + d] + pos[3 * eb[e] + d]) * 0.5;
      rph[d] += (phi[3 * ea[e] + d] + phi[3 * eb[e] + d]) * 0.5;
    }
  }
  for (int d = 0; d < 3; ++d) {
    fa[d] /= nf;
    fph[d] /= nf;
    ra[d] /= n;
    rph[d] /= n;
    opos[3 * i + d] = ((fa[d] + 2.0 * ra[d]) + (n - 3.0) * pos[3 * i + d]) / n;
    ophi[3 * i + d] = ((fph[d] + 2.0 * rph[d]) + (n - 3.0) * phi[3 * i + d]) / n;
  }
  const double cf = 1.0 / nf, cr = 0.5 / n;
  for (int l = 0; l < L; ++l) {
    double fw = 0.0, rw = 0.0;
    for (int k = f0; k < f1; ++k) fw += cf * oW[(static_cast<size_t>(face_base) + vf[k]) * L + l];
    for (int k = e0; k < e1; ++k) {
      const int e = ve[k];
      rw += cr * W[static_cast<size_t>(ea[e]) * L + l];
      rw += cr * W[static_cast<size_t>(eb[e]) * L + l];
    }
    oW[Li + l] = (((1.0 / n) * fw) + (2.0 / n) * rw) + ((n - 3.0) / n) * W[Li + l];
  }
}

// new faces: one quad per original corner, in (face, side) order
__global__ void k_new_faces(int H, const int* foff, const int* items, const int* face_of, const int* side_of,
                            const int* face_edge, int* ofitems, int edge_base, int face_base) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= H) return;
  const int f = face_of[h], s = side_of[h];
  const int o = foff[f], n = foff[f + 1] - o;
  ofitems[4 * h] = items[h];
  ofitems[4 * h + 1] = edge_base + face_edge[h];
  ofitems[4 * h + 2] = face_base + f;
  ofitems[4 * h + 3] = edge_base + face_edge[o + (s + n - 1) % n];
}

__global__ void k_iota_times(int n, int step, int* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j <= n) out[j] = j * step;
}

// truncate_weights (skinmesh.cpp:265-280): the four largest entries (ties to
// the lower link), summed in that order, re-sorted by link, zeros dropped,
// each divided by the sum
__global__ void k_truncate(int V, int L, const double* W, int* wc, int* wl, double* wv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const double* row = W + static_cast<size_t>(i) * L;
  int top[4];
  double tw[4];
  int nt = 0;
  for (int l = 0; l < L; ++l) {
    const double w = row[l];
    // lexicographic (w descending, link ascending): insert into the sorted top list
    int pos = nt;
    while (pos > 0 && (w > tw[pos - 1])) --pos;
    if (pos >= 4) continue;
    const int last = nt < 4 ? nt : 3;
    for (int q = last; q > pos; --q) {
      top[q] = top[q - 1];
      tw[q] = tw[q - 1];
    }
    top[pos] = l;
    tw[pos] = w;
    if (nt < 4) ++nt;
  }
  double sum = 0.0;
  for (int q = 0; q < nt; ++q) sum += tw[q];
  // by link
  for (int a = 1; a < nt; ++a)
    for (int b = a; b > 0 && top[b] < top[b - 1]; --b) {
      const int t = top[b];
      top[b] = top[b - 1];
      top[b - 1] = t;
      const double x = tw[b];
      tw[b] = tw[b - 1];
      tw[b - 1] = x;
    }
  int c = 0;
  for (int q = 0; q < 4; ++q) {
    wl[4 * i + q] = -1;
    wv[4 * i + q] = 0.0;
  }
  for (int q = 0; q < nt; ++q)
    if (tw[q] > 0.0) {
      wl[4 * i + c] = top[q];
      wv[4 * i + c] = tw[q] / sum;
      ++c;
    }
  wc[i] = c;
}

// ---- finalize (skinmesh.cpp:13-58) ------------------------------------------

__global__ void k_tri_counts(int F, int V, const int* foff, const int* items, int* cnt) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const int o = foff[f], n = foff[f + 1] - o;
  bool in_range = true;
  for (int s = 0; s < n; ++s) in_range = in_range && items[o + s] >= 0 && items[o + s] < V;
  cnt[f] = !in_range ? 0 : (n == 3 ? 1 : (n == 4 ? 2 : max(0, n - 2)));
}

__device__ __forceinline__ double sq_dist(const double* v0, int a, int b) {
  const double dx = v0[3 * a] - v0[3 * b], dy = v0[3 * a + 1] - v0[3 * b + 1], dz = v0[3 * a + 2] - v0[3 * b + 2];
  return (dx * dx + dy * dy) + dz * dz;
}

__global__ void k_triangulate(int F, const int* foff, const int* items, const int* toff, const double* v0, int* tri) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const int o = foff[f], n = foff[f + 1] - o;
  int t = toff[f];
  if (toff[f + 1] == t) return;
  const int* p = items + o;
  auto put = [&](int a, int b, int c) {
    tri[3 * t] = a;
    tri[3 * t + 1] = b;
    tri[3 * t + 2] = c;
    ++t;
  };
  if (n == 3) {
    put(p[0], p[1], p[2]);
  } else if (n == 4) {
    if (sq_dist(v0, p[0], p[2]) <= sq_dist(v0, p[1], p[3])) {
      put(p[0], p[1], p[2]);
      put(p[0], p[2], p[3]);
    } else {
      put(p[0], p[1], p[3]);
      put(p[1], p[2], p[3]);
    }
  } else {
    for (int s = 1; s + 1 < n; ++s) put(p[0], p[s], p[s + 1]);
  }
}

__global__ void k_vtri_fill(int T, const int* tri, const int* off, int* cursor, int* items) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  for (int c = 0; c < 3; ++c) {
    const int v = tri[3 * t + c];
    items[off[v] + atomicAdd(&cursor[v], 1)] = t;
  }
}

// each vertex's list ascending by triangle (the reference fills in triangle order)
__global__ void k_sort_segments(int V, const int* off, int* items) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int a = off[v], b = off[v + 1];
  for (int i = a + 1; i < b; ++i)
    for (int j = i; j > a && items[j] < items[j - 1]; --j) {
      const int x = items[j];
      items[j] = items[j - 1];
      items[j - 1] = x;
    }
}

// ---- build_neighbors (skinmesh.cpp:145-247) -----------------------------------

struct Grid {
  double ox, oy, oz, cell;
  int nx, ny, nz;
};

__device__ __forceinline__ int clampi(int v, int n) { return min(max(v, 0), n - 1); }

__global__ void k_cells(int V, const double* v0, Grid g, int* cell) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int ix = clampi(static_cast<int>((v0[3 * i] - g.ox) / g.cell), g.nx);
  const int iy = clampi(static_cast<int>((v0[3 * i + 1] - g.oy) / g.cell), g.ny);
  const int iz = clampi(static_cast<int>((v0[3 * i + 2] - g.oz) / g.cell), g.nz);
  cell[i] = (iz * g.ny + iy) * g.nx + ix;
}

// exact k nearest (squared distance, index) of every vertex, by rings of
// grid cells until the next ring cannot beat the k-th best (the reference's
// rule, conservative in the cell bounds)
template <int KMAX>
__global__ void k_knn(int V, int want, const double* v0, Grid g, const int* coff, const int* citems, int* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const double qx = v0[3 * i], qy = v0[3 * i + 1], qz = v0[3 * i + 2];
  const int cx = clampi(static_cast<int>((qx - g.ox) / g.cell), g.nx);
  const int cy = clampi(static_cast<int>((qy - g.oy) / g.cell), g.ny);
  const int cz = clampi(static_cast<int>((qz - g.oz) / g.cell), g.nz);
  double bd[KMAX];
  int bi[KMAX];
  int nb = 0;
  const int max_ring = max(g.nx, max(g.ny, g.nz));
  for (int ring = 0; ring <= max_ring; ++ring) {
    if (nb == want) {
      const double rmin = (ring - 1) > 0 ? (ring - 1) * g.cell : 0.0;
      if (rmin * rmin > bd[want - 1]) break;
    }
    for (int dz = -ring; dz <= ring; ++dz)
      for (int dy = -ring; dy <= ring; ++dy)
        for (int dx = -ring; dx <= ring; ++dx) {
          if (max(abs(dx), max(abs(dy), abs(dz))) != ring) continue;
          const int ix = cx + dx, iy = cy + dy, iz = cz + dz;
          if (ix < 0 || iy < 0 || iz < 0 || ix >= g.nx || iy >= g.ny || iz >= g.nz) continue;
          const int c = (iz * g.ny + iy) * g.nx + ix;
          for (int s = coff[c]; s < coff[c + 1]; ++s) {
            const int j = citems[s];
            if (j == i) continue;
            const double ddx = v0[3 * j] - qx, ddy = v0[3 * j + 1] - qy, ddz = v0[3 * j + 2] - qz;
            const double d2 = (ddx * ddx + ddy * ddy) + ddz * ddz;
            // lexicographic (d2, j) insertion into the sorted best list
            int pos = nb;
            while (pos > 0 && (d2 < bd[pos - 1] || (d2 == bd[pos - 1] && j < bi[pos - 1]))) --pos;
            if (pos >= want) continue;
            const int last = nb < want ? nb : want - 1;
            for (int q = last; q > pos; --q) {
              bd[q] = bd[q - 1];
              bi[q] = bi[q - 1];
            }
            bd[pos] = d2;
            bi[pos] = j;
            if (nb < want) ++nb;
          }
        }
  }
  for (int q = 0; q < want; ++q) out[static_cast<size_t>(i) * want + q] = q < nb ? bi[q] : -1;
}

}  // namespace wt_model

namespace {

using namespace wt_model;

// the GridKnn of the reference (skinmesh.cpp:151-176): bounding box, cell size
// from the volume heuristic with the O(n)-cells floor
Grid make_grid(const std::vector<double>& v0, int V) {
  double lo[3] = {v0[0], v0[1], v0[2]}, hi[3] = {v0[0], v0[1], v0[2]};
  for (int i = 0; i < V; ++i)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], v0[3 * i + d]);
      hi[d] = std::max(hi[d], v0[3 * i + d]);
    }
  const double n = static_cast<double>(V);
  double span[3];
  for (int d = 0; d < 3; ++d) span[d] = std::max(hi[d] - lo[d], 1e-9);
  const double mx = std::max(span[0], std::max(span[1], span[2]));
  Grid g;
  g.cell = std::max({1e-9, std::cbrt(span[0] * span[1] * span[2] / n) * 1.5, mx / (2.0 * std::cbrt(n) + 1.0)});
  g.ox = lo[0];
  g.oy = lo[1];
  g.oz = lo[2];
  g.nx = static_cast<int>(span[0] / g.cell) + 1;
  g.ny = static_cast<int>(span[1] / g.cell) + 1;
  g.nz = static_cast<int>(span[2] / g.cell) + 1;
  return g;
}

void knn(int V, const DArr<double>& v0, int k, DArr<int>& out, int& want) {
  want = std::min(k, V - 1);
  if (V <= 1 || k < 1) {
    want = 0;
    out.resize(0);
    return;
  }
  if (want > 16) throw Fail{WT_EINVAL, "build_neighbors: at most 16 neighbours on the GPU path"};
  std::vector<double> h(3 * static_cast<size_t>(V));
  v0.download(h.data(), h.size());
  const Grid g = make_grid(h, V);
  const long long ncell = static_cast<long long>(g.nx) * g.ny * g.nz;
  if (ncell > (1LL << 30)) throw Fail{WT_EINVAL, "build_neighbors: degenerate grid"};
  DArr<int> cell(V), cnt(ncell + 1), coff(ncell + 1), citems(V);
  k_cells<<<blocks(V), 256>>>(V, v0.p, g, cell.p);
  WM_CUDA(cudaMemset(cnt.p, 0, sizeof(int) * (ncell + 1)));
  k_count<<<blocks(V), 256>>>(V, cell.p, cnt.p);
  check_launch();
  exclusive_scan(cnt.p, coff.p, static_cast<int>(ncell));
  // the vertices in cell order (order inside a cell is irrelevant: the minimum is exact)
  {
    DArr<int> iota(V), sorted_cell(V);
    std::vector<int> hi(static_cast<size_t>(V));
    for (int i = 0; i < V; ++i) hi[static_cast<size_t>(i)] = i;
    iota.upload(hi.data(), hi.size());
    sort_pairs<int>(cell.p, sorted_cell.p, iota.p, citems.p, V, bits_for(ncell));
  }
  out.resize(static_cast<size_t>(V) * want);
  if (want <= 4) k_knn<4><<<blocks(V, 128), 128>>>(V, want, v0.p, g, coff.p, citems.p, out.p);
  else if (want <= 8) k_knn<8><<<blocks(V, 128), 128>>>(V, want, v0.p, g, coff.p, citems.p, out.p);
  else k_knn<16><<<blocks(V, 128), 128>>>(V, want, v0.p, g, coff.p, citems.p, out.p);
  check_launch();
  WM_CUDA(cudaDeviceSynchronize());
}

void subdivide_once(wt_mesh& m) {
  const int V = m.V, L = m.L, F = m.F, H = m.NI;
  DArr<int> face_of(H), side_of(H), sh(H), iota(H), is_first(H + 1), eid_first(H + 1), face_edge(H), err(1);
  DArr<unsigned long long> key(H), skey(H);
  k_halfedges<<<blocks(F), 256>>>(F, m.foff.p, m.fitems.p, face_of.p, side_of.p, key.p);
  check_launch();
  {
    std::vector<int> h(static_cast<size_t>(H));
    for (int j = 0; j < H; ++j) h[static_cast<size_t>(j)] = j;
    iota.upload(h.data(), h.size());
  }
  sort_pairs<unsigned long long>(key.p, skey.p, iota.p, sh.p, H, 64);
  WM_CUDA(cudaMemset(is_first.p, 0, sizeof(int) * (H + 1)));
  WM_CUDA(cudaMemset(err.p, 0, sizeof(int)));
  k_edge_heads<<<blocks(H), 256>>>(H, skey.p, sh.p, is_first.p, err.p);
  check_launch();
  int herr = 0;
  err.download(&herr, 1);
  if (herr) throw Fail{WT_EINVAL, "subdivide: an edge has more than two incident faces (NonManifold)"};
  exclusive_scan(is_first.p, eid_first.p, H);
  int NE = 0;
  WM_CUDA(cudaMemcpy(&NE, eid_first.p + H, sizeof(int), cudaMemcpyDeviceToHost));
  DArr<int> ea(NE), eb(NE), ef0(NE), ef1(NE), nfe(NE);
  k_edges<<<blocks(H), 256>>>(H, skey.p, sh.p, eid_first.p, face_of.p, face_edge.p, ea.p, eb.p, ef0.p, ef1.p,
                              nfe.p);
  check_launch();

  const int NV = V + NE + F, face_base = V + NE, edge_base = V;
  DArr<double> opos(3 * static_cast<size_t>(NV)), ophi(3 * static_cast<size_t>(NV)), oW(static_cast<size_t>(NV) * L);
  k_face_points<<<blocks(F), 256>>>(F, L, m.foff.p, m.fitems.p, m.pos.p, m.phi.p, m.W.p, opos.p, ophi.p, oW.p,
                                    face_base);
  check_launch();
  k_edge_points<<<blocks(NE), 256>>>(NE, L, ea.p, eb.p, ef0.p, ef1.p, nfe.p, m.pos.p, m.phi.p, m.W.p, opos.p,
                                     ophi.p, oW.p, edge_base, face_base);
  check_launch();
  // vertex -> edges (ascending edge), vertex -> faces (ascending face)
  DArr<int> pv(2 * static_cast<size_t>(NE)), pe(2 * static_cast<size_t>(NE)), spv(2 * static_cast<size_t>(NE)),
      ve(2 * static_cast<size_t>(NE)), vcnt(V + 1), ve_off(V + 1);
  k_vertex_edge_pairs<<<blocks(NE), 256>>>(NE, ea.p, eb.p, pv.p, pe.p);
  check_launch();
  sort_pairs<int>(pv.p, spv.p, pe.p, ve.p, 2 * NE, bits_for(V));
  WM_CUDA(cudaMemset(vcnt.p, 0, sizeof(int) * (V + 1)));
  k_count<<<blocks(2 * NE), 256>>>(2 * NE, pv.p, vcnt.p);
  check_launch();
  exclusive_scan(vcnt.p, ve_off.p, V);
  DArr<int> svf(H), vf(H), fcnt(V + 1), vf_off(V + 1);
  sort_pairs<int>(m.fitems.p, svf.p, face_of.p, vf.p, H, bits_for(V));
  WM_CUDA(cudaMemset(fcnt.p, 0, sizeof(int) * (V + 1)));
  k_count<<<blocks(H), 256>>>(H, m.fitems.p, fcnt.p);
  check_launch();
  exclusive_scan(fcnt.p, vf_off.p, V);
  k_vertex_points<<<blocks(V), 256>>>(V, L, ve_off.p, ve.p, vf_off.p, vf.p, ea.p, eb.p, nfe.p, m.pos.p, m.phi.p,
                                      m.W.p, opos.p, ophi.p, oW.p, face_base);
  check_launch();
  DArr<int> ofoff(H + 1), ofitems(4 * static_cast<size_t>(H));
  k_new_faces<<<blocks(H), 256>>>(H, m.foff.p, m.fitems.p, face_of.p, side_of.p, face_edge.p, ofitems.p, edge_base,
                                  face_base);
  k_iota_times<<<blocks(H + 1), 256>>>(H, 4, ofoff.p);
  check_launch();
  WM_CUDA(cudaDeviceSynchronize());
  m.V = NV;
  m.F = H;
  m.NI = 4 * H;
  m.pos = std::move(opos);
  m.phi = std::move(ophi);
  m.W = std::move(oW);
  m.foff = std::move(ofoff);
  m.fitems = std::move(ofitems);
}

void finalize(wt_mesh& m) {
  const int V = m.V, F = m.F;
  DArr<int> cnt(F + 1), toff(F + 1);
  k_tri_counts<<<blocks(F), 256>>>(F, V, m.foff.p, m.fitems.p, cnt.p);
  check_launch();
  exclusive_scan(cnt.p, toff.p, F);
  WM_CUDA(cudaMemcpy(&m.T, toff.p + F, sizeof(int), cudaMemcpyDeviceToHost));
  m.tri.resize(3 * static_cast<size_t>(m.T));
  k_triangulate<<<blocks(F), 256>>>(F, m.foff.p, m.fitems.p, toff.p, m.pos.p, m.tri.p);
  check_launch();
  DArr<int> vc(V + 1), cursor(V);
  WM_CUDA(cudaMemset(vc.p, 0, sizeof(int) * (V + 1)));
  k_count<<<blocks(3LL * m.T), 256>>>(3 * m.T, m.tri.p, vc.p);
  check_launch();
  m.vtri_off.resize(V + 1);
  exclusive_scan(vc.p, m.vtri_off.p, V);
  m.vtri_items.resize(3 * static_cast<size_t>(m.T));
  WM_CUDA(cudaMemset(cursor.p, 0, sizeof(int) * V));
  k_vtri_fill<<<blocks(m.T), 256>>>(m.T, m.tri.p, m.vtri_off.p, cursor.p, m.vtri_items.p);
  check_launch();
  k_sort_segments<<<blocks(V), 256>>>(V, m.vtri_off.p, m.vtri_items.p);
  check_launch();
  WM_CUDA(cudaDeviceSynchronize());
}

thread_local std::string g_model_err;

template <class Fn>
int run(Fn&& fn) {
  try {
    fn();
    return WT_OK;
  } catch (const Fail& f) {
    g_model_err = f.msg;
    return f.code;
  } catch (const std::exception& e) {
    g_model_err = e.what();
    return WT_EINVAL;
  }
}

}  // namespace

extern "C" {

const char* wt_gpu_mesh_last_error(void) { return g_model_err.c_str(); }

int wt_gpu_mesh_subdivide(int device, int32_t n_vertices, int32_t n_links, const double* v0, const double* phi,
                          const int32_t* weight_count, const int32_t* weight_link, const double* weight,
                          int32_t n_polys, const int32_t* poly_offsets, const int32_t* poly_items,
                          int32_t iterations, int32_t k_neighbors, wt_mesh** out) {
  if (!out) return WT_EINVAL;
  *out = nullptr;
  auto* m = new wt_mesh();
  const int rc = run([&] {
    if (n_vertices < 0 || n_links <= 0 || n_polys < 0 || iterations < 0 || !v0 || !weight_count || !weight_link ||
        !weight || (n_polys > 0 && (!poly_offsets || !poly_items)))
      throw Fail{WT_EINVAL, "subdivide: bad arguments"};
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw Fail{WT_ENODEV, "no CUDA device available"};
    }
    WM_CUDA(cudaSetDevice(device));
    const int V = n_vertices, L = n_links;
    m->device = device;
    m->V = V;
    m->L = L;
    m->F = n_polys;
    m->NI = n_polys > 0 ? poly_offsets[n_polys] : 0;
    m->pos.upload(v0, 3 * static_cast<size_t>(V));
    std::vector<double> ph(3 * static_cast<size_t>(V), 0.0);
    if (phi) std::copy(phi, phi + 3 * static_cast<size_t>(V), ph.begin());
    m->phi.upload(ph.data(), ph.size());
    m->foff.upload(poly_offsets, static_cast<size_t>(n_polys) + 1);
    m->fitems.upload(poly_items, static_cast<size_t>(m->NI));
    for (int k = 0; k < m->NI; ++k)
      if (poly_items[k] < 0 || poly_items[k] >= V) throw Fail{WT_EINVAL, "subdivide: polygon vertex out of range"};
    if (iterations > 0) {
      // the WeightMap of every vertex, dense (accumulate_weights(m, w, 1.0))
      std::vector<double> W(static_cast<size_t>(V) * L, 0.0);
      for (int i = 0; i < V; ++i)
        for (int s = 0; s < weight_count[i] && s < 4; ++s) {
          const int l = weight_link[4 * i + s];
          if (l < 0 || l >= L) throw Fail{WT_EINVAL, "subdivide: weight link out of range"};
          W[static_cast<size_t>(i) * L + l] += 1.0 * weight[4 * i + s];
        }
      m->W.upload(W.data(), W.size());
      for (int it = 0; it < iterations; ++it) subdivide_once(*m);
      m->wcount.resize(m->V);
      m->wlink.resize(4 * static_cast<size_t>(m->V));
      m->wval.resize(4 * static_cast<size_t>(m->V));
      k_truncate<<<blocks(m->V), 256>>>(m->V, L, m->W.p, m->wcount.p, m->wlink.p, m->wval.p);
      check_launch();
      m->W.resize(0);
    } else {  // finalize / neighbours only: the weight rows as given
      m->weights_dense = false;
      m->wcount.upload(weight_count, static_cast<size_t>(V));
      m->wlink.upload(weight_link, 4 * static_cast<size_t>(V));
      m->wval.upload(weight, 4 * static_cast<size_t>(V));
    }
    finalize(*m);
    if (k_neighbors > 0) knn(m->V, m->pos, k_neighbors, m->nbr, m->K);
    WM_CUDA(cudaDeviceSynchronize());
  });
  if (rc != WT_OK) {
    delete m;
    return rc;
  }
  *out = m;
  return WT_OK;
}

int wt_gpu_mesh_sizes(const wt_mesh* m, int32_t* n_vertices, int32_t* n_polys, int32_t* n_poly_items,
                      int32_t* n_triangles, int32_t* n_neighbors_per_vertex) {
  if (!m) return WT_EINVAL;
  if (n_vertices) *n_vertices = m->V;
  if (n_polys) *n_polys = m->F;
  if (n_poly_items) *n_poly_items = m->NI;
  if (n_triangles) *n_triangles = m->T;
  if (n_neighbors_per_vertex) *n_neighbors_per_vertex = m->K;
  return WT_OK;
}

int wt_gpu_mesh_export(const wt_mesh* m, double* v0, double* phi, int32_t* weight_count, int32_t* weight_link,
                       double* weight, int32_t* poly_offsets, int32_t* poly_items, int32_t* triangles,
                       int32_t* vtri_offsets, int32_t* vtri_items, int32_t* neighbors) {
  if (!m) return WT_EINVAL;
  return run([&] {
    WM_CUDA(cudaSetDevice(m->device));
    const size_t V = static_cast<size_t>(m->V);
    m->pos.download(v0, 3 * V);
    m->phi.download(phi, 3 * V);
    m->wcount.download(weight_count, V);
    m->wlink.download(weight_link, 4 * V);
    m->wval.download(weight, 4 * V);
    m->foff.download(poly_offsets, static_cast<size_t>(m->F) + 1);
    m->fitems.download(poly_items, static_cast<size_t>(m->NI));
    m->tri.download(triangles, 3 * static_cast<size_t>(m->T));
    m->vtri_off.download(vtri_offsets, V + 1);
    m->vtri_items.download(vtri_items, 3 * static_cast<size_t>(m->T));
    if (m->K > 0) m->nbr.download(neighbors, V * m->K);
  });
}

void wt_gpu_mesh_free(wt_mesh* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  delete m;
}

int wt_gpu_build_neighbors(int device, int32_t n, const double* v0, int32_t k, int32_t* out) {
  return run([&] {
    if (n < 0 || (n > 0 && !v0) || !out) throw Fail{WT_EINVAL, "build_neighbors: bad arguments"};
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw Fail{WT_ENODEV, "no CUDA device available"};
    }
    WM_CUDA(cudaSetDevice(device));
    DArr<double> dv;
    dv.upload(v0, 3 * static_cast<size_t>(n));
    DArr<int> nb;
    int want = 0;
    knn(n, dv, k, nb, want);
    nb.download(out, static_cast<size_t>(n) * want);
  });
}

}  // extern "C"
