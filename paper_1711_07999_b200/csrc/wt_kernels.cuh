// wt_kernels.cuh -- sm_100a kernels for one tracking frame.
//
// Per pose iteration (kinopt.cpp:139-170) the frame graph runs
//   k_skin -> k_normals(+bin histogram, last CTA scans) -> k_scatter
//   -> k_search(+scatter-average) -> k_pose_system(last CTA: reduce, damped
//   Cholesky, theta update, FK/dchain for the next iteration)
// and per shape iteration (shapeopt.cpp:58-110)
//   k_skin -> k_normals -> k_scatter -> k_search -> k_shape(last CTA: stats).
// Everything stays on the device; reductions are deterministic (fixed-point
// integer atomics are associative), so a frame is bitwise reproducible.
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>
#include <cstdint>

#include "wt_dq.cuh"

namespace wt {

constexpr int kVThreads = 256;    // per-vertex / per-pixel kernels
// Fixed-point reductions. Every cross-thread sum of the frame is a 64-bit
// integer sum (associative, so bitwise reproducible whatever the schedule),
// at a power-of-two scale chosen so no sum can leave the int64 range in any
// length unit (the reference sums in fp64 and works in metres or
// millimetres alike):
//  - observation sums: 2^e per frame, from the largest coordinate magnitude of
//    the frame's valid points (k_ingest) -- a vertex collects at most
//    (2*16+1)^2 < 2^11 points, so e = min(44, 51 - ceil(log2 max|x|)): 2^-44 m
//    for metre-scale scenes, 2^-39 mm for millimetre depth;
//  - JtJ / Jtr and sum r^2: per call from the vertex count, the model's lever
//    arm and the cutoff (pose_scales, wt_gpu.cu): 2^-40 / 2^-44 at metre scale;
//    k_pose_solve still checks the non-negative sums (diagonal, sum r^2) for
//    wrap-around and reports WT_ERANGE instead of taking a garbage step;
//  - the shape statistics are fp64 per-CTA partials folded in CTA order.
constexpr int kObsExpMax = 44, kObsExpBudget = 51;
constexpr int kRedCopies = 8;  // CTAs spread their fixed-point atomics over this many slot copies

struct DevModel {
  int V, L, NP, K;
  const double4* v0;       // template vertices (x,y,z,0), fp64
  const double4* wgt;      // skin weights, entry order kept (entry 0 = pivot)
  const uchar4* wlink;     // skin links, 0xFF = unused
  const int* ring_off;     // [V+1] incident triangles of each vertex (CSR order)
  const int2* ring;        // (b,c) follow i in its triangle; bits 30-31 of b: position of i
  const int* fan_nb;       // [V*8] ring neighbours in fan order n_0..n_{k-1}, then n_0 again (k < 8),
                           // -1 padded; -2 in slot 0: not a closed fan of <= 8 triangles, use the CSR
  const unsigned long long* fan_code;  // [V] bits 2j..2j+1: rot of fan triangle j = (i, n_j, n_j+1);
                                       // bits 16+3t..: fan position of CSR triangle t; bits 40..43: k
  const int* nbr;          // [K][V] neighbour ELL, -1 padded
  const LinkDesc* links;   // [L]
  const int* pair_off;     // [L+1] dchain pairs of each link
  const int* pair_theta;   // [NP] theta index k of the pair
  const int* pair_link;    // [NP] link driven by theta k
  const int* pair_owner;   // [NP] link j the pair belongs to
  const double* s_diag;    // [L] influence counts S
  const int* link_depth;   // [L] depth in the tree (root 0)
  int max_depth;
  const unsigned* pose_e;  // [NE] JtJ/Jtr entry e -> (row | col << 16), col = L for Jtr
};

struct DevIntr {
  double fx, fy, cx, cy;
  int W, H;
};

struct KinStat {      // per pose iteration (device)
  double residual_sum;
  double step_norm;
  int associated;
  int skipped;
};

struct ShapeStat {    // per shape iteration (device)
  double mean_phi, max_phi, mean_abs_r_before, mean_abs_r_after;
  int singular;
  int pad;
};

struct DevState {
  double* theta;      // [L]
  double* fk;         // [L*8]
  double* offsets;    // [L*8] H_jD = H_0j * inverse(bind_j)
  double* dchain;     // [NP*8]
  double4* pv;        // posed vertices (x,y,z, blend ok), fp64
  float4* pn;         // normals (x,y,z, valid)
  int* vpix;          // bucket pixel (row-major) or -1
  int* pix_cnt;       // [P] bucket sizes (self-cleaning: k_scatter counts them back down to 0)
  int* row_cnt;       // [H] bucketed vertices per image row (cleared by k_scatter)
  int* poff;          // [P+1] row-major pixel offsets: the VertexBuckets CSR
  double4* items;     // bucketed vertices in pixel order (x,y,z, bits: vertex index)
  unsigned long long* acc;   // [V*4] fixed-point sums x,y,z + count (one 256-bit record)
  unsigned long long* red;   // reduction slots (self-cleaning)
  unsigned* tickets;         // last-CTA tickets (self-cleaning)
  KinStat* kin_stats;
  ShapeStat* shape_stats;
  double* sys_out;           // optional JtJ/Jtr dump [L*L + L]
  const int* fwords;         // the frame's words: [0] valid-pixel list length, [2..3] max |coordinate| bits
  double* spart;             // shape statistics: 5 fp64 partials per CTA
  long long bstride;         // bytes between the arenas of consecutive sequences of a batch
};

struct DevFrame {
  const uint8_t* valid;  // per pixel
  const double* pts_hi;  // per pixel fp64 point (valid pixels only)
  const double4* vpts;   // valid-pixel list: the pixel's point and index (bits of .w; -1 padding)
  const int* n_valid;
  long long bstride;
};

// ---------------------------------------------------------------------------
// Batched sequences. Every per-sequence buffer (state, phi, frame) of a
// batch of B independent sequences lives in one arena per sequence, all
// arenas the same layout and `bstride` bytes apart, so sequence b's buffers
// are sequence 0's pointers + b * bstride. A batched launch puts the
// sequence in blockIdx.y (gridDim.y = B) and every frame kernel rebases its
// pointers on entry; the model (DevModel) is shared. Every frame kernel is
// instantiated twice: B = false (one sequence, no rebasing -- the pointers
// stay in the constant bank) and B = true (batched launches).
template <class T>
__device__ __forceinline__ T* seq_ptr(T* p, long long off) {
  return p ? reinterpret_cast<T*>(reinterpret_cast<unsigned long long>(p) + off) : p;
}

// A negative stride walks the batch backwards: blockIdx.y = 0 is the last
// sequence (the host alternates the direction from launch to launch, seq_walk).
__device__ __forceinline__ long long seq_off(long long bstride) {
  return bstride >= 0 ? static_cast<long long>(blockIdx.y) * bstride
                      : static_cast<long long>(gridDim.y - 1 - blockIdx.y) * -bstride;
}

__device__ inline DevState seq_state(DevState s) {
  const long long o = seq_off(s.bstride);
  if (o == 0) return s;
  s.theta = seq_ptr(s.theta, o);
  s.fk = seq_ptr(s.fk, o);
  s.offsets = seq_ptr(s.offsets, o);
  s.dchain = seq_ptr(s.dchain, o);
  s.pv = seq_ptr(s.pv, o);
  s.pn = seq_ptr(s.pn, o);
  s.vpix = seq_ptr(s.vpix, o);
  s.pix_cnt = seq_ptr(s.pix_cnt, o);
  s.row_cnt = seq_ptr(s.row_cnt, o);
  s.poff = seq_ptr(s.poff, o);
  s.items = seq_ptr(s.items, o);
  s.acc = seq_ptr(s.acc, o);
  s.red = seq_ptr(s.red, o);
  s.tickets = seq_ptr(s.tickets, o);
  s.kin_stats = seq_ptr(s.kin_stats, o);
  s.shape_stats = seq_ptr(s.shape_stats, o);
  s.sys_out = seq_ptr(s.sys_out, o);
  s.fwords = seq_ptr(s.fwords, o);
  s.spart = seq_ptr(s.spart, o);
  return s;
}

__device__ inline DevFrame seq_frame(DevFrame f) {
  const long long o = seq_off(f.bstride);
  if (o == 0) return f;
  f.valid = seq_ptr(f.valid, o);
  f.pts_hi = seq_ptr(f.pts_hi, o);
  f.vpts = seq_ptr(f.vpts, o);
  f.n_valid = seq_ptr(f.n_valid, o);
  return f;
}

// ---------------------------------------------------------------------------
// 256-bit global accesses. sm_100 has 32-byte vector loads and stores
// (LDG/STG.E.ENL2.256): a double4 record (posed vertex, bucket item, phi,
// skin weights, observation sums) moves in ONE L1 wavefront instead of the two
// 128-bit halves the compiler emits for a double4, which halves the L1 work
// of the gather-heavy kernels (normals, search, shape). Every buffer these
// touch is 32-byte aligned (256-byte carve, wt_gpu.cu). The loads go through
// the non-coherent path: nothing a kernel reads this way is written by the
// same kernel. They are volatile so they stay behind the PDL wait
// (pdl_entry) like every other access.
__device__ __forceinline__ double4 ld256(const double4* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
// From L2 (reads issued before a PDL wait: never a stale L1 line).
__device__ __forceinline__ double4 ld256_cg(const double4* p) {
  double4 v;
  asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ ulonglong4 ld256(const ulonglong4* p) {
  ulonglong4 v;
  asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st256(double4* p, double4 v) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
               : "memory");
}
__device__ __forceinline__ void st256(ulonglong4* p, ulonglong4 v) {
  asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v.x), "l"(v.y), "l"(v.z), "l"(v.w)
               : "memory");
}

// The observation sums are self-cleaning: the kernel that consumes an
// association last (the pose system before the next re-association, the
// shape step, the stats pass) zeroes the sums it read, so k_normals need not
// clear all V of them before every search.
__device__ __forceinline__ void clear_obs(const DevState& s, int i) {
  st256(reinterpret_cast<ulonglong4*>(s.acc) + i, make_ulonglong4(0ull, 0ull, 0ull, 0ull));
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch: the frame graph's kernels are launched with
// programmatic stream serialisation, so kernel N+1's CTAs become resident
// while kernel N drains (hiding the launch gap); each kernel lets its
// successor launch right away and waits for its predecessor's memory before
// touching any of it. Without PDL both instructions are no-ops.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// k_search and k_normals release their dependents only after their own
// wait: once a CTA of their successor runs, every kernel before its
// predecessor has completed, and it may read that output before its own
// wait (pdl_wait) -- k_pose_system and k_pose_solve the FK output of the
// previous pose solve, k_shape phi and the posed mesh.
__device__ __forceinline__ void pdl_entry_ordered() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool use_pdl = getenv("WT_NO_PDL") == nullptr;  // A/B switch for measurements
  cfg.attrs = attr;
  cfg.numAttrs = use_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------------------
// small helpers

__device__ __forceinline__ long long fix(double x, double scale) {
  return __double2ll_rn(x * scale);
}

// Global-memory atomics in explicit PTX. A batched kernel rebases its
// pointers per sequence (seq_state), after which the compiler can no longer
// prove they address global memory: atomicAdd then compiles to a generic
// ATOM.E plus a shared-memory CAS fallback path, and a result-less add no
// longer becomes the fire-and-forget RED. Every pointer passed here is global.
__device__ __forceinline__ void red_add(unsigned long long* p, long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)),
               "l"(static_cast<unsigned long long>(v))
               : "memory");
}

__device__ __forceinline__ void red_add(int* p, int v) {
  asm volatile("red.global.add.s32 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "r"(v) : "memory");
}

__device__ __forceinline__ void red_max(unsigned long long* p, unsigned long long v) {
  asm volatile("red.global.max.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
}

__device__ __forceinline__ int atom_add(int* p, int v) {
  int old;
  asm volatile("atom.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(__cvta_generic_to_global(p)), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ unsigned atom_add(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(__cvta_generic_to_global(p)), "r"(v) : "memory");
  return old;
}

// inv_scale = 1 / scale, exact: every fixed-point scale is a power of two
// (a multiplication instead of an fp64 division per value)
__device__ __forceinline__ double unfix(unsigned long long v, double inv_scale) {
  return static_cast<double>(static_cast<long long>(v)) * inv_scale;
}

// Scale of the frame's observation sums (see kObsExpBudget) from the largest
// coordinate magnitude k_ingest recorded in frame words [2..3]: 2^e with
// e = min(44, 51 - ex), max_abs < 2^ex, built from the exponent bits.
// (inverse = true: 2^-e, for unfix)
__host__ __device__ inline double obs_scale_of_bits(long long bits, bool inverse = false) {
  const int biased = static_cast<int>((bits >> 52) & 0x7FF);
  const int ex = biased == 0 ? 0 : biased - 1022;  // frexp's exponent (0 for zero / subnormal)
  const int e = kObsExpBudget - ex < kObsExpMax ? kObsExpBudget - ex : kObsExpMax;
  union {
    long long i;
    double d;
  } u;
  u.i = static_cast<long long>((inverse ? -e : e) + 1023) << 52;
  return u.d;
}

// 2^n for -1022 <= n <= 1023, from the exponent bits
__host__ __device__ inline double exp2i(int n) {
  union {
    long long i;
    double d;
  } u;
  u.i = static_cast<long long>(n + 1023) << 52;
  return u.d;
}

__device__ __forceinline__ double obs_scale(const int* fwords, bool inverse = false) {
  return obs_scale_of_bits(__ldcg(reinterpret_cast<const long long*>(fwords + 2)), inverse);
}

// Returns true in every thread of the CTA that finished last (grid-wide),
// after a fence; resets the ticket.
__device__ __forceinline__ bool last_block(unsigned* ticket) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atom_add(ticket, 1u);
    is_last = (t == gridDim.x - 1);  // per sequence (blockIdx.y)
    if (is_last) *ticket = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// Block-wide exclusive scan over n ints in shared memory (in place);
// returns the total. blockDim.x must be a multiple of 32.
__device__ inline int block_exclusive_scan(int* a, int n) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int x = i < n ? a[i] : 0;
    int s = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane == 31) warp_tot[wid] = s;
    __syncthreads();
    if (wid == 0) {
      int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      if (lane < nw) warp_tot[lane] = t;
    }
    __syncthreads();
    const int excl = carry + (wid > 0 ? warp_tot[wid - 1] : 0) + s - x;
    if (i < n) a[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + x;
    __syncthreads();
  }
  return carry;
}

// Block-wide sum of a double and an int (result valid in thread 0).
__device__ __forceinline__ void block_sum2(double& d, long long& n) {
  __shared__ double sd[32];
  __shared__ long long sn[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    n += __shfl_xor_sync(0xffffffffu, n, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) {
    sd[wid] = d;
    sn[wid] = n;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    d = 0.0;
    n = 0;
    for (int k = 0; k < nw; ++k) {  // fixed order
      d += sd[k];
      n += sn[k];
    }
  }
  __syncthreads();
}

// Loads link offsets (and optionally the dchain) into shared memory.
__device__ __forceinline__ void load_offsets(const DevModel& m, const DevState& s, double* s_off) {
  for (int i = threadIdx.x; i < m.L * 8; i += blockDim.x) s_off[i] = s.offsets[i];
}

// Dual-quaternion blend of one vertex (skinmesh.cpp:60-77): raw sum with the
// antipodality signs. Returns false when the real part collapsed.
__device__ __forceinline__ bool blend_vertex(const double* s_off, double4 w, uchar4 lk, DQ& raw,
                                             double sign[4]) {
  const unsigned char li[4] = {lk.x, lk.y, lk.z, lk.w};
  const double wi[4] = {w.x, w.y, w.z, w.w};
  for (int c = 0; c < 4; ++c) raw.r[c] = raw.d[c] = 0.0;
  sign[0] = sign[1] = sign[2] = sign[3] = 1.0;
  if (li[0] == 0xFF) return false;  // no weights: blend not ok
  const double* pivot = s_off + 8 * li[0];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (li[e] == 0xFF) break;
    const double* h = s_off + 8 * li[e];
    const double dot = pivot[0] * h[0] + pivot[1] * h[1] + pivot[2] * h[2] + pivot[3] * h[3];
    const double sg = dot < 0.0 ? -1.0 : 1.0;
    sign[e] = sg;
    const double k = sg * wi[e];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      raw.r[c] += h[c] * k;
      raw.d[c] += h[4 + c] * k;
    }
  }
  const double n = sqrt(raw.r[0] * raw.r[0] + raw.r[1] * raw.r[1] + raw.r[2] * raw.r[2] +
                        raw.r[3] * raw.r[3]);
  return n > 1e-12;
}

// ---------------------------------------------------------------------------
// FK / link offsets / dchain for the current theta (skeleton.cpp:56-108),
// executed by one whole CTA. Also used by the pose-solve tail.

// The link table and tree depths block_fk reads, staged in shared memory
// ahead of time (the pose kernel stages them in its prologue so its solve
// tail pays no global-memory latency for them).
struct FkTables {
  LinkDesc sl[64];
  int dep[64];
};

__device__ __forceinline__ void fk_stage(const DevModel& m, FkTables& t) {
  const int n4 = m.L * static_cast<int>(sizeof(LinkDesc) / sizeof(double));
  const double* src = reinterpret_cast<const double*>(m.links);
  double* dst = reinterpret_cast<double*>(t.sl);
  for (int k = threadIdx.x; k < n4; k += blockDim.x) dst[k] = src[k];
  for (int j = threadIdx.x; j < m.L; j += blockDim.x) t.dep[j] = m.link_depth[j];
}

// Requires fk_stage(m, t) and a barrier before the call.
__device__ inline void fk_run(const DevModel& m, const DevState& s, const double* theta_in, const FkTables& t,
                       long long* stamps = nullptr) {
  __shared__ DQ fk[64];
  __shared__ DQ loc[64];
  __shared__ double cs[64][2];
  const int L = m.L;
  const LinkDesc* sl = t.sl;
  // this thread's first dchain pair indices, in flight during the FK chain
  const int p0 = threadIdx.x;
  const int own0 = p0 < m.NP ? __ldg(m.pair_owner + p0) : 0;
  const int lnk0 = p0 < m.NP ? __ldg(m.pair_link + p0) : 0;
  // joint transforms and local offsets in parallel (one link per thread);
  // each joint's half-angle sincos is evaluated once ...
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    const LinkDesc& l = sl[j];
    const double th = theta_in[l.theta_index];
    double sn, cn;
    sincos(th * 0.5, &sn, &cn);
    cs[j][0] = cn;
    cs[j][1] = sn;
    loc[j] = dq_compose(dq_load(l.offset), dq_joint_cs(l.kind, l.axis, th, cn, sn));
  }
  __syncthreads();
  if (stamps && threadIdx.x == 0) stamps[0] = clock64();
  // ... then every link's chain independently, composed from the root down
  // (the same left fold as forward_kinematics, so bitwise the same result)
  // with no barrier per tree level ...
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    int path[64];
    int n = 0;
    for (int q = j; q >= 0; q = sl[q].parent) path[n++] = q;
    DQ acc = loc[path[n - 1]];
    for (int d = n - 2; d >= 0; --d) acc = dq_compose(acc, loc[path[d]]);
    fk[j] = acc;
  }
  __syncthreads();
  if (stamps && threadIdx.x == 0) stamps[1] = clock64();
  // ... then offsets and the dchain blocks in parallel (skeleton.cpp:71-108)
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    dq_store(fk[j], s.fk + 8 * j);
    dq_store(dq_compose(fk[j], dq_load(sl[j].bind_inv)), s.offsets + 8 * j);
  }
  for (int p = threadIdx.x; p < m.NP; p += blockDim.x) {
    const int j = p == p0 ? own0 : m.pair_owner[p], kl = p == p0 ? lnk0 : m.pair_link[p];
    const LinkDesc& lk = sl[kl];
    const DQ off = dq_load(lk.offset);
    const DQ pre = lk.parent < 0 ? off : dq_compose(fk[lk.parent], off);
    const DQ dj = dq_djoint_cs(lk.kind, lk.axis, cs[kl][0], cs[kl][1]);
    const DQ k_to_j = dq_compose(dq_inverse(fk[kl]), fk[j]);
    dq_store(dq_compose(dq_compose(pre, dj), dq_compose(k_to_j, dq_load(sl[j].bind_inv))), s.dchain + 8 * p);
  }
}

__device__ inline void block_fk(const DevModel& m, const DevState& s, const double* theta_in) {
  __shared__ FkTables t;
  fk_stage(m, t);
  __syncthreads();
  fk_run(m, s, theta_in, t);
}

template <bool B>
static __global__ void k_fk(DevModel m, DevState s) {
  pdl_entry();
  if constexpr (B) s = seq_state(s);
  block_fk(m, s, s.theta);
}


// ---------------------------------------------------------------------------
// frame ingest: depth_to_cloud (seqio.cpp:419-437) in fp64 and the list of
// valid pixels. CTAs cover 256-pixel segments of one image row; each warp
// compacts the valid pixels of its 32 columns in image order into a run
// padded with -1 to a multiple of 4 entries, so the 4 pixels of a search
// warp are row neighbours from at most two 32-column segments.

constexpr int kIngestSeg = 256;
constexpr int kRunAlign = 4;  // valid-pixel runs padded to 4 entries (a batch search warp's pixels)

template <bool B>
static __global__ void __launch_bounds__(kIngestSeg) k_ingest(DevIntr in, const float* depth, double scale,
                                                      const double* cloud, const uint8_t* cloud_valid,
                                                      uint8_t* pvalid, double* pts_hi, double4* vpts,
                                                      int* n_valid, long long bstride) {
  if constexpr (B) {  // sequence blockIdx.y of a batch (see seq_state)
    const long long o = seq_off(bstride);
    depth = seq_ptr(depth, o);
    cloud = seq_ptr(cloud, o);
    cloud_valid = seq_ptr(cloud_valid, o);
    pvalid = seq_ptr(pvalid, o);
    pts_hi = seq_ptr(pts_hi, o);
    vpts = seq_ptr(vpts, o);
    n_valid = seq_ptr(n_valid, o);
  }
  const int segs = (in.W + kIngestSeg - 1) / kIngestSeg;
  const int v = blockIdx.x / segs;
  const int u = (blockIdx.x % segs) * kIngestSeg + threadIdx.x;
  const int i = v * in.W + u;
  int valid = 0;
  double mx = 0.0;  // max |coordinate| of this pixel's point
  double x = 0, y = 0, z = 0;
  if (u < in.W) {
    if (depth) {
      const float d = depth[i];
      if (d > 0.0f && isfinite(d)) {
        z = static_cast<double>(d) * scale;
        x = (u - in.cx) / in.fx * z;
        y = (v - in.cy) / in.fy * z;
        valid = 1;
      }
    } else {
      valid = cloud_valid[i] != 0;
      if (valid) {
        x = cloud[3 * i];
        y = cloud[3 * i + 1];
        z = cloud[3 * i + 2];
      }
    }
    pvalid[i] = static_cast<uint8_t>(valid);
    if (valid) {
      pts_hi[3 * i] = x;
      pts_hi[3 * i + 1] = y;
      pts_hi[3 * i + 2] = z;
      mx = fmax(fabs(x), fmax(fabs(y), fabs(z)));
    }
  }
  const int lane = threadIdx.x & 31;
  {
    // largest coordinate magnitude of the frame (the observation-sum scale):
    // a warp maximum, then one integer atomicMax on the bits (non-negative
    // doubles order like their bit patterns)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx > 0.0)
      red_max(reinterpret_cast<unsigned long long*>(n_valid + 2), static_cast<unsigned long long>(__double_as_longlong(mx)));
  }
  const unsigned m = __ballot_sync(0xffffffffu, valid);
  if (m) {
    // a run padded to a multiple of kRunAlign (the pixels of one search warp)
    const int n = __popc(m), padded = (n + kRunAlign - 1) & ~(kRunAlign - 1);
    int base = 0;
    if (lane == 0) base = atom_add(n_valid, padded);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (valid)
      st256(vpts + base + __popc(m & ((1u << lane) - 1u)),
            make_double4(x, y, z, __longlong_as_double(static_cast<long long>(i))));
    if (lane >= n && lane < padded) st256(vpts + base + lane, make_double4(0.0, 0.0, 0.0, __longlong_as_double(-1ll)));
  }
}


// ---------------------------------------------------------------------------
// K1 skinning: v = normalize(blend)(v0 + phi) (skinmesh.cpp:112-121).

// One vertex: offsets in shared memory, every load issued before the arithmetic.
// The model's weights and template vertex (constants) may come preloaded.
struct SkinConst {
  double4 wv, a;
  uchar4 lk;
};
__device__ __forceinline__ SkinConst skin_const(const DevModel& m, int i) {
  return {ld256(m.wgt + i), ld256(m.v0 + i), m.wlink[i]};
}
__device__ __forceinline__ void skin_vertex(const DevModel& m, const DevState& s, const double4* phi,
                                            const double* s_off, int i, const SkinConst& k) {
  const double4 f = ld256(phi + i);
  const double4 wv = k.wv, a = k.a;
  const uchar4 lk = k.lk;
  const double rest[3] = {a.x + f.x, a.y + f.y, a.z + f.z};
  DQ raw;
  double sign[4];
  double4 out;
  if (blend_vertex(s_off, wv, lk, raw, sign)) {
    double p[3];
    dq_transform_point(dq_normalize(raw), rest, p);
    out = make_double4(p[0], p[1], p[2], 1.0);
  } else {
    out = make_double4(rest[0], rest[1], rest[2], 0.0);  // placeholder, excluded downstream
  }
  st256(s.pv + i, out);
}

template <bool B>
static __global__ void __launch_bounds__(kVThreads) k_skin(DevModel m, DevState s, const double4* phi) {
  // the first vertex's model constants load before the wait, under the
  // predecessor's tail (the one-CTA pose solve, at C3 ~10 us)
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  SkinConst k0{};
  if (i0 < m.V) k0 = skin_const(m, i0);
  pdl_entry();
  if constexpr (B) s = seq_state(s);
  if constexpr (B) phi = seq_ptr(phi, seq_off(s.bstride));
  extern __shared__ double s_off[];
  load_offsets(m, s, s_off);
  __syncthreads();
  if (i0 < m.V) skin_vertex(m, s, phi, s_off, i0, k0);
  // grid-stride: a batch launches fewer, longer-lived CTAs per sequence
  for (int i = i0 + gridDim.x * blockDim.x; i < m.V; i += gridDim.x * blockDim.x)
    skin_vertex(m, s, phi, s_off, i, skin_const(m, i));
}

// One of eight register values by a 3-bit slot (a select tree, no local memory).
__device__ __forceinline__ double pick8(const double (&a)[8], unsigned k) {
  const double l0 = (k & 1u) ? a[1] : a[0], l1 = (k & 1u) ? a[3] : a[2];
  const double l2 = (k & 1u) ? a[5] : a[4], l3 = (k & 1u) ? a[7] : a[6];
  const double m0 = (k & 2u) ? l1 : l0, m1 = (k & 2u) ? l3 : l2;
  return (k & 4u) ? m1 : m0;
}

// acc += (f1 - f0) x (f2 - f0) for one incident triangle; (b, c) follow i in
// the triangle cyclically and rot is the position of i in it.
__device__ __forceinline__ void add_cross(unsigned rot, double vx, double vy, double vz, double bx, double by,
                                          double bz, double cx, double cy, double cz, double& ax, double& ay,
                                          double& az) {
  const double f0x = rot == 0 ? vx : (rot == 1 ? cx : bx), f1x = rot == 0 ? bx : (rot == 1 ? vx : cx),
               f2x = rot == 0 ? cx : (rot == 1 ? bx : vx);
  const double f0y = rot == 0 ? vy : (rot == 1 ? cy : by), f1y = rot == 0 ? by : (rot == 1 ? vy : cy),
               f2y = rot == 0 ? cy : (rot == 1 ? by : vy);
  const double f0z = rot == 0 ? vz : (rot == 1 ? cz : bz), f1z = rot == 0 ? bz : (rot == 1 ? vz : cz),
               f2z = rot == 0 ? cz : (rot == 1 ? bz : vz);
  const double ex = f1x - f0x, ey = f1y - f0y, ez = f1z - f0z;
  const double fx = f2x - f0x, fy = f2y - f0y, fz = f2z - f0z;
  ax += ey * fz - ez * fy;
  ay += ez * fx - ex * fz;
  az += ex * fy - ey * fx;
}

// The cross product (f1 - f0) x (f2 - f0) of one incident triangle, as add_cross.
__device__ __forceinline__ void fan_cross(unsigned rot, double vx, double vy, double vz, double bx, double by,
                                          double bz, double cx, double cy, double cz, double& ox, double& oy,
                                          double& oz) {
  const double f0x = rot == 0 ? vx : (rot == 1 ? cx : bx), f1x = rot == 0 ? bx : (rot == 1 ? vx : cx),
               f2x = rot == 0 ? cx : (rot == 1 ? bx : vx);
  const double f0y = rot == 0 ? vy : (rot == 1 ? cy : by), f1y = rot == 0 ? by : (rot == 1 ? vy : cy),
               f2y = rot == 0 ? cy : (rot == 1 ? by : vy);
  const double f0z = rot == 0 ? vz : (rot == 1 ? cz : bz), f1z = rot == 0 ? bz : (rot == 1 ? vz : cz),
               f2z = rot == 0 ? cz : (rot == 1 ? bz : vz);
  const double ex = f1x - f0x, ey = f1y - f0y, ez = f1z - f0z;
  const double fx = f2x - f0x, fy = f2y - f0y, fz = f2z - f0z;
  ox = ey * fz - ez * fy;
  oy = ez * fx - ex * fz;
  oz = ex * fy - ey * fx;
}

// Vertex normal exactly as skin() (skinmesh.cpp:125-139): per incident
// triangle (f0, f1, f2) in CSR order, acc += (v1 - v0) x (v2 - v0), then
// acc / |acc|; returns the PosedMesh valid flag (blend ok and |acc| > 1e-20).
// Bitwise the reference's when compiled without FMA contraction (wt_exact.cu).
//
// Fan path (closed fans of <= 8 triangles: every vertex of the meshes here):
// the k incident triangles of a closed, consistently wound fan are
// (i, n_j, n_j+1) around the ring, so the k distinct neighbours are gathered
// once, all in flight, one 256-bit load each (6 for 97 % of the vertices, not
// the 12 a per-triangle gather makes). Each fan triangle's cross product is
// formed from registers with static indices; only the CSR-order summation
// picks them by fan position (a select tree), so the arithmetic and its order
// are the reference's.
// q: the vertex's fan ids (fan_nb row, a model constant; k_normals loads
// the first vertex's before its PDL wait).
__device__ __forceinline__ bool vertex_normal_q(const DevModel& m, const double4* pv, int i, const double4& v,
                                                const ulonglong4& q, double& nx, double& ny, double& nz) {
  double ax = 0, ay = 0, az = 0;
  const int id[8] = {static_cast<int>(q.x), static_cast<int>(q.x >> 32), static_cast<int>(q.y),
                     static_cast<int>(q.y >> 32), static_cast<int>(q.z), static_cast<int>(q.z >> 32),
                     static_cast<int>(q.w), static_cast<int>(q.w >> 32)};
  if (id[0] != -2) {
    const unsigned long long code = __ldg(m.fan_code + i);
    const int k = static_cast<int>(code >> 40) & 15;
    double px[8], py[8], pz[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double4 g = id[j] >= 0 ? ld256(pv + id[j]) : v;  // padding slots load nothing
      px[j] = g.x;
      py[j] = g.y;
      pz[j] = g.z;
    }
    double cx[8], cy[8], cz[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int j1 = (j + 1) & 7;  // slot k holds n_0 again (k < 8); k = 8 wraps to slot 0
      cx[j] = cy[j] = cz[j] = 0.0;
      if (j < k) {
        const unsigned rot = static_cast<unsigned>(code >> (2 * j)) & 3u;
        fan_cross(rot, v.x, v.y, v.z, px[j], py[j], pz[j], px[j1], py[j1], pz[j1], cx[j], cy[j], cz[j]);
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (t >= k) break;
      const unsigned f = static_cast<unsigned>(code >> (16 + 3 * t)) & 7u;
      ax += pick8(cx, f);
      ay += pick8(cy, f);
      az += pick8(cz, f);
    }
  } else {
    // many-triangle vertices: the CSR, four triangles' gathers in flight at a time
    const int r0 = m.ring_off[i], r1 = m.ring_off[i + 1];
    for (int r = r0; r < r1; r += 4) {
      int2 bc[4];
      double4 pb[4], pc[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        bc[k] = r + k < r1 ? m.ring[r + k] : make_int2(-1, -1);
        const bool ok = bc[k].x != -1;
        pb[k] = ok ? ld256(pv + (bc[k].x & 0x3FFFFFFF)) : v;
        pc[k] = ok ? ld256(pv + bc[k].y) : v;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (r + k >= r1) break;
        add_cross(static_cast<unsigned>(bc[k].x) >> 30, v.x, v.y, v.z, pb[k].x, pb[k].y, pb[k].z, pc[k].x,
                  pc[k].y, pc[k].z, ax, ay, az);
      }
    }
  }
  const double len = sqrt(ax * ax + ay * ay + az * az);
  nx = ny = nz = 0.0;
  if (!(len > 1e-20)) return false;
  nx = ax / len;
  ny = ay / len;
  nz = az / len;
  return v.w != 0.0;
}
__device__ __forceinline__ ulonglong4 fan_ids(const DevModel& m, int i) {
  return ld256(reinterpret_cast<const ulonglong4*>(m.fan_nb + 8 * static_cast<size_t>(i)));
}
__device__ __forceinline__ bool vertex_normal(const DevModel& m, const double4* pv, int i, const double4& v,
                                              double& nx, double& ny, double& nz) {
  return vertex_normal_q(m, pv, i, v, fan_ids(m, i), nx, ny, nz);
}

// ---------------------------------------------------------------------------
// K2 normals (skinmesh.cpp:125-139) fused with K3a: back-face cull, projection
// with lround semantics (association.cpp:29-37,49-51) and the bin histogram.

// A batch is throughput-bound: three CTAs per SM (the register cap spills a
// little, which costs less than the lost occupancy). A lone sequence is
// latency-bound: two CTAs per SM, no spills.
template <bool B>
static __global__ void __launch_bounds__(kVThreads, B ? 3 : 2) k_normals(DevModel m, DevState s, DevIntr in,
                                                       int do_bucket, int zero_acc, int compute) {
  // the first vertex's fan ids (model constants) load before the wait
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  ulonglong4 q0 = make_ulonglong4(0ull, 0ull, 0ull, 0ull);
  if (compute && i0 < m.V) q0 = fan_ids(m, i0);
  pdl_entry_ordered();
  if constexpr (B) s = seq_state(s);
  // grid-stride: a batch launches fewer, longer-lived CTAs per sequence
  for (int i = i0; i < m.V; i += gridDim.x * blockDim.x) {
    const double4 v = ld256(s.pv + i);
    const double vx = v.x, vy = v.y, vz = v.z;
    double nx = 0, ny = 0, nz = 0;
    bool valid;
    if (compute) {
      valid = vertex_normal_q(m, s.pv, i, v, i == i0 ? q0 : fan_ids(m, i), nx, ny, nz);
      s.pn[i] = make_float4(static_cast<float>(nx), static_cast<float>(ny), static_cast<float>(nz),
                            valid ? 1.0f : 0.0f);
    } else {  // normals given (loose-vertex association)
      const float4 n = s.pn[i];
      nx = n.x;
      ny = n.y;
      nz = n.z;
      valid = n.w != 0.0f;
    }
    if (zero_acc) clear_obs(s, i);
    if (do_bucket) {
      // bucket_occupancy (association.cpp:39-56): per-pixel and per-row
      // counts as fire-and-forget reductions (no value comes back, so no
      // round trip); the slot inside the pixel is taken later, in k_scatter
      int pix = -1, row = -1;
      if (valid && !(nx * vx + ny * vy + nz * vz > 0.0) && vz > 0.0) {
        const double pu = in.fx * vx / vz + in.cx;
        const double pvv = in.fy * vy / vz + in.cy;
        const double ru = round(pu), rv = round(pvv);  // half away from zero, like lround
        if (ru >= 0.0 && rv >= 0.0 && ru < in.W && rv < in.H) {
          row = static_cast<int>(rv);
          pix = row * in.W + static_cast<int>(ru);
        }
      }
      if (pix >= 0) {
        red_add(&s.pix_cnt[pix], 1);
        red_add(&s.row_cnt[row], 1);
      }
      s.vpix[i] = pix;
    }
  }
}

// K3b: row-major pixel offsets of the bucket CSR (association.cpp:58-59),
// one warp per image row, no block barriers: the row's base is the sum of
// the preceding rows' counts (warp reduction); the row is read in coalesced
// 32-pixel chunks, all loads first, then scanned chunk by chunk with
// shuffles. (k_scatter counts the per-pixel sizes back down to zero.)

constexpr int kRowChunks = 64;  // rows up to 2048 pixels

template <bool B>
static __global__ void __launch_bounds__(kVThreads) k_pixoff(DevState s, int W, int H) {
  pdl_entry();
  if constexpr (B) s = seq_state(s);
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= H) return;
  // this row's counts first: their loads and the preceding rows' sums below
  // are in flight together
  int* cnt = s.pix_cnt + row * W;
  int* off = s.poff + row * W;
  const int nch = (W + 31) / 32;
  int v[kRowChunks];
#pragma unroll
  for (int t = 0; t < kRowChunks; ++t) {
    const int c = t * 32 + lane;
    v[t] = (t < nch && c < W) ? __ldcg(cnt + c) : 0;
  }
  int base = 0;
  {
    // sum of the preceding rows' counts: 16 loads in flight per lane
    constexpr int U = 16;
    for (int k0 = lane; k0 < row; k0 += 32 * U) {
      int v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + 32 * u;
        v[u] = k < row ? __ldcg(s.row_cnt + k) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) base += v[u];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) base += __shfl_xor_sync(0xffffffffu, base, o);
  int run = base;
#pragma unroll
  for (int t = 0; t < kRowChunks; ++t) {
    if (t >= nch) break;
    int incl = v[t];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int c = t * 32 + lane;
    if (c < W) {
      off[c] = run + incl - v[t];
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (row == H - 1 && lane == 0) s.poff[W * H] = run;
}

// K3c: scatter into pixel order (association.cpp:60-66; unordered within a
// pixel -- the winner rule is a lexicographic (d^2, index) minimum, so bucket
// order never changes a result). Clears the row counts for the next pass.
// One vertex (or row counter) of the scatter.
__device__ __forceinline__ void scatter_vertex(const DevModel& m, const DevState& s, int H, int i) {
  if (i < H) s.row_cnt[i] = 0;
  if (i >= m.V) return;
  const int pix = s.vpix[i];
  if (pix < 0) return;
  const double4 v = ld256(s.pv + i);
  // the bucket's slots are poff[pix] + (count - 1) .. poff[pix]: taken by
  // counting the bucket size back down, which leaves the counts at zero for
  // the next association (no cursor array, no clearing pass)
  st256(s.items + __ldg(s.poff + pix) + atom_add(&s.pix_cnt[pix], -1) - 1,
        make_double4(v.x, v.y, v.z, __longlong_as_double(static_cast<long long>(i))));
}

template <bool B>
static __global__ void __launch_bounds__(kVThreads) k_scatter(DevModel m, DevState s, int H) {
  pdl_entry();
  if constexpr (B) s = seq_state(s);
  const int n = max(m.V, H);
  // grid-stride: a batch launches fewer, longer-lived CTAs per sequence
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    scatter_vertex(m, s, H, i);
}


// ---------------------------------------------------------------------------
// K4 + K5: windowed nearest-vertex search (associate_winners,
// association.cpp:69-109) and the scatter-average accumulation
// (association.cpp:124-131), one thread per valid pixel. Window rows are
// contiguous spans of the bucket CSR as in the reference, and every distance
// is the reference's exact fp64 ((dx*dx + dy*dy) + dz*dz) (no FMA), so the
// winner map equals the reference's whenever the posed vertices do.
//
// Rings: for depth frames every point lies on its pixel's centre ray, so a
// vertex bucketed in Chebyshev ring k is at least lb(k) away (lround buckets
// put it (k - 1/2)/f off the ray in normalised coordinates on one axis; the
// half-space {x/z >= t + d} is d z / sqrt(1 + (t + d)^2) from the point).
// Scanning rings outward and stopping once lb(k)^2 exceeds the best (or the
// cutoff) yields the full-window answer from a few rings.

__device__ __forceinline__ double exact_d2(double4 v, double px, double py, double pz) {
  const double dx = __dsub_rn(v.x, px), dy = __dsub_rn(v.y, py), dz = __dsub_rn(v.z, pz);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

struct SearchArgs {
  double fx, fy, cx, cy;
  int prune;  // points lie on their pixel's centre ray (depth frames)
  int W, H;
  int window;
  double cut2;  // cutoff^2 (association.cpp:75,98)
  int write_winners;
  int* winners;
};

__device__ __forceinline__ double ring_lb2(int k, double atx, double aty, double ifx, double ify, double z) {
  const double dx = (k - 0.5) * ifx, dy = (k - 0.5) * ify;
  const double tx = atx + dx, ty = aty + dy;
  const double b = fmin(dx * rsqrt(1.0 + tx * tx), dy * rsqrt(1.0 + ty * ty)) * z;
  return b * b * (1.0 - 1e-9);
}

// Squared distances are non-negative doubles (never -0 or NaN for finite
// inputs), whose IEEE bit patterns order exactly like their values as signed
// 64-bit integers: the (d^2, index) minimum runs on integer compares, which
// keeps the loop-carried dependency a few cycles instead of a chain of fp64
// compares.
__device__ __forceinline__ long long d2_key(double x) { return __double_as_longlong(x); }

__device__ __forceinline__ void scan_span(const DevState& s, int e0, int e1, double px, double py, double pz,
                                          double cut2, double& best_x, int& best_i, int step = 1) {
  const long long ck = d2_key(cut2);
  long long bk = best_i < 0 ? LLONG_MAX : d2_key(best_x);
  auto consider = [&](const double4& it) {
    const long long xk = d2_key(exact_d2(it, px, py, pz));
    const int vi = static_cast<int>(__double_as_longlong(it.w));
    if (xk <= ck && (xk < bk || (xk == bk && vi < best_i))) {
      bk = xk;
      best_i = vi;
    }
  };
  for (int e = e0; e < e1; e += step) consider(ld256(s.items + e));
  if (best_i >= 0) best_x = __longlong_as_double(bk);
}

// Per-pixel result: the winner map entry and the scatter-average sums.
__device__ __forceinline__ void search_emit(const DevState& s, const SearchArgs& a, int pix, int best_i, double px,
                                            double py, double pz, double oscale) {
  if (a.write_winners) a.winners[pix] = best_i;
  if (best_i >= 0) {
    unsigned long long* acc = s.acc + 4 * static_cast<size_t>(best_i);
    red_add(acc + 0, fix(px, oscale));
    red_add(acc + 1, fix(py, oscale));
    red_add(acc + 2, fix(pz, oscale));
    red_add(acc + 3, 1ll);
  }
}

// k_search: a group of G lanes per valid pixel (32 / G pixels per warp, taken
// from the image-ordered 32-column runs of the valid-pixel list, so a warp's
// pixels are row neighbours and share cache lines). Phase 1: lane r of the
// group scans row r of the pixel's (2 K1 + 1)^2 core -- one span of the
// row-major bucket CSR each, all rows in parallel -- and the group reduces
// the lexicographic (d^2, index) minimum with shuffles. The pixel is finished
// when the exact ring bound lb(K1 + 1) exceeds that best (or the cutoff).
// Phase 2 (rare): the outermost ring K* that can still hold a winner or a tie
// is fixed from the phase-1 best, and the group's lanes scan the rows of the
// (2K*+1)^2 box outside the core, G rows at a time.
// Two instantiations (the result is the same exact minimum either way):
//  - one sequence (latency-bound): K1 = 2, G = 16, SPL = 3 -- a 5x5 core,
//    three lanes per core row each taking every third item of the row's
//    span, so a lane's dependent load chain is a third of the row (measured:
//    C3 1747 -> 1937 frames/s against one lane per row, G = 8);
//  - a batch (L1-throughput-bound): K1 = 1, G = 4, SPL = 1 -- a 3x3 core,
//    which already closes ~89 % of the pixels (the nearest vertex is usually
//    well inside lb(2)), so a pixel loads ~2.7x fewer bucket items; splitting
//    rows there only costs issue slots (G = 8 / SPL = 2: -4 %).
#ifndef WT_SEARCH_SOLO_G
#define WT_SEARCH_SOLO_G 16
#endif
#ifndef WT_SEARCH_SOLO_SPL
#define WT_SEARCH_SOLO_SPL 3
#endif
#ifndef WT_SEARCH_BATCH_G
#define WT_SEARCH_BATCH_G 4
#endif
#ifndef WT_SEARCH_BATCH_SPL
#define WT_SEARCH_BATCH_SPL 1
#endif
constexpr int kNearRingsSolo = 2, kSearchGroupSolo = WT_SEARCH_SOLO_G, kSearchSplitSolo = WT_SEARCH_SOLO_SPL;
constexpr int kNearRingsBatch = 1, kSearchGroupBatch = WT_SEARCH_BATCH_G, kSearchSplitBatch = WT_SEARCH_BATCH_SPL;

// Lexicographic (d^2, index) minimum over the G lanes of a group (lanes
// [g*G, g*G + G) of the warp); every lane of the group ends with it. A
// butterfly for power-of-two G, a fold over the group's lanes otherwise (the
// minimum does not depend on the order).
template <int G>
__device__ __forceinline__ void group_min(double& bx, int& bi) {
  auto take = [&](double ox, int oi) {
    if (oi >= 0 && (bi < 0 || ox < bx || (ox == bx && oi < bi))) {
      bx = ox;
      bi = oi;
    }
  };
  if constexpr ((G & (G - 1)) == 0) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) take(__shfl_xor_sync(0xffffffffu, bx, o), __shfl_xor_sync(0xffffffffu, bi, o));
  } else {
    const int lane = threadIdx.x & 31, base = lane - lane % G;
    const double x0 = bx;
    const int i0 = bi;
    bx = INFINITY;
    bi = -1;
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int src = min(base + t, 31);
      const double ox = __shfl_sync(0xffffffffu, x0, src);
      const int oi = __shfl_sync(0xffffffffu, i0, src);
      if (base + t < 32) take(ox, oi);
    }
  }
}

#ifndef WT_SEARCH_MINB_BATCH
#define WT_SEARCH_MINB_BATCH 5  // resident CTAs per SM the batch search is compiled for
#endif
template <bool B, int NR = B ? kNearRingsBatch : kNearRingsSolo, int G = B ? kSearchGroupBatch : kSearchGroupSolo,
          int SPL = B ? kSearchSplitBatch : kSearchSplitSolo>
static __global__ void __launch_bounds__(kVThreads, B ? WT_SEARCH_MINB_BATCH : 4) k_search(DevState s, DevFrame f,
                                                                                        SearchArgs a) {
  if constexpr (B) s = seq_state(s);
  if constexpr (B) f = seq_frame(f);
  if constexpr (B) a.winners = seq_ptr(a.winners, seq_off(s.bstride));
  const int lane = threadIdx.x & 31, sub = lane % G;
  constexpr int PPW = 32 / G;  // pixels per warp (lanes from PPW * G on idle)
  const int TW = gridDim.x * (blockDim.x >> 5);
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // The frame's pixel list and points (k_ingest, at the frame start: several
  // kernels back, complete once this CTA runs -- pdl_entry_ordered) of the
  // first pixel are read before the wait, from L2; the bucket lists after.
  // (A lone sequence only: a batch's CTAs loop over many pixels.)
  const int nv = __ldcg(f.n_valid);
  const double oscale = obs_scale(f.n_valid);
  // the list record (point, pixel) of this lane's pixel; a lone sequence
  // loads it one grid-stride step ahead: the first before the wait, the
  // next one as each step starts
  double4 rec = make_double4(0.0, 0.0, 0.0, __longlong_as_double(-1ll));
  const bool lane_on = lane < PPW * G;
  if constexpr (!B) {
    const int j = gw * PPW + lane / G;
    if (lane_on && j < nv) rec = ld256_cg(f.vpts + j);
  }
  pdl_entry_ordered();
  const int w = a.window;
  const int K1 = min(NR, w);
  const double ifx = 1.0 / a.fx, ify = 1.0 / a.fy;
  for (int base = gw * PPW; base < nv; base += TW * PPW) {
    if constexpr (B) {  // a batch: no registers to spare for the step ahead
      const int j = base + lane / G;
      rec = make_double4(0.0, 0.0, 0.0, __longlong_as_double(-1ll));
      if (lane_on && j < nv) rec = ld256(f.vpts + j);
    }
    const int pix = static_cast<int>(__double_as_longlong(rec.w));
    const double px = rec.x, py = rec.y, pz = rec.z;
    if constexpr (!B) {
      const int j = base + TW * PPW + lane / G;
      rec = make_double4(0.0, 0.0, 0.0, __longlong_as_double(-1ll));
      if (lane_on && j < nv) rec = ld256(f.vpts + j);
    }
    const bool act = pix >= 0;
    const int pu = pix % a.W, pv = pix / a.W;
    double best_x = INFINITY;
    int best_i = -1;
#ifndef WT_SEARCH_CORE_DEAL
#define WT_SEARCH_CORE_DEAL 1
#endif
    // the batch form (3x3 core, 4 lanes): the three core-row spans as one
    // list dealt round-robin to all 4 lanes (longest lane ~n/4 items, not the
    // longest row's n/3 with a lane idle)
    constexpr bool kDeal = WT_SEARCH_CORE_DEAL && B && G == 4 && SPL == 1 && NR == 1;
    if (kDeal && K1 == 1) {
      if (act) {
        const int c0 = max(pu - 1, 0), c1 = min(pu + 1, a.W - 1);
        int lo[3], n[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int rr = pv - 1 + q;
          const bool in = rr >= 0 && rr < a.H;
          lo[q] = in ? __ldg(s.poff + rr * a.W + c0) : 0;
          n[q] = in ? __ldg(s.poff + rr * a.W + c1 + 1) - lo[q] : 0;
        }
        const long long ck = d2_key(a.cut2);
        long long bk = LLONG_MAX;
        const int n01 = n[0] + n[1], nt = n01 + n[2];
        for (int t = sub; t < nt; t += G) {
          const int e = t < n[0] ? lo[0] + t : (t < n01 ? lo[1] + (t - n[0]) : lo[2] + (t - n01));
          const double4 it = ld256(s.items + e);
          const long long xk = d2_key(exact_d2(it, px, py, pz));
          const int vi = static_cast<int>(__double_as_longlong(it.w));
          if (xk <= ck && (xk < bk || (xk == bk && vi < best_i))) {
            bk = xk;
            best_i = vi;
          }
        }
        if (best_i >= 0) best_x = __longlong_as_double(bk);
      }
    } else if (act && sub < (2 * K1 + 1) * SPL) {
      // SPL lanes per core row, each scanning every SPL-th item of its span
      const int rr = pv - K1 + sub / SPL;
      if (rr >= 0 && rr < a.H) {
        const int r = rr * a.W;
        const int c0 = max(pu - K1, 0), c1 = min(pu + K1, a.W - 1);
        scan_span(s, __ldg(s.poff + r + c0) + sub % SPL, __ldg(s.poff + r + c1 + 1), px, py, pz, a.cut2, best_x,
                  best_i, SPL);
      }
    }
    group_min<G>(best_x, best_i);
    bool open = false;
    if (act) {
      bool done = K1 == w;
      if (!done && a.prune) {
        const double atx = fabs((pu - a.cx) * ifx), aty = fabs((pv - a.cy) * ify);
        const double lb = ring_lb2(K1 + 1, atx, aty, ifx, ify, pz);
        done = lb > a.cut2 || lb > best_x;  // no vertex outside the core can win or tie
      }
      open = !done;
    }
    if (__any_sync(0xffffffffu, open)) {
      // phase 2 for the open pixels of this warp (groups work independently)
      double bx = INFINITY;
      int bi = -1;
      if (open) {
        const double atx = fabs((pu - a.cx) * ifx), aty = fabs((pv - a.cy) * ify);
        int ks = w;
        if (a.prune) {
          ks = K1;
          for (int k = K1 + 1; k <= w; ++k) {
            const double lb = ring_lb2(k, atx, aty, ifx, ify, pz);
            if (lb > a.cut2 || lb > best_x) break;
            ks = k;
          }
        }
        const int c0 = max(pu - ks, 0), c1 = min(pu + ks, a.W - 1);
#ifndef WT_RING_UNITS
#define WT_RING_UNITS 1
#endif
        if (WT_RING_UNITS) {
          // The (2ks+1)^2 box outside the core as work units dealt round-robin
          // to the group's lanes: each full ring row (|dr| > K1) split into two
          // interleaved halves (every other item of its span), then the left
          // and right side spans of the core rows. The long full rows no
          // longer land on one lane (ks = 2, G = 4: 11 -> ~5 items on the
          // slowest lane).
          // pieces per full ring row: 2 for 4-lane groups (measured best at
          // C5), 3 for 16-lane groups (ks = K1 + 1: 6 row pieces + 10 side
          // spans = one unit per lane; C3 1903 -> 1917 frames/s)
          constexpr int SP = G >= 16 ? 3 : 2;
          const int nrow = ks - K1;  // full rows above (and below) the core band
          const int nunits = 2 * SP * nrow + 2 * (2 * K1 + 1);
          for (int u = sub; u < nunits; u += G) {
            int dr, lo, hi, off = 0, step = 1;
            if (u < 2 * SP * nrow) {
              const int fr = u / SP;
              dr = fr < nrow ? -ks + fr : K1 + 1 + (fr - nrow);
              lo = c0;
              hi = c1;
              off = u % SP;
              step = SP;
            } else {
              const int v = u - 2 * SP * nrow;
              dr = -K1 + (v >> 1);
              lo = (v & 1) ? max(pu + K1 + 1, c0) : c0;
              hi = (v & 1) ? c1 : min(pu - K1 - 1, c1);
            }
            const int rr = pv + dr;
            if (lo > hi || rr < 0 || rr >= a.H) continue;
            const int r = rr * a.W;
            scan_span(s, s.poff[r + lo] + off, s.poff[r + hi + 1], px, py, pz, a.cut2, bx, bi, step);
          }
        } else {
          for (int dr = sub - ks; dr <= ks; dr += G) {
            const int rr = pv + dr;
            if (rr < 0 || rr >= a.H) continue;
            const int r = rr * a.W;
            if (dr >= -K1 && dr <= K1) {  // the core columns were scanned in phase 1
              const int l1 = min(pu - K1 - 1, c1), r0 = max(pu + K1 + 1, c0);
              if (l1 >= c0) scan_span(s, s.poff[r + c0], s.poff[r + l1 + 1], px, py, pz, a.cut2, bx, bi);
              if (r0 <= c1) scan_span(s, s.poff[r + r0], s.poff[r + c1 + 1], px, py, pz, a.cut2, bx, bi);
            } else {
              scan_span(s, s.poff[r + c0], s.poff[r + c1 + 1], px, py, pz, a.cut2, bx, bi);
            }
          }
        }
      }
      group_min<G>(bx, bi);
      if (open && bi >= 0 && (best_i < 0 || bx < best_x || (bx == best_x && bi < best_i))) {
        best_x = bx;
        best_i = bi;
      }
    }
    if (act && sub == 0) search_emit(s, a, pix, best_i, px, py, pz, oscale);
  }
}

// p~_i = mean of the observations won by vertex i; count in *cnt.
__device__ __forceinline__ ulonglong4 load_obs(const unsigned long long* acc, int i) {
  return ld256(reinterpret_cast<const ulonglong4*>(acc) + i);
}

__device__ __forceinline__ bool observed_mean(const ulonglong4& q, double oinv, double* pt) {
  const ulonglong2 a01 = make_ulonglong2(q.x, q.y), a23 = make_ulonglong2(q.z, q.w);
  const long long c = static_cast<long long>(a23.y);
  if (c <= 0) return false;
  const double inv = 1.0 / static_cast<double>(c);
  pt[0] = unfix(a01.x, oinv) * inv;
  pt[1] = unfix(a01.y, oinv) * inv;
  pt[2] = unfix(a23.x, oinv) * inv;
  return true;
}


// ---------------------------------------------------------------------------
// Dense fp64 solve of the damped L x L pose system by one CTA (solve_step,
// kinopt.cpp:121-130) as an LDL^T factorisation: A = L D L^T with unit L.
// D_k is exactly the pivot Eigen's LLT takes the square root of, so the
// factorisation fails (returns 0) under the same condition -- the first pivot
// that is not strictly positive. No square roots; one barrier per pivot: every
// thread updates trailing entries (i,j) listed in the (ea, eb) upper-triangle
// table. A is row-major (lower triangle used, overwritten); b is overwritten;
// x receives the solution. Must be called by all threads of the CTA.
__device__ inline int block_ldlt_solve(int L, int lda, double* A, double* b, double* x, const unsigned short* ea,
                                const unsigned short* eb, int NT) {
  __shared__ int s_ok;
  __shared__ double inv_d[64];
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  for (int k = 0; k < L; ++k) {
    const double dk = A[k * lda + k];
    if (!(dk > 0.0)) {  // uniform: every thread read the same pivot
      if (threadIdx.x == 0) s_ok = 0;
      break;
    }
    const double inv = __drcp_rn(dk);
    for (int e = threadIdx.x; e < NT; e += blockDim.x) {
      const int r = ea[e], c = eb[e];  // r <= c: update lower entry (c, r)
      if (r > k) A[c * lda + r] -= A[c * lda + k] * A[r * lda + k] * inv;
    }
    if (threadIdx.x == 0) inv_d[k] = inv;
    __syncthreads();
  }
  __syncthreads();
  const int ok = s_ok;
  if (ok && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int k = 0; k < L; ++k) {  // forward: (unit) L z = b
      const double zk = b[k];
      __syncwarp();
      for (int i = k + 1 + lane; i < L; i += 32) b[i] -= A[i * lda + k] * inv_d[k] * zk;
      __syncwarp();
    }
    for (int k = lane; k < L; k += 32) b[k] *= inv_d[k];  // D y = z
    __syncwarp();
    for (int k = L - 1; k >= 0; --k) {  // backward: L^T x = y
      const double xk = b[k];
      __syncwarp();
      for (int i = lane; i < k; i += 32) b[i] -= A[k * lda + i] * inv_d[i] * xk;
      if (lane == 0) x[k] = xk;
      __syncwarp();
    }
  }
  __syncthreads();
  return ok;
}

// One-warp LDL^T solve for L <= N <= 32 (N a compile-time padding, the
// system is extended with an identity block), with the same factorisation
// and failure rule as block_ldlt_solve: lane i holds row i in registers,
// column k travels by shuffles (cheap on sm_100: ~9 cycles), the forward
// substitution is fused into the elimination and the backward one reads the
// unit-L factor written back to A (row stride lda). Returns 1 on success (x
// written), 0 when a pivot is not strictly positive. Call from a full warp.
//
// The pivot loop is NOT unrolled: a fully unrolled N = 20 elimination is
// ~10k straight-line instructions that run once per launch from a cold
// instruction cache (ncu: stall_no_instruction dominated the solving warp,
// 18k cycles). Instead each lane's register row is rotated by one after
// every pivot so the pivot column is always a[0] and the body indexes
// registers statically; it does N-1 (instead of N-1-k) shuffle/FMA pairs per
// pivot but stays a few hundred instructions, resident after the first pass.
// The arithmetic (operands and order of every FMA) is unchanged.
template <int N>
__device__ inline int warp_ldlt_solve(int L, int lda, double* A, const double* b, double* x, double (*scol)[32]) {
  const int lane = threadIdx.x & 31;
  const bool row = lane < L;
  double a[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    a[j] = row ? (j < L ? A[lane * lda + j] : 0.0) : (j == lane ? 1.0 : 0.0);
  }
  double bi = row ? b[lane] : 0.0;
  double dinv = 1.0;
  int ok = 1;
  // Fully unrolled over the pivots: a[j] is this lane's entry of column j
  // (static register indices, no shifting), and pivot k updates only the
  // trailing columns k+1..N-1. Column k of the current Schur complement
  // (every lane's a[k]) and the right-hand side are published through
  // shared memory -- one store per lane, then broadcast loads -- instead of
  // one 64-bit shuffle per entry (two SHFLs each); the two column buffers
  // alternate, so one warp barrier per pivot suffices. Same FMAs, same
  // operands as a shuffle broadcast.
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double* col = scol[2 * (k & 1)];
    double* rhs = scol[2 * (k & 1) + 1];
    col[lane] = a[k];
    rhs[lane] = bi;
    __syncwarp();
    const double dk = col[k];
    ok &= dk > 0.0 ? 1 : 0;  // uniform; padded pivots are 1
    const double inv = __drcp_rn(dk);
    const double zk = rhs[k];
    const bool act = lane > k;
    const double lik = a[k] * inv;
    if (lane == k) dinv = inv;
    // Unpredicated: entries with t > lane (or lane <= k) are upper-triangle
    // values no later pivot reads, so updating them is harmless; every entry
    // that is read gets exactly the FMA the predicated form did.
#pragma unroll
    for (int t = k + 1; t < N; ++t) a[t] = __fma_rn(-lik, col[t], a[t]);  // A[t][k], unscaled
    if (act) {
      bi = __fma_rn(-lik, zk, bi);
      if (row) A[lane * lda + k] = lik;
    }
  }
  if (!ok) return 0;
  __syncwarp();
  double yi = bi * dinv;
  for (int k = L - 1; k >= 0; --k) {
    const double xk = __shfl_sync(0xffffffffu, yi, k);
    if (lane < k) yi = __fma_rn(-A[k * lda + lane], xk, yi);
  }
  if (row) x[lane] = yi;
  __syncwarp();
  return 1;
}

// warp_ldlt_solve with the pivots taken two at a time: one publish / warp
// barrier / broadcast round per pair. The pair's second pivot D1 = d1 - e^2/d0
// comes from the 2x2 determinant, det = d0 d1 - e^2, so its reciprocal
// d0 / det and 1/d0 are two independent reciprocals, not a chain; the pivot
// tests are d0 > 0 and det > 0 (D1 > 0). Row i then takes pivot k's and pivot
// k+1's updates in one pass: a_t -= l_ik c_k[t] + l_i,k+1 w[t], with
// w[t] = c_k+1[t] - l_k+1,k c_k[t] (column k+1 after pivot k, formed by every
// lane). The L factors, D^-1 and the substitutions are those of the
// one-pivot form; the rounding differs by the order of the pivot-k update.
// scol: three pairs of 32-double buffers (column k, column k+1, rhs), alternating.
template <int N>
__device__ inline int warp_ldlt_solve2(int L, int lda, double* A, const double* b, double* x, double (*scol)[32]) {
  static_assert(N % 2 == 0, "pivot pairs");
  const int lane = threadIdx.x & 31;
  const bool row = lane < L;
  double a[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    a[j] = row ? (j < L ? A[lane * lda + j] : 0.0) : (j == lane ? 1.0 : 0.0);
  }
  double bi = row ? b[lane] : 0.0;
  double dinv = 1.0;
  int ok = 1;
#pragma unroll
  for (int k = 0; k < N; k += 2) {
    double* ck = scol[3 * ((k >> 1) & 1)];
    double* ck1 = scol[3 * ((k >> 1) & 1) + 1];
    double* rhs = scol[3 * ((k >> 1) & 1) + 2];
    ck[lane] = a[k];
    ck1[lane] = a[k + 1];
    rhs[lane] = bi;
    __syncwarp();
    const double d0 = ck[k], e = ck[k + 1], d1 = ck1[k + 1];
    const double z0 = rhs[k], z1 = rhs[k + 1];
    const double det = __fma_rn(d0, d1, -(e * e));
    ok &= (d0 > 0.0 && det > 0.0) ? 1 : 0;  // uniform; padded pivots are 1
    const double inv0 = __drcp_rn(d0);
    const double inv1 = d0 * __drcp_rn(det);  // 1 / D1
    const double lk1 = e * inv0;              // l_k+1,k
    const double lik = a[k] * inv0;
    const double lik1 = __fma_rn(-lik, e, a[k + 1]) * inv1;
    const double z1p = __fma_rn(-lk1, z0, z1);  // rhs k+1 after pivot k
#pragma unroll
    for (int t = k + 2; t < N; ++t) {
      const double w = __fma_rn(-lk1, ck[t], ck1[t]);
      a[t] = __fma_rn(-lik1, w, __fma_rn(-lik, ck[t], a[t]));
    }
    if (lane == k) dinv = inv0;
    if (lane == k + 1) {
      dinv = inv1;
      bi = z1p;
      if (row) A[lane * lda + k] = lk1;
    }
    if (lane > k + 1) {
      bi = __fma_rn(-lik1, z1p, __fma_rn(-lik, z0, bi));
      if (row) {
        A[lane * lda + k] = lik;
        A[lane * lda + k + 1] = lik1;
      }
    }
  }
  if (!ok) return 0;
  __syncwarp();
  double yi = bi * dinv;
  for (int k = L - 1; k >= 0; --k) {
    const double xk = __shfl_sync(0xffffffffu, yi, k);
    if (lane < k) yi = __fma_rn(-A[k * lda + lane], xk, yi);
  }
  if (row) x[lane] = yi;
  __syncwarp();
  return 1;
}

// ---------------------------------------------------------------------------
// K6 + K7 (+K0): pose normal equations (accumulate_normal_system,
// kinopt.cpp:72-119 with fill_row :29-47) for every associated vertex, then
// in the last CTA: prior (:113-117), damped Cholesky (solve_step :121-130),
// theta update (:161-165), iteration stats (:153-169) and FK/dchain for the
// new theta. JtJ rows of 128 vertices are staged in shared memory (fp64),
// compacted to the vertices that carry a row, and reduced entry-parallel.

struct PoseArgs {
  double lambda_k, lambda_s, diag_floor, limit;
  int clamp;
  int iteration;
  int solve;             // 0: only dump JtJ/Jtr (+prior) to s.sys_out (stage hook)
  int clean_acc;        // zero the sums read (last consumer of this association)
  const int* count_in;   // optional association override (stage hook)
  const double* res_in;
  long long* dbg;        // optional timing record of the last CTA (WT_DEBUG_POSE)
  signed char fexp[68];       // fixed-point exponent per theta (+ [L]: the residual column): entry (a, b)
                              // of [JtJ | Jtr] is scaled by 2^(fexp[a] + fexp[b]) (pose_scales, wt_gpu.cu)
  double res_scale, res_inv;  // ... of sum r^2
};

// k_pose_system runs 256-thread CTAs, two per SM (registers), or 128-thread
// CTAs when a large skeleton's row tiles do not fit 8 warps' shared memory
// (pose_threads, wt_gpu.cu): fewer CTAs, half the reduction atomics.
constexpr int kPoseThreads = 256;
// Shared-memory layout of k_pose_system for L links, NP dchain pairs and
// W warps: offsets, dchain, per-warp row tiles [W][32][L|1], per-warp
// residuals, per-warp entry partials [W][NE], pair tables, entry table.
__host__ __device__ inline size_t pose_smem_bytes(int L, int NP, int warps) {
  const int Lr = (L + 1) | 1;
  const int NE = L * (L + 1) / 2 + L;
  return sizeof(double) * (8 * L + 8 * NP + warps * 32 * Lr + warps * NE) +
         sizeof(int) * (L + 1 + NP) + sizeof(unsigned short) * 2 * NE + 64 +
         (sizeof(double) + sizeof(int)) * warps * 64 + 16;
}

// Upper T x T tiles of the L x (L+1) block [JtJ | Jtr]: tile (bi, bj), bj >= bi.
__host__ __device__ inline int pose_tiles(int L, int T = 4) {
  const int nbr = (L + T - 1) / T, nbc = (L + T) / T;
  int n = 0;
  for (int bi = 0; bi < nbr; ++bi) n += nbc - bi;
  return n;
}
// Tile edge of the pose kernel for L links: 3 while the 3x3 tiles fit one
// warp (L <= 20: 28 tiles, 9 FMAs per row per lane), else 4 (L <= 27), else
// 0 (lane-owned entries).
__host__ __device__ inline int pose_tile_edge(int L) {
  return pose_tiles(L, 3) <= 32 ? 3 : (pose_tiles(L, 4) <= 32 ? 4 : 0);
}

// TPL = T (3 or 4): every lane owns one T x T tile of [JtJ | Jtr]: per row
// 2T shared loads feed T^2 FMAs. TPL = 0: lane-owned entries
// e = lane + 32 q (Q of them), any L <= 64.
template <int Q, int TPL, bool B>
static __global__ void __launch_bounds__(kPoseThreads, 512 / kPoseThreads) k_pose_system(DevModel m, DevState s, const double4* phi, PoseArgs a) {
  // a lone sequence waits after staging the pose tables (pdl_entry_ordered);
  // a batch (thousands of rows per warp) keeps the plain entry
  if constexpr (B) pdl_entry();
  else pdl_trigger();
  if constexpr (B) s = seq_state(s);
  if constexpr (B) phi = seq_ptr(phi, seq_off(s.bstride));
  extern __shared__ __align__(16) double psm[];
  const int L = m.L;
  const int Lr = (L + 1) | 1;  // row stride: L Jacobian entries + the residual, odd
  const int NT = L * (L + 1) / 2;
  const int NE = NT + L;  // upper JtJ, then Jtr
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* s_off = psm;                       // 8L
  double* s_dch = s_off + 8 * L;             // 8NP
  double* rows = s_dch + 8 * m.NP;           // nw * 32 * Lr
  long long* part = reinterpret_cast<long long*>(rows + nw * 32 * Lr);  // nw * NE
  int* s_poff = reinterpret_cast<int*>(part + nw * NE);  // L+1
  int* s_pth = s_poff + (L + 1);                          // NP
  unsigned short* ea = reinterpret_cast<unsigned short*>(s_pth + m.NP);
  unsigned short* eb = ea + NE;
  double* qres = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(eb + NE) + 15) & ~static_cast<uintptr_t>(15));  // nw * 64
  int* qidx = reinterpret_cast<int*>(qres + nw * 64);                             // nw * 64

  const double oinv = a.count_in ? 1.0 : obs_scale(s.fwords, true);  // frame words (k_ingest)
  const long long t0 = clock64();
  if (a.dbg && threadIdx.x == 0) {
    unsigned long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    a.dbg[8 + 3 * 296 + (blockIdx.x % 296)] = static_cast<long long>(g0);
  }
  {
    // stage offsets, dchain and pair tables: all loads of a thread first
    constexpr int U = 4;
    const int n_off = 8 * L, n_dch = 8 * m.NP;
    for (int k0 = threadIdx.x; k0 < n_off + n_dch; k0 += U * blockDim.x) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * blockDim.x;
        if constexpr (B)
          v[u] = k < n_off ? __ldg(s.offsets + k) : (k < n_off + n_dch ? __ldg(s.dchain + (k - n_off)) : 0.0);
        else  // from L2: read before the wait (pdl_entry_ordered)
          v[u] = k < n_off ? __ldcg(s.offsets + k) : (k < n_off + n_dch ? __ldcg(s.dchain + (k - n_off)) : 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * blockDim.x;
        if (k < n_off + n_dch) s_off[k] = v[u];  // s_dch follows s_off contiguously
      }
    }
  }
  __shared__ int s_fexp[68];  // fixed-point exponents (PoseArgs::fexp), one 32-bit word each
  for (int k = threadIdx.x; k <= L; k += blockDim.x) s_fexp[k] = a.fexp[k];
  for (int k = threadIdx.x; k <= L; k += blockDim.x) s_poff[k] = __ldg(m.pair_off + k);
  for (int k = threadIdx.x; k < m.NP; k += blockDim.x) s_pth[k] = __ldg(m.pair_theta + k);
  if (TPL == 0) {
    for (int e = threadIdx.x; e < NE; e += blockDim.x) {
      if (e < NT) {  // row-major upper triangle
        int r = 0, rem = e;
        while (rem >= L - r) {
          rem -= L - r;
          ++r;
        }
        ea[e] = static_cast<unsigned short>(r);
        eb[e] = static_cast<unsigned short>(r + rem);
      } else {
        ea[e] = static_cast<unsigned short>(e - NT);
        eb[e] = static_cast<unsigned short>(L);  // pairs with the residual (row[L])
      }
    }
  }
  // this lane's tile (TPL > 0)
  int tbi = -1, tbj = -1;
  if (TPL > 0) {
    const int nbr = (L + TPL - 1) / TPL, nbc = (L + TPL) / TPL;
    int t = lane;
    for (int bi = 0; bi < nbr; ++bi) {
      if (t < nbc - bi) {
        tbi = bi;
        tbj = bi + t;
        break;
      }
      t -= nbc - bi;
    }
  }
  __syncthreads();
  if constexpr (!B) pdl_wait();
  // WT_POSE_SECTIONS builds (diagnostics, tools/diag_pose.py): cycles of
  // thread 0 in staging, scans, row builds and outer products
#ifndef WT_POSE_SECTIONS
#define WT_POSE_SECTIONS 0
#endif
  long long c_stage = 0, c_scan = 0, c_rows = 0, c_outer = 0, c_mark = 0;
  if (WT_POSE_SECTIONS && a.dbg) c_stage = clock64() - t0;

  // Warp g of TW owns vertices g, g + TW, g + 2 TW, ... (every warp gets the
  // same count to within one, spread over the whole mesh, so no warp holds a
  // region of expensive deep-chain vertices) and scans them 32 at a time,
  // queueing the associated ones; full batches of 32 queued vertices build
  // their rows (fill_row) in a warp-private shared tile, every lane busy, and
  // the batch's outer products are accumulated in fp64 registers in
  // ascending queue order, then added to 2^-40 fixed-point integers.
  constexpr int NACC = TPL > 0 ? TPL * TPL : Q;
  // fixed-point accumulators: the warp's NE entries in shared memory, each
  // owned by exactly one lane (no atomics)
  long long* wpart = part + warp * NE;
  for (int e = lane; e < NE; e += 32) wpart[e] = 0;
  int eidx[NACC];  // entry of each accumulator slot of this lane, -1 = none
#pragma unroll
  for (int q = 0; q < NACC; ++q) {
    int e = -1;
    if (TPL > 0) {
      const int ra = TPL * tbi + q / TPL, cb = TPL * tbj + q % TPL;
      if (tbi >= 0 && ra < L && cb <= L && (cb == L || ra <= cb))
        e = cb == L ? NT + ra : ra * L - ra * (ra - 1) / 2 + (cb - ra);
    } else {
      e = lane + 32 * q < NE ? lane + 32 * q : -1;
    }
    eidx[q] = e;
  }
  __syncwarp();
  long long rsq = 0, nassoc = 0;  // sum r^2 (fixed point at a.res_scale), associated count
  double* wrows = rows + warp * 32 * Lr;
  const int TW = gridDim.x * nw, gw = blockIdx.x * nw + warp;
  int* wq = qidx + warp * 64;       // warp-private queue of associated vertices
  double* wqr = qres + warp * 64;   // ... and their residuals
  int qn = 0;                       // warp-uniform queue length (< 32 between chunks)
  // A batch (long scans: thousands of owned vertices per warp at C5) loads
  // the next 32 owned vertices' sums one chunk ahead and the posed vertex and
  // normal only for the associated ones (C5: 322 -> 299 us per launch); a lone
  // sequence (two chunks per warp) keeps the one-round form (no spills).
#ifndef WT_POSE_AHEAD_MODE
#define WT_POSE_AHEAD_MODE 0  // 0: batch only, 1: always, 2: never (experiments)
#endif
  constexpr bool WT_POSE_SCAN_AHEAD = WT_POSE_AHEAD_MODE == 1 ? true : (WT_POSE_AHEAD_MODE == 2 ? false : B);
  ulonglong4 q_next = make_ulonglong4(0ull, 0ull, 0ull, 0ull);
  if (WT_POSE_SCAN_AHEAD && !a.count_in && gw + TW * lane < m.V)
    q_next = ld256(reinterpret_cast<const ulonglong4*>(s.acc) + gw + TW * lane);
  for (int jb = 0;; jb += 32) {
    const bool more = gw + TW * jb < m.V;
    if (WT_POSE_SECTIONS && a.dbg) c_mark = clock64();
    if (more) {
      // scan 32 owned vertices: association and residual (association.cpp:132-136);
      // the posed vertex and normal are fetched with the sums (one round trip)
      const int i = gw + TW * (jb + lane);
      bool have = false;
      double r = 0.0;
      ulonglong4 q_cur = q_next;
      if (WT_POSE_SCAN_AHEAD && !a.count_in) {
        const int inext = gw + TW * (jb + 32 + lane);
        if (inext < m.V) q_next = ld256(reinterpret_cast<const ulonglong4*>(s.acc) + inext);
      }
      if (i < m.V) {
        if (a.count_in) {
          have = a.count_in[i] > 0;
          r = have ? a.res_in[i] : 0.0;
        } else {
          const ulonglong4 q = WT_POSE_SCAN_AHEAD ? q_cur : ld256(reinterpret_cast<const ulonglong4*>(s.acc) + i);
          const ulonglong2 a01 = make_ulonglong2(q.x, q.y), a23 = make_ulonglong2(q.z, q.w);
          const long long c = static_cast<long long>(a23.y);
          have = c > 0;
          double4 v = make_double4(0, 0, 0, 0);
          float4 n = make_float4(0, 0, 0, 0);
          if (!WT_POSE_SCAN_AHEAD || have) {
            v = ld256(s.pv + i);
            n = s.pn[i];
          }
          if (have) {
            if (a.clean_acc) clear_obs(s, i);
            const double inv = 1.0 / static_cast<double>(c);
            const double px = unfix(a01.x, oinv) * inv, py = unfix(a01.y, oinv) * inv,
                         pz = unfix(a23.x, oinv) * inv;
            r = static_cast<double>(n.x) * (px - v.x) + static_cast<double>(n.y) * (py - v.y) +
                static_cast<double>(n.z) * (pz - v.z);
          }
        }
      }
      if (have) {
        rsq += fix(r * r, a.res_scale);
        ++nassoc;
      }
      const unsigned hm = __ballot_sync(0xffffffffu, have);
      if (have) {
        const int pos = qn + __popc(hm & ((1u << lane) - 1u));
        wq[pos] = i;
        wqr[pos] = r;
      }
      qn += __popc(hm);
      __syncwarp();
    }
    if (WT_POSE_SECTIONS && a.dbg) {
      const long long c = clock64();
      c_scan += c - c_mark;
      c_mark = c;
    }
    // rows of full batches (and of the remainder at the end), every lane busy
    while (qn >= 32 || (!more && qn > 0)) {
      const int nrows = qn < 32 ? qn : 32;
      // A short batch (a lone sequence's tail: ~8 rows per warp at C3) builds
      // each row with `split` lanes; lane qq of a row takes the chain positions
      // qq, qq + split, ... of every weight entry. theta_index is a permutation
      // (validated at create), so a theta sits at its joint's depth in every
      // chain that holds it: each row entry is still summed by one lane, in
      // entry order -- bitwise the one-lane row.
#ifndef WT_POSE_ROW_SPLIT
#define WT_POSE_ROW_SPLIT 1
#endif
      const int lsh = (B || !WT_POSE_ROW_SPLIT) ? 0 : (nrows <= 8 ? 2 : (nrows <= 16 ? 1 : 0));
      const int split = 1 << lsh, rt = lane >> lsh, qq = lane & (split - 1);
      for (int k = lane; k < nrows * Lr; k += 32) wrows[k] = 0.0;
      __syncwarp();
      bool has_row = false;
      if (rt < nrows) {
        const int i = wq[rt];
        const double r = wqr[rt];
        const float4 n = s.pn[i];
        DQ raw;
        double sign[4];
        const double4 wv = ld256(m.wgt + i);
        const uchar4 lk = m.wlink[i];
        const double4 a0 = ld256(m.v0 + i);
        const double4 f = ld256(phi + i);
        if (n.w != 0.0f && blend_vertex(s_off, wv, lk, raw, sign)) {
          const double rest[3] = {a0.x + f.x, a0.y + f.y, a0.z + f.z};
          const double nn[3] = {n.x, n.y, n.z};
          double r8[8];
          dq_point_plane_row(raw, rest, nn, r8);
          double* row = wrows + rt * Lr;
          if (qq == 0) row[L] = r;
          const unsigned char li[4] = {lk.x, lk.y, lk.z, lk.w};
          const double wi[4] = {wv.x, wv.y, wv.z, wv.w};
          for (int e = 0; e < 4; ++e) {
            if (li[e] == 0xFF) break;
            const double coeff = wi[e] * sign[e];
            for (int p = s_poff[li[e]] + qq; p < s_poff[li[e] + 1]; p += split) {
              const double* d8 = s_dch + 8 * p;
              const double dot = ((r8[0] * d8[0] + r8[1] * d8[1]) + (r8[2] * d8[2] + r8[3] * d8[3])) +
                                 ((r8[4] * d8[4] + r8[5] * d8[5]) + (r8[6] * d8[6] + r8[7] * d8[7]));
              row[s_pth[p]] += coeff * dot;
            }
          }
          has_row = qq == 0;
        }
      }
      unsigned mask = __ballot_sync(0xffffffffu, has_row);
      if (lsh) mask = __ballot_sync(0xffffffffu, lane < nrows && ((mask >> (lane << lsh)) & 1u));
      __syncwarp();
      if (WT_POSE_SECTIONS && a.dbg) {
        const long long c = clock64();
        c_rows += c - c_mark;
        c_mark = c;
      }
      if (mask) {
        double acc[NACC];
#pragma unroll
        for (int q = 0; q < NACC; ++q) acc[q] = 0.0;
        if (TPL > 0) {
          if (tbi >= 0) {
            const int ca = TPL * tbi, cb = TPL * tbj;
            while (mask) {
              const int t = __ffs(mask) - 1;
              mask &= mask - 1;
              const double* row = wrows + t * Lr;
              double ra[TPL > 0 ? TPL : 1], rb[TPL > 0 ? TPL : 1];
#pragma unroll
              for (int u = 0; u < TPL; ++u) {
                ra[u] = row[min(ca + u, L)];  // clamped: in-bounds, discarded beyond L
                rb[u] = row[min(cb + u, L)];
              }
#pragma unroll
              for (int u = 0; u < TPL; ++u)
#pragma unroll
                for (int v = 0; v < TPL; ++v) acc[TPL * u + v] += ra[u] * rb[v];
            }
          }
        } else {
          while (mask) {
            const int t = __ffs(mask) - 1;
            mask &= mask - 1;
            const double* row = wrows + t * Lr;
#pragma unroll
            for (int q = 0; q < NACC; ++q) {
              const int e = lane + 32 * q;
              if (e < NE) acc[q] += row[ea[e]] * row[eb[e]];
            }
          }
        }
#pragma unroll
        for (int q = 0; q < NACC; ++q)
          if (eidx[q] >= 0) {
            int ex;
            if (TPL > 0) {
              ex = s_fexp[TPL * tbi + q / TPL] + s_fexp[TPL * tbj + q % TPL];  // (row, col), col L = Jtr
            } else {
              const int e = lane + 32 * q;
              ex = s_fexp[ea[e]] + s_fexp[eb[e]];
            }
            wpart[eidx[q]] += fix(acc[q], exp2i(ex));
          }
      }
      if (WT_POSE_SECTIONS && a.dbg) {
        const long long c = clock64();
        c_outer += c - c_mark;
        c_mark = c;
      }
      // drop the processed rows from the queue
      const int rest_n = qn - nrows;
      int qi = 0;
      double qr = 0.0;
      if (lane < rest_n) {
        qi = wq[nrows + lane];
        qr = wqr[nrows + lane];
      }
      __syncwarp();
      if (lane < rest_n) {
        wq[lane] = qi;
        wqr[lane] = qr;
      }
      qn = rest_n;
      __syncwarp();
    }
    if (!more) break;
  }
  const long long t1 = clock64();
  unsigned long long g_main = 0;
  if (a.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_main));
  // per-CTA integer sums (exact), then fixed-point atomics spread over
  // kRedCopies slot copies to avoid same-address serialisation
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rsq += __shfl_xor_sync(0xffffffffu, rsq, o);
    nassoc += __shfl_xor_sync(0xffffffffu, nassoc, o);
  }
  __shared__ long long s_rsq[32], s_na[32];
  if (lane == 0) {
    s_rsq[warp] = rsq;
    s_na[warp] = nassoc;
  }
  __syncthreads();
  unsigned long long* red = s.red + (blockIdx.x % kRedCopies) * (NE + 2);
  for (int e = threadIdx.x; e < NE; e += blockDim.x) {
    long long sum = 0;
    for (int w = 0; w < nw; ++w) sum += part[w * NE + e];
    if (sum) red_add(red + e, sum);
  }
  if (threadIdx.x == 0) {
    long long r2 = 0, na = 0;
    for (int w = 0; w < nw; ++w) {
      r2 += s_rsq[w];
      na += s_na[w];
    }
    if (r2) red_add(red + NE, r2);
    if (na) red_add(red + NE + 1, na);
  }
  if (a.dbg && threadIdx.x == 0) {
    unsigned long long g_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    const int slot = blockIdx.x % 296;
    a.dbg[8 + 3 * slot] = static_cast<long long>(g_main);
    a.dbg[8 + 3 * slot + 1] = static_cast<long long>(g_end);
    a.dbg[8 + 3 * slot + 2] = t1 - t0;
    long long* sec = a.dbg + 8 + 4 * 296 + 4 * slot;
    sec[0] = c_stage;
    sec[1] = c_scan;
    sec[2] = c_rows;
    sec[3] = c_outer;
  }
  if (a.dbg && threadIdx.x == 0 && blockIdx.x == 0) a.dbg[0] = t1 - t0;
}


// K7 (+K0): the pose-solve step, one CTA right after k_pose_system in the
// same stream: fold the reduction copies into JtJ / Jtr, add the prior
// (kinopt.cpp:113-117), damp and factor (solve_step, kinopt.cpp:121-130;
// a failed factorisation skips the step, :166-168), theta -= x with the
// optional clamp (:161-165), the iteration stats (:153-169) and FK / offsets
// / dchain for the new theta (skeleton.cpp:56-108). A kernel of its own, so
// the serial solve is not register-capped by the reduction kernel.
__host__ __device__ inline size_t pose_solve_smem_bytes(int L) {
  const int NE = L * (L + 1) / 2 + L;
  return sizeof(double) * L * (L | 1) + sizeof(unsigned short) * 2 * NE + 16;
}

template <bool B>
static __global__ void __launch_bounds__(256, 1) k_pose_solve(DevModel m, DevState s, PoseArgs a) {
  pdl_trigger();  // the model tables, theta and S are read before the wait (pdl_entry_ordered)
  if constexpr (B) s = seq_state(s);
  __shared__ FkTables fkt;
  extern __shared__ __align__(16) double solve_sm[];  // pose_solve_smem_bytes(L)
  __shared__ double jtr[64];
  __shared__ double s_theta[64];
  __shared__ double s_x[64];
  __shared__ double s_rsum;
  __shared__ long long s_nassoc;
  __shared__ int s_finite;
  int wrapped = 0;  // a non-negative fixed-point sum (diagonal, sum r^2) left the int64 range
  const int L = m.L;
  const int Lp = L | 1;
  const int NT = L * (L + 1) / 2;
  const int NE = NT + L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* A = solve_sm;                                                // L * Lp
  unsigned short* ea = reinterpret_cast<unsigned short*>(A + L * Lp);  // NE
  unsigned short* eb = ea + NE;
  const long long t2 = clock64();
  // every global load of the prologue in one round: reduction copies, entry
  // table, theta, S, the link table
  unsigned long long sum[4] = {0ull, 0ull, 0ull, 0ull};
  unsigned ent[4] = {0u, 0u, 0u, 0u};
  {
    double th = 0.0, sd = 0.0;
    if (threadIdx.x < L) {
      th = __ldcg(s.theta + threadIdx.x);  // L2: written by the previous solve
      sd = __ldg(m.s_diag + threadIdx.x);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = threadIdx.x + q * blockDim.x;
      if (e < NE) ent[q] = __ldg(m.pose_e + e);
    }
    fk_stage(m, fkt);
    pdl_wait();
    unsigned long long v[4][kRedCopies];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = threadIdx.x + q * blockDim.x;
      if (e < NE) {
#pragma unroll
        for (int c = 0; c < kRedCopies; ++c) v[q][c] = __ldcg(s.red + c * (NE + 2) + e);
      }
    }
    unsigned long long rv[2 * kRedCopies];
    if (threadIdx.x == blockDim.x - 1) {
#pragma unroll
      for (int c = 0; c < kRedCopies; ++c) {
        rv[2 * c] = __ldcg(s.red + c * (NE + 2) + NE);
        rv[2 * c + 1] = __ldcg(s.red + c * (NE + 2) + NE + 1);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < kRedCopies; ++c) sum[q] += v[q][c];
    if (threadIdx.x < L) {
      s_theta[threadIdx.x] = th;
      s_x[threadIdx.x] = sd;  // staged S for the prior
    }
    if (threadIdx.x == blockDim.x - 1) {
      unsigned long long rs = 0ull, na = 0ull;
#pragma unroll
      for (int c = 0; c < kRedCopies; ++c) {
        rs += rv[2 * c];
        na += rv[2 * c + 1];
        s.red[c * (NE + 2) + NE] = 0ull;
        s.red[c * (NE + 2) + NE + 1] = 0ull;
      }
      s_rsum = unfix(rs, a.res_inv);
      s_nassoc = static_cast<long long>(na);
      s_finite = 1;
      wrapped |= static_cast<long long>(rs) < 0 ? 1 : 0;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + q * blockDim.x;
    if (e >= NE) continue;
#pragma unroll
    for (int c = 0; c < kRedCopies; ++c) s.red[c * (NE + 2) + e] = 0ull;  // self-cleaning
    const int ca = ent[q] & 0xFFFF, cb = ent[q] >> 16;
    ea[e] = static_cast<unsigned short>(ca);
    eb[e] = static_cast<unsigned short>(cb == L ? 0xFFFF : cb);
    if (ca == cb && static_cast<long long>(sum[q]) < 0) wrapped = 1;
    const double val = unfix(sum[q], exp2i(-(a.fexp[ca] + a.fexp[cb])));
    if (cb == L) {
      jtr[ca] = val;
    } else {
      A[ca * Lp + cb] = val;
      A[cb * Lp + ca] = val;
    }
  }
  for (int e = threadIdx.x + 4 * blockDim.x; e < NE; e += blockDim.x) {  // L > 43: the rest
    unsigned long long t = 0ull;
    for (int c = 0; c < kRedCopies; ++c) {
      t += __ldcg(s.red + c * (NE + 2) + e);
      s.red[c * (NE + 2) + e] = 0ull;
    }
    const unsigned en = __ldg(m.pose_e + e);
    const int ca = en & 0xFFFF, cb = en >> 16;
    ea[e] = static_cast<unsigned short>(ca);
    eb[e] = static_cast<unsigned short>(cb == L ? 0xFFFF : cb);
    if (ca == cb && static_cast<long long>(t) < 0) wrapped = 1;
    const double val = unfix(t, exp2i(-(a.fexp[ca] + a.fexp[cb])));
    if (cb == L) {
      jtr[ca] = val;
    } else {
      A[ca * Lp + cb] = val;
      A[cb * Lp + ca] = val;
    }
  }
  const int out_of_range = __syncthreads_or(wrapped);
  // default-pose prior (lambda_s S)^2 on the diagonal (kinopt.cpp:113-117),
  // then A = JtJ + lambda_k diag(JtJ) + floor I (kinopt.cpp:121-126)
  for (int k = threadIdx.x; k < L; k += blockDim.x) {
    const double p = a.lambda_s * s_x[k];
    const double jd = A[k * Lp + k] + p * p;
    jtr[k] += p * p * s_theta[k];
    A[k * Lp + k] = a.solve ? jd + a.lambda_k * jd + a.diag_floor : jd;
  }
  __syncthreads();
  if (!a.solve) {
    for (int e = threadIdx.x; e < L * L; e += blockDim.x) s.sys_out[e] = A[(e / L) * Lp + e % L];
    for (int k = threadIdx.x; k < L; k += blockDim.x) s.sys_out[L * L + k] = jtr[k];
    return;
  }
  if (out_of_range && threadIdx.x == 0) s_finite = 0;
  for (int e = threadIdx.x; e < L * L; e += blockDim.x)
    if (!isfinite(A[(e / L) * Lp + e % L])) s_finite = 0;
  for (int k = threadIdx.x; k < L; k += blockDim.x)
    if (!isfinite(jtr[k])) s_finite = 0;
  __syncthreads();
  const long long t3 = clock64();
#ifndef WT_POSE_BLOCK_SOLVE
#define WT_POSE_BLOCK_SOLVE 0
#endif
  if (L <= 32 && !WT_POSE_BLOCK_SOLVE) {
    if (warp == 0) {
      int ok = 0;
      if (s_finite) {
#ifndef WT_LDLT_PAIRS
#define WT_LDLT_PAIRS 1
#endif
        __shared__ double scol[6][32];
        if (WT_LDLT_PAIRS) {
          if (L <= 8) ok = warp_ldlt_solve2<8>(L, Lp, A, jtr, s_x, scol);
          else if (L <= 16) ok = warp_ldlt_solve2<16>(L, Lp, A, jtr, s_x, scol);
          else if (L <= 20) ok = warp_ldlt_solve2<20>(L, Lp, A, jtr, s_x, scol);
          else if (L <= 24) ok = warp_ldlt_solve2<24>(L, Lp, A, jtr, s_x, scol);
          else ok = warp_ldlt_solve2<32>(L, Lp, A, jtr, s_x, scol);
        } else {
          if (L <= 8) ok = warp_ldlt_solve<8>(L, Lp, A, jtr, s_x, scol);
          else if (L <= 16) ok = warp_ldlt_solve<16>(L, Lp, A, jtr, s_x, scol);
          else if (L <= 20) ok = warp_ldlt_solve<20>(L, Lp, A, jtr, s_x, scol);
          else if (L <= 24) ok = warp_ldlt_solve<24>(L, Lp, A, jtr, s_x, scol);
          else ok = warp_ldlt_solve<32>(L, Lp, A, jtr, s_x, scol);
        }
      }
      // theta -= x (kinopt.cpp:161-165), optional clamp, iteration stats
      double xk = 0.0;
      if (ok && lane < L) {
        xk = s_x[lane];
        double t = s_theta[lane] - xk;
        if (a.clamp && a.limit > 0.0) t = fmin(fmax(t, -a.limit), a.limit);
        s_theta[lane] = t;
      }
      double nrm = xk * xk;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      if (lane == 0) {
        KinStat st;
        st.residual_sum = s_rsum;
        st.associated = static_cast<int>(s_nassoc);
        st.step_norm = ok ? sqrt(nrm) : 0.0;
        st.skipped = ok ? 0 : (out_of_range ? 2 : 1);  // 2: reported as WT_ERANGE by the host
        s.kin_stats[a.iteration] = st;
      }
    }
    __syncthreads();
  } else {
    // general L (<= 64): block LDL^T over the (ea, eb) table
    const int ok = s_finite ? block_ldlt_solve(L, Lp, A, jtr, s_x, ea, eb, NT) : 0;
    if (threadIdx.x == 0) {
      double nrm = 0.0;
      if (ok) {
        for (int k = 0; k < L; ++k) {
          double t = s_theta[k] - s_x[k];
          if (a.clamp && a.limit > 0.0) t = fmin(fmax(t, -a.limit), a.limit);
          s_theta[k] = t;
          nrm += s_x[k] * s_x[k];
        }
      }
      KinStat st;
      st.residual_sum = s_rsum;
      st.associated = static_cast<int>(s_nassoc);
      st.step_norm = ok ? sqrt(nrm) : 0.0;
      st.skipped = ok ? 0 : (out_of_range ? 2 : 1);
      s.kin_stats[a.iteration] = st;
    }
    __syncthreads();
  }
  const long long t4 = clock64();
  for (int k = threadIdx.x; k < L; k += blockDim.x) s.theta[k] = s_theta[k];
  __shared__ long long fk_st[2];
  fk_run(m, s, s_theta, fkt, a.dbg ? fk_st : nullptr);
  if (a.dbg) __syncthreads();
  if (a.dbg && threadIdx.x == 0) {
    a.dbg[1] = 0;
    a.dbg[2] = t3 - t2;
    a.dbg[3] = t4 - t3;
    a.dbg[4] = clock64() - t4;
    a.dbg[5] = fk_st[0] - t4;        // sincos + local transforms
    a.dbg[6] = fk_st[1] - fk_st[0];  // level chain
  }
}


// ---------------------------------------------------------------------------
// K8: per-vertex regularised 3x3 shape step (optimize_shape body,
// shapeopt.cpp:78-96, solve_vertex :25-48), Jacobi: reads phi_in, writes
// phi_out. The last CTA writes the iteration's ShapeIterStats.

// solve_vertex with Eigen LLT semantics on the 3x3 system; returns false
// (singular) on non-finite input or a non-positive pivot.
__device__ __forceinline__ bool solve_vertex3(const double g[3], double r, const double phi[3],
                                              const double nd[3], int ncount, double lphi,
                                              double lnbr, double lw, double floor_,
                                              double delta[3]) {
  double A[3][3];
  for (int x = 0; x < 3; ++x)
    for (int y = 0; y < 3; ++y) A[x][y] = g[x] * g[y];
  const double reg = lphi + lnbr * ncount;
  for (int d = 0; d < 3; ++d) {
    A[d][d] += reg;
    A[d][d] += lw * A[d][d];
    A[d][d] += floor_;
  }
  double b[3];
  for (int d = 0; d < 3; ++d) b[d] = g[d] * r + lphi * phi[d] + lnbr * nd[d];
  bool finite = true;
  for (int x = 0; x < 3; ++x) {
    finite = finite && isfinite(b[x]);
    for (int y = 0; y < 3; ++y) finite = finite && isfinite(A[x][y]);
  }
  delta[0] = delta[1] = delta[2] = 0.0;
  if (!finite) return false;
  // LLT on the lower triangle (Eigen llt_inplace semantics: a pivot <= 0
  // fails). The factor's diagonal enters only through its reciprocals, so
  // each is one rsqrt of the pivot: no fp64 division or square root on the
  // chain (results within an ulp or two of the divided form; C5 shape step
  // 392 -> 301 us, C3 18.5 -> 15.1 us).
  const double p0 = A[0][0];
  if (!(p0 > 0.0)) return false;
  const double i0 = rsqrt(p0);
  const double l10 = A[1][0] * i0, l20 = A[2][0] * i0;
  const double p1 = A[1][1] - l10 * l10;
  if (!(p1 > 0.0)) return false;
  const double i1 = rsqrt(p1);
  const double l21 = (A[2][1] - l20 * l10) * i1;
  const double p2 = A[2][2] - l20 * l20 - l21 * l21;
  if (!(p2 > 0.0)) return false;
  const double i2 = rsqrt(p2);
  const double y0 = b[0] * i0;
  const double y1 = (b[1] - l10 * y0) * i1;
  const double y2 = (b[2] - l20 * y0 - l21 * y1) * i2;
  delta[2] = y2 * i2;
  delta[1] = (y1 - l21 * delta[2]) * i1;
  delta[0] = (y0 - l10 * delta[1] - l20 * delta[2]) * i0;
  return true;
}

// Shape statistics as fp64 per-CTA partials (sum |r|, observed, sum |phi|,
// singular, max |phi|), written by thread 0 of every CTA; the CTA that
// finishes last folds them in CTA order -- deterministic for a given grid and
// free of any fixed-point range (phi and r in any length unit).
constexpr int kStatParts = 5;

__device__ inline void stat_partials_put(double* spart, double a, double b, double c, double d, double mx) {
  double* p = spart + kStatParts * blockIdx.x;
  p[0] = a;
  p[1] = b;
  p[2] = c;
  p[3] = d;
  p[4] = mx;
}

// In the last CTA (all threads): a fixed-shape fold -- thread t sums CTAs
// t, t + T, ... in order, a shuffle butterfly per warp, then the warps in
// order -- deterministic for a given grid; result in out[] of thread 0.
__device__ inline void stat_partials_fold(const double* spart, double out[kStatParts]) {
  double acc[kStatParts] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    const double* p = spart + kStatParts * b;
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] += __ldcg(p + k);
    acc[4] = fmax(acc[4], __ldcg(p + 4));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    acc[4] = fmax(acc[4], __shfl_xor_sync(0xffffffffu, acc[4], o));
  }
  __shared__ double red[kStatParts][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < kStatParts; ++k) red[k][wid] = acc[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < kStatParts; ++k) out[k] = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {  // warp order
#pragma unroll
      for (int k = 0; k < 4; ++k) out[k] += red[k][w];
      out[4] = fmax(out[4], red[4][w]);
    }
  }
}

struct ShapeArgs {
  double lambda_phi, lambda_nbr, lambda_w, diag_floor;
  int iteration;
  int clean_acc;  // zero the observation sums read
};

constexpr int kNbrAhead = 4;  // neighbour gathers issued together in k_shape (kNN k = 4)

// The loads of one vertex of the shape step that do not depend on the
// association: phi and its neighbours' (the neighbour sum nd, in list order),
// and -- PRE: read before the PDL wait, from L2 -- the posed vertex, normal
// and skin weights, which otherwise load only for observed vertices.
struct ShapeIn {
  double ph[3], nd[3];
  int ncount;
  double4 v, wv;
  float4 n;
  uchar4 lk;
};
template <bool PRE>
__device__ __forceinline__ ShapeIn shape_gather(const DevModel& m, const DevState& s, const double4* phi_in, int i) {
  ShapeIn in;
  const double4 f = PRE ? ld256_cg(phi_in + i) : ld256(phi_in + i);
  if (PRE) {
    in.v = ld256_cg(s.pv + i);
    in.n = __ldcg(s.pn + i);
    in.wv = ld256(m.wgt + i);
    in.lk = m.wlink[i];
  }
  in.ph[0] = f.x;
  in.ph[1] = f.y;
  in.ph[2] = f.z;
  in.nd[0] = in.nd[1] = in.nd[2] = 0.0;
  in.ncount = 0;
  // the first kNbrAhead neighbour indices, then their phi, all in flight at
  // once; summed in list order up to the first -1 (as the loop below)
  int jn[kNbrAhead];
  double4 fn[kNbrAhead];
#pragma unroll
  for (int k = 0; k < kNbrAhead; ++k) jn[k] = k < m.K ? m.nbr[k * m.V + i] : -1;
#pragma unroll
  for (int k = 0; k < kNbrAhead; ++k) {
    const double4* q = phi_in + (jn[k] >= 0 ? jn[k] : i);
    fn[k] = PRE ? ld256_cg(q) : ld256(q);
  }
  bool more = true;
#pragma unroll
  for (int k = 0; k < kNbrAhead; ++k) {
    if (!more || jn[k] < 0) {
      more = false;
      continue;
    }
    in.nd[0] += in.ph[0] - fn[k].x;
    in.nd[1] += in.ph[1] - fn[k].y;
    in.nd[2] += in.ph[2] - fn[k].z;
    ++in.ncount;
  }
  for (int k = kNbrAhead; more && k < m.K; ++k) {
    const int j = m.nbr[k * m.V + i];
    if (j < 0) break;
    const double4 fj = PRE ? ld256_cg(phi_in + j) : ld256(phi_in + j);
    in.nd[0] += in.ph[0] - fj.x;
    in.nd[1] += in.ph[1] - fj.y;
    in.nd[2] += in.ph[2] - fj.z;
    ++in.ncount;
  }
  return in;
}

struct ShapeAcc {
  double abs_r = 0.0, sum_phi = 0.0, max_phi = 0.0;
  long long observed = 0, singular = 0;
};
// One vertex of the shape step given its gathered inputs (PRE: posed vertex,
// normal and weights included).
template <bool PRE>
__device__ __forceinline__ void shape_vertex(const DevModel& m, const DevState& s, const double* s_off,
                                             const ShapeArgs& a, double4* phi_out, double oinv, int i,
                                             const ShapeIn& in, ShapeAcc& acc) {
  const ulonglong4 obs = load_obs(s.acc, i);
  const double* ph = in.ph;
  double g[3] = {0.0, 0.0, 0.0};
  double r = 0.0;
  double pt[3];
  if (observed_mean(obs, oinv, pt)) {
    if (a.clean_acc) clear_obs(s, i);
    const double4 v = PRE ? in.v : ld256(s.pv + i);
    const float4 n = PRE ? in.n : s.pn[i];
    const double ro = static_cast<double>(n.x) * (pt[0] - v.x) + static_cast<double>(n.y) * (pt[1] - v.y) +
                      static_cast<double>(n.z) * (pt[2] - v.z);
    acc.abs_r += fabs(ro);
    ++acc.observed;
    DQ raw;
    double sign[4];
    if (n.w != 0.0f && blend_vertex(s_off, PRE ? in.wv : ld256(m.wgt + i), PRE ? in.lk : m.wlink[i], raw, sign)) {
      // dr/dphi = -(R^T n), R = rotation of the normalised blend
      double R[9];
      dq_rotation(dq_normalize(raw), R);
      g[0] = -(R[0] * n.x + R[3] * n.y + R[6] * n.z);
      g[1] = -(R[1] * n.x + R[4] * n.y + R[7] * n.z);
      g[2] = -(R[2] * n.x + R[5] * n.y + R[8] * n.z);
      r = ro;
    }
  }
  double delta[3];
  const bool ok = solve_vertex3(g, r, ph, in.nd, in.ncount, a.lambda_phi, a.lambda_nbr, a.lambda_w,
                                a.diag_floor, delta);
  acc.singular += ok ? 0 : 1;
  const double nx = ph[0] - delta[0], ny = ph[1] - delta[1], nz = ph[2] - delta[2];
  st256(phi_out + i, make_double4(nx, ny, nz, 0.0));
  const double len = sqrt(nx * nx + ny * ny + nz * nz);
  acc.sum_phi += len;
  acc.max_phi = fmax(acc.max_phi, len);
}

template <bool B>
static __global__ void __launch_bounds__(kVThreads) k_shape(DevModel m, DevState s, const double4* phi_in,
                                                     double4* phi_out, ShapeArgs a) {
  if constexpr (B) s = seq_state(s);
  if constexpr (B) phi_in = seq_ptr(phi_in, seq_off(s.bstride));
  if constexpr (B) phi_out = seq_ptr(phi_out, seq_off(s.bstride));
  extern __shared__ double s_off[];
  // A lone sequence gathers its first vertex and stages the pose offsets
  // before the PDL wait: phi (the previous shape step's), the posed vertex
  // and normal are several kernels back, complete once this CTA runs
  // (pdl_entry_ordered); only the association sums need the wait.
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  ShapeIn pre{};
  if constexpr (!B) {
    if (i0 < m.V) pre = shape_gather<true>(m, s, phi_in, i0);
    for (int k = threadIdx.x; k < m.L * 8; k += blockDim.x) s_off[k] = __ldcg(s.offsets + k);
  }
  const double oinv = obs_scale(s.fwords, true);  // frame words (k_ingest)
  pdl_entry();
  if constexpr (B) load_offsets(m, s, s_off);
  __syncthreads();
  ShapeAcc acc;
  int i = i0;
  if (!B && i0 < m.V) {
    shape_vertex<true>(m, s, s_off, a, phi_out, oinv, i0, pre, acc);
    i += gridDim.x * blockDim.x;
  }
  for (; i < m.V; i += gridDim.x * blockDim.x)
    shape_vertex<false>(m, s, s_off, a, phi_out, oinv, i, shape_gather<false>(m, s, phi_in, i), acc);
  double abs_r = acc.abs_r, sum_phi = acc.sum_phi, max_phi = acc.max_phi;
  long long observed = acc.observed, singular = acc.singular;
  // block reductions (fixed order), then per-CTA partials folded by the last CTA
  block_sum2(abs_r, observed);
  double sp = sum_phi;
  block_sum2(sp, singular);
  __shared__ double smax[32];
  double mx = max_phi;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < (blockDim.x >> 5); ++k) mx = fmax(mx, smax[k]);
    stat_partials_put(s.spart, abs_r, static_cast<double>(observed), sp, static_cast<double>(singular), mx);
  }
  if (!last_block(s.tickets + 2)) return;
  double tot[kStatParts];
  stat_partials_fold(s.spart, tot);
  if (threadIdx.x == 0) {
    const double sabs = tot[0];
    const long long nobs = static_cast<long long>(tot[1]);
    const double sphi = tot[2];
    const long long nsing = static_cast<long long>(tot[3]);
    const double mphi = tot[4];
    ShapeStat st;
    st.mean_phi = m.V > 0 ? sphi / static_cast<double>(m.V) : 0.0;
    st.max_phi = mphi;
    st.mean_abs_r_before = nobs > 0 ? sabs / static_cast<double>(nobs) : 0.0;
    st.mean_abs_r_after = 0.0;
    st.singular = static_cast<int>(nsing);
    st.pad = 0;
    s.shape_stats[a.iteration] = st;
  }
}

// Closing measurement pass of optimize_shape (shapeopt.cpp:112-129): mean
// |r| over observed vertices of a fresh association; fills mean_abs_r_after.
template <bool B>
static __global__ void __launch_bounds__(kVThreads, 5) k_shape_after(DevModel m, DevState s, int n_its, int clean_acc) {
  pdl_entry();
  if constexpr (B) s = seq_state(s);
  double abs_r = 0.0;
  long long observed = 0;
  const double oinv = obs_scale(s.fwords, true);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m.V; i += gridDim.x * blockDim.x) {
    double pt[3];
    if (observed_mean(load_obs(s.acc, i), oinv, pt)) {
      if (clean_acc) clear_obs(s, i);
      const double4 v = ld256(s.pv + i);
      const float4 n = s.pn[i];
      abs_r += fabs(static_cast<double>(n.x) * (pt[0] - v.x) + static_cast<double>(n.y) * (pt[1] - v.y) +
                    static_cast<double>(n.z) * (pt[2] - v.z));
      ++observed;
    }
  }
  block_sum2(abs_r, observed);
  if (threadIdx.x == 0) stat_partials_put(s.spart, abs_r, static_cast<double>(observed), 0.0, 0.0, 0.0);
  if (!last_block(s.tickets + 3)) return;
  double tot[kStatParts];
  stat_partials_fold(s.spart, tot);
  if (threadIdx.x == 0) {
    const double sabs = tot[0];
    const long long nobs = static_cast<long long>(tot[1]);
    for (int k = 0; k + 1 < n_its; ++k)
      s.shape_stats[k].mean_abs_r_after = s.shape_stats[k + 1].mean_abs_r_before;
    if (n_its > 0) s.shape_stats[n_its - 1].mean_abs_r_after = nobs > 0 ? sabs / nobs : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Stage-hook kernels.

// solve_step on an explicit system (kinopt.cpp:121-130): out[0..n) = x,
// out[n] = 1 on success, 0 for NotPositiveDefinite.
static __global__ void k_solve_step(int n, const double* jtj, const double* jtr, double lambda_k,
                             double diag_floor, double* out) {
  extern __shared__ double sm[];
  double* A = sm;
  double* b = A + n * n;
  double* x = b + n;
  unsigned short* ea = reinterpret_cast<unsigned short*>(x + n);
  const int NT = n * (n + 1) / 2;
  unsigned short* eb = ea + NT;
  __shared__ int fin;
  if (threadIdx.x == 0) fin = 1;
  for (int e = threadIdx.x; e < NT; e += blockDim.x) {
    int r = 0, rem = e;
    while (rem >= n - r) {
      rem -= n - r;
      ++r;
    }
    ea[e] = static_cast<unsigned short>(r);
    eb[e] = static_cast<unsigned short>(r + rem);
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) A[e] = jtj[e];
  for (int k = threadIdx.x; k < n; k += blockDim.x) b[k] = jtr[k];
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x)
    A[k * n + k] = jtj[k * n + k] + lambda_k * jtj[k * n + k] + diag_floor;
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x)
    if (!isfinite(A[e])) fin = 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x)
    if (!isfinite(b[k])) fin = 0;
  __syncthreads();
  const int ok = fin ? block_ldlt_solve(n, n, A, b, x, ea, eb, NT) : 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) out[k] = ok ? x[k] : 0.0;
  if (threadIdx.x == 0) out[n] = ok ? 1.0 : 0.0;
}

static __global__ void k_solve_vertices(int n, const double* dr, const double* r, const double* phi,
                                 const double* nd, const int* ncount, double lphi, double lnbr,
                                 double lw, double floor_, double* delta, uint8_t* singular) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d[3];
  const bool ok = solve_vertex3(dr + 3 * i, r[i], phi + 3 * i, nd + 3 * i, ncount[i], lphi, lnbr,
                                lw, floor_, d);
  delta[3 * i] = d[0];
  delta[3 * i + 1] = d[1];
  delta[3 * i + 2] = d[2];
  singular[i] = ok ? 0 : 1;
}

// run_tracking's per-frame record (tracker.cpp:84-90): theta and the world
// origin of every link, transform_point(H_0j, 0), from the FK the frame's
// last pose-solve tail (or k_fk) left in s.fk for the current theta.
static __global__ void k_record(DevModel m, DevState s, double* theta_out, double* joints_out) {
  const int j = threadIdx.x;
  if (j >= m.L) return;
  if (theta_out) theta_out[j] = s.theta[j];
  if (joints_out) {
    const double zero[3] = {0.0, 0.0, 0.0};
    dq_transform_point(dq_load(s.fk + 8 * j), zero, joints_out + 3 * j);
  }
}

}  // namespace wt
