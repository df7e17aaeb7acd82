// wt_gpu.cu -- host orchestration and the C-ABI (include/wt_gpu.h) of the
// B200 tracking path. One wt_gpu_ctx owns the uploaded model, the per-
// sequence state (theta, Phi) and one CUDA stream; every frame is one
// captured CUDA graph of fixed shape (iteration counts are static), so the
// host issues a single graph launch per track_frame.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "wt_gpu.h"
#include "wt_kernels.cuh"

namespace wt {
// wt_exact.cu (compiled without FMA contraction)
void launch_skin(cudaStream_t st, int grid, int nseq, int L, const DevModel& m, const DevState& s,
                 const double4* phi);
void launch_normals(cudaStream_t st, int grid, int nseq, const DevModel& m, const DevState& s, const DevIntr& in,
                    int do_bucket, int zero_acc, int compute);
void launch_fk(cudaStream_t st, int nseq, const DevModel& m, const DevState& s);
void recon_launch(cudaStream_t st, const DevModel& m, const DevState& s, const DevIntr& in, int T, const int* tri,
                  double* v3, unsigned long long* zbits, int* owner, const uint8_t* pvalid, const double* pts,
                  double* ox, double* oy, double* oz, int* vis_list, int* counters, double* dist);
void launch_pose_solve(cudaStream_t st, int nseq, int L, const DevModel& m, const DevState& s, const PoseArgs& a);
void render_launch(cudaStream_t st, int V, int L, int T, const double* offsets, const double* v0,
                   const double* phi, const double* wgt, const int* wlink, const int* wcount,
                   const int* tri, const int* dom, double fx, double fy, double cx, double cy,
                   int W, int H, double sigma, double dropout, double quant, uint64_t base,
                   double* vpos, unsigned long long* zbits, int* owner, float* depth,
                   uint8_t* vis);
}

namespace {

thread_local std::string g_err;

struct CudaError {
  int code;
  std::string msg;
};

#define WT_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw CudaError{WT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};   \
  } while (0)

struct ApiError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw ApiError{code, msg}; }

template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  const cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess)
    throw CudaError{WT_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e)};
  return static_cast<T*>(p);
}

template <class T>
void upload(T* dst, const T* src, size_t n, cudaStream_t st) {
  if (n) WT_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

struct DevBuf {
  std::vector<void*> ptrs;
  template <class T>
  T* alloc(size_t n) {
    T* p = dalloc<T>(n);
    ptrs.push_back(p);
    return p;
  }
  ~DevBuf() {
    for (void* p : ptrs) cudaFree(p);
  }
};

struct GraphKey {
  std::vector<double> v;
  bool operator<(const GraphKey& o) const { return v < o.v; }
};

}  // namespace

struct wt_gpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int V = 0, L = 0, NP = 0, K = 0, T = 0;
  double lever = 1.0;  // max(1, largest template distance vertex <-> joint origin), x4 margin (pose_scales)
  std::vector<char> theta_prismatic;  // per theta index: its joint is prismatic (row entries <= 1, pose_scales)
  wt_intrinsics intr{};
  wt::DevIntr din{};
  int P = 0;

  // host model copies
  std::vector<wt::LinkDesc> links;
  std::vector<int> pair_off, pair_theta, pair_link, pair_owner;
  std::vector<double> s_diag;
  std::vector<int> dominant;

  DevBuf mem;
  wt::DevModel dm{};
  wt::DevState ds{};   // tracking state
  wt::DevState hs{};   // stage-hook state (scratch theta / fk / offsets / dchain)
  double4* phi[2] = {nullptr, nullptr};
  double4* phi_scratch = nullptr;
  int cur = 0;
  // batch: nseq sequences in lockstep, each with its own arena of per-sequence
  // buffers (ds, phi, frame, stats), bstride bytes apart (wt_kernels.cuh seq_state)
  int nseq = 1;
  long long bstride = 0;
  void* arena = nullptr;
  int last_nk = 0, last_ns = 0;  // iterations recorded by the last batch frame
  int frame_index = 0;
  bool fk_valid = false;  // ds.fk / offsets / dchain are the FK of ds.theta (skips k_fk at frame start)

  // frame
  float* d_depth = nullptr;
  uint8_t* d_valid = nullptr;
  double* d_pts_hi = nullptr;
  double4* d_vpts = nullptr;  // valid-pixel list records (point, pixel; k_ingest -> k_search)
  int* d_nvalid = nullptr;
  int* d_winners = nullptr;
  bool frame_loaded = false;
  // a device depth frame handed to wt_gpu_load_depth and not yet ingested: the
  // next track call copies and ingests it on a branch of its frame graph that
  // joins before the first search (track_frame_overlapped); any other frame
  // consumer ingests it first (require_frame)
  const float* pending_depth = nullptr;
  double pending_scale = 1.0;
  bool frame_on_rays = false;  // depth frame: every point on its pixel's centre ray

  // stats
  int cap_kin = 0, cap_shape = 0;
  wt::KinStat* h_kin = nullptr;
  wt::ShapeStat* h_shape = nullptr;
  // host mirror of theta, read back with a tracked frame's stats (one round
  // trip per frame); valid until the next API call on the context
  double* h_theta = nullptr;
  bool theta_mirror = false;
  double4* h_phi4 = nullptr;  // page-locked staging of Phi transfers (set_state / get_state), lazily allocated

  // renderer (fp64 copies, lazily built)
  double* r_v0 = nullptr;
  double* r_wgt = nullptr;
  int* r_wlink = nullptr;
  int* r_wcount = nullptr;
  int* r_tri = nullptr;
  int* r_dom = nullptr;
  double* r_off = nullptr;
  double* r_phi = nullptr;
  double* r_vpos = nullptr;
  unsigned long long* r_zbits = nullptr;
  int* r_owner = nullptr;
  float* r_depth = nullptr;
  uint8_t* r_vis = nullptr;
  std::vector<double> h_v0, h_wgt;
  std::vector<int> h_wlink, h_wcount, h_tri;

  // reconstruction error buffers (lazily built)
  double* rc_obs = nullptr;  // [3P] observed points, SoA
  int* rc_vis = nullptr;     // [V] visible vertices
  int* rc_cnt = nullptr;     // [2] visible / observed counts
  double* rc_dist = nullptr; // [V]

  int* hook_cnt = nullptr;
  double* hook_res = nullptr;
  long long* pose_dbg = nullptr;  // WT_DEBUG_POSE: last-CTA timing of the pose kernel

  // profiling: when set during capture, an event is recorded after every
  // kernel so per-kernel device time inside the real frame graph is known
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_events;
  std::vector<int> prof_kind;

  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<const void*, int> resident;  // CTAs of 256 threads resident per SM, per kernel (occupancy API)
  int sms = 148;

  // sequence driver: pinned staging + device double buffer + copy stream
  cudaStream_t copy_stream = nullptr;
  float* seq_pinned[2] = {nullptr, nullptr};
  float* seq_depth[2] = {nullptr, nullptr};
  cudaEvent_t seq_h2d[2] = {nullptr, nullptr};     // upload from slot b finished
  cudaEvent_t seq_ingest[2] = {nullptr, nullptr};  // ingest of slot b finished
  double* rec_buf = nullptr;                       // [cap_rec * L * 4] theta + joints
  int cap_rec = 0;

  // per-frame API with a pinned host frame: the upload and ingest are forked
  // onto up_stream inside the frame graph and joined before the first
  // search, so they overlap the first skin / normals / bucket build
  struct H2DGraph {
    cudaGraph_t graph;                  // kept: its memcpy nodes are re-pointed per launch
    cudaGraphExec_t exec;
    std::vector<cudaGraphNode_t> copy;  // the upload of sequence b's frame
  };
  std::map<GraphKey, H2DGraph> h2d_graphs;
  cudaStream_t up_stream = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  std::function<void()> before_search;  // the join, run once by the next enq_search
  bool walk_back = false;               // seq_walk: the next batched launch walks the sequences backwards

  ~wt_gpu_ctx() {
    for (int b = 0; b < 2; ++b) {
      if (seq_pinned[b]) cudaFreeHost(seq_pinned[b]);
      if (seq_h2d[b]) cudaEventDestroy(seq_h2d[b]);
      if (seq_ingest[b]) cudaEventDestroy(seq_ingest[b]);
    }
    if (copy_stream) cudaStreamDestroy(copy_stream);
    for (auto& kv : h2d_graphs) {
      cudaGraphExecDestroy(kv.second.exec);
      cudaGraphDestroy(kv.second.graph);
    }
    if (up_stream) cudaStreamDestroy(up_stream);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (join_ev) cudaEventDestroy(join_ev);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    for (cudaEvent_t e : prof_events) cudaEventDestroy(e);
    if (h_kin) cudaFreeHost(h_kin);
    if (h_theta) cudaFreeHost(h_theta);
    if (h_phi4) cudaFreeHost(h_phi4);
    if (h_shape) cudaFreeHost(h_shape);
    if (stream) cudaStreamDestroy(stream);
    if (arena) cudaFree(arena);
  }
};

namespace {

template <class F>
int guarded(wt_gpu_ctx* ctx, F&& f, bool keep_mirror = false) {
  if (ctx && !keep_mirror) ctx->theta_mirror = false;  // any other call may move theta
  try {
    f();
    return WT_OK;
  } catch (const ApiError& e) {
    (ctx ? ctx->err : g_err) = e.msg;
    return e.code;
  } catch (const CudaError& e) {
    (ctx ? ctx->err : g_err) = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    (ctx ? ctx->err : g_err) = e.what();
    return WT_EINVAL;
  }
}

void check_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw CudaError{WT_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

// kernel kinds reported by wt_gpu_profile_frame
enum { K_FK = 0, K_SKIN, K_NORMALS, K_SCATTER, K_SEARCH, K_POSE, K_SHAPE, K_SHAPE_AFTER, K_POSE_SOLVE, K_PIXOFF, K_NKIND };

void mark(wt_gpu_ctx* c, int kind) {
  check_launch();
  if (!c->prof_on) return;
  cudaEvent_t e;
  WT_CUDA(cudaEventCreate(&e));
  // External: becomes an event-record node of the captured graph
  WT_CUDA(cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal));
  c->prof_events.push_back(e);
  c->prof_kind.push_back(kind);
}

int vgrid(int n) { return std::max(1, (n + wt::kVThreads - 1) / wt::kVThreads); }

// One wave of `kernel` (kVThreads per CTA) on this device: resident CTAs per
// SM from the occupancy calculator (registers and shared memory as compiled)
// times the SM count.
template <class K>
int full_wave(wt_gpu_ctx* c, K kernel, int threads = wt::kVThreads, size_t smem = 0) {
  const void* key = reinterpret_cast<const void*>(kernel);
  auto it = c->resident.find(key);
  if (it == c->resident.end()) {
    int n = 0;
    WT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem));
    it = c->resident.emplace(key, std::max(1, n)).first;
  }
  return it->second * c->sms;
}

// per-sequence CTAs of a one-wave grid of `ctas` CTAs shared by a batch,
// times batch_mult waves for a batch (WT_WAVE_<kind> overrides it, experiments)
int wave(const wt_gpu_ctx* c, int ctas, const char* kind, double batch_mult = 1.0) {
  if (c->nseq == 1) return ctas;
  double mult = batch_mult;
  const char* e = getenv((std::string("WT_WAVE_") + kind).c_str());
  if (e) mult = atof(e);
  return std::max(1, static_cast<int>(ctas * mult / c->nseq));
}

// ---- validation (Skeleton::build, skeleton.cpp:7-50; bundle invariants) ----

void validate_model(const wt_model_desc* d) {
  if (!d) fail(WT_EINVAL, "model is NULL");
  const int L = d->n_links, V = d->n_vertices, T = d->n_triangles;
  if (L <= 0) fail(WT_EINVAL, "skeleton has no links");
  if (L > 64) fail(WT_EINVAL, "at most 64 links are supported on the GPU path");
  if (V < 0 || T < 0) fail(WT_ELENGTH, "negative vertex / triangle count");
  if (V >= (1 << 26)) fail(WT_EINVAL, "at most 2^26 vertices are supported");
  int roots = 0;
  std::vector<char> seen(static_cast<size_t>(L), 0);
  for (int j = 0; j < L; ++j) {
    const int p = d->parent[j];
    if (p < 0) ++roots;
    else if (p >= j)
      fail(WT_EINVAL, "link " + std::to_string(j) +
                          ": links are not topologically sorted (cycle or forward parent)");
    const int ti = d->theta_index[j];
    if (ti < 0 || ti >= L) fail(WT_EINVAL, "link " + std::to_string(j) + ": theta index out of range");
    if (seen[static_cast<size_t>(ti)])
      fail(WT_EINVAL, "link " + std::to_string(j) + ": duplicate theta index " + std::to_string(ti));
    seen[static_cast<size_t>(ti)] = 1;
    const double* ax = d->joint_axis + 3 * j;
    const double n = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
    if (std::abs(n - 1.0) > 1e-9) fail(WT_EINVAL, "link " + std::to_string(j) + ": axis is not unit length");
    if (d->joint_kind[j] != WT_JOINT_HINGE && d->joint_kind[j] != WT_JOINT_PRISMATIC)
      fail(WT_EINVAL, "link " + std::to_string(j) + ": unknown joint kind");
  }
  if (roots != 1)
    fail(WT_EINVAL, "skeleton must have exactly one root, found " + std::to_string(roots));
  for (int i = 0; i < V; ++i) {
    const int c = d->weight_count[i];
    if (c < 0 || c > 4) fail(WT_EINVAL, "vertex " + std::to_string(i) + ": weight count must be 0..4");
    for (int s = 0; s < c; ++s) {
      const int l = d->weight_link[4 * i + s];
      if (l < 0 || l >= L)
        fail(WT_EINVAL, "vertex " + std::to_string(i) + ": weight references link " +
                            std::to_string(l) + " out of range");
    }
  }
  for (int t = 0; t < 3 * T; ++t)
    if (d->triangles[t] < 0 || d->triangles[t] >= V)
      fail(WT_EINVAL, "triangle " + std::to_string(t / 3) + ": vertex index out of range");
  if (d->vtri_offsets[0] != 0) fail(WT_ELENGTH, "vertex->triangle CSR must start at 0");
  for (int i = 0; i < V; ++i)
    if (d->vtri_offsets[i + 1] < d->vtri_offsets[i]) fail(WT_ELENGTH, "vertex->triangle CSR not monotone");
  for (int c = 0; c < d->vtri_offsets[V]; ++c)
    if (d->vtri_items[c] < 0 || d->vtri_items[c] >= T)
      fail(WT_EINVAL, "vertex->triangle CSR references a missing triangle");
  if (d->nbr_offsets[0] != 0) fail(WT_ELENGTH, "neighbour CSR must start at 0");
  for (int i = 0; i < V; ++i) {
    if (d->nbr_offsets[i + 1] < d->nbr_offsets[i]) fail(WT_ELENGTH, "neighbour CSR not monotone");
    for (int c = d->nbr_offsets[i]; c < d->nbr_offsets[i + 1]; ++c) {
      const int n = d->nbr_items[c];
      if (n < 0 || n >= V) fail(WT_EINVAL, "vertex " + std::to_string(i) + ": neighbour out of range");
      if (n == i) fail(WT_EINVAL, "vertex " + std::to_string(i) + ": neighbor set contains the vertex itself");
    }
  }
}

// stage-hook state: own theta / fk / offsets / dchain, sequence 0's per-vertex buffers
void alloc_hook_state(wt_gpu_ctx* c, wt::DevState& s) {
  s.theta = c->mem.alloc<double>(c->L);
  s.fk = c->mem.alloc<double>(8 * c->L);
  s.offsets = c->mem.alloc<double>(8 * c->L);
  s.dchain = c->mem.alloc<double>(8 * std::max(1, c->NP));
  s.bstride = 0;
}

// Bump allocator over one sequence's arena (a dry run with base = nullptr
// only measures it).
struct Carve {
  char* base = nullptr;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~static_cast<size_t>(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += sizeof(T) * std::max<size_t>(n, 1);
    return p;
  }
};

constexpr int kArenaKin = 64, kArenaShape = 32;  // stats slots per sequence arena

// Every per-sequence buffer, in arena order. Zero-initialised arenas are a
// valid initial state (theta = 0; the self-cleaning counters and slots 0).
void layout_seq(wt_gpu_ctx* c, Carve& a) {
  const int L = c->L, V = c->V, P = c->P, H = c->din.H;
  wt::DevState& s = c->ds;
  s.theta = a.take<double>(L);
  s.fk = a.take<double>(8 * L);
  s.offsets = a.take<double>(8 * L);
  s.dchain = a.take<double>(8 * std::max(1, c->NP));
  s.pv = a.take<double4>(V);
  s.pn = a.take<float4>(V);
  s.vpix = a.take<int>(V);
  s.pix_cnt = a.take<int>(P);
  s.row_cnt = a.take<int>(H);
  s.poff = a.take<int>(P + 1);
  s.items = a.take<double4>(V);
  s.acc = a.take<unsigned long long>(4 * static_cast<size_t>(std::max(1, V)));
  s.red = a.take<unsigned long long>(wt::kRedCopies * (L * (L + 1) / 2 + L + 2) + 8);
  s.tickets = a.take<unsigned>(8);
  s.sys_out = a.take<double>(L * L + L);
  s.kin_stats = a.take<wt::KinStat>(kArenaKin);
  s.shape_stats = a.take<wt::ShapeStat>(kArenaShape);
  c->phi[0] = a.take<double4>(V);
  c->phi[1] = a.take<double4>(V);
  c->d_depth = a.take<float>(P);
  c->d_valid = a.take<uint8_t>(P);
  c->d_pts_hi = a.take<double>(3 * static_cast<size_t>(P));
  // valid-pixel list: one run of 32 entries per 32-column row segment
  c->d_vpts = a.take<double4>(32 * H * ((c->din.W + 31) / 32));
  c->d_nvalid = a.take<int>(4);  // frame words: [0] list length, [2..3] max |coordinate| (k_ingest)
  s.fwords = c->d_nvalid;
  s.spart = a.take<double>(static_cast<size_t>(wt::kStatParts) * vgrid(V));
  c->d_winners = a.take<int>(P);
}

void alloc_arenas(wt_gpu_ctx* c) {
  Carve dry;
  layout_seq(c, dry);
  const size_t S = (dry.off + 4095) & ~static_cast<size_t>(4095);
  WT_CUDA(cudaMalloc(&c->arena, S * static_cast<size_t>(c->nseq)));
  WT_CUDA(cudaMemsetAsync(c->arena, 0, S * static_cast<size_t>(c->nseq), c->stream));
  Carve real;
  real.base = static_cast<char*>(c->arena);
  layout_seq(c, real);
  c->bstride = c->nseq > 1 ? static_cast<long long>(S) : 0;
  c->ds.bstride = c->bstride;
  c->cap_kin = kArenaKin;
  c->cap_shape = kArenaShape;
  WT_CUDA(cudaMallocHost(&c->h_kin, sizeof(wt::KinStat) * c->cap_kin * c->nseq));
  WT_CUDA(cudaMallocHost(&c->h_shape, sizeof(wt::ShapeStat) * c->cap_shape * c->nseq));
  WT_CUDA(cudaMallocHost(&c->h_theta, sizeof(double) * c->L));
}

template <class T>
T* seq_at(T* p, const wt_gpu_ctx* c, int seq) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(p) + static_cast<long long>(seq) * c->bstride);
}

void require_single(const wt_gpu_ctx* c) {
  if (c->nseq != 1) fail(WT_EINVAL, "not available on a batch context (use the wt_gpu_batch_* calls)");
}

// Every captured frame graph (plain and pinned-upload forms) bakes the stats
// buffers into its kernel parameters: a reallocation must drop them all.
void drop_graphs(wt_gpu_ctx* c) {
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  c->graphs.clear();
  for (auto& kv : c->h2d_graphs) {
    cudaGraphExecDestroy(kv.second.exec);
    cudaGraphDestroy(kv.second.graph);
  }
  c->h2d_graphs.clear();
}

void ensure_stats(wt_gpu_ctx* c, int nk, int ns) {
  if ((nk > c->cap_kin || ns > c->cap_shape) && c->nseq > 1)
    fail(WT_EINVAL, "a batch records at most " + std::to_string(kArenaKin) + " pose / " +
                        std::to_string(kArenaShape) + " surface iterations per frame");
  if (nk > c->cap_kin) {
    c->cap_kin = std::max(nk, 16);
    c->ds.kin_stats = c->mem.alloc<wt::KinStat>(c->cap_kin);
    if (c->h_kin) cudaFreeHost(c->h_kin);
    WT_CUDA(cudaMallocHost(&c->h_kin, sizeof(wt::KinStat) * c->cap_kin));
    drop_graphs(c);
  }
  if (ns > c->cap_shape) {
    c->cap_shape = std::max(ns, 8);
    c->ds.shape_stats = c->mem.alloc<wt::ShapeStat>(c->cap_shape);
    if (c->h_shape) cudaFreeHost(c->h_shape);
    WT_CUDA(cudaMallocHost(&c->h_shape, sizeof(wt::ShapeStat) * c->cap_shape));
    drop_graphs(c);
  }
}

// ---- kernel launch helpers (all on ctx->stream) ------------------------------

// A batch walks its sequences in alternating order from one launch to the
// next (blockIdx.y ascending, then descending: a negative stride, seq_off):
// the sequences a kernel touched last are still in L2 when the next kernel
// starts with them.
wt::DevState seq_walk(wt_gpu_ctx* c, wt::DevState s) {
  if (c->nseq > 1 && c->walk_back) s.bstride = -s.bstride;
  c->walk_back = !c->walk_back;
  return s;
}

void enq_fk(wt_gpu_ctx* c, const wt::DevState& s) {
  wt::launch_fk(c->stream, c->nseq, c->dm, seq_walk(c, s));
  mark(c, K_FK);
}

void enq_skin(wt_gpu_ctx* c, const wt::DevState& s, const double4* phi) {
  wt::launch_skin(c->stream, vgrid(c->V), c->nseq, c->L, c->dm, seq_walk(c, s), phi);
  mark(c, K_SKIN);
}

void enq_normals(wt_gpu_ctx* c, const wt::DevState& s, bool bucket, bool zero_acc,
                 bool compute = true) {
  wt::launch_normals(c->stream, vgrid(c->V), c->nseq, c->dm, seq_walk(c, s), c->din, bucket ? 1 : 0, zero_acc ? 1 : 0,
                     compute ? 1 : 0);
  mark(c, K_NORMALS);
}

void enq_scatter(wt_gpu_ctx* c, const wt::DevState& s) {
  WT_CUDA(wt::launch_pdl(c->nseq > 1 ? wt::k_pixoff<true> : wt::k_pixoff<false>, dim3((c->din.H + 7) / 8, c->nseq), dim3(wt::kVThreads), 0, c->stream,
                         seq_walk(c, s), c->din.W, c->din.H));
  mark(c, K_PIXOFF);
  WT_CUDA(wt::launch_pdl(c->nseq > 1 ? wt::k_scatter<true> : wt::k_scatter<false>,
                         dim3(vgrid(std::max(c->V, c->din.H)), c->nseq), dim3(wt::kVThreads), 0, c->stream, c->dm,
                         seq_walk(c, s), c->din.H));
  mark(c, K_SCATTER);
}

void enq_search(wt_gpu_ctx* c, const wt::DevState& s, const wt_assoc_config* a, int* winners) {
  if (c->before_search) {  // the frame's upload + ingest, forked off earlier in this graph
    auto join = std::move(c->before_search);
    c->before_search = nullptr;
    join();
  }
  wt::DevFrame f{c->d_valid, c->d_pts_hi, c->d_vpts, c->d_nvalid, c->bstride};
  wt::SearchArgs sa;
  sa.fx = c->din.fx;
  sa.fy = c->din.fy;
  sa.cx = c->din.cx;
  sa.cy = c->din.cy;
  sa.prune = c->frame_on_rays ? 1 : 0;
  sa.W = c->din.W;
  sa.H = c->din.H;
  sa.window = a->window_radius;
  sa.cut2 = a->cutoff * a->cutoff;
  sa.write_winners = winners ? 1 : 0;
  sa.winners = winners;
  // G lanes per valid pixel; at most P pixels (the list is padded per 32 columns)
  // one wave (5 CTAs per SM fit the registers); warps stride over the 4-pixel groups
  // (a batch shares the wave between its sequences)
  // the narrow 3x3-core form pays once the batch makes the search
  // throughput-bound; small batches stay latency-bound and keep the solo form
  static const int narrow_from = getenv("WT_NARROW_SEARCH_FROM") ? atoi(getenv("WT_NARROW_SEARCH_FROM")) : 8;
  const bool narrow = c->nseq > 1 && c->nseq >= narrow_from;
  const int G = narrow ? wt::kSearchGroupBatch : wt::kSearchGroupSolo;  // grid sizing
  // a lone frame of more than 2^20 pixels (C4) has enough pixels in flight to
  // be throughput-bound: one lane per core row, 8-lane groups (1080p: 572 ->
  // 647 frames/s against the VGA form)
  const bool big_frame = c->nseq == 1 && c->P > (1 << 20);
  auto kern = c->nseq > 1 ? (narrow ? wt::k_search<true>
                                    : wt::k_search<true, wt::kNearRingsSolo, wt::kSearchGroupSolo, wt::kSearchSplitSolo>)
                          : (big_frame ? wt::k_search<false, wt::kNearRingsSolo, 8, 1> : wt::k_search<false>);
  // one wave (warps stride over the pixel groups); a batch shares 8 waves between its sequences
  const int grid = std::max(1, std::min(c->P * G / wt::kVThreads + 1, wave(c, full_wave(c, kern), "SEARCH", 8.0)));
  const wt::DevState sw = seq_walk(c, s);
  f.bstride = sw.bstride;
  WT_CUDA(wt::launch_pdl(kern, dim3(grid, c->nseq), dim3(wt::kVThreads), 0, c->stream, sw, f, sa));
  mark(c, K_SEARCH);
}

// zero_acc: clear the observation sums first (stage hooks); the frame graphs
// rely on their consumers leaving them clean (clear_acc, wt_kernels.cuh)
void enq_associate(wt_gpu_ctx* c, const wt::DevState& s, const wt_assoc_config* a, int* winners,
                   bool zero_acc = false) {
  enq_normals(c, s, true, zero_acc);
  enq_scatter(c, s);
  enq_search(c, s, a, winners);
}

// 256-thread CTAs, two resident per SM (registers): one wave of 296 CTAs,
// ~43 vertices per warp at C3 (two scan chunks each) and half the per-CTA
// reduction atomics of 128-thread CTAs (C3 2119 -> 2141 frames/s); 128 when
// 8 warps' row tiles exceed the shared memory (L > ~50)
int pose_threads(const wt_gpu_ctx* c) {
  return wt::pose_smem_bytes(c->L, c->NP, wt::kPoseThreads / 32) <= 227 * 1024 ? wt::kPoseThreads : 128;
}

// one wave of the pose kernel (occupancy calculator: registers and the
// dynamic shared memory of this skeleton); a batch shares two waves between
// its sequences (C5 6714 -> 6733 frames/s against one)
template <class K>
int pose_grid(wt_gpu_ctx* c, K kernel) {
  const int warps = pose_threads(c) / 32;
  const int wave_ctas = full_wave(c, kernel, pose_threads(c), wt::pose_smem_bytes(c->L, c->NP, warps));
  return std::max(1, std::min((c->V + 32 * warps - 1) / (32 * warps), wave(c, wave_ctas, "POSE", 2.0)));
}

// JtJ entries per lane (upper triangle + Jtr) held in registers
int pose_q(int L) {
  const int ne = L * (L + 1) / 2 + L;
  return ne <= 32 * 8 ? 8 : ne <= 32 * 16 ? 16 : ne <= 32 * 32 ? 32 : 68;
}

template <int Q, int TPL>
void launch_pose(wt_gpu_ctx* c, const wt::DevState& s, const double4* phi, const wt::PoseArgs& pa) {
  auto kern = c->nseq > 1 ? wt::k_pose_system<Q, TPL, true> : wt::k_pose_system<Q, TPL, false>;
  WT_CUDA(wt::launch_pdl(kern, dim3(pose_grid(c, kern), c->nseq), dim3(pose_threads(c)),
                         wt::pose_smem_bytes(c->L, c->NP, pose_threads(c) / 32), c->stream, c->dm, seq_walk(c, s), phi,
                         pa));
}

template <int Q, int TPL>
void pose_attr(wt_gpu_ctx* c) {
  const int bytes = static_cast<int>(wt::pose_smem_bytes(c->L, c->NP, pose_threads(c) / 32));
  WT_CUDA(cudaFuncSetAttribute(wt::k_pose_system<Q, TPL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  WT_CUDA(cudaFuncSetAttribute(wt::k_pose_system<Q, TPL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

// Fixed-point scales of the pose reduction (wt_kernels.cuh): row entry k is
// n . dv/dtheta_k, at most b_k = the lever arm R for a hinge (c->lever, the
// template's with a 4x margin for pose and Phi) and 1 for a prismatic joint,
// and |r| <= cutoff = b_L; so over V vertices |JtJ_ab| <= V b_a b_b and
// |Jtr_a| <= V b_a cutoff. Entry (a, b) is scaled by 2^(x_a + x_b), per-theta
// exponents with x_k <= floor((62 - e_V) / 2) - e_k (V < 2^e_V, b_k < 2^e_k):
// every entry stays below 2^62, and a prismatic entry in millimetres keeps
// its own resolution instead of the hinges' (the widest entry's scale for all,
// before). x_k <= 20: at most 2^-40, the metre-scale value. sum r^2 <= V
// cutoff^2 has a scale of its own.
double pow2_below(double bound, int cap) {
  int ex = 0;
  std::frexp(std::max(bound, 1e-300), &ex);  // bound < 2^ex
  return std::ldexp(1.0, std::min(cap, 62 - ex));
}

int exp2_above(double b) {  // e with b < 2^e
  int ex = 0;
  std::frexp(std::max(b, 1e-300), &ex);
  return ex;
}

void pose_scales(const wt_gpu_ctx* c, double cutoff, wt::PoseArgs& pa) {
  const double V = std::max(1, c->V), R = c->lever;
  const int half = (62 - exp2_above(V)) / 2;
  for (int k = 0; k <= c->L; ++k) {
    const double b = k == c->L ? cutoff : (c->theta_prismatic[static_cast<size_t>(k)] ? 1.0 : R);
    pa.fexp[k] = static_cast<signed char>(std::max(-60, std::min(20, half - exp2_above(b))));
  }
  pa.res_scale = pow2_below(2.0 * V * cutoff * cutoff, 44);
  pa.res_inv = 1.0 / pa.res_scale;
}

void enq_pose(wt_gpu_ctx* c, const wt::DevState& s, const double4* phi, const wt_kin_config* k,
              int it, bool solve, const int* count_in, const double* res_in, double cutoff, bool clean_acc = false) {
  wt::PoseArgs pa;
  pose_scales(c, cutoff, pa);
  pa.lambda_k = k->lambda_k;
  pa.lambda_s = k->lambda_s;
  pa.diag_floor = k->diag_floor;
  pa.limit = k->limit;
  pa.clamp = k->clamp_limits;
  pa.iteration = it;
  pa.solve = solve ? 1 : 0;
  pa.clean_acc = clean_acc ? 1 : 0;
  pa.count_in = count_in;
  pa.res_in = res_in;
  pa.dbg = c->pose_dbg;
  const int edge = wt::pose_tile_edge(c->L);
  if (edge == 3) {
    launch_pose<1, 3>(c, s, phi, pa);
  } else if (edge == 4) {
    launch_pose<1, 4>(c, s, phi, pa);
  } else {
    switch (pose_q(c->L)) {
      case 8: launch_pose<8, 0>(c, s, phi, pa); break;
      case 16: launch_pose<16, 0>(c, s, phi, pa); break;
      case 32: launch_pose<32, 0>(c, s, phi, pa); break;
      default: launch_pose<68, 0>(c, s, phi, pa); break;
    }
  }
  mark(c, K_POSE);
  wt::launch_pose_solve(c->stream, c->nseq, c->L, c->dm, seq_walk(c, s), pa);
  mark(c, K_POSE_SOLVE);
}

// a batch: four waves of the 4-CTA/SM grid shared by its sequences (C5: 453 -> 366 us)
int shape_grid(const wt_gpu_ctx* c) { return std::max(1, std::min(vgrid(c->V), wave(c, 4 * 148, "SHAPE", 4.0))); }

void enq_shape(wt_gpu_ctx* c, const wt_shape_config* sc, int it, const double4* in, double4* out) {
  // the shape step is the association's only consumer: it leaves the sums clean
  wt::ShapeArgs sa;
  sa.lambda_phi = sc->lambda_phi;
  sa.lambda_nbr = sc->lambda_nbr;
  sa.lambda_w = sc->lambda_w;
  sa.diag_floor = sc->diag_floor;
  sa.iteration = it;
  sa.clean_acc = 1;
  WT_CUDA(wt::launch_pdl(c->nseq > 1 ? wt::k_shape<true> : wt::k_shape<false>, dim3(shape_grid(c), c->nseq), dim3(wt::kVThreads), sizeof(double) * 8 * c->L, c->stream,
                         c->dm, seq_walk(c, c->ds), in, out, sa));
  mark(c, K_SHAPE);
}

// optimize_pose (kinopt.cpp:132-171) as a static kernel sequence.
void enq_optimize_pose(wt_gpu_ctx* c, const wt_kin_config* k, const wt_assoc_config* a, bool need_fk) {
  if (need_fk) enq_fk(c, c->ds);
  const int refresh = std::max(1, k->assoc_refresh);
  for (int it = 0; it < k->iterations; ++it) {
    enq_skin(c, c->ds, c->phi[c->cur]);
    if (it % refresh == 0) {
      enq_associate(c, c->ds, a, nullptr);
    } else {
      // correspondences kept, residuals follow the moved surface (:145-150)
      enq_normals(c, c->ds, false, false);
    }
    // the last pose system before a re-association (or the end) cleans the sums
    const bool last_use = (it + 1) % refresh == 0 || it + 1 == k->iterations;
    enq_pose(c, c->ds, c->phi[c->cur], k, it, true, nullptr, nullptr, a->cutoff, last_use);
  }
}

// optimize_shape (shapeopt.cpp:50-130). Returns the new current phi index.
int enq_optimize_shape(wt_gpu_ctx* c, int cur, const wt_shape_config* sc, const wt_assoc_config* a,
                       bool stats_pass, bool need_fk) {
  if (need_fk) enq_fk(c, c->ds);
  for (int it = 0; it < sc->iterations; ++it) {
    enq_skin(c, c->ds, c->phi[cur]);
    enq_associate(c, c->ds, a, nullptr);
    enq_shape(c, sc, it, c->phi[cur], c->phi[cur ^ 1]);
    cur ^= 1;  // Jacobi swap (shapeopt.cpp:98)
  }
  if (stats_pass && sc->iterations > 0) {
    enq_skin(c, c->ds, c->phi[cur]);
    enq_associate(c, c->ds, a, nullptr);
    WT_CUDA(wt::launch_pdl(c->nseq > 1 ? wt::k_shape_after<true> : wt::k_shape_after<false>, dim3(shape_grid(c), c->nseq), dim3(wt::kVThreads), 0, c->stream, c->dm,
                           seq_walk(c, c->ds), sc->iterations, 1));
    mark(c, K_SHAPE_AFTER);
  }
  return cur;
}

void check_assoc(const wt_assoc_config* a) {
  if (!a) fail(WT_EINVAL, "assoc config is NULL");
  if (a->window_radius < 0 || a->window_radius > 16)
    fail(WT_EINVAL, "window_radius must be in [0, 16] on the GPU path");
  if (!(a->cutoff >= 0.0)) fail(WT_EINVAL, "cutoff must be >= 0");
}

void require_frame(wt_gpu_ctx* c) {
  if (!c->frame_loaded) fail(WT_EINVAL, "no frame loaded (call wt_gpu_load_depth / wt_gpu_load_cloud)");
}

void run_graph(wt_gpu_ctx* c, const GraphKey& key, const std::function<void()>& body) {
  auto it = c->graphs.find(key);
  if (it == c->graphs.end()) {
    cudaGraph_t g;
    WT_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      body();
    } catch (...) {
      cudaStreamEndCapture(c->stream, &g);
      throw;
    }
    WT_CUDA(cudaStreamEndCapture(c->stream, &g));
    cudaGraphExec_t ex;
    WT_CUDA(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    it = c->graphs.emplace(key, ex).first;
  }
  WT_CUDA(cudaGraphLaunch(it->second, c->stream));
}

void put_kin(const wt_gpu_ctx* c, int n, wt_kin_iter_stats* out, int cap, int seq = 0) {
  const wt::KinStat* h = c->h_kin + static_cast<size_t>(seq) * c->cap_kin;
  for (int k = 0; k < n && k < cap; ++k) {
    out[k].iteration = k;
    out[k].associated = h[k].associated;
    out[k].residual_sum = h[k].residual_sum;
    out[k].step_norm = h[k].step_norm;
    out[k].solver_skipped = h[k].skipped;
    out[k].pad_ = 0;
  }
}

void put_shape(const wt_gpu_ctx* c, int n, wt_shape_iter_stats* out, int cap, int seq = 0) {
  const wt::ShapeStat* h = c->h_shape + static_cast<size_t>(seq) * c->cap_shape;
  for (int k = 0; k < n && k < cap; ++k) {
    out[k].iteration = k;
    out[k].singular = h[k].singular;
    out[k].mean_phi = h[k].mean_phi;
    out[k].max_phi = h[k].max_phi;
    out[k].mean_abs_r_before = h[k].mean_abs_r_before;
    out[k].mean_abs_r_after = h[k].mean_abs_r_after;
  }
}


// A tracked frame's results back on the host: the stats (FrameStats) and
// theta (the host mirror), one synchronisation; then the frame counter.
// A pose iteration whose fixed-point normal equations left the int64 range
// (k_pose_solve, skipped == 2) is an error, not a silent skip.
void check_range(const wt_gpu_ctx* c, int nk) {
  for (int k = 0; k < nk; ++k)
    if (c->h_kin[k].skipped == 2)
      fail(WT_ERANGE, "pose iteration " + std::to_string(k) +
                          ": normal equations outside the fixed-point range of the device reduction");
}

void frame_readback(wt_gpu_ctx* c, int nk, int ns, wt_frame_stats* stats) {
  if (nk) WT_CUDA(cudaMemcpyAsync(c->h_kin, c->ds.kin_stats, sizeof(wt::KinStat) * nk, cudaMemcpyDeviceToHost,
                                  c->stream));
  if (stats && ns)
    WT_CUDA(cudaMemcpyAsync(c->h_shape, c->ds.shape_stats, sizeof(wt::ShapeStat) * ns, cudaMemcpyDeviceToHost,
                            c->stream));
  WT_CUDA(cudaMemcpyAsync(c->h_theta, c->ds.theta, sizeof(double) * c->L, cudaMemcpyDeviceToHost, c->stream));
  WT_CUDA(cudaStreamSynchronize(c->stream));
  c->theta_mirror = true;
  check_range(c, nk);
  if (stats) {
    stats->frame = c->frame_index;
    stats->n_kin = nk;
    stats->n_shape = ns;
    if (stats->kin) put_kin(c, nk, stats->kin, stats->cap_kin);
    if (stats->shape) put_shape(c, ns, stats->shape, stats->cap_shape);
  }
  ++c->frame_index;
}

// Phi moves between the caller's packed [V][3] array and the device's
// double4 records through a page-locked staging buffer (one DMA each way).
double4* phi_stage(wt_gpu_ctx* c) {
  if (!c->h_phi4) WT_CUDA(cudaMallocHost(&c->h_phi4, sizeof(double4) * std::max(1, c->V)));
  return c->h_phi4;
}

void phi_put(wt_gpu_ctx* c, double4* dst, const double* phi) {
  double4* h = phi_stage(c);
  WT_CUDA(cudaStreamSynchronize(c->stream));  // the staging buffer is free
  for (int i = 0; i < c->V; ++i) h[i] = make_double4(phi[3 * i], phi[3 * i + 1], phi[3 * i + 2], 0.0);
  WT_CUDA(cudaMemcpyAsync(dst, h, sizeof(double4) * c->V, cudaMemcpyHostToDevice, c->stream));
  WT_CUDA(cudaStreamSynchronize(c->stream));
}

// enqueues the download; phi_unpack after the stream synchronised
void phi_get_async(wt_gpu_ctx* c, const double4* src) {
  WT_CUDA(cudaMemcpyAsync(phi_stage(c), src, sizeof(double4) * c->V, cudaMemcpyDeviceToHost, c->stream));
}

void phi_unpack(const wt_gpu_ctx* c, double* phi) {
  const double4* h = c->h_phi4;
  for (int i = 0; i < c->V; ++i) {
    phi[3 * i] = h[i].x;
    phi[3 * i + 1] = h[i].y;
    phi[3 * i + 2] = h[i].z;
  }
}

// rows of `width` bytes, one per sequence arena, to / from a packed host array
void copy_from_seqs(const wt_gpu_ctx* c, void* dst, size_t dpitch, const void* src, size_t width) {
  if (width == 0) return;
  if (c->nseq == 1) {
    WT_CUDA(cudaMemcpyAsync(dst, src, width, cudaMemcpyDefault, c->stream));
  } else {
    WT_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, static_cast<size_t>(c->bstride), width, c->nseq, cudaMemcpyDefault,
                              c->stream));
  }
}

void copy_to_seqs(const wt_gpu_ctx* c, void* dst, const void* src, size_t spitch, size_t width,
                  cudaStream_t st = nullptr, cudaMemcpyKind kind = cudaMemcpyDefault) {
  if (width == 0) return;
  if (!st) st = c->stream;
  if (c->nseq == 1) {
    WT_CUDA(cudaMemcpyAsync(dst, src, width, kind, st));
  } else {
    WT_CUDA(cudaMemcpy2DAsync(dst, static_cast<size_t>(c->bstride), src, spitch, width, c->nseq, kind, st));
  }
}

void ensure_render(wt_gpu_ctx* c) {
  if (c->r_v0) return;
  const int V = c->V, P = c->P;
  c->r_v0 = c->mem.alloc<double>(3 * V);
  c->r_wgt = c->mem.alloc<double>(4 * V);
  c->r_wlink = c->mem.alloc<int>(4 * V);
  c->r_wcount = c->mem.alloc<int>(V);
  c->r_tri = c->mem.alloc<int>(3 * std::max(1, c->T));
  c->r_dom = c->mem.alloc<int>(V);
  c->r_off = c->mem.alloc<double>(8 * c->L);
  c->r_phi = c->mem.alloc<double>(3 * V);
  c->r_vpos = c->mem.alloc<double>(3 * V);
  c->r_zbits = c->mem.alloc<unsigned long long>(P);
  c->r_owner = c->mem.alloc<int>(P);
  c->r_depth = c->mem.alloc<float>(P);
  c->r_vis = c->mem.alloc<uint8_t>(c->L);
  upload(c->r_v0, c->h_v0.data(), 3 * V, c->stream);
  upload(c->r_wgt, c->h_wgt.data(), 4 * V, c->stream);
  upload(c->r_wlink, c->h_wlink.data(), 4 * V, c->stream);
  upload(c->r_wcount, c->h_wcount.data(), V, c->stream);
  upload(c->r_tri, c->h_tri.data(), 3 * c->T, c->stream);
  upload(c->r_dom, c->dominant.data(), V, c->stream);
}

void host_offsets(const wt_gpu_ctx* c, const double* theta, double* out) {
  std::vector<wt::DQ> fk(static_cast<size_t>(c->L));
  wt::fk_all(c->links.data(), c->L, theta, fk.data());
  for (int j = 0; j < c->L; ++j)
    wt::dq_store(wt::dq_compose(fk[j], wt::dq_load(c->links[j].bind_inv)), out + 8 * j);
}

}  // namespace

extern "C" {

int wt_gpu_abi_version(void) { return WT_ABI_VERSION; }

int wt_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

const char* wt_gpu_global_last_error(void) { return g_err.c_str(); }
const char* wt_gpu_last_error(const wt_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

}  // extern "C"

namespace {
int create_ctx(int device, const wt_model_desc* d, const wt_intrinsics* intr, int nseq, wt_gpu_ctx** out) {
  if (!out) {
    g_err = "out is NULL";
    return WT_EINVAL;
  }
  *out = nullptr;
  auto* c = new wt_gpu_ctx();
  const int rc = guarded(nullptr, [&] {
    if (nseq < 1 || nseq > 4096) fail(WT_EINVAL, "batch size must be in 1..4096");
    c->nseq = nseq;
    validate_model(d);
    if (!intr || intr->width <= 0 || intr->height <= 0) fail(WT_EINVAL, "bad intrinsics");
    if (intr->width > 32 * wt::kRowChunks) fail(WT_EINVAL, "image rows wider than 2048 pixels are not supported");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      fail(WT_ENODEV, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) fail(WT_ENODEV, "device index out of range");
    c->device = device;
    WT_CUDA(cudaSetDevice(device));
    WT_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    WT_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
    c->L = d->n_links;
    c->V = d->n_vertices;
    c->T = d->n_triangles;
    c->intr = *intr;
    c->din.fx = intr->fx;
    c->din.fy = intr->fy;
    c->din.cx = intr->cx;
    c->din.cy = intr->cy;
    c->din.W = intr->width;
    c->din.H = intr->height;
    c->P = intr->width * intr->height;
    const int L = c->L, V = c->V;

    // skeleton: bind pose = FK(0), ancestors, dchain pairs (skeleton.cpp:7-50)
    c->links.resize(static_cast<size_t>(L));
    std::vector<int> theta_to_link(static_cast<size_t>(L));
    for (int j = 0; j < L; ++j) {
      wt::LinkDesc& l = c->links[static_cast<size_t>(j)];
      l.parent = d->parent[j];
      l.kind = d->joint_kind[j];
      l.theta_index = d->theta_index[j];
      l.pad = 0;
      for (int k = 0; k < 3; ++k) l.axis[k] = d->joint_axis[3 * j + k];
      for (int k = 0; k < 8; ++k) l.offset[k] = d->parent_offset[8 * j + k];
      theta_to_link[static_cast<size_t>(l.theta_index)] = j;
    }
    c->theta_prismatic.assign(static_cast<size_t>(L), 0);
    for (int k = 0; k < L; ++k)
      c->theta_prismatic[static_cast<size_t>(k)] = d->joint_kind[theta_to_link[static_cast<size_t>(k)]] == WT_JOINT_PRISMATIC;
    std::vector<double> zero(static_cast<size_t>(L), 0.0);
    std::vector<wt::DQ> bind(static_cast<size_t>(L));
    wt::fk_all(c->links.data(), L, zero.data(), bind.data());
    for (int j = 0; j < L; ++j) wt::dq_store(wt::dq_inverse(bind[j]), c->links[j].bind_inv);
    {
      // lever arm bound of the pose rows: template vertex <-> bind-pose joint origin
      std::vector<double> org(3 * static_cast<size_t>(L));
      for (int j = 0; j < L; ++j) {
        const double zero[3] = {0.0, 0.0, 0.0};
        wt::dq_transform_point(bind[j], zero, &org[3 * j]);
      }
      double r2 = 0.0;
      for (int i = 0; i < d->n_vertices; ++i)
        for (int j = 0; j < L; ++j) {
          const double dx = d->v0[3 * i] - org[3 * j], dy = d->v0[3 * i + 1] - org[3 * j + 1],
                       dz = d->v0[3 * i + 2] - org[3 * j + 2];
          r2 = std::max(r2, dx * dx + dy * dy + dz * dz);
        }
      c->lever = std::max(1.0, 4.0 * std::sqrt(r2));
    }
    std::vector<std::vector<int>> anc(static_cast<size_t>(L));
    c->pair_off.assign(1, 0);
    for (int j = 0; j < L; ++j) {
      std::vector<int> path;
      for (int cur = j; cur >= 0; cur = d->parent[cur]) path.push_back(d->theta_index[cur]);
      std::reverse(path.begin(), path.end());
      anc[static_cast<size_t>(j)] = path;
      for (int k : path) {
        c->pair_theta.push_back(k);
        c->pair_link.push_back(theta_to_link[static_cast<size_t>(k)]);
        c->pair_owner.push_back(j);
      }
      c->pair_off.push_back(static_cast<int>(c->pair_theta.size()));
    }
    c->NP = static_cast<int>(c->pair_theta.size());
    // influence counts S (kinopt.cpp:58-70)
    c->s_diag.assign(static_cast<size_t>(L), 0.0);
    std::vector<char> hit(static_cast<size_t>(L));
    for (int i = 0; i < V; ++i) {
      std::fill(hit.begin(), hit.end(), 0);
      for (int s = 0; s < d->weight_count[i]; ++s)
        for (int k : anc[static_cast<size_t>(d->weight_link[4 * i + s])]) hit[static_cast<size_t>(k)] = 1;
      for (int k = 0; k < L; ++k)
        if (hit[static_cast<size_t>(k)]) c->s_diag[static_cast<size_t>(k)] += 1.0;
    }

    // per-vertex device layout
    std::vector<double4> v0(static_cast<size_t>(V)), wg(static_cast<size_t>(V)), ph(static_cast<size_t>(V));
    std::vector<uchar4> wl(static_cast<size_t>(V));
    c->h_v0.assign(d->v0, d->v0 + 3 * V);
    c->h_wgt.assign(static_cast<size_t>(4 * V), 0.0);
    c->h_wlink.assign(static_cast<size_t>(4 * V), 0);
    c->h_wcount.assign(d->weight_count, d->weight_count + V);
    c->dominant.assign(static_cast<size_t>(V), -1);
    for (int i = 0; i < V; ++i) {
      v0[i] = make_double4(d->v0[3 * i], d->v0[3 * i + 1], d->v0[3 * i + 2], 0.0);
      const double* p = d->phi ? d->phi + 3 * i : nullptr;
      ph[i] = p ? make_double4(p[0], p[1], p[2], 0.0) : make_double4(0, 0, 0, 0);
      double w[4] = {0, 0, 0, 0};
      unsigned char lk[4] = {0xFF, 0xFF, 0xFF, 0xFF};
      double best = -1.0;
      for (int s = 0; s < d->weight_count[i]; ++s) {
        w[s] = d->weight[4 * i + s];
        lk[s] = static_cast<unsigned char>(d->weight_link[4 * i + s]);
        c->h_wgt[4 * i + s] = d->weight[4 * i + s];
        c->h_wlink[4 * i + s] = d->weight_link[4 * i + s];
        // dominant link (synth.cpp:211-225): max weight, ties to lower link
        const double e = d->weight[4 * i + s];
        const int link = d->weight_link[4 * i + s];
        int& dom = c->dominant[static_cast<size_t>(i)];
        if (e > best || (e == best && link < dom)) {
          best = e;
          dom = link;
        }
      }
      wg[i] = make_double4(w[0], w[1], w[2], w[3]);
      wl[i] = make_uchar4(lk[0], lk[1], lk[2], lk[3]);
    }
    // one-ring: incident triangles in CSR order, rotated so vertex i leads
    std::vector<int> ring_off(static_cast<size_t>(V) + 1);
    std::vector<int2> ring(static_cast<size_t>(d->vtri_offsets[V]));
    for (int i = 0; i < V; ++i) {
      ring_off[i] = d->vtri_offsets[i];
      for (int k = d->vtri_offsets[i]; k < d->vtri_offsets[i + 1]; ++k) {
        const int* t = d->triangles + 3 * d->vtri_items[k];
        // (b, c) follow i cyclically; bits 30-31 of .x carry i's position in
        // the triangle so the kernel rebuilds (f0, f1, f2) in stored order
        if (t[0] == i) ring[k] = make_int2(t[1], t[2]);
        else if (t[1] == i) ring[k] = make_int2(t[2] | (1 << 30), t[0]);
        else if (t[2] == i) ring[k] = make_int2(t[0] | (2 << 30), t[1]);
        else fail(WT_EINVAL, "vertex->triangle CSR lists a triangle that does not contain the vertex");
      }
    }
    ring_off[V] = d->vtri_offsets[V];
    c->h_tri.assign(d->triangles, d->triangles + 3 * c->T);
    // neighbours as ELL [K][V]
    int K = 0;
    for (int i = 0; i < V; ++i) K = std::max(K, d->nbr_offsets[i + 1] - d->nbr_offsets[i]);
    c->K = K;
    std::vector<int> nbr(static_cast<size_t>(std::max(1, K)) * std::max(1, V), -1);
    for (int i = 0; i < V; ++i)
      for (int k = 0; k < d->nbr_offsets[i + 1] - d->nbr_offsets[i]; ++k)
        nbr[static_cast<size_t>(k) * V + i] = d->nbr_items[d->nbr_offsets[i] + k];

    // device model
    double4* d_v0 = c->mem.alloc<double4>(V);
    double4* d_wg = c->mem.alloc<double4>(V);
    uchar4* d_wl = c->mem.alloc<uchar4>(V);
    int* d_roff = c->mem.alloc<int>(V + 1);
    int2* d_ring = c->mem.alloc<int2>(ring.size());
    // fan table of k_normals: for a closed, consistently wound fan of k <= 8
    // triangles, the ring neighbours n_0..n_{k-1} such that fan triangle j is
    // (i, n_j, n_j+1) (n_0 = b of CSR triangle 0), n_0 repeated in slot k; the
    // rot of each fan triangle and the fan position of each CSR triangle.
    // Anything else (open fans, > 8 triangles) falls back to the CSR.
    std::vector<int> fan_nb(static_cast<size_t>(V) * 8, -1);
    std::vector<unsigned long long> fan_code(static_cast<size_t>(V), 0ull);
    for (int i = 0; i < V; ++i) {
      const int k = ring_off[i + 1] - ring_off[i];
      int* nb = fan_nb.data() + static_cast<size_t>(i) * 8;
      const int2* rg = ring.data() + ring_off[i];
      bool ok = k >= 1 && k <= 8;
      int fan_of[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // CSR triangle -> fan position
      unsigned long long code = 0ull;
      if (ok) {
        int cur = 0;  // CSR index of fan triangle j
        bool used[8] = {false, false, false, false, false, false, false, false};
        for (int j = 0; j < k && ok; ++j) {
          used[cur] = true;
          fan_of[cur] = j;
          nb[j] = rg[cur].x & 0x3FFFFFFF;
          code |= static_cast<unsigned long long>(static_cast<unsigned>(rg[cur].x) >> 30) << (2 * j);
          if (j + 1 == k) {
            ok = rg[cur].y == nb[0];  // the fan closes
            break;
          }
          int nxt = -1;  // the triangle whose b is this one's c
          for (int t = 0; t < k; ++t)
            if (!used[t] && (rg[t].x & 0x3FFFFFFF) == rg[cur].y) {
              nxt = nxt < 0 ? t : -2;
            }
          ok = nxt >= 0;
          cur = nxt;
        }
      }
      if (ok) {
        for (int t = 0; t < k; ++t) code |= static_cast<unsigned long long>(fan_of[t]) << (16 + 3 * t);
        code |= static_cast<unsigned long long>(k) << 40;
        if (k < 8) nb[k] = nb[0];
      } else {
        std::fill(nb, nb + 8, -1);
        nb[0] = -2;
        code = 0ull;
      }
      fan_code[i] = code;
    }
    int* d_fan_nb = c->mem.alloc<int>(fan_nb.size());
    unsigned long long* d_fan_code = c->mem.alloc<unsigned long long>(fan_code.size());
    upload(d_fan_nb, fan_nb.data(), fan_nb.size(), c->stream);
    upload(d_fan_code, fan_code.data(), fan_code.size(), c->stream);
    int* d_nbr = c->mem.alloc<int>(nbr.size());
    wt::LinkDesc* d_links = c->mem.alloc<wt::LinkDesc>(L);
    int* d_poff = c->mem.alloc<int>(L + 1);
    int* d_pth = c->mem.alloc<int>(std::max(1, c->NP));
    int* d_plk = c->mem.alloc<int>(std::max(1, c->NP));
    int* d_pow = c->mem.alloc<int>(std::max(1, c->NP));
    std::vector<int> depth(static_cast<size_t>(L), 0);
    int max_depth = 0;
    for (int j = 0; j < L; ++j) {
      depth[j] = d->parent[j] < 0 ? 0 : depth[d->parent[j]] + 1;
      max_depth = std::max(max_depth, depth[j]);
    }
    int* d_depth = c->mem.alloc<int>(L);
    upload(d_depth, depth.data(), L, c->stream);
    double* d_s = c->mem.alloc<double>(L);
    // JtJ / Jtr entry table of the pose kernels: row-major upper triangle, then Jtr
    std::vector<unsigned> pose_e;
    for (int r = 0; r < L; ++r)
      for (int cc = r; cc < L; ++cc) pose_e.push_back(static_cast<unsigned>(r) | (static_cast<unsigned>(cc) << 16));
    for (int r = 0; r < L; ++r) pose_e.push_back(static_cast<unsigned>(r) | (static_cast<unsigned>(L) << 16));
    unsigned* d_pe = c->mem.alloc<unsigned>(pose_e.size());
    upload(d_pe, pose_e.data(), pose_e.size(), c->stream);
    upload(d_v0, v0.data(), V, c->stream);
    upload(d_wg, wg.data(), V, c->stream);
    upload(d_wl, wl.data(), V, c->stream);
    upload(d_roff, ring_off.data(), V + 1, c->stream);
    upload(d_ring, ring.data(), ring.size(), c->stream);
    upload(d_nbr, nbr.data(), nbr.size(), c->stream);
    upload(d_links, c->links.data(), L, c->stream);
    upload(d_poff, c->pair_off.data(), L + 1, c->stream);
    upload(d_pth, c->pair_theta.data(), c->NP, c->stream);
    upload(d_plk, c->pair_link.data(), c->NP, c->stream);
    upload(d_pow, c->pair_owner.data(), c->NP, c->stream);
    upload(d_s, c->s_diag.data(), L, c->stream);
    c->dm = wt::DevModel{V, L, c->NP, K, d_v0, d_wg, d_wl, d_roff, d_ring, d_fan_nb, d_fan_code, d_nbr,
                         d_links, d_poff, d_pth, d_plk, d_pow, d_s, d_depth, max_depth, d_pe};

    alloc_arenas(c);
    c->hs = c->ds;  // hooks share sequence 0's per-vertex buffers, own theta/fk/offsets/dchain
    alloc_hook_state(c, c->hs);
    c->phi_scratch = c->mem.alloc<double4>(V);
    for (int b = 0; b < c->nseq; ++b) upload(seq_at(c->phi[0], c, b), ph.data(), V, c->stream);
    if (getenv("WT_DEBUG_POSE")) c->pose_dbg = c->mem.alloc<long long>(8 + 8 * 296 + 8);
    if (wt::pose_smem_bytes(L, c->NP, pose_threads(c) / 32) > 227 * 1024)
      fail(WT_EINVAL, "skeleton too large for the pose kernel's shared memory");
    const int edge = wt::pose_tile_edge(L);
    if (edge == 3) {
      pose_attr<1, 3>(c);
    } else if (edge == 4) {
      pose_attr<1, 4>(c);
    } else {
      switch (pose_q(L)) {
        case 8: pose_attr<8, 0>(c); break;
        case 16: pose_attr<16, 0>(c); break;
        case 32: pose_attr<32, 0>(c); break;
        default: pose_attr<68, 0>(c); break;
      }
    }
    WT_CUDA(cudaStreamSynchronize(c->stream));
  });
  if (rc != WT_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return WT_OK;
}
}  // namespace

extern "C" {

int wt_gpu_create(int device, const wt_model_desc* d, const wt_intrinsics* intr, wt_gpu_ctx** out) {
  return create_ctx(device, d, intr, 1, out);
}

int wt_gpu_create_batch(int device, const wt_model_desc* d, const wt_intrinsics* intr, int32_t n_seq,
                        wt_gpu_ctx** out) {
  return create_ctx(device, d, intr, n_seq, out);
}

int32_t wt_gpu_batch_size(const wt_gpu_ctx* c) { return c ? c->nseq : 0; }

void wt_gpu_destroy(wt_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  delete ctx;
}

int wt_gpu_set_state(wt_gpu_ctx* c, const double* theta, const double* phi, int32_t frame_index) {
  if (!c) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    if (theta) {
      upload(c->ds.theta, theta, c->L, c->stream);
      c->fk_valid = false;
    }
    if (phi) phi_put(c, c->phi[c->cur], phi);
    c->frame_index = frame_index;
    WT_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int wt_gpu_get_state(wt_gpu_ctx* c, double* theta, double* phi, int32_t* frame_index) {
  if (!c) return WT_EINVAL;
  if (c->theta_mirror && !phi) {  // right after a tracked frame: theta came back with its stats
    if (theta) std::memcpy(theta, c->h_theta, sizeof(double) * c->L);
    if (frame_index) *frame_index = c->frame_index;
    return WT_OK;
  }
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    if (theta)
      WT_CUDA(cudaMemcpyAsync(theta, c->ds.theta, sizeof(double) * c->L, cudaMemcpyDeviceToHost, c->stream));
    if (phi) phi_get_async(c, c->phi[c->cur]);
    WT_CUDA(cudaStreamSynchronize(c->stream));
    if (phi) phi_unpack(c, phi);
    if (frame_index) *frame_index = c->frame_index;
  });
}

static void ingest(wt_gpu_ctx* c, const float* depth_dev, double scale, const double* cloud_dev,
                   const uint8_t* valid_dev, cudaStream_t st = nullptr) {
  // batch: depth_dev / cloud_dev / valid_dev are the arena buffers (same stride)
  if (!st) st = c->stream;
  if (c->nseq == 1) WT_CUDA(cudaMemsetAsync(c->d_nvalid, 0, 4 * sizeof(int), st));
  else WT_CUDA(cudaMemset2DAsync(c->d_nvalid, static_cast<size_t>(c->bstride), 0, 4 * sizeof(int), c->nseq, st));
  const int segs = (c->din.W + wt::kIngestSeg - 1) / wt::kIngestSeg;
  (c->nseq > 1 ? wt::k_ingest<true> : wt::k_ingest<false>)<<<dim3(segs * c->din.H, c->nseq), wt::kIngestSeg, 0, st>>>(
      c->din, depth_dev, scale, cloud_dev, valid_dev, c->d_valid, c->d_pts_hi, c->d_vpts, c->d_nvalid, c->bstride);
  check_launch();
}

namespace {
void track_frame_overlapped(wt_gpu_ctx* c, const float* depth, double scale, const wt_track_config* cfg,
                            bool shape_now, bool device_frame = false);
}  // namespace

// the pending device frame (wt_gpu_load_depth), for a consumer that is not a
// track call
static void flush_pending(wt_gpu_ctx* c) {
  if (!c->pending_depth) return;
  const float* d = c->pending_depth;
  c->pending_depth = nullptr;
  ingest(c, d, c->pending_scale, nullptr, nullptr);
}

// device memory of this context's GPU (a frame the ingest may read in place)
bool on_device(const wt_gpu_ctx* c, const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice && at.device == c->device;
}

int wt_gpu_load_depth(wt_gpu_ctx* c, const float* depth, double depth_scale) {
  if (!c || !depth) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    c->pending_depth = nullptr;
    if (on_device(c, depth) && c->nseq == 1 && !getenv("WT_NO_H2D_OVERLAP")) {
      c->pending_depth = depth;  // ingested by the next track call's graph, or by require_frame
      c->pending_scale = depth_scale;
    } else if (on_device(c, depth)) {
      ingest(c, depth, depth_scale, nullptr, nullptr);  // read in place: the ingest is its only reader
    } else {
      WT_CUDA(cudaMemcpyAsync(c->d_depth, depth, sizeof(float) * c->P, cudaMemcpyDefault, c->stream));
      ingest(c, c->d_depth, depth_scale, nullptr, nullptr);
    }
    c->frame_loaded = true;
    c->frame_on_rays = true;
  });
}

int wt_gpu_load_cloud(wt_gpu_ctx* c, const double* points, const uint8_t* valid) {
  if (!c || !points || !valid) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    c->pending_depth = nullptr;
    WT_CUDA(cudaMemcpyAsync(c->d_pts_hi, points, sizeof(double) * 3 * c->P, cudaMemcpyDefault, c->stream));
    WT_CUDA(cudaMemcpyAsync(c->d_valid, valid, c->P, cudaMemcpyDefault, c->stream));
    ingest(c, nullptr, 1.0, c->d_pts_hi, c->d_valid);
    c->frame_loaded = true;
    c->frame_on_rays = false;
  });
}

int wt_gpu_track_loaded(wt_gpu_ctx* c, const wt_track_config* cfg, wt_frame_stats* stats) {
  if (!c || !cfg) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    require_frame(c);
    check_assoc(&cfg->assoc);
    if (cfg->kin.iterations < 0 || cfg->shape.iterations < 0) fail(WT_EINVAL, "negative iteration count");
    const bool shape_now = cfg->mode == WT_MODE_DYNAMIC ||
                           (cfg->mode == WT_MODE_SHAPE_MATCH && c->frame_index == 0);
    ensure_stats(c, cfg->kin.iterations, cfg->shape.iterations);
    const int start = c->cur;
    GraphKey key{{1.0, static_cast<double>(cfg->kin.iterations), static_cast<double>(cfg->kin.assoc_refresh),
                  cfg->kin.lambda_k, cfg->kin.lambda_s, cfg->kin.diag_floor,
                  static_cast<double>(cfg->kin.clamp_limits), cfg->kin.limit,
                  static_cast<double>(cfg->assoc.window_radius), cfg->assoc.cutoff,
                  shape_now ? 1.0 : 0.0, static_cast<double>(cfg->shape.iterations),
                  cfg->shape.lambda_phi, cfg->shape.lambda_nbr, cfg->shape.lambda_w,
                  cfg->shape.diag_floor, static_cast<double>(cfg->shape_stats), static_cast<double>(start),
                  c->fk_valid ? 0.0 : 1.0}};
    const bool need_fk = !c->fk_valid;
    if (c->pending_depth) {  // the frame's copy + ingest on a branch of the frame graph
      const float* d = c->pending_depth;
      c->pending_depth = nullptr;
      track_frame_overlapped(c, d, c->pending_scale, cfg, shape_now, true);
    } else {
      run_graph(c, key, [&] {
        enq_optimize_pose(c, &cfg->kin, &cfg->assoc, need_fk);
        if (shape_now) enq_optimize_shape(c, start, &cfg->shape, &cfg->assoc, cfg->shape_stats != 0, false);
      });
    }
    c->fk_valid = true;
    c->cur = (shape_now && (cfg->shape.iterations % 2)) ? start ^ 1 : start;
    frame_readback(c, cfg->kin.iterations, shape_now ? cfg->shape.iterations : 0, stats);
  });
}

namespace {
GraphKey track_key(const wt_gpu_ctx* c, const wt_track_config* cfg, bool shape_now, double tag) {
  return GraphKey{{tag, static_cast<double>(cfg->kin.iterations), static_cast<double>(cfg->kin.assoc_refresh),
                   cfg->kin.lambda_k, cfg->kin.lambda_s, cfg->kin.diag_floor,
                   static_cast<double>(cfg->kin.clamp_limits), cfg->kin.limit,
                   static_cast<double>(cfg->assoc.window_radius), cfg->assoc.cutoff, shape_now ? 1.0 : 0.0,
                   static_cast<double>(cfg->shape.iterations), cfg->shape.lambda_phi, cfg->shape.lambda_nbr,
                   cfg->shape.lambda_w, cfg->shape.diag_floor, static_cast<double>(cfg->shape_stats),
                   static_cast<double>(c->cur), c->fk_valid ? 0.0 : 1.0}};
}

// one frame; FK of the current theta is recomputed first unless still valid
void enq_track(wt_gpu_ctx* c, const wt_track_config* cfg, bool shape_now) {
  enq_optimize_pose(c, &cfg->kin, &cfg->assoc, !c->fk_valid);
  if (shape_now) enq_optimize_shape(c, c->cur, &cfg->shape, &cfg->assoc, cfg->shape_stats != 0, false);
}
}  // namespace

void* wt_gpu_stream(wt_gpu_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

// Debug: last pose kernel's last-CTA timing (needs WT_DEBUG_POSE at create).
int wt_gpu_debug_pose(wt_gpu_ctx* c, long long* out) {
  if (!c || !c->pose_dbg) return 0;
  cudaMemcpy(out, c->pose_dbg, sizeof(long long) * (8 + 8 * 296), cudaMemcpyDeviceToHost);
  return 5;
}

int wt_gpu_host_alloc(size_t bytes, void** out) {
  if (!out) return WT_EINVAL;
  *out = nullptr;
  return guarded(nullptr, [&] {
    const cudaError_t e = cudaMallocHost(out, std::max<size_t>(bytes, 1));
    if (e != cudaSuccess) throw CudaError{WT_ENOMEM, std::string("cudaMallocHost: ") + cudaGetErrorString(e)};
  });
}

void wt_gpu_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int wt_gpu_bucket_count(wt_gpu_ctx* c, int32_t seq, int32_t* n_bucketed) {
  if (!c || !n_bucketed) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    if (seq < 0 || seq >= c->nseq) fail(WT_EINVAL, "sequence index out of range");
    WT_CUDA(cudaMemcpyAsync(n_bucketed, seq_at(c->ds.poff, c, seq) + c->P, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
  }, true);
}

int wt_gpu_sync(wt_gpu_ctx* c) {
  if (!c) return WT_EINVAL;
  return guarded(c, [&] { WT_CUDA(cudaStreamSynchronize(c->stream)); });
}

int wt_gpu_track_async(wt_gpu_ctx* c, const wt_track_config* cfg) {
  if (!c || !cfg) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    require_frame(c);
    check_assoc(&cfg->assoc);
    const bool shape_now = cfg->mode == WT_MODE_DYNAMIC ||
                           (cfg->mode == WT_MODE_SHAPE_MATCH && c->frame_index == 0);
    ensure_stats(c, cfg->kin.iterations, cfg->shape.iterations);
    const int start = c->cur;
    if (c->pending_depth) {  // the frame's copy + ingest on a branch of the frame graph
      const float* d = c->pending_depth;
      c->pending_depth = nullptr;
      track_frame_overlapped(c, d, c->pending_scale, cfg, shape_now, true);
    } else {
      run_graph(c, track_key(c, cfg, shape_now, 1.0), [&] { enq_track(c, cfg, shape_now); });
    }
    c->fk_valid = true;
    c->cur = (shape_now && (cfg->shape.iterations % 2)) ? start ^ 1 : start;
    ++c->frame_index;
  });
}

int wt_gpu_profile_frame(wt_gpu_ctx* c, const wt_track_config* cfg, int32_t* kinds, float* ms, int32_t cap,
                         int32_t* n_out) {
  if (!c || !cfg) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_frame(c);
    flush_pending(c);
    check_assoc(&cfg->assoc);
    const bool shape_now = cfg->mode == WT_MODE_DYNAMIC ||
                           (cfg->mode == WT_MODE_SHAPE_MATCH && c->frame_index == 0);
    ensure_stats(c, cfg->kin.iterations, cfg->shape.iterations);
    for (cudaEvent_t e : c->prof_events) cudaEventDestroy(e);
    c->prof_events.clear();
    c->prof_kind.clear();
    const int start = c->cur;
    cudaEvent_t e0;
    WT_CUDA(cudaEventCreate(&e0));
    cudaGraph_t g;
    c->prof_on = true;
    WT_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      WT_CUDA(cudaEventRecordWithFlags(e0, c->stream, cudaEventRecordExternal));
      enq_track(c, cfg, shape_now);
    } catch (...) {
      c->prof_on = false;
      cudaStreamEndCapture(c->stream, &g);
      throw;
    }
    c->prof_on = false;
    WT_CUDA(cudaStreamEndCapture(c->stream, &g));
    cudaGraphExec_t ex;
    WT_CUDA(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    WT_CUDA(cudaGraphLaunch(ex, c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
    cudaGraphExecDestroy(ex);
    c->fk_valid = true;
    c->cur = (shape_now && (cfg->shape.iterations % 2)) ? start ^ 1 : start;
    ++c->frame_index;
    const int n = static_cast<int>(c->prof_events.size());
    cudaEvent_t prev = e0;
    for (int k = 0; k < n && k < cap; ++k) {
      float t = 0.0f;
      WT_CUDA(cudaEventElapsedTime(&t, prev, c->prof_events[k]));
      if (ms) ms[k] = t;
      if (kinds) kinds[k] = c->prof_kind[k];
      prev = c->prof_events[k];
    }
    cudaEventDestroy(e0);
    if (n_out) *n_out = n;
  });
}

namespace {
void ensure_seq(wt_gpu_ctx* c, int frames) {
  if (!c->copy_stream) {
    WT_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      WT_CUDA(cudaMallocHost(&c->seq_pinned[b], sizeof(float) * c->P));
      c->seq_depth[b] = c->mem.alloc<float>(c->P);
      WT_CUDA(cudaEventCreateWithFlags(&c->seq_h2d[b], cudaEventDisableTiming));
      WT_CUDA(cudaEventCreateWithFlags(&c->seq_ingest[b], cudaEventDisableTiming));
    }
  }
  if (frames > c->cap_rec) {
    c->cap_rec = std::max(frames, 64);
    c->rec_buf = c->mem.alloc<double>(static_cast<size_t>(c->cap_rec) * c->L * 4);
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
}  // namespace

int wt_gpu_track_sequence(wt_gpu_ctx* c, const float* frames, int32_t n_frames, double depth_scale,
                          const wt_track_config* cfg, double* theta_out, double* joints_out) {
  if (!c || !cfg || (n_frames > 0 && !frames) || n_frames < 0) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    check_assoc(&cfg->assoc);
    if (cfg->kin.iterations < 0 || cfg->shape.iterations < 0) fail(WT_EINVAL, "negative iteration count");
    if (n_frames == 0) return;
    ensure_stats(c, cfg->kin.iterations, cfg->shape.iterations);
    ensure_seq(c, n_frames);
    const bool on_device = is_device_ptr(frames);
    const size_t P = static_cast<size_t>(c->P);
    const int L = c->L;
    double* rec_theta = c->rec_buf;
    double* rec_joints = c->rec_buf + static_cast<size_t>(c->cap_rec) * L;
    for (int f = 0; f < n_frames; ++f) {
      const float* src = frames + static_cast<size_t>(f) * P;
      const float* dev_depth = src;
      const int b = f & 1;
      if (!on_device) {
        // the pinned slot is free once its previous upload (frame f-2) landed
        WT_CUDA(cudaEventSynchronize(c->seq_h2d[b]));
        std::memcpy(c->seq_pinned[b], src, sizeof(float) * P);
        // the device slot is free once frame f-2's ingest has read it
        WT_CUDA(cudaStreamWaitEvent(c->copy_stream, c->seq_ingest[b], 0));
        WT_CUDA(cudaMemcpyAsync(c->seq_depth[b], c->seq_pinned[b], sizeof(float) * P, cudaMemcpyHostToDevice,
                                c->copy_stream));
        WT_CUDA(cudaEventRecord(c->seq_h2d[b], c->copy_stream));
        WT_CUDA(cudaStreamWaitEvent(c->stream, c->seq_h2d[b], 0));
        dev_depth = c->seq_depth[b];
      }
      ingest(c, dev_depth, depth_scale, nullptr, nullptr);
      if (!on_device) WT_CUDA(cudaEventRecord(c->seq_ingest[b], c->stream));
      c->frame_loaded = true;
      c->frame_on_rays = true;
      const bool shape_now = cfg->mode == WT_MODE_DYNAMIC ||
                             (cfg->mode == WT_MODE_SHAPE_MATCH && c->frame_index == 0);
      const int start = c->cur;
      run_graph(c, track_key(c, cfg, shape_now, 1.0), [&] { enq_track(c, cfg, shape_now); });
      c->fk_valid = true;
      c->cur = (shape_now && (cfg->shape.iterations % 2)) ? start ^ 1 : start;
      ++c->frame_index;
      wt::k_record<<<1, 64, 0, c->stream>>>(c->dm, c->ds, rec_theta + static_cast<size_t>(f) * L,
                                            rec_joints + static_cast<size_t>(f) * L * 3);
      check_launch();
    }
    if (theta_out)
      WT_CUDA(cudaMemcpyAsync(theta_out, rec_theta, sizeof(double) * n_frames * L, cudaMemcpyDeviceToHost,
                              c->stream));
    if (joints_out)
      WT_CUDA(cudaMemcpyAsync(joints_out, rec_joints, sizeof(double) * n_frames * L * 3,
                              cudaMemcpyDeviceToHost, c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int wt_gpu_joint_positions(wt_gpu_ctx* c, double* joints_out) {
  if (!c || !joints_out) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    ensure_seq(c, 1);
    // FK of the current theta into the hook state, then the origins
    WT_CUDA(cudaMemcpyAsync(c->hs.theta, c->ds.theta, sizeof(double) * c->L, cudaMemcpyDeviceToDevice, c->stream));
    wt::launch_fk(c->stream, 1, c->dm, c->hs);
    wt::k_record<<<1, 64, 0, c->stream>>>(c->dm, c->hs, nullptr, c->rec_buf);
    check_launch();
    WT_CUDA(cudaMemcpyAsync(joints_out, c->rec_buf, sizeof(double) * c->L * 3, cudaMemcpyDeviceToHost,
                            c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
  });
}

namespace {
bool pinned_host(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// One frame from a pinned host depth image: the frame graph forks the upload
// and ingest onto copy_stream at its start and joins them before the first
// search; only the search and what follows need the frame.
void track_frame_overlapped(wt_gpu_ctx* c, const float* depth, double scale, const wt_track_config* cfg,
                            bool shape_now, bool device_frame) {
  if (!c->up_stream) WT_CUDA(cudaStreamCreateWithFlags(&c->up_stream, cudaStreamNonBlocking));
  if (!c->fork_ev) WT_CUDA(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
  if (!c->join_ev) WT_CUDA(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
  GraphKey key = track_key(c, cfg, shape_now, 4.0);
  key.v.push_back(scale);
  key.v.push_back(device_frame ? 1.0 : 0.0);  // the upload node copies from host or device memory
  const size_t bytes = sizeof(float) * c->P;
  auto it = c->h2d_graphs.find(key);
  if (it == c->h2d_graphs.end()) {
    cudaGraph_t g;
    WT_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      WT_CUDA(cudaEventRecord(c->fork_ev, c->stream));
      WT_CUDA(cudaStreamWaitEvent(c->up_stream, c->fork_ev, 0));
      for (int b = 0; b < c->nseq; ++b)  // one 1D upload per sequence (re-pointable per launch)
        WT_CUDA(cudaMemcpyAsync(seq_at(c->d_depth, c, b), depth + static_cast<size_t>(b) * c->P, bytes,
                                cudaMemcpyDefault, c->up_stream));  // pinned host or device frames
      ingest(c, c->d_depth, scale, nullptr, nullptr, c->up_stream);
      WT_CUDA(cudaEventRecord(c->join_ev, c->up_stream));
      c->before_search = [c] { WT_CUDA(cudaStreamWaitEvent(c->stream, c->join_ev, 0)); };
      enq_track(c, cfg, shape_now);
      if (c->before_search) {  // no search in this frame: join at the end
        c->before_search = nullptr;
        WT_CUDA(cudaStreamWaitEvent(c->stream, c->join_ev, 0));
      }
    } catch (...) {
      c->before_search = nullptr;
      cudaStreamEndCapture(c->stream, &g);
      throw;
    }
    WT_CUDA(cudaStreamEndCapture(c->stream, &g));
    size_t n = 0;
    WT_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    WT_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
    std::vector<cudaGraphNode_t> cp(static_cast<size_t>(c->nseq), nullptr);
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      WT_CUDA(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeMemcpy) continue;
      cudaMemcpy3DParms prm{};
      WT_CUDA(cudaGraphMemcpyNodeGetParams(nd, &prm));
      const long long off = static_cast<const char*>(prm.dstPtr.ptr) - reinterpret_cast<const char*>(c->d_depth);
      const long long b = c->nseq > 1 ? off / c->bstride : 0;
      if (b >= 0 && b < c->nseq) cp[static_cast<size_t>(b)] = nd;
    }
    for (cudaGraphNode_t nd : cp)
      if (!nd) fail(WT_ECUDA, "frame graph: upload node not found");
    cudaGraphExec_t ex;
    WT_CUDA(cudaGraphInstantiate(&ex, g, 0));
    it = c->h2d_graphs.emplace(key, wt_gpu_ctx::H2DGraph{g, ex, cp}).first;
  } else {  // re-point the uploads at this call's host frames
    for (int b = 0; b < c->nseq; ++b)
      WT_CUDA(cudaGraphExecMemcpyNodeSetParams1D(it->second.exec, it->second.copy[static_cast<size_t>(b)],
                                                 seq_at(c->d_depth, c, b), depth + static_cast<size_t>(b) * c->P,
                                                 bytes, cudaMemcpyDefault));
  }
  WT_CUDA(cudaGraphLaunch(it->second.exec, c->stream));
}
}  // namespace

int wt_gpu_track_frame(wt_gpu_ctx* c, const float* depth, double depth_scale,
                       const wt_track_config* cfg, wt_frame_stats* stats) {
  if (!c || !depth || !cfg) return WT_EINVAL;
  if (c->nseq != 1 || getenv("WT_NO_H2D_OVERLAP") || !pinned_host(depth)) {
    const int rc = wt_gpu_load_depth(c, depth, depth_scale);
    if (rc != WT_OK) return rc;
    return wt_gpu_track_loaded(c, cfg, stats);
  }
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    check_assoc(&cfg->assoc);
    if (cfg->kin.iterations < 0 || cfg->shape.iterations < 0) fail(WT_EINVAL, "negative iteration count");
    const bool shape_now = cfg->mode == WT_MODE_DYNAMIC ||
                           (cfg->mode == WT_MODE_SHAPE_MATCH && c->frame_index == 0);
    ensure_stats(c, cfg->kin.iterations, cfg->shape.iterations);
    const int start = c->cur;
    c->frame_loaded = true;
    c->frame_on_rays = true;
    track_frame_overlapped(c, depth, depth_scale, cfg, shape_now);
    c->fk_valid = true;
    c->cur = (shape_now && (cfg->shape.iterations % 2)) ? start ^ 1 : start;
    frame_readback(c, cfg->kin.iterations, shape_now ? cfg->shape.iterations : 0, stats);
  });
}

int wt_gpu_track_frame_cloud(wt_gpu_ctx* c, const double* points, const uint8_t* valid,
                             const wt_track_config* cfg, wt_frame_stats* stats) {
  const int rc = wt_gpu_load_cloud(c, points, valid);
  if (rc != WT_OK) return rc;
  return wt_gpu_track_loaded(c, cfg, stats);
}

int wt_gpu_optimize_pose(wt_gpu_ctx* c, const wt_kin_config* kin, const wt_assoc_config* assoc,
                         wt_kin_iter_stats* stats, int32_t cap, int32_t* n_out) {
  if (!c || !kin) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    require_frame(c);
    flush_pending(c);
    check_assoc(assoc);
    if (kin->iterations < 0) fail(WT_EINVAL, "negative iteration count");
    ensure_stats(c, kin->iterations, 0);
    GraphKey key{{2.0, static_cast<double>(kin->iterations), static_cast<double>(kin->assoc_refresh),
                  kin->lambda_k, kin->lambda_s, kin->diag_floor, static_cast<double>(kin->clamp_limits),
                  kin->limit, static_cast<double>(assoc->window_radius), assoc->cutoff,
                  static_cast<double>(c->cur), c->fk_valid ? 0.0 : 1.0}};
    const bool need_fk = !c->fk_valid;
    run_graph(c, key, [&] { enq_optimize_pose(c, kin, assoc, need_fk); });
    c->fk_valid = true;
    const int nk = kin->iterations;
    if (nk) WT_CUDA(cudaMemcpyAsync(c->h_kin, c->ds.kin_stats, sizeof(wt::KinStat) * nk,
                                    cudaMemcpyDeviceToHost, c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
    if (stats) put_kin(c, nk, stats, cap);
    if (n_out) *n_out = nk;
    check_range(c, nk);
  });
}

int wt_gpu_optimize_shape(wt_gpu_ctx* c, const wt_shape_config* shape, const wt_assoc_config* assoc,
                          int32_t with_stats_pass, wt_shape_iter_stats* stats, int32_t cap,
                          int32_t* n_out) {
  if (!c || !shape) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    require_frame(c);
    flush_pending(c);
    check_assoc(assoc);
    if (shape->iterations < 0) fail(WT_EINVAL, "negative iteration count");
    ensure_stats(c, 0, shape->iterations);
    const int start = c->cur;
    GraphKey key{{3.0, static_cast<double>(shape->iterations), shape->lambda_phi, shape->lambda_nbr,
                  shape->lambda_w, shape->diag_floor, static_cast<double>(assoc->window_radius),
                  assoc->cutoff, static_cast<double>(with_stats_pass), static_cast<double>(start),
                  c->fk_valid ? 0.0 : 1.0}};
    const bool need_fk = !c->fk_valid;
    run_graph(c, key, [&] { enq_optimize_shape(c, start, shape, assoc, with_stats_pass != 0, need_fk); });
    c->fk_valid = true;
    c->cur = (shape->iterations % 2) ? start ^ 1 : start;
    const int ns = shape->iterations;
    if (ns) WT_CUDA(cudaMemcpyAsync(c->h_shape, c->ds.shape_stats, sizeof(wt::ShapeStat) * ns,
                                    cudaMemcpyDeviceToHost, c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
    if (stats) put_shape(c, ns, stats, cap);
    if (n_out) *n_out = ns;
  });
}

// ---- stage hooks -----------------------------------------------------------------

int wt_gpu_skin(wt_gpu_ctx* c, const double* theta, const double* phi, double* v, double* n,
                uint8_t* valid) {
  if (!c || !theta) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    upload(c->hs.theta, theta, c->L, c->stream);
    const double4* ph = c->phi[c->cur];
    if (phi) {
      std::vector<double4> tmp(static_cast<size_t>(c->V));
      for (int i = 0; i < c->V; ++i) tmp[i] = make_double4(phi[3 * i], phi[3 * i + 1], phi[3 * i + 2], 0.0);
      upload(c->phi_scratch, tmp.data(), c->V, c->stream);
      WT_CUDA(cudaStreamSynchronize(c->stream));
      ph = c->phi_scratch;
    }
    enq_fk(c, c->hs);
    enq_skin(c, c->hs, ph);
    enq_normals(c, c->hs, false, false);
    std::vector<double4> pv(static_cast<size_t>(c->V));
    std::vector<float4> pn(static_cast<size_t>(c->V));
    WT_CUDA(cudaMemcpyAsync(pv.data(), c->hs.pv, sizeof(double4) * c->V, cudaMemcpyDeviceToHost, c->stream));
    WT_CUDA(cudaMemcpyAsync(pn.data(), c->hs.pn, sizeof(float4) * c->V, cudaMemcpyDeviceToHost, c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < c->V; ++i) {
      if (v) {
        v[3 * i] = pv[i].x;
        v[3 * i + 1] = pv[i].y;
        v[3 * i + 2] = pv[i].z;
      }
      if (n) {
        n[3 * i] = pn[i].x;
        n[3 * i + 1] = pn[i].y;
        n[3 * i + 2] = pn[i].z;
      }
      if (valid) valid[i] = pn[i].w != 0.0f ? 1 : 0;
    }
  });
}

// reconstruction_error_frame (metrics.cpp:110-142) of the current state
// against the loaded frame: dist[V], NaN for vertices that are not visible.
int wt_gpu_recon_error(wt_gpu_ctx* c, double* dist, int32_t* n_visible) {
  if (!c || !dist) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    require_frame(c);
    flush_pending(c);
    ensure_render(c);
    if (!c->rc_obs) {
      c->rc_obs = c->mem.alloc<double>(3 * static_cast<size_t>(c->P));
      c->rc_vis = c->mem.alloc<int>(c->V);
      c->rc_cnt = c->mem.alloc<int>(2);
      c->rc_dist = c->mem.alloc<double>(c->V);
    }
    enq_fk(c, c->ds);
    c->fk_valid = true;
    enq_skin(c, c->ds, c->phi[c->cur]);
    wt::recon_launch(c->stream, c->dm, c->ds, c->din, c->T, c->r_tri, c->r_vpos, c->r_zbits, c->r_owner, c->d_valid,
                     c->d_pts_hi, c->rc_obs, c->rc_obs + c->P, c->rc_obs + 2 * static_cast<size_t>(c->P), c->rc_vis,
                     c->rc_cnt, c->rc_dist);
    check_launch();
    WT_CUDA(cudaMemcpyAsync(dist, c->rc_dist, sizeof(double) * c->V, cudaMemcpyDeviceToHost, c->stream));
    int cnt[2] = {0, 0};
    WT_CUDA(cudaMemcpyAsync(cnt, c->rc_cnt, sizeof(int) * 2, cudaMemcpyDeviceToHost, c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
    if (n_visible) *n_visible = cnt[0];
  });
}

}  // extern "C"

namespace {

// Downloads an association (accumulators + posed mesh) and forms p~, count
// and r = n.(p~ - v) exactly as the device kernels do.
void read_association(cudaStream_t st, int V, const wt::DevState& s, double* p_tilde, int32_t* count,
                      double* residual) {
  std::vector<unsigned long long> acc(4 * static_cast<size_t>(V));
  std::vector<double4> pv(static_cast<size_t>(V));
  std::vector<float4> pn(static_cast<size_t>(V));
  long long max_abs = 0;  // bits of the frame's largest coordinate magnitude (k_ingest): the sums' scale
  WT_CUDA(cudaMemcpyAsync(&max_abs, s.fwords + 2, sizeof(long long), cudaMemcpyDeviceToHost, st));
  WT_CUDA(cudaMemcpyAsync(acc.data(), s.acc, sizeof(unsigned long long) * 4 * V, cudaMemcpyDeviceToHost, st));
  WT_CUDA(cudaMemcpyAsync(pv.data(), s.pv, sizeof(double4) * V, cudaMemcpyDeviceToHost, st));
  WT_CUDA(cudaMemcpyAsync(pn.data(), s.pn, sizeof(float4) * V, cudaMemcpyDeviceToHost, st));
  WT_CUDA(cudaStreamSynchronize(st));
  const double oscale = wt::obs_scale_of_bits(max_abs);
  for (int i = 0; i < V; ++i) {
    const long long cnt = static_cast<long long>(acc[4 * i + 3]);
    double pt[3] = {0, 0, 0}, r = 0.0;
    if (cnt > 0) {
      const double inv = 1.0 / static_cast<double>(cnt);
      for (int k = 0; k < 3; ++k)
        pt[k] = static_cast<double>(static_cast<long long>(acc[4 * i + k])) / oscale * inv;
      r = static_cast<double>(pn[i].x) * (pt[0] - pv[i].x) + static_cast<double>(pn[i].y) * (pt[1] - pv[i].y) +
          static_cast<double>(pn[i].z) * (pt[2] - pv[i].z);
    }
    if (p_tilde)
      for (int k = 0; k < 3; ++k) p_tilde[3 * i + k] = pt[k];
    if (count) count[i] = static_cast<int32_t>(cnt);
    if (residual) residual[i] = r;
  }
}

}  // namespace

extern "C" {

int wt_gpu_associate(wt_gpu_ctx* c, int32_t window_radius, double cutoff, int32_t* winners,
                     double* p_tilde, int32_t* count, double* residual) {
  if (!c) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    require_frame(c);
    flush_pending(c);
    wt_assoc_config a{window_radius, 0, cutoff};
    check_assoc(&a);
    if (winners) WT_CUDA(cudaMemsetAsync(c->d_winners, 0xFF, sizeof(int) * c->P, c->stream));
    enq_associate(c, c->hs, &a, winners ? c->d_winners : nullptr, /*zero_acc=*/true);
    if (winners)
      WT_CUDA(cudaMemcpyAsync(winners, c->d_winners, sizeof(int) * c->P, cudaMemcpyDeviceToHost, c->stream));
    read_association(c->stream, c->V, c->hs, p_tilde, count, residual);
    // leave the sums clean for the frame graphs (their consumers clean up)
    WT_CUDA(cudaMemsetAsync(c->hs.acc, 0, sizeof(unsigned long long) * 4 * std::max(1, c->V), c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int wt_gpu_associate_posed(int device, const wt_intrinsics* intr, int32_t nv, const double* v,
                           const double* n, const uint8_t* valid, const double* points,
                           const uint8_t* point_valid, int32_t window_radius, double cutoff,
                           int32_t* winners, double* p_tilde, int32_t* count, double* residual) {
  // A throwaway context with a link-free "loose vertex" model: normals are
  // taken as given (the reference tests' PosedMesh), so only the bucket /
  // search / average kernels run.
  wt_gpu_ctx* c = nullptr;
  const int rc = guarded(nullptr, [&] {
    if (!intr || nv < 0 || !v || !n || !valid || !points || !point_valid) fail(WT_EINVAL, "NULL argument");
    const int par[1] = {-1};
    const double off[8] = {1, 0, 0, 0, 0, 0, 0, 0};
    const int kind[1] = {WT_JOINT_HINGE};
    const double axis[3] = {0, 0, 1};
    const int tix[1] = {0};
    std::vector<double> v0(v, v + 3 * nv);
    std::vector<int> wc(static_cast<size_t>(nv), 0), wlk(4 * static_cast<size_t>(nv), -1);
    std::vector<double> w(4 * static_cast<size_t>(nv), 0.0);
    std::vector<int> zero_off(static_cast<size_t>(nv) + 1, 0);
    wt_model_desc d{};
    d.n_links = 1;
    d.n_vertices = nv;
    d.n_triangles = 0;
    d.parent = par;
    d.parent_offset = off;
    d.joint_kind = kind;
    d.joint_axis = axis;
    d.theta_index = tix;
    d.v0 = v0.data();
    d.phi = nullptr;
    d.weight_count = wc.data();
    d.weight_link = wlk.data();
    d.weight = w.data();
    d.triangles = nullptr;
    d.vtri_offsets = zero_off.data();
    d.vtri_items = nullptr;
    d.nbr_offsets = zero_off.data();
    d.nbr_items = nullptr;
    const int r = wt_gpu_create(device, &d, intr, &c);
    if (r != WT_OK) fail(r, g_err);
    std::vector<double4> pv(static_cast<size_t>(nv));
    std::vector<float4> pn(static_cast<size_t>(nv));
    for (int i = 0; i < nv; ++i) {
      pv[i] = make_double4(v[3 * i], v[3 * i + 1], v[3 * i + 2], 1.0);
      pn[i] = make_float4(static_cast<float>(n[3 * i]), static_cast<float>(n[3 * i + 1]),
                          static_cast<float>(n[3 * i + 2]), valid[i] ? 1.0f : 0.0f);
    }
    upload(c->ds.pv, pv.data(), nv, c->stream);
    upload(c->ds.pn, pn.data(), nv, c->stream);
    if (wt_gpu_load_cloud(c, points, point_valid) != WT_OK) fail(WT_ECUDA, c->err);
    wt_assoc_config a{window_radius, 0, cutoff};
    check_assoc(&a);
    if (winners) WT_CUDA(cudaMemsetAsync(c->d_winners, 0xFF, sizeof(int) * c->P, c->stream));
    enq_normals(c, c->ds, true, true, /*compute=*/false);  // bucket with the given normals
    enq_scatter(c, c->ds);
    enq_search(c, c->ds, &a, winners ? c->d_winners : nullptr);
    if (winners)
      WT_CUDA(cudaMemcpyAsync(winners, c->d_winners, sizeof(int) * c->P, cudaMemcpyDeviceToHost, c->stream));
    read_association(c->stream, nv, c->ds, p_tilde, count, residual);
  });
  if (c) wt_gpu_destroy(c);
  return rc;
}

int wt_gpu_normal_system(wt_gpu_ctx* c, const double* theta, const wt_kin_config* kin,
                         const int32_t* count, const double* residual, double* jtj, double* jtr) {
  if (!c || !theta || !kin || !count || !residual) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_single(c);
    const int V = c->V, L = c->L;
    if (!c->hook_cnt) {
      c->hook_cnt = c->mem.alloc<int>(V);
      c->hook_res = c->mem.alloc<double>(V);
    }
    int* d_cnt = c->hook_cnt;
    double* d_res = c->hook_res;
    upload(d_cnt, count, V, c->stream);
    upload(d_res, residual, V, c->stream);
    upload(c->hs.theta, theta, L, c->stream);
    enq_fk(c, c->hs);
    enq_skin(c, c->hs, c->phi[c->cur]);
    enq_normals(c, c->hs, false, false);
    double rmax = 0.0;  // the given residuals bound |r| (the role of the cutoff)
    for (int i = 0; i < V; ++i)
      if (count[i] > 0) rmax = std::max(rmax, std::fabs(residual[i]));
    enq_pose(c, c->hs, c->phi[c->cur], kin, 0, false, d_cnt, d_res, rmax);
    std::vector<double> out(static_cast<size_t>(L * L + L));
    WT_CUDA(cudaMemcpyAsync(out.data(), c->hs.sys_out, sizeof(double) * out.size(), cudaMemcpyDeviceToHost,
                            c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
    std::copy(out.begin(), out.begin() + L * L, jtj);
    std::copy(out.begin() + L * L, out.end(), jtr);
  });
}

int wt_gpu_solve_step(int device, int32_t n, const double* jtj, const double* jtr, double lambda_k,
                      double diag_floor, double* x) {
  int status = WT_OK;
  const int rc = guarded(nullptr, [&] {
    if (n <= 0 || n > 64 || !jtj || !jtr || !x) fail(WT_EINVAL, "solve_step: bad arguments (n in 1..64)");
    WT_CUDA(cudaSetDevice(device));
    double* d = dalloc<double>(n * n + n + n + 1);
    std::vector<double> out(static_cast<size_t>(n) + 1);
    cudaError_t e = cudaMemcpy(d, jtj, sizeof(double) * n * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + n * n, jtr, sizeof(double) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      wt::k_solve_step<<<1, 256, sizeof(double) * (n * n + 2 * n) + sizeof(unsigned short) * n * (n + 1) + 16>>>(n, d, d + n * n, lambda_k, diag_floor,
                                                                     d + n * n + n);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out.data(), d + n * n + n, sizeof(double) * (n + 1), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) throw CudaError{WT_ECUDA, cudaGetErrorString(e)};
    if (out[static_cast<size_t>(n)] == 0.0) {
      status = WT_ENOTPD;
      g_err = "Cholesky factorization of the damped system failed";
      return;
    }
    std::copy(out.begin(), out.begin() + n, x);
  });
  return rc != WT_OK ? rc : status;
}

int wt_gpu_solve_vertices(int device, int32_t n, const double* dr_dphi, const double* r,
                          const double* phi, const double* nbr_delta, const int32_t* nbr_count,
                          const wt_shape_config* cfg, double* delta, uint8_t* singular) {
  return guarded(nullptr, [&] {
    if (n < 0 || !cfg) fail(WT_EINVAL, "solve_vertices: bad arguments");
    if (n == 0) return;
    WT_CUDA(cudaSetDevice(device));
    DevBuf m;
    double* d_dr = m.alloc<double>(3 * n);
    double* d_r = m.alloc<double>(n);
    double* d_phi = m.alloc<double>(3 * n);
    double* d_nd = m.alloc<double>(3 * n);
    int* d_nc = m.alloc<int>(n);
    double* d_delta = m.alloc<double>(3 * n);
    uint8_t* d_sing = m.alloc<uint8_t>(n);
    WT_CUDA(cudaMemcpy(d_dr, dr_dphi, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
    WT_CUDA(cudaMemcpy(d_r, r, sizeof(double) * n, cudaMemcpyHostToDevice));
    WT_CUDA(cudaMemcpy(d_phi, phi, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
    WT_CUDA(cudaMemcpy(d_nd, nbr_delta, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
    WT_CUDA(cudaMemcpy(d_nc, nbr_count, sizeof(int) * n, cudaMemcpyHostToDevice));
    wt::k_solve_vertices<<<(n + 255) / 256, 256>>>(n, d_dr, d_r, d_phi, d_nd, d_nc, cfg->lambda_phi,
                                                   cfg->lambda_nbr, cfg->lambda_w, cfg->diag_floor,
                                                   d_delta, d_sing);
    check_launch();
    WT_CUDA(cudaMemcpy(delta, d_delta, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    WT_CUDA(cudaMemcpy(singular, d_sing, n, cudaMemcpyDeviceToHost));
  });
}

// ---- batched sequences (C5) -------------------------------------------------------
// n_seq independent sequences of one model, tracked in lockstep: every frame
// kernel runs once for the whole batch with the sequence in blockIdx.y.

int wt_gpu_batch_set_state(wt_gpu_ctx* c, int32_t seq, const double* theta, const double* phi) {
  if (!c) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    if (seq < 0 || seq >= c->nseq) fail(WT_EINVAL, "sequence index out of range");
    if (theta) {
      upload(seq_at(c->ds.theta, c, seq), theta, c->L, c->stream);
      c->fk_valid = false;
    }
    if (phi) phi_put(c, seq_at(c->phi[c->cur], c, seq), phi);
    WT_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int wt_gpu_batch_get_state(wt_gpu_ctx* c, int32_t seq, double* theta, double* phi) {
  if (!c) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    if (seq < 0 || seq >= c->nseq) fail(WT_EINVAL, "sequence index out of range");
    if (theta)
      WT_CUDA(cudaMemcpyAsync(theta, seq_at(c->ds.theta, c, seq), sizeof(double) * c->L, cudaMemcpyDeviceToHost,
                              c->stream));
    if (phi) phi_get_async(c, seq_at(c->phi[c->cur], c, seq));
    WT_CUDA(cudaStreamSynchronize(c->stream));
    if (phi) phi_unpack(c, phi);
  });
}

int wt_gpu_batch_load_depth(wt_gpu_ctx* c, const float* depth, double depth_scale) {
  if (!c || !depth) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    const size_t row = sizeof(float) * static_cast<size_t>(c->P);
    copy_to_seqs(c, c->d_depth, depth, row, row);
    ingest(c, c->d_depth, depth_scale, nullptr, nullptr);
    c->frame_loaded = true;
    c->frame_on_rays = true;
  });
}

int wt_gpu_batch_track_async(wt_gpu_ctx* c, const wt_track_config* cfg) {
  if (!c || !cfg) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    require_frame(c);
    check_assoc(&cfg->assoc);
    if (cfg->kin.iterations < 0 || cfg->shape.iterations < 0) fail(WT_EINVAL, "negative iteration count");
    const bool shape_now = cfg->mode == WT_MODE_DYNAMIC ||
                           (cfg->mode == WT_MODE_SHAPE_MATCH && c->frame_index == 0);
    ensure_stats(c, cfg->kin.iterations, cfg->shape.iterations);
    const int start = c->cur;
    run_graph(c, track_key(c, cfg, shape_now, 1.0), [&] { enq_track(c, cfg, shape_now); });
    c->fk_valid = true;
    c->cur = (shape_now && (cfg->shape.iterations % 2)) ? start ^ 1 : start;
    c->last_nk = cfg->kin.iterations;
    c->last_ns = shape_now ? cfg->shape.iterations : 0;
    ++c->frame_index;
  });
}

int wt_gpu_batch_stats(wt_gpu_ctx* c, wt_frame_stats* stats) {
  if (!c || !stats) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    const int nk = c->last_nk, ns = c->last_ns;
    copy_from_seqs(c, c->h_kin, sizeof(wt::KinStat) * c->cap_kin, c->ds.kin_stats, sizeof(wt::KinStat) * nk);
    copy_from_seqs(c, c->h_shape, sizeof(wt::ShapeStat) * c->cap_shape, c->ds.shape_stats,
                   sizeof(wt::ShapeStat) * ns);
    WT_CUDA(cudaStreamSynchronize(c->stream));
    for (int b = 0; b < c->nseq; ++b) {
      wt_frame_stats& st = stats[b];
      st.frame = c->frame_index - 1;
      st.n_kin = nk;
      st.n_shape = ns;
      if (st.kin) put_kin(c, nk, st.kin, st.cap_kin, b);
      if (st.shape) put_shape(c, ns, st.shape, st.cap_shape, b);
    }
  });
}

int wt_gpu_batch_track(wt_gpu_ctx* c, const float* depth, double depth_scale, const wt_track_config* cfg,
                       wt_frame_stats* stats) {
  if (c && depth && cfg && c->nseq > 1 && !getenv("WT_NO_H2D_OVERLAP") && pinned_host(depth)) {
    // pinned host frames: the uploads overlap the batch's first skin /
    // normals / bucket build inside the frame graph (track_frame_overlapped)
    int rc = guarded(c, [&] {
      WT_CUDA(cudaSetDevice(c->device));
      check_assoc(&cfg->assoc);
      if (cfg->kin.iterations < 0 || cfg->shape.iterations < 0) fail(WT_EINVAL, "negative iteration count");
      const bool shape_now = cfg->mode == WT_MODE_DYNAMIC ||
                             (cfg->mode == WT_MODE_SHAPE_MATCH && c->frame_index == 0);
      ensure_stats(c, cfg->kin.iterations, cfg->shape.iterations);
      const int start = c->cur;
      c->frame_loaded = true;
      c->frame_on_rays = true;
      track_frame_overlapped(c, depth, depth_scale, cfg, shape_now);
      c->fk_valid = true;
      c->cur = (shape_now && (cfg->shape.iterations % 2)) ? start ^ 1 : start;
      c->last_nk = cfg->kin.iterations;
      c->last_ns = shape_now ? cfg->shape.iterations : 0;
      ++c->frame_index;
    });
    if (rc == WT_OK && stats) rc = wt_gpu_batch_stats(c, stats);
    if (rc == WT_OK) rc = wt_gpu_sync(c);
    return rc;
  }
  int rc = wt_gpu_batch_load_depth(c, depth, depth_scale);
  if (rc == WT_OK) rc = wt_gpu_batch_track_async(c, cfg);
  if (rc == WT_OK && stats) rc = wt_gpu_batch_stats(c, stats);
  if (rc == WT_OK) rc = wt_gpu_sync(c);
  return rc;
}

int wt_gpu_render_depth(wt_gpu_ctx* c, const double* theta, const double* phi, const wt_noise* noise,
                        int32_t frame_index, float* depth, uint8_t* joint_visible) {
  if (!c || !theta || !depth) return WT_EINVAL;
  return guarded(c, [&] {
    WT_CUDA(cudaSetDevice(c->device));
    ensure_render(c);
    std::vector<double> off(static_cast<size_t>(8 * c->L));
    host_offsets(c, theta, off.data());
    upload(c->r_off, off.data(), off.size(), c->stream);
    if (phi) upload(c->r_phi, phi, 3 * static_cast<size_t>(c->V), c->stream);
    else WT_CUDA(cudaMemsetAsync(c->r_phi, 0, sizeof(double) * 3 * c->V, c->stream));
    const wt_noise nz = noise ? *noise : wt_noise{0, 0, 0, 0};
    // base = splitmix64(seed ^ frame) (synth.cpp:237)
    uint64_t x = nz.seed ^ static_cast<uint64_t>(static_cast<int64_t>(frame_index));
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    const uint64_t base = x ^ (x >> 31);
    wt::render_launch(c->stream, c->V, c->L, c->T, c->r_off, c->r_v0, c->r_phi, c->r_wgt, c->r_wlink,
                      c->r_wcount, c->r_tri, c->r_dom, c->intr.fx, c->intr.fy, c->intr.cx, c->intr.cy,
                      c->intr.width, c->intr.height, nz.sigma, nz.dropout, nz.quantization, base,
                      c->r_vpos, c->r_zbits, c->r_owner, c->r_depth, c->r_vis);
    check_launch();
    WT_CUDA(cudaMemcpyAsync(depth, c->r_depth, sizeof(float) * c->P, cudaMemcpyDefault, c->stream));
    if (joint_visible)
      WT_CUDA(cudaMemcpyAsync(joint_visible, c->r_vis, c->L, cudaMemcpyDefault, c->stream));
    WT_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
