// warptrack_gpu.cpp -- see warptrack_gpu.hpp. Marshals the reference structs
// (AoS fp64 Eigen vectors) into the flat C-ABI of include/wt_gpu.h and maps
// status codes back onto the reference's exception types (errors.hpp).
#include "warptrack_gpu.hpp"

#include <cstdint>
#include <cstring>
#include <list>
#include <mutex>
#include <string>
#include <type_traits>

#include "warptrack/errors.hpp"
#include "wt_gpu.h"

namespace warptrack::gpu {
namespace {

[[noreturn]] void raise(int rc, const std::string& what) {
  switch (rc) {
    case WT_ELENGTH: throw LengthMismatch(what);
    case WT_EINVAL: throw ValidationError(what);
    default: throw Error(what);
  }
}

void check(int rc, const wt_gpu_ctx* ctx, const char* call) {
  if (rc == WT_OK) return;
  const char* msg = ctx ? wt_gpu_last_error(ctx) : wt_gpu_global_last_error();
  raise(rc, std::string(call) + ": " + (msg ? msg : ""));
}

wt_intrinsics to_c(const Intrinsics& in) { return {in.fx, in.fy, in.cx, in.cy, in.width, in.height}; }

wt_kin_config to_c(const KinSolverConfig& k) {
  wt_kin_config c{};
  c.iterations = k.iterations;
  c.assoc_refresh = k.assoc_refresh;
  c.lambda_k = k.lambda_k;
  c.lambda_s = k.lambda_s;
  c.diag_floor = k.diag_floor;
  c.clamp_limits = k.clamp_limits ? 1 : 0;
  c.limit = k.limit;
  return c;
}

wt_shape_config to_c(const ShapeSolverConfig& s) {
  wt_shape_config c{};
  c.iterations = s.iterations;
  c.lambda_phi = s.lambda_phi;
  c.lambda_nbr = s.lambda_nbr;
  c.lambda_w = s.lambda_w;
  c.diag_floor = s.diag_floor;
  return c;
}

wt_assoc_config to_c(const AssocConfig& a) {
  wt_assoc_config c{};
  c.window_radius = a.window_radius;
  c.cutoff = a.cutoff;
  return c;
}

wt_track_config to_c(const TrackConfig& t) {
  wt_track_config c{};
  switch (t.mode) {
    case TrackMode::dynamic: c.mode = WT_MODE_DYNAMIC; break;
    case TrackMode::shape_match: c.mode = WT_MODE_SHAPE_MATCH; break;
    case TrackMode::smooth_bind: c.mode = WT_MODE_SMOOTH_BIND; break;
    case TrackMode::rigid: c.mode = WT_MODE_RIGID; break;
  }
  c.threads = t.threads;
  c.kin = to_c(t.kin);
  c.shape = to_c(t.shape);
  c.assoc = to_c(t.assoc);
  c.shape_stats = 1;  // track_frame always collects shape stats (tracker.cpp:64)
  return c;
}

KinIterStats from_c(const wt_kin_iter_stats& s) {
  KinIterStats o;
  o.iteration = s.iteration;
  o.residual_sum = s.residual_sum;
  o.step_norm = s.step_norm;
  o.associated = s.associated;
  o.solver_skipped = s.solver_skipped != 0;
  return o;
}

ShapeIterStats from_c(const wt_shape_iter_stats& s) {
  ShapeIterStats o;
  o.iteration = s.iteration;
  o.mean_phi = s.mean_phi;
  o.max_phi = s.max_phi;
  o.mean_abs_r_before = s.mean_abs_r_before;
  o.mean_abs_r_after = s.mean_abs_r_after;
  o.singular = s.singular;
  return o;
}

// Flat arrays of the model descriptor; kept alive for wt_gpu_create only.
struct DescArrays {
  std::vector<int32_t> parent, joint_kind, theta_index, weight_count, weight_link, triangles, vtri_off, vtri_items,
      nbr_off, nbr_items;
  std::vector<double> parent_offset, joint_axis, v0, phi, weight;
  wt_model_desc desc{};

  DescArrays(const Skeleton& sk, const SkinnedMesh& mesh) {
    const int L = sk.link_count();
    const std::size_t V = mesh.v0.size();
    for (int j = 0; j < L; ++j) {
      const Link& l = sk.link(j);
      parent.push_back(l.parent);
      const Vec8 o = to_vec8(l.parent_offset);
      for (int c = 0; c < 8; ++c) parent_offset.push_back(o[c]);
      joint_kind.push_back(l.joint.kind == JointKind::prismatic ? WT_JOINT_PRISMATIC : WT_JOINT_HINGE);
      joint_axis.insert(joint_axis.end(), {l.joint.axis.x, l.joint.axis.y, l.joint.axis.z});
      theta_index.push_back(l.joint.theta_index);
    }
    for (std::size_t i = 0; i < V; ++i) {
      v0.insert(v0.end(), {mesh.v0[i].x(), mesh.v0[i].y(), mesh.v0[i].z()});
      const Vec3 p = mesh.phi.size() == V ? mesh.phi[i] : Vec3::Zero();
      phi.insert(phi.end(), {p.x(), p.y(), p.z()});
      const VertexWeights& w = mesh.weights[i];
      weight_count.push_back(w.count);
      for (int s = 0; s < 4; ++s) {
        weight_link.push_back(s < w.count ? w.entry[static_cast<std::size_t>(s)].link : -1);
        weight.push_back(s < w.count ? w.entry[static_cast<std::size_t>(s)].w : 0.0);
      }
    }
    for (const auto& t : mesh.triangles) triangles.insert(triangles.end(), {t[0], t[1], t[2]});
    vtri_off.assign(mesh.vertex_tri_offsets.begin(), mesh.vertex_tri_offsets.end());
    vtri_items.assign(mesh.vertex_tri_items.begin(), mesh.vertex_tri_items.end());
    if (vtri_off.empty()) vtri_off.assign(V + 1, 0);
    nbr_off.push_back(0);
    for (std::size_t i = 0; i < V; ++i) {
      if (i < mesh.neighbors.size())
        for (int n : mesh.neighbors[i]) nbr_items.push_back(n);
      nbr_off.push_back(static_cast<int32_t>(nbr_items.size()));
    }
    auto nz = [](auto& v) { return v.empty() ? nullptr : v.data(); };
    desc.n_links = L;
    desc.n_vertices = static_cast<int32_t>(V);
    desc.n_triangles = static_cast<int32_t>(mesh.triangles.size());
    desc.parent = parent.data();
    desc.parent_offset = parent_offset.data();
    desc.joint_kind = joint_kind.data();
    desc.joint_axis = joint_axis.data();
    desc.theta_index = theta_index.data();
    desc.v0 = nz(v0);
    desc.phi = nz(phi);
    desc.weight_count = nz(weight_count);
    desc.weight_link = nz(weight_link);
    desc.weight = nz(weight);
    desc.triangles = nz(triangles);
    desc.vtri_offsets = vtri_off.data();
    desc.vtri_items = nz(vtri_items);
    desc.nbr_offsets = nbr_off.data();
    desc.nbr_items = nz(nbr_items);
  }
};

// The CloudFrame's points as the packed [P][3] doubles the C-ABI takes: a
// Vec3 (Eigen::Vector3d) is three unpadded doubles, so the vector's storage
// already is that array and nothing is copied; otherwise it is flattened.
const double* packed_points(const CloudFrame& f, std::vector<double>& tmp) {
  if constexpr (sizeof(Vec3) == 3 * sizeof(double) && std::is_standard_layout_v<Vec3>) {
    if (!f.points.empty()) return f.points.data()->data();
  }
  tmp.resize(3 * f.points.size());
  for (std::size_t i = 0; i < f.points.size(); ++i) {
    tmp[3 * i] = f.points[i].x();
    tmp[3 * i + 1] = f.points[i].y();
    tmp[3 * i + 2] = f.points[i].z();
  }
  return tmp.data();
}

// Does track_frame run optimize_shape this frame (tracker.cpp:63-66)?
bool shape_runs(const TrackConfig& cfg, int frame_index) {
  return cfg.mode == TrackMode::dynamic || (cfg.mode == TrackMode::shape_match && frame_index == 0);
}

}  // namespace

Sequence::Sequence(const Skeleton& skeleton, const SkinnedMesh& mesh, const Intrinsics& intr, int device)
    : links_(skeleton.link_count()), vertices_(mesh.vertex_count()), intr_(intr) {
  DescArrays d(skeleton, mesh);
  const wt_intrinsics ci = to_c(intr);
  check(wt_gpu_create(device, &d.desc, &ci, &ctx_), nullptr, "wt_gpu_create");
}

Sequence::~Sequence() {
  wt_gpu_destroy(ctx_);
  wt_gpu_host_free(pinned_depth_);
}

void Sequence::upload(const TrackerState& state) {
  if (state.theta.size() != links_) throw LengthMismatch("theta size differs from the skeleton");
  std::vector<double> th(static_cast<std::size_t>(links_));
  for (int k = 0; k < links_; ++k) th[static_cast<std::size_t>(k)] = state.theta[k];
  const double* php = nullptr;
  const std::size_t V = static_cast<std::size_t>(vertices_);
  if (state.mesh.phi.size() == V) {
    bool same = phi_known_;
    for (std::size_t i = 0; same && i < V; ++i)
      for (int c = 0; c < 3; ++c) same = same && phi_mirror_[3 * i + c] == state.mesh.phi[i][c];
    if (!same) {
      phi_mirror_.resize(3 * V);
      for (std::size_t i = 0; i < V; ++i)
        for (int c = 0; c < 3; ++c) phi_mirror_[3 * i + c] = state.mesh.phi[i][c];
      php = phi_mirror_.data();
      phi_known_ = true;
    }
  }
  check(wt_gpu_set_state(ctx_, th.data(), php, state.frame_index), ctx_, "wt_gpu_set_state");
}

void Sequence::download(TrackerState& state, bool with_phi) {
  std::vector<double> th(static_cast<std::size_t>(links_));
  const std::size_t V = static_cast<std::size_t>(vertices_);
  if (with_phi) phi_mirror_.resize(3 * V);
  int32_t fi = 0;
  check(wt_gpu_get_state(ctx_, th.data(), with_phi ? phi_mirror_.data() : nullptr, &fi), ctx_, "wt_gpu_get_state");
  state.theta.resize(links_);
  for (int k = 0; k < links_; ++k) state.theta[k] = th[static_cast<std::size_t>(k)];
  if (with_phi) {
    phi_known_ = true;
    state.mesh.phi.resize(V);
    for (std::size_t i = 0; i < V; ++i)
      state.mesh.phi[i] = Vec3(phi_mirror_[3 * i], phi_mirror_[3 * i + 1], phi_mirror_[3 * i + 2]);
  }
  state.frame_index = fi;
}

namespace {
FrameStats collect(const wt_frame_stats& st, const std::vector<wt_kin_iter_stats>& k,
                   const std::vector<wt_shape_iter_stats>& s) {
  FrameStats fs;
  fs.frame = st.frame;
  for (int i = 0; i < st.n_kin; ++i) fs.kin.push_back(from_c(k[static_cast<std::size_t>(i)]));
  for (int i = 0; i < st.n_shape; ++i) fs.shape.push_back(from_c(s[static_cast<std::size_t>(i)]));
  return fs;
}
}  // namespace

FrameStats Sequence::track_frame(const CloudFrame& frame, const TrackConfig& cfg) {
  if (frame.width != intr_.width || frame.height != intr_.height)
    throw LengthMismatch("frame size differs from the intrinsics grid");
  std::vector<double> tmp;
  const double* pts = packed_points(frame, tmp);
  std::vector<wt_kin_iter_stats> k(static_cast<std::size_t>(std::max(cfg.kin.iterations, 1)));
  std::vector<wt_shape_iter_stats> s(static_cast<std::size_t>(std::max(cfg.shape.iterations, 1)));
  wt_frame_stats st{0, 0, 0, static_cast<int32_t>(k.size()), static_cast<int32_t>(s.size()), 0, k.data(), s.data()};
  const wt_track_config c = to_c(cfg);
  check(wt_gpu_track_frame_cloud(ctx_, pts, frame.valid.data(), &c, &st), ctx_, "wt_gpu_track_frame_cloud");
  return collect(st, k, s);
}

FrameStats Sequence::track_depth(const std::vector<float>& depth, double scale, const TrackConfig& cfg) {
  if (depth.size() != static_cast<std::size_t>(intr_.width) * intr_.height)
    throw LengthMismatch("depth image size differs from the intrinsics grid");
  // staged in page-locked memory: the frame graph then uploads it on a side
  // stream, overlapped with the first skin / normals / bucket build
  if (!pinned_depth_) {
    void* p = nullptr;
    check(wt_gpu_host_alloc(sizeof(float) * depth.size(), &p), nullptr, "wt_gpu_host_alloc");
    pinned_depth_ = static_cast<float*>(p);
  }
  std::memcpy(pinned_depth_, depth.data(), sizeof(float) * depth.size());
  std::vector<wt_kin_iter_stats> k(static_cast<std::size_t>(std::max(cfg.kin.iterations, 1)));
  std::vector<wt_shape_iter_stats> s(static_cast<std::size_t>(std::max(cfg.shape.iterations, 1)));
  wt_frame_stats st{0, 0, 0, static_cast<int32_t>(k.size()), static_cast<int32_t>(s.size()), 0, k.data(), s.data()};
  const wt_track_config c = to_c(cfg);
  check(wt_gpu_track_frame(ctx_, pinned_depth_, scale, &c, &st), ctx_, "wt_gpu_track_frame");
  return collect(st, k, s);
}

void Sequence::optimize_pose(const CloudFrame& frame, const KinSolverConfig& cfg, const AssocConfig& assoc,
                             std::vector<KinIterStats>* stats) {
  std::vector<double> tmp;
  check(wt_gpu_load_cloud(ctx_, packed_points(frame, tmp), frame.valid.data()), ctx_, "wt_gpu_load_cloud");
  std::vector<wt_kin_iter_stats> k(static_cast<std::size_t>(std::max(cfg.iterations, 1)));
  int32_t n = 0;
  const wt_kin_config kc = to_c(cfg);
  const wt_assoc_config ac = to_c(assoc);
  check(wt_gpu_optimize_pose(ctx_, &kc, &ac, k.data(), static_cast<int32_t>(k.size()), &n), ctx_,
        "wt_gpu_optimize_pose");
  if (stats)  // appended, as kinopt.cpp:153-169 push_back onto the caller's vector
    for (int i = 0; i < n; ++i) stats->push_back(from_c(k[static_cast<std::size_t>(i)]));
}

void Sequence::optimize_shape(const CloudFrame& frame, const ShapeSolverConfig& cfg, const AssocConfig& assoc,
                              std::vector<ShapeIterStats>* stats) {
  std::vector<double> tmp;
  check(wt_gpu_load_cloud(ctx_, packed_points(frame, tmp), frame.valid.data()), ctx_, "wt_gpu_load_cloud");
  std::vector<wt_shape_iter_stats> s(static_cast<std::size_t>(std::max(cfg.iterations, 1)));
  int32_t n = 0;
  const wt_shape_config sc = to_c(cfg);
  const wt_assoc_config ac = to_c(assoc);
  check(wt_gpu_optimize_shape(ctx_, &sc, &ac, stats ? 1 : 0, s.data(), static_cast<int32_t>(s.size()), &n), ctx_,
        "wt_gpu_optimize_shape");
  if (stats)  // appended after the caller's entries (shapeopt.cpp:56,112-129 use stats_base = size())
    for (int i = 0; i < n; ++i) stats->push_back(from_c(s[static_cast<std::size_t>(i)]));
}

// ---- free functions with the reference signatures ----------------------------------

namespace {
// What a cached device context was built from: the state's address plus the
// identity of its model (a state at a reused address, or a different model
// of the same size -- e.g. rigidify(bundle) -- does not match).
struct ModelKey {
  const TrackerState* state = nullptr;
  const Skeleton* skeleton = nullptr;
  const void* v0 = nullptr;
  const void* weights = nullptr;
  const void* triangles = nullptr;
  const void* neighbors = nullptr;
  std::size_t V = 0, T = 0, N = 0;
  int L = 0;
  std::uint64_t fingerprint = 0;
  Intrinsics intr;

  bool operator==(const ModelKey& o) const {
    return state == o.state && skeleton == o.skeleton && v0 == o.v0 && weights == o.weights &&
           triangles == o.triangles && neighbors == o.neighbors && V == o.V && T == o.T && N == o.N && L == o.L &&
           fingerprint == o.fingerprint && intr.fx == o.intr.fx && intr.fy == o.intr.fy && intr.cx == o.intr.cx &&
           intr.cy == o.intr.cy && intr.width == o.intr.width && intr.height == o.intr.height;
  }
};

// FNV-1a over the link offsets and up to 1024 evenly sampled vertices'
// template positions and skin weights (cheap enough for every call).
std::uint64_t fingerprint(const Skeleton& sk, const SkinnedMesh& m) {
  std::uint64_t h = 1469598103934665603ull;
  auto mix = [&h](const void* p, std::size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (std::size_t k = 0; k < n; ++k) h = (h ^ b[k]) * 1099511628211ull;
  };
  for (int j = 0; j < sk.link_count(); ++j) {
    const Vec8 o = to_vec8(sk.link(j).parent_offset);
    for (int c = 0; c < 8; ++c) {
      const double x = o[c];
      mix(&x, sizeof x);
    }
  }
  const std::size_t V = m.v0.size(), step = V > 1024 ? V / 1024 : 1;
  for (std::size_t i = 0; i < V; i += step) {
    for (int c = 0; c < 3; ++c) {
      const double x = m.v0[i][c];
      mix(&x, sizeof x);
    }
    if (i < m.weights.size()) {
      const VertexWeights& w = m.weights[i];
      mix(&w.count, sizeof w.count);
      for (int s = 0; s < w.count && s < 4; ++s) {
        mix(&w.entry[static_cast<std::size_t>(s)].link, sizeof(int));
        mix(&w.entry[static_cast<std::size_t>(s)].w, sizeof(double));
      }
    }
  }
  return h;
}

ModelKey key_of(const TrackerState& state, const Intrinsics& intr) {
  ModelKey k;
  k.state = &state;
  k.skeleton = state.skeleton;
  k.v0 = state.mesh.v0.data();
  k.weights = state.mesh.weights.data();
  k.triangles = state.mesh.triangles.data();
  k.neighbors = state.mesh.neighbors.data();
  k.V = state.mesh.v0.size();
  k.T = state.mesh.triangles.size();
  k.N = state.mesh.neighbors.size();
  k.L = state.skeleton->link_count();
  k.fingerprint = fingerprint(*state.skeleton, state.mesh);
  k.intr = intr;
  return k;
}

struct Cached {
  ModelKey key;
  std::unique_ptr<Sequence> seq;
};
std::mutex g_mu;
std::list<Cached> g_cache;  // most recently used first, at most kMaxCachedStates

Sequence& sequence_for(const TrackerState& state, const Intrinsics& intr) {
  if (!state.skeleton) throw ValidationError("TrackerState has no skeleton");
  const ModelKey key = key_of(state, intr);
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
    if (it->key.state != &state) continue;
    if (it->key == key) {
      g_cache.splice(g_cache.begin(), g_cache, it);
      return *g_cache.front().seq;
    }
    g_cache.erase(it);  // same address, different model: rebuild
    break;
  }
  g_cache.push_front(Cached{key, std::make_unique<Sequence>(*state.skeleton, state.mesh, intr)});
  while (g_cache.size() > static_cast<std::size_t>(kMaxCachedStates)) g_cache.pop_back();
  return *g_cache.front().seq;
}
}  // namespace

void release(const TrackerState& state) {
  std::lock_guard<std::mutex> lock(g_mu);
  g_cache.remove_if([&](const Cached& c) { return c.key.state == &state; });
}

FrameStats track_frame(TrackerState& state, const CloudFrame& frame, const Intrinsics& intr,
                       const TrackConfig& cfg) {
  Sequence& s = sequence_for(state, intr);
  s.upload(state);
  const bool shape = shape_runs(cfg, state.frame_index);
  FrameStats fs = s.track_frame(frame, cfg);
  s.download(state, shape);  // phi only moved if optimize_shape ran
  return fs;
}

void optimize_pose(TrackerState& state, const CloudFrame& frame, const Intrinsics& intr,
                   const KinSolverConfig& cfg, const AssocConfig& assoc, int /*threads*/,
                   std::vector<KinIterStats>* stats) {
  Sequence& s = sequence_for(state, intr);
  s.upload(state);
  s.optimize_pose(frame, cfg, assoc, stats);
  s.download(state, false);
}

void optimize_shape(TrackerState& state, const CloudFrame& frame, const Intrinsics& intr,
                    const ShapeSolverConfig& cfg, const AssocConfig& assoc, int /*threads*/,
                    std::vector<ShapeIterStats>* stats) {
  Sequence& s = sequence_for(state, intr);
  s.upload(state);
  s.optimize_shape(frame, cfg, assoc, stats);
  s.download(state);
}

TrackOutputs run_tracking(const ModelBundle& bundle, SequenceReader& reader, const TrackConfig& cfg,
                          const Pose& init, const FrameCallback& callback) {
  // as tracker.cpp:75-77: the bundle is tracked as given (callers rigidify
  // for the rigid mode, e.g. bindings.cpp:250-251)
  TrackerState state = make_tracker(bundle, init);
  const Intrinsics intr = reader.header().intrinsics();
  Sequence seq(bundle, intr);
  seq.upload(state);
  const bool need_phi = static_cast<bool>(callback);

  TrackOutputs out;
  for (const Link& l : bundle.skeleton.links()) out.estimate.joint_names.push_back(l.name);
  const int L = bundle.skeleton.link_count();
  std::vector<double> joints(3 * static_cast<std::size_t>(L));
  for (int f = 0; f < reader.frame_count(); ++f) {
    const std::vector<float> depth = reader.read_depth(f);
    const bool shape = shape_runs(cfg, state.frame_index);
    out.stats.push_back(seq.track_depth(depth, reader.header().depth_scale, cfg));
    seq.download(state, need_phi && shape);
    check(wt_gpu_joint_positions(seq.handle(), joints.data()), seq.handle(), "wt_gpu_joint_positions");
    std::vector<Vec3> js(static_cast<std::size_t>(L));
    for (int j = 0; j < L; ++j)
      js[static_cast<std::size_t>(j)] = Vec3(joints[3 * static_cast<std::size_t>(j)],
                                             joints[3 * static_cast<std::size_t>(j) + 1],
                                             joints[3 * static_cast<std::size_t>(j) + 2]);
    out.estimate.theta.push_back(state.theta);
    out.estimate.joints.push_back(std::move(js));
    out.estimate.visible.emplace_back(static_cast<std::size_t>(L), 1);
    if (callback) callback(state, f, reader.read_frame(f));
  }
  seq.download(state);
  out.final_phi = state.mesh.phi;
  return out;
}

}  // namespace warptrack::gpu
