// warptrack_gpu.hpp -- the reference-side adapter: warptrack's own C++
// tracker API (tracker.hpp:36-37, kinopt.hpp:67-69, shapeopt.hpp:62-64,
// tracker.cpp:70-100) executed by libwt_gpu.so through include/wt_gpu.h.
//
// A maintainer adds adapter/warptrack_gpu.{hpp,cpp} to proj/src, links
// libwt_gpu.so, and routes callers through warptrack::gpu.
// The signatures are the reference's; only the namespace differs, so
// call sites change by one qualifier (or a using-declaration).
#pragma once

#include <memory>
#include <vector>

#include "warptrack/tracker.hpp"

struct wt_gpu_ctx;

namespace warptrack::gpu {

/// One GPU context per tracking sequence: the model uploaded once, theta /
/// Phi / frame index resident on the device. Not thread-safe; distinct
/// Sequences are independent (different host threads, streams, devices).
class Sequence {
 public:
  Sequence(const Skeleton& skeleton, const SkinnedMesh& mesh, const Intrinsics& intr, int device = 0);
  Sequence(const ModelBundle& bundle, const Intrinsics& intr, int device = 0)
      : Sequence(bundle.skeleton, bundle.mesh, intr, device) {}
  ~Sequence();
  Sequence(const Sequence&) = delete;
  Sequence& operator=(const Sequence&) = delete;

  /// TrackerState <-> device (theta, mesh.phi, frame_index). Phi crosses
  /// only when it differs from what the device holds (a host mirror of the
  /// last synchronised Phi), so a caller that leaves state.mesh.phi alone
  /// between frames pays no Phi upload.
  void upload(const TrackerState& state);
  void download(TrackerState& state, bool with_phi = true);

  FrameStats track_frame(const CloudFrame& frame, const TrackConfig& cfg);
  FrameStats track_depth(const std::vector<float>& depth, double scale, const TrackConfig& cfg);
  void optimize_pose(const CloudFrame& frame, const KinSolverConfig& cfg, const AssocConfig& assoc,
                     std::vector<KinIterStats>* stats);
  void optimize_shape(const CloudFrame& frame, const ShapeSolverConfig& cfg, const AssocConfig& assoc,
                      std::vector<ShapeIterStats>* stats);

  wt_gpu_ctx* handle() const { return ctx_; }
  int link_count() const { return links_; }
  int vertex_count() const { return vertices_; }

 private:
  wt_gpu_ctx* ctx_ = nullptr;
  int links_ = 0, vertices_ = 0;
  Intrinsics intr_;
  std::vector<double> phi_mirror_;  // packed [V][3]: the device's Phi as of the last upload / download
  bool phi_known_ = false;
  float* pinned_depth_ = nullptr;   // page-locked staging: track_depth takes the overlapped upload path
};

/// Drop-in replacements with the reference signatures. Each call keeps a
/// device context cached per TrackerState, keyed by the state's address AND
/// its model's identity (the skeleton pointer, the mesh arrays' addresses and
/// sizes, and a fingerprint of sampled template vertices, skin weights and
/// link offsets), so a new state at a reused address or a rigidified model
/// gets its own upload. At most kMaxCachedStates contexts are kept (least
/// recently used dropped). Each call synchronises theta / phi / frame_index
/// in and out, so the host TrackerState stays authoritative exactly as in
/// the reference (phi only moves when it changed, see Sequence::upload).
constexpr int kMaxCachedStates = 16;
FrameStats track_frame(TrackerState& state, const CloudFrame& frame, const Intrinsics& intr,
                       const TrackConfig& cfg);
void optimize_pose(TrackerState& state, const CloudFrame& frame, const Intrinsics& intr,
                   const KinSolverConfig& cfg, const AssocConfig& assoc, int threads,
                   std::vector<KinIterStats>* stats);
void optimize_shape(TrackerState& state, const CloudFrame& frame, const Intrinsics& intr,
                    const ShapeSolverConfig& cfg, const AssocConfig& assoc, int threads,
                    std::vector<ShapeIterStats>* stats);

/// run_tracking (tracker.cpp:70-100) with the state resident on the GPU for
/// the whole sequence: frames are read with the reference's SequenceReader,
/// theta comes back each frame (the callback sees a host TrackerState with
/// theta and frame_index current; phi is synchronised only when a callback
/// is given), Phi once at the end.
TrackOutputs run_tracking(const ModelBundle& bundle, SequenceReader& reader, const TrackConfig& cfg,
                          const Pose& init, const FrameCallback& callback = nullptr);

/// Drops the cached context of a TrackerState (e.g. before it is destroyed).
void release(const TrackerState& state);

}  // namespace warptrack::gpu
