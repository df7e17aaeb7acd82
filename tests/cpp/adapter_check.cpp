// adapter_check.cpp -- TEST: the reference's own C++ API driven through the
// GPU adapter (adapter/warptrack_gpu.*) against the unmodified reference CPU
// implementation on the same inputs. Built by `make -C oracle/ref adapter`
// (reference objects + adapter + libwt_gpu.so) and run on a GPU box by
// tests/test_adapter.py. Prints one line per check and exits non-zero on the
// first failure.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <string>

#include "warptrack/synth.hpp"
#include "warptrack_gpu.hpp"

using namespace warptrack;

namespace {

int failures = 0;

void expect(bool ok, const std::string& what, double got, double tol) {
  std::printf("%s %-58s %.3e (tol %.1e)\n", ok ? "PASS" : "FAIL", what.c_str(), got, tol);
  if (!ok) ++failures;
}

double max_abs(const Pose& a, const Pose& b) {
  double m = 0.0;
  for (int k = 0; k < a.size(); ++k) m = std::max(m, std::abs(a[k] - b[k]));
  return m;
}

double max_abs(const std::vector<Vec3>& a, const std::vector<Vec3>& b) {
  double m = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i)
    for (int c = 0; c < 3; ++c) m = std::max(m, std::abs(a[i][c] - b[i][c]));
  return m;
}

Pose pose_at(const Skeleton& sk, int f) {
  Pose p = sk.zero_pose();
  p[0] = -0.5;  // prismatic root toward the camera
  for (int k = 1; k < p.size(); ++k) p[k] = 0.25 * std::sin(0.35 * f + 0.7 * k);
  return p;
}

}  // namespace

int main(int argc, char** argv) {
  const std::filesystem::path dir = argc > 1 ? argv[1] : std::filesystem::temp_directory_path();
  ModelBundle bundle = make_biped_rig();
  bundle.mesh = subdivide(bundle.mesh, 1);
  bundle.mesh.neighbors = build_neighbors(bundle.mesh.v0, 4);
  Intrinsics intr;
  intr.width = 320;
  intr.height = 240;
  intr.fx = intr.fy = 365.456 * 320 / 512.0;
  intr.cx = 160;
  intr.cy = 120;
  const Skeleton& sk = bundle.skeleton;
  std::printf("biped sub1: %d vertices, %d links\n", bundle.mesh.vertex_count(), sk.link_count());

  // 1. track_frame drop-in on CloudFrames (dynamic 5 + 2), TrackerState stays on the host
  {
    TrackConfig cfg;
    cfg.kin.iterations = 5;
    cfg.shape.iterations = 2;
    TrackerState cpu = make_tracker(bundle, pose_at(sk, 0));
    TrackerState gpu_state = make_tracker(bundle, pose_at(sk, 0));
    for (int f = 1; f <= 3; ++f) {
      const CloudFrame frame = render_frame(bundle, pose_at(sk, f), {}, intr, NoiseSpec{}, f);
      const FrameStats a = track_frame(cpu, frame, intr, cfg);
      const FrameStats b = gpu::track_frame(gpu_state, frame, intr, cfg);
      expect(max_abs(cpu.theta, gpu_state.theta) <= 1e-6, "track_frame theta, frame " + std::to_string(f),
             max_abs(cpu.theta, gpu_state.theta), 1e-6);
      expect(max_abs(cpu.mesh.phi, gpu_state.mesh.phi) <= 1e-6, "track_frame phi, frame " + std::to_string(f),
             max_abs(cpu.mesh.phi, gpu_state.mesh.phi), 1e-6);
      bool same = a.kin.size() == b.kin.size() && a.frame == b.frame && gpu_state.frame_index == cpu.frame_index;
      for (std::size_t k = 0; same && k < a.kin.size(); ++k) same = a.kin[k].associated == b.kin[k].associated;
      expect(same, "track_frame stats (frame, associated per iteration)", same ? 0.0 : 1.0, 0.0);
    }
    gpu::release(gpu_state);
  }

  // 2. optimize_pose / optimize_shape drop-ins (test_kinopt / test_shapeopt call them directly)
  {
    const CloudFrame frame = render_frame(bundle, pose_at(sk, 2), {}, intr, NoiseSpec{}, 2);
    TrackerState cpu = make_tracker(bundle, pose_at(sk, 1));
    TrackerState gpu_state = make_tracker(bundle, pose_at(sk, 1));
    KinSolverConfig kin;
    kin.assoc_refresh = 3;
    std::vector<KinIterStats> sa, sb;
    optimize_pose(cpu, frame, intr, kin, AssocConfig{}, 1, &sa);
    gpu::optimize_pose(gpu_state, frame, intr, kin, AssocConfig{}, 1, &sb);
    expect(max_abs(cpu.theta, gpu_state.theta) <= 1e-6, "optimize_pose theta (12 its, assoc_refresh 3)",
           max_abs(cpu.theta, gpu_state.theta), 1e-6);
    double rs = 0.0;
    for (std::size_t k = 0; k < sa.size() && k < sb.size(); ++k)
      rs = std::max(rs, std::abs(sa[k].residual_sum - sb[k].residual_sum) / std::max(1e-30, sa[k].residual_sum));
    expect(sa.size() == sb.size() && rs <= 1e-6, "optimize_pose residual_sum per iteration (relative)", rs, 1e-6);
    ShapeSolverConfig shp;
    std::vector<ShapeIterStats> ta, tb;
    optimize_shape(cpu, frame, intr, shp, AssocConfig{}, 1, &ta);
    gpu::optimize_shape(gpu_state, frame, intr, shp, AssocConfig{}, 1, &tb);
    expect(max_abs(cpu.mesh.phi, gpu_state.mesh.phi) <= 1e-6, "optimize_shape phi",
           max_abs(cpu.mesh.phi, gpu_state.mesh.phi), 1e-6);
    bool same = ta.size() == tb.size();
    for (std::size_t k = 0; same && k < ta.size(); ++k) same = ta[k].singular == tb[k].singular;
    expect(same, "optimize_shape singular counts", same ? 0.0 : 1.0, 0.0);
    gpu::release(gpu_state);
  }

  // 3. run_tracking over a .wts written by the reference's SequenceWriter
  {
    const std::filesystem::path seq = dir / "adapter_check.wts";
    SequenceHeader h;
    h.width = static_cast<std::uint32_t>(intr.width);
    h.height = static_cast<std::uint32_t>(intr.height);
    h.fx = intr.fx;
    h.fy = intr.fy;
    h.cx = intr.cx;
    h.cy = intr.cy;
    h.frame_count = 6;
    {
      SequenceWriter w(seq, h);
      for (int f = 1; f <= 6; ++f)
        w.write_depth(synthesize_frame(bundle, pose_at(sk, f), {}, intr, NoiseSpec{}, f).depth);
      w.close();
    }
    for (TrackMode mode : {TrackMode::dynamic, TrackMode::smooth_bind, TrackMode::rigid}) {
      TrackConfig cfg;
      cfg.mode = mode;
      cfg.kin.iterations = 5;
      cfg.shape.iterations = 2;
      SequenceReader ra(seq), rb(seq);
      // callers rigidify for the rigid mode (bindings.cpp:250-251)
      const ModelBundle tracked = mode == TrackMode::rigid ? rigidify(bundle) : bundle;
      const TrackOutputs a = run_tracking(tracked, ra, cfg, pose_at(sk, 0));
      const TrackOutputs b = gpu::run_tracking(tracked, rb, cfg, pose_at(sk, 0));
      double th = 0.0, jt = 0.0;
      for (int f = 0; f < a.estimate.frame_count(); ++f) {
        th = std::max(th, max_abs(a.estimate.theta[static_cast<std::size_t>(f)], b.estimate.theta[static_cast<std::size_t>(f)]));
        jt = std::max(jt, max_abs(a.estimate.joints[static_cast<std::size_t>(f)], b.estimate.joints[static_cast<std::size_t>(f)]));
      }
      const std::string m = to_string(mode);
      expect(b.estimate.frame_count() == 6 && th <= 1e-6, "run_tracking theta, 6 frames, " + m, th, 1e-6);
      expect(jt <= 1e-6, "run_tracking joint positions, " + m, jt, 1e-6);
      const double ph = max_abs(a.final_phi, b.final_phi);
      expect(ph <= 1e-6, "run_tracking final phi, " + m, ph, 1e-6);
    }
  }

  // 4. the context cache follows the model, not just the state's address: the
  //    same TrackerState object re-pointed at a rigidified model (same vertex
  //    and link counts, different weights) must track with the new weights
  {
    TrackConfig cfg;
    cfg.kin.iterations = 5;
    cfg.shape.iterations = 2;
    const ModelBundle rigid = rigidify(bundle);
    TrackerState gpu_state = make_tracker(bundle, pose_at(sk, 0));
    const CloudFrame f1 = render_frame(bundle, pose_at(sk, 1), {}, intr, NoiseSpec{}, 1);
    gpu::track_frame(gpu_state, f1, intr, cfg);  // caches a context for the blended model
    gpu_state.mesh = rigid.mesh;                 // same object, another model
    gpu_state.theta = pose_at(sk, 1);
    TrackerState cpu = make_tracker(rigid, pose_at(sk, 1));
    cpu.frame_index = gpu_state.frame_index;
    const CloudFrame f2 = render_frame(rigid, pose_at(sk, 2), {}, intr, NoiseSpec{}, 2);
    track_frame(cpu, f2, intr, cfg);
    gpu::track_frame(gpu_state, f2, intr, cfg);
    expect(max_abs(cpu.theta, gpu_state.theta) <= 1e-6, "model swapped under the same TrackerState: theta",
           max_abs(cpu.theta, gpu_state.theta), 1e-6);
    expect(max_abs(cpu.mesh.phi, gpu_state.mesh.phi) <= 1e-6, "model swapped under the same TrackerState: phi",
           max_abs(cpu.mesh.phi, gpu_state.mesh.phi), 1e-6);
    // stats are appended to the caller's vector (kinopt.cpp:153-169)
    std::vector<KinIterStats> st;
    KinSolverConfig kin;
    kin.iterations = 3;
    gpu::optimize_pose(gpu_state, f2, intr, kin, AssocConfig{}, 1, &st);
    gpu::optimize_pose(gpu_state, f2, intr, kin, AssocConfig{}, 1, &st);
    expect(st.size() == 6, "optimize_pose appends its stats", static_cast<double>(st.size()), 6.0);
    gpu::release(gpu_state);
  }

  // 5. errors map onto the reference's exception types
  {
    TrackerState bad = make_tracker(bundle, sk.zero_pose());
    bad.theta.resize(2);
    bool threw = false;
    try {
      gpu::track_frame(bad, render_frame(bundle, sk.zero_pose(), {}, intr, NoiseSpec{}), intr, TrackConfig{});
    } catch (const LengthMismatch&) {
      threw = true;
    }
    expect(threw, "wrong theta size raises LengthMismatch", threw ? 0.0 : 1.0, 0.0);
    gpu::release(bad);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
