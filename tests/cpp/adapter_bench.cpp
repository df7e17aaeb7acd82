// adapter_bench.cpp -- TIMING TOOL: the reference's own C++ API for the hot
// path (track_frame, tracker.hpp:36-37; run_tracking, tracker.hpp:50-52)
// executed on the GPU through the drop-in adapter (adapter/warptrack_gpu.*)
// inside the reference library, as INTEGRATION.md links it. The model comes
// as a raw wt_model_desc dump (bench.py writes it; the driver's
// wtref_model_from_desc builds the reference ModelBundle from it), the frames
// as a .wts read by the reference's SequenceReader. Built by
// `make -C oracle/ref adapter`; bench.py reports it as `e2e_reference_api`.
//
//   adapter_bench <model.desc> <seq.wts> <warmup> <steps>
//
// Prints one JSON object: frames/s of gpu::track_frame on the reference's
// CloudFrames (each call uploads the frame and synchronises theta / phi of
// the host TrackerState, returning FrameStats) and of gpu::run_tracking over
// the file, host clock (steady_clock, as acceptance.cpp:718-726).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "warptrack/seqio.hpp"
#include "warptrack/tracker.hpp"
#include "warptrack_gpu.hpp"
#include "wt_gpu.h"

struct wtref_model;
extern "C" int wtref_model_from_desc(const wt_model_desc* d, wtref_model** out);
const warptrack::ModelBundle* wtref_bundle_of(const wtref_model* m);

using namespace warptrack;
using Clock = std::chrono::steady_clock;

namespace {
template <class T>
std::vector<T> take(std::ifstream& in, std::size_t n) {
  std::vector<T> v(std::max<std::size_t>(n, 1));
  in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(sizeof(T) * n));
  return v;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: adapter_bench model.desc seq.wts warmup steps\n");
    return 2;
  }
  std::ifstream in(argv[1], std::ios::binary);
  int32_t hdr[5];
  in.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
  const int L = hdr[0], V = hdr[1], T = hdr[2], NVT = hdr[3], NNB = hdr[4];
  auto parent = take<int32_t>(in, L);
  auto poff = take<double>(in, 8 * static_cast<std::size_t>(L));
  auto kind = take<int32_t>(in, L);
  auto axis = take<double>(in, 3 * static_cast<std::size_t>(L));
  auto tix = take<int32_t>(in, L);
  auto v0 = take<double>(in, 3 * static_cast<std::size_t>(V));
  auto phi = take<double>(in, 3 * static_cast<std::size_t>(V));
  auto wc = take<int32_t>(in, V);
  auto wl = take<int32_t>(in, 4 * static_cast<std::size_t>(V));
  auto ww = take<double>(in, 4 * static_cast<std::size_t>(V));
  auto tri = take<int32_t>(in, 3 * static_cast<std::size_t>(T));
  auto vto = take<int32_t>(in, static_cast<std::size_t>(V) + 1);
  auto vti = take<int32_t>(in, NVT);
  auto nbo = take<int32_t>(in, static_cast<std::size_t>(V) + 1);
  auto nbi = take<int32_t>(in, NNB);
  if (!in) {
    std::fprintf(stderr, "short model descriptor\n");
    return 2;
  }
  wt_model_desc d{};
  d.n_links = L;
  d.n_vertices = V;
  d.n_triangles = T;
  d.parent = parent.data();
  d.parent_offset = poff.data();
  d.joint_kind = kind.data();
  d.joint_axis = axis.data();
  d.theta_index = tix.data();
  d.v0 = v0.data();
  d.phi = phi.data();
  d.weight_count = wc.data();
  d.weight_link = wl.data();
  d.weight = ww.data();
  d.triangles = tri.data();
  d.vtri_offsets = vto.data();
  d.vtri_items = vti.data();
  d.nbr_offsets = nbo.data();
  d.nbr_items = nbi.data();
  wtref_model* h = nullptr;
  if (wtref_model_from_desc(&d, &h) != 0) {
    std::fprintf(stderr, "model rejected\n");
    return 2;
  }
  const ModelBundle& bundle = *wtref_bundle_of(h);

  SequenceReader reader(argv[2]);
  const int warm = std::atoi(argv[3]), steps = std::atoi(argv[4]);
  if (reader.frame_count() < warm + steps) {
    std::fprintf(stderr, "sequence too short\n");
    return 2;
  }
  const Intrinsics intr = reader.header().intrinsics();
  std::vector<CloudFrame> clouds;
  for (int f = 0; f < reader.frame_count(); ++f) clouds.push_back(reader.read_frame(f));
  TrackConfig cfg;  // dynamic, 5 pose + 2 surface iterations (the bench workload)
  cfg.mode = TrackMode::dynamic;
  cfg.kin.iterations = 5;
  cfg.shape.iterations = 2;

  // gpu::track_frame on the reference's CloudFrames: the TrackerState stays on the host
  TrackerState state = make_tracker(bundle, bundle.skeleton.zero_pose());
  for (int f = 0; f < warm; ++f) gpu::track_frame(state, clouds[static_cast<std::size_t>(f)], intr, cfg);
  const auto t0 = Clock::now();
  for (int f = 0; f < steps; ++f) gpu::track_frame(state, clouds[static_cast<std::size_t>(warm + f)], intr, cfg);
  const double dt = std::chrono::duration<double>(Clock::now() - t0).count();
  gpu::release(state);

  // gpu::run_tracking over the file (frame reads included)
  SequenceReader r2(argv[2]);
  const auto t1 = Clock::now();
  const TrackOutputs out = gpu::run_tracking(bundle, r2, cfg, bundle.skeleton.zero_pose());
  const double dt2 = std::chrono::duration<double>(Clock::now() - t1).count();
  std::printf(
      "{\"track_frame_cloud\": {\"value\": %.3f, \"unit\": \"frames/s\", \"frames\": %d, \"seconds\": %.4f, "
      "\"api\": \"warptrack::gpu::track_frame(TrackerState&, const CloudFrame&, const Intrinsics&, const "
      "TrackConfig&): the host TrackerState synchronised every call\"}, "
      "\"run_tracking\": {\"value\": %.3f, \"unit\": \"frames/s\", \"frames\": %d, \"seconds\": %.4f, "
      "\"api\": \"warptrack::gpu::run_tracking(const ModelBundle&, SequenceReader&, ...): .wts frames read "
      "each step\"}, \"vertices\": %d, \"width\": %d, \"height\": %d}\n",
      steps / dt, steps, dt, out.estimate.frame_count() / dt2, out.estimate.frame_count(), dt2,
      bundle.mesh.vertex_count(), intr.width, intr.height);
  return 0;
}
