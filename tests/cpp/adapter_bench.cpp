// adapter_bench.cpp -- TIMING TOOL: the reference's own C++ API for the hot
// path (track_frame, tracker.hpp:36-37; run_tracking, tracker.hpp:50-52)
// executed on the GPU through the drop-in adapter (adapter/warptrack_gpu.*),
// on a model and a .wts sequence the reference itself loads (load_model,
// SequenceReader). Built by `make -C oracle/ref adapter`; bench.py runs it
// and reports the numbers as `e2e_reference_api`.
//
//   adapter_bench <model.json> <seq.wts> <warmup> <steps>
//
// Prints one JSON object: frames/s of gpu::track_frame on reference
// CloudFrames (each call uploads the frame, syncs theta/phi of the host
// TrackerState, returns FrameStats), of gpu::run_tracking over the file, and
// the host clock of both (steady_clock, as acceptance.cpp:718-726).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "warptrack/seqio.hpp"
#include "warptrack/tracker.hpp"
#include "warptrack_gpu.hpp"

using namespace warptrack;
using Clock = std::chrono::steady_clock;

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: adapter_bench model.json seq.wts warmup steps\n");
    return 2;
  }
  const ModelBundle bundle = load_model(argv[1]);
  SequenceReader reader(argv[2]);
  const int warm = std::atoi(argv[3]), steps = std::atoi(argv[4]);
  if (reader.frame_count() < warm + steps + 1) {
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

  // gpu::track_frame with reference CloudFrames: the TrackerState stays on the host
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
      "TrackConfig&) -- host TrackerState synchronised every call\"}, "
      "\"run_tracking\": {\"value\": %.3f, \"unit\": \"frames/s\", \"frames\": %d, \"seconds\": %.4f, "
      "\"api\": \"warptrack::gpu::run_tracking(ModelBundle, SequenceReader&, ...) -- .wts frames read each step\"}, "
      "\"vertices\": %d, \"width\": %d, \"height\": %d}\n",
      steps / dt, steps, dt, out.estimate.frame_count() / dt2, out.estimate.frame_count(), dt2,
      bundle.mesh.vertex_count(), intr.width, intr.height);
  return 0;
}
