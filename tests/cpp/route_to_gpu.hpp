// route_to_gpu.hpp -- TEST: force-included (g++ -include) into the reference's
// own, unmodified tests/acceptance.cpp so that its tracking calls run on the
// GPU drop-in (adapter/warptrack_gpu.*):
//   acceptance.cpp:165  track_frame    (criteria 1-2, closed loop)
//   acceptance.cpp:541  optimize_pose  (criterion 6, prior relaxation)
//   acceptance.cpp:647  run_tracking   (criterion 8, CLI-equivalent pipeline)
//   acceptance.cpp:724  track_frame    (criterion 9, throughput)
// Every header acceptance.cpp includes is included here first (they are all
// #pragma once), then the three names are redirected for the rest of the
// translation unit -- i.e. only at acceptance.cpp's own call sites.
#pragma once

#include "oracles.hpp"
#include "warptrack/kinopt.hpp"
#include "warptrack/metrics.hpp"
#include "warptrack/parallel.hpp"
#include "warptrack/seqio.hpp"
#include "warptrack/shapeopt.hpp"
#include "warptrack/synth.hpp"
#include "warptrack/tracker.hpp"
#include "warptrack_gpu.hpp"

#define track_frame ::warptrack::gpu::track_frame
#define optimize_pose ::warptrack::gpu::optimize_pose
#define run_tracking ::warptrack::gpu::run_tracking
