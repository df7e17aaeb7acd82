// wt_exact.cu -- the geometry kernels whose rounding decides association:
// forward kinematics / link offsets (k_fk and the pose-solve tail,
// skeleton.cpp:56-108), skinning and vertex normals (skinmesh.cpp:60-139).
// This unit is compiled with -fmad=false: every product and sum rounds
// separately, in the reference's operation order, so given the same link
// offsets the posed vertices and fp64 normals are bitwise the reference's
// (device sin/cos of theta/2 may still differ from libm by an ulp).
#include <cuda_runtime.h>

#include "wt_kernels.cuh"

namespace wt {

void launch_skin(cudaStream_t st, int grid, int L, const DevModel& m, const DevState& s, const double4* phi) {
  k_skin<<<grid, kVThreads, sizeof(double) * 8 * L, st>>>(m, s, phi);
}

void launch_normals(cudaStream_t st, int grid, const DevModel& m, const DevState& s, const DevIntr& in,
                    int do_bucket, int zero_acc, int compute) {
  k_normals<<<grid, kVThreads, 0, st>>>(m, s, in, do_bucket, zero_acc, compute);
}

void launch_fk(cudaStream_t st, const DevModel& m, const DevState& s) { k_fk<<<1, 128, 0, st>>>(m, s); }

void launch_pose_solve(cudaStream_t st, int L, const DevModel& m, const DevState& s, const PoseArgs& a) {
  k_pose_solve<<<1, 256, pose_solve_smem_bytes(L), st>>>(m, s, a);
}

}  // namespace wt
