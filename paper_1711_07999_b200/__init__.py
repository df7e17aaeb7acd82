"""B200-native drop-in for the per-frame model-fitting hot path of warptrack
(Walsman et al., arXiv 1711.07999): track_frame / optimize_pose /
optimize_shape as sm_100a CUDA kernels behind the C-ABI in include/wt_gpu.h."""
