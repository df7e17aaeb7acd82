/*
 * wt_gpu.h -- C-ABI drop-in boundary for the per-frame model-fitting hot path
 * of warptrack (Walsman et al., arXiv 1711.07999) on NVIDIA B200 (sm_100a).
 *
 * Every entry point takes plain pointers and sizes; no C++ or torch types
 * cross this boundary and no exception escapes it. Status codes replace the
 * reference's exception taxonomy (proj/include/warptrack/errors.hpp:9-66):
 *   WT_EINVAL   <- ValidationError / bad arguments
 *   WT_ELENGTH  <- LengthMismatch
 *   WT_ENOTPD   <- NotPositiveDefinite (solve_step only; inside a frame a
 *                  Cholesky failure stays "skip the iteration + flag", exactly
 *                  like proj/src/kinopt.cpp:160-168)
 *   WT_ECUDA / WT_ENOMEM for device failures.
 *   WT_ERANGE   a frame's fixed-point normal equations left the int64 range
 *               (the device reduction's scales are chosen from the model and
 *               the cutoff so this needs a diverged pose; the reference, which
 *               sums in fp64, would take the step)
 * The message of the last failure is available from wt_gpu_last_error().
 *
 * Replaced reference interfaces (file:line into /root/reference/proj):
 *   wt_gpu_track_frame / _cloud  <- track_frame        include/warptrack/tracker.hpp:36-37
 *   wt_gpu_optimize_pose         <- optimize_pose      include/warptrack/kinopt.hpp:67-69
 *   wt_gpu_optimize_shape        <- optimize_shape     include/warptrack/shapeopt.hpp:62-64
 *   wt_gpu_skin                  <- skin / link_offsets include/warptrack/skinmesh.hpp:74-78,
 *                                                       include/warptrack/skeleton.hpp:73-75
 *   wt_gpu_associate(_posed)     <- associate / associate_winners
 *                                                      include/warptrack/association.hpp:63-71
 *   wt_gpu_normal_system         <- accumulate_normal_system include/warptrack/kinopt.hpp:47-50
 *   wt_gpu_solve_step            <- solve_step         include/warptrack/kinopt.hpp:54
 *   wt_gpu_solve_vertices        <- solve_vertex (batched) include/warptrack/shapeopt.hpp:48
 *   wt_gpu_render_depth          <- synthesize_frame   include/warptrack/synth.hpp:92-94
 *   wt_model_desc                <- Skeleton / SkinnedMesh (skeleton.hpp:14-63, skinmesh.hpp:31-48)
 *   wt_intrinsics                <- Intrinsics          association.hpp:11-15
 *   wt_track_config              <- TrackConfig         tracker.hpp:14-20 (+ KinSolverConfig
 *                                   kinopt.hpp:10-18, ShapeSolverConfig shapeopt.hpp:9-15,
 *                                   AssocConfig tracker_state.hpp:11-14)
 *   wt_frame_stats               <- FrameStats          tracker.hpp:28-32
 *
 * Threading: one context = one tracking sequence = one CUDA stream. A context
 * is not thread-safe; distinct contexts are independent (different host
 * threads, devices). The reference's `threads` field is accepted and ignored.
 */
#ifndef WT_GPU_H
#define WT_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WT_ABI_VERSION 2

enum {
  WT_OK = 0,
  WT_EINVAL = 1,
  WT_ELENGTH = 2,
  WT_ECUDA = 3,
  WT_ENOMEM = 4,
  WT_ENOTPD = 5,
  WT_ENODEV = 6,
  WT_ERANGE = 7
};

/* TrackMode, tracker_state.hpp:9 */
enum { WT_MODE_DYNAMIC = 0, WT_MODE_SHAPE_MATCH = 1, WT_MODE_SMOOTH_BIND = 2, WT_MODE_RIGID = 3 };
/* JointKind, skeleton.hpp:10 */
enum { WT_JOINT_HINGE = 0, WT_JOINT_PRISMATIC = 1 };

typedef struct wt_intrinsics {
  double fx, fy, cx, cy;
  int32_t width, height;
} wt_intrinsics;

typedef struct wt_kin_config {
  int32_t iterations;    /* 12 */
  int32_t assoc_refresh; /* 1 */
  double lambda_k;       /* 1e-2 */
  double lambda_s;       /* 1e-4 */
  double diag_floor;     /* 1e-9 */
  int32_t clamp_limits;  /* 0 */
  int32_t pad_;
  double limit;          /* 0 */
} wt_kin_config;

typedef struct wt_shape_config {
  int32_t iterations; /* 2 */
  int32_t pad_;
  double lambda_phi;  /* 0.05 */
  double lambda_nbr;  /* 0.5 */
  double lambda_w;    /* 1e-2 */
  double diag_floor;  /* 1e-9 */
} wt_shape_config;

typedef struct wt_assoc_config {
  int32_t window_radius; /* 5 */
  int32_t pad_;
  double cutoff;         /* 0.10 */
} wt_assoc_config;

typedef struct wt_track_config {
  int32_t mode;         /* WT_MODE_* (dynamic) */
  int32_t threads;      /* ignored on the GPU */
  wt_kin_config kin;
  wt_shape_config shape;
  wt_assoc_config assoc;
  int32_t shape_stats;  /* 1 = run optimize_shape's closing stats pass
                           (track_frame always does, tracker.cpp:64) */
  int32_t pad_;
} wt_track_config;

typedef struct wt_kin_iter_stats { /* KinIterStats, kinopt.hpp:56-62 */
  int32_t iteration;
  int32_t associated;
  double residual_sum;
  double step_norm;
  int32_t solver_skipped;
  int32_t pad_;
} wt_kin_iter_stats;

typedef struct wt_shape_iter_stats { /* ShapeIterStats, shapeopt.hpp:50-57 */
  int32_t iteration;
  int32_t singular;
  double mean_phi;
  double max_phi;
  double mean_abs_r_before;
  double mean_abs_r_after;
} wt_shape_iter_stats;

typedef struct wt_frame_stats { /* FrameStats, tracker.hpp:28-32 */
  int32_t frame;
  int32_t n_kin;     /* out */
  int32_t n_shape;   /* out */
  int32_t cap_kin;   /* capacity of kin[] */
  int32_t cap_shape; /* capacity of shape[] */
  int32_t pad_;
  wt_kin_iter_stats* kin;
  wt_shape_iter_stats* shape;
} wt_frame_stats;

typedef struct wt_noise { /* NoiseSpec, synth.hpp:34-39 */
  double sigma, dropout, quantization;
  uint64_t seed;
} wt_noise;

/* Flat mirror of ModelBundle {Skeleton, SkinnedMesh}. Weight rows hold up to
 * four (link, w) entries in the reference's entry order (entry 0 is the
 * blend pivot, skinmesh.cpp:64); unused slots are ignored. Triangles and the
 * vertex->triangle CSR are SkinnedMesh::finalize()'s output
 * (skinmesh.cpp:13-58); neighbours are build_neighbors(v0, 4)'s lists
 * (skinmesh.cpp:196-247) in CSR form. */
typedef struct wt_model_desc {
  int32_t n_links;
  int32_t n_vertices;
  int32_t n_triangles;
  int32_t pad_;
  const int32_t* parent;        /* [L] -1 for the root */
  const double* parent_offset;  /* [L*8] canonical (w,x,y,z | w,x,y,z) */
  const int32_t* joint_kind;    /* [L] WT_JOINT_* */
  const double* joint_axis;     /* [L*3] unit */
  const int32_t* theta_index;   /* [L] */
  const double* v0;             /* [V*3] */
  const double* phi;            /* [V*3] or NULL (zeros) */
  const int32_t* weight_count;  /* [V] 0..4 */
  const int32_t* weight_link;   /* [V*4] */
  const double* weight;         /* [V*4] */
  const int32_t* triangles;     /* [T*3] */
  const int32_t* vtri_offsets;  /* [V+1] */
  const int32_t* vtri_items;    /* [vtri_offsets[V]] */
  const int32_t* nbr_offsets;   /* [V+1] */
  const int32_t* nbr_items;     /* [nbr_offsets[V]] */
} wt_model_desc;

typedef struct wt_gpu_ctx wt_gpu_ctx;

/* ---- library / context ------------------------------------------------- */
int wt_gpu_abi_version(void);
int wt_gpu_device_count(void);
/* Message of the last failure of a context-free call on this thread. */
const char* wt_gpu_global_last_error(void);

/* Validates the skeleton like Skeleton::build (skeleton.cpp:7-50), computes
 * the bind pose (FK at theta = 0) and influence counts S (kinopt.cpp:58-70),
 * uploads the model once and allocates per-sequence device state. */
int wt_gpu_create(int device, const wt_model_desc* model, const wt_intrinsics* intr,
                  wt_gpu_ctx** out);
void wt_gpu_destroy(wt_gpu_ctx* ctx);
const char* wt_gpu_last_error(const wt_gpu_ctx* ctx);

/* TrackerState {theta, mesh.phi, frame_index} (tracker_state.hpp:18-23).
 * phi may be NULL (left unchanged on set / not read on get). */
int wt_gpu_set_state(wt_gpu_ctx* ctx, const double* theta, const double* phi, int32_t frame_index);
int wt_gpu_get_state(wt_gpu_ctx* ctx, double* theta, double* phi, int32_t* frame_index);

/* ---- frames -------------------------------------------------------------- */
/* Depth frame exactly as SequenceReader::read_depth returns it (row-major
 * float32, 0 = invalid); unprojected on the device like depth_to_cloud
 * (seqio.cpp:419-437). `depth` may be host (pageable or pinned) or device.
 * A device frame of the context's GPU is read by the next call that consumes
 * the frame (a track call copies and unprojects it inside its frame graph,
 * overlapped with the first skinning and bucketing), so it must stay valid
 * and unchanged until that call. */
int wt_gpu_load_depth(wt_gpu_ctx* ctx, const float* depth, double depth_scale);
/* Organized CloudFrame (association.hpp:19-29): points [P*3], valid [P]. */
int wt_gpu_load_cloud(wt_gpu_ctx* ctx, const double* points, const uint8_t* valid);

/* ---- the hot path ---------------------------------------------------------- */
/* track_frame (tracker.cpp:54-68) on the loaded frame. stats may be NULL. */
int wt_gpu_track_loaded(wt_gpu_ctx* ctx, const wt_track_config* cfg, wt_frame_stats* stats);
/* load_depth + track_loaded. With a pinned host frame the upload and its
 * unprojection run on a side stream inside the frame graph and are joined
 * before the first correspondence search, so they overlap the first skin /
 * normals / bucket build; theta comes back with the stats, so a
 * wt_gpu_get_state(theta only) right after costs no device round trip. */
int wt_gpu_track_frame(wt_gpu_ctx* ctx, const float* depth, double depth_scale,
                       const wt_track_config* cfg, wt_frame_stats* stats);
/* load_cloud + track_loaded. */
int wt_gpu_track_frame_cloud(wt_gpu_ctx* ctx, const double* points, const uint8_t* valid,
                             const wt_track_config* cfg, wt_frame_stats* stats);
/* run_tracking (tracker.cpp:70-100) over n_frames depth images laid out
 * back to back ([n_frames][H*W] float, host or device memory): track_frame on
 * each in order, recording theta [n_frames*L] and the link origins
 * transform_point(FK(theta)[j], 0) [n_frames*L*3] (either may be NULL).
 * Host frames are staged through pinned double buffers on a copy stream so
 * frame f+1's upload overlaps frame f's solve. frame_index advances by
 * n_frames; the final Phi stays in the context (wt_gpu_get_state). */
int wt_gpu_track_sequence(wt_gpu_ctx* ctx, const float* frames, int32_t n_frames, double depth_scale,
                          const wt_track_config* cfg, double* theta_out, double* joints_out);
/* reconstruction_error_frame (metrics.cpp:110-142) of the current state (theta,
 * Phi) against the loaded frame: for every vertex visible in the z-buffer of
 * the posed mesh (front-facing, in frame, within 1 mm of the depth at its
 * pixel) the distance to the nearest valid observed point, exact (brute force,
 * fp64). dist [V] receives NaN for vertices that are not visible; n_visible
 * (nullable) their count. */
int wt_gpu_recon_error(wt_gpu_ctx* ctx, double* dist, int32_t* n_visible);
/* Link origins at the current theta, [L*3] (tracker.cpp:84-86). */
int wt_gpu_joint_positions(wt_gpu_ctx* ctx, double* joints_out);
/* optimize_pose (kinopt.cpp:132-171) / optimize_shape (shapeopt.cpp:50-130)
 * on the loaded frame; stats arrays may be NULL. */
int wt_gpu_optimize_pose(wt_gpu_ctx* ctx, const wt_kin_config* kin, const wt_assoc_config* assoc,
                         wt_kin_iter_stats* stats, int32_t cap, int32_t* n_out);
int wt_gpu_optimize_shape(wt_gpu_ctx* ctx, const wt_shape_config* shape,
                          const wt_assoc_config* assoc, int32_t with_stats_pass,
                          wt_shape_iter_stats* stats, int32_t cap, int32_t* n_out);

/* ---- model preprocessing on the device ----------------------------------------- */
/* subdivide(mesh, iterations) (skinmesh.cpp:490-511: Catmull-Clark of
 * positions, phi and skin weights by catmull_clark_once :298-470, then
 * truncate_weights :265-280), SkinnedMesh::finalize() (skinmesh.cpp:13-58:
 * triangles + vertex->triangle CSR) and, for k_neighbors > 0,
 * build_neighbors(v0, k) (skinmesh.cpp:196-247) -- all on the device, bitwise
 * the reference's. iterations == 0 only finalizes (weights kept as given).
 * Inputs: template vertices, phi (NULL: zeros), weight rows as in
 * wt_model_desc, polygons as CSR. The result is read with wt_gpu_mesh_sizes /
 * wt_gpu_mesh_export (any output pointer may be NULL) and released with
 * wt_gpu_mesh_free. Errors: WT_EINVAL (bad input; an edge with more than two
 * faces, the reference's NonManifold), WT_ENODEV, WT_ECUDA / WT_ENOMEM; the
 * message is wt_gpu_mesh_last_error(). */
typedef struct wt_mesh wt_mesh;
int wt_gpu_mesh_subdivide(int device, int32_t n_vertices, int32_t n_links, const double* v0, const double* phi,
                          const int32_t* weight_count, const int32_t* weight_link, const double* weight,
                          int32_t n_polys, const int32_t* poly_offsets, const int32_t* poly_items,
                          int32_t iterations, int32_t k_neighbors, wt_mesh** out);
int wt_gpu_mesh_sizes(const wt_mesh* mesh, int32_t* n_vertices, int32_t* n_polys, int32_t* n_poly_items,
                      int32_t* n_triangles, int32_t* n_neighbors_per_vertex);
int wt_gpu_mesh_export(const wt_mesh* mesh, double* v0, double* phi, int32_t* weight_count, int32_t* weight_link,
                       double* weight, int32_t* poly_offsets, int32_t* poly_items, int32_t* triangles,
                       int32_t* vtri_offsets, int32_t* vtri_items, int32_t* neighbors);
void wt_gpu_mesh_free(wt_mesh* mesh);
const char* wt_gpu_mesh_last_error(void);
/* build_neighbors(v0, k) alone (skinmesh.cpp:196-247): out[n][min(k, n-1)],
 * each row ascending by (squared distance, index); k <= 16. */
int wt_gpu_build_neighbors(int device, int32_t n, const double* v0, int32_t k, int32_t* out);

/* ---- page-locked host staging ----------------------------------------------- */
/* Page-locked host memory (cudaMallocHost) for callers that do not link the
 * CUDA runtime (the reference-side adapter): a depth frame staged there takes
 * wt_gpu_track_frame's overlapped upload path. */
int wt_gpu_host_alloc(size_t bytes, void** out);
void wt_gpu_host_free(void* p);

/* ---- asynchronous use / measurement --------------------------------------- */
/* The context's CUDA stream (cudaStream_t) for event timing by the caller. */
void* wt_gpu_stream(wt_gpu_ctx* ctx);
/* Enqueues track_frame on the loaded frame without waiting and without
 * stats; wt_gpu_sync (or any synchronous call) waits for completion. */
int wt_gpu_track_async(wt_gpu_ctx* ctx, const wt_track_config* cfg);
int wt_gpu_sync(wt_gpu_ctx* ctx);
/* Runs one track_frame through an instrumented graph (a CUDA event after
 * every kernel) and returns each kernel's kind and device time in ms:
 * 0 fk, 1 skin, 2 normals+bucket, 3 scatter, 4 search+average,
 * 5 pose system, 6 shape step, 7 shape stats pass, 8 pose solve,
 * 9 pixel offsets (the bucket CSR scan). */
int wt_gpu_profile_frame(wt_gpu_ctx* ctx, const wt_track_config* cfg, int32_t* kinds, float* ms,
                         int32_t cap, int32_t* n_out);
/* Vertices bucketed by the last association of sequence `seq` (the size of
 * the VertexBuckets item list, association.cpp:39-67): measurement only. */
int wt_gpu_bucket_count(wt_gpu_ctx* ctx, int32_t seq, int32_t* n_bucketed);

/* ---- batched sequences --------------------------------------------------- */
/* n_seq independent tracking sequences of ONE model, tracked in lockstep
 * (run_tracking, tracker.cpp:73-90, for n_seq sequences at once): every
 * frame kernel runs once for the whole batch, the sequence index in
 * blockIdx.y, so a frame of the batch is one CUDA graph whatever n_seq is.
 * Each sequence has its own TrackerState (theta, phi) and frame; the frame
 * index and mode schedule are shared. The per-frame calls above return
 * WT_EINVAL on a batch context; wt_gpu_set_state / wt_gpu_get_state act on
 * sequence 0 and the shared frame index. */
int wt_gpu_create_batch(int device, const wt_model_desc* model, const wt_intrinsics* intr, int32_t n_seq,
                        wt_gpu_ctx** out);
int32_t wt_gpu_batch_size(const wt_gpu_ctx* ctx);
/* theta [L] / phi [V*3] of sequence seq (either may be NULL). */
int wt_gpu_batch_set_state(wt_gpu_ctx* ctx, int32_t seq, const double* theta, const double* phi);
int wt_gpu_batch_get_state(wt_gpu_ctx* ctx, int32_t seq, double* theta, double* phi);
/* depth [n_seq][H][W] (host or device), one frame per sequence. */
int wt_gpu_batch_load_depth(wt_gpu_ctx* ctx, const float* depth, double depth_scale);
/* track_frame for every sequence on the loaded frames, without waiting. */
int wt_gpu_batch_track_async(wt_gpu_ctx* ctx, const wt_track_config* cfg);
/* stats[n_seq] of the last batch frame (waits for it). */
int wt_gpu_batch_stats(wt_gpu_ctx* ctx, wt_frame_stats* stats);
/* load + track + (stats may be NULL) + wait. */
int wt_gpu_batch_track(wt_gpu_ctx* ctx, const float* depth, double depth_scale, const wt_track_config* cfg,
                       wt_frame_stats* stats);

/* ---- stage hooks (parity / tests) --------------------------------------- */
/* skin(mesh, link_offsets(theta)) with phi override (NULL = state phi).
 * Outputs are host arrays [V*3],[V*3],[V]; any may be NULL. */
int wt_gpu_skin(wt_gpu_ctx* ctx, const double* theta, const double* phi, double* v, double* n,
                uint8_t* valid);
/* associate() on the posed mesh of the last wt_gpu_skin call and the loaded
 * frame: winners [P] (-1 none), p_tilde [V*3], count [V], residual [V]. */
int wt_gpu_associate(wt_gpu_ctx* ctx, int32_t window_radius, double cutoff, int32_t* winners,
                     double* p_tilde, int32_t* count, double* residual);
/* Context-free association of arbitrary posed vertices (the reference's
 * "loose vertex" tests) against an organized cloud. */
int wt_gpu_associate_posed(int device, const wt_intrinsics* intr, int32_t n_vertices,
                           const double* v, const double* n, const uint8_t* valid,
                           const double* points, const uint8_t* point_valid,
                           int32_t window_radius, double cutoff, int32_t* winners,
                           double* p_tilde, int32_t* count, double* residual);
/* accumulate_normal_system at theta for a given association (count,
 * residual [V]); jtj [L*L] row-major, jtr [L]. */
int wt_gpu_normal_system(wt_gpu_ctx* ctx, const double* theta, const wt_kin_config* kin,
                         const int32_t* count, const double* residual, double* jtj, double* jtr);
/* solve_step: A = JtJ + lambda_k diag(JtJ) + floor I, x = A^-1 Jtr by a
 * device Cholesky; WT_ENOTPD on non-finite input or a failed factorisation. */
int wt_gpu_solve_step(int device, int32_t n, const double* jtj, const double* jtr,
                      double lambda_k, double diag_floor, double* x);
/* solve_vertex over a batch of independent problems (shapeopt.cpp:25-48). */
int wt_gpu_solve_vertices(int device, int32_t n, const double* dr_dphi, const double* r,
                          const double* phi, const double* nbr_delta, const int32_t* nbr_count,
                          const wt_shape_config* cfg, double* delta, uint8_t* singular);
/* synthesize_frame (synth.cpp:229-270): z-buffer render of the posed model
 * with the stateless splitmix64 noise; depth [H*W], joint_visible [L]. */
int wt_gpu_render_depth(wt_gpu_ctx* ctx, const double* theta, const double* phi,
                        const wt_noise* noise, int32_t frame_index, float* depth,
                        uint8_t* joint_visible);

#ifdef __cplusplus
}
#endif

#endif /* WT_GPU_H */
