// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (the CPU checker, never shipped).
//
// A thin extern "C" driver over the UNMODIFIED reference warptrack sources
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/ref/Makefile
// against the Eigen-subset shim in oracle/ref/eigen_shim). It exposes the
// reference's own hot-path functions with plain pointers so the Python tests
// and bench.py's CPU baseline can call them on exactly the inputs the GPU
// path receives. Nothing here re-implements reference behaviour: each entry
// point marshals arrays into the reference structs and calls the reference
// function named in its comment.
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "warptrack/association.hpp"
#include "warptrack/kinopt.hpp"
#include "warptrack/metrics.hpp"
#include "warptrack/parallel.hpp"
#include "warptrack/seqio.hpp"
#include "warptrack/shapeopt.hpp"
#include "warptrack/skinmesh.hpp"
#include "warptrack/synth.hpp"
#include "warptrack/tracker.hpp"
#include "wt_gpu.h"

using namespace warptrack;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return WT_OK;
  } catch (const LengthMismatch& e) {
    g_err = e.what();
    return WT_ELENGTH;
  } catch (const NotPositiveDefinite& e) {
    g_err = e.what();
    return WT_ENOTPD;
  } catch (const std::exception& e) {
    g_err = e.what();
    return WT_EINVAL;
  }
}

Intrinsics to_intr(const wt_intrinsics* i) {
  Intrinsics r;
  r.fx = i->fx;
  r.fy = i->fy;
  r.cx = i->cx;
  r.cy = i->cy;
  r.width = i->width;
  r.height = i->height;
  return r;
}

KinSolverConfig to_kin(const wt_kin_config* k) {
  KinSolverConfig c;
  c.iterations = k->iterations;
  c.lambda_k = k->lambda_k;
  c.lambda_s = k->lambda_s;
  c.diag_floor = k->diag_floor;
  c.assoc_refresh = k->assoc_refresh;
  c.clamp_limits = k->clamp_limits != 0;
  c.limit = k->limit;
  return c;
}

ShapeSolverConfig to_shape(const wt_shape_config* s) {
  ShapeSolverConfig c;
  c.iterations = s->iterations;
  c.lambda_phi = s->lambda_phi;
  c.lambda_nbr = s->lambda_nbr;
  c.lambda_w = s->lambda_w;
  c.diag_floor = s->diag_floor;
  return c;
}

AssocConfig to_assoc(const wt_assoc_config* a) {
  AssocConfig c;
  c.window_radius = a->window_radius;
  c.cutoff = a->cutoff;
  return c;
}

TrackConfig to_track(const wt_track_config* t) {
  TrackConfig c;
  c.mode = static_cast<TrackMode>(t->mode);
  c.kin = to_kin(&t->kin);
  c.shape = to_shape(&t->shape);
  c.assoc = to_assoc(&t->assoc);
  c.threads = t->threads;
  return c;
}

std::vector<Vec3> vec3s(const double* p, std::size_t n) {
  std::vector<Vec3> out(n);
  for (std::size_t i = 0; i < n; ++i) out[i] = Vec3(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
  return out;
}

void put_vec3s(const std::vector<Vec3>& v, double* out) {
  if (!out) return;
  for (std::size_t i = 0; i < v.size(); ++i) {
    out[3 * i] = v[i].x();
    out[3 * i + 1] = v[i].y();
    out[3 * i + 2] = v[i].z();
  }
}

Pose to_pose(const double* theta, int n) {
  Pose p = Pose::Zero(n);
  for (int k = 0; k < n; ++k) p[k] = theta[k];
  return p;
}

CloudFrame to_cloud(const Intrinsics& intr, const double* pts, const uint8_t* valid) {
  CloudFrame f;
  f.width = intr.width;
  f.height = intr.height;
  const std::size_t n = static_cast<std::size_t>(intr.width) * intr.height;
  f.points = vec3s(pts, n);
  f.valid.assign(valid, valid + n);
  return f;
}

PosedMesh to_posed(int nv, const double* v, const double* n, const uint8_t* valid) {
  PosedMesh p;
  p.v = vec3s(v, static_cast<std::size_t>(nv));
  p.n = vec3s(n, static_cast<std::size_t>(nv));
  p.valid.assign(valid, valid + nv);
  return p;
}

}  // namespace

struct wtref_model {
  ModelBundle bundle;
};

// The bundle behind a handle (C++ tools linking this driver, e.g. adapter_bench).
const warptrack::ModelBundle* wtref_bundle_of(const wtref_model* m) { return m ? &m->bundle : nullptr; }

struct wtref_tracker {
  std::shared_ptr<wtref_model> model;
  TrackerState state;
};

extern "C" {

const char* wtref_last_error(void) { return g_err.c_str(); }
int wtref_hardware_threads(void) { return resolve_threads(0); }

// ---- models ------------------------------------------------------------

// Builds a ModelBundle from the flat description. Skeleton::build validates
// (skeleton.cpp:7-50); triangles / CSR / neighbours are taken as given.
int wtref_model_from_desc(const wt_model_desc* d, wtref_model** out) {
  return guarded([&] {
    auto m = std::make_unique<wtref_model>();
    std::vector<Link> links(static_cast<std::size_t>(d->n_links));
    for (int j = 0; j < d->n_links; ++j) {
      Link& l = links[static_cast<std::size_t>(j)];
      l.name = "link" + std::to_string(j);
      l.parent = d->parent[j];
      Vec8 o;
      for (int c = 0; c < 8; ++c) o[c] = d->parent_offset[8 * j + c];
      l.parent_offset = from_vec8(o);
      l.joint.kind = d->joint_kind[j] == WT_JOINT_PRISMATIC ? JointKind::prismatic : JointKind::hinge;
      l.joint.axis = Axis(d->joint_axis[3 * j], d->joint_axis[3 * j + 1], d->joint_axis[3 * j + 2]);
      l.joint.theta_index = d->theta_index[j];
    }
    m->bundle.skeleton = Skeleton::build(std::move(links));
    SkinnedMesh& mesh = m->bundle.mesh;
    const std::size_t nv = static_cast<std::size_t>(d->n_vertices);
    mesh.v0 = vec3s(d->v0, nv);
    mesh.phi = d->phi ? vec3s(d->phi, nv) : std::vector<Vec3>(nv, Vec3::Zero());
    mesh.weights.resize(nv);
    for (std::size_t i = 0; i < nv; ++i)
      for (int s = 0; s < d->weight_count[i]; ++s)
        mesh.weights[i].add(d->weight_link[4 * i + s], d->weight[4 * i + s]);
    mesh.triangles.resize(static_cast<std::size_t>(d->n_triangles));
    mesh.polys.resize(static_cast<std::size_t>(d->n_triangles));
    for (int t = 0; t < d->n_triangles; ++t) {
      mesh.triangles[t] = {d->triangles[3 * t], d->triangles[3 * t + 1], d->triangles[3 * t + 2]};
      mesh.polys[t] = {d->triangles[3 * t], d->triangles[3 * t + 1], d->triangles[3 * t + 2]};
    }
    mesh.vertex_tri_offsets.assign(d->vtri_offsets, d->vtri_offsets + nv + 1);
    mesh.vertex_tri_items.assign(d->vtri_items, d->vtri_items + d->vtri_offsets[nv]);
    mesh.neighbors.resize(nv);
    for (std::size_t i = 0; i < nv; ++i)
      mesh.neighbors[i].assign(d->nbr_items + d->nbr_offsets[i], d->nbr_items + d->nbr_offsets[i + 1]);
    *out = m.release();
  });
}

// make_rig (synth.cpp:571-576).
int wtref_make_rig(const char* name, wtref_model** out) {
  return guarded([&] {
    auto m = std::make_unique<wtref_model>();
    m->bundle = make_rig(name);
    *out = m.release();
  });
}

// subdivide (skinmesh.cpp:490-511) + build_neighbors(v0, 4), as the Python
// binding subdivide_model does (bindings.cpp:154-161).
int wtref_subdivide(const wtref_model* in, int iterations, wtref_model** out) {
  return guarded([&] {
    auto m = std::make_unique<wtref_model>();
    m->bundle = in->bundle;
    m->bundle.mesh = subdivide(in->bundle.mesh, iterations);
    m->bundle.mesh.neighbors = build_neighbors(m->bundle.mesh.v0, 4);
    *out = m.release();
  });
}

// rigidify (tracker.cpp:24-43).
int wtref_rigidify(const wtref_model* in, wtref_model** out) {
  return guarded([&] {
    auto m = std::make_unique<wtref_model>();
    m->bundle = rigidify(in->bundle);
    *out = m.release();
  });
}

void wtref_model_free(wtref_model* m) { delete m; }

int wtref_model_sizes(const wtref_model* m, int* n_links, int* n_vertices, int* n_triangles,
                      int* n_vtri_items, int* n_nbr_items, int* n_polys, int* n_poly_items) {
  const SkinnedMesh& mesh = m->bundle.mesh;
  *n_links = m->bundle.skeleton.link_count();
  *n_vertices = mesh.vertex_count();
  *n_triangles = static_cast<int>(mesh.triangles.size());
  *n_vtri_items = static_cast<int>(mesh.vertex_tri_items.size());
  int nn = 0;
  for (const auto& nb : mesh.neighbors) nn += static_cast<int>(nb.size());
  *n_nbr_items = nn;
  *n_polys = static_cast<int>(mesh.polys.size());
  int np = 0;
  for (const auto& p : mesh.polys) np += static_cast<int>(p.size());
  *n_poly_items = np;
  return WT_OK;
}

// Exports the bundle in the wt_model_desc layout (caller-allocated arrays,
// sizes from wtref_model_sizes) plus the authored polygon list.
int wtref_model_export(const wtref_model* m, int* parent, double* parent_offset, int* joint_kind,
                       double* joint_axis, int* theta_index, double* v0, double* phi,
                       int* weight_count, int* weight_link, double* weight, int* triangles,
                       int* vtri_offsets, int* vtri_items, int* nbr_offsets, int* nbr_items,
                       int* poly_offsets, int* poly_items) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    for (int j = 0; j < sk.link_count(); ++j) {
      const Link& l = sk.link(j);
      parent[j] = l.parent;
      const Vec8 o = to_vec8(l.parent_offset);
      for (int c = 0; c < 8; ++c) parent_offset[8 * j + c] = o[c];
      joint_kind[j] = l.joint.kind == JointKind::prismatic ? WT_JOINT_PRISMATIC : WT_JOINT_HINGE;
      joint_axis[3 * j] = l.joint.axis.x;
      joint_axis[3 * j + 1] = l.joint.axis.y;
      joint_axis[3 * j + 2] = l.joint.axis.z;
      theta_index[j] = l.joint.theta_index;
    }
    const SkinnedMesh& mesh = m->bundle.mesh;
    const std::size_t nv = mesh.v0.size();
    put_vec3s(mesh.v0, v0);
    if (mesh.phi.size() == nv) put_vec3s(mesh.phi, phi);
    else std::memset(phi, 0, sizeof(double) * 3 * nv);
    for (std::size_t i = 0; i < nv; ++i) {
      const VertexWeights& w = mesh.weights[i];
      weight_count[i] = w.count;
      for (int s = 0; s < 4; ++s) {
        weight_link[4 * i + s] = s < w.count ? w.entry[static_cast<std::size_t>(s)].link : -1;
        weight[4 * i + s] = s < w.count ? w.entry[static_cast<std::size_t>(s)].w : 0.0;
      }
    }
    for (std::size_t t = 0; t < mesh.triangles.size(); ++t)
      for (int c = 0; c < 3; ++c) triangles[3 * t + c] = mesh.triangles[t][static_cast<std::size_t>(c)];
    std::copy(mesh.vertex_tri_offsets.begin(), mesh.vertex_tri_offsets.end(), vtri_offsets);
    std::copy(mesh.vertex_tri_items.begin(), mesh.vertex_tri_items.end(), vtri_items);
    int k = 0;
    for (std::size_t i = 0; i < nv; ++i) {
      nbr_offsets[i] = k;
      for (int n : mesh.neighbors[i]) nbr_items[k++] = n;
    }
    nbr_offsets[nv] = k;
    int p = 0;
    for (std::size_t f = 0; f < mesh.polys.size(); ++f) {
      poly_offsets[f] = p;
      for (int vi : mesh.polys[f]) poly_items[p++] = vi;
    }
    poly_offsets[mesh.polys.size()] = p;
  });
}

// SkinnedMesh::finalize (skinmesh.cpp:13-58) on an arbitrary polygon list.
// Outputs: n_triangles, then (after a second call with buffers) triangles and
// the vertex->triangle CSR. Pass NULL buffers to query the count.
int wtref_finalize(int nv, const double* v0, int npolys, const int* poly_offsets,
                   const int* poly_items, int* n_triangles, int* triangles, int* vtri_offsets,
                   int* vtri_items) {
  return guarded([&] {
    SkinnedMesh mesh;
    mesh.v0 = vec3s(v0, static_cast<std::size_t>(nv));
    mesh.polys.resize(static_cast<std::size_t>(npolys));
    for (int f = 0; f < npolys; ++f)
      mesh.polys[f].assign(poly_items + poly_offsets[f], poly_items + poly_offsets[f + 1]);
    mesh.finalize();
    *n_triangles = static_cast<int>(mesh.triangles.size());
    if (!triangles) return;
    for (std::size_t t = 0; t < mesh.triangles.size(); ++t)
      for (int c = 0; c < 3; ++c) triangles[3 * t + c] = mesh.triangles[t][static_cast<std::size_t>(c)];
    std::copy(mesh.vertex_tri_offsets.begin(), mesh.vertex_tri_offsets.end(), vtri_offsets);
    std::copy(mesh.vertex_tri_items.begin(), mesh.vertex_tri_items.end(), vtri_items);
  });
}

// build_neighbors (skinmesh.cpp:196-247): out_items [nv*k] padded with -1,
// out_counts [nv].
int wtref_build_neighbors(int nv, const double* v0, int k, int* out_items, int* out_counts) {
  return guarded([&] {
    const auto nb = build_neighbors(vec3s(v0, static_cast<std::size_t>(nv)), k);
    for (int i = 0; i < nv; ++i) {
      out_counts[i] = static_cast<int>(nb[static_cast<std::size_t>(i)].size());
      for (int s = 0; s < k; ++s)
        out_items[i * k + s] =
            s < out_counts[i] ? nb[static_cast<std::size_t>(i)][static_cast<std::size_t>(s)] : -1;
    }
  });
}

// ---- kinematics / skinning ------------------------------------------------

// forward_kinematics + link_offsets (skeleton.cpp:56-80): fk, offsets [L*8].
int wtref_fk(const wtref_model* m, const double* theta, double* fk_out, double* offsets_out) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    const auto fk = forward_kinematics(sk, to_pose(theta, sk.joint_count()));
    const auto off = link_offsets(sk, fk);
    for (std::size_t j = 0; j < fk.size(); ++j) {
      const Vec8 a = to_vec8(fk[j]), b = to_vec8(off[j]);
      for (int c = 0; c < 8; ++c) {
        if (fk_out) fk_out[8 * j + c] = a[c];
        if (offsets_out) offsets_out[8 * j + c] = b[c];
      }
    }
  });
}

// compute_pose_derivatives (kinopt.cpp:11-23): dchain as a dense [L*L*8]
// array, entry (j, k) = dH_jD/dtheta_k (zero for non-ancestors).
int wtref_pose_derivatives(const wtref_model* m, const double* theta, double* dchain) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    const int L = sk.link_count();
    const PoseDerivatives pd = compute_pose_derivatives(sk, to_pose(theta, L));
    std::memset(dchain, 0, sizeof(double) * static_cast<std::size_t>(L) * L * 8);
    for (int j = 0; j < L; ++j)
      for (const auto& [k, d8] : pd.dchain[static_cast<std::size_t>(j)])
        for (int c = 0; c < 8; ++c) dchain[(static_cast<std::size_t>(j) * L + k) * 8 + c] = d8[c];
  });
}

// skin(mesh, link_offsets(theta), phi) (skinmesh.cpp:104-141).
int wtref_skin(const wtref_model* m, const double* theta, const double* phi, int threads,
               double* v, double* n, uint8_t* valid) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    const auto off = link_offsets(sk, to_pose(theta, sk.joint_count()));
    const std::size_t nv = m->bundle.mesh.v0.size();
    const PosedMesh posed = phi ? skin(m->bundle.mesh, off, vec3s(phi, nv), threads)
                                : skin(m->bundle.mesh, off, threads);
    put_vec3s(posed.v, v);
    put_vec3s(posed.n, n);
    if (valid) std::copy(posed.valid.begin(), posed.valid.end(), valid);
  });
}

// influence_counts (kinopt.cpp:58-70).
int wtref_influence_counts(const wtref_model* m, double* s) {
  return guarded([&] {
    const Eigen::VectorXd v = influence_counts(m->bundle.skeleton, m->bundle.mesh);
    for (Eigen::Index k = 0; k < v.size(); ++k) s[k] = v[k];
  });
}

// vertex_jacobian (kinopt.cpp:51-56) with the posed mesh at theta.
int wtref_vertex_jacobian(const wtref_model* m, const double* theta, int i, double* row) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    const PoseDerivatives pd = compute_pose_derivatives(sk, to_pose(theta, sk.joint_count()));
    const PosedMesh posed = skin(m->bundle.mesh, pd.offsets);
    const Eigen::VectorXd r = vertex_jacobian(m->bundle.mesh, i, posed, pd, sk);
    for (Eigen::Index k = 0; k < r.size(); ++k) row[k] = r[k];
  });
}

// ---- association --------------------------------------------------------------

// project (association.cpp:29-37). Returns 1 and (u,v) when it lands.
int wtref_project(const wt_intrinsics* intr, double x, double y, double z, int* u, int* v) {
  const auto pc = project(to_intr(intr), Vec3(x, y, z));
  if (!pc) return 0;
  *u = pc->u;
  *v = pc->v;
  return 1;
}

// bucket_occupancy (association.cpp:39-67) on an explicit posed mesh.
// offsets [P+1], items [<= nv]; *n_items receives the item count.
int wtref_bucket_occupancy(const wt_intrinsics* intr, int nv, const double* v, const double* n,
                           const uint8_t* valid, int* offsets, int* items, int* n_items) {
  return guarded([&] {
    const VertexBuckets b = bucket_occupancy(to_posed(nv, v, n, valid), to_intr(intr));
    std::copy(b.offsets.begin(), b.offsets.end(), offsets);
    std::copy(b.items.begin(), b.items.end(), items);
    *n_items = static_cast<int>(b.items.size());
  });
}

// associate (association.cpp:111-138) + associate_winners (:69-109) on an
// explicit posed mesh and organized cloud.
int wtref_associate(const wt_intrinsics* intr, int nv, const double* v, const double* n,
                    const uint8_t* valid, const double* points, const uint8_t* point_valid,
                    int window, double cutoff, int threads, int* winners, double* p_tilde,
                    int* count, double* residual) {
  return guarded([&] {
    const Intrinsics in = to_intr(intr);
    const PosedMesh posed = to_posed(nv, v, n, valid);
    const CloudFrame frame = to_cloud(in, points, point_valid);
    if (winners) {
      const VertexBuckets b = bucket_occupancy(posed, in);
      const auto w = associate_winners(frame, b, posed, window, cutoff, threads);
      std::copy(w.begin(), w.end(), winners);
    }
    const AssociationResult r = associate(frame, in, posed, window, cutoff, threads);
    put_vec3s(r.p_tilde, p_tilde);
    if (count) std::copy(r.count.begin(), r.count.end(), count);
    if (residual) std::copy(r.residual.begin(), r.residual.end(), residual);
  });
}

// depth_to_cloud (seqio.cpp:419-437): points [P*3], valid [P].
int wtref_depth_to_cloud(const wt_intrinsics* intr, const float* depth, double scale,
                         double* points, uint8_t* valid) {
  return guarded([&] {
    const Intrinsics in = to_intr(intr);
    const std::size_t n = static_cast<std::size_t>(in.width) * in.height;
    const CloudFrame f = depth_to_cloud(in, std::vector<float>(depth, depth + n), scale);
    put_vec3s(f.points, points);
    std::copy(f.valid.begin(), f.valid.end(), valid);
  });
}

// ---- pose system ----------------------------------------------------------------

// accumulate_normal_system (kinopt.cpp:72-119) at theta with the model's phi,
// for a given association (count, residual); jtj row-major [L*L].
int wtref_normal_system(const wtref_model* m, const double* theta, const wt_kin_config* kin,
                        const int* count, const double* residual, int threads, double* jtj,
                        double* jtr) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    const int L = sk.joint_count();
    const Pose pose = to_pose(theta, L);
    const PoseDerivatives pd = compute_pose_derivatives(sk, pose);
    const PosedMesh posed = skin(m->bundle.mesh, pd.offsets, threads);
    const std::size_t nv = posed.v.size();
    AssociationResult assoc;
    assoc.p_tilde.assign(nv, Vec3::Zero());
    assoc.count.assign(count, count + nv);
    assoc.residual.assign(residual, residual + nv);
    const Eigen::VectorXd s = influence_counts(sk, m->bundle.mesh);
    const NormalSystem sys = accumulate_normal_system(m->bundle.mesh, posed, assoc, pd, sk, s,
                                                      to_kin(kin), pose, threads);
    for (int a = 0; a < L; ++a) {
      jtr[a] = sys.jtr[a];
      for (int b = 0; b < L; ++b) jtj[a * L + b] = sys.jtj(a, b);
    }
  });
}

// solve_step (kinopt.cpp:121-130). WT_ENOTPD mirrors NotPositiveDefinite.
int wtref_solve_step(int n, const double* jtj, const double* jtr, double lambda_k,
                     double diag_floor, double* x) {
  return guarded([&] {
    NormalSystem sys;
    sys.jtj = Eigen::MatrixXd::Zero(n, n);
    sys.jtr = Eigen::VectorXd::Zero(n);
    for (int a = 0; a < n; ++a) {
      sys.jtr[a] = jtr[a];
      for (int b = 0; b < n; ++b) sys.jtj(a, b) = jtj[a * n + b];
    }
    KinSolverConfig cfg;
    cfg.lambda_k = lambda_k;
    cfg.diag_floor = diag_floor;
    const Eigen::VectorXd r = solve_step(sys, cfg);
    for (int a = 0; a < n; ++a) x[a] = r[a];
  });
}

// solve_vertex (shapeopt.cpp:25-48) for one problem.
int wtref_solve_vertex(const double* dr_dphi, double r, const double* phi, const double* nbr_delta,
                       int nbr_count, const wt_shape_config* cfg, double* delta, int* singular) {
  return guarded([&] {
    VertexShapeProblem p;
    p.dr_dphi = Vec3(dr_dphi[0], dr_dphi[1], dr_dphi[2]);
    p.r = r;
    p.phi = Vec3(phi[0], phi[1], phi[2]);
    p.nbr_delta = Vec3(nbr_delta[0], nbr_delta[1], nbr_delta[2]);
    p.nbr_count = nbr_count;
    const VertexShapeStep s = solve_vertex(p, to_shape(cfg));
    delta[0] = s.delta.x();
    delta[1] = s.delta.y();
    delta[2] = s.delta.z();
    *singular = s.singular ? 1 : 0;
  });
}

// ---- tracker --------------------------------------------------------------------

// make_tracker (tracker.cpp:45-52). The tracker shares the model's bundle.
int wtref_tracker_create(wtref_model* m, const double* init_theta, wtref_tracker** out) {
  return guarded([&] {
    auto t = std::make_unique<wtref_tracker>();
    t->model = std::shared_ptr<wtref_model>(new wtref_model(*m));
    const int L = t->model->bundle.skeleton.joint_count();
    t->state = make_tracker(t->model->bundle, init_theta ? to_pose(init_theta, L) : Pose());
    *out = t.release();
  });
}

void wtref_tracker_free(wtref_tracker* t) { delete t; }

int wtref_tracker_get(const wtref_tracker* t, double* theta, double* phi, int* frame_index) {
  for (Eigen::Index k = 0; k < t->state.theta.size(); ++k) theta[k] = t->state.theta[k];
  if (phi) put_vec3s(t->state.mesh.phi, phi);
  if (frame_index) *frame_index = t->state.frame_index;
  return WT_OK;
}

int wtref_tracker_set(wtref_tracker* t, const double* theta, const double* phi, int frame_index) {
  const int L = t->model->bundle.skeleton.joint_count();
  t->state.theta = to_pose(theta, L);
  if (phi) t->state.mesh.phi = vec3s(phi, t->state.mesh.v0.size());
  t->state.frame_index = frame_index;
  return WT_OK;
}

namespace {
void put_kin_stats(const std::vector<KinIterStats>& in, wt_kin_iter_stats* out, int cap, int* n) {
  int k = 0;
  for (const auto& s : in) {
    if (out && k < cap) {
      out[k].iteration = s.iteration;
      out[k].associated = s.associated;
      out[k].residual_sum = s.residual_sum;
      out[k].step_norm = s.step_norm;
      out[k].solver_skipped = s.solver_skipped ? 1 : 0;
    }
    ++k;
  }
  if (n) *n = k;
}
void put_shape_stats(const std::vector<ShapeIterStats>& in, wt_shape_iter_stats* out, int cap,
                     int* n) {
  int k = 0;
  for (const auto& s : in) {
    if (out && k < cap) {
      out[k].iteration = s.iteration;
      out[k].singular = s.singular;
      out[k].mean_phi = s.mean_phi;
      out[k].max_phi = s.max_phi;
      out[k].mean_abs_r_before = s.mean_abs_r_before;
      out[k].mean_abs_r_after = s.mean_abs_r_after;
    }
    ++k;
  }
  if (n) *n = k;
}
}  // namespace

// track_frame (tracker.cpp:54-68) on an organized cloud.
int wtref_track_frame_cloud(wtref_tracker* t, const wt_intrinsics* intr, const double* points,
                            const uint8_t* valid, const wt_track_config* cfg, wt_frame_stats* st) {
  return guarded([&] {
    const Intrinsics in = to_intr(intr);
    const FrameStats fs = track_frame(t->state, to_cloud(in, points, valid), in, to_track(cfg));
    if (st) {
      st->frame = fs.frame;
      put_kin_stats(fs.kin, st->kin, st->cap_kin, &st->n_kin);
      put_shape_stats(fs.shape, st->shape, st->cap_shape, &st->n_shape);
    }
  });
}

// depth_to_cloud + track_frame: what run_tracking does per frame
// (tracker.cpp:80-81 via SequenceReader::read_frame, seqio.cpp:489-491).
int wtref_track_frame_depth(wtref_tracker* t, const wt_intrinsics* intr, const float* depth,
                            double scale, const wt_track_config* cfg, wt_frame_stats* st) {
  return guarded([&] {
    const Intrinsics in = to_intr(intr);
    const std::size_t n = static_cast<std::size_t>(in.width) * in.height;
    const CloudFrame cloud = depth_to_cloud(in, std::vector<float>(depth, depth + n), scale);
    const FrameStats fs = track_frame(t->state, cloud, in, to_track(cfg));
    if (st) {
      st->frame = fs.frame;
      put_kin_stats(fs.kin, st->kin, st->cap_kin, &st->n_kin);
      put_shape_stats(fs.shape, st->shape, st->cap_shape, &st->n_shape);
    }
  });
}

// optimize_pose (kinopt.cpp:132-171) on an organized cloud.
int wtref_optimize_pose(wtref_tracker* t, const wt_intrinsics* intr, const double* points,
                        const uint8_t* valid, const wt_kin_config* kin, const wt_assoc_config* assoc,
                        int threads, wt_kin_iter_stats* stats, int cap, int* n) {
  return guarded([&] {
    const Intrinsics in = to_intr(intr);
    std::vector<KinIterStats> st;
    optimize_pose(t->state, to_cloud(in, points, valid), in, to_kin(kin), to_assoc(assoc), threads,
                  &st);
    put_kin_stats(st, stats, cap, n);
  });
}

// optimize_shape (shapeopt.cpp:50-130); with_stats selects the stats path.
int wtref_optimize_shape(wtref_tracker* t, const wt_intrinsics* intr, const double* points,
                         const uint8_t* valid, const wt_shape_config* shape,
                         const wt_assoc_config* assoc, int threads, int with_stats,
                         wt_shape_iter_stats* stats, int cap, int* n) {
  return guarded([&] {
    const Intrinsics in = to_intr(intr);
    std::vector<ShapeIterStats> st;
    optimize_shape(t->state, to_cloud(in, points, valid), in, to_shape(shape), to_assoc(assoc),
                   threads, with_stats ? &st : nullptr);
    put_shape_stats(st, stats, cap, n);
  });
}

// ---- synthesis -----------------------------------------------------------------------

// synthesize_frame (synth.cpp:229-270): depth [H*W], joint_visible [L].
int wtref_render_depth(const wtref_model* m, const double* theta, const double* phi,
                       const wt_intrinsics* intr, const wt_noise* noise, int frame_index,
                       float* depth, uint8_t* joint_visible) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    NoiseSpec ns;
    ns.sigma = noise ? noise->sigma : 0.0;
    ns.dropout = noise ? noise->dropout : 0.0;
    ns.quantization = noise ? noise->quantization : 0.0;
    ns.seed = noise ? noise->seed : 0;
    const std::vector<Vec3> ph = phi ? vec3s(phi, m->bundle.mesh.v0.size()) : std::vector<Vec3>{};
    const FrameSynthesis fs = synthesize_frame(m->bundle, to_pose(theta, sk.joint_count()), ph,
                                               to_intr(intr), ns, frame_index);
    std::copy(fs.depth.begin(), fs.depth.end(), depth);
    if (joint_visible) std::copy(fs.joint_visible.begin(), fs.joint_visible.end(), joint_visible);
  });
}

// rasterize (synth.cpp:139-191) of the model posed at theta: depth (f64) and
// winning triangle per pixel.
int wtref_rasterize(const wtref_model* m, const double* theta, const double* phi,
                    const wt_intrinsics* intr, double* depth, int* tri) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    const auto off = link_offsets(sk, to_pose(theta, sk.joint_count()));
    const std::size_t nv = m->bundle.mesh.v0.size();
    const PosedMesh posed = phi ? skin(m->bundle.mesh, off, vec3s(phi, nv), 1)
                                : skin(m->bundle.mesh, off, 1);
    const RasterResult r = rasterize(posed.v, m->bundle.mesh.triangles, to_intr(intr));
    std::copy(r.depth.begin(), r.depth.end(), depth);
    std::copy(r.tri.begin(), r.tri.end(), tri);
  });
}

// ---- sequence files and the sequence driver ------------------------------------------

// SequenceWriter (seqio.cpp:493-535): n frames of H*W float depth.
int wtref_write_sequence(const char* path, const wt_intrinsics* intr, double depth_scale,
                         const float* frames, int n) {
  return guarded([&] {
    SequenceHeader h;
    h.width = static_cast<std::uint32_t>(intr->width);
    h.height = static_cast<std::uint32_t>(intr->height);
    h.fx = intr->fx;
    h.fy = intr->fy;
    h.cx = intr->cx;
    h.cy = intr->cy;
    h.frame_count = static_cast<std::uint32_t>(n);
    h.depth_scale = depth_scale;
    SequenceWriter w(path, h);
    const std::size_t px = static_cast<std::size_t>(intr->width) * intr->height;
    for (int f = 0; f < n; ++f)
      w.write_depth(std::vector<float>(frames + f * px, frames + (f + 1) * px));
    w.close();
  });
}

// SequenceReader::read_depth (seqio.cpp:476-487) of frame f; header out.
int wtref_read_depth(const char* path, int f, wt_intrinsics* intr, double* depth_scale, int* frame_count,
                     float* depth) {
  return guarded([&] {
    SequenceReader r(path);
    const SequenceHeader& h = r.header();
    if (intr) *intr = wt_intrinsics{h.fx, h.fy, h.cx, h.cy, static_cast<int>(h.width), static_cast<int>(h.height)};
    if (depth_scale) *depth_scale = h.depth_scale;
    if (frame_count) *frame_count = r.frame_count();
    if (depth) {
      const std::vector<float> d = r.read_depth(f);
      std::copy(d.begin(), d.end(), depth);
    }
  });
}

// run_tracking (tracker.cpp:70-100) over a .wts file: per-frame theta [F*L],
// joint origins [F*L*3], final phi [V*3].
int wtref_run_tracking(const wtref_model* m, const char* path, const wt_track_config* cfg,
                       const double* init_theta, double* theta_out, double* joints_out, double* phi_out) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    const TrackConfig tc = to_track(cfg);
    const ModelBundle tracked = tc.mode == TrackMode::rigid ? rigidify(m->bundle) : m->bundle;
    SequenceReader reader(path);
    const Pose init = init_theta ? to_pose(init_theta, sk.joint_count()) : sk.zero_pose();
    const TrackOutputs out = run_tracking(tracked, reader, tc, init);
    const int L = sk.link_count(), J = sk.joint_count();
    for (int f = 0; f < out.estimate.frame_count(); ++f) {
      for (int k = 0; k < J; ++k) theta_out[f * J + k] = out.estimate.theta[static_cast<std::size_t>(f)][k];
      for (int j = 0; j < L; ++j)
        for (int c = 0; c < 3; ++c)
          joints_out[(f * L + j) * 3 + c] =
              out.estimate.joints[static_cast<std::size_t>(f)][static_cast<std::size_t>(j)][c];
    }
    if (phi_out)
      for (std::size_t i = 0; i < out.final_phi.size(); ++i)
        for (int c = 0; c < 3; ++c) phi_out[i * 3 + c] = out.final_phi[i][c];
  });
}

// reconstruction_error_frame (metrics.cpp:110-142) of the model posed at
// (theta, phi) against an organized cloud: distances of the visible vertices
// in ascending vertex order, count in *n.
int wtref_recon_error(const wtref_model* m, const double* theta, const double* phi, const wt_intrinsics* intr,
                      const double* points, const uint8_t* valid, int threads, double* dist, int* n) {
  return guarded([&] {
    const Skeleton& sk = m->bundle.skeleton;
    const auto off = link_offsets(sk, to_pose(theta, sk.joint_count()));
    const std::size_t nv = m->bundle.mesh.v0.size();
    const PosedMesh posed = phi ? skin(m->bundle.mesh, off, vec3s(phi, nv), 1) : skin(m->bundle.mesh, off, 1);
    const Intrinsics in = to_intr(intr);
    const std::vector<double> d =
        reconstruction_error_frame(posed, m->bundle.mesh.triangles, to_cloud(in, points, valid), in, threads);
    std::copy(d.begin(), d.end(), dist);
    *n = static_cast<int>(d.size());
  });
}

}  // extern "C"

