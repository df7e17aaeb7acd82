/*
 * wt_oracle.c -- TEST INFRASTRUCTURE ONLY: a plain-C, fp64, single-threaded
 * restatement of the reference warptrack hot path (track_frame and
 * everything below it), used by tests/ and __graft_entry__.smoke() as the
 * checker for the CUDA path and by bench.py's CPU-baseline leg when the
 * reference itself (oracle/_ref) is not built. It is never linked into or
 * called by the product path.
 *
 * Every function cites the reference function it restates (file:line under
 * /root/reference/proj). The restatement is pinned against the reference's
 * own known-answer tests (tests/test_oracle_kat.py) and against the unmodified
 * reference built in oracle/_ref (tests/test_oracle_vs_ref.py, committed
 * fixtures in tests/golden/).
 *
 * Data layout: the model is the wt_model_desc of include/wt_gpu.h (the same
 * flat arrays the GPU context consumes); vectors are double[3], dual
 * quaternions double[8] in the canonical (w,x,y,z | w,x,y,z) layout.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "wt_gpu.h"

typedef struct { double r[4], d[4]; } dq_t;

/* ---- dual quaternions (dualquat.hpp:18-118, dualquat.cpp) ---------------- */

static void q_mul(const double* a, const double* b, double* o) { /* dualquat.hpp:29-34 */
  double w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  double x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  double y = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  double z = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
  o[0] = w; o[1] = x; o[2] = y; o[3] = z;
}
static void q_conj(const double* a, double* o) { o[0] = a[0]; o[1] = -a[1]; o[2] = -a[2]; o[3] = -a[3]; }
static double q_dot(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3]; }

static dq_t dq_ident(void) { dq_t h = {{1, 0, 0, 0}, {0, 0, 0, 0}}; return h; }
static dq_t dq_from(const double* v) { dq_t h; for (int c = 0; c < 4; ++c) { h.r[c] = v[c]; h.d[c] = v[4 + c]; } return h; }
static void dq_to(dq_t h, double* v) { for (int c = 0; c < 4; ++c) { v[c] = h.r[c]; v[4 + c] = h.d[c]; } }

static dq_t dq_compose(dq_t a, dq_t b) { /* dualquat.cpp:81-86: apply b, then a */
  dq_t o; double t1[4], t2[4];
  q_mul(a.r, b.r, o.r); q_mul(a.r, b.d, t1); q_mul(a.d, b.r, t2);
  for (int c = 0; c < 4; ++c) o.d[c] = t1[c] + t2[c];
  return o;
}
static dq_t dq_inv(dq_t h) { dq_t o; q_conj(h.r, o.r); q_conj(h.d, o.d); return o; } /* :110-112 */

static dq_t dq_joint(int kind, const double* ax, double th) { /* hinge/prismatic :65-79 */
  dq_t h = dq_ident();
  if (kind == WT_JOINT_HINGE) {
    double c = cos(th * 0.5), s = sin(th * 0.5);
    h.r[0] = c; h.r[1] = ax[0] * s; h.r[2] = ax[1] * s; h.r[3] = ax[2] * s;
  } else {
    h.d[1] = ax[0] * th * 0.5; h.d[2] = ax[1] * th * 0.5; h.d[3] = ax[2] * th * 0.5;
  }
  return h;
}
static dq_t dq_djoint(int kind, const double* ax, double th) { /* d_hinge/d_prismatic :183-195 */
  dq_t h; memset(&h, 0, sizeof h);
  if (kind == WT_JOINT_HINGE) {
    double c = 0.5 * cos(th * 0.5), s = -0.5 * sin(th * 0.5);
    h.r[0] = s; h.r[1] = ax[0] * c; h.r[2] = ax[1] * c; h.r[3] = ax[2] * c;
  } else {
    h.d[1] = ax[0] * 0.5; h.d[2] = ax[1] * 0.5; h.d[3] = ax[2] * 0.5;
  }
  return h;
}
static void dq_apply(dq_t h, const double* p, double* out) { /* transform_point :88-96 */
  const double* u = h.r + 1;
  double uxp[3] = {u[1] * p[2] - u[2] * p[1], u[2] * p[0] - u[0] * p[2], u[0] * p[1] - u[1] * p[0]};
  double uuxp[3] = {u[1] * uxp[2] - u[2] * uxp[1], u[2] * uxp[0] - u[0] * uxp[2], u[0] * uxp[1] - u[1] * uxp[0]};
  double rc[4], t[4];
  q_conj(h.r, rc); q_mul(h.d, rc, t);
  for (int c = 0; c < 3; ++c) out[c] = p[c] + 2.0 * (h.r[0] * uxp[c] + uuxp[c]) + 2.0 * t[1 + c];
}
static dq_t dq_normalize(dq_t h) { /* normalize :98-108 (caller checks |real| > 1e-12) */
  double n = sqrt(q_dot(h.r, h.r)), inv = 1.0 / n, s = q_dot(h.r, h.d);
  dq_t o;
  for (int c = 0; c < 4; ++c) { o.r[c] = h.r[c] * inv; o.d[c] = h.d[c] * inv - h.r[c] * (s * inv * inv * inv); }
  return o;
}
static void dq_rotation(dq_t h, double* m) { /* to_matrix :114-131 rotation block */
  double w = h.r[0], x = h.r[1], y = h.r[2], z = h.r[3];
  m[0] = 1 - 2 * (y * y + z * z); m[1] = 2 * (x * y - w * z); m[2] = 2 * (x * z + w * y);
  m[3] = 2 * (x * y + w * z); m[4] = 1 - 2 * (x * x + z * z); m[5] = 2 * (y * z - w * x);
  m[6] = 2 * (x * z - w * y); m[7] = 2 * (y * z + w * x); m[8] = 1 - 2 * (x * x + y * y);
}

/* d_normalized_transform (dualquat.cpp:197-223): the 3x8 Jacobian of
 * p(h) = vec(q u4 q* + 2 d q*) / |q|^2, restated element-wise with the
 * quaternion left/right product matrices L(p) v = p v, R(q) v = v q. */
static void left_mat(const double* p, double* m) {
  double v[16] = {p[0], -p[1], -p[2], -p[3], p[1], p[0], -p[3], p[2], p[2], p[3], p[0], -p[1], p[3], -p[2], p[1], p[0]};
  memcpy(m, v, sizeof v);
}
static void right_mat(const double* q, double* m) {
  double v[16] = {q[0], -q[1], -q[2], -q[3], q[1], q[0], q[3], -q[2], q[2], -q[3], q[0], q[1], q[3], q[2], -q[1], q[0]};
  memcpy(m, v, sizeof v);
}
static void mat4_mul(const double* a, const double* b, double* o) {
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) {
    double s = 0; for (int k = 0; k < 4; ++k) s += a[4 * i + k] * b[4 * k + j]; o[4 * i + j] = s;
  }
}
void wto_d_normalized_transform(const double* h8, const double* u, double* D /* 3x8 row-major */) {
  dq_t h = dq_from(h8);
  double n2 = q_dot(h.r, h.r), inv_n2 = 1.0 / n2;
  double u4[4] = {0, u[0], u[1], u[2]}, qc[4], a[4], g1[4], t[4];
  q_conj(h.r, qc); q_mul(u4, qc, a); q_mul(h.r, a, g1); q_mul(h.d, qc, t);
  double f[3]; for (int c = 0; c < 3; ++c) f[c] = (g1[1 + c] + 2.0 * t[1 + c]) * inv_n2;
  double C[16] = {1, 0, 0, 0, 0, -1, 0, 0, 0, 0, -1, 0, 0, 0, 0, -1};
  double Ra[16], Lq[16], Lu[16], Ld[16], Rqc[16], tmp[16], tmp2[16], dgq[16];
  right_mat(a, Ra); left_mat(h.r, Lq); left_mat(u4, Lu); left_mat(h.d, Ld); right_mat(qc, Rqc);
  mat4_mul(Lq, Lu, tmp); mat4_mul(tmp, C, tmp2);
  double LdC[16]; mat4_mul(Ld, C, LdC);
  for (int k = 0; k < 16; ++k) dgq[k] = Ra[k] + tmp2[k] + 2.0 * LdC[k];
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 4; ++j) {
    D[8 * i + j] = dgq[4 * (i + 1) + j] * inv_n2 - f[i] * (2.0 * inv_n2) * h.r[j];
    D[8 * i + 4 + j] = 2.0 * Rqc[4 * (i + 1) + j] * inv_n2;
  }
}

/* ---- skeleton (skeleton.cpp) -------------------------------------------------- */

typedef struct {
  int L, V, T, NP;
  const wt_model_desc* d;
  double bind_inv[64][8];
  int anc_off[65], anc[64 * 64], theta_to_link[64];
} model_t;

static void fk_all(const model_t* m, const double* th, dq_t* fk) { /* forward_kinematics :56-69 */
  const wt_model_desc* d = m->d;
  for (int j = 0; j < m->L; ++j) {
    dq_t local = dq_compose(dq_from(d->parent_offset + 8 * j), dq_joint(d->joint_kind[j], d->joint_axis + 3 * j, th[d->theta_index[j]]));
    fk[j] = d->parent[j] < 0 ? local : dq_compose(fk[d->parent[j]], local);
  }
}

static int model_init(model_t* m, const wt_model_desc* d) { /* Skeleton::build :7-50 (validation subset) */
  memset(m, 0, sizeof *m);
  m->d = d; m->L = d->n_links; m->V = d->n_vertices; m->T = d->n_triangles;
  if (m->L <= 0 || m->L > 64) return WT_EINVAL;
  int roots = 0;
  for (int j = 0; j < m->L; ++j) {
    if (d->parent[j] < 0) ++roots; else if (d->parent[j] >= j) return WT_EINVAL;
    m->theta_to_link[d->theta_index[j]] = j;
  }
  if (roots != 1) return WT_EINVAL;
  double zero[64] = {0};
  dq_t bind[64];
  fk_all(m, zero, bind);
  for (int j = 0; j < m->L; ++j) dq_to(dq_inv(bind[j]), m->bind_inv[j]);
  int k = 0;
  for (int j = 0; j < m->L; ++j) { /* ancestors: theta indices root -> j */
    int path[64], n = 0;
    for (int c = j; c >= 0; c = d->parent[c]) path[n++] = d->theta_index[c];
    m->anc_off[j] = k;
    for (int q = n - 1; q >= 0; --q) m->anc[k++] = path[q];
  }
  m->anc_off[m->L] = k;
  m->NP = k;
  return WT_OK;
}

static void link_offsets(const model_t* m, const dq_t* fk, dq_t* off) { /* :71-80 */
  for (int j = 0; j < m->L; ++j) off[j] = dq_compose(fk[j], dq_from(m->bind_inv[j]));
}

static dq_t d_link_offset(const model_t* m, const double* th, const dq_t* fk, int j, int k_theta) { /* :82-108 */
  const wt_model_desc* d = m->d;
  int kl = m->theta_to_link[k_theta];
  dq_t off = dq_from(d->parent_offset + 8 * kl);
  dq_t pre = d->parent[kl] < 0 ? off : dq_compose(fk[d->parent[kl]], off);
  dq_t dj = dq_djoint(d->joint_kind[kl], d->joint_axis + 3 * kl, th[k_theta]);
  dq_t k_to_j = dq_compose(dq_inv(fk[kl]), fk[j]);
  return dq_compose(dq_compose(pre, dj), dq_compose(k_to_j, dq_from(m->bind_inv[j])));
}

/* ---- skinning (skinmesh.cpp:60-141) ------------------------------------------------ */

typedef struct { dq_t raw, posed; double sign[4]; int ok; } blend_t;

static blend_t blend(const model_t* m, const dq_t* off, int i) { /* blend :60-77 */
  const wt_model_desc* d = m->d;
  blend_t b; memset(&b, 0, sizeof b);
  for (int s = 0; s < 4; ++s) b.sign[s] = 1.0;
  b.posed = dq_ident();
  int cnt = d->weight_count[i];
  if (cnt == 0) return b;
  const double* pivot = off[d->weight_link[4 * i]].r;
  for (int s = 0; s < cnt; ++s) {
    const dq_t* h = &off[d->weight_link[4 * i + s]];
    double sign = q_dot(pivot, h->r) < 0.0 ? -1.0 : 1.0;
    b.sign[s] = sign;
    double k = sign * d->weight[4 * i + s];
    for (int c = 0; c < 4; ++c) { b.raw.r[c] = b.raw.r[c] + h->r[c] * k; b.raw.d[c] = b.raw.d[c] + h->d[c] * k; }
  }
  if (sqrt(q_dot(b.raw.r, b.raw.r)) <= 1e-12) return b;
  b.posed = dq_normalize(b.raw);
  b.ok = 1;
  return b;
}

/* skin (skinmesh.cpp:104-141): v, n [V*3], valid [V]; phi [V*3]. */
static void skin(const model_t* m, const dq_t* off, const double* phi, double* v, double* n, uint8_t* valid) {
  const wt_model_desc* d = m->d;
  for (int i = 0; i < m->V; ++i) {
    blend_t b = blend(m, off, i);
    double rest[3];
    for (int c = 0; c < 3; ++c) rest[c] = d->v0[3 * i + c] + phi[3 * i + c];
    valid[i] = 1;
    if (b.ok) dq_apply(b.posed, rest, v + 3 * i);
    else { memcpy(v + 3 * i, rest, sizeof rest); valid[i] = 0; }
  }
  for (int i = 0; i < m->V; ++i) { /* area-weighted normals in CSR order :125-139 */
    double acc[3] = {0, 0, 0};
    for (int k = d->vtri_offsets[i]; k < d->vtri_offsets[i + 1]; ++k) {
      const int* f = d->triangles + 3 * d->vtri_items[k];
      const double *a = v + 3 * f[0], *bb = v + 3 * f[1], *cc = v + 3 * f[2];
      double e1[3] = {bb[0] - a[0], bb[1] - a[1], bb[2] - a[2]}, e2[3] = {cc[0] - a[0], cc[1] - a[1], cc[2] - a[2]};
      acc[0] += e1[1] * e2[2] - e1[2] * e2[1];
      acc[1] += e1[2] * e2[0] - e1[0] * e2[2];
      acc[2] += e1[0] * e2[1] - e1[1] * e2[0];
    }
    double len = sqrt(acc[0] * acc[0] + acc[1] * acc[1] + acc[2] * acc[2]);
    if (len > 1e-20) for (int c = 0; c < 3; ++c) n[3 * i + c] = acc[c] / len;
    else { n[3 * i] = n[3 * i + 1] = n[3 * i + 2] = 0.0; valid[i] = 0; }
  }
}

/* ---- association (association.cpp) ------------------------------------------- */

int wto_project(const wt_intrinsics* in, const double* p, int* u, int* v) { /* project :29-37 */
  if (p[2] <= 0.0) return 0;
  double uu = in->fx * p[0] / p[2] + in->cx, vv = in->fy * p[1] / p[2] + in->cy;
  double ru = round(uu), rv = round(vv); /* lround: half away from zero */
  if (ru < 0 || rv < 0 || ru >= in->width || rv >= in->height) return 0;
  *u = (int)ru; *v = (int)rv;
  return 1;
}

/* bucket_occupancy (association.cpp:39-67): offsets [P+1], items [<=V]. */
int wto_bucket_occupancy(const wt_intrinsics* in, int nv, const double* v, const double* n, const uint8_t* valid,
                         int* offsets, int* items) {
  int P = in->width * in->height;
  int* pix = (int*)malloc(sizeof(int) * (nv ? nv : 1));
  memset(offsets, 0, sizeof(int) * (P + 1));
  for (int i = 0; i < nv; ++i) {
    pix[i] = -1;
    if (!valid[i]) continue;
    const double* vi = v + 3 * i; const double* ni = n + 3 * i;
    if (ni[0] * vi[0] + ni[1] * vi[1] + ni[2] * vi[2] > 0.0) continue; /* back-facing */
    int pu, pv;
    if (!wto_project(in, vi, &pu, &pv)) continue;
    pix[i] = pv * in->width + pu;
    offsets[pix[i] + 1]++;
  }
  for (int p = 0; p < P; ++p) offsets[p + 1] += offsets[p];
  int* cur = (int*)malloc(sizeof(int) * (P ? P : 1));
  memcpy(cur, offsets, sizeof(int) * P);
  for (int i = 0; i < nv; ++i) if (pix[i] >= 0) items[cur[pix[i]]++] = i; /* ascending vertex index */
  int total = offsets[P];
  free(cur); free(pix);
  return total;
}

/* associate_winners (association.cpp:69-109) + associate (:111-138). */
void wto_associate(const wt_intrinsics* in, int nv, const double* v, const double* n, const uint8_t* valid,
                   const double* pts, const uint8_t* pvalid, int w, double cutoff, int* winners,
                   double* p_tilde, int* count, double* residual) {
  int W = in->width, H = in->height, P = W * H;
  int* off = (int*)malloc(sizeof(int) * (P + 1));
  int* items = (int*)malloc(sizeof(int) * (nv ? nv : 1));
  wto_bucket_occupancy(in, nv, v, n, valid, off, items);
  double cut2 = cutoff * cutoff;
  int* win = winners ? winners : (int*)malloc(sizeof(int) * P);
  for (int pi = 0; pi < P; ++pi) {
    win[pi] = -1;
    if (!pvalid[pi]) continue;
    const double* p = pts + 3 * pi;
    int pu = pi % W, pv = pi / W, best = -1;
    double best_sq = INFINITY;
    int u0 = pu - w < 0 ? 0 : pu - w, u1 = pu + w > W - 1 ? W - 1 : pu + w;
    int v0 = pv - w < 0 ? 0 : pv - w, v1 = pv + w > H - 1 ? H - 1 : pv + w;
    for (int r = v0; r <= v1; ++r)
      for (int s = off[r * W + u0]; s < off[r * W + u1 + 1]; ++s) { /* one span per window row */
        int vi = items[s];
        const double* q = v + 3 * vi;
        double dx = q[0] - p[0], dy = q[1] - p[1], dz = q[2] - p[2];
        double d = dx * dx + dy * dy + dz * dz;
        if (d > cut2) continue;
        if (d < best_sq || (d == best_sq && vi < best)) { best_sq = d; best = vi; }
      }
    win[pi] = best;
  }
  for (int i = 0; i < nv; ++i) { count[i] = 0; residual[i] = 0; p_tilde[3 * i] = p_tilde[3 * i + 1] = p_tilde[3 * i + 2] = 0; }
  for (int pi = 0; pi < P; ++pi) { /* sums in ascending observation order */
    int wv = win[pi];
    if (wv < 0) continue;
    for (int c = 0; c < 3; ++c) p_tilde[3 * wv + c] += pts[3 * pi + c];
    count[wv]++;
  }
  for (int i = 0; i < nv; ++i) {
    if (!count[i]) continue;
    for (int c = 0; c < 3; ++c) p_tilde[3 * i + c] /= (double)count[i];
    residual[i] = n[3 * i] * (p_tilde[3 * i] - v[3 * i]) + n[3 * i + 1] * (p_tilde[3 * i + 1] - v[3 * i + 1]) +
                  n[3 * i + 2] * (p_tilde[3 * i + 2] - v[3 * i + 2]);
  }
  if (!winners) free(win);
  free(off); free(items);
}

/* depth_to_cloud (seqio.cpp:419-437). */
void wto_depth_to_cloud(const wt_intrinsics* in, const float* depth, double scale, double* pts, uint8_t* valid) {
  for (int v = 0; v < in->height; ++v)
    for (int u = 0; u < in->width; ++u) {
      int i = v * in->width + u;
      float d = depth[i];
      pts[3 * i] = pts[3 * i + 1] = pts[3 * i + 2] = 0.0;
      valid[i] = 0;
      if (!(d > 0.0f) || !isfinite(d)) continue;
      double z = (double)d * scale;
      pts[3 * i] = (u - in->cx) / in->fx * z;
      pts[3 * i + 1] = (v - in->cy) / in->fy * z;
      pts[3 * i + 2] = z;
      valid[i] = 1;
    }
}

/* ---- pose system (kinopt.cpp) ------------------------------------------------------ */

static void influence_counts(const model_t* m, double* S) { /* influence_counts :58-70 */
  const wt_model_desc* d = m->d;
  for (int k = 0; k < m->L; ++k) S[k] = 0;
  for (int i = 0; i < m->V; ++i) {
    char hit[64] = {0};
    for (int e = 0; e < d->weight_count[i]; ++e) {
      int l = d->weight_link[4 * i + e];
      for (int q = m->anc_off[l]; q < m->anc_off[l + 1]; ++q) hit[m->anc[q]] = 1;
    }
    for (int k = 0; k < m->L; ++k) if (hit[k]) S[k] += 1.0;
  }
}

/* fill_row (kinopt.cpp:29-47); dchain [NP][8] indexed like anc[]. */
static int fill_row(const model_t* m, const dq_t* off, const double* dch, const double* phi, const double* n,
                    const uint8_t* valid, int i, double* row) {
  const wt_model_desc* d = m->d;
  for (int k = 0; k < m->L; ++k) row[k] = 0.0;
  if (!valid[i]) return 0;
  blend_t b = blend(m, off, i);
  if (!b.ok) return 0;
  double rest[3], D[24], r8[8], raw8[8];
  for (int c = 0; c < 3; ++c) rest[c] = d->v0[3 * i + c] + phi[3 * i + c];
  dq_to(b.raw, raw8);
  wto_d_normalized_transform(raw8, rest, D);
  for (int j = 0; j < 8; ++j) r8[j] = -(n[3 * i] * D[j] + n[3 * i + 1] * D[8 + j] + n[3 * i + 2] * D[16 + j]);
  for (int s = 0; s < d->weight_count[i]; ++s) {
    double coeff = d->weight[4 * i + s] * b.sign[s];
    int l = d->weight_link[4 * i + s];
    for (int q = m->anc_off[l]; q < m->anc_off[l + 1]; ++q) {
      double dot = 0; for (int c = 0; c < 8; ++c) dot += r8[c] * dch[8 * q + c];
      row[m->anc[q]] += coeff * dot;
    }
  }
  return 1;
}

static void pose_derivatives(const model_t* m, const double* th, dq_t* fk, dq_t* off, double* dch) { /* :11-23 */
  fk_all(m, th, fk);
  link_offsets(m, fk, off);
  for (int j = 0; j < m->L; ++j)
    for (int q = m->anc_off[j]; q < m->anc_off[j + 1]; ++q) dq_to(d_link_offset(m, th, fk, j, m->anc[q]), dch + 8 * q);
}

/* accumulate_normal_system (kinopt.cpp:72-119) in vertex order + prior. */
static void normal_system(const model_t* m, const dq_t* off, const double* dch, const double* phi, const double* n,
                          const uint8_t* valid, const int* count, const double* res, const double* S,
                          const double* th, double lambda_s, double* jtj, double* jtr) {
  int L = m->L;
  double row[64];
  memset(jtj, 0, sizeof(double) * L * L); memset(jtr, 0, sizeof(double) * L);
  for (int i = 0; i < m->V; ++i) {
    if (!count[i]) continue;
    if (!fill_row(m, off, dch, phi, n, valid, i, row)) continue;
    for (int a = 0; a < L; ++a) {
      if (row[a] == 0.0) continue;
      jtr[a] += row[a] * res[i];
      for (int b2 = 0; b2 < L; ++b2) if (row[b2] != 0.0) jtj[a * L + b2] += row[a] * row[b2];
    }
  }
  for (int k = 0; k < L; ++k) { double p = lambda_s * S[k]; jtj[k * L + k] += p * p; jtr[k] += p * p * th[k]; }
}

/* solve_step (kinopt.cpp:121-130): LLT failing at the first pivot <= 0. */
int wto_solve_step(int L, const double* jtj, const double* jtr, double lambda_k, double floor_, double* x) {
  double* a = (double*)malloc(sizeof(double) * L * L);
  for (int e = 0; e < L * L; ++e) a[e] = jtj[e];
  for (int k = 0; k < L; ++k) a[k * L + k] = jtj[k * L + k] + lambda_k * jtj[k * L + k] + floor_;
  for (int e = 0; e < L * L; ++e) if (!isfinite(a[e])) { free(a); return WT_ENOTPD; }
  for (int k = 0; k < L; ++k) if (!isfinite(jtr[k])) { free(a); return WT_ENOTPD; }
  for (int k = 0; k < L; ++k) {
    double s = a[k * L + k];
    for (int j = 0; j < k; ++j) s -= a[k * L + j] * a[k * L + j];
    if (!(s > 0.0)) { free(a); return WT_ENOTPD; }
    s = sqrt(s); a[k * L + k] = s;
    for (int i = k + 1; i < L; ++i) {
      double t = a[i * L + k];
      for (int j = 0; j < k; ++j) t -= a[i * L + j] * a[k * L + j];
      a[i * L + k] = t / s;
    }
  }
  for (int i = 0; i < L; ++i) { double s = jtr[i]; for (int j = 0; j < i; ++j) s -= a[i * L + j] * x[j]; x[i] = s / a[i * L + i]; }
  for (int i = L - 1; i >= 0; --i) { double s = x[i]; for (int j = i + 1; j < L; ++j) s -= a[j * L + i] * x[j]; x[i] = s / a[i * L + i]; }
  free(a);
  return WT_OK;
}

/* solve_vertex (shapeopt.cpp:25-48). Returns 1 when singular. */
int wto_solve_vertex(const double* g, double r, const double* phi, const double* nd, int ncount,
                     const wt_shape_config* c, double* delta) {
  double A[9];
  for (int x = 0; x < 3; ++x) for (int y = 0; y < 3; ++y) A[3 * x + y] = g[x] * g[y];
  double reg = c->lambda_phi + c->lambda_nbr * ncount;
  for (int k = 0; k < 3; ++k) { A[4 * k] += reg; A[4 * k] += c->lambda_w * A[4 * k]; A[4 * k] += c->diag_floor; }
  double b[3];
  for (int k = 0; k < 3; ++k) b[k] = g[k] * r + c->lambda_phi * phi[k] + c->lambda_nbr * nd[k];
  delta[0] = delta[1] = delta[2] = 0.0;
  for (int k = 0; k < 9; ++k) if (!isfinite(A[k])) return 1;
  for (int k = 0; k < 3; ++k) if (!isfinite(b[k])) return 1;
  double Lm[9] = {0};
  for (int k = 0; k < 3; ++k) {
    double s = A[4 * k];
    for (int j = 0; j < k; ++j) s -= Lm[3 * k + j] * Lm[3 * k + j];
    if (!(s > 0.0)) return 1;
    Lm[4 * k] = sqrt(s);
    for (int i = k + 1; i < 3; ++i) {
      double t = A[3 * i + k];
      for (int j = 0; j < k; ++j) t -= Lm[3 * i + j] * Lm[3 * k + j];
      Lm[3 * i + k] = t / Lm[4 * k];
    }
  }
  double y[3];
  for (int i = 0; i < 3; ++i) { double s = b[i]; for (int j = 0; j < i; ++j) s -= Lm[3 * i + j] * y[j]; y[i] = s / Lm[4 * i]; }
  for (int i = 2; i >= 0; --i) { double s = y[i]; for (int j = i + 1; j < 3; ++j) s -= Lm[3 * j + i] * delta[j]; delta[i] = s / Lm[4 * i]; }
  return 0;
}

/* ---- tracker (kinopt.cpp:132-171, shapeopt.cpp:50-130, tracker.cpp:54-68) ---- */

typedef struct wto_tracker {
  model_t m;
  wt_intrinsics in;
  double theta[64];
  double* phi;
  int frame_index;
  /* scratch */
  double *v, *n, *pts, *p_tilde, *res, *S, *dch;
  uint8_t *valid, *pvalid;
  int *count;
} wto_tracker;

int wto_create(const wt_model_desc* d, const wt_intrinsics* in, wto_tracker** out) {
  wto_tracker* t = (wto_tracker*)calloc(1, sizeof *t);
  if (model_init(&t->m, d) != WT_OK) { free(t); return WT_EINVAL; }
  t->in = *in;
  int V = d->n_vertices, P = in->width * in->height;
  t->phi = (double*)calloc((size_t)3 * V + 3, sizeof(double));
  if (d->phi) memcpy(t->phi, d->phi, sizeof(double) * 3 * V);
  t->v = (double*)calloc((size_t)3 * V + 3, sizeof(double));
  t->n = (double*)calloc((size_t)3 * V + 3, sizeof(double));
  t->p_tilde = (double*)calloc((size_t)3 * V + 3, sizeof(double));
  t->res = (double*)calloc((size_t)V + 1, sizeof(double));
  t->count = (int*)calloc((size_t)V + 1, sizeof(int));
  t->valid = (uint8_t*)calloc((size_t)V + 1, 1);
  t->pts = (double*)calloc((size_t)3 * P, sizeof(double));
  t->pvalid = (uint8_t*)calloc((size_t)P, 1);
  t->S = (double*)calloc(64, sizeof(double));
  t->dch = (double*)calloc((size_t)8 * (t->m.NP + 1), sizeof(double));
  influence_counts(&t->m, t->S);
  *out = t;
  return WT_OK;
}

void wto_destroy(wto_tracker* t) {
  if (!t) return;
  free(t->phi); free(t->v); free(t->n); free(t->p_tilde); free(t->res); free(t->count); free(t->valid);
  free(t->pts); free(t->pvalid); free(t->S); free(t->dch); free(t);
}

void wto_set_state(wto_tracker* t, const double* theta, const double* phi, int frame_index) {
  if (theta) memcpy(t->theta, theta, sizeof(double) * t->m.L);
  if (phi) memcpy(t->phi, phi, sizeof(double) * 3 * t->m.V);
  t->frame_index = frame_index;
}

void wto_get_state(const wto_tracker* t, double* theta, double* phi, int* frame_index) {
  if (theta) memcpy(theta, t->theta, sizeof(double) * t->m.L);
  if (phi) memcpy(phi, t->phi, sizeof(double) * 3 * t->m.V);
  if (frame_index) *frame_index = t->frame_index;
}

void wto_load_depth(wto_tracker* t, const float* depth, double scale) { wto_depth_to_cloud(&t->in, depth, scale, t->pts, t->pvalid); }
void wto_load_cloud(wto_tracker* t, const double* pts, const uint8_t* valid) {
  int P = t->in.width * t->in.height;
  memcpy(t->pts, pts, sizeof(double) * 3 * P); memcpy(t->pvalid, valid, (size_t)P);
}

/* skin at theta with phi (NULL = state phi): skin_mesh binding (bindings.cpp:185-201). */
void wto_skin(wto_tracker* t, const double* theta, const double* phi, double* v, double* n, uint8_t* valid) {
  dq_t fk[64], off[64];
  fk_all(&t->m, theta, fk); link_offsets(&t->m, fk, off);
  skin(&t->m, off, phi ? phi : t->phi, v, n, valid);
}

static void associate_state(wto_tracker* t, const wt_assoc_config* a, int* winners) {
  wto_associate(&t->in, t->m.V, t->v, t->n, t->valid, t->pts, t->pvalid, a->window_radius, a->cutoff, winners,
                t->p_tilde, t->count, t->res);
}

/* optimize_pose (kinopt.cpp:132-171). */
int wto_optimize_pose(wto_tracker* t, const wt_kin_config* k, const wt_assoc_config* a, wt_kin_iter_stats* st) {
  model_t* m = &t->m;
  int L = m->L, refresh = k->assoc_refresh > 1 ? k->assoc_refresh : 1;
  dq_t fk[64], off[64];
  double jtj[64 * 64], jtr[64], x[64];
  for (int it = 0; it < k->iterations; ++it) {
    pose_derivatives(m, t->theta, fk, off, t->dch);
    skin(m, off, t->phi, t->v, t->n, t->valid);
    if (it % refresh == 0) associate_state(t, a, NULL);
    else
      for (int i = 0; i < m->V; ++i)
        if (t->count[i] > 0)
          t->res[i] = t->n[3 * i] * (t->p_tilde[3 * i] - t->v[3 * i]) + t->n[3 * i + 1] * (t->p_tilde[3 * i + 1] - t->v[3 * i + 1]) +
                      t->n[3 * i + 2] * (t->p_tilde[3 * i + 2] - t->v[3 * i + 2]);
    double rsum = 0; int assoc = 0;
    for (int i = 0; i < m->V; ++i) if (t->count[i] > 0) { rsum += t->res[i] * t->res[i]; ++assoc; }
    normal_system(m, off, t->dch, t->phi, t->n, t->valid, t->count, t->res, t->S, t->theta, k->lambda_s, jtj, jtr);
    int rc = wto_solve_step(L, jtj, jtr, k->lambda_k, k->diag_floor, x);
    double nrm = 0;
    if (rc == WT_OK) {
      for (int q = 0; q < L; ++q) {
        t->theta[q] -= x[q];
        if (k->clamp_limits && k->limit > 0.0) t->theta[q] = fmin(fmax(t->theta[q], -k->limit), k->limit);
        nrm += x[q] * x[q];
      }
    }
    if (st) {
      st[it].iteration = it; st[it].associated = assoc; st[it].residual_sum = rsum;
      st[it].step_norm = rc == WT_OK ? sqrt(nrm) : 0.0; st[it].solver_skipped = rc != WT_OK;
    }
  }
  return WT_OK;
}

static double mean_abs_r(const wto_tracker* t) {
  double s = 0; int n = 0;
  for (int i = 0; i < t->m.V; ++i) if (t->count[i] > 0) { s += fabs(t->res[i]); ++n; }
  return n ? s / n : 0.0;
}

/* optimize_shape (shapeopt.cpp:50-130), with the closing stats pass. */
int wto_optimize_shape(wto_tracker* t, const wt_shape_config* c, const wt_assoc_config* a, int with_stats,
                       wt_shape_iter_stats* st) {
  model_t* m = &t->m;
  const wt_model_desc* d = m->d;
  int V = m->V;
  dq_t fk[64], off[64];
  double* next = (double*)malloc(sizeof(double) * 3 * (V + 1));
  fk_all(m, t->theta, fk); link_offsets(m, fk, off);
  for (int it = 0; it < c->iterations; ++it) {
    skin(m, off, t->phi, t->v, t->n, t->valid);
    associate_state(t, a, NULL);
    double before = mean_abs_r(t);
    int singular = 0;
    for (int i = 0; i < V; ++i) {
      double nd[3] = {0, 0, 0}, g[3] = {0, 0, 0}, r = 0, delta[3];
      int nc = d->nbr_offsets[i + 1] - d->nbr_offsets[i];
      for (int q = d->nbr_offsets[i]; q < d->nbr_offsets[i + 1]; ++q)
        for (int k = 0; k < 3; ++k) nd[k] += t->phi[3 * i + k] - t->phi[3 * d->nbr_items[q] + k];
      if (t->count[i] > 0 && t->valid[i]) {
        blend_t b = blend(m, off, i);
        if (b.ok) {
          double R[9];
          dq_rotation(dq_normalize(b.raw), R);
          for (int k = 0; k < 3; ++k) g[k] = -(R[k] * t->n[3 * i] + R[3 + k] * t->n[3 * i + 1] + R[6 + k] * t->n[3 * i + 2]);
          r = t->res[i];
        }
      }
      singular += wto_solve_vertex(g, r, t->phi + 3 * i, nd, nc, c, delta);
      for (int k = 0; k < 3; ++k) next[3 * i + k] = t->phi[3 * i + k] - delta[k];
    }
    memcpy(t->phi, next, sizeof(double) * 3 * V); /* Jacobi swap */
    if (st) {
      double sum = 0, mx = 0;
      for (int i = 0; i < V; ++i) {
        double l = sqrt(t->phi[3 * i] * t->phi[3 * i] + t->phi[3 * i + 1] * t->phi[3 * i + 1] + t->phi[3 * i + 2] * t->phi[3 * i + 2]);
        sum += l; if (l > mx) mx = l;
      }
      st[it].iteration = it; st[it].singular = singular; st[it].mean_phi = V ? sum / V : 0.0; st[it].max_phi = mx;
      st[it].mean_abs_r_before = before; st[it].mean_abs_r_after = 0.0;
    }
  }
  if (with_stats && st && c->iterations > 0) {
    skin(m, off, t->phi, t->v, t->n, t->valid);
    associate_state(t, a, NULL);
    for (int s = 0; s + 1 < c->iterations; ++s) st[s].mean_abs_r_after = st[s + 1].mean_abs_r_before;
    st[c->iterations - 1].mean_abs_r_after = mean_abs_r(t);
  }
  free(next);
  return WT_OK;
}

/* track_frame (tracker.cpp:54-68) on the loaded frame. */
int wto_track_loaded(wto_tracker* t, const wt_track_config* cfg, wt_frame_stats* st) {
  wt_kin_iter_stats kin[64];
  wt_shape_iter_stats shp[64];
  wto_optimize_pose(t, &cfg->kin, &cfg->assoc, kin);
  int shape_now = cfg->mode == WT_MODE_DYNAMIC || (cfg->mode == WT_MODE_SHAPE_MATCH && t->frame_index == 0);
  if (shape_now) wto_optimize_shape(t, &cfg->shape, &cfg->assoc, 1, shp);
  if (st) {
    st->frame = t->frame_index;
    st->n_kin = cfg->kin.iterations;
    st->n_shape = shape_now ? cfg->shape.iterations : 0;
    for (int k = 0; k < st->n_kin && k < st->cap_kin && st->kin; ++k) st->kin[k] = kin[k];
    for (int k = 0; k < st->n_shape && k < st->cap_shape && st->shape; ++k) st->shape[k] = shp[k];
  }
  ++t->frame_index;
  return WT_OK;
}

/* accumulate_normal_system at theta for an explicit (count, residual). */
int wto_normal_system(wto_tracker* t, const double* theta, const wt_kin_config* k, const int* count,
                      const double* res, double* jtj, double* jtr) {
  dq_t fk[64], off[64];
  pose_derivatives(&t->m, theta, fk, off, t->dch);
  skin(&t->m, off, t->phi, t->v, t->n, t->valid);
  normal_system(&t->m, off, t->dch, t->phi, t->n, t->valid, count, res, t->S, theta, k->lambda_s, jtj, jtr);
  return WT_OK;
}

/* fk / link offsets / dense dchain [L*L*8] at theta (for parity checks). */
void wto_pose_derivatives(wto_tracker* t, const double* theta, double* fk8, double* off8, double* dchain) {
  dq_t fk[64], off[64];
  pose_derivatives(&t->m, theta, fk, off, t->dch);
  int L = t->m.L;
  for (int j = 0; j < L; ++j) { if (fk8) dq_to(fk[j], fk8 + 8 * j); if (off8) dq_to(off[j], off8 + 8 * j); }
  if (dchain) {
    memset(dchain, 0, sizeof(double) * L * L * 8);
    for (int j = 0; j < L; ++j)
      for (int q = t->m.anc_off[j]; q < t->m.anc_off[j + 1]; ++q)
        memcpy(dchain + ((size_t)j * L + t->m.anc[q]) * 8, t->dch + 8 * q, sizeof(double) * 8);
  }
}
