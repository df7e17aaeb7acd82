// wt_dq.cuh -- dual-quaternion algebra, forward kinematics and pose
// derivatives in fp64, shared by host (context setup) and device (the
// per-frame FK/dchain step fused into the pose-solve tail).
//
// Layout: canonical 8-vector (real.w, real.x, real.y, real.z, dual.w,
// dual.x, dual.y, dual.z), proj/include/warptrack/dualquat.hpp:104-107.
#pragma once

#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define WT_HD __host__ __device__ __forceinline__
#else
#define WT_HD inline
#endif

namespace wt {

struct DQ {
  double r[4];
  double d[4];
};

// Hamilton product, dualquat.hpp:29-34.
WT_HD void qmul(const double* a, const double* b, double* o) {
  const double w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  const double x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  const double y = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  const double z = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
  o[0] = w;
  o[1] = x;
  o[2] = y;
  o[3] = z;
}

WT_HD void qconj(const double* a, double* o) {
  o[0] = a[0];
  o[1] = -a[1];
  o[2] = -a[2];
  o[3] = -a[3];
}

WT_HD DQ dq_identity() {
  DQ h;
  h.r[0] = 1.0;
  h.r[1] = h.r[2] = h.r[3] = 0.0;
  h.d[0] = h.d[1] = h.d[2] = h.d[3] = 0.0;
  return h;
}

WT_HD DQ dq_load(const double* v) {
  DQ h;
  for (int c = 0; c < 4; ++c) {
    h.r[c] = v[c];
    h.d[c] = v[4 + c];
  }
  return h;
}

WT_HD void dq_store(const DQ& h, double* v) {
  for (int c = 0; c < 4; ++c) {
    v[c] = h.r[c];
    v[4 + c] = h.d[c];
  }
}

// compose(a, b): apply b, then a (dualquat.cpp:81-86). Bilinear.
WT_HD DQ dq_compose(const DQ& a, const DQ& b) {
  DQ o;
  double t1[4], t2[4];
  qmul(a.r, b.r, o.r);
  qmul(a.r, b.d, t1);
  qmul(a.d, b.r, t2);
  for (int c = 0; c < 4; ++c) o.d[c] = t1[c] + t2[c];
  return o;
}

// inverse of a unit DQ (dualquat.cpp:110-112).
WT_HD DQ dq_inverse(const DQ& h) {
  DQ o;
  qconj(h.r, o.r);
  qconj(h.d, o.d);
  return o;
}

// hinge / prismatic joint transforms (dualquat.cpp:65-79).
WT_HD DQ dq_joint(int kind, const double* axis, double theta) {
  DQ h = dq_identity();
  if (kind == 0) {
    const double c = cos(theta * 0.5);
    const double s = sin(theta * 0.5);
    h.r[0] = c;
    h.r[1] = axis[0] * s;
    h.r[2] = axis[1] * s;
    h.r[3] = axis[2] * s;
  } else {
    h.d[1] = axis[0] * theta * 0.5;
    h.d[2] = axis[1] * theta * 0.5;
    h.d[3] = axis[2] * theta * 0.5;
  }
  return h;
}

// d_hinge / d_prismatic (dualquat.cpp:183-195).
WT_HD DQ dq_djoint(int kind, const double* axis, double theta) {
  DQ h;
  for (int c = 0; c < 4; ++c) h.r[c] = h.d[c] = 0.0;
  if (kind == 0) {
    const double c = 0.5 * cos(theta * 0.5);
    const double s = -0.5 * sin(theta * 0.5);
    h.r[0] = s;
    h.r[1] = axis[0] * c;
    h.r[2] = axis[1] * c;
    h.r[3] = axis[2] * c;
  } else {
    h.d[1] = axis[0] * 0.5;
    h.d[2] = axis[1] * 0.5;
    h.d[3] = axis[2] * 0.5;
  }
  return h;
}

// Joint transform / derivative from the precomputed half-angle cos/sin
// (c, s) = (cos(theta/2), sin(theta/2)); theta itself for prismatic joints.
WT_HD DQ dq_joint_cs(int kind, const double* axis, double theta, double c, double s) {
  DQ h = dq_identity();
  if (kind == 0) {
    h.r[0] = c;
    h.r[1] = axis[0] * s;
    h.r[2] = axis[1] * s;
    h.r[3] = axis[2] * s;
  } else {
    h.d[1] = axis[0] * theta * 0.5;
    h.d[2] = axis[1] * theta * 0.5;
    h.d[3] = axis[2] * theta * 0.5;
  }
  return h;
}

WT_HD DQ dq_djoint_cs(int kind, const double* axis, double c, double s) {
  DQ h;
  for (int k = 0; k < 4; ++k) h.r[k] = h.d[k] = 0.0;
  if (kind == 0) {
    h.r[0] = -0.5 * s;
    h.r[1] = axis[0] * (0.5 * c);
    h.r[2] = axis[1] * (0.5 * c);
    h.r[3] = axis[2] * (0.5 * c);
  } else {
    h.d[1] = axis[0] * 0.5;
    h.d[2] = axis[1] * 0.5;
    h.d[3] = axis[2] * 0.5;
  }
  return h;
}

// Rigid action of a unit DQ on a point (dualquat.cpp:88-96).
WT_HD void dq_transform_point(const DQ& h, const double* p, double* out) {
  const double ux = h.r[1], uy = h.r[2], uz = h.r[3], w = h.r[0];
  const double cx = uy * p[2] - uz * p[1];
  const double cy = uz * p[0] - ux * p[2];
  const double cz = ux * p[1] - uy * p[0];
  const double ccx = uy * cz - uz * cy;
  const double ccy = uz * cx - ux * cz;
  const double ccz = ux * cy - uy * cx;
  double rc[4], t[4];
  qconj(h.r, rc);
  qmul(h.d, rc, t);
  out[0] = p[0] + 2.0 * (w * cx + ccx) + 2.0 * t[1];
  out[1] = p[1] + 2.0 * (w * cy + ccy) + 2.0 * t[2];
  out[2] = p[2] + 2.0 * (w * cz + ccz) + 2.0 * t[3];
}

// normalize (dualquat.cpp:98-108); caller checks |real| > 1e-12.
WT_HD DQ dq_normalize(const DQ& h) {
  const double n = sqrt(h.r[0] * h.r[0] + h.r[1] * h.r[1] + h.r[2] * h.r[2] + h.r[3] * h.r[3]);
  const double inv = 1.0 / n;
  const double s = h.r[0] * h.d[0] + h.r[1] * h.d[1] + h.r[2] * h.d[2] + h.r[3] * h.d[3];
  DQ o;
  for (int c = 0; c < 4; ++c) {
    o.r[c] = h.r[c] * inv;
    o.d[c] = h.d[c] * inv - h.r[c] * (s * inv * inv * inv);
  }
  return o;
}

// Rotation block of a unit DQ (to_matrix, dualquat.cpp:114-131), row-major.
WT_HD void dq_rotation(const DQ& h, double* m) {
  const double w = h.r[0], x = h.r[1], y = h.r[2], z = h.r[3];
  m[0] = 1 - 2 * (y * y + z * z);
  m[1] = 2 * (x * y - w * z);
  m[2] = 2 * (x * z + w * y);
  m[3] = 2 * (x * y + w * z);
  m[4] = 1 - 2 * (x * x + z * z);
  m[5] = 2 * (y * z - w * x);
  m[6] = 2 * (x * z - w * y);
  m[7] = 2 * (y * z + w * x);
  m[8] = 1 - 2 * (x * x + y * y);
}

// r8 = -n^T * d_normalized_transform(h, u): the 1x8 row of dr/dH for a
// point-plane residual r = n.(p~ - v(H)) (kinopt.cpp:36-38 with
// dualquat.cpp:197-223). With L(p)vec(q) = vec(p q), R(q)vec(p) = vec(p q),
// C = diag(1,-1,-1,-1), n4 = (0, n), a = u4 conj(q):
//   n4^T R(a)           = vec(n4 conj(a))^T
//   n4^T L(q) L(u4) C   = (C vec(conj(u4) (conj(q) n4)))^T
//   n4^T 2 L(d) C       = 2 (C vec(conj(d) n4))^T
//   n4^T 2 R(conj q)    = 2 vec(n4 q)^T
// so the whole 3x8 Jacobian never has to be materialised.
WT_HD void dq_point_plane_row(const DQ& h, const double* u, const double* n, double* r8) {
  const double* q = h.r;
  const double n2 = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
  const double inv_n2 = 1.0 / n2;
  const double u4[4] = {0.0, u[0], u[1], u[2]};
  const double n4[4] = {0.0, n[0], n[1], n[2]};
  double qc[4], a[4], g[4], t[4], dc[4];
  qconj(q, qc);
  qmul(u4, qc, a);      // a = u4 conj(q)
  qmul(q, a, g);        // q a
  qmul(h.d, qc, t);     // d conj(q)
  const double fx = (g[1] + 2.0 * t[1]) * inv_n2;
  const double fy = (g[2] + 2.0 * t[2]) * inv_n2;
  const double fz = (g[3] + 2.0 * t[3]) * inv_n2;
  const double nf = n[0] * fx + n[1] * fy + n[2] * fz;

  double ac[4], t1[4], t2[4], t3[4], u4c[4];
  qconj(a, ac);
  qmul(n4, ac, t1);     // n4 conj(a)
  double qn[4];
  qmul(qc, n4, qn);     // conj(q) n4
  qconj(u4, u4c);
  qmul(u4c, qn, t2);    // conj(u4) conj(q) n4
  qconj(h.d, dc);
  qmul(dc, n4, t3);     // conj(d) n4
  // C = diag(1,-1,-1,-1) applied to t2 and t3.
  const double cs[4] = {1.0, -1.0, -1.0, -1.0};
  for (int c = 0; c < 4; ++c) {
    const double dg = t1[c] + cs[c] * t2[c] + 2.0 * cs[c] * t3[c];
    r8[c] = -(dg * inv_n2 - nf * 2.0 * inv_n2 * q[c]);
  }
  double t4[4];
  qmul(n4, q, t4);      // n4 q
  for (int c = 0; c < 4; ++c) r8[4 + c] = -(2.0 * t4[c] * inv_n2);
}

// ---- skeleton ------------------------------------------------------------

struct LinkDesc {
  int parent;
  int kind;
  int theta_index;
  int pad;
  double axis[3];
  double offset[8];
  double bind_inv[8];  // inverse(bind_pose[j])
};

// forward_kinematics (skeleton.cpp:56-69) for links in topological order.
WT_HD void fk_all(const LinkDesc* links, int L, const double* theta, DQ* fk) {
  for (int j = 0; j < L; ++j) {
    const LinkDesc& l = links[j];
    const DQ hj = dq_joint(l.kind, l.axis, theta[l.theta_index]);
    const DQ local = dq_compose(dq_load(l.offset), hj);
    fk[j] = l.parent < 0 ? local : dq_compose(fk[l.parent], local);
  }
}

// One d_link_offset block (skeleton.cpp:82-108): dH_jD / dtheta_k where
// k_link = link_of_joint(k) is an ancestor-or-self of link j.
WT_HD DQ d_link_offset(const LinkDesc* links, const DQ* fk, const double* theta, int j,
                       int k_link) {
  const LinkDesc& lk = links[k_link];
  const DQ off = dq_load(lk.offset);
  const DQ pre = lk.parent < 0 ? off : dq_compose(fk[lk.parent], off);
  const DQ dj = dq_djoint(lk.kind, lk.axis, theta[lk.theta_index]);
  const DQ k_to_j = dq_compose(dq_inverse(fk[k_link]), fk[j]);
  return dq_compose(dq_compose(pre, dj), dq_compose(k_to_j, dq_load(links[j].bind_inv)));
}

}  // namespace wt
