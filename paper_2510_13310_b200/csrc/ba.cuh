// ba.cuh -- per-observation bundle-adjustment math (reprojection residual and
// analytic Jacobian), restating ba.py:111-194 and scene.py:135-184, 368-408.
//
// The residual path (projection, diff, robust weight) is written with explicit
// round-to-nearest intrinsics in the same operation order as the reference's
// numpy expressions, so that residuals and costs on the reference's synthetic
// scenes reproduce its arithmetic (bit-zero residuals on exact scenes,
// ba.py/test_ba.py:48-52). Jacobian blocks use ordinary (FMA-contracted) fp64
// and match the reference to rounding.
#pragma once
#include "common.cuh"

#define MUL(a, b) __dmul_rn((a), (b))
#define ADD(a, b) __dadd_rn((a), (b))
#define SUB(a, b) __dsub_rn((a), (b))
#define DIV(a, b) __ddiv_rn((a), (b))

// DEPTH_EPS, scene.py:23
#define SSFM_DEPTH_EPS 1e-12

// Per-camera cache, rebuilt whenever theta changes (24 doubles = 192 B).
struct __align__(16) BACam {
  double R[9];      // R(q/|q|), scene.py:141-149
  double qh[4];     // q/|q|
  double qnorm;     // |q|
  double t[3];      // center
  double f;         // focal (theta or fixed)
  double pp[2];     // principal point
  double k[2];      // bal radial k1, k2
  double pad;       // 1/|q|
};

struct BAParams {
  int C, P;
  long long N;
  int model;          // 0 pinhole, 1 bal
  int focal_mode;     // 0 none (fixed focals), 1 per camera, 2 shared
  int loss_kind;      // 0 trivial, 1 huber, 2 cauchy
  double delta;
  long long off_pts;  // 7C
  long long off_foc;  // 7C + 3P
};

// quat_to_matrix_many on one quaternion (scene.py:135-150), normalization
// order of np.linalg.norm(axis=1) (sequential sum of squares).
__device__ __forceinline__ void ba_make_cam(const double* q, const double* t, double f,
                                            const double* pp, const double* k, BACam& c) {
  double n2 = ADD(ADD(ADD(MUL(q[0], q[0]), MUL(q[1], q[1])), MUL(q[2], q[2])), MUL(q[3], q[3]));
  double n = __dsqrt_rn(n2);
  double w = DIV(q[0], n), x = DIV(q[1], n), y = DIV(q[2], n), z = DIV(q[3], n);
  c.qh[0] = w; c.qh[1] = x; c.qh[2] = y; c.qh[3] = z;
  c.qnorm = n;
  c.R[0] = SUB(1.0, MUL(2.0, ADD(MUL(y, y), MUL(z, z))));
  c.R[1] = MUL(2.0, SUB(MUL(x, y), MUL(w, z)));
  c.R[2] = MUL(2.0, ADD(MUL(x, z), MUL(w, y)));
  c.R[3] = MUL(2.0, ADD(MUL(x, y), MUL(w, z)));
  c.R[4] = SUB(1.0, MUL(2.0, ADD(MUL(x, x), MUL(z, z))));
  c.R[5] = MUL(2.0, SUB(MUL(y, z), MUL(w, x)));
  c.R[6] = MUL(2.0, SUB(MUL(x, z), MUL(w, y)));
  c.R[7] = MUL(2.0, ADD(MUL(y, z), MUL(w, x)));
  c.R[8] = SUB(1.0, MUL(2.0, ADD(MUL(x, x), MUL(y, y))));
  c.t[0] = t[0]; c.t[1] = t[1]; c.t[2] = t[2];
  c.f = f;
  c.pp[0] = pp[0]; c.pp[1] = pp[1];
  c.k[0] = k[0]; c.k[1] = k[1];
  c.pad = 1.0 / n;   // 1/|q| for the factored operator (ba_pi_mul)
}

// Projection of one observation (ba.py:111-131). Returns camera point p,
// safe depth zs, mask and pixel uv.
struct BAProj {
  double v[3];    // X - t
  double p[3];    // R v
  double zs;      // safe z
  double uv[2];
  bool mask;
};

__device__ __forceinline__ void ba_project(const BACam& c, const double* X, int model, BAProj& o) {
  o.v[0] = SUB(X[0], c.t[0]);
  o.v[1] = SUB(X[1], c.t[1]);
  o.v[2] = SUB(X[2], c.t[2]);
  // np.einsum("nij,nj->ni") evaluates (R0 v0 + R2 v2) + R1 v1 for j = 3.
#pragma unroll
  for (int i = 0; i < 3; ++i)
    o.p[i] = ADD(ADD(MUL(c.R[3 * i + 0], o.v[0]), MUL(c.R[3 * i + 2], o.v[2])),
                 MUL(c.R[3 * i + 1], o.v[1]));
  const double z = o.p[2];
  o.zs = (fabs(z) < SSFM_DEPTH_EPS) ? 1.0 : z;
  if (model == 1) {
    o.mask = z < -SSFM_DEPTH_EPS;                       // scene.py:373-374
    double n0 = DIV(-o.p[0], o.zs), n1 = DIV(-o.p[1], o.zs);
    double r2 = ADD(MUL(n0, n0), MUL(n1, n1));
    double sc = ADD(ADD(1.0, MUL(c.k[0], r2)), MUL(MUL(c.k[1], r2), r2));
    double fs = MUL(c.f, sc);
    o.uv[0] = ADD(MUL(fs, n0), c.pp[0]);
    o.uv[1] = ADD(MUL(fs, n1), c.pp[1]);
  } else {
    o.mask = z > SSFM_DEPTH_EPS;                        // scene.py:375
    o.uv[0] = ADD(MUL(c.f, DIV(o.p[0], o.zs)), c.pp[0]);
    o.uv[1] = ADD(MUL(c.f, DIV(o.p[1], o.zs)), c.pp[1]);
  }
}

// robust_weight_many (scene.py:398-408): cost term and IRLS weight.
__device__ __forceinline__ void robust(int kind, double delta, double s, double& cost, double& w) {
  if (kind == 2) {   // Cauchy (an extension: scene.cauchy_cost_weight)
    const double d2 = MUL(delta, delta);
    const double r = DIV(s, d2);
    cost = MUL(d2, log1p(r));
    w = DIV(1.0, ADD(1.0, r));
    return;
  }
  if (kind == 1) {
    const double d2 = MUL(delta, delta);
    if (s > d2) {
      double root = __dsqrt_rn(s);
      cost = SUB(MUL(MUL(2.0, delta), root), d2);
      w = DIV(delta, root);
      return;
    }
  }
  cost = s;
  w = 1.0;
}

// Residual + robust cost term of one observation (ba.py:133-138, 148-151, 192-193).
__device__ __forceinline__ void ba_residual(const BAParams& bp, const BACam& c, const double* X,
                                            const double* pix, BAProj& pr, double r[2],
                                            double& sw, double& cost_term) {
  ba_project(c, X, bp.model, pr);
  const double d0 = SUB(pr.uv[0], pix[0]), d1 = SUB(pr.uv[1], pix[1]);
  const double s = ADD(MUL(d0, d0), MUL(d1, d1));
  double cst, w;
  robust(bp.loss_kind, bp.delta, s, cst, w);
  cost_term = pr.mask ? cst : 0.0;
  sw = pr.mask ? __dsqrt_rn(w) : 0.0;
  r[0] = MUL(d0, sw);
  r[1] = MUL(d1, sw);
}

// Compact Jacobian record of one observation (16 doubles):
//   pq[0..7]  sw * du_dp * dp_dq (2x4, row-major)            pose quaternion cols
//   jp[8..13] sw * du_dp * R     (2x3, row-major)            point block
//                                (pose center block == -jp, ba.py:187-188)
//   jf[14..15] sw * du_df        (2x1)                       focal block
#define BA_JREC 16

__device__ __forceinline__ void ba_jacobian(const BAParams& bp, const BACam& c, const BAProj& pr,
                                            double sw, double* J) {
  const double inv_z = 1.0 / pr.zs;
  const double f = c.f;
  const double px = pr.p[0], py = pr.p[1];
  double dup[6];   // du_dp 2x3
  double duf[2];
  if (bp.model == 1) {
    const double k1 = c.k[0], k2 = c.k[1];
    const double n0 = -px * inv_z, n1 = -py * inv_z;
    const double r2 = n0 * n0 + n1 * n1;
    const double sc = 1.0 + k1 * r2 + k2 * r2 * r2;
    // dn_dp = [[-iz, 0, px iz^2], [0, -iz, py iz^2]]
    const double a = f * sc, b = 2.0 * f * (k1 + 2.0 * k2 * r2);
    const double m00 = a + b * n0 * n0, m01 = b * n0 * n1, m11 = a + b * n1 * n1;
    const double iz2 = inv_z * inv_z;
    dup[0] = -m00 * inv_z; dup[1] = -m01 * inv_z; dup[2] = (m00 * px + m01 * py) * iz2;
    dup[3] = -m01 * inv_z; dup[4] = -m11 * inv_z; dup[5] = (m01 * px + m11 * py) * iz2;
    duf[0] = sc * n0; duf[1] = sc * n1;
  } else {
    dup[0] = f * inv_z; dup[1] = 0.0; dup[2] = -f * px * inv_z * inv_z;
    dup[3] = 0.0; dup[4] = f * inv_z; dup[5] = -f * py * inv_z * inv_z;
    duf[0] = px * inv_z; duf[1] = py * inv_z;
  }
  // d(R(q/|q|) v)/dq (scene.py:153-184)
  const double w = c.qh[0], u0 = c.qh[1], u1 = c.qh[2], u2 = c.qh[3];
  const double v0 = pr.v[0], v1 = pr.v[1], v2 = pr.v[2];
  double D[12];  // 3x4 row-major
  D[0] = 2.0 * (u1 * v2 - u2 * v1);
  D[4] = 2.0 * (u2 * v0 - u0 * v2);
  D[8] = 2.0 * (u0 * v1 - u1 * v0);
  const double ud = u0 * v0 + u1 * v1 + u2 * v2;
  const double u[3] = {u0, u1, u2}, v[3] = {v0, v1, v2};
  // -w [v]x
  const double vx[9] = {0.0, -v2, v1, v2, 0.0, -v0, -v1, v0, 0.0};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      D[4 * i + 1 + j] = 2.0 * (-w * vx[3 * i + j] + (i == j ? ud : 0.0) + u[i] * v[j] - 2.0 * v[i] * u[j]);
  // dp_dq = D (I - qh qh^T) / |q|
  double G[12];
  const double qh[4] = {w, u0, u1, u2};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double dq = D[4 * i] * qh[0] + D[4 * i + 1] * qh[1] + D[4 * i + 2] * qh[2] + D[4 * i + 3] * qh[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) G[4 * i + k] = (D[4 * i + k] - dq * qh[k]) / c.qnorm;
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      J[4 * r + k] = sw * (dup[3 * r] * G[k] + dup[3 * r + 1] * G[4 + k] + dup[3 * r + 2] * G[8 + k]);
#pragma unroll
    for (int k = 0; k < 3; ++k)
      J[8 + 3 * r + k] = sw * (dup[3 * r] * c.R[k] + dup[3 * r + 1] * c.R[3 + k] + dup[3 * r + 2] * c.R[6 + k]);
    J[14 + r] = (bp.focal_mode != 0) ? sw * duf[r] : 0.0;
  }
}

// Camera-side row view of a record: Jc (2x8) = [pq (2x4) | -jp (2x3) | jf (2x1)].
__device__ __forceinline__ void ba_jc_row(const double* J, int r, double* row8) {
#pragma unroll
  for (int k = 0; k < 4; ++k) row8[k] = J[4 * r + k];
#pragma unroll
  for (int k = 0; k < 3; ++k) row8[4 + k] = -J[8 + 3 * r + k];
  row8[7] = J[14 + r];
}

// Jc p (2-vector) for an 8-slot camera vector p.
__device__ __forceinline__ void ba_jc_mul(const double* J, const double* p, double* t) {
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    t[r] = J[4 * r] * p[0] + J[4 * r + 1] * p[1] + J[4 * r + 2] * p[2] + J[4 * r + 3] * p[3]
         - (J[8 + 3 * r] * p[4] + J[8 + 3 * r + 1] * p[5] + J[8 + 3 * r + 2] * p[6])
         + J[14 + r] * p[7];
  }
}

// Jc^T t (8-vector).
__device__ __forceinline__ void ba_jct_mul(const double* J, const double* t, double* o) {
#pragma unroll
  for (int k = 0; k < 4; ++k) o[k] = J[k] * t[0] + J[4 + k] * t[1];
#pragma unroll
  for (int k = 0; k < 3; ++k) o[4 + k] = -(J[8 + k] * t[0] + J[11 + k] * t[1]);
  o[7] = J[14] * t[0] + J[15] * t[1];
}

// Jp y (2-vector), Jp^T t (3-vector).
__device__ __forceinline__ void ba_jp_mul(const double* J, const double* y, double* t) {
  t[0] = J[8] * y[0] + J[9] * y[1] + J[10] * y[2];
  t[1] = J[11] * y[0] + J[12] * y[1] + J[13] * y[2];
}
__device__ __forceinline__ void ba_jpt_mul(const double* J, const double* t, double* o) {
  o[0] = J[8] * t[0] + J[11] * t[1];
  o[1] = J[9] * t[0] + J[12] * t[1];
  o[2] = J[10] * t[0] + J[13] * t[1];
}

// Factored operator record of one observation (6 doubles), for the two-pass
// Schur operator: with E = [[1, 0, -e0], [0, 1, -e1]] (e = p_xy / z_s) and a
// symmetric 2x2 S,   sw du_dp = S E,   sw du_df = phi e.   Then
//   Jp = S E R,   Jc = [S E D(v) Pi | -S E R | phi e]
// with Pi = (I - qh qh^T) / |q| and D(v) the 3x4 of scene.py:153-184; R, qh,
// |q| are per camera and v = X - t per observation, so an observation costs
// 6 doubles (+ v in the camera-major copy) instead of the 16 of BA_JREC.
// Rows: 0 s00, 1 e0, 2 e1, 3 phi, 4 s01, 5 s11 (pinhole: s01 = 0, s11 = s00,
// rows 4-5 unused).
#define BA_FREC 6
__device__ __forceinline__ void ba_factor(const BAParams& bp, const BACam& c, const BAProj& pr, double sw,
                                          double* F) {
  const double inv_z = 1.0 / pr.zs;
  const double e0 = pr.p[0] * inv_z, e1 = pr.p[1] * inv_z;
  F[1] = e0;
  F[2] = e1;
  if (bp.model == 1) {
    const double k1 = c.k[0], k2 = c.k[1];
    const double n0 = -e0, n1 = -e1;
    const double r2 = n0 * n0 + n1 * n1;
    const double sc = 1.0 + k1 * r2 + k2 * r2 * r2;
    const double a = c.f * sc, b = 2.0 * c.f * (k1 + 2.0 * k2 * r2);
    const double g = -sw * inv_z;
    F[0] = g * (a + b * n0 * n0);
    F[4] = g * (b * n0 * n1);
    F[5] = g * (a + b * n1 * n1);
    F[3] = bp.focal_mode != 0 ? -sw * sc : 0.0;
  } else {
    const double a = sw * (c.f * inv_z);
    F[0] = a;
    F[4] = 0.0;
    F[5] = a;
    F[3] = bp.focal_mode != 0 ? sw : 0.0;
  }
}

// (D(v) w)_i for a quaternion-space 4-vector w (D of scene.py:153-184):
//   2 [ (u x v)_i w0 - qw (v x w')_i + (u.v) w'_i + u_i (v.w') - 2 v_i (u.w') ]
__device__ __forceinline__ void ba_dq_mul(const double* qh, const double* v, const double* w, double* o) {
  const double u0 = qh[1], u1 = qh[2], u2 = qh[3], qw = qh[0];
  const double ud = u0 * v[0] + u1 * v[1] + u2 * v[2];
  const double vw = v[0] * w[1] + v[1] * w[2] + v[2] * w[3];
  const double uw = u0 * w[1] + u1 * w[2] + u2 * w[3];
  const double c0 = u1 * v[2] - u2 * v[1], c1 = u2 * v[0] - u0 * v[2], c2 = u0 * v[1] - u1 * v[0];
  const double x0 = v[1] * w[3] - v[2] * w[2], x1 = v[2] * w[1] - v[0] * w[3], x2 = v[0] * w[2] - v[1] * w[1];
  o[0] = 2.0 * (c0 * w[0] - qw * x0 + ud * w[1] + u0 * vw - 2.0 * v[0] * uw);
  o[1] = 2.0 * (c1 * w[0] - qw * x1 + ud * w[2] + u1 * vw - 2.0 * v[1] * uw);
  o[2] = 2.0 * (c2 * w[0] - qw * x2 + ud * w[3] + u2 * vw - 2.0 * v[2] * uw);
}

// D(v)^T g (4-vector):  [2 (u x v).g,  2 (qw (v x g)_j + (u.v) g_j + (u.g) v_j - 2 (v.g) u_j)]
__device__ __forceinline__ void ba_dqt_mul(const double* qh, const double* v, const double* g, double* o) {
  const double u0 = qh[1], u1 = qh[2], u2 = qh[3], qw = qh[0];
  const double ud = u0 * v[0] + u1 * v[1] + u2 * v[2];
  const double ug = u0 * g[0] + u1 * g[1] + u2 * g[2];
  const double vg = v[0] * g[0] + v[1] * g[1] + v[2] * g[2];
  const double c0 = u1 * v[2] - u2 * v[1], c1 = u2 * v[0] - u0 * v[2], c2 = u0 * v[1] - u1 * v[0];
  const double x0 = v[1] * g[2] - v[2] * g[1], x1 = v[2] * g[0] - v[0] * g[2], x2 = v[0] * g[1] - v[1] * g[0];
  o[0] = 2.0 * (c0 * g[0] + c1 * g[1] + c2 * g[2]);
  o[1] = 2.0 * (qw * x0 + ud * g[0] + ug * v[0] - 2.0 * vg * u0);
  o[2] = 2.0 * (qw * x1 + ud * g[1] + ug * v[1] - 2.0 * vg * u1);
  o[3] = 2.0 * (qw * x2 + ud * g[2] + ug * v[2] - 2.0 * vg * u2);
}

// Pi w = (w - qh (qh.w)) / |q|  (Pi symmetric); inv_qn = 1 / |q|
__device__ __forceinline__ void ba_pi_mul(const double* qh, double inv_qn, const double* w, double* o) {
  const double d = qh[0] * w[0] + qh[1] * w[1] + qh[2] * w[2] + qh[3] * w[3];
#pragma unroll
  for (int k = 0; k < 4; ++k) o[k] = (w[k] - d * qh[k]) * inv_qn;
}
