// On-device accuracy metrics of the reconstruction:
// pairwise relative-rotation AUC, the Umeyama moments of camera-centre
// registration, and the Sim(3) transform of a scene in place. The reference
// computes these in numpy (synth_metrics.py:210-309); rotation_auc is
// O(C^2) (12.5M camera pairs at C5) and align touches every point.
// Reductions are fixed-order (block per row, rows summed in order): results
// are deterministic run to run.
#pragma once
#include "common.cuh"

#define MET_MAX_TAU 16
#define MET_THREADS 256

struct AucArgs {
  int ntau;
  double inv_tau[MET_MAX_TAU];
};

struct Sim3Args {
  double R[9];     // row-major rotation
  double t[3];
  double s;
  double rqc[4];   // conj(quat_from_matrix(R)), (w, x, y, z)
};

// q / |q| per camera (quat_normalize, scene.py:30-32), both scenes
__global__ void k_met_qnorm(const double* __restrict__ qa, const double* __restrict__ qb, int C,
                            double* __restrict__ na, double* __restrict__ nb) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= 2 * C) return;
  const double* q = c < C ? qa + 4ll * c : qb + 4ll * (c - C);
  double* o = c < C ? na + 4ll * c : nb + 4ll * (c - C);
  const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
#pragma unroll
  for (int k = 0; k < 4; ++k) o[k] = q[k] / n;
}

// q_a * conj(q_b) (synth_metrics.py:294-300)
__device__ __forceinline__ void met_rel(const double* a, const double* b, double* o) {
  const double bw = b[0], bx = -b[1], by = -b[2], bz = -b[3];
  const double aw = a[0], ax = a[1], ay = a[2], az = a[3];
  o[0] = aw * bw - (ax * bx + ay * by + az * bz);
  o[1] = aw * bx + bw * ax + (ay * bz - az * by);
  o[2] = aw * by + bw * ay + (az * bx - ax * bz);
  o[3] = aw * bz + bw * az + (ax * by - ay * bx);
}

// block i: pairs (i, j > i); part[i][k] = sum_j max(0, 1 - err_ij / tau_k)
__global__ void __launch_bounds__(MET_THREADS) k_met_auc_rows(const double* __restrict__ qe,
                                                              const double* __restrict__ qt, int C, AucArgs a,
                                                              double* __restrict__ part) {
  __shared__ double sm[(MET_THREADS / 32) * MET_MAX_TAU];
  const int i = blockIdx.x;
  double v[MET_MAX_TAU];
#pragma unroll
  for (int k = 0; k < MET_MAX_TAU; ++k) v[k] = 0.0;
  double ei[4], ti[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { ei[k] = qe[4ll * i + k]; ti[k] = qt[4ll * i + k]; }
  const double r2d = 180.0 / 3.141592653589793;
  for (int j = i + 1 + threadIdx.x; j < C; j += blockDim.x) {
    double re[4], rt[4];
    met_rel(ei, qe + 4ll * j, re);
    met_rel(ti, qt + 4ll * j, rt);
    double d = fabs(re[0] * rt[0] + re[1] * rt[1] + re[2] * rt[2] + re[3] * rt[3]);
    d = fmin(fmax(d, 0.0), 1.0);
    const double err = 2.0 * acos(d) * r2d;
#pragma unroll
    for (int k = 0; k < MET_MAX_TAU; ++k)
      if (k < a.ntau) v[k] += fmax(0.0, 1.0 - err * a.inv_tau[k]);
  }
  block_reduce<MET_MAX_TAU>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < MET_MAX_TAU; ++k) part[(long long)MET_MAX_TAU * i + k] = v[k];
  }
}

// rows summed in order, one thread per threshold
__global__ void k_met_auc_final(const double* __restrict__ part, int rows, int ntau, double* __restrict__ out) {
  const int k = threadIdx.x;
  if (k >= ntau) return;
  double s = 0.0;
  for (int i = 0; i < rows; ++i) s += part[(long long)MET_MAX_TAU * i + k];
  out[k] = s;
}

// Umeyama moments (synth_metrics.py:225-238) in one block, two passes:
// out = [mx(3), my(3), cov = yc^T xc / n (9, row-major), var_x = sum|xc|^2 / n,
//        sum |x - y|^2 (uncentred, for center_rmse)]
__global__ void __launch_bounds__(1024) k_met_moments(const double* __restrict__ x, const double* __restrict__ y,
                                                      int n, double* __restrict__ out) {
  __shared__ double sm[32 * 11];
  __shared__ double mean[6];
  double v[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) v[k] = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v[k] += x[3ll * i + k];
      v[3 + k] += y[3ll * i + k];
      const double e = x[3ll * i + k] - y[3ll * i + k];
      v[6] += e * e;
    }
  }
  block_reduce<7>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) mean[k] = v[k] / n;
    out[16] = v[6];
  }
  __syncthreads();
  double w[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) w[k] = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double xc[3], yc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) { xc[k] = x[3ll * i + k] - mean[k]; yc[k] = y[3ll * i + k] - mean[3 + k]; }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) w[3 * r + c] += yc[r] * xc[c];
    w[9] += xc[0] * xc[0] + xc[1] * xc[1] + xc[2] * xc[2];
  }
  __syncthreads();
  block_reduce<10>(w, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) out[k] = mean[k];
#pragma unroll
    for (int k = 0; k < 10; ++k) out[6 + k] = w[k] / n;
  }
}

// x <- s (R x) + t for [n][3] positions (Alignment.apply, synth_metrics.py:206-207)
__device__ __forceinline__ void met_sim3(const Sim3Args& a, double* p) {
  const double x = p[0], y = p[1], z = p[2];
#pragma unroll
  for (int r = 0; r < 3; ++r) p[r] = a.s * (x * a.R[3 * r] + y * a.R[3 * r + 1] + z * a.R[3 * r + 2]) + a.t[r];
}

__global__ void k_met_apply_points(Sim3Args a, double* __restrict__ pts, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) met_sim3(a, pts + 3 * i);
}

// cameras: q <- normalize(q * conj(rq)), centre <- s R c + t (synth_metrics.py:248-251)
__global__ void k_met_apply_cameras(Sim3Args a, double* __restrict__ quats, double* __restrict__ centers, int C) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double* q = quats + 4ll * c;
  const double aw = q[0], ax = q[1], ay = q[2], az = q[3];
  const double bw = a.rqc[0], bx = a.rqc[1], by = a.rqc[2], bz = a.rqc[3];
  double o[4];
  o[0] = aw * bw - ax * bx - ay * by - az * bz;   // quat_multiply (scene.py:35-44)
  o[1] = aw * bx + ax * bw + ay * bz - az * by;
  o[2] = aw * by - ax * bz + ay * bw + az * bx;
  o[3] = aw * bz + ax * by - ay * bx + az * bw;
  const double n = sqrt(o[0] * o[0] + o[1] * o[1] + o[2] * o[2] + o[3] * o[3]);
#pragma unroll
  for (int k = 0; k < 4; ++k) q[k] = o[k] / n;
  met_sim3(a, centers + 3ll * c);
}

// make_rays (gp.py:150-177) per observation, in numpy's operation order
// (explicit round-to-nearest, no contraction): bit-identical to the host
// restatement. dirs = ((u - cx) / f, (v - cy) / f, 1); world = rotate_many(
// conj(q), dirs) (scene.py:126-132); rays = world / |world|; ray depth =
// depth * |dirs|.
__global__ void k_make_rays(long long n, const long long* __restrict__ cam, const double* __restrict__ pix,
                            const double* __restrict__ pps, const double* __restrict__ foc,
                            const double* __restrict__ quats, const double* __restrict__ depths,
                            double* __restrict__ rays, double* __restrict__ ray_depths) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long c = cam[i];
  const double f = foc[c];
  const double d0 = __ddiv_rn(__dsub_rn(pix[2 * i], pps[2 * c]), f);
  const double d1 = __ddiv_rn(__dsub_rn(pix[2 * i + 1], pps[2 * c + 1]), f);
  const double d2 = 1.0;
  const double* q = quats + 4 * c;
  double qn[4] = {q[0], -q[1], -q[2], -q[3]};
  const double qq = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(qn[0], qn[0]), __dmul_rn(qn[1], qn[1])),
                                        __dmul_rn(qn[2], qn[2])), __dmul_rn(qn[3], qn[3]));
  const double qnorm = __dsqrt_rn(qq);
#pragma unroll
  for (int k = 0; k < 4; ++k) qn[k] = __ddiv_rn(qn[k], qnorm);
  const double u0 = qn[1], u1 = qn[2], u2 = qn[3];
  const double t0 = __dsub_rn(__dmul_rn(u1, d2), __dmul_rn(u2, d1));
  const double t1 = __dsub_rn(__dmul_rn(u2, d0), __dmul_rn(u0, d2));
  const double t2 = __dsub_rn(__dmul_rn(u0, d1), __dmul_rn(u1, d0));
  const double c0 = __dsub_rn(__dmul_rn(u1, t2), __dmul_rn(u2, t1));
  const double c1 = __dsub_rn(__dmul_rn(u2, t0), __dmul_rn(u0, t2));
  const double c2 = __dsub_rn(__dmul_rn(u0, t1), __dmul_rn(u1, t0));
  const double w0 = __dadd_rn(d0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(qn[0], t0), c0)));
  const double w1 = __dadd_rn(d1, __dmul_rn(2.0, __dadd_rn(__dmul_rn(qn[0], t1), c1)));
  const double w2 = __dadd_rn(d2, __dmul_rn(2.0, __dadd_rn(__dmul_rn(qn[0], t2), c2)));
  const double wn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(w0, w0), __dmul_rn(w1, w1)), __dmul_rn(w2, w2)));
  rays[3 * i] = __ddiv_rn(w0, wn);
  rays[3 * i + 1] = __ddiv_rn(w1, wn);
  rays[3 * i + 2] = __ddiv_rn(w2, wn);
  if (depths) {
    const double dn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
    ray_depths[i] = __dmul_rn(depths[i], dn);
  }
}
