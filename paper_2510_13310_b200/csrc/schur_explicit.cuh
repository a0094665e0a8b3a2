// schur_explicit.cuh -- solve_normal(..., solver="schur_pcg") on an EXPLICIT,
// user-assembled BlockNormalSystem (lm.py:537-704 _solve_schur, lm.py:707-720).
//
// BAProblem / GPProblem never come here: they solve matrix-free from the
// compact Jacobian (ba_pcg*.cuh, gp_kernels.cuh). This path is for a caller
// that holds the block storage of a damped normal system (sparse_block.py:
// 162-216) -- a foreign problem provider under lm_solve, or a direct
// solve_normal call -- and it keeps the reference's algorithm:
//
//   stage 1  eliminate per-observation scale blocks (lm.py:563-597)
//   stage 2  invert the 3x3 point blocks with pinning / det > 0 (lm.py:495-513),
//            y = M b_pt, b_red = b_ret - sum U y (lm.py:599-622)
//   S        direct retained part, minus sum U_a M U_b^T per slot (schur_fill,
//            _core.pyx:100-160), pinned zero diagonals (lm.py:628-635); S is a
//            dense n_ret x n_ret matrix, like the reference's
//   PCG      block-Jacobi per retained block (lm.py:516-534), x0 = 0, the
//            reference's stop rule and CGStall conditions (lm.py:637-672)
//   back-substitution (lm.py:674-704)
//
// Index planning (block classification, U-entry gathers, slot schedule) is
// host integer work done once per pattern (generic._SchurXPlan); every
// floating-point step runs here. Each output has one owner that sums its
// contributions in the plan's order, so results are deterministic.
#pragma once
#include "common.cuh"

#include "../../include/ssfm.h"

typedef ssfm_schur_plan XsPlan;   // field meanings: include/ssfm.h

struct XsWork {
  double *S, *U, *dpt, *M, *y, *g, *bred, *x, *r, *z, *p, *q, *prec;
  int* status;
  struct Ctl {
    double tol, rho, rn;
    int iters, done;   // done: 0 running, 1 converged, 2 stalled (max iters), 3 breakdown
    int cg_max;
    int pad;
  }* ctl;
};

__device__ __forceinline__ double xs_inv_d(double d) { return d == 0.0 ? 0.0 : 1.0 / d; }

// S = direct part, U = gathered couplings, d_pt = point diagonals, g = gradient
__global__ void k_xs_init(XsPlan pl, const double* __restrict__ data, const double* __restrict__ grad, XsWork w) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  for (long long k = t; k < pl.n_direct; k += nt) w.S[pl.direct_dst[k]] = data[pl.direct_src[k]];
  const long long nu = pl.n_u ? pl.u_off[pl.n_u] : 0;
  for (long long k = t; k < nu; k += nt) w.U[k] = data[pl.u_gather[k]];
  for (long long k = t; k < 9 * pl.n_pt; k += nt) w.dpt[k] = data[pl.pt_diag[k / 9] + k % 9];
  for (long long k = t; k < pl.n_params; k += nt) w.g[k] = grad[k];
}

// ---- stage 1: scale elimination (lm.py:563-597) --------------------------
// masked scales (zero diagonal) must have no coupling and no gradient
__global__ void k_xs_sc_check(XsPlan pl, const double* __restrict__ data, const double* __restrict__ grad,
                              XsWork w) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= pl.n_sc) return;
  if (data[pl.sc_diag[s]] != 0.0) return;
  bool bad = grad[pl.sc_theta[s]] != 0.0;
  for (int i = 0; i < 3; ++i) bad |= data[pl.sc_uc[s] + i] != 0.0 || data[pl.sc_up[s] + i] != 0.0;
  if (bad) atomicOr(w.status, ST_PIN_SCALE);
}

// retained (width-3) diagonal blocks of S and their gradient rows
__global__ void k_xs_sc_cam(XsPlan pl, const double* __restrict__ data, const double* __restrict__ grad, XsWork w) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= pl.n_rblk) return;
  const long long a = pl.c_scseg[c], b = pl.c_scseg[c + 1];
  if (a == b) return;
  const long long r0 = pl.ret_s_off[c], n = pl.n_ret;
  for (long long k = a; k < b; ++k) {
    const int s = pl.sc_by_c[k];
    const double inv = xs_inv_d(data[pl.sc_diag[s]]);
    const double* u = data + pl.sc_uc[s];
    const double bs = grad[pl.sc_theta[s]];
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) w.S[(r0 + i) * n + r0 + j] -= inv * (u[i] * u[j]);
      w.g[pl.ret_theta[r0 + i]] -= (inv * bs) * u[i];
    }
  }
}

__global__ void k_xs_sc_pt(XsPlan pl, const double* __restrict__ data, const double* __restrict__ grad, XsWork w) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= pl.n_pt) return;
  for (long long k = pl.p_scseg[p]; k < pl.p_scseg[p + 1]; ++k) {
    const int s = pl.sc_by_p[k];
    const double inv = xs_inv_d(data[pl.sc_diag[s]]);
    const double* u = data + pl.sc_up[s];
    const double bs = grad[pl.sc_theta[s]];
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) w.dpt[9 * p + 3 * i + j] -= inv * (u[i] * u[j]);
      w.g[pl.pt_theta[p] + i] -= (inv * bs) * u[i];
    }
  }
}

__global__ void k_xs_sc_u(XsPlan pl, const double* __restrict__ data, XsWork w) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= pl.n_u) return;
  for (long long k = pl.u_scseg[e]; k < pl.u_scseg[e + 1]; ++k) {
    const int s = pl.sc_by_u[k];
    const double inv = xs_inv_d(data[pl.sc_diag[s]]);
    const double* uc = data + pl.sc_uc[s];
    const double* up = data + pl.sc_up[s];
    double* U = w.U + pl.u_off[e];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) U[3 * i + j] -= inv * (uc[i] * up[j]);
  }
}

// ---- stage 2: point blocks (lm.py:495-513, :599-606) ---------------------
__device__ __forceinline__ double det3(const double* a) {
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) + a[2] * (a[3] * a[7] - a[4] * a[6]);
}

__global__ void k_xs_ptinv(XsPlan pl, XsWork w) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= pl.n_pt) return;
  double a[9];
  for (int k = 0; k < 9; ++k) a[k] = w.dpt[9 * p + k];
  const double* b = w.g + pl.pt_theta[p];
  for (int i = 0; i < 3; ++i) {
    if (a[4 * i] == 0.0) {                // pinned direction: gradient must be zero
      if (b[i] != 0.0) atomicOr(w.status, ST_PIN_POINT);
      a[4 * i] = 1.0;
    }
  }
  const double det = det3(a);
  double m[9];
  if (!(det > 0.0) || !isfinite(det)) {
    atomicOr(w.status, ST_SINGULAR_POINT);
    for (int k = 0; k < 9; ++k) m[k] = 0.0;
  } else {
    const double id = 1.0 / det;
    m[0] = (a[4] * a[8] - a[5] * a[7]) * id;
    m[1] = (a[2] * a[7] - a[1] * a[8]) * id;
    m[2] = (a[1] * a[5] - a[2] * a[4]) * id;
    m[3] = (a[5] * a[6] - a[3] * a[8]) * id;
    m[4] = (a[0] * a[8] - a[2] * a[6]) * id;
    m[5] = (a[2] * a[3] - a[0] * a[5]) * id;
    m[6] = (a[3] * a[7] - a[4] * a[6]) * id;
    m[7] = (a[1] * a[6] - a[0] * a[7]) * id;
    m[8] = (a[0] * a[4] - a[1] * a[3]) * id;
  }
  for (int k = 0; k < 9; ++k) w.M[9 * p + k] = m[k];
  for (int i = 0; i < 3; ++i) w.y[3 * p + i] = m[3 * i] * b[0] + m[3 * i + 1] * b[1] + m[3 * i + 2] * b[2];
}

// b_red = g_ret - sum_U U y   (per retained block, U entries in entry order)
__global__ void k_xs_bred(XsPlan pl, XsWork w) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= pl.n_rblk) return;
  const long long r0 = pl.ret_s_off[c];
  const int wd = (int)(pl.ret_s_off[c + 1] - r0);
  for (int i = 0; i < wd; ++i) w.bred[r0 + i] = w.g[pl.ret_theta[r0 + i]];
  for (long long k = pl.ret_useg[c]; k < pl.ret_useg[c + 1]; ++k) {
    const int e = pl.u_by_ret[k];
    const double* U = w.U + pl.u_off[e];
    const double* y = w.y + 3ll * pl.u_pt[e];
    for (int i = 0; i < wd; ++i) w.bred[r0 + i] -= U[3 * i] * y[0] + U[3 * i + 1] * y[1] + U[3 * i + 2] * y[2];
  }
}

// S[slot] -= sum U_a M U_b^T (one warp per slot, lanes over the wa x wb
// elements; contributions in the slot's order), mirrored for ra != rb
__global__ void k_xs_fill(XsPlan pl, XsWork w) {
  const long long s = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= pl.n_slots) return;
  const int ra = pl.slot_ra[s], rb = pl.slot_rb[s];
  const long long r0 = pl.ret_s_off[ra], c0 = pl.ret_s_off[rb], n = pl.n_ret;
  const int wa = (int)(pl.ret_s_off[ra + 1] - r0), wb = (int)(pl.ret_s_off[rb + 1] - c0);
  for (int el = lane; el < wa * wb; el += 32) {
    const int i = el / wb, j = el - i * wb;
    double acc = 0.0;
    for (long long k = pl.slot_seg[s]; k < pl.slot_seg[s + 1]; ++k) {
      const int ea = pl.con_ua[k], eb = pl.con_ub[k];
      const double* Ua = w.U + pl.u_off[ea] + 3 * i;
      const double* Ub = w.U + pl.u_off[eb] + 3 * j;
      const double* M = w.M + 9ll * pl.u_pt[ea];
      double v = 0.0;
      for (int kk = 0; kk < 3; ++kk) {
        const double tm = __dadd_rn(__dadd_rn(__dmul_rn(Ua[0], M[kk]), __dmul_rn(Ua[1], M[3 + kk])),
                                    __dmul_rn(Ua[2], M[6 + kk]));
        v = __dadd_rn(v, __dmul_rn(tm, Ub[kk]));
      }
      acc = __dadd_rn(acc, v);
    }
    w.S[(r0 + i) * n + c0 + j] -= acc;
    if (r0 != c0) w.S[(c0 + j) * n + r0 + i] -= acc;
  }
}

// pin exactly-zero diagonals of S (lm.py:628-635)
__global__ void k_xs_pin(XsPlan pl, XsWork w) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= pl.n_ret) return;
  double* d = w.S + i * pl.n_ret + i;
  if (*d == 0.0) {
    if (w.bred[i] != 0.0) atomicOr(w.status, ST_PIN_RETAINED);
    *d = 1.0;
  }
}

// block-Jacobi factors: invert each retained block's w x w diagonal block of S
// (Gauss-Jordan with partial pivoting; exact-zero pivot or non-finite result
// = the reference's LinAlgError / non-finite SingularBlock, lm.py:516-534)
__global__ void k_xs_prec(XsPlan pl, XsWork w) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= pl.n_rblk) return;
  const long long r0 = pl.ret_s_off[c], n = pl.n_ret;
  const int wd = (int)(pl.ret_s_off[c + 1] - r0);
  double a[8][8], inv[8][8];
  for (int i = 0; i < wd; ++i)
    for (int j = 0; j < wd; ++j) {
      a[i][j] = w.S[(r0 + i) * n + r0 + j];
      inv[i][j] = i == j ? 1.0 : 0.0;
    }
  bool ok = true;
  for (int col = 0; col < wd && ok; ++col) {
    int piv = col;
    for (int i = col + 1; i < wd; ++i)
      if (fabs(a[i][col]) > fabs(a[piv][col])) piv = i;
    if (a[piv][col] == 0.0) { ok = false; break; }
    if (piv != col)
      for (int j = 0; j < wd; ++j) {
        double t = a[col][j]; a[col][j] = a[piv][j]; a[piv][j] = t;
        t = inv[col][j]; inv[col][j] = inv[piv][j]; inv[piv][j] = t;
      }
    const double ip = 1.0 / a[col][col];
    for (int j = 0; j < wd; ++j) { a[col][j] *= ip; inv[col][j] *= ip; }
    for (int i = 0; i < wd; ++i) {
      if (i == col) continue;
      const double f = a[i][col];
      if (f == 0.0) continue;
      for (int j = 0; j < wd; ++j) { a[i][j] -= f * a[col][j]; inv[i][j] -= f * inv[col][j]; }
    }
  }
  double* out = w.prec + pl.pre_off[c];
  for (int i = 0; i < wd; ++i)
    for (int j = 0; j < wd; ++j) {
      const double v = ok ? inv[i][j] : 0.0;
      if (!isfinite(v)) ok = false;
      out[i * wd + j] = v;
    }
  if (!ok) atomicOr(w.status, ST_SINGULAR_PRECOND);
}

// ---- PCG (lm.py:637-672) -------------------------------------------------
// q = S p: one warp per row, lanes stride the columns, fixed butterfly
__global__ void k_xs_matvec(XsPlan pl, XsWork w) {
  if (w.ctl->done) return;
  const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= pl.n_ret) return;
  const double* a = w.S + row * pl.n_ret;
  double v = 0.0;
  for (long long j = lane; j < pl.n_ret; j += 32) v += a[j] * w.p[j];
  v = warp_sum(v);
  if (lane == 0) w.q[row] = v;
}

__device__ __forceinline__ double xs_block_sum(double v, double* sm) {
  double a[1] = {v};
  block_reduce<1>(a, sm);
  if (threadIdx.x == 0) sm[32] = a[0];
  __syncthreads();
  const double s = sm[32];
  __syncthreads();
  return s;
}

// z = M r per retained block (threads over blocks)
__device__ __forceinline__ void xs_precond(const XsPlan& pl, const XsWork& w) {
  for (long long c = threadIdx.x; c < pl.n_rblk; c += blockDim.x) {
    const long long r0 = pl.ret_s_off[c];
    const int wd = (int)(pl.ret_s_off[c + 1] - r0);
    const double* m = w.prec + pl.pre_off[c];
    for (int i = 0; i < wd; ++i) {
      double v = 0.0;
      for (int j = 0; j < wd; ++j) v += m[i * wd + j] * w.r[r0 + j];
      w.z[r0 + i] = v;
    }
  }
}

// one CTA: x = 0, r = b_red, the stop test, z = M r, p = z, rho = r.z
__global__ void k_xs_cg_start(XsPlan pl, XsWork w, const double* __restrict__ grad, double cg_tol, int cg_max) {
  __shared__ double sm[40];
  const long long n = pl.n_ret;
  double gg = 0.0, rr = 0.0;
  for (long long k = threadIdx.x; k < pl.n_params; k += blockDim.x) gg += grad[k] * grad[k];
  for (long long k = threadIdx.x; k < n; k += blockDim.x) {
    w.x[k] = 0.0;
    w.r[k] = w.bred[k];
    rr += w.bred[k] * w.bred[k];
  }
  gg = xs_block_sum(gg, sm);
  rr = xs_block_sum(rr, sm);
  const double tol = cg_tol * fmax(sqrt(gg), 1e-300);
  const double rn = sqrt(rr);
  if (threadIdx.x == 0) {
    w.ctl->tol = tol;
    w.ctl->rn = rn;
    w.ctl->iters = 0;
    w.ctl->cg_max = cg_max;
    w.ctl->done = rn <= tol ? 1 : 0;
  }
  if (rn <= tol) return;
  __syncthreads();
  xs_precond(pl, w);
  __syncthreads();
  double rz = 0.0;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) {
    w.p[k] = w.z[k];
    rz += w.r[k] * w.z[k];
  }
  rz = xs_block_sum(rz, sm);
  if (threadIdx.x == 0) {
    w.ctl->rho = rz;
    if (cg_max <= 0) w.ctl->done = 2;
  }
}

// one CTA: alpha, x/r update, stop test, z = M r, beta, p update
__global__ void k_xs_cg_step(XsPlan pl, XsWork w) {
  __shared__ double sm[40];
  if (w.ctl->done) return;
  const long long n = pl.n_ret;
  double pq = 0.0;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) pq += w.p[k] * w.q[k];
  pq = xs_block_sum(pq, sm);
  if (!isfinite(pq) || pq <= 0.0) {
    if (threadIdx.x == 0) w.ctl->done = 3;
    return;
  }
  const double alpha = w.ctl->rho / pq;
  double rr = 0.0;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) {
    w.x[k] += alpha * w.p[k];
    const double rk = w.r[k] - alpha * w.q[k];
    w.r[k] = rk;
    rr += rk * rk;
  }
  rr = xs_block_sum(rr, sm);
  const int iters = w.ctl->iters + 1;
  const double rn = sqrt(rr);
  if (rn <= w.ctl->tol) {
    if (threadIdx.x == 0) { w.ctl->iters = iters; w.ctl->rn = rn; w.ctl->done = 1; }
    return;
  }
  xs_precond(pl, w);
  __syncthreads();
  double rz = 0.0;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) rz += w.r[k] * w.z[k];
  rz = xs_block_sum(rz, sm);
  const double beta = rz / w.ctl->rho;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) w.p[k] = w.p[k] * beta + w.z[k];
  if (threadIdx.x == 0) {
    w.ctl->iters = iters;
    w.ctl->rn = rn;
    w.ctl->rho = rz;
    if (iters >= w.ctl->cg_max) w.ctl->done = 2;
  }
}

// ---- back-substitution (lm.py:674-704) ------------------------------------
__global__ void k_xs_back_zero(XsPlan pl, double* delta) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  for (long long k = t; k < pl.n_params; k += nt) delta[k] = 0.0;
}
__global__ void k_xs_back_x(XsPlan pl, XsWork w, double* delta) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < pl.n_ret) delta[pl.ret_theta[k]] = w.x[k];
}
// delta_pt = y - M sum_U U^T x  (U entries of the point in entry order)
__global__ void k_xs_back_pt(XsPlan pl, XsWork w, double* delta) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= pl.n_pt) return;
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long k = pl.pt_useg[p]; k < pl.pt_useg[p + 1]; ++k) {
    const int e = pl.u_by_pt[k];
    const long long r0 = pl.ret_s_off[pl.u_ret[e]];
    const int wd = pl.u_w[e];
    const double* U = w.U + pl.u_off[e];
    for (int j = 0; j < 3; ++j) {
      double v = 0.0;
      for (int i = 0; i < wd; ++i) v += U[3 * i + j] * w.x[r0 + i];
      acc[j] += v;
    }
  }
  const double* m = w.M + 9 * p;
  for (int i = 0; i < 3; ++i)
    delta[pl.pt_theta[p] + i] = w.y[3 * p + i] - (m[3 * i] * acc[0] + m[3 * i + 1] * acc[1] + m[3 * i + 2] * acc[2]);
}
// delta_o = inv (b_o - u_c . delta_c - u_p . delta_p), original system values
__global__ void k_xs_back_sc(XsPlan pl, const double* __restrict__ data, const double* __restrict__ grad,
                             double* delta) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= pl.n_sc) return;
  const double inv = xs_inv_d(data[pl.sc_diag[s]]);
  const double* uc = data + pl.sc_uc[s];
  const double* up = data + pl.sc_up[s];
  const long long cr = pl.ret_s_off[pl.sc_c[s]];
  const long long pr = pl.pt_theta[pl.sc_p[s]];
  double dc = 0.0, dp = 0.0;
  for (int i = 0; i < 3; ++i) {
    dc += uc[i] * delta[pl.ret_theta[cr + i]];
    dp += up[i] * delta[pr + i];
  }
  delta[pl.sc_theta[s]] = inv * ((grad[pl.sc_theta[s]] - dc) - dp);
}
