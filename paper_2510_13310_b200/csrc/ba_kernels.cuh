// ba_kernels.cuh -- bundle-adjustment kernels: camera prep, cost, linearize
// (+ Jt r, J^T J blocks), damped elimination blocks, preconditioner, back
// substitution and the candidate update.
//
// Data layout in HBM (N observations, P points, C cameras):
//   Jpm[16][N]  compact Jacobian, SoA, point-major   (read by point passes)
//   Jcm[16][N]  same records, SoA, camera-major       (read by camera passes)
//   per point (AoS): Cpt[6] (Jp^T Jp), gpt[3] (Jp^T r), Cinv[6], y0[3], yv[4]
//   per camera (AoS): Bc[64] (Jc^T Jc, 8x8 full), gcam[8], Minv[64], bred[8]
// The compact record is 16 fp64 per observation instead of the reference's
// 22 (ba.py:63): the pose-center block equals -(point block) (ba.py:187-188).
#pragma once
#include "ba.cuh"
#include "topo.cuh"

struct BADev {
  BAParams bp;
  Topo topo;
  const double* pix_pm;   // [2N] interleaved, point-major
  const double* pix_cm;   // [2N] interleaved, camera-major
  const double* pps;      // [2C]
  const double* dists;    // [2C]
  const double* focals;   // [C] fixed focals (focal_mode 0)
  BACam* cams;            // [C]
  double* Jpm;            // [16 * Npad] (fused-operator handles)
  double* Gpm;            // [8 * Npad] point-major Jp (6) + Jf (2): omega-form handles (ba_wobs)
  double* Xl;             // [4P] points at the linearization (omega-form, padded: 32-byte gathers)
  double* Wc;             // [8C] per-camera omega-form vector of the current p / x (ba_wvec)
  double* Rpm;            // [4N] point-major weighted residual [r0, r1, 0, 0] (ba_k_lin_tile; full sectors)
  double* Jcm;            // [16 * Npad]
  double* Fcm;            // [9 * Npad] factored records (ba_factor) + v = X - t, camera-major (two-pass only)
  BACam* camlin;          // [C] camera cache at the linearization (cams is overwritten by trial costs)
  long long Npad;
  double* Cpt;            // [6P]
  double* gpt;            // [3P]
  double* Bc;             // [64C]
  double* gcam;           // [8C]
  double* tilebuf;        // [44 * nt]
  double* Cinv;           // [6P]
  double* y0;             // [3P]
  double* yv;             // [4P] (padded for 32-byte gathers)
  double* Minv;           // [64C]
  double* bred;           // [8C]
  double* fterm;          // [2C] shared focal: per-camera shares (operator row / precond)
  double* fpt;            // [3P] shared focal: a_j = sum_o Jp_o^T jf_o (nullptr otherwise)
  double* fwpart;         // [ptinv blocks] shared focal: sum_j a_j^T Cinv_j a_j partials
  unsigned char* pinned;  // [C] bitmask of pinned retained slots
  const double* lamp;     // device-resident lambda (LM loop as a CUDA graph) or nullptr: the argument
  double* scal;           // scalars: [0] gmax bits, [1] gnorm2, [2] cost, ...
  double* partials;       // [max(nb, blocks)] reduction scratch
  int* status;
};

enum { SC_GMAX = 0, SC_GNORM2 = 1, SC_COST = 2, SC_LAMBDA = 3, SC_GFOCAL = 4 };

// Omega-form point-major record Gpm of observation i: [Jp row 0 (3), Jp row 1
// (3), Jf (2)]. GPM_AOS=1: 64-byte records (whole sectors); 0: SoA rows.
#ifndef GPM_AOS
#define GPM_AOS 1
#endif
__device__ __forceinline__ void gpm_store(const BADev& d, long long i, const double* jp8) {
#if GPM_AOS
  double* g = d.Gpm + 8 * i;
  *reinterpret_cast<double4*>(g) = make_double4(jp8[0], jp8[1], jp8[2], jp8[3]);
  *reinterpret_cast<double4*>(g + 4) = make_double4(jp8[4], jp8[5], jp8[6], jp8[7]);
#else
#pragma unroll
  for (int k = 0; k < 8; ++k) d.Gpm[k * d.Npad + i] = jp8[k];
#endif
}
// Factored camera-major record Fcm of observation i (ba_factor + v = X - t).
// FCM_AOS=1: one record per observation, pinhole 64 bytes [s00, e0, e1, phi,
// v0, v1, v2, 0], bal 96 bytes [s00, e0, e1, phi, s01, s11, v0, v1, v2, 0 x3]
// (2 / 3 vector loads instead of 7 / 9 scalar ones); 0: SoA rows [9][Npad].
#ifndef FCM_AOS
#define FCM_AOS 1
#endif
__host__ __device__ __forceinline__ long long fcm_doubles(int model, long long Npad) {
#if FCM_AOS
  return (model == 1 ? 12ll : 8ll) * Npad;
#else
  (void)model;
  return 9ll * Npad;
#endif
}
// F[0..5] = s00, e0, e1, phi, s01, s11 (ba_factor), F[6..8] = v
__device__ __forceinline__ void fcm_store(const BADev& d, long long i, const double* F, unsigned long long pol) {
#if FCM_AOS
  (void)pol;
  if (d.bp.model == 1) {
    double* r = d.Fcm + 12 * i;
    *reinterpret_cast<double4*>(r) = make_double4(F[0], F[1], F[2], F[3]);
    *reinterpret_cast<double4*>(r + 4) = make_double4(F[4], F[5], F[6], F[7]);
    *reinterpret_cast<double4*>(r + 8) = make_double4(F[8], 0.0, 0.0, 0.0);
  } else {
    double* r = d.Fcm + 8 * i;
    *reinterpret_cast<double4*>(r) = make_double4(F[0], F[1], F[2], F[3]);
    *reinterpret_cast<double4*>(r + 4) = make_double4(F[6], F[7], F[8], 0.0);
  }
#else
  const long long Np = d.Npad;
#pragma unroll
  for (int k = 0; k < 9; ++k)
    if (d.bp.model == 1 || k < 4 || k > 5) st_hint(d.Fcm + k * Np + i, F[k], pol);
#endif
}
// f[0..5] = s00, e0, e1, phi, s01, s11 (pinhole: s01 = 0, s11 = s00), vv = v
__device__ __forceinline__ void fcm_load(const BADev& d, long long i, double* f, double* vv, unsigned long long pol) {
#if FCM_AOS
  if (d.bp.model == 1) {
    double a[4], b[4], c[4];
    ld_v4_ro(d.Fcm + 12 * i, a, pol);
    ld_v4_ro(d.Fcm + 12 * i + 4, b, pol);
    ld_v4_ro(d.Fcm + 12 * i + 8, c, pol);
    f[0] = a[0]; f[1] = a[1]; f[2] = a[2]; f[3] = a[3]; f[4] = b[0]; f[5] = b[1];
    vv[0] = b[2]; vv[1] = b[3]; vv[2] = c[0];
  } else {
    double a[4], b[4];
    ld_v4_ro(d.Fcm + 8 * i, a, pol);
    ld_v4_ro(d.Fcm + 8 * i + 4, b, pol);
    f[0] = a[0]; f[1] = a[1]; f[2] = a[2]; f[3] = a[3]; f[4] = 0.0; f[5] = a[0];
    vv[0] = b[0]; vv[1] = b[1]; vv[2] = b[2];
  }
#else
  const long long Np = d.Npad;
#pragma unroll
  for (int k = 0; k < 4; ++k) f[k] = ldg_stream(d.Fcm + k * Np + i, pol);
  if (d.bp.model == 1) {
    f[4] = ldg_stream(d.Fcm + 4 * Np + i, pol);
    f[5] = ldg_stream(d.Fcm + 5 * Np + i, pol);
  } else {
    f[4] = 0.0;
    f[5] = f[0];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) vv[k] = ldg_stream(d.Fcm + (6 + k) * Np + i, pol);
#endif
}

__device__ __forceinline__ void gpm_load(const BADev& d, long long i, double* G, unsigned long long pol) {
#if GPM_AOS
  ld_v4_ro(d.Gpm + 8 * i, G, pol);
  ld_v4_ro(d.Gpm + 8 * i + 4, G + 4, pol);
#else
#pragma unroll
  for (int k = 0; k < 8; ++k) G[k] = ldg_stream(d.Gpm + k * d.Npad + i, pol);
#endif
}

// ---------------------------------------------------------------------------
// camera cache from theta (quat_to_matrix_many per camera, ba.py:111-116)
// ---------------------------------------------------------------------------
__global__ void ba_k_prep(BADev d, const double* __restrict__ theta) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d.bp.C) return;
  const double* pose = theta + 7ll * c;
  double f;
  if (d.bp.focal_mode == 1) f = theta[d.bp.off_foc + c];
  else if (d.bp.focal_mode == 2) f = theta[d.bp.off_foc];
  else f = d.focals[c];
  BACam cc;
  ba_make_cam(pose, pose + 4, f, d.pps + 2 * c, d.dists + 2 * c, cc);
  d.cams[c] = cc;
}

// ---------------------------------------------------------------------------
// cost (ba.py:133-138): one thread per observation (point-major), fixed-tree
// block sums, then a single-block sum of the block partials in block order.
// ---------------------------------------------------------------------------
__global__ void ba_k_cost(BADev d, const double* __restrict__ theta, double* partials) {
  __shared__ double sm[32];
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  if (i < d.topo.N) {
    const int c = d.topo.pm_cam[i], j = d.topo.pm_pt[i];
    const BACam cc = d.cams[c];
    const double* X = theta + d.bp.off_pts + 3ll * j;
    BAProj pr;
    double r[2], sw, ct;
    ba_residual(d.bp, cc, X, d.pix_pm + 2 * i, pr, r, sw, ct);
    v[0] = ct;
  }
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
}

// reproj_rmse statistics (synth_metrics.py:312-325): unweighted squared
// pixel error and count over observations in front of their camera; block
// partials [2 * block] summed in fixed order by the host entry point.
__global__ void ba_k_reproj(BADev d, const double* __restrict__ theta, double* partials) {
  __shared__ double sm[64];
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double v[2] = {0.0, 0.0};
  if (i < d.topo.N) {
    const int c = d.topo.pm_cam[i], j = d.topo.pm_pt[i];
    const BACam cc = d.cams[c];
    BAProj pr;
    ba_project(cc, theta + d.bp.off_pts + 3ll * j, d.bp.model, pr);
    if (pr.mask) {
      const double d0 = SUB(pr.uv[0], d.pix_pm[2 * i]), d1 = SUB(pr.uv[1], d.pix_pm[2 * i + 1]);
      v[0] = ADD(MUL(d0, d0), MUL(d1, d1));
      v[1] = 1.0;
    }
  }
  block_reduce<2>(v, sm);
  if (threadIdx.x == 0) { partials[2ll * blockIdx.x] = v[0]; partials[2ll * blockIdx.x + 1] = v[1]; }
}

// Sum n partials in fixed order with one block (deterministic).
__global__ void k_sum_partials(const double* __restrict__ partials, int n, double* out) {
  __shared__ double sm[32];
  double v[1] = {0.0};
  // contiguous chunk per thread, chunks in thread order
  int per = (n + blockDim.x - 1) / blockDim.x;
  int a = threadIdx.x * per, b = min(n, a + per);
  for (int k = a; k < b; ++k) v[0] += partials[k];
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) *out = v[0];
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // order-preserving for non-negative doubles (and NaN sorts above +inf)
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// One observation's weighted residual, robust cost term and compact Jacobian
// record. The point-major and camera-major copies of the Jacobian are computed
// by two kernels from the same inputs with this one expression tree (same
// rounding and contraction), so they are bit-identical; ssfm_check_jacobian
// verifies it on the device (tests/test_gpu_ba.py).
__device__ __forceinline__ void ba_obs_eval(const BAParams& bp, const BACam* __restrict__ cam, const double* X,
                                         const double* pix, double* r, double* J, double* cost_term,
                                         double* F = nullptr) {
  const BACam cc = *cam;
  BAProj pr;
  double sw;
  ba_residual(bp, cc, X, pix, pr, r, sw, *cost_term);
  ba_jacobian(bp, cc, pr, sw, J);
  if (F) {   // factored record (+ v) for the two-pass operator
    ba_factor(bp, cc, pr, sw, F);
    F[6] = pr.v[0]; F[7] = pr.v[1]; F[8] = pr.v[2];
  }
}

// ---------------------------------------------------------------------------
// linearize (ba.py:140-194) fused with the point side of jtj/jtr
// (_core.pyx:18-97 for point keys): one warp per point batch.
// Writes Jpm (coalesced), Jcm/rcm (camera-major scatter), Cpt, gpt, and the
// optional reference-layout exports (r_out [2N], J_out [22N] in observation order).
// ---------------------------------------------------------------------------
#define LIN_V 12   // Jp^T Jp (6), Jp^T r (3), Jp^T jf (3, shared focal only)
#ifndef LP_V2
#define LP_V2 1
#endif
__global__ void __launch_bounds__(256) ba_k_linearize(BADev d, const double* __restrict__ theta,
                                                      double* r_out, double* J_out, double* gpt_norm_part) {
  __shared__ double sm[8][SSFM_BATCH][LIN_V];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long Np = d.Npad;
  double gn2 = 0.0;   // sum of squares of owned point gradients (lane-local)
  double gmax = 0.0;
  for (int b = gw; b < d.topo.nb; b += warps) {
    const int ob0 = d.topo.bat_obs[b], ob1 = d.topo.bat_obs[b + 1];
    const int pb0 = d.topo.bat_pt[b], pb1 = d.topo.bat_pt[b + 1];
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    if (my_pt < pb1) { ps = d.topo.pt_seg[my_pt]; pe = d.topo.pt_seg[my_pt + 1]; }
    double acc[LIN_V];
#pragma unroll
    for (int k = 0; k < LIN_V; ++k) acc[k] = 0.0;
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[LIN_V];
#pragma unroll
      for (int k = 0; k < LIN_V; ++k) val[k] = 0.0;
      if (i < ob1) {
        const int c = d.topo.pm_cam[i], j = d.topo.pm_pt[i];
        const double* X = theta + d.bp.off_pts + 3ll * j;
        double r[2], J[BA_JREC], ct;
        ba_obs_eval(d.bp, d.cams + c, X, d.pix_pm + 2ll * i, r, J, &ct);
        if (d.Gpm) {   // omega form: Jp and Jf only (the quaternion block is Jp (omega x v))
          gpm_store(d, i, J + 8);
        } else {
#pragma unroll
          for (int k = 0; k < BA_JREC; ++k) d.Jpm[k * Np + i] = J[k];
        }
        // point-side products: Jp^T Jp (upper 6) and Jp^T r
        const double* jp = J + 8;
        val[0] = jp[0] * jp[0] + jp[3] * jp[3];
        val[1] = jp[0] * jp[1] + jp[3] * jp[4];
        val[2] = jp[0] * jp[2] + jp[3] * jp[5];
        val[3] = jp[1] * jp[1] + jp[4] * jp[4];
        val[4] = jp[1] * jp[2] + jp[4] * jp[5];
        val[5] = jp[2] * jp[2] + jp[5] * jp[5];
        val[6] = jp[0] * r[0] + jp[3] * r[1];
        val[7] = jp[1] * r[0] + jp[4] * r[1];
        val[8] = jp[2] * r[0] + jp[5] * r[1];
        val[9] = jp[0] * J[14] + jp[3] * J[15];
        val[10] = jp[1] * J[14] + jp[4] * J[15];
        val[11] = jp[2] * J[14] + jp[5] * J[15];
        if (r_out) {
          const int o = d.topo.pm_obs[i];
          r_out[2ll * o] = r[0];
          r_out[2ll * o + 1] = r[1];
        }
        if (J_out) {
          // reference layout per observation: pose 2x7 | point 2x3 | focal 2x1
          const int o = d.topo.pm_obs[i];
          const int w = d.bp.focal_mode ? 22 : 20;
          double* dst = J_out + (long long)w * o;
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[7 * rr + k] = J[4 * rr + k];
#pragma unroll
            for (int k = 0; k < 3; ++k) dst[7 * rr + 4 + k] = -J[8 + 3 * rr + k];
#pragma unroll
            for (int k = 0; k < 3; ++k) dst[14 + 3 * rr + k] = J[8 + 3 * rr + k];
            if (d.bp.focal_mode) dst[20 + rr] = J[14 + rr];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < LIN_V; ++k) sm[wib][lane][k] = val[k];
      __syncwarp();
      // owner lane sums its point's observations of this round in order
      const int a = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a; o < e; ++o) {
#pragma unroll
        for (int k = 0; k < LIN_V; ++k) acc[k] += sm[wib][o - base][k];
      }
      __syncwarp();
    }
    if (my_pt < pb1) {
      if (d.fpt) {
#pragma unroll
        for (int k = 0; k < 3; ++k) d.fpt[3ll * my_pt + k] = acc[9 + k];
      }
      if (d.Xl) {
        const double* X = theta + d.bp.off_pts + 3ll * my_pt;
        double* xl = d.Xl + 4ll * my_pt;
        xl[0] = X[0]; xl[1] = X[1]; xl[2] = X[2]; xl[3] = 0.0;
      }
      double* C6 = d.Cpt + 6ll * my_pt;
#pragma unroll
      for (int k = 0; k < 6; ++k) C6[k] = acc[k];
      double* g3 = d.gpt + 3ll * my_pt;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        g3[k] = acc[6 + k];
        gn2 += acc[6 + k] * acc[6 + k];
        gmax = fmax(gmax, fabs(acc[6 + k]));
      }
    }
  }
  // per-warp partial of |g|^2 (fixed lane order) and global max
  gn2 = warp_sum(gn2);
  gmax = warp_max(gmax);
  if (lane == 0) {
    gpt_norm_part[gw] = gn2;
    atomic_max_nonneg(d.scal + SC_GMAX, gmax);
  }
}

// ---------------------------------------------------------------------------
// camera side of linearize + jtj/jtr: per camera tile (one CTA, <= 256
// observations of one camera, camera-major order) evaluate the observations
// again with the same compiled body (ba_obs_eval), write the camera-major
// Jacobian copy and residual coalesced, and reduce the tile's Jc^T Jc (36
// upper) and Jc^T r (8). Recomputing costs ~2x the linearize flops but
// replaces 16 scattered 8-byte stores per observation (sector read-modify-
// write: ~8x the bytes) by coalesced ones.
// ---------------------------------------------------------------------------
#define CAM_V 44
__global__ void __launch_bounds__(SSFM_TILE) ba_k_linearize_cm(BADev d, const double* __restrict__ theta) {
  __shared__ double sm[(SSFM_TILE / 32) * CAM_V];
  const int t = blockIdx.x;
  const int o0 = d.topo.tile_obs[t], o1 = d.topo.tile_obs[t + 1];
  const int c = d.topo.tile_cam[t];
  const int i = o0 + threadIdx.x;
  double v[CAM_V];
#pragma unroll
  for (int k = 0; k < CAM_V; ++k) v[k] = 0.0;
  if (i < o1) {
    const long long Np = d.Npad;
    const int j = d.topo.cm_pt[i];
    double r[2], J[BA_JREC], ct, F[BA_FREC + 3];
    ba_obs_eval(d.bp, d.cams + c, theta + d.bp.off_pts + 3ll * j, d.pix_cm + 2ll * i, r, J, &ct,
                d.Fcm ? F : nullptr);
    if (d.Jcm) {
#pragma unroll
      for (int k = 0; k < BA_JREC; ++k) d.Jcm[k * Np + i] = J[k];
    }
    if (d.Fcm) fcm_store(d, i, F, pol_evict_first());
    double a[8], b[8];
    ba_jc_row(J, 0, a);
    ba_jc_row(J, 1, b);
    int idx = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int q = p; q < 8; ++q) v[idx++] = a[p] * a[q] + b[p] * b[q];
#pragma unroll
    for (int p = 0; p < 8; ++p) v[36 + p] = a[p] * r[0] + b[p] * r[1];
  }
  block_reduce<CAM_V>(v, sm);
  if (threadIdx.x == 0) {
    double* dst = d.tilebuf + (long long)CAM_V * t;
#pragma unroll
    for (int k = 0; k < CAM_V; ++k) dst[k] = v[k];
  }
}

// ---------------------------------------------------------------------------
// linearize of omega-form handles in two passes that evaluate each
// observation ONCE (ba_k_linearize + ba_k_linearize_cm evaluate it twice, and
// the point-major one gathers a 192-byte camera cache per observation):
//  * ba_k_lin_tile, one CTA per camera tile (the tile's camera is uniform):
//    residual and Jacobian, the factored record Fcm (coalesced), the
//    point-major Jp + Jf record Gpm[8] and residual Rpm[4] (whole 64- / 32-
//    byte sectors at the observation's point-major position: no partial-
//    sector writes), and the tile's Jc^T Jc / Jc^T r (as ba_k_linearize_cm);
//  * ba_k_lin_points, one warp per point batch: Jp^T Jp, Jp^T r (and
//    Jp^T Jf) summed per point in observation order from Gpm / Rpm, as
//    ba_k_linearize does (the same values: the records are bit-identical).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ba_precond_f_entry(const double* cb, const double* w, int o);
#ifndef LIN_TR
#define LIN_TR 1   // warp transpose-reduction of the tile-group sums (C5 non-PCG 7.2 -> 5.9 ms per LM iteration)
#endif
#ifndef LIN_MINB
#define LIN_MINB (LIN_TR ? 2 : 1)   // CTAs per SM of ba_k_lin_tile (TR: 128 registers, no spills)
#endif
#ifndef LIN_STPOL
#define LIN_STPOL 1   // C5 non-PCG 5.62 -> 5.50 ms per LM iteration (profiles/r2b/ab_linearize_store_policy_c5.log)
#endif
#ifndef LIN_PF
#define LIN_PF 1   // ba_k_lin_tile / ba_k_precond_grp: point indices one step ahead
#endif
// one observation of ba_k_lin_tile: records out, its rows a, b of Jc and
// residual r (j = its point, ip = its point-major position)
__device__ __forceinline__ void ba_lin_obs_rows(const BADev& d, const double* __restrict__ theta, int c, long long i,
                                                int j, int ip, double* a, double* b, double* r) {
  const unsigned long long pst = pol_evict_first();
  double J[BA_JREC], ct, F[BA_FREC + 3];
  ba_obs_eval(d.bp, d.cams + c, theta + d.bp.off_pts + 3ll * j, d.pix_cm + 2ll * i, r, J, &ct, F);
  fcm_store(d, i, F, pst);   // pinhole: s01, s11 are implied
#if LIN_STPOL && GPM_AOS   // the scattered point-major records leave L2 first (the X gathers stay)
  st_v4_hint(d.Gpm + 8ll * ip, J[8], J[9], J[10], J[11], pst);
  st_v4_hint(d.Gpm + 8ll * ip + 4, J[12], J[13], J[14], J[15], pst);
  st_v4_hint(d.Rpm + 4ll * ip, r[0], r[1], 0.0, 0.0, pst);
#else
  gpm_store(d, ip, J + 8);
  *reinterpret_cast<double4*>(d.Rpm + 4ll * ip) = make_double4(r[0], r[1], 0.0, 0.0);
#endif
  ba_jc_row(J, 0, a);
  ba_jc_row(J, 1, b);
}
// ... and its J^T J / J^T r terms added to v
__device__ __forceinline__ void ba_lin_obs(const BADev& d, const double* __restrict__ theta, int c, long long i,
                                           int j, int ip, double* v) {
  double a[8], b[8], r[2];
  ba_lin_obs_rows(d, theta, c, i, j, ip, a, b, r);
  int idx = 0;
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int q = p; q < 8; ++q) v[idx++] += a[p] * a[q] + b[p] * b[q];
#pragma unroll
  for (int p = 0; p < 8; ++p) v[36 + p] += a[p] * r[0] + b[p] * r[1];
}

// ---------------------------------------------------------------------------
// Warp transpose-reduction of the 44 per-observation terms of a camera tile
// group (36 upper entries of an 8x8 block + an 8-vector), for the tile-group
// kernels of linearize and the preconditioner (LIN_TR). Each lane evaluates
// its observation's terms on demand (prod(k)); a halving butterfly leaves lane
// l with the warp sum of term l (terms 0..31) and lanes 2m, 2m+1 with the sum
// of term 32 + m: 47 shuffles per 32 observations, and 2 accumulators per lane
// across the loop instead of 44 (the scalar kernels hold 44 and run at 232 /
// 196 registers, 8 warps per SM). Fixed order: deterministic.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void warp_tr44_add(const double (&t)[CAM_V], double& acc1, double& acc2) {
  const int lane = threadIdx.x & 31;
  {   // terms 0..31
    double x[16];
    const bool h4 = lane & 16;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const double lo = t[m], hi = t[m + 16];
      x[m] = (h4 ? hi : lo) + __shfl_xor_sync(SSFM_FULL, h4 ? lo : hi, 16);
    }
#pragma unroll
    for (int w = 8, o = 8; w >= 1; w >>= 1, o >>= 1) {
      const bool hb = lane & o;
#pragma unroll
      for (int m = 0; m < w; ++m) {
        const double lo = x[m], hi = x[m + w];
        x[m] = (hb ? hi : lo) + __shfl_xor_sync(SSFM_FULL, hb ? lo : hi, o);
      }
    }
    acc1 += x[0];
  }
  {   // terms 32..43 (padded to 16)
    double x[8];
    const bool h4 = lane & 16;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const double lo = t[32 + m], hi = 40 + m < CAM_V ? t[40 + m] : 0.0;
      x[m] = (h4 ? hi : lo) + __shfl_xor_sync(SSFM_FULL, h4 ? lo : hi, 16);
    }
#pragma unroll
    for (int w = 4, o = 8; w >= 1; w >>= 1, o >>= 1) {
      const bool hb = lane & o;
#pragma unroll
      for (int m = 0; m < w; ++m) {
        const double lo = x[m], hi = x[m + w];
        x[m] = (hb ? hi : lo) + __shfl_xor_sync(SSFM_FULL, hb ? lo : hi, o);
      }
    }
    acc2 += x[0] + __shfl_xor_sync(SSFM_FULL, x[0], 1);
  }
}
// per-lane accumulators of every warp -> the 44 group sums (warp order) in smw
__device__ __forceinline__ void tr44_block_sum(double acc1, double acc2, double (*sred)[48], double* smw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  sred[wid][lane] = acc1;
  if (!(lane & 1)) sred[wid][32 + (lane >> 1)] = acc2;
  __syncthreads();
  if (threadIdx.x < CAM_V) {
    double x = sred[0][threadIdx.x];
    for (int w = 1; w < nw; ++w) x += sred[w][threadIdx.x];
    smw[threadIdx.x] = x;
  }
  __syncthreads();
}

// per tile group (topo.grp_tile: up to SSFM_GRP tiles of one camera; the
// camera is uniform, so no per-observation camera gather): every observation
// evaluated once; its records written; the group's J^T J / J^T r reduced
// once into its first tile's slot (the other tiles' slots zero)
__global__ void __launch_bounds__(SSFM_TILE, LIN_MINB) ba_k_lin_tile(BADev d, const double* __restrict__ theta) {
  __shared__ double smw[CAM_V];
  const int g = blockIdx.x;
  const int t0 = d.topo.grp_tile[g], t1 = d.topo.grp_tile[g + 1];
  const int o0 = d.topo.tile_obs[t0], o1 = d.topo.tile_obs[t1];
  const int c = d.topo.tile_cam[t0];
#if LIN_TR
  __shared__ double sred[SSFM_TILE / 32][48];
  const unsigned long long pst = pol_evict_first();
  const int lane = threadIdx.x & 31, wbase = o0 + (int)(threadIdx.x & ~31u);
  double acc1 = 0.0, acc2 = 0.0;
  int jn = 0, ipn = 0;
  if (wbase + lane < o1) {
    jn = ldg_stream_i(d.topo.cm_pt + wbase + lane, pst);
    ipn = ldg_stream_i(d.topo.cm_to_pm + wbase + lane, pst);
  }
  for (int base = wbase; base < o1; base += blockDim.x) {   // warp-uniform
    const int i = base + lane;
    const int j = jn, ip = ipn;
    if (i + (int)blockDim.x < o1) {
      jn = ldg_stream_i(d.topo.cm_pt + i + blockDim.x, pst);
      ipn = ldg_stream_i(d.topo.cm_to_pm + i + blockDim.x, pst);
    }
    double a[8], b[8], r[2] = {0.0, 0.0};
    if (i < o1) {
      ba_lin_obs_rows(d, theta, c, i, j, ip, a, b, r);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) { a[k] = 0.0; b[k] = 0.0; }
    }
    double t[CAM_V];
    int idx = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int q = p; q < 8; ++q) t[idx++] = a[p] * a[q] + b[p] * b[q];
#pragma unroll
    for (int p = 0; p < 8; ++p) t[36 + p] = a[p] * r[0] + b[p] * r[1];
    warp_tr44_add(t, acc1, acc2);
  }
  tr44_block_sum(acc1, acc2, sred, smw);
#else
  __shared__ double sm[(SSFM_TILE / 32) * CAM_V];
  double v[CAM_V];
#pragma unroll
  for (int k = 0; k < CAM_V; ++k) v[k] = 0.0;
#if LIN_PF   // the next observation's point index and point-major position one step ahead
  const unsigned long long pst = pol_evict_first();
  int jn = 0, ipn = 0;
  if (o0 + (int)threadIdx.x < o1) {
    jn = ldg_stream_i(d.topo.cm_pt + o0 + threadIdx.x, pst);
    ipn = ldg_stream_i(d.topo.cm_to_pm + o0 + threadIdx.x, pst);
  }
  for (int i = o0 + threadIdx.x; i < o1; i += blockDim.x) {
    const int j = jn, ip = ipn;
    if (i + (int)blockDim.x < o1) {
      jn = ldg_stream_i(d.topo.cm_pt + i + blockDim.x, pst);
      ipn = ldg_stream_i(d.topo.cm_to_pm + i + blockDim.x, pst);
    }
    ba_lin_obs(d, theta, c, i, j, ip, v);
  }
#else
  for (int i = o0 + threadIdx.x; i < o1; i += blockDim.x) ba_lin_obs(d, theta, c, i, d.topo.cm_pt[i], d.topo.cm_to_pm[i], v);
#endif
  block_reduce<CAM_V>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < CAM_V; ++k) smw[k] = v[k];
  }
  __syncthreads();
#endif
  if (threadIdx.x < 64) {
    double* dst = d.tilebuf + (long long)CAM_V * t0;
    for (int o = threadIdx.x; o < CAM_V; o += 64) dst[o] = smw[o];
  } else {
    for (int k = threadIdx.x - 64; k < CAM_V * (t1 - t0 - 1); k += blockDim.x - 64)
      d.tilebuf[(long long)CAM_V * (t0 + 1) + k] = 0.0;
  }
}

__global__ void __launch_bounds__(256) ba_k_lin_points(BADev d, const double* __restrict__ theta,
                                                       double* gpt_norm_part) {
  __shared__ __align__(16) double sm[8][SSFM_BATCH][LIN_V];
  const int nv2 = d.fpt ? LIN_V / 2 : 5;   // Jp^T jf only for the shared focal: 9 of the 12 values
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long pst = pol_evict_first();
  double gn2 = 0.0, gmax = 0.0;
  for (int b = gw; b < d.topo.nb; b += warps) {
    const int ob0 = d.topo.bat_obs[b], ob1 = d.topo.bat_obs[b + 1];
    const int pb0 = d.topo.bat_pt[b], pb1 = d.topo.bat_pt[b + 1];
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    if (my_pt < pb1) { ps = d.topo.pt_seg[my_pt]; pe = d.topo.pt_seg[my_pt + 1]; }
    double acc[LIN_V];
#pragma unroll
    for (int k = 0; k < LIN_V; ++k) acc[k] = 0.0;
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[LIN_V];
#pragma unroll
      for (int k = 0; k < LIN_V; ++k) val[k] = 0.0;
      if (i < ob1) {
        double G[8], r[4];
        gpm_load(d, i, G, pst);
        ld_v4_ro(d.Rpm + 4ll * i, r, pst);
        const double* jp = G;
        val[0] = jp[0] * jp[0] + jp[3] * jp[3];
        val[1] = jp[0] * jp[1] + jp[3] * jp[4];
        val[2] = jp[0] * jp[2] + jp[3] * jp[5];
        val[3] = jp[1] * jp[1] + jp[4] * jp[4];
        val[4] = jp[1] * jp[2] + jp[4] * jp[5];
        val[5] = jp[2] * jp[2] + jp[5] * jp[5];
        val[6] = jp[0] * r[0] + jp[3] * r[1];
        val[7] = jp[1] * r[0] + jp[4] * r[1];
        val[8] = jp[2] * r[0] + jp[5] * r[1];
        val[9] = jp[0] * G[6] + jp[3] * G[7];
        val[10] = jp[1] * G[6] + jp[4] * G[7];
        val[11] = jp[2] * G[6] + jp[5] * G[7];
      }
#if LP_V2   // 16-byte shared-memory accesses (half the L1 wavefronts of 8-byte ones: L1/TEX bound)
      double2* row = reinterpret_cast<double2*>(&sm[wib][lane][0]);
#pragma unroll
      for (int k = 0; k < LIN_V / 2; ++k)
        if (k < nv2) row[k] = make_double2(val[2 * k], val[2 * k + 1]);
      __syncwarp();
      const int a = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a; o < e; ++o) {
        const double2* src = reinterpret_cast<const double2*>(&sm[wib][o - base][0]);
#pragma unroll
        for (int k = 0; k < LIN_V / 2; ++k) {
          if (k < nv2) {
            const double2 x = src[k];
            acc[2 * k] += x.x;
            acc[2 * k + 1] += x.y;
          }
        }
      }
#else
#pragma unroll
      for (int k = 0; k < LIN_V; ++k) sm[wib][lane][k] = val[k];
      __syncwarp();
      const int a = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a; o < e; ++o) {
#pragma unroll
        for (int k = 0; k < LIN_V; ++k) acc[k] += sm[wib][o - base][k];
      }
#endif
      __syncwarp();
    }
    if (my_pt < pb1) {
      if (d.fpt) {
#pragma unroll
        for (int k = 0; k < 3; ++k) d.fpt[3ll * my_pt + k] = acc[9 + k];
      }
      const double* X = theta + d.bp.off_pts + 3ll * my_pt;
      *reinterpret_cast<double4*>(d.Xl + 4ll * my_pt) = make_double4(X[0], X[1], X[2], 0.0);
      double* C6 = d.Cpt + 6ll * my_pt;
#pragma unroll
      for (int k = 0; k < 6; ++k) C6[k] = acc[k];
      double* g3 = d.gpt + 3ll * my_pt;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        g3[k] = acc[6 + k];
        gn2 += acc[6 + k] * acc[6 + k];
        gmax = fmax(gmax, fabs(acc[6 + k]));
      }
    }
  }
  gn2 = warp_sum(gn2);
  gmax = warp_max(gmax);
  if (lane == 0) {
    gpt_norm_part[gw] = gn2;
    atomic_max_nonneg(d.scal + SC_GMAX, gmax);
  }
}

// cost over camera tiles (the tile's camera uniform, no per-observation
// camera gather): one partial per tile, summed in tile order
__global__ void __launch_bounds__(SSFM_TILE) ba_k_cost_tile(BADev d, const double* __restrict__ theta,
                                                            double* partials) {
  __shared__ double sm[32];
  const int t = blockIdx.x;
  const int o0 = d.topo.tile_obs[t], o1 = d.topo.tile_obs[t + 1];
  const int i = o0 + threadIdx.x;
  double v[1] = {0.0};
  if (i < o1) {
    const BACam cc = d.cams[d.topo.tile_cam[t]];
    const int j = d.topo.cm_pt[i];
    BAProj pr;
    double r[2], sw, ct;
    ba_residual(d.bp, cc, theta + d.bp.off_pts + 3ll * j, d.pix_cm + 2ll * i, pr, r, sw, ct);
    v[0] = ct;
  }
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) partials[t] = v[0];
}

// per camera: sum of its tile partials in tile order (the local part of a
// camera block when the observations are sharded over ranks)
__global__ void k_cam_tilesum(const Topo T, const double* __restrict__ tilebuf, int V, double* camsum) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= T.C) return;
  for (int k = 0; k < V; ++k) {
    double s = 0.0;
    for (int t = T.cam_tile[c]; t < T.cam_tile[c + 1]; ++t) s += tilebuf[(long long)V * t + k];
    camsum[(long long)V * c + k] = s;
  }
}

// camsum != nullptr: per-camera sums already reduced over ranks (k_cam_tilesum
// + allreduce); otherwise the local tiles are summed here.
__device__ __forceinline__ void cam_sums(const BADev& d, int c, const double* camsum, double* s) {
  if (camsum) {
#pragma unroll
    for (int k = 0; k < CAM_V; ++k) s[k] = camsum[(long long)CAM_V * c + k];
    return;
  }
#pragma unroll
  for (int k = 0; k < CAM_V; ++k) s[k] = 0.0;
  for (int t = d.topo.cam_tile[c]; t < d.topo.cam_tile[c + 1]; ++t) {
    const double* src = d.tilebuf + (long long)CAM_V * t;
#pragma unroll
    for (int k = 0; k < CAM_V; ++k) s[k] += src[k];
  }
}

__global__ void ba_k_camfin(BADev d, double* cam_norm_part, const double* camsum) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  double gn2 = 0.0, gmax = 0.0;
  if (c < d.bp.C) {
    double s[CAM_V];
    cam_sums(d, c, camsum, s);
    double* B = d.Bc + 64ll * c;
    int idx = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int q = p; q < 8; ++q) { B[8 * p + q] = s[idx]; B[8 * q + p] = s[idx]; ++idx; }
    double* g = d.gcam + 8ll * c;
    const int nown = d.bp.focal_mode == 2 ? 7 : 8;   // shared focal: summed over cameras later
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      g[p] = s[36 + p];
      if (p < nown) {
        gn2 += s[36 + p] * s[36 + p];
        gmax = fmax(gmax, fabs(s[36 + p]));
      }
    }
  }
  double v[1] = {gn2};
  __shared__ double sm[32];
  const double gm = warp_max(gmax);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(d.scal + SC_GMAX, gm);
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) cam_norm_part[blockIdx.x] = v[0];
}

// ---------------------------------------------------------------------------
// damped point blocks (apply_damping + _invert_elim_blocks, lm.py:495-513,
// sparse_block.py:406-426): Cinv = (C diag*(1+lam))^-1, y0 = Cinv b_j, b = -g.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool inv_sym3(const double* m, double* inv, double& det) {
  const double c00 = m[3] * m[5] - m[4] * m[4];
  const double c01 = m[2] * m[4] - m[1] * m[5];
  const double c02 = m[1] * m[4] - m[2] * m[3];
  det = m[0] * c00 + m[1] * c01 + m[2] * c02;
  if (!(det > 0.0) || !isfinite(det)) return false;
  const double id = 1.0 / det;
  inv[0] = c00 * id;
  inv[1] = c01 * id;
  inv[2] = c02 * id;
  inv[3] = (m[0] * m[5] - m[2] * m[2]) * id;
  inv[4] = (m[1] * m[2] - m[0] * m[4]) * id;
  inv[5] = (m[0] * m[3] - m[1] * m[1]) * id;
  return true;
}

__device__ __forceinline__ void ptinv_focal_part(const BADev& d, int j, const double* inv) {
  // shared focal: a_j^T Cinv_j a_j, block partials in block order (fixed tree)
  __shared__ double sm[32];
  double v[1] = {0.0};
  if (j < d.bp.P) {
    const double* a = d.fpt + 3ll * j;
    double w[3];
    sym3_matvec(inv, a, w);
    v[0] = a[0] * w[0] + a[1] * w[1] + a[2] * w[2];
  }
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) d.fwpart[blockIdx.x] = v[0];
}

__global__ void ba_k_ptinv(BADev d, double lam) {
  if (d.lamp) lam = *d.lamp;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double inv[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (j < d.bp.P) {
    double m[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) m[k] = d.Cpt[6ll * j + k];
    const double s = 1.0 + lam;
    m[0] *= s; m[3] *= s; m[5] *= s;
    double b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) b[k] = -d.gpt[3ll * j + k];
    const int di[3] = {0, 3, 5};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (m[di[k]] == 0.0) {
        if (b[k] != 0.0) atomicOr(d.status, ST_PIN_POINT);
        m[di[k]] = 1.0;
      }
    }
    double det;
    if (!inv_sym3(m, inv, det)) {
      atomicOr(d.status, ST_SINGULAR_POINT);
#pragma unroll
      for (int k = 0; k < 6; ++k) inv[k] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) d.Cinv[6ll * j + k] = inv[k];
    double y[3];
    sym3_matvec(inv, b, y);
#pragma unroll
    for (int k = 0; k < 3; ++k) d.y0[3ll * j + k] = y[k];
  }
  // every thread of the block, one code path (the reduction uses full-warp
  // shuffles and __syncthreads)
  if (d.fpt) ptinv_focal_part(d, j, inv);
}

// ---------------------------------------------------------------------------
// Schur preconditioner blocks and reduced rhs, per camera tile:
//   sum_o E_o Cinv_j E_o^T  (E_o = Jc^T Jp, 8x3)   -> 36 upper
//   sum_o E_o y0_j                                 -> 8
// (the diagonal slots of schur_fill_cy and b_red, lm.py:608-626)
// ---------------------------------------------------------------------------
// Factored form (two-pass handles, no Jcm): the rows of Jc in the camera
// frame, a~_r = [D(v)^T (SE)_r ; -(SE)_r ; phi e_r], are reduced over the
// tile and mapped once per tile by T = diag(Pi, R^T, 1): W = T W~ T^T.
// accumulates observation i's terms into v (the tile's camera cache cb)
// observation i's camera-frame rows a, b of Jc, K = Jp Cinv_j Jp^T (k00, k01,
// k11) and Jp y0_j (ty0, ty1); j = the observation's point
__device__ __forceinline__ void ba_precond_rows(const BADev& d, long long i, int j, const double* cb, double* a,
                                                double* b, double& k00, double& k01, double& k11, double& ty0,
                                                double& ty1) {
  double f[6], vv[3];
  fcm_load(d, i, f, vv, pol_evict_first());
  double qh[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) qh[k] = cb[9 + k];
  const double se[2][3] = {{f[0], f[4], -(f[0] * f[1] + f[4] * f[2])},
                           {f[4], f[5], -(f[4] * f[1] + f[5] * f[2])}};
  {
    double ci[6], y[3];
#pragma unroll
    for (int k = 0; k < 6; ++k) ci[k] = d.Cinv[6ll * j + k];
#pragma unroll
    for (int k = 0; k < 3; ++k) y[k] = d.y0[3ll * j + k];
    double jp[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k) jp[r][k] = se[r][0] * cb[k] + se[r][1] * cb[3 + k] + se[r][2] * cb[6 + k];
    double w0[3], w1[3];
    sym3_matvec(ci, jp[0], w0);
    sym3_matvec(ci, jp[1], w1);
    k00 = jp[0][0] * w0[0] + jp[0][1] * w0[1] + jp[0][2] * w0[2];
    k01 = jp[1][0] * w0[0] + jp[1][1] * w0[1] + jp[1][2] * w0[2];
    k11 = jp[1][0] * w1[0] + jp[1][1] * w1[1] + jp[1][2] * w1[2];
    ty0 = jp[0][0] * y[0] + jp[0][1] * y[1] + jp[0][2] * y[2];
    ty1 = jp[1][0] * y[0] + jp[1][1] * y[1] + jp[1][2] * y[2];
  }
  ba_dqt_mul(qh, vv, se[0], a);
  ba_dqt_mul(qh, vv, se[1], b);
#pragma unroll
  for (int k = 0; k < 3; ++k) { a[4 + k] = -se[0][k]; b[4 + k] = -se[1][k]; }
  a[7] = f[3] * f[1];
  b[7] = f[3] * f[2];
}
__device__ __forceinline__ void ba_precond_f(const BADev& d, long long i, int j, const double* cb, double* v) {
  double a[8], b[8], k00, k01, k11, ty0, ty1;
  ba_precond_rows(d, i, j, cb, a, b, k00, k01, k11, ty0, ty1);
  double ka[8], kb[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) { ka[p] = k00 * a[p] + k01 * b[p]; kb[p] = k01 * a[p] + k11 * b[p]; }
  int idx = 0;
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int q = p; q < 8; ++q) v[idx++] += a[p] * ka[q] + b[p] * kb[q];
#pragma unroll
  for (int p = 0; p < 8; ++p) v[36 + p] += a[p] * ty0 + b[p] * ty1;
}


// W = T W~ T^T, u = T u~ for the tile's camera, T = diag(Pi, R^T, 1): one
// output entry per lane of warp 0 (packed upper 36 + 8), from W~ in shared
__device__ __forceinline__ double ba_precond_t(const double* cb, int p, int a) {
  if (p < 4) return a < 4 ? ((p == a ? 1.0 : 0.0) - cb[9 + p] * cb[9 + a]) * cb[22] : 0.0;
  if (p < 7) return (a >= 4 && a < 7) ? cb[3 * (a - 4) + (p - 4)] : 0.0;   // R^T
  return a == 7 ? 1.0 : 0.0;
}
__device__ __forceinline__ int ba_pk(int a, int b) {   // packed upper index, a <= b
  return a * 8 - a * (a - 1) / 2 + (b - a);
}
__device__ __forceinline__ void ba_blk(int p, int* lo, int* hi) {
  if (p < 4) { *lo = 0; *hi = 4; } else if (p < 7) { *lo = 4; *hi = 7; } else { *lo = 7; *hi = 8; }
}
__device__ __forceinline__ double ba_precond_f_entry(const double* cb, const double* w, int o) {
  if (o >= 36) {
    const int p = o - 36;
    int lo, hi;
    ba_blk(p, &lo, &hi);
    double sacc = 0.0;
    for (int a = lo; a < hi; ++a) sacc += ba_precond_t(cb, p, a) * w[36 + a];
    return sacc;
  }
  int p = 0, rem = o;
  while (rem >= 8 - p) { rem -= 8 - p; ++p; }
  const int q = p + rem;
  int pl, ph, ql, qh_;
  ba_blk(p, &pl, &ph);
  ba_blk(q, &ql, &qh_);
  double sacc = 0.0;
  for (int a = pl; a < ph; ++a) {
    const double tpa = ba_precond_t(cb, p, a);
    for (int b = ql; b < qh_; ++b) {
      const double wab = a <= b ? w[ba_pk(a, b)] : w[ba_pk(b, a)];
      sacc += tpa * wab * ba_precond_t(cb, q, b);
    }
  }
  return sacc;
}

__global__ void __launch_bounds__(SSFM_TILE) ba_k_precond(BADev d) {
  __shared__ double sm[(SSFM_TILE / 32) * CAM_V];
  const int t = blockIdx.x;
  const int o0 = d.topo.tile_obs[t], o1 = d.topo.tile_obs[t + 1];
  const int i = o0 + threadIdx.x;
  double v[CAM_V];
#pragma unroll
  for (int k = 0; k < CAM_V; ++k) v[k] = 0.0;
  if (!d.Jcm) return;   // factored records: ba_k_precond_grp
  if (i < o1) {
    const long long Np = d.Npad;
    double J[BA_JREC];
#pragma unroll
    for (int k = 0; k < BA_JREC; ++k) J[k] = d.Jcm[k * Np + i];
    const int j = d.topo.cm_pt[i];
    double ci[6], y[3];
#pragma unroll
    for (int k = 0; k < 6; ++k) ci[k] = d.Cinv[6ll * j + k];
#pragma unroll
    for (int k = 0; k < 3; ++k) y[k] = d.y0[3ll * j + k];
    // K = Jp Cinv Jp^T (2x2)
    const double* jp = J + 8;
    double w0[3], w1[3];
    sym3_matvec(ci, jp, w0);
    sym3_matvec(ci, jp + 3, w1);
    const double k00 = jp[0] * w0[0] + jp[1] * w0[1] + jp[2] * w0[2];
    const double k01 = jp[3] * w0[0] + jp[4] * w0[1] + jp[5] * w0[2];
    const double k11 = jp[3] * w1[0] + jp[4] * w1[1] + jp[5] * w1[2];
    double a[8], b[8];
    ba_jc_row(J, 0, a);
    ba_jc_row(J, 1, b);
    double ka[8], kb[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) { ka[p] = k00 * a[p] + k01 * b[p]; kb[p] = k01 * a[p] + k11 * b[p]; }
    int idx = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int q = p; q < 8; ++q) v[idx++] = a[p] * ka[q] + b[p] * kb[q];
    double ty[2];
    ba_jp_mul(J, y, ty);
#pragma unroll
    for (int p = 0; p < 8; ++p) v[36 + p] = a[p] * ty[0] + b[p] * ty[1];
  }
  block_reduce<CAM_V>(v, sm);
  if (threadIdx.x == 0) {
    double* dst = d.tilebuf + (long long)CAM_V * t;
#pragma unroll
    for (int k = 0; k < CAM_V; ++k) dst[k] = v[k];
  }
}

// Factored preconditioner terms per tile GROUP (up to SSFM_GRP consecutive
// tiles of one camera, topo.grp_tile): each thread accumulates several
// observations, one block reduction and one mapping through
// T = diag(Pi, R^T, 1) per group instead of per tile. The group's sums land
// in its first tile's slot; its other tiles' slots are zero (the per-camera
// sums over tiles are unchanged).
#ifndef PRE_MINB
#define PRE_MINB (LIN_TR ? 2 : 1)   // CTAs per SM (scalar sums at 2: spills)
#endif
__global__ void __launch_bounds__(SSFM_TILE, PRE_MINB) ba_k_precond_grp(BADev d) {
  __shared__ double smw[CAM_V];
  const int g = blockIdx.x;
  const int t0 = d.topo.grp_tile[g], t1 = d.topo.grp_tile[g + 1];
  const int o0 = d.topo.tile_obs[t0], o1 = d.topo.tile_obs[t1];
  const double* cb = reinterpret_cast<const double*>(d.camlin + d.topo.tile_cam[t0]);
#if LIN_TR
  __shared__ double sred[SSFM_TILE / 32][48];
  const unsigned long long pst = pol_evict_first();
  const int lane = threadIdx.x & 31, wbase = o0 + (int)(threadIdx.x & ~31u);
  double acc1 = 0.0, acc2 = 0.0;
  int jn = wbase + lane < o1 ? ldg_stream_i(d.topo.cm_pt + wbase + lane, pst) : 0;
  for (int base = wbase; base < o1; base += blockDim.x) {   // warp-uniform
    const int i = base + lane;
    const int j = jn;
    if (i + (int)blockDim.x < o1) jn = ldg_stream_i(d.topo.cm_pt + i + blockDim.x, pst);
    double a[8], b[8], k00 = 0.0, k01 = 0.0, k11 = 0.0, ty0 = 0.0, ty1 = 0.0;
    if (i < o1) {
      ba_precond_rows(d, i, j, cb, a, b, k00, k01, k11, ty0, ty1);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) { a[k] = 0.0; b[k] = 0.0; }
    }
    double ka[8], kb[8], t[CAM_V];
#pragma unroll
    for (int p = 0; p < 8; ++p) { ka[p] = k00 * a[p] + k01 * b[p]; kb[p] = k01 * a[p] + k11 * b[p]; }
    int idx = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int q = p; q < 8; ++q) t[idx++] = a[p] * ka[q] + b[p] * kb[q];
#pragma unroll
    for (int p = 0; p < 8; ++p) t[36 + p] = a[p] * ty0 + b[p] * ty1;
    warp_tr44_add(t, acc1, acc2);
  }
  tr44_block_sum(acc1, acc2, sred, smw);
#else
  __shared__ double sm[(SSFM_TILE / 32) * CAM_V];
  double v[CAM_V];
#pragma unroll
  for (int k = 0; k < CAM_V; ++k) v[k] = 0.0;
#if LIN_PF
  const unsigned long long pst = pol_evict_first();
  int jn = o0 + (int)threadIdx.x < o1 ? ldg_stream_i(d.topo.cm_pt + o0 + threadIdx.x, pst) : 0;
  for (int i = o0 + threadIdx.x; i < o1; i += blockDim.x) {
    const int j = jn;
    if (i + (int)blockDim.x < o1) jn = ldg_stream_i(d.topo.cm_pt + i + blockDim.x, pst);
    ba_precond_f(d, i, j, cb, v);
  }
#else
  for (int i = o0 + threadIdx.x; i < o1; i += blockDim.x) ba_precond_f(d, i, d.topo.cm_pt[i], cb, v);
#endif
  block_reduce<CAM_V>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < CAM_V; ++k) smw[k] = v[k];
  }
  __syncthreads();
#endif
  if (threadIdx.x < 64) {
    double* dst = d.tilebuf + (long long)CAM_V * t0;
    for (int o = threadIdx.x; o < CAM_V; o += 64) dst[o] = ba_precond_f_entry(cb, smw, o);
  } else {
    for (int k = threadIdx.x - 64; k < CAM_V * (t1 - t0 - 1); k += blockDim.x - 64)
      d.tilebuf[(long long)CAM_V * (t0 + 1) + k] = 0.0;
  }
}

// Gauss-Jordan inverse with partial pivoting (n <= 8), like LAPACK getrf/getri
// used by np.linalg.inv. Returns false on an exactly zero pivot or non-finite.
__device__ bool gj_inverse(double* a, double* inv, int n, int lda) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) inv[i * lda + j] = (i == j) ? 1.0 : 0.0;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    double best = fabs(a[col * lda + col]);
    for (int r = col + 1; r < n; ++r) {
      double v = fabs(a[r * lda + col]);
      if (v > best) { best = v; piv = r; }
    }
    if (!(best > 0.0)) return false;
    if (piv != col) {
      for (int k = 0; k < n; ++k) {
        double t = a[col * lda + k]; a[col * lda + k] = a[piv * lda + k]; a[piv * lda + k] = t;
        t = inv[col * lda + k]; inv[col * lda + k] = inv[piv * lda + k]; inv[piv * lda + k] = t;
      }
    }
    const double ip = 1.0 / a[col * lda + col];
    for (int k = 0; k < n; ++k) { a[col * lda + k] *= ip; inv[col * lda + k] *= ip; }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = a[r * lda + col];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        a[r * lda + k] -= f * a[col * lda + k];
        inv[r * lda + k] -= f * inv[col * lda + k];
      }
    }
  }
  for (int i = 0; i < n * lda; ++i)
    if (!isfinite(inv[i])) return false;
  return true;
}

// per camera: S_cc = B_c(damped) - sum E Cinv E^T, b_red = b_c - sum E y0,
// pinning (lm.py:628-635), block-Jacobi factors for the 7x7 pose block and the
// 1x1 focal block separately (lm.py:473-483, 516-527).
__global__ void ba_k_camprec(BADev d, double lam, const double* camsum) {
  if (d.lamp) lam = *d.lamp;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d.bp.C) return;
  double s[CAM_V];
  cam_sums(d, c, camsum, s);
  const double* B = d.Bc + 64ll * c;
  double S[64];
  int idx = 0;
  for (int p = 0; p < 8; ++p)
    for (int q = p; q < 8; ++q) {
      double bpq = B[8 * p + q];
      if (p == q) bpq *= (1.0 + lam);
      const double v = bpq - s[idx++];
      S[8 * p + q] = v;
      S[8 * q + p] = v;
    }
  double br[8];
  for (int p = 0; p < 8; ++p) br[p] = -d.gcam[8ll * c + p] - s[36 + p];
  unsigned pin = 0;
  for (int p = 0; p < 8; ++p) {
    if (p == 7 && d.bp.focal_mode == 2) continue;   // shared focal: decided over all cameras
    if (S[9 * p] == 0.0) {
      // a zero diagonal of a PSD matrix implies a zero row: pin it (lm.py:628-635)
      if (br[p] != 0.0) atomicOr(d.status, ST_PIN_RETAINED);
      pin |= 1u << p;
      S[9 * p] = 1.0;
    }
  }
  if (d.bp.focal_mode == 2) {
    // shared focal: this camera's share of the 1x1 focal block and of its rhs;
    // ba_k_shared_focal_prec sums the shares and decides the pin
    d.fterm[2ll * c] = B[63] * (1.0 + lam);   // the point terms are not per camera:
    d.fterm[2ll * c + 1] = br[7];             // a_j couples every camera of point j
    pin = (pin & 0x7fu) | 0x80u;
    br[7] = 0.0;
  }
  d.pinned[c] = (unsigned char)pin;
  for (int p = 0; p < 8; ++p) d.bred[8ll * c + p] = (pin >> p & 1u) ? 0.0 : br[p];
  double A[49], I7[49];
  for (int p = 0; p < 7; ++p)
    for (int q = 0; q < 7; ++q) A[7 * p + q] = S[8 * p + q];
  double* M = d.Minv + 64ll * c;
  const bool ok = gj_inverse(A, I7, 7, 7);
  if (!ok) atomicOr(d.status, ST_SINGULAR_PRECOND);
  for (int p = 0; p < 8; ++p)
    for (int q = 0; q < 8; ++q) M[8 * p + q] = (p < 7 && q < 7 && ok) ? I7[7 * p + q] : 0.0;
  if (d.bp.focal_mode == 2) { M[63] = 1.0; return; }
  const double s77 = S[63];
  const double f = 1.0 / s77;
  if (!isfinite(f)) atomicOr(d.status, ST_SINGULAR_PRECOND);
  M[63] = f;
}

// Shared focal (ba.py:49, 61): one retained scalar coupled to every camera.
// Its damped Schur diagonal is the sum of the cameras' damped focal diagonals
// minus sum_j a_j^T Cinv_j a_j (a_j = sum over ALL observations of point j of
// Jp^T jf: the cross terms between cameras are part of it); its reduced rhs is
// the sum of the cameras' shares. Summed in fixed order (one block); pinned if
// the diagonal is exactly zero
// (lm.py:628-635), and set its 1x1 block-Jacobi factor (lm.py:516-527).
// wsum != nullptr: the point part summed over every rank's points (sharded).
__global__ void ba_k_shared_focal_prec(BADev d, int nwpart, const double* wsum) {
  __shared__ double sm[96];
  double v[3] = {0.0, 0.0, 0.0};
  const int C = d.bp.C;
  const int per = (C + blockDim.x - 1) / blockDim.x;
  const int a = threadIdx.x * per, b = min(C, a + per);
  for (int c = a; c < b; ++c) { v[0] += d.fterm[2ll * c]; v[1] += d.fterm[2ll * c + 1]; }
  if (!wsum) {
    const int perw = (nwpart + blockDim.x - 1) / blockDim.x;
    const int aw = threadIdx.x * perw, bw = min(nwpart, aw + perw);
    for (int k = aw; k < bw; ++k) v[2] += d.fwpart[k];
  }
  block_reduce<3>(v, sm);
  if (threadIdx.x == 0) {
    // S_ff = A_ff (1 + lam) - sum_j a_j^T Cinv_j a_j  (lm.py:608-626 for the focal row)
    const double sff = v[0] - (wsum ? *wsum : v[2]), bf = v[1];
    if (sff == 0.0) {
      if (bf != 0.0) atomicOr(d.status, ST_PIN_RETAINED);
      d.pinned[0] |= 0x80;
      d.bred[7] = 0.0;
      d.Minv[63] = 1.0;
    } else {
      d.pinned[0] &= 0x7f;
      d.bred[7] = bf;
      const double f = 1.0 / sff;
      if (!isfinite(f)) atomicOr(d.status, ST_SINGULAR_PRECOND);
      d.Minv[63] = f;
    }
  }
}

// Shared focal gradient: sum of the cameras' focal entries (camera order);
// adds it to |g|^2 and max|g| (camfin left it out).
__global__ void ba_k_shared_focal_grad(BADev d) {
  __shared__ double sm[32];
  double v[1] = {0.0};
  const int C = d.bp.C;
  const int per = (C + blockDim.x - 1) / blockDim.x;
  const int a = threadIdx.x * per, b = min(C, a + per);
  for (int c = a; c < b; ++c) v[0] += d.gcam[8ll * c + 7];
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) {
    d.scal[SC_GFOCAL] = v[0];
    d.scal[SC_GNORM2] += v[0] * v[0];
    atomic_max_nonneg(d.scal + SC_GMAX, fabs(v[0]));
  }
}

// ---------------------------------------------------------------------------
// Omega form of the point-side operator (two-pass handles with the factored
// camera pass). The quaternion block of an observation is the point block
// times a per-camera map: drotate_dq (scene.py:153-184) applied to a
// direction w is R (omega x v) with omega = (2/|q|) vec(qh^* (x) w) (the
// derivative of R(q/|q|) v along w), and the point block is
// Jp = sw du_dp R (ba.py:187-190), so
//   Jc_o p_c = Jp_o (omega_c x v_o - p_t,c) + Jf_o p_f,c
//            = Jp_o (omega_c x X_j - b_c) + Jf_o p_f,c,   b_c = omega_c x t_c + p_t,c.
// The point pass then streams Jp and Jf (8 doubles per observation instead
// of the 16-double record) and gathers W_c = [omega_c, b_c, p_f,c, 0] (64
// bytes, like the 8-slot p it replaces) and X_j at the linearization. The
// operator equals the stored Jacobian's to rounding.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ba_wvec(const BADev& d, const double* __restrict__ v, int c,
                                        double* __restrict__ W) {
  const double* cb = reinterpret_cast<const double*>(d.camlin + c);
  const double* pc = v + 8ll * c;
  const double qw = cb[9], qx = cb[10], qy = cb[11], qz = cb[12], s2 = 2.0 * cb[22];
  const double pw = pc[0], px = pc[1], py = pc[2], pz = pc[3];
  // vec(qh^* (x) p) = qw p_v - pw q_v - q_v x p_v
  const double o0 = s2 * (qw * px - pw * qx - (qy * pz - qz * py));
  const double o1 = s2 * (qw * py - pw * qy - (qz * px - qx * pz));
  const double o2 = s2 * (qw * pz - pw * qz - (qx * py - qy * px));
  const double t0 = cb[14], t1 = cb[15], t2 = cb[16];
  double* w = W + 8ll * c;
  w[0] = o0; w[1] = o1; w[2] = o2;
  w[3] = (o1 * t2 - o2 * t1) + pc[4];
  w[4] = (o2 * t0 - o0 * t2) + pc[5];
  w[5] = (o0 * t1 - o1 * t0) + pc[6];
  w[6] = d.bp.focal_mode == 2 ? v[7] : (d.bp.focal_mode == 1 ? pc[7] : 0.0);
  w[7] = 0.0;
}

__global__ void k_cam_wvec(BADev d, const double* __restrict__ v, double* W) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < d.bp.C) ba_wvec(d, v, c, W);
}

// One observation's Jp^T (Jc p_c) in the omega form (point-major index i):
// the AoS record Gpm[8i..8i+7] = [Jp row 0, Jp row 1, Jf], the camera's W
// (of p) and the observation's point X at the linearization.
__device__ __forceinline__ void ba_wobs_math(const double* G, const double* w, const double* X, double* val) {
  const double u0 = (w[1] * X[2] - w[2] * X[1]) - w[3];
  const double u1 = (w[2] * X[0] - w[0] * X[2]) - w[4];
  const double u2 = (w[0] * X[1] - w[1] * X[0]) - w[5];
  const double t0 = G[0] * u0 + G[1] * u1 + G[2] * u2 + G[6] * w[6];
  const double t1 = G[3] * u0 + G[4] * u1 + G[5] * u2 + G[7] * w[6];
  val[0] = G[0] * t0 + G[3] * t1;
  val[1] = G[1] * t0 + G[4] * t1;
  val[2] = G[2] * t0 + G[5] * t1;
}
template <bool RO>
__device__ __forceinline__ void ba_wobs(const BADev& d, long long i, int c, const double* __restrict__ W,
                                        const double* X, double* val) {
  const unsigned long long pstream = pol_evict_first(), pkeep = pol_evict_last();
  double G[8], w[8];
  gpm_load(d, i, G, pstream);
  if constexpr (RO) {
    ld_v4_ro(W + 8ll * c, w, pkeep);
    ld_v4_ro(W + 8ll * c + 4, w + 4, pkeep);
  } else {
    ld_v4(W + 8ll * c, w);
    ld_v4(W + 8ll * c + 4, w + 4);
  }
  const double u0 = (w[1] * X[2] - w[2] * X[1]) - w[3];
  const double u1 = (w[2] * X[0] - w[0] * X[2]) - w[4];
  const double u2 = (w[0] * X[1] - w[1] * X[0]) - w[5];
  const double t0 = G[0] * u0 + G[1] * u1 + G[2] * u2 + G[6] * w[6];
  const double t1 = G[3] * u0 + G[4] * u1 + G[5] * u2 + G[7] * w[6];
  val[0] = G[0] * t0 + G[3] * t1;
  val[1] = G[1] * t0 + G[4] * t1;
  val[2] = G[2] * t0 + G[5] * t1;
}

// ---------------------------------------------------------------------------
// back-substitution (lm.py:674-690): delta_j = y0_j - Cinv_j sum_o Jp^T Jc x_c
// one warp per point batch; camera part of delta scattered by ba_k_camdelta.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ba_k_backsub(BADev d, const double* __restrict__ x,
                                                    double* delta) {
  __shared__ double sm[8][SSFM_BATCH][3];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long Np = d.Npad;
  for (int b = gw; b < d.topo.nb; b += warps) {
    const int ob0 = d.topo.bat_obs[b], ob1 = d.topo.bat_obs[b + 1];
    const int pb0 = d.topo.bat_pt[b], pb1 = d.topo.bat_pt[b + 1];
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    if (my_pt < pb1) { ps = d.topo.pt_seg[my_pt]; pe = d.topo.pt_seg[my_pt + 1]; }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[3] = {0.0, 0.0, 0.0};
      if (i < ob1 && d.Gpm) {
        const int c = d.topo.pm_cam[i], j = d.topo.pm_pt[i];
        ba_wobs<false>(d, i, c, d.Wc, d.Xl + 4ll * j, val);
      } else if (i < ob1) {
        double J[BA_JREC];
#pragma unroll
        for (int k = 0; k < BA_JREC; ++k) J[k] = d.Jpm[k * Np + i];
        const int c = d.topo.pm_cam[i];
        double pc[8];
        ld_v4(x + 8ll * c, pc);
        ld_v4(x + 8ll * c + 4, pc + 4);
        if (d.bp.focal_mode == 2) pc[7] = x[7];
        double t[2];
        ba_jc_mul(J, pc, t);
        ba_jpt_mul(J, t, val);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) sm[wib][lane][k] = val[k];
      __syncwarp();
      const int a = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a; o < e; ++o) {
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] += sm[wib][o - base][k];
      }
      __syncwarp();
    }
    if (my_pt < pb1) {
      double ci[6], w[3];
#pragma unroll
      for (int k = 0; k < 6; ++k) ci[k] = d.Cinv[6ll * my_pt + k];
      sym3_matvec(ci, acc, w);
      double* dst = delta + d.bp.off_pts + 3ll * my_pt;
#pragma unroll
      for (int k = 0; k < 3; ++k) dst[k] = d.y0[3ll * my_pt + k] - w[k];
    }
  }
}

__global__ void ba_k_camdelta(BADev d, const double* __restrict__ x, double* delta) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d.bp.C) return;
#pragma unroll
  for (int k = 0; k < 7; ++k) delta[7ll * c + k] = x[8ll * c + k];
  if (d.bp.focal_mode == 1) delta[d.bp.off_foc + c] = x[8ll * c + 7];
  if (d.bp.focal_mode == 2 && c == 0) delta[d.bp.off_foc] = x[7];
}

// candidate = theta + delta (lm.py:770)
__global__ void k_axpy_theta(const double* __restrict__ theta, const double* __restrict__ delta,
                             double* out, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = theta[i] + delta[i];
}

// renormalize (lm.py:104-117): unit quaternion per camera_pose block
__global__ void ba_k_renorm(int C, double* theta, int* status) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double* q = theta + 7ll * c;
  const double n = __dsqrt_rn(ADD(ADD(ADD(MUL(q[0], q[0]), MUL(q[1], q[1])), MUL(q[2], q[2])), MUL(q[3], q[3])));
  if (n < 1e-12) { atomicOr(status, ST_ZERO_QUAT); return; }
#pragma unroll
  for (int k = 0; k < 4; ++k) q[k] = DIV(q[k], n);
}

// diagnostic: count (observation, entry) pairs where the camera-major copy of
// the Jacobian differs from the point-major one (bitwise)
__global__ void k_check_jcopies(BADev d, unsigned long long* mism) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= d.topo.N) return;
  const int ic = d.topo.pm_to_cm[i];
  int bad = 0;
  for (int k = 0; k < BA_JREC; ++k)
    bad += __double_as_longlong(d.Jpm[k * d.Npad + i]) != __double_as_longlong(d.Jcm[k * d.Npad + ic]);
  if (bad) atomicAdd(mism, (unsigned long long)bad);
}
