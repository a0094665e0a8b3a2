// gp_kernels.cuh -- global positioning (gp.py): ray residual
//   u_o = sqrt(w) (v_o - d_o (X_j - t_i))
// with per-observation scale d_o (or fixed 1/depth in depth mode), its compact
// Jacobian, the two-stage Schur elimination (scales, then points; lm.py:563-606)
// and the matrix-free PCG on the 3C camera-centre system.
//
// Compact Jacobian per observation (gp.py:118-124): the centre block is a_t I,
// the point block -a I and the scale column g, with a = d sqrt(w),
// a_t = a (0 for camera 0 when the gauge is fixed, gp.py:120-121) and
// g = -sqrt(w) (X - t). Stored as 4 fp64 {a, g0, g1, g2} per observation
// instead of the reference's 21 (gp.py:65).
//
// Folded per-observation quantities (Appendix C of SURVEY.md; lm.py:563-597):
//   inv_o = 1 / ((1+lam) |g|^2)   (0 when that is 0)
//   U'_o  = -a_t a I + inv_o a_t a g g^T           (camera x point coupling)
//   B'_c  = (1+lam) sum a_t^2 I - sum inv_o a_t^2 g g^T
//   C'_j  = (1+lam) sum a^2 I   - sum inv_o a^2 g g^T
#pragma once
#include "ba_kernels.cuh"
#include "comm.cuh"
#include "fused.cuh"
#include <cooperative_groups.h>

#define GP_JREC 4
#define GP_SCALE_FLOOR 1e-6   // gp.py:298

struct GPParams {
  int C, P;
  long long N;
  int depth_mode, gauge_fixed;
  int loss_kind;
  double delta;
  long long off_pts;   // 3C
  long long off_sc;    // 3C + 3P
};

struct GPDev {
  GPParams gp;
  Topo topo;
  const double* ray_pm;   // [3N] point-major rays
  const double* dep_pm;   // [N] point-major ray depths (depth mode)
  const double* ray_cm;   // [3N] camera-major rays
  const double* dep_cm;   // [N] camera-major ray depths (depth mode)
  double* Jpm;            // [4 * Npad]
  double* Jcm;            // [4 * Npad]
  double* rcm;            // [3 * Npad]
  double* bo_pm;          // [N] b_o = -(g . r) point-major
  double* bo_cm;          // [N] camera-major
  long long Npad;
  double* Apt;            // [P]  sum a^2
  double* gpt;            // [3P] J^T r point part
  double* Acam;           // [C]  sum a_t^2
  double* gcam;           // [3C] J^T r camera part
  double* Minv_pt;        // [6P] C'_j^-1
  double* y0;             // [3P]
  double* yv;             // [4P] (padded for 32-byte gathers)
  double* Bp;             // [6C] B'_c (upper)
  double* Minv;           // [16C] preconditioner (4x4 slots, 3x3 used)
  double* bred;           // [4C]
  unsigned char* pinned;  // [C]
  double* tilebuf;        // [18 * nt]
  double* gsc;            // [N] scale gradient (original order)
  double* scal;
  double* partials;
  int* status;
  double lam;
  const double* lamp;     // device-resident lambda (LM loop as a CUDA graph) or nullptr: lam / the argument
};

// GP observation record {a, g0, g1, g2} in the point- or camera-major array:
// GP_AOS=1 one 32-byte record per observation (one vector load), 0: SoA rows.
#ifndef GP_AOS
#define GP_AOS 1
#endif
__device__ __forceinline__ void gp_rec_st(double* base, long long Np, long long i, const double* rec) {
#if GP_AOS
  (void)Np;
  *reinterpret_cast<double4*>(base + 4 * i) = make_double4(rec[0], rec[1], rec[2], rec[3]);
#else
#pragma unroll
  for (int k = 0; k < 4; ++k) base[k * Np + i] = rec[k];
#endif
}
// STREAM: L2 evict_first, no L1 allocation (the PCG passes)
template <bool STREAM>
__device__ __forceinline__ void gp_rec_ld(const double* base, long long Np, long long i, double* rec) {
#if GP_AOS
  (void)Np;
  if constexpr (STREAM) ld_v4_ro(base + 4 * i, rec, pol_evict_first());
  else ld_v4(base + 4 * i, rec);
#else
#pragma unroll
  for (int k = 0; k < 4; ++k) rec[k] = __ldg(base + k * Np + i);
#endif
}

__device__ __forceinline__ double gp_at(const GPDev& g, int cam, double a) {
  return (g.gp.gauge_fixed && cam == 0) ? 0.0 : a;
}

__device__ __forceinline__ double gp_inv(double lam, const double* rec) {
  const double g2 = rec[1] * rec[1] + rec[2] * rec[2] + rec[3] * rec[3];
  const double D = (1.0 + lam) * g2;
  return D == 0.0 ? 0.0 : 1.0 / D;
}

// residual block of one observation (gp.py:96-107), numpy operation order;
// camera c, point j, original observation o, its ray v and depth
__device__ __forceinline__ void gp_residual_at(const GPDev& g, int c, int j, int o, const double* v, double dep,
                                               const double* __restrict__ theta, double span[3], double blk[3],
                                               double& dsc, double& s) {
  const double* X = theta + g.gp.off_pts + 3ll * j;
  const double* t = theta + 3ll * c;
  if (g.gp.depth_mode) dsc = DIV(1.0, dep);
  else dsc = theta[g.gp.off_sc + o];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    span[k] = SUB(X[k], t[k]);
    blk[k] = SUB(v[k], MUL(dsc, span[k]));
  }
  // np.einsum("ni,ni->n") evaluates (b0 b0 + b2 b2) + b1 b1 for 3 terms
  s = ADD(ADD(MUL(blk[0], blk[0]), MUL(blk[2], blk[2])), MUL(blk[1], blk[1]));
}

// point-major observation i
__device__ __forceinline__ void gp_residual(const GPDev& g, long long i, const double* __restrict__ theta,
                                            double span[3], double blk[3], double& dsc, double& s) {
  gp_residual_at(g, g.topo.pm_cam[i], g.topo.pm_pt[i], g.topo.pm_obs[i], g.ray_pm + 3 * i,
                 g.gp.depth_mode ? g.dep_pm[i] : 0.0, theta, span, blk, dsc, s);
}

// compact record {a, g}, weighted residual and b_o = -(g . r) of one
// observation (gp.py:109-128); shared by the point-major and camera-major
// linearize passes (one expression tree -> bit-identical copies)
__device__ __forceinline__ void gp_record(const GPDev& g, int c, const double span[3], const double blk[3],
                                          double d, double s, double rec[4], double r[3], double& bo) {
  double cst, w;
  robust(g.gp.loss_kind, g.gp.delta, s, cst, w);
  const double sw = __dsqrt_rn(w);
  rec[0] = d * sw;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    rec[1 + k] = g.gp.depth_mode ? 0.0 : -span[k] * sw;
    r[k] = MUL(blk[k], sw);
  }
  bo = -(rec[1] * r[0] + rec[2] * r[1] + rec[3] * r[2]);
  (void)c;
}

__global__ void gp_k_cost(GPDev g, const double* __restrict__ theta, double* partials) {
  __shared__ double sm[32];
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  if (i < g.topo.N) {
    double span[3], blk[3], d, s, cst, w;
    gp_residual(g, i, theta, span, blk, d, s);
    robust(g.gp.loss_kind, g.gp.delta, s, cst, w);
    v[0] = cst;
  }
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
}

// linearize (gp.py:109-128) + point side of J^T J / J^T r; one warp per batch
#define GPL_V 4
__global__ void __launch_bounds__(256) gp_k_linearize(GPDev g, const double* __restrict__ theta,
                                                      double* r_out, double* J_out, double* norm_part) {
  __shared__ double sm[8][SSFM_BATCH][GPL_V];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long Np = g.Npad;
  double gn2 = 0.0, gmax = 0.0;
  for (int b = gw; b < g.topo.nb; b += warps) {
    const int ob0 = g.topo.bat_obs[b], ob1 = g.topo.bat_obs[b + 1];
    const int pb0 = g.topo.bat_pt[b], pb1 = g.topo.bat_pt[b + 1];
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    if (my_pt < pb1) { ps = g.topo.pt_seg[my_pt]; pe = g.topo.pt_seg[my_pt + 1]; }
    double acc[GPL_V] = {0.0, 0.0, 0.0, 0.0};
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[GPL_V] = {0.0, 0.0, 0.0, 0.0};
      if (i < ob1) {
        double span[3], blk[3], d, s;
        gp_residual(g, i, theta, span, blk, d, s);
        const int c = g.topo.pm_cam[i];
        double rec[4], r[3], bo;
        gp_record(g, c, span, blk, d, s, rec, r, bo);
        const double a = rec[0];
        const double at = gp_at(g, c, a);
        gp_rec_st(g.Jpm, Np, i, rec);
        g.bo_pm[i] = bo;
        const int o = g.topo.pm_obs[i];
        if (!g.gp.depth_mode) {
          g.gsc[o] = -bo;    // squared norm summed by gp_k_scale_norm
          gmax = fmax(gmax, fabs(bo));
        }
        // point block is -a I: J^T r = -a r, J^T J diag = a^2
        val[0] = a * a;
        val[1] = -a * r[0];
        val[2] = -a * r[1];
        val[3] = -a * r[2];
        if (r_out) {
#pragma unroll
          for (int k = 0; k < 3; ++k) r_out[3ll * o + k] = r[k];
        }
        if (J_out) {
          const int wdt = g.gp.depth_mode ? 18 : 21;
          double* dst = J_out + (long long)wdt * o;
#pragma unroll
          for (int k = 0; k < 9; ++k) {
            const bool dg = (k % 4) == 0;
            dst[k] = dg ? at : 0.0;
            dst[9 + k] = dg ? -a : 0.0;
          }
          if (!g.gp.depth_mode) {
#pragma unroll
            for (int k = 0; k < 3; ++k) dst[18 + k] = rec[1 + k];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < GPL_V; ++k) sm[wib][lane][k] = val[k];
      __syncwarp();
      const int a0 = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a0; o < e; ++o) {
#pragma unroll
        for (int k = 0; k < GPL_V; ++k) acc[k] += sm[wib][o - base][k];
      }
      __syncwarp();
    }
    if (my_pt < pb1) {
      g.Apt[my_pt] = acc[0];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        g.gpt[3ll * my_pt + k] = acc[1 + k];
        gn2 += acc[1 + k] * acc[1 + k];
        gmax = fmax(gmax, fabs(acc[1 + k]));
      }
    }
  }
  gn2 = warp_sum(gn2);
  gmax = warp_max(gmax);
  if (lane == 0) {
    norm_part[gw] = gn2;
    atomic_max_nonneg(g.scal + SC_GMAX, gmax);
  }
}

// camera side at linearize, per camera tile (camera-major): evaluate the
// observations again with the same expressions, write the camera-major
// record / residual / b_o copies coalesced, and reduce sum a_t^2 and
// sum a_t r (J^T r camera part). Replaces scattered 8-byte stores.
#define GPC_V 4
__global__ void __launch_bounds__(SSFM_TILE) gp_k_linearize_cm(GPDev g, const double* __restrict__ theta) {
  __shared__ double sm[(SSFM_TILE / 32) * GPC_V];
  const int t = blockIdx.x;
  const int o0 = g.topo.tile_obs[t], o1 = g.topo.tile_obs[t + 1];
  const int c = g.topo.tile_cam[t];
  const int i = o0 + threadIdx.x;
  double v[GPC_V] = {0.0, 0.0, 0.0, 0.0};
  if (i < o1) {
    const long long Np = g.Npad;
    double span[3], blk[3], d, s;
    gp_residual_at(g, c, g.topo.cm_pt[i], g.topo.cm_obs[i], g.ray_cm + 3ll * i,
                   g.gp.depth_mode ? g.dep_cm[i] : 0.0, theta, span, blk, d, s);
    double rec[4], r[3], bo;
    gp_record(g, c, span, blk, d, s, rec, r, bo);
    gp_rec_st(g.Jcm, Np, i, rec);
#pragma unroll
    for (int k = 0; k < 3; ++k) g.rcm[k * Np + i] = r[k];
    g.bo_cm[i] = bo;
    const double at = gp_at(g, c, rec[0]);
    v[0] = at * at;
#pragma unroll
    for (int k = 0; k < 3; ++k) v[1 + k] = at * r[k];
  }
  block_reduce<GPC_V>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < GPC_V; ++k) g.tilebuf[(long long)GPC_V * t + k] = v[k];
  }
}

__global__ void gp_k_camfin(GPDev g, double* norm_part, const double* camsum) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  double gn2 = 0.0, gmax = 0.0;
  if (c < g.gp.C) {
    double s[GPC_V] = {0.0, 0.0, 0.0, 0.0};
    if (camsum) {   // per-camera sums already reduced over the ranks
#pragma unroll
      for (int k = 0; k < GPC_V; ++k) s[k] = camsum[(long long)GPC_V * c + k];
    } else {
      for (int t = g.topo.cam_tile[c]; t < g.topo.cam_tile[c + 1]; ++t)
#pragma unroll
        for (int k = 0; k < GPC_V; ++k) s[k] += g.tilebuf[(long long)GPC_V * t + k];
    }
    g.Acam[c] = s[0];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      g.gcam[3ll * c + k] = s[1 + k];
      gn2 += s[1 + k] * s[1 + k];
      gmax = fmax(gmax, fabs(s[1 + k]));
    }
  }
  double v[1] = {gn2};
  __shared__ double sm[32];
  const double gm = warp_max(gmax);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(g.scal + SC_GMAX, gm);
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) norm_part[blockIdx.x] = v[0];
}

// sum of squares of the scale gradient in fixed order (block partials)
__global__ void gp_k_scale_norm(GPDev g, double* part) {
  __shared__ double sm[32];
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  if (i < g.topo.N && !g.gp.depth_mode) { const double x = g.gsc[i]; v[0] = x * x; }
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// ---------------------------------------------------------------------------
// per lambda: stage 1 (scales) folded into the point blocks + stage 2 inverse
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gp_k_pt_elim(GPDev g, double lam) {
  if (g.lamp) lam = *g.lamp;
  __shared__ double sm[8][SSFM_BATCH][9];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long Np = g.Npad;
  for (int b = gw; b < g.topo.nb; b += warps) {
    const int ob0 = g.topo.bat_obs[b], ob1 = g.topo.bat_obs[b + 1];
    const int pb0 = g.topo.bat_pt[b], pb1 = g.topo.bat_pt[b + 1];
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    if (my_pt < pb1) { ps = g.topo.pt_seg[my_pt]; pe = g.topo.pt_seg[my_pt + 1]; }
    double acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = 0.0;
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) val[k] = 0.0;
      if (i < ob1) {
        double rec[4];
        gp_rec_ld<false>(g.Jpm, Np, i, rec);
        const double inv = gp_inv(lam, rec);
        const double a = rec[0], bo = g.bo_pm[i];
        const double f = inv * a * a;
        const double* gg = rec + 1;
        val[0] = f * gg[0] * gg[0]; val[1] = f * gg[0] * gg[1]; val[2] = f * gg[0] * gg[2];
        val[3] = f * gg[1] * gg[1]; val[4] = f * gg[1] * gg[2]; val[5] = f * gg[2] * gg[2];
        const double h = inv * bo * a;
        val[6] = h * gg[0]; val[7] = h * gg[1]; val[8] = h * gg[2];
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) sm[wib][lane][k] = val[k];
      __syncwarp();
      const int a0 = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a0; o < e; ++o) {
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] += sm[wib][o - base][k];
      }
      __syncwarp();
    }
    if (my_pt < pb1) {
      const double A = g.Apt[my_pt] * (1.0 + lam);
      double m[6] = {A - acc[0], -acc[1], -acc[2], A - acc[3], -acc[4], A - acc[5]};
      double b[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) b[k] = -g.gpt[3ll * my_pt + k] + acc[6 + k];
      const int di[3] = {0, 3, 5};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (m[di[k]] == 0.0) {
          if (b[k] != 0.0) atomicOr(g.status, ST_PIN_POINT);
          m[di[k]] = 1.0;
        }
      }
      double inv[6], det;
      if (!inv_sym3(m, inv, det)) {
        atomicOr(g.status, ST_SINGULAR_POINT);
#pragma unroll
        for (int k = 0; k < 6; ++k) inv[k] = 0.0;
      }
      double y[3];
      sym3_matvec(inv, b, y);
#pragma unroll
      for (int k = 0; k < 6; ++k) g.Minv_pt[6ll * my_pt + k] = inv[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) g.y0[3ll * my_pt + k] = y[k];
    }
  }
}

// U'_o v for a 3-vector v
__device__ __forceinline__ void gp_u_mul(double at, double a, double inv, const double* gg,
                                         const double* v, double* o) {
  const double gv = gg[0] * v[0] + gg[1] * v[1] + gg[2] * v[2];
  const double s = at * a;
#pragma unroll
  for (int k = 0; k < 3; ++k) o[k] = s * (-v[k] + inv * gg[k] * gv);
}

// per camera tile at lambda: sum inv a_t^2 g g^T (6), sum inv b_o a_t g (3),
// sum U' M U'^T (6), sum U' y0 (3)
#define GPE_V 18
__global__ void __launch_bounds__(SSFM_TILE) gp_k_cam_elim(GPDev g, double lam) {
  if (g.lamp) lam = *g.lamp;
  __shared__ double sm[(SSFM_TILE / 32) * GPE_V];
  const int t = blockIdx.x;
  const int o0 = g.topo.tile_obs[t], o1 = g.topo.tile_obs[t + 1];
  const int c = g.topo.tile_cam[t];
  const int i = o0 + threadIdx.x;
  double v[GPE_V];
#pragma unroll
  for (int k = 0; k < GPE_V; ++k) v[k] = 0.0;
  if (i < o1) {
    const long long Np = g.Npad;
    double rec[4];
    gp_rec_ld<false>(g.Jcm, Np, i, rec);
    const double a = rec[0], at = gp_at(g, c, a);
    const double inv = gp_inv(lam, rec);
    const double* gg = rec + 1;
    const double bo = g.bo_cm[i];
    const double f = inv * at * at;
    v[0] = f * gg[0] * gg[0]; v[1] = f * gg[0] * gg[1]; v[2] = f * gg[0] * gg[2];
    v[3] = f * gg[1] * gg[1]; v[4] = f * gg[1] * gg[2]; v[5] = f * gg[2] * gg[2];
    const double h = inv * bo * at;
    v[6] = h * gg[0]; v[7] = h * gg[1]; v[8] = h * gg[2];
    const int j = g.topo.cm_pt[i];
    double M[6], y[3];
#pragma unroll
    for (int k = 0; k < 6; ++k) M[k] = g.Minv_pt[6ll * j + k];
#pragma unroll
    for (int k = 0; k < 3; ++k) y[k] = g.y0[3ll * j + k];
    // U' (sym) columns e_k -> U' M U'
    double U[9];
    {
      const double s = at * a;
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = 0; q < 3; ++q) U[3 * p + q] = s * ((p == q ? -1.0 : 0.0) + inv * gg[p] * gg[q]);
    }
    double MU[9];   // M U (M sym)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double col[3] = {U[q], U[3 + q], U[6 + q]};
      double o[3];
      sym3_matvec(M, col, o);
      MU[q] = o[0]; MU[3 + q] = o[1]; MU[6 + q] = o[2];
    }
    int idx = 9;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int q = p; q < 3; ++q)
        v[idx++] = U[3 * p] * MU[q] + U[3 * p + 1] * MU[3 + q] + U[3 * p + 2] * MU[6 + q];
    double uy[3];
    gp_u_mul(at, a, inv, gg, y, uy);
    v[15] = uy[0]; v[16] = uy[1]; v[17] = uy[2];
  }
  block_reduce<GPE_V>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < GPE_V; ++k) g.tilebuf[(long long)GPE_V * t + k] = v[k];
  }
}

__global__ void gp_k_camprec(GPDev g, double lam, const double* camsum) {
  if (g.lamp) lam = *g.lamp;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.gp.C) return;
  double s[GPE_V];
#pragma unroll
  for (int k = 0; k < GPE_V; ++k) s[k] = camsum ? camsum[(long long)GPE_V * c + k] : 0.0;
  if (!camsum)
    for (int t = g.topo.cam_tile[c]; t < g.topo.cam_tile[c + 1]; ++t)
#pragma unroll
      for (int k = 0; k < GPE_V; ++k) s[k] += g.tilebuf[(long long)GPE_V * t + k];
  const double A = g.Acam[c] * (1.0 + lam);
  double Bp[6] = {A - s[0], -s[1], -s[2], A - s[3], -s[4], A - s[5]};
#pragma unroll
  for (int k = 0; k < 6; ++k) g.Bp[6ll * c + k] = Bp[k];
  double S[9];
  {
    int idx = 0;
    for (int p = 0; p < 3; ++p)
      for (int q = p; q < 3; ++q) {
        const double val = Bp[idx] - s[9 + idx];
        S[3 * p + q] = val; S[3 * q + p] = val; ++idx;
      }
  }
  double br[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) br[k] = (-g.gcam[3ll * c + k] - s[6 + k]) - s[15 + k];
  unsigned pin = 0;
  for (int p = 0; p < 3; ++p) {
    if (S[4 * p] == 0.0) {
      if (br[p] != 0.0) atomicOr(g.status, ST_PIN_RETAINED);
      pin |= 1u << p;
      S[4 * p] = 1.0;
    }
  }
  pin |= 1u << 3;   // 4th slot is padding
  g.pinned[c] = (unsigned char)pin;
  for (int p = 0; p < 3; ++p) g.bred[4ll * c + p] = (pin >> p & 1u) ? 0.0 : br[p];
  g.bred[4ll * c + 3] = 0.0;
  double I3[9];
  const bool ok = gj_inverse(S, I3, 3, 3);
  if (!ok) atomicOr(g.status, ST_SINGULAR_PRECOND);
  double* M = g.Minv + 16ll * c;
  for (int p = 0; p < 4; ++p)
    for (int q = 0; q < 4; ++q) M[4 * p + q] = (p < 3 && q < 3) ? (ok ? I3[3 * p + q] : 0.0) : (p == q ? 1.0 : 0.0);
}

// ---------------------------------------------------------------------------
// PCG (same structure as ba_k_pcg, 4 slots per camera, slot 3 padding)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double grp4_get(double v, int k) {
  const int base = (threadIdx.x & 31) & ~3;
  return __shfl_sync(SSFM_FULL, v, base + k);
}

#ifndef GP_PIPE
#define GP_PIPE 1   // index prefetch one round ahead (as ba_point_pass_w / ba_camera_pass_f)
#endif
#if GP_PIPE
// Each warp owns a contiguous range of point batches, so the next round's
// observation range is known without a load and its camera indices are
// requested one round ahead: a round issues its record stream and its camera
// gather together (one DRAM latency per round instead of index -> gather).
// Same arithmetic and per-point order as before: bit-identical output.
__device__ __forceinline__ void gp_point_pass(const GPDev& g, const double* v, double* y,
                                              double (*sm)[SSFM_BATCH][3]) {
  const unsigned long long pstream = pol_evict_first();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long Np = g.Npad;
  const double lam = g.lam;
  const int nb = g.topo.nb;
  const int b0 = (int)((long long)nb * gw / warps), b1 = (int)((long long)nb * (gw + 1) / warps);
  if (b0 >= b1) return;   // warp-uniform
  int ob0 = g.topo.bat_obs[b0], ob1 = g.topo.bat_obs[b0 + 1], pb0 = g.topo.bat_pt[b0];
  int cn = ob0 + lane < ob1 ? ldg_stream_i(g.topo.pm_cam + ob0 + lane, pstream) : 0;
  for (int b = b0; b < b1; ++b) {
    const int pb1 = g.topo.bat_pt[b + 1];
    const int nob1 = b + 1 < b1 ? g.topo.bat_obs[b + 2] : ob1;   // end of the next batch
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    if (my_pt < pb1) { ps = g.topo.pt_seg[my_pt]; pe = g.topo.pt_seg[my_pt + 1]; }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      const int c = cn;
      const bool act = i < ob1;
      double rec[4], pc[4];
      if (act) {
        gp_rec_ld<true>(g.Jpm, Np, i, rec);
        ld_v4(v + 4ll * c, pc);   // 4 slots per camera: one 32-byte gather
      }
      const bool more = base + SSFM_BATCH < ob1;
      const int ni = more ? i + SSFM_BATCH : ob1 + lane, nend = more ? ob1 : nob1;
      if (ni < nend) cn = ldg_stream_i(g.topo.pm_cam + ni, pstream);
      double val[3] = {0.0, 0.0, 0.0};
      if (act) {
        const double at = gp_at(g, c, rec[0]);
        const double inv = gp_inv(lam, rec);
        gp_u_mul(at, rec[0], inv, rec + 1, pc, val);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) sm[wib][lane][k] = val[k];
      __syncwarp();
      const int a0 = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a0; o < e; ++o) {
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] += sm[wib][o - base][k];
      }
      __syncwarp();
    }
    if (my_pt < pb1) {
      double M[6], w[3];
#pragma unroll
      for (int k = 0; k < 6; ++k) M[k] = __ldg(g.Minv_pt + 6ll * my_pt + k);
      sym3_matvec(M, acc, w);
#pragma unroll
      for (int k = 0; k < 3; ++k) y[4ll * my_pt + k] = w[k];   // padded: one 32-byte gather
    }
    ob0 = ob1; ob1 = nob1; pb0 = pb1;
  }
}

__device__ __forceinline__ void gp_camera_pass(const GPDev& g, const double* y, double* tile4,
                                               double* smred) {
  // one warp per camera tile, register accumulation, one butterfly; the point
  // index is requested one round ahead so the y gather leaves with the record
  (void)smred;
  const unsigned long long pstream = pol_evict_first();
  const long long Np = g.Npad;
  const double lam = g.lam;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int t = gw; t < g.topo.nt; t += warps) {
    const int o0 = __ldg(g.topo.tile_obs + t), o1 = __ldg(g.topo.tile_obs + t + 1);
    const int c = __ldg(g.topo.tile_cam + t);
    double o[3] = {0.0, 0.0, 0.0};
    int jn = o0 + lane < o1 ? ldg_stream_i(g.topo.cm_pt + o0 + lane, pstream) : 0;
    for (int i = o0 + lane; i < o1; i += 32) {
      const int j = jn;
      double rec[4], yj[4], u[3];
      gp_rec_ld<true>(g.Jcm, Np, i, rec);
      ld_v4(y + 4ll * j, yj);
      if (i + 32 < o1) jn = ldg_stream_i(g.topo.cm_pt + i + 32, pstream);
      const double at = gp_at(g, c, rec[0]);
      const double inv = gp_inv(lam, rec);
      gp_u_mul(at, rec[0], inv, rec + 1, yj, u);
#pragma unroll
      for (int k = 0; k < 3; ++k) o[k] += u[k];
    }
    warp_allreduce<3>(o);
    if (lane < 3) tile4[4ll * t + lane] = lane == 0 ? o[0] : (lane == 1 ? o[1] : o[2]);
  }
}
#else
__device__ __forceinline__ void gp_point_pass(const GPDev& g, const double* v, double* y,
                                              double (*sm)[SSFM_BATCH][3]) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long Np = g.Npad;
  const double lam = g.lam;
  for (int b = gw; b < g.topo.nb; b += warps) {
    const int ob0 = g.topo.bat_obs[b], ob1 = g.topo.bat_obs[b + 1];
    const int pb0 = g.topo.bat_pt[b], pb1 = g.topo.bat_pt[b + 1];
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    if (my_pt < pb1) { ps = g.topo.pt_seg[my_pt]; pe = g.topo.pt_seg[my_pt + 1]; }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[3] = {0.0, 0.0, 0.0};
      if (i < ob1) {
        double rec[4];
        gp_rec_ld<true>(g.Jpm, Np, i, rec);
        const int c = __ldg(g.topo.pm_cam + i);
        const double at = gp_at(g, c, rec[0]);
        const double inv = gp_inv(lam, rec);
        double pc[4];
        ld_v4(v + 4ll * c, pc);   // 4 slots per camera: one 32-byte gather
        gp_u_mul(at, rec[0], inv, rec + 1, pc, val);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) sm[wib][lane][k] = val[k];
      __syncwarp();
      const int a0 = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a0; o < e; ++o) {
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] += sm[wib][o - base][k];
      }
      __syncwarp();
    }
    if (my_pt < pb1) {
      double M[6], w[3];
#pragma unroll
      for (int k = 0; k < 6; ++k) M[k] = __ldg(g.Minv_pt + 6ll * my_pt + k);
      sym3_matvec(M, acc, w);
#pragma unroll
      for (int k = 0; k < 3; ++k) y[4ll * my_pt + k] = w[k];   // padded: one 32-byte gather
    }
  }
}

__device__ __forceinline__ void gp_camera_pass(const GPDev& g, const double* y, double* tile4,
                                               double* smred) {
  // one warp per camera tile, register accumulation, one butterfly (no CTA
  // barriers; same structure as ba_camera_pass)
  (void)smred;
  const long long Np = g.Npad;
  const double lam = g.lam;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int t = gw; t < g.topo.nt; t += warps) {
    const int o0 = __ldg(g.topo.tile_obs + t), o1 = __ldg(g.topo.tile_obs + t + 1);
    const int c = __ldg(g.topo.tile_cam + t);
    double o[3] = {0.0, 0.0, 0.0};
    for (int i = o0 + lane; i < o1; i += 32) {
      double rec[4];
      gp_rec_ld<true>(g.Jcm, Np, i, rec);
      const int j = __ldg(g.topo.cm_pt + i);
      const double at = gp_at(g, c, rec[0]);
      const double inv = gp_inv(lam, rec);
      double yj[4], u[3];
      ld_v4(y + 4ll * j, yj);
      gp_u_mul(at, rec[0], inv, rec + 1, yj, u);
#pragma unroll
      for (int k = 0; k < 3; ++k) o[k] += u[k];
    }
    warp_allreduce<3>(o);
    if (lane < 3) tile4[4ll * t + lane] = lane == 0 ? o[0] : (lane == 1 ? o[1] : o[2]);
  }
}

#endif

// Fused single pass for GP (the BA version is ba_fused_pass, fused.cuh): y_j
// for every point of the warp's batch, then each observation's camera term
// U'_o y_j added into the CTA's shared copy of the camera vector (4 slots per
// camera) in ticket order. The GP camera vector always fits one CTA.
// Dynamic shared memory: acc [4C] | stage [FZ_WARPS][4][32] | cnt [C] ints.
__device__ __forceinline__ void gp_fused_pass(const GPDev& g, const FusedTopo& fz, const double* __restrict__ v,
                                              double* dyn, double (*smv)[SSFM_BATCH][3],
                                              double (*smy)[SSFM_BATCH][3], int (*smown)[SSFM_BATCH]) {
  constexpr int SL = 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = blockIdx.x, ngrp = gridDim.x;
  const int C = g.gp.C;
  const long long Np = g.Npad;
  const double lam = g.lam;
  double* acc = dyn;
  double* stage = dyn + (long long)SL * C + (long long)warp * 32 * SL;
  int* cnt = reinterpret_cast<int*>(dyn + (long long)SL * C + FZ_WARPS * 32 * SL);
  for (int k = threadIdx.x; k < SL * C; k += blockDim.x) acc[k] = 0.0;
  for (int k = threadIdx.x; k < C; k += blockDim.x) cnt[k] = 0;
  __syncthreads();
  const int sstride = ngrp * FZ_WARPS;
  for (int b = grp * FZ_WARPS + warp; b < g.topo.nb; b += sstride) {
    const int ob0 = __ldg(g.topo.bat_obs + b), ob1 = __ldg(g.topo.bat_obs + b + 1);
    const int pb0 = __ldg(g.topo.bat_pt + b), pb1 = __ldg(g.topo.bat_pt + b + 1);
    const int rounds = (ob1 - ob0 + 31) >> 5;
    const int my_pt = pb0 + lane;
    const bool own = my_pt < pb1;
    int ps = 0, pe = 0;
    if (own) { ps = __ldg(g.topo.pt_seg + my_pt); pe = __ldg(g.topo.pt_seg + my_pt + 1); }
    double rec[4] = {0.0, 0.0, 0.0, 0.0};
    int c = 0, tk = 0;
    double a3[3] = {0.0, 0.0, 0.0};
    for (int r = 0; r < rounds; ++r) {
      const int base = ob0 + 32 * r;
      const int i = base + lane;
      double val[3] = {0.0, 0.0, 0.0};
      if (i < ob1) {
        c = __ldg(g.topo.pm_cam + i);
        gp_rec_ld<true>(g.Jpm, Np, i, rec);
        tk = __ldg(fz.tick + i);
        double pc[4];
        ld_v4(v + 4ll * c, pc);
        gp_u_mul(gp_at(g, c, rec[0]), rec[0], gp_inv(lam, rec), rec + 1, pc, val);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) smv[warp][lane][k] = val[k];
      __syncwarp();
      const int lo = max(ps, base), hi = min(pe, base + SSFM_BATCH);
      for (int o = lo; o < hi; ++o) {
#pragma unroll
        for (int k = 0; k < 3; ++k) a3[k] += smv[warp][o - base][k];
        smown[warp][o - base] = lane;
      }
      __syncwarp();
    }
    if (own) {
      double M[6], w[3];
#pragma unroll
      for (int k = 0; k < 6; ++k) M[k] = __ldg(g.Minv_pt + 6ll * my_pt + k);
      sym3_matvec(M, a3, w);
#pragma unroll
      for (int k = 0; k < 3; ++k) smy[warp][lane][k] = w[k];
    }
    __syncwarp();
    for (int r = 0; r < rounds; ++r) {
      const int i = ob0 + 32 * r + lane;
      const bool have = i < ob1;
      double u[SL] = {0.0, 0.0, 0.0, 0.0};
      if (have) {
        if (rounds > 1) {
          c = __ldg(g.topo.pm_cam + i);
          gp_rec_ld<true>(g.Jpm, Np, i, rec);
          tk = __ldg(fz.tick + i);
        }
        const int owner = rounds > 1 ? 0 : smown[warp][lane];
        double y[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) y[k] = smy[warp][owner][k];
        gp_u_mul(gp_at(g, c, rec[0]), rec[0], gp_inv(lam, rec), rec + 1, y, u);
      }
      const unsigned same = __match_any_sync(SSFM_FULL, have ? c : -1);
      const bool dup = __popc(same) > 1;
      if (__any_sync(SSFM_FULL, dup && have)) {
#pragma unroll
        for (int j = 0; j < SL; ++j) stage[j * 32 + lane] = u[j];
        __syncwarp();
        if (have && dup && lane == __ffs(same) - 1) {
#pragma unroll
          for (int j = 0; j < SL; ++j) u[j] = 0.0;
          for (unsigned m = same; m; m &= m - 1) {
            const int l = __ffs(m) - 1;
#pragma unroll
            for (int j = 0; j < SL; ++j) u[j] += stage[j * 32 + l];
          }
        }
        __syncwarp();
      }
      if (have && lane == __ffs(same) - 1) {
        int spins = 0;
        while (ld_acquire_smem(cnt + c) != tk) {
          if (++spins > FZ_SPIN_LIMIT) { atomicOr(g.status, ST_SCHEDULE); break; }
        }
        fz_add<SL>(acc, c, u);
        st_release_smem(cnt + c, tk + 1);
      }
    }
    __syncwarp();
  }
  __syncthreads();
  double* dst = fz.gpart + (long long)grp * SL * C;
  for (int k = threadIdx.x; k < SL * C; k += blockDim.x) {
    const int cc = k / SL, j = k - cc * SL;
    dst[k] = acc[fz_slot<SL>(cc, j)];
  }
}

// FUSED: one-pass operator (gp_fused_pass, 512 threads, dynamic shared
// camera vector, 2 CTAs per SM: 62 registers, no spills; 1 CTA per SM at 101
// registers was 0.207 vs 0.158 ms per C4 GP CG iteration); otherwise the
// two-pass operator (256 threads).
template <bool FUSED>
__global__ void __launch_bounds__(FUSED ? FZ_THREADS : PCG_THREADS, FUSED ? 2 : 4)
gp_k_pcg(GPDev g, FusedTopo fz, CommDev cm, double lam, int max_iters, double cg_tol, double* x, double* r,
         double* z, double* p, double* q, double* part, CGCtl* ctl) {
  constexpr int NT = FUSED ? FZ_THREADS : PCG_THREADS;
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ double smp[NT / 32][SSFM_BATCH][3];
  __shared__ double smy[FUSED ? NT / 32 : 1][SSFM_BATCH][3];
  __shared__ int smown[FUSED ? NT / 32 : 1][SSFM_BATCH];
  __shared__ double smred[(NT / 32) * 8];
  __shared__ double smb[4];
  extern __shared__ double gdyn[];
  if (g.lamp) lam = *g.lamp;
  g.lam = lam;
  const int S = 4 * g.gp.C;
  const int stride = gridDim.x * blockDim.x;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  double* tile4 = g.tilebuf;
  const int NP = gridDim.x;
  auto local_cam = [&](int s) -> double {   // local camera half of S*p, slot s = 4c + k
    double a = 0.0;
    if constexpr (FUSED) {
      for (int gq = 0; gq < NP; ++gq) a += fz.gpart[(long long)gq * S + s];
    } else {
      const int c = s >> 2, k = s & 3;
      a = tiles_sum<4>(tile4, k, g.topo.cam_tile[c], g.topo.cam_tile[c + 1]);
    }
    return a;
  };
  unsigned long long ep = cm.nranks > 1 ? *cm.epoch : 0ull;
  {
    double v[2] = {0.0, 0.0};
    for (int base = 0; base < S; base += stride) {
      const int s = base + gid;
      if (base + (gid & ~31) >= S) continue;
      const bool ok = s < S;
      const int c = ok ? s >> 2 : 0, k = s & 3;
      const double rk = ok ? g.bred[s] : 0.0;
      double zk = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double rm = grp4_get(rk, m);
        if (ok) zk += g.Minv[16ll * c + 4 * k + m] * rm;
      }
      if (ok && ((g.pinned[c] >> k) & 1)) zk = rk;
      if (ok) { x[s] = 0.0; r[s] = rk; z[s] = zk; p[s] = zk; }
      v[0] += rk * rk;
      v[1] += rk * zk;
    }
    block_reduce<2>(v, smred);
    if (threadIdx.x == 0) { part[2ll * blockIdx.x] = v[0]; part[2ll * blockIdx.x + 1] = v[1]; }
  }
  grid.sync();
  const double gn = sqrt(g.scal[SC_GNORM2]);
  const double tol = cg_tol * fmax(gn, 1e-300);
  double rr = cta_partials_sum(part, NP, 2, 0, &smb[0]);
  double rho = cta_partials_sum(part, NP, 2, 1, &smb[1]);
  double rn = sqrt(rr);
  int iters = 0, flag = 0;
  if (rn > tol) {
    while (true) {
      if (iters >= max_iters) { flag = ST_CG_MAXITER; break; }
      if constexpr (FUSED) {
        gp_fused_pass(g, fz, p, gdyn, smp, smy, smown);
      } else {
        gp_point_pass(g, p, g.yv, smp);
        grid.sync();
        gp_camera_pass(g, g.yv, tile4, smred);
      }
      grid.sync();
      if (cm.nranks > 1) {   // exchange the camera half of S*p with the peers (comm.cuh)
        ++ep;
        double* mine = cm.buf[cm.rank] + (long long)(ep & 1) * cm.cap;
        for (int s = gid; s < S; s += stride) mine[s] = local_cam(s);
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) comm_signal_wait(cm, ep);
        grid.sync();
      }
      {
        double v[1] = {0.0};
        for (int base = 0; base < S; base += stride) {
          const int s = base + gid;
          if (base + (gid & ~31) >= S) continue;
          const bool ok = s < S;
          const int c = ok ? s >> 2 : 0, k = s & 3;
          const double pk = ok ? p[s] : 0.0;
          const double p0 = grp4_get(pk, 0), p1 = grp4_get(pk, 1), p2 = grp4_get(pk, 2);
          if (ok) {
            double qk = 0.0;
            if (k < 3) {
              const double* B = g.Bp + 6ll * c;
              const double row[3][3] = {{B[0], B[1], B[2]}, {B[1], B[3], B[4]}, {B[2], B[4], B[5]}};
              double acc;
              if (cm.nranks > 1) {
                const long long off = (long long)(ep & 1) * cm.cap + s;
                acc = comm_peer_load(cm.buf[0] + off);
                for (int rk = 1; rk < cm.nranks; ++rk) acc += comm_peer_load(cm.buf[rk] + off);
              } else {
                acc = local_cam(s);
              }
              qk = row[k][0] * p0 + row[k][1] * p1 + row[k][2] * p2 - acc;
            }
            if ((g.pinned[c] >> k) & 1) qk = pk;
            q[s] = qk;
            v[0] += pk * qk;
          }
        }
        block_reduce<1>(v, smred);
        if (threadIdx.x == 0) part[2ll * NP + blockIdx.x] = v[0];
      }
      grid.sync();
      const double pq = cta_partials_sum(part + 2ll * NP, NP, 1, 0, &smb[0]);
      if (!isfinite(pq) || pq <= 0.0) { flag = ST_CG_BREAKDOWN; break; }
      const double alpha = rho / pq;
      {
        double v[2] = {0.0, 0.0};
        for (int base = 0; base < S; base += stride) {
          const int s = base + gid;
          if (base + (gid & ~31) >= S) continue;
          const bool ok = s < S;
          const int c = ok ? s >> 2 : 0, k = s & 3;
          double rk = 0.0;
          if (ok) { x[s] += alpha * p[s]; rk = r[s] - alpha * q[s]; r[s] = rk; }
          double zk = 0.0;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const double rm = grp4_get(rk, m);
            if (ok) zk += g.Minv[16ll * c + 4 * k + m] * rm;
          }
          if (ok) z[s] = zk;
          v[0] += rk * rk;
          v[1] += rk * zk;
        }
        block_reduce<2>(v, smred);
        if (threadIdx.x == 0) { part[2ll * blockIdx.x] = v[0]; part[2ll * blockIdx.x + 1] = v[1]; }
      }
      grid.sync();
      rr = cta_partials_sum(part, NP, 2, 0, &smb[0]);
      const double rz = cta_partials_sum(part, NP, 2, 1, &smb[1]);
      ++iters;
      rn = sqrt(rr);
      if (rn <= tol) break;
      const double beta = rz / rho;
      rho = rz;
      for (int s = gid; s < S; s += stride) p[s] = z[s] + beta * p[s];
      grid.sync();
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (cm.nranks > 1) *cm.epoch = ep;
    ctl->tol = tol; ctl->rho = rho; ctl->rn = rn; ctl->iters = iters; ctl->flag = flag;
    if (flag) atomicOr(g.status, flag);
  }
}

// back-substitution: points then scales (lm.py:674-704)
__global__ void __launch_bounds__(256) gp_k_backsub(GPDev g, const double* __restrict__ x,
                                                    double* delta) {
  __shared__ double sm[8][SSFM_BATCH][3];
  __shared__ double dpt[8][SSFM_BATCH][3];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long Np = g.Npad;
  const double lam = g.lamp ? *g.lamp : g.lam;   // LM graph: lambda on the device
  for (int b = gw; b < g.topo.nb; b += warps) {
    const int ob0 = g.topo.bat_obs[b], ob1 = g.topo.bat_obs[b + 1];
    const int pb0 = g.topo.bat_pt[b], pb1 = g.topo.bat_pt[b + 1];
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    if (my_pt < pb1) { ps = g.topo.pt_seg[my_pt]; pe = g.topo.pt_seg[my_pt + 1]; }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[3] = {0.0, 0.0, 0.0};
      if (i < ob1) {
        double rec[4];
        gp_rec_ld<false>(g.Jpm, Np, i, rec);
        const int c = g.topo.pm_cam[i];
        const double at = gp_at(g, c, rec[0]);
        const double inv = gp_inv(lam, rec);
        double xc[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) xc[k] = x[4ll * c + k];
        gp_u_mul(at, rec[0], inv, rec + 1, xc, val);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) sm[wib][lane][k] = val[k];
      __syncwarp();
      const int a0 = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a0; o < e; ++o)
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] += sm[wib][o - base][k];
      __syncwarp();
    }
    if (my_pt < pb1) {
      double M[6], w[3];
#pragma unroll
      for (int k = 0; k < 6; ++k) M[k] = g.Minv_pt[6ll * my_pt + k];
      sym3_matvec(M, acc, w);
      double* dst = delta + g.gp.off_pts + 3ll * my_pt;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double dv = g.y0[3ll * my_pt + k] - w[k];
        dst[k] = dv;
        dpt[wib][lane][k] = dv;
      }
    }
    __syncwarp();
    if (!g.gp.depth_mode) {
      // scales: delta_o = inv (b_o - a_t g.dc + a g.dj) with the original b_o
      for (int base = ob0; base < ob1; base += SSFM_BATCH) {
        const int i = base + lane;
        if (i < ob1) {
          double rec[4];
          gp_rec_ld<false>(g.Jpm, Np, i, rec);
          const int c = g.topo.pm_cam[i], j = g.topo.pm_pt[i];
          const double at = gp_at(g, c, rec[0]);
          const double inv = gp_inv(lam, rec);
          const double* dj = dpt[wib][j - pb0];
          double gc = 0.0, gj = 0.0;
#pragma unroll
          for (int k = 0; k < 3; ++k) { gc += rec[1 + k] * x[4ll * c + k]; gj += rec[1 + k] * dj[k]; }
          const double bo = g.bo_pm[i];
          delta[g.gp.off_sc + g.topo.pm_obs[i]] = inv * (bo - at * gc + rec[0] * gj);
        }
      }
    }
    __syncwarp();
  }
}

__global__ void gp_k_camdelta(GPDev g, const double* __restrict__ x, double* delta) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.gp.C) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) delta[3ll * c + k] = x[4ll * c + k];
}

// post_step (gp.py:130-147): mean scale, gauge transform, floor
__global__ void gp_k_scale_sum(GPDev g, const double* __restrict__ theta, double* part) {
  __shared__ double sm[32];
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  if (i < g.topo.N) v[0] = theta[g.gp.off_sc + i];
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

__global__ void gp_k_gauge_prep(GPDev g, const double* __restrict__ part, int n, const double* __restrict__ theta,
                                double* sum_cnt) {
  __shared__ double sm[32];
  double v[1] = {0.0};
  int per = (n + blockDim.x - 1) / blockDim.x;
  int a = threadIdx.x * per, b = min(n, a + per);
  for (int k = a; k < b; ++k) v[0] += part[k];
  block_reduce<1>(v, sm);
  if (threadIdx.x == 0) {
    if (sum_cnt) {   // sharded: (sum, count) for the allreduce, mean in gp_k_gauge_mean
      sum_cnt[0] = v[0];
      sum_cnt[1] = (double)g.topo.N;
    } else {
      g.scal[4] = v[0] / (double)g.topo.N;   // mean
    }
    g.scal[5] = theta[0]; g.scal[6] = theta[1]; g.scal[7] = theta[2];   // t0 copy
  }
}

__global__ void gp_k_gauge_mean(GPDev g, const double* sum_cnt) { g.scal[4] = sum_cnt[0] / sum_cnt[1]; }

__global__ void gp_k_gauge_apply(GPDev g, double* theta, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double m = g.scal[4];
  const bool xf = g.gp.gauge_fixed && m > 0.0 && isfinite(m);
  if (i >= g.gp.off_sc) {
    double s = theta[i];
    if (xf) s = s / m;
    theta[i] = fmax(s, GP_SCALE_FLOOR);
  } else if (xf) {
    const double t0 = g.scal[5 + (int)(i % 3)];
    theta[i] = MUL(theta[i], m) + MUL(SUB(1.0, m), t0);
  }
}

__global__ void k_export_grad_gp(GPDev g, double* grad, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i < g.gp.off_pts) grad[i] = g.gcam[i];
  else if (i < g.gp.off_sc) grad[i] = g.gpt[i - g.gp.off_pts];
  else grad[i] = g.gsc[i - g.gp.off_sc];
}

// ---------------------------------------------------------------------------
// host-side launch sequences for GP
// ---------------------------------------------------------------------------
static inline int gp_nblk(long long n, int t) { return (int)((n + t - 1) / t); }

static int gp_launch_linearize(GPDev& g, const double* theta, double* r_out, double* J_out,
                               double* red, int lin_blocks, int cam_blocks, cudaStream_t st) {
  gp_k_linearize<<<lin_blocks, 256, 0, st>>>(g, theta, r_out, J_out, red);
  if (g.topo.nt) gp_k_linearize_cm<<<g.topo.nt, SSFM_TILE, 0, st>>>(g, theta);
  const long long off = (long long)lin_blocks * 8;
  gp_k_camfin<<<cam_blocks, 256, 0, st>>>(g, red + off, nullptr);
  const int sb = gp_nblk(g.topo.N, 256);
  gp_k_scale_norm<<<sb, 256, 0, st>>>(g, red + off + cam_blocks);
  k_sum_partials<<<1, 1024, 0, st>>>(red, (int)(off + cam_blocks + sb), g.scal + SC_GNORM2);
  return cudaGetLastError() != cudaSuccess;
}

static int gp_launch_elim(GPDev& g, double lam, int cam_blocks, cudaStream_t st) {
  g.lam = lam;
  const int lin_blocks = std::max(1, gp_nblk(g.topo.nb, 8));
  gp_k_pt_elim<<<std::min(lin_blocks, 148 * 16), 256, 0, st>>>(g, lam);
  if (g.topo.nt) gp_k_cam_elim<<<g.topo.nt, SSFM_TILE, 0, st>>>(g, lam);
  gp_k_camprec<<<gp_nblk(g.gp.C, 64), 64, 0, st>>>(g, lam, nullptr);
  (void)cam_blocks;
  return cudaGetLastError() != cudaSuccess;
}

static int gp_launch_backsub(GPDev& g, const double* x, double* delta, int lin_blocks, int cam_blocks,
                             cudaStream_t st) {
  gp_k_backsub<<<lin_blocks, 256, 0, st>>>(g, x, delta);
  gp_k_camdelta<<<cam_blocks, 256, 0, st>>>(g, x, delta);
  return cudaGetLastError() != cudaSuccess;
}

static int gp_launch_post_step(GPDev& g, double* theta, double* red, cudaStream_t st) {
  if (g.gp.depth_mode) return 0;
  const int sb = gp_nblk(g.topo.N, 256);
  gp_k_scale_sum<<<sb, 256, 0, st>>>(g, theta, red);
  gp_k_gauge_prep<<<1, 1024, 0, st>>>(g, red, sb, theta, nullptr);
  const long long n = g.gp.off_sc + g.topo.N;
  gp_k_gauge_apply<<<gp_nblk(n, 256), 256, 0, st>>>(g, theta, n);
  return cudaGetLastError() != cudaSuccess;
}

static void gp_export_grad(GPDev& g, double* grad, cudaStream_t st) {
  const long long n = g.gp.off_sc + (g.gp.depth_mode ? 0 : g.topo.N);
  k_export_grad_gp<<<gp_nblk(n, 256), 256, 0, st>>>(g, grad, n);
}
