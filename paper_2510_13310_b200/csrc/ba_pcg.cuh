// ba_pcg.cuh -- the whole block-Jacobi PCG on the reduced camera system as
// ONE persistent cooperative kernel (lm.py:637-672), with the Schur operator
// applied matrix-free (replaces schur_fill_cy + the dense S@p at lm.py:656):
//
//   y_j      = Cinv_j  sum_{o in j} Jp_o^T (Jc_o p_c)          point pass  (P1)
//   t_tile   = sum_{o in tile} Jc_o^T (Jp_o y_j)               camera pass (P2)
//   (S p)_c  = B_c p_c + lam diag(B_c) p_c - sum_tiles t_tile  per camera  (P3)
//
// The reduced vector keeps 8 slots per camera (7 pose + 1 focal). Pinned
// slots (zero Schur diagonal) behave as identity rows, as in lm.py:628-635.
// All CTAs evaluate the scalar recurrences redundantly from the same partials
// in the same order, so control decisions are identical everywhere without
// extra broadcasts. No floating-point atomics.
#pragma once
#include <cooperative_groups.h>
#include "ba_kernels.cuh"
#include "fused.cuh"
#include "comm.cuh"

namespace cg = cooperative_groups;

struct CGCtl {
  double tol;
  double rho;
  double rn;
  double pq;
  int iters;
  int flag;     // 0 running/converged, ST_CG_* on failure
  int pad[2];
  // per-phase time of block 0 (ns, %globaltimer), accumulated over CG
  // iterations: [0] point / fused pass, [1] camera pass, [2] q = S p + p.q,
  // [3] x, r, z + r.r, r.z, [4] p update; each includes its grid barrier
  unsigned long long phase_ns[5];
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

#define PCG_THREADS 256

// Sum of per-CTA partials (n of them, stride ns) component k, evaluated by warp 0
// in a fixed order and broadcast through shared memory.
__device__ __forceinline__ double cta_partials_sum(const double* part, int n, int ns, int k,
                                                   double* smslot) {
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) s += part[(long long)i * ns + k];
    s = warp_sum(s);
    if (threadIdx.x == 0) *smslot = s;
  }
  __syncthreads();
  const double v = *smslot;
  __syncthreads();
  return v;
}

// Factored camera pass (ba_factor records, ba.cuh). Per observation it
// streams 7 (pinhole) / 9 (bal) doubles (S, e, phi, v = X - t) + 1 index
// instead of the 16-double Jacobian record, and applies the tile's camera
// (R, Pi from camlin, the linearization's camera cache) once per tile: C5
// camera pass 0.535 -> 0.329 ms. The operator is the stored Jacobian's to
// rounding. (A factored point pass lost, 0.555 -> 0.832 ms: every observation
// gathers its camera's R, qh, t through L1, which saturates at 89 %; the
// point pass keeps the Jacobian record.)

#ifndef CAMF_MINB
#define CAMF_MINB 2      // CTAs per SM of the factored camera pass
#endif
#ifndef CAMF_UNROLL
#define CAMF_UNROLL 2
#endif
constexpr int kCamfUnroll = CAMF_UNROLL;
#ifndef CAMF_HOIST
#define CAMF_HOIST 1     // keep the tile camera's R, qh in registers across the loop
#endif
#ifndef CAMF_PF
#define CAMF_PF 1        // point indices CAMF_PFD rounds ahead (ba_camera_pass_f)
#endif
#ifndef CAMF_PFD
#define CAMF_PFD 4        // C5 camera pass 0.259 -> 0.252 ms (2 and 3 equal)
#endif
template <bool RO>
__device__ __forceinline__ void ba_camera_pass_f(const BADev& d, const double* y, double* tile8) {
  const unsigned long long pstream = pol_evict_first(), pkeep = pol_evict_last();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int t = gw; t < d.topo.nt; t += warps) {
    const int o0 = __ldg(d.topo.tile_obs + t), o1 = __ldg(d.topo.tile_obs + t + 1);
    const int c = __ldg(d.topo.tile_cam + t);
    const double* cb = reinterpret_cast<const double*>(d.camlin + c);
    double o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = 0.0;
#if CAMF_HOIST
    double R[9], qh[4];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(cb + k);
#pragma unroll
    for (int k = 0; k < 4; ++k) qh[k] = __ldg(cb + 9 + k);
#endif
#if CAMF_PF
    // the point index one round ahead: a round's y gather is issued together
    // with its record stream instead of behind the index's DRAM latency
    // (CAMF_PFD rounds ahead: the loop is unrolled by two)
    int jq[CAMF_PFD];
#pragma unroll
    for (int q = 0; q < CAMF_PFD; ++q) jq[q] = o0 + lane + 32 * q < o1 ? ldg_stream_i(d.topo.cm_pt + o0 + lane + 32 * q, pstream) : 0;
#endif
#pragma unroll kCamfUnroll
    for (int i = o0 + lane; i < o1; i += 32) {
#if !CAMF_HOIST
      // the tile's camera: warp-uniform addresses, L1 broadcasts (not kept
      // in registers across the loop: register budget)
      double R[9], qh[4];
#pragma unroll
      for (int k = 0; k < 9; ++k) R[k] = __ldg(cb + k);
#pragma unroll
      for (int k = 0; k < 4; ++k) qh[k] = __ldg(cb + 9 + k);
#endif
      double f[6], vv[3];
#if CAMF_PF
      const int j = jq[0];
      double yj[4];
      if constexpr (RO) ld_v4_ro(y + 4ll * j, yj, pkeep);
      else ld_v4_hint(y + 4ll * j, yj, pkeep);
      fcm_load(d, i, f, vv, pstream);
#pragma unroll
      for (int q = 0; q + 1 < CAMF_PFD; ++q) jq[q] = jq[q + 1];
      if (i + 32 * CAMF_PFD < o1) jq[CAMF_PFD - 1] = ldg_stream_i(d.topo.cm_pt + i + 32 * CAMF_PFD, pstream);
#else
      fcm_load(d, i, f, vv, pstream);
      const int j = ldg_stream_i(d.topo.cm_pt + i, pstream);
      double yj[4];
      if constexpr (RO) ld_v4_ro(y + 4ll * j, yj, pkeep);
      else ld_v4_hint(y + 4ll * j, yj, pkeep);
#endif
      double ry[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) ry[r] = R[3 * r] * yj[0] + R[3 * r + 1] * yj[1] + R[3 * r + 2] * yj[2];
      const double h0 = ry[0] - f[1] * ry[2], h1 = ry[1] - f[2] * ry[2];
      const double s0 = f[0] * h0 + f[4] * h1, s1 = f[4] * h0 + f[5] * h1;
      const double k0 = f[0] * s0 + f[4] * s1, k1 = f[4] * s0 + f[5] * s1;
      const double g[3] = {k0, k1, -(f[1] * k0 + f[2] * k1)};
      double dt[4];
      ba_dqt_mul(qh, vv, g, dt);
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] += dt[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) o[4 + k] += g[k];
      o[7] += f[3] * (f[1] * s0 + f[2] * s1);
    }
    warp_allreduce<8>(o);
    // camera frame -> theta slots: quaternion Pi (.), centre -R^T (.)
#if !CAMF_HOIST
    double R[9], qh[4];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(cb + k);
#pragma unroll
    for (int k = 0; k < 4; ++k) qh[k] = __ldg(cb + 9 + k);
#endif
    double out[8];
    ba_pi_mul(qh, __ldg(cb + 22), o, out);
#pragma unroll
    for (int m = 0; m < 3; ++m) out[4 + m] = -(R[m] * o[4] + R[3 + m] * o[5] + R[6 + m] * o[6]);
    out[7] = o[7];
    if (lane < 8) {
      double x = out[0];
#pragma unroll
      for (int k = 1; k < 8; ++k) x = lane == k ? out[k] : x;
      tile8[8ll * t + lane] = x;
    }
  }
}

#ifndef PTP_PF
#define PTP_PF 0         // L2 bulk prefetch of the next batch's records
#endif
#ifndef PTP_PIPE
#define PTP_PIPE 0       // software-pipelined point pass (ba_point_pass_pipe)
#endif
#if PTP_PIPE
#define PTP_THREADS 128
#ifndef PTP_MINB
#define PTP_MINB 6
#endif
#else
#ifndef PTP_THREADS
#define PTP_THREADS PCG_THREADS
#endif
#ifndef PTP_MINB
#define PTP_MINB (4 * PCG_THREADS / PTP_THREADS)
#endif
#endif
// P1 for a camera vector v -> y (per point): y_j = Cinv_j sum_o Jp^T (Jc v_c)
template <bool RO = false>
__device__ __forceinline__ void ba_point_pass(const BADev& d, const double* v, double* y,
                                              double (*sm)[SSFM_BATCH][3]) {
  const unsigned long long pstream = pol_evict_first(), pkeep = pol_evict_last();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long Np = d.Npad;
#if PTP_PF
  // batch bounds carried one batch ahead; the next batch's Jacobian rows,
  // camera ids and Cinv blocks are prefetched into L2 (bulk requests, one per
  // lane) while this batch runs
  int nb0 = 0, nb1 = 0, np0 = 0, np1 = 0;
  if (gw + warps < d.topo.nb) {
    nb0 = d.topo.bat_obs[gw + warps]; nb1 = d.topo.bat_obs[gw + warps + 1];
    np0 = d.topo.bat_pt[gw + warps]; np1 = d.topo.bat_pt[gw + warps + 1];
  }
#endif
  for (int b = gw; b < d.topo.nb; b += warps) {
    const int ob0 = d.topo.bat_obs[b], ob1 = d.topo.bat_obs[b + 1];
    const int pb0 = d.topo.bat_pt[b], pb1 = d.topo.bat_pt[b + 1];
#if PTP_PF
    if (b + warps < d.topo.nb) {
      if (lane < BA_JREC) pf_l2_bulk(d.Jpm + lane * Np + nb0, 8ll * (nb1 - nb0));
      else if (lane == BA_JREC) pf_l2_bulk(d.topo.pm_cam + nb0, 4ll * (nb1 - nb0));
      else if (lane == BA_JREC + 1) pf_l2_bulk(d.Cinv + 6ll * np0, 48ll * (np1 - np0));
      const int bn = b + 2 * warps;
      if (bn < d.topo.nb) {
        nb0 = d.topo.bat_obs[bn]; nb1 = d.topo.bat_obs[bn + 1];
        np0 = d.topo.bat_pt[bn]; np1 = d.topo.bat_pt[bn + 1];
      }
    }
#endif
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    if (my_pt < pb1) { ps = d.topo.pt_seg[my_pt]; pe = d.topo.pt_seg[my_pt + 1]; }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[3] = {0.0, 0.0, 0.0};
      if (i < ob1) {
        double J[BA_JREC];
#pragma unroll
        for (int k = 0; k < BA_JREC; ++k) J[k] = ldg_stream(d.Jpm + k * Np + i, pstream);
        const int c = ldg_stream_i(d.topo.pm_cam + i, pstream);
        double pc[8];
        if constexpr (RO) {
          ld_v4_ro(v + 8ll * c, pc, pkeep);
          ld_v4_ro(v + 8ll * c + 4, pc + 4, pkeep);
        } else {
          ld_v4(v + 8ll * c, pc);
          ld_v4(v + 8ll * c + 4, pc + 4);
        }
        if (d.bp.focal_mode == 2) pc[7] = v[7];   // shared focal (camera 0, slot 7)
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
      for (int k = 0; k < 6; ++k) ci[k] = __ldg(d.Cinv + 6ll * my_pt + k);
      sym3_matvec(ci, acc, w);
#pragma unroll
      for (int k = 0; k < 3; ++k) st_hint(y + 4ll * my_pt + k, w[k], pkeep);
    }
  }
}

#ifndef PTW_PIPE
#define PTW_PIPE 1      // index prefetch one round ahead, contiguous batch ranges per warp
#endif
#ifndef PTW_CIEARLY
// owners load Cinv at the batch start (C5 point pass 0.46 -> 0.45 ms without
// PTW_PIPE; with it the 12 registers spill)
#define PTW_CIEARLY (!PTW_PIPE)
#endif
#if PTW_PIPE
// P1 in the omega form (ba_wobs): W = the per-camera vector of p (ba_wvec).
// Streams the 64-byte Jp + Jf record and the camera and point indices per
// observation, gathers W_c (64 bytes, L2-resident) and X_j (32 bytes).
//
// Latency structure. The loads are issued in program order (volatile asm), so
// a gather whose address comes from an index loaded in the same round puts
// the index's DRAM latency in front of everything after it. Here each warp
// owns a contiguous range of batches, so the next round's observation range
// is known without a load, and its camera / point indices are requested one
// round ahead. A round then issues the record stream and both gathers at once
// (their addresses are already in registers): one DRAM latency per round
// instead of index -> record -> gather. Same per-point summation order and
// arithmetic as before: the output is bit-identical.
// BS: back-substitution (lm.py:674-690) instead of y: delta_j = y0_j - Cinv_j
// sum_o Jp^T (Jc x_c), W = the per-camera vector of x, written at
// y + off_pts + 3j
template <bool RO = false, bool BS = false>
__device__ __forceinline__ void ba_point_pass_w(const BADev& d, const double* W, double* y,
                                                double (*sm)[SSFM_BATCH][3]) {
  const unsigned long long pstream = pol_evict_first(), pkeep = pol_evict_last();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nb = d.topo.nb;
  const int b0 = (int)((long long)nb * gw / warps), b1 = (int)((long long)nb * (gw + 1) / warps);
  if (b0 >= b1) return;   // warp-uniform
  int ob0 = d.topo.bat_obs[b0], ob1 = d.topo.bat_obs[b0 + 1], pb0 = d.topo.bat_pt[b0];
  int cn = 0, jn = 0;
  if (ob0 + lane < ob1) {
    cn = ldg_stream_i(d.topo.pm_cam + ob0 + lane, pstream);
    jn = ldg_stream_i(d.topo.pm_pt + ob0 + lane, pstream);
  }
  for (int b = b0; b < b1; ++b) {
    const int pb1 = d.topo.bat_pt[b + 1];
    const int nob1 = b + 1 < b1 ? d.topo.bat_obs[b + 2] : ob1;   // end of the next batch
    const int my_pt = pb0 + lane;
    const bool own = my_pt < pb1;
    int ps = 0, pe = 0;
#if PTW_CIEARLY
    double ci[6];
#endif
    if (own) {
      ps = d.topo.pt_seg[my_pt]; pe = d.topo.pt_seg[my_pt + 1];
#if PTW_CIEARLY
#pragma unroll
      for (int k = 0; k < 6; ++k) ci[k] = __ldg(d.Cinv + 6ll * my_pt + k);
#endif
    }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      const int c = cn, j = jn;
      const bool act = i < ob1;
      double G[8], w[8], X[4];
      if (act) gpm_load(d, i, G, pstream);
      // the next round's indices: this batch's next round or the next batch's first
      const bool more = base + SSFM_BATCH < ob1;
      const int ni = more ? i + SSFM_BATCH : ob1 + lane, nend = more ? ob1 : nob1;
      if (ni < nend) {
        cn = ldg_stream_i(d.topo.pm_cam + ni, pstream);
        jn = ldg_stream_i(d.topo.pm_pt + ni, pstream);
      }
      double val[3] = {0.0, 0.0, 0.0};
      if (act) {
        if constexpr (RO) {
          ld_v4_ro(W + 8ll * c, w, pkeep);
          ld_v4_ro(W + 8ll * c + 4, w + 4, pkeep);
        } else {
          ld_v4(W + 8ll * c, w);
          ld_v4(W + 8ll * c + 4, w + 4);
        }
        ld_v4_ro(d.Xl + 4ll * j, X, pkeep);
        ba_wobs_math(G, w, X, val);
      }
      const int a = max(ps, base), e = min(pe, base + SSFM_BATCH);
#pragma unroll
      for (int k = 0; k < 3; ++k) sm[wib][lane][k] = val[k];
      __syncwarp();
      for (int o = a; o < e; ++o) {
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] += sm[wib][o - base][k];
      }
      __syncwarp();
    }
    if (own) {
      double w3[3];
#if !PTW_CIEARLY
      double ci[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) ci[k] = __ldg(d.Cinv + 6ll * my_pt + k);
#endif
      sym3_matvec(ci, acc, w3);
      if constexpr (BS) {
        double* dst = y + d.bp.off_pts + 3ll * my_pt;
#pragma unroll
        for (int k = 0; k < 3; ++k) dst[k] = d.y0[3ll * my_pt + k] - w3[k];
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) st_hint(y + 4ll * my_pt + k, w3[k], pkeep);
      }
    }
    ob0 = ob1; ob1 = nob1; pb0 = pb1;
  }
}
#else
// P1 in the omega form (ba_wobs): W = the per-camera vector of p (ba_wvec).
// Streams the 64-byte Jp + Jf record and the camera and point indices per
// observation (the 16-double record and one index before), gathers W_c (64
// bytes, L2-resident) and X_j (32 bytes).
// BS: back-substitution (lm.py:674-690) instead of y: delta_j = y0_j - Cinv_j
// sum_o Jp^T (Jc x_c), W = the per-camera vector of x, written at
// y + off_pts + 3j
template <bool RO = false, bool BS = false>
__device__ __forceinline__ void ba_point_pass_w(const BADev& d, const double* W, double* y,
                                                double (*sm)[SSFM_BATCH][3]) {
  const unsigned long long pstream = pol_evict_first(), pkeep = pol_evict_last();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int b = gw; b < d.topo.nb; b += warps) {
    const int ob0 = d.topo.bat_obs[b], ob1 = d.topo.bat_obs[b + 1];
    const int pb0 = d.topo.bat_pt[b], pb1 = d.topo.bat_pt[b + 1];
    const int my_pt = pb0 + lane;
    const bool own = my_pt < pb1;
    int ps = 0, pe = 0;
#if PTW_CIEARLY
    double ci[6];
#endif
    if (own) {
      ps = d.topo.pt_seg[my_pt]; pe = d.topo.pt_seg[my_pt + 1];
#if PTW_CIEARLY   // the owner's Cinv in flight during the batch (not after its reduction)
#pragma unroll
      for (int k = 0; k < 6; ++k) ci[k] = __ldg(d.Cinv + 6ll * my_pt + k);
#endif
    }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[3] = {0.0, 0.0, 0.0};
      if (i < ob1) {
        const int c = ldg_stream_i(d.topo.pm_cam + i, pstream);
        const int j = ldg_stream_i(d.topo.pm_pt + i, pstream);
        double X[4];
        ld_v4_ro(d.Xl + 4ll * j, X, pkeep);
        ba_wobs<RO>(d, i, c, W, X, val);
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
    if (own) {
      double w[3];
#if !PTW_CIEARLY
      double ci[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) ci[k] = __ldg(d.Cinv + 6ll * my_pt + k);
#endif
      sym3_matvec(ci, acc, w);
      if constexpr (BS) {
        double* dst = y + d.bp.off_pts + 3ll * my_pt;
#pragma unroll
        for (int k = 0; k < 3; ++k) dst[k] = d.y0[3ll * my_pt + k] - w[k];
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) st_hint(y + 4ll * my_pt + k, w[k], pkeep);
      }
    }
  }
}
#endif

// P1, software-pipelined: while a warp works on batch b, the Jacobian rows
// and camera ids of its next batch are already in flight into a second
// shared-memory stage (cp.async, no registers held), and batch b's Cinv
// blocks are requested at the top of the batch instead of after the
// reduction. Batch bounds are carried two batches ahead, so no load in the
// loop head waits on another load. Batches with more than 32 observations (a
// point seen more than 32 times) are read directly, round by round.
struct PtpStage {
  double J[BA_JREC][SSFM_BATCH];
  int cam[SSFM_BATCH];
};

__device__ __forceinline__ void ptp_issue(const BADev& d, int o0, int o1, PtpStage& s, unsigned long long pol,
                                          int lane) {
  const long long Np = d.Npad;
  const int i = o0 + lane;
  if (o1 - o0 <= SSFM_BATCH && i < o1) {
#pragma unroll
    for (int k = 0; k < BA_JREC; ++k) cp_async8(&s.J[k][lane], d.Jpm + k * Np + i, pol);
    cp_async4(&s.cam[lane], d.topo.pm_cam + i, pol);
  }
  cp_commit();
}

template <bool RO>
__device__ __forceinline__ void ptp_obs(const BADev& d, const double* v, const double* J, int c, double* val) {
  double pc[8];
  if constexpr (RO) {
    const unsigned long long pkeep = pol_evict_last();
    ld_v4_ro(v + 8ll * c, pc, pkeep);
    ld_v4_ro(v + 8ll * c + 4, pc + 4, pkeep);
  } else {
    ld_v4(v + 8ll * c, pc);
    ld_v4(v + 8ll * c + 4, pc + 4);
  }
  if (d.bp.focal_mode == 2) pc[7] = v[7];   // shared focal (camera 0, slot 7)
  double t[2];
  ba_jc_mul(J, pc, t);
  ba_jpt_mul(J, t, val);
}

template <bool RO = false>
__device__ __forceinline__ void ba_point_pass_pipe(const BADev& d, const double* v, double* y, PtpStage (*stg)[2],
                                                   double (*sm)[SSFM_BATCH][3]) {
  const unsigned long long pstream = pol_evict_first(), pkeep = pol_evict_last();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long Np = d.Npad;
  const int nb = d.topo.nb;
  auto bounds = [&](int b, int& o0, int& o1, int& p0, int& p1) {
    if (b < nb) {
      o0 = d.topo.bat_obs[b]; o1 = d.topo.bat_obs[b + 1];
      p0 = d.topo.bat_pt[b]; p1 = d.topo.bat_pt[b + 1];
    } else {
      o0 = o1 = p0 = p1 = 0;
    }
  };
  int ob0, ob1, pb0, pb1, nb0, nb1, np0, np1;
  bounds(gw, ob0, ob1, pb0, pb1);
  bounds(gw + warps, nb0, nb1, np0, np1);
  int st = 0;
  ptp_issue(d, ob0, ob1, stg[wib][0], pstream, lane);
  for (int b = gw; b < nb; b += warps) {
    ptp_issue(d, nb0, nb1, stg[wib][st ^ 1], pstream, lane);   // next batch (empty group past the end)
    int xb0, xb1, xp0, xp1;
    bounds(b + 2 * warps, xb0, xb1, xp0, xp1);
    const int my_pt = pb0 + lane;
    int ps = 0, pe = 0;
    double ci[6];
    if (my_pt < pb1) {
      ps = d.topo.pt_seg[my_pt];
      pe = d.topo.pt_seg[my_pt + 1];
#pragma unroll
      for (int k = 0; k < 6; ++k) ci[k] = __ldg(d.Cinv + 6ll * my_pt + k);
    }
    double acc[3] = {0.0, 0.0, 0.0};
    const bool staged = ob1 - ob0 <= SSFM_BATCH;
    cp_wait<1>();
    __syncwarp();
    for (int base = ob0; base < ob1; base += SSFM_BATCH) {
      const int i = base + lane;
      double val[3] = {0.0, 0.0, 0.0};
      if (i < ob1) {
        double J[BA_JREC];
        int c;
        if (staged) {
#pragma unroll
          for (int k = 0; k < BA_JREC; ++k) J[k] = stg[wib][st].J[k][lane];
          c = stg[wib][st].cam[lane];
        } else {
#pragma unroll
          for (int k = 0; k < BA_JREC; ++k) J[k] = ldg_stream(d.Jpm + k * Np + i, pstream);
          c = ldg_stream_i(d.topo.pm_cam + i, pstream);
        }
        ptp_obs<RO>(d, v, J, c, val);
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
      double w[3];
      sym3_matvec(ci, acc, w);
#pragma unroll
      for (int k = 0; k < 3; ++k) st_hint(y + 4ll * my_pt + k, w[k], pkeep);
    }
    ob0 = nb0; ob1 = nb1; pb0 = np0; pb1 = np1;
    nb0 = xb0; nb1 = xb1; np0 = xp0; np1 = xp1;
    st ^= 1;
  }
  cp_wait<0>();
}

// P2: per camera tile, sum Jc^T (Jp y_j) -> tile8[t][8]. One WARP per tile:
// lanes accumulate the tile's observations round by round in registers, then
// one butterfly reduction; no CTA barriers (a block reduction per 256-obs
// tile left 30 % of the warps waiting at __syncthreads). Fixed order:
// deterministic.
template <bool RO = false>
__device__ __forceinline__ void ba_camera_pass(const BADev& d, const double* y, double* tile8,
                                               double* smred) {
  (void)smred;
  const unsigned long long pstream = pol_evict_first(), pkeep = pol_evict_last();
  const long long Np = d.Npad;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int t = gw; t < d.topo.nt; t += warps) {
    const int o0 = __ldg(d.topo.tile_obs + t), o1 = __ldg(d.topo.tile_obs + t + 1);
    double o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = 0.0;
#pragma unroll 2
    for (int i = o0 + lane; i < o1; i += 32) {
      double J[BA_JREC];
#pragma unroll
      for (int k = 0; k < BA_JREC; ++k) J[k] = ldg_stream(d.Jcm + k * Np + i, pstream);
      const int j = ldg_stream_i(d.topo.cm_pt + i, pstream);
      double yj[4];
      if constexpr (RO) ld_v4_ro(y + 4ll * j, yj, pkeep);
      else ld_v4_hint(y + 4ll * j, yj, pkeep);
      double tt[2], u[8];
      ba_jp_mul(J, yj, tt);
      ba_jct_mul(J, tt, u);
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] += u[k];
    }
    warp_allreduce<8>(o);
    if (lane < 8) {
      double v = o[0];
#pragma unroll
      for (int k = 1; k < 8; ++k) v = lane == k ? o[k] : v;
      tile8[8ll * t + lane] = v;
    }
  }
}


// Fused single pass (fused.cuh): y_j for every point of the warp's batch,
// then the camera terms Jc^T Jp y_j added into the CTA's slot group of the
// shared-memory camera vector `acc` (SL slots per camera) in ticket order.
// Finally the CTA writes its slot group to gpart[grp][8C].
// Dynamic shared memory: acc [SL*C] doubles | stage [FZ_WARPS][32][SL] doubles |
// cnt [C] ints.
template <int SL>
__device__ __forceinline__ void ba_fused_pass(const BADev& d, const FusedTopo& fz,
                                              const double* __restrict__ v, double* dyn,
                                              double (*smv)[SSFM_BATCH][3],
                                              double (*smy)[SSFM_BATCH][3],
                                              int (*smown)[SSFM_BATCH]) {
  constexpr int G = 8 / SL;
  const unsigned long long pstream = pol_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x % G, grp = blockIdx.x / G, ngrp = gridDim.x / G;
  const int C = d.bp.C;
  const long long Np = d.Npad;
  double* acc = dyn;
  double* stage = dyn + (long long)SL * C + (long long)warp * 32 * SL;   // [SL][32] per warp
  int* cnt = reinterpret_cast<int*>(dyn + (long long)SL * C + FZ_WARPS * 32 * SL);
  for (int k = threadIdx.x; k < SL * C; k += blockDim.x) acc[k] = 0.0;
  for (int k = threadIdx.x; k < C; k += blockDim.x) cnt[k] = 0;
  __syncthreads();
  // batch metadata is prefetched one batch ahead; Cinv, ticket and J of a
  // batch are issued together so each batch costs ~2 dependent latencies
  // (J/cam -> p gather) instead of a chain of five.
  const int sstride = ngrp * FZ_WARPS;
  int b = grp * FZ_WARPS + warp;
  int nob0 = 0, nob1 = 0, npb0 = 0, npb1 = 0;
  if (b < d.topo.nb) {
    nob0 = __ldg(d.topo.bat_obs + b); nob1 = __ldg(d.topo.bat_obs + b + 1);
    npb0 = __ldg(d.topo.bat_pt + b); npb1 = __ldg(d.topo.bat_pt + b + 1);
  }
  for (; b < d.topo.nb; b += sstride) {
    const int ob0 = nob0, ob1 = nob1, pb0 = npb0, pb1 = npb1;
    const int my_pt = pb0 + lane;
    const bool own = my_pt < pb1;
    int ps = 0, pe = 0;
    double ci[6];
    if (own) {
      ps = __ldg(d.topo.pt_seg + my_pt); pe = __ldg(d.topo.pt_seg + my_pt + 1);
#pragma unroll
      for (int k = 0; k < 6; ++k) ci[k] = __ldg(d.Cinv + 6ll * my_pt + k);
    }
    {
      const int bn = b + sstride;
      if (bn < d.topo.nb) {
        nob0 = __ldg(d.topo.bat_obs + bn); nob1 = __ldg(d.topo.bat_obs + bn + 1);
        npb0 = __ldg(d.topo.bat_pt + bn); npb1 = __ldg(d.topo.bat_pt + bn + 1);
      }
    }
    const int rounds = (ob1 - ob0 + 31) >> 5;
    double J[BA_JREC];
    int c = 0, tk = 0;
    double a3[3] = {0.0, 0.0, 0.0};
    // phase 1: per-point sums of Jp^T Jc p (observation order)
    for (int r = 0; r < rounds; ++r) {
      const int base = ob0 + 32 * r;
      const int i = base + lane;
      double val[3] = {0.0, 0.0, 0.0};
      if (i < ob1) {
        c = __ldg(d.topo.pm_cam + i);
#pragma unroll
        for (int k = 0; k < BA_JREC; ++k) J[k] = ldg_stream(d.Jpm + k * Np + i, pstream);
        tk = __ldg(fz.tick + i);
        double pc[8];
        ld_v4(v + 8ll * c, pc);
        ld_v4(v + 8ll * c + 4, pc + 4);
        if (d.bp.focal_mode == 2) pc[7] = v[7];   // shared focal (camera 0, slot 7)
        double t[2];
        ba_jc_mul(J, pc, t);
        ba_jpt_mul(J, t, val);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) smv[warp][lane][k] = val[k];
      __syncwarp();
      const int a = max(ps, base), e = min(pe, base + SSFM_BATCH);
      for (int o = a; o < e; ++o) {
#pragma unroll
        for (int k = 0; k < 3; ++k) a3[k] += smv[warp][o - base][k];
        smown[warp][o - base] = lane;
      }
      __syncwarp();
    }
    if (own) {
      double w[3];
      sym3_matvec(ci, a3, w);
#pragma unroll
      for (int k = 0; k < 3; ++k) smy[warp][lane][k] = w[k];
    }
    __syncwarp();
    // phase 2: camera terms, ticket-ordered accumulation
    for (int r = 0; r < rounds; ++r) {
      const int i = ob0 + 32 * r + lane;
      const bool have = i < ob1;
      double u[SL];
#pragma unroll
      for (int j = 0; j < SL; ++j) u[j] = 0.0;
      int t = 0;
      if (have) {
        if (rounds > 1) {   // a single point with > 32 observations: reload its round
#pragma unroll
          for (int k = 0; k < BA_JREC; ++k) J[k] = ldg_stream(d.Jpm + k * Np + i, pstream);
          c = __ldg(d.topo.pm_cam + i);
          tk = __ldg(fz.tick + i);
        }
        t = tk;
        const int owner = rounds > 1 ? 0 : smown[warp][lane];
        double y[3], t2[2], o[8];
#pragma unroll
        for (int k = 0; k < 3; ++k) y[k] = smy[warp][owner][k];
        ba_jp_mul(J, y, t2);
        ba_jct_mul(J, t2, o);
#pragma unroll
        for (int m = 0; m < 8; ++m)
          if (m / SL == g) u[m % SL] = o[m];
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
        while (ld_acquire_smem(cnt + c) != t) {
          if (++spins > FZ_SPIN_LIMIT) { atomicOr(d.status, ST_SCHEDULE); break; }
        }
        fz_add<SL>(acc, c, u);
        st_release_smem(cnt + c, t + 1);
      }
    }
    __syncwarp();
  }
  __syncthreads();
  double* dst = fz.gpart + (long long)grp * 8 * C;
  for (int k = threadIdx.x; k < SL * C; k += blockDim.x) {
    const int c = k / SL, j = k - c * SL;
    dst[8ll * c + g * SL + j] = acc[fz_slot<SL>(c, j)];
  }
}

// The whole PCG as one persistent cooperative kernel. SL = 0: two-pass
// operator (P1 point pass, P2 camera tiles). SL > 0: fused single pass with
// 8/SL slot groups (fused.cuh); needs SL*C doubles of dynamic shared memory.
template <int SL, bool FAC = false>
__global__ void __launch_bounds__(SL ? FZ_THREADS : PCG_THREADS, SL ? 1 : 4)
ba_k_pcg(BADev d, FusedTopo fz, CommDev cm, double lam, int max_iters, double cg_tol, double* x,
         double* r, double* z, double* p, double* q, double* part, CGCtl* ctl) {
  constexpr int NT = SL ? FZ_THREADS : PCG_THREADS;
  if (d.lamp) lam = *d.lamp;   // LM loop as a CUDA graph: lambda lives on the device
  cg::grid_group grid = cg::this_grid();
  __shared__ double smp[NT / 32][SSFM_BATCH][3];
  __shared__ double smy[SL ? NT / 32 : 1][SSFM_BATCH][3];
  __shared__ int smown[SL ? NT / 32 : 1][SSFM_BATCH];
  __shared__ double smred[(NT / 32) * 8];
  __shared__ double smb[4];
  extern __shared__ double dyn_acc[];
  const int S = 8 * d.bp.C;
  const int stride = gridDim.x * blockDim.x;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  double* tile8 = d.tilebuf;
  const int NP = gridDim.x;
  const int ngrp = SL ? gridDim.x / (8 / (SL ? SL : 8)) : 0;
  // local camera half of S*p for slot s = 8c + k (tile or group partials in order)
  auto local_cam = [&](int s) -> double {
    double a = 0.0;
    if constexpr (SL == 0) {
      const int c = s >> 3, k = s & 7;
      a = tiles_sum<8>(tile8, k, d.topo.cam_tile[c], d.topo.cam_tile[c + 1]);
    } else {
      for (int gq = 0; gq < ngrp; ++gq) a += fz.gpart[(long long)gq * S + s];
    }
    return a;
  };
  unsigned long long ep = cm.nranks > 1 ? *cm.epoch : 0ull;
  // phase timers of block 0 live in shared memory (no registers held across
  // the passes)
  __shared__ unsigned long long ph[5], pt0;
  if (threadIdx.x == 0) { for (int k = 0; k < 5; ++k) ph[k] = 0ull; }
  const bool shared = d.bp.focal_mode == 2;
  double qf = 0.0;

  // ---- init: x = 0, r = b_red, z = M r, p = z
  {
    double v[2] = {0.0, 0.0};
    for (int base = 0; base < S; base += stride) {
      const int s = base + gid;
      const bool ok = s < S;
      if (base + (gid & ~31) >= S) continue;   // whole warp out of range
      const int c = ok ? s >> 3 : 0, k = s & 7;
      const double rk = ok ? d.bred[s] : 0.0;
      double zk = 0.0;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const double rm = grp8_get(rk, m);
        if (ok) zk += d.Minv[64ll * c + 8 * k + m] * rm;
      }
      if (ok) { x[s] = 0.0; r[s] = rk; z[s] = zk; p[s] = zk; }
      v[0] += rk * rk;
      v[1] += rk * zk;
    }
    block_reduce<2>(v, smred);
    if (threadIdx.x == 0) { part[2ll * blockIdx.x] = v[0]; part[2ll * blockIdx.x + 1] = v[1]; }
  }
  grid.sync();
  if (d.Gpm) {   // omega-form point pass: the per-camera vector of p
    for (int c = gid; c < d.bp.C; c += stride) ba_wvec(d, p, c, d.Wc);
    grid.sync();
  }
  const double gn = sqrt(d.scal[SC_GNORM2]);
  const double tol = cg_tol * fmax(gn, 1e-300);
  double rr = cta_partials_sum(part, NP, 2, 0, &smb[0]);
  double rho = cta_partials_sum(part, NP, 2, 1, &smb[1]);
  double pf = shared ? p[7] : 0.0;
  double rn = sqrt(rr);
  int iters = 0;
  int flag = 0;
  if (rn > tol) {
    while (true) {
      if (iters >= max_iters) { flag = ST_CG_MAXITER; break; }
      const bool tim = blockIdx.x == 0 && threadIdx.x == 0;
      if (tim) pt0 = gtimer();
      if constexpr (SL == 0) {
        // P1: point pass
        if (d.Gpm) ba_point_pass_w(d, d.Wc, d.yv, smp);
        else ba_point_pass(d, p, d.yv, smp);
        grid.sync();
        if (tim) { const unsigned long long t1 = gtimer(); ph[0] += t1 - pt0; pt0 = t1; }
        // P2: camera tiles
        if constexpr (FAC) ba_camera_pass_f<false>(d, d.yv, tile8);
        else ba_camera_pass(d, d.yv, tile8, smred);
      } else {
        ba_fused_pass<SL>(d, fz, p, dyn_acc, smp, smy, smown);
      }
      grid.sync();
      if (tim) { const unsigned long long t1 = gtimer(); ph[SL == 0 ? 1 : 0] += t1 - pt0; pt0 = t1; }
      // P2x (sharded): exchange the local camera half of S*p with the peer
      // ranks inside the kernel (comm.cuh); P3 then sums the ranks in order.
      if (cm.nranks > 1) {
        ++ep;
        double* mine = cm.buf[cm.rank] + (long long)(ep & 1) * cm.cap;
        if constexpr (SL == 0) {
          for (int s = gid; s < S; s += stride) mine[s] = local_cam(s);
        } else {   // one warp per slot (see P3)
          const int lane = threadIdx.x & 31;
          for (int s = gid >> 5; s < S; s += stride >> 5) {
            double a = 0.0;
#pragma unroll 4
            for (int g = lane; g < ngrp; g += 32) a += fz.gpart[(long long)g * S + s];
            a = warp_sum(a);
            if (lane == 0) mine[s] = a;
          }
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) comm_signal_wait(cm, ep);
        grid.sync();
      }
      // P3: q = S p per slot, p.q partials
      {
      double v[1] = {0.0};
      if (SL > 0 && cm.nranks == 1) {
        // fused, one rank: one warp per slot sums the slot groups (lanes
        // stride the groups with independent loads, then a butterfly), lane 0
        // finishes the slot. A thread per slot waited on ngrp loads in turn.
        const int lane = threadIdx.x & 31;
        for (int s = gid >> 5; s < S; s += stride >> 5) {
          double a = 0.0;
#pragma unroll 4
          for (int g = lane; g < ngrp; g += 32) a += fz.gpart[(long long)g * S + s];
          a = warp_sum(a);
          if (lane == 0) {
            const int c = s >> 3, k = s & 7;
            const double pk = p[s];
            double bp = 0.0;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
              const double pm = (shared && m == 7) ? pf : p[8ll * c + m];
              bp += d.Bc[64ll * c + 8 * k + m] * pm;
            }
            if (shared && k == 7) {
              d.fterm[c] = bp + lam * d.Bc[64ll * c + 63] * pf - a;
              if (c) q[s] = 0.0;
            } else {
              double qk = bp + lam * d.Bc[64ll * c + 9 * k] * pk - a;
              if ((d.pinned[c] >> k) & 1) qk = pk;
              q[s] = qk;
              v[0] += pk * qk;
            }
          }
        }
      } else {
        for (int base = 0; base < S; base += stride) {
          const int s = base + gid;
          if (base + (gid & ~31) >= S) continue;
          const bool ok = s < S;
          const int c = ok ? s >> 3 : 0, k = s & 7;
          const double pk = ok ? p[s] : 0.0;
          // shared focal: the focal slot of every camera reads the one shared
          // unknown, stored in camera 0's slot 7 (the others are pinned zeros)
          const double pkt = (shared && k == 7) ? pf : pk;
          double bp = 0.0;
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            const double pm = grp8_get(pkt, m);
            if (ok) bp += d.Bc[64ll * c + 8 * k + m] * pm;
          }
          if (ok) {
            double acc;
            if (cm.nranks > 1) {
              const long long off = (long long)(ep & 1) * cm.cap + s;
              acc = comm_peer_load(cm.buf[0] + off);
              for (int rk = 1; rk < cm.nranks; ++rk) acc += comm_peer_load(cm.buf[rk] + off);
            } else {
              acc = local_cam(s);
            }
            if (shared && k == 7) {
              // camera c's share of the shared-focal row; summed below
              d.fterm[c] = bp + lam * d.Bc[64ll * c + 63] * pf - acc;
              if (c) q[s] = 0.0;
            } else {
              double qk = bp + lam * d.Bc[64ll * c + 9 * k] * pk - acc;
              if ((d.pinned[c] >> k) & 1) qk = pk;
              q[s] = qk;
              v[0] += pk * qk;
            }
          }
        }
      }
      block_reduce<1>(v, smred);
      if (threadIdx.x == 0) part[2ll * NP + blockIdx.x] = v[0];
      }
      grid.sync();
      if (tim) { const unsigned long long t1 = gtimer(); ph[2] += t1 - pt0; pt0 = t1; }
      double pq = cta_partials_sum(part + 2ll * NP, NP, 1, 0, &smb[0]);
      if (shared) {   // every CTA sums the cameras' shares in the same order
        qf = (d.pinned[0] >> 7 & 1) ? pf : cta_partials_sum(d.fterm, d.bp.C, 1, 0, &smb[2]);
        pq += pf * qf;
      }
      if (!isfinite(pq) || pq <= 0.0) { flag = ST_CG_BREAKDOWN; break; }
      const double alpha = rho / pq;
      // P4: x += a p, r -= a q, z = M r; partials r.r, r.z
      {
        double v[2] = {0.0, 0.0};
        for (int base = 0; base < S; base += stride) {
          const int s = base + gid;
          if (base + (gid & ~31) >= S) continue;
          const bool ok = s < S;
          const int c = ok ? s >> 3 : 0, k = s & 7;
          double rk = 0.0;
          if (ok) {
            x[s] += alpha * p[s];
            rk = r[s] - alpha * ((shared && s == 7) ? qf : q[s]);
            r[s] = rk;
          }
          double zk = 0.0;
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            const double rm = grp8_get(rk, m);
            if (ok) zk += d.Minv[64ll * c + 8 * k + m] * rm;
          }
          if (ok) z[s] = zk;
          v[0] += rk * rk;
          v[1] += rk * zk;
        }
        block_reduce<2>(v, smred);
        if (threadIdx.x == 0) { part[2ll * blockIdx.x] = v[0]; part[2ll * blockIdx.x + 1] = v[1]; }
      }
      grid.sync();
      if (tim) { const unsigned long long t1 = gtimer(); ph[3] += t1 - pt0; pt0 = t1; }
      rr = cta_partials_sum(part, NP, 2, 0, &smb[0]);
      const double rz = cta_partials_sum(part, NP, 2, 1, &smb[1]);
      ++iters;
      rn = sqrt(rr);
      if (rn <= tol) break;
      const double beta = rz / rho;
      rho = rz;
      // P5: p = z + beta p (omega form: one camera per thread, then its W)
      if (d.Gpm) {
        if (shared && gid == 0) p[7] = z[7] + beta * p[7];   // camera 0 slot 7: read by every camera's W
        grid.sync();
        for (int c = gid; c < d.bp.C; c += stride) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (!(shared && c == 0 && k == 7)) p[8ll * c + k] = z[8ll * c + k] + beta * p[8ll * c + k];
          ba_wvec(d, p, c, d.Wc);
        }
      } else {
        for (int s = gid; s < S; s += stride) p[s] = z[s] + beta * p[s];
      }
      grid.sync();
      if (tim) ph[4] += gtimer() - pt0;
      if (shared) pf = p[7];   // every thread tracks the shared focal of p
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (cm.nranks > 1) *cm.epoch = ep;
    for (int k = 0; k < 5; ++k) ctl->phase_ns[k] = ph[k];
    ctl->tol = tol;
    ctl->rho = rho;
    ctl->rn = rn;
    ctl->iters = iters;
    ctl->flag = flag;
    if (flag) atomicOr(d.status, flag);
  }
}

// Diagnostic wrappers: the two passes of the two-pass operator as standalone
// kernels (per-pass timing and roofline, ssfm_bench_operator).
__global__ void __launch_bounds__(PTP_THREADS, PTP_MINB) k_op_point(BADev d, const double* v, double* y) {
  __shared__ double smp[PTP_THREADS / 32][SSFM_BATCH][3];
  if (d.Gpm) { ba_point_pass_w<true>(d, d.Wc, y, smp); return; }   // W of v: k_cam_wvec first
#if PTP_PIPE
  __shared__ PtpStage stg[PTP_THREADS / 32][2];
  ba_point_pass_pipe<true>(d, v, y, stg, smp);
#else
  ba_point_pass<true>(d, v, y, smp);
#endif
}
template <bool FAC>
__global__ void __launch_bounds__(PCG_THREADS, FAC ? CAMF_MINB : 4) k_op_camera(BADev d, const double* y, double* tile8) {
  __shared__ double smred[(PCG_THREADS / 32) * 8];
  if constexpr (FAC) ba_camera_pass_f<true>(d, y, tile8);
  else ba_camera_pass<true>(d, y, tile8, smred);
}

// back-substitution of omega-form handles: the point pass with the W of x
// (k_cam_wvec first) and the delta_j = y0_j - Cinv_j (.) finaliser
__global__ void __launch_bounds__(PTP_THREADS, PTP_MINB) ba_k_backsub_w(BADev d, double* delta) {
  __shared__ double smp[PTP_THREADS / 32][SSFM_BATCH][3];
  ba_point_pass_w<true, true>(d, d.Wc, delta, smp);
}
