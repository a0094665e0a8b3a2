// ba_pcg_graph.cuh -- the block-Jacobi PCG (lm.py:637-672) as a CUDA graph:
// one conditional WHILE node whose body is one CG iteration split into
// kernels, each with the occupancy that suits it (no grid-wide barriers; the
// kernel boundaries order the phases):
//
//   point pass (or fused pass) -> camera pass -> q = S p, p.q partials ->
//   alpha, x, r, z, r.r / r.z partials -> beta, p update -> scalars + loop
//   condition (one block, cudaGraphSetConditional)
//
// The same arithmetic, partial layout and summation order as ba_k_pcg, so
// results are identical to the persistent kernel's (tests compare them
// bitwise). lambda, the tolerance and the iteration cap live in device memory:
// the instantiated graph is reused for every damped solve of the handle.
// Sharded handles add two kernels between the passes and q: k_gx_post (this
// rank's camera sums into its exchange buffer) and k_gx_barrier (signal and
// wait, comm.cuh); k_g_q then sums the ranks in rank order.
#pragma once
#include "ba_pcg.cuh"
#include "comm.cuh"

#define CGV_BLOCKS 148   // vector-phase grid (partials per reduction)

// device scalar state of the graph PCG
struct CGGraphDev {
  double* x; double* r; double* z; double* p; double* q;
  double* partA;   // [2 * CGV_BLOCKS] p.q (and init r.r / r.z)
  double* partB;   // [2 * CGV_BLOCKS] r.r / r.z
  double* sc;      // [8]: 0 lam, 1 cg_tol, 2 tol, 3 rho, 4 rn, 5 rz (pending), 6 qf, 7 shared focal p
  int* ic;         // [8]: 0 max_iters, 1 iters, 2 flag, 3 done, 4 shared focal p pending (sc[7])
  CGCtl* ctl;
  int fused;       // 0 two-pass (tile8), 1 fused (gpart, ngrp groups)
  int ngrp;
};

// sum of n per-block partials component k in fixed order (warp 0), broadcast
__device__ __forceinline__ double g_partials_sum(const double* part, int n, int k, double* smslot) {
  return cta_partials_sum(part, n, 2, k, smslot);
}

// ---- init: x = 0, r = b_red, z = M r, p = z; partials r.r, r.z -> partA
__global__ void __launch_bounds__(256) k_g_init(BADev d, CGGraphDev g) {
  __shared__ double smred[64];
  const int S = 8 * d.bp.C;
  const int stride = gridDim.x * blockDim.x;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  double v[2] = {0.0, 0.0};
  for (int base = 0; base < S; base += stride) {
    const int s = base + gid;
    const bool ok = s < S;
    if (base + (gid & ~31) >= S) continue;
    const int c = ok ? s >> 3 : 0, k = s & 7;
    const double rk = ok ? d.bred[s] : 0.0;
    double zk = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const double rm = grp8_get(rk, m);
      if (ok) zk += d.Minv[64ll * c + 8 * k + m] * rm;
    }
    if (ok) { g.x[s] = 0.0; g.r[s] = rk; g.z[s] = zk; g.p[s] = zk; }
    v[0] += rk * rk;
    v[1] += rk * zk;
  }
  block_reduce<2>(v, smred);
  if (threadIdx.x == 0) { g.partA[2ll * blockIdx.x] = v[0]; g.partA[2ll * blockIdx.x + 1] = v[1]; }
}

// init scalars: rho, tol, done (rn <= tol), iteration cap
template <typename Dev>   // BADev or GPDev: scal
__global__ void k_g_init2(Dev d, CGGraphDev g, int nblk) {
  __shared__ double smb[4];
  const double rr = g_partials_sum(g.partA, nblk, 0, &smb[0]);
  const double rho = g_partials_sum(g.partA, nblk, 1, &smb[1]);
  if (threadIdx.x == 0) {
    const double gn = sqrt(d.scal[SC_GNORM2]);
    const double tol = g.sc[1] * fmax(gn, 1e-300);
    const double rn = sqrt(rr);
    g.sc[2] = tol; g.sc[3] = rho; g.sc[4] = rn;
    g.ic[1] = 0;
    int flag = 0, done = !(rn > tol);
    if (!done && g.ic[0] <= 0) { flag = ST_CG_MAXITER; done = 1; }
    g.ic[2] = flag;
    g.ic[3] = done;
  }
}

// ---- body kernels (each returns at once when the solve is done)
__global__ void __launch_bounds__(PTP_THREADS, PTP_MINB) k_g_point(BADev d, CGGraphDev g) {
  if (*(volatile int*)(g.ic + 3)) return;
  __shared__ double smp[PTP_THREADS / 32][SSFM_BATCH][3];
  if (d.Gpm) { ba_point_pass_w<true>(d, d.Wc, d.yv, smp); return; }   // W (of p) is constant here
#if PTP_PIPE
  __shared__ PtpStage stg[PTP_THREADS / 32][2];
  ba_point_pass_pipe<true>(d, g.p, d.yv, stg, smp);   // p is constant during this kernel
#else
  ba_point_pass<true>(d, g.p, d.yv, smp);   // p is constant during this kernel
#endif
}

// FAC: the factored camera pass (ba_camera_pass_f)
template <bool FAC>
__global__ void __launch_bounds__(PCG_THREADS, FAC ? CAMF_MINB : 4) k_g_camera(BADev d, CGGraphDev g) {
  if (*(volatile int*)(g.ic + 3)) return;
  __shared__ double smred[(PCG_THREADS / 32) * 8];
  if constexpr (FAC) ba_camera_pass_f<true>(d, d.yv, d.tilebuf);   // y is constant during this kernel
  else ba_camera_pass<true>(d, d.yv, d.tilebuf, smred);
}

template <int SL>
__global__ void __launch_bounds__(FZ_THREADS, 1) k_g_fused(BADev d, FusedTopo fz, CGGraphDev g) {
  if (*(volatile int*)(g.ic + 3)) return;
  __shared__ double smp[FZ_WARPS][SSFM_BATCH][3];
  __shared__ double smy[FZ_WARPS][SSFM_BATCH][3];
  __shared__ int smown[FZ_WARPS][SSFM_BATCH];
  extern __shared__ double dyn_acc[];
  ba_fused_pass<SL>(d, fz, g.p, dyn_acc, smp, smy, smown);
}

// q = S p per slot (P3 of ba_k_pcg), p.q partials -> partA, shared-focal shares
__global__ void __launch_bounds__(256) k_g_q(BADev d, FusedTopo fz, CGGraphDev g, CommDev cm) {
  if (*(volatile int*)(g.ic + 3)) return;
  const long long xoff = cm.nranks > 1 ? (long long)(*cm.epoch & 1) * cm.cap : 0;
  __shared__ double smred[64];
  const int S = 8 * d.bp.C;
  const int stride = gridDim.x * blockDim.x;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const double lam = g.sc[0];
  const bool shared = d.bp.focal_mode == 2;
  const double pf = shared ? g.p[7] : 0.0;
  double v[1] = {0.0};
  for (int base = 0; base < S; base += stride) {
    const int s = base + gid;
    if (base + (gid & ~31) >= S) continue;
    const bool ok = s < S;
    const int c = ok ? s >> 3 : 0, k = s & 7;
    const double pk = ok ? g.p[s] : 0.0;
    const double pkt = (shared && k == 7) ? pf : pk;
    double bp = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const double pm = grp8_get(pkt, m);
      if (ok) bp += d.Bc[64ll * c + 8 * k + m] * pm;
    }
    if (ok) {
      double acc = 0.0;
      if (cm.nranks > 1) {            // camera sums exchanged by k_gx_post / k_gx_barrier
        acc = comm_peer_load(cm.buf[0] + xoff + s);
        for (int rk = 1; rk < cm.nranks; ++rk) acc += comm_peer_load(cm.buf[rk] + xoff + s);
      } else if (!g.fused) {
        acc = tiles_sum<8>(d.tilebuf, k, d.topo.cam_tile[c], d.topo.cam_tile[c + 1]);
      } else {
        for (int gq = 0; gq < g.ngrp; ++gq) acc += fz.gpart[(long long)gq * S + s];
      }
      if (shared && k == 7) {
        d.fterm[c] = bp + lam * d.Bc[64ll * c + 63] * pf - acc;
        if (c) g.q[s] = 0.0;
      } else {
        double qk = bp + lam * d.Bc[64ll * c + 9 * k] * pk - acc;
        if ((d.pinned[c] >> k) & 1) qk = pk;
        g.q[s] = qk;
        v[0] += pk * qk;
      }
    }
  }
  block_reduce<1>(v, smred);
  if (threadIdx.x == 0) g.partA[2ll * blockIdx.x] = v[0];
}

// sharded: this rank's camera sums -> own exchange buffer of the next epoch
__global__ void __launch_bounds__(256) k_gx_post(BADev d, FusedTopo fz, CGGraphDev g, CommDev cm) {
  if (*(volatile int*)(g.ic + 3)) return;
  const int S = 8 * d.bp.C;
  double* mine = cm.buf[cm.rank] + (long long)((*cm.epoch + 1) & 1) * cm.cap;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const int c = s >> 3, k = s & 7;
    double a = 0.0;
    if (!g.fused) {
      a = tiles_sum<8>(d.tilebuf, k, d.topo.cam_tile[c], d.topo.cam_tile[c + 1]);
    } else {
      for (int gq = 0; gq < g.ngrp; ++gq) a += fz.gpart[(long long)gq * S + s];
    }
    mine[s] = a;
  }
}

// sharded: signal this epoch and wait for the peers (skipped identically on
// every rank once the solve is done)
__global__ void k_gx_barrier(CGGraphDev g, CommDev cm) {
  if (*(volatile int*)(g.ic + 3)) return;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const unsigned long long e = *cm.epoch + 1;
    comm_signal_wait(cm, e);
    *cm.epoch = e;
  }
}

// alpha = rho / p.q (every block, same order); x += a p, r -= a q, z = M r;
// partials r.r, r.z -> partB
__global__ void __launch_bounds__(256) k_g_update(BADev d, CGGraphDev g, int nblk) {
  if (*(volatile int*)(g.ic + 3)) return;
  __shared__ double smred[64];
  __shared__ double smb[4];
  const int S = 8 * d.bp.C;
  const int stride = gridDim.x * blockDim.x;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const bool shared = d.bp.focal_mode == 2;
  double pq = g_partials_sum(g.partA, nblk, 0, &smb[0]);
  double qf = 0.0;
  if (shared) {
    const double pf = g.p[7];
    qf = (d.pinned[0] >> 7 & 1) ? pf : cta_partials_sum(d.fterm, d.bp.C, 1, 0, &smb[2]);
    pq += pf * qf;
  }
  if (!isfinite(pq) || pq <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) g.ic[2] = ST_CG_BREAKDOWN;
    return;
  }
  const double alpha = g.sc[3] / pq;
  double v[2] = {0.0, 0.0};
  for (int base = 0; base < S; base += stride) {
    const int s = base + gid;
    if (base + (gid & ~31) >= S) continue;
    const bool ok = s < S;
    const int c = ok ? s >> 3 : 0, k = s & 7;
    double rk = 0.0;
    if (ok) {
      g.x[s] += alpha * g.p[s];
      rk = g.r[s] - alpha * ((shared && s == 7) ? qf : g.q[s]);
      g.r[s] = rk;
    }
    double zk = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const double rm = grp8_get(rk, m);
      if (ok) zk += d.Minv[64ll * c + 8 * k + m] * rm;
    }
    if (ok) g.z[s] = zk;
    v[0] += rk * rk;
    v[1] += rk * zk;
  }
  block_reduce<2>(v, smred);
  if (threadIdx.x == 0) { g.partB[2ll * blockIdx.x] = v[0]; g.partB[2ll * blockIdx.x + 1] = v[1]; }
}

// beta = r.z / rho (every block, same order); p = z + beta p
__global__ void __launch_bounds__(256) k_g_pupdate(BADev d, CGGraphDev g, int nblk) {
  if (*(volatile int*)(g.ic + 3) || *(volatile int*)(g.ic + 2)) return;
  __shared__ double smb[4];
  const double rr = g_partials_sum(g.partB, nblk, 0, &smb[0]);
  const double rz = g_partials_sum(g.partB, nblk, 1, &smb[1]);
  if (sqrt(rr) <= g.sc[2]) return;   // converged: the loop ends, p is not used again
  const double beta = rz / g.sc[3];
  const int S = 8 * d.bp.C;
  if (d.Gpm) {
    // omega form: one camera per thread, p then its W. Shared focal: every
    // camera's W reads camera 0's slot 7, so each thread computes it itself.
    const bool shared = d.bp.focal_mode == 2;
    const double pf = shared ? g.z[7] + beta * g.p[7] : 0.0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d.bp.C; c += gridDim.x * blockDim.x) {
      double pc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pc[k] = g.z[8ll * c + k] + beta * g.p[8ll * c + k];
      if (shared && c == 0) {   // slot 7 of camera 0 is read by every thread: k_g_scalars writes it
        pc[7] = g.p[7];
        g.sc[7] = pf;
        g.ic[4] = 1;
      }
      double* w = d.Wc + 8ll * c;
      // ba_wvec on registers: W of this camera from pc (and the shared focal)
      const double* cb = reinterpret_cast<const double*>(d.camlin + c);
      const double qw = cb[9], qx = cb[10], qy = cb[11], qz = cb[12], s2 = 2.0 * cb[22];
      const double o0 = s2 * (qw * pc[1] - pc[0] * qx - (qy * pc[3] - qz * pc[2]));
      const double o1 = s2 * (qw * pc[2] - pc[0] * qy - (qz * pc[1] - qx * pc[3]));
      const double o2 = s2 * (qw * pc[3] - pc[0] * qz - (qx * pc[2] - qy * pc[1]));
      const double t0 = cb[14], t1 = cb[15], t2 = cb[16];
      w[0] = o0; w[1] = o1; w[2] = o2;
      w[3] = (o1 * t2 - o2 * t1) + pc[4];
      w[4] = (o2 * t0 - o0 * t2) + pc[5];
      w[5] = (o0 * t1 - o1 * t0) + pc[6];
      w[6] = shared ? pf : (d.bp.focal_mode == 1 ? pc[7] : 0.0);
      w[7] = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) g.p[8ll * c + k] = pc[k];
    }
    return;
  }
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x)
    g.p[s] = g.z[s] + beta * g.p[s];
}

// ---------------------------------------------------------------------------
// The vector phases of one CG iteration (q = S p and p.q, alpha, x / r / z
// and r.r / r.z, beta, p (+ its omega-form W), the scalars and the loop
// condition) as ONE kernel: a thread-block cluster of GV_CL CTAs, each owning
// a contiguous range of cameras. The only cross-CTA dependencies are the
// three scalar reductions; they go through distributed shared memory (each
// CTA's partial in its own shared memory, every CTA sums the GV_CL partials in
// rank order after a cluster barrier), so every CTA takes identical
// decisions. Replaces k_g_q, k_g_update, k_g_pupdate and k_g_scalars (four
// launches and their grid-wide gaps per CG iteration).
// ---------------------------------------------------------------------------
#ifndef GV_CL
#define GV_CL 8
#endif
// 16 (a non-portable cluster) was measured at the end of round 2: BA -1 % at C5,
// but the GP vector phase then ends its CG loops at once (wrong steps)
static_assert(GV_CL >= 1 && GV_CL <= 8, "GV_CL > 8 breaks the GP vector phase (k_gg_vec)");
#define GV_THREADS 1024

template <int NV>
__device__ __forceinline__ void gv_cluster_sum(cg::cluster_group& cl, double (&v)[NV], double* smred, double* slot) {
  block_reduce<NV>(v, smred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) slot[k] = v[k];
  }
  cl.sync();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (int r = 0; r < GV_CL; ++r) {
    const double* rs = cl.map_shared_rank(slot, r);
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += rs[k];
  }
}

__global__ void __cluster_dims__(GV_CL, 1, 1) __launch_bounds__(GV_THREADS, 1)
k_g_vec(BADev d, FusedTopo fz, CGGraphDev g, CommDev cm, cudaGraphConditionalHandle hc) {
  if (*(volatile int*)(g.ic + 3)) {   // solved before this iteration (uniform over the cluster):
    if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(hc, 0u);   // end the WHILE loop
    return;
  }
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double smred[(GV_THREADS / 32) * 2];
  __shared__ double slot_pq[2], slot_rr[2];
  const int rank = (int)cl.block_rank();
  const int C = d.bp.C;
  const int c0 = (int)((long long)C * rank / GV_CL), c1 = (int)((long long)C * (rank + 1) / GV_CL);
  const int s0 = 8 * c0, s1 = 8 * c1;
  const long long xoff = cm.nranks > 1 ? (long long)(*cm.epoch & 1) * cm.cap : 0;
  const double lam = g.sc[0];
  const bool shared = d.bp.focal_mode == 2;
  const double pf = shared ? g.p[7] : 0.0;
  // ---- q = S p (slot-major: 8 consecutive lanes hold one camera), p.q
  double v1[2] = {0.0, 0.0};
  for (int base = s0; base < s1; base += GV_THREADS) {
    const int s = base + threadIdx.x;
    if (base + (int)(threadIdx.x & ~31u) >= s1) continue;
    const bool ok = s < s1;
    const int c = ok ? s >> 3 : c0, k = s & 7;
    const double pk = ok ? g.p[s] : 0.0;
    const double pkt = (shared && k == 7) ? pf : pk;
    double bp = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const double pm = grp8_get(pkt, m);
      if (ok) bp += d.Bc[64ll * c + 8 * k + m] * pm;
    }
    if (ok) {
      double acc = 0.0;
      if (cm.nranks > 1) {
        acc = comm_peer_load(cm.buf[0] + xoff + s);
        for (int rk = 1; rk < cm.nranks; ++rk) acc += comm_peer_load(cm.buf[rk] + xoff + s);
      } else if (!g.fused) {
        acc = tiles_sum<8>(d.tilebuf, k, d.topo.cam_tile[c], d.topo.cam_tile[c + 1]);
      } else {
        for (int gq = 0; gq < g.ngrp; ++gq) acc += fz.gpart[(long long)gq * (8 * C) + s];
      }
      if (shared && k == 7) {
        const double ft = bp + lam * d.Bc[64ll * c + 63] * pf - acc;
        v1[1] += ft;             // the shared focal row: the cameras' shares
        if (c) g.q[s] = 0.0;
      } else {
        double qk = bp + lam * d.Bc[64ll * c + 9 * k] * pk - acc;
        if ((d.pinned[c] >> k) & 1) qk = pk;
        g.q[s] = qk;
        v1[0] += pk * qk;
      }
    }
  }
  gv_cluster_sum<2>(cl, v1, smred, slot_pq);
  double pq = v1[0], qf = 0.0;
  if (shared) {
    qf = (d.pinned[0] >> 7 & 1) ? pf : v1[1];
    pq += pf * qf;
  }
  if (!isfinite(pq) || pq <= 0.0) {
    if (rank == 0 && threadIdx.x == 0) {
      g.ic[2] = ST_CG_BREAKDOWN;
      g.ic[3] = 1;
      CGCtl* ctl = g.ctl;
      ctl->tol = g.sc[2]; ctl->rho = g.sc[3]; ctl->rn = g.sc[4];
      ctl->iters = g.ic[1]; ctl->flag = ST_CG_BREAKDOWN;
      atomicOr(d.status, ST_CG_BREAKDOWN);
      cudaGraphSetConditional(hc, 0u);
    }
    cl.sync();   // no CTA may exit while its shared slots are read
    return;
  }
  const double alpha = g.sc[3] / pq;
  // ---- x += a p, r -= a q, z = M r; r.r, r.z
  double v2[2] = {0.0, 0.0};
  for (int base = s0; base < s1; base += GV_THREADS) {
    const int s = base + threadIdx.x;
    if (base + (int)(threadIdx.x & ~31u) >= s1) continue;
    const bool ok = s < s1;
    const int c = ok ? s >> 3 : c0, k = s & 7;
    double rk = 0.0;
    if (ok) {
      g.x[s] += alpha * g.p[s];
      rk = g.r[s] - alpha * ((shared && s == 7) ? qf : g.q[s]);
      g.r[s] = rk;
    }
    double zk = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const double rm = grp8_get(rk, m);
      if (ok) zk += d.Minv[64ll * c + 8 * k + m] * rm;
    }
    if (ok) g.z[s] = zk;
    v2[0] += rk * rk;
    v2[1] += rk * zk;
  }
  gv_cluster_sum<2>(cl, v2, smred, slot_rr);
  const double rr = v2[0], rz = v2[1];
  const int iters = g.ic[1] + 1;
  const double rn = sqrt(rr);
  int flag = 0, done = 0;
  if (rn <= g.sc[2]) done = 1;
  else if (iters >= g.ic[0]) { flag = ST_CG_MAXITER; done = 1; }
  if (!done) {
    // ---- p = z + beta p (+ W of p for the omega-form point pass)
    const double beta = rz / g.sc[3];
    const double pf_new = shared ? g.z[7] + beta * pf : 0.0;   // pf: p[7] read at entry
    for (int base = s0; base < s1; base += GV_THREADS) {
      const int s = base + threadIdx.x;
      if (base + (int)(threadIdx.x & ~31u) >= s1) continue;
      const bool ok = s < s1;
      const int c = ok ? s >> 3 : c0, k = s & 7;
      double pk = ok ? g.z[s] + beta * g.p[s] : 0.0;
      if (ok) g.p[s] = pk;
      if (d.Gpm) {
        const double pc0 = grp8_get(pk, 0), pc1 = grp8_get(pk, 1), pc2 = grp8_get(pk, 2), pc3 = grp8_get(pk, 3);
        const double pc4 = grp8_get(pk, 4), pc5 = grp8_get(pk, 5), pc6 = grp8_get(pk, 6), pc7 = grp8_get(pk, 7);
        if (ok && k == 0) {
          const double* cb = reinterpret_cast<const double*>(d.camlin + c);
          const double qw = cb[9], qx = cb[10], qy = cb[11], qz = cb[12], s2 = 2.0 * cb[22];
          const double o0 = s2 * (qw * pc1 - pc0 * qx - (qy * pc3 - qz * pc2));
          const double o1 = s2 * (qw * pc2 - pc0 * qy - (qz * pc1 - qx * pc3));
          const double o2 = s2 * (qw * pc3 - pc0 * qz - (qx * pc2 - qy * pc1));
          const double t0 = cb[14], t1 = cb[15], t2 = cb[16];
          double* w = d.Wc + 8ll * c;
          w[0] = o0; w[1] = o1; w[2] = o2;
          w[3] = (o1 * t2 - o2 * t1) + pc4;
          w[4] = (o2 * t0 - o0 * t2) + pc5;
          w[5] = (o0 * t1 - o1 * t0) + pc6;
          w[6] = shared ? pf_new : (d.bp.focal_mode == 1 ? pc7 : 0.0);
          w[7] = 0.0;
        }
      }
    }
  }
  if (rank == 0 && threadIdx.x == 0) {
    g.ic[1] = iters;
    g.sc[4] = rn;
    if (!done) g.sc[3] = rz;   // rho of the next iteration
    g.ic[2] = flag;
    g.ic[3] = done;
    if (done) {
      CGCtl* ctl = g.ctl;
      ctl->tol = g.sc[2]; ctl->rho = g.sc[3]; ctl->rn = rn;
      ctl->iters = iters; ctl->flag = flag;
      if (flag) atomicOr(d.status, flag);
    }
    cudaGraphSetConditional(hc, done ? 0u : 1u);
  }
  cl.sync();   // the shared slots stay valid until every CTA has read them
}

// scalars of the iteration and the loop condition (one block)
template <typename Dev>   // BADev or GPDev: status
__global__ void k_g_scalars(Dev d, CGGraphDev g, int nblk, cudaGraphConditionalHandle hc) {
  __shared__ double smb[4];
  int done = *(volatile int*)(g.ic + 3);
  if (threadIdx.x == 0 && g.ic[4]) {   // omega form, shared focal: p's shared slot (k_g_pupdate)
    g.p[7] = g.sc[7];
    g.ic[4] = 0;
  }
  if (!done) {
    int flag = g.ic[2];
    if (!flag) {
      const double rr = g_partials_sum(g.partB, nblk, 0, &smb[0]);
      const double rz = g_partials_sum(g.partB, nblk, 1, &smb[1]);
      if (threadIdx.x == 0) {
        const int iters = g.ic[1] + 1;
        const double rn = sqrt(rr);
        g.ic[1] = iters;
        g.sc[4] = rn;
        if (rn <= g.sc[2]) done = 1;
        else if (iters >= g.ic[0]) { flag = ST_CG_MAXITER; done = 1; }
        else g.sc[3] = rz;   // rho of the next iteration
        g.ic[2] = flag;
        g.ic[3] = done;
      }
    } else if (threadIdx.x == 0) {
      g.ic[3] = done = 1;
    }
  }
  if (threadIdx.x == 0) {
    if (g.ic[3]) {
      CGCtl* ctl = g.ctl;
      ctl->tol = g.sc[2]; ctl->rho = g.sc[3]; ctl->rn = g.sc[4];
      ctl->iters = g.ic[1]; ctl->flag = g.ic[2];
      if (g.ic[2]) atomicOr(d.status, g.ic[2]);
    }
    cudaGraphSetConditional(hc, g.ic[3] ? 0u : 1u);
  }
}
