// gp_pcg_graph.cuh -- the GP damped solve's PCG as a CUDA graph (the BA
// version is ba_pcg_graph.cuh): one conditional WHILE node whose body runs the
// two passes of the GP Schur operator (gp_point_pass / gp_camera_pass), q,
// the x / r / z update and the p update as separate kernels, each at its own
// occupancy with no grid barrier. Same recurrences, fixed-order sums and stop
// rule as gp_k_pcg (gp_kernels.cuh); lambda, the tolerance and the cap come
// from device memory (k_g_setparams), so one instantiated graph serves every
// damped solve of the handle. Single-rank handles only (sharded GP handles
// keep the persistent kernel with its in-kernel exchange).
#pragma once
#include "ba_pcg_graph.cuh"
#include "gp_kernels.cuh"

// x = 0, r = b_red, z = M r (pinned: z = r), p = z; partials r.r, r.z -> partA
__global__ void __launch_bounds__(256) k_gg_init(GPDev d, CGGraphDev g) {
  __shared__ double smred[64];
  const int S = 4 * d.gp.C;
  const int stride = gridDim.x * blockDim.x;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  double v[2] = {0.0, 0.0};
  for (int base = 0; base < S; base += stride) {
    const int s = base + gid;
    if (base + (gid & ~31) >= S) continue;
    const bool ok = s < S;
    const int c = ok ? s >> 2 : 0, k = s & 3;
    const double rk = ok ? d.bred[s] : 0.0;
    double zk = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double rm = grp4_get(rk, m);
      if (ok) zk += d.Minv[16ll * c + 4 * k + m] * rm;
    }
    if (ok && ((d.pinned[c] >> k) & 1)) zk = rk;
    if (ok) { g.x[s] = 0.0; g.r[s] = rk; g.z[s] = zk; g.p[s] = zk; }
    v[0] += rk * rk;
    v[1] += rk * zk;
  }
  block_reduce<2>(v, smred);
  if (threadIdx.x == 0) { g.partA[2ll * blockIdx.x] = v[0]; g.partA[2ll * blockIdx.x + 1] = v[1]; }
}

__global__ void __launch_bounds__(PCG_THREADS, 4) k_gg_point(GPDev d, CGGraphDev g) {
  if (*(volatile int*)(g.ic + 3)) return;
  __shared__ double smp[PCG_THREADS / 32][SSFM_BATCH][3];
  d.lam = g.sc[0];
  gp_point_pass(d, g.p, d.yv, smp);
}

__global__ void __launch_bounds__(PCG_THREADS, 4) k_gg_camera(GPDev d, CGGraphDev g) {
  if (*(volatile int*)(g.ic + 3)) return;
  __shared__ double smred[(PCG_THREADS / 32) * 8];
  d.lam = g.sc[0];
  gp_camera_pass(d, d.yv, d.tilebuf, smred);
}

// q = S p per slot (gp_k_pcg's q phase), p.q partials -> partA
__global__ void __launch_bounds__(256) k_gg_q(GPDev d, CGGraphDev g) {
  if (*(volatile int*)(g.ic + 3)) return;
  __shared__ double smred[64];
  const int S = 4 * d.gp.C;
  const int stride = gridDim.x * blockDim.x;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  for (int base = 0; base < S; base += stride) {
    const int s = base + gid;
    if (base + (gid & ~31) >= S) continue;
    const bool ok = s < S;
    const int c = ok ? s >> 2 : 0, k = s & 3;
    const double pk = ok ? g.p[s] : 0.0;
    const double p0 = grp4_get(pk, 0), p1 = grp4_get(pk, 1), p2 = grp4_get(pk, 2);
    if (ok) {
      double qk = 0.0;
      if (k < 3) {
        const double* B = d.Bp + 6ll * c;
        const double row[3][3] = {{B[0], B[1], B[2]}, {B[1], B[3], B[4]}, {B[2], B[4], B[5]}};
        double acc = 0.0;
        acc = tiles_sum<4>(d.tilebuf, k, d.topo.cam_tile[c], d.topo.cam_tile[c + 1]);
        qk = row[k][0] * p0 + row[k][1] * p1 + row[k][2] * p2 - acc;
      }
      if ((d.pinned[c] >> k) & 1) qk = pk;
      g.q[s] = qk;
      v[0] += pk * qk;
    }
  }
  block_reduce<1>(v, smred);
  if (threadIdx.x == 0) g.partA[2ll * blockIdx.x] = v[0];
}

// alpha = rho / p.q; x += a p, r -= a q, z = M r; partials r.r, r.z -> partB
__global__ void __launch_bounds__(256) k_gg_update(GPDev d, CGGraphDev g, int nblk) {
  if (*(volatile int*)(g.ic + 3)) return;
  __shared__ double smred[64];
  __shared__ double smb[4];
  const int S = 4 * d.gp.C;
  const int stride = gridDim.x * blockDim.x;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const double pq = g_partials_sum(g.partA, nblk, 0, &smb[0]);
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
    const int c = ok ? s >> 2 : 0, k = s & 3;
    double rk = 0.0;
    if (ok) { g.x[s] += alpha * g.p[s]; rk = g.r[s] - alpha * g.q[s]; g.r[s] = rk; }
    double zk = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double rm = grp4_get(rk, m);
      if (ok) zk += d.Minv[16ll * c + 4 * k + m] * rm;
    }
    if (ok) g.z[s] = zk;
    v[0] += rk * rk;
    v[1] += rk * zk;
  }
  block_reduce<2>(v, smred);
  if (threadIdx.x == 0) { g.partB[2ll * blockIdx.x] = v[0]; g.partB[2ll * blockIdx.x + 1] = v[1]; }
}

// beta = r.z / rho; p = z + beta p
__global__ void __launch_bounds__(256) k_gg_pupdate(GPDev d, CGGraphDev g, int nblk) {
  if (*(volatile int*)(g.ic + 3) || *(volatile int*)(g.ic + 2)) return;
  __shared__ double smb[4];
  const double rr = g_partials_sum(g.partB, nblk, 0, &smb[0]);
  const double rz = g_partials_sum(g.partB, nblk, 1, &smb[1]);
  if (sqrt(rr) <= g.sc[2]) return;
  const double beta = rz / g.sc[3];
  const int S = 4 * d.gp.C;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x)
    g.p[s] = g.z[s] + beta * g.p[s];
}

// The GP vector phases as one thread-block cluster kernel (k_g_vec for GP):
// q = S p and p.q, alpha, x / r / z and r.r / r.z, beta, p, the scalars and
// the loop condition; the three scalar reductions through distributed shared
// memory. Replaces k_gg_q, k_gg_update, k_gg_pupdate and k_g_scalars.
__global__ void __cluster_dims__(GV_CL, 1, 1) __launch_bounds__(GV_THREADS, 1)
k_gg_vec(GPDev d, CGGraphDev g, cudaGraphConditionalHandle hc) {
  if (*(volatile int*)(g.ic + 3)) {   // solved before this iteration (uniform over the cluster):
    if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(hc, 0u);   // end the WHILE loop
    return;
  }
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double smred[(GV_THREADS / 32) * 2];
  __shared__ double slot_pq[2], slot_rr[2];
  const int rank = (int)cl.block_rank();
  const int C = d.gp.C;
  const int c0 = (int)((long long)C * rank / GV_CL), c1 = (int)((long long)C * (rank + 1) / GV_CL);
  const int s0 = 4 * c0, s1 = 4 * c1;
  double v1[2] = {0.0, 0.0};
  for (int base = s0; base < s1; base += GV_THREADS) {
    const int s = base + threadIdx.x;
    if (base + (int)(threadIdx.x & ~31u) >= s1) continue;
    const bool ok = s < s1;
    const int c = ok ? s >> 2 : c0, k = s & 3;
    const double pk = ok ? g.p[s] : 0.0;
    const double p0 = grp4_get(pk, 0), p1 = grp4_get(pk, 1), p2 = grp4_get(pk, 2);
    if (ok) {
      double qk = 0.0;
      if (k < 3) {
        const double* B = d.Bp + 6ll * c;
        const double row[3][3] = {{B[0], B[1], B[2]}, {B[1], B[3], B[4]}, {B[2], B[4], B[5]}};
        double acc = 0.0;
        acc = tiles_sum<4>(d.tilebuf, k, d.topo.cam_tile[c], d.topo.cam_tile[c + 1]);
        qk = row[k][0] * p0 + row[k][1] * p1 + row[k][2] * p2 - acc;
      }
      if ((d.pinned[c] >> k) & 1) qk = pk;
      g.q[s] = qk;
      v1[0] += pk * qk;
    }
  }
  gv_cluster_sum<2>(cl, v1, smred, slot_pq);
  const double pq = v1[0];
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
    cl.sync();
    return;
  }
  const double alpha = g.sc[3] / pq;
  double v2[2] = {0.0, 0.0};
  for (int base = s0; base < s1; base += GV_THREADS) {
    const int s = base + threadIdx.x;
    if (base + (int)(threadIdx.x & ~31u) >= s1) continue;
    const bool ok = s < s1;
    const int c = ok ? s >> 2 : c0, k = s & 3;
    double rk = 0.0;
    if (ok) { g.x[s] += alpha * g.p[s]; rk = g.r[s] - alpha * g.q[s]; g.r[s] = rk; }
    double zk = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double rm = grp4_get(rk, m);
      if (ok) zk += d.Minv[16ll * c + 4 * k + m] * rm;
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
    const double beta = rz / g.sc[3];
    for (int s = s0 + threadIdx.x; s < s1; s += GV_THREADS) g.p[s] = g.z[s] + beta * g.p[s];
  }
  if (rank == 0 && threadIdx.x == 0) {
    g.ic[1] = iters;
    g.sc[4] = rn;
    if (!done) g.sc[3] = rz;
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
  cl.sync();
}
