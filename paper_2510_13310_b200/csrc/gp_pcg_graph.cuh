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
        for (int t = d.topo.cam_tile[c]; t < d.topo.cam_tile[c + 1]; ++t) acc += d.tilebuf[4ll * t + k];
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
