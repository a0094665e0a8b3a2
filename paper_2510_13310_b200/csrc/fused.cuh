// fused.cuh -- schedule for the single-pass (fused) Schur operator.
//
// The two-pass operator (ba_pcg.cuh P1/P2) reads the compact Jacobian twice
// per CG iteration: point-major for y_j = Cinv_j sum Jp^T Jc p, camera-major
// for sum Jc^T Jp y_j. The camera term of an observation only needs its own
// point's y_j, so one point-major pass can produce both while J is still in
// registers. The camera side is accumulated into a per-CTA shared-memory copy
// of the camera vector, deterministically and without CTA-wide barriers:
//
//   step   = 16 consecutive point batches; CTA group grp processes steps
//            grp, grp + ngrp, ... and warp w of the CTA takes batch 16 s + w
//   unit   = one 32-observation round of a batch (a batch holding a point with
//            > 32 observations has several rounds); units of one CTA are
//            totally ordered by their first point-major observation index,
//            which is consistent with every warp's program order
//   ticket = for each (CTA group, camera), the rank of the unit among the
//            group's units that observe that camera
//
// Inside a unit the lanes that share a camera are summed in lane order by
// the lowest such lane (__match_any_sync); that lane then waits until the
// camera's shared-memory counter equals its ticket, adds, and bumps the
// counter. Every camera slot therefore receives its adds in one fixed order
// (bit-stable results, no floating-point atomics), while warps otherwise run
// independently (a unit only waits on units that precede it in the total
// order, so the wait graph is acyclic). Waits are bounded: a schedule error
// sets ST_SCHEDULE instead of hanging.
//
// When 8C fp64 does not fit one CTA's shared memory, the 8 camera slots are
// split into G groups (G = 2, 4, 8); the G CTAs of a group-set process the
// same steps (their J reads hit L2 for all but the first) and each owns 8/G
// slots of every camera.
#pragma once
#include "topo.cuh"

#define FZ_WARPS 16
#define FZ_THREADS (FZ_WARPS * 32)
#define FZ_MAX_CAMERAS (1 << 24)
#define FZ_SPIN_LIMIT (1 << 26)

struct FusedTopo {
  int nsteps = 0;
  int G = 0;                      // slot groups (0 = fused operator disabled)
  int SL = 0;                     // slots per group = 8 / G (BA) or 4 / G (GP)
  int ngrp = 0;                   // number of CTA groups in the PCG grid (gridDim / G)
  unsigned short* tick = nullptr; // [N] point-major: ticket of the observation's unit
  double* gpart = nullptr;        // [ngrp * slots_per_cam * C] per-group camera partials
};

#define FZ_MAX_TICKET 65535

// Ticket counters live in shared memory; acquire/release at CTA scope on the
// shared window (generic atomics would go through the generic LSU path). As
// atomics (an OR with 0 to read, an exchange to write) so that racecheck sees
// the flag protocol as synchronisation, not as racing plain accesses.
__device__ __forceinline__ int ld_acquire_smem(const int* p) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  int v;
  asm volatile("atom.acquire.cta.shared::cta.or.b32 %0, [%1], 0;" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_smem(int* p, int v) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("{ .reg .b32 old; atom.release.cta.shared::cta.exch.b32 old, [%0], %1; }" ::"r"(a), "r"(v) : "memory");
}

// Camera accumulator layout: SL doubles per camera, its 16-byte chunks XOR-
// swizzled by the camera id so that lanes updating random cameras spread over
// all 32 banks (an unswizzled 64-byte record maps every camera onto 2 bank
// groups: 16-way conflicts).
template <int SL>
__device__ __forceinline__ int fz_slot(int c, int j) {
  if constexpr (SL >= 4) {
    constexpr int M = SL / 2 - 1;
    return c * SL + ((((j >> 1) ^ (c & M))) << 1) + (j & 1);
  } else {
    return c * SL + j;
  }
}

template <int SL>
__device__ __forceinline__ void fz_add(double* acc, int c, const double* u) {
  if constexpr (SL >= 2) {
    constexpr int M = SL / 2 - 1;
    double2* a2 = reinterpret_cast<double2*>(acc + (long long)c * SL);
#pragma unroll
    for (int q = 0; q < SL / 2; ++q) {   // logical chunk q lives at physical chunk q ^ (c & M)
      const int pq = q ^ (c & M);
      double2 cur = a2[pq];
      cur.x += u[2 * q];
      cur.y += u[2 * q + 1];
      a2[pq] = cur;
    }
  } else {
    acc[c] += u[0];
  }
}

// per observation: sort key (CTA group, camera) and unit id (first observation
// index of its 32-round). One warp per batch.
__global__ void k_fz_keys(Topo T, int ngrp, unsigned long long* key, int* unit, int* idx) {
  const int lane = threadIdx.x & 31;
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= T.nb) return;
  const int ob0 = T.bat_obs[b], ob1 = T.bat_obs[b + 1];
  const int grp = (b / FZ_WARPS) % ngrp;
  for (int i = ob0 + lane; i < ob1; i += 32) {
    key[i] = (unsigned long long)grp * (unsigned long long)T.C + (unsigned long long)T.pm_cam[i];
    unit[i] = ob0 + ((i - ob0) & ~31);
    idx[i] = i;
  }
}

// one thread per sorted run head: walk the run, count distinct units
__global__ void k_fz_tickets(const unsigned long long* __restrict__ skey, const int* __restrict__ sidx,
                             const int* __restrict__ unit, long long n, unsigned short* tick, int* status) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  if (k > 0 && skey[k - 1] == skey[k]) return;
  int t = 0;
  int prev = unit[sidx[k]];
  for (long long m = k; m < n && skey[m] == skey[k]; ++m) {
    const int i = sidx[m];
    const int u = unit[i];
    if (u != prev) { ++t; prev = u; }
    if (t > FZ_MAX_TICKET) { atomicOr(status, ST_SCHEDULE); return; }
    tick[i] = (unsigned short)t;
  }
}

