// fused.cuh -- schedule for the single-pass (fused) Schur operator.
//
// The two-pass operator (ba_pcg.cuh P1/P2) reads the compact Jacobian twice
// per CG iteration: point-major for y_j = Cinv_j sum Jp^T Jc p, camera-major
// for sum Jc^T Jp y_j. The camera term of an observation only needs its own
// point's y_j, so one point-major pass can produce both while J is still in
// registers. The camera side is then accumulated into a per-CTA shared-memory
// copy of the camera vector, deterministically:
//
//   step       = 16 consecutive point batches (one per warp of a 512-thread CTA)
//   CTA-round  = round r of every warp's batch in the step (a batch with a
//                point of > 32 observations has several rounds)
//   rank       = number of earlier observations (warp-major, lane-minor) of
//                the same camera in the same CTA-round
//
// In the accumulation, ranks are applied in order with a __syncthreads()
// between them, so each camera slot receives at most one add per rank and the
// order of adds is fixed by the static step -> CTA schedule (no floating-point
// atomics, bit-stable results). The rank is packed into the camera id word
// (pm_camr = cam | rank << FZ_RSHIFT), so the schedule costs no extra bytes per
// observation inside the CG loop.
//
// When 8C fp64 does not fit one CTA's shared memory, the 8 camera slots are
// split into G groups (G = 2, 4, 8); the G CTAs of a group-set process the
// same steps (their J reads hit L2 for all but the first) and each owns 8/G
// slots of every camera.
#pragma once
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include "topo.cuh"

#define FZ_WARPS 16
#define FZ_THREADS (FZ_WARPS * 32)
#define FZ_RSHIFT 22
#define FZ_CMASK ((1 << FZ_RSHIFT) - 1)
#define FZ_MAX_CAMERAS (1 << FZ_RSHIFT)

struct FusedTopo {
  int nsteps = 0;
  int G = 0;               // slot groups (0 = fused operator disabled)
  int SL = 0;              // slots per group = 8 / G (BA) or 4 / G (GP)
  int ngrp = 0;            // number of CTA groups in the PCG grid (gridDim / G)
  int* camr = nullptr;     // [N] point-major: cam | rank << FZ_RSHIFT
  int* step_info = nullptr;// [nsteps]: rounds | (maxrank + 1) << 16
  double* gpart = nullptr; // [ngrp * slots_per_cam * C] per-group camera partials
};

// One CTA (FZ_THREADS) per step: ranks of every observation within its CTA-round.
__global__ void __launch_bounds__(FZ_THREADS) k_fz_ranks(Topo T, int* camr, int* step_info, int nsteps) {
  typedef cub::BlockRadixSort<int, FZ_THREADS, 1, int> Sort;
  typedef cub::BlockScan<int, FZ_THREADS> Scan;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ int s_rank[FZ_THREADS];
  __shared__ int s_max;
  __shared__ int s_rounds;
  const int s = blockIdx.x;
  if (s >= nsteps) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = s * FZ_WARPS + warp;
  int ob0 = 0, ob1 = 0;
  if (b < T.nb) { ob0 = T.bat_obs[b]; ob1 = T.bat_obs[b + 1]; }
  const int my_rounds = (ob1 - ob0 + 31) / 32;
  if (threadIdx.x == 0) { s_max = 0; s_rounds = 0; }
  __syncthreads();
  if (lane == 0) atomicMax(&s_rounds, my_rounds);
  __syncthreads();
  const int R = s_rounds;
  int maxrank = 0;
  for (int r = 0; r < R; ++r) {
    const int i = ob0 + 32 * r + lane;
    const bool have = r < my_rounds && i < ob1;
    // key: camera (valid) or a sentinel above every camera id; value: thread
    int key[1] = {have ? T.pm_cam[i] : FZ_MAX_CAMERAS};
    int val[1] = {(int)threadIdx.x};
    __syncthreads();
    Sort(tmp.sort).Sort(key, val, 0, FZ_RSHIFT + 1);
    __syncthreads();
    // sorted position k = threadIdx.x holds (key[0], val[0]); run start by max-scan of heads
    s_rank[threadIdx.x] = key[0];
    __syncthreads();
    const int k = threadIdx.x;
    const bool head = (k == 0) || (s_rank[k - 1] != key[0]);
    int start = head ? k : 0;
    int run_start[1] = {start};
    __syncthreads();
    Scan(tmp.scan).InclusiveScan(run_start, run_start, cub::Max());
    const int rank = k - run_start[0];
    __syncthreads();
    s_rank[val[0]] = rank;   // stable sort: equal cameras keep thread order
    __syncthreads();
    if (have) {
      const int rk = s_rank[threadIdx.x];
      camr[i] = T.pm_cam[i] | (rk << FZ_RSHIFT);
      maxrank = max(maxrank, rk);
    }
  }
  atomicMax(&s_max, maxrank);
  __syncthreads();
  if (threadIdx.x == 0) step_info[s] = R | ((s_max + 1) << 16);
}
