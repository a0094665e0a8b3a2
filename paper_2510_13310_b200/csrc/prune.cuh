// prune.cuh -- ba.prune (ba.py:223-261) on the device: drop points seen by
// fewer than two cameras and cameras left without observations, repeating to
// a fixed point, then the old -> new index maps and the observation mask.
// Integer work only (counts by integer atomics, maps by exclusive scans), so
// the result is bit-identical to the reference's.
#pragma once
#include "common.cuh"

// per alive observation: +1 to its point's and camera's view counts
__global__ void k_prune_count(const int* __restrict__ cam, const int* __restrict__ pt, long long n,
                              const unsigned char* __restrict__ cam_ok, const unsigned char* __restrict__ pt_ok,
                              int* cnt_cam, int* cnt_pt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = cam[i], j = pt[i];
    if (cam_ok[c] && pt_ok[j]) {
      atomicAdd(cnt_pt + j, 1);
      atomicAdd(cnt_cam + c, 1);
    }
  }
}

// drop_pt = alive & views < 2, drop_cam = alive & views == 0 (ba.py:237-240);
// *changed |= any drop; the counts are reset for the next round
__global__ void k_prune_drop(int* cnt, unsigned char* ok, int n, int min_views, int* changed) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  if (ok[k] && cnt[k] < min_views) {
    ok[k] = 0;
    *changed = 1;
  }
  cnt[k] = 0;
}

__global__ void k_prune_flags(const unsigned char* __restrict__ ok, int n, int* flag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) flag[k] = ok[k];
}

// old -> new index (-1 when removed) from the exclusive scan of the flags
__global__ void k_prune_map(const unsigned char* __restrict__ ok, const int* __restrict__ scan, int n, int* map) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) map[k] = ok[k] ? scan[k] : -1;
}

__global__ void k_prune_obs(const int* __restrict__ cam, const int* __restrict__ pt, long long n,
                            const unsigned char* __restrict__ cam_ok, const unsigned char* __restrict__ pt_ok,
                            unsigned char* mask, unsigned long long* alive) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned char m = cam_ok[cam[i]] && pt_ok[pt[i]];
    mask[i] = m;
    if (m) atomicAdd(alive, 1ull);
  }
}
