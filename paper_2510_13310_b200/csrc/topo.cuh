// topo.cuh -- one-time device construction of the observation orderings,
// segments and work units shared by the BA and GP problems.
//
// Replaces the reference's per-problem pattern/plan construction
// (JtJPattern sparse_block.py:219-323, JtrPattern :326-363, _SchurPlan
// lm.py:236-483), which sorts contributions on the host, with two stable
// device radix sorts:
//   point-major order  = stable sort of observations by point   (ties keep
//                        observation order: the reference's per-point
//                        contribution order, lm.py:340 lexsort)
//   camera-major order = stable sort by camera
// plus work units:
//   point batches  : runs of whole points with <= 32 observations and <= 32
//                    points (one warp each; a point with > 32 observations is
//                    a batch on its own and is processed in rounds)
//   camera tiles   : <= TILE observations of a single camera (one CTA each)
#pragma once
#include <cub/cub.cuh>
#include "common.cuh"

#define SSFM_TILE 256
#define SSFM_BATCH 32
#define SSFM_CHUNK 128

struct Topo {
  int C = 0, P = 0;
  long long N = 0;
  // point-major
  int* pm_obs = nullptr;    // [N] original observation id
  int* pm_pt = nullptr;     // [N] point id
  int* pm_cam = nullptr;    // [N] camera id
  int* pm_to_cm = nullptr;  // [N] camera-major position
  int* cm_to_pm = nullptr;  // [N] point-major position of a camera-major observation
  int* pt_seg = nullptr;    // [P+1]
  int* bat_obs = nullptr;   // [nb+1]
  int* bat_pt = nullptr;    // [nb+1]
  int nb = 0;
  // camera-major
  int* cm_obs = nullptr;    // [N]
  int* cm_pt = nullptr;     // [N]
  int* cam_seg = nullptr;   // [C+1]
  int* tile_obs = nullptr;  // [nt+1]
  int* tile_cam = nullptr;  // [nt]
  int* cam_tile = nullptr;  // [C+1]
  int nt = 0;
  // tile groups: up to SSFM_GRP consecutive tiles of one camera (one CTA of
  // the per-camera reductions: linearize, preconditioner)
  int* grp_tile = nullptr;  // [ng+1] first tile of each group
  int ng = 0;
};

__global__ void k_check_index(const int* __restrict__ cam, const int* __restrict__ pt,
                              long long n, int C, int P, int* status) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) {
    int c = cam[i], p = pt[i];
    if (c < 0 || c >= C || p < 0 || p >= P) atomicOr(status, ST_BAD_INDEX);
  }
}

__global__ void k_iota(int* out, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int)i;
}

__global__ void k_count(const int* __restrict__ key, long long n, int* counts) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&counts[key[i]], 1);
}

// Segment offsets from sorted keys (no atomics): observation i opens the
// segments of every key in (key[i-1], key[i]]; the last one closes the rest.
__global__ void k_seg_from_sorted(const int* __restrict__ key, long long n, int nkeys, int* seg) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int prev = i == 0 ? -1 : key[i - 1];
  for (int k = prev + 1; k <= key[i]; ++k) seg[k] = (int)i;
  if (i == n - 1)
    for (int k = key[i] + 1; k <= nkeys; ++k) seg[k] = (int)n;
}

// gather helpers for the permuted views
__global__ void k_perm_views(const int* __restrict__ perm_pm, const int* __restrict__ perm_cm,
                             const int* __restrict__ cam, const int* __restrict__ pt, long long n,
                             int* pm_pt, int* pm_cam, int* cm_pt, int* inv_cm) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) {
    int o = perm_pm[i];
    pm_pt[i] = pt[o];
    pm_cam[i] = cam[o];
    int oc = perm_cm[i];
    cm_pt[i] = pt[oc];
    inv_cm[oc] = (int)i;      // camera-major position of observation oc
  }
}

__global__ void k_pm_to_cm(const int* __restrict__ perm_pm, const int* __restrict__ inv_cm,
                           long long n, int* pm_to_cm) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) pm_to_cm[i] = inv_cm[perm_pm[i]];
}

__global__ void k_invert_perm(const int* __restrict__ perm, long long n, int* inv) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) inv[perm[i]] = (int)i;
}

// Greedy packing of consecutive points into warp batches, chunk-parallel.
// pass 0 counts batches per chunk, pass 1 writes their first point/observation.
__global__ void k_batches(const int* __restrict__ pt_seg, int P, int pass,
                          int* chunk_cnt, const int* chunk_off, int* bat_pt, int* bat_obs) {
  int ch = blockIdx.x * blockDim.x + threadIdx.x;
  int p0 = ch * SSFM_CHUNK;
  if (p0 >= P) return;
  int p1 = min(P, p0 + SSFM_CHUNK);
  int nb = 0;
  int out = pass ? chunk_off[ch] : 0;
  int p = p0;
  while (p < p1) {
    int s = pt_seg[p];
    int q = p + 1;
    // add points while the batch stays within 32 observations and 32 points
    while (q < p1 && (q - p) < SSFM_BATCH && pt_seg[q + 1] - s <= SSFM_BATCH) ++q;
    if (pass) { bat_pt[out + nb] = p; bat_obs[out + nb] = s; }
    ++nb;
    p = q;
  }
  if (!pass) chunk_cnt[ch] = nb;
}

__global__ void k_tile_count(const int* __restrict__ cam_seg, int C, int* cnt) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) {
    int n = cam_seg[c + 1] - cam_seg[c];
    cnt[c] = (n + SSFM_TILE - 1) / SSFM_TILE;
  }
}

__global__ void k_tile_write(const int* __restrict__ cam_seg, const int* __restrict__ cam_tile, int C,
                             int* tile_obs, int* tile_cam) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) {
    int t0 = cam_tile[c], t1 = cam_tile[c + 1];
    for (int t = t0; t < t1; ++t) {
      tile_obs[t] = cam_seg[c] + (t - t0) * SSFM_TILE;
      tile_cam[t] = c;
    }
  }
}

__global__ void k_set_last(int* a, int idx, int v) { a[idx] = v; }

#ifndef SSFM_GRP
#define SSFM_GRP 4
#endif
