// pattern.cuh -- reference-equivalent integer structures, built on the device
// for bit-exact comparison with the reference:
//   JtJPattern.off_keys  (sparse_block.py:260-266): sorted unique (a<b)
//                         param-block pairs co-occurring in a residual block
//   _SchurPlan slots     (lm.py:338-384): unique retained pairs (ra<=rb) per
//                         point, ordered by (shape code, slot code)
#pragma once
#include <cub/cub.cuh>
#include "topo.cuh"

// kind: 0 BA, 1 GP. F: number of focal blocks (BA) ; S: scale blocks (GP)
__global__ void k_offkey_codes(const int* __restrict__ pm_cam, const int* __restrict__ pm_pt,
                               const int* __restrict__ pm_obs, long long N, int kind, int C, int P,
                               int F, int nscale, long long nblocks, unsigned long long* codes) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const long long c = pm_cam[i], j = (long long)C + pm_pt[i];
  const int per = (kind == 0) ? (F ? 3 : 1) : (nscale ? 3 : 1);
  unsigned long long* out = codes + per * i;
  out[0] = (unsigned long long)(c * nblocks + j);
  if (per == 3) {
    long long x;
    if (kind == 0) x = (long long)C + P + (F == 1 ? 0 : c);
    else x = (long long)C + P + pm_obs[i];
    out[1] = (unsigned long long)(c * nblocks + x);
    out[2] = (unsigned long long)(j * nblocks + x);
  }
}

// retained list of a point: BA poses c then focal ids; GP centres
__device__ __forceinline__ int ret_item(const int* pm_cam, int s, int k, int m, int kind, int C, int F) {
  if (k < m) return pm_cam[s + k];
  return (F == 1) ? C : C + pm_cam[s + k - m];   // focal ret-local id
}

__global__ void k_slot_count(const int* __restrict__ pt_seg, int P, int kind, int F, long long* cnt) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P) return;
  const long long m = pt_seg[j + 1] - pt_seg[j];
  const long long L = (kind == 0 && F) ? 2 * m : m;
  cnt[j] = L * (L + 1) / 2;
}

__global__ void k_slot_codes(const int* __restrict__ pt_seg, const int* __restrict__ pm_cam, int P, int kind,
                             int C, int F, const long long* __restrict__ off, unsigned long long* codes) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P) return;
  const int s = pt_seg[j];
  const int m = pt_seg[j + 1] - s;
  const int L = (kind == 0 && F) ? 2 * m : m;
  // F: 2 per-camera focal (C focal blocks), 1 shared focal, 0 none
  const long long nret = (long long)C + (kind == 0 ? (F == 1 ? 1 : (F == 2 ? C : 0)) : 0);
  long long o = off[j];
  for (int a = 0; a < L; ++a) {
    const long long ra0 = ret_item(pm_cam, s, a, m, kind, C, F);
    for (int b = a; b < L; ++b) {
      const long long rb0 = ret_item(pm_cam, s, b, m, kind, C, F);
      const long long ra = ra0 < rb0 ? ra0 : rb0, rb = ra0 < rb0 ? rb0 : ra0;
      const int wa = (kind == 1) ? 3 : (ra < C ? 7 : 1);
      const int wb = (kind == 1) ? 3 : (rb < C ? 7 : 1);
      const unsigned long long shape = (unsigned long long)(wa * 8 + wb);
      codes[o++] = (shape << 56) | (unsigned long long)(ra * nret + rb);
    }
  }
}

__global__ void k_decode_pairs(const unsigned long long* __restrict__ codes, long long n, long long base,
                               int* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long v = codes[i] & ((1ull << 56) - 1);
  out[2 * i] = (int)(v / base);
  out[2 * i + 1] = (int)(v % base);
}
