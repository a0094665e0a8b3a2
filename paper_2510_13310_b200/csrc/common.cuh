// common.cuh -- shared device utilities for the sparse LM core.
//
// Determinism contract (mirrors _kernels/_core.pyx:1-8 and SPEC's "fixed
// summation order"): every output block is reduced by exactly one owner in a
// fixed order. Point segments are summed sequentially in observation order by
// one lane; camera segments are split into fixed tiles, each tile reduced by a
// fixed butterfly tree, and the tile partials are summed in tile order. No
// floating-point atomics anywhere, so results are bit-stable run to run.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define SSFM_WARP 32
#define SSFM_FULL 0xffffffffu

// Device status bits (accumulated with atomicOr on an int in device memory).
enum : int {
  ST_SINGULAR_POINT = 1 << 0,     // lm.py:508-512 det<=0 / non-finite
  ST_PIN_POINT = 1 << 1,          // lm.py:503-505 masked point dir with gradient
  ST_SINGULAR_PRECOND = 1 << 2,   // lm.py:520-525
  ST_PIN_RETAINED = 1 << 3,       // lm.py:631-633
  ST_CG_MAXITER = 1 << 4,         // lm.py:652-655
  ST_CG_BREAKDOWN = 1 << 5,       // lm.py:657-659
  ST_ZERO_QUAT = 1 << 6,          // lm.py:114-115
  ST_PIN_SCALE = 1 << 7,          // lm.py:569-575
  ST_BAD_INDEX = 1 << 8,
  ST_SCHEDULE = 1 << 9,           // fused-operator ticket schedule violated (internal error)
  ST_COMM_TIMEOUT = 1 << 10,      // a peer rank did not reach the exchange (comm.cuh)
};

__device__ __forceinline__ double shfl_xor_d(double v, int m) {
  return __shfl_xor_sync(SSFM_FULL, v, m);
}

// Butterfly all-reduce of V doubles inside a warp (fixed tree -> deterministic,
// every lane ends with the same bits).
template <int V>
__device__ __forceinline__ void warp_allreduce(double (&v)[V]) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] += shfl_xor_d(v[k], m);
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += shfl_xor_d(v, m);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = fmax(v, shfl_xor_d(v, m));
  return v;
}

// Block reduction of V doubles: warp butterflies, then warp 0 sums the warp
// results in warp order. `sm` needs (blockDim/32)*V doubles. Result valid in
// thread 0 only (returned in v for tid 0). Must be called by all threads.
template <int V>
__device__ __forceinline__ void block_reduce(double (&v)[V], double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  warp_allreduce<V>(v);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < V; ++k) sm[warp * V + k] = v[k];
  }
  __syncthreads();
  if (V <= 4) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        double s = sm[k];
        for (int w = 1; w < nw; ++w) s += sm[w * V + k];
        v[k] = s;
      }
    }
  } else {
    // wide reductions: lane k of warp 0 sums component k over the warps (same
    // warp order as the sequential loop, so the same bits), results back
    // through shared memory for thread 0
    if (warp == 0) {
      for (int k = lane; k < V; k += 32) {
        double s = sm[k];
        for (int w = 1; w < nw; ++w) s += sm[w * V + k];
        sm[k] = s;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < V; ++k) v[k] = sm[k];
    }
  }
  __syncthreads();
}

// 32-byte vector load (LDG.E.ENL2.256 on sm_100a): 4 consecutive doubles, the
// address must be 32-byte aligned. One instruction per 4 doubles of a gathered
// camera/point block instead of four 8-byte gathers (L1 wavefronts dominate
// scattered gathers). Coherent (no .nc): the vectors gathered this way are
// rewritten between grid barriers inside the persistent PCG kernels.
__device__ __forceinline__ void ld_v4(const double* a, double* x) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3]) : "l"(a));
}

// L2 eviction policies (createpolicy): the per-observation Jacobian streams
// through L2 once per pass (evict_first, and no L1 allocation: it lives in
// registers), while the small per-point / per-camera vectors that are
// gathered at random (y, p) should survive the stream (evict_last).
__device__ __forceinline__ unsigned long long pol_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ldg_stream(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int ldg_stream_i(const int* a, unsigned long long pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void ld_v4_hint(const double* a, double* x, unsigned long long pol) {
  asm volatile("ld.global.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3]) : "l"(a), "l"(pol));
}
// read-only variant for kernels in which the gathered vector is constant (the
// graph-PCG passes): non-coherent path, no L1 allocation (random 32-byte
// gathers have little L1 reuse and the fills compete with the streams)
__device__ __forceinline__ void ld_v4_ro(const double* a, double* x, unsigned long long pol) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3]) : "l"(a), "l"(pol));
}

// L2 prefetch of the byte range [a, a + bytes) with one bulk (TMA) request:
// the range is widened to 16-byte alignment (cp.async.bulk.prefetch needs it;
// device allocations are 256-byte granular, so the widened range stays mapped)
__device__ __forceinline__ void pf_l2_bulk(const void* a, long long bytes) {
  if (bytes <= 0) return;
  const unsigned long long s = reinterpret_cast<unsigned long long>(a);
  const unsigned long long lo = s & ~15ull, hi = (s + (unsigned long long)bytes + 15ull) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((unsigned)(hi - lo)) : "memory");
}

// LDGSTS: asynchronous global -> shared copies (per thread; groups committed
// and waited on per thread, so a warp needs __syncwarp before reading a
// peer's element). The L2 policy rides along.
__device__ __forceinline__ void cp_async8(void* s, const void* g, unsigned long long pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(sa), "l"(g), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async4(void* s, const void* g, unsigned long long pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(sa), "l"(g), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Stream-ordered fills and copies for the solve paths (instead of
// cudaMemsetAsync / device-to-device cudaMemcpyAsync: with several shards on
// one device those are implicit synchronisation points between streams, so a
// shard's memset would wait behind a peer's kernel that spins in an exchange
// waiting for this very shard).
__global__ void k_fill_u32(unsigned* p, long long n, unsigned v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void k_copy_f64(double* __restrict__ dst, const double* __restrict__ src, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// sum of buf[V t + k] over the tiles t in [t0, t1) of one camera, in t order
// (bit-identical to the plain loop) with the loads issued eight at a time: the
// plain loop waits one L2 round trip per tile (16 tiles per camera at C5)
template <int V>
__device__ __forceinline__ double tiles_sum(const double* buf, int k, int t0, int t1) {
  double s = 0.0;
  for (int t = t0; t < t1; t += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = t + u < t1 ? buf[(long long)V * (t + u) + k] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (t + u < t1) s += v[u];
  }
  return s;
}

// 32-byte store with an L2 eviction policy (a whole sector)
__device__ __forceinline__ void st_v4_hint(double* a, double x0, double x1, double x2, double x3,
                                           unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "d"(x0), "d"(x1), "d"(x2),
               "d"(x3), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

// Symmetric 3x3 stored as upper triangle {00,01,02,11,12,22}.
__device__ __forceinline__ void sym3_matvec(const double* m, const double* x, double* y) {
  y[0] = m[0] * x[0] + m[1] * x[1] + m[2] * x[2];
  y[1] = m[1] * x[0] + m[3] * x[1] + m[4] * x[2];
  y[2] = m[2] * x[0] + m[4] * x[1] + m[5] * x[2];
}

// Upper-triangle index of (i<=j) in an n x n symmetric matrix stored row-wise.
__host__ __device__ constexpr int sym_idx(int n, int i, int j) {
  return i * n - (i * (i - 1)) / 2 + (j - i);
}

// Warp-level 8-lane group helpers (4 cameras per warp, one lane per retained
// slot): broadcast slot k of the group.
__device__ __forceinline__ double grp8_get(double v, int k) {
  const int base = (threadIdx.x & 31) & ~7;
  return __shfl_sync(SSFM_FULL, v, base + k);
}
