// comm.cuh -- cross-GPU exchange for the point-sharded solver.
//
// Observations are sharded by point ownership: each rank holds all cameras
// (replicated) and a contiguous range of points with every observation of
// those points. Camera-side sums (J^T J camera blocks, J^T r, the Schur
// preconditioner blocks, the camera half of S*p every CG iteration) and the
// scalar reductions (cost, |g|^2, max|g|, status bits) are the only exchange.
//
// Transport: peer memory. Every rank owns one exchange region in its HBM:
//   [ flag u64 | pad to 256 B | buffer 0 (cap doubles) | buffer 1 (cap doubles) ]
// and maps every peer's region (CUDA IPC across processes over NVLink 5 /
// NVSwitch, or plain device pointers for several handles in one process).
// An allreduce with epoch e:
//   1. write the local contribution into own buffer[e & 1]
//   2. fence.sys; st.release.sys own flag = e
//   3. wait until every peer's flag >= e (ld.acquire.sys, bounded spin)
//   4. read buffer[e & 1] of ranks 0..R-1 and combine IN RANK ORDER
// Step 4 runs the same operations in the same order on every rank, so every
// replicated quantity stays bitwise identical across ranks and all ranks take
// the same LM / CG control decisions with no broadcast. Double buffering is
// safe: a peer can only reach epoch e + 2 (overwriting buffer[e & 1]) after it
// has seen our flag at e + 1, which we publish only after finishing step 4.
//
// Inside the persistent PCG kernels steps 1-4 are fused with the operator:
// CTAs write their slice, grid.sync, one thread does 2-3, grid.sync, every
// CTA reads the peers' slices it needs -- the exchange of the camera half of
// S*p needs no extra kernel launch and no host round trip per CG iteration.
// Between kernels, the same protocol runs as three small kernels
// (k_ar_post / k_ar_barrier / k_ar_reduce).
#pragma once
#include "common.cuh"

#define SSFM_MAX_RANKS 16
#define COMM_TIMEOUT_NS 60000000000ull   // 60 s (SSFM_COMM_TIMEOUT_S): a lost peer is an error, not a hang

enum { AR_SUM = 0, AR_MAX = 1, AR_OR = 2 };

struct CommDev {
  int rank = 0;
  int nranks = 1;
  long long cap = 0;                                  // doubles per buffer
  unsigned long long* flag[SSFM_MAX_RANKS] = {};      // every rank's epoch flag (own at [rank])
  double* buf[SSFM_MAX_RANKS] = {};                   // every rank's 2 x cap buffers
  unsigned long long* epoch = nullptr;                // own epoch counter (local memory)
  int* status = nullptr;
  unsigned long long timeout_ns = COMM_TIMEOUT_NS;
};

__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// steps 2-3; called by ONE thread after the local contribution is written
__device__ __forceinline__ void comm_signal_wait(const CommDev& cm, unsigned long long e) {
  __threadfence_system();
  st_release_sys_u64(cm.flag[cm.rank], e);
  const unsigned long long t0 = globaltimer_ns();
  for (int r = 0; r < cm.nranks; ++r) {
    if (r == cm.rank) continue;
    while (ld_acquire_sys_u64(cm.flag[r]) < e) {
      if (globaltimer_ns() - t0 > cm.timeout_ns) {
        atomicOr(cm.status, ST_COMM_TIMEOUT);
        // diagnostic: where the peers are (a peer behind e never arrived; one
        // ahead means the ranks ran different collective sequences)
        printf("[ssfm comm] rank %d timed out at epoch %llu waiting for rank %d (flag %llu)\n", cm.rank, e, r,
               ld_acquire_sys_u64(cm.flag[r]));
        return;
      }
    }
  }
}

__device__ __forceinline__ double comm_peer_load(const double* p) { return __ldcv(p); }

__device__ __forceinline__ double ar_combine(int op, double a, double b) {
  if (op == AR_MAX) return fmax(a, b);
  if (op == AR_OR) return (double)((long long)a | (long long)b);
  return a + b;
}

// 1. own buffer[(epoch + 1) & 1] <- src
__global__ void k_ar_post(CommDev cm, const double* __restrict__ src, long long n) {
  const unsigned long long e = *cm.epoch + 1;
  double* dst = cm.buf[cm.rank] + (e & 1) * cm.cap;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// 2-3, then advance the local epoch
__global__ void k_ar_barrier(CommDev cm) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const unsigned long long e = *cm.epoch + 1;
    comm_signal_wait(cm, e);
    *cm.epoch = e;
  }
}

// 4. dst <- combine over ranks in rank order
__global__ void k_ar_reduce(CommDev cm, double* dst, long long n, int op) {
  const unsigned long long e = *cm.epoch;
  const long long off = (e & 1) * cm.cap;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double v = comm_peer_load(cm.buf[0] + off + i);
    for (int r = 1; r < cm.nranks; ++r) v = ar_combine(op, v, comm_peer_load(cm.buf[r] + off + i));
    dst[i] = v;
  }
}

// int status word <-> double for the OR reduction
__global__ void k_status_to_double(const int* s, double* d) { *d = (double)*s; }
__global__ void k_double_to_status(const double* d, int* s) { *s = (int)(long long)*d; }
