// dense.cuh -- the reference's dense solver (lm.py:124-220 _DensePlan,
// materialize_dense, _solve_dense) on the device, for small problems and the
// LMConfig(solver="dense") option:
//   assemble A from the block storage (scatter, the caller's _DensePlan
//   indices), pin exactly-zero diagonals (the gradient entry must be zero),
//   reject negative diagonals, Jacobi-equilibrate, Cholesky (cuSOLVER potrf,
//   loaded on first use with dlopen: no load-time dependency of the library),
//   solve, un-scale.
#pragma once
#include <dlfcn.h>
#include <cusolverDn.h>
#include "common.cuh"

__global__ void k_dense_scatter(const double* __restrict__ src_data, const long long* __restrict__ dst,
                                const long long* __restrict__ src, long long m, double* A) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < m) A[dst[k]] = src_data[src[k]];
}

// pin zero diagonals, check signs, s = 1 / sqrt(diag), rhs = s * b
__global__ void k_dense_prep(double* A, const double* __restrict__ b, long long n, double* s, double* rhs,
                             int* flag) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = A[i * n + i];
  if (d == 0.0) {
    if (b[i] != 0.0) atomicOr(flag, 1);   // zero diagonal with non-zero gradient
    A[i * n + i] = 1.0;
    d = 1.0;
  }
  if (d < 0.0) atomicOr(flag, 2);        // negative diagonal in damped system
  const double si = 1.0 / sqrt(d);
  s[i] = si;
  rhs[i] = si * b[i];
}

// A_ij *= s_j, then *= s_i (the reference's order)
__global__ void k_dense_scale(double* A, const double* __restrict__ s, long long n) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n * n) return;
  const long long i = k / n, j = k - i * n;
  A[k] = (A[k] * s[j]) * s[i];
}

__global__ void k_dense_unscale(const double* __restrict__ s, const double* __restrict__ y, long long n,
                                double* x) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) x[i] = s[i] * y[i];
}

struct CuSolverApi {
  bool tried = false, ok = false;
  cusolverStatus_t (*create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*destroy)(cusolverDnHandle_t) = nullptr;
  cusolverStatus_t (*set_stream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*potrf_bs)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*potrf)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*potrs)(cusolverDnHandle_t, cublasFillMode_t, int, int, const double*, int, double*, int,
                            int*) = nullptr;
};

static CuSolverApi& cusolver_api() {
  static CuSolverApi api;
  if (api.tried) return api;
  api.tried = true;
  void* lib = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_LOCAL);
  if (!lib) lib = dlopen("/usr/local/cuda/lib64/libcusolver.so.11", RTLD_NOW | RTLD_LOCAL);
  if (!lib) return api;
  api.create = (decltype(api.create))dlsym(lib, "cusolverDnCreate");
  api.destroy = (decltype(api.destroy))dlsym(lib, "cusolverDnDestroy");
  api.set_stream = (decltype(api.set_stream))dlsym(lib, "cusolverDnSetStream");
  api.potrf_bs = (decltype(api.potrf_bs))dlsym(lib, "cusolverDnDpotrf_bufferSize");
  api.potrf = (decltype(api.potrf))dlsym(lib, "cusolverDnDpotrf");
  api.potrs = (decltype(api.potrs))dlsym(lib, "cusolverDnDpotrs");
  api.ok = api.create && api.destroy && api.set_stream && api.potrf_bs && api.potrf && api.potrs;
  return api;
}
