// block_algebra.cuh -- the generic block-sparse products of the reference's
// public sparse_block API on the device: jtj (sparse_block.py:370-385 ->
// _core.pyx:18-58 jtj_fill_cy), jtr (sparse_block.py:388-403 -> _core.pyx:61-97
// jtr_fill_cy) and the diagonal scaling of apply_damping / scale_diag_inplace
// (sparse_block.py:406-439), for any BlockSparseJacobian.
//
// The contribution schedule (JtJPattern / JtrPattern: which entry pairs feed
// which output block, in which order) is integer index work done once per
// pattern by the host wrapper, exactly as the reference builds it. The kernels
// then reproduce the reference's arithmetic bit for bit: one owner per output
// scalar, contributions in schedule order, and within a contribution the
// residual-row dot product in row order with separate round-to-nearest multiply
// and add (the Cython loops are compiled without FMA contraction).
#pragma once
#include "common.cuh"

// one thread per output block (key): out[key_out_off[k] + i*wb + j] =
//   sum over contributions c of sum_r A_c[r][i] * B_c[r][j]
__global__ void k_block_jtj(const double* __restrict__ entry_data, const long long* __restrict__ entry_off,
                            const int* __restrict__ entry_h, const int* __restrict__ entry_w,
                            const long long* __restrict__ contrib_a, const long long* __restrict__ contrib_b,
                            const long long* __restrict__ seg_start, const long long* __restrict__ key_out_off,
                            long long nkeys, double* out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= nkeys) return;
  const long long c0 = seg_start[k], c1 = seg_start[k + 1];
  const long long ea0 = contrib_a[c0], eb0 = contrib_b[c0];
  const int wa = entry_w[ea0], wb = entry_w[eb0];
  const long long base = key_out_off[k];
  for (int i = 0; i < wa; ++i) {
    for (int j = 0; j < wb; ++j) {
      double acc = 0.0;
      for (long long c = c0; c < c1; ++c) {
        const long long ea = contrib_a[c], eb = contrib_b[c];
        const double* A = entry_data + entry_off[ea];
        const double* B = entry_data + entry_off[eb];
        const int h = entry_h[ea];
        double s = 0.0;
        for (int r = 0; r < h; ++r) s = __dadd_rn(s, __dmul_rn(A[r * wa + i], B[r * wb + j]));
        acc = __dadd_rn(acc, s);
      }
      out[base + (long long)i * wb + j] = acc;
    }
  }
}

// one thread per param segment: out[seg_out[s] + i] = sum over entries c of
//   sum_r J_c[r][i] * res[res_row[c] + r]
__global__ void k_block_jtr(const double* __restrict__ entry_data, const long long* __restrict__ entry_off,
                            const int* __restrict__ entry_h, const int* __restrict__ entry_w,
                            const int* __restrict__ by_entry, const long long* __restrict__ seg_start,
                            const long long* __restrict__ seg_out, const long long* __restrict__ res_row,
                            long long nsegs, const double* __restrict__ res, double* out) {
  const long long sg = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (sg >= nsegs) return;
  const long long c0 = seg_start[sg], c1 = seg_start[sg + 1];
  const int w = entry_w[by_entry[c0]];
  for (int i = 0; i < w; ++i) {
    double acc = 0.0;
    for (long long c = c0; c < c1; ++c) {
      const int e = by_entry[c];
      const int h = entry_h[e];
      const double* J = entry_data + entry_off[e];
      const long long ro = res_row[c];
      double v = 0.0;
      for (int r = 0; r < h; ++r) v = __dadd_rn(v, __dmul_rn(J[r * w + i], res[ro + r]));
      acc = __dadd_rn(acc, v);
    }
    out[seg_out[sg] + i] = acc;
  }
}

// data[idx[k]] *= factor (diagonal scalars of the diagonal blocks)
__global__ void k_block_scale_diag(double* data, const long long* __restrict__ idx, long long n, double factor) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < n) data[idx[k]] = __dmul_rn(data[idx[k]], factor);
}
