// K4: dense all-pairs double sums for the exact cosine (reference
// inner_product.cpp:179-236, `dense_self_norm_sq` and `exact_cosine`):
//   S(A, B) = sum_a sum_b c(a, b) * sigma^2 exp(-|p_a - p_b|^2 / (2 l^2)),
//   c = prod_k (linear: <u, v> | SE: sigma_k^2 exp(-|u - v|^2 / (2 l_k^2)))
// (kernels.cpp:18-53, kernels.hpp:45-47), in FP64 throughout (B200 runs FP64
// at half the FP32 rate; the reference's own tests hold the cosine to 1e-12).
//
// One thread per point a (position + feature row in registers), B streamed
// through shared memory in tiles of kDenseTile points; the exponents of the
// geometric and SE factors are added so each pair costs one exp. Each block
// writes one FP64 partial per (a-block, b-chunk); the host adds them in a
// fixed order, so results are deterministic.
#include <cuda_runtime.h>

#include "engine.cuh"

namespace kreg_dev {

namespace {

constexpr int kDenseThreads = 128;
constexpr int kDenseTile = 32;
#ifndef KREG_DENSE_J
#define KREG_DENSE_J 2
#endif
constexpr int kDenseJ = KREG_DENSE_J;  // target points per inner iteration (divides kDenseTile)

template <int DMAX>
__global__ void __launch_bounds__(kDenseThreads) k_dense(const DenseReq* reqs) {
  const DenseReq& R = reqs[blockIdx.z];
  const int a = blockIdx.x * kDenseThreads + threadIdx.x;
  const int D = R.D;
  __shared__ double bp[kDenseTile][3];
  __shared__ double bf[kDenseTile][DMAX > 0 ? DMAX : 1];
  __shared__ double su[DMAX > 0 ? DMAX : 1][kDenseThreads];  // a's feature row, one column per thread
  double px = 0, py = 0, pz = 0;
  const bool active = a < R.n_a;
  if (active) {
    px = R.a[3 * (long long)a];
    py = R.a[3 * (long long)a + 1];
    pz = R.a[3 * (long long)a + 2];
    for (int d = 0; d < D; ++d) su[d][threadIdx.x] = R.af[(long long)a * D + d];
  }
  const long long b0 = (long long)R.n_b * blockIdx.y / gridDim.y;
  const long long b1 = (long long)R.n_b * (blockIdx.y + 1) / gridDim.y;
  double acc = 0.0;
  for (long long t0 = b0; t0 < b1; t0 += kDenseTile) {
    const int nt = (int)min((long long)kDenseTile, b1 - t0);
    __syncthreads();
    for (int k = threadIdx.x; k < nt * 3; k += kDenseThreads) bp[k / 3][k % 3] = R.b[3 * t0 + k];
    if (DMAX > 0)
      for (int k = threadIdx.x; k < nt * D; k += kDenseThreads) bf[k / D][k % D] = R.bf[t0 * D + k];
    __syncthreads();
    if (!active) continue;
    // kDenseJ target points at a time: independent FP64 dependency chains
    // (the per-pair dot products and exponent sums are serial otherwise)
    for (int j0 = 0; j0 < nt; j0 += kDenseJ) {
      double expo[kDenseJ], c[kDenseJ];
#pragma unroll
      for (int q = 0; q < kDenseJ; ++q) {
        const int j = min(j0 + q, nt - 1);
        const double dx = px - bp[j][0], dy = py - bp[j][1], dz = pz - bp[j][2];
        expo[q] = (dx * dx + dy * dy + dz * dz) * R.neg_inv_2l2;  // kernels.hpp:45-47
        c[q] = 1.0;
      }
      if (DMAX > 0) {
        for (int k = 0; k < R.n_channels; ++k) {  // kernels.cpp:34-52
          const DenseChannel& ch = R.ch[k];
          double sq[kDenseJ];
#pragma unroll
          for (int q = 0; q < kDenseJ; ++q) sq[q] = 0.0;
          if (ch.linear) {
            for (int d = 0; d < ch.dim; ++d) {
              const double u = su[ch.offset + d][threadIdx.x];
#pragma unroll
              for (int q = 0; q < kDenseJ; ++q) sq[q] += u * bf[min(j0 + q, nt - 1)][ch.offset + d];
            }
#pragma unroll
            for (int q = 0; q < kDenseJ; ++q) c[q] *= sq[q];
          } else {
            for (int d = 0; d < ch.dim; ++d) {
              const double u = su[ch.offset + d][threadIdx.x];
#pragma unroll
              for (int q = 0; q < kDenseJ; ++q) {
                const double e = u - bf[min(j0 + q, nt - 1)][ch.offset + d];
                sq[q] += e * e;
              }
            }
#pragma unroll
            for (int q = 0; q < kDenseJ; ++q) expo[q] += sq[q] * ch.neg_inv_2l2;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kDenseJ; ++q)
        if (j0 + q < nt) acc += c[q] * exp(expo[q]);
    }
  }
  // fixed-order block reduction
  __shared__ double red[kDenseThreads];
  red[threadIdx.x] = acc * R.pref;
  __syncthreads();
  for (int s = kDenseThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) R.partials[(long long)blockIdx.y * gridDim.x + blockIdx.x] = red[0];
}

}  // namespace

void dense_sums(const DenseReq* h, const DenseReq* d, int n, int b_chunks, cudaStream_t st) {
  int max_a = 1, max_d = 0;
  for (int r = 0; r < n; ++r) {
    max_a = max(max_a, h[r].n_a);
    max_d = max(max_d, h[r].D);
  }
  const dim3 grid((max_a + kDenseThreads - 1) / kDenseThreads, b_chunks, n);
  if (max_d == 0) k_dense<0><<<grid, kDenseThreads, 0, st>>>(d);
  else if (max_d <= 8) k_dense<8><<<grid, kDenseThreads, 0, st>>>(d);
  else k_dense<kMaxDenseDim><<<grid, kDenseThreads, 0, st>>>(d);
  note_launches(1);
}

int dense_blocks_a(int n_a) { return (n_a + kDenseThreads - 1) / kDenseThreads; }

}  // namespace kreg_dev
