// kNN regression through the k-th order statistic of the distances (NEXT row §8f-4):
// "by adapting the function rho in (med_reg), we obtain an indicator function, which returns a
// non-zero value for those data that are no further from x than the k-order statistic d_(k). Then
// the weighted sum of k nearest neighbours is calculated by reduction."
//
// Three steps, no sort of the distances:
//   1. knn_dist_kernel: D[j][i] = sum_l (q_jl - x_il)^2 for every query j and reference point i,
//      float32 with explicit round-to-nearest operations in the order l = 0..p-1 (no FMA
//      contraction), so the oracle reproduces every distance bit for bit;
//   2. the batched k-th selection (batched_select, step a8) of every row of D -> d2_(k);
//   3. knn_reduce_kernel: the indicator reduction rho(d) = 1 (d < d_(k)), a/b (d = d_(k)), 0
//      (else) with a = k - #{d < d_(k)}, b = #{d = d_(k)} (the LTS rho of P:L469-476 at rank k), so
//      exactly k neighbours carry weight even with ties; f(q) = sum rho w f / sum rho w, fp64,
//      fixed-order block reduction.  w = 1 (plain mean) or 1/(d2 + 1e-12) (inverse squared distance).
#include <cuda_runtime.h>

#include <cstdint>

#include "cpsel_knn.h"

namespace cpsel {
namespace {

constexpr int kDistThreads = 256;
constexpr int kDistQ = 16;  // queries per CTA (in shared memory)

__global__ void __launch_bounds__(kDistThreads) knn_dist_kernel(const float* __restrict__ X,
                                                                const float* __restrict__ Q, uint64_t n,
                                                                uint32_t p, uint32_t nq, float* __restrict__ D,
                                                                unsigned long long* bad) {
  __shared__ float qs[kDistQ * kKnnMaxP];
  const uint32_t j0 = blockIdx.y * kDistQ;
  const uint32_t nj = min((uint32_t)kDistQ, nq - j0);
  for (uint32_t t = threadIdx.x; t < nj * p; t += blockDim.x) qs[t] = Q[(size_t)j0 * p + t];
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    float xi[kKnnMaxP];
#pragma unroll
    for (int l = 0; l < kKnnMaxP; ++l)
      if (l < (int)p) xi[l] = X[i * p + l];
    for (uint32_t j = 0; j < nj; ++j) {
      float d = 0.f;
#pragma unroll
      for (int l = 0; l < kKnnMaxP; ++l) {
        if (l < (int)p) {
          const float e = __fsub_rn(qs[j * p + l], xi[l]);
          d = __fadd_rn(d, __fmul_rn(e, e));
        }
      }
      D[(size_t)(j0 + j) * n + i] = d;
      if (!isfinite(d)) atomicAdd(bad, 1ull);  // NaN/Inf in X or Q, or an overflowing distance
    }
  }
}

__device__ __forceinline__ double knn_w(float d, int weighting) {
  return weighting ? 1.0 / ((double)d + kKnnEps) : 1.0;
}

// One CTA per query (grid-stride): the rho/a,b reduction of row j of D against d2_(k) = dk[j].
__global__ void __launch_bounds__(256) knn_reduce_kernel(const float* __restrict__ D, const float* __restrict__ f,
                                                         uint64_t n, uint32_t nq, uint64_t k,
                                                         const float* __restrict__ dk, int weighting,
                                                         float* __restrict__ out, unsigned long long* bad) {
  __shared__ double s_sum[4][8];
  __shared__ unsigned long long s_cnt[3][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t j = blockIdx.x; j < nq; j += gridDim.x) {
    const float t = dk[j];
    const float* row = D + (size_t)j * n;
    double s_lt = 0.0, w_lt = 0.0, s_eq = 0.0, w_eq = 0.0;
    unsigned long long c_lt = 0, c_eq = 0, nonfin = 0;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const float d = __ldcs(row + i);
      const float fi = f[i];
      if (!isfinite(fi)) ++nonfin;
      if (d < t) {
        const double wi = knn_w(d, weighting);
        s_lt += wi * (double)fi;
        w_lt += wi;
        ++c_lt;
      } else if (d == t) {
        const double wi = knn_w(d, weighting);
        s_eq += wi * (double)fi;
        w_eq += wi;
        ++c_eq;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s_lt += __shfl_xor_sync(0xffffffffu, s_lt, o);
      w_lt += __shfl_xor_sync(0xffffffffu, w_lt, o);
      s_eq += __shfl_xor_sync(0xffffffffu, s_eq, o);
      w_eq += __shfl_xor_sync(0xffffffffu, w_eq, o);
      c_lt += __shfl_xor_sync(0xffffffffu, c_lt, o);
      c_eq += __shfl_xor_sync(0xffffffffu, c_eq, o);
      nonfin += __shfl_xor_sync(0xffffffffu, nonfin, o);
    }
    if (lane == 0) {
      s_sum[0][w] = s_lt; s_sum[1][w] = w_lt; s_sum[2][w] = s_eq; s_sum[3][w] = w_eq;
      s_cnt[0][w] = c_lt; s_cnt[1][w] = c_eq; s_cnt[2][w] = nonfin;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a4[4] = {0, 0, 0, 0};
      unsigned long long c3[3] = {0, 0, 0};
      for (int q = 0; q < 8; ++q) {
        for (int u = 0; u < 4; ++u) a4[u] += s_sum[u][q];
        for (int u = 0; u < 3; ++u) c3[u] += s_cnt[u][q];
      }
      // rho = a/b on the ties at d_(k): exactly k neighbours' worth of weight (P:L476 with h = k)
      const double a = (double)(k - c3[0]), b = (double)c3[1];
      const double r = b > 0 ? a / b : 0.0;
      out[j] = (float)((a4[0] + r * a4[2]) / (a4[1] + r * a4[3]));
      if (c3[2] && j == 0) atomicAdd(bad, c3[2]);
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t knn_distances(const float* X, const float* Q, uint64_t n, uint32_t p, uint32_t nq, float* D,
                          unsigned long long* bad, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned gy = (nq + kDistQ - 1) / kDistQ;
  uint64_t gx = (n + kDistThreads - 1) / kDistThreads;
  const uint64_t cap = (uint64_t)sms * 8 * 4 / (gy > 0 ? gy : 1) + 1;  // ~4 waves of 8 CTAs per SM
  if (gx > cap) gx = cap;
  knn_dist_kernel<<<dim3((unsigned)gx, gy), kDistThreads, 0, st>>>(X, Q, n, p, nq, D, bad);
  return cudaGetLastError();
}

cudaError_t knn_reduce(const float* D, const float* f, uint64_t n, uint32_t nq, uint64_t k, const float* dk,
                       int weighting, float* out, unsigned long long* bad, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = sms * 8;
  if ((uint32_t)grid > nq) grid = (int)nq;
  knn_reduce_kernel<<<grid, 256, 0, st>>>(D, f, n, nq, k, dk, weighting, out, bad);
  return cudaGetLastError();
}

}  // namespace cpsel
