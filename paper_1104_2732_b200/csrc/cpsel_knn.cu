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

// P: the dimension (compile-time, 1..32); the queries sit in shared memory padded to PP = P rounded
// up to 4 and are read as 16-byte broadcasts; only the P real coordinates enter the sum
template <int P>
__global__ void __launch_bounds__(kDistThreads) knn_dist_kernel(const float* __restrict__ X,
                                                                const float* __restrict__ Q, uint64_t n,
                                                                uint32_t nq, float* __restrict__ D,
                                                                unsigned long long* bad) {
  constexpr int PP = (P + 3) / 4 * 4;
  __shared__ float4 qs[kDistQ][PP / 4];
  const uint32_t j0 = blockIdx.y * kDistQ;
  const uint32_t nj = min((uint32_t)kDistQ, nq - j0);
  for (uint32_t t = threadIdx.x; t < kDistQ * PP; t += blockDim.x) {
    const uint32_t j = t / PP, l = t % PP;
    reinterpret_cast<float*>(&qs[j][0])[l] = (j < nj && l < (uint32_t)P) ? Q[(size_t)(j0 + j) * P + l] : 0.f;
  }
  __syncthreads();
  unsigned nonfin = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    float xi[P];
#pragma unroll
    for (int l = 0; l < P; ++l) xi[l] = __ldg(X + i * P + l);
    float* out = D + (size_t)j0 * n + i;
#pragma unroll 4
    for (uint32_t j = 0; j < nj; ++j) {
      float d = 0.f;
#pragma unroll
      for (int l4 = 0; l4 < PP / 4; ++l4) {
        const float4 q = qs[j][l4];  // shared-memory broadcast
        const float qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (4 * l4 + c < P) {
            const float e = __fsub_rn(qv[c], xi[4 * l4 + c]);
            d = __fadd_rn(d, __fmul_rn(e, e));
          }
        }
      }
      __stcs(out + (size_t)j * n, d);
      nonfin += isfinite(d) ? 0u : 1u;  // NaN/Inf in X or Q, or an overflowing distance
    }
  }
  if (nonfin) atomicAdd(bad, (unsigned long long)nonfin);
}

__device__ __forceinline__ double knn_w(float d, int weighting) {
  return weighting ? 1.0 / ((double)d + kKnnEps) : 1.0;
}

// One CTA per query (grid-stride): the rho/a,b reduction of row j of D against d2_(k) = dk[j].
// Branch-free accumulation; 16-byte loads of the row and of f when both are aligned.
__global__ void __launch_bounds__(256) knn_reduce_kernel(const float* __restrict__ D, const float* __restrict__ f,
                                                         uint64_t n, uint32_t nq, uint64_t k,
                                                         const float* __restrict__ dk, int weighting,
                                                         float* __restrict__ out) {
  __shared__ double s_sum[4][8];
  __shared__ unsigned long long s_cnt[2][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t j = blockIdx.x; j < nq; j += gridDim.x) {
    const float t = dk[j];
    const float* row = D + (size_t)j * n;
    double s_lt = 0.0, w_lt = 0.0, s_eq = 0.0, w_eq = 0.0;
    unsigned long long c_lt = 0, c_eq = 0;
    // only d <= d_(k) carries weight: f is read for those alone (k of n per row, plus ties)
    auto acc = [&](float d, uint64_t i) {
      if (d <= t) {
        const float fi = __ldg(f + i);
        const double wi = knn_w(d, weighting), wf = wi * (double)fi;
        if (d < t) {
          s_lt += wf;
          w_lt += wi;
          ++c_lt;
        } else {
          s_eq += wf;
          w_eq += wi;
          ++c_eq;
        }
      }
    };
    uint64_t i0 = 0;
    if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
      const uint64_t nv = n / 4;
      const float4* r4 = reinterpret_cast<const float4*>(row);
      uint64_t v = threadIdx.x;
      for (; v + 3 * blockDim.x < nv; v += 4 * blockDim.x) {  // four 16-byte loads in flight per thread
        float4 d4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) d4[u] = __ldcs(r4 + v + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t b = 4 * (v + u * blockDim.x);
          acc(d4[u].x, b);
          acc(d4[u].y, b + 1);
          acc(d4[u].z, b + 2);
          acc(d4[u].w, b + 3);
        }
      }
      for (; v < nv; v += blockDim.x) {
        const float4 d4 = __ldcs(r4 + v);
        acc(d4.x, 4 * v);
        acc(d4.y, 4 * v + 1);
        acc(d4.z, 4 * v + 2);
        acc(d4.w, 4 * v + 3);
      }
      i0 = nv * 4;
    }
    for (uint64_t i = i0 + threadIdx.x; i < n; i += blockDim.x) acc(__ldcs(row + i), i);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s_lt += __shfl_xor_sync(0xffffffffu, s_lt, o);
      w_lt += __shfl_xor_sync(0xffffffffu, w_lt, o);
      s_eq += __shfl_xor_sync(0xffffffffu, s_eq, o);
      w_eq += __shfl_xor_sync(0xffffffffu, w_eq, o);
      c_lt += __shfl_xor_sync(0xffffffffu, c_lt, o);
      c_eq += __shfl_xor_sync(0xffffffffu, c_eq, o);
    }
    if (lane == 0) {
      s_sum[0][w] = s_lt; s_sum[1][w] = w_lt; s_sum[2][w] = s_eq; s_sum[3][w] = w_eq;
      s_cnt[0][w] = c_lt; s_cnt[1][w] = c_eq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a4[4] = {0, 0, 0, 0};
      unsigned long long c3[2] = {0, 0};
      for (int q = 0; q < 8; ++q) {
        for (int u = 0; u < 4; ++u) a4[u] += s_sum[u][q];
        for (int u = 0; u < 2; ++u) c3[u] += s_cnt[u][q];
      }
      // rho = a/b on the ties at d_(k): exactly k neighbours' worth of weight (P:L476 with h = k)
      const double a = (double)(k - c3[0]), b = (double)c3[1];
      const double r = b > 0 ? a / b : 0.0;
      out[j] = (float)((a4[0] + r * a4[2]) / (a4[1] + r * a4[3]));
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) knn_check_kernel(const float* __restrict__ f, uint64_t n,
                                                        unsigned long long* bad) {
  unsigned c = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    c += isfinite(f[i]) ? 0u : 1u;
  if (c) atomicAdd(bad, (unsigned long long)c);
}


// kNN classification ("the majority vote (among the k nearest neighbours)"): per query the
// rho-weighted votes of the classes, rho as in the regression (1 below d_(k), a/b at it), the
// winner = the largest vote, the smallest class index among equal votes.  Votes in fp64 shared
// memory (per-CTA; only the d <= d_(k) elements vote).
constexpr int kKnnMaxClasses = 64;
__global__ void __launch_bounds__(256) knn_vote_kernel(const float* __restrict__ D, const int* __restrict__ labels,
                                                       uint64_t n, uint32_t nq, uint64_t k, uint32_t nclass,
                                                       const float* __restrict__ dk, int weighting,
                                                       int* __restrict__ out, double* __restrict__ votes_out,
                                                       unsigned long long* bad) {
  __shared__ double v_lt[kKnnMaxClasses], v_eq[kKnnMaxClasses];
  __shared__ unsigned long long s_c[2];
  for (uint32_t j = blockIdx.x; j < nq; j += gridDim.x) {
    for (int c = threadIdx.x; c < kKnnMaxClasses; c += blockDim.x) v_lt[c] = v_eq[c] = 0.0;
    if (threadIdx.x < 2) s_c[threadIdx.x] = 0ull;
    __syncthreads();
    const float t = dk[j];
    const float* row = D + (size_t)j * n;
    unsigned long long c_lt = 0, c_eq = 0;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const float d = __ldcs(row + i);
      if (d <= t) {
        const int lab = labels[i];
        if (lab < 0 || (uint32_t)lab >= nclass) {
          atomicAdd(bad, 1ull);
          continue;
        }
        const double wi = knn_w(d, weighting);
        if (d < t) {
          atomicAdd(&v_lt[lab], wi);
          ++c_lt;
        } else {
          atomicAdd(&v_eq[lab], wi);
          ++c_eq;
        }
      }
    }
    atomicAdd(&s_c[0], c_lt);
    atomicAdd(&s_c[1], c_eq);
    __syncthreads();
    if (threadIdx.x == 0) {
      const double a = (double)(k - s_c[0]), b = (double)s_c[1];
      const double r = b > 0 ? a / b : 0.0;
      int best = 0;
      double bv = -1.0;
      for (uint32_t c = 0; c < nclass; ++c) {
        const double v = v_lt[c] + r * v_eq[c];
        if (votes_out) votes_out[(size_t)j * nclass + c] = v;
        if (v > bv) { bv = v; best = (int)c; }
      }
      out[j] = best;
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
  const dim3 g((unsigned)gx, gy);
  switch (p) {
#define KD(PV) \
  case PV: knn_dist_kernel<PV><<<g, kDistThreads, 0, st>>>(X, Q, n, nq, D, bad); break;
    KD(1) KD(2) KD(3) KD(4) KD(5) KD(6) KD(7) KD(8) KD(9) KD(10) KD(11) KD(12) KD(13) KD(14) KD(15) KD(16)
    KD(17) KD(18) KD(19) KD(20) KD(21) KD(22) KD(23) KD(24) KD(25) KD(26) KD(27) KD(28) KD(29) KD(30) KD(31) KD(32)
#undef KD
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t knn_reduce(const float* D, const float* f, uint64_t n, uint32_t nq, uint64_t k, const float* dk,
                       int weighting, float* out, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = sms * 8;
  if ((uint32_t)grid > nq) grid = (int)nq;
  knn_reduce_kernel<<<grid, 256, 0, st>>>(D, f, n, nq, k, dk, weighting, out);
  return cudaGetLastError();
}

cudaError_t knn_vote(const float* D, const int* labels, uint64_t n, uint32_t nq, uint64_t k, uint32_t nclass,
                     const float* dk, int weighting, int* out, double* votes, unsigned long long* bad, cudaStream_t st) {
  if (nclass == 0 || nclass > (uint32_t)kKnnMaxClasses) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = sms * 8;
  if ((uint32_t)grid > nq) grid = (int)nq;
  knn_vote_kernel<<<grid, 256, 0, st>>>(D, labels, n, nq, k, nclass, dk, weighting, out, votes, bad);
  return cudaGetLastError();
}

cudaError_t knn_check_f(const float* f, uint64_t n, unsigned long long* bad, cudaStream_t st) {
  knn_check_kernel<<<148 * 4, 256, 0, st>>>(f, n, bad);
  return cudaGetLastError();
}

}  // namespace cpsel
