// kNN regression via d_(k) (internal; NEXT row §8f-4).  See cpsel_knn.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cpsel {

constexpr int kKnnMaxP = 32;        // dimensions of a point
constexpr double kKnnEps = 1e-12;   // inverse-distance weight 1/(d^2 + eps)

// D (nq x n row-major): squared Euclidean distances, float32, explicit rn ops in order l = 0..p-1;
// *bad += #non-finite distances
cudaError_t knn_distances(const float* X, const float* Q, uint64_t n, uint32_t p, uint32_t nq, float* D,
                          unsigned long long* bad, cudaStream_t st);
// out[j] = sum rho_i w_i f_i / sum rho_i w_i, rho = 1 below dk[j], a/b at it
cudaError_t knn_reduce(const float* D, const float* f, uint64_t n, uint32_t nq, uint64_t k, const float* dk,
                       int weighting, float* out, cudaStream_t st);
// classification: out[j] = argmax_c sum rho_i w_i [label_i = c] (smallest c among equal votes), the
// votes (nullable) nq x nclass; *bad += #labels outside [0, nclass)
cudaError_t knn_vote(const float* D, const int* labels, uint64_t n, uint32_t nq, uint64_t k, uint32_t nclass,
                     const float* dk, int weighting, int* out, double* votes, unsigned long long* bad, cudaStream_t st);
// *bad += #non-finite f_i
cudaError_t knn_check_f(const float* f, uint64_t n, unsigned long long* bad, cudaStream_t st);

}  // namespace cpsel
