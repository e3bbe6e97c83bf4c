// LMS robust-regression stage (internal): batched residuals X.Theta on the tensor cores and the
// batched cutting-plane selection over the C columns of S.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cpsel {

constexpr int kLmsMaxP = 16;

struct LmsWorkspace {
  float* S = nullptr;          // n x C column-major squared residuals (cpsel_lms_objective)
  size_t S_bytes = 0;
  void* dev = nullptr;         // batched-select scratch (per-CTA ping-pong buffers) + counters
  size_t dev_bytes = 0;
  void* img = nullptr;         // packed TF32 hi/lo operand images of X and Theta
  size_t img_bytes = 0;
  void* host = nullptr;        // pinned mirror
  size_t host_bytes = 0;
};

struct LmsReport {
  uint32_t passes = 0, cp_iters = 0;
  uint64_t z_total = 0, bytes = 0, nonfinite = 0;
  double ms = 0;
};

cudaError_t lms_residuals(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p,
                          const float* thetas, uint32_t C, float* S, cudaStream_t st);
// Per column j of S (n x C column-major): the k-th smallest -> out[j].  Returns
// cudaErrorNotSupported if the iteration cap is reached.
cudaError_t batched_select(LmsWorkspace& w, const float* S, uint64_t n, uint32_t C, uint64_t k, float* out,
                           uint32_t max_iters, LmsReport* rep, cudaStream_t st);
// LTS objective per column from its h-th order statistic m[j] (fp64 out).
cudaError_t lts_reduce(const float* S, uint64_t n, uint32_t C, uint64_t h, const float* m, double* out,
                       cudaStream_t st);
void lms_free(LmsWorkspace& w);

}  // namespace cpsel
