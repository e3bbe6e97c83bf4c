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
  // fused path (§8f-2): no S
  void* fimg = nullptr;        // Theta (A operand, 128 candidates/tile) + X (B operand, 256 rows/tile) images, padded y
  size_t fimg_bytes = 0;
  void* fcol = nullptr;        // per-column cuts / counters / slot map / fail list, LTS partial sums
  size_t fcol_bytes = 0;
  float* fz = nullptr;         // per-column copies of ]t_lo, t_hi[ (C x zcap)
  size_t fz_bytes = 0;
  float* fS = nullptr;         // stored S of the columns the fused input could not finish
  size_t fS_bytes = 0;
  void* fsamp = nullptr;       // sample rows (X, y, B image) and their residuals for the R23 cuts
  size_t fsamp_bytes = 0;
};

struct LmsReport {
  uint32_t passes = 0, cp_iters = 0;
  uint64_t z_total = 0, bytes = 0, nonfinite = 0;
  double ms = 0;
  uint32_t fallback = 0;       // fused path: columns finished from a stored S
  double ms_fused = 0;         // fused path: cuts + fused tensor-core pass (CUDA events)
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
// Fused path (no S in HBM): the k-th smallest of every column of S = (X Theta - y 1^T)^2, taken on
// the residuals of fused_tc_kernel (3xTF32 tcgen05, recomputed in its epilogue).  rep->fallback =
// columns finished from a stored S (target outside the sample cuts or copy overflow).
cudaError_t lms_fused_select(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p,
                             const float* thetas, uint32_t C, uint64_t k, float* out, uint32_t max_iters,
                             LmsReport* rep, cudaStream_t st);
// Input check for the fused path: 0 = finite and overflow-free (fused path valid), 1 = NaN/Inf in
// X, y or Theta, 2 = finite but some s might overflow (use the stored-S path), -1 = CUDA error (*err).
int lms_fused_check(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p, const float* thetas,
                    uint32_t C, cudaStream_t st, cudaError_t* err);
// The S the fused path selects on (store mode of the same kernel, every column).
cudaError_t lms_fused_residuals(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p,
                                const float* thetas, uint32_t C, float* S, cudaStream_t st);
// LTS on the fused path: out[j] = sum_{s < m_j} s + (h - #{s < m_j}) m_j, one more fused pass.
cudaError_t lms_fused_lts(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p,
                          const float* thetas, uint32_t C, uint64_t h, const float* m, double* out, cudaStream_t st);
void lms_free(LmsWorkspace& w);

}  // namespace cpsel
