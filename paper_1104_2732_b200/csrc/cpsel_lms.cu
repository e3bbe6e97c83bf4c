// LMS stage: placeholder residual kernel (replaced by the tcgen05 kernel) + batched selection.
#include "cpsel_lms.h"

namespace cpsel {

__global__ void residual_ffma_kernel(const float* __restrict__ X, const float* __restrict__ y, uint64_t n, uint32_t p,
                                     const float* __restrict__ th, uint32_t C, float* __restrict__ S) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t j = blockIdx.y;
  if (i >= n) return;
  float acc = 0.f;
  for (uint32_t l = 0; l < p; ++l) acc = fmaf(X[i * p + l], th[(uint64_t)j * p + l], acc);
  const float r = acc - y[i];
  S[(uint64_t)j * n + i] = r * r;
}

cudaError_t lms_residuals(LmsWorkspace&, const float* X, const float* y, uint64_t n, uint32_t p, const float* thetas,
                          uint32_t C, float* S, cudaStream_t st) {
  dim3 grid((unsigned)((n + 255) / 256), C);
  residual_ffma_kernel<<<grid, 256, 0, st>>>(X, y, n, p, thetas, C, S);
  return cudaGetLastError();
}

cudaError_t batched_select(LmsWorkspace&, const float*, uint64_t, uint32_t, uint64_t, float*, uint32_t, LmsReport*,
                           cudaStream_t) {
  return cudaErrorNotSupported;
}

void lms_free(LmsWorkspace& w) {
  if (w.S) cudaFree(w.S);
  if (w.dev) cudaFree(w.dev);
  if (w.host) cudaFreeHost(w.host);
  w = LmsWorkspace{};
}

}  // namespace cpsel
