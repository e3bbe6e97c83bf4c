// Micro-benchmark (not product code): the HBM read ceiling of the init pass's access pattern —
// warp-strided groups of 4 float4 per lane, the next group's loads issued before the current group's
// work, a min over the values so nothing is optimized away.  Built and timed by scripts/micro/readbw.py.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ld_nc(const float4* p) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

template <int U, int PD>
__global__ void __launch_bounds__(256, 4) read_kernel(const float4* __restrict__ x, uint64_t nvec, float* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t W = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5), Wt = (uint64_t)gridDim.x * 8;
  const uint64_t GV = 32 * U, nfull = nvec / GV;
  float m = 3.4e38f;
  float4 v[U];
  if (W < nfull)
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_nc(x + W * GV + u * 32 + lane);
  if (PD > 0 && lane == 0)
    for (int d = 1; d <= PD; ++d)
      if (W + d * Wt < nfull)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + (W + d * Wt) * GV), "r"((unsigned)(GV * 16)) : "memory");
  for (uint64_t g = W; g < nfull; g += Wt) {
    if (PD > 0 && lane == 0 && g + (PD + 1) * Wt < nfull)  // keep PD groups beyond the next one prefetched
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + (g + (PD + 1) * Wt) * GV), "r"((unsigned)(GV * 16)) : "memory");
    float4 c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = v[u];
    if (g + Wt < nfull)
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_nc(x + (g + Wt) * GV + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < U; ++u) m = fminf(m, fminf(fminf(c[u].x, c[u].y), fminf(c[u].z, c[u].w)));
  }
  if (m < -1e38f) out[0] = m;
}

extern "C" int run_read(const void* x, uint64_t n, float* out, int grid, int u, int pd, float* ms, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t nvec = n / 4;
  auto go = [&]() {
    if (u == 4 && pd == 0) read_kernel<4, 0><<<grid, 256>>>((const float4*)x, nvec, out);
    else if (u == 4 && pd == 1) read_kernel<4, 1><<<grid, 256>>>((const float4*)x, nvec, out);
    else if (u == 4 && pd == 2) read_kernel<4, 2><<<grid, 256>>>((const float4*)x, nvec, out);
    else if (u == 4) read_kernel<4, 4><<<grid, 256>>>((const float4*)x, nvec, out);
    else if (u == 8) read_kernel<8, 0><<<grid, 256>>>((const float4*)x, nvec, out);
    else read_kernel<2, 0><<<grid, 256>>>((const float4*)x, nvec, out);
  };
  go();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) go();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  *ms /= reps;
  return (int)cudaGetLastError();
}
