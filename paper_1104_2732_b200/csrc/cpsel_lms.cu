// LMS robust-regression stage: S = (X Theta - y 1^T)^2 on the 5th-generation tensor
// cores (step a7), then the batched cutting-plane selection of every column (step a8, kernel in
// cpsel_kernels.cu).
//
// a7 design: X (n x p) and Theta (p x C) are split once into TF32 hi/lo parts and
// packed into the tcgen05 K-major no-swizzle core-matrix image (8 rows x 16 B per core matrix,
// K padded to 16).  A persistent kernel (one CTA per SM) walks the (128-row x 256-candidate) tiles:
//   warp 0  : producer — cp.async.bulk (TMA bulk copy) of the A and B images into a 2-stage smem
//             ring, completion on mbarriers (expect_tx);
//   warp 1  : MMA issuer — one elected thread issues 6 tcgen05.mma.kind::tf32 (M=128, N=256, K=8):
//             hi*hi + hi*lo + lo*hi for each K-half (3xTF32, ~fp32-accurate products), into one of
//             two TMEM accumulators (2 x 256 columns), then tcgen05.commit to the smem-empty and the
//             TMEM-full barriers;
//   warps 2-9: epilogue — two warps per TMEM lane quarter, each on 128 of the 256 columns:
//             tcgen05.ld 32x32b.x32 (TMEM lane = row), r = acc - y_i, s = r*r, and a coalesced
//             store into column-major S (each warp-store = 32 consecutive rows of one column =
//             128 B, pointer-stepped by n), then arrive on the TMEM-empty barrier.
// The stage is HBM-write bound (4 bytes of S per 2p flops); the tensor cores keep the contraction
// off the FP32 pipes so the epilogue can stream S at full bandwidth.
#include <cstdint>

#include "cpsel_kernels.h"
#include "cpsel_ptx.h"
#include "cpsel_lms.h"

namespace cpsel {
namespace {

constexpr int TM = 128;              // rows per tile (TMEM lanes)
constexpr int TN = 256;              // candidates per tile (TMEM columns per accumulator)
constexpr int KP = 16;               // padded K
constexpr int A_HALF = TM * KP * 4;  // 8 KB (hi or lo)
constexpr int B_HALF = TN * KP * 4;  // 16 KB
constexpr int A_IMG = 2 * A_HALF;    // 16 KB per M tile
constexpr int B_IMG = 2 * B_HALF;    // 32 KB per N tile
constexpr int STAGE = A_IMG + B_IMG; // 48 KB
constexpr int kEpiWarps = 8;         // 2 per TMEM lane quarter, each on half of the 256 columns
constexpr int kThreads = 32 * (2 + kEpiWarps);

// byte offset of element (row, k) in a K-major no-swizzle core-matrix image
__host__ __device__ constexpr uint32_t core_off(int row, int k) {
  return (uint32_t)((row >> 3) * 512 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__global__ void pack_rows_kernel(const float* __restrict__ src, uint64_t rows, uint32_t p, int tile_rows,
                                 unsigned char* __restrict__ img) {
  const uint64_t tile = blockIdx.x;
  const int r = threadIdx.x;
  const uint64_t row = tile * tile_rows + r;
  const int half = tile_rows * KP * 4;
  unsigned char* base = img + tile * (uint64_t)(2 * half);
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const float v = (row < rows && k < (int)p) ? src[row * p + k] : 0.f;
    const uint32_t hi = tf32_rna(v);
    const uint32_t lo = tf32_rna(v - __uint_as_float(hi));
    *reinterpret_cast<uint32_t*>(base + core_off(r, k)) = hi;
    *reinterpret_cast<uint32_t*>(base + half + core_off(r, k)) = lo;
  }
}

// K-major, no swizzle: LBO = 128 B (between the two 16-B K chunks), SBO = 512 B (between 8-row groups)
__device__ __forceinline__ uint64_t sdesc(const void* p) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3FFFull) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) | (1ull << 46);
}
constexpr uint32_t kIdesc = (1u << 4)              // D: f32
                            | (2u << 7)            // A: tf32
                            | (2u << 10)           // B: tf32
                            | ((uint32_t)(TN >> 3) << 17)
                            | ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define TMEM_LD32(taddr, r)                                                                                     \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                       \
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                      \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                     \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),         \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),     \
                 "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),  \
                 "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),  \
                 "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                           \
               : "r"(taddr))

struct ResidualArgs {
  const unsigned char* a_img;   // n_mt x 16 KB
  const unsigned char* b_img;   // n_nt x 32 KB
  const float* y;
  float* S;                     // C x n (column-major n x C)
  uint64_t n;
  uint32_t C;
  uint32_t n_mt, n_nt;
};

__global__ void __launch_bounds__(kThreads, 1) residual_tc_kernel(ResidualArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* stage[2] = {smem, smem + STAGE};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);
  uint64_t* full = bars;           // [2]
  uint64_t* empty = bars + 2;      // [2]
  uint64_t* tfull = bars + 4;      // [2]
  uint64_t* tempty = bars + 6;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tiles = a.n_mt * a.n_nt;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const uint32_t s = it & 1, ph = (it >> 1) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        const uint32_t mt = t / a.n_nt, nt = t % a.n_nt;
        mbar_expect_tx(&full[s], STAGE);
        bulk_g2s(stage[s], a.a_img + (size_t)mt * A_IMG, A_IMG, &full[s]);
        bulk_g2s(stage[s] + A_IMG, a.b_img + (size_t)nt * B_IMG, B_IMG, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const uint32_t s = it & 1, ph = (it >> 1) & 1;
      mbar_wait(&tempty[s], ph ^ 1);
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const uint32_t d = tmem_base + s * TN;
        const unsigned char* A = stage[s];
        const unsigned char* B = stage[s] + A_IMG;
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t ahi = sdesc(A + ks * 256), alo = sdesc(A + A_HALF + ks * 256);
          const uint64_t bhi = sdesc(B + ks * 256), blo = sdesc(B + B_HALF + ks * 256);
          mma_tf32(d, alo, bhi, ks > 0 ? 1u : 0u);  // small terms first
          mma_tf32(d, ahi, blo, 1u);
          mma_tf32(d, ahi, bhi, 1u);
        }
        mma_commit(&empty[s]);
        mma_commit(&tfull[s]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: warps 2..9 -> TMEM lane quarter (warp % 4), column half
    const int q = warp & 3;
    const uint32_t cbeg = (uint32_t)((warp - 2) >> 2) * (TN / 2);
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const uint32_t s = it & 1, ph = (it >> 1) & 1;
      const uint32_t mt = t / a.n_nt, nt = t % a.n_nt;
      const uint64_t row = (uint64_t)mt * TM + q * 32 + lane;
      const bool row_ok = row < a.n;
      const float yi = row_ok ? a.y[row] : 0.f;
      const uint32_t col_first = nt * TN + cbeg;
      const bool full = col_first + TN / 2 <= a.C;
      float* p = a.S + (size_t)col_first * a.n + row;
      mbar_wait(&tfull[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + s * TN + cbeg;
#pragma unroll 1
      for (uint32_t c0 = 0; c0 < TN / 2; c0 += 32) {
        uint32_t r[32];
        TMEM_LD32(taddr + c0, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row_ok) {
          if (full) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float res = __uint_as_float(r[j]) - yi;
              __stcs(p, res * res);
              p += a.n;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float res = __uint_as_float(r[j]) - yi;
              if (col_first + c0 + j < a.C) __stcs(p, res * res);
              p += a.n;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[s]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

constexpr size_t kResidualSmem = 2 * STAGE + 1024 + 128 + 40 * 1024;  // ring + align + barriers; pad => 1 CTA/SM

}  // namespace

cudaError_t lms_residuals(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p, const float* thetas,
                          uint32_t C, float* S, cudaStream_t st) {
  const uint32_t n_mt = (uint32_t)((n + TM - 1) / TM), n_nt = (C + TN - 1) / TN;
  const size_t need = (size_t)n_mt * A_IMG + (size_t)n_nt * B_IMG;
  if (w.img_bytes < need) {
    if (w.img) cudaFree(w.img);
    w.img = nullptr;
    w.img_bytes = 0;
    cudaError_t e = cudaMalloc(&w.img, need);
    if (e != cudaSuccess) return e;
    w.img_bytes = need;
  }
  unsigned char* a_img = static_cast<unsigned char*>(w.img);
  unsigned char* b_img = a_img + (size_t)n_mt * A_IMG;
  pack_rows_kernel<<<n_mt, TM, 0, st>>>(X, n, p, TM, a_img);
  pack_rows_kernel<<<n_nt, TN, 0, st>>>(thetas, C, p, TN, b_img);
  cudaError_t e = cudaFuncSetAttribute(residual_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kResidualSmem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  ResidualArgs a{a_img, b_img, y, S, n, C, n_mt, n_nt};
  const uint32_t tiles = n_mt * n_nt;
  const int grid = (int)(tiles < (uint32_t)sms ? tiles : (uint32_t)sms);
  residual_tc_kernel<<<grid, kThreads, kResidualSmem, st>>>(a);
  return cudaGetLastError();
}

// LTS (NEXT row §8f-2): given m_j = the h-th smallest of column j of S,
// F_j = sum_{s < m_j} s + (h - #{s < m_j}) * m_j  (= the sum of the h smallest squared residuals,
// the rho/a,b form with every s = m_j equal to m_j).  One CTA per column (grid-stride), fp64
// accumulation, fixed-order block reduction.
__global__ void __launch_bounds__(256) lts_reduce_kernel(const float* __restrict__ S, uint64_t n, uint32_t C,
                                                         uint64_t h, const float* __restrict__ m,
                                                         double* __restrict__ out) {
  __shared__ double ws[8];
  __shared__ unsigned long long wc[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t j = blockIdx.x; j < C; j += gridDim.x) {
    const float mj = m[j];
    const float* col = S + (size_t)j * n;
    double acc = 0.0;
    unsigned long long cnt = 0;
    // 16-byte body (columns are 4-float aligned when n % 4 == 0; else scalar)
    const bool vec = ((reinterpret_cast<uintptr_t>(col) & 15) == 0);
    uint64_t i0 = 0;
    if (vec) {
      const float4* c4 = reinterpret_cast<const float4*>(col);
      const uint64_t nv = n / 4;
      for (uint64_t v = threadIdx.x; v < nv; v += blockDim.x) {
        const float4 q = __ldcs(c4 + v);
        unsigned c = 0;
        if (q.x < mj) { acc += (double)q.x; ++c; }
        if (q.y < mj) { acc += (double)q.y; ++c; }
        if (q.z < mj) { acc += (double)q.z; ++c; }
        if (q.w < mj) { acc += (double)q.w; ++c; }
        cnt += c;
      }
      i0 = nv * 4;
    }
    for (uint64_t i = i0 + threadIdx.x; i < n; i += blockDim.x) {
      const float v = col[i];
      if (v < mj) { acc += (double)v; ++cnt; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if (lane == 0) { ws[w] = acc; wc[w] = cnt; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0;
      unsigned long long c = 0;
      for (int q = 0; q < 8; ++q) { a += ws[q]; c += wc[q]; }
      out[j] = a + (double)(h - c) * (double)mj;
    }
    __syncthreads();
  }
}

cudaError_t lts_reduce(const float* S, uint64_t n, uint32_t C, uint64_t h, const float* m, double* out,
                       cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = sms * 8;
  if ((uint32_t)grid > C) grid = (int)C;
  lts_reduce_kernel<<<grid, 256, 0, st>>>(S, n, C, h, m, out);
  return cudaGetLastError();
}

cudaError_t batched_select(LmsWorkspace& w, const float* S, uint64_t n, uint32_t C, uint64_t k, float* out,
                           uint32_t max_iters, LmsReport* rep, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = sms * batched_blocks_per_sm();
  if ((uint32_t)grid > C) grid = (int)C;
  const uint64_t cap = n / 8 * 5 + 1;  // a column compacts once its bracket holds <= 5/8 of it
  const size_t scratch = (size_t)grid * 2 * cap * sizeof(float);
  const size_t need = scratch + 256;
  if (w.dev_bytes < need) {
    if (w.dev) cudaFree(w.dev);
    w.dev = nullptr;
    w.dev_bytes = 0;
    cudaError_t e = cudaMalloc(&w.dev, need);
    if (e != cudaSuccess) return e;
    w.dev_bytes = need;
  }
  if (!w.host) {
    cudaError_t e = cudaHostAlloc(&w.host, 256, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    w.host_bytes = 256;
  }
  unsigned char* base = static_cast<unsigned char*>(w.dev);
  unsigned* next_col = reinterpret_cast<unsigned*>(base + scratch);
  unsigned long long* stats = reinterpret_cast<unsigned long long*>(base + scratch + 64);
  cudaError_t e = cudaMemsetAsync(base + scratch, 0, 256, st);
  if (e != cudaSuccess) return e;
  BatchArgs a{S, n, C, k, out, reinterpret_cast<float*>(base), cap, next_col, stats, max_iters};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  e = launch_batched_select(a, grid, st);
  if (e != cudaSuccess) return e;
  cudaEventRecord(e1, st);
  e = cudaMemcpyAsync(w.host, stats, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const unsigned long long* h = static_cast<const unsigned long long*>(w.host);
  if (rep) {
    rep->passes = (uint32_t)h[0];
    rep->cp_iters = (uint32_t)(h[0] - C);
    rep->bytes = h[1];
    rep->nonfinite = h[3];
    rep->ms = ms;
  }
  if (h[2]) return cudaErrorNotSupported;  // safeguard tripped on some column
  return cudaSuccess;
}

void lms_free(LmsWorkspace& w) {
  if (w.S) cudaFree(w.S);
  if (w.dev) cudaFree(w.dev);
  if (w.img) cudaFree(w.img);
  if (w.host) cudaFreeHost(w.host);
  w = LmsWorkspace{};
}

}  // namespace cpsel
