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
//
// The default LMS/LTS path never stores S: fused_tc_kernel (below) runs the same product transposed
// and takes the selection's first pass in its epilogue.
#include <cstdint>
#include <cstring>
#include <vector>

#include "cpsel_kernels.h"
#include "cpsel_ptx.h"
#include "cpsel_lms.h"

namespace cpsel {
namespace {

// a start/end CUDA-event pair, destroyed on every return path
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  EventPair() {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  float ms() const {
    float v = 0.f;
    cudaEventElapsedTime(&v, a, b);
    return v;
  }
};

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

// extra (fold): column p carries extra_v[row] (X: y_i) or extra_c (Theta: -1), so the product is
// x_i . theta_j - y_i — the residual itself comes out of the tensor core (p <= 15)
__global__ void pack_rows_kernel(const float* __restrict__ src, uint64_t rows, uint32_t p, int tile_rows,
                                 unsigned char* __restrict__ img, int extra = 0, const float* extra_v = nullptr,
                                 float extra_c = 0.f) {
  const uint64_t tile = blockIdx.x;
  const int r = threadIdx.x;
  const uint64_t row = tile * tile_rows + r;
  const int half = tile_rows * KP * 4;
  unsigned char* base = img + tile * (uint64_t)(2 * half);
  // four consecutive k of one row are one 16-byte chunk of the core-matrix image: 16-byte stores
#pragma unroll
  for (int kq = 0; kq < KP; kq += 4) {
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k = kq + c;
      float v = (row < rows && k < (int)p) ? src[row * p + k] : 0.f;
      if (extra && k == (int)p && row < rows) v = extra_v ? extra_v[row] : extra_c;
      hi[c] = tf32_rna(v);
      lo[c] = tf32_rna(v - __uint_as_float(hi[c]));
    }
    *reinterpret_cast<uint4*>(base + core_off(r, kq)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(base + half + core_off(r, kq)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
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

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate,
                                         uint32_t idesc = kIdesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
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

// ------------------------------------------------------------------------------------------
// Fused residual pass (§8f-2 "fused GEMM-epilogue recompute"): the same 3xTF32 tcgen05 product,
// transposed — candidates on the TMEM lanes (A = Theta image, 128 candidates per tile), rows on
// the TMEM columns (B = X image, 256 rows per operand tile, issued as FS-row sub-tiles into
// kTStages TMEM accumulators) — so each epilogue thread owns ONE candidate column j and walks 32
// consecutive rows per tcgen05.ld.  An epilogue warp releases a sub-tile's accumulator (and its y)
// as soon as both are in registers, before the element work, so the MMA refills it while the
// warps compute.  Nothing of S is stored: per element s = (acc - y_i)^2 is counted against the
// column's two sample cuts (R23: #s <= t_lo), and the ones strictly between them are appended to
// the column's own buffer z_j (thread-private slots in shared memory; a thread holding kFlush
// writes them out itself behind one atomicAdd on the column cursor).  Work is cut into units
// (candidate tile, chunk of row tiles) so the per-column counters stay in registers for a whole
// unit and are flushed once per unit.  (NaN/Inf: the inputs are checked instead, lms_fused_check.)
//   MODE kFuseCuts : the statistics above (the init pass a1 + R23 cuts + a4 copy of every column)
//   MODE kFuseStore: s stored to S[slot[j]*n + row] for the columns with slot[j] >= 0 (fallback
//                    columns, and the parity hook: the S the fused statistics were taken on)
//   MODE kFuseLts  : sum_{s < m_j} s (fp64) and #{s < m_j} per column (LTS)
constexpr int kFuseCuts = 0, kFuseStore = 1, kFuseLts = 2;
constexpr int FN = 256;                    // rows per operand tile (the X image's 256-row tiles)
#ifndef CPSEL_LMS_FS
#define CPSEL_LMS_FS 128
#endif
constexpr int FS = CPSEL_LMS_FS;           // rows per sub-tile = TMEM columns per accumulator (128 or 256)
constexpr int kTStages = 512 / FS;         // TMEM accumulator stages (all 512 columns)
constexpr int kSubs = FN / FS;             // sub-tiles per operand tile
constexpr int kWR = FS / 4;                // rows per epilogue warp per sub-tile
constexpr int kChunks = kWR / 32;          // 32-row chunks (one tcgen05.ld each) per warp per sub-tile
constexpr int kFEpiWarps = 16;             // 4 per TMEM lane quarter, each on 32 of a sub-tile's 128 rows
constexpr int kFYWarp = 2 + kFEpiWarps;    // the warp that stages y for each accumulator stage
constexpr int kFStages = 2;                // operand (Theta + X tile) stages in shared memory
constexpr int kFThreads = 32 * (3 + kFEpiWarps);
constexpr int kRing = 48;                  // staging slots per epilogue thread (kFlush - 1 pending + 16 of a half chunk)
constexpr int kFlush = 32;                 // elements per flush (one thread's 128 bytes)
constexpr uint32_t kSlot = 4;              // a thread's slots are consecutive words ...
constexpr uint32_t kLaneStage = 4 * (kRing + 4);  // ... 16-byte aligned per thread (conflict-free LDS.128 quarter-warps)
constexpr int kFBarBytes = 256;            // mbarriers + the TMEM address slot
// M = 128 candidates, N = FS rows
constexpr uint32_t kIdescSub = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(FS >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

struct FusedArgs {
  const unsigned char* a_img;   // Theta: n_ct x 16 KB (128 candidates per tile)
  const unsigned char* b_img;   // X: n_rt x 32 KB (256 rows per tile)
  const float* y;               // y, padded with zeros to n_rt * 256
  uint64_t n;
  uint32_t C, n_rt, rt_per_unit, n_chunks;
  const uint32_t* ct_list;      // candidate tiles to run
  uint32_t n_ct_list;
  uint32_t b_ct_stride;         // 0: one X (and y) for all candidate tiles; else candidate tile ct reads
                                // its own row tiles ct * b_ct_stride + rt (per-tile sample rows)
  const float* cuts;            // kFuseCuts: 4 floats per column (t_lo, t_hi, t_mid, -)
  unsigned long long* le;       // kFuseCuts: #s <= t_lo per column      | kFuseLts: #s < m_j
  unsigned long long* cursor;   // kFuseCuts: elements of ]t_lo, t_hi[
  float* z;                     // kFuseCuts: column j's interior at z + j * zcap
  uint64_t zcap;
  const int* slot;              // kFuseStore
  float* S;                     // kFuseStore: slot-major columns of n
  const float* m;               // kFuseLts: per column threshold m_j
  double* sum;                  // kFuseLts: fp64 sum of s < m_j per (chunk, row quarter, column)
};

// s = (acc - y)^2 for two rows at once (FADD2/FMUL2: the same IEEE round-to-nearest results as
// the scalar residual kernel's FADD, FMUL)
__device__ __forceinline__ void resid2(uint32_t a0, uint32_t a1, unsigned long long y01, float& s0, float& s1) {
  unsigned long long acc = ((unsigned long long)a1 << 32) | a0, d, sq;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(acc), "l"(y01));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(sq) : "l"(d));
  s0 = __uint_as_float((uint32_t)sq);
  s1 = __uint_as_float((uint32_t)(sq >> 32));
}

// FOLD (y folded into the product, p <= 15): the accumulator already holds the residuals r — only
// the squares remain (one FMUL2 per two rows, the same IEEE round-to-nearest as FMUL)
template <bool FOLD>
__device__ __forceinline__ void resid2x(uint32_t a0, uint32_t a1, unsigned long long y01, float& s0, float& s1) {
  if (FOLD) {
    unsigned long long acc = ((unsigned long long)a1 << 32) | a0, sq;
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(sq) : "l"(acc));
    s0 = __uint_as_float((uint32_t)sq);
    s1 = __uint_as_float((uint32_t)(sq >> 32));
  } else {
    resid2(a0, a1, y01, s0, s1);
  }
}

// The per-element step of the fused cut pass (a1 + R23 + a4 on one residual).  Every s is >= 0 (or
// +Inf for a padded row), so float order is unsigned order of the bits: with d = bits(s) - lo1,
// lo1 = bits(t_lo) + 1, s <= t_lo iff d wraps (its top bit is set: #s <= t_lo += d >> 31) and
// t_lo < s < t_hi iff d < w, w = bits(t_hi) - lo1 (unsigned).  Interior s are appended to the
// thread's staging slots at shared address ta.  5 instructions per element after the residual.
__device__ __forceinline__ void cut_elem(float s, uint32_t lo1, uint32_t w, uint32_t& le, uint32_t& ta) {
  asm volatile(
      "{\n\t.reg .pred in;\n\t.reg .u32 d, c;\n\t"
      "sub.u32 d, %2, %3;\n\t"
      "shr.u32 c, d, 31;\n\t"
      "add.u32 %0, %0, c;\n\t"
      "setp.lt.u32 in, d, %4;\n\t"
      "@in st.shared.f32 [%1], %5;\n\t"
      "@in add.u32 %1, %1, %6;\n\t}"
      : "+r"(le), "+r"(ta)
      : "r"(__float_as_uint(s)), "r"(lo1), "r"(w), "f"(s), "n"(kSlot)
      : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// Write `cnt` staged elements of this thread (its slots from base_sa on) to zc[0..cnt) within room.
__device__ __forceinline__ void stage_out(uint32_t base_sa, uint32_t cnt, float* zc, uint64_t room) {
  for (uint32_t o = 0; o < cnt; o += 4) {
    const float4 q = lds128(base_sa + o * kSlot);
    const float qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (o + i < cnt && o + i < room) zc[o + i] = qv[i];
  }
}

// The 16 elements r[h*16 .. h*16+15] of a chunk (rows beyond nvalid enter as +Inf), then the flush
// of every thread holding >= kFlush staged elements (at most kFlush - 1 + 16 < kRing pending): all
// such threads at once, each writing ITS first kFlush to its column's copy (16-byte shared loads of
// its own slots, no cross-lane traffic: one pass of the warp however many lanes flush) and moving
// the rest to the front of its slots.
template <bool FULL, bool FOLD>
__device__ __forceinline__ void cut_half(const uint32_t* r, int h, const ulonglong2* yv, int nvalid, uint32_t lo1,
                                         uint32_t wcut, uint32_t& le, uint32_t& le2, uint32_t& ta,
                                         uint32_t base_sa, const FusedArgs& a, uint32_t j, float* zcol) {
#pragma unroll
  for (int jj = 0; jj < 16; jj += 2) {
    const int i = h * 16 + jj;
    const unsigned long long y01 = (i & 2) ? yv[i >> 2].y : yv[i >> 2].x;
    float s0, s1;
    resid2x<FOLD>(r[i], r[i + 1], y01, s0, s1);
    if (FULL) {
      cut_elem(s0, lo1, wcut, le, ta);
      cut_elem(s1, lo1, wcut, le2, ta);  // two counters: half the dependent chain
    } else {
      cut_elem(i < nvalid ? s0 : __int_as_float(0x7f800000), lo1, wcut, le, ta);
      cut_elem(i + 1 < nvalid ? s1 : __int_as_float(0x7f800000), lo1, wcut, le, ta);
    }
  }
  const uint32_t cnt = (ta - base_sa) / kSlot;
  if (__any_sync(0xffffffffu, cnt >= kFlush)) {
    if (cnt >= kFlush) {
      const unsigned long long pos = atomicAdd(a.cursor + j, (unsigned long long)kFlush);
      float* dst = zcol + pos;
      if (pos + kFlush <= a.zcap) {
#pragma unroll
        for (int v = 0; v < kFlush / 4; ++v) {
          const float4 q = lds128(base_sa + v * 16);
          dst[4 * v] = q.x;
          dst[4 * v + 1] = q.y;
          dst[4 * v + 2] = q.z;
          dst[4 * v + 3] = q.w;
        }
      } else {
        stage_out(base_sa, kFlush, dst, pos < a.zcap ? a.zcap - pos : 0);
      }
#pragma unroll
      for (int v = 0; v < (kRing - kFlush) / 4; ++v)  // the rest (<= 15) to the front
        if ((uint32_t)(kFlush + 4 * v) < cnt) sts128(base_sa + v * 16, lds128(base_sa + kFlush * kSlot + v * 16));
      ta -= kFlush * kSlot;
    }
  }
}

template <int MODE, bool FOLD>
__global__ void __launch_bounds__(kFThreads, 1) fused_tc_kernel(FusedArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // kFStages operand stages (the loads run up to kFStages-1 tiles ahead); kTStages TMEM
  // accumulators of one 128-row sub-tile each (the epilogue warps may drift up to kTStages-1
  // sub-tiles apart before the MMA has to wait for the slowest)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kFStages * STAGE);
  uint64_t* full = bars;                    // [kFStages]
  uint64_t* empty = bars + kFStages;        // [kFStages]
  uint64_t* tfull = bars + 2 * kFStages;    // [kTStages]
  uint64_t* tempty = tfull + kTStages;      // [kTStages]
  uint64_t* yfull = tempty + kTStages;      // [kTStages]: y of the sub-tile in accumulator stage s is in ybuf[s]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(yfull + kTStages);
  float* ybuf = reinterpret_cast<float*>(smem + kFStages * STAGE + kFBarBytes);  // [kTStages][FS]
  const uint32_t ring_sa = smem_u32(smem + kFStages * STAGE + kFBarBytes + kTStages * FS * 4);  // 512 threads x kLaneStage B
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t units = a.n_ct_list * a.n_chunks;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kFStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kTStages; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kFEpiWarps);
      mbar_init(&yfull[i], 1);
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

  if (!FOLD && warp == kFYWarp) {
    // ---------------- y stager: the sub-tile's 128 y values into ybuf[s] once the epilogue released
    //                  accumulator stage s (the epilogue reads them as shared-memory broadcasts).
    //                  A plain warp copy (512 B per sub-tile; 16 B per lane), released to the
    //                  epilogue by an mbarrier arrive: ordinary generic-proxy accesses ordered by
    //                  the stage barriers (a bulk copy here was an async-proxy write racecheck
    //                  cannot see ordered behind the epilogue's reads)
    uint32_t it = 0;
    for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
      const uint32_t ct = a.ct_list[u % a.n_ct_list], ch = u / a.n_ct_list;
      const uint32_t r0 = ch * a.rt_per_unit, r1 = min(a.n_rt, r0 + a.rt_per_unit);
      for (uint32_t rt = r0; rt < r1; ++rt) {
        const float4* src = reinterpret_cast<const float4*>(a.y + ((size_t)ct * a.b_ct_stride + rt) * FN);
        const float4 yh[2] = {__ldg(src + lane), __ldg(src + 32 + lane)};  // loads ahead of the waits
#pragma unroll
        for (int h = 0; h < kSubs; ++h, ++it) {
          const uint32_t s = it % kTStages, ph = (it / kTStages) & 1;
          mbar_wait_sleep(&tempty[s], ph ^ 1);
#pragma unroll
          for (int c = 0; c < FS / 128; ++c) reinterpret_cast<float4*>(ybuf + s * FS)[c * 32 + lane] = yh[h * (FS / 128) + c];
          __syncwarp();
          if (lane == 0) mbar_arrive(&yfull[s]);
        }
      }
    }
  } else if (warp == 0) {
    // ---------------- producer: Theta tile (A) + X tile (B) per stage
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
        const uint32_t ct = a.ct_list[u % a.n_ct_list], ch = u / a.n_ct_list;
        const uint32_t r0 = ch * a.rt_per_unit, r1 = min(a.n_rt, r0 + a.rt_per_unit);
        for (uint32_t rt = r0; rt < r1; ++rt, ++it) {
          const uint32_t s = it % kFStages, ph = (it / kFStages) & 1;
          mbar_wait_sleep(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], STAGE);
          bulk_g2s(smem + s * STAGE, a.a_img + (size_t)ct * A_IMG, A_IMG, &full[s]);
          bulk_g2s(smem + s * STAGE + A_IMG, a.b_img + ((size_t)ct * a.b_ct_stride + rt) * B_IMG, B_IMG, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: D[j][i] = theta_j . x_i, the residual kernel's three products, per
    //                  128-row half of the operand tile (rows 128h.. of the hi / lo images start
    //                  8 KB in: 16 core-matrix row groups of 512 B)
    uint32_t it = 0, ot = 0;
    for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
      const uint32_t ch = u / a.n_ct_list;
      const uint32_t r0 = ch * a.rt_per_unit, r1 = min(a.n_rt, r0 + a.rt_per_unit);
      for (uint32_t rt = r0; rt < r1; ++rt, ++ot) {
        const uint32_t ss = ot % kFStages, sph = (ot / kFStages) & 1;  // operand stage
        mbar_wait_sleep(&full[ss], sph);
        const unsigned char* A = smem + ss * STAGE;
        const unsigned char* B = smem + ss * STAGE + A_IMG;
#pragma unroll
        for (int h = 0; h < kSubs; ++h, ++it) {
          const uint32_t s = it % kTStages, ph = (it / kTStages) & 1;  // TMEM stage
          mbar_wait_sleep(&tempty[s], ph ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
            const uint32_t d = tmem_base + s * FS;
            for (int ks = 0; ks < 2; ++ks) {
              const uint64_t ahi = sdesc(A + ks * 256), alo = sdesc(A + A_HALF + ks * 256);
              const uint64_t bhi = sdesc(B + h * (FS * 64) + ks * 256);
              const uint64_t blo = sdesc(B + B_HALF + h * (FS * 64) + ks * 256);
              mma_tf32(d, ahi, blo, ks > 0 ? 1u : 0u, kIdescSub);  // x_lo * theta_hi (small terms first)
              mma_tf32(d, alo, bhi, 1u, kIdescSub);                // x_hi * theta_lo
              mma_tf32(d, ahi, bhi, 1u, kIdescSub);
            }
            mma_commit(&tfull[s]);
          }
          __syncwarp();
        }
        if (lane == 0) mma_commit(&empty[ss]);
        __syncwarp();
      }
    }
  } else if (warp >= 2 && warp < 2 + kFEpiWarps) {
    // ---------------- epilogue: warps 2..17 -> TMEM lane quarter (warp % 4) = 32 candidates,
    //                  row quarter rq: rows [rq*32, rq*32+32) of each 128-row sub-tile
    const int q = warp & 3;
    const int rq = (warp - 2) >> 2;
    const int e = threadIdx.x - 64;  // 0..511: this thread's staging slots
    const uint32_t base_sa = ring_sa + kLaneStage * (uint32_t)e;
    uint32_t it = 0;
    for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
      const uint32_t ct = a.ct_list[u % a.n_ct_list], ch = u / a.n_ct_list;
      const uint32_t r0 = ch * a.rt_per_unit, r1 = min(a.n_rt, r0 + a.rt_per_unit);
      const uint32_t j = ct * TM + q * 32 + lane;
      const bool col_ok = j < a.C;
      float mj = 0.f;
      uint32_t lo1 = 0x80000000u, wcut = 0u;  // a column past C: copies nothing (its counts are dropped)
      int slot = -1;
      if (MODE == kFuseCuts && col_ok) {
        const uint32_t bl = __float_as_uint(a.cuts[4 * (size_t)j]), bh = __float_as_uint(a.cuts[4 * (size_t)j + 1]);
        lo1 = bl + 1u;
        wcut = bh - lo1;  // the cuts are >= +0 and t_lo < t_hi
      }
      if (MODE == kFuseStore && col_ok) slot = a.slot[j];
      if (MODE == kFuseLts && col_ok) mj = a.m[j];
      uint32_t le = 0, le2 = 0;
      double lsum = 0.0;
      uint32_t ta = base_sa;  // next free staging slot
      float* zcol = a.z + (size_t)(col_ok ? j : 0) * a.zcap;
      // rows left in x from this unit's first row of this warp (only the last row tile is ragged)
      const uint64_t urow = (uint64_t)r0 * FN + rq * kWR;
      const uint64_t ur_left = a.n > urow ? a.n - urow : 0;
      for (uint32_t cc = 0; cc < kSubs * kChunks * (r1 - r0); ++cc) {
        const uint32_t c = cc % kChunks;  // chunk of this warp's rows in the sub-tile
        const uint32_t s = it % kTStages, ph = (it / kTStages) & 1;
        const uint64_t roff = (uint64_t)(cc / kChunks) * FS + c * 32;  // this chunk starts at urow + roff
        const int nvalid = ur_left >= roff + 32 ? 32 : (ur_left > roff ? (int)(ur_left - roff) : 0);
        if (c == 0) {
          mbar_wait_sleep(&tfull[s], ph);
          if (!FOLD) mbar_wait_sleep(&yfull[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + s * FS + rq * kWR + c * 32;
        const uint32_t ys_sa = smem_u32(ybuf + s * FS + rq * kWR + c * 32);
        uint32_t r[32];
        TMEM_LD32(taddr, r);
        ulonglong2 yv[8];
        if (!FOLD) {
#pragma unroll
          for (int v = 0; v < 8; ++v)  // shared-memory broadcast (LDS.128)
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(yv[v].x), "=l"(yv[v].y) : "r"(ys_sa + v * 16));
        } else {
#pragma unroll
          for (int v = 0; v < 8; ++v) yv[v].x = yv[v].y = 0ull;  // unused
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c == kChunks - 1) {
          // the sub-tile's last accumulator columns and y are in registers: release the stage
          // before the element work
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[s]);
          ++it;
        }
        if (MODE == kFuseCuts) {
          if (nvalid == 32) {
            cut_half<true, FOLD>(r, 0, yv, 32, lo1, wcut, le, le2, ta, base_sa, a, j, zcol);
            cut_half<true, FOLD>(r, 1, yv, 32, lo1, wcut, le, le2, ta, base_sa, a, j, zcol);
          } else {  // the ragged end of x: padded rows enter as +Inf
            cut_half<false, FOLD>(r, 0, yv, nvalid, lo1, wcut, le, le2, ta, base_sa, a, j, zcol);
            cut_half<false, FOLD>(r, 1, yv, nvalid, lo1, wcut, le, le2, ta, base_sa, a, j, zcol);
          }
        } else if (MODE == kFuseStore) {
          // the warp's 32 columns x 32 rows transposed through its staging slots (row stride 33
          // words: conflict-free both ways), so every store writes 32 consecutive rows (128 bytes)
          // of one column instead of 16 bytes of 32 columns
          if (__any_sync(0xffffffffu, slot >= 0)) {
            const uint32_t tb = ring_sa + kLaneStage * 32u * (uint32_t)(warp - 2);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const unsigned long long y01 = (i & 2) ? yv[i >> 2].y : yv[i >> 2].x;
              float s0, s1;
              resid2x<FOLD>(r[i], r[i + 1], y01, s0, s1);
              asm volatile("st.shared.f32 [%0], %1;" ::"r"(tb + (uint32_t)(i * 33 + lane) * 4u), "f"(s0) : "memory");
              asm volatile("st.shared.f32 [%0], %1;" ::"r"(tb + (uint32_t)((i + 1) * 33 + lane) * 4u), "f"(s1) : "memory");
            }
            __syncwarp();
            const uint64_t rowc = urow + roff;
#pragma unroll 4
            for (int cc2 = 0; cc2 < 32; ++cc2) {
              const int sl = __shfl_sync(0xffffffffu, slot, cc2);
              float v;
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(tb + (uint32_t)(lane * 33 + cc2) * 4u));
              if (sl >= 0 && lane < nvalid) __stcs(a.S + (size_t)sl * a.n + rowc + lane, v);
            }
            __syncwarp();  // the slots are rewritten by the next chunk
          }
        } else {
          unsigned c = 0;
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const unsigned long long y01 = (i & 2) ? yv[i >> 2].y : yv[i >> 2].x;
            float s0, s1;
            resid2x<FOLD>(r[i], r[i + 1], y01, s0, s1);
            if (i < nvalid && s0 < mj) { lsum += (double)s0; ++c; }
            if (i + 1 < nvalid && s1 < mj) { lsum += (double)s1; ++c; }
          }
          le += c;
        }
      }
      // end of unit: flush this column's counters and the rest of its staging slots
      if (MODE == kFuseCuts) {
        const uint32_t cnt = (ta - base_sa) / kSlot;
        if (col_ok) {
          atomicAdd(a.le + j, (unsigned long long)le + le2);
          if (cnt) {
            const unsigned long long pos = atomicAdd(a.cursor + j, (unsigned long long)cnt);
            stage_out(base_sa, cnt, zcol + pos, pos < a.zcap ? a.zcap - pos : 0);
          }
        }
      } else if (MODE == kFuseLts && col_ok) {
        atomicAdd(a.le + j, (unsigned long long)le);
        a.sum[((size_t)ch * 4 + rq) * a.C + j] = lsum;  // fixed-order reduction afterwards
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

constexpr size_t kFusedSmem = kFStages * STAGE + 1024 + kFBarBytes + kTStages * FS * 4 + (size_t)kFEpiWarps * 32 * kLaneStage;  // ring, barriers, y, staging

__global__ void pad_copy_kernel(const float* __restrict__ src, uint64_t n, float* __restrict__ dst, uint64_t n_pad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = i < n ? src[i] : 0.f;
}

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

// Scratch (per-CTA ping-pong buffers) + the counter block: next_col @0, stats[4] @64, fail_count @96.
static cudaError_t run_batched(LmsWorkspace& w, BatchArgs a, LmsReport* rep, uint32_t* fail_count,
                               cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = sms * batched_blocks_per_sm();
  if ((uint32_t)grid > a.C) grid = (int)a.C;
  const uint64_t cap = a.n / 8 * 5 + 1;  // a column compacts once its bracket holds <= 5/8 of it
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
  a.scratch = reinterpret_cast<float*>(base);
  a.cap = cap;
  a.next_col = reinterpret_cast<unsigned*>(base + scratch);
  a.stats = reinterpret_cast<unsigned long long*>(base + scratch + 64);
  if (a.f_le) a.fail_count = reinterpret_cast<unsigned*>(base + scratch + 96);
  cudaError_t e = cudaMemsetAsync(base + scratch, 0, 256, st);
  if (e != cudaSuccess) return e;
  EventPair ev;
  cudaEventRecord(ev.a, st);
  e = launch_batched_select(a, grid, st);
  if (e != cudaSuccess) return e;
  cudaEventRecord(ev.b, st);
  e = cudaMemcpyAsync(w.host, base + scratch + 64, 40, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  const float ms = ev.ms();
  const unsigned long long* h = static_cast<const unsigned long long*>(w.host);
  if (rep) {
    rep->passes += (uint32_t)h[0];
    rep->cp_iters += (uint32_t)(h[0] - a.C);
    rep->bytes += h[1];
    rep->nonfinite += h[3];
    rep->ms += ms;
  }
  if (fail_count) *fail_count = (uint32_t)(h[4] & 0xffffffffull);
  if (h[2]) return cudaErrorNotSupported;  // safeguard tripped on some column
  return cudaSuccess;
}

cudaError_t batched_select(LmsWorkspace& w, const float* S, uint64_t n, uint32_t C, uint64_t k, float* out,
                           uint32_t max_iters, LmsReport* rep, cudaStream_t st) {
  BatchArgs a{S, n, C, k, out, nullptr, 0, nullptr, nullptr, max_iters};
  if (rep) *rep = LmsReport{};
  return run_batched(w, a, rep, nullptr, st);
}

// ------------------------------------------------------------------------------------------
// Fused path.  Geometry: candidate tiles of 128 (A = Theta), row tiles of 256 (B = X), units of
// kRtPerUnit row tiles x one candidate tile.
namespace {
constexpr uint32_t kRtPerUnit = 16;

struct FusedGeom {
  uint32_t n_ct, n_rt, n_chunks, rt_per_unit = kRtPerUnit, b_ct_stride = 0;
  unsigned char *a_img, *b_img;
  float* y_pad;
  bool fold = false;  // y folded into the images (column p): the product is the residual (p < 16)
};

__global__ void slot_map_kernel(int* slot, uint32_t C, const unsigned* list, uint32_t nlist) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < C; j += gridDim.x * blockDim.x) slot[j] = -1;
  __syncthreads();  // (one CTA: launched with grid 1)
  for (uint32_t i = threadIdx.x; i < nlist; i += blockDim.x) slot[list ? list[i] : i] = (int)i;
}

__global__ void lts_finish_kernel(const double* part, uint32_t nparts, uint32_t C, const unsigned long long* cnt,
                                  uint64_t h, const float* m, double* out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < C; j += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (uint32_t q = 0; q < nparts; ++q) acc += part[(size_t)q * C + j];  // fixed order
    out[j] = acc + (double)(h - cnt[j]) * (double)m[j];
  }
}

cudaError_t ensure_buf(void** p, size_t* have, size_t need) {
  if (*have >= need) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(p, need);
  if (e == cudaSuccess) *have = need;
  return e;
}

cudaError_t fused_prepare(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p,
                          const float* thetas, uint32_t C, FusedGeom& g, cudaStream_t st) {
  g.n_ct = (C + TM - 1) / TM;
  g.n_rt = (uint32_t)((n + FN - 1) / FN);
  g.n_chunks = (g.n_rt + kRtPerUnit - 1) / kRtPerUnit;
  const size_t need = (size_t)g.n_ct * A_IMG + (size_t)g.n_rt * B_IMG + (size_t)g.n_rt * FN * sizeof(float);
  cudaError_t e = ensure_buf(&w.fimg, &w.fimg_bytes, need);
  if (e != cudaSuccess) return e;
  g.a_img = static_cast<unsigned char*>(w.fimg);
  g.b_img = g.a_img + (size_t)g.n_ct * A_IMG;
  g.y_pad = reinterpret_cast<float*>(g.b_img + (size_t)g.n_rt * B_IMG);
  g.fold = p < (uint32_t)KP;
  if (g.fold) {  // r = [x_i, y_i] . [theta_j, -1]: the residual comes out of the tensor core
    pack_rows_kernel<<<g.n_ct, TM, 0, st>>>(thetas, C, p, TM, g.a_img, 1, nullptr, -1.f);
    pack_rows_kernel<<<g.n_rt, FN, 0, st>>>(X, n, p, FN, g.b_img, 1, y, 0.f);
  } else {
    pack_rows_kernel<<<g.n_ct, TM, 0, st>>>(thetas, C, p, TM, g.a_img);
    pack_rows_kernel<<<g.n_rt, FN, 0, st>>>(X, n, p, FN, g.b_img);
    pad_copy_kernel<<<512, 256, 0, st>>>(y, n, g.y_pad, (uint64_t)g.n_rt * FN);
  }
  return cudaGetLastError();
}

template <int MODE, bool FOLD>
cudaError_t fused_launch_t(const FusedGeom& g, FusedArgs a, uint32_t n_ct_list, cudaStream_t st) {
  a.a_img = g.a_img;
  a.b_img = g.b_img;
  a.y = g.y_pad;
  a.n_rt = g.n_rt;
  a.rt_per_unit = g.rt_per_unit;
  a.n_chunks = g.n_chunks;
  a.b_ct_stride = g.b_ct_stride;
  a.n_ct_list = n_ct_list;
  cudaError_t e = cudaFuncSetAttribute(fused_tc_kernel<MODE, FOLD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kFusedSmem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t units = n_ct_list * g.n_chunks;
  const int grid = (int)(units < (uint32_t)sms ? units : (uint32_t)sms);
  fused_tc_kernel<MODE, FOLD><<<grid, kFThreads, kFusedSmem, st>>>(a);
  return cudaGetLastError();
}
template <int MODE>
cudaError_t fused_launch(const FusedGeom& g, FusedArgs a, uint32_t n_ct_list, cudaStream_t st) {
  return g.fold ? fused_launch_t<MODE, true>(g, a, n_ct_list, st) : fused_launch_t<MODE, false>(g, a, n_ct_list, st);
}

// per-column arrays in w.fcol
struct FusedCols {
  float* cuts;                 // 4C
  unsigned long long* le;      // C
  unsigned long long* cursor;  // C
  int* slot;                   // C
  unsigned* fail_list;         // C
  unsigned* ct_list;           // n_ct
  double* part;                // LTS partials (2 n_chunks x C)
};

cudaError_t fused_cols(LmsWorkspace& w, uint32_t C, const FusedGeom& g, bool lts, FusedCols& c) {
  const size_t fixed = (size_t)C * (16 + 8 + 8 + 4 + 4 + 4) + (size_t)g.n_ct * 4 + 256;
  const size_t part = lts ? (size_t)4 * g.n_chunks * C * sizeof(double) : 0;
  cudaError_t e = ensure_buf(&w.fcol, &w.fcol_bytes, fixed + part);
  if (e != cudaSuccess) return e;
  unsigned char* b = static_cast<unsigned char*>(w.fcol);
  c.part = reinterpret_cast<double*>(b);  // 8-byte aligned first
  b += part;
  c.le = reinterpret_cast<unsigned long long*>(b); b += (size_t)C * 8;
  c.cursor = reinterpret_cast<unsigned long long*>(b); b += (size_t)C * 8;
  c.cuts = reinterpret_cast<float*>(b); b += (size_t)C * 16;
  c.slot = reinterpret_cast<int*>(b); b += (size_t)C * 4;
  c.fail_list = reinterpret_cast<unsigned*>(b); b += (size_t)C * 4;
  c.ct_list = reinterpret_cast<unsigned*>(b);
  return cudaSuccess;
}

__global__ void iota_kernel(unsigned* v, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}

// R23 cuts of every column: the residuals of kLmsSamples evenly strided rows, computed by the fused
// kernel in store mode (the same arithmetic: exactly elements of S), then the per-column cut search.
// Each candidate tile draws its own rows (stride n/ms, a phase of its own): one shared row set would
// make the sample error common to all columns, and near-identical candidates (close theta_j) would
// then miss their cut window together.
constexpr uint32_t kLmsSamples = 16384;
__global__ void gather_sample_kernel(const float* __restrict__ X, const float* __restrict__ y, uint64_t n,
                                     uint32_t p, uint32_t ms, float* __restrict__ Xs, float* __restrict__ ys) {
  const uint32_t ct = blockIdx.y;
  const uint64_t stride = n / ms;
  const uint64_t phase = ((uint64_t)ct * 2654435761ull) % stride;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ms; i += gridDim.x * blockDim.x) {
    const uint64_t row = ((uint64_t)i * n) / ms + phase;  // < n: i*n/ms + stride - 1 < n
    float* xo = Xs + ((size_t)ct * ms + i) * p;
    for (uint32_t l = 0; l < p; ++l) xo[l] = X[row * p + l];
    ys[(size_t)ct * ms + i] = y[row];
  }
}

// The same rows packed straight into the fold image (X with y as column p), no gathered copy: tile t
// of candidate tile ct = t / (ms / FN) holds sample rows (i * n) / ms + phase(ct) of X.
__global__ void pack_sample_fold_kernel(const float* __restrict__ X, const float* __restrict__ y, uint64_t n,
                                        uint32_t p, uint32_t ms, unsigned char* __restrict__ img) {
  const uint32_t tiles_per_ct = ms / FN;
  const uint64_t tile = blockIdx.x;
  const uint32_t ct = (uint32_t)(tile / tiles_per_ct);
  const uint32_t i = (uint32_t)(tile % tiles_per_ct) * FN + threadIdx.x;  // sample index within ct
  const uint64_t stride = n / ms;
  const uint64_t phase = ((uint64_t)ct * 2654435761ull) % stride;
  const uint64_t row = ((uint64_t)i * n) / ms + phase;  // < n (as gather_sample_kernel)
  const int half = FN * KP * 4;
  unsigned char* base = img + tile * (uint64_t)(2 * half);
  const int r = threadIdx.x;
#pragma unroll
  for (int kq = 0; kq < KP; kq += 4) {
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k = kq + c;
      float v = k < (int)p ? X[row * p + k] : 0.f;
      if (k == (int)p) v = y[row];
      hi[c] = tf32_rna(v);
      lo[c] = tf32_rna(v - __uint_as_float(hi[c]));
    }
    *reinterpret_cast<uint4*>(base + core_off(r, kq)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(base + half + core_off(r, kq)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

cudaError_t fused_sample_cuts(LmsWorkspace& w, const FusedGeom& g, const float* X, const float* y, uint64_t n,
                              uint32_t p, uint32_t C, uint64_t k, const FusedCols& c, cudaStream_t st) {
  const uint32_t ms = kLmsSamples;
  FusedGeom gs;
  gs.n_ct = g.n_ct;
  gs.n_rt = ms / FN;
  gs.rt_per_unit = 1;
  gs.n_chunks = gs.n_rt;
  gs.b_ct_stride = gs.n_rt;
  const size_t ss_bytes = (size_t)C * ms * sizeof(float);
  const size_t img_bytes = (size_t)gs.n_ct * gs.n_rt * B_IMG;
  const size_t need = ss_bytes + img_bytes + (size_t)gs.n_ct * ms * (p + 1) * sizeof(float);
  cudaError_t e = ensure_buf(&w.fsamp, &w.fsamp_bytes, need);
  if (e != cudaSuccess) return e;
  unsigned char* b = static_cast<unsigned char*>(w.fsamp);
  float* Ss = reinterpret_cast<float*>(b);
  gs.b_img = b + ss_bytes;
  float* ys = reinterpret_cast<float*>(gs.b_img + img_bytes);
  float* Xs = ys + (size_t)gs.n_ct * ms;
  gs.y_pad = ys;  // ms is a multiple of the row tile: no padding
  gs.a_img = g.a_img;
  gs.fold = g.fold;
  if (gs.fold) {  // y is column p of the image: the strided rows packed directly
    pack_sample_fold_kernel<<<gs.n_ct * gs.n_rt, FN, 0, st>>>(X, y, n, p, ms, gs.b_img);
  } else {
    gather_sample_kernel<<<dim3(ms / 256, gs.n_ct), 256, 0, st>>>(X, y, n, p, ms, Xs, ys);
    pack_rows_kernel<<<gs.n_ct * gs.n_rt, FN, 0, st>>>(Xs, (uint64_t)gs.n_ct * ms, p, FN, gs.b_img);
  }
  slot_map_kernel<<<1, 1024, 0, st>>>(c.slot, C, nullptr, C);
  FusedArgs a{};
  a.n = ms; a.C = C; a.ct_list = c.ct_list; a.slot = c.slot; a.S = Ss;
  if ((e = fused_launch<kFuseStore>(gs, a, gs.n_ct, st)) != cudaSuccess) return e;
  return launch_lms_cuts(Ss, ms, n, C, k, c.cuts, st);
}
}  // namespace

// Input check of the fused path: the fused pass does not test its residuals for NaN/Inf, so the
// inputs are checked instead — every s = (x.theta - y)^2 is finite when X, y, Theta are finite and
// B = p max|X| max|theta| + max|y| < 2^60 (|r| <= sum_l |x_l||theta_l| + |y| <= B, times (1 + 2^-20)
// for the 3xTF32 split and fp32 accumulation, so s < 2^121 < FLT_MAX).  One flat, 16-byte-load pass
// over each array (the per-coordinate maxima of round 1 cost a strided walk: 48 us at configs[4]).
// out: [0] non-finite count, [1] max|X|, [2] max|theta|, [3] max|y| (float bits; all values >= 0,
// so unsigned order = float order).
__device__ __forceinline__ void check_span(const float* __restrict__ a, uint64_t m, unsigned& bad, float& mx) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x, t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t mis = (reinterpret_cast<uintptr_t>(a) / 4) & 3;
  uint64_t head = mis ? 4 - mis : 0;
  if (head > m) head = m;
  const float4* a4 = reinterpret_cast<const float4*>(a + head);
  const uint64_t nv = (m - head) / 4;
  for (uint64_t i = t; i < nv; i += stride) {
    const float4 q = __ldg(a4 + i);  // (cached: the pack reads X right after)
    const float v[4] = {fabsf(q.x), fabsf(q.y), fabsf(q.z), fabsf(q.w)};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      bad += !(v[c] <= 3.4028235e38f);
      mx = fmaxf(mx, v[c]);
    }
  }
  const uint64_t tail0 = head + nv * 4;
  if (t < head) {
    const float v = fabsf(a[t]);
    bad += !(v <= 3.4028235e38f);
    mx = fmaxf(mx, v);
  }
  if (t < m - tail0) {
    const float v = fabsf(a[tail0 + t]);
    bad += !(v <= 3.4028235e38f);
    mx = fmaxf(mx, v);
  }
}
__global__ void lms_check_kernel(const float* __restrict__ X, const float* __restrict__ y,
                                 const float* __restrict__ th, uint64_t n, uint32_t p, uint32_t C,
                                 unsigned* __restrict__ out) {
  unsigned bad = 0;
  float mX = 0.f, mT = 0.f, mY = 0.f;
  check_span(X, n * p, bad, mX);
  check_span(th, (uint64_t)C * p, bad, mT);
  check_span(y, n, bad, mY);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    mX = fmaxf(mX, __shfl_xor_sync(0xffffffffu, mX, o));
    mT = fmaxf(mT, __shfl_xor_sync(0xffffffffu, mT, o));
    mY = fmaxf(mY, __shfl_xor_sync(0xffffffffu, mY, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(out, bad);
    atomicMax(out + 1, __float_as_uint(mX));
    atomicMax(out + 2, __float_as_uint(mT));
    atomicMax(out + 3, __float_as_uint(mY));
  }
}

int lms_fused_check(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p, const float* thetas,
                    uint32_t C, cudaStream_t st, cudaError_t* err) {
  *err = ensure_buf(&w.fcol, &w.fcol_bytes, 256);
  if (*err != cudaSuccess) return -1;
  if (!w.host) {
    *err = cudaHostAlloc(&w.host, 256, cudaHostAllocDefault);
    if (*err != cudaSuccess) return -1;
    w.host_bytes = 256;
  }
  unsigned* d = static_cast<unsigned*>(w.fcol);
  if ((*err = cudaMemsetAsync(d, 0, 256, st)) != cudaSuccess) return -1;
  lms_check_kernel<<<296 * 4, 256, 0, st>>>(X, y, thetas, n, p, C, d);
  if ((*err = cudaMemcpyAsync(w.host, d, 16, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return -1;
  if ((*err = cudaStreamSynchronize(st)) != cudaSuccess) return -1;
  const unsigned* h = static_cast<const unsigned*>(w.host);
  if (h[0]) return 1;
  float mX, mT, mY;
  memcpy(&mX, h + 1, 4);
  memcpy(&mT, h + 2, 4);
  memcpy(&mY, h + 3, 4);
  const double B = (double)p * (double)mX * (double)mT + (double)mY;
  return B < 1152921504606846976.0 /* 2^60 */ ? 0 : 2;
}

cudaError_t lms_fused_residuals(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p,
                                const float* thetas, uint32_t C, float* S, cudaStream_t st) {
  FusedGeom g;
  cudaError_t e = fused_prepare(w, X, y, n, p, thetas, C, g, st);
  if (e != cudaSuccess) return e;
  FusedCols c;
  if ((e = fused_cols(w, C, g, false, c)) != cudaSuccess) return e;
  slot_map_kernel<<<1, 1024, 0, st>>>(c.slot, C, nullptr, C);
  iota_kernel<<<1, 256, 0, st>>>(c.ct_list, g.n_ct);
  FusedArgs a{};
  a.n = n; a.C = C; a.ct_list = c.ct_list; a.slot = c.slot; a.S = S;
  return fused_launch<kFuseStore>(g, a, g.n_ct, st);
}

cudaError_t lms_fused_select(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p,
                             const float* thetas, uint32_t C, uint64_t k, float* out, uint32_t max_iters,
                             LmsReport* rep, cudaStream_t st) {
  if (rep) *rep = LmsReport{};
  FusedGeom g;
  cudaError_t e = fused_prepare(w, X, y, n, p, thetas, C, g, st);
  if (e != cudaSuccess) return e;
  FusedCols c;
  if ((e = fused_cols(w, C, g, false, c)) != cudaSuccess) return e;
  // per-column copy of ]t_lo, t_hi[: the cuts keep ~2 x 3.5 sd of 16384 samples (~2.8% of n);
  // n/8 leaves room for any k (an overflowing column falls back, counts stay exact)
  const uint64_t zcap = n / 8 + 64;
  if ((e = ensure_buf(reinterpret_cast<void**>(&w.fz), &w.fz_bytes, (size_t)C * zcap * sizeof(float))) != cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(c.le, 0, (size_t)C * 16, st)) != cudaSuccess) return e;  // le + cursor
  iota_kernel<<<1, 256, 0, st>>>(c.ct_list, g.n_ct);
  EventPair ev;
  cudaEventRecord(ev.a, st);
  if ((e = fused_sample_cuts(w, g, X, y, n, p, C, k, c, st)) != cudaSuccess) return e;
  FusedArgs a{};
  a.n = n; a.C = C; a.ct_list = c.ct_list;
  a.cuts = c.cuts; a.le = c.le; a.cursor = c.cursor; a.z = w.fz; a.zcap = zcap;
  if ((e = fused_launch<kFuseCuts>(g, a, g.n_ct, st)) != cudaSuccess) return e;
  cudaEventRecord(ev.b, st);
  // continuation on the per-column copies
  BatchArgs b{nullptr, n, C, k, out, nullptr, 0, nullptr, nullptr, max_iters};
  b.f_cuts = c.cuts; b.f_le = c.le; b.f_cursor = c.cursor; b.f_z = w.fz; b.f_zcap = zcap;
  b.fail_list = c.fail_list;
  uint32_t nfail = 0;
  e = run_batched(w, b, rep, &nfail, st);
  if (rep) { rep->ms_fused = ev.ms(); rep->fallback = nfail; }
  if (e != cudaSuccess) return e;
  if (nfail == 0) return cudaSuccess;
  // fallback: store S for the failed columns only (same kernel, same arithmetic), select from it
  std::vector<unsigned> fl(nfail);
  if ((e = cudaMemcpy(fl.data(), c.fail_list, nfail * sizeof(unsigned), cudaMemcpyDeviceToHost)) != cudaSuccess)
    return e;
  std::vector<unsigned> cts;
  for (unsigned j : fl) {
    const unsigned t = j / TM;
    bool seen = false;
    for (unsigned u : cts) seen |= (u == t);
    if (!seen) cts.push_back(t);
  }
  if ((e = cudaMemcpyAsync(c.ct_list, cts.data(), cts.size() * sizeof(unsigned), cudaMemcpyHostToDevice, st)) !=
      cudaSuccess)
    return e;
  if ((e = ensure_buf(reinterpret_cast<void**>(&w.fS), &w.fS_bytes, (size_t)nfail * n * sizeof(float))) != cudaSuccess)
    return e;
  slot_map_kernel<<<1, 1024, 0, st>>>(c.slot, C, c.fail_list, nfail);
  FusedArgs sa{};
  sa.n = n; sa.C = C; sa.ct_list = c.ct_list; sa.slot = c.slot; sa.S = w.fS;
  if ((e = fused_launch<kFuseStore>(g, sa, (uint32_t)cts.size(), st)) != cudaSuccess) return e;
  BatchArgs f{w.fS, n, nfail, k, out, nullptr, 0, nullptr, nullptr, max_iters};
  f.out_map = c.fail_list;
  return run_batched(w, f, rep, nullptr, st);
}

cudaError_t lms_fused_lts(LmsWorkspace& w, const float* X, const float* y, uint64_t n, uint32_t p,
                          const float* thetas, uint32_t C, uint64_t h, const float* m, double* out, cudaStream_t st) {
  FusedGeom g;
  cudaError_t e = fused_prepare(w, X, y, n, p, thetas, C, g, st);
  if (e != cudaSuccess) return e;
  FusedCols c;
  if ((e = fused_cols(w, C, g, true, c)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.le, 0, (size_t)C * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.part, 0, (size_t)4 * g.n_chunks * C * sizeof(double), st)) != cudaSuccess) return e;
  iota_kernel<<<1, 256, 0, st>>>(c.ct_list, g.n_ct);
  FusedArgs a{};
  a.n = n; a.C = C; a.ct_list = c.ct_list; a.le = c.le; a.m = m; a.sum = c.part;
  if ((e = fused_launch<kFuseLts>(g, a, g.n_ct, st)) != cudaSuccess) return e;
  lts_finish_kernel<<<(C + 255) / 256, 256, 0, st>>>(c.part, 4 * g.n_chunks, C, c.le, h, m, out);
  return cudaGetLastError();
}

void lms_free(LmsWorkspace& w) {
  if (w.S) cudaFree(w.S);
  if (w.dev) cudaFree(w.dev);
  if (w.img) cudaFree(w.img);
  if (w.host) cudaFreeHost(w.host);
  if (w.fimg) cudaFree(w.fimg);
  if (w.fcol) cudaFree(w.fcol);
  if (w.fz) cudaFree(w.fz);
  if (w.fS) cudaFree(w.fS);
  if (w.fsamp) cudaFree(w.fsamp);
  w = LmsWorkspace{};
}

}  // namespace cpsel
