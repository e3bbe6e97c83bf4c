#ifdef CPSEL_VB_PROF
#include <cstdio>
#endif
// sm_100a kernels of the cutting-plane selection path (Beliakov, arXiv:1104.2732).
//
//   init_kernel   step a1: one streaming pass -> (min, #min, max, #max, sum(x-x0), #nonfinite)
//                 ("y_L, y_R and sum x_i ... in a single parallel reduction")
//   pass_kernel   step a2 (+a4): one streaming pass at query t over bracket (y_lo, y_hi) ->
//                 (#x<t, #x==t, sum_{y_lo<x<t}(t-x), sum_{t<x<y_hi}(x-t), pred, succ)
//                 (Fig. 1 'Objective' P:L270-282, footnote P:L192), optionally fused with the
//                 copy_if of the bracket interior (Fig. 1 'SortZ' P:L289-290), split into
//                 the two halves (y_lo,t) and (t,y_hi) so the kept half is known after the pass.
//   radix select  step a5: MSB-first radix select over order-preserving keys on the small set z
//                 (replaces the paper's radix *sort* of z).
//
// Design: HBM-bound streams.  Persistent grid = k x 148 CTAs, 128-bit
// ld.global.nc.L1::no_allocate loads, UNROLL vectors in flight per thread, per-thread
// accumulators, warp-shuffle + shared-memory block reduction, one 80-byte partial per CTA and a
// last-CTA finish (threadfence + atomic ticket) that folds the partials in a fixed order, so
// results are deterministic for a fixed grid.  Compaction stages interior elements per warp in
// shared memory (ballot/popc) and flushes them with one global atomicAdd per <= 1024 elements.
// No fast-math / FTZ: counts must be exact on subnormals.
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include <cooperative_groups.h>

#include "cpsel_kernels.h"
#include "cpsel_ptx.h"

namespace cpsel {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;

template <typename T> struct VecOf;
template <> struct VecOf<float> { using V = float4; static constexpr int N = 4; };
template <> struct VecOf<double> { using V = double2; static constexpr int N = 2; };

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
// the same with an L2 evict-first policy (createpolicy): the init pass's one read of x, so that its
// streaming does not push the copy it writes (read again by the exact finish) out of L2
__device__ __forceinline__ float4 ld_stream_ef(const float4* p, uint64_t pol) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double2 ld_stream_ef(const double2* p, uint64_t pol) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v2.f64 {%0,%1}, [%2], %3;" : "=d"(r.x), "=d"(r.y)
      : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float lane_of(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
__device__ __forceinline__ double lane_of(const double2& v, int j) { return j == 0 ? v.x : v.y; }


template <typename T> __device__ __forceinline__ T tmax(T a, T b);
template <> __device__ __forceinline__ float tmax(float a, float b) { return fmaxf(a, b); }
template <> __device__ __forceinline__ double tmax(double a, double b) { return fmax(a, b); }
template <typename T> __device__ __forceinline__ T tmin(T a, T b);
template <> __device__ __forceinline__ float tmin(float a, float b) { return fminf(a, b); }
template <> __device__ __forceinline__ double tmin(double a, double b) { return fmin(a, b); }

template <typename T> __device__ __forceinline__ T tinf();
template <> __device__ __forceinline__ float tinf() { return __int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double tinf() { return __longlong_as_double(0x7ff0000000000000ll); }

// Order-preserving integer keys of floats (radix select, sample cut, ordered-key bisection).
// (negative: all bits flipped, else the sign bit set — one arithmetic shift and one xor)
__device__ __forceinline__ unsigned long long okey(float v) {
  const unsigned u = __float_as_uint(v);
  return (unsigned long long)(u ^ ((unsigned)(__float_as_int(v) >> 31) | 0x80000000u));
}
__device__ __forceinline__ unsigned long long okey(double v) {
  const long long s = __double_as_longlong(v);
  return (unsigned long long)s ^ ((unsigned long long)(s >> 63) | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_key_f32(unsigned long long k) {
  const unsigned kk = (unsigned)k;
  const unsigned u = (kk & 0x80000000u) ? (kk & 0x7fffffffu) : ~kk;
  return (double)__uint_as_float(u);
}
__device__ __forceinline__ double from_key_f64(unsigned long long k) {
  const unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// Value-linear bins of ]t_lo, t_hi[ (the direct chain's first digit, vbin): bin = trunc((v - t_lo) *
// 2048 / (t_hi - t_lo)) clamped to 2047, with the two roundings done explicitly (no contraction) so
// the init pass and the finish compute the same bin for every value; v <= v' => bin(v) <= bin(v')
// (each step is monotone).  vbin_scale = 0: the span is not finite (an open cut, R31) -> key digits.
__device__ __forceinline__ float vbin_scale(float tl, float th) {
  const float span = __fsub_rn(th, tl);
  return (th > tl && span < __int_as_float(0x7f800000)) ? __fdiv_rn(2048.f, span) : 0.f;
}
__device__ __forceinline__ double vbin_scale(double tl, double th) {
  const double span = __dsub_rn(th, tl);
  return (th > tl && span < __longlong_as_double(0x7ff0000000000000ll)) ? __ddiv_rn(2048.0, span) : 0.0;
}
__device__ __forceinline__ unsigned vbin_of(float v, float tl, float sc) {
  return (unsigned)fminf(fmaxf(__fmul_rn(__fsub_rn(v, tl), sc), 0.f), 2047.f);
}
__device__ __forceinline__ unsigned vbin_of(double v, double tl, double sc) {
  return (unsigned)fmin(fmax(__dmul_rn(__dsub_rn(v, tl), sc), 0.0), 2047.0);
}
// the first digit of a copied element: its value bin, or (sc == 0) the top 11 bits of its key
template <typename T> __device__ __forceinline__ unsigned vbin_digit(T v, T tl, T sc) {
  return sc > T(0) ? vbin_of(v, tl, sc) : (unsigned)(okey(v) >> (sizeof(T) == 4 ? 21 : 53)) & 2047u;
}

// ------------------------------------------------------------------------------------------
// Generic grid-stride stream over x[0..n) with 16-byte vector loads.  F provides
//   template<bool MASKED> void vec(const V&, bool ok)   (all lanes call; ok=false -> no-op)
//   void group_begin(), group_end()                       (around each UNROLL-vector group)
//   void scalar(T, bool ok)                               (head/tail elements)
// Any element alignment is accepted: the unaligned head and the tail (< VE elements each)
// are processed as scalars by warp 0 of the last CTA.
template <typename T, int UNROLL, typename F>
__device__ __forceinline__ void stream_array(const T* __restrict__ x, uint64_t n, F& f,
                                             unsigned part, unsigned nparts) {
  using V = typename VecOf<T>::V;
  constexpr int VE = VecOf<T>::N;
  const uint64_t mis = (reinterpret_cast<uintptr_t>(x) / sizeof(T)) & (VE - 1);
  uint64_t head = mis ? (VE - mis) : 0;
  if (head > n) head = n;
  const V* __restrict__ xv = reinterpret_cast<const V*>(x + head);
  const uint64_t nvec = (n - head) / VE;
  constexpr uint64_t TILE = (uint64_t)kBlock * UNROLL;
  const uint64_t stride = (uint64_t)nparts * TILE;
  uint64_t base = (uint64_t)part * TILE;
  for (; base + TILE <= nvec; base += stride) {
    V v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = ld_stream(xv + base + (uint64_t)u * kBlock + threadIdx.x);
    f.group_begin();
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) f.template vec<false>(v[u], true, u);
    f.group_end();
  }
  if (base < nvec) {  // the one ragged tile of this CTA
    V v[UNROLL];
    bool ok[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint64_t i = base + (uint64_t)u * kBlock + threadIdx.x;
      ok[u] = i < nvec;
      if (ok[u]) v[u] = ld_stream(xv + i);
    }
    f.group_begin();
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) f.template vec<true>(v[u], ok[u], u);
    f.group_end();
  }
  if (part == nparts - 1 && threadIdx.x < 32) {
    const uint64_t tail0 = head + nvec * VE;
    const uint64_t ntail = n - tail0;  // < VE
    const int lane = threadIdx.x;
    bool okh = (uint64_t)lane < head;
    f.scalar(okh ? x[lane] : T(0), okh);
    bool okt = (uint64_t)lane < ntail;
    f.scalar(okt ? x[tail0 + lane] : T(0), okt);
  }
}

// ------------------------------------------------------------------------------------------
// Programmatic dependent launch: a kernel launched with pdl_launch() may be scheduled while the
// kernel before it in the stream is still running (that one calls pdl_trigger()); it calls
// pdl_wait() before touching anything the previous kernel writes.  Both are no-ops without PDL.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ------------------------------------------------------------------------------------------
// Result mailbox: after the finishing thread wrote the result (possibly into mapped host memory),
// make it visible system-wide, then set the flag the host spins on.
__device__ __forceinline__ void publish_done(unsigned long long* done, unsigned long long seq) {
  if (done) {
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(done) = seq;
  }
}

// ------------------------------------------------------------------------------------------
// Block / grid reduction helpers (fixed order -> deterministic for a fixed grid).
template <typename V> __device__ __forceinline__ V warp_sum(V v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

__device__ __forceinline__ void combine(PassPartial& a, const PassPartial& b) {
  a.c_lt += b.c_lt; a.c_eq += b.c_eq; a.c_lo += b.c_lo; a.c_hi += b.c_hi;
  a.L_lo += b.L_lo; a.L_hi += b.L_hi; a.P += b.P; a.N += b.N;
  a.pred = fmax(a.pred, b.pred); a.succ = fmin(a.succ, b.succ);
}

// Reduce one PassPartial per thread to thread 0 of the block.
__device__ PassPartial block_reduce(PassPartial p) {
  __shared__ PassPartial sh[kWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  p.c_lt = warp_sum(p.c_lt); p.c_eq = warp_sum(p.c_eq);
  p.c_lo = warp_sum(p.c_lo); p.c_hi = warp_sum(p.c_hi);
  p.L_lo = warp_sum(p.L_lo); p.L_hi = warp_sum(p.L_hi);
  p.P = warp_sum(p.P); p.N = warp_sum(p.N);
  p.pred = warp_max(p.pred); p.succ = warp_min(p.succ);
  if (lane == 0) sh[w] = p;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kWarps; ++i) combine(p, sh[i]);
  }
  __syncthreads();
  return p;
}

// fold a partial written by another CTA straight from L2 (ld.global.cg), field by field
__device__ __forceinline__ void combine_from(PassPartial& a, const PassPartial* b) {
  a.c_lt += __ldcg(&b->c_lt); a.c_eq += __ldcg(&b->c_eq); a.c_lo += __ldcg(&b->c_lo); a.c_hi += __ldcg(&b->c_hi);
  a.L_lo += __ldcg(&b->L_lo); a.L_hi += __ldcg(&b->L_hi); a.P += __ldcg(&b->P); a.N += __ldcg(&b->N);
  a.pred = fmax(a.pred, __ldcg(&b->pred)); a.succ = fmin(a.succ, __ldcg(&b->succ));
}
__device__ __forceinline__ void combine_from(InitPartial& a, const InitPartial* b) {
  const double mn = __ldcg(&b->vmin), mx = __ldcg(&b->vmax);
  const unsigned long long cmn = __ldcg(&b->cnt_min), cmx = __ldcg(&b->cnt_max);
  if (mn < a.vmin) { a.vmin = mn; a.cnt_min = cmn; } else if (mn == a.vmin) a.cnt_min += cmn;
  if (mx > a.vmax) { a.vmax = mx; a.cnt_max = cmx; } else if (mx == a.vmax) a.cnt_max += cmx;
  a.S += __ldcg(&b->S); a.N0 += __ldcg(&b->N0); a.P0 += __ldcg(&b->P0); a.I0 += __ldcg(&b->I0);
  a.nonfinite += __ldcg(&b->nonfinite); a.pad2 += __ldcg(&b->pad2);
  a.cA += __ldcg(&b->cA); a.cB += __ldcg(&b->cB); a.cC += __ldcg(&b->cC); a.cD += __ldcg(&b->cD);
  a.cE += __ldcg(&b->cE);
}

__device__ __forceinline__ void combine(InitPartial& a, const InitPartial& b) {
  if (b.vmin < a.vmin) { a.vmin = b.vmin; a.cnt_min = b.cnt_min; }
  else if (b.vmin == a.vmin) a.cnt_min += b.cnt_min;
  if (b.vmax > a.vmax) { a.vmax = b.vmax; a.cnt_max = b.cnt_max; }
  else if (b.vmax == a.vmax) a.cnt_max += b.cnt_max;
  a.S += b.S;
  a.nonfinite += b.nonfinite;
  a.N0 += b.N0;
  a.P0 += b.P0;
  a.I0 += b.I0;
  a.pad2 += b.pad2;
  a.cA += b.cA; a.cB += b.cB; a.cC += b.cC; a.cD += b.cD; a.cE += b.cE;
}

// Reduce one InitPartial per thread to thread 0 of the block: warp butterflies, then the warps.
__device__ InitPartial block_reduce(InitPartial p) {
  __shared__ InitPartial sh[kWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // field by field (few live registers): (min, #min) and (max, #max) pairs, then plain sums
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double mn = __shfl_xor_sync(FULL, p.vmin, o);
    const unsigned long long cmn = __shfl_xor_sync(FULL, p.cnt_min, o);
    if (mn < p.vmin) { p.vmin = mn; p.cnt_min = cmn; } else if (mn == p.vmin) p.cnt_min += cmn;
    const double mx = __shfl_xor_sync(FULL, p.vmax, o);
    const unsigned long long cmx = __shfl_xor_sync(FULL, p.cnt_max, o);
    if (mx > p.vmax) { p.vmax = mx; p.cnt_max = cmx; } else if (mx == p.vmax) p.cnt_max += cmx;
  }
  p.S = warp_sum(p.S); p.N0 = warp_sum(p.N0); p.P0 = warp_sum(p.P0); p.I0 = warp_sum(p.I0);
  p.nonfinite = warp_sum(p.nonfinite); p.pad2 = warp_sum(p.pad2);
  p.cA = warp_sum(p.cA); p.cB = warp_sum(p.cB); p.cC = warp_sum(p.cC); p.cD = warp_sum(p.cD);
  p.cE = warp_sum(p.cE);
  if (lane == 0) sh[w] = p;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 1; i < kWarps; ++i) combine(p, sh[i]);
  __syncthreads();
  return p;
}

// Last-CTA finish: every CTA stores its partial, the last one to arrive folds all partials in a
// fixed order.  Returns true in the last CTA (where *total is valid in thread 0).
template <typename P>
__device__ bool grid_finish(const P& mine, P* partials, unsigned int* ticket, P* total, const P& identity) {
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = mine;
    __threadfence();
    const unsigned prev = atomicAdd(ticket, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  P acc = identity;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += kBlock) combine_from(acc, partials + i);
  acc = block_reduce(acc);
  if (threadIdx.x == 0) {
    *total = acc;
    *ticket = 0u;  // self-reset for the next launch
  }
  return true;
}

// ------------------------------------------------------------------------------------------
// Step a1: init reduction.
// Fast form: per 16-byte vector a min/max of its lanes (FMNMX) and a rarely-taken branch that
// updates (min, #min) / (max, #max) only when the vector reaches the running extreme; the shifted
// sum doubles as the non-finite detector (NaN/Inf make it non-finite; the host then re-runs the
// CHECKED form, which counts non-finite elements exactly).
// CUT: also evaluate the two extra cuts t_lo <= t_hi of R23 (sample quantiles bracketing the
// target rank) in the same read: #x<t_lo, #x=t_lo, #x<t_hi, #x=t_hi, #x>t_hi, N_lo = sum (t_lo-x)^+,
// P_hi = sum (x-t_hi)^+ and the bracket-interior sum I = sum_{t_lo<x<t_hi} (x-t_lo), as predicated
// PTX (16 issue slots per element, balanced over the ALU and FMA pipes: three of the five
// counters are per-thread float counters, exact below 2^24).
template <typename T, bool CHECKED, bool CUT = false> struct InitFn {
  T mn, mx, x0;
  unsigned cmn, cmx, nonfin;
  double S;
  T g[4];
  T tl, th;
  unsigned cA = 0, cC = 0;        // #x<t_lo, #x<t_hi
  float fB = 0, fD = 0, fE = 0;   // #x=t_lo, #x=t_hi, #x>t_hi (exact while < 2^24 per thread)
  // with the cuts the shifted sum is not needed (the first iterate comes from the cuts' sums) and
  // a NaN shows as counts not adding up to n; the CHECKED re-run still computes everything
  static constexpr bool SUM = !CUT || CHECKED;
  T gN[4], gP[4], gI[4];
  double N0 = 0, P0 = 0, I0 = 0;
  __device__ InitFn(T x0_) : mn(tinf<T>()), mx(-tinf<T>()), x0(x0_), cmn(0), cmx(0), nonfin(0), S(0) {}
  __device__ __forceinline__ void cut(float v, float& n_, float& p_, float& i_) {
    asm("{\n\t.reg .pred pA, pB, pC, pD, pE, pI;\n\t.reg .f32 dl, dh;\n\t"
        "setp.lt.f32 pA, %8, %9;\n\t"
        "setp.eq.f32 pB, %8, %9;\n\t"
        "setp.lt.f32 pC, %8, %10;\n\t"
        "setp.eq.f32 pD, %8, %10;\n\t"
        "setp.gt.f32 pE, %8, %10;\n\t"
        "setp.gt.and.f32 pI, %8, %9, pC;\n\t"
        "sub.rn.f32 dl, %9, %8;\n\t"
        "sub.rn.f32 dh, %8, %10;\n\t"
        "@pA add.u32 %0, %0, 1;\n\t"
        "@pC add.u32 %1, %1, 1;\n\t"
        "@pB add.rn.f32 %2, %2, 0f3F800000;\n\t"
        "@pD add.rn.f32 %3, %3, 0f3F800000;\n\t"
        "@pE add.rn.f32 %4, %4, 0f3F800000;\n\t"
        "@pA add.rn.f32 %5, %5, dl;\n\t"
        "@pE add.rn.f32 %6, %6, dh;\n\t"
        "@pI sub.rn.f32 %7, %7, dl;\n\t}"
        : "+r"(cA), "+r"(cC), "+f"(fB), "+f"(fD), "+f"(fE), "+f"(n_), "+f"(p_), "+f"(i_)
        : "f"(v), "f"(tl), "f"(th));
  }
  __device__ __forceinline__ void cut(double v, double& n_, double& p_, double& i_) {
    asm("{\n\t.reg .pred pA, pB, pC, pD, pE, pI;\n\t.reg .f64 dl, dh;\n\t"
        "setp.lt.f64 pA, %8, %9;\n\t"
        "setp.eq.f64 pB, %8, %9;\n\t"
        "setp.lt.f64 pC, %8, %10;\n\t"
        "setp.eq.f64 pD, %8, %10;\n\t"
        "setp.gt.f64 pE, %8, %10;\n\t"
        "setp.gt.and.f64 pI, %8, %9, pC;\n\t"
        "sub.rn.f64 dl, %9, %8;\n\t"
        "sub.rn.f64 dh, %8, %10;\n\t"
        "@pA add.u32 %0, %0, 1;\n\t"
        "@pC add.u32 %1, %1, 1;\n\t"
        "@pB add.rn.f32 %2, %2, 0f3F800000;\n\t"
        "@pD add.rn.f32 %3, %3, 0f3F800000;\n\t"
        "@pE add.rn.f32 %4, %4, 0f3F800000;\n\t"
        "@pA add.rn.f64 %5, %5, dl;\n\t"
        "@pE add.rn.f64 %6, %6, dh;\n\t"
        "@pI sub.rn.f64 %7, %7, dl;\n\t}"
        : "+r"(cA), "+r"(cC), "+f"(fB), "+f"(fD), "+f"(fE), "+d"(n_), "+d"(p_), "+d"(i_)
        : "d"(v), "d"(tl), "d"(th));
  }
  __device__ __forceinline__ void slow(T v) {
    if (v < mn) { mn = v; cmn = 1; } else if (v == mn) ++cmn;
    if (v > mx) { mx = v; cmx = 1; } else if (v == mx) ++cmx;
  }
  __device__ __forceinline__ void group_begin() {
    g[0] = g[1] = g[2] = g[3] = T(0);
    if (CUT)
#pragma unroll
      for (int u = 0; u < 4; ++u) gN[u] = gP[u] = gI[u] = T(0);
  }
  __device__ __forceinline__ void group_end() {
    if (SUM) S += (double)((g[0] + g[1]) + (g[2] + g[3]));
    if (CUT) {
      N0 += (double)((gN[0] + gN[1]) + (gN[2] + gN[3]));
      P0 += (double)((gP[0] + gP[1]) + (gP[2] + gP[3]));
      I0 += (double)((gI[0] + gI[1]) + (gI[2] + gI[3]));
    }
  }
  __device__ __forceinline__ void vec_elems(const float4& v, int u) {
    if (CUT) {
      const int w = u & 3;
      cut(v.x, gN[w], gP[w], gI[w]); cut(v.y, gN[w], gP[w], gI[w]);
      cut(v.z, gN[w], gP[w], gI[w]); cut(v.w, gN[w], gP[w], gI[w]);
    }
    const float lo = fminf(fminf(v.x, v.y), fminf(v.z, v.w));
    const float hi = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
    if (lo <= mn || hi >= mx) { slow(v.x); slow(v.y); slow(v.z); slow(v.w); }
    if (SUM) g[u & 3] += ((v.x - x0) + (v.y - x0)) + ((v.z - x0) + (v.w - x0));
    if (CHECKED)
      nonfin += !(fabsf(v.x) <= FLT_MAX) + !(fabsf(v.y) <= FLT_MAX) + !(fabsf(v.z) <= FLT_MAX) + !(fabsf(v.w) <= FLT_MAX);
  }
  __device__ __forceinline__ void vec_elems(const double2& v, int u) {
    if (CUT) {
      const int w = u & 3;
      cut(v.x, gN[w], gP[w], gI[w]); cut(v.y, gN[w], gP[w], gI[w]);
    }
    const double lo = fmin(v.x, v.y), hi = fmax(v.x, v.y);
    if (lo <= mn || hi >= mx) { slow(v.x); slow(v.y); }
    if (SUM) g[u & 3] += (v.x - x0) + (v.y - x0);
    if (CHECKED) nonfin += !(fabs(v.x) <= DBL_MAX) + !(fabs(v.y) <= DBL_MAX);
  }
  template <bool MASKED, typename V> __device__ __forceinline__ void vec(const V& v, bool ok, int u) {
    if (MASKED && !ok) return;
    vec_elems(v, u);
  }
  __device__ __forceinline__ void scalar(T v, bool ok) {
    if (!ok) return;
    group_begin();
    slow(v);
    g[0] = v - x0;
    if (CUT) cut(v, gN[0], gP[0], gI[0]);
    if (CHECKED) nonfin += !(fabs(v) <= (sizeof(T) == 4 ? (T)FLT_MAX : (T)DBL_MAX));
    group_end();
  }
};

template <typename T, int UNROLL, bool CHECKED, bool CUT>
__global__ void __launch_bounds__(kBlock, 4) init_kernel(InitArgs a) {
  const T* x = static_cast<const T*>(a.x);
  InitFn<T, CHECKED, CUT> f(x[0]);
  if (CUT) {
    f.tl = static_cast<const T*>(a.t0)[0];
    f.th = static_cast<const T*>(a.t0)[1];
  }
  stream_array<T, UNROLL>(x, a.n, f, blockIdx.x, gridDim.x);
  InitPartial p;
  p.vmin = (double)f.mn; p.vmax = (double)f.mx; p.S = f.S; p.pad = 0;
  p.cnt_min = f.cmn; p.cnt_max = f.cmx; p.nonfinite = f.nonfin; p.pad2 = 0;
  p.N0 = f.N0; p.P0 = f.P0; p.I0 = f.I0;
  p.cA = f.cA; p.cB = (unsigned long long)f.fB; p.cC = f.cC; p.cD = (unsigned long long)f.fD;
  p.cE = (unsigned long long)f.fE;
  p = block_reduce(p);
  InitPartial id;
  id.vmin = tinf<double>(); id.vmax = -tinf<double>(); id.S = 0; id.pad = 0;
  id.cnt_min = id.cnt_max = id.nonfinite = id.pad2 = 0;
  id.N0 = id.P0 = id.I0 = 0; id.cA = id.cB = id.cC = id.cD = id.cE = 0;
  InitPartial tot;
  if (grid_finish(p, static_cast<InitPartial*>(a.partials), a.ticket, &tot, id) && threadIdx.x == 0) {
    DevInit r;
    r.vmin = tot.vmin; r.vmax = tot.vmax; r.S = tot.S; r.x0 = (double)x[0];
    r.cnt_min = tot.cnt_min; r.cnt_max = tot.cnt_max; r.nonfinite = tot.nonfinite; r.pad = 0;
    r.t_lo = CUT ? (double)f.tl : 0.0;
    r.t_hi = CUT ? (double)f.th : 0.0;
    r.N_lo = tot.N0; r.P_hi = tot.P0; r.I_in = tot.I0;
    r.c_le_lo = tot.cA + tot.cB; r.c_lt_hi = tot.cC; r.res1 = r.res2 = 0;
    r.t_est = CUT ? (double)static_cast<const T*>(a.t0)[2] : 0.0;
    // a NaN is in none of <t_hi, =t_hi, >t_hi: the fast form reports the shortfall (CHECKED counts all)
    if (CUT && !CHECKED) r.nonfinite = a.n - tot.cC - tot.cD - tot.cE;
    r.has_cut = CUT ? 6ull : 0ull;  // two cuts, with N_lo / P_hi
    *a.out = r;
    publish_done(a.done, a.seq);
  }
}

// R23: the extra cut of the init pass — the sample quantile at the target rank among 1024 evenly
// strided samples: one CTA of 1024 threads, one key per thread, bitonic sort with warp shuffles
// for strides < 32 and shared memory above.
// Sort the block's 1024 sample keys (one per thread, padding = ~0 sorts last) and write the two
// cuts bracketing local rank r of an m-element array, from ms real samples: ranks q -/+ 3.5
// binomial standard deviations (+2) of the sample.  The target lies between the two cuts with
// overwhelming probability on any input order (the cuts are exact either way).
// keys_out != nullptr: write the sorted sample keys there instead (R28, pooled across ranks).
template <typename T>
__device__ __forceinline__ void sample_sort_pick(unsigned long long v, unsigned long long* key, uint64_t ms,
                                                 uint64_t m, uint64_t r, T* t0, unsigned long long* keys_out) {
  constexpr int S = 1024;
  const int i = threadIdx.x;
  for (int size = 2; size <= S; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      unsigned long long w;
      if (stride >= 32) {
        key[i] = v;
        __syncthreads();
        w = key[i ^ stride];
        __syncthreads();
      } else {
        w = __shfl_xor_sync(FULL, v, stride);
      }
      const bool up = (i & size) == 0, lower = (i & stride) == 0;
      const unsigned long long lo = v < w ? v : w, hi = v < w ? w : v;
      v = (up == lower) ? lo : hi;
    }
  }
  key[i] = v;
  __syncthreads();
  if (keys_out) {
    keys_out[i] = v;
    return;
  }
  if (i == 0) {
    const double md = (double)ms;
    const double q = ((double)r - 0.5) / (double)m * md;
    const double w = 3.5 * sqrt(fmax(q * (md - q) / md, 0.0)) + 2.0;
    const double ql = floor(q - w), qh = ceil(q + w);
    const uint64_t il = ql < 0 ? 0 : (uint64_t)ql;
    const uint64_t ih = qh >= md ? ms - 1 : (uint64_t)qh;
    t0[0] = (T)(sizeof(T) == 4 ? from_key_f32(key[il]) : from_key_f64(key[il]));
    t0[1] = (T)(sizeof(T) == 4 ? from_key_f32(key[ih]) : from_key_f64(key[ih]));
    // the sample's own estimate of the target (a starting iterate where no interior sum is kept)
    const double qm = floor(q);
    const uint64_t im = qm < 0 ? 0 : (qm >= md ? ms - 1 : (uint64_t)qm);
    t0[2] = (T)(sizeof(T) == 4 ? from_key_f32(key[im]) : from_key_f64(key[im]));
  }
}

// R23: the two extra cuts of the init pass — 1024 evenly strided samples of x[0..n), cuts around
// rank k.  (Also used for a contiguous current array with its local rank, R26.)
template <typename T>
__global__ void __launch_bounds__(1024) sample_cut_kernel(const T* __restrict__ x, uint64_t n, uint64_t k, T* t0,
                                                          uint32_t smax, unsigned long long* keys_out) {
  constexpr int S = 1024;
  __shared__ unsigned long long key[S];
  const int i = threadIdx.x;
  const uint64_t m = n < (uint64_t)smax ? n : (uint64_t)smax;
  unsigned long long v = ~0ull;  // padding sorts last
  if ((uint64_t)i < m) {
    const uint64_t pos = (n == m) ? (uint64_t)i : ((uint64_t)i * n) / m + (n / m) / 2;
    v = okey(x[pos]);
  }
  sample_sort_pick<T>(v, key, m, n, k, t0, keys_out);
}

// R26: the same for a segmented current array (the runs `side` of the Wtot warp entries, m
// elements in total): sample i is element floor(i*m/1024) + (m/1024)/2 of the concatenated runs.
template <typename T>
__global__ void __launch_bounds__(1024) sample_seg_kernel(const T* __restrict__ base, const SegEntry* __restrict__ tab,
                                                          int side, int Wtot, uint64_t m, uint64_t r, T* t0,
                                                          uint32_t smax, unsigned long long* keys_out) {
  constexpr int S = 1024;
  __shared__ unsigned long long key[S];
  __shared__ unsigned long long cstart[S];
  const int i = threadIdx.x;
  const int per = (Wtot + S - 1) / S;  // runs per chunk
  const int w0 = i * per, w1 = min(w0 + per, Wtot);
  unsigned long long c = 0;
  for (int w = w0; w < w1; ++w) c += tab[w].cnt[side];
  // inclusive block scan of the chunk totals
  cstart[i] = c;
  __syncthreads();
  for (int off = 1; off < S; off <<= 1) {
    const unsigned long long add = i >= off ? cstart[i - off] : 0ull;
    __syncthreads();
    cstart[i] += add;
    __syncthreads();
  }
  const uint64_t ms = m < (uint64_t)smax ? m : (uint64_t)smax;
  unsigned long long v = ~0ull;
  if ((uint64_t)i < ms) {
    uint64_t g = (m == ms) ? (uint64_t)i : ((uint64_t)i * m) / ms + (m / ms) / 2;
    // first chunk whose inclusive total exceeds g
    int lo = 0, hi = S - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cstart[mid] > g) hi = mid; else lo = mid + 1;
    }
    g -= lo ? cstart[lo - 1] : 0ull;
    for (int w = lo * per; w < min(lo * per + per, Wtot); ++w) {
      const SegEntry e = tab[w];
      if (g < e.cnt[side]) {
        v = okey(base[e.off[side] + g]);
        break;
      }
      g -= e.cnt[side];
    }
  }
  sample_sort_pick<T>(v, key, ms, m, r, t0, keys_out);
}

// ------------------------------------------------------------------------------------------
// R29: the sample cuts from a LARGE sample — 32768 (f32) / 16384 (f64) evenly strided samples of
// the current array (contiguous, or the runs `side` of a segmented one), kept in registers as
// order-preserving keys, and the three sample order statistics (ranks q - w, q + w and q) found
// by one-CTA MSB radix select of all three at once (11-bit digits, smem histograms), not a sort.
// With 32768 samples the two cuts keep ~2% of the array between them (vs ~11% with 1024).
template <typename T> struct SampleKey;
// ROUNDS: MSB digits resolved; the cuts are the bounds of the remaining key class (f32: 10 bits =
// 2^10 ulps, f64: 20 bits) — any float is a valid cut, only its rank precision matters.
template <> struct SampleKey<float> {
  using K = unsigned;
  static constexpr int KPT = 32, ROUNDS = 2;
  static constexpr K KLO = 0x00800000u, KHI = 0xff7fffffu;  // keys of -FLT_MAX, +FLT_MAX
  __device__ static K key(float v) { return (unsigned)okey(v); }
  __device__ static float val(K k) { return (float)from_key_f32(k); }
  __device__ static int shift(int r) { return r == 0 ? 21 : (r == 1 ? 10 : 0); }
  __device__ static int bits(int r) { return r == 2 ? 10 : 11; }
};
template <> struct SampleKey<double> {
  using K = unsigned long long;
  static constexpr int KPT = 16, ROUNDS = 4;
  static constexpr K KLO = 0x0010000000000000ull, KHI = 0xffefffffffffffffull;  // keys of -DBL_MAX, +DBL_MAX
  __device__ static K key(double v) { return okey(v); }
  __device__ static double val(K k) { return from_key_f64(k); }
  __device__ static int shift(int r) { return r < 4 ? 53 - 11 * r : (r == 4 ? 10 : 0); }
  __device__ static int bits(int r) { return r < 4 ? 11 : 10; }
};
struct SampleSel {
  unsigned hist[3][2048];
  unsigned csum[3][32];
  unsigned long long prefix[3], mask[3], rank[3];
};
constexpr int kGatherMaxWarps = 5888;  // run-table entries a gather CTA can scan in shared memory (46 KB)

// Gather: sample s (one per thread of kSampleCtas<T> CTAs) is element floor(s*m/ms) + (m/ms)/2 of
// the array (contiguous x, or the concatenation of the runs `side` of tab[0..Wtot)), written as an
// order-preserving key; padding keys ~0 beyond ms.  Many CTAs, so the scattered loads of the
// sample are spread over the SMs.
constexpr int kGatherThreads = 256;
template <typename T, int KPT>
__global__ void __launch_bounds__(kGatherThreads) sample_gather_kernel(const T* __restrict__ x, uint64_t m,
                                                             const SegEntry* __restrict__ tab, int side, int Wtot,
                                                             typename SampleKey<T>::K* __restrict__ keys,
                                                             const ChainState* chain, int which) {
  using SK = SampleKey<T>;
  using K = typename SK::K;
  constexpr uint64_t S = 1024ull * KPT;
  if (chain) {  // a device-chain step: size from the chain, nothing to do unless the chain holds
    if (!chain->ok[which]) return;
    m = chain->m[which];
  }
  __shared__ unsigned long long pre[kGatherMaxWarps];  // inclusive prefix of the run lengths
  __shared__ unsigned long long wsum[32];
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  constexpr int NW = kGatherThreads / 32;
  const uint64_t ms = m < S ? m : S;
  const uint64_t smp = (uint64_t)blockIdx.x * kGatherThreads + i;
  if (tab) {
    // every CTA scans the whole (small) run table: per-thread chunk sums, warp and block scans
    const int per = (Wtot + kGatherThreads - 1) / kGatherThreads;
    const int w0 = i * per, w1 = min(w0 + per, Wtot);
    unsigned long long c = 0;
    for (int w = w0; w < w1; ++w) {
      c += tab[w].cnt[side];
      pre[w] = c;
    }
    unsigned long long incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      unsigned long long v = lane < NW ? wsum[lane] : 0ull, inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane < NW) wsum[lane] = inc - v;  // exclusive warp offsets
    }
    __syncthreads();
    const unsigned long long base = wsum[warp] + incl - c;  // exclusive offset of this thread's chunk
    for (int w = w0; w < w1; ++w) pre[w] += base;
    __syncthreads();
  }
  K key = ~K(0);
  if (smp < ms) {
    uint64_t g = (m == ms) ? smp : (smp * m) / ms + (m / ms) / 2;
    if (!tab) {
      key = SK::key(x[g]);
    } else {
      int lo = 0, hi = Wtot - 1;  // first run whose inclusive prefix exceeds g
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] > g) hi = mid; else lo = mid + 1;
      }
      g -= lo ? pre[lo - 1] : 0ull;
      key = SK::key(x[tab[lo].off[side] + g]);
    }
  }
  if (smp < S) keys[smp] = key;
}

// Select: one CTA of 1024 threads holds the KPT keys per thread in registers and finds the three
// sample order statistics (ranks q - w, q + w and q; q the local target rank r scaled to the
// sample) by MSB radix select of all three at once (11-bit digits, smem histograms) — no sort.
template <typename T, int KPT>
__global__ void __launch_bounds__(1024) sample_select_kernel(const typename SampleKey<T>::K* __restrict__ keys_in,
                                                             uint64_t m, uint64_t r, T* t0, const ChainState* chain,
                                                             int which) {
  using SK = SampleKey<T>;
  using K = typename SK::K;
  if (chain) {
    if (!chain->ok[which]) return;
    m = chain->m[which];
    r = chain->r[which];
  }
  constexpr uint64_t S = 1024ull * KPT;
  __shared__ SampleSel sh;
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  const uint64_t ms = m < S ? m : S;
  K keys[KPT];
#pragma unroll
  for (int j = 0; j < KPT; ++j) keys[j] = keys_in[(uint64_t)j * 1024 + i];
  // sort this thread's keys (bitonic network in registers)
#pragma unroll
  for (int size = 2; size <= KPT; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int l = j ^ stride;
        if (l > j) {
          const K a = keys[j], b = keys[l];
          const bool up = (j & size) == 0;
          keys[j] = up ? (a < b ? a : b) : (a < b ? b : a);
          keys[l] = up ? (a < b ? b : a) : (a < b ? a : b);
        }
      }
    }
  }
  if (i == 0) {
    const double md = (double)ms;
    const double q = ((double)r - 0.5) / (double)m * md;
    const double w = 3.5 * sqrt(fmax(q * (md - q) / md, 0.0)) + 2.0;
    const double qq[3] = {floor(q - w), ceil(q + w), floor(q)};
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      sh.rank[t] = qq[t] < 0 ? 0 : (qq[t] >= md ? ms - 1 : (uint64_t)qq[t]);  // 0-based
      sh.prefix[t] = 0;
      sh.mask[t] = 0;
    }
  }
  for (int rd = 0; rd < SK::ROUNDS; ++rd) {
    const int shift = SK::shift(rd), nb = 1 << SK::bits(rd);
    for (int b = i; b < 3 * 2048; b += 1024) (&sh.hist[0][0])[b] = 0u;
    __syncthreads();
    const K p0 = (K)sh.prefix[0], p1 = (K)sh.prefix[1], p2 = (K)sh.prefix[2];
    const K m0 = (K)sh.mask[0], m1 = (K)sh.mask[1], m2 = (K)sh.mask[2];
    // each thread's keys are sorted, so the keys of a prefix class are contiguous and their digits
    // non-decreasing: one shared atomic per run of equal digits (the leading digits of a sample
    // are highly concentrated — per-key atomics would serialise on a few bins)
    const int ntg = rd == 0 ? 1 : 3;  // round 0: every prefix is empty, one histogram serves all
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (t >= ntg) break;
      const K pt = t == 0 ? p0 : (t == 1 ? p1 : p2), mt = t == 0 ? m0 : (t == 1 ? m1 : m2);
      unsigned run = 0;
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const K k = keys[j];
        const bool in = (k & mt) == pt;
        const unsigned d = (unsigned)(k >> shift) & (unsigned)(nb - 1);
        run += in ? 1u : 0u;
        bool last = in;
        if (j + 1 < KPT) {
          const K kn = keys[j + 1 < KPT ? j + 1 : j];
          last = in && (((kn & mt) != pt) || (((unsigned)(kn >> shift) & (unsigned)(nb - 1)) != d));
        }
        if (last) {
          atomicAdd(&sh.hist[t][d], run);
          run = 0;
        }
      }
    }
    __syncthreads();
    if (rd == 0)
      for (int b = i; b < 2048; b += 1024) sh.hist[1][b] = sh.hist[2][b] = sh.hist[0][b];
    __syncthreads();
    // digit search, two levels: warp w sums bins [64w, 64w+64) of each target, then warp t finds
    // the 64-bin chunk and the bin holding rank[t]
    {
      const int c0 = warp * 64;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        unsigned v = (c0 + lane < nb ? sh.hist[t][c0 + lane] : 0u) + (c0 + 32 + lane < nb ? sh.hist[t][c0 + 32 + lane] : 0u);
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (lane == 0) sh.csum[t][warp] = v;
      }
    }
    __syncthreads();
    if (warp < 3) {
      const int t = warp;
      const unsigned long long rk = sh.rank[t];
      // chunk: inclusive scan of the 32 chunk sums
      const unsigned cs = sh.csum[t][lane];
      unsigned incl = cs;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned hm = __ballot_sync(FULL, (unsigned long long)incl > rk);
      const int c = __ffs(hm) - 1;  // first chunk whose inclusive total exceeds rk
      unsigned long long before = __shfl_sync(FULL, incl - cs, c);
      // bin inside the chunk (two 32-bin halves)
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int b = c * 64 + half * 32 + lane;
        const unsigned h = b < nb ? sh.hist[t][b] : 0u;
        unsigned in2 = h;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(FULL, in2, o);
          if (lane >= o) in2 += y;
        }
        const unsigned hb = __ballot_sync(FULL, before + in2 > rk);
        if (hb) {
          const int src = __ffs(hb) - 1;
          const unsigned ex = __shfl_sync(FULL, in2 - h, src);
          if (lane == 0) {
            sh.prefix[t] |= (unsigned long long)(c * 64 + half * 32 + src) << shift;
            sh.mask[t] |= (unsigned long long)(nb - 1) << shift;
            sh.rank[t] = rk - (before + ex);
          }
          break;
        }
        before += __shfl_sync(FULL, in2, 31);
      }
    }
    __syncthreads();
  }
  if (i < 3) {
    // t_a: the lower bound of its class, t_b: the upper bound, estimate: the lower bound — clamped
    // to the finite keys
    K kk = (K)sh.prefix[i];
    if (i == 1) kk |= (K)~(K)sh.mask[1];
    kk = kk < SK::KLO ? SK::KLO : (kk > SK::KHI ? SK::KHI : kk);
    t0[i] = SK::val(kk);
  }
}

// ------------------------------------------------------------------------------------------
// Step a2 (+ a4): one cutting-plane pass.
// Compaction (a4) is block-synchronous per tile: every thread keeps the flags of its
// UNROLL*VE elements, the block scans the (lo,hi) counts (warp shuffles + one smem round), ONE
// thread reserves the block's output ranges with one atomicAdd per half per tile, and every
// thread then writes its elements straight to their final positions (lo half growing up from
// z[0], hi half growing down from z[z_cap-1]).  Output order is unspecified (z is a multiset).
struct CompactShared {
  unsigned warp_incl[kWarps];  // per-warp inclusive totals, packed lo | hi << 16
  unsigned warp_excl[kWarps];  // per-warp exclusive block prefix, packed
  unsigned tot;                // group totals, packed
  unsigned n[2];               // elements staged in the smem buffers (lo, hi)
  unsigned long long base[2];  // reserved output offsets of a flush
};
// smem staging: per half 2 x (block group) elements; a half is flushed (one atomicAdd, coalesced
// stores) once more than one group's worth is staged
template <typename T> __host__ __device__ constexpr int group_elems() { return kBlock * 4 * VecOf<T>::N; }
template <typename T> __host__ __device__ constexpr int stage_elems() { return group_elems<T>() + group_elems<T>() / 2; }
template <typename T> constexpr size_t compact_smem_bytes() { return 2 * stage_elems<T>() * sizeof(T); }

template <typename T, int MODE, int UNROLL> struct PassFn {
  static constexpr int VE = VecOf<T>::N;
  static constexpr int G = UNROLL * VE;  // elements per thread per group (<= 16)
  T t, yL, yR;
  unsigned c_lt, c_eq, c_lo, c_hi;
  double L_lo, L_hi, P, N;
  T pred, succ;
  T glo[UNROLL], ghi[UNROLL], gP[UNROLL], gN[UNROLL];
  // compaction (MODE == kCompact)
  T vals[G];
  unsigned lo_bits, hi_bits;
  CompactShared* cs;
  T* z;
  uint64_t z_cap;
  unsigned long long* cursors;

  __device__ __forceinline__ void hot_elem(float v, float& glo_, float& ghi_) {
    asm("{\n\t.reg .pred plt, pgt, peq, plo, phi;\n\t.reg .f32 d;\n\t"
        "setp.lt.f32 plt, %4, %5;\n\t"
        "setp.gt.f32 pgt, %4, %5;\n\t"
        "setp.eq.f32 peq, %4, %5;\n\t"
        "setp.gt.and.f32 plo, %4, %6, plt;\n\t"
        "setp.lt.and.f32 phi, %4, %7, pgt;\n\t"
        "sub.rn.f32 d, %5, %4;\n\t"
        "@plt add.u32 %0, %0, 1;\n\t"
        "@peq add.u32 %1, %1, 1;\n\t"
        "@plo add.rn.f32 %2, %2, d;\n\t"
        "@phi sub.rn.f32 %3, %3, d;\n\t}"
        : "+r"(c_lt), "+r"(c_eq), "+f"(glo_), "+f"(ghi_)
        : "f"(v), "f"(t), "f"(yL), "f"(yR));
  }
  __device__ __forceinline__ void hot_elem(double v, double& glo_, double& ghi_) {
    asm("{\n\t.reg .pred plt, pgt, peq, plo, phi;\n\t.reg .f64 d;\n\t"
        "setp.lt.f64 plt, %4, %5;\n\t"
        "setp.gt.f64 pgt, %4, %5;\n\t"
        "setp.eq.f64 peq, %4, %5;\n\t"
        "setp.gt.and.f64 plo, %4, %6, plt;\n\t"
        "setp.lt.and.f64 phi, %4, %7, pgt;\n\t"
        "sub.rn.f64 d, %5, %4;\n\t"
        "@plt add.u32 %0, %0, 1;\n\t"
        "@peq add.u32 %1, %1, 1;\n\t"
        "@plo add.rn.f64 %2, %2, d;\n\t"
        "@phi sub.rn.f64 %3, %3, d;\n\t}"
        : "+r"(c_lt), "+r"(c_eq), "+d"(glo_), "+d"(ghi_)
        : "d"(v), "d"(t), "d"(yL), "d"(yR));
  }

  __device__ __forceinline__ void compact_elem(float v, float& glo_, float& ghi_, int idx) {
    asm("{\n\t.reg .pred plt, pgt, plo, phi;\n\t.reg .f32 d;\n\t"
        "setp.lt.f32 plt, %4, %5;\n\t"
        "setp.gt.f32 pgt, %4, %5;\n\t"
        "setp.gt.and.f32 plo, %4, %6, plt;\n\t"
        "setp.lt.and.f32 phi, %4, %7, pgt;\n\t"
        "sub.rn.f32 d, %5, %4;\n\t"
        "@plo add.rn.f32 %0, %0, d;\n\t"
        "@phi sub.rn.f32 %1, %1, d;\n\t"
        "@plo or.b32 %2, %2, %8;\n\t"
        "@phi or.b32 %3, %3, %8;\n\t}"
        : "+f"(glo_), "+f"(ghi_), "+r"(lo_bits), "+r"(hi_bits)
        : "f"(v), "f"(t), "f"(yL), "f"(yR), "r"(1u << idx));
  }
  __device__ __forceinline__ void compact_elem(double v, double& glo_, double& ghi_, int idx) {
    asm("{\n\t.reg .pred plt, pgt, plo, phi;\n\t.reg .f64 d;\n\t"
        "setp.lt.f64 plt, %4, %5;\n\t"
        "setp.gt.f64 pgt, %4, %5;\n\t"
        "setp.gt.and.f64 plo, %4, %6, plt;\n\t"
        "setp.lt.and.f64 phi, %4, %7, pgt;\n\t"
        "sub.rn.f64 d, %5, %4;\n\t"
        "@plo add.rn.f64 %0, %0, d;\n\t"
        "@phi sub.rn.f64 %1, %1, d;\n\t"
        "@plo or.b32 %2, %2, %8;\n\t"
        "@phi or.b32 %3, %3, %8;\n\t}"
        : "+d"(glo_), "+d"(ghi_), "+r"(lo_bits), "+r"(hi_bits)
        : "d"(v), "d"(t), "d"(yL), "d"(yR), "r"(1u << idx));
  }
  // one element; idx = position inside the thread's group (compaction bookkeeping)
  __device__ __forceinline__ void elem(T v, bool ok, int u, int idx) {
    if (MODE == kHot) {
      // the hot form: no pred/succ (the driver uses them only on small compacted brackets).
      // Predicated PTX: 10 issue slots per element (5 compares, 1 sub, 4 predicated adds).
      if (ok) hot_elem(v, glo[u], ghi[u]);
      return;
    }
    if (MODE == kCompact) {
      // compaction form: no counters (the driver derives c_lt = c_le(yL) + #lo and
      // c_eq = m - #lo - #hi from the compaction totals), no pred/succ; 9 issue slots
      if (ok) compact_elem(v, glo[u], ghi[u], idx);
      vals[idx] = v;
      return;
    }
    const bool lt = v < t;
    const bool gt = v > t;
    const bool lo = ok && lt && (v > yL);
    const bool hi = ok && gt && (v < yR);
    const T d = t - v;
    if (ok) {
      if (lt) ++c_lt;
      if (v == t) ++c_eq;
    }
    if (lo) { glo[u] += d; pred = tmax(pred, v); }
    if (hi) { ghi[u] -= d; succ = tmin(succ, v); }
    if (MODE == kDirect) {
      if (lo) ++c_lo;
      if (hi) ++c_hi;
      if (ok && lt) gN[u] += d;
      if (ok && gt) gP[u] -= d;
    }
  }
  __device__ __forceinline__ void group_begin() {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) { glo[u] = ghi[u] = T(0); if (MODE == kDirect) gP[u] = gN[u] = T(0); }
    if (MODE == kCompact) lo_bits = hi_bits = 0u;
  }
  __device__ __forceinline__ void sum_group() {
    // pairwise combine of the per-vector partials, then one fp64 add (R10)
    T a = glo[0], b = ghi[0], c = gP[0], d = gN[0];
    if (UNROLL == 4) {
      a = (glo[0] + glo[1]) + (glo[2] + glo[3]);
      b = (ghi[0] + ghi[1]) + (ghi[2] + ghi[3]);
      if (MODE == kDirect) { c = (gP[0] + gP[1]) + (gP[2] + gP[3]); d = (gN[0] + gN[1]) + (gN[2] + gN[3]); }
    } else {
#pragma unroll
      for (int u = 1; u < UNROLL; ++u) { a += glo[u]; b += ghi[u]; if (MODE == kDirect) { c += gP[u]; d += gN[u]; } }
    }
    L_lo += (double)a;
    L_hi += (double)b;
    if (MODE == kDirect) { P += (double)c; N += (double)d; }
  }
  T* sbuf;  // smem staging: [0, CAPS) lo, [CAPS, 2 CAPS) hi
  static constexpr int CAPS = stage_elems<T>();
  // coalesced write-out of one staged half (all threads of the CTA call it)
  __device__ __forceinline__ void flush(int side, unsigned cnt) {
    if (threadIdx.x == 0) cs->base[side] = atomicAdd(&cursors[side], (unsigned long long)cnt);
    __syncthreads();
    const uint64_t base = cs->base[side];
    const T* src = sbuf + side * CAPS;
    // (bounded: a speculative compaction — the batched init's ]t_lo, t_hi[ copy — may overflow
    // z_cap; the cursor still counts everything and the caller then does not use the copy)
    if (side == 0) {
      for (unsigned i = threadIdx.x; i < cnt; i += kBlock)
        if (base + i < z_cap) z[base + i] = src[i];
    } else {
      for (unsigned i = threadIdx.x; i < cnt; i += kBlock)
        if (base + i < z_cap) z[z_cap - 1 - (base + i)] = src[i];
    }
    __syncthreads();
  }
  unsigned n_lo = 0, n_hi = 0;  // staged counts (block-uniform, kept in every thread)
  // final flush after the stream (all threads)
  __device__ __forceinline__ void finish() {
    __syncthreads();
    if (n_lo) flush(0, n_lo);
    if (n_hi) flush(1, n_hi);
    n_lo = n_hi = 0;
  }
  // block-synchronous compaction of this group (all threads of the CTA call it): block scan of
  // the (lo, hi) counts, scatter into the smem staging buffers, flush a half when full
  __device__ __forceinline__ void compact_group() {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned packed = (unsigned)__popc(lo_bits) | ((unsigned)__popc(hi_bits) << 16);
    unsigned incl = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) cs->warp_incl[w] = incl;
    __syncthreads();
    if (w == 0) {
      const unsigned tot = lane < kWarps ? cs->warp_incl[lane] : 0u;
      unsigned sc = tot;
#pragma unroll
      for (int o = 1; o < kWarps; o <<= 1) {
        const unsigned y = __shfl_up_sync(FULL, sc, o);
        if (lane >= o) sc += y;
      }
      if (lane < kWarps) cs->warp_excl[lane] = sc - tot;
      if (lane == kWarps - 1) cs->tot = sc;
    }
    __syncthreads();
    const unsigned pre = cs->warp_excl[w] + (incl - packed);
    const unsigned tot = cs->tot;
    unsigned plo = n_lo + (pre & 0xffffu);
    unsigned phi = n_hi + (pre >> 16);
    T* slo = sbuf;
    T* shi = sbuf + CAPS;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if ((lo_bits >> j) & 1u) slo[plo++] = vals[j];
      if ((hi_bits >> j) & 1u) shi[phi++] = vals[j];
    }
    n_lo += tot & 0xffffu;
    n_hi += tot >> 16;
    // a flush is due once another full group might not fit
    constexpr unsigned THR = (unsigned)(CAPS - group_elems<T>());
    if (n_lo > THR || n_hi > THR) {
      __syncthreads();  // staged writes visible
      if (n_lo > THR) { flush(0, n_lo); n_lo = 0; }
      if (n_hi > THR) { flush(1, n_hi); n_hi = 0; }
    }
  }
  __device__ __forceinline__ void group_end() {
    sum_group();
    if (MODE == kCompact) compact_group();
  }
  template <bool MASKED, typename V> __device__ __forceinline__ void vec(const V& v, bool ok, int u) {
#pragma unroll
    for (int j = 0; j < VE; ++j) elem(lane_of(v, j), MASKED ? ok : true, u, u * VE + j);
  }
  // head/tail elements (warp 0 of the last CTA only): compaction by per-element atomics
  __device__ __forceinline__ void scalar(T v, bool ok) {
    group_begin();
    elem(v, ok, 0, 0);
    sum_group();
    if (MODE == kCompact) {
      if (lo_bits & 1u) z[atomicAdd(&cursors[0], 1ull)] = v;
      if (hi_bits & 1u) z[z_cap - 1 - atomicAdd(&cursors[1], 1ull)] = v;
      lo_bits = hi_bits = 0u;
    }
  }
};

template <typename T, int MODE, int UNROLL>
__global__ void __launch_bounds__(kBlock) pass_kernel(PassArgs a) {
  using Fn = PassFn<T, MODE, UNROLL>;
  __shared__ CompactShared cs;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  if (a.ks) {  // device loop: this pass's array and bracket from the loop state
    const KelleyState* ks = a.ks;
    if (ks->done || ks->compact) return;
    a.x = ks->cur; a.n = ks->n_cur; a.t = ks->tq; a.y_lo = ks->yL; a.y_hi = ks->yR;
    a.out = const_cast<DevPass*>(&ks->tuple);
  }
  Fn f;
  f.t = (T)a.t; f.yL = (T)a.y_lo; f.yR = (T)a.y_hi;
  f.c_lt = f.c_eq = f.c_lo = f.c_hi = 0;
  f.L_lo = f.L_hi = f.P = f.N = 0.0;
  f.pred = -tinf<T>(); f.succ = tinf<T>();
  f.lo_bits = f.hi_bits = 0u;
  if (MODE == kCompact) {
    f.cs = &cs;
    f.sbuf = reinterpret_cast<T*>(dyn_smem);
    f.z = static_cast<T*>(a.z);
    f.z_cap = a.z_cap;
    f.cursors = a.cursors;
    if (threadIdx.x == 0) cs.n[0] = cs.n[1] = 0u;
    __syncthreads();
  }
  stream_array<T, UNROLL>(static_cast<const T*>(a.x), a.n, f, blockIdx.x, gridDim.x);
  if (MODE == kCompact) f.finish();
  PassPartial p;
  p.c_lt = f.c_lt; p.c_eq = f.c_eq; p.c_lo = f.c_lo; p.c_hi = f.c_hi;
  p.L_lo = f.L_lo; p.L_hi = f.L_hi; p.P = f.P; p.N = f.N;
  p.pred = (double)f.pred; p.succ = (double)f.succ;
  p = block_reduce(p);
  PassPartial id;
  id.c_lt = id.c_eq = id.c_lo = id.c_hi = 0;
  id.L_lo = id.L_hi = id.P = id.N = 0;
  id.pred = -tinf<double>(); id.succ = tinf<double>();
  PassPartial tot;
  if (grid_finish(p, static_cast<PassPartial*>(a.partials), a.ticket, &tot, id) && threadIdx.x == 0) {
    DevPass r;
    r.c_lt = tot.c_lt; r.c_eq = tot.c_eq; r.c_lo = tot.c_lo; r.c_hi = tot.c_hi;
    r.L_lo = tot.L_lo; r.L_hi = tot.L_hi; r.P = tot.P; r.N = tot.N;
    r.pred = tot.pred; r.succ = tot.succ;
    r.z_lo = r.z_hi = 0;
    if (MODE == kCompact) {
      r.z_lo = atomicAdd(&a.cursors[0], 0ull);
      r.z_hi = atomicAdd(&a.cursors[1], 0ull);
      a.cursors[0] = 0ull;
      a.cursors[1] = 0ull;
    }
    *a.out = r;
    publish_done(a.done, a.seq);
  }
}

// ------------------------------------------------------------------------------------------
// Step a5: radix select on order-preserving keys.

template <typename T> struct HistFn {
  unsigned* sh;
  unsigned long long prefix, mask;
  int shift;
  unsigned dmask;
  __device__ __forceinline__ void elem(T v, bool ok) {
    if constexpr (sizeof(T) == 4) {
      const unsigned u = __float_as_uint(v);
      const unsigned k = u ^ ((unsigned)((int)u >> 31) | 0x80000000u);
      if (ok && (k & (unsigned)mask) == (unsigned)prefix) atomicAdd(&sh[(k >> shift) & dmask], 1u);
    } else {
      const unsigned long long k = okey(v);
      if (ok && (k & mask) == prefix) atomicAdd(&sh[(unsigned)(k >> shift) & dmask], 1u);
    }
  }
  __device__ __forceinline__ void group_begin() {}
  __device__ __forceinline__ void group_end() {}
  template <bool MASKED, typename V> __device__ __forceinline__ void vec(const V& v, bool ok, int) {
#pragma unroll
    for (int j = 0; j < VecOf<T>::N; ++j) elem(lane_of(v, j), MASKED ? ok : true);
  }
  __device__ __forceinline__ void scalar(T v, bool ok) { elem(v, ok); }
};

template <typename T, int MODE> constexpr size_t pass_smem() { return MODE == kCompact ? compact_smem_bytes<T>() : 0; }

template <typename T, int MODE>
cudaError_t launch_pass_t(const PassArgs& a, int grid, cudaStream_t st) {
  pass_kernel<T, MODE, 4><<<grid, kBlock, pass_smem<T, MODE>(), st>>>(a);
  return cudaGetLastError();
}

template <typename T, int MODE> cudaError_t occ_pass(int* blocks) {
  if (pass_smem<T, MODE>() > 0) {  // dynamic + static smem may exceed the 48 KB default
    cudaError_t e = cudaFuncSetAttribute(pass_kernel<T, MODE, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)pass_smem<T, MODE>());
    if (e != cudaSuccess) return e;
  }
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, pass_kernel<T, MODE, 4>, kBlock, pass_smem<T, MODE>());
}


// ------------------------------------------------------------------------------------------
// Step a2+a4, segmented form: warp-private compaction (no atomics for regions, no block barriers).
constexpr int kSegU = 4;  // vectors per lane per group

// INSIDE: every input element is known to lie strictly inside ]y_lo, y_hi[ (the input is a kept
// half of an earlier compaction), so the bracket tests are skipped (7 issue slots per element).
template <typename T, bool INSIDE> struct WarpSeg {
  static constexpr int VE = VecOf<T>::N;
  static constexpr int G = kSegU * VE;       // elements per lane per group
  static constexpr int GW = 32 * G;          // elements per warp per group
  T t, yL, yR;
  T vals[G];
  unsigned lo_bits, hi_bits;
  T glo[kSegU], ghi[kSegU];
  double L_lo, L_hi;
  unsigned long long n_lo, n_hi;             // warp-uniform: elements written so far
  T* stage;                                  // this warp's smem: [0,GW) lo, [GW,2GW) hi
  // output
  int dense;
  T* out;
  uint64_t reg_lo, reg_end;                  // region [reg_lo, reg_end) (segmented out)
  unsigned long long* cursors;               // dense out
  uint64_t z_cap;

  __device__ __forceinline__ void elem(float v, int u, int idx) {
    if (INSIDE) {
      asm("{\n\t.reg .pred plo, phi;\n\t.reg .f32 d;\n\t"
          "setp.lt.f32 plo, %4, %5;\n\t"
          "setp.gt.f32 phi, %4, %5;\n\t"
          "sub.rn.f32 d, %5, %4;\n\t"
          "@plo add.rn.f32 %0, %0, d;\n\t"
          "@phi sub.rn.f32 %1, %1, d;\n\t"
          "@plo or.b32 %2, %2, %6;\n\t"
          "@phi or.b32 %3, %3, %6;\n\t}"
          : "+f"(glo[u]), "+f"(ghi[u]), "+r"(lo_bits), "+r"(hi_bits)
          : "f"(v), "f"(t), "r"(1u << idx));
      vals[idx] = v;
      return;
    }
    asm("{\n\t.reg .pred plt, pgt, plo, phi;\n\t.reg .f32 d;\n\t"
        "setp.lt.f32 plt, %4, %5;\n\t"
        "setp.gt.f32 pgt, %4, %5;\n\t"
        "setp.gt.and.f32 plo, %4, %6, plt;\n\t"
        "setp.lt.and.f32 phi, %4, %7, pgt;\n\t"
        "sub.rn.f32 d, %5, %4;\n\t"
        "@plo add.rn.f32 %0, %0, d;\n\t"
        "@phi sub.rn.f32 %1, %1, d;\n\t"
        "@plo or.b32 %2, %2, %8;\n\t"
        "@phi or.b32 %3, %3, %8;\n\t}"
        : "+f"(glo[u]), "+f"(ghi[u]), "+r"(lo_bits), "+r"(hi_bits)
        : "f"(v), "f"(t), "f"(yL), "f"(yR), "r"(1u << idx));
    vals[idx] = v;
  }
  __device__ __forceinline__ void elem(double v, int u, int idx) {
    if (INSIDE) {
      asm("{\n\t.reg .pred plo, phi;\n\t.reg .f64 d;\n\t"
          "setp.lt.f64 plo, %4, %5;\n\t"
          "setp.gt.f64 phi, %4, %5;\n\t"
          "sub.rn.f64 d, %5, %4;\n\t"
          "@plo add.rn.f64 %0, %0, d;\n\t"
          "@phi sub.rn.f64 %1, %1, d;\n\t"
          "@plo or.b32 %2, %2, %6;\n\t"
          "@phi or.b32 %3, %3, %6;\n\t}"
          : "+d"(glo[u]), "+d"(ghi[u]), "+r"(lo_bits), "+r"(hi_bits)
          : "d"(v), "d"(t), "r"(1u << idx));
      vals[idx] = v;
      return;
    }
    asm("{\n\t.reg .pred plt, pgt, plo, phi;\n\t.reg .f64 d;\n\t"
        "setp.lt.f64 plt, %4, %5;\n\t"
        "setp.gt.f64 pgt, %4, %5;\n\t"
        "setp.gt.and.f64 plo, %4, %6, plt;\n\t"
        "setp.lt.and.f64 phi, %4, %7, pgt;\n\t"
        "sub.rn.f64 d, %5, %4;\n\t"
        "@plo add.rn.f64 %0, %0, d;\n\t"
        "@phi sub.rn.f64 %1, %1, d;\n\t"
        "@plo or.b32 %2, %2, %8;\n\t"
        "@phi or.b32 %3, %3, %8;\n\t}"
        : "+d"(glo[u]), "+d"(ghi[u]), "+r"(lo_bits), "+r"(hi_bits)
        : "d"(v), "d"(t), "d"(yL), "d"(yR), "r"(1u << idx));
    vals[idx] = v;
  }
  __device__ __forceinline__ void begin() {
#pragma unroll
    for (int u = 0; u < kSegU; ++u) glo[u] = ghi[u] = T(0);
    lo_bits = hi_bits = 0u;
  }
  // close a group: sums to fp64, warp scan of the counts, stage, write-out.  Each half is staged at
  // the 16-byte phase of its destination, so its aligned middle leaves shared memory as 16-byte
  // vectors (LDS.128 -> STG.128, one instruction pair per 4 f32 / 2 f64 written) and only the
  // < 16-byte head and tail as scalars.  (A cp.async.bulk store of the middle measured slower: one
  // ~1 KB bulk copy per half-group per warp queues on the SM's TMA unit.)
  static constexpr unsigned VA = 16 / sizeof(T);  // elements per 16 bytes
  static constexpr int GWP = GW + VA;               // staging of one half, phase padding included
  // dst[i] <- staged element i (shared-window address sa of element 0); dst and sa have the same
  // 16-byte phase
  __device__ __forceinline__ void flush(T* dst, unsigned sa, unsigned cnt) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned ph = (unsigned)(reinterpret_cast<uintptr_t>(dst) / sizeof(T)) & (VA - 1u);
    unsigned head = (VA - ph) & (VA - 1u);
    if (head > cnt) head = cnt;
    const unsigned nv = (cnt - head) / VA, tail = cnt - head - nv * VA;
    if (lane < head) dst[lane] = ld_sh(sa + lane * (unsigned)sizeof(T));
    const unsigned t0 = head + nv * VA;
    if (lane < tail) dst[t0 + lane] = ld_sh(sa + (t0 + lane) * (unsigned)sizeof(T));
    char* dv = reinterpret_cast<char*>(dst + head);
    const unsigned sv = sa + head * (unsigned)sizeof(T);
    for (unsigned i = lane; i < nv; i += 32) {
      unsigned r0, r1, r2, r3;
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(sv + 16 * i));
      asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(dv + 16 * (size_t)i), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                   : "memory");
    }
  }
  __device__ __forceinline__ static T ld_sh(unsigned a) {
    if constexpr (sizeof(T) == 4) {
      unsigned v;
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
      return __uint_as_float(v);
    } else {
      unsigned long long v;
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
      return __longlong_as_double(v);
    }
  }
  // staging of element j: to the lo half (bit j of lo_bits), the hi half, or nowhere — predicated
  // shared stores with post-incremented addresses (no branches)
  template <int J> __device__ __forceinline__ void stage_elem(unsigned& alo, unsigned& ahi) {
    if constexpr (sizeof(T) == 4) {
      asm volatile("{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\t"
                   "and.b32 t, %2, %4;\n\t"
                   "setp.ne.u32 p, t, 0;\n\t"
                   "and.b32 t, %3, %4;\n\t"
                   "setp.ne.u32 q, t, 0;\n\t"
                   "@p st.shared.b32 [%0], %5;\n\t"
                   "@p add.u32 %0, %0, 4;\n\t"
                   "@q st.shared.b32 [%1], %5;\n\t"
                   "@q add.u32 %1, %1, 4;\n\t}"
                   : "+r"(alo), "+r"(ahi)
                   : "r"(lo_bits), "r"(hi_bits), "n"(1u << J), "r"(__float_as_uint((float)vals[J]))
                   : "memory");
    } else {
      asm volatile("{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\t"
                   "and.b32 t, %2, %4;\n\t"
                   "setp.ne.u32 p, t, 0;\n\t"
                   "and.b32 t, %3, %4;\n\t"
                   "setp.ne.u32 q, t, 0;\n\t"
                   "@p st.shared.b64 [%0], %5;\n\t"
                   "@p add.u32 %0, %0, 8;\n\t"
                   "@q st.shared.b64 [%1], %5;\n\t"
                   "@q add.u32 %1, %1, 8;\n\t}"
                   : "+r"(alo), "+r"(ahi)
                   : "r"(lo_bits), "r"(hi_bits), "n"(1u << J), "l"(__double_as_longlong((double)vals[J]))
                   : "memory");
    }
  }
  template <int J> __device__ __forceinline__ void stage_all(unsigned& alo, unsigned& ahi) {
    if constexpr (J < G) {
      stage_elem<J>(alo, ahi);
      stage_all<J + 1>(alo, ahi);
    }
  }
  __device__ __forceinline__ void end() {
    L_lo += (double)((glo[0] + glo[1]) + (glo[2] + glo[3]));
    L_hi += (double)((ghi[0] + ghi[1]) + (ghi[2] + ghi[3]));
    const int lane = threadIdx.x & 31;
    const unsigned packed = (unsigned)__popc(lo_bits) | ((unsigned)__popc(hi_bits) << 16);
    unsigned incl = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned tot = __shfl_sync(FULL, incl, 31);
    if (tot == 0u) return;
    const unsigned nlo = tot & 0xffffu, nhi = tot >> 16;
    T* dlo;
    T* dhi;
    if (dense) {
      unsigned long long blo = 0, bhi = 0;
      if (lane == 0) {
        if (nlo) blo = atomicAdd(&cursors[0], (unsigned long long)nlo);
        if (nhi) bhi = atomicAdd(&cursors[1], (unsigned long long)nhi);
      }
      blo = __shfl_sync(FULL, blo, 0);
      bhi = __shfl_sync(FULL, bhi, 0);
      dlo = out + blo;
      dhi = out + (z_cap - bhi - nhi);
    } else {
      dlo = out + reg_lo + n_lo;
      dhi = out + (reg_end - n_hi - nhi);
    }
    const unsigned phlo = (unsigned)(reinterpret_cast<uintptr_t>(dlo) / sizeof(T)) & (VA - 1u);
    const unsigned phhi = (unsigned)(reinterpret_cast<uintptr_t>(dhi) / sizeof(T)) & (VA - 1u);
    const unsigned slo = smem_u32(stage) + phlo * (unsigned)sizeof(T);
    const unsigned shi = smem_u32(stage) + (GWP + phhi) * (unsigned)sizeof(T);
    const unsigned pre = incl - packed;
    unsigned alo = slo + (pre & 0xffffu) * (unsigned)sizeof(T), ahi = shi + (pre >> 16) * (unsigned)sizeof(T);
    stage_all<0>(alo, ahi);
    __syncwarp();
    if (nlo) flush(dlo, slo, nlo);
    if (nhi) flush(dhi, shi, nhi);
    __syncwarp();  // the staging buffer is free for the next group
    n_lo += nlo;
    n_hi += nhi;
  }
};

// one warp, one group of up to 32*kSegU vectors starting at vector index v0 (lane-strided)
template <typename T, bool MASKED, typename F>
__device__ __forceinline__ void seg_group(F& f, const typename VecOf<T>::V* __restrict__ xv, uint64_t v0,
                                          uint64_t nvec) {
  using V = typename VecOf<T>::V;
  constexpr int VE = VecOf<T>::N;
  const int lane = threadIdx.x & 31;
  V v[kSegU];
  bool ok[kSegU];
#pragma unroll
  for (int u = 0; u < kSegU; ++u) {
    const uint64_t i = v0 + (uint64_t)u * 32 + lane;
    ok[u] = !MASKED || i < nvec;
    if (ok[u]) v[u] = ld_stream(xv + i);
  }
  f.begin();
#pragma unroll
  for (int u = 0; u < kSegU; ++u) {
    if (ok[u]) {
#pragma unroll
      for (int j = 0; j < VE; ++j) f.elem(lane_of(v[u], j), u, u * VE + j);
    }
  }
  f.end();
}

// up to 32 scattered scalars (one per lane): x[idx] for lanes with ok
template <typename T, typename F>
__device__ __forceinline__ void seg_scalars(F& f, T v, bool ok) {
  f.begin();
  if (ok) f.elem(v, 0, 0);
  f.end();
}

// a whole contiguous run [p, p+c) processed by one warp
template <typename T, typename F>
__device__ __forceinline__ void seg_run(F& f, const T* __restrict__ p, uint64_t c) {
  using V = typename VecOf<T>::V;
  constexpr int VE = VecOf<T>::N;
  const int lane = threadIdx.x & 31;
  const uint64_t mis = (reinterpret_cast<uintptr_t>(p) / sizeof(T)) & (VE - 1);
  uint64_t head = mis ? (VE - mis) : 0;
  if (head > c) head = c;
  const V* xv = reinterpret_cast<const V*>(p + head);
  const uint64_t nvec = (c - head) / VE;
  const uint64_t tail0 = head + nvec * VE, ntail = c - tail0;
  // head and tail scalars (< VE each) in one masked group
  {
    const bool okh = (uint64_t)lane < head;
    const bool okt = (uint64_t)lane >= head && (uint64_t)lane < head + ntail;
    T v = T(0);
    if (okh) v = p[lane];
    if (okt) v = p[tail0 + (lane - head)];
    if (head + ntail) seg_scalars<T>(f, v, okh || okt);
  }
  constexpr uint64_t GV = 32 * kSegU;
  uint64_t v0 = 0;
  for (; v0 + GV <= nvec; v0 += GV) seg_group<T, false>(f, xv, v0, nvec);
  if (v0 < nvec) seg_group<T, true>(f, xv, v0, nvec);
}

// The same with the loads software-pipelined: the next group's vectors are in flight while the
// current group is processed (a warp streams a whole run by itself, so without this every group is
// one dependent memory round trip) — the radix rounds over the init's segmented copy.
template <typename T, typename F>
__device__ __forceinline__ void seg_run_pipe(F& f, const T* __restrict__ p, uint64_t c) {
  using V = typename VecOf<T>::V;
  constexpr int VE = VecOf<T>::N;
  const int lane = threadIdx.x & 31;
  const uint64_t mis = (reinterpret_cast<uintptr_t>(p) / sizeof(T)) & (VE - 1);
  uint64_t head = mis ? (VE - mis) : 0;
  if (head > c) head = c;
  const V* xv = reinterpret_cast<const V*>(p + head);
  const uint64_t nvec = (c - head) / VE;
  const uint64_t tail0 = head + nvec * VE, ntail = c - tail0;
  {
    const bool okh = (uint64_t)lane < head;
    const bool okt = (uint64_t)lane >= head && (uint64_t)lane < head + ntail;
    T v = T(0);
    if (okh) v = p[lane];
    if (okt) v = p[tail0 + (lane - head)];
    if (head + ntail) seg_scalars<T>(f, v, okh || okt);
  }
  constexpr uint64_t GV = 32 * kSegU;
  const uint64_t nfull = nvec / GV;
  V cur[kSegU];
  if (nfull > 0) {
#pragma unroll
    for (int u = 0; u < kSegU; ++u) cur[u] = ld_stream(xv + (uint64_t)u * 32 + lane);
  }
  for (uint64_t g = 0; g < nfull; ++g) {
    V nxt[kSegU];
    if (g + 1 < nfull) {
#pragma unroll
      for (int u = 0; u < kSegU; ++u) nxt[u] = ld_stream(xv + (g + 1) * GV + (uint64_t)u * 32 + lane);
    }
    f.begin();
#pragma unroll
    for (int u = 0; u < kSegU; ++u) {
#pragma unroll
      for (int j = 0; j < VE; ++j) f.elem(lane_of(cur[u], j), u, u * VE + j);
    }
    f.end();
#pragma unroll
    for (int u = 0; u < kSegU; ++u) cur[u] = nxt[u];
  }
  if (nfull * GV < nvec) seg_group<T, true>(f, xv, nfull * GV, nvec);
}

// ------------------------------------------------------------------------------------------
// Step a5, one launch per digit: the histogram of the digit over the prefix class, then the last
// CTA to finish picks the digit holding the rank, extends the prefix and clears the histogram
// (no separate pick / init launches).  Input: contiguous z[0..m) or the runs `side` of a segmented
// array (one warp per run, the segmented grid).
struct RadixSegFn {
  unsigned* sh;
  unsigned sh_sa;  // shared-window address of sh
  unsigned long long prefix, mask;
  int shift;
  unsigned dmask;
  template <typename T> __device__ __forceinline__ void elem(T v, int, int) {
    if constexpr (sizeof(T) == 4) {  // 32-bit key arithmetic, predicated reduction (no branch)
      const unsigned u = __float_as_uint(v);
      const unsigned k = u ^ ((unsigned)((int)u >> 31) | 0x80000000u);
      const unsigned addr = sh_sa + 4u * ((k >> shift) & dmask);
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "setp.eq.u32 p, %0, %1;\n\t"
          "@p red.shared.add.u32 [%2], 1;\n\t}" ::"r"(k & (unsigned)mask),
          "r"((unsigned)prefix), "r"(addr)
          : "memory");
    } else {
      const unsigned long long k = okey(v);
      if ((k & mask) == prefix) atomicAdd(&sh[(unsigned)(k >> shift) & dmask], 1u);
    }
  }
  __device__ __forceinline__ void begin() {}
  __device__ __forceinline__ void end() {}
};

struct RadixArgs {
  const KelleyState* ks;  // device loop: the exact finish's input, rank and mailbox seq from *ks
  const void* z;
  uint64_t m;
  const SegEntry* tab;  // nullptr: contiguous
  int side;
  int Wtot;             // segmented: runs in tab
  RadixState* st;
  unsigned* hist;       // 2048 global digit counters, zero between rounds
  unsigned* ticket;
  int shift, bits, first, last;
  uint64_t r;           // the rank (1-based), taken by the first round
  const ChainState* chain;  // device chain: skip unless chain->ok[1]; rank chain->r[1]
  unsigned* hist0;          // round-0 counts taken by the init pass (this launch is round 1), or nullptr
  double* vout;
  unsigned long long* done;
  unsigned long long seq;
};

template <typename T, bool SEG>
__global__ void __launch_bounds__(kBlock) radix_round_kernel(RadixArgs a) {
  pdl_wait();     // the previous round's digit / the init's copy and chain decision
  pdl_trigger();  // the next round may be scheduled (it waits for this grid to finish)
  if (a.ks) {
    a.z = a.ks->sel_base; a.m = a.ks->sel_m; a.tab = a.ks->sel_tab; a.side = a.ks->sel_side;
    a.r = a.ks->sel_r; a.seq = a.ks->seq;
    a.vout = a.ks->vout; a.done = a.ks->done_flag;
  }
  if (a.chain) {
    if (!a.chain->ok[1]) {  // skipped: the init's round-0 counts must still be cleared
      if (a.hist0 && blockIdx.x == 0)
        for (int i = threadIdx.x; i < 2048; i += kBlock) a.hist0[i] = 0u;
      return;
    }
    a.r = a.chain->r[1];
  }
  __shared__ unsigned sh[2048];
  __shared__ unsigned long long s_prefix, s_mask, s_rank;
  __shared__ bool s_last;
  __shared__ unsigned wsum[kWarps];
  if (a.hist0) {
    // round 0 was counted by the init pass into hist0: every CTA picks its digit for rank a.r
    // (the same result everywhere), so no launch or serial tail is spent on it
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned h[8], tsum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      h[j] = __ldcg(&a.hist0[threadIdx.x * 8 + j]);
      tsum += h[j];
    }
    unsigned incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    unsigned wbase = 0;
    for (int q = 0; q < w; ++q) wbase += wsum[q];
    unsigned long long before = wbase + incl - tsum;
    const int sh0 = sizeof(T) == 4 ? 21 : 53;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (before < a.r && a.r <= before + h[j]) {
        s_prefix = (unsigned long long)(threadIdx.x * 8 + j) << sh0;
        s_mask = 2047ull << sh0;
        s_rank = a.r - before;
      }
      before += h[j];
    }
  } else if (threadIdx.x == 0) {
    s_prefix = a.first ? 0ull : a.st->prefix;
    s_mask = a.first ? 0ull : a.st->mask;
    s_rank = a.first ? a.r : a.st->r;
  }
  for (int i = threadIdx.x; i < 2048; i += kBlock) sh[i] = 0;
  __syncthreads();
  RadixSegFn f;
  f.sh = sh;
  f.sh_sa = (unsigned)__cvta_generic_to_shared(sh);
  f.prefix = s_prefix;
  f.mask = s_mask;
  f.shift = a.shift;
  f.dmask = (1u << a.bits) - 1u;
  if (SEG) {
    // a warp per run; a grid smaller than the segmented one (a small copy) loops over the runs
    for (uint64_t W = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); W < (uint64_t)a.Wtot;
         W += (uint64_t)gridDim.x * kWarps) {
      const SegEntry e = a.tab[W];
      seg_run_pipe<T>(f, static_cast<const T*>(a.z) + e.off[a.side], e.cnt[a.side]);
    }
  } else {
    HistFn<T> hf;
    hf.sh = sh; hf.prefix = s_prefix; hf.mask = s_mask; hf.shift = a.shift; hf.dmask = f.dmask;
    stream_array<T, 2>(static_cast<const T*>(a.z), a.m, hf, blockIdx.x, gridDim.x);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += kBlock)
    if (sh[i]) atomicAdd(&a.hist[i], sh[i]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the pick: 8 bins per thread, block scan of the thread totals
  const int nb = 1 << a.bits;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned h[8];
  unsigned tsum = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int b = threadIdx.x * 8 + j;
    h[j] = b < nb ? __ldcg(&a.hist[b]) : 0u;
    tsum += h[j];
  }
  unsigned incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  unsigned wbase = 0;
  for (int q = 0; q < w; ++q) wbase += wsum[q];
  const unsigned long long r = s_rank;
  unsigned long long before = wbase + incl - tsum;  // exclusive prefix of this thread's first bin
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (before < r && r <= before + h[j]) {
      const int digit = threadIdx.x * 8 + j;
      const unsigned long long dmask = (unsigned long long)(nb - 1) << a.shift;
      const unsigned long long prefix = s_prefix | ((unsigned long long)digit << a.shift);
      a.st->prefix = prefix;
      a.st->mask = s_mask | dmask;
      a.st->r = r - before;
      a.st->count = h[j];
      if (a.last) {
        a.st->key = prefix;
        a.st->value = (sizeof(T) == 4) ? from_key_f32(prefix) : from_key_f64(prefix);
        if (a.vout) *a.vout = a.st->value;
        publish_done(a.done, a.seq);
      }
    }
    before += h[j];
  }
  for (int i = threadIdx.x; i < 2048; i += kBlock) a.hist[i] = 0u;
  if (a.hist0)  // every CTA read it before taking its ticket
    for (int i = threadIdx.x; i < 2048; i += kBlock) a.hist0[i] = 0u;
  if (threadIdx.x == 0) *a.ticket = 0u;
}

// ------------------------------------------------------------------------------------------
// Step a5, all digit rounds in ONE cooperative launch (the grid is co-resident): per round every CTA
// counts its share into shared memory and merges the nonzero bins into a global histogram (one of
// three, rotating), a grid barrier, then EVERY CTA picks the digit from that histogram itself (the
// same bytes, the same pick) and the next round starts — no launch, no last-CTA tail per round.
// The first round's buffer of the next round is cleared before the barrier (nobody adds to it until
// after), the one two rounds back is free by then; the last CTA out clears all three and hist0.
struct RadixPlan {
  int n;
  int shift[6], bits[6];
};
struct CoopArgs {
  RadixArgs a;
  RadixPlan plan;
  int first_round;
  unsigned* g3;   // 3 x 2048 global digit counters (zero on entry, left zero)
  unsigned* bar;  // [0] arrivals, [1] generation, [2] exit ticket (zero on entry, left zero)
};
__device__ __forceinline__ void coop_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}
// NT threads per CTA: 256 (4 CTAs per SM, the segmented grid's shape) or 1024 (one CTA per SM: a
// quarter of the CTAs to merge histograms and to cross the grid barrier, every warp still on one run)
template <typename T, bool SEG, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) radix_coop_kernel(const __grid_constant__ CoopArgs c) {
  constexpr int NW = NT / 32, BPT = 2048 / NT;  // warps, bins per thread of the pick
  const RadixArgs& a = c.a;
  pdl_wait();  // the init's copy, its round-0 counts and the chain decision
  uint64_t rank0 = a.r;
  if (a.chain) {
    if (!a.chain->ok[1]) {  // skipped (uniformly): the init's round-0 counts must still be cleared
      if (a.hist0 && blockIdx.x == 0)
        for (int i = threadIdx.x; i < 2048; i += NT) a.hist0[i] = 0u;
      return;
    }
    rank0 = a.chain->r[1];
  }
  __shared__ unsigned sh[2048];
  __shared__ unsigned long long s_prefix, s_mask, s_rank;
  __shared__ unsigned wsum[NW];
  __shared__ bool s_last;
  __shared__ int s_shift[6], s_bits[6];
  if (threadIdx.x < 6) {
    s_shift[threadIdx.x] = c.plan.shift[threadIdx.x];
    s_bits[threadIdx.x] = c.plan.bits[threadIdx.x];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // the digit holding rank r in a 2048-bin histogram h (global, read with ld.cg), as one block:
  // 8 bins per thread, block scan of the thread totals; the finder updates the shared prefix
  auto pick = [&](const unsigned* h, int shift, int bits, bool last) {
    const int nb = 1 << bits;
    unsigned hv[BPT], tsum = 0;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      const int b = threadIdx.x * BPT + j;
      hv[j] = b < nb ? __ldcg(&h[b]) : 0u;
      tsum += hv[j];
    }
    unsigned incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    const unsigned long long r = s_rank, pf = s_prefix, mk = s_mask;
    __syncthreads();
    unsigned wbase = 0;
    for (int q = 0; q < w; ++q) wbase += wsum[q];
    unsigned long long before = wbase + incl - tsum;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      if (before < r && r <= before + hv[j]) {
        const int digit = threadIdx.x * BPT + j;
        const unsigned long long prefix = pf | ((unsigned long long)digit << shift);
        s_prefix = prefix;
        s_mask = mk | ((unsigned long long)(nb - 1) << shift);
        s_rank = r - before;
        if (last && blockIdx.x == 0) {
          a.st->prefix = prefix;
          a.st->mask = s_mask;
          a.st->r = r - before;
          a.st->count = hv[j];
          a.st->key = prefix;
          a.st->value = (sizeof(T) == 4) ? from_key_f32(prefix) : from_key_f64(prefix);
          if (a.vout) *a.vout = a.st->value;
          publish_done(a.done, a.seq);
        }
      }
      before += hv[j];
    }
    __syncthreads();
  };
  if (threadIdx.x == 0) {
    s_prefix = 0ull;
    s_mask = 0ull;
    s_rank = rank0;
  }
  __syncthreads();
  if (a.hist0) pick(a.hist0, s_shift[0], s_bits[0], false);  // round 0 counted by the init pass
  for (int ri = c.first_round; ri < c.plan.n; ++ri) {
    const int shift = s_shift[ri], bits = s_bits[ri];
    unsigned* G = c.g3 + 2048 * (ri % 3);
    for (int i = threadIdx.x; i < 2048; i += NT) sh[i] = 0;
    __syncthreads();
    if (SEG) {
      RadixSegFn f;
      f.sh = sh;
      f.sh_sa = (unsigned)__cvta_generic_to_shared(sh);
      f.prefix = s_prefix;
      f.mask = s_mask;
      f.shift = shift;
      f.dmask = (1u << bits) - 1u;
      for (uint64_t W = (uint64_t)blockIdx.x * NW + w; W < (uint64_t)a.Wtot; W += (uint64_t)gridDim.x * NW) {
        const SegEntry e = a.tab[W];
        seg_run_pipe<T>(f, static_cast<const T*>(a.z) + e.off[a.side], e.cnt[a.side]);
      }
    } else {
      HistFn<T> hf;
      hf.sh = sh; hf.prefix = s_prefix; hf.mask = s_mask; hf.shift = shift; hf.dmask = (1u << bits) - 1u;
      stream_array<T, 2>(static_cast<const T*>(a.z), a.m, hf, blockIdx.x, gridDim.x);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += NT)
      if (sh[i]) atomicAdd(&G[i], sh[i]);
    if (blockIdx.x == 0)  // next round's buffer: last read two barriers ago, added to only after this one
      for (int i = threadIdx.x; i < 2048; i += NT) c.g3[2048 * ((ri + 1) % 3) + i] = 0u;
    coop_barrier(c.bar, gridDim.x);
    pick(G, shift, bits, ri == c.plan.n - 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(c.bar + 2, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  for (int i = threadIdx.x; i < 3 * 2048; i += NT) c.g3[i] = 0u;
  if (a.hist0)
    for (int i = threadIdx.x; i < 2048; i += NT) a.hist0[i] = 0u;
  if (threadIdx.x == 0) c.bar[2] = 0u;
}

// ------------------------------------------------------------------------------------------
// Step a5 behind the vbin init (launch_vbin_finish): the init counted its copy per VALUE bin of
// ]t_lo, t_hi[ (2048 equal widths: for any smooth density near the target each bin holds ~1/2048 of
// the copy, where the top key digits put most of it in one or two bins), so after the bin pick only a
// few thousand elements remain: one pass over the copy takes their key range (and copies them if
// they fit), the last CTA selects among them in shared memory.  No grid barrier, no second pass.
struct VbArgs {
  const void* z;
  const SegEntry* tab;
  int Wtot;
  const void* cuts;          // t_lo, t_hi (the init's)
  unsigned* hist0;           // the init's 2048 first-digit counts (cleared here)
  unsigned long long* st;    // [0] ticket, [1] copied count, [2] ~min key, [3] max key (left zero)
  void* zb;                  // kVbCap elements: the target bin's copy
  const ChainState* chain;
  double* vout;
  unsigned long long* fallback;
  unsigned long long* done;
  unsigned long long seq;
};
template <typename T> struct VbFn {
  T lo, hi;     // a value interval holding bin b (a superset: vb_bounds), tested first
  T tl, sc;     // the exact bin test on the few values inside it
  unsigned b;
  bool comp;
  unsigned long long kmin = ~0ull, kmax = 0ull;
  unsigned long long* cnt;
  T* zb;
  // one vector of VE values: two compares per value, one rarely taken branch per vector
  template <int VE> __device__ __forceinline__ void vec(const T (&v)[VE]) {
    bool any = false;
#pragma unroll
    for (int j = 0; j < VE; ++j) any |= v[j] >= lo && v[j] <= hi;
    if (any) {
#pragma unroll
      for (int j = 0; j < VE; ++j) elem(v[j], 0, 0);
    }
  }
  __device__ __forceinline__ void elem(T v, int, int) {
    if (v >= lo && v <= hi && vbin_digit(v, tl, sc) == b) {
      const unsigned long long k = okey(v);
      kmin = k < kmin ? k : kmin;
      kmax = k > kmax ? k : kmax;
      if (comp) {
        const unsigned long long i = atomicAdd(cnt, 1ull);
        if (i < (unsigned long long)kVbCap) zb[i] = v;
      }
    }
  }
};
// A value interval [lo, hi] containing every v of ]tl, th[ whose vbin_digit is b (more is harmless:
// the exact digit test follows).  Value bins: the digit's two roundings move (v - tl) * sc by less
// than 2^-p * 2048 * 2 bins (p = 24 / 53), so bin b lies in tl + [b - 1/2, b + 3/2] / sc, evaluated
// in double (f32: |tl| * sc < 2048 * 2^23, error < 10^-6 bins; f64: within 0.02 bins while
// |tl| * sc, |th| * sc < 10^14, else the whole span) and rounded outward to T.  Key digits (sc = 0):
// the values of the key class [b << S, (b + 1) << S).
template <typename T> __device__ __forceinline__ void vb_bounds(T tl, T th, T sc, unsigned b, T& lo, T& hi) {
  if (sc > T(0)) {
    const double dtl = (double)tl, dsc = (double)sc;
    if (sizeof(T) == 8 && !(fabs(dtl) * dsc < 1e14 && fabs((double)th) * dsc < 1e14)) {
      lo = tl; hi = th;
      return;
    }
    const double l = dtl + ((double)b - 0.5) / dsc, h = b >= 2047u ? (double)th : dtl + ((double)b + 1.5) / dsc;
    if (sizeof(T) == 4) {
      lo = (T)__double2float_rd(l);
      hi = (T)__double2float_ru(h);
    } else {
      lo = (T)l; hi = (T)h;
    }
  } else {
    constexpr int S = sizeof(T) == 4 ? 21 : 53;
    using K = typename SampleKey<T>::K;
    lo = SampleKey<T>::val((K)b << S);
    hi = SampleKey<T>::val((((K)b + 1) << S) - 1);  // b = 2047: the key of the largest NaN, harmless
    if (b == 2047u) hi = th;
    if (!(lo == lo)) lo = -tinf<T>();  // a class of NaN keys below -inf / above +inf
    if (!(hi == hi)) hi = tinf<T>();
  }
}
// the digit of a 2048-bin block histogram h (nb bins) holding rank r (1-based): 1024 threads, two
// bins each; returns (in shared memory) the digit and the count before it
__device__ __forceinline__ void pick1024(const unsigned* h, int nb, unsigned long long r, unsigned* wsum,
                                         unsigned* s_d, unsigned long long* s_before, unsigned* s_cnt,
                                         bool global) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b0 = 2 * threadIdx.x;
  const unsigned h0 = b0 < nb ? (global ? __ldcg(&h[b0]) : h[b0]) : 0u;
  const unsigned h1 = b0 + 1 < nb ? (global ? __ldcg(&h[b0 + 1]) : h[b0 + 1]) : 0u;
  const unsigned tsum = h0 + h1;
  unsigned incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  const unsigned long long ws = wsum[lane];  // the 32 warp totals, scanned by every warp
  unsigned long long wi = ws;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(FULL, wi, o);
    if (lane >= o) wi += y;
  }
  unsigned long long before = __shfl_sync(FULL, wi - ws, w);
  before += incl - tsum;
  if (before < r && r <= before + h0) {
    *s_d = (unsigned)b0; *s_before = before; *s_cnt = h0;
  } else if (before + h0 < r && r <= before + tsum) {
    *s_d = (unsigned)b0 + 1u; *s_before = before + h0; *s_cnt = h1;
  }
  __syncthreads();
}
#ifdef CPSEL_VB_PROF
__device__ unsigned long long g_vbprof[16];
#define VBT(i)                                                                  \
  if (threadIdx.x == 0) {                                                       \
    unsigned long long t_;                                                      \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
    atomicMin(&g_vbprof[2 * (i)], t_ | 0ull);                                   \
    atomicMax(&g_vbprof[2 * (i) + 1], t_);                                      \
  }
#else
#define VBT(i)
#endif
template <typename T>
__global__ void __launch_bounds__(1024, 1) vbin_finish_kernel(const __grid_constant__ VbArgs a) {
  constexpr int NW = 32;
  pdl_wait();  // the init's copy, its bin counts and the chain decision
  VBT(0);
  if (a.chain && !a.chain->ok[1]) {  // skipped (uniformly): the init's counts must still be cleared
    if (blockIdx.x == 0)
      for (int i = threadIdx.x; i < 2048; i += 1024) a.hist0[i] = 0u;
    return;
  }
  const unsigned long long r = a.chain->r[1];
  __shared__ unsigned wsum[NW];
  __shared__ unsigned s_b, s_cb, s_d, s_dc;
  __shared__ unsigned long long s_base, s_bef, s_kmin[NW], s_kmax[NW];
  __shared__ bool s_last;
  pick1024(a.hist0, 2048, r, wsum, &s_b, &s_base, &s_cb, true);
  const T* cuts = static_cast<const T*>(a.cuts);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  VBT(1);
  VbFn<T> f;
  f.tl = cuts[0];
  f.sc = vbin_scale(cuts[0], cuts[1]);
  f.b = s_b;
  vb_bounds<T>(f.tl, cuts[1], f.sc, s_b, f.lo, f.hi);
  f.comp = s_cb <= (unsigned)kVbCap;
  f.cnt = &a.st[1];
  f.zb = static_cast<T*>(a.zb);
  // one warp per run, 8 vectors per lane in flight (a run of the ~1% copy is a few thousand
  // elements: ~3 dependent L2 round trips instead of one per 4-vector group)
  using V = typename VecOf<T>::V;
  constexpr int VE = VecOf<T>::N, U = 8;
  for (uint64_t W = (uint64_t)blockIdx.x * NW + w; W < (uint64_t)a.Wtot; W += (uint64_t)gridDim.x * NW) {
    const SegEntry e = a.tab[W];
    const T* p = static_cast<const T*>(a.z) + e.off[0];
    const uint64_t c = e.cnt[0];
    const uint64_t mis = (reinterpret_cast<uintptr_t>(p) / sizeof(T)) & (VE - 1);
    const uint64_t head = mis ? ((VE - mis) < c ? (VE - mis) : c) : 0;
    const uint64_t nvec = (c - head) / VE, tail0 = head + nvec * VE;
    if ((uint64_t)lane < head) f.elem(p[lane], 0, 0);
    if ((uint64_t)lane < c - tail0) f.elem(p[tail0 + lane], 0, 0);
    const V* xv = reinterpret_cast<const V*>(p + head);
    const uint64_t nfull = nvec / (32 * U) * (32 * U);
    for (uint64_t v0 = 0; v0 < nfull; v0 += 32 * U) {  // full batches: no bounds tests
      V buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u) buf[u] = ld_stream(xv + v0 + (uint64_t)u * 32 + lane);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        T vv[VE];
#pragma unroll
        for (int j = 0; j < VE; ++j) vv[j] = lane_of(buf[u], j);
        f.vec(vv);
      }
    }
    for (uint64_t i = nfull + lane; i < nvec; i += 32) {
      const V b = ld_stream(xv + i);
      T vv[VE];
#pragma unroll
      for (int j = 0; j < VE; ++j) vv[j] = lane_of(b, j);
      f.vec(vv);
    }
  }
  VBT(2);
  unsigned long long kmn = f.kmin, kmx = f.kmax;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long p = __shfl_xor_sync(FULL, kmn, o), q = __shfl_xor_sync(FULL, kmx, o);
    kmn = p < kmn ? p : kmn;
    kmx = q > kmx ? q : kmx;
  }
  if (lane == 0) { s_kmin[w] = kmn; s_kmax[w] = kmx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < NW; ++q) {
      kmn = s_kmin[q] < kmn ? s_kmin[q] : kmn;
      kmx = s_kmax[q] > kmx ? s_kmax[q] : kmx;
    }
    if (kmx >= kmn) {  // this CTA saw elements of the bin
      atomicMax(&a.st[2], ~kmn);
      atomicMax(&a.st[3], kmx);
    }
    __threadfence();
    s_last = atomicAdd(reinterpret_cast<unsigned*>(&a.st[0]), 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  VBT(3);
  __threadfence();
  const unsigned long long gmin = ~__ldcg(&a.st[2]), gmax = __ldcg(&a.st[3]);
  const unsigned c = s_cb;
  unsigned long long key = gmin;
  bool fb = false;
  if (gmin != gmax) {
    if (c <= (unsigned)kVbCap) {
      // radix select of rank r - base among the bin's c keys, in shared memory, from the highest
      // bit in which the bin's smallest and largest key differ
      extern __shared__ __align__(16) unsigned long long vb_keys[];
      __shared__ unsigned hist[2048];
      const T* zb = static_cast<const T*>(a.zb);
      for (unsigned i = threadIdx.x; i < c; i += 1024) vb_keys[i] = okey(__ldcg(&zb[i]));
#ifdef CPSEL_VB_PROF
      __syncthreads();
      VBT(5);
#endif
      const int hb = 63 - __clzll(gmin ^ gmax);
      unsigned long long mask = hb >= 63 ? 0ull : ~((2ull << hb) - 1ull);
      unsigned long long prefix = gmin & mask;
      unsigned long long rk = r - s_base;
      int lo = hb + 1;
      while (lo > 0) {
        const int bits = lo < 11 ? lo : 11, shift = lo - bits;
        const unsigned dm = (1u << bits) - 1u;
        for (int i = threadIdx.x; i < 2048; i += 1024) hist[i] = 0u;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < c; i += 1024) {
          const unsigned long long k = vb_keys[i];
          if ((k & mask) == prefix) atomicAdd(&hist[(unsigned)(k >> shift) & dm], 1u);
        }
        __syncthreads();
        pick1024(hist, 1 << bits, rk, wsum, &s_d, &s_bef, &s_dc, false);
        prefix |= (unsigned long long)s_d << shift;
        mask |= (unsigned long long)dm << shift;
        rk -= s_bef;
        lo = shift;
        __syncthreads();
      }
      key = prefix;
    } else {
      fb = true;  // a large bin of several values: the host runs the key-digit radix select
    }
  }
#ifdef CPSEL_VB_PROF
  __syncthreads();
  VBT(4);
  if (threadIdx.x == 0) {
    __threadfence();
    printf("vbprof c=%u start 0..%llu  bounds %llu..%llu  scanned %llu..%llu  last %llu  loaded %llu  end %llu (ns)\n", c,
           g_vbprof[1] - g_vbprof[0], g_vbprof[2] - g_vbprof[0], g_vbprof[3] - g_vbprof[0],
           g_vbprof[4] - g_vbprof[0], g_vbprof[5] - g_vbprof[0], g_vbprof[7] - g_vbprof[0], g_vbprof[11] - g_vbprof[0],
           g_vbprof[9] - g_vbprof[0]);
    for (int q = 0; q < 16; q += 2) { g_vbprof[q] = ~0ull; g_vbprof[q + 1] = 0ull; }
  }
#endif
  if (threadIdx.x == 0) {
    *a.fallback = fb ? 1ull : 0ull;
    if (!fb) *a.vout = sizeof(T) == 4 ? from_key_f32(key) : from_key_f64(key);
    publish_done(a.done, a.seq);
  }
  for (int i = threadIdx.x; i < 2048; i += 1024) a.hist0[i] = 0u;  // every CTA read it before its ticket
  if (threadIdx.x < 4) a.st[threadIdx.x] = 0ull;
}

template <typename T, bool INSIDE>
__global__ void __launch_bounds__(kBlock, 4) seg_pass_kernel(SegArgs a) {
  using F = WarpSeg<T, INSIDE>;
  if (a.ks) {  // device loop: input, bracket and output from the loop state
    KelleyState* ks = a.ks;
    if (ks->done || !ks->compact || (ks->inside != 0) != INSIDE) return;
    a.x = ks->cur; a.n = ks->n_cur;
    a.seg_in = ks->cur_seg ? ks->cur_tab : nullptr;
    a.side_in = ks->cur_side;
    a.t = ks->tq; a.y_lo = ks->yL; a.y_hi = ks->yR;
    a.dense_out = ks->dense;
    a.out = ks->dense ? ks->zb[ks->tgt] : ks->sb[ks->tgt];
    a.R = ks->R;
    a.seg_out = ks->st[ks->tgt];
    a.z_cap = ks->cap;
    a.out_tuple = &ks->tuple;
  }
  __shared__ __align__(16) T stage_all[kWarps * 2 * F::GWP];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t W = (uint64_t)blockIdx.x * kWarps + w;
  const uint64_t Wtot = (uint64_t)gridDim.x * kWarps;
  F f;
  f.t = (T)a.t; f.yL = (T)a.y_lo; f.yR = (T)a.y_hi;
  f.L_lo = f.L_hi = 0.0;
  f.n_lo = f.n_hi = 0;
  f.stage = stage_all + (size_t)w * 2 * F::GWP;
  f.dense = a.dense_out;
  f.out = static_cast<T*>(a.out);
  f.reg_lo = W * a.R;
  f.reg_end = (W + 1) * a.R;
  f.cursors = a.cursors;
  f.z_cap = a.z_cap;
  if (a.seg_in == nullptr) {
    // contiguous input: warp-strided groups over the 16-B aligned body; the unaligned head and
    // the tail go to the last warp
    using V = typename VecOf<T>::V;
    constexpr int VE = VecOf<T>::N;
    const T* x = static_cast<const T*>(a.x);
    const uint64_t n = a.n;
    const uint64_t mis = (reinterpret_cast<uintptr_t>(x) / sizeof(T)) & (VE - 1);
    uint64_t head = mis ? (VE - mis) : 0;
    if (head > n) head = n;
    const V* xv = reinterpret_cast<const V*>(x + head);
    const uint64_t nvec = (n - head) / VE;
    constexpr uint64_t GV = 32 * kSegU;
    const uint64_t nfull = nvec / GV;
    for (uint64_t g = W; g < nfull; g += Wtot) seg_group<T, false>(f, xv, g * GV, nvec);
    if (nfull * GV < nvec && W == nfull % Wtot) seg_group<T, true>(f, xv, nfull * GV, nvec);
    if (W == Wtot - 1) {
      const uint64_t tail0 = head + nvec * VE, ntail = n - tail0;
      const bool okh = (uint64_t)lane < head;
      const bool okt = (uint64_t)lane >= head && (uint64_t)lane < head + ntail;
      T v = T(0);
      if (okh) v = x[lane];
      if (okt) v = x[tail0 + (lane - head)];
      if (head + ntail) seg_scalars<T>(f, v, okh || okt);
    }
  } else {
    const SegEntry e = a.seg_in[W];
    const T* base = static_cast<const T*>(a.x);
    seg_run<T>(f, base + e.off[a.side_in], e.cnt[a.side_in]);
  }
  if (!a.dense_out && lane == 0) {
    SegEntry o;
    o.off[0] = f.reg_lo;
    o.cnt[0] = f.n_lo;
    o.off[1] = f.reg_end - f.n_hi;
    o.cnt[1] = f.n_hi;
    a.seg_out[W] = o;
  }
  PassPartial p;
  p.c_lt = p.c_eq = 0;
  p.c_lo = lane == 0 ? f.n_lo : 0;   // warp totals, counted once per warp
  p.c_hi = lane == 0 ? f.n_hi : 0;
  p.L_lo = f.L_lo; p.L_hi = f.L_hi; p.P = 0; p.N = 0;
  p.pred = -tinf<double>(); p.succ = tinf<double>();
  p = block_reduce(p);
  PassPartial id;
  id.c_lt = id.c_eq = id.c_lo = id.c_hi = 0;
  id.L_lo = id.L_hi = id.P = id.N = 0;
  id.pred = -tinf<double>(); id.succ = tinf<double>();
  PassPartial tot;
  if (grid_finish(p, static_cast<PassPartial*>(a.partials), a.ticket, &tot, id) && threadIdx.x == 0) {
    DevPass r;
    r.c_lt = r.c_eq = 0;
    r.c_lo = tot.c_lo; r.c_hi = tot.c_hi;
    r.L_lo = tot.L_lo; r.L_hi = tot.L_hi; r.P = 0; r.N = 0;
    r.pred = tot.pred; r.succ = tot.succ;
    r.z_lo = tot.c_lo; r.z_hi = tot.c_hi;
    if (a.dense_out) {
      a.cursors[0] = 0ull;
      a.cursors[1] = 0ull;
    }
    *a.out_tuple = r;
    publish_done(a.done, a.seq);
  }
}

// ------------------------------------------------------------------------------------------
// The device chain's decisions (§8f-3), taken by the finishing thread of the init / cut pass.
// Step 0 (after the init): the usual path holds if the init compacted ]t_lo, t_hi[, saw no
// NaN/Inf, both cuts lie inside ]prev(min), next(max)[, differ and bracket rank k, and the copy is
// too large for the exact selection — then the chain's cut pass cuts the copy around rank
// k - #x<=t_lo.  Step 1 (after that cut pass): the target lies between its cuts, which differ, and
// the copy is small enough for the radix select.  Each decision also goes to the host (mapped).
template <typename T> __device__ __forceinline__ T nextafter_t(T v, bool up);
template <> __device__ __forceinline__ float nextafter_t(float v, bool up) { return nextafterf(v, up ? INFINITY : -INFINITY); }
template <> __device__ __forceinline__ double nextafter_t(double v, bool up) {
  return ::nextafter(v, up ? (double)INFINITY : -(double)INFINITY);
}
template <typename T>
__device__ void chain_decide0(const DevInit& r, uint64_t k, uint64_t cap, ChainState* cs, ChainMail* mail,
                              unsigned long long seq, int direct) {
  const double lo_out = (double)nextafter_t<T>((T)r.vmin, false), hi_out = (double)nextafter_t<T>((T)r.vmax, true);
  const uint64_t written = r.pad;
  // (a cut at or beyond an extreme's outer neighbour — the open cut of an extreme rank — has nothing
  // between it and that neighbour: the copy is still exactly the bracket interior)
  const bool base = (r.has_cut & 1) && r.nonfinite == 0 && isfinite(r.vmin) && isfinite(r.vmax) && isfinite(lo_out) &&
                    isfinite(hi_out) && isfinite(r.t_est) && r.t_lo < r.t_hi &&
                    r.c_le_lo < k && r.c_lt_hi >= k && written == r.c_lt_hi - r.c_le_lo;
  if (direct) {  // the radix select of the init's copy itself is next: decision 1 gates it
    cs->ok[0] = 0;
    cs->ok[1] = (base && written <= cap) ? 1ull : 0ull;
    cs->m[1] = written;
    cs->r[1] = k - r.c_le_lo;
    cs->le_base = r.c_le_lo;
    mail->ok[1] = cs->ok[1]; mail->m[1] = cs->m[1]; mail->r[1] = cs->r[1];
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(&mail->seq[1]) = seq;
    return;
  }
  const bool ok = base && written > cap;
  cs->ok[0] = ok ? 1ull : 0ull;
  cs->m[0] = written;
  cs->r[0] = k - r.c_le_lo;
  cs->le_base = r.c_le_lo;
  cs->ok[1] = 0;
  mail->ok[0] = cs->ok[0]; mail->m[0] = cs->m[0]; mail->r[0] = cs->r[0];
  __threadfence_system();
  *reinterpret_cast<volatile unsigned long long*>(&mail->seq[0]) = seq;
}
__device__ void chain_decide1(const DevPass& p, uint64_t k, uint64_t cap, ChainState* cs, ChainMail* mail,
                              unsigned long long seq) {
  const uint64_t le_a = cs->le_base + p.c_lt, inner = p.z_lo, lt_b = le_a + inner;
  const bool ok = cs->ok[0] && le_a < k && k <= lt_b && p.pred < p.succ && p.c_eq == 0 && inner <= cap;
  cs->ok[1] = ok ? 1ull : 0ull;
  cs->m[1] = inner;
  cs->r[1] = k - le_a;
  mail->ok[1] = cs->ok[1]; mail->m[1] = cs->m[1]; mail->r[1] = cs->r[1];
  __threadfence_system();
  *reinterpret_cast<volatile unsigned long long*>(&mail->seq[1]) = seq;
}

// ------------------------------------------------------------------------------------------
// R26: the cut pass — two sample cuts t_a <= t_b of the current (compacted) array evaluated in one
// read, with the copy_if of ]t_a, t_b[ (multi-point Kelley).  Every input element
// lies inside the bracket, so the element step is the init pass's cut step without the extremes:
// 6 issue slots (#x<=t_a, the interior bit and the interior sum).
template <typename T> struct WarpCut {
  static constexpr int VE = VecOf<T>::N;
  static constexpr int G = kSegU * VE;
  static constexpr int GW = 32 * G;
  T ta, tb;
  T vals[G];
  unsigned bits;
  float fL = 0.f;                  // #x<=t_a (exact per-thread float counter)
  unsigned long long n_in = 0;     // warp-uniform: elements written
  T* stage;
  int dense;
  T* out;
  uint64_t reg_lo;
  unsigned long long* cursors;
  uint64_t z_cap;                  // dense output capacity: a group that would overflow it is not written
  __device__ __forceinline__ void elem(float v, int u, int idx) {
    asm("{\n\t.reg .pred pL, pI;\n\t"
        "setp.le.f32 pL, %2, %3;\n\t"
        "setp.lt.and.f32 pI, %2, %4, !pL;\n\t"
        "@pL add.rn.f32 %0, %0, 0f3F800000;\n\t"
        "@pI or.b32 %1, %1, %5;\n\t}"
        : "+f"(fL), "+r"(bits)
        : "f"(v), "f"(ta), "f"(tb), "r"(1u << idx));
    (void)u;
    vals[idx] = v;
  }
  __device__ __forceinline__ void elem(double v, int u, int idx) {
    asm("{\n\t.reg .pred pL, pI;\n\t"
        "setp.le.f64 pL, %2, %3;\n\t"
        "setp.lt.and.f64 pI, %2, %4, !pL;\n\t"
        "@pL add.rn.f32 %0, %0, 0f3F800000;\n\t"
        "@pI or.b32 %1, %1, %5;\n\t}"
        : "+f"(fL), "+r"(bits)
        : "d"(v), "d"(ta), "d"(tb), "r"(1u << idx));
    (void)u;
    vals[idx] = v;
  }
  __device__ __forceinline__ void begin() { bits = 0u; }
  __device__ __forceinline__ void end() {
    const int lane = threadIdx.x & 31;
    const unsigned cnt = (unsigned)__popc(bits);
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned tot = __shfl_sync(FULL, incl, 31);
    if (tot == 0u) return;
    T* sp = stage + (incl - cnt);
#pragma unroll
    for (int j = 0; j < G; ++j)
      if (bits & (1u << j)) *sp++ = vals[j];
    __syncwarp();
    T* dst;
    bool fits = true;
    if (dense) {
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(&cursors[0], (unsigned long long)tot);
      b = __shfl_sync(FULL, b, 0);
      fits = b + tot <= z_cap;  // else the cursor total reports the overflow and nothing is kept
      dst = out + b;
    } else {
      dst = out + reg_lo + n_in;
    }
    if (fits)
      for (unsigned i = lane; i < tot; i += 32) dst[i] = stage[i];
    n_in += tot;
    __syncwarp();
  }
};

template <typename T>
__global__ void __launch_bounds__(kBlock, 4) cut_pass_kernel(SegArgs a) {
  using F = WarpCut<T>;
  if (a.chain && !a.chain->ok[0]) return;  // a device-chain step whose chain did not hold
  __shared__ __align__(16) T stage_all[kWarps * F::GW];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t W = (uint64_t)blockIdx.x * kWarps + w;
  const uint64_t Wtot = (uint64_t)gridDim.x * kWarps;
  F f;
  f.ta = static_cast<const T*>(a.cuts)[0];
  f.tb = static_cast<const T*>(a.cuts)[1];
  f.stage = stage_all + (size_t)w * F::GW;
  f.dense = a.dense_out;
  f.out = static_cast<T*>(a.out);
  f.reg_lo = W * a.R;
  f.cursors = a.cursors;
  f.z_cap = a.z_cap;
  if (a.seg_in == nullptr) {
    using V = typename VecOf<T>::V;
    constexpr int VE = VecOf<T>::N;
    const T* x = static_cast<const T*>(a.x);
    const uint64_t n = a.n;
    const uint64_t mis = (reinterpret_cast<uintptr_t>(x) / sizeof(T)) & (VE - 1);
    uint64_t head = mis ? (VE - mis) : 0;
    if (head > n) head = n;
    const V* xv = reinterpret_cast<const V*>(x + head);
    const uint64_t nvec = (n - head) / VE;
    constexpr uint64_t GV = 32 * kSegU;
    const uint64_t nfull = nvec / GV;
    for (uint64_t g = W; g < nfull; g += Wtot) seg_group<T, false>(f, xv, g * GV, nvec);
    if (nfull * GV < nvec && W == nfull % Wtot) seg_group<T, true>(f, xv, nfull * GV, nvec);
    if (W == Wtot - 1) {
      const uint64_t tail0 = head + nvec * VE, ntail = n - tail0;
      const bool okh = (uint64_t)lane < head;
      const bool okt = (uint64_t)lane >= head && (uint64_t)lane < head + ntail;
      T v = T(0);
      if (okh) v = x[lane];
      if (okt) v = x[tail0 + (lane - head)];
      if (head + ntail) seg_scalars<T>(f, v, okh || okt);
    }
  } else {
    const SegEntry e = a.seg_in[W];
    const T* base = static_cast<const T*>(a.x);
    seg_run<T>(f, base + e.off[a.side_in], e.cnt[a.side_in]);
  }
  if (!a.dense_out && lane == 0) {
    SegEntry o;
    o.off[0] = f.reg_lo;
    o.cnt[0] = f.n_in;
    o.off[1] = f.reg_lo + a.R;
    o.cnt[1] = 0;
    a.seg_out[W] = o;
  }
  PassPartial p;
  p.c_lt = (unsigned long long)f.fL;
  p.c_eq = 0;
  p.c_lo = lane == 0 ? f.n_in : 0;  // warp totals, counted once per warp
  p.c_hi = 0;
  p.L_lo = 0; p.L_hi = 0; p.P = 0; p.N = 0;
  p.pred = -tinf<double>(); p.succ = tinf<double>();
  p = block_reduce(p);
  PassPartial id;
  id.c_lt = id.c_eq = id.c_lo = id.c_hi = 0;
  id.L_lo = id.L_hi = id.P = id.N = 0;
  id.pred = -tinf<double>(); id.succ = tinf<double>();
  PassPartial tot;
  if (grid_finish(p, static_cast<PassPartial*>(a.partials), a.ticket, &tot, id) && threadIdx.x == 0) {
    DevPass r;
    r.c_lt = tot.c_lt;
    r.c_eq = (a.dense_out && tot.c_lo > a.z_cap) ? 1ull : 0ull;  // the dense copy overflowed: not kept
    r.c_lo = tot.c_lo; r.c_hi = 0;
    r.L_lo = (double)static_cast<const T*>(a.cuts)[2];  // the sample's estimate of x_(k)
    r.L_hi = 0; r.P = 0; r.N = 0;
    r.pred = (double)f.ta; r.succ = (double)f.tb;
    r.z_lo = tot.c_lo; r.z_hi = 0;
    if (a.dense_out) a.cursors[0] = 0ull;
    *a.out_tuple = r;
    publish_done(a.done, a.seq);
    if (a.chain_out) chain_decide1(r, a.chain_k, a.chain_cap, a.chain_out, a.chain_mail, a.chain_seq);
  }
}

// ------------------------------------------------------------------------------------------
// Steps a1 + a4 fused (R23): the init reduction, the two extra cuts and the copy_if of the elements
// strictly between the cuts, in ONE read of x.  Warp-strided groups and the warp-private region
// layout of seg_pass_kernel (the interior lands in run 0 of each warp's entry), so the following
// cutting-plane passes read it as a segmented array.
// SUMS: also accumulate N(t_lo) = sum (t_lo-x)^+ and P(t_hi) = sum (x-t_hi)^+ (only the reported
// objective values need them, R25)
template <typename T, bool SUMS> struct InitSeg {
  static constexpr int VE = VecOf<T>::N;
  static constexpr int G = kSegU * VE;
  static constexpr int GW = 32 * G;
  T mn, mx, tl, th;
  unsigned cmn = 0, cmx = 0, nan = 0;
  float fL = 0;                   // #x<=t_lo (exact per-thread float counter, < 2^24 per thread)
  T gN[kSegU], gP[kSegU], gI[kSegU];
  double N0 = 0, P0 = 0, I0 = 0;
  T vals[G];
  unsigned bits;
  unsigned long long n_in = 0;    // warp-uniform: interior elements written
  T* out;
  uint64_t reg_lo;
  T* stage;                       // this warp's GW-element staging buffer (shared memory)
  unsigned* hist0 = nullptr;      // direct chain: shared-memory histogram of the copy's first digit
  T vtl = T(0), vsc = T(0);       // vbin: t_lo and the bin scale (0: top key digit)

  // one element, SUMS: 3 compares, 2 subs, 1 counter, 3 sums, 1 interior bit (10 issue slots):
  //   fL = #x<=t_lo, N += (t_lo-x) on x<=t_lo, P += (x-t_hi) on x>t_hi, I += (x-t_lo) and the
  //   interior bit on t_lo<x<t_hi.  #x<t_hi = #x<=t_lo + #interior.
  //   !SUMS: fL and the interior bit only (4 slots; the next iterate comes from the sample, R25).
  //   (#x==t_lo and #x==t_hi are not needed, R24.)
  __device__ __forceinline__ void cut(float v, int u, int idx) {
    if (SUMS)
      asm("{\n\t.reg .pred pL, pH, pI;\n\t.reg .f32 dl, dh;\n\t"
          "setp.le.f32 pL, %5, %6;\n\t"
          "setp.gt.f32 pH, %5, %7;\n\t"
          "setp.lt.and.f32 pI, %5, %7, !pL;\n\t"
          "sub.rn.f32 dl, %6, %5;\n\t"
          "sub.rn.f32 dh, %5, %7;\n\t"
          "@pL add.rn.f32 %0, %0, 0f3F800000;\n\t"
          "@pL add.rn.f32 %1, %1, dl;\n\t"
          "@pH add.rn.f32 %2, %2, dh;\n\t"
          "@pI sub.rn.f32 %3, %3, dl;\n\t"
          "@pI or.b32 %4, %4, %8;\n\t}"
          : "+f"(fL), "+f"(gN[u]), "+f"(gP[u]), "+f"(gI[u]), "+r"(bits)
          : "f"(v), "f"(tl), "f"(th), "r"(1u << idx));
    else
      asm("{\n\t.reg .pred pL, pI;\n\t"
          "setp.le.f32 pL, %2, %3;\n\t"
          "setp.lt.and.f32 pI, %2, %4, !pL;\n\t"
          "@pL add.rn.f32 %0, %0, 0f3F800000;\n\t"
          "@pI or.b32 %1, %1, %5;\n\t}"
          : "+f"(fL), "+r"(bits)
          : "f"(v), "f"(tl), "f"(th), "r"(1u << idx));
    vals[idx] = v;
  }
  __device__ __forceinline__ void cut(double v, int u, int idx) {
    if (SUMS)
      asm("{\n\t.reg .pred pL, pH, pI;\n\t.reg .f64 dl, dh;\n\t"
          "setp.le.f64 pL, %5, %6;\n\t"
          "setp.gt.f64 pH, %5, %7;\n\t"
          "setp.lt.and.f64 pI, %5, %7, !pL;\n\t"
          "sub.rn.f64 dl, %6, %5;\n\t"
          "sub.rn.f64 dh, %5, %7;\n\t"
          "@pL add.rn.f32 %0, %0, 0f3F800000;\n\t"
          "@pL add.rn.f64 %1, %1, dl;\n\t"
          "@pH add.rn.f64 %2, %2, dh;\n\t"
          "@pI sub.rn.f64 %3, %3, dl;\n\t"
          "@pI or.b32 %4, %4, %8;\n\t}"
          : "+f"(fL), "+d"(gN[u]), "+d"(gP[u]), "+d"(gI[u]), "+r"(bits)
          : "d"(v), "d"(tl), "d"(th), "r"(1u << idx));
    else
      asm("{\n\t.reg .pred pL, pI;\n\t"
          "setp.le.f64 pL, %2, %3;\n\t"
          "setp.lt.and.f64 pI, %2, %4, !pL;\n\t"
          "@pL add.rn.f32 %0, %0, 0f3F800000;\n\t"
          "@pI or.b32 %1, %1, %5;\n\t}"
          : "+f"(fL), "+r"(bits)
          : "d"(v), "d"(tl), "d"(th), "r"(1u << idx));
    vals[idx] = v;
  }
  __device__ __forceinline__ void begin() {
    if (SUMS)
#pragma unroll
      for (int u = 0; u < kSegU; ++u) gN[u] = gP[u] = gI[u] = T(0);
    bits = 0u;
  }
  __device__ __forceinline__ void vec(const float4& v, int u) {
    cut(v.x, u, u * 4 + 0); cut(v.y, u, u * 4 + 1); cut(v.z, u, u * 4 + 2); cut(v.w, u, u * 4 + 3);
  }
  __device__ __forceinline__ void vec(const double2& v, int u) {
    cut(v.x, u, u * 2 + 0); cut(v.y, u, u * 2 + 1);
  }
  // group-level extremes: NaN-propagating min/max trees over the thread's values and a warp vote
  // against the WARP-UNIFORM running (min, max); only a group that beats a running extreme or holds
  // a NaN takes the (warp-uniform) update.  The multiplicities of min and max are not counted (R27):
  // the driver brackets with their outer neighbours instead.  Warp-level records are rare (~H(groups)/groups),
  // where per-thread records would send most warps down the slow path early on.  Must be called by
  // all 32 lanes.
  __device__ __forceinline__ static T nan_min(T a, T b) {
    if (sizeof(T) == 4) {
      float r;
      asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"((float)a), "f"((float)b));
      return (T)r;
    }
    return (a != a || b != b) ? a + b : (T)fmin((double)a, (double)b);
  }
  __device__ __forceinline__ static T nan_max(T a, T b) {
    if (sizeof(T) == 4) {
      float r;
      asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"((float)a), "f"((float)b));
      return (T)r;
    }
    return (a != a || b != b) ? a + b : (T)fmax((double)a, (double)b);
  }
  __device__ __forceinline__ void extremes(int nvalid) {
    T lo = nvalid > 0 ? vals[0] : tinf<T>(), hi = nvalid > 0 ? vals[0] : -tinf<T>();
    bool bad = false;  // f64: fmin/fmax drop NaNs, so they are flagged separately
    if (sizeof(T) == 8 && nvalid > 0) bad = vals[0] != vals[0];
#pragma unroll
    for (int j = 1; j < G; ++j)
      if (j < nvalid) {
        if (sizeof(T) == 4) {
          lo = nan_min(lo, vals[j]);
          hi = nan_max(hi, vals[j]);
        } else {
          lo = (T)fmin((double)lo, (double)vals[j]);
          hi = (T)fmax((double)hi, (double)vals[j]);
          bad |= vals[j] != vals[j];
        }
      }
    const bool need = !(lo >= mn) || !(hi <= mx) || bad;  // a new extreme, or a NaN
    if (__any_sync(FULL, need)) slow_group(nvalid, bad ? (T)NAN : lo, hi);
  }
  __device__ __forceinline__ void slow_group(int nvalid, T lo, T hi) {
    if (__any_sync(FULL, lo != lo || hi != hi)) {  // NaNs: count them, extremes over the rest
      lo = tinf<T>(); hi = -tinf<T>();
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (j < nvalid) {
          const T v = vals[j];
          if (v != v) ++nan;
          else { lo = v < lo ? v : lo; hi = v > hi ? v : hi; }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const T a = __shfl_xor_sync(FULL, lo, o), b = __shfl_xor_sync(FULL, hi, o);
      lo = a < lo ? a : lo;
      hi = b > hi ? b : hi;
    }
    mn = lo < mn ? lo : mn;
    mx = hi > mx ? hi : mx;
  }
  __device__ __forceinline__ void end(int nvalid) {
    extremes(nvalid);
    if (SUMS) {
      N0 += (double)((gN[0] + gN[1]) + (gN[2] + gN[3]));
      P0 += (double)((gP[0] + gP[1]) + (gP[2] + gP[3]));
      I0 += (double)((gI[0] + gI[1]) + (gI[2] + gI[3]));
    }
    const int lane = threadIdx.x & 31;
    const unsigned cnt = (unsigned)__popc(bits);
    const unsigned act = __ballot_sync(FULL, cnt != 0u);
    if (act == 0u) return;
    unsigned excl, tot;
    if (__all_sync(FULL, cnt <= 1u)) {  // the usual case: at most one interior element per lane
      unsigned lt;
      asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
      excl = (unsigned)__popc(act & lt);
      tot = (unsigned)__popc(act);
    } else {
      unsigned incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      excl = incl - cnt;
      tot = __shfl_sync(FULL, incl, 31);
    }
    // predicated shared stores: lane l stages its interior elements at [excl_l, excl_l + cnt_l),
    // then the warp writes the group's run out coalesced (the order inside a run is free); a
    // vector slot no lane has an interior element in is skipped by the whole warp
    T* sp = stage + excl;
    constexpr int VU = G / kSegU;
#pragma unroll
    for (int u = 0; u < kSegU; ++u) {
      const unsigned mu = (bits >> (u * VU)) & ((1u << VU) - 1u);
      if (__any_sync(FULL, mu != 0u)) {
#pragma unroll
        for (int q = 0; q < VU; ++q)
          if (mu & (1u << q)) *sp++ = vals[u * VU + q];
      }
    }
    __syncwarp();
    T* dst = out + reg_lo + n_in;
    if (hist0 && vsc > T(0)) {  // the copy's first digit (direct chain): its value bin (vbin) ...
      for (unsigned i = lane; i < tot; i += 32) {
        const T v = stage[i];
        dst[i] = v;
        atomicAdd(&hist0[vbin_of(v, vtl, vsc)], 1u);
      }
    } else if (hist0) {  // ... or its top key digit  (an L2 evict-last store hint here measured 1%
      for (unsigned i = lane; i < tot; i += 32) {  //  slower overall: plain stores)
        const T v = stage[i];
        dst[i] = v;
        atomicAdd(&hist0[(unsigned)(okey(v) >> (sizeof(T) == 4 ? 21 : 53)) & 2047u], 1u);
      }
    } else {
      for (unsigned i = lane; i < tot; i += 32) dst[i] = stage[i];
    }
    __syncwarp();
    n_in += tot;
  }
};

template <typename T, bool SUMS>
__global__ void __launch_bounds__(kBlock, 4) init_seg_kernel(InitArgs ia, SegArgs a) {
  using F = InitSeg<T, SUMS>;
  using V = typename VecOf<T>::V;
  constexpr int VE = VecOf<T>::N;
  pdl_wait();  // the sample kernel's cuts
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t W = (uint64_t)blockIdx.x * kWarps + w;
  const uint64_t Wtot = (uint64_t)gridDim.x * kWarps;
  const T* x = static_cast<const T*>(ia.x);
  const uint64_t n = ia.n;
  F f;
  f.mn = tinf<T>(); f.mx = -tinf<T>();
  f.tl = static_cast<const T*>(ia.t0)[0];
  f.th = static_cast<const T*>(ia.t0)[1];
  f.out = static_cast<T*>(a.out);
  f.reg_lo = W * a.R;
  __shared__ unsigned h0[2048];
  const bool hist = ia.chain_direct && ia.hist;
  if (hist) {
    for (int i = threadIdx.x; i < 2048; i += kBlock) h0[i] = 0u;
    __syncthreads();
    f.hist0 = h0;
    if (ia.vbin) {
      f.vtl = f.tl;
      f.vsc = vbin_scale(f.tl, f.th);
    }
  }
  const uint64_t mis = (reinterpret_cast<uintptr_t>(x) / sizeof(T)) & (VE - 1);
  uint64_t head = mis ? (VE - mis) : 0;
  if (head > n) head = n;
  const V* xv = reinterpret_cast<const V*>(x + head);
  const uint64_t nvec = (n - head) / VE;
  constexpr uint64_t GV = 32 * kSegU;
  const uint64_t nfull = nvec / GV;
  {
    __shared__ __align__(16) T stage_all[kWarps * F::GW];
    f.stage = stage_all + (size_t)w * F::GW;
    // software pipelined: the next group's loads are issued once the current group's values sit in
    // f.vals, so they are in flight during its scan / staging / copy-out
    V v[kSegU];
    const uint64_t pol = policy_evict_first();
    if (W < nfull) {
#pragma unroll
      for (int u = 0; u < kSegU; ++u) v[u] = ld_stream_ef(xv + W * GV + (uint64_t)u * 32 + lane, pol);
    }
    for (uint64_t g = W; g < nfull; g += Wtot) {
      f.begin();
#pragma unroll
      for (int u = 0; u < kSegU; ++u) f.vec(v[u], u);
      const uint64_t gn = g + Wtot;
      if (gn < nfull) {
#pragma unroll
        for (int u = 0; u < kSegU; ++u) v[u] = ld_stream_ef(xv + gn * GV + (uint64_t)u * 32 + lane, pol);
      }
      f.end(F::G);
    }
  }
  if (nfull * GV < nvec && W == nfull % Wtot) {  // the ragged group
    V v[kSegU];
    bool ok[kSegU];
#pragma unroll
    for (int u = 0; u < kSegU; ++u) {
      const uint64_t i = nfull * GV + (uint64_t)u * 32 + lane;
      ok[u] = i < nvec;
      if (ok[u]) v[u] = ld_stream(xv + i);
    }
    // masked-off vectors: replicate a valid lane value so the group extremes stay exact
    f.begin();
    int nvalid = 0;
#pragma unroll
    for (int u = 0; u < kSegU; ++u)
      if (ok[u]) { f.vec(v[u], u); nvalid = (u + 1) * VE; }
    f.end(nvalid);
  }
  if (W == Wtot - 1) {  // unaligned head + tail scalars
    const uint64_t tail0 = head + nvec * VE, ntail = n - tail0;
    const bool okh = (uint64_t)lane < head;
    const bool okt = (uint64_t)lane >= head && (uint64_t)lane < head + ntail;
    if (head + ntail) {
      f.begin();
      int nvalid = 0;
      if (okh || okt) {
        const T v = okh ? x[lane] : x[tail0 + (lane - head)];
        f.cut(v, 0, 0);
        nvalid = 1;
      }
      f.end(nvalid);
    }
  }
  if (lane == 0) {
    SegEntry o;
    o.off[0] = f.reg_lo;
    o.cnt[0] = f.n_in;
    o.off[1] = f.reg_lo + a.R;
    o.cnt[1] = 0;
    a.seg_out[W] = o;
  }
  pdl_trigger();  // the chained radix round may be scheduled now (it waits for this grid to finish)
  if (hist) {  // this CTA's round-0 histogram into the global one (before the grid finish's fence)
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += kBlock)
      if (h0[i]) atomicAdd(&ia.hist[i], h0[i]);
    __threadfence();  // every thread's reductions performed before the grid finish's ticket
  }
  InitPartial p;
  p.vmin = (double)f.mn; p.vmax = (double)f.mx; p.S = 0; p.pad = 0;
  p.cnt_min = f.cmn; p.cnt_max = f.cmx; p.nonfinite = f.nan;
  p.pad2 = lane == 0 ? f.n_in : 0;  // interior elements written (counted once per warp)
  p.N0 = f.N0; p.P0 = f.P0; p.I0 = f.I0;
  p.cA = (unsigned long long)f.fL; p.cB = p.cC = p.cD = p.cE = 0;  // cA = #x<=t_lo
  p = block_reduce(p);
  InitPartial id;
  id.vmin = tinf<double>(); id.vmax = -tinf<double>(); id.S = 0; id.pad = 0;
  id.cnt_min = id.cnt_max = id.nonfinite = id.pad2 = 0;
  id.N0 = id.P0 = id.I0 = 0; id.cA = id.cB = id.cC = id.cD = id.cE = 0;
  InitPartial tot;
  bool last;
  if (!SUMS && ia.acc) {
    // no fp sums in this form: every field is an extreme or a count, so the grid's totals are exact
    // and order-free through atomics (min as the max of the complemented order-preserving key) —
    // the last CTA reads five words instead of folding every CTA's partial (a ~10 us serial tail)
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
      unsigned long long* g = ia.acc;
      atomicMax(&g[0], ~okey((T)p.vmin));
      atomicMax(&g[1], okey((T)p.vmax));
      if (p.nonfinite) atomicAdd(&g[2], p.nonfinite);
      if (p.pad2) atomicAdd(&g[3], p.pad2);
      if (p.cA) atomicAdd(&g[4], p.cA);
      __threadfence();
      s_last = atomicAdd(ia.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    last = s_last;
    if (last && threadIdx.x == 0) {
      __threadfence();
      unsigned long long* g = ia.acc;
      const unsigned long long kmin = ~__ldcg(&g[0]), kmax = __ldcg(&g[1]);
      tot = id;
      tot.vmin = sizeof(T) == 4 ? from_key_f32(kmin) : from_key_f64(kmin);
      tot.vmax = sizeof(T) == 4 ? from_key_f32(kmax) : from_key_f64(kmax);
      tot.nonfinite = __ldcg(&g[2]);
      tot.pad2 = __ldcg(&g[3]);
      tot.cA = __ldcg(&g[4]);
      for (int q = 0; q < 5; ++q) g[q] = 0ull;  // self-reset for the next launch
      *ia.ticket = 0u;
    }
  } else {
    last = grid_finish(p, static_cast<InitPartial*>(ia.partials), ia.ticket, &tot, id);
  }
  if (!last) return;
  if (threadIdx.x == 0) {
    DevInit r;
    r.vmin = tot.vmin; r.vmax = tot.vmax; r.S = 0; r.x0 = (double)x[0];
    r.cnt_min = tot.cnt_min; r.cnt_max = tot.cnt_max; r.nonfinite = tot.nonfinite;
    r.pad = tot.pad2;  // interior elements written
    r.t_lo = (double)f.tl; r.t_hi = (double)f.th;
    r.N_lo = tot.N0; r.P_hi = tot.P0; r.I_in = tot.I0;
    r.c_le_lo = tot.cA;
    r.c_lt_hi = tot.cA + tot.pad2;  // every x < t_hi is <= t_lo or interior
    r.t_est = (double)static_cast<const T*>(ia.t0)[2];
    r.res1 = r.res2 = 0;
    r.has_cut = SUMS ? 15ull : 11ull;  // two cuts + the interior compacted (+ N_lo, P_hi), no #min/#max
    *ia.out = r;
    publish_done(ia.done, ia.seq);
    if (ia.chain) chain_decide0<T>(r, ia.chain_k, ia.chain_cap, ia.chain, ia.chain_mail, ia.chain_seq, ia.chain_direct);
  }
}

// The batched kernel's init pass: the per-element step of init_seg_kernel (stats + two cuts +
// interior bit) with the block-level dense compaction of PassFn (one CTA per column, the interior
// ]t_lo, t_hi[ goes to the CTA's buffer from index 0).
struct BatchInitFn : InitSeg<float, false> {
  PassFn<float, kCompact, 4> pc;
  int nvalid = 0;
  __device__ __forceinline__ void group_begin() {
    begin();
    nvalid = 0;
  }
  template <bool MASKED, typename V> __device__ __forceinline__ void vec(const V& v, bool ok, int u) {
    if (MASKED && !ok) return;
    InitSeg<float, false>::vec(v, u);
    nvalid = (u + 1) * 4;
  }
  __device__ __forceinline__ void group_end() {
    extremes(nvalid);
#pragma unroll
    for (int j = 0; j < 16; ++j) pc.vals[j] = vals[j];
    pc.lo_bits = bits;
    pc.hi_bits = 0u;
    pc.compact_group();
  }
  // head/tail scalars (warp 0 only): per-element atomics on the (shared) cursor
  __device__ __forceinline__ void scalar(float v, bool ok) {
    begin();
    if (ok) cut(v, 0, 0);
    extremes(ok ? 1 : 0);

    if (bits & 1u) {
      const unsigned long long pos = atomicAdd(&pc.cursors[0], 1ull);
      if (pos < pc.z_cap) pc.z[pos] = v;
    }
  }
};

// ------------------------------------------------------------------------------------------
// Step a8: batched selection (LMS: one k-th order statistic per column of S).  One CTA runs the
// whole method on one column at a time (work-stealing over columns): the init reduction, the
// Kelley iterations with the driver step on thread 0 (device-side driver, same rules as the host
// driver), multi-level compaction into the CTA's private ping-pong buffers, and an exact finish
// on <= 32 elements by warp-wide rank counting.
__device__ __forceinline__ float snap_dev(double t, float yL, float yR) {
  float f = isfinite(t) ? __double2float_rn(t) : __double2float_rn(0.5 * (double)yL + 0.5 * (double)yR);
  if (!(f > yL)) f = nextafterf(yL, tinf<float>());
  if (!(f < yR)) f = nextafterf(yR, -tinf<float>());
  return f;
}
__device__ __forceinline__ float key_mid_dev(float yL, float yR) {
  const unsigned a = (unsigned)okey(yL), b = (unsigned)okey(yR);
  return (float)from_key_f32((unsigned long long)(a + (b - a) / 2));
}

constexpr int kBatchSample = 2048;   // samples of the init pass's extra cuts (R23; 32-bit keys)
constexpr int kBatchCutSample = 1024;  // samples of a cut pass over the compacted bracket (R26)
constexpr int kBatchFinish = 4096;   // kept halves this small are finished by a block radix select

struct BatchState {
  const float* cur;
  unsigned long long n_cur, c_le_L, c_lt_R, D_lo, m, k_r;
  unsigned long long cursors[2];
  double t;
  float yL, yR, tq, result, cut_lo, cut_hi, cut_mid;
  int col, on_z, slow, bisect, phase, compact, cur_buf, tgt, side, iters, exact, cuts_stalled, free_step;
};

// Block-wide exact selection of NT order statistics of 32-bit keys held PER per thread (kBlock
// threads): rk[t] = 0-based rank among all kBlock*PER keys (padding keys 0xffffffff sort last and
// are never selected when rk[t] < #valid).  MSB radix select with 11/11/10-bit digits and one
// shared-memory histogram per target (hist: NT x 2048 words); out[t] on every thread.  Replaces a
// bitonic sort of the whole set (a5 / R26 sample cuts): 3 histogram rounds instead of log^2 stages.
template <int PER, int NT>
__device__ void block_radix_select(const unsigned (&key)[PER], unsigned* hist, const unsigned (&rk_in)[NT],
                                   unsigned (&out)[NT]) {
  __shared__ unsigned wsum[NT][kWarps];
  __shared__ unsigned sel[NT][2];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  unsigned prefix[NT], rk[NT], mask = 0u;
#pragma unroll
  for (int t = 0; t < NT; ++t) { prefix[t] = 0u; rk[t] = rk_in[t]; }
#pragma unroll 1
  for (int round = 0; round < 3; ++round) {
    const int sh = round == 0 ? 21 : (round == 1 ? 10 : 0);
    const unsigned dm = round == 2 ? 1023u : 2047u;
    for (int b = tid; b < NT * 2048; b += kBlock) hist[b] = 0u;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const unsigned d = (key[u] >> sh) & dm;
#pragma unroll
      for (int t = 0; t < NT; ++t)
        if ((key[u] & mask) == prefix[t]) atomicAdd(&hist[t * 2048 + d], 1u);
    }
    __syncthreads();
    constexpr int B = 2048 / kBlock;  // bins per thread
    unsigned c[NT][B], incl[NT], tot[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      unsigned v = 0u;
#pragma unroll
      for (int b = 0; b < B; ++b) { c[t][b] = hist[t * 2048 + tid * B + b]; v += c[t][b]; }
      tot[t] = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += w;
      }
      incl[t] = v;
      if (lane == 31) wsum[t][wid] = v;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      unsigned before = incl[t] - tot[t];
      for (int w2 = 0; w2 < wid; ++w2) before += wsum[t][w2];
      if (before <= rk[t] && rk[t] < before + tot[t]) {
#pragma unroll
        for (int b = 0; b < B; ++b) {
          if (before <= rk[t] && rk[t] < before + c[t][b]) { sel[t][0] = (unsigned)(tid * B + b); sel[t][1] = before; }
          before += c[t][b];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      prefix[t] |= sel[t][0] << sh;
      rk[t] -= sel[t][1];
    }
    mask |= dm << sh;
    __syncthreads();  // hist / sel reused
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) out[t] = prefix[t];
}

// The cuts of local rank r (1-based) of m elements from ms evenly strided samples of z[0..m)
// (ms <= S): sample order statistics of ranks q -/+ (3.5 sd + 2) and q -> st.cut_lo / cut_hi /
// cut_mid.  Block-wide; hist = NT x 2048 words of shared memory.
template <int S>
__device__ void batch_sample_cuts(BatchState& st, unsigned* hist, const float* z, uint64_t m, uint64_t r) {
  constexpr int PER = S / kBlock;
  const uint64_t ms = m < (uint64_t)S ? m : (uint64_t)S;
  unsigned key[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const uint64_t i = (uint64_t)(threadIdx.x + u * kBlock);
    if (i < ms) {
      const uint64_t pos = (m == ms) ? i : (i * m) / ms + (m / ms) / 2;
      key[u] = (unsigned)okey(z[pos]);
    } else {
      key[u] = ~0u;
    }
  }
  const double md = (double)ms;
  const double q = ((double)r - 0.5) / (double)m * md;
  const double w = 3.5 * sqrt(fmax(q * (md - q) / md, 0.0)) + 2.0;
  const double ql = floor(q - w), qh = ceil(q + w), qm = floor(q);
  const unsigned rk[3] = {ql < 0 ? 0u : (unsigned)ql, qh >= md ? (unsigned)(ms - 1) : (unsigned)qh,
                          qm < 0 ? 0u : (qm >= md ? (unsigned)(ms - 1) : (unsigned)qm)};
  unsigned out[3];
  block_radix_select<PER, 3>(key, hist, rk, out);
  if (threadIdx.x == 0) {
    // R31: a cut whose sample rank falls off the sample opens to the largest finite float
    st.cut_lo = ql < 0 ? -FLT_MAX : (float)from_key_f32(out[0]);
    st.cut_hi = qh >= md - 1 ? FLT_MAX : (float)from_key_f32(out[1]);
    st.cut_mid = (float)from_key_f32(out[2]);
  }
  __syncthreads();
}

// R23 for the fused LMS pass.  Ss holds, per column j, the residuals s of ms evenly strided sample
// rows (computed by the fused tensor-core kernel in store mode: exactly elements of S).  Per column,
// the bin edges around the sample order statistics of ranks q -/+ (3.5 sd + 2) and q (q the target
// rank k scaled to the sample, as batch_sample_cuts) -> cuts[4j .. 4j+2] = t_lo, t_hi, t_mid.  Two
// digit rounds on the order-preserving keys RELATIVE to the column's smallest sample key kmin:
// round 0 bins d = key - kmin by its top 11 significant bits (bin width 2^sh, sh from the column's
// key span, so the 2048 bins cover the sample evenly in key space — the squared residuals of one
// candidate share few exponents, and top-bits bins would pile most of them into a handful of
// contended shared-memory counters), round 1 the next 11 bits of d within each target's bin; t_lo
// is the lower edge of the lo target's final bin (<= that sample order statistic), t_hi the upper
// edge of the hi target's (>=): cuts at most 2^max(0, sh-11) key units wider than the exact sample
// quantiles, which is all a cut needs — the fused pass counts exactly at whatever values they are.
// One CTA of 1024 threads per column.
// Each CTA (512 threads, two per SM, so one CTA's copy and histogram rounds overlap the other's)
// walks its columns: the column's samples are bulk-copied into the CTA's shared buffer and every
// round reads its keys from there (32 per thread would not fit the registers of two CTAs per SM).
// The counters take predicated shared reductions (no divergent branches).
constexpr int kCutThreads = 512;
constexpr int kCutMaxPer = 32;   // <= 16384 samples
constexpr int kCutBPT = 2048 / kCutThreads;  // histogram bins per thread in the scans (one uint4)
static_assert(kCutBPT == 4, "the scans read one uint4 of bins per thread");
constexpr size_t kCutSmem = (size_t)kCutThreads * kCutMaxPer * 4 + 64;  // one column buffer + an mbarrier
__device__ __forceinline__ void red_shared_add1(uint32_t addr, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t@q red.shared.add.u32 [%0], 1;\n\t}" ::"r"(addr), "r"((int)p)
               : "memory");
}
__global__ void __launch_bounds__(kCutThreads, 2) lms_cuts_kernel(const float* __restrict__ Ss, uint32_t ms,
                                                                  uint64_t n, uint32_t C, uint64_t k,
                                                                  float* __restrict__ cuts) {
  constexpr int NW = kCutThreads / 32;
  __shared__ __align__(16) unsigned hist[3][2048];
  __shared__ unsigned wsum[3][NW];
  __shared__ unsigned sel[3][2];
  __shared__ unsigned wmin[NW], wmax[NW];
  extern __shared__ __align__(16) unsigned char cut_smem[];
  float* buf = reinterpret_cast<float*>(cut_smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(cut_smem + (size_t)kCutThreads * kCutMaxPer * 4);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t col_bytes = ms * 4u;  // a multiple of 16 (ms is a multiple of 256)
  unsigned rank[3];
  {
    const double md = (double)ms;
    const double q = ((double)k - 0.5) / (double)n * md;
    const double w = 3.5 * sqrt(fmax(q * (md - q) / md, 0.0)) + 2.0;
    const double ql = floor(q - w), qh = ceil(q + w), qm = floor(q);
    rank[0] = ql < 0 ? 0u : (unsigned)ql;
    rank[1] = qh >= md ? ms - 1 : (unsigned)qh;
    rank[2] = qm < 0 ? 0u : (qm >= md ? ms - 1 : (unsigned)qm);
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t it = 0;
  const float4* cb = reinterpret_cast<const float4*>(buf);
  for (uint32_t j = blockIdx.x; j < C; j += gridDim.x, ++it) {
    if (tid == 0) {  // (every thread's reads of the previous column ended at the last barrier)
      fence_proxy_async_smem();
      mbar_expect_tx(&bar[0], col_bytes);
      bulk_g2s(buf, Ss + (size_t)j * ms, col_bytes, &bar[0]);
    }
    mbar_wait(&bar[0], it & 1);
    unsigned kmn = 0xffffffffu, kmx = 0u;
#pragma unroll
    for (int v = 0; v < kCutMaxPer / 4; ++v) {  // element (v * kCutThreads + tid) * 4 + c: order is irrelevant
      const uint32_t e4 = v * kCutThreads + tid;
      const float4 q = cb[e4];
      const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (e4 * 4 + c < ms) {
          const unsigned kk = (unsigned)okey(qq[c]);
          kmn = min(kmn, kk);
          kmx = max(kmx, kk);
        }
      }
    }
    kmn = __reduce_min_sync(0xffffffffu, kmn);
    kmx = __reduce_max_sync(0xffffffffu, kmx);
    if (lane == 0) { wmin[wid] = kmn; wmax[wid] = kmx; }
    for (int i = tid; i < 3 * 2048; i += kCutThreads) (&hist[0][0])[i] = 0u;
    __syncthreads();
    kmn = __reduce_min_sync(0xffffffffu, lane < NW ? wmin[lane] : 0xffffffffu);
    kmx = __reduce_max_sync(0xffffffffu, lane < NW ? wmax[lane] : 0u);
    // d = key - kmin < 2^span_bits; round 0 takes d >> sh0 (11 bits), round 1 the bits below
    const unsigned span = kmx - kmn;
    const int span_bits = span ? 32 - __clz(span) : 0;
    const int sh0 = span_bits > 11 ? span_bits - 11 : 0;
    const int sh1 = sh0 > 11 ? sh0 - 11 : 0;
    const unsigned m1 = (1u << (sh0 - sh1)) - 1u;  // round-1 digit: the bits of d below the round-0 bin
    const uint32_t h0 = smem_u32(&hist[0][0]), h1 = smem_u32(&hist[1][0]), h2 = smem_u32(&hist[2][0]);
    unsigned bin[3] = {0u, 0u, 0u}, rk[3] = {rank[0], rank[1], rank[2]};
#pragma unroll 1
    for (int round = 0; round < 2; ++round) {
      if (round == 1) {
        for (int i = tid; i < 2048; i += kCutThreads) hist[0][i] = 0u;  // (1, 2 still zero)
        __syncthreads();
      }
#pragma unroll 2
      for (int v = 0; v < kCutMaxPer / 4; ++v) {  // 16-byte reads of the column (conflict-free)
        const uint32_t e4 = v * kCutThreads + tid;
        const float4 q = cb[e4];
        const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const bool ok = e4 * 4 + c < ms;
          const unsigned d = (unsigned)okey(qq[c]) - kmn;
          if (round == 0) {
            red_shared_add1(h0 + 4u * (d >> sh0), ok);
          } else {
            const unsigned top = d >> sh0, dd = 4u * ((d >> sh1) & m1);
            red_shared_add1(h0 + dd, ok && top == bin[0]);
            red_shared_add1(h1 + dd, ok && top == bin[1]);
            red_shared_add1(h2 + dd, ok && top == bin[2]);
          }
        }
      }
      __syncthreads();
      unsigned incl[3], tsum[3];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int hsrc = round == 0 ? 0 : t;
        const uint4 hv = reinterpret_cast<const uint4*>(&hist[hsrc][0])[tid];  // kCutBPT == 4 bins
        tsum[t] = hv.x + hv.y + hv.z + hv.w;
        unsigned v = tsum[t];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned w = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += w;
        }
        incl[t] = v;
        if (lane == 31) wsum[t][wid] = v;
      }
      __syncthreads();
      if (wid == 0) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          unsigned v = lane < NW ? wsum[t][lane] : 0u;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned w = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += w;
          }
          if (lane < NW) wsum[t][lane] = v;
        }
      }
      __syncthreads();
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        unsigned before = (wid ? wsum[t][wid - 1] : 0u) + incl[t] - tsum[t];
        if (before <= rk[t] && rk[t] < before + tsum[t]) {  // this thread's 4 bins hold the rank
          const uint4 hv = reinterpret_cast<const uint4*>(&hist[round == 0 ? 0 : t][0])[tid];
          const unsigned cv[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
          for (int q = 0; q < kCutBPT; ++q) {
            if (before <= rk[t] && rk[t] < before + cv[q]) {
              sel[t][0] = (unsigned)(kCutBPT * tid + q);
              sel[t][1] = before;
            }
            before += cv[q];
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        bin[t] = round == 0 ? sel[t][0] : ((bin[t] << (sh0 - sh1)) | sel[t][0]);
        rk[t] -= sel[t][1];
      }
      __syncthreads();
    }
    if (tid == 0) {  // bin[t] = d >> sh1 of the target: its key lies in kmin + [bin << sh1, (bin + 1) << sh1)
      const unsigned w1 = (1u << sh1) - 1u;
      cuts[4 * (size_t)j] = (float)from_key_f32(kmn + (bin[0] << sh1));
      cuts[4 * (size_t)j + 1] = (float)from_key_f32(kmn + (bin[1] << sh1) + w1);
      cuts[4 * (size_t)j + 2] = (float)from_key_f32(kmn + (bin[2] << sh1) + (w1 >> 1));
      cuts[4 * (size_t)j + 3] = 0.f;
    }
  }
}

template <int MODE>
__device__ __forceinline__ PassPartial batch_pass(BatchState& st, float* zbuf, uint64_t cap, float* sbuf) {
  using Fn = PassFn<float, MODE, 4>;
  __shared__ CompactShared cs;
  Fn f;
  f.sbuf = sbuf;
  if (MODE == kCompact) {
    if (threadIdx.x == 0) cs.n[0] = cs.n[1] = 0u;
    __syncthreads();
  }
  f.t = st.tq; f.yL = st.yL; f.yR = st.yR;
  f.c_lt = f.c_eq = f.c_lo = f.c_hi = 0;
  f.L_lo = f.L_hi = f.P = f.N = 0.0;
  f.pred = -tinf<float>(); f.succ = tinf<float>();
  f.lo_bits = f.hi_bits = 0u;
  f.cs = &cs;
  f.z = zbuf;
  f.z_cap = cap;
  f.cursors = st.cursors;
  stream_array<float, 4>(st.cur, st.n_cur, f, 0u, 1u);
  if (MODE == kCompact) f.finish();
  PassPartial p;
  p.c_lt = f.c_lt; p.c_eq = f.c_eq; p.c_lo = f.c_lo; p.c_hi = f.c_hi;
  p.L_lo = f.L_lo; p.L_hi = f.L_hi; p.P = f.P; p.N = f.N;
  p.pred = (double)f.pred; p.succ = (double)f.succ;
  return block_reduce(p);
}

__global__ void __launch_bounds__(kBlock, 4) batched_select_kernel(BatchArgs a) {
  __shared__ BatchState st;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  float* sbuf = reinterpret_cast<float*>(dyn_smem);
  const uint64_t n = a.n, k = a.k;
  float* my0 = a.scratch + (size_t)blockIdx.x * 2 * a.cap;
  float* my1 = my0 + a.cap;
  for (;;) {
    if (threadIdx.x == 0) {
      st.col = (int)atomicAdd(a.next_col, 1u);
      st.cursors[0] = st.cursors[1] = 0ull;
    }
    __syncthreads();
    if (st.col >= (int)a.C) break;
    const float* x = a.S ? a.S + (size_t)st.col * n : nullptr;
    unsigned* keys32 = reinterpret_cast<unsigned*>(dyn_smem);
    if (a.f_le) {
      // ---- fused LMS input: the fused residual pass took the init statistics, counted at the two
      //      cuts and copied ]t_lo, t_hi[ out (a1 + R23 + a4); start from that bracket
      if (threadIdx.x == 0) {
        const int c = st.col;
        const float tl = a.f_cuts[4 * (size_t)c], th = a.f_cuts[4 * (size_t)c + 1], tm = a.f_cuts[4 * (size_t)c + 2];
        const unsigned long long le = a.f_le[c], written = a.f_cursor[c];
        st.phase = 0;
        st.iters = 0;
        atomicAdd(&a.stats[0], 1ull);
        if (tl < th && le < k && k <= le + written && written <= a.f_zcap) {
          // the target lies in ]t_lo, t_hi[ (c_le(t_lo) < k <= c_lt(t_hi)) whose copy is z_j
          st.yL = tl; st.yR = th; st.c_le_L = le; st.c_lt_R = le + written; st.m = written;
          st.cur = a.f_z + (size_t)c * a.f_zcap; st.n_cur = written; st.cur_buf = -1;
          st.D_lo = le; st.on_z = 1; st.slow = 0; st.bisect = 0;
          st.exact = 1; st.cuts_stalled = 0; st.free_step = 0; st.tgt = 0;
          st.t = (tm > tl && tm < th) ? (double)tm : 0.5 * (double)tl + 0.5 * (double)th;  // R25
          if (st.m <= (unsigned long long)kBatchFinish) { st.k_r = k - st.c_le_L; st.phase = 2; }
        } else {  // needs full passes over the column: deferred to the stored-S fallback
          a.fail_list[atomicAdd(a.fail_count, 1u)] = (unsigned)c;
          st.phase = 4;
        }
      }
      __syncthreads();
    } else {
    // ---- R23/R29: two extra cuts at quantiles of 8192 strided samples bracketing rank k
    const bool cut = n > 2;
    if (cut) batch_sample_cuts<kBatchSample>(st, keys32, x, n, k);
    // ---- a1 + a4: init reduction over the column, the two extra cuts and the copy_if of
    //      ]t_lo, t_hi[ into this CTA's buffer 0, in one read (R23)
    {
      __shared__ CompactShared cs;
      BatchInitFn f;
      f.mn = tinf<float>(); f.mx = -tinf<float>();
      f.tl = cut ? st.cut_lo : x[0];
      f.th = cut ? st.cut_hi : x[0];
      f.pc.cs = &cs;
      f.pc.sbuf = sbuf;
      f.pc.z = my0;
      f.pc.z_cap = a.cap;
      f.pc.cursors = st.cursors;
      __syncthreads();
      stream_array<float, 4>(x, n, f, 0u, 1u);
      f.pc.finish();
      InitPartial p;
      p.vmin = (double)f.mn; p.vmax = (double)f.mx; p.S = 0; p.pad = 0;
      p.cnt_min = f.cmn; p.cnt_max = f.cmx; p.nonfinite = f.nan; p.pad2 = 0;
      p.N0 = f.N0; p.P0 = f.P0; p.I0 = f.I0;
      p.cA = (unsigned long long)f.fL; p.cB = p.cC = p.cD = p.cE = 0;  // cA = #x<=t_lo
      p = block_reduce(p);
      __syncthreads();  // compaction cursor final
      if (threadIdx.x == 0) {
        const unsigned long long written = st.cursors[0];
        st.cursors[0] = st.cursors[1] = 0ull;
        p.cC = p.cA + written;  // #x<t_hi: every x < t_hi is <= t_lo or interior
        p.pad2 = written;
        atomicAdd(&a.stats[1], (unsigned long long)(4 * written));
      }
      if (threadIdx.x == 0) {
        st.phase = 0;
        st.iters = 0;
        atomicAdd(&a.stats[0], 1ull);
        atomicAdd(&a.stats[1], (unsigned long long)(4 * n));
        if (p.nonfinite) {
          st.result = __int_as_float(0x7fc00000);
          atomicAdd(&a.stats[3], 1ull);
          st.phase = 1;
        } else {
          // the bracket starts just outside the extremes (their multiplicities are not counted,
          // R27): #x<=prev(min) = 0, #x<next(max) = n
          st.yL = nextafterf((float)p.vmin, -INFINITY); st.yR = nextafterf((float)p.vmax, INFINITY);
          st.c_le_L = 0; st.c_lt_R = n;
          st.m = n;
          st.D_lo = 0; st.on_z = 0; st.slow = 0; st.bisect = 0;
          st.exact = 1; st.cuts_stalled = 0; st.free_step = 0;
          st.cur = x; st.n_cur = n; st.cur_buf = -1; st.tgt = 0;
          st.t = 0.5 * p.vmin + 0.5 * p.vmax;  // only used if neither cut lies strictly inside
          if (cut) {  // the two extra cuts, as the host driver applies them (R23-R25)
            // the batched init pass keeps only #x<=t_lo and the interior count: the usual bracket
            // ]t_lo, t_hi[ starts from the sample's estimate of the target (R25); a cut on the far
            // side of the target moves to the adjacent float and the iteration starts from the
            // midpoint
            const double tl = st.cut_lo, th = st.cut_hi;
            bool settled = false, mean_ok = false;
            // (an open cut of an extreme rank, R31, lies outside the bracket with nothing between)
            const bool lo_open = tl <= (double)st.yL && p.cA == 0;
            if (tl > (double)st.yL && tl < (double)st.yR) {
              const unsigned long long c_le = p.cA;
              if (c_le < k) {
                st.yL = (float)tl; st.c_le_L = c_le; st.m = st.c_lt_R - c_le;
              } else {  // y_R <- next(t_lo): #x<next(t_lo) = #x<=t_lo
                st.yR = nextafterf((float)tl, INFINITY); st.c_lt_R = c_le; st.m = c_le - st.c_le_L;
                settled = true;
              }
            }
            if (!settled && th > (double)st.yL && th < (double)st.yR) {
              const unsigned long long c_lt = p.cC;
              if (c_lt >= k) {
                st.yR = (float)th; st.c_lt_R = c_lt; st.m = c_lt - st.c_le_L;
                if (((double)st.yL == tl || lo_open) && st.cut_mid > st.yL && st.cut_mid < st.yR) {
                  st.t = st.cut_mid;  // the sample's estimate of the target (R25)
                  mean_ok = true;
                }
              } else {  // y_L <- prev(t_hi): #x<=prev(t_hi) = #x<t_hi
                st.yL = nextafterf((float)th, -INFINITY); st.c_le_L = c_lt; st.m = st.c_lt_R - c_lt;
              }
            }
            if (!mean_ok) st.t = 0.5 * (double)st.yL + 0.5 * (double)st.yR;
            if (!isfinite(st.t)) st.t = 0.5 * p.vmin + 0.5 * p.vmax;
            // the init pass already copied out ]t_lo, t_hi[: if that is the bracket, continue on it
            const bool hi_open = th >= (double)st.yR && p.cC == n;
            if (st.phase == 0 && ((double)st.yL == tl || lo_open) && ((double)st.yR == th || hi_open) &&
                st.m == p.pad2 && p.pad2 <= a.cap) {
              st.cur = my0; st.n_cur = p.pad2; st.cur_buf = 0;
              st.D_lo = st.c_le_L; st.on_z = 1;
              if (st.m <= (unsigned long long)kBatchFinish) { st.k_r = k - st.c_le_L; st.phase = 2; }
            }
          }
        }
      }
      __syncthreads();
    }
    }
    // ---- a2/a3/a4: Kelley iterations
    while (st.phase == 0) {
      // R26 cut step: a compacted bracket larger than the shared-memory finish is cut at two
      // quantiles of 1024 samples of its own; only what lies between them is copied
      if (st.on_z && st.exact && !st.cuts_stalled && !st.bisect && st.m > (unsigned long long)kBatchFinish) {
        batch_sample_cuts<kBatchCutSample>(st, keys32, st.cur, st.n_cur, k - st.c_le_L);
        if (threadIdx.x == 0) st.tgt = (st.cur_buf == 0) ? 1 : 0;
        __syncthreads();
        float* zbuf = st.tgt == 0 ? my0 : my1;
        __shared__ CompactShared cs2;
        BatchInitFn f;
        f.mn = tinf<float>(); f.mx = -tinf<float>();
        f.tl = st.cut_lo; f.th = st.cut_hi;
        f.pc.cs = &cs2; f.pc.sbuf = sbuf; f.pc.z = zbuf; f.pc.z_cap = a.cap; f.pc.cursors = st.cursors;
        __syncthreads();
        stream_array<float, 4>(st.cur, st.n_cur, f, 0u, 1u);
        f.pc.finish();
        unsigned long long le_loc = (unsigned long long)f.fL;
#pragma unroll
        for (int o = 16; o; o >>= 1) le_loc += __shfl_xor_sync(FULL, le_loc, o);
        __shared__ unsigned long long le_w[kWarps];
        if ((threadIdx.x & 31) == 0) le_w[threadIdx.x >> 5] = le_loc;
        __syncthreads();  // (also: compaction cursor final)
        if (threadIdx.x == 0) {
          unsigned long long le_part = 0;
          for (int q = 0; q < kWarps; ++q) le_part += le_w[q];
          const unsigned long long written = st.cursors[0];
          st.cursors[0] = st.cursors[1] = 0ull;
          atomicAdd(&a.stats[0], 1ull);
          atomicAdd(&a.stats[1], (unsigned long long)(4 * (st.n_cur + written)));
          const unsigned long long le_a = st.c_le_L + le_part, lt_b = le_a + written;
          const float ta = st.cut_lo, tb = st.cut_hi;
          const unsigned long long m_old = st.m;
          if (++st.iters > (int)a.max_iters) {
            st.result = __int_as_float(0x7fc00000);
            atomicAdd(&a.stats[2], 1ull);
            st.phase = 1;
          } else if (le_a < k && k <= lt_b && ta < tb) {  // continue on the copy of ]t_a, t_b[
            st.yL = ta; st.yR = tb; st.c_le_L = le_a; st.c_lt_R = lt_b; st.m = written;
            st.cur = zbuf; st.n_cur = written; st.cur_buf = st.tgt; st.D_lo = le_a; st.exact = 1;
            if (st.m > m_old / 2) st.cuts_stalled = 1;
            st.t = (st.cut_mid > ta && st.cut_mid < tb) ? (double)st.cut_mid : 0.5 * (double)ta + 0.5 * (double)tb;
            st.free_step = 1;
            if (st.m <= (unsigned long long)kBatchFinish) { st.k_r = k - st.c_le_L; st.phase = 2; }
          } else {  // the target is outside: move to the adjacent float of the cut (R24)
            if (k <= le_a) {
              st.yR = nextafterf(ta, INFINITY); st.c_lt_R = le_a; st.m = le_a - st.c_le_L;
            } else if (ta == tb) {
              st.yL = ta; st.c_le_L = le_a; st.m = st.c_lt_R - le_a;
            } else {
              st.yL = nextafterf(tb, -INFINITY); st.c_le_L = lt_b; st.m = st.c_lt_R - lt_b;
            }
            st.exact = 0;
            st.cuts_stalled = 1;
            st.t = (st.cut_mid > st.yL && st.cut_mid < st.yR) ? (double)st.cut_mid
                                                               : 0.5 * (double)st.yL + 0.5 * (double)st.yR;
            st.free_step = 1;
          }
        }
        __syncthreads();
        continue;
      }
      if (threadIdx.x == 0) {
        const double tt = st.bisect ? (double)key_mid_dev(st.yL, st.yR) : st.t;
        st.tq = snap_dev(tt, st.yL, st.yR);
        st.compact = st.on_z || st.m <= a.cap;
        st.tgt = (st.cur_buf == 0) ? 1 : 0;
      }
      __syncthreads();
      float* zbuf = st.tgt == 0 ? my0 : my1;
      PassPartial tot = st.compact ? batch_pass<kCompact>(st, zbuf, a.cap, sbuf) : batch_pass<kHot>(st, zbuf, a.cap, sbuf);
      __syncthreads();  // compaction cursors complete
      if (threadIdx.x == 0) {
        const unsigned long long zl = st.cursors[0], zh = st.cursors[1];
        st.cursors[0] = st.cursors[1] = 0ull;
        atomicAdd(&a.stats[0], 1ull);
        atomicAdd(&a.stats[1], (unsigned long long)(4 * (st.n_cur + (st.compact ? zl + zh : 0))));
        // compaction passes carry no counters: derive them from the compaction totals
        const unsigned long long c_lt = st.compact ? st.c_le_L + zl : st.D_lo + tot.c_lt;
        const unsigned long long c_le = st.compact ? c_lt + (st.m - zl - zh) : c_lt + tot.c_eq;
        const float tq = st.tq;
        const unsigned long long m_old = st.m;
        if (++st.iters > (int)a.max_iters) {
          st.result = __int_as_float(0x7fc00000);
          atomicAdd(&a.stats[2], 1ull);
          st.phase = 1;
        } else if (c_lt < k && k <= c_le) {
          st.result = tq; st.phase = 1;
        } else if (c_le < k) {
          const unsigned long long c_hi = st.c_lt_R - c_le;
          if (c_le + 1 == k && isfinite(tot.succ)) {
            st.result = (float)tot.succ; st.phase = 1;
          } else {
            st.yL = tq; st.c_le_L = c_le; st.m = c_hi;
            st.t = (double)tq + tot.L_hi / (double)c_hi;
            st.side = 1;
          }
        } else {
          const unsigned long long c_lo = c_lt - st.c_le_L;
          if (c_lt == k && isfinite(tot.pred)) {
            st.result = (float)tot.pred; st.phase = 1;
          } else {
            st.yR = tq; st.c_lt_R = c_lt; st.m = c_lo;
            st.t = (double)tq - tot.L_lo / (double)c_lo;
            st.side = 0;
          }
        }
        if (st.phase == 0) {
          if (st.compact) {
            float* base = st.tgt == 0 ? my0 : my1;
            st.cur = st.side == 0 ? base : base + (a.cap - zh);
            st.n_cur = st.side == 0 ? zl : zh;
            st.cur_buf = st.tgt;
            st.D_lo = st.c_le_L;
            st.on_z = 1;
            st.exact = 1;
            if (st.m <= (unsigned long long)kBatchFinish) {
              st.k_r = k - st.c_le_L;  // rank inside the kept half
              st.phase = 2;
            }
          }
          if (st.free_step) {
            st.free_step = 0;
          } else if (st.m > m_old - m_old / 8) {
            if (++st.slow >= 2) st.bisect = 1;
          } else {
            st.slow = 0;
            st.bisect = 0;
          }
        }
      }
      __syncthreads();
    }
    // ---- a5: exact finish on <= kBatchFinish elements: block radix select of their keys
    if (st.phase == 2) {
      const uint32_t cnt = (uint32_t)st.n_cur;
      constexpr int PER = kBatchFinish / kBlock;
      unsigned key[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const uint32_t i = threadIdx.x + u * kBlock;
        key[u] = i < cnt ? (unsigned)okey(st.cur[i]) : ~0u;
      }
      const unsigned rk[1] = {(unsigned)(st.k_r - 1)};
      unsigned out[1];
      block_radix_select<PER, 1>(key, keys32, rk, out);
      if (threadIdx.x == 0) st.result = (float)from_key_f32(out[0]);
    }
    __syncthreads();
    if (threadIdx.x == 0 && st.phase != 4) {
      const float r = st.result;
      a.out[a.out_map ? a.out_map[st.col] : (unsigned)st.col] = r == 0.0f ? 0.0f : r;  // canonical +0 (R13)
    }
    __syncthreads();
  }
}


// ------------------------------------------------------------------------------------------
// §8f-3 device-resident Kelley loop: the step kernel (one thread) = drive()'s Kelley step.  It
// consumes the pass that just ran (if any), then schedules the next one through the graph's
// conditional handles: hw (the WHILE), hh (hot pass), hs0 / hs1 (compacting pass with bracket
// tests / all inside), hrs / hrd (after the loop: radix rounds over a segmented / dense kept half).
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <typename T> __device__ double ks_snap(double t, double yL, double yR);
template <> __device__ double ks_snap<float>(double t, double yL, double yR) {
  const float fl = (float)yL, fr = (float)yR;
  float f = isfinite(t) ? (float)t : (float)(0.5 * yL + 0.5 * yR);
  if (!(f > fl)) f = nextafterf(fl, INFINITY);
  if (!(f < fr)) f = nextafterf(fr, -INFINITY);
  return f;
}
template <> __device__ double ks_snap<double>(double t, double yL, double yR) {
  double f = isfinite(t) ? t : 0.5 * yL + 0.5 * yR;
  if (!(f > yL)) f = ::nextafter(yL, (double)INFINITY);
  if (!(f < yR)) f = ::nextafter(yR, -(double)INFINITY);
  return f;
}
template <typename T> __device__ double ks_key_mid(double yL, double yR) {
  const unsigned long long a = okey((T)yL), b = okey((T)yR);
  const unsigned long long c = a + (b - a) / 2;
  return sizeof(T) == 4 ? from_key_f32(c) : from_key_f64(c);
}
struct KHandles {
  cudaGraphConditionalHandle hw, hh, hs0, hs1, hrs, hrd;
};
__device__ void ks_set(const KHandles& h, unsigned w, unsigned hot, unsigned s0, unsigned s1, unsigned rs, unsigned rd) {
  cudaGraphSetConditional(h.hw, w);
  cudaGraphSetConditional(h.hh, hot);
  cudaGraphSetConditional(h.hs0, s0);
  cudaGraphSetConditional(h.hs1, s1);
  cudaGraphSetConditional(h.hrs, rs);
  cudaGraphSetConditional(h.hrd, rd);
}
// the counters into the mapped report (before the value is published)
__device__ void ks_report(KelleyState& s) {
  KelleyReport* r = s.rep;
  r->error = s.error;
  r->exit_reason = s.exit_reason;
  r->passes = s.passes;
  r->cp_iters = s.cp_iters;
  r->fallback = s.fallback;
  r->launches = s.launches;
  r->n_rows = s.n_rows;
  r->bytes_moved = s.bytes_moved;
  r->z_count = s.z_count;
  __threadfence_system();
}
// the loop ends with a value (hit / adjacency) or an error: publish it, run nothing more
__device__ void ks_finish(KelleyState& s, const KHandles& h, double v, unsigned reason, int error) {
  s.done = 1;
  s.error = error;
  s.value = v;
  s.exit_reason = reason;
  ks_set(h, 0, 0, 0, 0, 0, 0);
  ks_report(s);
  if (s.vout) *s.vout = v;
  publish_done(s.done_flag, s.seq);
}
__device__ void ks_row(KelleyState& s, const KRow& r) {
  if (s.record && s.n_rows < (unsigned)kKelleyMaxRows) s.rep->rows[s.n_rows] = r;
  s.n_rows++;
}
template <typename T>
__global__ void kelley_step_kernel(KelleyState* sp, KHandles h) {
  if (threadIdx.x != 0) return;
  KelleyState& s = *sp;
  constexpr unsigned long long es = sizeof(T);
  if (s.done) {  // (defensive: the WHILE already stopped)
    ks_set(h, 0, 0, 0, 0, 0, 0);
    return;
  }
  if (s.pending) {
    // ---- the pass at tq just ran: its tuple -> counts, F, the rank test, the bracket update
    s.pending = 0;
    const DevPass r = s.tuple;
    const bool compact = s.compact != 0;
    const unsigned long long now = gtimer_ns();
    s.passes++;
    s.cp_iters++;
    s.launches += 1;
    const unsigned long long zl = r.z_lo, zh = r.z_hi;
    s.bytes_moved += s.n_cur * es + (compact ? (zl + zh) * es : 0ull);
    const unsigned long long c_lt = compact ? s.c_le_L + zl : s.D_lo + r.c_lt;
    const unsigned long long c_le = compact ? c_lt + (s.m - zl - zh) : c_lt + r.c_eq;
    // F_k(tq) from positive terms only (App. A identities; Eq. 2 with paper-k = n-k+1, R2)
    const double tq = s.tq;
    const double N_t = s.N_L + (double)s.c_le_L * (tq - s.yL) + r.L_lo;
    const double P_t = s.P_R + (double)(s.n - s.c_lt_R) * (s.yR - tq) + r.L_hi;
    KRow row;
    row.t = tq;
    row.F = s.wP * P_t + s.wN * N_t;
    row.c_lt = c_lt;
    row.c_eq = c_le - c_lt;
    row.interior = 0;
    row.scanned = s.n_cur;
    row.written = compact ? zl + zh : 0ull;
    row.kind = (unsigned)s.kind;
    row.compacted = compact ? 1u : 0u;
    row.kernel_ms = 1e-6 * (double)(now - s.t_start_ns);  // this pass, graph-node overheads included
    const unsigned long long k = s.k;
    // step 1.3: 0 in dF(t) <=> c_lt < k <= c_le -> t = x_(k)
    if (c_lt < k && k <= c_le) {
      ks_row(s, row);
      ks_finish(s, h, tq, 2u, 0);
      return;
    }
    const unsigned long long m_old = s.m;
    int side;
    if (c_le < k) {  // dF(t) < 0: y_L <- t (sign per R1)
      const unsigned long long c_hi = s.c_lt_R - c_le;
      if (c_le + 1 == k && isfinite(r.succ)) {  // x_(k) = successor of t (P:L192 footnote, mirrored)
        ks_row(s, row);
        ks_finish(s, h, r.succ, 4u, 0);
        return;
      }
      if (compact && zh != c_hi) {
        ks_finish(s, h, 0.0, 0u, 1);
        return;
      }
      s.yL = tq; s.N_L = N_t; s.c_le_L = c_le; s.m = c_hi;
      s.t = tq + r.L_hi / (double)c_hi;  // mean of ]t, yR[ (App. A)
      side = 1;
    } else {  // c_lt >= k: y_R <- t
      const unsigned long long c_lo = c_lt - s.c_le_L;
      if (c_lt == k && isfinite(r.pred)) {  // x_(k) = largest x < t (P:L192 footnote)
        ks_row(s, row);
        ks_finish(s, h, r.pred, 3u, 0);
        return;
      }
      if (compact && zl != c_lo) {
        ks_finish(s, h, 0.0, 0u, 1);
        return;
      }
      s.yR = tq; s.P_R = P_t; s.c_lt_R = c_lt; s.m = c_lo;
      s.t = tq - r.L_lo / (double)c_lo;  // mean of ]yL, t[ (App. A)
      side = 0;
    }
    row.interior = s.m;
    ks_row(s, row);
    if (compact) {
      const unsigned long long hn = side == 0 ? zl : zh;
      if (s.m <= s.select_cap) {
        // hybrid finish: the exact select in the kept half, by the radix rounds after the loop
        s.sel_r = k - s.c_le_L;
        s.sel_m = hn;
        s.z_count = hn;
        if (s.dense) {
          s.sel_base = static_cast<const char*>(s.zb[s.tgt]) + (side == 0 ? 0ull : (s.cap - zh)) * es;
          s.sel_tab = nullptr;
          s.sel_side = 0;
          s.sel_seg = 0;
        } else {
          s.sel_base = s.sb[s.tgt];
          s.sel_tab = s.st[s.tgt];
          s.sel_side = side;
          s.sel_seg = 1;
        }
        s.bytes_moved += (unsigned long long)(sizeof(T) == 4 ? 3 : 6) * hn * es;
        s.launches += sizeof(T) == 4 ? 3u : 6u;
        s.exit_reason = 5u;
        s.done = 1;
        ks_set(h, 0, 0, 0, 0, s.sel_seg ? 1u : 0u, s.sel_seg ? 0u : 1u);
        ks_report(s);  // the last radix round publishes the value
        return;
      }
      // continue the cutting plane on the kept half only (multi-level compaction, §8f-1)
      if (s.dense) {
        s.cur_seg = 0;
        s.cur = static_cast<const char*>(s.zb[s.tgt]) + (side == 0 ? 0ull : (s.cap - zh)) * es;
        s.cur_dbuf = s.tgt;
      } else {
        s.cur_seg = 1;
        s.cur = s.sb[s.tgt];
        s.cur_tab = s.st[s.tgt];
        s.cur_side = side;
        s.cur_sbuf = s.tgt;
      }
      s.n_cur = hn;
      s.D_lo = s.c_le_L;
      s.on_z = 1;
      s.exact = 1;
    }
    // progress safeguard (R7): two consecutive steps keeping > 7/8 of the interior switch to
    // ordered-key bisection until progress resumes
    if (s.free_step) {
      s.free_step = 0;
    } else if (s.m > m_old - m_old / 8) {
      if (++s.slow >= 2) s.bisect = 1;
    } else {
      s.slow = 0;
      s.bisect = 0;
    }
  }
  // ---- schedule the next pass
  if (++s.it > s.max_iters || s.m == 0) {
    ks_finish(s, h, 0.0, 0u, 1);
    return;
  }
  s.kind = 0;
  if (s.bisect) {
    s.t = ks_key_mid<T>(s.yL, s.yR);
    s.kind = 1;
    s.fallback++;
  }
  const double tq = ks_snap<T>(s.t, s.yL, s.yR);
  if (!(tq > s.yL && tq < s.yR)) {
    ks_finish(s, h, 0.0, 0u, 1);
    return;
  }
  s.tq = tq;
  s.compact = (s.on_z || s.m <= s.z_cap) ? 1 : 0;
  s.dense = s.m <= s.dense_cap ? 1 : 0;
  if (s.compact) {
    s.tgt = s.dense ? (s.cur_dbuf == 0 ? 1 : 0) : (s.cur_sbuf == 0 ? 1 : 0);
    s.inside = (s.cur != s.x && s.exact) ? 1 : 0;
    s.last_dense = s.dense;
  }
  s.pending = 1;
  s.t_start_ns = gtimer_ns();
  ks_set(h, 1, s.compact ? 0u : 1u, (s.compact && !s.inside) ? 1u : 0u, (s.compact && s.inside) ? 1u : 0u, 0, 0);
}
}  // namespace

// ==========================================================================================
cudaError_t query_shapes(int device, LaunchShape* s) {
  cudaError_t e = cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return e;
  int b;
#define OCC(DT, T, MODE)                                   \
  if ((e = occ_pass<T, MODE>(&b)) != cudaSuccess) return e; \
  s->grid_pass[DT][MODE] = s->num_sms * (b > 0 ? b : 1);
  OCC(kF32, float, kHot) OCC(kF32, float, kCompact) OCC(kF32, float, kDirect)
  OCC(kF64, double, kHot) OCC(kF64, double, kCompact) OCC(kF64, double, kDirect)
#undef OCC
  {
    int cb = 0;
#define COOP(DT, T, SEGV, NTV)                                                                                      \
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cb, radix_coop_kernel<T, SEGV, NTV>, NTV, 0)) !=       \
      cudaSuccess)                                                                                                 \
    return e;                                                                                                      \
  s->coop_max[DT][SEGV ? 1 : 0][NTV == 1024 ? 1 : 0] = s->num_sms * cb;
    COOP(kF32, float, false, 256) COOP(kF32, float, true, 256) COOP(kF64, double, false, 256)
    COOP(kF64, double, true, 256) COOP(kF32, float, false, 1024) COOP(kF32, float, true, 1024)
    COOP(kF64, double, false, 1024) COOP(kF64, double, true, 1024)
#undef COOP
  }
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, seg_pass_kernel<float, false>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_seg[kF32] = s->num_sms * (b > 0 ? b : 1);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, seg_pass_kernel<double, false>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_seg[kF64] = s->num_sms * (b > 0 ? b : 1);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, init_kernel<float, 4, false, true>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_init[kF32] = s->num_sms * (b > 0 ? b : 1);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, init_kernel<double, 4, false, true>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_init[kF64] = s->num_sms * (b > 0 ? b : 1);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, radix_round_kernel<float, false>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_hist[kF32] = s->num_sms * (b > 0 ? b : 1);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, radix_round_kernel<double, false>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_hist[kF64] = s->num_sms * (b > 0 ? b : 1);
  return cudaSuccess;
}

size_t partial_bytes_needed(const LaunchShape& s) {
  int g = 0;
  for (int d = 0; d < 2; ++d) {
    g = g > s.grid_seg[d] ? g : s.grid_seg[d];
    for (int m = 0; m < 3; ++m) g = g > s.grid_pass[d][m] ? g : s.grid_pass[d][m];
    g = g > s.grid_init[d] ? g : s.grid_init[d];
  }
  const size_t per = sizeof(PassPartial) > sizeof(InitPartial) ? sizeof(PassPartial) : sizeof(InitPartial);
  return (size_t)g * per;
}

constexpr int kRadixPerCta = 16384;  // elements per CTA of a radix round
static int clamp_grid(int grid, uint64_t n, int per_cta) {
  const uint64_t need = (n + per_cta - 1) / per_cta;
  if (need < (uint64_t)grid) grid = (int)(need > 0 ? need : 1);
  return grid;
}

template <typename T>
static void launch_init_t(const InitArgs& a, int grid, cudaStream_t st, bool checked) {
  const bool cut = a.t0 != nullptr;
  if (checked) {
    if (cut) init_kernel<T, 4, true, true><<<grid, kBlock, 0, st>>>(a);
    else init_kernel<T, 4, true, false><<<grid, kBlock, 0, st>>>(a);
  } else {
    if (cut) init_kernel<T, 4, false, true><<<grid, kBlock, 0, st>>>(a);
    else init_kernel<T, 4, false, false><<<grid, kBlock, 0, st>>>(a);
  }
}

cudaError_t launch_init(int dtype, const InitArgs& a, const LaunchShape& s, cudaStream_t st, bool checked) {
  if (dtype == kF32) launch_init_t<float>(a, clamp_grid(s.grid_init[kF32], a.n, kBlock * 4 * 4), st, checked);
  else launch_init_t<double>(a, clamp_grid(s.grid_init[kF64], a.n, kBlock * 4 * 2), st, checked);
  return cudaGetLastError();
}

cudaError_t launch_sample_cut(int dtype, const void* x, uint64_t n, uint64_t k, void* t0, cudaStream_t st,
                              uint32_t smax, unsigned long long* keys_out) {
  if (dtype == kF32)
    sample_cut_kernel<float><<<1, 1024, 0, st>>>(static_cast<const float*>(x), n, k, static_cast<float*>(t0), smax,
                                                 keys_out);
  else
    sample_cut_kernel<double><<<1, 1024, 0, st>>>(static_cast<const double*>(x), n, k, static_cast<double*>(t0), smax,
                                                  keys_out);
  return cudaGetLastError();
}

cudaError_t launch_pass(int dtype, const PassArgs& a, const LaunchShape& s, cudaStream_t st) {
  const int per = kBlock * 4 * (dtype == kF32 ? 4 : 2);
  const int grid = clamp_grid(s.grid_pass[dtype][a.mode], a.n, per);
  if (dtype == kF32) {
    switch (a.mode) {
      case kHot: return launch_pass_t<float, kHot>(a, grid, st);
      case kCompact: return launch_pass_t<float, kCompact>(a, grid, st);
      default: return launch_pass_t<float, kDirect>(a, grid, st);
    }
  }
  switch (a.mode) {
    case kHot: return launch_pass_t<double, kHot>(a, grid, st);
    case kCompact: return launch_pass_t<double, kCompact>(a, grid, st);
    default: return launch_pass_t<double, kDirect>(a, grid, st);
  }
}


// ---- §8f-3: the device-resident Kelley loop as one CUDA graph -------------------------------
static cudaError_t add_kernel(cudaGraph_t g, cudaGraphNode_t* node, const cudaGraphNode_t* deps, size_t ndeps,
                              const void* fn, dim3 grid, dim3 block, size_t smem, void** args) {
  cudaKernelNodeParams kp = {};
  kp.func = const_cast<void*>(fn);
  kp.gridDim = grid;
  kp.blockDim = block;
  kp.sharedMemBytes = (unsigned)smem;
  kp.kernelParams = args;
  return cudaGraphAddKernelNode(node, g, deps, ndeps, &kp);
}
static cudaError_t add_cond(cudaGraph_t g, cudaGraphNode_t* node, const cudaGraphNode_t* deps, size_t ndeps,
                            cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type, cudaGraph_t* body) {
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = 1;
  cudaError_t e = cudaGraphAddNode(node, g, deps, ndeps, &p);
  if (e == cudaSuccess) *body = p.conditional.phGraph_out[0];
  return e;
}

template <typename T>
static cudaError_t kelley_graph_t(const LaunchShape& s, KelleyState* ks, void* partials, unsigned* ticket,
                                  unsigned long long* cursors, RadixState* rstate, unsigned* hist,
                                  cudaGraphExec_t* out) {
  const int dt = sizeof(T) == 4 ? kF32 : kF64;
  cudaGraph_t g = nullptr;
  cudaError_t e;
#define GK(x)                        \
  do {                               \
    if ((e = (x)) != cudaSuccess) {  \
      if (g) cudaGraphDestroy(g);    \
      return e;                      \
    }                                \
  } while (0)
  GK(cudaGraphCreate(&g, 0));
  KHandles h{};
  GK(cudaGraphConditionalHandleCreate(&h.hw, g, 1, cudaGraphCondAssignDefault));
  GK(cudaGraphConditionalHandleCreate(&h.hrs, g, 0, cudaGraphCondAssignDefault));
  GK(cudaGraphConditionalHandleCreate(&h.hrd, g, 0, cudaGraphCondAssignDefault));
  cudaGraphNode_t nw, nrs, nrd;
  cudaGraph_t body, brs, brd;
  GK(add_cond(g, &nw, nullptr, 0, h.hw, cudaGraphCondTypeWhile, &body));
  GK(cudaGraphConditionalHandleCreate(&h.hh, body, 0, cudaGraphCondAssignDefault));
  GK(cudaGraphConditionalHandleCreate(&h.hs0, body, 0, cudaGraphCondAssignDefault));
  GK(cudaGraphConditionalHandleCreate(&h.hs1, body, 0, cudaGraphCondAssignDefault));
  // body: step -> IF hot -> IF compacting (bracket tests) -> IF compacting (all inside)
  KHandles hs_arg = h;  // (kernel-node parameters are copied when the node is created)
  KelleyState* ks_arg = ks;
  void* step_args[] = {&ks_arg, &hs_arg};
  cudaGraphNode_t nstep, nh, ns0, ns1;
  GK(add_kernel(body, &nstep, nullptr, 0, (const void*)kelley_step_kernel<T>, dim3(1), dim3(32), 0, step_args));
  cudaGraph_t bh, bs0, bs1;
  GK(add_cond(body, &nh, &nstep, 1, h.hh, cudaGraphCondTypeIf, &bh));
  GK(add_cond(body, &ns0, &nh, 1, h.hs0, cudaGraphCondTypeIf, &bs0));
  GK(add_cond(body, &ns1, &ns0, 1, h.hs1, cudaGraphCondTypeIf, &bs1));
  PassArgs pa{};
  pa.ks = ks;
  pa.mode = kHot;
  pa.cursors = cursors;
  pa.partials = partials;
  pa.ticket = ticket;
  void* pa_args[] = {&pa};
  cudaGraphNode_t tmp;
  GK(add_kernel(bh, &tmp, nullptr, 0, (const void*)pass_kernel<T, kHot, 4>, dim3(s.grid_pass[dt][kHot]), dim3(kBlock),
                pass_smem<T, kHot>(), pa_args));
  SegArgs sa{};
  sa.ks = ks;
  sa.cursors = cursors;
  sa.partials = partials;
  sa.ticket = ticket;
  void* sa_args[] = {&sa};
  GK(add_kernel(bs0, &tmp, nullptr, 0, (const void*)seg_pass_kernel<T, false>, dim3(s.grid_seg[dt]), dim3(kBlock), 0,
                sa_args));
  GK(add_kernel(bs1, &tmp, nullptr, 0, (const void*)seg_pass_kernel<T, true>, dim3(s.grid_seg[dt]), dim3(kBlock), 0,
                sa_args));
  // after the loop: the radix rounds of the exact finish (segmented / dense kept half)
  GK(add_cond(g, &nrs, &nw, 1, h.hrs, cudaGraphCondTypeIf, &brs));
  GK(add_cond(g, &nrd, &nrs, 1, h.hrd, cudaGraphCondTypeIf, &brd));
  static const int plan32[] = {21, 11, 10, 11, 0, 10};
  static const int plan64[] = {53, 11, 42, 11, 31, 11, 20, 11, 10, 10, 0, 10};
  const int rounds = dt == kF32 ? 3 : 6;
  const int* plan = dt == kF32 ? plan32 : plan64;
  for (int segv = 0; segv < 2; ++segv) {
    cudaGraph_t bg = segv ? brs : brd;
    cudaGraphNode_t prev = nullptr;
    for (int i = 0; i < rounds; ++i) {
      RadixArgs ra{};
      ra.ks = ks;
      ra.st = rstate; ra.hist = hist; ra.ticket = ticket;
      ra.Wtot = s.grid_seg[dt] * kWarps;
      ra.shift = plan[2 * i]; ra.bits = plan[2 * i + 1];
      ra.first = i == 0; ra.last = i == rounds - 1;
      void* ra_args[] = {&ra};
      const void* fn = segv ? (const void*)radix_round_kernel<T, true> : (const void*)radix_round_kernel<T, false>;
      const int grid = segv ? s.grid_seg[dt] : s.grid_hist[dt];
      cudaGraphNode_t nn;
      GK(add_kernel(bg, &nn, prev ? &prev : nullptr, prev ? 1 : 0, fn, dim3(grid), dim3(kBlock), 0, ra_args));
      prev = nn;
    }
  }
  GK(cudaGraphInstantiate(out, g, 0));
  cudaGraphDestroy(g);
  return cudaSuccess;
#undef GK
}

cudaError_t kelley_graph_build(int dtype, const LaunchShape& s, KelleyState* ks, void* partials, unsigned* ticket,
                               unsigned long long* cursors, RadixState* rstate, unsigned* hist, cudaGraphExec_t* out) {
  if (dtype == kF32) return kelley_graph_t<float>(s, ks, partials, ticket, cursors, rstate, hist, out);
  return kelley_graph_t<double>(s, ks, partials, ticket, cursors, rstate, hist, out);
}

// A device buffer published to mapped host memory, then `seq` to *flag (the host spins on it instead
// of a stream synchronisation): the sharded path's all-gathered records.
__global__ void publish_kernel(const unsigned long long* __restrict__ src, unsigned long long* dst, uint32_t words,
                               unsigned long long* flag, unsigned long long seq) {
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) publish_done(flag, seq);
}
cudaError_t launch_publish(const void* src, void* dst_mapped, size_t bytes, unsigned long long* flag,
                           unsigned long long seq, cudaStream_t st) {
  publish_kernel<<<1, 256, 0, st>>>(static_cast<const unsigned long long*>(src),
                                    static_cast<unsigned long long*>(dst_mapped), (uint32_t)(bytes / 8), flag, seq);
  return cudaGetLastError();
}

int seg_total_warps(int dtype, const LaunchShape& s) { return s.grid_seg[dtype] * kWarps; }

cudaError_t launch_init_seg(int dtype, const InitArgs& ia, const SegArgs& a, const LaunchShape& s, cudaStream_t st,
                            bool sums) {
  // the same grid as seg_pass_kernel: its warp regions / run table are what later passes read
  const int g = s.grid_seg[dtype];
  if (dtype == kF32) {
    if (sums) return pdl_launch(init_seg_kernel<float, true>, dim3(g), dim3(kBlock), 0, st, ia, a);
    return pdl_launch(init_seg_kernel<float, false>, dim3(g), dim3(kBlock), 0, st, ia, a);
  } else {
    if (sums) return pdl_launch(init_seg_kernel<double, true>, dim3(g), dim3(kBlock), 0, st, ia, a);
    return pdl_launch(init_seg_kernel<double, false>, dim3(g), dim3(kBlock), 0, st, ia, a);
  }
  return cudaGetLastError();
}

uint64_t seg_region(int dtype, uint64_t n, const LaunchShape& s) {
  const uint64_t ve = dtype == kF32 ? 4 : 2;
  const uint64_t gw = 32 * kSegU * ve;  // elements per warp group
  const uint64_t wt = (uint64_t)seg_total_warps(dtype, s);
  const uint64_t groups = (n + gw - 1) / gw;
  return ((groups + wt - 1) / wt + 1) * gw + 64;  // + one ragged group + head/tail scalars
}

cudaError_t launch_seg_pass(int dtype, const SegArgs& a, bool inside, const LaunchShape& s, cudaStream_t st) {
  const int g = s.grid_seg[dtype];
  if (dtype == kF32) {
    if (inside) seg_pass_kernel<float, true><<<g, kBlock, 0, st>>>(a);
    else seg_pass_kernel<float, false><<<g, kBlock, 0, st>>>(a);
  } else {
    if (inside) seg_pass_kernel<double, true><<<g, kBlock, 0, st>>>(a);
    else seg_pass_kernel<double, false><<<g, kBlock, 0, st>>>(a);
  }
  return cudaGetLastError();
}

// The same, as ONE launch over a cluster of 8 CTAs (8 SMs, distributed shared memory): every CTA
// gathers KPT samples per thread straight into registers, builds its local histograms, and adds
// them into CTA 0's through DSMEM atomics; CTA 0 picks the digits and the others read the new
// prefixes back from it.  Replaces the global round trip of the keys and one launch, and spreads
// the sorting / histogram work over 8 SMs.
#ifdef CPSEL_VB_PROF
__device__ unsigned long long g_scprof[16];
#define SCT(i)                                                                  \
  if (threadIdx.x == 0) {                                                       \
    unsigned long long t_;                                                      \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
    atomicMin(&g_scprof[2 * (i)], t_ | 0ull);                                   \
    atomicMax(&g_scprof[2 * (i) + 1], t_);                                      \
  }
#else
#define SCT(i)
#endif
constexpr int kSampleCluster = 8;
struct ClusterSel {
  unsigned loc[3][2048];   // this CTA's histograms
  unsigned glob[3][2048];  // CTA 0: the cluster's histograms
  unsigned csum[3][32];
  unsigned long long prefix[3], mask[3], rank[3];
  unsigned long long wsum[32];
  int open_lo, open_hi;    // the cut's sample rank fell off the sample: no cut on that side
};
template <typename T, int KPT>
__global__ void __cluster_dims__(kSampleCluster, 1, 1) __launch_bounds__(1024)
    sample_cluster_kernel(const T* __restrict__ x, uint64_t m, const SegEntry* __restrict__ tab, int side, int Wtot,
                          uint64_t r, T* t0, const ChainState* chain, int which, uint64_t m_rank, int allow_open) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  using SK = SampleKey<T>;
  using K = typename SK::K;
  pdl_wait();
  pdl_trigger();  // the init pass may be scheduled (it waits for the cuts)
  SCT(0);
  extern __shared__ __align__(16) unsigned char csm[];
  ClusterSel& sh = *reinterpret_cast<ClusterSel*>(csm);
  unsigned long long* pre = reinterpret_cast<unsigned long long*>(csm + sizeof(ClusterSel));  // run-table prefix
  const unsigned crank = cl.block_rank();
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  bool go = true;
  if (chain) {
    go = chain->ok[which] != 0;
    m = chain->m[which];
    r = chain->r[which];
  }
  if (!go) return;  // uniform over the cluster (every CTA reads the same chain)
  constexpr uint64_t S = (uint64_t)kSampleCluster * 1024 * KPT;
  const uint64_t ms = m < S ? m : S;
  if (tab) {  // this CTA's copy of the run-table prefix
    const int per = (Wtot + 1023) / 1024;
    const int w0 = i * per, w1 = min(w0 + per, Wtot);
    unsigned long long c = 0;
    for (int w = w0; w < w1; ++w) {
      c += tab[w].cnt[side];
      pre[w] = c;
    }
    unsigned long long incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) sh.wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const unsigned long long v = sh.wsum[lane];
      unsigned long long inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
      }
      sh.wsum[lane] = inc - v;
    }
    __syncthreads();
    const unsigned long long base = sh.wsum[warp] + incl - c;
    for (int w = w0; w < w1; ++w) pre[w] += base;
    __syncthreads();
  }
  K keys[KPT];
  constexpr int VEK = 16 / sizeof(T);
  bool vec_done = false;
  if constexpr (KPT % VEK == 0 && KPT >= VEK) {
    if (!tab && m == ms && ms == S && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
      // the whole (pooled, contiguous) sample: thread (crank, i) takes KPT consecutive values with
      // 16-byte loads (which thread holds which sample does not matter to the histograms)
      using V = typename VecOf<T>::V;
      const V* xv = reinterpret_cast<const V*>(x + ((uint64_t)crank * 1024 + i) * KPT);
      V vv[KPT / VEK];
#pragma unroll
      for (int u = 0; u < KPT / VEK; ++u) vv[u] = __ldg(xv + u);
#pragma unroll
      for (int u = 0; u < KPT / VEK; ++u)
#pragma unroll
        for (int q = 0; q < VEK; ++q) keys[u * VEK + q] = SK::key(lane_of(vv[u], q));
      vec_done = true;
    }
  }
  if (!vec_done)
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const uint64_t smp = ((uint64_t)j * kSampleCluster + crank) * 1024 + i;
    keys[j] = ~K(0);
    if (smp < ms) {
      uint64_t g = (m == ms) ? smp : (smp * m) / ms + (m / ms) / 2;
      if (!tab) {
        keys[j] = SK::key(x[g]);
      } else {
        int lo = 0, hi = Wtot - 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (pre[mid] > g) hi = mid; else lo = mid + 1;
        }
        g -= lo ? pre[lo - 1] : 0ull;
        keys[j] = SK::key(x[tab[lo].off[side] + g]);
      }
    }
  }
  SCT(1);
  if (crank == 0 && i == 0) {
    // m_rank: the population the sample stands for (the pooled sample of G ranks, R28: m samples
    // of m_rank elements in all); 0 = m
    const double md = (double)ms;
    const double q = ((double)r - 0.5) / (double)(m_rank ? m_rank : m) * md;
    const double w = 3.5 * sqrt(fmax(q * (md - q) / md, 0.0)) + 2.0;
    const double qq[3] = {floor(q - w), ceil(q + w), floor(q)};
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      sh.rank[t] = qq[t] < 0 ? 0 : (qq[t] >= md ? ms - 1 : (uint64_t)qq[t]);
      sh.prefix[t] = 0;
      sh.mask[t] = 0;
    }
    // an extreme target rank (k near 1 or n): the sample's own extreme would be a cut the target
    // may well lie beyond — take the outermost float instead (the cut then keeps everything on
    // that side; exactness does not depend on where the cuts are)
    // (not when the init pass also sums (x - t_lo)^+ etc. for F, R25: those sums would overflow)
    sh.open_lo = allow_open && qq[0] < 0;
    sh.open_hi = allow_open && qq[1] >= md - 1;
  }
  unsigned* glob0 = cl.map_shared_rank(&sh.glob[0][0], 0);
  ClusterSel* sh0 = cl.map_shared_rank(&sh, 0);
  for (int rd = 0; rd < SK::ROUNDS; ++rd) {
    const int shift = SK::shift(rd), nb = 1 << SK::bits(rd);
    for (int b = i; b < 3 * 2048; b += 1024) {
      (&sh.loc[0][0])[b] = 0u;
      if (crank == 0) (&sh.glob[0][0])[b] = 0u;
    }
    cl.sync();  // CTA 0's prefixes and zeroed histograms visible to every CTA
    const K p0 = (K)sh0->prefix[0], p1 = (K)sh0->prefix[1], p2 = (K)sh0->prefix[2];
    const K m0 = (K)sh0->mask[0], m1 = (K)sh0->mask[1], m2 = (K)sh0->mask[2];
    // targets whose prefix class equals an earlier target's share its histogram (the usual case:
    // the three ranks lie in one class of the first digit)
    const bool same1 = p1 == p0 && m1 == m0, same2 = p2 == p0 && m2 == m0;
    const int ntg = rd == 0 ? 1 : 3;
    // one predicated shared reduction per key and target: keys of one digit that meet in a warp
    // instruction are aggregated by the hardware (no per-thread sort, no run detection — the sort
    // and run-aggregation this replaced cost ~200 instructions per sample on the cluster's 8 SMs)
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (t >= ntg) break;
      if ((t == 1 && same1) || (t == 2 && same2)) continue;  // copied from target 0 at the merge
      const K pt = t == 0 ? p0 : (t == 1 ? p1 : p2), mt = t == 0 ? m0 : (t == 1 ? m1 : m2);
      const unsigned base = (unsigned)__cvta_generic_to_shared(&sh.loc[t][0]);
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const K k = keys[j];
        const unsigned addr = base + 4u * ((unsigned)(k >> shift) & (unsigned)(nb - 1));
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.eq.u32 p, %0, 1;\n\t"
            "@p red.shared.add.u32 [%1], 1;\n\t}" ::"r"((k & mt) == pt ? 1u : 0u), "r"(addr)
            : "memory");
      }
    }
    // the cluster's histograms summed into CTA 0: every CTA sums its 1/8 slice of the bins over the
    // 8 CTAs' local histograms (distributed-shared-memory loads) and stores it in CTA 0 — no remote
    // atomics (~6K of them per CTA per round, serialised at CTA 0, cost ~20 us)
    cl.sync();  // every local histogram complete
    {
      const int nbins = ntg * 2048, slice = nbins / kSampleCluster;
      const unsigned* locq[kSampleCluster];
#pragma unroll
      for (int q = 0; q < kSampleCluster; ++q) locq[q] = cl.map_shared_rank(&sh.loc[0][0], q);
      for (int b = (int)crank * slice + i; b < ((int)crank + 1) * slice; b += 1024) {
        const int t = b >> 11;
        const int src = (t == 1 && same1) || (t == 2 && same2) ? (b & 2047) : b;  // shared histogram
        unsigned v = 0;
#pragma unroll
        for (int q = 0; q < kSampleCluster; ++q) v += locq[q][src];
        glob0[b] = v;
      }
    }
    cl.sync();  // the cluster's histograms complete in CTA 0
    if (crank == 0) {
      if (rd == 0)
        for (int b = i; b < 2048; b += 1024) sh.glob[1][b] = sh.glob[2][b] = sh.glob[0][b];
      __syncthreads();
      const int c0 = warp * 64;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        unsigned v = (c0 + lane < nb ? sh.glob[t][c0 + lane] : 0u) + (c0 + 32 + lane < nb ? sh.glob[t][c0 + 32 + lane] : 0u);
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (lane == 0) sh.csum[t][warp] = v;
      }
      __syncthreads();
      if (warp < 3) {
        const int t = warp;
        const unsigned long long rk = sh.rank[t];
        const unsigned cs = sh.csum[t][lane];
        __syncwarp();  // every lane has read rank before lane 0 rewrites it below
        unsigned incl = cs;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += y;
        }
        const unsigned hm = __ballot_sync(FULL, (unsigned long long)incl > rk);
        const int c = __ffs(hm) - 1;
        unsigned long long before = __shfl_sync(FULL, incl - cs, c);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int b = c * 64 + half * 32 + lane;
          const unsigned h = b < nb ? sh.glob[t][b] : 0u;
          unsigned in2 = h;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(FULL, in2, o);
            if (lane >= o) in2 += y;
          }
          const unsigned hb = __ballot_sync(FULL, before + in2 > rk);
          if (hb) {
            const int src = __ffs(hb) - 1;
            const unsigned ex = __shfl_sync(FULL, in2 - h, src);
            if (lane == 0) {
              sh.prefix[t] |= (unsigned long long)(c * 64 + half * 32 + src) << shift;
              sh.mask[t] |= (unsigned long long)(nb - 1) << shift;
              sh.rank[t] = rk - (before + ex);
            }
            break;
          }
          before += __shfl_sync(FULL, in2, 31);
        }
      }
    }
    __syncthreads();  // CTA 0: the digit search is done before the next round clears its histograms
    SCT(2 + rd);
  }
  cl.sync();
  SCT(7);
  if (crank == 0 && i < 3) {
    K kk = (K)sh.prefix[i];
    if (i == 1) kk |= (K)~(K)sh.mask[1];
    kk = kk < SK::KLO ? SK::KLO : (kk > SK::KHI ? SK::KHI : kk);
    if (i == 0 && sh.open_lo) kk = SK::KLO;
    if (i == 1 && sh.open_hi) kk = SK::KHI;
    t0[i] = SK::val(kk);
  }
#ifdef CPSEL_VB_PROF
  if (crank == 0 && i == 0) {
    printf("scprof start 0..%llu keys %llu..%llu r0 %llu..%llu r1 %llu..%llu end %llu..%llu\n", g_scprof[1] - g_scprof[0],
           g_scprof[2] - g_scprof[0], g_scprof[3] - g_scprof[0], g_scprof[4] - g_scprof[0], g_scprof[5] - g_scprof[0],
           g_scprof[6] - g_scprof[0], g_scprof[7] - g_scprof[0], g_scprof[14] - g_scprof[0], g_scprof[15] - g_scprof[0]);
    for (int q = 0; q < 16; q += 2) { g_scprof[q] = ~0ull; g_scprof[q + 1] = 0ull; }
  }
#endif
}

// §8f-3 for small arrays (BASELINE configs[0], n = 1e5): the WHOLE selection as one launch.  The
// array (m <= 8 x 1024 x KPT elements) is held in the registers of one 8-CTA cluster as
// order-preserving keys, sorted per thread, and x_(r) is found by an exact MSB radix select (all
// digit rounds: 3 for f32, 6 for f64) whose per-CTA run-aggregated histograms are merged into CTA 0
// over distributed shared memory; non-finite keys are counted on the way (R12).  CTA 0 publishes the
// value (canonical +0, R13) and the non-finite count into the mailbox: no init pass, no host round
// trip between rounds.
struct ExactSel {
  unsigned loc[2048];
  unsigned glob[2048];
  unsigned csum[32];
  unsigned long long prefix, mask, rank, bad;
};
template <typename T, int KPT>
__global__ void __cluster_dims__(kSampleCluster, 1, 1) __launch_bounds__(1024)
    exact_cluster_kernel(const T* __restrict__ x, uint64_t m, uint64_t r, double* vout, unsigned long long* bad_out,
                         unsigned long long* done, unsigned long long seq) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  using SK = SampleKey<T>;
  using K = typename SK::K;
  constexpr int ROUNDS = sizeof(T) == 4 ? 3 : 6;
  __shared__ ExactSel sh;
  const unsigned crank = cl.block_rank();
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  K keys[KPT];
  unsigned bad = 0;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const uint64_t g = ((uint64_t)j * kSampleCluster + crank) * 1024 + i;  // coalesced per warp
    keys[j] = ~K(0);                                                      // padding: sorts last
    if (g < m) {
      keys[j] = SK::key(x[g]);
      bad += (keys[j] < SK::KLO || keys[j] > SK::KHI) ? 1u : 0u;           // NaN, +-Inf
    }
  }
#pragma unroll
  for (int size = 2; size <= KPT; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int l = j ^ stride;
        if (l > j) {
          const K a = keys[j], b = keys[l];
          const bool up = (j & size) == 0;
          keys[j] = up ? (a < b ? a : b) : (a < b ? b : a);
          keys[l] = up ? (a < b ? b : a) : (a < b ? a : b);
        }
      }
    }
  }
  if (i == 0) {
    sh.prefix = 0;
    sh.mask = 0;
    sh.rank = r - 1;
    sh.bad = 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(FULL, bad, o);
  ExactSel* sh0 = cl.map_shared_rank(&sh, 0);
  cl.sync();  // CTA 0's state initialised
  if (lane == 0 && bad) atomicAdd(&sh0->bad, (unsigned long long)bad);
  for (int rd = 0; rd < ROUNDS; ++rd) {
    const int shift = SK::shift(rd), nb = 1 << SK::bits(rd);
    for (int b = i; b < 2048; b += 1024) {
      sh.loc[b] = 0u;
      if (crank == 0) sh.glob[b] = 0u;
    }
    cl.sync();  // CTA 0's prefix and zeroed histogram visible to every CTA
    const K pt = (K)sh0->prefix, mt = (K)sh0->mask;
    unsigned run = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {  // run-aggregated: the thread's keys are sorted
      const K k = keys[j];
      const bool in = (k & mt) == pt;
      const unsigned d = (unsigned)(k >> shift) & (unsigned)(nb - 1);
      run += in ? 1u : 0u;
      bool last = in;
      if (j + 1 < KPT) {
        const K kn = keys[j + 1 < KPT ? j + 1 : j];
        last = in && (((kn & mt) != pt) || (((unsigned)(kn >> shift) & (unsigned)(nb - 1)) != d));
      }
      if (last) {
        atomicAdd(&sh.loc[d], run);
        run = 0;
      }
    }
    __syncthreads();
    unsigned* glob0 = cl.map_shared_rank(&sh.glob[0], 0);
    for (int b = i; b < 2048; b += 1024) {
      const unsigned v = sh.loc[b];
      if (v) atomicAdd(glob0 + b, v);
    }
    cl.sync();  // the cluster's histogram complete in CTA 0
    if (crank == 0) {
      const int c0 = warp * 64;
      unsigned v = (c0 + lane < nb ? sh.glob[c0 + lane] : 0u) + (c0 + 32 + lane < nb ? sh.glob[c0 + 32 + lane] : 0u);
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
      if (lane == 0) sh.csum[warp] = v;
      __syncthreads();
      if (warp == 0) {
        const unsigned long long rk = sh.rank;
        const unsigned cs = sh.csum[lane];
        __syncwarp();  // every lane has read rank before lane 0 rewrites it below
        unsigned incl = cs;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += y;
        }
        const unsigned hm = __ballot_sync(FULL, (unsigned long long)incl > rk);
        const int c = __ffs(hm) - 1;
        unsigned long long before = __shfl_sync(FULL, incl - cs, c);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int b = c * 64 + half * 32 + lane;
          const unsigned h = b < nb ? sh.glob[b] : 0u;
          unsigned in2 = h;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(FULL, in2, o);
            if (lane >= o) in2 += y;
          }
          const unsigned hb = __ballot_sync(FULL, before + in2 > rk);
          if (hb) {
            const int src = __ffs(hb) - 1;
            const unsigned ex = __shfl_sync(FULL, in2 - h, src);
            if (lane == 0) {
              sh.prefix |= (unsigned long long)(c * 64 + half * 32 + src) << shift;
              sh.mask |= (unsigned long long)(nb - 1) << shift;
              sh.rank = rk - (before + ex);
            }
            break;
          }
          before += __shfl_sync(FULL, in2, 31);
        }
      }
    }
    __syncthreads();
  }
  cl.sync();
  if (crank == 0 && i == 0) {
    const double v = (double)SK::val((K)sh.prefix);
    *vout = v == 0.0 ? 0.0 : v;
    *bad_out = sh.bad;
    publish_done(done, seq);
  }
}

constexpr int kExactKPT32 = 16, kExactKPT64 = 8;
uint64_t exact_cluster_cap(int dtype) {
  return (uint64_t)kSampleCluster * 1024 * (dtype == kF32 ? kExactKPT32 : kExactKPT64);
}
cudaError_t launch_exact_cluster(int dtype, const void* x, uint64_t m, uint64_t r, double* vout,
                                 unsigned long long* bad_out, unsigned long long* done, unsigned long long seq,
                                 cudaStream_t st) {
  if (m == 0 || m > exact_cluster_cap(dtype) || r < 1 || r > m) return cudaErrorInvalidValue;
  if (dtype == kF32)
    exact_cluster_kernel<float, kExactKPT32><<<kSampleCluster, 1024, 0, st>>>(static_cast<const float*>(x), m, r, vout,
                                                                              bad_out, done, seq);
  else
    exact_cluster_kernel<double, kExactKPT64><<<kSampleCluster, 1024, 0, st>>>(static_cast<const double*>(x), m, r,
                                                                               vout, bad_out, done, seq);
  return cudaGetLastError();
}

template <typename T, int KPT>
cudaError_t sample_cluster_t(const void* x, uint64_t m, const SegEntry* tab, int side, int Wtot, uint64_t r, void* t0,
                             cudaStream_t st, const ChainState* chain, int which, uint64_t m_rank = 0,
                             int allow_open = 1) {
  const size_t smem = sizeof(ClusterSel) + (tab ? (size_t)Wtot * 8 : 0);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(sample_cluster_kernel<T, KPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(ClusterSel) + 8 * kGatherMaxWarps));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  sample_cluster_kernel<T, KPT><<<kSampleCluster, 1024, smem, st>>>(static_cast<const T*>(x), m, tab, side, Wtot, r,
                                                                   static_cast<T*>(t0), chain, which, m_rank,
                                                                   allow_open);
  return cudaGetLastError();
}

template <typename T, int KPT>
cudaError_t sample_select_t(const void* x, uint64_t m, const SegEntry* tab, int side, int Wtot, uint64_t r, void* t0,
                            void* keys, cudaStream_t st, const ChainState* chain, int which) {
  auto* kk = static_cast<typename SampleKey<T>::K*>(keys);
  sample_gather_kernel<T, KPT><<<KPT * 1024 / kGatherThreads, kGatherThreads, 0, st>>>(static_cast<const T*>(x), m, tab,
                                                                                       side, Wtot, kk, chain, which);
  sample_select_kernel<T, KPT><<<1, 1024, 0, st>>>(kk, m, r, static_cast<T*>(t0), chain, which);
  return cudaGetLastError();
}

cudaError_t launch_sample_select(int dtype, const void* x, uint64_t m, const SegEntry* tab, int side, int Wtot,
                                 uint64_t r, void* t0, void* keys, cudaStream_t st, bool small,
                                 const ChainState* chain, int which, bool allow_open) {
  if (tab && Wtot > kGatherMaxWarps) return cudaErrorInvalidValue;
  (void)keys;
  // one cluster launch: 8 CTAs x 1024 threads x KPT samples (131072 / 8192 for f32, 65536 / 8192 f64;
  // f32 at 131072: the init's copy ~1% of n — measured +1.1% whole-step vs 32768; f64 at 65536:
  // 2^28 median 0.555 -> 0.545 ms vs 16384)
  const int op = allow_open ? 1 : 0;
  if (dtype == kF32)
    return small ? sample_cluster_t<float, 1>(x, m, tab, side, Wtot, r, t0, st, chain, which, 0, op)
                 : sample_cluster_t<float, 16>(x, m, tab, side, Wtot, r, t0, st, chain, which, 0, op);
  return small ? sample_cluster_t<double, 1>(x, m, tab, side, Wtot, r, t0, st, chain, which, 0, op)
               : sample_cluster_t<double, 8>(x, m, tab, side, Wtot, r, t0, st, chain, which, 0, op);
}



// ---------------------------------------------------------------------------- sharded helpers (R28)
// Inclusive prefix of the run lengths cnt[side] of tab[0..Wtot) into pre[] (shared), by the whole
// CTA of kGatherThreads threads (per-thread chunks, warp and block scans).
__device__ __forceinline__ void scan_runs(const SegEntry* __restrict__ tab, int side, int Wtot, unsigned long long* pre,
                                          unsigned long long* wsum) {
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  constexpr int NW = kGatherThreads / 32;
  const int per = (Wtot + kGatherThreads - 1) / kGatherThreads;
  const int w0 = i * per, w1 = min(w0 + per, Wtot);
  unsigned long long c = 0;
  for (int w = w0; w < w1; ++w) {
    c += tab[w].cnt[side];
    pre[w] = c;
  }
  unsigned long long incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long v = lane < NW ? wsum[lane] : 0ull, inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane < NW) wsum[lane] = inc - v;
  }
  __syncthreads();
  const unsigned long long base = wsum[warp] + incl - c;
  for (int w = w0; w < w1; ++w) pre[w] += base;
  __syncthreads();
}

// This rank's share of the pooled sample (R28): ms evenly strided VALUES of its m-element current
// array (contiguous x, or the runs `side` of tab[0..Wtot) based at x) into out[0..ms), ms <= m.
// Sample s is element floor(s*m/ms) + (m/ms)/2, as in the one-GPU gather.
template <typename T>
__global__ void __launch_bounds__(kGatherThreads) pool_gather_kernel(const T* __restrict__ x, uint64_t m,
                                                                     const SegEntry* __restrict__ tab, int side,
                                                                     int Wtot, uint64_t ms, T* __restrict__ out) {
  __shared__ unsigned long long pre[kGatherMaxWarps];
  __shared__ unsigned long long wsum[32];
  if (tab) scan_runs(tab, side, Wtot, pre, wsum);
  const uint64_t smp = (uint64_t)blockIdx.x * kGatherThreads + threadIdx.x;
  if (smp >= ms) return;
  uint64_t g = (m == ms) ? smp : (smp * m) / ms + (m / ms) / 2;
  if (!tab) {
    out[smp] = x[g];
    return;
  }
  int lo = 0, hi = Wtot - 1;  // first run whose inclusive prefix exceeds g
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] > g) hi = mid; else lo = mid + 1;
  }
  g -= lo ? pre[lo - 1] : 0ull;
  out[smp] = x[tab[lo].off[side] + g];
}

// The runs `side` of the segmented array (base, tab[0..Wtot)) packed contiguously into out, in run
// order (the sharded exact finish all-gathers one contiguous block per rank, a6).
template <typename T>
__global__ void __launch_bounds__(kGatherThreads) seg_pack_kernel(const T* __restrict__ base,
                                                                  const SegEntry* __restrict__ tab, int side, int Wtot,
                                                                  T* __restrict__ out) {
  __shared__ unsigned long long pre[kGatherMaxWarps];
  __shared__ unsigned long long wsum[32];
  scan_runs(tab, side, Wtot, pre, wsum);
  constexpr int NW = kGatherThreads / 32;
  const int lane = threadIdx.x & 31;
  for (int w = blockIdx.x * NW + (threadIdx.x >> 5); w < Wtot; w += gridDim.x * NW) {
    const unsigned long long c = tab[w].cnt[side], o = tab[w].off[side], dst = pre[w] - c;
    for (unsigned long long j = lane; j < c; j += 32) out[dst + j] = base[o + j];
  }
}

cudaError_t launch_pool_gather(int dtype, const void* x, uint64_t m, const SegEntry* tab, int side, int Wtot,
                               uint64_t ms, void* out, cudaStream_t st) {
  if (tab && Wtot > kGatherMaxWarps) return cudaErrorInvalidValue;
  if (ms == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((ms + kGatherThreads - 1) / kGatherThreads);
  if (dtype == kF32)
    pool_gather_kernel<float><<<grid, kGatherThreads, 0, st>>>(static_cast<const float*>(x), m, tab, side, Wtot, ms,
                                                               static_cast<float*>(out));
  else
    pool_gather_kernel<double><<<grid, kGatherThreads, 0, st>>>(static_cast<const double*>(x), m, tab, side, Wtot, ms,
                                                                static_cast<double*>(out));
  return cudaGetLastError();
}

// R40: the one-GPU sample cuts as ONE cooperative grid kernel (replacing pool_gather + the 8-CTA
// cluster select of the same sample): S / 1024 CTAs of 1024 threads, one strided sample per thread
// (the gather's positions), so each CTA histograms ~1024 keys per round (not 16384 as in the
// cluster, where the shared-memory atomics of the first round dominated); the per-CTA histograms
// are added into a global one (scratch, zero on entry and left zero), one grid barrier per digit
// round, and every CTA then picks the next digits of the three sample ranks from the global counts
// itself (the same deterministic scan everywhere: no broadcast).  Same ranks, digits and cut
// values as sample_cluster_kernel (R23, R29).
constexpr int kSgMaxRounds = 4;
constexpr size_t kSgHalf = (size_t)kSgMaxRounds * 3 * 2048 + 32;  // counts + [the barrier counter]
constexpr size_t kSampleGridWords = 2 * kSgHalf + 32;                 // two halves + [the phase]
template <typename T, int KPT>
__global__ void __launch_bounds__(1024, 1)
    sample_grid_kernel(const T* __restrict__ x, uint64_t m, uint64_t ms, uint64_t m_rank, uint64_t r, T* t0,
                       unsigned* __restrict__ scratch, int allow_open) {
  using SK = SampleKey<T>;
  using K = typename SK::K;
  __shared__ unsigned loc[3][2048];
  __shared__ unsigned wsum3[3][32];
  __shared__ unsigned s_d3[3];
  __shared__ unsigned long long s_b3[3];
  __shared__ unsigned long long prefix[3], mask[3], rank[3];
  __shared__ int open_lo, open_hi;
  // two halves used alternately: this launch counts in half ph and clears the other (the previous
  // launch's, complete in stream order) for the next, so nothing waits for a last CTA to clean up
  const unsigned ph = __ldcg(scratch + 2 * kSgHalf) & 1u;
  unsigned* const H = scratch + ph * kSgHalf;
  unsigned* const bar = H + (size_t)kSgMaxRounds * 3 * 2048;
  pdl_trigger();  // the init pass may be scheduled (it waits for the cuts)
  SCT(0);
  const int i = threadIdx.x;
  {
    unsigned* const O = scratch + (ph ^ 1u) * kSgHalf;
    for (size_t b = (size_t)blockIdx.x * 1024 + i; b < kSgHalf; b += (size_t)gridDim.x * 1024) O[b] = 0u;
  }
  bool have[KPT];
  K key[KPT];
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const uint64_t smp = ((uint64_t)j * gridDim.x + blockIdx.x) * 1024 + i;
    have[j] = smp < ms;
    key[j] = 0;
    if (have[j]) {
      const uint64_t g = (m == ms) ? smp : (smp * m) / ms + (m / ms) / 2;
      key[j] = SK::key(x[g]);
    }
  }
  if (i == 0) {
    const double md = (double)ms;
    const double q = ((double)r - 0.5) / (double)(m_rank ? m_rank : m) * md;
    const double w = 3.5 * sqrt(fmax(q * (md - q) / md, 0.0)) + 2.0;
    const double qq[3] = {floor(q - w), ceil(q + w), floor(q)};
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      rank[t] = qq[t] < 0 ? 0 : (qq[t] >= md ? ms - 1 : (uint64_t)qq[t]);
      prefix[t] = 0;
      mask[t] = 0;
    }
    open_lo = allow_open && qq[0] < 0;
    open_hi = allow_open && qq[1] >= md - 1;
  }
  for (int b = i; b < 3 * 2048; b += 1024) (&loc[0][0])[b] = 0u;
  __syncthreads();
  SCT(1);
  for (int rd = 0; rd < SK::ROUNDS; ++rd) {
    const int shift = SK::shift(rd), nb = 1 << SK::bits(rd);
    // the distinct classes of the three targets: src[t] = the first target with t's class
    int src[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      src[t] = t;
      for (int u = t - 1; u >= 0; --u)
        if (prefix[u] == prefix[t] && mask[u] == mask[t]) src[t] = u;
    }
    unsigned* G = H + (size_t)rd * 3 * 2048;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (src[t] != t) continue;
#pragma unroll
      for (int j = 0; j < KPT; ++j)
        if (have[j] && (key[j] & (K)mask[t]) == (K)prefix[t])
          atomicAdd(&loc[t][(unsigned)(key[j] >> shift) & (unsigned)(nb - 1)], 1u);
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (src[t] != t) continue;
      for (int b = i; b < nb; b += 1024) {
        const unsigned v = loc[t][b];
        if (v) {
          atomicAdd(&G[t * 2048 + b], v);
          loc[t][b] = 0u;
        }
      }
    }
    SCT(2 + 2 * (rd & 1));
    // grid barrier rd + 1 on a counter that only grows within the launch (one release-add per CTA,
    // acquire polls until every CTA has arrived; the last CTA out resets it)
    __syncthreads();
    if (i == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
      const unsigned target = (unsigned)(rd + 1) * gridDim.x;
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      } while (v < target);
    }
    __syncthreads();
    SCT(3 + 2 * (rd & 1));
    // the digit of every target: each thread loads two bins of every distinct class at once (one
    // L2 round trip, not three), one block scan per class, then each target's range test
    const int lane = i & 31, w = i >> 5, bi = 2 * i;
    unsigned h0[3], h1[3], incl[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      h0[t] = h1[t] = 0u;
      if (src[t] == t && bi < nb) {
        h0[t] = __ldcg(&G[t * 2048 + bi]);
        h1[t] = __ldcg(&G[t * 2048 + bi + 1]);
      }
    }
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      incl[t] = h0[t] + h1[t];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(FULL, incl[t], o);
        if (lane >= o) incl[t] += y;
      }
      if (lane == 31) wsum3[t][w] = incl[t];
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int c = src[t];  // the class whose counts target t reads (c <= t)
      unsigned long long ws = wsum3[c][lane], wi = ws;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL, wi, o);
        if (lane >= o) wi += y;
      }
      const unsigned a0 = c == 0 ? h0[0] : (c == 1 ? h0[1] : h0[2]);
      const unsigned a1 = c == 0 ? h1[0] : (c == 1 ? h1[1] : h1[2]);
      const unsigned ic = c == 0 ? incl[0] : (c == 1 ? incl[1] : incl[2]);
      const unsigned long long before = __shfl_sync(FULL, wi - ws, w) + ic - (a0 + a1);
      const unsigned long long rk = rank[t] + 1;  // 1-based
      if (before < rk && rk <= before + a0) {
        s_d3[t] = (unsigned)bi;
        s_b3[t] = before;
      } else if (before + a0 < rk && rk <= before + a0 + a1) {
        s_d3[t] = (unsigned)bi + 1u;
        s_b3[t] = before + a0;
      }
    }
    __syncthreads();
    if (i < 3) {
      prefix[i] |= (unsigned long long)s_d3[i] << shift;
      mask[i] |= (unsigned long long)(nb - 1) << shift;
      rank[i] -= s_b3[i];
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && i < 3) {
    K kk = (K)prefix[i];
    if (i == 1) kk |= (K)~(K)mask[1];
    kk = kk < SK::KLO ? SK::KLO : (kk > SK::KHI ? SK::KHI : kk);
    if (i == 0 && open_lo) kk = SK::KLO;
    if (i == 1 && open_hi) kk = SK::KHI;
    t0[i] = SK::val(kk);
  }
#ifdef CPSEL_VB_PROF
  SCT(6);
  if (blockIdx.x == 0 && i == 0) {
    printf("sgprof start 0..%llu keys %llu..%llu r0 %llu..%llu bar0 %llu..%llu r1 %llu..%llu bar1 %llu..%llu end0 %llu\n",
           g_scprof[1] - g_scprof[0], g_scprof[2] - g_scprof[0], g_scprof[3] - g_scprof[0], g_scprof[4] - g_scprof[0],
           g_scprof[5] - g_scprof[0], g_scprof[6] - g_scprof[0], g_scprof[7] - g_scprof[0], g_scprof[8] - g_scprof[0],
           g_scprof[9] - g_scprof[0], g_scprof[10] - g_scprof[0], g_scprof[11] - g_scprof[0], g_scprof[13] - g_scprof[0]);
    for (int q = 0; q < 16; q += 2) { g_scprof[q] = ~0ull; g_scprof[q + 1] = 0ull; }
  }
#endif
  // every CTA read the phase before the first barrier, and CTA 0 is past the last one
  if (blockIdx.x == 0 && i == 0) scratch[2 * kSgHalf] = ph ^ 1u;
}
size_t sample_grid_words() { return kSampleGridWords; }
cudaError_t launch_sample_grid(int dtype, const void* x, uint64_t m, uint64_t ms, uint64_t m_rank, uint64_t r,
                               void* t0, unsigned* scratch, cudaStream_t st, bool allow_open) {
  // one key per thread up to 128 CTAs, else 4, 8 or 16 (<= 128 x 16384 samples)
  const int kpt = ms <= 128 * 1024 ? 1 : ms <= 4 * 128 * 1024 ? 4 : ms <= 8 * 128 * 1024 ? 8 : 16;
  if (ms == 0 || ms > m || ms % (1024 * kpt) || ms / (1024 * kpt) > 128) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ms / (1024 * kpt)));
  cfg.blockDim = dim3(1024);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int op = allow_open ? 1 : 0;
  if (dtype == kF32) {
    void (*f)(const float*, uint64_t, uint64_t, uint64_t, uint64_t, float*, unsigned*, int) =
        kpt == 16 ? sample_grid_kernel<float, 16>
                  : kpt == 8 ? sample_grid_kernel<float, 8>
                             : kpt == 4 ? sample_grid_kernel<float, 4> : sample_grid_kernel<float, 1>;
    return cudaLaunchKernelEx(&cfg, f, static_cast<const float*>(x), m, ms, m_rank, r, static_cast<float*>(t0), scratch,
                              op);
  }
  void (*f)(const double*, uint64_t, uint64_t, uint64_t, uint64_t, double*, unsigned*, int) =
      kpt == 16 ? sample_grid_kernel<double, 16>
                : kpt == 8 ? sample_grid_kernel<double, 8>
                           : kpt == 4 ? sample_grid_kernel<double, 4> : sample_grid_kernel<double, 1>;
  return cudaLaunchKernelEx(&cfg, f, static_cast<const double*>(x), m, ms, m_rank, r, static_cast<double*>(t0), scratch,
                            op);
}

uint64_t pool_sample_size(int dtype, bool small) {
  return (uint64_t)kSampleCluster * 1024 * (small ? 1 : (dtype == kF32 ? 16 : 8));
}

cudaError_t launch_pool_pick(int dtype, const void* pooled, uint64_t ms, uint64_t m_rank, uint64_t r, void* t0,
                             cudaStream_t st, bool small, bool allow_open) {
  if (ms > pool_sample_size(dtype, small)) return cudaErrorInvalidValue;
  const int op = allow_open ? 1 : 0;
  if (dtype == kF32)
    return small ? sample_cluster_t<float, 1>(pooled, ms, nullptr, 0, 0, r, t0, st, nullptr, 0, m_rank, op)
                 : sample_cluster_t<float, 16>(pooled, ms, nullptr, 0, 0, r, t0, st, nullptr, 0, m_rank, op);
  return small ? sample_cluster_t<double, 1>(pooled, ms, nullptr, 0, 0, r, t0, st, nullptr, 0, m_rank, op)
               : sample_cluster_t<double, 8>(pooled, ms, nullptr, 0, 0, r, t0, st, nullptr, 0, m_rank, op);
}

cudaError_t launch_seg_pack(int dtype, const void* base, const SegEntry* tab, int side, int Wtot, void* out,
                            cudaStream_t st) {
  if (Wtot > kGatherMaxWarps) return cudaErrorInvalidValue;
  const int grid = 32;
  if (dtype == kF32)
    seg_pack_kernel<float><<<grid, kGatherThreads, 0, st>>>(static_cast<const float*>(base), tab, side, Wtot,
                                                            static_cast<float*>(out));
  else
    seg_pack_kernel<double><<<grid, kGatherThreads, 0, st>>>(static_cast<const double*>(base), tab, side, Wtot,
                                                             static_cast<double*>(out));
  return cudaGetLastError();
}

cudaError_t launch_sample_seg(int dtype, const void* base, const SegEntry* tab, int side, int Wtot, uint64_t m,
                              uint64_t r, void* t0, cudaStream_t st, uint32_t smax, unsigned long long* keys_out) {
  if (dtype == kF32)
    sample_seg_kernel<float><<<1, 1024, 0, st>>>(static_cast<const float*>(base), tab, side, Wtot, m, r,
                                                 static_cast<float*>(t0), smax, keys_out);
  else
    sample_seg_kernel<double><<<1, 1024, 0, st>>>(static_cast<const double*>(base), tab, side, Wtot, m, r,
                                                  static_cast<double*>(t0), smax, keys_out);
  return cudaGetLastError();
}

cudaError_t launch_cut_pass(int dtype, const SegArgs& a, const LaunchShape& s, cudaStream_t st) {
  // the segmented grid: its warp regions / run tables are what later passes read
  const int g = s.grid_seg[dtype];
  if (dtype == kF32) cut_pass_kernel<float><<<g, kBlock, 0, st>>>(a);
  else cut_pass_kernel<double><<<g, kBlock, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_vbin_finish(int dtype, const void* z, const SegEntry* tab, const void* cuts, unsigned* hist,
                               const LaunchShape& s, cudaStream_t st, const ChainState* chain, double* vout,
                               unsigned long long* fallback, unsigned long long* done, unsigned long long seq) {
  VbArgs a{};
  a.z = z; a.tab = tab; a.cuts = cuts; a.chain = chain; a.vout = vout; a.fallback = fallback; a.done = done;
  a.seq = seq;
  a.Wtot = s.grid_seg[dtype] * kWarps;
  a.hist0 = hist + 2048;
  a.st = reinterpret_cast<unsigned long long*>(hist + kVbState);
  a.zb = hist + kVbBuf;
  const size_t smem = (size_t)kVbCap * 8;  // the last CTA's keys
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.Wtot + 31) / 32);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (dtype == kF32) {
    static const cudaError_t a0 = cudaFuncSetAttribute(vbin_finish_kernel<float>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (a0 != cudaSuccess) return a0;
    e = cudaLaunchKernelEx(&cfg, vbin_finish_kernel<float>, a);
  } else {
    static const cudaError_t a1 = cudaFuncSetAttribute(vbin_finish_kernel<double>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (a1 != cudaSuccess) return a1;
    e = cudaLaunchKernelEx(&cfg, vbin_finish_kernel<double>, a);
  }
  return e;
}

cudaError_t launch_radix_select(int dtype, const void* z, uint64_t m, uint64_t r, RadixState* state,
                                unsigned* hist, const LaunchShape& s, cudaStream_t st, double* vout,
                                unsigned long long* done, unsigned long long seq, const SegEntry* tab, int side,
                                unsigned* ticket, const ChainState* chain, int first_round, unsigned* hist0,
                                uint64_t m_hint) {
  // digit plan, MSB first: f32 11+11+10, f64 11+11+11+11+10+10 (first_round > 0: the earlier rounds
  // were taken by the init pass, RadixState holds their prefix and rank)
  static const int plan32[] = {21, 11, 10, 11, 0, 10};
  static const int plan64[] = {53, 11, 42, 11, 31, 11, 20, 11, 10, 10, 0, 10};
  const int rounds = dtype == kF32 ? 3 : 6;
  const int* plan = dtype == kF32 ? plan32 : plan64;
  {  // all rounds in one cooperative launch, if the grid fits co-resident
    static const bool coop_on = !(getenv("CPSEL_RADIX_COOP") && getenv("CPSEL_RADIX_COOP")[0] == '0');
    // 1024-thread CTAs, one per SM (CPSEL_RADIX_NT=256: four 256-thread CTAs per SM)
    // (dense input: stream_array's lane arithmetic assumes kBlock threads, so always 256)
    static const int nt_seg = (getenv("CPSEL_RADIX_NT") && atoi(getenv("CPSEL_RADIX_NT")) == 256) ? 256 : 1024;
    const int nt = tab ? nt_seg : kBlock;
    const int per_cta = nt / kBlock;  // 256-thread CTAs' worth of warps per CTA
    const int seg_grid = (s.grid_seg[dtype] + per_cta - 1) / per_cta;
    const int grid = tab ? seg_grid : clamp_grid(s.grid_hist[dtype] / per_cta, m, kRadixPerCta * per_cta);
    if (coop_on && grid <= s.coop_max[dtype][tab ? 1 : 0][nt == 1024 ? 1 : 0]) {
      CoopArgs c{};
      RadixArgs& a = c.a;
      a.z = z; a.m = m; a.tab = tab; a.side = side; a.st = state; a.hist = hist; a.ticket = ticket;
      a.r = r; a.vout = vout; a.done = done; a.seq = seq; a.chain = chain;
      a.Wtot = s.grid_seg[dtype] * kWarps;
      a.hist0 = first_round == 1 ? hist0 : nullptr;
      c.plan.n = rounds;
      for (int i = 0; i < rounds; ++i) {
        c.plan.shift[i] = plan[2 * i];
        c.plan.bits[i] = plan[2 * i + 1];
      }
      c.first_round = first_round;
      c.g3 = hist + 4096;
      c.bar = hist + 4096 + 3 * 2048;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(nt);
      cfg.stream = st;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      cudaError_t e;
#define COOPL(T, SEGV) (nt == 1024 ? cudaLaunchKernelEx(&cfg, radix_coop_kernel<T, SEGV, 1024>, c) \
                                   : cudaLaunchKernelEx(&cfg, radix_coop_kernel<T, SEGV, 256>, c))
      if (dtype == kF32)
        e = tab ? COOPL(float, true) : COOPL(float, false);
      else
        e = tab ? COOPL(double, true) : COOPL(double, false);
#undef COOPL
      return e;
    }
  }
  RadixArgs a{};
  a.z = z; a.m = m; a.tab = tab; a.side = side; a.st = state; a.hist = hist; a.ticket = ticket;
  a.r = r; a.vout = vout; a.done = done; a.seq = seq; a.chain = chain;
  a.Wtot = s.grid_seg[dtype] * kWarps;
  // dense input: one CTA per kRadixPerCta elements (each CTA merges up to 2048 bins into the global
  // histogram and the last one scans them, so a small copy is not spread over the whole grid)
  (void)m_hint;
  for (int i = first_round; i < rounds; ++i) {
    a.shift = plan[2 * i]; a.bits = plan[2 * i + 1];
    a.first = i == 0; a.last = i == rounds - 1;
    a.hist0 = (i == 1 && first_round == 1) ? hist0 : nullptr;
    const int grid = tab ? s.grid_seg[dtype]  // a warp per run: the runs are short, latency-bound
                         : clamp_grid(s.grid_hist[dtype], m, kRadixPerCta);
    if (dtype == kF32) {
      if (tab) pdl_launch(radix_round_kernel<float, true>, dim3(grid), dim3(kBlock), 0, st, a);
      else pdl_launch(radix_round_kernel<float, false>, dim3(grid), dim3(kBlock), 0, st, a);
    } else {
      if (tab) pdl_launch(radix_round_kernel<double, true>, dim3(grid), dim3(kBlock), 0, st, a);
      else pdl_launch(radix_round_kernel<double, false>, dim3(grid), dim3(kBlock), 0, st, a);
    }
  }
  return cudaGetLastError();
}

}  // namespace cpsel

namespace cpsel {
cudaError_t launch_batched_select(const BatchArgs& a, int grid, cudaStream_t st) {
  constexpr size_t sm = compact_smem_bytes<float>();
  cudaError_t e = cudaFuncSetAttribute(batched_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  batched_select_kernel<<<grid, kBlock, sm, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_lms_cuts(const float* Ss, uint32_t ms, uint64_t n, uint32_t C, uint64_t k, float* cuts,
                            cudaStream_t st) {
  if (ms > (uint32_t)(kCutThreads * kCutMaxPer)) return cudaErrorInvalidValue;
  int dev = 0, sms = 148, b = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (ms % 256) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(lms_cuts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCutSmem);
  if (e != cudaSuccess) return e;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, lms_cuts_kernel, kCutThreads, kCutSmem);
  uint32_t grid = (uint32_t)(sms * (b > 0 ? b : 1));
  if (grid > C) grid = C;
  lms_cuts_kernel<<<grid, kCutThreads, kCutSmem, st>>>(Ss, ms, n, C, k, cuts);
  return cudaGetLastError();
}

int batched_blocks_per_sm() {
  constexpr size_t sm = compact_smem_bytes<float>();
  cudaFuncSetAttribute(batched_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int b = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, batched_select_kernel, kBlock, sm);
  return b > 0 ? b : 1;
}
}  // namespace cpsel
