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

#include "cpsel_kernels.h"

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
__device__ __forceinline__ float lane_of(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
__device__ __forceinline__ double lane_of(const double2& v, int j) { return j == 0 ? v.x : v.y; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T> __device__ __forceinline__ T tmax(T a, T b);
template <> __device__ __forceinline__ float tmax(float a, float b) { return fmaxf(a, b); }
template <> __device__ __forceinline__ double tmax(double a, double b) { return fmax(a, b); }
template <typename T> __device__ __forceinline__ T tmin(T a, T b);
template <> __device__ __forceinline__ float tmin(float a, float b) { return fminf(a, b); }
template <> __device__ __forceinline__ double tmin(double a, double b) { return fmin(a, b); }

template <typename T> __device__ __forceinline__ T tinf();
template <> __device__ __forceinline__ float tinf() { return __int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double tinf() { return __longlong_as_double(0x7ff0000000000000ll); }

// ------------------------------------------------------------------------------------------
// Generic grid-stride stream over x[0..n) with 16-byte vector loads.  F provides
//   template<bool MASKED> void vec(const V&, bool ok)   (all lanes call; ok=false -> no-op)
//   void group_begin(), group_end()                       (around each UNROLL-vector group)
//   void scalar(T, bool ok)                               (head/tail elements)
// Any element alignment is accepted: the unaligned head and the tail (< VE elements each)
// are processed as scalars by warp 0 of the last CTA.
template <typename T, int UNROLL, typename F>
__device__ __forceinline__ void stream_array(const T* __restrict__ x, uint64_t n, F& f) {
  using V = typename VecOf<T>::V;
  constexpr int VE = VecOf<T>::N;
  const uint64_t mis = (reinterpret_cast<uintptr_t>(x) / sizeof(T)) & (VE - 1);
  uint64_t head = mis ? (VE - mis) : 0;
  if (head > n) head = n;
  const V* __restrict__ xv = reinterpret_cast<const V*>(x + head);
  const uint64_t nvec = (n - head) / VE;
  constexpr uint64_t TILE = (uint64_t)kBlock * UNROLL;
  const uint64_t stride = (uint64_t)gridDim.x * TILE;
  uint64_t base = (uint64_t)blockIdx.x * TILE;
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
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < 32) {
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

__device__ __forceinline__ void combine(InitPartial& a, const InitPartial& b) {
  if (b.vmin < a.vmin) { a.vmin = b.vmin; a.cnt_min = b.cnt_min; }
  else if (b.vmin == a.vmin) a.cnt_min += b.cnt_min;
  if (b.vmax > a.vmax) { a.vmax = b.vmax; a.cnt_max = b.cnt_max; }
  else if (b.vmax == a.vmax) a.cnt_max += b.cnt_max;
  a.S += b.S;
  a.nonfinite += b.nonfinite;
}

__device__ InitPartial block_reduce(InitPartial p) {
  __shared__ InitPartial sh[kBlock];
  sh[threadIdx.x] = p;
  __syncthreads();
  // fixed-shape tree over the block
  for (int s = kBlock / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) combine(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  InitPartial r = sh[0];
  __syncthreads();
  return r;
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
  static_assert(sizeof(P) % 8 == 0, "partial must be 8-byte words");
  for (unsigned i = threadIdx.x; i < gridDim.x; i += kBlock) {
    P q;
    // ld.global.cg: read at L2 (the partials were written by other CTAs)
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(partials + i);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&q);
#pragma unroll
    for (int w = 0; w < (int)(sizeof(P) / 8); ++w) dst[w] = __ldcg(src + w);
    combine(acc, q);
  }
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
template <typename T, bool CHECKED> struct InitFn {
  T mn, mx, x0;
  unsigned cmn, cmx, nonfin;
  double S;
  T g[4];
  __device__ InitFn(T x0_) : mn(tinf<T>()), mx(-tinf<T>()), x0(x0_), cmn(0), cmx(0), nonfin(0), S(0) {}
  __device__ __forceinline__ void slow(T v) {
    if (v < mn) { mn = v; cmn = 1; } else if (v == mn) ++cmn;
    if (v > mx) { mx = v; cmx = 1; } else if (v == mx) ++cmx;
  }
  __device__ __forceinline__ void group_begin() { g[0] = g[1] = g[2] = g[3] = T(0); }
  __device__ __forceinline__ void group_end() { S += (double)((g[0] + g[1]) + (g[2] + g[3])); }
  __device__ __forceinline__ void vec_elems(const float4& v, int u) {
    const float lo = fminf(fminf(v.x, v.y), fminf(v.z, v.w));
    const float hi = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
    if (lo <= mn || hi >= mx) { slow(v.x); slow(v.y); slow(v.z); slow(v.w); }
    g[u & 3] += ((v.x - x0) + (v.y - x0)) + ((v.z - x0) + (v.w - x0));
    if (CHECKED)
      nonfin += !(fabsf(v.x) <= FLT_MAX) + !(fabsf(v.y) <= FLT_MAX) + !(fabsf(v.z) <= FLT_MAX) + !(fabsf(v.w) <= FLT_MAX);
  }
  __device__ __forceinline__ void vec_elems(const double2& v, int u) {
    const double lo = fmin(v.x, v.y), hi = fmax(v.x, v.y);
    if (lo <= mn || hi >= mx) { slow(v.x); slow(v.y); }
    g[u & 3] += (v.x - x0) + (v.y - x0);
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
    if (CHECKED) nonfin += !(fabs(v) <= (sizeof(T) == 4 ? (T)FLT_MAX : (T)DBL_MAX));
    group_end();
  }
};

template <typename T, int UNROLL, bool CHECKED>
__global__ void __launch_bounds__(kBlock) init_kernel(InitArgs a) {
  const T* x = static_cast<const T*>(a.x);
  InitFn<T, CHECKED> f(x[0]);
  stream_array<T, UNROLL>(x, a.n, f);
  InitPartial p;
  p.vmin = (double)f.mn; p.vmax = (double)f.mx; p.S = f.S; p.pad = 0;
  p.cnt_min = f.cmn; p.cnt_max = f.cmx; p.nonfinite = f.nonfin; p.pad2 = 0;
  p = block_reduce(p);
  InitPartial id;
  id.vmin = tinf<double>(); id.vmax = -tinf<double>(); id.S = 0; id.pad = 0;
  id.cnt_min = id.cnt_max = id.nonfinite = id.pad2 = 0;
  InitPartial tot;
  if (grid_finish(p, static_cast<InitPartial*>(a.partials), a.ticket, &tot, id) && threadIdx.x == 0) {
    DevInit r;
    r.vmin = tot.vmin; r.vmax = tot.vmax; r.S = tot.S; r.x0 = (double)x[0];
    r.cnt_min = tot.cnt_min; r.cnt_max = tot.cnt_max; r.nonfinite = tot.nonfinite; r.pad = 0;
    *a.out = r;
  }
}

// ------------------------------------------------------------------------------------------
// Step a2 (+ a4): one cutting-plane pass.
template <typename T> constexpr int stage_cap() { return sizeof(T) == 4 ? 1024 : 512; }

template <typename T, int MODE, int UNROLL> struct PassFn {
  static constexpr int VE = VecOf<T>::N;
  static constexpr int CAPW = stage_cap<T>();
  static constexpr int GROUP_MAX = 32 * UNROLL * VE;  // elements a warp can add per group
  T t, yL, yR;
  unsigned c_lt, c_eq, c_lo, c_hi;
  double L_lo, L_hi, P, N;
  T pred, succ;
  T glo[UNROLL], ghi[UNROLL], gP[UNROLL], gN[UNROLL];
  // compaction (MODE == kCompact)
  T* s_lo; T* s_hi;
  int n_lo, n_hi;
  T* z;
  uint64_t z_cap;
  unsigned long long* cursors;

  __device__ __forceinline__ void elem(T v, bool ok, int u) {
    const bool lt = v < t;
    const bool gt = v > t;
    const bool lo = lt && (v > yL);
    const bool hi = gt && (v < yR);
    const T d = t - v;
    if (MODE == kHot) {
      // the hot form: no pred/succ (the driver uses them only on small compacted brackets).
      // Written as predicated PTX so every accumulation is ONE predicated instruction
      // (10 issue slots per element: 5 compares, 1 sub, 4 predicated adds).
      if (ok) hot_elem(v, glo[u], ghi[u]);
    } else if (MODE == kCompact) {
      // ok is always true here for unmasked calls; masked calls pass ok explicitly
      if (ok) {
        if (lt) ++c_lt;
        if (v == t) ++c_eq;
        if (lo) { glo[u] += d; pred = tmax(pred, v); }
        if (hi) { ghi[u] -= d; succ = tmin(succ, v); }
      }
    } else {
      if (ok) {
        c_lt += lt;
        c_eq += (v == t);
        c_lo += lo;
        c_hi += hi;
        if (lo) { glo[u] += d; pred = tmax(pred, v); }
        if (hi) { ghi[u] -= d; succ = tmin(succ, v); }
        if (lt) gN[u] += d;
        if (gt) gP[u] -= d;
      }
    }
    if (MODE == kCompact) {
      push(ok && lo, v, s_lo, n_lo);
      push(ok && hi, v, s_hi, n_hi);
    }
  }
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
  __device__ __forceinline__ void push(bool f, T v, T* s, int& cnt) {
    const unsigned m = __ballot_sync(FULL, f);
    if (f) s[cnt + __popc(m & lanemask_lt())] = v;
    cnt += __popc(m);
  }
  __device__ __forceinline__ void flush(T* s, int& cnt, int side) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0 && cnt) base = atomicAdd(&cursors[side], (unsigned long long)cnt);
    base = __shfl_sync(FULL, base, 0);
    for (int i = lane; i < cnt; i += 32) {
      const uint64_t pos = base + (uint64_t)i;
      if (side == 0) z[pos] = s[i];
      else z[z_cap - 1 - pos] = s[i];
    }
    __syncwarp();
    cnt = 0;
  }
  __device__ __forceinline__ void group_begin() {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) { glo[u] = ghi[u] = T(0); if (MODE == kDirect) gP[u] = gN[u] = T(0); }
  }
  __device__ __forceinline__ void group_end() {
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
    if (MODE == kCompact) {
      if (n_lo > CAPW - GROUP_MAX) flush(s_lo, n_lo, 0);
      if (n_hi > CAPW - GROUP_MAX) flush(s_hi, n_hi, 1);
    }
  }
  template <bool MASKED, typename V> __device__ __forceinline__ void vec(const V& v, bool ok, int u) {
#pragma unroll
    for (int j = 0; j < VE; ++j) elem(lane_of(v, j), MASKED ? ok : true, u);
  }
  __device__ __forceinline__ void scalar(T v, bool ok) {
    group_begin();
    elem(v, ok, 0);
    group_end();
  }
};

template <typename T, int MODE, int UNROLL>
__global__ void __launch_bounds__(kBlock) pass_kernel(PassArgs a) {
  using Fn = PassFn<T, MODE, UNROLL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Fn f;
  f.t = (T)a.t; f.yL = (T)a.y_lo; f.yR = (T)a.y_hi;
  f.c_lt = f.c_eq = f.c_lo = f.c_hi = 0;
  f.L_lo = f.L_hi = f.P = f.N = 0.0;
  f.pred = -tinf<T>(); f.succ = tinf<T>();
  f.n_lo = f.n_hi = 0;
  if (MODE == kCompact) {
    T* base = reinterpret_cast<T*>(smem_raw) + (size_t)(threadIdx.x >> 5) * 2 * Fn::CAPW;
    f.s_lo = base;
    f.s_hi = base + Fn::CAPW;
    f.z = static_cast<T*>(a.z);
    f.z_cap = a.z_cap;
    f.cursors = a.cursors;
  }
  stream_array<T, UNROLL>(static_cast<const T*>(a.x), a.n, f);
  if (MODE == kCompact) {
    f.flush(f.s_lo, f.n_lo, 0);
    f.flush(f.s_hi, f.n_hi, 1);
  }
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
  }
}

// ------------------------------------------------------------------------------------------
// Step a5: radix select on order-preserving keys.
__device__ __forceinline__ unsigned long long okey(float v) {
  const unsigned u = __float_as_uint(v);
  return (unsigned long long)((u & 0x80000000u) ? ~u : (u | 0x80000000u));
}
__device__ __forceinline__ unsigned long long okey(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
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

constexpr int kRadixBits = 11;
constexpr int kBins = 1 << kRadixBits;

template <typename T> struct HistFn {
  unsigned* sh;
  unsigned long long prefix, mask;
  int shift;
  unsigned dmask;
  __device__ __forceinline__ void elem(T v, bool ok) {
    const unsigned long long k = okey(v);
    if (ok && (k & mask) == prefix) atomicAdd(&sh[(unsigned)(k >> shift) & dmask], 1u);
  }
  __device__ __forceinline__ void group_begin() {}
  __device__ __forceinline__ void group_end() {}
  template <bool MASKED, typename V> __device__ __forceinline__ void vec(const V& v, bool ok, int) {
#pragma unroll
    for (int j = 0; j < VecOf<T>::N; ++j) elem(lane_of(v, j), MASKED ? ok : true);
  }
  __device__ __forceinline__ void scalar(T v, bool ok) { elem(v, ok); }
};

template <typename T>
__global__ void __launch_bounds__(kBlock) hist_kernel(const T* z, uint64_t m, const RadixState* st,
                                                      int shift, int bits, unsigned* hist) {
  __shared__ unsigned sh[kBins];
  for (int i = threadIdx.x; i < kBins; i += kBlock) sh[i] = 0;
  __syncthreads();
  HistFn<T> f;
  f.sh = sh;
  f.prefix = st->prefix;
  f.mask = st->mask;
  f.shift = shift;
  f.dmask = (1u << bits) - 1u;
  stream_array<T, 2>(z, m, f);
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += kBlock)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// One CTA of 1024 threads: find the digit holding rank r, extend the prefix, clear hist.
template <typename T>
__global__ void __launch_bounds__(1024) pick_kernel(RadixState* st, unsigned* hist, int shift, int bits,
                                                    int last) {
  __shared__ unsigned long long scan[1024];
  const int tid = threadIdx.x;
  const int nb = 1 << bits;  // <= 2048: two bins per thread
  const unsigned h0 = (2 * tid < nb) ? hist[2 * tid] : 0u;
  const unsigned h1 = (2 * tid + 1 < nb) ? hist[2 * tid + 1] : 0u;
  scan[tid] = (unsigned long long)h0 + h1;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele scan
    const unsigned long long v = tid >= off ? scan[tid - off] : 0ull;
    __syncthreads();
    scan[tid] += v;
    __syncthreads();
  }
  const unsigned long long r = st->r;
  const unsigned long long before = scan[tid] - h0 - h1;  // exclusive prefix of bin 2*tid
  int digit = -1;
  unsigned long long below = 0, cnt = 0;
  if (before < r && r <= before + h0) { digit = 2 * tid; below = before; cnt = h0; }
  else if (before + h0 < r && r <= before + h0 + h1) { digit = 2 * tid + 1; below = before + h0; cnt = h1; }
  __syncthreads();
  if (digit >= 0) {
    const unsigned long long dmask = (unsigned long long)(nb - 1) << shift;
    st->prefix |= (unsigned long long)digit << shift;
    st->mask |= dmask;
    st->r = r - below;
    st->count = cnt;
    if (last) {
      st->key = st->prefix;
      st->value = (sizeof(T) == 4) ? from_key_f32(st->prefix) : from_key_f64(st->prefix);
    }
  }
  if (2 * tid < kBins) hist[2 * tid] = 0u;
  if (2 * tid + 1 < kBins) hist[2 * tid + 1] = 0u;
}

__global__ void radix_init_kernel(RadixState* st, unsigned long long r, unsigned long long m) {
  st->prefix = 0; st->mask = 0; st->r = r; st->count = m; st->value = 0; st->key = 0;
}

template <typename T, int MODE, int UNROLL> constexpr size_t pass_smem() {
  return MODE == kCompact ? (size_t)kWarps * 2 * stage_cap<T>() * sizeof(T) : 0;
}

template <typename T, int MODE>
cudaError_t launch_pass_t(const PassArgs& a, int grid, cudaStream_t st) {
  constexpr int U = 4;
  constexpr size_t sm = pass_smem<T, MODE, U>();
  pass_kernel<T, MODE, U><<<grid, kBlock, sm, st>>>(a);
  return cudaGetLastError();
}

template <typename T, int MODE> cudaError_t set_attrs() {
  constexpr size_t sm = pass_smem<T, MODE, 4>();
  if (sm > 48 * 1024)
    return cudaFuncSetAttribute(pass_kernel<T, MODE, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  return cudaSuccess;
}

template <typename T, int MODE> cudaError_t occ_pass(int* blocks) {
  cudaError_t e = set_attrs<T, MODE>();
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, pass_kernel<T, MODE, 4>, kBlock,
                                                       pass_smem<T, MODE, 4>());
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
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, init_kernel<float, 4, false>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_init[kF32] = s->num_sms * (b > 0 ? b : 1);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, init_kernel<double, 4, false>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_init[kF64] = s->num_sms * (b > 0 ? b : 1);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, hist_kernel<float>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_hist[kF32] = s->num_sms * (b > 0 ? b : 1);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, hist_kernel<double>, kBlock, 0)) != cudaSuccess) return e;
  s->grid_hist[kF64] = s->num_sms * (b > 0 ? b : 1);
  return cudaSuccess;
}

size_t partial_bytes_needed(const LaunchShape& s) {
  int g = 0;
  for (int d = 0; d < 2; ++d) {
    for (int m = 0; m < 3; ++m) g = g > s.grid_pass[d][m] ? g : s.grid_pass[d][m];
    g = g > s.grid_init[d] ? g : s.grid_init[d];
  }
  const size_t per = sizeof(PassPartial) > sizeof(InitPartial) ? sizeof(PassPartial) : sizeof(InitPartial);
  return (size_t)g * per;
}

static int clamp_grid(int grid, uint64_t n, int per_cta) {
  const uint64_t need = (n + per_cta - 1) / per_cta;
  if (need < (uint64_t)grid) grid = (int)(need > 0 ? need : 1);
  return grid;
}

cudaError_t launch_init(int dtype, const InitArgs& a, const LaunchShape& s, cudaStream_t st, bool checked) {
  if (dtype == kF32) {
    const int grid = clamp_grid(s.grid_init[kF32], a.n, kBlock * 4 * 4);
    if (checked) init_kernel<float, 4, true><<<grid, kBlock, 0, st>>>(a);
    else init_kernel<float, 4, false><<<grid, kBlock, 0, st>>>(a);
  } else {
    const int grid = clamp_grid(s.grid_init[kF64], a.n, kBlock * 4 * 2);
    if (checked) init_kernel<double, 4, true><<<grid, kBlock, 0, st>>>(a);
    else init_kernel<double, 4, false><<<grid, kBlock, 0, st>>>(a);
  }
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

cudaError_t launch_radix_select(int dtype, const void* z, uint64_t m, uint64_t r, RadixState* state,
                                unsigned* hist, const LaunchShape& s, cudaStream_t st) {
  radix_init_kernel<<<1, 1, 0, st>>>(state, r, m);
  // digit plan, MSB first: f32 11+11+10, f64 11+11+11+11+10+10
  static const int plan32[] = {21, 11, 10, 11, 0, 10};
  static const int plan64[] = {53, 11, 42, 11, 31, 11, 20, 11, 10, 10, 0, 10};
  const int rounds = dtype == kF32 ? 3 : 6;
  const int* plan = dtype == kF32 ? plan32 : plan64;
  for (int i = 0; i < rounds; ++i) {
    const int shift = plan[2 * i], bits = plan[2 * i + 1];
    const int last = (i == rounds - 1);
    if (dtype == kF32) {
      const int grid = clamp_grid(s.grid_hist[kF32], m, kBlock * 2 * 4);
      hist_kernel<float><<<grid, kBlock, 0, st>>>(static_cast<const float*>(z), m, state, shift, bits, hist);
      pick_kernel<float><<<1, 1024, 0, st>>>(state, hist, shift, bits, last);
    } else {
      const int grid = clamp_grid(s.grid_hist[kF64], m, kBlock * 2 * 2);
      hist_kernel<double><<<grid, kBlock, 0, st>>>(static_cast<const double*>(z), m, state, shift, bits, hist);
      pick_kernel<double><<<1, 1024, 0, st>>>(state, hist, shift, bits, last);
    }
  }
  return cudaGetLastError();
}

}  // namespace cpsel
