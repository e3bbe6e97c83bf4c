// Host side of libcpsel.so: the cutting-plane driver (Algorithm 1, with the hybrid
// finish of P:L196), its three back ends (one GPU, G GPUs over NCCL, host callbacks) and the
// C ABI declared in include/cpsel.h.
//
// The driver is a pure host state machine; every step over the data is a kernel launch
// (cpsel_kernels.cu) whose 96-byte result tuple comes back to the host once per pass
// (P:L426 'partial sums ... added together on the CPU').  Readings R1-R20: DESIGN.md §3.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cpsel.h"
#include "cpsel_kernels.h"
#include "cpsel_lms.h"
#include "cpsel_comm.h"
#include "cpsel_knn.h"
#include "cpsel_nccl.h"

using namespace cpsel;

// ============================================================================================
// context
struct cpsel_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  LaunchShape shape{};
  cpsel_config cfg{};
  std::string err;
  // device scratch
  void* d_partials = nullptr;
  unsigned int* d_ticket = nullptr;
  unsigned long long* d_cursors = nullptr;
  DevPass* d_pass = nullptr;
  DevInit* d_init = nullptr;
  void* d_t0 = nullptr;              // the two extra cuts of the init pass (R23)
  void* d_skeys = nullptr;           // gathered sample keys (R29)
  void* d_pool1 = nullptr;           // the one-GPU gathered sample values (R29, two-kernel form)
  ChainState* d_chain = nullptr;     // device chain state (§8f-3)
  RadixState* d_radix = nullptr;
  unsigned int* d_hist = nullptr;
  DevPass* d_gather = nullptr;       // G x DevPass (sharded)
  DevInit* d_gather_init = nullptr;  // G x DevInit (sharded)
  void* d_zb[2] = {nullptr, nullptr}; // dense ping-pong compaction buffers
  size_t zb_bytes[2] = {0, 0};
  void* d_sb[2] = {nullptr, nullptr}; // segmented (warp-private) compaction buffers
  size_t sb_bytes[2] = {0, 0};
  void* d_st[2] = {nullptr, nullptr}; // their run tables (SegEntry per warp)
  size_t st_bytes[2] = {0, 0};
  void* d_zall = nullptr;            // all-gathered bracket contents (sharded)
  size_t zall_bytes = 0;
  void* d_stage = nullptr;           // H2D staging (cpsel_select_kth_host)
  size_t stage_bytes = 0;
  // pinned host mirrors
  DevPass* h_pass = nullptr;
  DevInit* h_init = nullptr;
  RadixState* h_radix = nullptr;
  DevPass* h_gather = nullptr;
  DevInit* h_gather_init = nullptr;
  // sharded records published to mapped memory (gather_records): host view, device view, the flag
  unsigned char* h_rec = nullptr;
  unsigned char* d_rec = nullptr;
  size_t rec_bytes = 0;
  unsigned long long* h_rec_flag = nullptr;
  unsigned long long* d_rec_flag = nullptr;
  // sharded sample cuts (R28): the pooled sample (every rank's share of evenly strided values), shard sizes
  void* d_pool = nullptr;
  unsigned long long* d_sizes = nullptr;     // [0] this rank's, [1..G] all ranks'
  unsigned long long* h_sizes = nullptr;
  // LMS workspace
  LmsWorkspace lms;
  // multi-GPU
  Comm comm;  // NCCL communicator or loopback group (cpsel_comm.h)
  // last trace
  std::vector<cpsel_trace_row> trace;
  // kernel timing (record_timing): a pool of (start, end) event pairs, one pair per step of a
  // selection, resolved once the selection is over (no synchronisation between steps)
  std::vector<cudaEvent_t> evpool;
  // record_timing == 2 ("light"): only the init kernel of each selection is bracketed by events,
  // appended to this ring and resolved when the caller asks (cpsel_init_timings) — nothing is read
  // back inside a selection, so the timing does not delay the next call
  std::vector<cudaEvent_t> light_ev;
  uint32_t light_n = 0;
  // result mailbox in mapped pinned memory: the finishing thread of a pass/init/select kernel
  // writes its result here and then bumps the flag the host spins on (no copy, no stream sync)
  struct Mailbox {
    DevPass pass;
    DevInit init;
    double radix_value;
    unsigned long long seq_pass, seq_init, seq_radix;
    unsigned long long radix_fallback;          // the value-binned finish left it to the radix select
    double direct_value;                        // exact_cluster_kernel (small arrays, §8f-3)
    unsigned long long direct_bad, seq_direct;
    ChainMail chain;  // the device chain's step decisions (§8f-3)
  };
  Mailbox* mb = nullptr;      // host view
  Mailbox* mb_dev = nullptr;  // device view of the same memory
  unsigned long long seq = 0;
  // device-resident Kelley loop (§8f-3): its state (device), the host staging of it (pinned), the
  // report it writes (mapped) and one instantiated graph per dtype
  KelleyState* d_ks = nullptr;
  KelleyState* h_ks = nullptr;
  KelleyReport* h_rep = nullptr;
  KelleyReport* d_rep = nullptr;
  cudaGraphExec_t kgraph[2] = {nullptr, nullptr};
  // kNN (§8f-4): the distance matrix, the d2_(k) per query, the non-finite counter
  void* d_knn = nullptr;
  size_t knn_bytes = 0;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

cpsel_status fail(cpsel_ctx* c, cpsel_status s, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return s;
}

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? CPSEL_ENOMEM : CPSEL_ECUDA,     \
                  "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__);   \
  } while (0)

#define NK(expr)                                                                                 \
  do {                                                                                           \
    ncclResult_t r_ = (expr);                                                                    \
    if (r_ != ncclSuccess)                                                                       \
      return fail(ctx, CPSEL_ENCCL, "%s: %s", #expr, nccl_api().GetErrorString(r_));             \
  } while (0)

size_t elem_size(int dt) { return dt == kF32 ? 4 : 8; }

cpsel_status ensure(cpsel_ctx* ctx, void** p, size_t* have, size_t need) {
  if (*have >= need && *p) return CPSEL_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  size_t sz = std::max<size_t>(need, 256);
  CK(cudaMalloc(p, sz));
  *have = sz;
  return CPSEL_OK;
}

// ---------------------------------------------------------------------------------- keys
uint64_t key_of(double v, int dt) {
  if (dt == kF32) {
    float f = (float)v;
    uint32_t u;
    memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? (uint32_t)~u : (u | 0x80000000u);
  }
  uint64_t u;
  memcpy(&u, &v, 8);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
double from_key(uint64_t k, int dt) {
  if (dt == kF32) {
    uint32_t kk = (uint32_t)k;
    uint32_t u = (kk & 0x80000000u) ? (kk & 0x7fffffffu) : ~kk;
    float f;
    memcpy(&f, &u, 4);
    return f;
  }
  uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double v;
  memcpy(&v, &u, 8);
  return v;
}

// Round t to the dtype and nudge it strictly inside ]yL, yR[ (R9).
double snap(double t, double yL, double yR, int dt) {
  if (dt == kF32) {
    const float fl = (float)yL, fr = (float)yR;
    float f = std::isfinite(t) ? (float)t : (float)(0.5 * yL + 0.5 * yR);
    if (!(f > fl)) f = std::nextafterf(fl, INFINITY);
    if (!(f < fr)) f = std::nextafterf(fr, -INFINITY);
    return f;
  }
  double f = std::isfinite(t) ? t : 0.5 * yL + 0.5 * yR;
  if (!(f > yL)) f = std::nextafter(yL, INFINITY);
  if (!(f < yR)) f = std::nextafter(yR, -INFINITY);
  return f;
}

// Brent's root finder (Numerical Recipes' zbrent, the paper's [NR]: P:L136), the comparison
// driver 2: its interpolation proposes the next point on f(t) = c_lt(t) + c_le(t) - 2k + 1 (negative
// below x_(k), positive above, an integer), the passes and the exact bracket stay the cutting
// plane's.  Step by step the same as oracle.brent_root (same operations in double).
struct BrentRoot {
  double a = 0, b = 0, c = 0, fa = 0, fb = 0, fc = 0, d = 0, e = 0;
  void init(double yl, double fl, double yr, double fr) {
    a = yl; fa = fl; b = yr; fb = fr; c = b; fc = fb;
    d = e = b - a;
  }
  double propose() {
    if ((fb > 0.0 && fc > 0.0) || (fb < 0.0 && fc < 0.0)) {
      c = a; fc = fa;
      e = d = b - a;
    }
    if (std::fabs(fc) < std::fabs(fb)) {
      a = b; b = c; c = a;
      fa = fb; fb = fc; fc = fa;
    }
    const double tol1 = 2.0 * 2.220446049250313e-16 * std::fabs(b);
    const double xm = 0.5 * (c - b);
    if (std::fabs(e) >= tol1 && std::fabs(fa) > std::fabs(fb)) {
      const double s = fb / fa;
      double p, q;
      if (a == c) {
        p = 2.0 * xm * s;
        q = 1.0 - s;
      } else {
        const double qq = fa / fc, r = fb / fc;
        p = s * (2.0 * xm * qq * (qq - r) - (b - a) * (r - 1.0));
        q = (qq - 1.0) * (r - 1.0) * (s - 1.0);
      }
      if (p > 0.0) q = -q;
      p = std::fabs(p);
      const double min1 = 3.0 * xm * q - std::fabs(tol1 * q), min2 = std::fabs(e * q);
      if (2.0 * p < (min1 < min2 ? min1 : min2)) {
        e = d;
        d = p / q;
      } else {
        d = xm;
        e = d;
      }
    } else {
      d = xm;
      e = d;
    }
    return b + (std::fabs(d) > tol1 ? d : (xm >= 0.0 ? tol1 : -tol1));
  }
  void accept(double t, double ft) {
    a = b; fa = fb;
    b = t; fb = ft;
  }
};

// Brent's minimisation (Numerical Recipes' brent: parabolic interpolation, golden section when the
// parabola is rejected; the paper's "Brent's method of optimization", P:L113, P:L136, P:L204,
// P:L229), the comparison driver 3, on F_k from the passes' sums.  Reading R37: Brent's own bracket
// [a, b] is kept as NR keeps it and intersected with the exact bracket the counts give; the first
// point is NR's golden-section point.  Step by step the same as oracle.BrentMinStep (the same
// operations in double), so a trace replays exactly from its F values.
struct BrentMin {
  static constexpr double kCgold = 0.3819660, kTol = 1.4901161193847656e-08, kZeps = 1.0e-10;
  double a = 0, b = 0, x = 0, w = 0, v = 0, fx = 0, fw = 0, fv = 0, d = 0, e = 0;
  bool started = false;
  void init(double yl, double yr) {
    a = yl; b = yr;
    x = w = v = yl + kCgold * (yr - yl);
    d = e = 0.0;
    started = false;
  }
  // false once NR's convergence test holds (brent would return x)
  bool propose(double* u) {
    if (!started) {
      *u = x;
      return true;
    }
    const double xm = 0.5 * (a + b);
    const double tol1 = kTol * std::fabs(x) + kZeps, tol2 = 2.0 * tol1;
    if (std::fabs(x - xm) <= tol2 - 0.5 * (b - a)) return false;
    if (std::fabs(e) > tol1) {
      const double r = (x - w) * (fx - fv);
      double q = (x - v) * (fx - fw);
      double p = (x - v) * q - (x - w) * r;
      q = 2.0 * (q - r);
      if (q > 0.0) p = -p;
      q = std::fabs(q);
      const double etemp = e;
      e = d;
      if (std::fabs(p) >= std::fabs(0.5 * q * etemp) || p <= q * (a - x) || p >= q * (b - x)) {
        e = (x >= xm) ? a - x : b - x;
        d = kCgold * e;
      } else {
        d = p / q;
        const double uu = x + d;
        if (uu - a < tol2 || b - uu < tol2) d = (xm - x >= 0.0) ? std::fabs(tol1) : -std::fabs(tol1);
      }
    } else {
      e = (x >= xm) ? a - x : b - x;
      d = kCgold * e;
    }
    *u = std::fabs(d) >= tol1 ? x + d : x + (d >= 0.0 ? std::fabs(tol1) : -std::fabs(tol1));
    return true;
  }
  // F(u) = fu; [yl, yr]: the exact bracket after u's counts
  void accept(double u, double fu, double yl, double yr) {
    if (!started) {
      x = w = v = u;
      fx = fw = fv = fu;
      started = true;
    } else if (fu <= fx) {
      if (u >= x) a = x; else b = x;
      v = w; w = x; x = u;
      fv = fw; fw = fx; fx = fu;
    } else {
      if (u < x) a = u; else b = u;
      if (fu <= fw || w == x) {
        v = w; w = u;
        fv = fw; fw = fu;
      } else if (fu <= fv || v == x || v == w) {
        v = u; fv = fu;
      }
    }
    a = std::max(a, yl);
    b = std::min(b, yr);
  }
};

// Ordered-key bisection point of ]yL, yR[ (safeguard, R7).
double key_mid(double yL, double yR, int dt) {
  const uint64_t a = key_of(yL, dt), b = key_of(yR, dt);
  return from_key(a + (b - a) / 2, dt);
}

double canonical_zero(double v) { return v == 0.0 ? 0.0 : v; }

// ============================================================================================
// Back ends: what one 'reduction' means on a given substrate.
//
// A back end owns a "current array": x at first; after a compacting pass the driver may adopt
// one half of it (multi-level compaction), so later passes read only the bracket
// contents.  Counts a back end returns are local to the current array; the driver adds the
// number of elements dropped below it (D_lo) to get global counts.
struct Backend {
  virtual ~Backend() = default;
  // k: the target rank (for the extra cut, R23)
  virtual cpsel_status init(cpsel_init_stats* out, uint64_t k) = 0;
  // one pass at t over the current array; if compact, also copy ]yL,t[ and ]t,yR[ out
  // (z_lo/z_hi: elements written, summed over ranks)
  // dense: write the halves contiguously (else the back end may keep them segmented)
  virtual cpsel_status pass(double t, double yL, double yR, bool compact, bool dense, cpsel_pass_stats* out,
                            uint64_t* z_lo, uint64_t* z_hi) = 0;
  // are the halves of the last compacting pass contiguous (selectable)?
  virtual bool kept_dense() const { return true; }
  // did the init pass also copy out the elements strictly between its two cuts (R23)?  If so,
  // adopt_init() makes them the current array.
  virtual bool init_compacted() const { return false; }
  virtual uint64_t init_written() const { return 0; }
  virtual cpsel_status adopt_init() { return CPSEL_EINTERNAL; }
  // current array <- half `side` (0: ]yL,t[, 1: ]t,yR[) of the last compacting pass
  virtual cpsel_status adopt(int side) = 0;
  // R26 cut pass over the current array (exactly the bracket interior, m elements): two sample
  // cuts t_a <= t_b around local rank r, #x<=t_a, the copy_if of ]t_a, t_b[ (dense if asked) and
  // its sum of (x - t_a).  adopt(0) then makes the copy the current array.
  struct CutResult {
    double ta, tb, t_est;  // the cuts and the sample's estimate of x_(k)
    uint64_t le_a, inner;  // local #x<=t_a, #]t_a,t_b[
    bool overflow;         // the (dense) copy did not fit: counts valid, nothing kept
  };
  virtual bool has_cut_pass() const { return false; }
  virtual cpsel_status cut_pass(uint64_t /*r*/, bool /*dense*/, CutResult*) { return CPSEL_EINTERNAL; }
  // the bracket shrank without a compaction: the current array now also holds elements outside it
  virtual void set_inexact() {}
  // r-th smallest (1-based) of half `side` of the last compacting pass, or of the current array (2)
  virtual cpsel_status select(int side, uint64_t r, double* out) = 0;
  virtual std::string message() const = 0;
  // kernels launched / timing slot (record_timing; -1: none) / local elements read, of the last step
  uint32_t launches = 0;
  int slot = -1;
  int sample_slot = -1;  // the sample-cut kernels of the last step (R29), if timed separately
  uint64_t scanned = 0;
  // CUDA-event milliseconds of a step's timing slot (waits for it); 0 if none
  virtual double slot_ms(int) { return 0.0; }
  // §8f-3: the rest of the Kelley iterations (no cut passes) and the exact finish on the device
  struct LoopIn {
    double yL, yR, t, N_L, P_R;
    uint64_t c_le_L, c_lt_R, m, D_lo, it, k, n, z_cap, select_cap, dense_cap, max_iters;
    int on_z, exact, bisect, slow, free_step, record;
    double wP, wN;
  };
  struct LoopOut {
    double value = 0.0, loop_ms = 0.0;
    uint32_t exit_reason = 0, passes = 0, cp_iters = 0, fallback = 0, launches = 0;
    int error = 0;
    uint64_t bytes_moved = 0, z_count = 0;
    std::vector<cpsel_trace_row> rows;
  };
  virtual bool has_device_loop() const { return false; }
  virtual cpsel_status device_loop(const LoopIn&, LoopOut*) { return CPSEL_EINTERNAL; }
};

// ------------------------------------------------------------------------ one GPU
// The current array is contiguous (x, or a dense compaction buffer) or segmented (the warp-private
// runs of a segmented compaction: buffer sb[i] + table st[i] + side).  Large brackets are
// compacted into warp-private regions (seg_pass_kernel, no atomics/barriers); once the interior
// is <= the dense threshold the compaction appends to a dense buffer, which the radix select reads.
struct GpuBackend : Backend {
  cpsel_ctx* ctx;
  const void* x;
  uint64_t n;
  int dt;
  // current array
  bool cur_seg = false;
  const void* cur;           // contiguous base, or segmented buffer base
  uint64_t n_cur;            // elements in the current array
  const SegEntry* cur_tab = nullptr;
  int cur_side = 0;
  int cur_dbuf = -1, cur_sbuf = -1;  // dense / segmented buffer in use as input (-1: none)
  // last compaction
  bool last_dense = true;
  int tgt = 0;               // buffer written by the last compacting pass
  uint64_t zlo = 0, zhi = 0; // local halves written by the last compacting pass
  uint64_t cap = 0;          // capacity (elements) of each dense buffer
  uint64_t R = 0;            // segmented region size
  bool init_seg_done = false;  // the init pass wrote ]t_lo, t_hi[ into segmented buffer 0
  uint64_t init_n_in = 0;
  unsigned long long mail_seq = 0;
  bool cur_exact = true;     // a compacted current array holds exactly the bracket interior
  // the device chain (§8f-3): with the fused init the usual continuation (a cut pass on the init's
  // copy, the radix select of its copy) is launched right behind the init; the driver's requests
  // take those results when they ask for exactly those steps
  struct Spec {
    bool active = false, cut_used = false, small = false, direct = false, vbin = false;
    unsigned long long seq_c0 = 0, seq_cut = 0, seq_c1 = 0, seq_radix = 0;
    int sample_slot = -1, cut_slot = -1, radix_slot = -1;
  } spec;
  uint64_t chain_select_cap = 0;  // 0: no device chain
  GpuBackend(cpsel_ctx* c, const void* x_, uint64_t n_, int dt_)
      : ctx(c), x(x_), n(n_), dt(dt_), cur(x_), n_cur(n_) {}
  std::string message() const override { return ctx->err; }
  bool timed() const { return ctx->cfg.record_timing == 1; }
  bool light() const { return ctx->cfg.record_timing == 2; }
  // f32 only (f64 keys crowd into few top-digit bins: the init slows by more than the round saves);
  // measured at 2^30 f32: +1.6% whole-step throughput, init kernel 1% slower.  CPSEL_INIT_HIST0=0: off
  bool init_hist0() const {
    static const bool on = !(getenv("CPSEL_INIT_HIST0") && getenv("CPSEL_INIT_HIST0")[0] == '0');
    return on && dt == kF32;
  }
  // the direct chain's finish by value bins (launch_vbin_finish: the init counts its copy per value
  // bin of ]t_lo, t_hi[, one pass over the copy and a shared-memory select of the target bin), both
  // dtypes; CPSEL_VBIN=0: the key-digit radix select (init_hist0 for f32)
  bool sample_grid_on() const {  // R40; CPSEL_SAMPLE_GRID=0: pool_gather + the cluster select
    static const bool on = !(getenv("CPSEL_SAMPLE_GRID") && getenv("CPSEL_SAMPLE_GRID")[0] == '0');
    return on;
  }
  // R40: the grid kernel's sample, as a multiple of the cluster's (f32 131072, f64 65536 values):
  // f32 4x (524288) — the cuts' rank window narrows by 2 (1/sqrt(S)), so the init copies ~0.5% of
  // x instead of ~1% and the finish reads half as much; measured at 2^30 f32: 700 -> 672 us per
  // median (the init 35 us faster, the sample kernel 10 us slower; 8x and 16x: slower again, the
  // sample's scattered loads cost more than the smaller copy saves); f64 8x (524288 values too):
  // 2^28 f64 medians 429 -> 422 us against 4x.  CPSEL_SAMPLE_X=1|4|8|16 overrides both
  uint64_t sample_grid_x() const {
    static const long env = [] {
      const char* e = getenv("CPSEL_SAMPLE_X");
      const long v = e ? atol(e) : 0;
      return v == 1 || v == 4 || v == 8 || v == 16 ? v : 0L;
    }();
    return (uint64_t)(env ? env : (dt == kF32 ? 4 : 8));
  }
  bool vbin_on() const {
    static const bool on = !(getenv("CPSEL_VBIN") && getenv("CPSEL_VBIN")[0] == '0');
    return on;
  }
  // start/end of the init kernel in the light ring: at most kLightPairs pairs are kept until the
  // caller reads them (further selections go untimed); a start whose end was never recorded (an
  // error in between) is overwritten by the next start, so pairs stay aligned
  static constexpr uint32_t kLightPairs = 4096;
  cudaError_t light_mark(bool start) {
    if (start) {
      ctx->light_n &= ~1u;
      if (ctx->light_n >= 2 * kLightPairs) return cudaSuccess;
    } else if ((ctx->light_n & 1u) == 0) {
      return cudaSuccess;  // its start was not recorded
    }
    if (ctx->light_ev.size() <= ctx->light_n) {
      cudaEvent_t e;
      cudaError_t err = cudaEventCreate(&e);
      if (err != cudaSuccess) return err;
      ctx->light_ev.push_back(e);
    }
    return cudaEventRecord(ctx->light_ev[ctx->light_n++], ctx->stream);
  }
  int next_slot = 0;
  bool use_mail = true;  // results through the mapped mailbox (one GPU); false: device tuple + copy
  cudaError_t tic() {
    slot = -1;
    if (!timed()) return cudaSuccess;
    while (ctx->evpool.size() < 2 * (size_t)(next_slot + 1)) {
      cudaEvent_t e;
      cudaError_t err = cudaEventCreate(&e);
      if (err != cudaSuccess) return err;
      ctx->evpool.push_back(e);
    }
    return cudaEventRecord(ctx->evpool[2 * next_slot], ctx->stream);
  }
  cudaError_t toc() {
    if (!timed()) return cudaSuccess;
    slot = next_slot++;
    return cudaEventRecord(ctx->evpool[2 * slot + 1], ctx->stream);
  }
  double slot_ms(int s) override {
    if (s < 0 || 2 * (size_t)s + 1 >= ctx->evpool.size()) return 0.0;
    float ms = 0.f;
    if (cudaEventSynchronize(ctx->evpool[2 * s + 1]) != cudaSuccess) return 0.0;
    if (cudaEventElapsedTime(&ms, ctx->evpool[2 * s], ctx->evpool[2 * s + 1]) != cudaSuccess) return 0.0;
    return ms;
  }
  // spin until the kernel published `seq` into the mailbox flag (a failed launch or a kernel that
  // ended without publishing is detected through the stream)
  // With a communicator attached (sharded calls) the wait also watches the collectives: an NCCL
  // asynchronous error (a peer process died, a network fault) or no progress for comm.timeout_s
  // aborts the communicator and fails the call with CPSEL_ENCCL instead of spinning forever.
  cpsel_status wait_mail(const unsigned long long* flag, unsigned long long seq) {
    const volatile unsigned long long* f = flag;
    const bool watch = ctx->comm.active();
    const auto t0 = watch ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point();
    for (uint32_t i = 1;; ++i) {
      if (*f == seq) {
        std::atomic_thread_fence(std::memory_order_acquire);
        return CPSEL_OK;
      }
      if ((i & 255u) == 0u) {
        const cudaError_t e = cudaStreamQuery(ctx->stream);
        if (e == cudaSuccess) {
          if (*f == seq) {
            std::atomic_thread_fence(std::memory_order_acquire);
            return CPSEL_OK;
          }
          return fail(ctx, CPSEL_EINTERNAL, "kernel finished without publishing its result");
        }
        if (e != cudaErrorNotReady) return fail(ctx, CPSEL_ECUDA, "%s", cudaGetErrorString(e));
        if (watch && (i & 4095u) == 0u) {
          const char* bad = ctx->comm.health();
          const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          if (bad || waited > ctx->comm.timeout_s) {
            ctx->comm.abort();
            return fail(ctx, CPSEL_ENCCL, "sharded collective failed: %s (communicator aborted; re-run comm init)",
                        bad ? bad : "no progress within the timeout (CPSEL_COMM_TIMEOUT_S)");
          }
        }
      }
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
    }
  }
  char* dbuf(int i) const { return static_cast<char*>(ctx->d_zb[i]); }
  const void* half_ptr(int side) const {  // dense halves of the last (dense) compaction
    return side == 0 ? (const void*)dbuf(tgt) : (const void*)(dbuf(tgt) + (cap - zhi) * elem_size(dt));
  }
  uint64_t half_n(int side) const { return side == 0 ? zlo : zhi; }

  // init kernel (fast form, then the checked form if anything came out non-finite)
  // presampled: d_t0 already holds the cuts (sharded: pooled across ranks, R28)
  cpsel_status run_init(bool sync_result, uint64_t k, bool cut, bool presampled = false) {
    InitArgs a{x, n, ctx->d_partials, ctx->d_ticket, ctx->d_init, cut ? ctx->d_t0 : nullptr};
    a.acc = reinterpret_cast<unsigned long long*>(ctx->d_ticket) + 8;  // words 8..15 of the ticket block
    if (use_mail) {
      a.out = &ctx->mb_dev->init;
      a.done = &ctx->mb_dev->seq_init;
      a.seq = ++ctx->seq;
    }
    // with the segmented buffers in place the init pass also copies out ]t_lo, t_hi[ (R23)
    const bool fuse = cut && R > 0;
    init_seg_done = false;
    CK(tic());
    sample_slot = -1;
    int sample_launches = 0;
    if (cut && !presampled) {
      sample_launches = 1;
      const bool small = n <= (1ull << 26);
      const uint64_t S = pool_sample_size(dt, small);
      if (n > 4 * S) {
        // R29: the strided sample gathered by a many-CTA kernel (every SM's load slots, not just the
        // cluster's 8: the gather was latency-bound there), then the cluster select reads it
        // contiguously from L2 — the same sample and the same cuts as the one-launch form
        if (sample_grid_on()) {
          // R40: the same sample and cuts in one cooperative launch (d_pool1 as its zeroed scratch)
          const uint64_t Sg = small ? S : S * sample_grid_x();
          CK(launch_sample_grid(dt, x, n, n > 4 * Sg ? Sg : S, n, k, ctx->d_t0, static_cast<unsigned*>(ctx->d_pool1),
                                ctx->stream, !ctx->cfg.objective));
        } else {
          CK(launch_pool_gather(dt, x, n, nullptr, 0, 0, S, ctx->d_pool1, ctx->stream));
          CK(launch_pool_pick(dt, ctx->d_pool1, S, n, k, ctx->d_t0, ctx->stream, small, !ctx->cfg.objective));
          sample_launches = 2;
        }
      } else {
        CK(launch_sample_select(dt, x, n, nullptr, 0, 0, k, ctx->d_t0, ctx->d_skeys, ctx->stream, small, nullptr, 0,
                                /*allow_open=*/!ctx->cfg.objective));
      }
      CK(toc());
      sample_slot = slot;
      CK(tic());
    }
    if (light()) CK(light_mark(true));
    // the device chain (§8f-3) when its continuation is likely: the init's copy (~1-4% of n) will
    // exceed the exact-selection cap
    spec = Spec{};
    // the init's copy holds ~2% of n: radix-select it right behind the init when it will fit the
    // select cap (direct), else chain the R26 cut pass first
    const bool chain_ok = fuse && use_mail && !presampled && chain_select_cap > 0 && !ctx->cfg.objective;
    const bool direct = chain_ok && n / 25 <= chain_select_cap && n > (1ull << 22);
    const bool chain = chain_ok && (direct || (ctx->cfg.pass_cuts && n / 100 > chain_select_cap));
    if (fuse) {
      SegArgs sa{};
      sa.out = ctx->d_sb[0];
      sa.R = R;
      sa.seg_out = static_cast<SegEntry*>(ctx->d_st[0]);
      if (chain) {
        a.chain = ctx->d_chain;
        a.chain_mail = &ctx->mb_dev->chain;
        a.chain_seq = ++ctx->seq;
        if (direct) spec.seq_c1 = a.chain_seq; else spec.seq_c0 = a.chain_seq;
        a.chain_k = k;
        a.chain_cap = chain_select_cap;
        a.chain_direct = direct ? 1 : 0;
        // vbin: the init counts its copy per value bin for the value-binned finish; else (init_hist0)
        // radix round 0 of its copy (one radix round fewer)
        a.vbin = (direct && vbin_on()) ? 1 : 0;
        a.hist = (direct && (vbin_on() || init_hist0())) ? ctx->d_hist + 2048 : nullptr;
      }
      CK(launch_init_seg(dt, a, sa, ctx->shape, ctx->stream, ctx->cfg.objective != 0));
    } else {
      CK(launch_init(dt, a, ctx->shape, ctx->stream, false));
    }
    CK(toc());
    if (light()) CK(light_mark(false));
    const int init_slot_ = slot;
    if (chain) CK(direct ? launch_chain_direct() : launch_chain(k));
    slot = init_slot_;
    launches = 1 + sample_launches;  // the init and the sample kernels before it
    scanned = n;
    if (use_mail) {
      cpsel_status w = wait_mail(&ctx->mb->seq_init, a.seq);
      if (w != CPSEL_OK) return w;
      *ctx->h_init = ctx->mb->init;
    } else if (sync_result) {
      CK(cudaMemcpyAsync(ctx->h_init, ctx->d_init, sizeof(DevInit), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    } else {
      // the caller reads the record from d_init itself (sharded: all-gathered, checked after it)
      init_seg_done = fuse;
      return CPSEL_OK;
    }
    const DevInit& r = *ctx->h_init;
    // fast form: no non-finite count; NaN/Inf surface as a non-finite sum/extreme or, with the
    // cuts (which skip the shifted sum), as #x<t_hi + #x=t_hi + #x>t_hi < n
    // R27: without the extremes' multiplicities the driver brackets with their outer neighbours,
    // which must be finite (else the checked form below counts them)
    const bool f32 = dt == kF32;
    const double out_lo = f32 ? (double)std::nextafterf((float)r.vmin, -INFINITY) : std::nextafter(r.vmin, -INFINITY);
    const double out_hi = f32 ? (double)std::nextafterf((float)r.vmax, INFINITY) : std::nextafter(r.vmax, INFINITY);
    const bool suspicious = cut ? (!std::isfinite(r.N_lo) || !std::isfinite(r.P_hi) || !std::isfinite(r.I_in) ||
                                   !std::isfinite(r.t_est) ||
                                   ((r.has_cut & 8) && !(std::isfinite(out_lo) && std::isfinite(out_hi))) ||
                                   !std::isfinite(r.vmin) || !std::isfinite(r.vmax) || r.nonfinite != 0)
                                : (!std::isfinite(r.S) || !std::isfinite(r.vmin) || !std::isfinite(r.vmax));
    if (!suspicious && fuse) {
      init_seg_done = true;
      init_n_in = r.pad;
    }
    if (suspicious) {
      if (use_mail) a.seq = ++ctx->seq;
      CK(launch_init(dt, a, ctx->shape, ctx->stream, true));
      launches += 1;
      if (use_mail) {
        cpsel_status w = wait_mail(&ctx->mb->seq_init, a.seq);
        if (w != CPSEL_OK) return w;
        *ctx->h_init = ctx->mb->init;
      } else if (sync_result) {
        CK(cudaMemcpyAsync(ctx->h_init, ctx->d_init, sizeof(DevInit), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
      }
    }
    return CPSEL_OK;
  }
  // launch the usual continuation behind the init (kernels read m, r and go/no-go from the chain)
  // direct chain: the radix select of the init's segmented copy, gated by decision 1
  cudaError_t launch_chain_direct() {
    cudaError_t e;
    spec.active = true;
    spec.direct = true;
    spec.seq_radix = ++ctx->seq;
    spec.vbin = vbin_on();
    if ((e = tic()) != cudaSuccess) return e;
    if (spec.vbin) {
      e = launch_vbin_finish(dt, ctx->d_sb[0], static_cast<const SegEntry*>(ctx->d_st[0]), ctx->d_t0, ctx->d_hist,
                             ctx->shape, ctx->stream, ctx->d_chain, &ctx->mb_dev->radix_value,
                             &ctx->mb_dev->radix_fallback, &ctx->mb_dev->seq_radix, spec.seq_radix);
    } else {
      e = launch_radix_select(dt, ctx->d_sb[0], 0, 0, ctx->d_radix, ctx->d_hist, ctx->shape, ctx->stream,
                              &ctx->mb_dev->radix_value, &ctx->mb_dev->seq_radix, spec.seq_radix,
                              static_cast<const SegEntry*>(ctx->d_st[0]), 0, ctx->d_ticket, ctx->d_chain,
                              /*first_round=*/init_hist0() ? 1 : 0, init_hist0() ? ctx->d_hist + 2048 : nullptr,
                              /*m_hint: the expected copy*/ n / (n <= (1ull << 26) ? 25 : 100));
    }
    if (e != cudaSuccess) return e;
    if ((e = toc()) != cudaSuccess) return e;
    spec.radix_slot = slot;
    return cudaSuccess;
  }
  cudaError_t launch_chain(uint64_t k) {
    cudaError_t e;
    spec.active = true;
    spec.small = true;  // the init's copy holds ~2% of n (the driver's own choice is checked on use)
    const int W = seg_total_warps(dt, ctx->shape);
    if ((e = tic()) != cudaSuccess) return e;
    if ((e = launch_sample_select(dt, ctx->d_sb[0], 0, static_cast<const SegEntry*>(ctx->d_st[0]), 0, W, 0, ctx->d_t0,
                                  ctx->d_skeys, ctx->stream, spec.small, ctx->d_chain, 0)) != cudaSuccess) return e;
    if ((e = toc()) != cudaSuccess) return e;
    spec.sample_slot = slot;
    SegArgs a{};
    a.x = ctx->d_sb[0]; a.n = 0;
    a.seg_in = static_cast<const SegEntry*>(ctx->d_st[0]);
    a.side_in = 0;
    a.cuts = ctx->d_t0;
    a.dense_out = 0;
    a.out = ctx->d_sb[1];
    a.R = R;
    a.seg_out = static_cast<SegEntry*>(ctx->d_st[1]);
    a.cursors = ctx->d_cursors;
    a.partials = ctx->d_partials; a.ticket = ctx->d_ticket;
    a.out_tuple = &ctx->mb_dev->pass;
    a.done = &ctx->mb_dev->seq_pass;
    a.seq = spec.seq_cut = ++ctx->seq;
    a.chain = ctx->d_chain;
    a.chain_out = ctx->d_chain;
    a.chain_mail = &ctx->mb_dev->chain;
    a.chain_seq = spec.seq_c1 = ++ctx->seq;
    a.chain_k = k;
    a.chain_cap = chain_select_cap;
    if ((e = tic()) != cudaSuccess) return e;
    if ((e = launch_cut_pass(dt, a, ctx->shape, ctx->stream)) != cudaSuccess) return e;
    if ((e = toc()) != cudaSuccess) return e;
    spec.cut_slot = slot;
    spec.seq_radix = ++ctx->seq;
    if ((e = tic()) != cudaSuccess) return e;
    if ((e = launch_radix_select(dt, ctx->d_sb[1], 0, 0, ctx->d_radix, ctx->d_hist, ctx->shape, ctx->stream,
                                 &ctx->mb_dev->radix_value, &ctx->mb_dev->seq_radix, spec.seq_radix,
                                 static_cast<const SegEntry*>(ctx->d_st[1]), 0, ctx->d_ticket, ctx->d_chain, 0, nullptr,
                                 /*m_hint: ~4% of the init's ~1% copy*/ n / 2500)) != cudaSuccess)
      return e;
    if ((e = toc()) != cudaSuccess) return e;
    spec.radix_slot = slot;
    return cudaSuccess;
  }
  // the chain's decision `which` (0: after the init, 1: after the cut pass), once published
  cpsel_status chain_decision(int which, unsigned long long seq, bool* ok, uint64_t* m, uint64_t* r) {
    cpsel_status w = wait_mail(&ctx->mb->chain.seq[which], seq);
    if (w != CPSEL_OK) return w;
    *ok = ctx->mb->chain.ok[which] != 0;
    *m = ctx->mb->chain.m[which];
    *r = ctx->mb->chain.r[which];
    return CPSEL_OK;
  }
  cpsel_status init(cpsel_init_stats* o, uint64_t k) override {
    // (an array the driver selects directly gets the plain init: the cuts would not be used)
    cpsel_status st = run_init(true, k, ctx->cfg.init_cut != 0 && n > 2 &&
                                            (n > ctx->cfg.direct_threshold || ctx->cfg.force_cp));
    if (st != CPSEL_OK) return st;
    const DevInit& r = *ctx->h_init;
    o->vmin = r.vmin; o->vmax = r.vmax; o->cnt_min = r.cnt_min; o->cnt_max = r.cnt_max;
    o->nonfinite = r.nonfinite; o->x0 = r.x0; o->S = r.S;
    o->has_cut = r.has_cut; o->t_lo = r.t_lo; o->t_hi = r.t_hi;
    o->c_le_lo = r.c_le_lo; o->c_lt_hi = r.c_lt_hi; o->t_est = r.t_est;
    o->N_lo = r.N_lo; o->P_hi = r.P_hi; o->I_in = r.I_in;
    return CPSEL_OK;
  }
  // two dense ping-pong buffers of m_dense elements; two segmented buffers (+ run tables) able to
  // hold any compaction of the n-element array
  cpsel_status ensure_z(uint64_t m_dense, bool need_seg) {
    const size_t es = elem_size(dt);
    for (int i = 0; i < 2; ++i) {
      cpsel_status s = ensure(ctx, &ctx->d_zb[i], &ctx->zb_bytes[i], (size_t)std::max<uint64_t>(m_dense, 1) * es);
      if (s != CPSEL_OK) return s;
    }
    cap = std::min(ctx->zb_bytes[0], ctx->zb_bytes[1]) / es;
    if (need_seg) {
      R = seg_region(dt, n, ctx->shape);
      const size_t W = (size_t)seg_total_warps(dt, ctx->shape);
      for (int i = 0; i < 2; ++i) {
        cpsel_status s = ensure(ctx, &ctx->d_sb[i], &ctx->sb_bytes[i], W * R * es);
        if (s != CPSEL_OK) return s;
        s = ensure(ctx, &ctx->d_st[i], &ctx->st_bytes[i], W * sizeof(SegEntry));
        if (s != CPSEL_OK) return s;
      }
    }
    return CPSEL_OK;
  }
  cpsel_status launch_local_pass(double t, double yL, double yR, bool compact, bool dense) {
    if (!compact) {  // only ever on a contiguous array (before the first compaction)
      PassArgs a{};
      a.x = cur; a.n = n_cur; a.t = t; a.y_lo = yL; a.y_hi = yR;
      a.mode = kHot;
      a.cursors = ctx->d_cursors;
      a.partials = ctx->d_partials; a.ticket = ctx->d_ticket; a.out = ctx->d_pass;
      if (use_mail) {
        a.out = &ctx->mb_dev->pass;
        a.done = &ctx->mb_dev->seq_pass;
        a.seq = mail_seq = ++ctx->seq;
      }
      CK(tic());
      CK(launch_pass(dt, a, ctx->shape, ctx->stream));
      CK(toc());
    } else {
      SegArgs a{};
      a.x = cur; a.n = n_cur;
      a.seg_in = cur_seg ? cur_tab : nullptr;
      a.side_in = cur_side;
      a.t = t; a.y_lo = yL; a.y_hi = yR;
      a.dense_out = dense ? 1 : 0;
      if (dense) {
        tgt = (cur_dbuf == 0) ? 1 : 0;
        a.out = ctx->d_zb[tgt];
        a.z_cap = cap;
      } else {
        tgt = (cur_sbuf == 0) ? 1 : 0;
        a.out = ctx->d_sb[tgt];
        a.R = R;
        a.seg_out = static_cast<SegEntry*>(ctx->d_st[tgt]);
      }
      a.cursors = ctx->d_cursors;
      a.partials = ctx->d_partials; a.ticket = ctx->d_ticket; a.out_tuple = ctx->d_pass;
      if (use_mail) {
        a.out_tuple = &ctx->mb_dev->pass;
        a.done = &ctx->mb_dev->seq_pass;
        a.seq = mail_seq = ++ctx->seq;
      }
      CK(tic());
      // a compacted current array holds only bracket-interior elements (unless a cut pass moved
      // the bracket without compacting, R26)
      CK(launch_seg_pass(dt, a, /*inside=*/cur != x && cur_exact, ctx->shape, ctx->stream));
      CK(toc());
      last_dense = dense;
    }
    launches = 1;
    scanned = n_cur;
    return CPSEL_OK;
  }
  cpsel_status pass(double t, double yL, double yR, bool compact, bool dense, cpsel_pass_stats* o, uint64_t* z_lo,
                    uint64_t* z_hi) override {
    cpsel_status st = launch_local_pass(t, yL, yR, compact, dense);
    if (st != CPSEL_OK) return st;
    st = wait_mail(&ctx->mb->seq_pass, mail_seq);
    if (st != CPSEL_OK) return st;
    const DevPass r = ctx->mb->pass;
    o->c_lt = r.c_lt; o->c_eq = r.c_eq; o->c_lo = r.c_lo; o->c_hi = r.c_hi;
    o->L_lo = r.L_lo; o->L_hi = r.L_hi; o->P = r.P; o->N = r.N; o->pred = r.pred; o->succ = r.succ;
    if (compact) { zlo = r.z_lo; zhi = r.z_hi; }
    *z_lo = r.z_lo; *z_hi = r.z_hi;
    return CPSEL_OK;
  }
  bool init_compacted() const override { return init_seg_done; }
  uint64_t init_written() const override { return init_n_in; }
  void set_inexact() override { cur_exact = false; }
  bool has_cut_pass() const override { return use_mail && R > 0; }
  cpsel_status cut_pass(uint64_t r, bool dense, CutResult* o) override {
    dense = false;  // one GPU: the radix select reads the segmented copy directly (no atomics)
    if (spec.active && !spec.direct && !spec.cut_used && cur_seg && cur_sbuf == 0 && cur == ctx->d_sb[0]) {
      bool ok;
      uint64_t cm, cr;
      cpsel_status w = chain_decision(0, spec.seq_c0, &ok, &cm, &cr);
      if (w != CPSEL_OK) return w;
      if (ok && cr == r && cm == n_cur && spec.small == (n_cur <= (1ull << 26))) {  // the chain ran this pass
        w = wait_mail(&ctx->mb->seq_pass, spec.seq_cut);
        if (w != CPSEL_OK) return w;
        const DevPass rr = ctx->mb->pass;
        o->ta = rr.pred; o->tb = rr.succ; o->t_est = rr.L_lo;
        o->le_a = rr.c_lt; o->inner = rr.z_lo;
        o->overflow = rr.c_eq != 0;
        tgt = 1;
        last_dense = false;
        zlo = rr.z_lo; zhi = 0;
        launches = 3;
        scanned = n_cur;
        slot = spec.cut_slot;
        sample_slot = spec.sample_slot;
        spec.cut_used = true;
        return CPSEL_OK;
      }
      spec.active = false;
    }
    CK(tic());
    // a bracket already cut once holds ~2% of x: 8192 samples cut it to ~4% of itself, below select_cap
    CK(launch_sample_select(dt, cur, n_cur, cur_seg ? cur_tab : nullptr, cur_side, seg_total_warps(dt, ctx->shape), r,
                            ctx->d_t0, ctx->d_skeys, ctx->stream, /*small=*/n_cur <= (1ull << 26)));
    CK(toc());
    sample_slot = slot;
    SegArgs a{};
    a.x = cur; a.n = n_cur;
    a.seg_in = cur_seg ? cur_tab : nullptr;
    a.side_in = cur_side;
    a.cuts = ctx->d_t0;
    a.dense_out = dense ? 1 : 0;
    if (dense) {
      tgt = (cur_dbuf == 0) ? 1 : 0;
      a.out = ctx->d_zb[tgt];
      a.z_cap = cap;
    } else {
      tgt = (cur_sbuf == 0) ? 1 : 0;
      a.out = ctx->d_sb[tgt];
      a.R = R;
      a.seg_out = static_cast<SegEntry*>(ctx->d_st[tgt]);
    }
    a.cursors = ctx->d_cursors;
    a.partials = ctx->d_partials; a.ticket = ctx->d_ticket;
    a.out_tuple = &ctx->mb_dev->pass;
    a.done = &ctx->mb_dev->seq_pass;
    a.seq = mail_seq = ++ctx->seq;
    CK(tic());
    CK(launch_cut_pass(dt, a, ctx->shape, ctx->stream));
    CK(toc());
    launches = 2;
    scanned = n_cur;
    cpsel_status st = wait_mail(&ctx->mb->seq_pass, mail_seq);
    if (st != CPSEL_OK) return st;
    const DevPass rr = ctx->mb->pass;
    o->ta = rr.pred; o->tb = rr.succ; o->t_est = rr.L_lo;
    o->le_a = rr.c_lt; o->inner = rr.z_lo;
    o->overflow = rr.c_eq != 0;
    last_dense = dense;
    zlo = rr.z_lo; zhi = 0;
    return CPSEL_OK;
  }
  cpsel_status adopt_init() override {
    cur_exact = true;
    cur_seg = true;
    cur = ctx->d_sb[0];
    cur_tab = static_cast<const SegEntry*>(ctx->d_st[0]);
    cur_side = 0;
    cur_sbuf = 0;
    n_cur = init_n_in;
    return CPSEL_OK;
  }
  cpsel_status adopt(int side) override {
    cur_exact = true;
    if (last_dense) {
      cur_seg = false;
      cur = half_ptr(side);
      cur_dbuf = tgt;
    } else {
      cur_seg = true;
      cur = ctx->d_sb[tgt];
      cur_tab = static_cast<const SegEntry*>(ctx->d_st[tgt]);
      cur_side = side;
      cur_sbuf = tgt;
    }
    n_cur = half_n(side);
    return CPSEL_OK;
  }
  // tab != nullptr: the runs `side` of a segmented array based at `base`
  cpsel_status select_on(const void* base, uint64_t m, uint64_t r, double* out, const SegEntry* tab = nullptr,
                         int side = 0) {
    CK(tic());
    // the value comes back through the ctx's mapped mailbox (also on the sharded path: every rank's
    // own select)
    const unsigned long long seq = ++ctx->seq;
    CK(launch_radix_select(dt, base, m, r, ctx->d_radix, ctx->d_hist, ctx->shape, ctx->stream,
                           &ctx->mb_dev->radix_value, &ctx->mb_dev->seq_radix, seq, tab, side, ctx->d_ticket));
    CK(toc());
    cpsel_status w = wait_mail(&ctx->mb->seq_radix, seq);
    if (w != CPSEL_OK) return w;
    *out = ctx->mb->radix_value;
    launches = dt == kF32 ? 3 : 6;
    scanned = m;
    return CPSEL_OK;
  }
  // §8f-3: hand the remaining Kelley passes and the exact finish to the device (one graph launch)
  bool has_device_loop() const override { return use_mail; }
  cpsel_status device_loop(const LoopIn& li, LoopOut* lo) override {
    static_assert(sizeof(KRow) == sizeof(cpsel_trace_row), "trace row layout");
    if (!ctx->d_ks) {
      CK(cudaMalloc(&ctx->d_ks, sizeof(KelleyState)));
      CK(cudaHostAlloc(&ctx->h_ks, sizeof(KelleyState), cudaHostAllocDefault));
      CK(cudaHostAlloc(&ctx->h_rep, sizeof(KelleyReport), cudaHostAllocMapped));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->d_rep), ctx->h_rep, 0));
    }
    if (!ctx->kgraph[dt])
      CK(kelley_graph_build(dt, ctx->shape, ctx->d_ks, ctx->d_partials, ctx->d_ticket, ctx->d_cursors, ctx->d_radix,
                            ctx->d_hist, &ctx->kgraph[dt]));
    KelleyState& h = *ctx->h_ks;
    memset(&h, 0, sizeof h);
    h.n = li.n; h.k = li.k; h.z_cap = li.z_cap; h.select_cap = li.select_cap; h.dense_cap = li.dense_cap;
    h.max_iters = li.max_iters;
    h.seq = ++ctx->seq;
    h.wP = li.wP; h.wN = li.wN;
    h.x = x;
    for (int i = 0; i < 2; ++i) {
      h.sb[i] = ctx->d_sb[i];
      h.st[i] = static_cast<SegEntry*>(ctx->d_st[i]);
      h.zb[i] = ctx->d_zb[i];
    }
    h.cap = cap; h.R = R;
    h.dt = dt; h.record = li.record;
    h.vout = &ctx->mb_dev->radix_value;
    h.done_flag = &ctx->mb_dev->seq_radix;
    h.rep = ctx->d_rep;
    h.yL = li.yL; h.yR = li.yR; h.t = li.t; h.N_L = li.N_L; h.P_R = li.P_R;
    h.c_le_L = li.c_le_L; h.c_lt_R = li.c_lt_R; h.m = li.m; h.D_lo = li.D_lo; h.it = li.it;
    h.on_z = li.on_z; h.exact = li.exact && cur_exact; h.bisect = li.bisect; h.slow = li.slow;
    h.free_step = li.free_step;
    h.cur = cur; h.n_cur = n_cur; h.cur_tab = cur_seg ? cur_tab : nullptr;
    h.cur_seg = cur_seg; h.cur_side = cur_side; h.cur_sbuf = cur_sbuf; h.cur_dbuf = cur_dbuf;
    h.tgt = tgt; h.last_dense = last_dense;
    CK(cudaMemcpyAsync(ctx->d_ks, &h, sizeof h, cudaMemcpyHostToDevice, ctx->stream));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed()) {
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, ctx->stream));
    }
    const cudaError_t le = cudaGraphLaunch(ctx->kgraph[dt], ctx->stream);
    if (le != cudaSuccess) {
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
      return fail(ctx, CPSEL_ECUDA, "cudaGraphLaunch: %s", cudaGetErrorString(le));
    }
    if (e1) cudaEventRecord(e1, ctx->stream);
    cpsel_status w = wait_mail(&ctx->mb->seq_radix, h.seq);
    if (w == CPSEL_OK && e1) {
      float ms = 0.f;
      if (cudaEventSynchronize(e1) == cudaSuccess && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess) lo->loop_ms = ms;
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (w != CPSEL_OK) return w;
    const KelleyReport& r = *ctx->h_rep;
    lo->value = ctx->mb->radix_value;
    lo->error = r.error;
    lo->exit_reason = r.exit_reason;
    lo->passes = r.passes; lo->cp_iters = r.cp_iters; lo->fallback = r.fallback; lo->launches = r.launches;
    lo->bytes_moved = r.bytes_moved; lo->z_count = r.z_count;
    lo->rows.clear();
    const unsigned nr = std::min<unsigned>(r.n_rows, (unsigned)kKelleyMaxRows);
    for (unsigned i = 0; li.record && i < nr; ++i) {
      cpsel_trace_row row;
      memcpy(&row, &r.rows[i], sizeof row);
      lo->rows.push_back(row);
    }
    launches = 1;
    return CPSEL_OK;
  }
  // the radix select reads dense and segmented arrays alike
  bool kept_dense() const override { return true; }
  cpsel_status select(int side, uint64_t r, double* out) override {
    if (spec.active && spec.direct && side == 2 && cur_seg && cur_sbuf == 0 && cur == ctx->d_sb[0] && cur_side == 0) {
      bool ok;
      uint64_t cm, cr;
      cpsel_status w = chain_decision(1, spec.seq_c1, &ok, &cm, &cr);
      if (w != CPSEL_OK) return w;
      spec.active = false;
      if (ok && cr == r && cm == n_cur) {  // the chain ran this select right behind the init
        w = wait_mail(&ctx->mb->seq_radix, spec.seq_radix);
        if (w != CPSEL_OK) return w;
        if (!(spec.vbin && ctx->mb->radix_fallback)) {
          *out = ctx->mb->radix_value;
          launches = spec.vbin ? 1 : (dt == kF32 ? 3 : 6) - (init_hist0() ? 1 : 0);  // round 0 by the init?
          scanned = cm;
          slot = spec.radix_slot;
          return CPSEL_OK;
        }
        // a large target bin of several values: the key-digit radix select below (it left everything clean)
      }
    }
    if (spec.active && spec.cut_used && side == 0 && !last_dense && tgt == 1) {
      bool ok;
      uint64_t cm, cr;
      cpsel_status w = chain_decision(1, spec.seq_c1, &ok, &cm, &cr);
      if (w != CPSEL_OK) return w;
      spec.active = false;
      if (ok && cr == r && cm == half_n(0)) {  // the chain ran this select
        w = wait_mail(&ctx->mb->seq_radix, spec.seq_radix);
        if (w != CPSEL_OK) return w;
        *out = ctx->mb->radix_value;
        launches = dt == kF32 ? 4 : 7;  // + the chain step kernels
        scanned = cm;
        slot = spec.radix_slot;
        return CPSEL_OK;
      }
    }
    if (side == 2) return cur_seg ? select_on(cur, n_cur, r, out, cur_tab, cur_side) : select_on(cur, n_cur, r, out);
    if (last_dense) return select_on(half_ptr(side), half_n(side), r, out);
    return select_on(ctx->d_sb[tgt], half_n(side), r, out, static_cast<const SegEntry*>(ctx->d_st[tgt]), side);
  }
};

// ------------------------------------------------------------------------ G GPUs (NCCL)
// R28: cuts common to all ranks from their pooled samples.  keys: G blocks of 1024 sorted sample
// keys (block g holds ms_g = min(m_g, 1024) samples of rank g's m_g elements, padding after them);
// each sample of rank g stands for m_g / ms_g elements.  Same ranks q -/+ (3.5 sd + 2) as the
// one-array pick, in units of the pooled sample; every rank computes the same cuts from the same
// bytes.  Returns false if there is no sample at all.
bool pooled_pick(const unsigned long long* keys, const std::vector<uint64_t>& m, uint64_t r, int dt, double out[3]) {
  const int G = (int)m.size();
  std::vector<std::pair<unsigned long long, double>> smp;
  uint64_t M = 0, S = 0;
  for (int g = 0; g < G; ++g) {
    const uint64_t ms = std::min<uint64_t>(m[g], 1024);
    M += m[g];
    S += ms;
    for (uint64_t i = 0; i < ms; ++i) smp.emplace_back(keys[(size_t)g * 1024 + i], (double)m[g] / (double)ms);
  }
  if (smp.empty() || M == 0) return false;
  std::sort(smp.begin(), smp.end());
  const double Sd = (double)S;
  const double qs = ((double)r - 0.5) / (double)M * Sd;
  const double ws = 3.5 * std::sqrt(std::max(qs * (Sd - qs) / Sd, 0.0)) + 2.0;
  const double scale = (double)M / Sd;  // elements per pooled sample
  const double pos[3] = {(qs - ws) * scale, (qs + ws) * scale, qs * scale};
  for (int j = 0; j < 3; ++j) {
    double c = 0.0;
    size_t i = 0;
    for (; i + 1 < smp.size(); ++i) {
      c += smp[i].second;
      if (c > pos[j]) break;
    }
    out[j] = from_key(smp[i].first, dt);
  }
  return true;
}

struct ShardedBackend : GpuBackend {
  std::vector<uint64_t> n_rank;               // shard sizes
  std::vector<uint64_t> cur_rank;             // current-array sizes per rank
  std::vector<uint64_t> zlo_rank, zhi_rank;   // per-rank halves of the last compacting pass
  cpsel_init_stats combined{};
  uint64_t n_global = 0;
  ShardedBackend(cpsel_ctx* c, const void* x_, uint64_t n_local, int dt_) : GpuBackend(c, x_, n_local, dt_) {
    use_mail = false;  // the per-rank tuples are all-gathered from device memory
  }
  Comm& comm() const { return ctx->comm; }
  int G() const { return ctx->comm.world; }
  bool has_device_loop() const override { return false; }  // every pass ends in a collective
  // every kept part is selectable: select() packs a segmented one before the all-gather-v
  bool kept_dense() const override { return true; }

#define CM(expr)                                                                 \
  do {                                                                           \
    const char* m_ = (expr);                                                     \
    if (m_) return fail(ctx, CPSEL_ENCCL, "%s: %s", #expr, m_);                  \
  } while (0)

  // all-gather `bytes` per rank from d_src into d_all and bring the G records to h_all: published
  // into mapped memory by a one-CTA kernel behind the collective, the host spins on its flag (no
  // stream synchronisation per exchange)
  cpsel_status gather_records(const void* d_src, void* d_all, void* h_all, size_t bytes) {
    CM(comm().allgather(d_src, d_all, bytes, ctx->stream));
    const size_t tot = (size_t)G() * bytes;
    if (tot > ctx->rec_bytes) return fail(ctx, CPSEL_EINTERNAL, "record mailbox too small");
    const unsigned long long seq = ++ctx->seq;
    CK(launch_publish(d_all, ctx->d_rec, tot, ctx->d_rec_flag, seq, ctx->stream));
    cpsel_status w = wait_mail(ctx->h_rec_flag, seq);
    if (w != CPSEL_OK) return w;
    memcpy(h_all, ctx->h_rec, tot);
    return CPSEL_OK;
  }

  // the fast init's record needs the checked form (same test as the one-GPU path)
  static bool suspicious(const DevInit& r, bool cut, int dt) {
    const bool f32 = dt == kF32;
    const double out_lo = f32 ? (double)std::nextafterf((float)r.vmin, -INFINITY) : std::nextafter(r.vmin, -INFINITY);
    const double out_hi = f32 ? (double)std::nextafterf((float)r.vmax, INFINITY) : std::nextafter(r.vmax, INFINITY);
    return cut ? (!std::isfinite(r.N_lo) || !std::isfinite(r.P_hi) || !std::isfinite(r.I_in) || !std::isfinite(r.t_est) ||
                  ((r.has_cut & 8) && !(std::isfinite(out_lo) && std::isfinite(out_hi))) || !std::isfinite(r.vmin) ||
                  !std::isfinite(r.vmax) || r.nonfinite != 0)
               : (!std::isfinite(r.S) || !std::isfinite(r.vmin) || !std::isfinite(r.vmax));
  }

  // All-gather the per-rank init records and combine them in rank order (R17).
  cpsel_status gather_init() {
    if (n > 0) {
      cpsel_status st = run_init(true, 0, false);  // leaves the (checked) record in d_init
      if (st != CPSEL_OK) return st;
    } else {
      launches = 0;
      DevInit e{};
      e.vmin = INFINITY; e.vmax = -INFINITY;
      *ctx->h_init = e;
      CK(cudaMemcpyAsync(ctx->d_init, ctx->h_init, sizeof(DevInit), cudaMemcpyHostToDevice, ctx->stream));
    }
    // carry the shard size in the pad word
    *reinterpret_cast<uint64_t*>(&ctx->h_init[0].pad) = n;
    CK(cudaMemcpyAsync(&ctx->d_init->pad, &ctx->h_init[0].pad, sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
    cpsel_status st = gather_records(ctx->d_init, ctx->d_gather_init, ctx->h_gather_init, sizeof(DevInit));
    if (st != CPSEL_OK) return st;
    if (n == 0) slot = -1;
    scanned = n;
    const int Gn = G();
    n_rank.assign(Gn, 0);
    combined = cpsel_init_stats{};
    combined.vmin = INFINITY; combined.vmax = -INFINITY;
    n_global = 0;
    bool have_x0 = false;
    double S = 0.0;
    for (int q = 0; q < Gn; ++q) {
      const DevInit& r = ctx->h_gather_init[q];
      n_rank[q] = r.pad;
      n_global += r.pad;
      if (r.pad == 0) continue;
      if (r.vmin < combined.vmin) { combined.vmin = r.vmin; combined.cnt_min = r.cnt_min; }
      else if (r.vmin == combined.vmin) combined.cnt_min += r.cnt_min;
      if (r.vmax > combined.vmax) { combined.vmax = r.vmax; combined.cnt_max = r.cnt_max; }
      else if (r.vmax == combined.vmax) combined.cnt_max += r.cnt_max;
      combined.nonfinite += r.nonfinite;
      if (!have_x0) { combined.x0 = r.x0; have_x0 = true; }
      S += r.S + (double)r.pad * (r.x0 - combined.x0);
    }
    combined.S = S;
    cur_rank = n_rank;
    return CPSEL_OK;
  }
  // every rank's shard size (one tiny all-gather), before the buffers are sized
  cpsel_status exchange_sizes() {
    const int Gn = G();
    ctx->h_sizes[0] = n;
    CK(cudaMemcpyAsync(ctx->d_sizes, ctx->h_sizes, sizeof(unsigned long long), cudaMemcpyHostToDevice, ctx->stream));
    cpsel_status st = gather_records(ctx->d_sizes, ctx->d_sizes + 1, ctx->h_sizes + 1, sizeof(unsigned long long));
    if (st != CPSEL_OK) return st;
    n_rank.assign(ctx->h_sizes + 1, ctx->h_sizes + 1 + Gn);
    n_global = 0;
    for (uint64_t v : n_rank) n_global += v;
    return CPSEL_OK;
  }
  // R28: the pooled sample.  The S samples of the one-GPU cut kernel (R29) are apportioned to the
  // ranks in proportion to their current arrays (largest remainders, ties to the lower rank: the
  // same numbers on every rank), each rank gathers its share of evenly strided values into its
  // block of the pooled array, the blocks are all-gathered, and every rank runs the same cluster
  // select on the same bytes -> identical cuts t0 = {t_a, t_b, estimate} around global rank r.
  cpsel_status pooled_t0(bool on_x, const std::vector<uint64_t>& m_rank, uint64_t r) {
    const int Gn = G();
    const size_t es = elem_size(dt);
    uint64_t M = 0;
    for (uint64_t v : m_rank) M += v;
    const bool small = M <= (1ull << 26) && !on_x;
    // R40 for the init's cuts: the grid kernel's larger pooled sample (same apportioning).  Not for
    // loopback ranks: they share one GPU and run at once, and a cooperative grid per virtual rank
    // could spin on CTAs that cannot become resident while another rank's grid holds the SMs
    const bool grid = on_x && !small && sample_grid_on() && !ctx->comm.loop &&
                      M > 4 * pool_sample_size(dt, false) * sample_grid_x();
    const uint64_t S = pool_sample_size(dt, small) * (grid ? sample_grid_x() : 1);
    std::vector<uint64_t> s(Gn, 0);
    if (M <= S) {
      s = m_rank;
    } else {
      uint64_t tot = 0;
      std::vector<std::pair<unsigned long long, int>> rem;
      for (int q = 0; q < Gn; ++q) {
        const unsigned __int128 a = (unsigned __int128)S * m_rank[q];
        s[q] = (uint64_t)(a / M);
        tot += s[q];
        rem.emplace_back((unsigned long long)(a % M), q);
      }
      std::sort(rem.begin(), rem.end(), [](const auto& u, const auto& v) {
        return u.first != v.first ? u.first > v.first : u.second < v.second;
      });
      for (size_t i = 0; tot < S && i < rem.size(); ++i, ++tot) s[rem[i].second] += 1;
    }
    std::vector<size_t> bytes(Gn);
    uint64_t off = 0, total = 0;
    for (int q = 0; q < Gn; ++q) {
      bytes[q] = (size_t)s[q] * es;
      if (q < comm().rank) off += s[q];
      total += s[q];
    }
    char* mine = static_cast<char*>(ctx->d_pool) + off * es;
    const int W = seg_total_warps(dt, ctx->shape);
    const bool seg = !on_x && cur_seg;
    CK(launch_pool_gather(dt, on_x ? x : cur, on_x ? n : n_cur, seg ? cur_tab : nullptr, cur_side, W, s[comm().rank],
                          mine, ctx->stream));
    CM(comm().allgatherv(mine, ctx->d_pool, bytes.data(), ctx->stream));
    if (grid)  // the pooled array is the sample itself (m = ms: every value, in order)
      CK(launch_sample_grid(dt, ctx->d_pool, total, total, M, r, ctx->d_t0, static_cast<unsigned*>(ctx->d_pool1),
                            ctx->stream, !ctx->cfg.objective));
    else
      CK(launch_pool_pick(dt, ctx->d_pool, total, M, r, ctx->d_t0, ctx->stream, small, !ctx->cfg.objective));
    return CPSEL_OK;
  }
  // the init pass: with cuts (R23/R28) every rank runs the fused init at the pooled cuts and the
  // records are all-gathered and combined in rank order; else the plain init (gather_init)
  bool sharded_fused = false;
  uint64_t init_total = 0;
  std::vector<uint64_t> init_rank;
  cpsel_status init(cpsel_init_stats* o, uint64_t k) override {
    const bool cut = ctx->cfg.init_cut != 0 && n_global > 2 && R > 0;
    sharded_fused = false;
    if (!cut) {
      cpsel_status st = gather_init();
      if (st != CPSEL_OK) return st;
      *o = combined;
      return CPSEL_OK;
    }
    const int Gn = G();
    cpsel_status st = pooled_t0(true, n_rank, k);
    if (st != CPSEL_OK) return st;
    if (n > 0) {
      // launches: the pooled sample (gather + cluster select) and the init; the record is checked
      // after the all-gather (every rank takes the same fallback decision)
      st = run_init(false, k, true, /*presampled=*/true);
      if (st != CPSEL_OK) return st;
      launches = 3;
    } else {
      launches = 1;
      slot = -1;
      DevInit e{};
      e.vmin = INFINITY; e.vmax = -INFINITY;
      e.has_cut = 11;  // an empty shard: nothing below, inside or above the cuts
      *ctx->h_init = e;
      CK(cudaMemcpyAsync(ctx->d_init, ctx->h_init, sizeof(DevInit), cudaMemcpyHostToDevice, ctx->stream));
      // every warp of the (empty) segmented array has an empty run
      CK(cudaMemsetAsync(ctx->d_st[0], 0, seg_total_warps(dt, ctx->shape) * sizeof(SegEntry), ctx->stream));
      init_seg_done = true;
      init_n_in = 0;
    }
    st = gather_records(ctx->d_init, ctx->d_gather_init, ctx->h_gather_init, sizeof(DevInit));
    if (st != CPSEL_OK) return st;
    scanned = n;
    cpsel_init_stats c{};
    c.vmin = INFINITY; c.vmax = -INFINITY;
    c.has_cut = 11;  // two cuts, the interior compacted, no sums, no #min/#max (R27)
    init_rank.assign(Gn, 0);
    init_total = 0;
    bool all_fused = true, have_cuts = false;
    for (int q = 0; q < Gn; ++q) {
      const DevInit& r = ctx->h_gather_init[q];
      if (n_rank[q] == 0) continue;
      if (!have_cuts) {  // the cuts: identical on every rank (same pooled bytes, same select)
        c.t_lo = r.t_lo; c.t_hi = r.t_hi; c.t_est = r.t_est;
        have_cuts = true;
      }
      c.vmin = std::min(c.vmin, r.vmin);
      c.vmax = std::max(c.vmax, r.vmax);
      c.nonfinite += r.nonfinite;
      c.c_le_lo += r.c_le_lo;
      c.c_lt_hi += r.c_lt_hi;
      if ((r.has_cut & 11) != 11 || suspicious(r, true, dt)) all_fused = false;
      init_rank[q] = r.pad;
      init_total += r.pad;
    }
    if (!all_fused || !std::isfinite(c.vmin) || !std::isfinite(c.vmax)) {
      // a rank saw NaN/Inf (or could not bracket from the extremes' neighbours): the plain path
      init_seg_done = false;
      cpsel_status s2 = gather_init();
      if (s2 != CPSEL_OK) return s2;
      *o = combined;
      return CPSEL_OK;
    }
    sharded_fused = true;
    init_seg_done = true;
    init_n_in = init_rank[comm().rank];
    cur_rank = n_rank;
    *o = c;
    return CPSEL_OK;
  }
  bool init_compacted() const override { return sharded_fused; }
  uint64_t init_written() const override { return init_total; }
  cpsel_status adopt_init() override {
    cpsel_status st = GpuBackend::adopt_init();
    cur_rank = init_rank;
    return st;
  }
  // R26 + R28: the cut pass with cuts pooled across ranks; tuples all-gathered, combined in rank order
  bool has_cut_pass() const override { return R > 0; }
  cpsel_status cut_pass(uint64_t r, bool /*dense*/, CutResult* o) override {
    const int Gn = G();
    CK(tic());
    cpsel_status st = pooled_t0(false, cur_rank, r);
    if (st != CPSEL_OK) return st;
    CK(toc());
    sample_slot = slot;
    SegArgs a{};
    a.x = cur; a.n = n_cur;
    a.seg_in = cur_seg ? cur_tab : nullptr;
    a.side_in = cur_side;
    a.cuts = ctx->d_t0;
    a.dense_out = 0;  // segmented (warp-private) copy; select() packs it
    tgt = (cur_sbuf == 0) ? 1 : 0;
    a.out = ctx->d_sb[tgt];
    a.R = R;
    a.seg_out = static_cast<SegEntry*>(ctx->d_st[tgt]);
    a.cursors = ctx->d_cursors;
    a.partials = ctx->d_partials; a.ticket = ctx->d_ticket;
    a.out_tuple = ctx->d_pass;
    CK(tic());
    CK(launch_cut_pass(dt, a, ctx->shape, ctx->stream));  // also for an empty array: run tables
    CK(toc());
    launches = 3;
    scanned = n_cur;
    st = gather_records(ctx->d_pass, ctx->d_gather, ctx->h_gather, sizeof(DevPass));
    if (st != CPSEL_OK) return st;
    const DevPass& me = ctx->h_gather[comm().rank];
    o->ta = me.pred; o->tb = me.succ; o->t_est = me.L_lo;  // the cuts (identical on every rank)
    o->le_a = 0; o->inner = 0;
    o->overflow = false;
    zlo_rank.assign(Gn, 0);
    zhi_rank.assign(Gn, 0);
    for (int q = 0; q < Gn; ++q) {
      const DevPass& rr = ctx->h_gather[q];
      o->le_a += rr.c_lt;
      o->inner += rr.z_lo;
      o->overflow |= rr.c_eq != 0;
      zlo_rank[q] = rr.z_lo;
    }
    last_dense = false;
    zlo = me.z_lo;
    zhi = 0;
    return CPSEL_OK;
  }
  cpsel_status pass(double t, double yL, double yR, bool compact, bool dense, cpsel_pass_stats* o, uint64_t* z_lo,
                    uint64_t* z_hi) override {
    const int Gn = G();
    if (n_cur > 0 || (compact && cur_seg)) {
      // (a segmented current array is processed even when empty so every warp writes its run table)
      cpsel_status st = launch_local_pass(t, yL, yR, compact, dense);
      if (st != CPSEL_OK) return st;
    } else {
      launches = 0;
      scanned = 0;
      slot = -1;
      if (compact) {
        tgt = dense ? ((cur_dbuf == 0) ? 1 : 0) : ((cur_sbuf == 0) ? 1 : 0);
        last_dense = dense;
        if (!dense) CK(cudaMemsetAsync(ctx->d_st[tgt], 0, seg_total_warps(dt, ctx->shape) * sizeof(SegEntry), ctx->stream));
      }
      DevPass e{};
      e.pred = -INFINITY; e.succ = INFINITY;
      *ctx->h_pass = e;
      CK(cudaMemcpyAsync(ctx->d_pass, ctx->h_pass, sizeof(DevPass), cudaMemcpyHostToDevice, ctx->stream));
    }
    cpsel_status st = gather_records(ctx->d_pass, ctx->d_gather, ctx->h_gather, sizeof(DevPass));
    if (st != CPSEL_OK) return st;
    // fixed rank-order combine: identical bytes on every rank (R17)
    cpsel_pass_stats s{};
    s.pred = -INFINITY; s.succ = INFINITY;
    uint64_t tlo = 0, thi = 0;
    if (compact) {
      zlo_rank.assign(Gn, 0);
      zhi_rank.assign(Gn, 0);
    }
    for (int q = 0; q < Gn; ++q) {
      const DevPass& r = ctx->h_gather[q];
      s.c_lt += r.c_lt; s.c_eq += r.c_eq; s.c_lo += r.c_lo; s.c_hi += r.c_hi;
      s.L_lo += r.L_lo; s.L_hi += r.L_hi; s.P += r.P; s.N += r.N;
      s.pred = std::max(s.pred, r.pred); s.succ = std::min(s.succ, r.succ);
      if (compact) { zlo_rank[q] = r.z_lo; zhi_rank[q] = r.z_hi; }
      tlo += r.z_lo; thi += r.z_hi;
    }
    *o = s;
    if (compact) {
      zlo = ctx->h_gather[comm().rank].z_lo;
      zhi = ctx->h_gather[comm().rank].z_hi;
    }
    *z_lo = tlo; *z_hi = thi;
    return CPSEL_OK;
  }
  cpsel_status adopt(int side) override {
    cur_rank = side == 0 ? zlo_rank : zhi_rank;
    return GpuBackend::adopt(side);
  }
  // the exact finish (north_star "the final bracket contents are allgathered"): every
  // rank's kept part (packed contiguously if it is segmented) all-gathered in rank order (an
  // all-gather-v), then the same radix select on every rank.  One rank: the all-gather is the
  // identity, the one-GPU select reads the kept part where it is.
  cpsel_status select(int side, uint64_t r, double* out) override {
    if (G() == 1) return GpuBackend::select(side, r, out);
    const int Gn = G();
    const size_t es = elem_size(dt);
    const std::vector<uint64_t>& cnt = side == 2 ? cur_rank : side == 0 ? zlo_rank : zhi_rank;
    uint64_t total = 0, off = 0;
    std::vector<size_t> bytes(Gn);
    for (int q = 0; q < Gn; ++q) {
      if (q < comm().rank) off += cnt[q];
      total += cnt[q];
      bytes[q] = (size_t)cnt[q] * es;
    }
    cpsel_status st = ensure(ctx, &ctx->d_zall, &ctx->zall_bytes, (size_t)total * es);
    if (st != CPSEL_OK) return st;
    char* mine = static_cast<char*>(ctx->d_zall) + off * es;
    const void* send = mine;
    const uint64_t cm = cnt[comm().rank];
    const int W = seg_total_warps(dt, ctx->shape);
    if (side == 2 ? cur_seg : !last_dense) {  // segmented: pack into this rank's block
      const void* base = side == 2 ? cur : ctx->d_sb[tgt];
      const SegEntry* tab = side == 2 ? cur_tab : static_cast<const SegEntry*>(ctx->d_st[tgt]);
      if (cm) CK(launch_seg_pack(dt, base, tab, side == 2 ? cur_side : side, W, mine, ctx->stream));
    } else {
      send = side == 2 ? cur : half_ptr(side);
    }
    CM(comm().allgatherv(send, ctx->d_zall, bytes.data(), ctx->stream));
    st = select_on(ctx->d_zall, total, r, out);
    launches += 1;
    return st;
  }
#undef CM
};

// ------------------------------------------------------------------------ host callbacks
struct HostBackend : Backend {
  const cpsel_host_backend* be;
  std::string msg;
  explicit HostBackend(const cpsel_host_backend* b) : be(b) {}
  std::string message() const override { return msg; }
  cpsel_status init(cpsel_init_stats* o, uint64_t) override {
    if (be->init(be->user, o) != 0) { msg = "init callback failed"; return CPSEL_EINTERNAL; }
    return CPSEL_OK;
  }
  cpsel_status pass(double t, double yL, double yR, bool compact, bool /*dense*/, cpsel_pass_stats* o,
                    uint64_t* z_lo, uint64_t* z_hi) override {
    if (be->pass(be->user, t, yL, yR, compact ? 1 : 0, o) != 0) { msg = "pass callback failed"; return CPSEL_EINTERNAL; }
    // the callback reports c_lo/c_hi over its current array; those are the compacted halves
    *z_lo = compact ? o->c_lo : 0;
    *z_hi = compact ? o->c_hi : 0;
    return CPSEL_OK;
  }
  cpsel_status adopt(int side) override {
    if (be->adopt(be->user, side) != 0) { msg = "adopt callback failed"; return CPSEL_EINTERNAL; }
    return CPSEL_OK;
  }
  cpsel_status select(int side, uint64_t r, double* out) override {
    if (be->select(be->user, side, r, out) != 0) { msg = "select callback failed"; return CPSEL_EINTERNAL; }
    return CPSEL_OK;
  }
  bool has_cut_pass() const override { return be->cut != nullptr; }
  cpsel_status cut_pass(uint64_t r, bool, CutResult* o) override {
    cpsel_cut_stats c{};
    if (be->cut(be->user, r, &c) != 0) { msg = "cut callback failed"; return CPSEL_EINTERNAL; }
    o->ta = c.t_a; o->tb = c.t_b; o->t_est = c.t_est; o->le_a = c.le_a; o->inner = c.inner;
    o->overflow = false;
    return CPSEL_OK;
  }
};

// brackets up to this size are compacted densely (4 x 2^20: independent of a larger select cap — the
// radix select reads segmented arrays as well, and the fused init needs the segmented buffers)
uint64_t dense_threshold(uint64_t select_cap) { return std::max<uint64_t>(4 * std::min<uint64_t>(select_cap, 1ull << 20), 1ull << 20); }

// ============================================================================================
// The cutting-plane driver (Algorithm 1 + hybrid finish), shared by all back ends.
//
// Bracket invariant: c_le(yL) < k <= c_lt(yR), i.e. yL < x_(k) < yR, interior m = c_lt(yR)-c_le(yL).
// Cuts: F_k's right derivative at yL, left derivative at yR (R4, tightest cuts).  Kelley's step
// 1.1 with those cuts is exactly the mean of the open-bracket interior (App. A / pinned in
// tests/test_oracle_pins.py::test_appendix_A_kelley_step_is_interior_mean_exact_rationals);
// the driver evaluates it from bracket-local sums (no cancellation, R11).
//
// Compaction (P:L196 copy_if, R8): the first pass whose interior m <= z_cap copies both halves
// of the bracket (split at t) out; the kept half becomes the array of all later passes (every
// later pass compacts again), until the kept half has <= select_cap elements, which are then
// selected exactly by radix select (P:L196 'sort z', R21).
cpsel_status drive(Backend& be, uint64_t n, int dt, uint64_t k, const cpsel_config& cfg, uint64_t z_cap,
                   uint64_t select_cap, double* value, cpsel_info* info, std::vector<cpsel_trace_row>* trace) {
  const uint64_t dense_cap = dense_threshold(select_cap);
  const auto t0 = std::chrono::steady_clock::now();
  const size_t es = elem_size(dt);
  cpsel_info inf{};
  if (trace) trace->clear();
  // record_timing: timing slots of the steps (init, each pass with its trace row, select), resolved
  // once the selection is over
  int init_slot = -1, select_slot = -1;
  std::vector<std::pair<int, long>> pass_slots;
  std::vector<int> sample_slots;
  auto done = [&](double v, uint32_t reason) {
    *value = canonical_zero(v);
    inf.exit_reason = reason;
    inf.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (cfg.record_timing == 1) {
      inf.kernel_ms_init = be.slot_ms(init_slot);
      inf.kernel_ms_select = be.slot_ms(select_slot);
      inf.kernel_ms_sample = 0.0;
      for (int ss : sample_slots) inf.kernel_ms_sample += be.slot_ms(ss);
      inf.kernel_ms_passes = 0.0;
      for (const auto& ps : pass_slots) {
        const double ms = be.slot_ms(ps.first);
        inf.kernel_ms_passes += ms;
        if (trace && ps.second >= 0 && ps.second < (long)trace->size()) (*trace)[ps.second].kernel_ms = ms;
      }
    }
    if (info) *info = inf;
    return CPSEL_OK;
  };
  auto do_select = [&](int side, uint64_t r, double* v) {
    cpsel_status s2 = be.select(side, r, v);
    if (s2 != CPSEL_OK) return s2;
    inf.launches += be.launches;
    select_slot = be.slot;
    inf.z_count = be.scanned;
    inf.bytes_moved += (uint64_t)(dt == kF32 ? 3 : 6) * be.scanned * es;
    return CPSEL_OK;
  };
  // step 0: one reduction -> x_(1), x_(n), sum
  cpsel_init_stats rec{};
  cpsel_status st = be.init(&rec, k);
  if (st != CPSEL_OK) return st;
  inf.passes = 1;
  inf.launches += be.launches;
  init_slot = be.slot;
  if (be.sample_slot >= 0) sample_slots.push_back(be.sample_slot);
  inf.bytes_moved = be.scanned * es;
  if (rec.nonfinite) return CPSEL_ENONFINITE;
  const bool f32 = dt == kF32;
  auto next_up = [&](double v) { return f32 ? (double)std::nextafterf((float)v, INFINITY) : std::nextafter(v, INFINITY); };
  auto next_dn = [&](double v) { return f32 ? (double)std::nextafterf((float)v, -INFINITY) : std::nextafter(v, -INFINITY); };
  // R27: a fused init pass does not count the multiplicities of min and max; the bracket then
  // starts at their outer neighbours, where the counts are known: #x<=prev(min) = 0, #x<next(max) = n
  const bool ext_counts = (rec.has_cut & 8) == 0;
  if (ext_counts && k <= rec.cnt_min) return done(rec.vmin, 0);
  if (ext_counts && k > n - rec.cnt_max) return done(rec.vmax, 1);
  if (n <= cfg.direct_threshold && !cfg.force_cp) {
    double v;
    st = do_select(2, k, &v);
    if (st != CPSEL_OK) return st;
    return done(v, 6);
  }
  double yL = ext_counts ? rec.vmin : next_dn(rec.vmin), yR = ext_counts ? rec.vmax : next_up(rec.vmax);
  uint64_t c_le_L = ext_counts ? rec.cnt_min : 0, c_lt_R = ext_counts ? n - rec.cnt_max : n;
  long double N_L = 0.0L, P_R = 0.0L;  // N(yL) = sum (yL-x)^+ = 0 at (or below) the min; P(yR) = 0 at (or above) the max
  uint64_t m = c_lt_R - c_le_L;       // >= 1
  uint64_t D_lo = 0;                   // elements of x below the current array
  bool on_z = false;                   // the current array is a compacted bracket
  // first iterate: mean of the interior (App. A) from the shifted sum (replaced below when the init
  // pass also evaluated the two extra cuts, R23)
  double t = rec.x0 + (rec.S - (double)rec.cnt_min * (rec.vmin - rec.x0) - (double)rec.cnt_max * (rec.vmax - rec.x0)) /
                          (double)m;
  int slow = 0;
  bool bisect = false;
  BrentRoot brent;  // driver 2
  bool brent_on = false;
  BrentMin bmin;    // driver 3
  bool bmin_on = false;
  const long double wP = (long double)k - 0.5L, wN = (long double)n - (long double)k + 0.5L;
  constexpr uint64_t kUnknown = ~0ull;
  bool exact = true;  // the current (compacted) array holds exactly the bracket interior
  bool cuts_stalled = false;  // R26 cut passes stopped making progress
  bool free_step = false;     // the next pass's iterate was not a Kelley step (progress not judged)
  // R23: the init pass's two extra cuts t_lo <= t_hi (sample quantiles bracketing rank k) — two more
  // cuts of the cutting-plane model, evaluated in the same read of x as the init reduction.  N and P
  // at both cuts follow from the pass's sums: N(t_lo) = N_lo, P(t_hi) = P_hi,
  // P(t_lo) = I + P_hi + #{x>=t_hi}(t_hi-t_lo), N(t_hi) = N_lo + #{x<t_hi}(t_hi-t_lo) - I.
  if (rec.has_cut) {
    const long double tl = rec.t_lo, th = rec.t_hi, dlh = th - tl;
    // R25: without the init pass's positive-part sums, F_k (and so every later row's F) is unknown;
    // the iterate never needs it: the usual bracket ]t_lo, t_hi[ starts from its interior mean
    // t_lo + I/m, any other from the midpoint
    const bool sums = (rec.has_cut & 4) != 0;
    const long double N_tl = sums ? (long double)rec.N_lo : (long double)NAN;
    const long double P_th = sums ? (long double)rec.P_hi : (long double)NAN;
    t = NAN;
    const long double P_tl = (long double)rec.I_in + P_th + (long double)(n - rec.c_lt_hi) * dlh;  // R24
    const long double N_th = N_tl + (long double)rec.c_lt_hi * dlh - (long double)rec.I_in;
    auto row_of = [&](double tt, uint64_t clt, uint64_t ceq, long double Nt, long double Pt) {
      cpsel_trace_row r{};
      r.t = tt; r.F = (double)(wP * Pt + wN * Nt); r.c_lt = clt; r.c_eq = ceq; r.kind = 2;
      return r;
    };
    bool settled = false;  // the target is below t_lo: t_hi carries no further information
    // R24: the pass counts #x<=t_lo and #x<t_hi only — what the bracket update needs when the
    // target lies between the cuts (the usual case).  A cut on the far side of the target moves to
    // the adjacent float, where the missing count is the known one: #x<next(t_lo) = #x<=t_lo,
    // #x<=prev(t_hi) = #x<t_hi (no element lies strictly between a float and its neighbour).
    if (rec.t_lo > yL && rec.t_lo < yR) {
      const uint64_t c_le = rec.c_le_lo;
      cpsel_trace_row row = row_of(rec.t_lo, kUnknown, kUnknown, N_tl, P_tl);
      if (c_le < k) {  // y_L <- t_lo
        yL = rec.t_lo; N_L = N_tl; c_le_L = c_le; m = c_lt_R - c_le;
        const long double L_hi = P_tl - (long double)(n - c_lt_R) * ((long double)yR - tl);  // P_R = 0
        t = rec.t_lo + (double)(L_hi / (long double)m);
      } else {  // y_R <- next(t_lo): interior ]min, next(t_lo)[
        const double yr = next_up(rec.t_lo);
        const long double N_r = N_tl + (long double)c_le * ((long double)yr - tl);
        const long double L_lo = N_r - (long double)c_le_L * ((long double)yr - (long double)yL);  // N_L = 0
        yR = yr; P_R = P_tl - (long double)(n - c_le) * ((long double)yr - tl); c_lt_R = c_le; m = c_le - c_le_L;
        t = yr - (double)(L_lo / (long double)m);
        settled = true;
      }
      row.interior = m;
      if (trace && cfg.record_trace) trace->push_back(row);
    }
    if (!settled && rec.t_hi > yL && rec.t_hi < yR) {
      const uint64_t c_lt = rec.c_lt_hi;
      cpsel_trace_row row = row_of(rec.t_hi, c_lt, kUnknown, N_th, P_th);
      if (c_lt >= k) {  // y_R <- t_hi: interior ]y_L, t_hi[
        // sum_{y_L<x<t_hi} (x - y_L): the pass's I when y_L = t_lo, else via N (App. A identity)
        const long double L_lo = (yL == rec.t_lo) ? (long double)(c_lt - c_le_L) * dlh - (long double)rec.I_in
                                                  : N_th - N_L - (long double)c_le_L * (th - (long double)yL);
        yR = rec.t_hi; P_R = P_th; c_lt_R = c_lt; m = c_lt - c_le_L;
        t = rec.t_hi - (double)(L_lo / (long double)m);
      } else {  // y_L <- prev(t_hi): interior ]prev(t_hi), max[
        const double yl = next_dn(rec.t_hi);
        const long double P_l = P_th + (long double)(n - c_lt) * (th - (long double)yl);
        const long double L_hi = P_l - (long double)(n - c_lt_R) * ((long double)yR - (long double)yl);  // P_R = 0
        yL = yl; N_L = N_th - (long double)c_lt * (th - (long double)yl); c_le_L = c_lt; m = c_lt_R - c_lt;
        t = yl + (double)(L_hi / (long double)m);
      }
      row.interior = m;
      if (trace && cfg.record_trace) trace->push_back(row);
    }
    // without the sums the interior sum I is not kept either: start from the sample's estimate
    if (!sums) t = (rec.t_est > yL && rec.t_est < yR) ? rec.t_est : (double)NAN;
    free_step = !sums;
    if (!std::isfinite(t)) t = 0.5 * yL + 0.5 * yR;
    // the init pass already copied out ]t_lo, t_hi[: if that is the bracket, continue on it (a cut
    // outside the bracket with no element between it and the bracket end — the open cut of an
    // extreme rank — copies the same set)
    const bool lo_ok = yL == rec.t_lo || (rec.t_lo < yL && rec.c_le_lo == c_le_L);
    const bool hi_ok = yR == rec.t_hi || (rec.t_hi > yR && rec.c_lt_hi == c_lt_R);
    if (be.init_compacted() && lo_ok && hi_ok) {
      if (m != be.init_written()) {
        if (info) *info = inf;
        return CPSEL_EINTERNAL;
      }
      st = be.adopt_init();
      if (st != CPSEL_OK) return st;
      inf.bytes_moved += m * es;
      inf.init_written = m;
      D_lo = c_le_L;
      on_z = true;
      if (m <= select_cap && be.kept_dense()) {  // the init's copy is already small: select in it
        double v;
        st = do_select(2, k - c_le_L, &v);
        if (st != CPSEL_OK) return st;
        return done(v, 5);
      }
    }
  }
  for (uint32_t it = 1;; ++it) {
    if (it > cfg.max_iters) {
      if (info) *info = inf;
      return CPSEL_EINTERNAL;
    }
    // §8f-3: once no R26 cut pass can follow (pass_cuts off, objective on, or the cuts stalled), the
    // remaining Kelley passes and the exact finish run on the device as one graph launch; the step
    // kernel there is this loop's Kelley step (same iterates, same decisions, same trace rows)
    if (cfg.device_loop && cfg.driver == 0 && be.has_device_loop() &&
        (!cfg.pass_cuts || cfg.objective || !be.has_cut_pass() || cuts_stalled)) {
      Backend::LoopIn li{};
      li.yL = yL; li.yR = yR; li.t = t; li.N_L = (double)N_L; li.P_R = (double)P_R;
      li.c_le_L = c_le_L; li.c_lt_R = c_lt_R; li.m = m; li.D_lo = D_lo; li.it = it - 1;
      li.k = k; li.n = n; li.z_cap = z_cap; li.select_cap = select_cap; li.dense_cap = dense_cap;
      li.max_iters = cfg.max_iters;
      li.on_z = on_z; li.exact = exact; li.bisect = bisect; li.slow = slow; li.free_step = free_step;
      li.record = (trace && cfg.record_trace) ? 1 : 0;
      li.wP = (double)wP; li.wN = (double)wN;
      Backend::LoopOut lo;
      st = be.device_loop(li, &lo);
      if (st != CPSEL_OK) return st;
      inf.passes += lo.passes;
      inf.cp_iters += lo.cp_iters;
      inf.fallback_steps += lo.fallback;
      inf.launches += lo.launches;
      inf.bytes_moved += lo.bytes_moved;
      if (lo.exit_reason == 5) inf.z_count = lo.z_count;
      double rows_ms = 0.0;
      for (const auto& r : lo.rows) rows_ms += r.kernel_ms;
      if (trace && cfg.record_trace) trace->insert(trace->end(), lo.rows.begin(), lo.rows.end());
      if (lo.error) {
        if (info) *info = inf;
        return CPSEL_EINTERNAL;
      }
      done(lo.value, lo.exit_reason);
      if (cfg.record_timing == 1 && info) {  // the loop's passes (device timestamps) and the rest of it
        info->kernel_ms_passes += rows_ms;
        info->kernel_ms_select += std::max(0.0, lo.loop_ms - rows_ms);
      }
      return CPSEL_OK;
    }
    // R26 (multi-point step): a compacted current array that is exactly the bracket
    // interior and too large for the exact selection is cut at two sample quantiles of its own
    // around the local target rank; the copy keeps only ]t_a, t_b[ (~10% of the array) instead of
    // both halves of a Kelley split.  Not with objective=1 (F at the sample cuts would need two
    // more sums per element).
    if (cfg.pass_cuts && !cfg.objective && cfg.driver == 0 && on_z && exact && !bisect && !cuts_stalled &&
        m > select_cap && be.has_cut_pass()) {
      const uint64_t m_before = m;
      Backend::CutResult cr{};
      // dense output (selectable right away) when the expected copy (~2-4% of m) surely fits; a
      // copy that overflows the dense buffer is dropped and the pass still counts exactly
      st = be.cut_pass(k - c_le_L, m <= 8 * dense_cap, &cr);
      if (st != CPSEL_OK) return st;
      inf.launches += be.launches;
      inf.passes++;
      inf.cp_iters++;
      inf.bytes_moved += be.scanned * es + cr.inner * es;
      pass_slots.emplace_back(be.slot, (trace && cfg.record_trace) ? (long)trace->size() : -1L);
      if (be.sample_slot >= 0) sample_slots.push_back(be.sample_slot);
      const uint64_t le_a = c_le_L + cr.le_a, lt_b = le_a + cr.inner;
      cpsel_trace_row row{};
      row.t = cr.ta;
      row.F = NAN;
      row.c_lt = kUnknown; row.c_eq = kUnknown;  // #x<=t_a = le_a and #x<t_b = lt_b, see below
      row.kind = 3;
      row.compacted = 1;
      row.scanned = be.scanned;
      row.written = cr.inner;
      N_L = P_R = NAN;  // F is not tracked through sample cuts
      if (le_a < k && k <= lt_b && cr.ta < cr.tb && cr.overflow) {
        // the target is between the cuts but the copy was not kept: the bracket still shrinks
        yL = cr.ta; yR = cr.tb; c_le_L = le_a; c_lt_R = lt_b; m = cr.inner;
        row.interior = m;
        if (trace && cfg.record_trace) trace->push_back(row);
        exact = false;
        be.set_inexact();
        cuts_stalled = true;
        t = (cr.t_est > yL && cr.t_est < yR) ? cr.t_est : 0.5 * yL + 0.5 * yR;
        free_step = true;
        continue;
      }
      if (le_a < k && k <= lt_b && cr.ta < cr.tb) {  // the usual case: continue on the copy of ]t_a, t_b[
        yL = cr.ta; yR = cr.tb; c_le_L = le_a; c_lt_R = lt_b; m = cr.inner;
        // a sample that cannot split the bracket (e.g. one repeated value inside it) hands over to
        // Kelley passes for the rest of the selection
        if (m > m_before / 2) cuts_stalled = true;
        row.interior = m;
        if (trace && cfg.record_trace) trace->push_back(row);
        st = be.adopt(0);
        if (st != CPSEL_OK) return st;
        D_lo = c_le_L;
        exact = true;
        if (m <= select_cap && be.kept_dense()) {
          double v;
          st = do_select(0, k - c_le_L, &v);
          if (st != CPSEL_OK) return st;
          return done(v, 5);
        }
        // next iterate (if any pass still needs one): the sample's estimate of x_(k)
        t = (cr.t_est > cr.ta && cr.t_est < cr.tb) ? cr.t_est : 0.5 * cr.ta + 0.5 * cr.tb;
        slow = 0;
        free_step = true;
        continue;
      }
      // the target is outside the sample cuts: the bracket moves to the adjacent float of the cut
      // (R24); the current array is kept and now holds elements outside the bracket.  (With
      // t_a == t_b — duplicates in the sample — #x<t_b is not le_a + inner: one cut at t_a.)
      if (k <= le_a) {
        yR = next_up(cr.ta); c_lt_R = le_a; m = le_a - c_le_L;
      } else if (cr.ta == cr.tb) {
        yL = cr.ta; c_le_L = le_a; m = c_lt_R - le_a;
      } else {
        yL = next_dn(cr.tb); c_le_L = lt_b; m = c_lt_R - lt_b;
      }
      row.interior = m;
      if (trace && cfg.record_trace) trace->push_back(row);
      exact = false;
      be.set_inexact();
      cuts_stalled = true;  // the rest of this selection runs Kelley passes
      // next iterate: the sample's estimate of x_(k) if it lies inside (it is typically the value
      // a one-sided miss came from, e.g. a repeated value), else the midpoint; not a Kelley step,
      // so it does not count towards the progress safeguard
      t = (cr.t_est > yL && cr.t_est < yR) ? cr.t_est : 0.5 * yL + 0.5 * yR;
      free_step = true;
      continue;
    }
    uint32_t kind = 0;
    if (cfg.driver == 1) {  // the bisection comparison driver: the bracket's value midpoint
      t = 0.5 * yL + 0.5 * yR;
      kind = 4;
    } else if (cfg.driver == 2) {  // Brent's root finder: its interpolation's next point
      if (!brent_on) {
        brent.init(yL, 2.0 * (double)c_le_L - 2.0 * (double)k + 1.0, yR, 2.0 * (double)c_lt_R - 2.0 * (double)k + 1.0);
        brent_on = true;
      }
      t = brent.propose();
      kind = 5;
    } else if (cfg.driver == 3 && !bisect) {  // Brent's minimisation: its next point
      if (!bmin_on) {
        bmin.init(yL, yR);
        bmin_on = true;
      }
      double u;
      if (bmin.propose(&u)) {
        t = u;
        kind = 6;
      } else {  // NR's convergence test: ordered-key bisection of the exact bracket finishes it
        bisect = true;
        t = key_mid(yL, yR, dt);
        kind = 1;
        inf.fallback_steps++;
      }
    } else if (bisect) {
      t = key_mid(yL, yR, dt);
      kind = 1;
      inf.fallback_steps++;
    }
    const double tq = snap(t, yL, yR, dt);
    if (!(tq > yL && tq < yR)) {
      if (info) *info = inf;
      return CPSEL_EINTERNAL;  // impossible while m >= 1
    }
    const bool compact = on_z || m <= z_cap;
    const bool dense = m <= dense_cap;  // small brackets are compacted contiguously (selectable)
    cpsel_pass_stats s{};
    uint64_t zl = 0, zh = 0;
    st = be.pass(tq, yL, yR, compact, dense, &s, &zl, &zh);
    if (st != CPSEL_OK) return st;
    inf.launches += be.launches;
    // the pass's trace row (if recorded) is the next one pushed
    pass_slots.emplace_back(be.slot, (trace && cfg.record_trace) ? (long)trace->size() : -1L);
    inf.passes++;
    inf.cp_iters++;
    inf.bytes_moved += be.scanned * es + (compact ? (zl + zh) * es : 0);
    // global counts at t; a compaction pass carries no counters: they follow exactly from the
    // compaction totals (#lo = #{yL<x<t}, #hi = #{t<x<yR}, and every x == t is interior)
    const uint64_t c_lt = compact ? c_le_L + zl : D_lo + s.c_lt;
    const uint64_t c_le = compact ? c_lt + (m - zl - zh) : c_lt + s.c_eq;
    // F_k(t) from positive terms only (App. A identities; Eq. 2 with paper-k = n-k+1, R2)
    const long double N_t = N_L + (long double)c_le_L * ((long double)tq - yL) + s.L_lo;
    const long double P_t = P_R + (long double)(n - c_lt_R) * ((long double)yR - tq) + s.L_hi;
    cpsel_trace_row row{};
    row.t = tq;
    row.F = (double)(wP * P_t + wN * N_t);
    row.c_lt = c_lt;
    row.c_eq = c_le - c_lt;
    row.kind = kind;
    row.compacted = compact ? 1 : 0;
    row.kernel_ms = 0.0;  // filled from the timing slot when the selection ends
    row.scanned = be.scanned;
    row.written = compact ? zl + zh : 0;
    if (cfg.driver == 2) brent.accept(tq, (double)c_lt + (double)c_le - 2.0 * (double)k + 1.0);
    if (cfg.driver == 3 && !std::isfinite(row.F)) {  // F untracked (init cuts without their sums, R25)
      if (info) *info = inf;
      return CPSEL_EINVAL;
    }
    // step 1.3: 0 in dF(t) <=> c_lt < k <= c_le -> t = x_(k)
    if (c_lt < k && k <= c_le) {
      if (trace && cfg.record_trace) trace->push_back(row);
      return done(tq, 2);
    }
    const uint64_t m_old = m;
    int side;
    if (c_le < k) {  // dF(t) < 0: y_L <- t (sign per R1)
      const uint64_t c_hi = c_lt_R - c_le;
      if (c_le + 1 == k && std::isfinite(s.succ)) {  // x_(k) = successor of t (P:L192 footnote, mirrored)
        row.interior = 0;
        if (trace && cfg.record_trace) trace->push_back(row);
        return done(s.succ, 4);
      }
      if (compact && zh != c_hi) {
        if (info) *info = inf;
        return CPSEL_EINTERNAL;
      }
      yL = tq; N_L = N_t; c_le_L = c_le; m = c_hi;
      t = tq + s.L_hi / (double)c_hi;  // mean of ]t, yR[ (App. A)
      side = 1;
    } else {  // c_lt >= k: y_R <- t
      const uint64_t c_lo = c_lt - c_le_L;
      if (c_lt == k && std::isfinite(s.pred)) {  // x_(k) = largest x < t (P:L192 footnote)
        row.interior = 0;
        if (trace && cfg.record_trace) trace->push_back(row);
        return done(s.pred, 3);
      }
      if (compact && zl != c_lo) {
        if (info) *info = inf;
        return CPSEL_EINTERNAL;
      }
      yR = tq; P_R = P_t; c_lt_R = c_lt; m = c_lo;
      t = tq - s.L_lo / (double)c_lo;  // mean of ]yL, t[ (App. A)
      side = 0;
    }
    row.interior = m;
    if (trace && cfg.record_trace) trace->push_back(row);
    if (cfg.driver == 3 && kind == 6) bmin.accept(tq, row.F, yL, yR);
    if (compact) {
      if (m <= select_cap && be.kept_dense()) {  // hybrid finish: exact selection in the kept half
        double v;
        st = do_select(side, k - c_le_L, &v);
        if (st != CPSEL_OK) return st;
        return done(v, 5);
      }
      st = be.adopt(side);  // continue the cutting plane on the kept half only
      if (st != CPSEL_OK) return st;
      D_lo = c_le_L;
      on_z = true;
      exact = true;
    }
    // progress safeguard (R7): two consecutive steps keeping > 7/8 of the interior switch to
    // ordered-key bisection until progress resumes (bounds the pass count on any input); not for
    // the bisection driver, whose slow progress on wide data is what it demonstrates
    if (cfg.driver != 0) {
      free_step = false;
    } else if (free_step) {
      free_step = false;
    } else if (m > m_old - m_old / 8) {
      if (++slow >= 2) bisect = true;
    } else {
      slow = 0;
      bisect = false;
    }
  }
}

uint64_t auto_z_cap(uint64_t n, const cpsel_config& cfg) {
  if (cfg.z_cap) return std::min<uint64_t>(cfg.z_cap, n);
  return std::max<uint64_t>(n / 8 * 5, 1);  // compact once the bracket holds <= 5/8 of x
}

uint64_t auto_select_cap(const cpsel_config& cfg) { return cfg.select_cap ? cfg.select_cap : (1ull << 26); }

cpsel_status check_common(cpsel_ctx* ctx, const void* p, uint64_t n, cpsel_dtype dtype) {
  if (!ctx) return CPSEL_EINVAL;
  if (!p) return fail(ctx, CPSEL_EINVAL, "null array pointer");
  if (n == 0) return fail(ctx, CPSEL_EINVAL, "n == 0");
  if (dtype != CPSEL_F32 && dtype != CPSEL_F64) return fail(ctx, CPSEL_EINVAL, "bad dtype %d", (int)dtype);
  if (reinterpret_cast<uintptr_t>(p) % elem_size(dtype)) return fail(ctx, CPSEL_EINVAL, "misaligned element pointer");
  return CPSEL_OK;
}

void store_value(double v, cpsel_dtype dt, void* h_out) {
  if (dt == CPSEL_F32) {
    float f = (float)v;
    memcpy(h_out, &f, 4);
  } else {
    memcpy(h_out, &v, 8);
  }
}

// Small arrays (n <= direct_threshold and <= the cluster's register capacity): the whole selection
// is one exact_cluster_kernel launch and one mailbox wait (§8f-3, BASELINE configs[0]).
cpsel_status run_direct(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype, uint64_t k, void* h_out,
                        cpsel_info* info) {
  const auto t0 = std::chrono::steady_clock::now();
  struct Ev {  // destroyed on every return path
    cudaEvent_t e = nullptr;
    ~Ev() { if (e) cudaEventDestroy(e); }
  } e0, e1;
  const bool timed = ctx->cfg.record_timing == 1;
  if (timed) {
    CK(cudaEventCreate(&e0.e));
    CK(cudaEventCreate(&e1.e));
    CK(cudaEventRecord(e0.e, ctx->stream));
  }
  const unsigned long long seq = ++ctx->seq;
  CK(launch_exact_cluster((int)dtype, d_x, n, k, &ctx->mb_dev->direct_value, &ctx->mb_dev->direct_bad,
                          &ctx->mb_dev->seq_direct, seq, ctx->stream));
  if (timed) CK(cudaEventRecord(e1.e, ctx->stream));
  const volatile unsigned long long* f = &ctx->mb->seq_direct;
  for (uint32_t i = 1; *f != seq; ++i) {
    if ((i & 255u) == 0u) {
      const cudaError_t e = cudaStreamQuery(ctx->stream);
      if (e == cudaSuccess && *f != seq) return fail(ctx, CPSEL_EINTERNAL, "kernel finished without publishing its result");
      if (e != cudaSuccess && e != cudaErrorNotReady) return fail(ctx, CPSEL_ECUDA, "%s", cudaGetErrorString(e));
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  const double v = ctx->mb->direct_value;
  const unsigned long long bad = ctx->mb->direct_bad;
  float kms = 0.f;
  if (timed) {
    CK(cudaEventSynchronize(e1.e));
    cudaEventElapsedTime(&kms, e0.e, e1.e);
  }
  ctx->trace.clear();
  if (bad) return fail(ctx, CPSEL_ENONFINITE, "input holds NaN or Inf");
  if (info) {
    memset(info, 0, sizeof *info);
    info->passes = 1;
    info->exit_reason = 6;  // direct select
    info->z_count = n;
    info->bytes_moved = n * elem_size(dtype);
    info->launches = 1;
    info->kernel_ms_select = kms;
    info->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  store_value(v, dtype, h_out);
  return CPSEL_OK;
}

cpsel_status run_single(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype, uint64_t k, void* h_out,
                        cpsel_info* info) {
  if (!ctx->cfg.force_cp && n <= ctx->cfg.direct_threshold && n <= exact_cluster_cap((int)dtype))
    return run_direct(ctx, d_x, n, dtype, k, h_out, info);
  GpuBackend be(ctx, d_x, n, (int)dtype);
  be.chain_select_cap = auto_select_cap(ctx->cfg);
  const uint64_t zc = auto_z_cap(n, ctx->cfg);
  cpsel_status s = CPSEL_OK;
  if (n > ctx->cfg.direct_threshold || ctx->cfg.force_cp)
    s = be.ensure_z(std::min<uint64_t>(zc, dense_threshold(auto_select_cap(ctx->cfg))), zc > dense_threshold(auto_select_cap(ctx->cfg)));
  if (s != CPSEL_OK) return s;
  double v = 0;
  s = drive(be, n, (int)dtype, k, ctx->cfg, zc, auto_select_cap(ctx->cfg), &v, info, &ctx->trace);
  if (s == CPSEL_ENONFINITE) return fail(ctx, s, "input holds NaN or Inf");
  if (s == CPSEL_EINTERNAL) return fail(ctx, s, "cutting-plane safeguard tripped (iteration cap / inconsistent counts)");
  if (s != CPSEL_OK) return s;
  store_value(v, dtype, h_out);
  return CPSEL_OK;
}

}  // namespace

// ============================================================================================
// C ABI
extern "C" {

const char* cpsel_status_string(cpsel_status s) {
  switch (s) {
    case CPSEL_OK: return "ok";
    case CPSEL_EINVAL: return "invalid argument";
    case CPSEL_ERANK: return "rank out of range";
    case CPSEL_ENONFINITE: return "non-finite input";
    case CPSEL_ECUDA: return "CUDA error";
    case CPSEL_ENCCL: return "NCCL error";
    case CPSEL_ENOMEM: return "out of memory";
    case CPSEL_EINTERNAL: return "internal safeguard";
  }
  return "unknown status";
}

void cpsel_config_default(cpsel_config* c) {
  if (!c) return;
  memset(c, 0, sizeof *c);
  c->z_cap = 0;
  c->direct_threshold = 1ull << 17;
  c->select_cap = 0;
  c->max_iters = 200;
  c->force_cp = 0;
  c->record_trace = 1;
  c->record_timing = 0;
  c->init_cut = 1;
  c->pass_cuts = 1;
  c->lms_fused = 1;
  c->device_loop = 0;  // measured slower than the mailbox loop (cpsel.h)
  // operator overrides: CPSEL_ZCAP, CPSEL_MAXIT (unsigned integers)
  auto env_u64 = [](const char* name, uint64_t* dst) {
    const char* e = getenv(name);
    if (!e || !*e) return;
    char* end = nullptr;
    const unsigned long long v = strtoull(e, &end, 0);
    if (end && *end == '\0') *dst = v;
  };
  uint64_t v = c->z_cap;
  env_u64("CPSEL_ZCAP", &v);
  c->z_cap = v;
  v = c->max_iters;
  env_u64("CPSEL_MAXIT", &v);
  if (v >= 1 && v <= 100000) c->max_iters = static_cast<uint32_t>(v);
}

cpsel_status cpsel_create(int device, void* cuda_stream, cpsel_ctx** out) {
  if (!out) return CPSEL_EINVAL;
  *out = nullptr;
  cpsel_ctx* ctx = new cpsel_ctx();
  ctx->device = device;
  cpsel_config_default(&ctx->cfg);
  DeviceGuard g(device);
  auto bail = [&](cpsel_status s) {
    // keep ctx for the message? the caller has no handle yet: print to stderr
    fprintf(stderr, "cpsel_create: %s\n", ctx->err.c_str());
    cpsel_destroy(ctx);
    return s;
  };
#define CKC(expr)                                                                         \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      fail(ctx, CPSEL_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_));                    \
      return bail(e_ == cudaErrorMemoryAllocation ? CPSEL_ENOMEM : CPSEL_ECUDA);          \
    }                                                                                     \
  } while (0)
  CKC(cudaSetDevice(device));
  // NULL selects the legacy default stream (the stream torch's default "current stream" is)
  ctx->stream = static_cast<cudaStream_t>(cuda_stream);
  CKC(query_shapes(device, &ctx->shape));
  CKC(cudaMalloc(&ctx->d_partials, partial_bytes_needed(ctx->shape)));
  CKC(cudaMalloc(&ctx->d_ticket, 256));
  CKC(cudaMemset(ctx->d_ticket, 0, 256));
  CKC(cudaMalloc(&ctx->d_cursors, 256));
  CKC(cudaMemset(ctx->d_cursors, 0, 256));
  CKC(cudaMalloc(&ctx->d_pass, sizeof(DevPass)));
  CKC(cudaMalloc(&ctx->d_init, sizeof(DevInit)));
  CKC(cudaMalloc(&ctx->d_t0, 32));  // t_lo, t_hi, the sample estimate
  CKC(cudaMalloc(&ctx->d_skeys, kSampleKeyBytes));
  CKC(cudaMalloc(&ctx->d_pool1, std::max(pool_sample_size(kF32, false) * 4, pool_sample_size(kF64, false) * 8)));
  // R40's scratch (zero between uses; the two-kernel form, CPSEL_SAMPLE_GRID=0, never runs in the same process)
  CKC(cudaMemset(ctx->d_pool1, 0, sample_grid_words() * sizeof(unsigned)));
  CKC(cudaMalloc(&ctx->d_chain, sizeof(ChainState)));
  CKC(cudaMalloc(&ctx->d_radix, sizeof(RadixState)));
  // radix rounds | round 0 counted by the init | the cooperative rounds' histograms and barrier
  CKC(cudaMalloc(&ctx->d_hist, kRadixHistWords * sizeof(unsigned)));
  CKC(cudaMemset(ctx->d_hist, 0, kRadixHistWords * sizeof(unsigned)));
  CKC(cudaHostAlloc(&ctx->h_pass, sizeof(DevPass), cudaHostAllocDefault));
  CKC(cudaHostAlloc(&ctx->h_init, sizeof(DevInit), cudaHostAllocDefault));
  CKC(cudaHostAlloc(&ctx->h_radix, sizeof(RadixState), cudaHostAllocDefault));
  CKC(cudaHostAlloc(&ctx->mb, sizeof(cpsel_ctx::Mailbox), cudaHostAllocMapped));
  memset(ctx->mb, 0, sizeof(cpsel_ctx::Mailbox));
  CKC(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->mb_dev), ctx->mb, 0));
  CKC(cudaDeviceSynchronize());
#undef CKC
  *out = ctx;
  return CPSEL_OK;
}

void cpsel_destroy(cpsel_ctx* ctx) {
  if (!ctx) return;
  {
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->comm.release();
    void* dev[] = {ctx->d_t0, ctx->d_skeys, ctx->d_pool1, ctx->d_chain, ctx->d_partials, ctx->d_ticket, ctx->d_cursors, ctx->d_pass, ctx->d_init, ctx->d_radix,
                   ctx->d_hist, ctx->d_gather, ctx->d_gather_init, ctx->d_zb[0], ctx->d_zb[1], ctx->d_zall,
                   ctx->d_pool, ctx->d_sizes,
                   ctx->d_stage, ctx->d_sb[0], ctx->d_sb[1], ctx->d_st[0], ctx->d_st[1]};
    for (void* p : dev)
      if (p) cudaFree(p);
    lms_free(ctx->lms);
    void* host[] = {ctx->h_pass, ctx->h_init, ctx->h_radix, ctx->h_gather, ctx->h_gather_init, ctx->mb,
                    ctx->h_sizes, ctx->h_rec};
    for (void* p : host)
      if (p) cudaFreeHost(p);
    for (cudaGraphExec_t g : ctx->kgraph)
      if (g) cudaGraphExecDestroy(g);
    if (ctx->d_ks) cudaFree(ctx->d_ks);
    if (ctx->d_knn) cudaFree(ctx->d_knn);
    if (ctx->h_ks) cudaFreeHost(ctx->h_ks);
    if (ctx->h_rep) cudaFreeHost(ctx->h_rep);
    for (cudaEvent_t e : ctx->evpool) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->light_ev) cudaEventDestroy(e);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
}

const char* cpsel_last_error(const cpsel_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

cpsel_status cpsel_set_config(cpsel_ctx* ctx, const cpsel_config* cfg) {
  if (!ctx || !cfg) return CPSEL_EINVAL;
  if (cfg->max_iters == 0) return fail(ctx, CPSEL_EINVAL, "max_iters must be >= 1");
  if (cfg->driver < 0 || cfg->driver > 3) return fail(ctx, CPSEL_EINVAL, "driver must be 0, 1, 2 or 3");
  ctx->cfg = *cfg;
  return CPSEL_OK;
}

cpsel_status cpsel_get_config(const cpsel_ctx* ctx, cpsel_config* cfg) {
  if (!ctx || !cfg) return CPSEL_EINVAL;
  *cfg = ctx->cfg;
  return CPSEL_OK;
}

cpsel_status cpsel_set_stream(cpsel_ctx* ctx, void* cuda_stream) {
  if (!ctx) return CPSEL_EINVAL;
  DeviceGuard g(ctx->device);
  if (ctx->own_stream && ctx->stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
    ctx->own_stream = false;
  }
  ctx->stream = static_cast<cudaStream_t>(cuda_stream);  // NULL: the legacy default stream
  return CPSEL_OK;
}

cpsel_status cpsel_select_kth(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype, uint64_t k,
                              void* h_out, cpsel_info* info) {
  cpsel_status s = check_common(ctx, d_x, n, dtype);
  if (s != CPSEL_OK) return s;
  if (!h_out) return fail(ctx, CPSEL_EINVAL, "null h_out");
  if (k < 1 || k > n) return fail(ctx, CPSEL_ERANK, "k=%llu outside [1,%llu]", (unsigned long long)k, (unsigned long long)n);
  DeviceGuard g(ctx->device);
  return run_single(ctx, d_x, n, dtype, k, h_out, info);
}

cpsel_status cpsel_median(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype, void* h_out,
                          cpsel_info* info) {
  return cpsel_select_kth(ctx, d_x, n, dtype, (n + 1) / 2, h_out, info);
}

cpsel_status cpsel_select_kth_host(cpsel_ctx* ctx, const void* h_x, uint64_t n, cpsel_dtype dtype, uint64_t k,
                                   void* h_out, cpsel_info* info) {
  cpsel_status s = check_common(ctx, h_x, n, dtype);
  if (s != CPSEL_OK) return s;
  if (!h_out) return fail(ctx, CPSEL_EINVAL, "null h_out");
  if (k < 1 || k > n) return fail(ctx, CPSEL_ERANK, "k=%llu outside [1,%llu]", (unsigned long long)k, (unsigned long long)n);
  DeviceGuard g(ctx->device);
  const size_t bytes = (size_t)n * elem_size(dtype);
  s = ensure(ctx, &ctx->d_stage, &ctx->stage_bytes, bytes);
  if (s != CPSEL_OK) return s;
  CK(cudaMemcpyAsync(ctx->d_stage, h_x, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return run_single(ctx, ctx->d_stage, n, dtype, k, h_out, info);
}

cpsel_status cpsel_eval(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype, double t, double y_lo,
                        double y_hi, cpsel_pass_stats* out) {
  cpsel_status s = check_common(ctx, d_x, n, dtype);
  if (s != CPSEL_OK) return s;
  if (!out) return fail(ctx, CPSEL_EINVAL, "null out");
  auto representable = [&](double v) { return dtype == CPSEL_F64 || (double)(float)v == v; };
  if (std::isnan(t) || std::isnan(y_lo) || std::isnan(y_hi) || !representable(t) || !representable(y_lo) ||
      !representable(y_hi))
    return fail(ctx, CPSEL_EINVAL, "t / bracket not representable in the dtype");
  DeviceGuard g(ctx->device);
  PassArgs a{};
  a.x = d_x; a.n = n; a.t = t; a.y_lo = y_lo; a.y_hi = y_hi; a.mode = kDirect;
  a.cursors = ctx->d_cursors; a.partials = ctx->d_partials; a.ticket = ctx->d_ticket; a.out = ctx->d_pass;
  CK(launch_pass((int)dtype, a, ctx->shape, ctx->stream));
  CK(cudaMemcpyAsync(ctx->h_pass, ctx->d_pass, sizeof(DevPass), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const DevPass& r = *ctx->h_pass;
  out->c_lt = r.c_lt; out->c_eq = r.c_eq; out->c_lo = r.c_lo; out->c_hi = r.c_hi;
  out->L_lo = r.L_lo; out->L_hi = r.L_hi; out->P = r.P; out->N = r.N; out->pred = r.pred; out->succ = r.succ;
  return CPSEL_OK;
}

cpsel_status cpsel_init(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype, cpsel_init_stats* out) {
  cpsel_status s = check_common(ctx, d_x, n, dtype);
  if (s != CPSEL_OK) return s;
  if (!out) return fail(ctx, CPSEL_EINVAL, "null out");
  DeviceGuard g(ctx->device);
  GpuBackend be(ctx, d_x, n, (int)dtype);
  return be.init(out, (n + 1) / 2);  // the extra cut (if enabled) targets the median rank
}

cpsel_status cpsel_small_select(cpsel_ctx* ctx, const void* d_z, uint64_t m, cpsel_dtype dtype, uint64_t r,
                                void* h_out) {
  cpsel_status s = check_common(ctx, d_z, m, dtype);
  if (s != CPSEL_OK) return s;
  if (!h_out) return fail(ctx, CPSEL_EINVAL, "null h_out");
  if (r < 1 || r > m) return fail(ctx, CPSEL_ERANK, "r outside [1,m]");
  DeviceGuard g(ctx->device);
  GpuBackend be(ctx, d_z, m, (int)dtype);
  double v;
  s = be.select_on(d_z, m, r, &v);
  if (s != CPSEL_OK) return s;
  store_value(canonical_zero(v), dtype, h_out);
  return CPSEL_OK;
}

cpsel_status cpsel_init_timings(cpsel_ctx* ctx, double* ms, uint32_t max, uint32_t* n_out, int32_t reset) {
  if (!ctx || !n_out) return CPSEL_EINVAL;
  DeviceGuard g(ctx->device);
  const uint32_t pairs = ctx->light_n / 2;
  *n_out = pairs;
  for (uint32_t i = 0; ms && i < pairs && i < max; ++i) {
    float f = 0.f;
    CK(cudaEventSynchronize(ctx->light_ev[2 * i + 1]));
    CK(cudaEventElapsedTime(&f, ctx->light_ev[2 * i], ctx->light_ev[2 * i + 1]));
    ms[i] = f;
  }
  if (reset) ctx->light_n = 0;
  return CPSEL_OK;
}

cpsel_status cpsel_get_trace(const cpsel_ctx* ctx, cpsel_trace_row* rows, uint32_t max_rows, uint32_t* n_rows) {
  if (!ctx || !n_rows) return CPSEL_EINVAL;
  *n_rows = (uint32_t)ctx->trace.size();
  if (rows)
    for (uint32_t i = 0; i < max_rows && i < ctx->trace.size(); ++i) rows[i] = ctx->trace[i];
  return CPSEL_OK;
}

// ------------------------------------------------------------------------ multi-GPU
cpsel_status cpsel_nccl_unique_id(void* id_out128) {
  if (!id_out128) return CPSEL_EINVAL;
  const NcclApi& nc = nccl_api();
  if (!nc.ok) return CPSEL_ENCCL;
  ncclUniqueId id;
  if (nc.GetUniqueId(&id) != ncclSuccess) return CPSEL_ENCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(id_out128, &id, 128);
  return CPSEL_OK;
}

// per-world buffers of the sharded path (tuples, records, sizes, the pooled sample)
static cpsel_status comm_buffers(cpsel_ctx* ctx, int world) {
  if (ctx->d_gather) cudaFree(ctx->d_gather);
  if (ctx->d_gather_init) cudaFree(ctx->d_gather_init);
  if (ctx->h_gather) cudaFreeHost(ctx->h_gather);
  if (ctx->h_gather_init) cudaFreeHost(ctx->h_gather_init);
  if (ctx->d_pool) cudaFree(ctx->d_pool);
  if (ctx->d_sizes) cudaFree(ctx->d_sizes);
  if (ctx->h_sizes) cudaFreeHost(ctx->h_sizes);
  if (ctx->h_rec) cudaFreeHost(ctx->h_rec);
  ctx->h_rec = ctx->d_rec = nullptr;
  ctx->h_rec_flag = ctx->d_rec_flag = nullptr;
  ctx->d_gather = nullptr; ctx->d_gather_init = nullptr; ctx->h_gather = nullptr; ctx->h_gather_init = nullptr;
  ctx->d_pool = nullptr; ctx->d_sizes = nullptr; ctx->h_sizes = nullptr;
  CK(cudaMalloc(&ctx->d_gather, world * sizeof(DevPass)));
  CK(cudaMalloc(&ctx->d_gather_init, world * sizeof(DevInit)));
  CK(cudaHostAlloc(&ctx->h_gather, world * sizeof(DevPass), cudaHostAllocDefault));
  CK(cudaHostAlloc(&ctx->h_gather_init, world * sizeof(DevInit), cudaHostAllocDefault));
  // the pooled sample: up to 16x the cluster's (R40's CPSEL_SAMPLE_X), f64
  CK(cudaMalloc(&ctx->d_pool, pool_sample_size(kF64, false) * 16 * 8));
  CK(cudaMalloc(&ctx->d_sizes, (size_t)(world + 1) * sizeof(unsigned long long)));
  CK(cudaHostAlloc(&ctx->h_sizes, (size_t)(world + 1) * sizeof(unsigned long long), cudaHostAllocDefault));
  ctx->rec_bytes = (size_t)world * std::max(sizeof(DevPass), sizeof(DevInit));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_rec), ctx->rec_bytes + 64, cudaHostAllocMapped));
  memset(ctx->h_rec, 0, ctx->rec_bytes + 64);
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->d_rec), ctx->h_rec, 0));
  ctx->h_rec_flag = reinterpret_cast<unsigned long long*>(ctx->h_rec + ctx->rec_bytes);
  ctx->d_rec_flag = reinterpret_cast<unsigned long long*>(ctx->d_rec + ctx->rec_bytes);
  return CPSEL_OK;
}

cpsel_status cpsel_comm_init(cpsel_ctx* ctx, const void* id128, int rank, int world) {
  if (!ctx || !id128 || world < 1 || rank < 0 || rank >= world) return CPSEL_EINVAL;
  const NcclApi& nc = nccl_api();
  if (!nc.ok) return fail(ctx, CPSEL_ENCCL, "NCCL unavailable: %s", nc.load_error);
  DeviceGuard g(ctx->device);
  ctx->comm.release();
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  NK(nc.CommInitRank(&ctx->comm.nccl, world, id, rank));
  ctx->comm.rank = rank;
  ctx->comm.world = world;
  ctx->comm.timeout_s = comm_timeout_from_env(120.0);
  return comm_buffers(ctx, world);
}

struct cpsel_loopback {
  std::shared_ptr<LoopGroup> g;
};

cpsel_status cpsel_loopback_create(int world, cpsel_loopback** out) {
  if (!out || world < 1) return CPSEL_EINVAL;
  *out = new cpsel_loopback{std::make_shared<LoopGroup>(world)};
  return CPSEL_OK;
}

void cpsel_loopback_destroy(cpsel_loopback* g) { delete g; }

cpsel_status cpsel_comm_init_loopback(cpsel_ctx* ctx, cpsel_loopback* group, int rank) {
  if (!ctx || !group || rank < 0 || rank >= group->g->world) return CPSEL_EINVAL;
  DeviceGuard g(ctx->device);
  if (const char* m = ctx->comm.attach_loop(group->g, rank)) return fail(ctx, CPSEL_ENCCL, "loopback: %s", m);
  ctx->comm.timeout_s = comm_timeout_from_env(120.0);
  return comm_buffers(ctx, group->g->world);
}

cpsel_status cpsel_select_kth_sharded(cpsel_ctx* ctx, const void* d_shard, uint64_t n_local, cpsel_dtype dtype,
                                      uint64_t k, void* h_out, cpsel_info* info) {
  if (!ctx) return CPSEL_EINVAL;
  if (!ctx->comm.active()) return fail(ctx, CPSEL_ENCCL, "cpsel_comm_init has not been called");
  if (n_local > 0 && !d_shard) return fail(ctx, CPSEL_EINVAL, "null shard pointer");
  if (dtype != CPSEL_F32 && dtype != CPSEL_F64) return fail(ctx, CPSEL_EINVAL, "bad dtype");
  if (!h_out) return fail(ctx, CPSEL_EINVAL, "null h_out");
  DeviceGuard g(ctx->device);
  ShardedBackend be(ctx, d_shard, n_local, (int)dtype);
  cpsel_status s = be.exchange_sizes();
  if (s != CPSEL_OK) return s;
  const uint64_t n = be.n_global;
  if (n == 0) return fail(ctx, CPSEL_EINVAL, "global n == 0");
  if (k < 1 || k > n) return fail(ctx, CPSEL_ERANK, "k outside [1,n]");
  const uint64_t zc = auto_z_cap(n, ctx->cfg);
  {
    const uint64_t dc = dense_threshold(auto_select_cap(ctx->cfg));
    s = be.ensure_z(std::max<uint64_t>(std::min<uint64_t>(std::min(zc, dc), n_local), 1), zc > dc);
  }
  if (s != CPSEL_OK) return s;
  double v = 0;
  // sharded: the kept bracket is all-gathered to every rank before its exact selection, so one more
  // cut pass (a few-% tuple exchange) beats gathering a large copy — the cap is 2^22 elements
  // (16 MB of f32 gathered); one rank gathers nothing and keeps the one-GPU cap
  const uint64_t scap = ctx->cfg.select_cap ? ctx->cfg.select_cap
                                            : (ctx->comm.world == 1 ? auto_select_cap(ctx->cfg) : (1ull << 22));
  s = drive(be, n, (int)dtype, k, ctx->cfg, zc, scap, &v, info, &ctx->trace);
  if (s == CPSEL_ENONFINITE) return fail(ctx, s, "input holds NaN or Inf");
  if (s == CPSEL_EINTERNAL) return fail(ctx, s, "cutting-plane safeguard tripped");
  if (s != CPSEL_OK) return s;
  store_value(v, dtype, h_out);
  return CPSEL_OK;
}

cpsel_status cpsel_pooled_cuts(const uint64_t* keys, const uint64_t* m, uint32_t G, uint64_t r, cpsel_dtype dtype,
                               double* out3) {
  if (!keys || !m || !out3 || G == 0) return CPSEL_EINVAL;
  if (dtype != CPSEL_F32 && dtype != CPSEL_F64) return CPSEL_EINVAL;
  std::vector<uint64_t> mm(m, m + G);
  return pooled_pick(reinterpret_cast<const unsigned long long*>(keys), mm, r, (int)dtype, out3) ? CPSEL_OK
                                                                                                 : CPSEL_EINVAL;
}

// ------------------------------------------------------------------------ host-only driver
cpsel_status cpsel_drive_host(const cpsel_host_backend* be, uint64_t n, cpsel_dtype dtype, uint64_t k,
                              const cpsel_config* cfg, double* value_out, cpsel_info* info, cpsel_trace_row* trace,
                              uint32_t max_rows, uint32_t* n_rows) {
  if (!be || !be->init || !be->pass || !be->adopt || !be->select || !value_out) return CPSEL_EINVAL;
  if (dtype != CPSEL_F32 && dtype != CPSEL_F64) return CPSEL_EINVAL;
  if (n == 0) return CPSEL_EINVAL;
  if (k < 1 || k > n) return CPSEL_ERANK;
  cpsel_config c;
  if (cfg) c = *cfg; else cpsel_config_default(&c);
  HostBackend hb(be);
  std::vector<cpsel_trace_row> tr;
  const uint64_t zc = auto_z_cap(n, c);
  cpsel_status s = drive(hb, n, (int)dtype, k, c, zc, auto_select_cap(c), value_out, info, &tr);
  if (n_rows) *n_rows = (uint32_t)tr.size();
  if (trace)
    for (uint32_t i = 0; i < max_rows && i < tr.size(); ++i) trace[i] = tr[i];
  return s;
}

// ------------------------------------------------------------------------ LMS
static constexpr uint64_t kLmsFusedMinN = 1ull << 14;
static bool lms_use_fused(const cpsel_ctx* ctx, uint64_t n) { return ctx->cfg.lms_fused && n >= kLmsFusedMinN; }

static cpsel_status lms_validate(cpsel_ctx* ctx, const float* d_X, const float* d_y, uint64_t n, uint32_t p,
                                 const float* d_thetas, uint32_t C, const void* d_out) {
  if (!d_X || !d_y || !d_thetas || !d_out) return fail(ctx, CPSEL_EINVAL, "null pointer");
  if (n == 0 || p == 0 || C == 0) return fail(ctx, CPSEL_EINVAL, "empty problem");
  if (p > kLmsMaxP) return fail(ctx, CPSEL_EINVAL, "p=%u > %d", p, kLmsMaxP);
  return CPSEL_OK;
}

static void lms_info(cpsel_info* info, const LmsReport& rep, bool fused) {
  if (!info) return;
  memset(info, 0, sizeof *info);
  info->passes = rep.passes;
  info->cp_iters = rep.cp_iters;
  info->z_count = rep.z_total;
  info->bytes_moved = rep.bytes;
  info->ms_total = rep.ms + rep.ms_fused;
  info->kernel_ms_init = rep.ms_fused;
  info->kernel_ms_passes = rep.ms;
  info->fallback_steps = rep.fallback;
  info->launches = fused ? 2 : 1;
}

cpsel_status cpsel_lms_residuals(cpsel_ctx* ctx, const float* d_X, const float* d_y, uint64_t n, uint32_t p,
                                 const float* d_thetas, uint32_t C, float* d_S) {
  if (!ctx) return CPSEL_EINVAL;
  cpsel_status s = lms_validate(ctx, d_X, d_y, n, p, d_thetas, C, d_S);
  if (s != CPSEL_OK) return s;
  DeviceGuard g(ctx->device);
  if (lms_use_fused(ctx, n)) CK(lms_fused_residuals(ctx->lms, d_X, d_y, n, p, d_thetas, C, d_S, ctx->stream));
  else CK(lms_residuals(ctx->lms, d_X, d_y, n, p, d_thetas, C, d_S, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return CPSEL_OK;
}

cpsel_status cpsel_select_kth_batched(cpsel_ctx* ctx, const float* d_S, uint64_t n, uint32_t C, uint64_t k,
                                      float* d_out, cpsel_info* info) {
  if (!ctx) return CPSEL_EINVAL;
  if (!d_S || !d_out) return fail(ctx, CPSEL_EINVAL, "null pointer");
  if (n == 0 || C == 0) return fail(ctx, CPSEL_EINVAL, "empty problem");
  if (k < 1 || k > n) return fail(ctx, CPSEL_ERANK, "k outside [1,n]");
  DeviceGuard g(ctx->device);
  LmsReport rep{};
  cudaError_t e = batched_select(ctx->lms, d_S, n, C, k, d_out, ctx->cfg.max_iters, &rep, ctx->stream);
  if (e == cudaErrorNotSupported) return fail(ctx, CPSEL_EINTERNAL, "batched select: safeguard tripped on a column");
  CK(e);
  if (rep.nonfinite) return fail(ctx, CPSEL_ENONFINITE, "input holds NaN or Inf");
  lms_info(info, rep, false);
  return CPSEL_OK;
}

// k-th smallest squared residual of every candidate (the fused path or residuals + batched select)
static cpsel_status lms_kth(cpsel_ctx* ctx, const float* d_X, const float* d_y, uint64_t n, uint32_t p,
                            const float* d_thetas, uint32_t C, uint64_t k, float* d_out, cpsel_info* info,
                            bool* used_fused = nullptr) {
  bool fused = lms_use_fused(ctx, n);
  if (used_fused) *used_fused = false;
  if (fused) {
    cudaError_t ce = cudaSuccess;
    const int chk = lms_fused_check(ctx->lms, d_X, d_y, n, p, d_thetas, C, ctx->stream, &ce);
    if (chk < 0) CK(ce);
    if (chk == 1) return fail(ctx, CPSEL_ENONFINITE, "X, y or thetas hold NaN or Inf");
    fused = chk == 0;
  }
  if (fused) {
    if (used_fused) *used_fused = true;
    LmsReport rep{};
    cudaError_t e = lms_fused_select(ctx->lms, d_X, d_y, n, p, d_thetas, C, k, d_out, ctx->cfg.max_iters, &rep,
                                     ctx->stream);
    if (e == cudaErrorNotSupported) return fail(ctx, CPSEL_EINTERNAL, "batched select: safeguard tripped on a column");
    CK(e);
    if (rep.nonfinite) return fail(ctx, CPSEL_ENONFINITE, "residuals hold NaN or Inf");
    lms_info(info, rep, true);
    return CPSEL_OK;
  }
  cpsel_status s = ensure(ctx, reinterpret_cast<void**>(&ctx->lms.S), &ctx->lms.S_bytes, (size_t)n * C * sizeof(float));
  if (s != CPSEL_OK) return s;
  CK(lms_residuals(ctx->lms, d_X, d_y, n, p, d_thetas, C, ctx->lms.S, ctx->stream));
  return cpsel_select_kth_batched(ctx, ctx->lms.S, n, C, k, d_out, info);
}

cpsel_status cpsel_lms_objective(cpsel_ctx* ctx, const float* d_X, const float* d_y, uint64_t n, uint32_t p,
                                 const float* d_thetas, uint32_t C, float* d_out, cpsel_info* info) {
  if (!ctx) return CPSEL_EINVAL;
  cpsel_status s = lms_validate(ctx, d_X, d_y, n, p, d_thetas, C, d_out);
  if (s != CPSEL_OK) return s;
  DeviceGuard g(ctx->device);
  const auto t0 = std::chrono::steady_clock::now();
  s = lms_kth(ctx, d_X, d_y, n, p, d_thetas, C, (n + 1) / 2, d_out, info);
  if (info) info->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return s;
}

cpsel_status cpsel_lts_objective(cpsel_ctx* ctx, const float* d_X, const float* d_y, uint64_t n, uint32_t p,
                                 const float* d_thetas, uint32_t C, uint64_t h, double* d_out, float* d_m,
                                 cpsel_info* info) {
  if (!ctx) return CPSEL_EINVAL;
  cpsel_status s = lms_validate(ctx, d_X, d_y, n, p, d_thetas, C, d_out);
  if (s != CPSEL_OK) return s;
  if (!d_m) return fail(ctx, CPSEL_EINVAL, "null pointer");
  if (h < 1 || h > n) return fail(ctx, CPSEL_ERANK, "h outside [1,n]");
  DeviceGuard g(ctx->device);
  const auto t0 = std::chrono::steady_clock::now();
  bool fused = false;
  s = lms_kth(ctx, d_X, d_y, n, p, d_thetas, C, h, d_m, info, &fused);
  if (s != CPSEL_OK) return s;
  if (fused) CK(lms_fused_lts(ctx->lms, d_X, d_y, n, p, d_thetas, C, h, d_m, d_out, ctx->stream));
  else CK(lts_reduce(ctx->lms.S, n, C, h, d_m, d_out, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (info) info->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return CPSEL_OK;
}

// ------------------------------------------------------------------------ kNN (§8f-4)
// steps 1-2 of kNN (distances, d2_(k) per query) shared by regression and classification; on
// success D and dk hold them and *bad points at two zeroed/used counters
static cpsel_status knn_select(cpsel_ctx* ctx, const float* d_X, uint64_t n, uint32_t p, const float* d_Q,
                               uint32_t nq, uint64_t k, float* d_dk, float** D_out, float** dk_out,
                               unsigned long long** bad_out, LmsReport* rep) {
  const size_t dbytes = (size_t)n * nq * sizeof(float), off_dk = (dbytes + 255) / 256 * 256;
  const size_t off_bad = off_dk + ((size_t)nq * sizeof(float) + 255) / 256 * 256;
  cpsel_status s = ensure(ctx, &ctx->d_knn, &ctx->knn_bytes, off_bad + 256);
  if (s != CPSEL_OK) return s;
  char* base = static_cast<char*>(ctx->d_knn);
  float* D = reinterpret_cast<float*>(base);
  float* dk = d_dk ? d_dk : reinterpret_cast<float*>(base + off_dk);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(base + off_bad);
  CK(cudaMemsetAsync(bad, 0, 2 * sizeof *bad, ctx->stream));
  CK(knn_distances(d_X, d_Q, n, p, nq, D, bad, ctx->stream));            // 1. distances
  unsigned long long hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (hbad) return fail(ctx, CPSEL_ENONFINITE, "X or Q hold NaN or Inf (or a distance overflows)");
  cudaError_t e = batched_select(ctx->lms, D, n, nq, k, dk, ctx->cfg.max_iters, rep, ctx->stream);  // 2. d2_(k)
  if (e == cudaErrorNotSupported) return fail(ctx, CPSEL_EINTERNAL, "batched select: safeguard tripped on a query");
  CK(e);
  if (rep->nonfinite) return fail(ctx, CPSEL_ENONFINITE, "X or Q hold NaN or Inf");
  *D_out = D; *dk_out = dk; *bad_out = bad;
  return CPSEL_OK;
}

cpsel_status cpsel_knn_classify(cpsel_ctx* ctx, const float* d_X, const int32_t* d_labels, uint64_t n, uint32_t p,
                                const float* d_Q, uint32_t nq, uint64_t k, uint32_t n_classes, int32_t weighting,
                                int32_t* d_out, double* d_votes, cpsel_info* info) {
  if (!ctx) return CPSEL_EINVAL;
  if (!d_X || !d_labels || !d_Q || !d_out) return fail(ctx, CPSEL_EINVAL, "null pointer");
  if (n == 0 || nq == 0 || p == 0) return fail(ctx, CPSEL_EINVAL, "empty problem");
  if (p > (uint32_t)kKnnMaxP) return fail(ctx, CPSEL_EINVAL, "p > %d", kKnnMaxP);
  if (nq > 65535u * 16u) return fail(ctx, CPSEL_EINVAL, "nq > 1048560");
  if (n_classes == 0 || n_classes > 64) return fail(ctx, CPSEL_EINVAL, "n_classes must be in [1, 64]");
  if (weighting != 0 && weighting != 1) return fail(ctx, CPSEL_EINVAL, "weighting must be 0 or 1");
  if (k < 1 || k > n) return fail(ctx, CPSEL_ERANK, "k outside [1,n]");
  DeviceGuard g(ctx->device);
  const auto t0 = std::chrono::steady_clock::now();
  float *D, *dk;
  unsigned long long* bad;
  LmsReport rep{};
  cpsel_status s = knn_select(ctx, d_X, n, p, d_Q, nq, k, nullptr, &D, &dk, &bad, &rep);
  if (s != CPSEL_OK) return s;
  CK(knn_vote(D, d_labels, n, nq, k, n_classes, dk, weighting, d_out, d_votes, bad + 1, ctx->stream));  // 3. votes
  unsigned long long hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad + 1, sizeof hbad, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (hbad) return fail(ctx, CPSEL_EINVAL, "a label of a voting neighbour is outside [0, n_classes)");
  lms_info(info, rep, false);
  if (info) {
    info->launches += 2;
    info->bytes_moved += 2 * (uint64_t)n * nq * sizeof(float);
    info->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return CPSEL_OK;
}

cpsel_status cpsel_knn_regress(cpsel_ctx* ctx, const float* d_X, const float* d_f, uint64_t n, uint32_t p,
                               const float* d_Q, uint32_t nq, uint64_t k, int32_t weighting, float* d_out,
                               float* d_dk, cpsel_info* info) {
  if (!ctx) return CPSEL_EINVAL;
  if (!d_X || !d_f || !d_Q || !d_out) return fail(ctx, CPSEL_EINVAL, "null pointer");
  if (n == 0 || nq == 0 || p == 0) return fail(ctx, CPSEL_EINVAL, "empty problem");
  if (p > (uint32_t)kKnnMaxP) return fail(ctx, CPSEL_EINVAL, "p > %d", kKnnMaxP);
  if (nq > 65535u * 16u) return fail(ctx, CPSEL_EINVAL, "nq > 1048560");
  if (weighting != 0 && weighting != 1) return fail(ctx, CPSEL_EINVAL, "weighting must be 0 or 1");
  if (k < 1 || k > n) return fail(ctx, CPSEL_ERANK, "k outside [1,n]");
  DeviceGuard g(ctx->device);
  const auto t0 = std::chrono::steady_clock::now();
  const size_t dbytes = (size_t)n * nq * sizeof(float);
  float *D, *dk;
  unsigned long long* bad;
  LmsReport rep{};
  cpsel_status s = knn_select(ctx, d_X, n, p, d_Q, nq, k, d_dk, &D, &dk, &bad, &rep);
  if (s != CPSEL_OK) return s;
  CK(knn_check_f(d_f, n, bad + 1, ctx->stream));                         // NaN/Inf in f
  unsigned long long hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad + 1, sizeof hbad, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (hbad) return fail(ctx, CPSEL_ENONFINITE, "f holds NaN or Inf");
  CK(knn_reduce(D, d_f, n, nq, k, dk, weighting, d_out, ctx->stream));  // 3. the rho reduction
  CK(cudaStreamSynchronize(ctx->stream));
  lms_info(info, rep, false);
  if (info) {
    info->launches += 2;
    info->bytes_moved += 2 * dbytes;  // D written once, read once more by the reduction
    info->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return CPSEL_OK;
}

}  // extern "C"
