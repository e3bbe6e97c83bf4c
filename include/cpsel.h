/*
 * cpsel.h — C ABI of libcpsel.so: exact k-th order statistics (median) of large device
 * arrays by Kelley's cutting-plane method (Beliakov, arXiv:1104.2732), B200 / sm_100a.
 *
 * Citations: P:Lnnn = line nnn of the paper's text (/root/reference/PAPER.md, not shipped);
 * "R<n>" = numbered reading of the paper in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Every call returns cpsel_status; nothing aborts or throws.  On error the ctx keeps a
 *    message readable with cpsel_last_error().  Validation happens before any launch.
 *  - Ranks k are 1-based and select the k-th SMALLEST element (R2 maps Eq. 2).
 *  - The median is the lower median k = floor((n+1)/2) (R3).
 *  - d_* pointers are device pointers on the ctx's device, h_* pointers are host pointers.
 *    Input arrays are read-only for the duration of the call (the caller owns them and must
 *    not modify them concurrently).  The ctx owns all scratch; it grows lazily, is cached
 *    across calls and is freed by cpsel_destroy.  No allocation happens inside the
 *    iteration loop.
 *  - Work is enqueued on the ctx stream.  Calls are host-blocking (the cutting-plane driver
 *    needs each pass's tuple on the host, P:L426 'partial sums ... added on the CPU').
 *  - A ctx is not thread-safe; distinct ctxs may be used from distinct threads.
 *  - Non-finite inputs (NaN, +-Inf) are rejected with CPSEL_ENONFINITE (R12).
 *  - Returned values are elements of the input, bit-exact, with -0.0 canonicalised to +0.0 (R13).
 */
#ifndef CPSEL_H
#define CPSEL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CPSEL_OK = 0,
  CPSEL_EINVAL = 1,     /* null pointer, n == 0, bad dtype, misaligned element pointer, bad config */
  CPSEL_ERANK = 2,      /* k < 1 or k > n */
  CPSEL_ENONFINITE = 3, /* the input holds NaN or +-Inf */
  CPSEL_ECUDA = 4,      /* a CUDA runtime error (message in cpsel_last_error) */
  CPSEL_ENCCL = 5,      /* an NCCL error, or NCCL not loadable / comm not initialised; also a sharded
                           call whose collectives reported an asynchronous error or made no progress
                           for CPSEL_COMM_TIMEOUT_S seconds (default 120): the communicator is then
                           aborted and must be re-initialised */
  CPSEL_ENOMEM = 6,     /* device or pinned allocation failed */
  CPSEL_EINTERNAL = 7   /* a safeguard tripped (iteration cap); never expected */
} cpsel_status;

typedef enum { CPSEL_F32 = 0, CPSEL_F64 = 1 } cpsel_dtype;

typedef struct cpsel_ctx cpsel_ctx;

/* Tunables.  cpsel_config_default() fills the defaults noted here, then applies the operator
 * overrides CPSEL_ZCAP (z_cap) and CPSEL_MAXIT (max_iters, 1..100000) from the environment when
 * they are set to an unsigned integer (malformed values are ignored). */
typedef struct {
  uint64_t z_cap;            /* compaction threshold on the bracket interior count m: the first
                                pass whose interior m <= z_cap also copies the two halves of the
                                bracket (split at t) out (P:L196 copy_if, R8); later passes run on
                                the kept half only and compact again.  0 = auto (5/8 n). */
  uint64_t direct_threshold; /* n <= this: skip the cutting plane, select on x directly
                                (P:L311 'radix sort ... most efficient up to 2^21').  Default 2^17 */
  uint64_t select_cap;       /* a kept half of <= select_cap elements is finished by the exact
                                radix select (P:L196 'sort z', R21).  0 = auto (2^26: the init's copy of
                                ~2% of n is radix-selected directly up to n ~ 2^30). */
  uint32_t max_iters;        /* safety cap on cutting-plane passes (P:L169 maxit).  Default 200 */
  int32_t force_cp;          /* 1: always run cutting-plane passes (parity runs), ignore direct_threshold */
  int32_t record_trace;      /* 1: keep the per-iteration trace (cpsel_get_trace).  Default 1 */
  int32_t record_timing;     /* 2: light — only each selection's init kernel is bracketed by CUDA
                                events, kept in a ring read by cpsel_init_timings (nothing is read
                                back during the calls).
                                1: time every kernel with CUDA events on the ctx stream (info / trace
                                kernel_ms fields).  Default 0 */
  int32_t init_cut;          /* 1: the init pass also evaluates two extra cuts at sample quantiles
                                bracketing the target rank (R23), saving passes.  Default 1 */
  int32_t objective;         /* 1: every trace row carries F_k(t): the init pass also sums
                                (t_lo-x)^+ and (x-t_hi)^+ (4 more issue slots per element).
                                0: rows after the init cuts report F = NaN — the iterates never
                                need F (App. A: interior means), R25.  Default 0 */
  int32_t pass_cuts;         /* 1: a compacted bracket larger than select_cap is cut at two sample
                                quantiles of its own, keeping only what lies between them (R26,
                                multi-point step).  Ignored with objective=1.  Default 1 */
  int32_t lms_fused;         /* 1: LMS/LTS objectives never store S: the residuals are recomputed
                                on the tensor cores inside one fused pass that takes the init
                                statistics, counts at two sample cuts per candidate and copies
                                what lies between them (§8f-2); columns the copy cannot finish
                                are stored and selected from S.  Used for n >= 16384.  Default 1 */
  int32_t device_loop;       /* 1: once only Kelley passes remain (pass_cuts=0 or objective=1, or the
                                sample cuts missed), the rest of the selection runs as ONE CUDA graph
                                launch — a WHILE node over {Kelley step kernel, IF pass kernels} and
                                the exact select behind it — with no host round trip per pass (§8f-3).
                                0: the host drives every pass through the mapped mailbox.  Default 0:
                                measured on B200, a WHILE iteration costs ~9.7 us of device-side
                                relaunch, more than the mailbox round trip (+35 us per selection at
                                2^20..2^27, +2% at 2^30) */
  int32_t driver;            /* 0: Kelley's cutting plane (Algorithm 1, the method).  1: bisection, the
                                paper's comparison: t = (y_L + y_R)/2 in value, the
                                same passes, exact rank test and finish; no R26 cut passes, no
                                ordered-key safeguard (its pass count grows with log2 of the data
                                range, P:L413 — the outlier-sensitivity demonstration).  2: Brent's
                                root finder (Numerical Recipes' zbrent) on
                                f(t) = c_lt(t) + c_le(t) - 2k + 1 proposing the points instead, the
                                same passes and exact bracket.  3: Brent's minimisation (Numerical
                                Recipes' brent on F_k: parabolic steps, golden section
                                when they fail; its own bracket intersected with the exact one, R37)
                                proposing the points; needs F at every pass (init_cut = 0, or
                                objective = 1), else the call fails with CPSEL_EINVAL.  Default 0 */
} cpsel_config;

/* Per-call report (SPEC 'SelectionResult': iterations, reductions). */
typedef struct {
  uint32_t passes;         /* full passes over x (init + cutting-plane), P:L194 'maxit+1 reductions' */
  uint32_t cp_iters;       /* cutting-plane iterations (Algorithm 1 step 1) */
  uint32_t fallback_steps; /* safeguard steps (ordered-key bisection), R7 */
  uint32_t exit_reason;    /* 0 init_min, 1 init_max, 2 hit, 3 pred, 4 succ, 5 compact+select, 6 direct select */
  uint64_t z_count;        /* elements in the final selection set (0 if none) */
  uint64_t bytes_moved;    /* algorithmic HBM bytes of all passes (reads of x + writes/reads of z) */
  double ms_total;         /* host wall time of the call */
  uint32_t launches;       /* kernels this call launched */
  uint32_t reserved;
  double kernel_ms_init;   /* record_timing: CUDA-event time of the init kernel */
  double kernel_ms_passes; /* record_timing: sum over the cutting-plane pass kernels */
  double kernel_ms_select; /* record_timing: the small-set selection kernels */
  uint64_t init_written;   /* elements the init pass copied out (fused compaction of ]t_lo, t_hi[, R23) */
  double kernel_ms_sample; /* record_timing: the sample-cut kernels (gather + select, R29), not in the above */
} cpsel_info;

/* One objective pass at t (Fig. 1 'Objective'), see cpsel_eval. */
typedef struct {
  uint64_t c_lt, c_eq;   /* #{x < t}, #{x == t}: dF(t) = [n(c_lt-k+1/2), n(c_lt+c_eq-k+1/2)] */
  uint64_t c_lo, c_hi;   /* #{y_lo < x < t}, #{t < x < y_hi} */
  double L_lo, L_hi;     /* sum_{y_lo<x<t} (t-x),  sum_{t<x<y_hi} (x-t)   (fp64 accumulation) */
  double P, N;           /* sum (x-t)^+, sum (t-x)^+ over all x (direct, as Fig. 1 does) */
  double pred, succ;     /* max{x: y_lo<x<t} (-inf if none), min{x: t<x<y_hi} (+inf if none) */
} cpsel_pass_stats;

/* The init reduction (x_(1), x_(n) and sum x in ONE pass; R5 multiplicities). */
typedef struct {
  double vmin, vmax;      /* exact */
  uint64_t cnt_min, cnt_max, nonfinite;
  double x0;              /* the shift x[0] */
  double S;               /* sum_i (x_i - x0), fp64 (0 when has_cut: the first iterate then comes
                             from the cut's sums and the pass skips this sum) */
  uint64_t has_cut;       /* bit 1 (2): the pass also evaluated the two extra cuts t_lo <= t_hi (R23);
                             bit 0 (1): it also copied ]t_lo, t_hi[ out; bit 2 (4): N_lo, P_hi valid */
  double t_lo, t_hi;      /*   sample quantiles bracketing rank k (elements of x) */
  uint64_t c_le_lo, c_lt_hi; /* #{x<=t_lo}, #{x<t_hi}: the counts a bracket update needs at each cut
                             when the target lies between them; a cut beyond the target moves to the
                             adjacent float, where the missing count is the known one (R24) */
  double t_est;           /*   the sample's estimate of x_(k) (starting iterate when I_in is not kept) */
  uint64_t reserved_cut;
  double N_lo;            /*   sum (t_lo - x)^+ */
  double P_hi;            /*   sum (x - t_hi)^+ */
  double I_in;            /*   sum over t_lo < x < t_hi of (x - t_lo)  (with N_lo, P_hi: bit 2 of has_cut) */
} cpsel_init_stats;

/* One row per cutting-plane pass (R7 trace). */
typedef struct {
  double t;               /* query point (an element of the dtype) */
  double F;               /* F_k(t) = (k-1/2) P(t) + (n-k+1/2) N(t)  (Eq. 2, R2) via App. A identities */
  uint64_t c_lt, c_eq;    /* exact counts at t (UINT64_MAX: not evaluated — the init cuts, R24) */
  uint64_t interior;      /* bracket interior count after the update */
  uint64_t scanned;       /* elements this pass read (x, or the compacted bracket) */
  uint64_t written;       /* elements this pass wrote (compaction of both bracket halves) */
  uint32_t kind;          /* 0 Kelley step (interior mean, R4), 1 ordered-key bisection safeguard,
                             2 the init pass's extra cut (R23), 3 a two-cut pass (R26), 4 a step of
                             the bisection driver (driver = 1), 5 of Brent's root finder (driver 2),
                             6 of Brent's minimisation (driver 3) */
  uint32_t compacted;     /* 1 if this pass also wrote z */
  double kernel_ms;       /* record_timing: CUDA-event duration of this pass's kernel */
} cpsel_trace_row;

/* ---- context ------------------------------------------------------------------------- */
/* device: CUDA ordinal; cuda_stream: a cudaStream_t on that device, or NULL for the legacy
 * default stream (so work is ordered after whatever the caller enqueued there).  *out receives
 * the new ctx. */
cpsel_status cpsel_create(int device, void* cuda_stream, cpsel_ctx** out);
void cpsel_destroy(cpsel_ctx* ctx);
const char* cpsel_last_error(const cpsel_ctx* ctx);
const char* cpsel_status_string(cpsel_status s);
void cpsel_config_default(cpsel_config* cfg);
cpsel_status cpsel_set_config(cpsel_ctx* ctx, const cpsel_config* cfg);
cpsel_status cpsel_get_config(const cpsel_ctx* ctx, cpsel_config* cfg);
/* Re-target the ctx stream (e.g. torch's current stream; NULL = legacy default stream) without
 * recreating scratch. */
cpsel_status cpsel_set_stream(cpsel_ctx* ctx, void* cuda_stream);

/* ---- selection (north_star: select_kth(x, n, k), median(x, n)) -------------------------- */
/* d_x: device array of n elements of dtype (element-aligned, any 16-byte phase).
 * k in [1, n].  *h_out receives one element (4 or 8 bytes).  info may be NULL. */
cpsel_status cpsel_select_kth(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype,
                              uint64_t k, void* h_out, cpsel_info* info);
/* k = floor((n+1)/2). */
cpsel_status cpsel_median(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype,
                          void* h_out, cpsel_info* info);
/* Same as cpsel_select_kth for a HOST array h_x (pinned memory recommended): the H2D copy
 * into ctx-owned device staging is part of the call (end-to-end path). */
cpsel_status cpsel_select_kth_host(cpsel_ctx* ctx, const void* h_x, uint64_t n, cpsel_dtype dtype,
                                   uint64_t k, void* h_out, cpsel_info* info);

/* ---- LMS (north_star: lms_objective(X, y, thetas)) -------------------------- */
/* d_X: float32 n x p row-major; d_y: float32[n]; d_thetas: float32 p x C column-major
 * (theta_j = d_thetas[j*p .. j*p+p)).  d_out: float32[C] (device) receives, per candidate,
 * Med_i (x_i . theta_j - y_i)^2 (R19: median of squared residuals, lower median).
 * p <= 16.  Host-blocking; d_out is complete on return. */
cpsel_status cpsel_lms_objective(cpsel_ctx* ctx, const float* d_X, const float* d_y, uint64_t n,
                                 uint32_t p, const float* d_thetas, uint32_t C, float* d_out,
                                 cpsel_info* info);
/* The residual stage alone: d_S (float32, n x C column-major, column j at d_S + j*n) receives
 * (x_i . theta_j - y_i)^2 computed on the tensor cores (tcgen05, 3xTF32 split) — by the kernel
 * the objectives use under the current config (lms_fused), so the objectives are exactly the
 * order statistics of this S. */
cpsel_status cpsel_lms_residuals(cpsel_ctx* ctx, const float* d_X, const float* d_y, uint64_t n,
                                 uint32_t p, const float* d_thetas, uint32_t C, float* d_S);
/* LTS (NEXT row): d_out[j] (float64, device) = the sum of the h smallest squared
 * residuals of candidate j, computed as sum_{s<m_j} s + (h - #{s<m_j}) m_j (the rho/a,b form of
 * P:L464-478, every s = m_j equal to m_j) with m_j = the h-th smallest squared residual, written to
 * d_m[j] (float32, device).  Same residual and batched-selection stages as cpsel_lms_objective,
 * then one fp64-accumulated reduction over S.  1 <= h <= n (the paper's h = [(n+p)/2] or
 * (n+1)/2 is the caller's choice, R20).  Host-blocking. */
cpsel_status cpsel_lts_objective(cpsel_ctx* ctx, const float* d_X, const float* d_y, uint64_t n,
                                 uint32_t p, const float* d_thetas, uint32_t C, uint64_t h,
                                 double* d_out, float* d_m, cpsel_info* info);
/* Batched selection: for each column j of d_S (n x C column-major) the k-th smallest
 * -> d_out[j] (float32, device). */
cpsel_status cpsel_select_kth_batched(cpsel_ctx* ctx, const float* d_S, uint64_t n, uint32_t C,
                                      uint64_t k, float* d_out, cpsel_info* info);

/* ---- parity hooks ------------------------------------------------------------------------ */
/* One pass at t with bracket (y_lo, y_hi).  t, y_lo, y_hi must be representable in dtype
 * (else CPSEL_EINVAL).  Computes every field of cpsel_pass_stats in a single read of x. */
cpsel_status cpsel_eval(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype, double t,
                        double y_lo, double y_hi, cpsel_pass_stats* out);
/* The init reduction alone (step a1); with init_cut it also evaluates the two extra cuts at the
 * sample quantiles bracketing the median rank (R23). */
cpsel_status cpsel_init(cpsel_ctx* ctx, const void* d_x, uint64_t n, cpsel_dtype dtype,
                        cpsel_init_stats* out);
/* The small-set exact selection alone (step a5): r-th smallest (1-based) of d_z[0..m). */
cpsel_status cpsel_small_select(cpsel_ctx* ctx, const void* d_z, uint64_t m, cpsel_dtype dtype,
                                uint64_t r, void* h_out);
/* Copy up to max_rows rows of the last call's trace into rows; *n_rows = rows available. */
/* record_timing == 2: *n_out = init-kernel durations recorded since the last reset; ms[0..min(n,max))
 * receives them (CUDA-event ms, in call order; waits for the events).  reset != 0 empties the ring.
 * ms may be NULL (count only).  Errors: EINVAL (null ctx / n_out), ECUDA. */
cpsel_status cpsel_init_timings(cpsel_ctx* ctx, double* ms, uint32_t max, uint32_t* n_out, int32_t reset);
cpsel_status cpsel_get_trace(const cpsel_ctx* ctx, cpsel_trace_row* rows, uint32_t max_rows,
                             uint32_t* n_rows);

/* ---- multi-GPU (one process per GPU) -------------------------------------- */
/* Writes a fresh 128-byte ncclUniqueId into id_out (call on rank 0, broadcast it yourself,
 * e.g. torch.distributed.broadcast_object_list).  NCCL is resolved at run time from the
 * libnccl.so.2 already loaded in the process (torch's), else from the system. */
cpsel_status cpsel_nccl_unique_id(void* id_out128);
/* Collective: every rank calls with the same id, its rank and the world size.  Failure detection:
 * while a sharded call waits on its collectives it polls ncclCommGetAsyncError and a deadline of
 * CPSEL_COMM_TIMEOUT_S seconds (read here; default 120); either aborts the communicator
 * (ncclCommAbort) and fails the call with ENCCL, after which this function must be called again. */
cpsel_status cpsel_comm_init(cpsel_ctx* ctx, const void* id128, int rank, int world);
/* Loopback transport (SURVEY §4 "G virtual shards on one GPU"): `world` virtual ranks inside ONE
 * process, each a host thread with its own ctx (and stream) on the same device.  The sharded driver
 * runs unchanged; its all-gathers become device-to-device copies ordered by CUDA events between
 * two host barriers.  create: *out <- a group handle owned by the caller (destroy it after every
 * ctx attached to it has been destroyed or re-initialised; the ctxs keep the group alive until
 * then).  comm_init_loopback: attach ctx as `rank` (each rank exactly once).  A rank that does not
 * reach a collective within CPSEL_COMM_TIMEOUT_S seconds (read at attach; default 120) breaks the group: every rank's call then fails with ENCCL.
 * Errors: EINVAL (null pointers, rank outside [0, world)), ENCCL (rank already attached). */
typedef struct cpsel_loopback cpsel_loopback;
cpsel_status cpsel_loopback_create(int world, cpsel_loopback** out);
void cpsel_loopback_destroy(cpsel_loopback* group);
cpsel_status cpsel_comm_init_loopback(cpsel_ctx* ctx, cpsel_loopback* group, int rank);
/* Collective: x is the concatenation over ranks (in rank order) of the shards d_shard
 * (n_local elements each, may differ per rank, may be 0).  k is the global rank.  Every
 * rank receives the same *h_out.  Init: the pooled sample (R28: each rank's share of 131072
 * (f32) / 65536 (f64) evenly strided values, proportional to its shard, all-gathered; every rank
 * picks the same two cuts with the same cluster select), the fused init pass per rank, and an
 * all-gather of the 128-byte init records.  Per iteration one 96-byte-per-rank all-gather of the
 * pass tuples, combined in rank order; at the end an all-gather-v of the bracket contents
 * (north_star; <= 2^22 elements in all unless select_cap says otherwise) and the same radix select
 * on every rank. */
cpsel_status cpsel_select_kth_sharded(cpsel_ctx* ctx, const void* d_shard, uint64_t n_local,
                                      cpsel_dtype dtype, uint64_t k, void* h_out, cpsel_info* info);

/* R28: cuts common to all ranks from their pooled samples — the host step of the sharded init and
 * cut passes, exported for the CPU (gloo) tests.  keys: G blocks of 1024 order-preserving sample
 * keys (f32: sign-flipped bits in the low 32; f64: sign-flipped 64 bits), block g sorted ascending
 * with its min(m[g], 1024) valid keys first; m[g]: elements of rank g's array; r: the target rank
 * (1-based) in the concatenation.  out3 <- t_a, t_b, the pooled estimate of the target.
 * Errors: CPSEL_EINVAL (null pointers, G == 0, no element at all). */
cpsel_status cpsel_pooled_cuts(const uint64_t* keys, const uint64_t* m, uint32_t G, uint64_t r, cpsel_dtype dtype,
                               double* out3);

/* ---- kNN regression via d_(k) (NEXT row §8f-4) --------------------------------- */
/* For every query q_j (row j of Q, nq x p float32 row-major) and the n reference points x_i (rows of
 * X, n x p float32 row-major) with ordinates f_i (float32[n]), all device pointers:
 *   d2_ij = sum_l (q_jl - x_il)^2            float32, round-to-nearest in the order l = 0..p-1
 *   d2_(k)j = the k-th smallest of row j     (the batched cutting-plane selection, step a8)
 *   out[j] = sum_i rho_ij w_ij f_i / sum_i rho_ij w_ij,  rho = 1 if d2 < d2_(k), a/b if d2 = d2_(k),
 *            0 otherwise, a = k - #{d2 < d2_(k)}, b = #{d2 = d2_(k)}  (the paper's indicator rho,
 *            P:L469-476 at rank k: exactly k neighbours' worth of weight, ties shared);
 *            w = 1 (weighting 0) or 1/(d2 + 1e-12) (weighting 1, decreasing in the distance);
 *            fp64 accumulation, written as float32.
 * d_dk (nullable, float32[nq]) receives d2_(k) per query.  1 <= p <= 32.  The call owns an
 * nq x n float32 scratch matrix (grown lazily, freed with the ctx) and returns after completion.
 * Errors: EINVAL (null pointers, n/nq/p == 0, p > 32, nq > 1048560, weighting not 0/1), ERANK (k outside [1, n]),
 * ENONFINITE (NaN/Inf in X, Q or f), ENOMEM, ECUDA. */
cpsel_status cpsel_knn_regress(cpsel_ctx* ctx, const float* d_X, const float* d_f, uint64_t n, uint32_t p,
                               const float* d_Q, uint32_t nq, uint64_t k, int32_t weighting, float* d_out,
                               float* d_dk, cpsel_info* info);

/* kNN classification ("the majority vote (among the k nearest neighbours) is applied"): the
 * same distances and d2_(k) as cpsel_knn_regress; per query the votes
 *   V_c = sum_i rho_ij w_ij [labels_i = c]   (rho as above: exactly k neighbours' worth, ties shared)
 * and d_out[j] = the class with the largest vote (the smallest index among equal votes).
 * d_labels: int32[n] in [0, n_classes), 1 <= n_classes <= 64; d_votes (nullable): f64 nq x n_classes
 * row-major (fp64 shared-memory atomics: with weighting 1 the summation order, and so the last bits
 * of a vote, may vary run to run).  Errors as cpsel_knn_regress, plus EINVAL for n_classes outside
 * [1, 64] or a voting neighbour's label outside [0, n_classes). */
cpsel_status cpsel_knn_classify(cpsel_ctx* ctx, const float* d_X, const int32_t* d_labels, uint64_t n, uint32_t p,
                                const float* d_Q, uint32_t nq, uint64_t k, uint32_t n_classes, int32_t weighting,
                                int32_t* d_out, double* d_votes, cpsel_info* info);

/* ---- host-only driver (no GPU needed) ------------------------------------------------------ */
/* The same cutting-plane driver, with the three device steps supplied as callbacks.  Used by
 * the CPU tests (world-size-2 gloo tests of the sharded combine) to exercise the exact host
 * logic the GPU path runs.  Each callback returns 0 on success. */
typedef struct {
  double t_a, t_b;        /* the two cuts */
  double t_est;           /* the sample's estimate of x_(k) (the next starting iterate) */
  uint64_t le_a, inner;   /* #{x <= t_a}, #{t_a < x < t_b} (local to the current array) */
} cpsel_cut_stats;
typedef struct {
  void* user;
  /* init reduction over the whole (possibly sharded) array: fill *out. */
  int (*init)(void* user, cpsel_init_stats* out);
  /* one pass at t over bracket (y_lo, y_hi) of the current array (x at first); fill c_lt, c_eq,
     c_lo, c_hi, L_lo, L_hi, pred, succ of *out, counts local to the current array.  If
     compact != 0 the callee must also retain {y_lo < x < t} and {t < x < y_hi}. */
  int (*pass)(void* user, double t, double y_lo, double y_hi, int compact, cpsel_pass_stats* out);
  /* make the retained half `side` (0: (y_lo,t), 1: (t,y_hi)) of the last compacting pass the
     array every later pass (and select side 2) runs on. */
  int (*adopt)(void* user, int side);
  /* exact selection of the r-th smallest (1-based) of the retained half `side` of the last
     compacting pass, or of the current array if side == 2. */
  int (*select)(void* user, int side, uint64_t r, double* value_out);
  /* optional (NULL: none): the R26 cut pass over the current array, which is exactly the bracket
     interior — two sample cuts t_a <= t_b (elements of it) around its local rank r; fill *out with
     them, the sample's estimate of the target, #{x <= t_a} and #{t_a < x < t_b}, and retain the
     latter set as half 0 of a compacting pass. */
  int (*cut)(void* user, uint64_t r, cpsel_cut_stats* out);
} cpsel_host_backend;
cpsel_status cpsel_drive_host(const cpsel_host_backend* be, uint64_t n, cpsel_dtype dtype,
                              uint64_t k, const cpsel_config* cfg, double* value_out,
                              cpsel_info* info, cpsel_trace_row* trace, uint32_t max_rows,
                              uint32_t* n_rows);

#ifdef __cplusplus
}
#endif
#endif /* CPSEL_H */
