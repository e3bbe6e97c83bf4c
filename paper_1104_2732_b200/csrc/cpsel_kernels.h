// Internal interface between the host driver (cpsel_driver.cpp) and the sm_100a kernels
// (cpsel_kernels.cu).  Not part of the public ABI (include/cpsel.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cpsel {

enum Dtype : int { kF32 = 0, kF64 = 1 };

// Result of one pass at t over bracket (y_lo, y_hi) (step a2), written by the last CTA.
struct DevPass {
  unsigned long long c_lt, c_eq;   // #{x<t}, #{x==t}  (global)
  unsigned long long c_lo, c_hi;   // #{y_lo<x<t}, #{t<x<y_hi} (direct mode only; else 0)
  double L_lo, L_hi;               // sum_{y_lo<x<t}(t-x), sum_{t<x<y_hi}(x-t)
  double P, N;                     // direct mode only: sum (x-t)^+, sum (t-x)^+
  double pred, succ;               // max{y_lo<x<t}, min{t<x<y_hi}
  unsigned long long z_lo, z_hi;   // elements written by the fused compaction (a4)
};
static_assert(sizeof(DevPass) == 96, "DevPass layout");

// Result of the init pass (step a1).
struct DevInit {
  double vmin, vmax, S, x0;
  unsigned long long cnt_min, cnt_max, nonfinite, pad;
  // the two extra cuts t_lo <= t_hi evaluated in the same pass (R23)
  double t_lo, t_hi, N_lo, P_hi, I_in;
  // #x<=t_lo and #x<t_hi: the counts the bracket update needs at each cut (R24)
  unsigned long long c_le_lo, c_lt_hi;
  double t_est;                    // the sample's estimate of x_(k) (a starting iterate)
  unsigned long long res1, res2, has_cut;
};

// Per-CTA partial of a pass (grid reduction scratch).
struct PassPartial {
  unsigned long long c_lt, c_eq, c_lo, c_hi;
  double L_lo, L_hi, P, N, pred, succ;
};
struct InitPartial {
  double vmin, vmax, S, pad;
  unsigned long long cnt_min, cnt_max, nonfinite, pad2;
  double N0, P0, I0, pad3;
  unsigned long long cA, cB, cC, cD, cE, pad4;
};

// Device-side state of the radix select (step a5).
struct RadixState {
  unsigned long long prefix, mask;   // ordered-key bits fixed so far
  unsigned long long r;              // remaining 1-based rank inside the prefix class
  unsigned long long count;          // candidates in the prefix class (diagnostic)
  double value;                      // the selected element (after the last round)
  unsigned long long key;
};

enum PassMode : int { kHot = 0, kCompact = 1, kDirect = 2 };

struct KelleyState;

struct PassArgs {
  const struct KelleyState* ks;      // device loop (§8f-3): x, n, t, y_lo, y_hi, out taken from *ks
  const void* x;
  uint64_t n;
  double t, y_lo, y_hi;              // representable in the dtype
  int mode;
  void* z;                           // compaction target (mode kCompact), capacity z_cap
  uint64_t z_cap;
  unsigned long long* cursors;       // [0]=lo count, [1]=hi count; self-resetting
  void* partials;                    // >= grid PassPartial
  unsigned int* ticket;              // self-resetting grid ticket
  DevPass* out;                      // device (or mapped host) result
  unsigned long long* done;          // optional (mapped host) mailbox flag: set to seq after *out is written
  unsigned long long seq;
};

// Segmented compaction (a4, warp-private output regions).  The compacting pass is run by a fixed
// number of warps Wtot; warp W writes the ]y_lo,t[ elements it sees upward from out[W*R] and the
// ]t,y_hi[ elements downward from out[(W+1)*R - 1], and records both runs in seg[W].  A later pass
// over the kept half lets warp W read run `side` of seg[W] (same Wtot, same R), so no atomics, no
// block barriers and no data movement between warps are ever needed.
struct SegEntry {
  unsigned long long off[2];  // start offset (elements) of the lo / hi run
  unsigned long long cnt[2];  // lengths
};
struct SegArgs {
  struct KelleyState* ks;      // device loop (§8f-3): input, bracket, output taken from *ks
  // input: contiguous (seg_in == nullptr: x[0..n), warp-strided groups) or segmented
  const void* x;
  uint64_t n;                  // contiguous: elements; segmented: total (diagnostic)
  const SegEntry* seg_in;
  int side_in;
  double t, y_lo, y_hi;
  // output: dense_out == 0: warp regions of R elements in `out`, runs recorded in seg_out;
  //         dense_out == 1: appended to z (lo up from 0, hi down from z_cap-1) via cursors
  int dense_out;
  void* out;
  uint64_t R;
  SegEntry* seg_out;
  unsigned long long* cursors;
  uint64_t z_cap;
  void* partials;
  unsigned int* ticket;
  DevPass* out_tuple;
  unsigned long long* done;    // optional mailbox flag (see PassArgs)
  unsigned long long seq;
  const void* cuts;            // cut pass (R26): device pointer to the two cuts t_a <= t_b
  const struct ChainState* chain;  // device chain (§8f-3): skip unless chain->ok[0]
  // device chain: the finishing thread also takes the chain's next decision (step 1)
  struct ChainState* chain_out;
  struct ChainMail* chain_mail;
  unsigned long long chain_seq;
  uint64_t chain_k, chain_cap;
};

// Device-side chain of the usual selection (NEXT row §8f-3): init -> cut pass -> radix select,
// launched back to back; the step kernels between them decide on the device whether the usual
// path holds (ok) and hand the next kernel its array size m and rank r.  The host consumes a
// step's result only if its own driver asks for exactly that step.
struct ChainState {
  unsigned long long ok[2];   // [0]: cut pass on the init's copy, [1]: radix select of the cut's copy
  unsigned long long m[2], r[2];
  unsigned long long le_base;  // #x <= t_lo of the init (global count below the current array)
};
// the host-visible copy the step kernels publish (mapped memory), with a sequence flag each
struct ChainMail {
  unsigned long long ok[2], m[2], r[2];
  unsigned long long seq[2];
};

struct InitArgs {
  const void* x;
  uint64_t n;
  void* partials;
  unsigned int* ticket;
  DevInit* out;
  const void* t0;   // device pointer to the two extra cuts t_lo, t_hi (elements of the dtype), or nullptr
  unsigned long long* done;  // optional mailbox flag (see PassArgs)
  unsigned long long seq;
  // device chain (§8f-3, init_seg_kernel): the finishing thread also takes the chain's step 0
  struct ChainState* chain;
  struct ChainMail* chain_mail;
  unsigned long long chain_seq;
  uint64_t chain_k, chain_cap;
  int chain_direct;  // 1: the radix select runs right behind the init on its copy (gated by decision 1)
  // chain_direct: the init also counts the radix select's first digit round on its copy — a shared-
  // memory histogram of the copied elements' top digit, merged into hist (2048 words); the chained
  // radix select starts at round 1 and picks that digit itself
  unsigned int* hist;
  // vbin: the copy's first digit is its VALUE-LINEAR bin in ]t_lo, t_hi[ (2048 equal-width bins,
  // monotone in the value) instead of the top 11 key bits, whenever t_hi - t_lo is finite (an open
  // cut, R31, falls back to the key digit); the chained finish is vbin_finish_kernel
  int vbin;
  // init_seg_kernel without the fp sums: the grid's totals accumulated by atomics here (8 words,
  // zero on entry, left zero) instead of a last-CTA fold of every CTA's partial; nullptr: the fold
  unsigned long long* acc;
};

struct LaunchShape {
  int num_sms;
  int grid_pass[2][3];   // [dtype][mode]
  int grid_init[2];
  int grid_hist[2];
  int grid_seg[2];
  int coop_max[2][2][2];  // [dtype][segmented][1024-thread]: co-resident CTAs of the cooperative radix select
};

// ---- device-resident Kelley loop (NEXT row §8f-3) ---------------------------------------------
// The Kelley iterations of Algorithm 1 without a host round trip: ONE CUDA graph per
// (ctx, dtype) whose WHILE node runs {step kernel; IF hot: pass_kernel; IF compacting:
// seg_pass_kernel (bracket tests / all inside)} until the step kernel ends the loop, followed by
// the radix rounds of the exact finish (segmented or dense input) under IF nodes.  Every kernel
// reads its array, bracket and output from this state; the step kernel (one thread) is drive()'s
// Kelley step: exact rank test, tightest cuts, interior-mean iterate, snap to the dtype, ordered-key
// safeguard, compaction / adoption of the kept half, the hand-off to the exact select.
struct KRow {  // == cpsel_trace_row
  double t, F;
  unsigned long long c_lt, c_eq, interior, scanned, written;
  unsigned kind, compacted;
  double kernel_ms;
};
constexpr int kKelleyMaxRows = 256;
// what the host reads when the loop is over (mapped pinned memory, written by the step kernel)
struct KelleyReport {
  int error;
  unsigned exit_reason, passes, cp_iters, fallback, launches, n_rows, pad;
  unsigned long long bytes_moved, z_count;
  KRow rows[kKelleyMaxRows];
};
struct KelleyState {
  // configuration (host-written)
  unsigned long long n, k, z_cap, select_cap, dense_cap, max_iters, seq;
  double wP, wN;
  const void* x;
  void* sb[2];
  SegEntry* st[2];
  void* zb[2];
  unsigned long long cap, R;
  int dt, record;
  double* vout;                   // mapped mailbox: the value, then `seq` into *done_flag
  unsigned long long* done_flag;
  KelleyReport* rep;              // mapped: the trace rows and counters
  // driver state (host-written at the hand-off, then the step kernel's)
  double yL, yR, t, N_L, P_R, tq;
  unsigned long long c_le_L, c_lt_R, m, D_lo, it;
  int on_z, exact, bisect, slow, free_step, kind;
  // current array / the pass being run
  const void* cur;
  unsigned long long n_cur;
  const SegEntry* cur_tab;
  int cur_seg, cur_side, cur_sbuf, cur_dbuf, tgt, last_dense, compact, dense, inside, pending;
  DevPass tuple;                  // the pass's result (grid finish)
  // outcome
  int done, error;
  unsigned exit_reason, passes, cp_iters, fallback, launches, n_rows;
  double value;
  unsigned long long bytes_moved, t_start_ns, z_count;
  // the exact finish handed to the radix rounds
  const void* sel_base;
  const SegEntry* sel_tab;
  int sel_side, sel_seg;
  unsigned long long sel_m, sel_r;
};
// Build the graph for dtype on ctx scratch (partials, ticket, cursors, radix state / histogram).
cudaError_t kelley_graph_build(int dtype, const struct LaunchShape& s, KelleyState* ks, void* partials,
                               unsigned* ticket, unsigned long long* cursors, RadixState* rstate, unsigned* hist,
                               cudaGraphExec_t* out);

// Query occupancy and fill the persistent grid sizes (multiples of the SM count).
cudaError_t query_shapes(int device, LaunchShape* shape);
size_t partial_bytes_needed(const LaunchShape& shape);

// checked=false: fast form (nonfinite stays 0; a non-finite input shows as a non-finite S/min/max);
// checked=true: counts non-finite elements exactly.
// Warps of the segmented kernel (fixed per dtype; every level of one selection uses the same).
int seg_total_warps(int dtype, const LaunchShape& s);
// Region size R (elements per warp) able to hold any compaction of an n-element contiguous array.
uint64_t seg_region(int dtype, uint64_t n, const LaunchShape& s);
// The init reduction + both extra cuts + the copy_if of ]t_lo, t_hi[ into run 0 of each warp's
// region (a.out / a.R / a.seg_out) in one read (R23); DevInit.pad = interior elements written,
// has_cut = 3.  ia.t0 must hold the two cuts.
// sums: also N_lo = sum (t_lo-x)^+ and P_hi = sum (x-t_hi)^+ (has_cut = 7), else has_cut = 3 (R25).
cudaError_t launch_init_seg(int dtype, const InitArgs& ia, const SegArgs& a, const LaunchShape& s, cudaStream_t st,
                            bool sums);
// inside: every input element lies strictly inside the bracket (input = a kept half)
cudaError_t launch_seg_pass(int dtype, const SegArgs& a, bool inside, const LaunchShape& s, cudaStream_t st);
// R26: sample cuts of a compacted current array and the cut pass over it.
// launch_sample_seg: t0[0..1] <- the two sample cuts around local rank r of the m-element
// segmented array (runs `side` of tab[0..Wtot)).
// R29: t0[0..2] <- the cuts around local rank r (1-based) of the m-element current array and the
// sample estimate, from 32768 (f32) / 16384 (f64) evenly strided samples: contiguous x (tab ==
// nullptr) or the runs `side` of the segmented array (base x, tab[0..Wtot)).
// keys: device scratch of kSampleKeyBytes (the gathered sample).  Two launches: a many-CTA gather of
// the sample keys and a one-CTA radix select of the three sample order statistics.
constexpr size_t kSampleKeyBytes = 32768 * 4 > 16384 * 8 ? 32768 * 4 : 16384 * 8;
// small: 8192 (f32) / 4096 (f64) samples instead (the cut passes over an already small bracket).
// allow_open: a cut whose sample rank falls off the sample (extreme k) becomes -/+FLT_MAX (DBL_MAX),
// so the target cannot lie beyond it; off when the init pass sums (x - t_lo)^+ etc. for F (R25).
cudaError_t launch_sample_select(int dtype, const void* x, uint64_t m, const SegEntry* tab, int side, int Wtot,
                                 uint64_t r, void* t0, void* keys, cudaStream_t st, bool small = false,
                                 const ChainState* chain = nullptr, int which = 0, bool allow_open = true);

// smax (<= 1024): samples drawn; keys_out != nullptr: write the sorted sample keys (order-preserving
// 64-bit keys, padding ~0) there instead of picking cuts (pooled across ranks, R28).
cudaError_t launch_sample_seg(int dtype, const void* base, const SegEntry* tab, int side, int Wtot, uint64_t m,
                              uint64_t r, void* t0, cudaStream_t st, uint32_t smax = 1024,
                              unsigned long long* keys_out = nullptr);
// launch_cut_pass: one read of the current array (a.x / a.seg_in / a.side_in as for
// launch_seg_pass, every element inside the bracket) at the two cuts a.cuts = {t_a, t_b}:
// #x<=t_a, the copy_if of ]t_a, t_b[ (segmented run 0 of each warp region, or dense from z[0]) and
// the sample estimate.  Result tuple: c_lt = #x<=t_a, c_lo = z_lo = #]t_a,t_b[, L_lo = estimate,
// pred = t_a, succ = t_b, c_eq = 1 if a dense copy would not fit z_cap (then it is not kept).
cudaError_t launch_cut_pass(int dtype, const SegArgs& a, const LaunchShape& s, cudaStream_t st);

// Sharded sample cuts (R28): each rank gathers ms <= m evenly strided VALUES of its current array
// (contiguous x, or runs `side` of tab[0..Wtot)) into out[0..ms); the ranks' shares are all-gathered
// into one pooled array of <= pool_sample_size() values, and launch_pool_pick finds, on every rank
// from the same bytes, t0[0..2] = the cuts around rank r of the m_rank-element global array and the
// estimate (the one-GPU cluster select, with the rank scaled by m_rank instead of the sample size).
// launch_seg_pack: the runs `side` of a segmented array packed contiguously into out (run order).
uint64_t pool_sample_size(int dtype, bool small);
// R40: the one-GPU sample cuts in one cooperative launch (ms / 1024 <= 148 CTAs; ms % 1024 == 0):
// the ms strided samples of x[0..m) (launch_pool_gather's positions) and the three sample ranks of
// launch_pool_pick, written to t0[0..2] — the same values as gather + pick.  scratch:
// sample_grid_words() words, zero on entry, left zero.
size_t sample_grid_words();
cudaError_t launch_sample_grid(int dtype, const void* x, uint64_t m, uint64_t ms, uint64_t m_rank, uint64_t r,
                               void* t0, unsigned* scratch, cudaStream_t st, bool allow_open);
cudaError_t launch_pool_gather(int dtype, const void* x, uint64_t m, const SegEntry* tab, int side, int Wtot,
                               uint64_t ms, void* out, cudaStream_t st);
cudaError_t launch_pool_pick(int dtype, const void* pooled, uint64_t ms, uint64_t m_rank, uint64_t r, void* t0,
                             cudaStream_t st, bool small, bool allow_open = true);
cudaError_t launch_seg_pack(int dtype, const void* base, const SegEntry* tab, int side, int Wtot, void* out,
                            cudaStream_t st);
// bytes (a multiple of 8) of device src copied to mapped host memory (device view dst_mapped), then
// seq published to *flag (mapped): the host spins on the flag instead of synchronising the stream
cudaError_t launch_publish(const void* src, void* dst_mapped, size_t bytes, unsigned long long* flag,
                           unsigned long long seq, cudaStream_t st);

cudaError_t launch_init(int dtype, const InitArgs& a, const LaunchShape& s, cudaStream_t st, bool checked);
// t0[0], t0[1] <- the sample quantiles bracketing rank k (1024 strided samples of x, one CTA)
cudaError_t launch_sample_cut(int dtype, const void* x, uint64_t n, uint64_t k, void* t0, cudaStream_t st,
                              uint32_t smax = 1024, unsigned long long* keys_out = nullptr);
cudaError_t launch_pass(int dtype, const PassArgs& a, const LaunchShape& s, cudaStream_t st);

// Radix select of the r-th smallest (1-based) of z[0..m) (any element alignment).
// hist: >= kRadixHistWords unsigned ints, zero on entry, left zeroed ([0, 2048): the per-launch
// rounds; [2048, 4096): hist0, the round-0 counts of the init pass; [4096, ...): the cooperative
// form's three rotating histograms and its grid barrier).  state: device RadixState.
// All rounds run in ONE cooperative launch when the grid fits co-resident (CPSEL_RADIX_COOP=0: one
// launch per round).
// On completion state->value holds the element (as double).
// vout/done/seq (optional): the last round also writes the value to *vout (mapped host memory)
// and then sets *done = seq.
// tab != nullptr: the input is the runs `side` of the segmented array based at z (tab[0..Wtot),
// the segmented grid).  One launch per digit (f32: 3, f64: 6); the last CTA of each picks the digit
// (ticket: a self-resetting grid counter).
// §8f-3 small arrays: x_(r) of x[0..m) (m <= exact_cluster_cap) by ONE 8-CTA cluster launch (exact
// radix select in registers + DSMEM histograms); *vout = value (canonical +0), *bad_out = #NaN/Inf,
// then `seq` published to *done.
// + the value-binned finish (launch_vbin_finish): 16 state words at kVbState, then kVbCap elements
// (8 bytes each) of the target bin's copy at kVbBuf
constexpr int kVbState = 4096 + 3 * 2048 + 64;
constexpr int kVbCap = 16384;
constexpr int kVbBuf = kVbState + 16;
constexpr int kRadixHistWords = kVbBuf + 2 * kVbCap;
uint64_t exact_cluster_cap(int dtype);
cudaError_t launch_exact_cluster(int dtype, const void* x, uint64_t m, uint64_t r, double* vout,
                                 unsigned long long* bad_out, unsigned long long* done, unsigned long long seq,
                                 cudaStream_t st);
// The direct chain's exact finish behind an init pass with vbin = 1 (§8f-3, a5): every CTA picks the
// bin holding the rank from the init's 2048 counts (value-linear bins, or top key digits after an
// open cut), ONE pass over the init's segmented copy takes the bin's key range and, when the bin holds
// <= kVbCap elements, copies them; the last CTA finishes: a bin of one value is the answer, a small
// bin is radix-selected in shared memory from the common prefix of its key range on; a larger bin of
// several values sets *fallback (the host then runs launch_radix_select on the copy).  hist: the
// context's kRadixHistWords block (hist0 at +2048 is cleared, the state left zero).
cudaError_t launch_vbin_finish(int dtype, const void* z, const SegEntry* tab, const void* cuts, unsigned* hist,
                               const LaunchShape& s, cudaStream_t st, const ChainState* chain, double* vout,
                               unsigned long long* fallback, unsigned long long* done, unsigned long long seq);
cudaError_t launch_radix_select(int dtype, const void* z, uint64_t m, uint64_t r, RadixState* state,
                                unsigned int* hist, const LaunchShape& s, cudaStream_t st,
                                double* vout, unsigned long long* done, unsigned long long seq,
                                const SegEntry* tab, int side, unsigned int* ticket,
                                const ChainState* chain = nullptr, int first_round = 0,
                                unsigned int* hist0 = nullptr, uint64_t m_hint = 0);

// Step a8: per-column k-th smallest of S (n x C column-major, float32), one CTA per column.
struct BatchArgs {
  const float* S;
  uint64_t n;
  uint32_t C;
  uint64_t k;
  float* out;                  // device, C results
  float* scratch;              // grid x 2 x cap floats (per-CTA ping-pong compaction buffers)
  uint64_t cap;                // elements per buffer; a column compacts once its interior <= cap
  unsigned* next_col;          // work counter, zero on entry
  unsigned long long* stats;   // [0] passes, [1] bytes, [2] safeguard trips, [3] non-finite columns
  uint32_t max_iters;
  // fused LMS input (§8f-2): the fused residual pass already evaluated, per column, the two sample
  // cuts f_cuts[4j], f_cuts[4j+1] (R23) — #s <= t_lo in f_le[j], the copy of ]t_lo, t_hi[ at
  // f_z + j*f_zcap (f_cursor[j] elements) — so the kernel starts from that bracket instead of
  // reading a column of S (the inputs were checked finite and overflow-free beforehand).  A column the copy cannot finish
  // (target outside the cuts, copy overflow) is appended to fail_list and gets no output.
  const float* f_cuts = nullptr;
  const unsigned long long* f_le = nullptr;
  const unsigned long long* f_cursor = nullptr;
  const float* f_z = nullptr;
  uint64_t f_zcap = 0;
  unsigned* fail_list = nullptr;
  unsigned* fail_count = nullptr;
  const unsigned* out_map = nullptr;  // result of column c goes to out[out_map[c]] (nullable)
};
cudaError_t launch_batched_select(const BatchArgs& a, int grid, cudaStream_t st);
// Per column j of the LMS problem: t_lo, t_hi, t_mid (cuts[4j..4j+2]) around the sample order
// statistics bracketing rank k (R23 applied to the fused residual pass), from the residuals of ms
// sample rows per column (Ss: C x ms, column-major).  ms <= 16384.
cudaError_t launch_lms_cuts(const float* Ss, uint32_t ms, uint64_t n, uint32_t C, uint64_t k, float* cuts,
                            cudaStream_t st);
int batched_blocks_per_sm();

}  // namespace cpsel
