// kernels.cuh -- device state, filters, the exact candidate pipeline, and the
// per-round commit of the round-synchronous propagation on sm_100a.
//
// One round = run_round + process_block of the reference
// (par_engine.cpp:126-200), in three launches:
//
//   k_sell    phase 1 (sell.cuh): every activity chain of the round -- a row
//             of <= nnz_budget entries, or a chunk of a longer row -- by one
//             thread over a sliced-ELL copy, in entry order; row check,
//             filters, and queueing of the rows that may tighten.
//   k_cand    phase 2 (cand.cuh): the queued rows' entries, spread over lanes,
//             filtered, the survivors through the exact candidate pipeline
//             and committed by 64-bit atomics.
//   k_commit  per variable: change count, crossing check, next snapshot
//             record; the last CTA takes the round decision and sets the CUDA
//             graph's WHILE condition (no host round trip per round).
//
// All activity sums follow cpu_par's order exactly, so results are
// bit-identical to the reference (tests/test_gpu_parity.py).
#pragma once

#include <math_constants.h>

#include "propcore.cuh"

namespace pgb {

constexpr int kCommitThreads = 256;

// Device-resident loop state.
struct DevState {
  unsigned long long round_changes;  // changes of the current round
  long long total_changes;
  int32_t infeasible;                // raised by any kernel of the current round
  int32_t round;                     // rounds executed
  int32_t status;                    // -1 running, else PG_* status
  int32_t done;
  uint32_t ticket;                   // last-CTA election in k_commit
  uint32_t ticket_reset;             // last-CTA election in k_reset
  int32_t crossed;
  int32_t wl_short;                  // phase-2 queue lengths of the current round
  int32_t wl_long;
  int32_t work;                      // k_sell slice counter
  int32_t work2;                     // k_sell unit-batch counter (worklist rounds)
  int32_t cand_work;                 // k_cand ticket counter
  int32_t full;                      // 1: every work item is dirty (first round)
  int32_t frac_any;                  // an integral column has a fractional start bound
  int32_t frac_tmp;                  // k_reset's accumulator of frac_any
  int32_t nchg[2];                   // changed-column list lengths, by round parity
  long long chg_deg[2];              // sum of the listed columns' degrees (rows to mark)
  long long unit_wsum;               // sum of the units' worklist weights (set up once)
  int32_t nwide[2];                  // marked multi-lane unit list lengths, by round parity
  int32_t nmid[2];                   //   of which mid-length units (at the list's back)
  int32_t nunit[2];                  // marked one-lane unit list lengths, by round parity
  int32_t ntouch;                    // columns merged into this (worklist) round
  int32_t sparse_commit;             // the last commit visited only the touched columns
  int32_t sparse_round;              // this round is a worklist round (set by the dense k_sell)
  long long last_changes;            // changes of the previous round (worklist heuristics)
  uint32_t bar_count;                // grid barrier of the persistent round loop (loop.cuh)
  uint32_t bar_gen;
  int32_t bad_input;                 // a col_idx outside [0, n) (set at session setup, sticky)
  // row shards, unrolled graphs (engine.cu build_shard_graphs)
  int32_t stall;                     // a delta exchange overflowed its capacity: the round is
                                     // held (not committed) until the host resumes it densely
  int32_t resume;                    // the next round resumes a held one: exchange + commit only
  int32_t delta_rounds;              // rounds merged by the sparse delta exchange (this solve)
};

// Row shards run graphs of R unrolled rounds (no conditional nodes around
// NCCL calls); a round's kernels return at once once the solve is decided
// (done) or held (stall), and the compute phases also in a resumed round.
// Only those sessions pay the state loads (kUnrolledFlag in the kernel's
// DevCfg); the other loops never launch a round after the decision.
constexpr uint32_t kUnrolledFlag = 0x40000000u;
// Programmatic dependent launch (engine.cu pdl()): wait until the previous
// kernel of the stream has completed and its writes are visible, then let
// the next kernel's CTAs be scheduled.  Both are no-ops for a kernel
// launched without the attribute.  Every round kernel starts with this,
// before any access to data an earlier kernel wrote.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ bool round_off(DevState* st, const DevCfg& c) {
  return (c.flags & kUnrolledFlag) && (ld_gpu(&st->done) | ld_gpu(&st->stall)) != 0;
}
// the exchange kernels of row-sharded rounds always check
__device__ __forceinline__ bool state_off(DevState* st) {
  return (ld_gpu(&st->done) | ld_gpu(&st->stall)) != 0;
}
__device__ __forceinline__ bool compute_off(DevState* st, const DevCfg& c) {
  return (c.flags & kUnrolledFlag) &&
         (ld_gpu(&st->done) | ld_gpu(&st->stall) | ld_gpu(&st->resume)) != 0;
}

// Device-side worklist (PG_FLAG_WORKLIST): a round only
// visits work items containing a row with a variable changed in the previous
// round.  Exact under snapshot semantics: a row none of whose bounds changed
// yields the same candidates, already accepted or rejected against the same
// bounds (the reference's marking, seq_engine.cpp:29,37-38,77, by analogy).
// Rows are marked: k_commit lists the changed columns (warp-aggregated
// appends), k_mark walks each changed column's rows (column index built at
// session init) and sets the row's flag for the next round.  k_tiles
// compacts the marked rows of each warp tile; a segment group is processed
// when a row of one of its segments is marked.
struct Dirty {
  const int32_t* col_ptr;   // [n+1] column -> rows (sorted row space) containing it
  const int32_t* col_row;
  uint8_t* row_flag;        // [2][ms], by round parity (ms = m rounded up to 16)
  int32_t* chg_list;        // [2][n] changed columns of a round
  int32_t m, ms, n, first_seg_row;
  int32_t enabled;
  // the units of the marked rows, so a worklist round visits only those
  // (sell.cuh): row / chunk -> sliced-ELL unit
  const int32_t* row_unit;   // [m] unit of a whole row, -1 for a split row
  const int32_t* part_unit;  // [partials] unit of each chunk of a split row
  const int32_t* sfirst;     // split-row slot -> first partial (+1 sentinel)
  const int32_t* unit_slice; // [units] slice of a multi-lane unit, -1 for a one-lane unit
  int32_t* wide_list;        // [2][nunits] marked multi-lane units, by round parity
  int32_t* unit_list;        // [2][nunits] marked one-lane units
  int32_t nslices, nunits;
  int32_t dense_nchg;        // more changed columns than this: next round is a full sweep
  double dense_deg;          //   or when (entries to mark) x (mean unit weight) > dense_deg (F m)
  long long list_gate;       // a full sweep after more changes than this builds no list
  // a worklist round while w_lane nunit + w_wide nwide + w_mid nmid <= w_all nunits
  int32_t w_lane, w_wide, w_mid, w_all;
  int32_t unrolled;          // row-shard graphs of unrolled rounds (round_off)
  int32_t mark_batch;        // k_mark: B columns per warp once there are mark_batch x B per warp
};

// Row r (sorted) becomes marked for the round of parity `par` (exactly once:
// the byte flag is set with an atomic on its word).  Its units go on that
// round's lists: one-lane units (lg = 0, the bulk of the rows) on the unit
// list (a lane each), longer units on the wide list (a warp each).
__device__ __forceinline__ bool mark_row(uint8_t* flag, int r) {
  uint32_t* w = reinterpret_cast<uint32_t*>(flag) + (r >> 2);
  const uint32_t bit = 1u << (8 * (r & 3));
  if (ld_gpu(w) & bit) return false;
  return !(atomicOr(w, bit) & bit);
}
__device__ __forceinline__ void mark_row_units(const Dirty& D, int r, int par, DevState* st) {
  int32_t* ul = D.unit_list + (size_t)par * D.nunits;
  int32_t* wl = D.wide_list + (size_t)par * D.nunits;
  // unit_slice: -1 one-lane unit, -2 mid-length unit (appended from the
  // wide list's back), else a long unit
  auto one = [&](int u) {
    const int us = D.unit_slice[u];
    if (us == -1) ul[atomicAdd(&st->nunit[par], 1)] = u;
    else if (us == -2) wl[D.nunits - 1 - atomicAdd(&st->nmid[par], 1)] = u;
    else wl[atomicAdd(&st->nwide[par], 1)] = u;
  };
  const int u = D.row_unit[r];
  if (u >= 0) {
    one(u);
  } else {
    const int rs = r - D.first_seg_row;
    for (int p = D.sfirst[rs]; p < D.sfirst[rs + 1]; ++p) one(D.part_unit[p]);
  }
}

// Start of the next solve (device memory, set by stream-ordered copies):
// warm = 1 for a branch-and-bound node started from the session's root
// fixpoint, with `nvars` overridden columns vars[i] -> [lo[i], up[i]].
struct NodeCtl {
  int32_t warm;
  int32_t nvars;
  const int32_t* vars;
  const double* lo;
  const double* up;
};

// Per-column snapshot record, gathered with one 256-bit load per entry.
//   lo, up  the round's input bounds (bounds_in of par_engine.cpp:162)
//   q       filter coefficient (see entry_x), +inf = always examine
//   flags   bit 0: integral column
struct __align__(32) Snap {
  double lo;
  double up;
  double q;
  long long flags;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// read-only path: the snapshot is constant for the kernel's lifetime (every
// per-round kernel; NOT the persistent loop, see ld_snap_coh)
__device__ __forceinline__ void ld_snap(const Snap* p, double& lo, double& up, double& q) {
  [[maybe_unused]] long long f;  // the flags word rides along in the 256-bit load
  asm volatile("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];"
               : "=d"(lo), "=d"(up), "=d"(q), "=l"(f)
               : "l"(p));
}
// coherent path (L2, weak loads ordered by the grid barrier's fences): the
// persistent loop rewrites the snapshot between its rounds inside one kernel
__device__ __forceinline__ void ld_snap_coh(const Snap* p, double& lo, double& up, double& q) {
  const double2 b = __ldcg(reinterpret_cast<const double2*>(p));
  lo = b.x;
  up = b.y;
  q = __ldcg(&p->q);
}

// ---- exactness-preserving filters -----------------------------------------------
// (only compute candidates that may improve.)  For an entry
// with slack S = rhs - min_activity, the rhs-side candidate of the bound it
// touches (ub for a > 0, lb for a < 0) equals lb + S/a resp. ub - S/|a|, and
// tighten() can accept it only if S < |a| (ub - lb - thr), where thr >=
// abs + rel (the smallest possible step, propcore.hpp:168) for continuous
// variables and thr = integrality_eps for integral ones with integral bounds
// (floor(c + eps) < ub - step forces c < ub - eps).  Symmetrically for the
// lhs side with S = max_activity - lhs.  The tests keep a margin of 2^-40
// times the operand magnitudes, far above the few-ulp rounding error of the
// reference pipeline, so whatever they skip the reference would have
// rejected too.  q precomputes, per column,
//   q = (ub - lb - thr) + 2^-40 (|lb| + |ub|)
// (+inf for an infinite bound or an integral column with a fractional
// bound), so an entry's term is x = |a| q.
constexpr double kMargin = 0x1p-40;

__device__ __forceinline__ double column_q(double lo, double up, bool integral,
                                           const DevCfg& c) {
  if (isinf(lo) || isinf(up)) return CUDART_INF;
  if (integral && (lo != floor(lo) || up != ceil(up))) return CUDART_INF;
  const double thr = integral ? c.int_eps : c.imp_abs + c.imp_rel;
  return ((up - lo) - thr) + (fabs(lo) + fabs(up)) * kMargin;
}

// Row thresholds: an entry can tighten through the rhs side only if
// x >= tr (or, with exactly one infinite min-contribution, if it is that
// entry), likewise lhs.  A side that cannot tighten anything (infinite side,
// or two or more infinite contributions) is switched off.
struct RowFilter {
  double tr, tl;
  uint8_t mode;  // bit0 rhs threshold on, bit1 lhs threshold on, bit2 rhs one-inf, bit3 lhs one-inf
};

__device__ __forceinline__ RowFilter row_filter(const Act& act, double lhs, double rhs) {
  RowFilter f = {0.0, 0.0, 0};
  if (!isinf(rhs)) {
    if (act.min_i == 0) {
      f.tr = (rhs - act.min_f) - (fabs(rhs) + fabs(act.min_f)) * kMargin;
      if (isnan(f.tr)) f.tr = -CUDART_INF;  // must not skip anything
      f.mode |= 1;
    } else if (act.min_i == 1) {
      f.mode |= 4;
    }
  }
  if (!isinf(lhs)) {
    if (act.max_i == 0) {
      f.tl = (act.max_f - lhs) - (fabs(lhs) + fabs(act.max_f)) * kMargin;
      if (isnan(f.tl)) f.tl = -CUDART_INF;
      f.mode |= 2;
    } else if (act.max_i == 1) {
      f.mode |= 8;
    }
  }
  return f;
}

__device__ __forceinline__ bool row_may(const RowFilter& f, double xmax) {
  return (f.mode & 12) || ((f.mode & 1) && !(f.tr > xmax)) || ((f.mode & 2) && !(f.tl > xmax));
}

// pmin_inf / pmax_inf: the entry's min/max contribution is infinite
__device__ __forceinline__ bool entry_may(const RowFilter& f, double x, bool pmin_inf,
                                          bool pmax_inf) {
  return ((f.mode & 1) && !(f.tr > x)) || ((f.mode & 2) && !(f.tl > x)) ||
         ((f.mode & 4) && pmin_inf) || ((f.mode & 8) && pmax_inf);
}

// ---- exact candidate pipeline ---------------------------------------------------
// fire-and-forget 64-bit max at L2 (no load before it: a candidate never
// waits on the current merged value)
__device__ __forceinline__ void red_max(long long* p, long long k) {
  asm volatile("red.relaxed.gpu.global.max.s64 [%0], %1;" ::"l"(p), "l"(k) : "memory");
}

// A work ticket taken by one lane.  An add of 1 in a one-lane branch (even
// as inline PTX) is turned by ptxas into a warp-aggregated atomic whose
// result is shuffled to the active lanes right away, so the issuing warp
// waits for the atomic's round trip there (4-5 % of the full sweep's stall
// samples); an increment with a wrap bound is not aggregated, and its result
// waits in a register until the caller's shuffle, after the work it was
// taken under.  (The counters are reset every round, far below the bound.)
__device__ __forceinline__ int ticket(int32_t* p) {
  unsigned r;
  asm volatile("atom.relaxed.gpu.global.inc.u32 %0, [%1], 0x7fffffff;" : "=r"(r) : "l"(p) : "memory");
  return (int)r;
}

// Worklist rounds: the columns a round merged into, so the commit visits
// only those (each column listed once per round).
struct Touch {
  uint32_t* flag;   // [n]
  int32_t* list;    // [n]
  int32_t* count;
};
__device__ __forceinline__ void touch_col(const Touch* t, int j) {
  if (t && !atomicOr(&t->flag[j], 1u)) t->list[atomicAdd(t->count, 1)] = j;
}

__device__ __forceinline__ void commit_side(long long* key_out, int j, int kind, double cl,
                                            double cu, const Touch* t = nullptr) {
  if (kind) touch_col(t, j);
  // merge_lower / merge_upper (par_engine.cpp:56-71) as exact 64-bit max/min
  if (kind & 1) {
    const long long k = key_enc(canon0(cl));
    long long* p = key_out + 2 * (size_t)j;
    red_max(p, k);
  }
  if (kind & 2) {
    // upper bounds are kept as NEGATED keys so that one max-reduction merges
    // both sides (one NCCL all-reduce on the row-sharded path)
    const long long k = -key_enc(canon0(cu));
    long long* p = key_out + 2 * (size_t)j + 1;
    red_max(p, k);
  }
}

// residual -> candidates -> tighten vs the snapshot -> merge
// (propcore.hpp:78-208, par_engine.cpp:158-168).  Returns true on EmptyDomain.
__device__ __forceinline__ bool entry_pipeline(const Act& act, double a, double lo, double up,
                                               double lhs, double rhs, int32_t cx,
                                               long long* key_out, const DevCfg& c,
                                               const Touch* t = nullptr) {
  double min_res, max_res, cl, cu;
  residual(act, a, lo, up, min_res, max_res);
  candidates(a, lhs, rhs, min_res, max_res, cx < 0, c, cl, cu);
  const int kind = tighten(lo, up, cl, cu, c);
  if (kind == 4) return true;  // EmptyDomain: flag, skip the merge (par_engine.cpp:163-166)
  if (kind) commit_side(key_out, cx & 0x7fffffff, kind, cl, cu, t);
  return false;
}


// ---- round work items -----------------------------------------------------------
constexpr int kShortMax = 16;  // length classes of short rows (session row order)

// a chunk of nnz_budget entries of a row longer than nnz_budget (or the
// whole row when it is not split): wide_row_activities, par_engine.cpp:99-123
struct SegDesc {
  int32_t k0;
  int32_t len;
  int32_t out;    // partial index = first chunk of the row + chunk number
  int32_t rslot;  // segment-row slot
};

struct SegPartial {
  double min_f;
  double max_f;
  double xmax;
  int32_t min_i;
  int32_t max_i;
};

// sliced-ELL storage of the phase-1 chains (sell.cuh).  A slice holds
// H = 32 >> lg units of near-equal length; G = 1 << lg lanes share a unit
// (long units), lane = j * H + u takes entries i = t * G + j of unit u, and
// entry i of unit u lives at off + 32 * (i >> lg) + lane: every step of the
// warp is one contiguous 256 B (values) / 128 B (columns) request.
struct __align__(8) SliceDesc {
  long long off;    // first element of the slice in sv / sc / sw
  int32_t first;    // first unit
  int32_t width;    // longest unit of the slice
  int32_t steps;    // ceil(width / G)
  int16_t count;    // units in the slice (<= H)
  int8_t lg;        // log2 G
  int8_t pad;
};

// len entries; ref >= 0: the unit is the whole sorted row `ref`; ref < 0: it
// is chunk segment -(ref + 1) of a split row
struct UnitDesc {
  int32_t len;
  int32_t ref;
};

// pass-2 work: a piece (<= kCandPiece entries) of a row that may tighten
struct CandItem {
  int32_t row;  // sorted row
  int32_t k0;
  int32_t len;
  int32_t pad;
};
constexpr int kCandShort = 32;    // rows up to this length: batched 32 per warp
constexpr int kCandPiece = 128;   // longer rows: one warp per piece (one pass of 4 x 32)

struct RoundArgs {
  // phase 1: chains over the sliced-ELL copy
  const SliceDesc* slices;
  int32_t nslices;
  int32_t group_start;    // first slice of the grouped narrow region (sell.cuh)
  int32_t lg0_ustart;     // first unit / slice of the one-lane region
  int32_t lg0_sstart;
  int32_t nunits;
  const UnitDesc* units;
  const double* sv;
  const int32_t* sc;
  uint32_t* sw;           // per element: filter word of the round (sell.cuh)
  int32_t pad_col;        // = n: snapshot record {0, 0, 0, 0} of the padding entries
  // split rows: chunk partials, combined by the last chunk
  const SegDesc* segs;
  const int32_t* srow;    // segment-row slot -> sorted row
  const int32_t* sfirst;  // segment-row slot -> first partial (+1 sentinel)
  int32_t* row_done;      // per segment row: chunks finished this round
  SegPartial* partial;
  // phase 2 over the CSR copy (rows sorted by length class)
  const int32_t* row_ptr;
  const int32_t* colx;    // column | integral flag in bit 31
  const double* vals;
  const double* lhs;
  const double* rhs;
  Act* ract;              // [m] activity of the rows queued for phase 2
  int32_t* wl_short;      // queued rows with <= kCandShort entries
  CandItem* wl_long;      // pieces of longer queued rows
  const Snap* snap;
  const double2* bnd;     // [n+1] {lb, ub} of the round's input bounds (compact gathers)
  long long* key_out;
  DevState* st;
  Dirty dirty;
  Touch touch;            // worklist rounds: merged-into columns (kernels.cuh)
};

// RoundArgs with the gather record fixed at compile time (sell.cuh ld_col):
// kG = 0: 32 B snapshot records (q precomputed), 1: 16 B bounds records for
// rows dense in the columns or columns too many for 32 B records in L2,
// 2: 8 B float records (DevCfg::bf) when the bounds are floats (integral
// columns; C5: 5M columns = 40 MB instead of 80 MB); plain RoundArgs
// gathers the snapshot records
template <int kG>
struct RoundArgsG : RoundArgs {};
template <class RA>
constexpr bool gather16_v = false;
template <>
constexpr bool gather16_v<RoundArgsG<1>> = true;
template <class RA>
constexpr bool gather8_v = false;
template <>
constexpr bool gather8_v<RoundArgsG<2>> = true;
// the persistent round loop (loop.cuh): snapshot and bounds records are
// rewritten by the commit phase inside the same kernel, so its gathers use
// coherent loads (never ld.global.nc)
struct RoundArgsL : RoundArgs {};
template <class RA>
constexpr bool coherent_v = false;
template <>
constexpr bool coherent_v<RoundArgsL> = true;

// A row's activity is complete: row check (propcore.hpp:147-156, cpu_seq's
// verdicts), exactness-preserving row filter, and -- if some entry may
// tighten -- queue the row for phase 2.
template <bool kRowCheck>
__device__ __forceinline__ void finish_row(const RoundArgs& A, int r, const Act& act, double xmax,
                                           bool& inf_flag, const DevCfg& cfg) {
  const double l = A.lhs[r], h = A.rhs[r];
  if (kRowCheck && row_infeasible(act, l, h, cfg)) inf_flag = true;
  if (!row_may(row_filter(act, l, h), xmax)) return;
  A.ract[r] = act;
  const int k0 = A.row_ptr[r], len = A.row_ptr[r + 1] - k0;
  if (len <= kCandShort) {
    A.wl_short[atomicAdd(&A.st->wl_short, 1)] = r;
  } else {
    const int np = (len + kCandPiece - 1) / kCandPiece;
    const int pos = atomicAdd(&A.st->wl_long, np);
    for (int i = 0; i < np; ++i)
      A.wl_long[pos + i] = CandItem{r, k0 + i * kCandPiece, min(kCandPiece, len - i * kCandPiece), 0};
  }
}

// Last chunk of a split row: pairwise tree over its chunk partials in chunk
// order (par_engine.cpp:117-121), then finish_row.
template <bool kRowCheck>
__device__ void finish_split_row(const RoundArgs& A, int rs, bool& inf_flag, const DevCfg& cfg) {
  const int first = A.sfirst[rs];
  int np = A.sfirst[rs + 1] - first;
  volatile SegPartial* P = A.partial + first;
  double xmax = -CUDART_INF;
  for (int i = 0; i < np; ++i) xmax = fmax(xmax, P[i].xmax);
  while (np > 1) {
    int out = 0;
    for (int i = 0; i + 1 < np; i += 2) {
      const Act a = {P[i].min_f, P[i].max_f, P[i].min_i, P[i].max_i};
      const Act b = {P[i + 1].min_f, P[i + 1].max_f, P[i + 1].min_i, P[i + 1].max_i};
      const Act r = act_combine(a, b);
      P[out].min_f = r.min_f;
      P[out].max_f = r.max_f;
      P[out].min_i = r.min_i;
      P[out].max_i = r.max_i;
      ++out;
    }
    if (np & 1) {
      P[out].min_f = P[np - 1].min_f;
      P[out].max_f = P[np - 1].max_f;
      P[out].min_i = P[np - 1].min_i;
      P[out].max_i = P[np - 1].max_i;
      ++out;
    }
    np = out;
  }
  const Act act = {P[0].min_f, P[0].max_f, P[0].min_i, P[0].max_i};
  finish_row<kRowCheck>(A, A.srow[rs], act, xmax, inf_flag, cfg);
}

// ---- commit + round decision ------------------------------------------------------
template <int kThreads>
__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, int& f) {
  __shared__ unsigned long long s_sum[kThreads / 32];
  __shared__ int s_f[kThreads / 32];
  // the previous call's reads (thread 0) precede this call's writes
  // (compute-sanitizer racecheck: the persistent loop calls this every round)
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    f |= __shfl_xor_sync(0xffffffffu, f, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_sum[w] = v;
    s_f[w] = f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    int ff = 0;
    for (int i = 0; i < kThreads / 32; ++i) {
      t += s_sum[i];
      ff |= s_f[i];
    }
    v = t;
    f = ff;
  }
  return v;
}

// Per variable (par_engine.cpp:191-197): count sides with out != in, flag
// lo_out > up_out + abs, and write the next round's snapshot record.  The
// last CTA takes the round decision of run_parallel (par_engine.cpp:248-266).
// A worklist round visits only the marked rows' units when few are marked
// (sell.cuh); otherwise it is a full sweep.  Evaluated identically by the
// sweep and the commit of the round.
__device__ __forceinline__ bool round_is_sparse(DevState* st, const Dirty& D) {
  if (!D.enabled || ld_gpu(&st->full)) return false;
  const int par = (ld_gpu(&st->round) + 1) & 1;
  // worklist round while the marked units, weighted by their cost per unit
  // against a full sweep's (tuned on C2 / C5), stay below the full sweep
  const long long work = (long long)D.w_lane * ld_gpu(&st->nunit[par]) +
                         (long long)D.w_wide * ld_gpu(&st->nwide[par]) +
                         (long long)D.w_mid * ld_gpu(&st->nmid[par]);
  return work <= (long long)D.w_all * D.nunits;
}

// kList: a worklist round -- only the columns on the touched list (their
// flags are cleared); otherwise every column.
template <bool kList = false>
__device__ __forceinline__ void commit_body(Snap* __restrict__ snap, double2* __restrict__ bnd,
                                            const longlong2* __restrict__ key_out, int n,
                                            DevState* __restrict__ st, long long* __restrict__ per_round,
                                            const DevCfg& cfg, const Dirty& D,
                                            cudaGraphConditionalHandle cond, int use_graph,
                                            const Touch* touch = nullptr) {
  unsigned long long changes = 0, deg = 0;
  int inf = 0;
  const int R = ld_gpu(&st->round);  // rounds before this one
  const int nb = R & 1;                             // buffer of the next round's lists
  const int cb = nb ^ 1;                            // buffer this round consumed
  const int gstride = gridDim.x * blockDim.x;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int U = 4;  // columns in flight per thread
  const int lane = threadIdx.x & 31;
  const int nj = kList ? ld_gpu(touch->count) : n;
  // a full-sweep round after a round with many changes will have many too:
  // skip the changed-column list (the next round is a full sweep anyway)
  const bool list = D.enabled && (kList || !ld_gpu(&st->full) ||
                                  ld_gpu(&st->last_changes) <= D.list_gate);
  // the loop bound is warp-uniform (j0 - lane is), so the warp stays
  // converged for the list appends
  for (int j0 = gtid; j0 - lane < nj; j0 += U * gstride) {
    longlong2 kob[U];
    double2 inb[U];
    int jj[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = j0 + u * gstride;
      jj[u] = i < nj ? (kList ? touch->list[i] : i) : -1;
      if (jj[u] >= 0) {
        kob[u] = key_out[jj[u]];
        // the round's input bounds from the 16 B records (kept equal to
        // the snapshot's lo/up): half the bytes of the 32 B records' sectors
        inb[u] = bnd[jj[u]];
        if (kList) touch->flag[jj[u]] = 0u;
      }
    }
    int cu[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jj[u];
      int c = 0;
      if (j >= 0) {
        const longlong2 ko = kob[u];
        const double lo = key_dec(ko.x), up = key_dec(-ko.y);
        const double2 in = inb[u];
        // a change is a strict improvement, so comparing values is exact
        c = (lo != in.x) + (up != in.y);
        if (c) {
          changes += c;
          const long long fl = snap[j].flags;
          snap[j] = Snap{lo, up, column_q(lo, up, fl & 1, cfg), fl};
          bnd[j] = make_double2(lo, up);
          if (cfg.bf) cfg.bf[j] = fpair(lo, up);
        }
        if (lo > __dadd_rn(up, cfg.imp_abs)) inf = 1;
      }
      cu[u] = c;
    }
    if (list) {
      // changed columns of this round -> list (one atomic per warp for its
      // U columns per lane: the counter is a single address every warp of
      // the grid appends to), and the number of entries their marks will
      // visit (summed per thread, one atomic per CTA below)
      unsigned chm[U];
      int tot = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        chm[u] = __ballot_sync(0xffffffffu, cu[u] != 0);
        tot += __popc(chm[u]);
      }
      if (tot) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&st->nchg[cb], tot);
        base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (cu[u]) {
            const int j = jj[u];
            D.chg_list[(size_t)cb * D.n + base + __popc(chm[u] & ((1u << lane) - 1u))] = j;
            deg += (unsigned long long)(D.col_ptr[j + 1] - D.col_ptr[j]);
          }
          base += __popc(chm[u]);
        }
      }
    }
  }
  if (D.enabled) {
    // the consumed marks become the round-after-next's mark set
    uint32_t* f = reinterpret_cast<uint32_t*>(D.row_flag + (size_t)cb * D.ms);
    for (int i = gtid; i < D.ms / 4; i += gstride) f[i] = 0u;
  }
  int unused = 0;
  deg = block_sum<kCommitThreads>(deg, unused);
  changes = block_sum<kCommitThreads>(changes, inf);
  if (threadIdx.x == 0) {
    if (deg) atomicAdd(reinterpret_cast<unsigned long long*>(&st->chg_deg[cb]), deg);
    if (changes) atomicAdd(&st->round_changes, changes);
    if (inf) st->infeasible = 1;
    __threadfence();
    const uint32_t t = atomicAdd(&st->ticket, 1u);
    if (t == gridDim.x - 1) {
      // last CTA: the round decision of run_parallel (par_engine.cpp:248-266)
      __threadfence();
      const long long ch = (long long)atomicAdd(&st->round_changes, 0ull);
      // key_out[n].x: the all-reduced infeasibility of every rank (row shards)
      long long* slot = const_cast<long long*>(&key_out[n].x);
      const int infeasible = atomicAdd(&st->infeasible, 0) | (ld_gpu(slot) != 0);
      st_gpu(slot, 0);
      const int r = R + 1;
      st->round = r;
      if (r - 1 < cfg.round_limit) per_round[r - 1] = ch;
      st->total_changes += ch;
      int status = -1;
      if (infeasible) status = 2;                 // PG_INFEASIBLE
      else if (ch == 0) status = 0;               // PG_CONVERGED
      else if (r >= cfg.round_limit) status = 1;  // PG_ROUNDLIMIT
      st->status = status;
      st->done = status >= 0;
      st->round_changes = 0;
      st->infeasible = 0;
      st->ticket = 0;
      st->wl_short = 0;
      st->wl_long = 0;
      st->work = 0;
      st->work2 = 0;
      st->cand_work = 0;
      // many changed columns (or no list): the next round is a full sweep (no marks)
      // marks cost about their entries, and the rows they mark cost their
      // units' weights (round_is_sparse): with many, a full sweep is cheaper
      st->full = (!list || ld_gpu(&st->nchg[cb]) > D.dense_nchg ||
                  (double)ld_gpu(&st->chg_deg[cb]) * (double)ld_gpu(&st->unit_wsum) >
                      D.dense_deg * (double)D.nunits) ? 1 : 0;
      st->last_changes = ch;
      st->nchg[nb] = 0;  // the list k_mark consumed after the previous commit
      st->chg_deg[nb] = 0;
      st->nwide[cb] = 0;  // this round's unit lists
      st->nmid[cb] = 0;
      st->nunit[cb] = 0;
      st->ntouch = 0;
      st->sparse_commit = kList;
      st->resume = 0;
      __threadfence();
      if (use_graph) cudaGraphSetConditional(cond, status >= 0 ? 0u : 1u);
    }
  }
}

__global__ void __launch_bounds__(kCommitThreads)
    k_commit(Snap* __restrict__ snap, double2* __restrict__ bnd, const longlong2* __restrict__ key_out,
             int n, DevState* __restrict__ st, long long* __restrict__ per_round, const DevCfg cfg,
             const Dirty D, cudaGraphConditionalHandle cond, int use_graph, int allow_list) {
  // a worklist round of a single session is committed by k_commit_list; with
  // row shards every column may have moved on another rank: always in full
  pdl_begin();
  if (round_off(st, cfg)) return;
  if (allow_list && ld_gpu(&st->sparse_round)) return;
  commit_body(snap, bnd, key_out, n, st, per_round, cfg, D, cond, use_graph);
}

// the commit of a worklist round: only the columns merged into
__global__ void __launch_bounds__(kCommitThreads)
    k_commit_list(Snap* __restrict__ snap, double2* __restrict__ bnd,
                  const longlong2* __restrict__ key_out, int n, DevState* __restrict__ st,
                  long long* __restrict__ per_round, const DevCfg cfg, const Dirty D, const Touch T,
                  cudaGraphConditionalHandle cond, int use_graph) {
  pdl_begin();
  if (round_off(st, cfg) || !ld_gpu(&st->sparse_round)) return;
  commit_body<true>(snap, bnd, key_out, n, st, per_round, cfg, D, cond, use_graph, &T);
}

// Start of a solve: snapshot records and merge keys from the (normalised)
// start bounds, state reset, bounds_crossed pre-check (engine_common.hpp:51-58).
__global__ void __launch_bounds__(kCommitThreads)
    k_reset(const double* __restrict__ lo0, const double* __restrict__ up0,
            const uint8_t* __restrict__ integral, Snap* __restrict__ snap, double2* __restrict__ bnd,
            longlong2* __restrict__ key_out, int n, DevState* __restrict__ st, const DevCfg cfg,
            const Dirty D, const NodeCtl* __restrict__ ctl, int check_crossed,
            cudaGraphConditionalHandle cond, int use_graph) {
  int crossed = 0, frac = 0;
  {
    const int gstride = gridDim.x * blockDim.x, gtid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gtid == 0) key_out[n] = make_longlong2(0, 0);  // infeasibility slot
    uint32_t* f = reinterpret_cast<uint32_t*>(D.row_flag);
    for (int i = gtid; i < D.ms / 2; i += gstride) f[i] = 0u;
  }
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double l = lo0[j], u = up0[j];
    const bool in = integral[j] != 0;
    snap[j] = Snap{l, u, column_q(l, u, in, cfg), in ? 1LL : 0LL};
    bnd[j] = make_double2(l, u);
    if (cfg.bf) cfg.bf[j] = fpair(l, u);
    key_out[j] = make_longlong2(key_enc(l), -key_enc(u));
    if (l > __dadd_rn(u, cfg.imp_abs)) crossed = 1;
    if (in && (l != floor(l) || u != ceil(u))) frac = 1;  // floor(+-inf) = +-inf
  }
  if (frac) atomicOr(&st->frac_tmp, 1);
  unsigned long long dummy = 0;
  block_sum<kCommitThreads>(dummy, crossed);
  if (threadIdx.x == 0) {
    if (crossed) atomicOr(&st->crossed, 1);
    __threadfence();
    const uint32_t t = atomicAdd(&st->ticket_reset, 1u);
    if (t == gridDim.x - 1) {
      __threadfence();
      const int cr = check_crossed && atomicAdd(&st->crossed, 0);
      st->round_changes = 0;
      st->total_changes = 0;
      st->infeasible = 0;
      st->round = 0;
      st->status = cr ? 2 : -1;
      st->done = cr;
      st->ticket = 0;
      st->crossed = 0;
      st->wl_short = 0;
      st->wl_long = 0;
      st->work = 0;
      st->work2 = 0;
      st->cand_work = 0;
      // warm start from a root fixpoint: round 1 visits only the rows that
      // k_mark_vars marks (see NodeCtl)
      st->full = (D.enabled && ctl->warm) ? 0 : 1;
      st->nchg[0] = st->nchg[1] = 0;
      st->chg_deg[0] = st->chg_deg[1] = 0;
      st->ntouch = 0;
      st->sparse_round = 0;
      st->last_changes = 0x7fffffffffffffffLL;  // round 1 is a full sweep: no list
      st->nwide[0] = st->nwide[1] = 0;
      st->nmid[0] = st->nmid[1] = 0;
      st->nunit[0] = st->nunit[1] = 0;
      st->frac_any = atomicAdd(&st->frac_tmp, 0);
      st->frac_tmp = 0;
      st->ticket_reset = 0;
      st->stall = 0;
      st->resume = 0;
      st->delta_rounds = 0;
      __threadfence();
      if (use_graph) cudaGraphSetConditional(cond, cr ? 0u : 1u);
    }
  }
}

// Row-sharded rounds: this rank's infeasibility into the slot that rides the
// bound all-reduce (max over {lb key, -ub key, flag}).
__global__ void k_flag_to_slot(DevState* __restrict__ st, longlong2* __restrict__ slot) {
  if (threadIdx.x == 0 && !state_off(st)) slot->x = ld_gpu(&st->infeasible) ? 1 : 0;
}

// ---- row shards: sparse delta exchange ---------------
// A round's local merges as (column, lb key, negated ub key) items; the ranks
// all-gather them and apply them with the same max merges as the dense
// all-reduce, so key_out ends identical on every rank either way.
struct DeltaItem {
  long long col, lo, nup;
};

// cnt[0] = this rank's changed columns (items past `cap` are not written),
// cnt[1] = its infeasibility flag; cnt zeroed before the launch
__global__ void __launch_bounds__(256)
    k_delta_compact(const double2* __restrict__ bnd, const longlong2* __restrict__ key_out, int n,
                    DevState* __restrict__ st, DeltaItem* __restrict__ out, int cap,
                    int* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  if (state_off(st)) return;  // counts stay zero (memset before the launch)
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[1] = ld_gpu(&st->infeasible) ? 1 : 0;
  for (int j0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; j0 < n; j0 += gridDim.x * blockDim.x) {
    const int j = j0 + lane;
    bool ch = false;
    longlong2 k = make_longlong2(0, 0);
    if (j < n) {
      const double2 b = bnd[j];
      k = key_out[j];
      ch = k.x != key_enc(b.x) || k.y != -key_enc(b.y);
    }
    const unsigned m = __ballot_sync(0xffffffffu, ch);
    if (!m) continue;
    int base = 0;
    if (lane == 0) base = atomicAdd(cnt, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0) + __popc(m & ((1u << lane) - 1u));
    if (ch && base < cap) out[base] = DeltaItem{j, k.x, k.y};
  }
}

// every rank's items (rank r: all[r * stride .. + cnt_all[2r]]) merged by max
// held_ok: an overflow (some rank changed more than `stride` columns; the
// items were all-gathered at a fixed capacity) holds the round instead of
// applying a partial set -- the host resumes it with the dense all-reduce
// (unrolled graphs); without it the caller sized the gather to the counts
__global__ void __launch_bounds__(256)
    k_delta_apply(const DeltaItem* __restrict__ all, const int* __restrict__ cnt_all, int world,
                  int stride, longlong2* __restrict__ key_out, DevState* __restrict__ st,
                  int held_ok) {
  if (state_off(st)) return;
  if (held_ok) {
    int maxc = 0;
    for (int r = 0; r < world; ++r) maxc = max(maxc, cnt_all[2 * r]);
    if (maxc > stride) {
      if (blockIdx.x == 0 && threadIdx.x == 0) st->stall = 1;
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < world && cnt_all[2 * threadIdx.x + 1]) st->infeasible = 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->delta_rounds += 1;
  for (int r = 0; r < world; ++r) {
    const int c = min(cnt_all[2 * r], stride);
    const DeltaItem* a = all + (size_t)r * stride;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
      const DeltaItem d = a[i];
      long long* k = reinterpret_cast<long long*>(key_out + d.col);
      red_max(k, d.lo);
      red_max(k + 1, d.nup);
    }
  }
}

// the host resumes a held round (unrolled row-shard graphs): the next round
// skips its compute phases and merges the held local results densely
__global__ void k_shard_resume(DevState* __restrict__ st) {
  if (threadIdx.x == 0) {
    st->stall = 0;
    st->resume = 1;
  }
}

// Hybrid loop (engine.cu build_graph): the graph's WHILE rounds run while
// the rounds are full sweeps; once the next round would be a worklist round
// the loop hands over to the persistent kernel (k_loop), whose rounds are
// separated by grid barriers instead of half a dozen launches.  Runs after
// the round's marks, when the next round's kind is known.
__global__ void k_hybrid_decide(DevState* __restrict__ st, const Dirty D,
                                cudaGraphConditionalHandle cond) {
  if (threadIdx.x == 0 && !ld_gpu(&st->done) && round_is_sparse(st, D))
    cudaGraphSetConditional(cond, 0u);
}

// keys -> doubles (result download)
__global__ void k_decode(const longlong2* __restrict__ key, double* __restrict__ lo,
                         double* __restrict__ up, int n) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const longlong2 k = key[j];
    lo[j] = key_dec(k.x);
    up[j] = key_dec(-k.y);
  }
}

// |v| >= threshold -> +-inf (model.hpp:147-151), in place
__global__ void k_normalize(double* __restrict__ v, int n, double thr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = v[i];
    v[i] = x >= thr ? CUDART_INF : (x <= -thr ? -CUDART_INF : x);
  }
}

// Entry-balanced walk over a CSR: warp-cooperative, each warp takes chunks
// of kWalkChunk consecutive entries, so a 100k-entry row costs the same as
// 100k entries of short rows (a warp per row would leave one warp walking
// the longest row while the rest of the GPU idles).  f(valid, k, r) is called
// by every lane for entry k of row r.
constexpr int kWalkChunk = 512;

// last r in [0, m) with rp[r] <= k (same k on all lanes, rp[0] <= k):
// 32-ary search, four dependent probes for a million rows
__device__ __forceinline__ int warp_row_search(const int32_t* __restrict__ rp, int m, int64_t k) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = m;
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) >> 5;
    const int p = lo + lane * step;
    const bool ok = p < hi && rp[p] <= k;
    const int cnt = __popc(__ballot_sync(0xffffffffu, ok));
    lo += (cnt - 1) * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

template <class F>
__device__ __forceinline__ void walk_entries(const int32_t* __restrict__ rp, int m, int64_t nnz,
                                             F&& f) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c * kWalkChunk < nnz;
       c += nwarps) {
    const int64_t kb = c * kWalkChunk, ke = min(kb + kWalkChunk, nnz);
    int r = warp_row_search(rp, m, kb);
    for (int64_t k0 = kb; k0 < ke;) {
      // rows r .. r+31 and where row r+32 starts: the window covers entries
      // [k0, wend) -- all of the next 32 unless empty rows sit in between
      const int rr = r + lane;
      const int64_t s = rr < m ? rp[rr] : INT64_MAX;
      const int64_t s_end = rr < m ? rp[rr + 1] : INT64_MAX;
      const int64_t wend = min(min(k0 + 32, ke), __shfl_sync(0xffffffffu, s_end, 31));
      const int64_t k = k0 + lane;
      int j = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const int64_t v = __shfl_sync(0xffffffffu, s, j + step);
        if (v <= k) j += step;
      }
      f(k < wend, k, r + j);
      // row of entry wend
      k0 = wend;
      const int cnt = __popc(__ballot_sync(0xffffffffu, s <= k0));
      r += cnt - 1;
      if (cnt == 32)
        while (r + 1 < m && rp[r + 1] <= k0) ++r;
    }
  }
}

// Session init: rows into length-sorted order (perm[new] = old), lhs/rhs
// normalised (model.hpp:147-151), integrality packed into bit 31 of the
// column index (no per-entry byte gather).  Entries walked in the new order
// (coalesced stores, entry-balanced), each gathered from its old position.
__global__ void k_permute_rows(const int32_t* __restrict__ rp, const int32_t* __restrict__ cols,
                               const double* __restrict__ vals, const double* __restrict__ lhs,
                               const double* __restrict__ rhs, const int32_t* __restrict__ perm,
                               const int32_t* __restrict__ new_rp,
                               const uint8_t* __restrict__ integral, int32_t* __restrict__ colx,
                               double* __restrict__ new_vals, double* __restrict__ new_lhs,
                               double* __restrict__ new_rhs, int m, int n, double thr,
                               DevState* __restrict__ st) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int old = perm[i];
    const double l = lhs[old], h = rhs[old];
    new_lhs[i] = l >= thr ? CUDART_INF : (l <= -thr ? -CUDART_INF : l);
    new_rhs[i] = h >= thr ? CUDART_INF : (h <= -thr ? -CUDART_INF : h);
  }
  walk_entries(new_rp, m, new_rp[m], [&](bool valid, int64_t k, int r) {
    if (!valid) return;
    const int64_t src = rp[perm[r]] + (k - new_rp[r]);
    int32_t c = cols[src];
    if ((uint32_t)c >= (uint32_t)n) {
      // an out-of-range column index (undefined behaviour in the reference):
      // reported as PG_EINVAL after the solve; the entry is parked on the
      // padding column so that no kernel reads outside the arrays
      st->bad_input = 1;
      colx[k] = n;
    } else {
      colx[k] = integral[c] ? (int32_t)(c | 0x80000000u) : c;
    }
    new_vals[k] = vals[src];
  });
}

// Warm start of a branch-and-bound node (config C4): the start bounds are a
// converged root fixpoint with a few bounds overridden.  Every row of the
// root had all of its candidates rejected against the root bounds in the
// root's confirming round, so in the node's round 1 only rows containing an
// overridden column can produce anything; marking exactly those keeps the
// trajectory identical to a full sweep.
__global__ void __launch_bounds__(256)
    k_mark_vars(const Dirty D, const NodeCtl* __restrict__ ctl, DevState* __restrict__ st) {
  if (!D.enabled || !ctl->warm) return;
  uint8_t* flag = D.row_flag + (size_t)1 * D.ms;  // round 1 reads buffer (0 + 1) & 1
  const int lane = threadIdx.x & 31;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ctl->nvars;
       w += (gridDim.x * blockDim.x) >> 5) {
    const int j = ctl->vars[w];
    for (int e = D.col_ptr[j] + lane; e < D.col_ptr[j + 1]; e += 32) {
      const int r = D.col_row[e];
      if (mark_row(flag, r)) mark_row_units(D, r, 1, st);
    }
  }
}

// start bounds of a node: the root fixpoint (copied before) + its overrides
__global__ void k_apply_node(double* __restrict__ lo0, double* __restrict__ up0,
                             const NodeCtl* __restrict__ ctl, double thr, int f32) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ctl->nvars; i += gridDim.x * blockDim.x) {
    const int j = ctl->vars[i];
    const double l = ctl->lo[i], u = ctl->up[i];
    double nl = l >= thr ? CUDART_INF : (l <= -thr ? -CUDART_INF : l);
    double nu = u >= thr ? CUDART_INF : (u <= -thr ? -CUDART_INF : u);
    if (f32) {  // Narrow32 working copy (engine_common.hpp:24-38)
      nl = (double)(float)nl;
      nu = (double)(float)nu;
    }
    lo0[j] = nl;
    up0[j] = nu;
  }
}

// After the commit of round r: mark, for round r + 1, every row containing a
// column changed in round r (one warp per changed column).
__device__ __forceinline__ void mark_body(const Dirty& D, DevState* __restrict__ st) {
  const int r = ld_gpu(&st->round);
  if (!D.enabled || (D.unrolled && state_off(st)) || ld_gpu(&st->full)) return;
  const int cb = r & 1, nb = (r + 1) & 1;
  const int nchg = ld_gpu(&st->nchg[cb]);
  uint8_t* flag = D.row_flag + (size_t)nb * D.ms;
  const int lane = threadIdx.x & 31;
  // a warp takes B changed columns and walks their rows flattened over the
  // lanes (a column has few rows: one column per warp leaves most lanes idle
  // and pays one list append per column on the shared counters); B = 1 while
  // the columns are fewer than the warps, up to 32 with many
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int B = 1;
  while (B < 32 && (long long)nchg >= (long long)max(D.mark_batch, 1) * 2 * B * nwarps) B <<= 1;
  for (int w0 = B * ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); w0 < nchg; w0 += B * nwarps) {
    int e0 = 0, d = 0;
    if (lane < B && w0 + lane < nchg) {
      const int j = D.chg_list[(size_t)cb * D.n + w0 + lane];
      e0 = D.col_ptr[j];
      d = D.col_ptr[j + 1] - e0;
    }
    int incl = d;  // inclusive scan of the degrees
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int excl = incl - d;
    for (int t0 = 0; t0 < total; t0 += 32) {
      const int t = t0 + lane;
      // the column of flattened entry t: the last lane whose start is <= t
      // (fixed five steps, every lane shuffles)
      int pos = 0;
#pragma unroll
      for (int b = 16; b; b >>= 1)
        if (__shfl_sync(0xffffffffu, excl, pos + b) <= t) pos += b;
      const int e = __shfl_sync(0xffffffffu, e0, pos) + t - __shfl_sync(0xffffffffu, excl, pos);
      bool single = false;
      int u = -1;
      if (t < total) {
        const int row = D.col_row[e];
        if (mark_row(flag, row)) {
          u = D.row_unit[row];
          single = u >= 0 && D.unit_slice[u] == -1;
          if (!single) mark_row_units(D, row, nb, st);
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, single);
      if (bal) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&st->nunit[nb], __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (single)
          D.unit_list[(size_t)nb * D.nunits + base + __popc(bal & ((1u << lane) - 1u))] = u;
      }
    }
  }
}
__global__ void __launch_bounds__(256) k_mark(const Dirty D, DevState* __restrict__ st) {
  pdl_begin();
  mark_body(D, st);
}

__global__ void k_max_row_len(const int32_t* __restrict__ rp, int m, int32_t* __restrict__ out) {
  int mx = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    mx = max(mx, rp[i + 1] - rp[i]);
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// ---- worklist index (session init) -----------------------------------------------

// column counts (flat over the entries)
__global__ void k_csc_count(const int32_t* __restrict__ colx, int64_t nnz, int n,
                            int32_t* __restrict__ cnt) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x)
  {
    const uint32_t c = (uint32_t)colx[k] & 0x7fffffffu;
    if (c < (uint32_t)n) atomicAdd(&cnt[c], 1);  // out of range: rejected at setup
  }
}

// rows into their columns' ranges (entry-balanced walk); row r is named
// rowmap[r] when given (a CSR in the caller's row order)
__global__ void k_csc_fill(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ colx,
                           int m, int n, int32_t* __restrict__ cursor,
                           const int32_t* __restrict__ rowmap, int32_t* __restrict__ col_row) {
  walk_entries(row_ptr, m, row_ptr[m], [&](bool valid, int64_t k, int r) {
    if (!valid) return;  // k may be past the last entry
    const uint32_t c = (uint32_t)colx[k] & 0x7fffffffu;
    if (c < (uint32_t)n) col_row[atomicAdd(&cursor[c], 1)] = rowmap ? rowmap[r] : r;
  });
}

// inv[perm[i]] = i
__global__ void k_invert_perm(const int32_t* __restrict__ perm, int m, int32_t* __restrict__ inv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    inv[perm[i]] = i;
}

}  // namespace pgb
