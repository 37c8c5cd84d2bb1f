// kernels.cuh -- the round-synchronous propagation round on sm_100a.
//
// One round = run_round + process_block of the reference
// (par_engine.cpp:126-200), in three launches:
//
//   k_round   persistent, work-stealing over two kinds of items:
//             * segment groups (longest first): 32 segments of long rows
//               (chunks of nnz_budget entries, wide_row_activities,
//               par_engine.cpp:99-123); the CTA's 8 warps stage 32 entries of
//               every segment through shared memory, one lane per segment
//               sums in entry order;
//             * short-row tiles: 8 warp tiles of <= 32 rows / <= 128 entries,
//               one lane per row sums in entry order.
//             Then the exact candidate pipeline for the entries that pass an
//             exactness-preserving filter, committed by 64-bit atomics.
//   k_seg_cand  pass 2 over the segments of long rows that may tighten.
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

#ifndef PG_ROUND_MINB
#define PG_ROUND_MINB 2
#endif

constexpr int kCommitThreads = 256;
constexpr int kRoundThreads = 256;
constexpr int kRoundWarps = kRoundThreads / 32;

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
  int32_t wl_count;                  // pass-2 worklist length of the current round
  int32_t work;                      // k_round work-stealing counter
  int32_t full;                      // 1: every work item is dirty (first round)
  int32_t frac_any;                  // an integral column has a fractional start bound
  int32_t frac_tmp;                  // k_reset's accumulator of frac_any
  int32_t nchg[2];                   // changed-column list lengths, by round parity
};

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
};

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

__device__ __forceinline__ void ld_snap(const Snap* p, double& lo, double& up, double& q) {
  long long f;
  asm("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];"
      : "=d"(lo), "=d"(up), "=d"(q), "=l"(f)
      : "l"(p));
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
__device__ __forceinline__ void commit_side(long long* key_out, int j, int kind, double cl,
                                            double cu) {
  // merge_lower / merge_upper (par_engine.cpp:56-71) as exact 64-bit max/min
  if (kind & 1) {
    const long long k = key_enc(canon0(cl));
    long long* p = key_out + 2 * (size_t)j;
    if (*((volatile long long*)p) < k) atomicMax(p, k);
  }
  if (kind & 2) {
    // upper bounds are kept as NEGATED keys so that one max-reduction merges
    // both sides (one NCCL all-reduce on the row-sharded path)
    const long long k = -key_enc(canon0(cu));
    long long* p = key_out + 2 * (size_t)j + 1;
    if (*((volatile long long*)p) < k) atomicMax(p, k);
  }
}

// residual -> candidates -> tighten vs the snapshot -> merge
// (propcore.hpp:78-208, par_engine.cpp:158-168).  Returns true on EmptyDomain.
__device__ __forceinline__ bool entry_pipeline(const Act& act, double a, double lo, double up,
                                               double lhs, double rhs, int32_t cx,
                                               long long* key_out, const DevCfg& c) {
  double min_res, max_res, cl, cu;
  residual(act, a, lo, up, min_res, max_res);
  candidates(a, lhs, rhs, min_res, max_res, cx < 0, c, cl, cu);
  const int kind = tighten(lo, up, cl, cu, c);
  if (kind == 4) return true;  // EmptyDomain: flag, skip the merge (par_engine.cpp:163-166)
  if (kind) commit_side(key_out, cx & 0x7fffffff, kind, cl, cu);
  return false;
}

// min/max contributions (NaN = infinite) and the filter term of one entry
__device__ __forceinline__ void entry_terms(double a, const Snap* snap, int32_t cx,
                                            double& pmin, double& pmax, double& x) {
  double lo, up, q;
  ld_snap(snap + (cx & 0x7fffffff), lo, up, q);
  contrib(a, lo, up, pmin, pmax);
  x = fabs(a) * q;
}

// ---- work items of k_round ------------------------------------------------------
constexpr int kShortMax = 16;   // rows up to this length go to warp tiles
constexpr int kWItems = 4;
constexpr int kWNnz = 32 * kWItems;
constexpr int kLongSeg = 256;     // segments longer than this form groups of 8

struct TileDesc {
  int32_t r0;  // first row (sorted row space)
  int32_t nr;  // rows (<= 32)
  int32_t k0;  // first entry
  int32_t nz;  // entries (<= kWNnz)
};

struct SegDesc {
  int32_t k0;
  int32_t len;
  int32_t out;    // partial index = first chunk of the row + chunk number
  int32_t rslot;  // segment-row slot
};

struct SegGroup {
  int32_t first;  // first segment (segments sorted by length, descending)
  int32_t count;  // 32, or 8 for long segments (shorter tail per group)
};

struct SegPartial {
  double min_f;
  double max_f;
  double xmax;
  int32_t min_i;
  int32_t max_i;
};

// transposed staging of a segment group: [entry][segment], padded
constexpr int kSegStage = 2304;  // >= 64 x 33 and >= 256 x 9
struct SegGroupSmem {
  double pmin[kSegStage];
  double pmax[kSegStage];
  double xmax[32];
  int32_t cmin[32], cmax[32];
  SegDesc desc[32];
};

struct RoundArgs {
  const TileDesc* tiles;  // warp tiles of short rows (sorted row space)
  int32_t num_tiles;
  const SegDesc* segs;    // segments sorted by length, descending
  int32_t nseg;
  const SegGroup* groups;
  int32_t ngroups;
  const int32_t* srow;    // segment-row slot -> sorted row
  const int32_t* sfirst;  // segment-row slot -> first partial (+1 sentinel)
  const int32_t* chunk_seg;  // partial index -> segment index
  int32_t* row_done;      // per segment row: chunks finished this round
  SegPartial* partial;
  Act* row_act;
  int32_t* worklist;
  const int32_t* row_ptr;
  const int32_t* colx;
  const double* vals;
  const double* lhs;
  const double* rhs;
  const Snap* snap;
  long long* key_out;
  DevState* st;
  Dirty dirty;
};

// finite contributions (0 for an infinite bound: adding +-0 to a sum that
// starts at +0 is exact) and infinity flags, propcore.hpp:50-62
__device__ __forceinline__ void entry_terms_clean(double a, const Snap* snap, int32_t cx,
                                                  double& pmin, double& pmax, double& x,
                                                  bool& imin, bool& imax) {
  double lo, up, q;
  ld_snap(snap + (cx & 0x7fffffff), lo, up, q);
  const double bmin = a > 0 ? lo : up;
  const double bmax = a > 0 ? up : lo;
  imin = isinf(bmin);
  imax = isinf(bmax);
  pmin = imin ? 0.0 : __dmul_rn(a, bmin);
  pmax = imax ? 0.0 : __dmul_rn(a, bmax);
  x = fabs(a) * q;
}

// Row of a segment finished: tree over its chunk partials (in chunk order,
// par_engine.cpp:117-121), row check, filter; rows that may tighten push
// their segments onto the pass-2 worklist.
template <bool kRowCheck>
__device__ void finish_seg_row(const RoundArgs& A, int rs, const DevCfg& cfg) {
  const int first = A.sfirst[rs];
  int np = A.sfirst[rs + 1] - first;
  const int nch = np;
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
  A.row_act[rs] = act;
  const int row = A.srow[rs];
  const double l = A.lhs[row], h = A.rhs[row];
  if (kRowCheck && row_infeasible(act, l, h, cfg)) A.st->infeasible = 1;
  if (row_may(row_filter(act, l, h), xmax)) {
    const int pos = atomicAdd(&A.st->wl_count, nch);
    for (int i = 0; i < nch; ++i) A.worklist[pos + i] = A.chunk_seg[first + i];
  }
}

// One group of G segments of near-equal length by the whole CTA: the 8
// warps stage SC = (256/G) x 8 entries of every segment per step
// (coalesced runs per segment), one lane per segment sums them in entry
// order.  G = 8 for long segments keeps the per-group critical path short.
template <bool kRowCheck, int G>
__device__ void seg_group(const RoundArgs& A, SegGroupSmem& S, const SegGroup grp,
                          const uint8_t* sflag, const DevCfg& cfg) {
  constexpr int TPS = kRoundThreads / G;  // threads per segment
  constexpr int E = 8;                    // entries per thread per step
  constexpr int SC = TPS * E;             // entries per segment per step
  constexpr int LD = G + 1;               // padded stride
  static_assert(SC * LD <= kSegStage, "staging too small");
  const int tid = threadIdx.x;
  if (tid < G) S.desc[tid] = tid < grp.count ? A.segs[grp.first + tid] : SegDesc{0, 0, -1, -1};
  __syncthreads();
  const int L = S.desc[0].len;  // sorted descending
  const int ls = tid / TPS, sub = tid % TPS;
  const int my_k0 = S.desc[ls].k0, my_len = S.desc[ls].len;
  double smin = 0.0, smax = 0.0;  // chain sums (lanes < G of warp 0)
  double xm = -CUDART_INF;
  int cmin = 0, cmax = 0;
  for (int c0 = 0; c0 < L; c0 += SC) {
    double av[E];
    int32_t cv[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int i = c0 + sub + TPS * j;
      if (i < my_len) {
        cv[j] = __ldg(A.colx + my_k0 + i);
        av[j] = __ldg(A.vals + my_k0 + i);
      }
    }
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int i = c0 + sub + TPS * j;
      if (i < my_len) {
        double pmin, pmax, x;
        bool imin, imax;
        entry_terms_clean(av[j], A.snap, cv[j], pmin, pmax, x, imin, imax);
        S.pmin[(sub + TPS * j) * LD + ls] = pmin;
        S.pmax[(sub + TPS * j) * LD + ls] = pmax;
        xm = fmax(xm, x);
        cmin += imin;
        cmax += imax;
      }
    }
    __syncthreads();
    if (tid < G) {
      const int n = min(SC, S.desc[tid].len - c0);
      for (int i = 0; i < n; ++i) {
        smin = __dadd_rn(smin, S.pmin[i * LD + tid]);
        smax = __dadd_rn(smax, S.pmax[i * LD + tid]);
      }
    }
    __syncthreads();
  }
  // per-segment reduction of the order-free parts over its TPS threads
#pragma unroll
  for (int o = 1; o < TPS && o < 32; o <<= 1) {
    xm = fmax(xm, __shfl_xor_sync(0xffffffffu, xm, o));
    cmin += __shfl_xor_sync(0xffffffffu, cmin, o);
    cmax += __shfl_xor_sync(0xffffffffu, cmax, o);
  }
  if (sub == 0) {
    S.xmax[ls] = xm;
    S.cmin[ls] = cmin;
    S.cmax[ls] = cmax;
  }
  __syncthreads();
  // with the worklist, a dirty group may hold clean rows: only dirty rows are
  // finished (a clean multi-chunk row may be missing chunks of clean groups)
  if (tid < G && S.desc[tid].out >= 0 && (!sflag || sflag[S.desc[tid].rslot])) {
    const SegDesc d = S.desc[tid];
    const Act acc = {smin, smax, S.cmin[tid], S.cmax[tid]};
    const double xmax = S.xmax[tid];
    const int first = A.sfirst[d.rslot];
    const int nch = A.sfirst[d.rslot + 1] - first;
    if (nch == 1) {
      // the segment is the whole row: finish it here
      A.row_act[d.rslot] = acc;
      const int row = A.srow[d.rslot];
      const double l = A.lhs[row], h = A.rhs[row];
      if (kRowCheck && row_infeasible(acc, l, h, cfg)) A.st->infeasible = 1;
      if (row_may(row_filter(acc, l, h), xmax)) {
        const int pos = atomicAdd(&A.st->wl_count, 1);
        A.worklist[pos] = grp.first + tid;
      }
    } else {
      volatile SegPartial* P = A.partial + d.out;
      P->min_f = acc.min_f;
      P->max_f = acc.max_f;
      P->xmax = xmax;
      P->min_i = acc.min_i;
      P->max_i = acc.max_i;
      __threadfence();
      if (atomicAdd(&A.row_done[d.rslot], 1) == nch - 1) {
        __threadfence();
        A.row_done[d.rslot] = 0;
        finish_seg_row<kRowCheck>(A, d.rslot, cfg);
      }
    }
  }
  __syncthreads();
}

// number of set bits of the 128-bit mask m[0..3] in [b, e)
__device__ __forceinline__ int popc_range(const unsigned (&m)[kWItems], int b, int e) {
  int c = 0;
#pragma unroll
  for (int q = 0; q < kWItems; ++q) {
    const int lo = max(b - 32 * q, 0), hi = min(e - 32 * q, 32);
    if (lo < hi) {
      const unsigned keep = (hi == 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
      c += __popc(m[q] & keep);
    }
  }
  return c;
}

// ---- short rows: warp tiles with per-warp asynchronous staging -------------------
// Each warp owns a contiguous run of warp tiles (<= 32 consecutive rows of
// the SAME length L <= kShortMax, <= 128 entries) and pipelines them three
// deep:
//   tile i+2: TMA bulk copies of its vals/col streams -> shared memory
//   tile i+1: cp.async gathers of the 16 B {lb, ub} snapshot of every entry
//   tile i:   compute (one lane per row, sums in entry order)
// Neither stage holds registers, so a warp keeps ~256 gathers in flight with
// no CTA barrier.  Rows are stored sorted by length (session init).

struct __align__(16) TileStage {
  double vals[kWNnz + 2];   // +2 / +4: the bulk copies start 16 B aligned
  int32_t cols[kWNnz + 4];
  double2 rec[kWNnz];       // {lb, ub} of every entry's column
  double lhs[34];
  double rhs[34];
  TileDesc d;
};

struct TileWork {
  double pmin[kWNnz];       // finite min contributions, [position][row]
  double pmax[kWNnz];
  double x[kWNnz];          // filter terms
  double minf[32], maxf[32], lhs[32], rhs[32], tr[32], tl[32];
  int32_t mini[32], maxi[32];
  uint32_t cmin[32], cmax[32];  // per row: positions with an infinite contribution
  uint8_t qe[kWNnz];        // queue: entry index
  uint8_t mode[32];
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// lane 0: bulk copies of tile t's entry streams and row data into a stage
// (device arrays carry >= 16 B of tail padding for the widened ranges)
__device__ __forceinline__ void tile_issue_tma(const RoundArgs& A, TileStage& S, uint64_t* bar,
                                               const TileDesc d) {
  S.d = d;
  const int kv = d.k0 & ~1, kc = d.k0 & ~3, k1 = d.k0 + d.nz;
  const uint32_t bv = (uint32_t)(((k1 - kv) * 8 + 15) & ~15);
  const uint32_t bc = (uint32_t)(((k1 - kc) * 4 + 15) & ~15);
  const int rd = d.r0 & ~1;
  const uint32_t bs = (uint32_t)(((d.r0 + d.nr - rd) * 8 + 15) & ~15);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(bar, bc + bv + 2 * bs);
  bulk_g2s(S.vals, A.vals + kv, bv, bar);
  bulk_g2s(S.cols, A.colx + kc, bc, bar);
  bulk_g2s(S.lhs, A.lhs + rd, bs, bar);
  bulk_g2s(S.rhs, A.rhs + rd, bs, bar);
}

// all lanes: 16 B snapshot gathers of a staged tile (one cp.async group)
__device__ __forceinline__ void tile_issue_gathers(const RoundArgs& A, TileStage& S, int lane) {
  const int oc = S.d.k0 & 3;
#pragma unroll
  for (int q = 0; q < kWItems; ++q) {
    const int e = lane + 32 * q;
    if (e < S.d.nz) cp_async16(&S.rec[e], &A.snap[S.cols[oc + e] & 0x7fffffff].lo);
  }
  cp_async_commit();
}

// filter coefficient of a column computed from its bounds (column_q);
// frac_any = some integral column may carry a fractional bound
__device__ __forceinline__ double column_q_fast(double lo, double up, bool integral,
                                                bool frac_any, const DevCfg& c) {
  // an infinite bound makes both terms +inf (lb <= ub): no test needed
  const double thr = integral ? c.int_eps : c.imp_abs + c.imp_rel;
  const double q = ((up - lo) - thr) + (fabs(lo) + fabs(up)) * kMargin;
  if (frac_any && integral && (lo != floor(lo) || up != ceil(up))) return CUDART_INF;
  return q;
}

template <bool kRowCheck>
__device__ void tile_compute(const RoundArgs& A, TileWork& W, const TileStage& S,
                             bool frac_any, bool& inf_flag, const DevCfg& cfg) {
  const int lane = threadIdx.x & 31;
  const TileDesc d = S.d;
  const int nr = d.nr, nz = d.nz;
  const int L = nr ? nz / nr : 0;  // every row of a warp tile has L entries
  const float invL = L ? 1.0f / (float)L : 0.0f;
  const int ov = d.k0 & 1, oc = d.k0 & 3, ors = d.r0 & 1;
  W.cmin[lane] = 0u;
  W.cmax[lane] = 0u;
  __syncwarp();

  // phase 1: contributions and filter terms of the staged entries, written
  // transposed ([position][row]) so that phase 2 reads are conflict-free
  double xq[kWItems];
  int rq[kWItems];
  unsigned infq = 0;  // bit 2q: min contribution infinite, bit 2q+1: max
#pragma unroll
  for (int q = 0; q < kWItems; ++q) {
    const int e = lane + 32 * q;
    rq[q] = 0;
    xq[q] = 0.0;
    if (e < nz) {
      const int r = __float2int_rz(((float)e + 0.5f) * invL);
      const int i = e - r * L;
      rq[q] = r;
      const double a = S.vals[ov + e];
      const double2 b = S.rec[e];
      const double bmin = a > 0 ? b.x : b.y;
      const double bmax = a > 0 ? b.y : b.x;
      const bool imin = isinf(bmin), imax = isinf(bmax);
      W.pmin[i * nr + r] = imin ? 0.0 : __dmul_rn(a, bmin);
      W.pmax[i * nr + r] = imax ? 0.0 : __dmul_rn(a, bmax);
      const double x = fabs(a) * column_q_fast(b.x, b.y, S.cols[oc + e] < 0, frac_any, cfg);
      W.x[i * nr + r] = x;
      xq[q] = x;
      if (imin) atomicOr(&W.cmin[r], 1u << i);
      if (imax) atomicOr(&W.cmax[r], 1u << i);
      infq |= (imin ? 1u : 0u) << (2 * q) | (imax ? 2u : 0u) << (2 * q);
    }
  }
  __syncwarp();

  // phase 2: one lane per row, L sums in entry order (propcore.hpp:50-63)
  bool may = false;
  if (lane < nr) {
    double smin = 0.0, smax = 0.0, xmax = -CUDART_INF;
    for (int i = 0; i < L; ++i) {
      smin = __dadd_rn(smin, W.pmin[i * nr + lane]);
      smax = __dadd_rn(smax, W.pmax[i * nr + lane]);
      xmax = fmax(xmax, W.x[i * nr + lane]);
    }
    const Act act = {smin, smax, __popc(W.cmin[lane]), __popc(W.cmax[lane])};
    const double l = S.lhs[ors + lane], h = S.rhs[ors + lane];
    if (kRowCheck && row_infeasible(act, l, h, cfg)) inf_flag = true;
    const RowFilter f = row_filter(act, l, h);
    may = row_may(f, xmax);
    W.minf[lane] = act.min_f;
    W.maxf[lane] = act.max_f;
    W.mini[lane] = act.min_i;
    W.maxi[lane] = act.max_i;
    W.lhs[lane] = l;
    W.rhs[lane] = h;
    W.tr[lane] = f.tr;
    W.tl[lane] = f.tl;
    W.mode[lane] = f.mode;
  }
  const unsigned may_rows = __ballot_sync(0xffffffffu, may);
  __syncwarp();
  if (may_rows == 0) return;  // no row of this tile can tighten anything

  // phase 3: entry filter, compaction into a warp queue, dense exact pipeline
  int qn = 0;
#pragma unroll
  for (int q = 0; q < kWItems; ++q) {
    const int e = lane + 32 * q;
    bool pass = false;
    if (e < nz && ((may_rows >> rq[q]) & 1u)) {
      const int r = rq[q];
      const RowFilter f = {W.tr[r], W.tl[r], W.mode[r]};
      pass = entry_may(f, xq[q], (infq >> (2 * q)) & 1u, (infq >> (2 * q + 1)) & 1u);
    }
    const unsigned m = __ballot_sync(0xffffffffu, pass);
    if (pass) W.qe[qn + __popc(m & ((1u << lane) - 1u))] = (uint8_t)e;
    qn += __popc(m);
  }
  __syncwarp();
  for (int i = lane; i < qn; i += 32) {
    const int e = W.qe[i];
    const int r = __float2int_rz(((float)e + 0.5f) * invL);
    const double2 b = S.rec[e];
    const Act act = {W.minf[r], W.maxf[r], W.mini[r], W.maxi[r]};
    if (entry_pipeline(act, S.vals[ov + e], b.x, b.y, W.lhs[r], W.rhs[r], S.cols[oc + e],
                       A.key_out, cfg))
      inf_flag = true;
  }
  __syncwarp();
}

// Warp-specialised dense path: per CTA one producer warp and kWsConsumers
// consumer warps share a ring of kWsStages tile stages.
//   producer: TMA bulk copies of tile i (vals/col/lhs/rhs), then -- kWsLag
//             tiles behind -- cp.async gathers of the {lb, ub} records of
//             tile i - lag, completing on the stage's `full` mbarrier
//             (cp.async.mbarrier.arrive.noinc from every producer lane);
//   consumer c: tiles c, c + C, ... : wait `full`, compute, release `empty`.
// Memory parallelism is set by the ring depth, not by the number of
// resident compute warps.
#ifndef PG_WS_CONSUMERS
#define PG_WS_CONSUMERS 6
#endif
#ifndef PG_WS_STAGES
#define PG_WS_STAGES 8
#endif
constexpr int kWsConsumers = PG_WS_CONSUMERS;
constexpr int kWsWarps = kWsConsumers + 1;
constexpr int kWsStages = PG_WS_STAGES;
constexpr int kWsLag = 2;

struct TileRing {
  TileStage stage[kWsStages];
  uint64_t tma_bar[kWsStages];
  uint64_t full_bar[kWsStages];
  uint64_t empty_bar[kWsStages];
  TileWork work[kWsConsumers];
};
struct TileSparseSmem {
  TileStage stage[kWsWarps];
  TileWork work[kWsWarps];
};
union TilesSmem {
  TileRing ring;
  TileSparseSmem sparse;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// sparse round: per tile, the marked rows only, as a compacted virtual tile
// staged with plain loads (uniform row length keeps the layout)
template <bool kRowCheck>
__device__ void tiles_sparse(const RoundArgs& A, TileStage& S, TileWork& W, int tb, int te,
                             const uint8_t* rflag, bool frac_any, bool& inf_flag,
                             const DevCfg& cfg) {
  const int lane = threadIdx.x & 31;
  for (int t0 = tb; t0 < te; t0 += 32) {
    TileDesc wd = {0, 0, 0, 0};
    if (t0 + lane < te) wd = A.tiles[t0 + lane];
    for (int u = 0; u < 32 && t0 + u < te; ++u) {
      TileDesc d;
      d.r0 = __shfl_sync(0xffffffffu, wd.r0, u);
      d.nr = __shfl_sync(0xffffffffu, wd.nr, u);
      d.k0 = __shfl_sync(0xffffffffu, wd.k0, u);
      d.nz = __shfl_sync(0xffffffffu, wd.nz, u);
      const unsigned m = __ballot_sync(0xffffffffu, lane < d.nr && rflag[d.r0 + lane]);
      if (!m) continue;
      const int L = d.nz / d.nr, nv = __popc(m);
      // lane p of a marked row takes slot rank(p) of the virtual tile
      if ((m >> lane) & 1u) {
        const int rank = __popc(m & ((1u << lane) - 1u));
        W.qe[rank] = (uint8_t)lane;
        S.lhs[rank] = A.lhs[d.r0 + lane];
        S.rhs[rank] = A.rhs[d.r0 + lane];
      }
      __syncwarp();
      const float invL = 1.0f / (float)L;
      for (int e = lane; e < nv * L; e += 32) {
        const int r = __float2int_rz(((float)e + 0.5f) * invL);
        const int k = d.k0 + W.qe[r] * L + (e - r * L);
        const int32_t c = __ldg(A.colx + k);
        S.vals[e] = __ldg(A.vals + k);
        S.cols[e] = c;
        S.rec[e] = __ldg(reinterpret_cast<const double2*>(&A.snap[c & 0x7fffffff].lo));
      }
      if (lane == 0) S.d = TileDesc{0, nv, 0, nv * L};
      __syncwarp();
      tile_compute<kRowCheck>(A, W, S, frac_any, inf_flag, cfg);
    }
  }
}

template <bool kRowCheck>
__global__ void __launch_bounds__(kWsWarps * 32) k_tiles(const RoundArgs A, const DevCfg cfg) {
  extern __shared__ __align__(16) unsigned char tiles_smem[];
  TilesSmem& sm = *reinterpret_cast<TilesSmem*>(tiles_smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // contiguous run of tiles of this CTA (static: no global counter)
  const int per = (A.num_tiles + gridDim.x - 1) / gridDim.x;
  const int tb = min((int)blockIdx.x * per, A.num_tiles), te = min(tb + per, A.num_tiles);
  if (tb >= te) return;
  const bool full = !A.dirty.enabled || *((volatile int32_t*)&A.st->full);
  const bool frac_any = *((volatile int32_t*)&A.st->frac_any) != 0;
  bool inf_flag = false;
  if (!full) {
    const int par = (*((volatile int32_t*)&A.st->round) + 1) & 1;
    const uint8_t* rflag = A.dirty.row_flag + (size_t)par * A.dirty.ms;
    // every warp takes a slice of the CTA's tiles
    const int wper = (te - tb + kWsWarps - 1) / kWsWarps;
    const int wb = min(tb + warp * wper, te), we = min(wb + wper, te);
    tiles_sparse<kRowCheck>(A, sm.sparse.stage[warp], sm.sparse.work[warp], wb, we, rflag,
                            frac_any, inf_flag, cfg);
    if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
    return;
  }
  TileRing& R = sm.ring;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kWsStages; ++i) {
      mbar_init(&R.tma_bar[i], 1);
      mbar_init(&R.full_bar[i], 32);
      mbar_init(&R.empty_bar[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int N = te - tb;
  if (warp == kWsConsumers) {
    // ---- producer -----------------------------------------------------------
    int wbase = -1;
    TileDesc wdesc = {0, 0, 0, 0};
    for (int it = 0; it < N + kWsLag; ++it) {
      if (it < N) {
        const int t = tb + it;
        if (wbase < 0 || t >= wbase + 32) {  // descriptors, a 32-tile window per load
          wbase = t;
          if (t + lane < te) wdesc = A.tiles[t + lane];
        }
        TileDesc d;
        d.r0 = __shfl_sync(0xffffffffu, wdesc.r0, t - wbase);
        d.nr = __shfl_sync(0xffffffffu, wdesc.nr, t - wbase);
        d.k0 = __shfl_sync(0xffffffffu, wdesc.k0, t - wbase);
        d.nz = __shfl_sync(0xffffffffu, wdesc.nz, t - wbase);
        const int slot = it % kWsStages, use = it / kWsStages;
        if (use > 0) mbar_wait(&R.empty_bar[slot], (uint32_t)((use - 1) & 1));
        if (lane == 0) tile_issue_tma(A, R.stage[slot], &R.tma_bar[slot], d);
      }
      const int g = it - kWsLag;
      if (g >= 0 && g < N) {
        const int slot = g % kWsStages, use = g / kWsStages;
        mbar_wait(&R.tma_bar[slot], (uint32_t)(use & 1));
        TileStage& S = R.stage[slot];
        const int oc = S.d.k0 & 3;
#pragma unroll
        for (int q = 0; q < kWItems; ++q) {
          const int e = lane + 32 * q;
          if (e < S.d.nz) cp_async16(&S.rec[e], &A.snap[S.cols[oc + e] & 0x7fffffff].lo);
        }
        cp_async_arrive_noinc(&R.full_bar[slot]);
      }
    }
  } else {
    // ---- consumers ----------------------------------------------------------
    TileWork& W = R.work[warp];
    for (int i = warp; i < N; i += kWsConsumers) {
      const int slot = i % kWsStages, use = i / kWsStages;
      mbar_wait(&R.full_bar[slot], (uint32_t)(use & 1));
      tile_compute<kRowCheck>(A, W, R.stage[slot], frac_any, inf_flag, cfg);
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.empty_bar[slot]);
    }
    if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
  }
}

template <bool kRowCheck>
__global__ void __launch_bounds__(kRoundThreads, PG_ROUND_MINB) k_round(const RoundArgs A, const DevCfg cfg) {
  extern __shared__ __align__(16) unsigned char round_smem[];
  SegGroupSmem& sm = *reinterpret_cast<SegGroupSmem*>(round_smem);
  __shared__ int32_t s_item;
  const int lane = threadIdx.x & 31;
  // full sweep (first round, or no worklist), else skip clean work items
  const bool full = !A.dirty.enabled || *((volatile int32_t*)&A.st->full);
  const int par = (*((volatile int32_t*)&A.st->round) + 1) & 1;
  const uint8_t* sflag = A.dirty.row_flag + (size_t)par * A.dirty.ms + A.dirty.first_seg_row;
  const int total = A.ngroups;
  bool inf_flag = false;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(&A.st->work, 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= total) break;
    const SegGroup grp = A.groups[item];
    if (!full) {
      // dirty iff a row of one of its segments is marked
      const bool d = threadIdx.x < grp.count && sflag[A.segs[grp.first + threadIdx.x].rslot];
      if (!__syncthreads_or(d)) continue;
    }
    if (grp.count == 8 || grp.count < 8 && A.segs[grp.first].len > kLongSeg)
      seg_group<kRowCheck, 8>(A, sm, grp, full ? nullptr : sflag, cfg);
    else
      seg_group<kRowCheck, 32>(A, sm, grp, full ? nullptr : sflag, cfg);
  }
  if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
}

// Pass 2 over the worklist: one warp per segment, coalesced re-read (mostly
// L2 hits), entry filter, exact pipeline, atomic commit.
// Pass 2 over the worklist: the segments of rows that may tighten.  Each
// warp takes one segment (a short segment is one or two coalesced steps; a
// long one is split over the CTA's warps in 32-entry strides).
__device__ __forceinline__ bool seg_cand_entries(const RoundArgs& A, const SegDesc& d,
                                                 const Act& act, const RowFilter& f, double l,
                                                 double h, int first, int stride,
                                                 const DevCfg& cfg) {
  bool inf_flag = false;
  for (int i = first; i < d.len; i += stride) {
    const int k = d.k0 + i;
    const int32_t c = __ldg(A.colx + k);
    const double a = __ldg(A.vals + k);
    double lo, up, q;
    ld_snap(A.snap + (c & 0x7fffffff), lo, up, q);
    double pmin, pmax;
    contrib(a, lo, up, pmin, pmax);
    if (entry_may(f, fabs(a) * q, isnan(pmin), isnan(pmax)) &&
        entry_pipeline(act, a, lo, up, l, h, c, A.key_out, cfg))
      inf_flag = true;
  }
  return inf_flag;
}

__global__ void __launch_bounds__(256)
    k_seg_cand(const RoundArgs A, const DevCfg cfg) {
  const int nwl = *((volatile int32_t*)&A.st->wl_count);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  bool inf_flag = false;
  // long segments: one CTA each (worklist order is arbitrary, test per entry)
  for (int w = blockIdx.x; w < nwl; w += gridDim.x) {
    const SegDesc d = A.segs[A.worklist[w]];
    if (d.len <= kLongSeg) continue;
    const Act act = A.row_act[d.rslot];
    const int row = A.srow[d.rslot];
    const double l = A.lhs[row], h = A.rhs[row];
    inf_flag |= seg_cand_entries(A, d, act, row_filter(act, l, h), l, h, threadIdx.x,
                                 blockDim.x, cfg);
  }
  // short segments: one warp each
  for (int w = blockIdx.x * (blockDim.x >> 5) + warp; w < nwl;
       w += gridDim.x * (blockDim.x >> 5)) {
    const SegDesc d = A.segs[A.worklist[w]];
    if (d.len > kLongSeg) continue;
    const Act act = A.row_act[d.rslot];
    const int row = A.srow[d.rslot];
    const double l = A.lhs[row], h = A.rhs[row];
    inf_flag |= seg_cand_entries(A, d, act, row_filter(act, l, h), l, h, lane, 32, cfg);
  }
  if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
}

// ---- commit + round decision ------------------------------------------------------
template <int kThreads>
__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, int& f) {
  __shared__ unsigned long long s_sum[kThreads / 32];
  __shared__ int s_f[kThreads / 32];
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
__global__ void __launch_bounds__(kCommitThreads)
    k_commit(Snap* __restrict__ snap, const longlong2* __restrict__ key_out, int n,
             DevState* __restrict__ st, long long* __restrict__ per_round, const DevCfg cfg,
             const Dirty D, cudaGraphConditionalHandle cond, int use_graph) {
  unsigned long long changes = 0;
  int inf = 0;
  const int R = *((volatile int32_t*)&st->round);  // rounds before this one
  const int nb = R & 1;                             // buffer of the next round's lists
  const int cb = nb ^ 1;                            // buffer this round consumed
  const int gstride = gridDim.x * blockDim.x;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int j = gtid; j < n; j += gstride) {
    const longlong2 ko = key_out[j];
    const double lo = key_dec(ko.x), up = key_dec(-ko.y);
    const double2 in = *reinterpret_cast<const double2*>(&snap[j].lo);
    // a change is a strict improvement, so comparing values is exact
    const int c = (lo != in.x) + (up != in.y);
    if (c) {
      changes += c;
      const bool integral = snap[j].flags & 1;
      Snap s = {lo, up, column_q(lo, up, integral, cfg), snap[j].flags};
      snap[j] = s;
    }
    if (D.enabled) {
      // changed columns of this round -> list (one atomic per warp)
      const unsigned act = __activemask();
      const unsigned chm = __ballot_sync(act, c != 0);
      if (chm) {
        const int leader = __ffs(act) - 1;
        int base = 0;
        if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(&st->nchg[cb], __popc(chm));
        base = __shfl_sync(act, base, leader);
        if (c) D.chg_list[(size_t)cb * D.n + base + __popc(chm & ((1u << (threadIdx.x & 31)) - 1u))] = j;
      }
    }
    if (lo > __dadd_rn(up, cfg.imp_abs)) inf = 1;
  }
  if (D.enabled) {
    // the consumed marks become the round-after-next's mark set
    uint32_t* f = reinterpret_cast<uint32_t*>(D.row_flag + (size_t)cb * D.ms);
    for (int i = gtid; i < D.ms / 4; i += gstride) f[i] = 0u;
  }
  changes = block_sum<kCommitThreads>(changes, inf);
  if (threadIdx.x == 0) {
    if (changes) atomicAdd(&st->round_changes, changes);
    if (inf) st->infeasible = 1;
    __threadfence();
    const uint32_t t = atomicAdd(&st->ticket, 1u);
    if (t == gridDim.x - 1) {
      // last CTA: the round decision of run_parallel (par_engine.cpp:248-266)
      __threadfence();
      const long long ch = (long long)atomicAdd(&st->round_changes, 0ull);
      // key_out[n].x: the all-reduced infeasibility of every rank (row shards)
      volatile long long* slot = (volatile long long*)&key_out[n].x;
      const int infeasible = atomicAdd(&st->infeasible, 0) | (*slot != 0);
      *slot = 0;
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
      st->wl_count = 0;
      st->work = 0;
      st->full = 0;
      st->nchg[nb] = 0;  // the list k_mark consumed after the previous commit
      __threadfence();
      if (use_graph) cudaGraphSetConditional(cond, status >= 0 ? 0u : 1u);
    }
  }
}

// Start of a solve: snapshot records and merge keys from the (normalised)
// start bounds, state reset, bounds_crossed pre-check (engine_common.hpp:51-58).
__global__ void __launch_bounds__(kCommitThreads)
    k_reset(const double* __restrict__ lo0, const double* __restrict__ up0,
            const uint8_t* __restrict__ integral, Snap* __restrict__ snap,
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
      st->wl_count = 0;
      st->work = 0;
      // warm start from a root fixpoint: round 1 visits only the rows that
      // k_mark_vars marks (see NodeCtl)
      st->full = (D.enabled && ctl->warm) ? 0 : 1;
      st->nchg[0] = st->nchg[1] = 0;
      st->frac_any = atomicAdd(&st->frac_tmp, 0);
      st->frac_tmp = 0;
      st->ticket_reset = 0;
      __threadfence();
      if (use_graph) cudaGraphSetConditional(cond, cr ? 0u : 1u);
    }
  }
}

// Row-sharded rounds: this rank's infeasibility into the slot that rides the
// bound all-reduce (max over {lb key, -ub key, flag}).
__global__ void k_flag_to_slot(const DevState* __restrict__ st, longlong2* __restrict__ slot) {
  if (threadIdx.x == 0) slot->x = *((volatile const int32_t*)&st->infeasible) ? 1 : 0;
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

// Session init: rows into length-sorted order (perm[new] = old), lhs/rhs
// normalised (model.hpp:147-151), integrality packed into bit 31 of the
// column index (no per-entry byte gather).  One warp per row.
__global__ void k_permute_rows(const int32_t* __restrict__ rp, const int32_t* __restrict__ cols,
                               const double* __restrict__ vals, const double* __restrict__ lhs,
                               const double* __restrict__ rhs, const int32_t* __restrict__ perm,
                               const int32_t* __restrict__ new_rp,
                               const uint8_t* __restrict__ integral, int32_t* __restrict__ colx,
                               double* __restrict__ new_vals, double* __restrict__ new_lhs,
                               double* __restrict__ new_rhs, int m, double thr) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m;
       i += (gridDim.x * blockDim.x) >> 5) {
    const int old = perm[i];
    const int b = rp[old], len = rp[old + 1] - b, nb = new_rp[i];
    for (int k = lane; k < len; k += 32) {
      const int32_t c = cols[b + k];
      colx[nb + k] = integral[c] ? (int32_t)(c | 0x80000000u) : c;
      new_vals[nb + k] = vals[b + k];
    }
    if (lane == 0) {
      const double l = lhs[old], h = rhs[old];
      new_lhs[i] = l >= thr ? CUDART_INF : (l <= -thr ? -CUDART_INF : l);
      new_rhs[i] = h >= thr ? CUDART_INF : (h <= -thr ? -CUDART_INF : h);
    }
  }
}

// Warm start of a branch-and-bound node (config C4): the start bounds are a
// converged root fixpoint with a few bounds overridden.  Every row of the
// root had all of its candidates rejected against the root bounds in the
// root's confirming round, so in the node's round 1 only rows containing an
// overridden column can produce anything; marking exactly those keeps the
// trajectory identical to a full sweep.
__global__ void __launch_bounds__(256)
    k_mark_vars(const Dirty D, const NodeCtl* __restrict__ ctl) {
  if (!D.enabled || !ctl->warm) return;
  uint8_t* flag = D.row_flag + (size_t)1 * D.ms;  // round 1 reads buffer (0 + 1) & 1
  const int lane = threadIdx.x & 31;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ctl->nvars;
       w += (gridDim.x * blockDim.x) >> 5) {
    const int j = ctl->vars[w];
    for (int e = D.col_ptr[j] + lane; e < D.col_ptr[j + 1]; e += 32) flag[D.col_row[e]] = 1;
  }
}

// start bounds of a node: the root fixpoint (copied before) + its overrides
__global__ void k_apply_node(double* __restrict__ lo0, double* __restrict__ up0,
                             const NodeCtl* __restrict__ ctl, double thr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ctl->nvars; i += gridDim.x * blockDim.x) {
    const int j = ctl->vars[i];
    const double l = ctl->lo[i], u = ctl->up[i];
    lo0[j] = l >= thr ? CUDART_INF : (l <= -thr ? -CUDART_INF : l);
    up0[j] = u >= thr ? CUDART_INF : (u <= -thr ? -CUDART_INF : u);
  }
}

// After the commit of round r: mark, for round r + 1, every row containing a
// column changed in round r (one warp per changed column).
__global__ void __launch_bounds__(256) k_mark(const Dirty D, DevState* __restrict__ st) {
  const int r = *((volatile int32_t*)&st->round);
  if (!D.enabled || *((volatile int32_t*)&st->done)) return;
  const int cb = r & 1, nb = (r + 1) & 1;
  const int nchg = *((volatile int32_t*)&st->nchg[cb]);
  uint8_t* flag = D.row_flag + (size_t)nb * D.ms;
  const int lane = threadIdx.x & 31;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nchg;
       w += (gridDim.x * blockDim.x) >> 5) {
    const int j = D.chg_list[(size_t)cb * D.n + w];
    for (int e = D.col_ptr[j] + lane; e < D.col_ptr[j + 1]; e += 32) {
      const int row = D.col_row[e];
      if (!flag[row]) flag[row] = 1;  // read first: most rows are marked repeatedly
    }
  }
}

// ---- worklist index (session init) -----------------------------------------------

// column counts (one warp per row)
__global__ void k_csc_count(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ colx,
                            int m, int32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m;
       i += (gridDim.x * blockDim.x) >> 5)
    for (int k = row_ptr[i] + lane; k < row_ptr[i + 1]; k += 32)
      atomicAdd(&cnt[colx[k] & 0x7fffffff], 1);
}

__global__ void k_csc_fill(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ colx,
                           int m, int32_t* __restrict__ cursor, int32_t* __restrict__ col_row) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m;
       i += (gridDim.x * blockDim.x) >> 5)
    for (int k = row_ptr[i] + lane; k < row_ptr[i + 1]; k += 32)
      col_row[atomicAdd(&cursor[colx[k] & 0x7fffffff], 1)] = i;
}

}  // namespace pgb
