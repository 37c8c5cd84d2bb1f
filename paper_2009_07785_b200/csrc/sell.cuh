// sell.cuh -- one propagation round over a sliced-ELL copy of the matrix.
//
// Work units are the serial activity chains of cpu_par (par_engine.cpp:
// 126-146, 99-123): every row of at most nnz_budget entries is ONE chain
// (compute_row_activities in entry order, propcore.hpp:45-65), and a longer
// row is split into chains of nnz_budget entries whose partial records are
// combined pairwise afterwards (wide_row_activities).  Units are sorted by
// length, descending, and cut into slices (kernels.cuh, SliceDesc): short
// units one per lane, long units spread over G = 2/4/8 lanes so that no
// warp carries a 1024-step dependent chain.
//
// Phase 1 (per slice, one warp): every lane loads its entries (coalesced,
// one 256 B / 128 B request per step), gathers the column's record (32 B
// snapshot, 16 B bounds or 8 B float bounds, chosen per session; one L2
// sector, kept resident with an evict_last policy while the matrix streams
// through with evict_first), and forms the entry's min/max contributions.
// The G lanes of a unit hand their products to the unit's owner lanes in
// entry order (a padded shared-memory step buffer), so each sum is the
// reference's sequential chain, bit for bit.  Each entry also stores a 4-byte filter
// word: its filter term |a| q rounded up to float, with the two infinity
// flags in the low mantissa bits (always >= the exact term, so a test on it
// never drops an entry the exact test keeps).
//
// Phase 2 (same warp, whole rows only): row check (propcore.hpp:147-156),
// row filter, then one pass over the slice's filter words; the entries that
// may tighten are compacted into a per-warp queue and run through the exact
// candidate pipeline 32 at a time (re-loading only those entries).  Chunks
// of split rows write partial records; the last chunk combines them in
// chunk order and queues the row's pieces for k_cand (cand.cuh).
#pragma once

#include "kernels.cuh"
#include "setup.cuh"
#include "split.cuh"

namespace pgb {

#ifndef PG_SELL_UNROLL
#define PG_SELL_UNROLL 4
#endif
#ifndef PG_SELL_HINTS
#define PG_SELL_HINTS 1
#endif
#ifndef PG_SELL_PF
// lane 0 bulk-prefetching a slice's streams into L2 ahead of its loads:
// measured slower on the final kernels (C2 first round 163.8 -> 161.6 us,
// C3 687 -> 668 us without; long-row sweeps are L1-throughput-bound and each
// prefetch is an LSU instruction), so off by default
#define PG_SELL_PF 0
#endif
#ifndef PG_SELL_GROUP
#define PG_SELL_GROUP 2  // narrow one-lane slices per work item
#endif
#ifndef PG_SELL_GROUPW
#define PG_SELL_GROUPW 16  // slices at most this wide are grouped
#endif
#ifndef PG_SELL_LANEUNIT
#define PG_SELL_LANEUNIT 32
#endif
#ifndef PG_SELL_MIDMAX
#define PG_SELL_MIDMAX 128
#endif
#ifndef PG_SELL_XSMEM
#define PG_SELL_XSMEM 1  // multi-lane chains: products to the owner lane through shared memory
#endif
#ifndef PG_SELL_DEBUG
#define PG_SELL_DEBUG 0  // 1: cfg.flags 0x10000 skips phase 2 (timing experiments)
#endif
#ifndef PG_SELL_UL0
#define PG_SELL_UL0 PG_SELL_UNROLL  // full sweeps, one-lane slices: steps in flight per lane
#endif
#ifndef PG_SELL_LGU
#define PG_SELL_LGU 2  // slices with lg >= this use PG_SELL_ULONG steps per group
#endif
#ifndef PG_SELL_ULONG
#define PG_SELL_ULONG 2
#endif
#ifndef PG_SELL_LGMAX
#define PG_SELL_LGMAX 3
#endif
#ifndef PG_SELL_MINB_DENSE
#define PG_SELL_MINB_DENSE 2  // resident CTAs per SM the full sweep is compiled for
#endif
#ifndef PG_SELL_DISCARD
#define PG_SELL_DISCARD 1  // drop the filter words' L2 lines after phase 2 (no write-back)
#endif
#ifndef PG_SELL_WPF
#define PG_SELL_WPF 0
#endif
#ifndef PG_SELL_XPAD
#define PG_SELL_XPAD 1  // padded step buffer of multi-lane chains (bank-conflict free loads)
#endif
#ifndef PG_SELL_GNA
#define PG_SELL_GNA 1  // snapshot gathers with L1::no_allocate (C2 first round 179 -> 176 us)
#endif
#ifndef PG_SELL_MINB
#define PG_SELL_MINB 2
#endif
constexpr int kSellUnroll = PG_SELL_UNROLL;
constexpr int kSellThreads = 256;
constexpr int kSellWarps = kSellThreads / 32;
constexpr int kSellGroup = PG_SELL_GROUP;
#ifndef PG_MID_UNROLL
#define PG_MID_UNROLL 4  // C5 worklist rounds: 7.70 -> 7.46 ms (2: round-1 value, 8: 7.66)
#endif
constexpr int kMidU = PG_MID_UNROLL;
#ifndef PG_UNITS_UNROLL
#define PG_UNITS_UNROLL 4
#endif
constexpr int kUnitsU = PG_UNITS_UNROLL;  // worklist lane units: chain steps in flight  // worklist mid units: 8-entry steps in flight
constexpr int kSellLaneUnit = PG_SELL_LANEUNIT;  // worklist rounds: longer units get a warp each
constexpr int kSellMidMax = PG_SELL_MIDMAX;      //   (up to this length: 8 lanes each)
// lanes per unit by unit length: > 256 -> 8, > 128 -> 4, > 64 -> 2, else 1
#ifndef PG_SELL_G8
#define PG_SELL_G8 256
#endif
#ifndef PG_SELL_G4
#define PG_SELL_G4 128
#endif
constexpr int kSellG8 = PG_SELL_G8, kSellG4 = PG_SELL_G4, kSellG2 = 64;

// ---- memory access helpers ------------------------------------------------------
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void ld_snap_keep(const Snap* p, uint64_t pol, double& lo, double& up,
                                             double& q) {
#if !PG_SELL_HINTS
  ld_snap(p, lo, up, q);
  return;
#endif
  [[maybe_unused]] long long f;  // the flags word rides along in the 256-bit load
#if PG_SELL_GNA
  // no L1 allocation: the records have no reuse within an SM's L1 lifetime
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(lo), "=d"(up), "=d"(q), "=l"(f)
               : "l"(p), "l"(pol));
  return;
#endif
  asm volatile("ld.global.nc.L2::cache_hint.v4.b64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(lo), "=d"(up), "=d"(q), "=l"(f)
               : "l"(p), "l"(pol));
}
__device__ __forceinline__ double ld_stream_f64(const double* p, uint64_t pol) {
#if !PG_SELL_HINTS
  return __ldg(p);
#endif
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ld_stream_s32(const int32_t* p, uint64_t pol) {
#if !PG_SELL_HINTS
  return __ldg(p);
#endif
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// filter coefficient from the bounds (column_q): an infinite bound makes
// (up - lo) infinite; a NaN (both bounds the same infinity) reads as +inf
__device__ __forceinline__ double column_q_inline(double lo, double up, bool integral,
                                                  bool frac_any, const DevCfg& c) {
  const double thr = integral ? c.int_eps : c.imp_abs + c.imp_rel;
  double q = ((up - lo) - thr) + (fabs(lo) + fabs(up)) * kMargin;
  if (frac_any && integral && (lo != floor(lo) || up != ceil(up))) q = CUDART_INF;
  return q == q ? q : CUDART_INF;
}

// the gathered record of column c: {lb, ub} and the filter coefficient q --
// 16 B from the compact bounds array (two columns per sector: rows dense in
// the columns, config C3; q recomputed, column_q) or the 32 B snapshot record
// (q precomputed: sparse rows, one sector per entry either way)
template <class RA>
__device__ __forceinline__ void ld_col(const RA& A, int32_t c, uint64_t pol, bool frac_any,
                                       const DevCfg& cfg, double& lo, double& up, double& q) {
  if constexpr (coherent_v<RA>) {
    ld_snap_coh(A.snap + (c & 0x7fffffff), lo, up, q);
  } else if constexpr (gather8_v<RA>) {
    const int32_t j = c & 0x7fffffff;
    float2 f;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                 : "=f"(f.x), "=f"(f.y)
                 : "l"(cfg.bf + j), "l"(pol));
    if (f.x == f.x) {
      lo = f.x;
      up = f.y;
    } else {
      // a bound that is not a float: the exact record
      double2 b;
      asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                   : "=d"(b.x), "=d"(b.y)
                   : "l"(A.bnd + j), "l"(pol));
      lo = b.x;
      up = b.y;
    }
    q = column_q_inline(lo, up, c < 0, frac_any, cfg);
  } else if constexpr (gather16_v<RA>) {
    double2 b;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(b.x), "=d"(b.y)
                 : "l"(A.bnd + (c & 0x7fffffff)), "l"(pol));
    lo = b.x;
    up = b.y;
    q = column_q_inline(lo, up, c < 0, frac_any, cfg);
  } else {
    ld_snap_keep(A.snap + (c & 0x7fffffff), pol, lo, up, q);
  }
}

// ---- filter words -----------------------------------------------------------------
// Per entry a 32-bit word: the filter term x = |a| q rounded up to float as
// a monotone int32 key (negative floats bit-reversed), the two low bits
// replaced by the infinity flags (bit 0: min contribution infinite, bit 1:
// max contribution infinite).  (w | 3) is the key of a float >= x, the row
// thresholds are keyed after rounding down, so a test on a word is never
// stricter than the exact one (kernels.cuh entry_may) and all tests are
// integer compares.  A NaN term (a = 0 with an infinite bound, which never
// yields a candidate) keys as -inf, so it cannot mask the row's maximum.
__device__ __forceinline__ int32_t fkey_of(float f) {
  const int32_t b = __float_as_int(f);
  return b ^ ((b >> 31) & 0x7fffffff);
}
constexpr int32_t kFKeyMin = (int32_t)0x807fffff;  // key of -inf: the empty maximum
__device__ __forceinline__ int32_t fword(double x, bool imin, bool imax) {
  const float f = fmaxf(__double2float_ru(x), -CUDART_INF_F);
  return (fkey_of(f) & ~3) | (imin ? 1 : 0) | (imax ? 2 : 0);
}
// a double >= every term behind the largest word xk (+inf's key | 3 is a NaN pattern)
__device__ __forceinline__ double fkey_bound(int32_t xk) {
  const int32_t k = xk | 3;
  const float f = __int_as_float(k ^ ((k >> 31) & 0x7fffffff));
  return f == f ? (double)f : CUDART_INF;
}
// per-unit form of the row filter: each enabled side's threshold rounded
// down to float and keyed (a disabled side keys above every word), and the
// flag mask of the one-infinite-entry sides
struct FTest {
  int32_t tr, tl, fm;
};
__device__ __forceinline__ FTest ftest(const RowFilter& f) {
  FTest r;
  r.tr = (f.mode & 1) ? fkey_of(__double2float_rd(f.tr)) : 0x7fffffff;
  r.tl = (f.mode & 2) ? fkey_of(__double2float_rd(f.tl)) : 0x7fffffff;
  r.fm = ((f.mode & 4) ? 1 : 0) | ((f.mode & 8) ? 2 : 0);
  return r;
}
__device__ __forceinline__ bool fpass(const FTest& t, int32_t w) {
  const int32_t x = w | 3;
  return x >= t.tr || x >= t.tl || (w & t.fm) != 0;
}
__device__ __forceinline__ bool frow_may(const FTest& t, int32_t xk) {
  return t.fm != 0 || (xk | 3) >= min(t.tr, t.tl);
}
__device__ __forceinline__ bool is_inf(double x) { return fabs(x) == CUDART_INF; }

// The slice's filter words are dead once its phase 2 has read them (every
// round writes them again before reading): their L2 lines are dropped
// without a write-back (one 128 B line per step: 32 words of one step).
// sw points at this lane's word of step 0.
__device__ __forceinline__ void discard_words(const int32_t* sw, int steps, int lane) {
  if (!PG_SELL_DISCARD) return;
  const int32_t* p = sw - lane;
  for (int t = lane; t < steps; t += 32)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p + 32 * t) : "memory");
}

// ---- per-warp shared state ----------------------------------------------------------
struct SellWarpSmem {
  double min_f[32], max_f[32], lhs[32], rhs[32];
  int32_t min_i[32], max_i[32];
  int32_t tkr[32], tkl[32], fmask[32];
  uint8_t mode[32], may[32];
  // entries that survive the filter: element offset in the slice, unit
  int32_t qe[64];
  uint8_t qu[64];
  double2 xb[48];  // one step's {min, max} products of a multi-lane slice (padded, sell_step)
  double2 wbuf[256];  // worklist rounds: {min, max} contributions of a wide unit's block
  double2 wbuf2[256];
};

constexpr size_t kSellSmem = sizeof(SellWarpSmem) * kSellWarps;
// full sweeps never touch the wide-unit buffers: their warps' records are
// packed at this stride (the dynamic shared memory of the dense kernel)
constexpr size_t kSellDenseStride = __builtin_offsetof(SellWarpSmem, wbuf);
constexpr size_t kSellSmemDense = kSellDenseStride * kSellWarps;
static_assert(kSellDenseStride % 16 == 0, "warp records stay 16 B aligned");

// exact pipeline over queue entries [0, cnt), one per lane
template <class RA>
__device__ __forceinline__ bool sell_drain(const RA& A, const SellWarpSmem& W,
                                           long long off, int cnt, int lane, uint64_t pol_keep,
                                           const DevCfg& cfg) {
  bool inf_flag = false;
  if (lane < cnt) {
    const int u = W.qu[lane];
    const long long e = off + W.qe[lane];
    const double a = A.sv[e];
    const int32_t c = A.sc[e];
    double lo, up, q;
    ld_col(A, c, pol_keep, ld_gpu(&A.st->frac_any) != 0, cfg, lo, up, q);
    const Act act = {W.min_f[u], W.max_f[u], W.min_i[u], W.max_i[u]};
    inf_flag = entry_pipeline(act, a, lo, up, W.lhs[u], W.rhs[u], c, A.key_out, cfg);
  }
  return inf_flag;
}

// One step of a unit's chain on this lane: contributions (propcore.hpp:50-62:
// b by the sign of a; an infinite b is counted, a finite one adds a*b),
// filter term and word.  Adding +0.0 (an infinite b, or a padding entry) is
// exact: the sums start at +0.0 and never become -0.0.  With G = 2^LG lanes
// per unit, the G entries of the step sit on lanes u, u + H, .. and are
// added in entry order: through the warp's shared step buffer by the owner
// lane (j = 0) alone, the only lane whose sums are used (PG_SELL_XSMEM; one
// store and G 16-byte loads instead of 2G shuffles, which made long-row
// sweeps L1-bound), or through shuffles by every lane of the unit.
template <int LG>
__device__ __forceinline__ void sell_step(double a, double lo, double up, double q, int u, Act& act,
                                          int32_t& xk, int32_t* pw, double2* xb = nullptr) {
  constexpr int G = 1 << LG, H = 32 >> LG;
  const double bmin = a > 0 ? lo : up;
  const double bmax = a > 0 ? up : lo;
  const bool imin = is_inf(bmin), imax = is_inf(bmax);
  const double pmin = imin ? 0.0 : __dmul_rn(a, bmin);
  const double pmax = imax ? 0.0 : __dmul_rn(a, bmax);
  act.min_i += imin;
  act.max_i += imax;
  const int32_t w = fword(fabs(a) * q, imin, imax);
  xk = max(xk, w);
  *pw = w;
  if (LG == 0) {
    act.min_f = __dadd_rn(act.min_f, pmin);
    act.max_f = __dadd_rn(act.max_f, pmax);
  } else if (PG_SELL_XSMEM) {
    // unit u's G products of the step land contiguously (min and max
    // arrays); lane u runs the min chain, lane H + u the max chain
    // (slice_max_to_owner hands it to lane u after the chains)
    const int lane = threadIdx.x & 31;
    const int j = lane >> (5 - LG);
    // unit u's products at stride XS: with G >= 4 two doubles of padding
    // put the owner lanes' 16-byte loads on disjoint banks (G = 8: the min
    // and max lanes' loads are one conflict-free wavefront; unpadded, four)
    constexpr int XS = (PG_SELL_XPAD && G >= 4) ? G + 2 : G;
    double* xmin = reinterpret_cast<double*>(xb);
    double* xmax = xmin + H * XS;
    __syncwarp();  // the previous step's loads are done
    xmin[u * XS + j] = pmin;
    xmax[u * XS + j] = pmax;
    __syncwarp();
    if (lane < 2 * H) {
      const double2* src = reinterpret_cast<const double2*>((lane < H ? xmin : xmax) + u * XS);
      double v[G];
#pragma unroll
      for (int i = 0; i < G / 2; ++i) {
        const double2 p = src[i];
        v[2 * i] = p.x;
        v[2 * i + 1] = p.y;
      }
      double acc = lane < H ? act.min_f : act.max_f;
#pragma unroll
      for (int jj = 0; jj < G; ++jj) acc = __dadd_rn(acc, v[jj]);
      if (lane < H) act.min_f = acc;
      else act.max_f = acc;
    }
  } else {
#pragma unroll
    for (int jj = 0; jj < G; ++jj) {
      const double vmin = __shfl_sync(0xffffffffu, pmin, u + H * jj);
      const double vmax = __shfl_sync(0xffffffffu, pmax, u + H * jj);
      act.min_f = __dadd_rn(act.min_f, vmin);
      act.max_f = __dadd_rn(act.max_f, vmax);
    }
  }
}

// after the chains of a multi-lane slice (PG_SELL_XSMEM): the max chain ran
// on lane H + u; the owner lane u takes it
template <int LG>
__device__ __forceinline__ void slice_max_to_owner(Act& act) {
  if (LG == 0 || !PG_SELL_XSMEM) return;
  constexpr int H = 32 >> LG;
  const int lane = threadIdx.x & 31;
  const double mx = __shfl_sync(0xffffffffu, act.max_f, (lane + H) & 31);
  if (lane < H) act.max_f = mx;
}

// a chunk of a split row: its partial record; after the sweep,
// k_split_finish combines the partials of every row whose chunks all ran
template <bool kRowCheck>
__device__ __forceinline__ void chunk_done(const RoundArgs& A, const UnitDesc& ud, const Act& act,
                                           double xmax, bool& inf_flag, const DevCfg& cfg) {
  const SegDesc d = A.segs[-ud.ref - 1];
  SegPartial* P = A.partial + d.out;
  P->min_f = act.min_f;
  P->max_f = act.max_f;
  P->xmax = xmax;
  P->min_i = act.min_i;
  P->max_i = act.max_i;
  atomicAdd(&A.row_done[d.rslot], 1);  // k_split_finish combines complete rows
}

// Second half of a slice, after its chains: order-free reductions over a
// unit's lanes, row finish on the owner lanes (row check, filter; chunks of
// split rows: partial record, last chunk combines), then phase 2 over the
// slice's filter words.
template <bool kRowCheck, int LG, class RA>
__device__ __forceinline__ void slice_tail(const RA& A, SellWarpSmem& W, const SliceDesc& sd,
                                           const UnitDesc& ud, bool active, int len, int lane,
                                           Act act, int32_t xk, double lhs_r, double rhs_r,
                                           uint64_t pol_keep, bool& inf_flag, const DevCfg& cfg) {
  constexpr int H = 32 >> LG;
  const int j = lane >> (5 - LG), u = lane & (H - 1);
  const bool whole = ud.ref >= 0;
  const int steps = sd.steps;
  const int32_t* sw = reinterpret_cast<const int32_t*>(A.sw) + sd.off + lane;
  // order-free parts over the unit's lanes
#pragma unroll
  for (int o = H; o < 32; o <<= 1) {
    act.min_i += __shfl_xor_sync(0xffffffffu, act.min_i, o);
    act.max_i += __shfl_xor_sync(0xffffffffu, act.max_i, o);
    xk = max(xk, __shfl_xor_sync(0xffffffffu, xk, o));
  }

  // ---- row finish (owner lanes) ----------------------------------------------------
  bool may = false;
  if (j == 0 && active) {
    if (whole) {
      const double l = lhs_r, h = rhs_r;
      if (kRowCheck && row_infeasible(act, l, h, cfg)) inf_flag = true;
      const RowFilter f = row_filter(act, l, h);
      const FTest ft = ftest(f);
      may = frow_may(ft, xk);
      W.tkr[u] = ft.tr;
      W.tkl[u] = ft.tl;
      W.fmask[u] = ft.fm;
      W.min_f[u] = act.min_f;
      W.max_f[u] = act.max_f;
      W.min_i[u] = act.min_i;
      W.max_i[u] = act.max_i;
      W.lhs[u] = l;
      W.rhs[u] = h;
      W.mode[u] = f.mode;
    } else {
      chunk_done<kRowCheck>(A, ud, act, fkey_bound(xk), inf_flag, cfg);
    }
  }
  if (j == 0) W.may[u] = may;
  if (PG_SELL_DEBUG && (cfg.flags & 0x10000u)) return;  // timing experiments only: no phase 2
  if (!__any_sync(0xffffffffu, may)) {
    discard_words(sw, steps, lane);
    return;
  }

  // ---- phase 2: filter words -> queue -> exact pipeline ------------------------------
  __syncwarp();
  const bool umay = W.may[u] != 0;
  FTest ft = {0x7fffffff, 0x7fffffff, 0};
  if (umay) ft = FTest{W.tkr[u], W.tkl[u], W.fmask[u]};
  int qn = 0;
  // PG_SELL_WPF: the next group's words are in flight while this group is
  // tested (their latency was exposed once per group of every slice)
  int32_t bn[kSellUnroll];
  if (PG_SELL_WPF) {
#pragma unroll
    for (int k = 0; k < kSellUnroll; ++k) bn[k] = umay && (k << LG) + j < len ? sw[32 * k] : 0;
  }
  for (int t0 = 0; t0 < steps; t0 += kSellUnroll) {
    int32_t b[kSellUnroll];
    bool in[kSellUnroll];
#pragma unroll
    for (int k = 0; k < kSellUnroll; ++k) {
      in[k] = umay && ((t0 + k) << LG) + j < len;
      if (PG_SELL_WPF) {
        b[k] = bn[k];
        const int tn = t0 + kSellUnroll + k;
        bn[k] = umay && (tn << LG) + j < len ? sw[32 * tn] : 0;
      } else {
        b[k] = in[k] ? sw[32 * (t0 + k)] : 0;
      }
    }
#pragma unroll
    for (int k = 0; k < kSellUnroll; ++k) {
      const bool pass = in[k] && fpass(ft, b[k]);
      const unsigned m = __ballot_sync(0xffffffffu, pass);
      if (!m) continue;
      if (pass) {
        const int slot = qn + __popc(m & ((1u << lane) - 1u));
        W.qe[slot] = 32 * (t0 + k) + lane;
        W.qu[slot] = (uint8_t)u;
      }
      qn += __popc(m);
      if (qn >= 32) {
        __syncwarp();
        inf_flag |= sell_drain(A, W, sd.off, 32, lane, pol_keep, cfg);
        __syncwarp();
        qn -= 32;
        if (lane < qn) {
          W.qe[lane] = W.qe[32 + lane];
          W.qu[lane] = W.qu[32 + lane];
        }
        __syncwarp();
      }
    }
  }
  if (qn) {
    __syncwarp();
    inf_flag |= sell_drain(A, W, sd.off, qn, lane, pol_keep, cfg);
  }
  __syncwarp();
  discard_words(sw, steps, lane);
}

// One slice by one warp.  LG = log2(lanes per unit); kDense: a full sweep
// (no worklist), every lane walks every step of the slice.
template <bool kRowCheck, int LG, bool kDense, class RA>
__device__ __forceinline__ void sell_slice(const RA& A, SellWarpSmem& W, const SliceDesc& sd,
                                           int lane, bool full, const uint8_t* rflag,
                                           uint64_t pol_keep, uint64_t pol_stream, bool& inf_flag,
                                           const DevCfg& cfg) {
  constexpr int H = 32 >> LG;
  const int j = lane >> (5 - LG), u = lane & (H - 1);
  UnitDesc ud = {0, -1};
  bool active = u < sd.count;
  if (active) ud = A.units[sd.first + u];
  if (!full && active) {
    // worklist: the unit's row must carry a mark (split rows: all chunks of a
    // marked row are marked, so its finisher sees every partial)
    const int fr = ud.ref >= 0 ? ud.ref : A.srow[A.segs[-ud.ref - 1].rslot];
    active = rflag[fr] != 0;
  }
  if (!__any_sync(0xffffffffu, active)) return;
  const int len = active ? ud.len : 0;
  const double* sv = A.sv + sd.off + lane;
  const int32_t* sc = A.sc + sd.off + lane;
  int32_t* sw = reinterpret_cast<int32_t*>(A.sw) + sd.off + lane;
  const int steps = sd.steps;
  const bool frac_any = ld_gpu(&A.st->frac_any) != 0;

  // ---- phase 1: the chains ------------------------------------------------------
  Act act = {0.0, 0.0, 0, 0};
  int32_t xk = kFKeyMin;
  if (kDense) {
    constexpr int UL = LG >= PG_SELL_LGU ? PG_SELL_ULONG : LG == 0 ? PG_SELL_UL0 : kSellUnroll;
    // every lane walks all `steps` of the slice: entries past a unit's end are
    // padding (value 0, the padding column with bounds [0, 0]) and add +0.0
    const double* pa = sv;
    const int32_t* pc = sc;
    int32_t* pw = sw;
    int t = 0;
    double a[UL];
    int32_t c[UL];
    if (UL <= steps) {
#pragma unroll
      for (int k = 0; k < UL; ++k) {
        a[k] = ld_stream_f64(pa + 32 * k, pol_stream);
        c[k] = ld_stream_s32(pc + 32 * k, pol_stream);
      }
    }
    for (; t + UL <= steps; t += UL) {
      if (PG_SELL_PF && lane == 0 && t + 5 * UL <= steps) {
        prefetch_l2(pa + 32 * 4 * UL, 256u * UL);
        prefetch_l2(pc + 32 * 4 * UL, 128u * UL);
      }
      double lo[UL], up[UL], q[UL];
#pragma unroll
      for (int k = 0; k < UL; ++k)
        ld_col(A, c[k], pol_keep, frac_any, cfg, lo[k], up[k], q[k]);
      // the next group's values and columns are in flight during this one
      double an[UL];
      int32_t cn[UL];
      const bool more = t + 2 * UL <= steps;
#pragma unroll
      for (int k = 0; k < UL; ++k) {
        an[k] = 0.0;
        cn[k] = 0;
        if (more) {
          an[k] = ld_stream_f64(pa + 32 * (UL + k), pol_stream);
          cn[k] = ld_stream_s32(pc + 32 * (UL + k), pol_stream);
        }
      }
#pragma unroll
      for (int k = 0; k < UL; ++k)
        sell_step<LG>(a[k], lo[k], up[k], q[k], u, act, xk, pw + 32 * k, W.xb);
#pragma unroll
      for (int k = 0; k < UL; ++k) {
        a[k] = an[k];
        c[k] = cn[k];
      }
      pa += 32 * UL;
      pc += 32 * UL;
      pw += 32 * UL;
    }
    for (; t < steps; ++t) {
      const double a1 = ld_stream_f64(pa, pol_stream);
      const int32_t c1 = ld_stream_s32(pc, pol_stream);
      double lo1, up1, q1;
      ld_col(A, c1, pol_keep, frac_any, cfg, lo1, up1, q1);
      sell_step<LG>(a1, lo1, up1, q1, u, act, xk, pw, W.xb);
      pa += 32;
      pc += 32;
      pw += 32;
    }
  } else {
    // worklist rounds: only the marked units' entries
    for (int t0 = 0; t0 < steps; t0 += kSellUnroll) {
      double a[kSellUnroll], lo[kSellUnroll], up[kSellUnroll], q[kSellUnroll];
      int32_t c[kSellUnroll];
      bool in[kSellUnroll];
#pragma unroll
      for (int k = 0; k < kSellUnroll; ++k) {
        in[k] = ((t0 + k) << LG) + j < len;
        a[k] = 0.0;
        c[k] = A.pad_col;
        if (in[k]) {
          a[k] = ld_stream_f64(sv + 32 * (t0 + k), pol_stream);
          c[k] = ld_stream_s32(sc + 32 * (t0 + k), pol_stream);
        }
      }
#pragma unroll
      for (int k = 0; k < kSellUnroll; ++k)
        ld_col(A, c[k], pol_keep, frac_any, cfg, lo[k], up[k], q[k]);
#pragma unroll
      for (int k = 0; k < kSellUnroll; ++k)
        if (t0 + k < steps) sell_step<LG>(a[k], lo[k], up[k], q[k], u, act, xk, sw + 32 * (t0 + k), W.xb);
    }
  }
  if (PG_SELL_DEBUG && (cfg.flags & 0x40000u)) {  // timing experiments only: chains alone
    if (act.min_f == 12345.678 && xk == 1) A.st->infeasible = 1;
    return;
  }
  slice_max_to_owner<LG>(act);
  slice_tail<kRowCheck, LG>(A, W, sd, ud, active, len, lane, act, xk, ud.ref >= 0 ? A.lhs[ud.ref] : 0.0,
                            ud.ref >= 0 ? A.rhs[ud.ref] : 0.0, pol_keep, inf_flag, cfg);
}

// R narrow slices (one lane per unit) by one warp: every lane runs R
// independent chains, interleaved, so each step has R entries in flight per
// lane and the per-slice latencies (descriptors, row sides, the ticket)
// are paid once per R slices.  Full sweeps only.
template <bool kRowCheck, int R, class RA>
__device__ __forceinline__ void sell_group(const RA& A, SellWarpSmem& W, int s0, int nr,
                                           int lane, uint64_t pol_keep, uint64_t pol_stream,
                                           bool& inf_flag, const DevCfg& cfg) {
  long long off[R];
  int steps[R], cnt[R];
  UnitDesc ud[R];
  double l[R], h[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    SliceDesc d = {0, 0, 0, 0, 0, 0, 0};
    if (r < nr) d = A.slices[s0 + r];
    off[r] = d.off + lane;
    steps[r] = d.steps;
    cnt[r] = d.count;
    ud[r] = UnitDesc{0, -1};
    if (lane < d.count) ud[r] = A.units[d.first + lane];
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    l[r] = h[r] = 0.0;
    if (ud[r].ref >= 0) {
      l[r] = A.lhs[ud[r].ref];
      h[r] = A.rhs[ud[r].ref];
    }
  }
  Act act[R];
  int32_t xk[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    act[r] = Act{0.0, 0.0, 0, 0};
    xk[r] = kFKeyMin;
  }
  const int tmax = steps[0];  // the group's first slice is its widest
  const bool frac_any = ld_gpu(&A.st->frac_any) != 0;
  double a[R];
  int32_t c[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    a[r] = 0.0;
    c[r] = A.pad_col;
    if (0 < steps[r]) {
      a[r] = ld_stream_f64(A.sv + off[r], pol_stream);
      c[r] = ld_stream_s32(A.sc + off[r], pol_stream);
    }
  }
  for (int t = 0; t < tmax; ++t) {
    double lo[R], up[R], q[R];
#pragma unroll
    for (int r = 0; r < R; ++r) ld_col(A, c[r], pol_keep, frac_any, cfg, lo[r], up[r], q[r]);
    double an[R];
    int32_t cn[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      an[r] = 0.0;
      cn[r] = A.pad_col;
      if (t + 1 < steps[r]) {
        an[r] = ld_stream_f64(A.sv + off[r] + 32 * (t + 1), pol_stream);
        cn[r] = ld_stream_s32(A.sc + off[r] + 32 * (t + 1), pol_stream);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (t < steps[r]) sell_step<0>(a[r], lo[r], up[r], q[r], lane, act[r], xk[r], reinterpret_cast<int32_t*>(A.sw) + off[r] + 32 * t);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      a[r] = an[r];
      c[r] = cn[r];
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r < nr) {
      const SliceDesc d = {off[r] - lane, 0, 0, steps[r], (int16_t)cnt[r], 0, 0};
      slice_tail<kRowCheck, 0>(A, W, d, ud[r], lane < cnt[r], ud[r].len, lane, act[r], xk[r],
                               l[r], h[r], pol_keep, inf_flag, cfg);
    }
  }
}

// Persistent, one warp per slice (longest first).  kDense: a full sweep;
// otherwise a worklist round (only the marked rows' units).  Both are
// launched when the worklist is on; the one that does not match the round
// returns at once (the round's kind is known on the device only).
// Worklist round, multi-lane (long) units: a warp per unit over its CSR
// entries (coalesced), 256 entries per block; the lanes form the
// contributions, lane 0 adds them in entry order from shared memory (the
// reference's chain), then row finish and phase 2 with the exact filter.
template <bool kRowCheck, class RA>
__device__ __forceinline__ void sell_wide(const RA& A, SellWarpSmem& W, int par,
                                          uint64_t pol_keep, bool& inf_flag, const DevCfg& cfg) {
  const int lane = threadIdx.x & 31;
  const int nw = ld_gpu(&A.st->nwide[par]);  // the list's front: long units
  const int32_t* wl = A.dirty.wide_list + (size_t)par * A.dirty.nunits;
  const bool frac_any = ld_gpu(&A.st->frac_any) != 0;
  // static striding by warp (few, similar items: no ticket contention)
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < nw; t += nwarps) {
    const int u = wl[t];
    const UnitDesc ud = A.units[u];
    const int k0 = ud.ref >= 0 ? A.row_ptr[ud.ref] : A.segs[-ud.ref - 1].k0;
    const int len = ud.len;
#if PG_SELL_DEBUG
    const long long dbg_t0 = clock64();
    long long dbg_t1 = 0;
#endif
    int cmin = 0, cmax = 0;
    double xm = -CUDART_INF, smin = 0.0, smax = 0.0;
    // double-buffered blocks of 256 entries: the loads and gathers of block
    // b + 1 are in flight while lanes 0 / 1 add block b's contributions
    double a8[8];
    int32_t c8[8];
    auto load_block = [&](int base) {
#pragma unroll
      for (int s8 = 0; s8 < 8; ++s8) {
        const int e = base + 32 * s8 + lane;
        a8[s8] = 0.0;
        c8[s8] = A.pad_col;
        if (e < len) {
          a8[s8] = A.vals[k0 + e];
          c8[s8] = A.colx[k0 + e];
        }
      }
    };
    auto product_block = [&](int base, double2* buf) {
#pragma unroll
      for (int s8 = 0; s8 < 8; ++s8) {
        const int e = base + 32 * s8 + lane;
        double lo, up, q;
        ld_col(A, c8[s8], pol_keep, frac_any, cfg, lo, up, q);
        double pmin = 0.0, pmax = 0.0;
        if (e < len) {
          const double a = a8[s8];
          const double bmin = a > 0 ? lo : up;
          const double bmax = a > 0 ? up : lo;
          const bool imin = isinf(bmin), imax = isinf(bmax);
          pmin = imin ? 0.0 : __dmul_rn(a, bmin);
          pmax = imax ? 0.0 : __dmul_rn(a, bmax);
          cmin += imin;
          cmax += imax;
          xm = fmax(xm, fabs(a) * q);
        }
        buf[32 * s8 + lane] = make_double2(pmin, pmax);
      }
    };
    load_block(0);
    product_block(0, W.wbuf);
    __syncwarp();
    for (int base = 0; base < len; base += 256) {
      double2* cur = base & 256 ? W.wbuf2 : W.wbuf;
      double2* nxt = base & 256 ? W.wbuf : W.wbuf2;
      const bool more = base + 256 < len;
      if (more) load_block(base + 256);
      if (lane < 2) {
        // lane 0 runs the min chain, lane 1 the max chain, in entry order
        // (entries past the end are +0.0, which adds exactly)
        const double* wb = reinterpret_cast<const double*>(cur) + lane;
        const int nb = min(256, len - base);
        double acc = lane ? smax : smin;
        for (int i = 0; i < nb; i += 8) {
          double v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = wb[2 * (i + k)];
#pragma unroll
          for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, v[k]);
        }
        if (lane) smax = acc; else smin = acc;
      }
      if (more) product_block(base + 256, nxt);
      __syncwarp();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      cmin += __shfl_xor_sync(0xffffffffu, cmin, o);
      cmax += __shfl_xor_sync(0xffffffffu, cmax, o);
      xm = fmax(xm, __shfl_xor_sync(0xffffffffu, xm, o));
    }
    const Act act = {__shfl_sync(0xffffffffu, smin, 0), __shfl_sync(0xffffffffu, smax, 1), cmin, cmax};
#if PG_SELL_DEBUG
    dbg_t1 = clock64();
#endif
    if (ud.ref < 0) {
      if (lane == 0) chunk_done<kRowCheck>(A, ud, act, xm, inf_flag, cfg);
#if PG_SELL_DEBUG
      if (lane == 0 && (cfg.flags & 0x200000u))
        printf("[wide] chunk len %d phase1 %lld cyc\n", len, dbg_t1 - dbg_t0);
#endif
      continue;
    }
    const double l = A.lhs[ud.ref], h = A.rhs[ud.ref];
    if (kRowCheck && lane == 0 && row_infeasible(act, l, h, cfg)) inf_flag = true;
    const RowFilter f = row_filter(act, l, h);
    if (!row_may(f, xm)) continue;
    // phase 2: 8 entries per lane in flight, then the survivors' pipeline
    for (int e0 = 0; e0 < len; e0 += 256) {
      double a[8], lo[8], up[8];
      int32_t c[8];
      unsigned pass = 0;
#pragma unroll
      for (int s8 = 0; s8 < 8; ++s8) {
        const int e = e0 + 32 * s8 + lane;
        a[s8] = 0.0;
        c[s8] = A.pad_col;
        if (e < len) {
          a[s8] = A.vals[k0 + e];
          c[s8] = A.colx[k0 + e];
        }
      }
#pragma unroll
      for (int s8 = 0; s8 < 8; ++s8) {
        double q;
        ld_col(A, c[s8], pol_keep, frac_any, cfg, lo[s8], up[s8], q);
        const double bmin = a[s8] > 0 ? lo[s8] : up[s8];
        const double bmax = a[s8] > 0 ? up[s8] : lo[s8];
        if (e0 + 32 * s8 + lane < len && entry_may(f, fabs(a[s8]) * q, isinf(bmin), isinf(bmax)))
          pass |= 1u << s8;
      }
#pragma unroll
      for (int s8 = 0; s8 < 8; ++s8)
        if ((pass >> s8) & 1u)
          if (entry_pipeline(act, a[s8], lo[s8], up[s8], l, h, c[s8], A.key_out, cfg, &A.touch))
            inf_flag = true;
    }
#if PG_SELL_DEBUG
    if (lane == 0 && (cfg.flags & 0x200000u))
      printf("[wide] row len %d phase1 %lld phase2 %lld cyc\n", len, dbg_t1 - dbg_t0, clock64() - dbg_t1);
#endif
  }
}

// Worklist round, mid-length units (longer than a lane unit, at most
// kSellMidMax entries: C5's 50-entry rows, C2's medium rows): 8 lanes per
// unit, four units per warp, over the unit's CSR entries.  Lane j of a group
// holds entries j, j + 8, ..; every lane of the group adds the 8 products of
// a step in entry order through shuffles (the reference's sequential chain,
// as sell_step<3>), so the group's lanes all hold the row record.  Phase 2
// re-reads the entries of a row that may tighten and applies the exact
// filter per entry.
template <bool kRowCheck, class RA>
__device__ __forceinline__ void sell_mid(const RA& A, int par, uint64_t pol_keep, bool& inf_flag,
                                         const DevCfg& cfg) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 3, j = lane & 7;
  const int nm = ld_gpu(&A.st->nmid[par]);
  const int32_t* ml = A.dirty.wide_list + (size_t)par * A.dirty.nunits + A.dirty.nunits - 1;
  const bool frac_any = ld_gpu(&A.st->frac_any) != 0;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  // warps count down from the last one, so the first warps (long units) and
  // the mid units start at once
  for (int b = nwarps - 1 - gw; 4 * b < nm; b += nwarps) {
    const int t = 4 * b + g;
    const bool have = t < nm;
    UnitDesc ud = {0, -1};
    int k0 = 0;
    if (have) {
      ud = A.units[ml[-t]];
      k0 = ud.ref >= 0 ? A.row_ptr[ud.ref] : A.segs[-ud.ref - 1].k0;
    }
    const int len = have ? ud.len : 0;
    int maxlen = len;
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    Act act = {0.0, 0.0, 0, 0};
    double xm = -CUDART_INF;
    // steps of 8 entries, kMidU in flight: loads of steps s .. s + kMidU - 1,
    // then their gathers, then the ordered adds
    for (int s0 = 0; 8 * s0 < maxlen; s0 += kMidU) {
      double a[kMidU], lo[kMidU], up[kMidU], q[kMidU];
      int32_t c[kMidU];
#pragma unroll
      for (int k = 0; k < kMidU; ++k) {
        const int e = 8 * (s0 + k) + j;
        a[k] = 0.0;
        c[k] = A.pad_col;
        if (e < len) {
          a[k] = A.vals[k0 + e];
          c[k] = A.colx[k0 + e];
        }
      }
#pragma unroll
      for (int k = 0; k < kMidU; ++k) ld_col(A, c[k], pol_keep, frac_any, cfg, lo[k], up[k], q[k]);
#pragma unroll
      for (int k = 0; k < kMidU; ++k) {
        if (8 * (s0 + k) >= maxlen) break;  // warp-uniform
        const bool in = 8 * (s0 + k) + j < len;
        const double bmin = a[k] > 0 ? lo[k] : up[k];
        const double bmax = a[k] > 0 ? up[k] : lo[k];
        const bool imin = in && is_inf(bmin), imax = in && is_inf(bmax);
        const double pmin = (!in || imin) ? 0.0 : __dmul_rn(a[k], bmin);
        const double pmax = (!in || imax) ? 0.0 : __dmul_rn(a[k], bmax);
        act.min_i += imin;
        act.max_i += imax;
        if (in) xm = fmax(xm, fabs(a[k]) * q[k]);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const double vmin = __shfl_sync(0xffffffffu, pmin, jj, 8);
          const double vmax = __shfl_sync(0xffffffffu, pmax, jj, 8);
          act.min_f = __dadd_rn(act.min_f, vmin);
          act.max_f = __dadd_rn(act.max_f, vmax);
        }
      }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      act.min_i += __shfl_xor_sync(0xffffffffu, act.min_i, o);
      act.max_i += __shfl_xor_sync(0xffffffffu, act.max_i, o);
      xm = fmax(xm, __shfl_xor_sync(0xffffffffu, xm, o));
    }
    if (!have) continue;
    if (ud.ref < 0) {
      if (j == 0) chunk_done<kRowCheck>(A, ud, act, xm, inf_flag, cfg);
      continue;
    }
    const double l = A.lhs[ud.ref], h = A.rhs[ud.ref];
    if (kRowCheck && j == 0 && row_infeasible(act, l, h, cfg)) inf_flag = true;
    const RowFilter f = row_filter(act, l, h);
    if (!row_may(f, xm)) continue;
    // phase 2 (no shuffles: the groups may diverge here)
    for (int e0 = j; e0 < len; e0 += 32) {
      double a[4], lo[4], up[4];
      int32_t c[4];
      unsigned pass = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = e0 + 8 * k;
        a[k] = 0.0;
        c[k] = A.pad_col;
        if (e < len) {
          a[k] = A.vals[k0 + e];
          c[k] = A.colx[k0 + e];
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double q;
        ld_col(A, c[k], pol_keep, frac_any, cfg, lo[k], up[k], q);
        const double bmin = a[k] > 0 ? lo[k] : up[k];
        const double bmax = a[k] > 0 ? up[k] : lo[k];
        if (e0 + 8 * k < len && entry_may(f, fabs(a[k]) * q, isinf(bmin), isinf(bmax)))
          pass |= 1u << k;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((pass >> k) & 1u)
          if (entry_pipeline(act, a[k], lo[k], up[k], l, h, c[k], A.key_out, cfg, &A.touch))
            inf_flag = true;
    }
  }
}

// Worklist round, one-lane units: a warp takes 32 marked units (any slices),
// one per lane; the chain reads the unit's column of its slice (entry i at
// off + 32 i + position), then row finish and an in-lane phase 2 over the
// unit's filter words.  Exact like the slice path; used when few rows are
// marked, so the uncoalesced lane streams do not matter.
template <bool kRowCheck, class RA>
__device__ __forceinline__ void sell_units(const RA& A, int par, uint64_t pol_keep,
                                           bool& inf_flag, const DevCfg& cfg) {
  const int lane = threadIdx.x & 31;
  const int nu = ld_gpu(&A.st->nunit[par]);
  const int32_t* ul = A.dirty.unit_list + (size_t)par * A.dirty.nunits;
  const bool frac_any = ld_gpu(&A.st->frac_any) != 0;
  // static striding: warp w takes batches w, w + W, .. of 32 units (the
  // batches after the wide units' warps, so both kinds start at once)
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nwide = ld_gpu(&A.st->nwide[par]);
  for (int b = (gw + nwarps - nwide % nwarps) % nwarps; 32 * b < nu; b += nwarps) {
    const int i = 32 * b + lane;
    if (i >= nu) continue;
    const int u = ul[i];
    const UnitDesc ud = A.units[u];
    const int k = u - A.lg0_ustart;
    const long long off = A.slices[A.lg0_sstart + (k >> 5)].off + (k & 31);
    const double* sv = A.sv + off;
    const int32_t* sc = A.sc + off;
    int32_t* sw = reinterpret_cast<int32_t*>(A.sw) + off;
    Act act = {0.0, 0.0, 0, 0};
    int32_t xk = kFKeyMin;
    for (int t0 = 0; t0 < ud.len; t0 += kUnitsU) {
      double a[kUnitsU], lo[kUnitsU], up[kUnitsU], q[kUnitsU];
      int32_t c[kUnitsU];
#pragma unroll
      for (int k = 0; k < kUnitsU; ++k) {
        a[k] = 0.0;
        c[k] = A.pad_col;
        if (t0 + k < ud.len) {
          a[k] = sv[32 * (t0 + k)];
          c[k] = sc[32 * (t0 + k)];
        }
      }
#pragma unroll
      for (int k = 0; k < kUnitsU; ++k) ld_col(A, c[k], pol_keep, frac_any, cfg, lo[k], up[k], q[k]);
#pragma unroll
      for (int k = 0; k < kUnitsU; ++k)
        if (t0 + k < ud.len) sell_step<0>(a[k], lo[k], up[k], q[k], 0, act, xk, sw + 32 * (t0 + k));
    }
    if (ud.ref < 0) {
      chunk_done<kRowCheck>(A, ud, act, fkey_bound(xk), inf_flag, cfg);
      continue;
    }
    const double l = A.lhs[ud.ref], h = A.rhs[ud.ref];
    if (kRowCheck && row_infeasible(act, l, h, cfg)) inf_flag = true;
    const FTest ft = ftest(row_filter(act, l, h));
    if (!frow_may(ft, xk)) continue;
    for (int t0 = 0; t0 < ud.len; t0 += 4) {
      // four entries' filter words, then the survivors' loads, then pipelines
      bool pass[4];
      double a[4], lo[4], up[4], q[4];
      int32_t c[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) pass[k] = t0 + k < ud.len && fpass(ft, sw[32 * (t0 + k)]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        a[k] = 0.0;
        c[k] = A.pad_col;
        if (pass[k]) {
          a[k] = sv[32 * (t0 + k)];
          c[k] = sc[32 * (t0 + k)];
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (pass[k]) ld_col(A, c[k], pol_keep, frac_any, cfg, lo[k], up[k], q[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (pass[k] && entry_pipeline(act, a[k], lo[k], up[k], l, h, c[k], A.key_out, cfg, &A.touch))
          inf_flag = true;
    }
  }
}

template <bool kRowCheck, bool kDense, class RA>
__device__ __forceinline__ void sell_sweep(const RA& A, const DevCfg& cfg,
                                           SellWarpSmem* smem) {
  const int lane = threadIdx.x & 31;
  SellWarpSmem& W = *reinterpret_cast<SellWarpSmem*>(
      reinterpret_cast<unsigned char*>(smem) +
      (size_t)(threadIdx.x >> 5) * (kDense ? kSellDenseStride : sizeof(SellWarpSmem)));
  const bool full = kDense;
  const int par = (ld_gpu(&A.st->round) + 1) & 1;
  const uint8_t* rflag = A.dirty.row_flag + (size_t)par * A.dirty.ms;
  const uint64_t pk = l2_policy_evict_last();
  const uint64_t ps = l2_policy_evict_first();
  bool inf_flag = false;
  if (!kDense) {
    // worklist round: only the units of the marked rows
    if (!(PG_SELL_DEBUG && (cfg.flags & 0x80000u))) sell_wide<kRowCheck>(A, W, par, pk, inf_flag, cfg);
    sell_mid<kRowCheck>(A, par, pk, inf_flag, cfg);
    if (!(PG_SELL_DEBUG && (cfg.flags & 0x100000u))) sell_units<kRowCheck>(A, par, pk, inf_flag, cfg);
    if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
    return;
  }
  // work items by ticket, longest first; the next ticket is taken when an
  // item starts and read when it ends (its latency hides under the item)
  int next = 0;
  if (lane == 0) next = ticket(&A.st->work);
  next = __shfl_sync(0xffffffffu, next, 0);
  const int nitems = A.group_start + (A.nslices - A.group_start + kSellGroup - 1) / kSellGroup;
  while (next < nitems) {
    const int s = next;
    int nxt = 0;
    if (lane == 0) nxt = ticket(&A.st->work);
    if (s >= A.group_start) {
      // a group of narrow one-lane slices
      const int s0 = A.group_start + (s - A.group_start) * kSellGroup;
      const int nr = min(kSellGroup, A.nslices - s0);
      if (kDense) {
        sell_group<kRowCheck, kSellGroup>(A, W, s0, nr, lane, pk, ps, inf_flag, cfg);
      } else {
        for (int r = 0; r < nr; ++r)
          sell_slice<kRowCheck, 0, kDense>(A, W, A.slices[s0 + r], lane, full, rflag, pk, ps,
                                           inf_flag, cfg);
      }
    } else {
      const SliceDesc sd = A.slices[s];
      if (PG_SELL_LGMAX >= 3 && sd.lg == 3)
        sell_slice<kRowCheck, (PG_SELL_LGMAX >= 3 ? 3 : 0), kDense>(A, W, sd, lane, full, rflag, pk, ps, inf_flag, cfg);
      else if (PG_SELL_LGMAX >= 2 && sd.lg == 2)
        sell_slice<kRowCheck, (PG_SELL_LGMAX >= 2 ? 2 : 0), kDense>(A, W, sd, lane, full, rflag, pk, ps, inf_flag, cfg);
      else if (PG_SELL_LGMAX >= 1 && sd.lg == 1)
        sell_slice<kRowCheck, (PG_SELL_LGMAX >= 1 ? 1 : 0), kDense>(A, W, sd, lane, full, rflag, pk, ps, inf_flag, cfg);
      else
        sell_slice<kRowCheck, 0, kDense>(A, W, sd, lane, full, rflag, pk, ps, inf_flag, cfg);
    }
    next = __shfl_sync(0xffffffffu, nxt, 0);
  }
  if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
}

// a full sweep: no worklist, the first round, or more than half of the
// slices dirty (then visiting all of them is cheaper than the list; exact
// either way)
__device__ __forceinline__ bool sell_dense_round(const RoundArgs& A) {
  return !round_is_sparse(A.st, A.dirty);
}

template <bool kRowCheck, bool kDense, int kG>
__global__ void __launch_bounds__(kSellThreads, kDense ? PG_SELL_MINB_DENSE : PG_SELL_MINB)
    k_sell(const RoundArgsG<kG> A,
                                                                     const DevCfg cfg) {
  extern __shared__ __align__(16) unsigned char sell_dyn[];  // kSellWarps x SellWarpSmem
  SellWarpSmem* smem = reinterpret_cast<SellWarpSmem*>(sell_dyn);
  pdl_begin();
  if (compute_off(A.st, cfg)) return;
  const bool dense = sell_dense_round(A);
  // the round's kind, for the commit kernels (written before any of them runs)
  if (kDense && blockIdx.x == 0 && threadIdx.x == 0) A.st->sparse_round = dense ? 0 : 1;
  if (dense != kDense) return;
  sell_sweep<kRowCheck, kDense>(A, cfg, smem);
}

// ---- session setup: units, slices, the sliced-ELL copy ---------------------------

// every chain as a unit: the segments (a segment that is a whole row becomes
// a row unit), then the short rows; key = descending length
__global__ void k_make_units(const SegDesc* __restrict__ segs, int nseg,
                             const int32_t* __restrict__ srow, const int32_t* __restrict__ sfirst,
                             const TileLayout lay, const int32_t* __restrict__ row_ptr,
                             int nunits, int maxlen, UnitDesc* __restrict__ units,
                             int32_t* __restrict__ k0, uint32_t* __restrict__ key,
                             int32_t* __restrict__ idx) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < nunits; u += gridDim.x * blockDim.x) {
    UnitDesc d;
    if (u < nseg) {
      const SegDesc g = segs[u];
      const bool whole = sfirst[g.rslot + 1] - sfirst[g.rslot] == 1;
      d = UnitDesc{g.len, whole ? srow[g.rslot] : -(u + 1)};
      k0[u] = g.k0;
    } else {
      int i = u - nseg, L = lay.nclass - 1;
      while (L > 0 && i >= lay.class_start[L + 1] - lay.class_start[L]) {
        i -= lay.class_start[L + 1] - lay.class_start[L];
        --L;
      }
      const int r = lay.class_start[L] + i;
      d = UnitDesc{L, r};
      k0[u] = row_ptr[r];
    }
    units[u] = d;
    key[u] = (uint32_t)(maxlen - d.len);
    idx[u] = u;
  }
}

// units and their CSR starts into sorted order
__global__ void k_order_units(const UnitDesc* __restrict__ in, const int32_t* __restrict__ k0in,
                              const int32_t* __restrict__ order, int nunits,
                              UnitDesc* __restrict__ out, int32_t* __restrict__ k0out) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < nunits; u += gridDim.x * blockDim.x) {
    out[u] = in[order[u]];
    k0out[u] = k0in[order[u]];
  }
}

// lanes per unit: by length, and at least 2^lg_min (small instances: more
// lanes per unit, shorter chains, enough warps to fill the GPU)
__host__ __device__ inline int sell_lg(int len, int lg_min) {
  const int lg = len > kSellG8 ? 3 : len > kSellG4 ? 2 : len > kSellG2 ? 1 : 0;
  return lg > lg_min ? lg : lg_min;
}

// region ends: cnt[lg] = one past the last unit with lanes-per-unit 2^lg
// (units sorted by descending length; cnt must start zeroed)
__global__ void k_unit_regions(const UnitDesc* __restrict__ units, int nunits, int lg_min,
                               int32_t* __restrict__ cnt) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < nunits; u += gridDim.x * blockDim.x) {
    const int lg = sell_lg(units[u].len, lg_min);
    if (u + 1 == nunits || sell_lg(units[u + 1].len, lg_min) != lg) cnt[lg] = u + 1;
    // cnt[4]: units longer than the grouping width (sorted descending)
    if (units[u].len > PG_SELL_GROUPW && (u + 1 == nunits || units[u + 1].len <= PG_SELL_GROUPW))
      cnt[4] = u + 1;
  }
}

struct SellRegions {
  int32_t ustart[5];  // first unit of region k (lg = 3 - k), + end
  int32_t sstart[5];  // first slice of region k, + total
};

// per slice: first unit, count, width, steps; elements for the scan
__global__ void k_slice_desc(const UnitDesc* __restrict__ units, const SellRegions R,
                             SliceDesc* __restrict__ slices, long long* __restrict__ elems) {
  const int nslices = R.sstart[4];
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s <= nslices; s += gridDim.x * blockDim.x) {
    if (s == nslices) {
      elems[s] = 0;
      continue;
    }
    int k = 0;
    while (k < 3 && s >= R.sstart[k + 1]) ++k;
    const int lg = 3 - k, H = 32 >> lg;
    const int first = R.ustart[k] + (s - R.sstart[k]) * H;
    const int count = min(H, R.ustart[k + 1] - first);
    const int width = units[first].len;  // sorted descending
    const int steps = (width + (1 << lg) - 1) >> lg;
    slices[s] = SliceDesc{0, first, width, steps, (int16_t)count, (int8_t)lg, 0};
    elems[s] = 32LL * steps;
  }
}

// the transposed copy (padding: value 0 in the padding column, bounds [0, 0])
__global__ void k_fill_sell(const UnitDesc* __restrict__ units, const int32_t* __restrict__ k0,
                            int nslices, const long long* __restrict__ off,
                            const double* __restrict__ vals, const int32_t* __restrict__ colx,
                            int32_t pad_col, SliceDesc* __restrict__ slices,
                            double* __restrict__ sv, int32_t* __restrict__ sc) {
  const int lane = threadIdx.x & 31;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nslices;
       s += (gridDim.x * blockDim.x) >> 5) {
    const long long o = off[s];
    SliceDesc d = slices[s];
    const int lg = d.lg, H = 32 >> lg;
    const int j = lane >> (5 - lg), u = lane & (H - 1);
    const int len = u < d.count ? units[d.first + u].len : 0;
    const int b = u < d.count ? k0[d.first + u] : 0;
    for (int t = 0; t < d.steps; ++t) {
      const int i = (t << lg) + j;
      sv[o + 32LL * t + lane] = i < len ? vals[b + i] : 0.0;
      sc[o + 32LL * t + lane] = i < len ? colx[b + i] : pad_col;
    }
    __syncwarp();
    if (lane == 0) {
      d.off = o;
      slices[s] = d;
    }
  }
}

// worklist maps: whole row -> unit, chunk (partial index) -> unit, unit -> slice
__global__ void k_unit_maps(const UnitDesc* __restrict__ units, int nunits,
                            const SegDesc* __restrict__ segs, int32_t* __restrict__ row_unit,
                            int32_t* __restrict__ part_unit) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < nunits; u += gridDim.x * blockDim.x) {
    const UnitDesc d = units[u];
    if (d.ref >= 0) row_unit[d.ref] = u;
    else part_unit[segs[-d.ref - 1].out] = u;
  }
}
// unit_slice < 0: a short one-lane unit, visited by a lane in worklist
// rounds; otherwise (longer units) by a warp
__global__ void k_slice_units(const SliceDesc* __restrict__ slices, int nslices,
                              const UnitDesc* __restrict__ units, int32_t* __restrict__ unit_slice,
                              const Dirty D, DevState* __restrict__ st) {
  long long w = 0;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nslices; s += gridDim.x * blockDim.x) {
    const SliceDesc d = slices[s];
    for (int i = 0; i < d.count; ++i) {
      const int len = units[d.first + i].len;
      const int k = (d.lg == 0 && len <= kSellLaneUnit) ? -1 : len <= kSellMidMax ? -2 : s;
      unit_slice[d.first + i] = k;
      w += k == -1 ? D.w_lane : k == -2 ? D.w_mid : D.w_wide;
    }
  }
  if (w) atomicAdd(reinterpret_cast<unsigned long long*>(&st->unit_wsum), (unsigned long long)w);
}

}  // namespace pgb
