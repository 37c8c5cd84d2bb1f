// narrow_sell.cuh -- ScalarMode::Narrow32 rounds over the sliced-ELL copy.
//
// The reference's run_parallel<float> (par_engine.cpp:317-319,
// engine_common.hpp:24-38): activities, residuals and candidates in float
// (propcore.hpp templates on T = float), acceptance and EmptyDomain in
// double (propcore.hpp:160-208).  The float working values live in the f64
// arrays (a float is exact in a double).  Three launches per round:
//
//   k_sellf_act    phase 1: per slice (ticket), every lane runs its units'
//                  float chains in entry order over the sliced-ELL copy
//                  (coalesced values / columns, 16 B bound gathers); G > 1
//                  lanes per unit hand their products to the unit in entry
//                  order (shuffles), so each sum is the reference's chain.
//                  Whole rows -> ractf[row] (+ the Step-2 row check), chunks
//                  of split rows -> partf[chunk].
//   k_sellf_split  rows longer than nnz_budget: chunk partials combined
//                  pairwise in chunk order (wide_row_activities).
//   k_sellf_cand   phase 2: per slice again, every entry of a row that can
//                  yield a finite candidate (a finite side with at most one
//                  infinite contribution) through the float pipeline.
//
// There is no exactness-preserving filter in this mode: the f64 filter's
// margins do not cover float rounding, so every entry of a live row is
// examined (the set of examined entries is a superset of the reference's
// accepted ones, each decided by the same float/double arithmetic).
#pragma once

#include "narrow.cuh"
#include "sell.cuh"

namespace pgb {

// one step of a unit's float chain on this lane (propcore.hpp:50-62 on float)
template <int LG>
__device__ __forceinline__ void f32_step(float a, float lo, float up, int u, ActF& act) {
  constexpr int G = 1 << LG, H = 32 >> LG;
  const float bmin = a > 0 ? lo : up;
  const float bmax = a > 0 ? up : lo;
  const bool imin = isinf(bmin), imax = isinf(bmax);
  const float pmin = imin ? 0.0f : __fmul_rn(a, bmin);
  const float pmax = imax ? 0.0f : __fmul_rn(a, bmax);
  act.min_i += imin;
  act.max_i += imax;
  if (LG == 0) {
    act.min_f = __fadd_rn(act.min_f, pmin);
    act.max_f = __fadd_rn(act.max_f, pmax);
  } else {
#pragma unroll
    for (int jj = 0; jj < G; ++jj) {
      act.min_f = __fadd_rn(act.min_f, __shfl_sync(0xffffffffu, pmin, u + H * jj));
      act.max_f = __fadd_rn(act.max_f, __shfl_sync(0xffffffffu, pmax, u + H * jj));
    }
  }
}

// classify_constraint<float> Step 2 (propcore.hpp:147-156), in double
__device__ __forceinline__ bool f32_row_infeasible(const ActF& act, float l, float h,
                                                   const DevCfg& cfg) {
  const Act ad = {(double)act.min_f, (double)act.max_f, act.min_i, act.max_i};
  return row_infeasible(ad, (double)l, (double)h, cfg);
}

template <bool kRowCheck, int LG>
__device__ __forceinline__ void f32_slice_act(const RoundArgs& A, const SliceDesc& sd, int lane,
                                              ActF* ractf, ActF* partf, bool& inf_flag,
                                              const DevCfg& cfg) {
  constexpr int H = 32 >> LG;
  const int j = lane >> (5 - LG), u = lane & (H - 1);
  const bool active = u < sd.count;
  UnitDesc ud = {0, -1};
  if (active) ud = A.units[sd.first + u];
  const double* pa = A.sv + sd.off + lane;
  const int32_t* pc = A.sc + sd.off + lane;
  ActF act = {0.0f, 0.0f, 0, 0};
  constexpr int U = 4;
  int t = 0;
  for (; t + U <= sd.steps; t += U) {
    double a[U];
    int32_t c[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      a[k] = __ldg(pa + 32 * (t + k));
      c[k] = __ldg(pc + 32 * (t + k));
    }
    double2 b[U];
#pragma unroll
    for (int k = 0; k < U; ++k) b[k] = __ldg(A.bnd + (c[k] & 0x7fffffff));
#pragma unroll
    for (int k = 0; k < U; ++k) f32_step<LG>((float)a[k], (float)b[k].x, (float)b[k].y, u, act);
  }
  for (; t < sd.steps; ++t) {
    const double a = __ldg(pa + 32 * t);
    const double2 b = __ldg(A.bnd + (__ldg(pc + 32 * t) & 0x7fffffff));
    f32_step<LG>((float)a, (float)b.x, (float)b.y, u, act);
  }
#pragma unroll
  for (int o = H; o < 32; o <<= 1) {
    act.min_i += __shfl_xor_sync(0xffffffffu, act.min_i, o);
    act.max_i += __shfl_xor_sync(0xffffffffu, act.max_i, o);
  }
  if (j == 0 && active) {
    if (ud.ref >= 0) {
      ractf[ud.ref] = act;
      if (kRowCheck && f32_row_infeasible(act, (float)A.lhs[ud.ref], (float)A.rhs[ud.ref], cfg))
        inf_flag = true;
    } else {
      const SegDesc d = A.segs[-ud.ref - 1];
      partf[d.out] = act;
      atomicAdd(&A.row_done[d.rslot], 1);
    }
  }
}

template <bool kRowCheck>
__global__ void __launch_bounds__(kSellThreads) k_sellf_act(const RoundArgs A, const DevCfg cfg,
                                                            ActF* __restrict__ ractf,
                                                            ActF* __restrict__ partf) {
  if (compute_off(A.st, cfg)) return;
  const int lane = threadIdx.x & 31;
  bool inf_flag = false;
  int cur = 0;
  if (lane == 0) cur = ticket(&A.st->work);
  cur = __shfl_sync(0xffffffffu, cur, 0);
  while (cur < A.nslices) {
    int nxt = 0;
    if (lane == 0) nxt = ticket(&A.st->work);
    const SliceDesc sd = A.slices[cur];
    if (sd.lg == 3) f32_slice_act<kRowCheck, 3>(A, sd, lane, ractf, partf, inf_flag, cfg);
    else if (sd.lg == 2) f32_slice_act<kRowCheck, 2>(A, sd, lane, ractf, partf, inf_flag, cfg);
    else if (sd.lg == 1) f32_slice_act<kRowCheck, 1>(A, sd, lane, ractf, partf, inf_flag, cfg);
    else f32_slice_act<kRowCheck, 0>(A, sd, lane, ractf, partf, inf_flag, cfg);
    cur = __shfl_sync(0xffffffffu, nxt, 0);
  }
  if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
}

// split rows whose chunks all ran: the chunk records combined pairwise in
// chunk order, level by level (par_engine.cpp:117-121), in float; one
// thread per row (a few hundred rows, each tree ~log2(chunks) levels)
template <bool kRowCheck>
__global__ void k_sellf_split(const RoundArgs A, const int32_t* __restrict__ split, int nsplit,
                              ActF* __restrict__ ractf, ActF* __restrict__ partf, const DevCfg cfg) {
  if (compute_off(A.st, cfg)) return;
  bool inf_flag = false;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nsplit; w += gridDim.x * blockDim.x) {
    const int rs = split[w];
    const int first = A.sfirst[rs];
    int np = A.sfirst[rs + 1] - first;
    if (ld_gpu(&A.row_done[rs]) != np) continue;
    A.row_done[rs] = 0;
    ActF* P = partf + first;
    while (np > 1) {
      int out = 0;
      for (int i = 0; i + 1 < np; i += 2) {
        ActF c;
        c.min_f = __fadd_rn(P[i].min_f, P[i + 1].min_f);
        c.max_f = __fadd_rn(P[i].max_f, P[i + 1].max_f);
        c.min_i = P[i].min_i + P[i + 1].min_i;
        c.max_i = P[i].max_i + P[i + 1].max_i;
        P[out++] = c;
      }
      if (np & 1) P[out++] = P[np - 1];
      np = out;
    }
    const int r = A.srow[rs];
    ractf[r] = P[0];
    if (kRowCheck && f32_row_infeasible(P[0], (float)A.lhs[r], (float)A.rhs[r], cfg))
      inf_flag = true;
  }
  if (inf_flag) A.st->infeasible = 1;
}

// residual_activities<float> -> compute_bound_candidates<float> (float)
// -> tighten (double) -> merge, for one entry (k_round_f32's pipeline)
__device__ __forceinline__ bool f32_entry(const ActF& act, float a, float lo, float up, float l,
                                          float h, int32_t cx, long long* key_out,
                                          const DevCfg& cfg) {
  const float inf = CUDART_INF_F;
  const float eps = (float)cfg.int_eps;
  const float huge = (float)cfg.inf_thr;
  const float bmin = a > 0 ? lo : up;
  const float bmax = a > 0 ? up : lo;
  float min_res = -inf, max_res = inf;
  if (act.min_i == 0) min_res = __fsub_rn(act.min_f, __fmul_rn(a, bmin));
  else if (act.min_i == 1 && isinf(bmin)) min_res = act.min_f;
  if (act.max_i == 0) max_res = __fsub_rn(act.max_f, __fmul_rn(a, bmax));
  else if (act.max_i == 1 && isinf(bmax)) max_res = act.max_f;
  const bool rhs_side = !isinf(h) && !isinf(min_res);
  const bool lhs_side = !isinf(l) && !isinf(max_res);
  float cl = -inf, cu = inf;
  if (a > 0) {
    if (rhs_side) cu = __fdiv_rn(__fsub_rn(h, min_res), a);
    if (lhs_side) cl = __fdiv_rn(__fsub_rn(l, max_res), a);
  } else {
    if (rhs_side) cl = __fdiv_rn(__fsub_rn(h, min_res), a);
    if (lhs_side) cu = __fdiv_rn(__fsub_rn(l, max_res), a);
  }
  if (cx < 0) {
    if (isfinite(cl)) cl = ceilf(__fsub_rn(cl, eps));
    if (isfinite(cu)) cu = floorf(__fadd_rn(cu, eps));
  }
  if (!(cl > -huge && cl < huge)) cl = -inf;
  if (!(cu > -huge && cu < huge)) cu = inf;
  const int kind = tighten((double)lo, (double)up, (double)cl, (double)cu, cfg);
  if (kind == 4) return true;  // EmptyDomain: flag, no merge (par_engine.cpp:163-166)
  if (kind) commit_side(key_out, cx & 0x7fffffff, kind, (double)cl, (double)cu);
  return false;
}

template <int LG>
__device__ __forceinline__ void f32_slice_cand(const RoundArgs& A, const SliceDesc& sd, int lane,
                                               const ActF* ractf, bool& inf_flag,
                                               const DevCfg& cfg) {
  constexpr int H = 32 >> LG;
  const int j = lane >> (5 - LG), u = lane & (H - 1);
  int len = 0, r = -1;
  if (u < sd.count) {
    const UnitDesc ud = A.units[sd.first + u];
    len = ud.len;
    r = ud.ref >= 0 ? ud.ref : A.srow[A.segs[-ud.ref - 1].rslot];
  }
  ActF act = {0.0f, 0.0f, 2, 2};
  float l = -CUDART_INF_F, h = CUDART_INF_F;
  if (r >= 0) {
    act = ractf[r];
    l = (float)A.lhs[r];
    h = (float)A.rhs[r];
  }
  // a finite candidate needs a finite side whose residual can be finite
  const bool live = (!isinf(h) && act.min_i <= 1) || (!isinf(l) && act.max_i <= 1);
  if (!__any_sync(0xffffffffu, live)) return;
  const double* pa = A.sv + sd.off + lane;
  const int32_t* pc = A.sc + sd.off + lane;
  for (int t0 = 0; t0 < sd.steps; t0 += 4) {
    double a[4];
    int32_t c[4];
    bool in[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      in[k] = live && ((t0 + k) << LG) + j < len;
      a[k] = 0.0;
      c[k] = A.pad_col;
      if (in[k]) {
        a[k] = __ldg(pa + 32 * (t0 + k));
        c[k] = __ldg(pc + 32 * (t0 + k));
      }
    }
    double2 b[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) b[k] = in[k] ? __ldg(A.bnd + (c[k] & 0x7fffffff)) : make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (in[k] && f32_entry(act, (float)a[k], (float)b[k].x, (float)b[k].y, l, h, c[k], A.key_out, cfg))
        inf_flag = true;
  }
}

__global__ void __launch_bounds__(kSellThreads) k_sellf_cand(const RoundArgs A, const DevCfg cfg,
                                                             const ActF* __restrict__ ractf) {
  if (compute_off(A.st, cfg)) return;
  const int lane = threadIdx.x & 31;
  bool inf_flag = false;
  int cur = 0;
  if (lane == 0) cur = ticket(&A.st->cand_work);
  cur = __shfl_sync(0xffffffffu, cur, 0);
  while (cur < A.nslices) {
    int nxt = 0;
    if (lane == 0) nxt = ticket(&A.st->cand_work);
    const SliceDesc sd = A.slices[cur];
    if (sd.lg == 3) f32_slice_cand<3>(A, sd, lane, ractf, inf_flag, cfg);
    else if (sd.lg == 2) f32_slice_cand<2>(A, sd, lane, ractf, inf_flag, cfg);
    else if (sd.lg == 1) f32_slice_cand<1>(A, sd, lane, ractf, inf_flag, cfg);
    else f32_slice_cand<0>(A, sd, lane, ractf, inf_flag, cfg);
    cur = __shfl_sync(0xffffffffu, nxt, 0);
  }
  if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
}

}  // namespace pgb
