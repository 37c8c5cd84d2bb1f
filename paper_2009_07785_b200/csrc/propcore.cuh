// propcore.cuh -- device-side constraint math of the GPU-atomic round.
//
// Mirrors the reference's propcore (/root/reference/proj/core/include/
// propgate/propcore.hpp) operation for operation, with every rounding made
// explicit (__dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn) so nvcc can never
// contract a*b+c into an FMA: the reference is compiled for x86-64 without
// FMA, and these functions are bit-exact with it.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pgb {

// Run-time constants of one engine instance (EngineConfig, model.hpp:131-144).
struct DevCfg {
  double inf_thr;   // infinity_threshold
  double imp_abs;   // improvement_abs
  double imp_rel;   // improvement_rel
  double int_eps;   // integrality_eps
  int32_t chunk;    // nnz_budget: chunk length of long-row sums
  int32_t round_limit;
  uint32_t flags;
  int32_t pad;
  // compact {lb, ub} records of the round's input bounds as floats, {NaN,
  // NaN} where a bound is not a float (sell.cuh ld_col then reads the exact
  // 16 B record); null when the session does not keep them
  float2* bf;
};

// the compact record of [lo, up] (exact or the NaN marker)
__device__ __forceinline__ float2 fpair(double lo, double up) {
  const float fl = __double2float_rn(lo), fu = __double2float_rn(up);
  if ((double)fl == lo && (double)fu == up) return make_float2(fl, fu);
  return make_float2(__int_as_float(0x7fffffff), __int_as_float(0x7fffffff));
}

// ---- GPU-scope relaxed loads -------------------------------------------------
// Device state written by other CTAs (earlier kernels, or before a grid
// barrier) is read with ld.relaxed.gpu: coherent at L2, without the
// system-scope (STRONG.SYS) cost of a volatile access.
__device__ __forceinline__ int32_t ld_gpu(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_gpu(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_gpu(long long* p, long long v) {
  asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- ordered-bits keys ------------------------------------------------------
// A monotone map double -> int64 so that exact bound merges (merge_lower /
// merge_upper, par_engine.cpp:56-71) become single 64-bit atomicMax/atomicMin.
// -0.0 maps below +0.0, so candidates are canonicalised first.
__device__ __forceinline__ long long key_enc(double x) {
  const long long b = __double_as_longlong(x);
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double key_dec(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7fffffffffffffffLL));
}
__device__ __forceinline__ double canon0(double x) { return x == 0.0 ? 0.0 : x; }

// ActivityRecordT<double> (model.hpp:84-96)
struct Act {
  double min_f;
  double max_f;
  int32_t min_i;
  int32_t max_i;
};

__device__ __forceinline__ Act act_combine(const Act& a, const Act& b) {  // par_engine.cpp:46-50
  Act r;
  r.min_f = __dadd_rn(a.min_f, b.min_f);
  r.max_f = __dadd_rn(a.max_f, b.max_f);
  r.min_i = a.min_i + b.min_i;
  r.max_i = a.max_i + b.max_i;
  return r;
}

// One entry's contribution to compute_row_activities (propcore.hpp:50-62):
// b chosen by a > 0; an infinite b is counted, not summed.  Encoded as the
// product, or NaN for "infinite contribution" (a finite a*b is never NaN).
__device__ __forceinline__ void contrib(double a, double lo, double up, double& pmin,
                                        double& pmax) {
  const double bmin = a > 0 ? lo : up;
  const double bmax = a > 0 ? up : lo;
  pmin = isinf(bmin) ? __longlong_as_double(0x7ff8000000000000LL) : __dmul_rn(a, bmin);
  pmax = isinf(bmax) ? __longlong_as_double(0x7ff8000000000000LL) : __dmul_rn(a, bmax);
}
__device__ __forceinline__ void act_add(Act& act, double pmin, double pmax) {
  if (isnan(pmin)) ++act.min_i; else act.min_f = __dadd_rn(act.min_f, pmin);
  if (isnan(pmax)) ++act.max_i; else act.max_f = __dadd_rn(act.max_f, pmax);
}

// residual_activities (propcore.hpp:78-94)
__device__ __forceinline__ void residual(const Act& act, double a, double lo, double up,
                                         double& min_res, double& max_res) {
  const double bmin = a > 0 ? lo : up;
  const double bmax = a > 0 ? up : lo;
  min_res = -CUDART_INF;
  max_res = CUDART_INF;
  if (act.min_i == 0)
    min_res = __dsub_rn(act.min_f, __dmul_rn(a, bmin));
  else if (act.min_i == 1 && isinf(bmin))
    min_res = act.min_f;
  if (act.max_i == 0)
    max_res = __dsub_rn(act.max_f, __dmul_rn(a, bmax));
  else if (act.max_i == 1 && isinf(bmax))
    max_res = act.max_f;
}

// compute_bound_candidates (propcore.hpp:102-132)
__device__ __forceinline__ void candidates(double a, double lhs, double rhs, double min_res,
                                           double max_res, bool integral, const DevCfg& c,
                                           double& lo, double& up) {
  const bool rhs_side = !isinf(rhs) && !isinf(min_res);
  const bool lhs_side = !isinf(lhs) && !isinf(max_res);
  lo = -CUDART_INF;
  up = CUDART_INF;
  if (a > 0) {
    if (rhs_side) up = __ddiv_rn(__dsub_rn(rhs, min_res), a);
    if (lhs_side) lo = __ddiv_rn(__dsub_rn(lhs, max_res), a);
  } else {
    if (rhs_side) lo = __ddiv_rn(__dsub_rn(rhs, min_res), a);
    if (lhs_side) up = __ddiv_rn(__dsub_rn(lhs, max_res), a);
  }
  if (integral) {
    if (isfinite(lo)) lo = ceil(__dsub_rn(lo, c.int_eps));
    if (isfinite(up)) up = floor(__dadd_rn(up, c.int_eps));
  }
  if (!(lo > -c.inf_thr && lo < c.inf_thr)) lo = -CUDART_INF;
  if (!(up > -c.inf_thr && up < c.inf_thr)) up = CUDART_INF;
}

// improvement step abs + rel * max(1, |old|) (propcore.hpp:168-169, 176-177)
__device__ __forceinline__ double step_of(double old, const DevCfg& c) {
  return __dadd_rn(c.imp_abs, __dmul_rn(c.imp_rel, fmax(1.0, fabs(old))));
}

// tighten (propcore.hpp:185-208) with improves_lower/upper (:165-179).
// Returns bit0 = take lower, bit1 = take upper, or 4 = EmptyDomain.
__device__ __forceinline__ int tighten(double old_lo, double old_up, double cl, double cu,
                                       const DevCfg& c) {
  bool take_lo, take_up;
  if (isinf(cl)) take_lo = false;
  else if (isinf(old_lo)) take_lo = true;
  else take_lo = cl > __dadd_rn(old_lo, step_of(old_lo, c));
  if (isinf(cu)) take_up = false;
  else if (isinf(old_up)) take_up = true;
  else take_up = cu < __dsub_rn(old_up, step_of(old_up, c));
  const double lower = take_lo ? cl : old_lo;
  const double upper = take_up ? cu : old_up;
  if ((take_lo || take_up) && lower > __dadd_rn(upper, c.imp_abs)) return 4;
  return (take_lo ? 1 : 0) | (take_up ? 2 : 0);
}

// Step 2 of classify_constraint (propcore.hpp:147-156): the row cannot be
// satisfied under the current bounds.  (Step 1, Redundant, cannot coexist
// with Step 2 and never matters for the verdict.)
__device__ __forceinline__ bool row_infeasible(const Act& act, double lhs, double rhs,
                                               const DevCfg& c) {
  const double min_act = act.min_i == 0 ? act.min_f : -CUDART_INF;
  const double max_act = act.max_i == 0 ? act.max_f : CUDART_INF;
  if (lhs <= min_act && max_act <= rhs) return false;
  if (isfinite(rhs)) {
    const double slack = __dadd_rn(c.imp_abs, __dmul_rn(c.imp_rel, fmax(1.0, fabs(rhs))));
    if (min_act > __dadd_rn(rhs, slack)) return true;
  }
  if (isfinite(lhs)) {
    const double slack = __dadd_rn(c.imp_abs, __dmul_rn(c.imp_rel, fmax(1.0, fabs(lhs))));
    if (lhs > __dadd_rn(max_act, slack)) return true;
  }
  return false;
}

}  // namespace pgb
