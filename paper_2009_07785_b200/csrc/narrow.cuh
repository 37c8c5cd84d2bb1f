// narrow.cuh -- ScalarMode::Narrow32 rounds (model.hpp:129, the reference's
// run_parallel<float>, par_engine.cpp:317-319).
//
// The working copy is float (engine_common.hpp:24-38: values cast to float,
// sides and bounds normalised at infinity_threshold, then cast); activities,
// residuals and candidates are computed in float (propcore.hpp templates on
// T = float), acceptance and the EmptyDomain test in double
// (propcore.hpp:160-208).  On the device the float working values live in
// the f64 arrays (a float is exactly representable), bounds merge through
// the same ordered 64-bit keys (max over doubles of floats = max over the
// floats), and a round is one thread per row over the CSR copy, every entry
// through the float pipeline -- the f64 filters are not used in this mode.
#pragma once

#include "kernels.cuh"

namespace pgb {

struct ActF {
  float min_f, max_f;
  int32_t min_i, max_i;
};

__device__ __forceinline__ ActF actf_chain(const RoundArgs& A, int k0, int k1) {
  ActF a = {0.0f, 0.0f, 0, 0};
  for (int k = k0; k < k1; ++k) {
    const float v = (float)A.vals[k];
    const Snap& sn = A.snap[A.colx[k] & 0x7fffffff];
    const float lo = (float)sn.lo, up = (float)sn.up;
    const float bmin = v > 0 ? lo : up;
    const float bmax = v > 0 ? up : lo;
    if (isinf(bmin)) ++a.min_i; else a.min_f = __fadd_rn(a.min_f, __fmul_rn(v, bmin));
    if (isinf(bmax)) ++a.max_i; else a.max_f = __fadd_rn(a.max_f, __fmul_rn(v, bmax));
  }
  return a;
}

// cpu_par's summation order: one chain, or nnz_budget chunks combined
// pairwise in chunk order (par_engine.cpp:99-123); scratch: this thread's
// chunk partials
__device__ __forceinline__ ActF actf_row(const RoundArgs& A, int r, int chunk, ActF* part) {
  const int k0 = A.row_ptr[r], k1 = A.row_ptr[r + 1];
  if (k1 - k0 <= chunk) return actf_chain(A, k0, k1);
  int np = 0;
  for (int b = k0; b < k1; b += chunk) part[np++] = actf_chain(A, b, min(k1, b + chunk));
  while (np > 1) {
    int out = 0;
    for (int i = 0; i + 1 < np; i += 2) {
      ActF c;
      c.min_f = __fadd_rn(part[i].min_f, part[i + 1].min_f);
      c.max_f = __fadd_rn(part[i].max_f, part[i + 1].max_f);
      c.min_i = part[i].min_i + part[i + 1].min_i;
      c.max_i = part[i].max_i + part[i + 1].max_i;
      part[out++] = c;
    }
    if (np & 1) part[out++] = part[np - 1];
    np = out;
  }
  return part[0];
}

template <bool kRowCheck>
__global__ void __launch_bounds__(256) k_round_f32(const RoundArgs A, const DevCfg cfg, int m,
                                                   ActF* scratch, int maxc) {
  if (compute_off(A.st, cfg)) return;
  const float inf = CUDART_INF_F;
  const float eps = (float)cfg.int_eps;
  const float huge = (float)cfg.inf_thr;
  bool inf_flag = false;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  ActF* part = scratch + (size_t)gtid * maxc;
  for (int r = gtid; r < m; r += gstride) {
    const ActF act = actf_row(A, r, cfg.chunk, part);
    const float l = (float)A.lhs[r], h = (float)A.rhs[r];
    if (kRowCheck) {
      // classify_constraint<float> Step 2 (propcore.hpp:147-156), in double
      const Act ad = {(double)act.min_f, (double)act.max_f, act.min_i, act.max_i};
      if (row_infeasible(ad, (double)l, (double)h, cfg)) inf_flag = true;
    }
    for (int k = A.row_ptr[r]; k < A.row_ptr[r + 1]; ++k) {
      const float a = (float)A.vals[k];
      const int32_t cx = A.colx[k];
      const Snap& sn = A.snap[cx & 0x7fffffff];
      const float lo = (float)sn.lo, up = (float)sn.up;
      // residual_activities<float> (propcore.hpp:78-94)
      const float bmin = a > 0 ? lo : up;
      const float bmax = a > 0 ? up : lo;
      float min_res = -inf, max_res = inf;
      if (act.min_i == 0) min_res = __fsub_rn(act.min_f, __fmul_rn(a, bmin));
      else if (act.min_i == 1 && isinf(bmin)) min_res = act.min_f;
      if (act.max_i == 0) max_res = __fsub_rn(act.max_f, __fmul_rn(a, bmax));
      else if (act.max_i == 1 && isinf(bmax)) max_res = act.max_f;
      // compute_bound_candidates<float> (propcore.hpp:102-132)
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
      // tighten: acceptance in double (propcore.hpp:160-208)
      const int kind = tighten((double)lo, (double)up, (double)cl, (double)cu, cfg);
      if (kind == 4) inf_flag = true;
      else if (kind) commit_side(A.key_out, cx & 0x7fffffff, kind, (double)cl, (double)cu);
    }
  }
  if (__any_sync(__activemask(), inf_flag)) A.st->infeasible = 1;
}

// the float working copy (engine_common.hpp:24-38), in place: values cast,
// sides / bounds (already normalised) cast
__global__ void k_to_f32(double* __restrict__ v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = (double)(float)v[i];
}

}  // namespace pgb
