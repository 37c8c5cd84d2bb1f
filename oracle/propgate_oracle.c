/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY, NOT PART OF THE PRODUCT.
 *
 * Plain-C restatement of the reference's CPU propagation path (arXiv
 * 2009.07785 reference `propgate`, paths relative to /root/reference/proj):
 *   propcore        core/include/propgate/propcore.hpp:45-208
 *   cpu_par         core/src/par_engine.cpp:14-41, 46-71, 99-200, 203-273, 277-312
 *   cpu_seq         core/src/seq_engine.cpp:12-99
 *   init semantics  core/src/engine_common.hpp:24-58, model.hpp:147-151
 *   validate()      core/src/model.cpp:21-35
 *
 * Parity is pinned: tests/test_oracle.py checks this file bit-for-bit against
 * golden vectors produced by the reference itself (compiled from its own
 * sources into oracle/_ref/ by oracle/build_ref.sh; fixtures and generator
 * script under tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the CPU baseline.  The product path (paper_2009_07785_b200/) never does.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (see oracle/Makefile).
 * -ffp-contract=off keeps a*b + c as two roundings, like the reference
 * compiled for baseline x86-64 (no FMA).
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../include/propgate_b200.h"

static double orc_now(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static double ceil__f64(double x) { return ceil(x); }
static double floor__f64(double x) { return floor(x); }
static float ceil__f32(float x) { return ceilf(x); }
static float floor__f32(float x) { return floorf(x); }

#define T double
#define SFX(x) x##_f64
#include "oracle_body.h"
#undef T
#undef SFX

#define T float
#define SFX(x) x##_f32
#include "oracle_body.h"
#undef T
#undef SFX

/* ---- exported entry points -------------------------------------------- */

/* EngineConfig::validate, model.cpp:21-35 (0 ok, PG_EINVAL otherwise) */
int orc_validate(const pg_config* c) {
  if (c->round_limit < 1) return PG_EINVAL;
  if (!(c->infinity_threshold > 0)) return PG_EINVAL;
  if (!(c->improvement_abs > 0) || !(c->improvement_rel > 0)) return PG_EINVAL;
  if (!(c->integrality_eps > 0)) return PG_EINVAL;
  if (c->vector_threshold < 1) return PG_EINVAL;
  if (c->nnz_budget < c->vector_threshold) return PG_EINVAL;
  if (c->worker_count < 0) return PG_EINVAL;
  return PG_OK;
}

/* engine: 0 = cpu_seq (propagate_sequential), 1 = cpu_par (propagate_parallel).
 * lo0/up0 NULL = the problem's own bounds. */
int orc_propagate(int engine, const pg_problem* p, const pg_config* cfg, const double* lo0,
                  const double* up0, pg_result* res) {
  int rc = orc_validate(cfg);
  if (rc) return rc;
  if (!lo0) lo0 = p->lower;
  if (!up0) up0 = p->upper;
  if (cfg->scalar_mode == PG_NARROW32)
    return engine == 0 ? propagate_seq_f32(p, cfg, lo0, up0, res)
                       : propagate_par_f32(p, cfg, lo0, up0, res);
  return engine == 0 ? propagate_seq_f64(p, cfg, lo0, up0, res)
                     : propagate_par_f64(p, cfg, lo0, up0, res);
}

/* propagate_round_parallel, par_engine.cpp:277-312: one round on a caller
 * snapshot (normalised at entry), double precision. */
int orc_round(const pg_problem* p, const pg_config* cfg, const double* lb_in,
              const double* ub_in, double* lb_out, double* ub_out, int32_t* changed,
              int32_t* infeasible, int64_t* changes) {
  int rc = orc_validate(cfg);
  if (rc) return rc;
  work_f64 w;
  if (work_make_f64(p, cfg, lb_in, ub_in, &w)) return PG_ENOMEM;
  const int64_t n = p->num_cols;
  memcpy(lb_out, w.lo, sizeof(double) * (size_t)n);
  memcpy(ub_out, w.up, sizeof(double) * (size_t)n);
  act_f64* scratch = (act_f64*)malloc(sizeof(act_f64) * (size_t)max_chunks_f64(p, cfg->nnz_budget));
  int inf = 0;
  round_rows_f64(p, &w, cfg, 0, p->num_rows, w.lo, w.up, lb_out, ub_out, &inf, scratch);
  const int64_t ch = commit_f64(w.lo, w.up, lb_out, ub_out, n, cfg->improvement_abs, &inf);
  *changes = ch;
  *changed = ch > 0;
  *infeasible = inf;
  free(scratch);
  work_free_f64(&w);
  return PG_OK;
}

/* process_block over the row range [r0, r1) of an already-normalised
 * snapshot, merging into lb_out/ub_out (no commit).  Used by the row-shard
 * tests: shards merged by max/min must equal the unsharded round. */
int orc_round_rows(const pg_problem* p, const pg_config* cfg, int32_t r0, int32_t r1,
                   const double* lb_in, const double* ub_in, double* lb_out, double* ub_out,
                   int32_t* infeasible) {
  work_f64 w;
  if (work_make_f64(p, cfg, lb_in, ub_in, &w)) return PG_ENOMEM;
  act_f64* scratch = (act_f64*)malloc(sizeof(act_f64) * (size_t)max_chunks_f64(p, cfg->nnz_budget));
  int inf = 0;
  round_rows_f64(p, &w, cfg, r0, r1, w.lo, w.up, lb_out, ub_out, &inf, scratch);
  *infeasible = inf;
  free(scratch);
  work_free_f64(&w);
  return PG_OK;
}

/* run_round's post-pass, par_engine.cpp:191-197 */
int64_t orc_commit(int64_t n, const double* lb_in, const double* ub_in, const double* lb_out,
                   const double* ub_out, double slack, int32_t* infeasible) {
  int inf = 0;
  const int64_t ch = commit_f64(lb_in, ub_in, lb_out, ub_out, n, slack, &inf);
  if (inf) *infeasible = 1;
  return ch;
}

/* partition_row_blocks, par_engine.cpp:14-41 (0 Stream, 1 Narrow, 2 Wide) */
int orc_partition_row_blocks(const pg_problem* p, const pg_config* cfg, int32_t* starts,
                             int32_t* kinds, int32_t* num_blocks) {
  int32_t nb = 0, row = 0;
  starts[0] = 0;
  while (row < p->num_rows) {
    int32_t end = row;
    int64_t acc = 0;
    while (end < p->num_rows && acc + (p->row_ptr[end + 1] - p->row_ptr[end]) <= cfg->nnz_budget) {
      acc += p->row_ptr[end + 1] - p->row_ptr[end];
      ++end;
    }
    if (end - row >= 2) {
      kinds[nb] = 0;
      starts[++nb] = end;
      row = end;
    } else {
      kinds[nb] = (p->row_ptr[row + 1] - p->row_ptr[row]) < cfg->vector_threshold ? 1 : 2;
      starts[++nb] = row + 1;
      row = row + 1;
    }
  }
  *num_blocks = nb;
  return PG_OK;
}

/* ---- propcore entry points for the unit KATs (test_propcore.cpp) ------ */

/* out[4] = {min_finite, max_finite, min_inf_count, max_inf_count} */
void orc_row_activities(const int32_t* cols, const double* coefs, int64_t len,
                        const double* lower, const double* upper, double* out) {
  const act_f64 a = row_act_f64(cols, coefs, len, lower, upper);
  out[0] = a.min_finite;
  out[1] = a.max_finite;
  out[2] = a.min_inf;
  out[3] = a.max_inf;
}

void orc_residual(const double* act4, double a, double lo, double up, double* out2) {
  act_f64 act = {act4[0], act4[1], (int32_t)act4[2], (int32_t)act4[3]};
  residual_f64(&act, a, lo, up, &out2[0], &out2[1]);
}

void orc_candidates(double a, double lhs, double rhs, double min_res, double max_res,
                    int32_t integral, const pg_config* cfg, double* out2) {
  candidates_f64(a, lhs, rhs, min_res, max_res, integral, cfg, &out2[0], &out2[1]);
}

int32_t orc_classify(const double* act4, double lhs, double rhs, const pg_config* cfg) {
  act_f64 act = {act4[0], act4[1], (int32_t)act4[2], (int32_t)act4[3]};
  return classify_f64(&act, lhs, rhs, cfg);
}

int32_t orc_tighten(double old_lo, double old_up, double cand_lo, double cand_up,
                    const pg_config* cfg, double* out2) {
  out2[0] = 0;
  out2[1] = 0;
  const int32_t kind = tighten_f64(old_lo, old_up, cand_lo, cand_up, cfg, &out2[0], &out2[1]);
  /* like TightenOutcome: values meaningful only for the accepted sides */
  if (kind == 4 || !(kind & 1)) out2[0] = 0;
  if (kind == 4 || !(kind & 2)) out2[1] = 0;
  return kind;
}

/* Batch form of the propcore entry points over many independent rows (row t
 * uses columns 0..len-1 of its own slice), for the golden-vector tests:
 * act[4t..], klass[t]; per entry k: res[2k..], cand[4k..] (integral 0 then
 * 1, {lo, up}), tight[2k..] and tkind[k] of tighten(lo, up, cand(integral 0)). */
void orc_propcore_rows(int32_t nrows, const int32_t* row_len, const double* coefs,
                       const double* lower, const double* upper, const double* sides,
                       const pg_config* cfg, double* act, int32_t* klass, double* res,
                       double* cand, double* tight, int32_t* tkind) {
  int64_t off = 0;
  int32_t cols[64];
  for (int i = 0; i < 64; ++i) cols[i] = i;
  for (int32_t t = 0; t < nrows; ++t) {
    const int32_t L = row_len[t];
    const act_f64 a = row_act_f64(cols, coefs + off, L, lower + off, upper + off);
    act[4 * t + 0] = a.min_finite;
    act[4 * t + 1] = a.max_finite;
    act[4 * t + 2] = a.min_inf;
    act[4 * t + 3] = a.max_inf;
    const double lhs = sides[2 * t], rhs = sides[2 * t + 1];
    klass[t] = classify_f64(&a, lhs, rhs, cfg);
    for (int32_t k = 0; k < L; ++k) {
      const int64_t e = off + k;
      double mn, mx;
      residual_f64(&a, coefs[e], lower[e], upper[e], &mn, &mx);
      res[2 * e] = mn;
      res[2 * e + 1] = mx;
      for (int integ = 0; integ < 2; ++integ)
        candidates_f64(coefs[e], lhs, rhs, mn, mx, integ, cfg, &cand[4 * e + 2 * integ],
                       &cand[4 * e + 2 * integ + 1]);
      double o2[2];
      tkind[e] = orc_tighten(lower[e], upper[e], cand[4 * e], cand[4 * e + 1], cfg, o2);
      tight[2 * e] = o2[0];
      tight[2 * e + 1] = o2[1];
    }
    off += L;
  }
}

/* ---- csr_from_triplets (core/src/model.cpp:37-80) -------------------------
 * Range check over the triplets in input order (row before column, the first
 * bad triplet decides: returns 1 for a bad row, 2 for a bad column), then a
 * stable order by (row, col) -- here an LSD counting sort, columns first,
 * then rows -- and a sequential `sum += value` from 0.0 over each run of equal
 * (row, col); runs summing to 0.0 are dropped.  row_ptr [m + 1], col_idx /
 * values_out [count]; *nnz receives the entries kept.  -1 on allocation
 * failure. */
int orc_csr_from_triplets(int32_t m, int32_t n, int64_t count, const int32_t* rows,
                          const int32_t* cols, const double* vals, int32_t* row_ptr,
                          int32_t* col_idx, double* values_out, int64_t* nnz) {
  for (int64_t i = 0; i < count; ++i) {
    if (rows[i] < 0 || rows[i] >= m) return 1;
    if (cols[i] < 0 || cols[i] >= n) return 2;
  }
  int64_t* a = malloc(sizeof(int64_t) * (size_t)(count ? count : 1));
  int64_t* b = malloc(sizeof(int64_t) * (size_t)(count ? count : 1));
  int64_t* cnt = malloc(sizeof(int64_t) * ((size_t)(m > n ? m : n) + 1));
  if (!a || !b || !cnt) {
    free(a);
    free(b);
    free(cnt);
    return -1;
  }
  /* pass 1: stable by column */
  memset(cnt, 0, sizeof(int64_t) * ((size_t)n + 1));
  for (int64_t i = 0; i < count; ++i) ++cnt[cols[i] + 1];
  for (int32_t j = 0; j < n; ++j) cnt[j + 1] += cnt[j];
  for (int64_t i = 0; i < count; ++i) a[cnt[cols[i]]++] = i;
  /* pass 2: stable by row */
  memset(cnt, 0, sizeof(int64_t) * ((size_t)m + 1));
  for (int64_t i = 0; i < count; ++i) ++cnt[rows[i] + 1];
  for (int32_t r = 0; r < m; ++r) cnt[r + 1] += cnt[r];
  for (int64_t t = 0; t < count; ++t) b[cnt[rows[a[t]]]++] = a[t];
  int64_t out = 0, t = 0;
  row_ptr[0] = 0;
  for (int32_t r = 0; r < m; ++r) {
    while (t < count && rows[b[t]] == r) {
      const int32_t c = cols[b[t]];
      double sum = 0.0;
      while (t < count && rows[b[t]] == r && cols[b[t]] == c) sum += vals[b[t++]];
      if (sum != 0.0) {
        col_idx[out] = c;
        values_out[out++] = sum;
      }
    }
    row_ptr[r + 1] = (int32_t)out;
  }
  *nnz = out;
  free(a);
  free(b);
  free(cnt);
  return 0;
}
