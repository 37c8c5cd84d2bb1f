/*
 * ORACLE (test infrastructure only) -- scalar-generic body of the CPU
 * restatement, included twice by propgate_oracle.c with
 *   T = double, SFX(x) = x##_f64   (ScalarMode::Wide64)
 *   T = float,  SFX(x) = x##_f32   (ScalarMode::Narrow32)
 * mirroring the reference's templates on T (core/include/propgate/propcore.hpp,
 * core/src/par_engine.cpp, core/src/seq_engine.cpp, core/src/engine_common.hpp).
 * Acceptance comparisons always run in double, as in propcore.hpp:160-179.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * call this code, and only as the checker.
 */

typedef struct {
  T min_finite;
  T max_finite;
  int32_t min_inf;
  int32_t max_inf;
} SFX(act);

/* propcore.hpp:45-65 compute_row_activities: b chosen by a > 0 (not >=),
 * infinite contributions counted, finite ones summed a*b in entry order. */
static SFX(act) SFX(row_act)(const int32_t* cols, const T* coefs, int64_t len,
                             const T* lower, const T* upper) {
  SFX(act) r = {0, 0, 0, 0};
  for (int64_t k = 0; k < len; ++k) {
    const int32_t j = cols[k];
    const T a = coefs[k];
    const T bmin = a > 0 ? lower[j] : upper[j];
    const T bmax = a > 0 ? upper[j] : lower[j];
    if (isinf(bmin))
      ++r.min_inf;
    else
      r.min_finite += a * bmin;
    if (isinf(bmax))
      ++r.max_inf;
    else
      r.max_finite += a * bmax;
  }
  return r;
}

/* par_engine.cpp:46-50 combine */
static SFX(act) SFX(combine)(SFX(act) a, SFX(act) b) {
  SFX(act) r;
  r.min_finite = a.min_finite + b.min_finite;
  r.max_finite = a.max_finite + b.max_finite;
  r.min_inf = a.min_inf + b.min_inf;
  r.max_inf = a.max_inf + b.max_inf;
  return r;
}

/* Activity of one row with cpu_par's summation order.  partition_row_blocks
 * (par_engine.cpp:14-41) leaves every row longer than nnz_budget alone in a
 * VectorWide block, whose activity is reduced over nnz_budget-sized chunks
 * combined pairwise in index order (wide_row_activities, par_engine.cpp:99-123).
 * Every other row (Stream, Narrow, or Wide with a single chunk) is summed in
 * entry order (propcore.hpp:50-63). */
static SFX(act) SFX(par_row_act)(const int32_t* row_ptr, const int32_t* col_idx,
                                 const T* vals, int32_t row, const T* lower,
                                 const T* upper, int32_t chunk,
                                 SFX(act) * scratch) {
  const int64_t b = row_ptr[row], e = row_ptr[row + 1];
  if (e - b <= chunk) return SFX(row_act)(col_idx + b, vals + b, e - b, lower, upper);
  int64_t np = 0;
  for (int64_t k = b; k < e; k += chunk) {
    const int64_t len = (e - k) < chunk ? (e - k) : chunk;
    scratch[np++] = SFX(row_act)(col_idx + k, vals + k, len, lower, upper);
  }
  while (np > 1) {
    int64_t out = 0;
    for (int64_t i = 0; i + 1 < np; i += 2) scratch[out++] = SFX(combine)(scratch[i], scratch[i + 1]);
    if (np % 2 == 1) scratch[out++] = scratch[np - 1];
    np = out;
  }
  return scratch[0];
}

/* propcore.hpp:78-94 residual_activities */
static void SFX(residual)(const SFX(act) * act, T a, T lo, T up, T* min_res, T* max_res) {
  const T bmin = a > 0 ? lo : up;
  const T bmax = a > 0 ? up : lo;
  *min_res = -(T)INFINITY;
  *max_res = (T)INFINITY;
  if (act->min_inf == 0)
    *min_res = act->min_finite - a * bmin;
  else if (act->min_inf == 1 && isinf(bmin))
    *min_res = act->min_finite;
  if (act->max_inf == 0)
    *max_res = act->max_finite - a * bmax;
  else if (act->max_inf == 1 && isinf(bmax))
    *max_res = act->max_finite;
}

/* propcore.hpp:102-132 compute_bound_candidates */
static void SFX(candidates)(T a, T lhs, T rhs, T min_res, T max_res, int integral,
                            const pg_config* cfg, T* new_lo, T* new_up) {
  const T inf = (T)INFINITY;
  const int rhs_side = !isinf(rhs) && !isinf(min_res);
  const int lhs_side = !isinf(lhs) && !isinf(max_res);
  T lo = -inf, up = inf;
  if (a > 0) {
    if (rhs_side) up = (rhs - min_res) / a;
    if (lhs_side) lo = (lhs - max_res) / a;
  } else {
    if (rhs_side) lo = (rhs - min_res) / a;
    if (lhs_side) up = (lhs - max_res) / a;
  }
  if (integral) {
    const T eps = (T)cfg->integrality_eps;
    if (isfinite(lo)) lo = SFX(ceil_)(lo - eps);
    if (isfinite(up)) up = SFX(floor_)(up + eps);
  }
  const T huge = (T)cfg->infinity_threshold;
  if (!(lo > -huge && lo < huge)) lo = -inf;
  if (!(up > -huge && up < huge)) up = inf;
  *new_lo = lo;
  *new_up = up;
}

/* propcore.hpp:138-158 classify_constraint: 0 Redundant, 1 Infeasible,
 * 2 Propagatable. */
static int SFX(classify)(const SFX(act) * act, T lhs, T rhs, const pg_config* cfg) {
  const double min_act = act->min_inf == 0 ? (double)act->min_finite : -INFINITY;
  const double max_act = act->max_inf == 0 ? (double)act->max_finite : INFINITY;
  const double l = (double)lhs, r = (double)rhs;
  if (l <= min_act && max_act <= r) return 0;
  if (isfinite(r)) {
    const double slack = cfg->improvement_abs + cfg->improvement_rel * fmax(1.0, fabs(r));
    if (min_act > r + slack) return 1;
  }
  if (isfinite(l)) {
    const double slack = cfg->improvement_abs + cfg->improvement_rel * fmax(1.0, fabs(l));
    if (l > max_act + slack) return 1;
  }
  return 2;
}

/* propcore.hpp:185-208 tighten (with improves_lower/upper, :165-179).
 * Returns 0 NoChange, 1 NewLower, 2 NewUpper, 3 Both, 4 EmptyDomain. */
static int SFX(tighten)(T old_lo, T old_up, T cand_lo, T cand_up, const pg_config* cfg,
                        T* out_lo, T* out_up) {
  const double ol = (double)old_lo, ou = (double)old_up;
  const double cl = (double)cand_lo, cu = (double)cand_up;
  int take_lo, take_up;
  if (isinf(cl))
    take_lo = 0;
  else if (isinf(ol))
    take_lo = 1;
  else
    take_lo = cl > ol + (cfg->improvement_abs + cfg->improvement_rel * fmax(1.0, fabs(ol)));
  if (isinf(cu))
    take_up = 0;
  else if (isinf(ou))
    take_up = 1;
  else
    take_up = cu < ou - (cfg->improvement_abs + cfg->improvement_rel * fmax(1.0, fabs(ou)));
  const double lower = take_lo ? cl : ol;
  const double upper = take_up ? cu : ou;
  if ((take_lo || take_up) && lower > upper + cfg->improvement_abs) return 4;
  *out_lo = cand_lo;
  *out_up = cand_up;
  return (take_lo ? 1 : 0) | (take_up ? 2 : 0);
}

/* Working copy, engine_common.hpp:24-38: lhs/rhs/bounds with |v| >= the
 * infinity threshold mapped to +-inf (model.hpp:147-151); values untouched
 * except for the scalar conversion. */
typedef struct {
  T* vals;
  T* lhs;
  T* rhs;
  T* lo;
  T* up;
} SFX(work);

static double SFX(norm)(double v, double thr) {
  if (v >= thr) return INFINITY;
  if (v <= -thr) return -INFINITY;
  return v;
}

static int SFX(work_make)(const pg_problem* p, const pg_config* cfg, const double* lo,
                          const double* up, SFX(work) * w) {
  const int64_t nnz = p->nnz, m = p->num_rows, n = p->num_cols;
  w->vals = (T*)malloc(sizeof(T) * (size_t)(nnz ? nnz : 1));
  w->lhs = (T*)malloc(sizeof(T) * (size_t)(m ? m : 1));
  w->rhs = (T*)malloc(sizeof(T) * (size_t)(m ? m : 1));
  w->lo = (T*)malloc(sizeof(T) * (size_t)(n ? n : 1));
  w->up = (T*)malloc(sizeof(T) * (size_t)(n ? n : 1));
  if (!w->vals || !w->lhs || !w->rhs || !w->lo || !w->up) return -1;
  const double thr = cfg->infinity_threshold;
  for (int64_t k = 0; k < nnz; ++k) w->vals[k] = (T)p->values[k];
  for (int64_t i = 0; i < m; ++i) {
    w->lhs[i] = (T)SFX(norm)(p->lhs[i], thr);
    w->rhs[i] = (T)SFX(norm)(p->rhs[i], thr);
  }
  for (int64_t j = 0; j < n; ++j) {
    w->lo[j] = (T)SFX(norm)(lo[j], thr);
    w->up[j] = (T)SFX(norm)(up[j], thr);
  }
  return 0;
}

static void SFX(work_free)(SFX(work) * w) {
  free(w->vals);
  free(w->lhs);
  free(w->rhs);
  free(w->lo);
  free(w->up);
}

/* engine_common.hpp:51-58 bounds_crossed */
static int SFX(crossed)(const T* lo, const T* up, int64_t n, double slack) {
  for (int64_t j = 0; j < n; ++j)
    if ((double)lo[j] > (double)up[j] + slack) return 1;
  return 0;
}

/* One cpu_par round over rows [r0, r1) without the commit: process_block
 * (par_engine.cpp:126-171).  Reads only the snapshot lo_in/up_in; accepted
 * sides merge into lo_out/up_out by exact max/min (merge_lower/upper,
 * par_engine.cpp:56-71: replace only on strict improvement).  EmptyDomain
 * raises *infeasible and skips that entry's merge (:163-166). */
static void SFX(round_rows)(const pg_problem* p, const SFX(work) * w, const pg_config* cfg,
                            int32_t r0, int32_t r1, const T* lo_in, const T* up_in,
                            T* lo_out, T* up_out, int* infeasible, SFX(act) * scratch) {
  for (int32_t i = r0; i < r1; ++i) {
    const SFX(act) act = SFX(par_row_act)(p->row_ptr, p->col_idx, w->vals, i, lo_in,
                                          up_in, cfg->nnz_budget, scratch);
    for (int64_t k = p->row_ptr[i]; k < p->row_ptr[i + 1]; ++k) {
      const int32_t j = p->col_idx[k];
      const T a = w->vals[k];
      T min_res, max_res, cl, cu, nl = 0, nu = 0;
      SFX(residual)(&act, a, lo_in[j], up_in[j], &min_res, &max_res);
      SFX(candidates)(a, w->lhs[i], w->rhs[i], min_res, max_res, p->integral[j] != 0,
                      cfg, &cl, &cu);
      const int kind = SFX(tighten)(lo_in[j], up_in[j], cl, cu, cfg, &nl, &nu);
      if (kind == 4) {
        *infeasible = 1;
        continue;
      }
      if ((kind & 1) && lo_out[j] < nl) lo_out[j] = nl;
      if ((kind & 2) && up_out[j] > nu) up_out[j] = nu;
    }
  }
}

/* run_round's serial post-pass (par_engine.cpp:191-197). */
static int64_t SFX(commit)(const T* lo_in, const T* up_in, const T* lo_out,
                           const T* up_out, int64_t n, double slack, int* infeasible) {
  int64_t changes = 0;
  for (int64_t j = 0; j < n; ++j) {
    if (lo_out[j] != lo_in[j]) ++changes;
    if (up_out[j] != up_in[j]) ++changes;
    if ((double)lo_out[j] > (double)up_out[j] + slack) *infeasible = 1;
  }
  return changes;
}

static int64_t SFX(max_chunks)(const pg_problem* p, int32_t chunk) {
  int64_t mx = 1;
  for (int32_t i = 0; i < p->num_rows; ++i) {
    const int64_t len = (int64_t)p->row_ptr[i + 1] - p->row_ptr[i];
    const int64_t c = (len + chunk - 1) / chunk;
    if (c > mx) mx = c;
  }
  return mx;
}

static void SFX(store_bounds)(const T* lo, const T* up, int64_t n, pg_result* res) {
  if (res->lower)
    for (int64_t j = 0; j < n; ++j) res->lower[j] = (double)lo[j];
  if (res->upper)
    for (int64_t j = 0; j < n; ++j) res->upper[j] = (double)up[j];
}

static void SFX(push_round)(pg_result* res, int32_t round, int64_t changes) {
  if (res->per_round_changes && round - 1 < res->per_round_capacity)
    res->per_round_changes[round - 1] = changes;
  res->total_bound_changes += changes;
  res->rounds_executed = round;
}

/* run_parallel (par_engine.cpp:203-273), single-threaded: the merge is
 * exact max/min, so worker scheduling cannot change the result
 * (test_par_engine.cpp:183-210).  Optional Step-2 row check (flag
 * PG_FLAG_ROWCHECK) mirrors the GPU engine's verdict mode. */
static int SFX(propagate_par)(const pg_problem* p, const pg_config* cfg, const double* lo0,
                              const double* up0, pg_result* res) {
  const int64_t n = p->num_cols;
  SFX(work) w;
  if (SFX(work_make)(p, cfg, lo0, up0, &w)) return PG_ENOMEM;
  res->status = PG_CONVERGED;
  res->rounds_executed = 0;
  res->total_bound_changes = 0;
  res->constraints_processed = 0;
  if (SFX(crossed)(w.lo, w.up, n, cfg->improvement_abs)) {
    res->status = PG_INFEASIBLE;
    SFX(store_bounds)(w.lo, w.up, n, res);
    SFX(work_free)(&w);
    return PG_OK;
  }
  T* const lo_b = (T*)malloc(sizeof(T) * (size_t)(n ? n : 1));
  T* const up_b = (T*)malloc(sizeof(T) * (size_t)(n ? n : 1));
  T* lo_out = lo_b;
  T* up_out = up_b;
  SFX(act)* scratch = (SFX(act)*)malloc(sizeof(SFX(act)) * (size_t)SFX(max_chunks)(p, cfg->nnz_budget));
  const int rowcheck = (cfg->flags & PG_FLAG_ROWCHECK) != 0;
  T* lo_in = w.lo;
  T* up_in = w.up;
  const double t0 = orc_now();
  for (int32_t round = 1; round <= cfg->round_limit; ++round) {
    memcpy(lo_out, lo_in, sizeof(T) * (size_t)n);
    memcpy(up_out, up_in, sizeof(T) * (size_t)n);
    int infeasible = 0;
    SFX(round_rows)(p, &w, cfg, 0, p->num_rows, lo_in, up_in, lo_out, up_out, &infeasible,
                    scratch);
    if (rowcheck) {
      for (int32_t i = 0; i < p->num_rows && !infeasible; ++i) {
        const SFX(act) act = SFX(par_row_act)(p->row_ptr, p->col_idx, w.vals, i, lo_in, up_in,
                                              cfg->nnz_budget, scratch);
        if (SFX(classify)(&act, w.lhs[i], w.rhs[i], cfg) == 1) infeasible = 1;
      }
    }
    const int64_t changes =
        SFX(commit)(lo_in, up_in, lo_out, up_out, n, cfg->improvement_abs, &infeasible);
    SFX(push_round)(res, round, changes);
    res->constraints_processed += p->num_rows;
    if (infeasible) {
      res->status = PG_INFEASIBLE;
      break;
    }
    if (changes == 0) {
      res->status = PG_CONVERGED;
      break;
    }
    if (round == cfg->round_limit) {
      res->status = PG_ROUNDLIMIT;
      break;
    }
    T* t = lo_in; lo_in = lo_out; lo_out = t;
    t = up_in; up_in = up_out; up_out = t;
  }
  res->elapsed_ns = (int64_t)((orc_now() - t0) * 1e9);
  /* returned bounds are the last round's output (par_engine.cpp:271) */
  SFX(store_bounds)(lo_out, up_out, n, res);
  free(lo_b);
  free(up_b);
  free(scratch);
  SFX(work_free)(&w);
  return PG_OK;
}

/* run_sequential (seq_engine.cpp:12-99): Alg. 1 with marking; all rows start
 * marked (:29), ascending scan with immediate updates (:36-79), Step-1/2
 * row classification (:47-53), re-marking through the CSC (:77). */
static int SFX(propagate_seq)(const pg_problem* p, const pg_config* cfg, const double* lo0,
                              const double* up0, pg_result* res) {
  const int32_t m = p->num_rows;
  const int64_t n = p->num_cols;
  SFX(work) w;
  if (SFX(work_make)(p, cfg, lo0, up0, &w)) return PG_ENOMEM;
  res->status = PG_CONVERGED;
  res->rounds_executed = 0;
  res->total_bound_changes = 0;
  res->constraints_processed = 0;
  if (SFX(crossed)(w.lo, w.up, n, cfg->improvement_abs)) {
    res->status = PG_INFEASIBLE;
    SFX(store_bounds)(w.lo, w.up, n, res);
    SFX(work_free)(&w);
    return PG_OK;
  }
  /* column view for marking (model.cpp:82-104) */
  int64_t* col_ptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t* col_rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(p->nnz ? p->nnz : 1));
  for (int64_t k = 0; k < p->nnz; ++k) ++col_ptr[p->col_idx[k] + 1];
  for (int64_t j = 0; j < n; ++j) col_ptr[j + 1] += col_ptr[j];
  int64_t* next = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  memcpy(next, col_ptr, sizeof(int64_t) * (size_t)n);
  for (int32_t i = 0; i < m; ++i)
    for (int64_t k = p->row_ptr[i]; k < p->row_ptr[i + 1]; ++k) col_rows[next[p->col_idx[k]]++] = i;
  free(next);
  char* marked = (char*)malloc((size_t)(m ? m : 1));
  memset(marked, 1, (size_t)m);

  const double t0 = orc_now();
  for (int32_t round = 1; round <= cfg->round_limit; ++round) {
    int64_t changes = 0;
    int infeasible = 0;
    for (int32_t c = 0; c < m && !infeasible; ++c) {
      if (!marked[c]) continue;
      marked[c] = 0;
      ++res->constraints_processed;
      const int64_t b = p->row_ptr[c], e = p->row_ptr[c + 1];
      const SFX(act) act = SFX(row_act)(p->col_idx + b, w.vals + b, e - b, w.lo, w.up);
      const int rs = SFX(classify)(&act, w.lhs[c], w.rhs[c], cfg);
      if (rs == 1) {
        infeasible = 1;
        break;
      }
      if (rs == 0) continue;
      for (int64_t k = b; k < e; ++k) {
        const int32_t j = p->col_idx[k];
        const T a = w.vals[k];
        T min_res, max_res, cl, cu, nl = 0, nu = 0;
        SFX(residual)(&act, a, w.lo[j], w.up[j], &min_res, &max_res);
        SFX(candidates)(a, w.lhs[c], w.rhs[c], min_res, max_res, p->integral[j] != 0, cfg,
                        &cl, &cu);
        const int kind = SFX(tighten)(w.lo[j], w.up[j], cl, cu, cfg, &nl, &nu);
        if (kind == 4) {
          infeasible = 1;
          break;
        }
        if (kind == 0) continue;
        if (kind & 1) {
          w.lo[j] = nl;
          ++changes;
        }
        if (kind & 2) {
          w.up[j] = nu;
          ++changes;
        }
        for (int64_t q = col_ptr[j]; q < col_ptr[j + 1]; ++q) marked[col_rows[q]] = 1;
      }
    }
    SFX(push_round)(res, round, changes);
    if (infeasible) {
      res->status = PG_INFEASIBLE;
      break;
    }
    if (changes == 0) {
      res->status = PG_CONVERGED;
      break;
    }
    if (round == cfg->round_limit) res->status = PG_ROUNDLIMIT;
  }
  res->elapsed_ns = (int64_t)((orc_now() - t0) * 1e9);
  SFX(store_bounds)(w.lo, w.up, n, res);
  free(marked);
  free(col_rows);
  free(col_ptr);
  SFX(work_free)(&w);
  return PG_OK;
}
