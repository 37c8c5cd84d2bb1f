// ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// C-ABI shim over the UNMODIFIED reference library, compiled together with
// the reference's own sources (/root/reference/proj/core/src/*.cpp) into
// oracle/_ref/libpropgate_ref.so by oracle/build_ref.sh.  It only converts
// between the flat pg_* structs (include/propgate_b200.h) and the
// reference's types, then calls the reference entry points:
//   propagate_sequential  core/include/propgate/seq_engine.hpp:15
//   propagate_parallel    core/include/propgate/par_engine.hpp:41
//   propagate_round_parallel / partition_row_blocks  par_engine.hpp:12-36
//   gen_random / gen_cascade / permute_instance       generators.hpp:17-50
//   parse_mps_file                                    mps.hpp:28-39
//   propcore functions                                propcore.hpp:45-208
// Used to generate golden vectors (tests/golden/make_golden.py), to pin the
// C restatement (oracle/propgate_oracle.c), and as the CPU baseline
// ("kind": "reference") in bench.py.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../include/propgate_b200.h"
#include "propgate/generators.hpp"
#include "propgate/model.hpp"
#include "propgate/mps.hpp"
#include "propgate/par_engine.hpp"
#include "propgate/propcore.hpp"
#include "propgate/seq_engine.hpp"

using namespace propgate;

namespace {

thread_local std::string g_err;

EngineConfig to_cfg(const pg_config* c) {
  EngineConfig cfg;
  cfg.round_limit = c->round_limit;
  cfg.infinity_threshold = c->infinity_threshold;
  cfg.improvement_abs = c->improvement_abs;
  cfg.improvement_rel = c->improvement_rel;
  cfg.integrality_eps = c->integrality_eps;
  cfg.nnz_budget = c->nnz_budget;
  cfg.vector_threshold = c->vector_threshold;
  cfg.worker_count = c->worker_count;
  cfg.scalar_mode = c->scalar_mode == PG_NARROW32 ? ScalarMode::Narrow32 : ScalarMode::Wide64;
  return cfg;
}

ProblemInstance to_inst(const pg_problem* p, const double* lo, const double* up) {
  ProblemInstance inst;
  inst.matrix.num_rows = p->num_rows;
  inst.matrix.num_cols = p->num_cols;
  inst.matrix.row_ptr.assign(p->row_ptr, p->row_ptr + p->num_rows + 1);
  inst.matrix.col_idx.assign(p->col_idx, p->col_idx + p->nnz);
  inst.matrix.values.assign(p->values, p->values + p->nnz);
  inst.lhs.assign(p->lhs, p->lhs + p->num_rows);
  inst.rhs.assign(p->rhs, p->rhs + p->num_rows);
  inst.bounds.lower.assign(lo ? lo : p->lower, (lo ? lo : p->lower) + p->num_cols);
  inst.bounds.upper.assign(up ? up : p->upper, (up ? up : p->upper) + p->num_cols);
  inst.integral.assign(p->integral, p->integral + p->num_cols);
  return inst;
}

int status_code(PropagationStatus s) {
  switch (s) {
    case PropagationStatus::Converged: return PG_CONVERGED;
    case PropagationStatus::RoundLimit: return PG_ROUNDLIMIT;
    case PropagationStatus::Infeasible: return PG_INFEASIBLE;
  }
  return -1;
}

void fill(const PropagationResult& r, pg_result* out) {
  const size_t n = r.bounds.lower.size();
  if (out->lower) std::memcpy(out->lower, r.bounds.lower.data(), n * sizeof(double));
  if (out->upper) std::memcpy(out->upper, r.bounds.upper.data(), n * sizeof(double));
  if (out->per_round_changes)
    for (size_t i = 0; i < r.per_round_changes.size() && i < (size_t)out->per_round_capacity; ++i)
      out->per_round_changes[i] = r.per_round_changes[i];
  out->status = status_code(r.status);
  out->rounds_executed = r.rounds_executed;
  out->total_bound_changes = r.total_bound_changes;
  out->constraints_processed = r.constraints_processed;
  out->elapsed_ns = r.elapsed.count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_hardware_concurrency(void) { return (int)std::thread::hardware_concurrency(); }

// engine 0 = propagate_sequential, 1 = propagate_parallel
int ref_propagate(int engine, const pg_problem* p, const pg_config* c, const double* lo,
                  const double* up, pg_result* out) {
  try {
    const ProblemInstance inst = to_inst(p, lo, up);
    const EngineConfig cfg = to_cfg(c);
    const PropagationResult r =
        engine == 0 ? propagate_sequential(inst, cfg) : propagate_parallel(inst, cfg);
    fill(r, out);
    return PG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PG_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PG_ECUDA;
  }
}

int ref_round(const pg_problem* p, const pg_config* c, const double* lb_in, const double* ub_in,
              double* lb_out, double* ub_out, int32_t* changed, int32_t* infeasible,
              int64_t* changes) {
  try {
    const ProblemInstance inst = to_inst(p, nullptr, nullptr);
    const EngineConfig cfg = to_cfg(c);
    RoundSnapshot snap;
    snap.bounds_in.lower.assign(lb_in, lb_in + p->num_cols);
    snap.bounds_in.upper.assign(ub_in, ub_in + p->num_cols);
    const RowBlockPartition part = partition_row_blocks(inst.matrix, cfg);
    const RoundOutcome o = propagate_round_parallel(inst, snap, part, cfg);
    std::memcpy(lb_out, snap.bounds_out.lower.data(), sizeof(double) * p->num_cols);
    std::memcpy(ub_out, snap.bounds_out.upper.data(), sizeof(double) * p->num_cols);
    *changed = o.changed;
    *infeasible = o.infeasible;
    *changes = o.changes;
    return PG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PG_EINVAL;
  }
}

int ref_partition(const pg_problem* p, const pg_config* c, int32_t* starts, int32_t* kinds,
                  int32_t* num_blocks) {
  const ProblemInstance inst = to_inst(p, nullptr, nullptr);
  const RowBlockPartition part = partition_row_blocks(inst.matrix, to_cfg(c));
  for (size_t i = 0; i < part.block_starts.size(); ++i) starts[i] = part.block_starts[i];
  for (size_t i = 0; i < part.kinds.size(); ++i) kinds[i] = (int32_t)part.kinds[i];
  *num_blocks = part.num_blocks();
  return PG_OK;
}

// ---- instance handles (generators, MPS fixtures) -------------------------

void* ref_gen_random(int32_t rows, int32_t cols, uint64_t seed, double mean_row_nnz,
                     double integral_fraction, double inf_bound_frac, double inf_side_frac,
                     int64_t max_nnz) {
  RandomInstanceOptions o;
  o.num_rows = rows;
  o.num_cols = cols;
  o.seed = seed;
  o.mean_row_nnz = mean_row_nnz;
  o.integral_fraction = integral_fraction;
  o.infinite_bound_fraction = inf_bound_frac;
  o.infinite_side_fraction = inf_side_frac;
  o.max_nnz = max_nnz;
  return new ProblemInstance(gen_random(o));
}

void* ref_gen_cascade(int32_t m) { return new ProblemInstance(gen_cascade(m)); }

void* ref_parse_mps(const char* path) {
  try {
    return new ProblemInstance(parse_mps_file(path));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// permute_instance; col_perm_out [num_cols] receives perm.col_perm
void* ref_permute(void* h, uint64_t seed, int32_t* col_perm_out) {
  auto pr = permute_instance(*static_cast<ProblemInstance*>(h), seed);
  for (size_t j = 0; j < pr.second.col_perm.size(); ++j) col_perm_out[j] = pr.second.col_perm[j];
  return new ProblemInstance(std::move(pr.first));
}

void ref_inst_view(void* h, pg_problem* out) {
  auto* inst = static_cast<ProblemInstance*>(h);
  out->num_rows = inst->matrix.num_rows;
  out->num_cols = inst->matrix.num_cols;
  out->nnz = inst->matrix.nnz();
  out->row_ptr = inst->matrix.row_ptr.data();
  out->col_idx = inst->matrix.col_idx.data();
  out->values = inst->matrix.values.data();
  out->lhs = inst->lhs.data();
  out->rhs = inst->rhs.data();
  out->lower = inst->bounds.lower.data();
  out->upper = inst->bounds.upper.data();
  out->integral = inst->integral.data();
}

void ref_inst_free(void* h) { delete static_cast<ProblemInstance*>(h); }

// ---- csr_from_triplets (model.cpp:37-80) ----------------------------------
// 0 ok, 1 std::out_of_range (message in ref_last_error), -1 other error
int ref_csr_from_triplets(int32_t m, int32_t n, int64_t count, const int32_t* rows,
                          const int32_t* cols, const double* vals, int32_t* row_ptr,
                          int32_t* col_idx, double* values_out, int64_t* nnz) {
  try {
    std::vector<std::tuple<int, int, double>> t((size_t)count);
    for (int64_t i = 0; i < count; ++i) t[(size_t)i] = {rows[i], cols[i], vals[i]};
    const SparseMatrix mat = csr_from_triplets(t, m, n);
    std::copy(mat.row_ptr.begin(), mat.row_ptr.end(), row_ptr);
    std::copy(mat.col_idx.begin(), mat.col_idx.end(), col_idx);
    std::copy(mat.values.begin(), mat.values.end(), values_out);
    *nnz = (int64_t)mat.col_idx.size();
    return 0;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---- propcore (for golden vectors of the unit KATs) ----------------------

void ref_row_activities(const int32_t* cols, const double* coefs, int64_t len,
                        const double* lower, const double* upper, int32_t n, double* out4) {
  const std::span<const int> c(cols, (size_t)len);
  const std::span<const double> a(coefs, (size_t)len);
  const auto act = compute_row_activities<double>(c, a, std::span<const double>(lower, n),
                                                  std::span<const double>(upper, n));
  out4[0] = act.min_finite;
  out4[1] = act.max_finite;
  out4[2] = act.min_inf_count;
  out4[3] = act.max_inf_count;
}

void ref_residual(const double* act4, double a, double lo, double up, double* out2) {
  ActivityRecordT<double> act{act4[0], act4[1], (int)act4[2], (int)act4[3]};
  const auto r = residual_activities<double>(act, a, lo, up);
  out2[0] = r.min_res;
  out2[1] = r.max_res;
}

void ref_candidates(double a, double lhs, double rhs, double min_res, double max_res,
                    int32_t integral, const pg_config* c, double* out2) {
  const auto cand =
      compute_bound_candidates<double>(a, lhs, rhs, min_res, max_res, integral != 0, to_cfg(c));
  out2[0] = cand.new_lower;
  out2[1] = cand.new_upper;
}

int32_t ref_classify(const double* act4, double lhs, double rhs, const pg_config* c) {
  ActivityRecordT<double> act{act4[0], act4[1], (int)act4[2], (int)act4[3]};
  return (int32_t)classify_constraint<double>(act, lhs, rhs, to_cfg(c));
}

int32_t ref_tighten(double old_lo, double old_up, double cand_lo, double cand_up,
                    const pg_config* c, double* out2) {
  BoundCandidate<double> cand;
  cand.new_lower = cand_lo;
  cand.new_upper = cand_up;
  const auto o = tighten<double>(old_lo, old_up, cand, to_cfg(c));
  out2[0] = o.new_lower;
  out2[1] = o.new_upper;
  return (int32_t)o.kind;
}

}  // extern "C"
