// propgate_b200.hpp -- header-only C++ adapter: the reference's propagator
// API (namespace propgate, /root/reference/proj/core/include/propgate/) on
// top of the C-ABI in propgate_b200.h.
//
// A maintainer of the reference adds this header to the include path, links
// libpropgate_b200.so, and calls
//
//   propgate::propagate_gpu(instance, cfg)            ~ propagate_parallel
//                                                     (par_engine.hpp:41-42)
//   propgate::propagate_round_gpu(instance, snap, partition, cfg)
//                                                     ~ propagate_round_parallel
//                                                     (par_engine.hpp:33-36)
//   propgate::csr_from_triplets_gpu(entries, m, n)     ~ csr_from_triplets
//                                                     (model.cpp:37-80), built on the GPU
//
// with the reference's own ProblemInstance / EngineConfig / PropagationResult
// (model.hpp:68-144).  Semantics follow the reference: EngineConfig::validate
// failures throw std::invalid_argument (core/src/model.cpp:21-35);
// Infeasible / RoundLimit are statuses; elapsed covers the round loop only.
// CUDA / NCCL failures throw std::runtime_error (there is no CPU fallback).
// See INTEGRATION.md for the EngineId::Gpu wiring of harness.cpp / the CLI.
#pragma once

#include <chrono>
#include <stdexcept>
#include <span>
#include <string>
#include <tuple>
#include <vector>

#include "propgate/model.hpp"
#include "propgate/par_engine.hpp"
#include "propgate_b200.h"

namespace propgate {

// GPU-only knobs; the defaults give cpu_par's bounds and cpu_seq's verdicts.
struct GpuOptions {
  int device = 0;
  bool row_check = true;   // Step-2 row check: cpu_seq infeasibility verdicts
  bool worklist = false;   // device-side worklist (exact)
  int loop_mode = PG_LOOP_GRAPH;
};

namespace b200_detail {

inline pg_config to_c(const EngineConfig& cfg, const GpuOptions& opt) {
  pg_config c;
  pg_config_default(&c);
  c.round_limit = cfg.round_limit;
  c.infinity_threshold = cfg.infinity_threshold;
  c.improvement_abs = cfg.improvement_abs;
  c.improvement_rel = cfg.improvement_rel;
  c.integrality_eps = cfg.integrality_eps;
  c.nnz_budget = cfg.nnz_budget;
  c.vector_threshold = cfg.vector_threshold;
  c.worker_count = cfg.worker_count;
  c.scalar_mode = cfg.scalar_mode == ScalarMode::Narrow32 ? PG_NARROW32 : PG_WIDE64;
  c.device = opt.device;
  c.loop_mode = opt.loop_mode;
  c.flags = (opt.row_check ? PG_FLAG_ROWCHECK : 0u) | (opt.worklist ? PG_FLAG_WORKLIST : 0u);
  return c;
}

inline pg_problem to_c(const ProblemInstance& inst) {
  pg_problem p;
  p.num_rows = inst.matrix.num_rows;
  p.num_cols = inst.matrix.num_cols;
  p.nnz = inst.matrix.nnz();
  p.row_ptr = inst.matrix.row_ptr.data();
  p.col_idx = inst.matrix.col_idx.data();
  p.values = inst.matrix.values.data();
  p.lhs = inst.lhs.data();
  p.rhs = inst.rhs.data();
  p.lower = inst.bounds.lower.data();
  p.upper = inst.bounds.upper.data();
  p.integral = inst.integral.data();
  return p;
}

inline void check(int rc, const char* what) {
  if (rc == PG_OK) return;
  const std::string msg = std::string(what) + ": " + pg_last_error();
  if (rc == PG_EINVAL) throw std::invalid_argument(pg_last_error());
  if (rc == PG_ERANGE) throw std::out_of_range(pg_last_error());
  throw std::runtime_error(msg);
}

inline PropagationStatus status_of(int s) {
  return s == PG_INFEASIBLE ? PropagationStatus::Infeasible
         : s == PG_ROUNDLIMIT ? PropagationStatus::RoundLimit
                              : PropagationStatus::Converged;
}

}  // namespace b200_detail

inline PropagationResult propagate_gpu(const ProblemInstance& instance, const EngineConfig& cfg,
                                       const GpuOptions& opt = {}) {
  cfg.validate();  // the reference's own validation and exceptions
  const pg_config c = b200_detail::to_c(cfg, opt);
  const pg_problem p = b200_detail::to_c(instance);
  PropagationResult out;
  out.bounds.lower.resize(static_cast<size_t>(instance.num_cols()));
  out.bounds.upper.resize(static_cast<size_t>(instance.num_cols()));
  std::vector<int64_t> prc(static_cast<size_t>(cfg.round_limit));
  pg_result r{};
  r.lower = out.bounds.lower.data();
  r.upper = out.bounds.upper.data();
  r.per_round_changes = prc.data();
  r.per_round_capacity = cfg.round_limit;
  b200_detail::check(pg_propagate(&p, &c, &r), "pg_propagate");
  out.status = b200_detail::status_of(r.status);
  out.rounds_executed = r.rounds_executed;
  out.total_bound_changes = r.total_bound_changes;
  out.per_round_changes.assign(prc.begin(), prc.begin() + r.rounds_executed);
  out.constraints_processed = r.constraints_processed;
  out.elapsed = std::chrono::nanoseconds(r.elapsed_ns);
  return out;
}

// One round on the caller's snapshot.  The partition argument is accepted
// for signature compatibility; the GPU uses its own tiling of the rows.
inline RoundOutcome propagate_round_gpu(const ProblemInstance& instance, RoundSnapshot& snap,
                                        const RowBlockPartition& /*partition*/,
                                        const EngineConfig& cfg, const GpuOptions& opt = {}) {
  cfg.validate();
  const pg_config c = b200_detail::to_c(cfg, opt);
  const pg_problem p = b200_detail::to_c(instance);
  snap.bounds_out.lower.resize(snap.bounds_in.lower.size());
  snap.bounds_out.upper.resize(snap.bounds_in.upper.size());
  int32_t changed = 0, infeasible = 0;
  int64_t changes = 0;
  b200_detail::check(pg_round(&p, &c, snap.bounds_in.lower.data(), snap.bounds_in.upper.data(),
                              snap.bounds_out.lower.data(), snap.bounds_out.upper.data(), &changed,
                              &infeasible, &changes),
                     "pg_round");
  RoundOutcome o;
  o.changed = changed != 0;
  o.infeasible = infeasible != 0;
  o.changes = changes;
  return o;
}

// csr_from_triplets (model.cpp:37-80) with the CSR built on the device:
// same order, duplicate sums and dropped zeros; std::out_of_range with the
// reference's messages
inline SparseMatrix csr_from_triplets_gpu(std::span<const std::tuple<int, int, double>> entries,
                                          int num_rows, int num_cols, int device = 0) {
  const size_t k = entries.size();
  std::vector<int32_t> rows(k), cols(k);
  std::vector<double> vals(k);
  for (size_t i = 0; i < k; ++i) {
    rows[i] = std::get<0>(entries[i]);
    cols[i] = std::get<1>(entries[i]);
    vals[i] = std::get<2>(entries[i]);
  }
  SparseMatrix m;
  m.num_rows = num_rows;
  m.num_cols = num_cols;
  m.row_ptr.assign(static_cast<size_t>(num_rows) + 1, 0);
  m.col_idx.resize(k);
  m.values.resize(k);
  int64_t nnz = 0;
  b200_detail::check(pg_csr_from_triplets(num_rows, num_cols, (int64_t)k, rows.data(),
                                          cols.data(), vals.data(), device, m.row_ptr.data(),
                                          m.col_idx.data(), m.values.data(), &nnz),
                     "pg_csr_from_triplets");
  m.col_idx.resize(static_cast<size_t>(nnz));
  m.values.resize(static_cast<size_t>(nnz));
  return m;
}

}  // namespace propgate
