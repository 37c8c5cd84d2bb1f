// Drop-in check (GPU box): the reference's own types, generators, engines and
// comparator with the GPU engine substituted through include/propgate_b200.hpp
// -- what EngineId::Gpu in the reference harness would run.
// Built by oracle/build_ref.sh against the unmodified reference sources.
// Exit code = number of failed checks.
#include <cstring>
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "propgate/generators.hpp"
#include "propgate/harness.hpp"
#include "propgate/par_engine.hpp"
#include "propgate/seq_engine.hpp"
#include "propgate_b200.hpp"

using namespace propgate;

static int failures = 0;
static void report(const char* what, bool ok, const std::string& detail) {
  std::printf("%s  %s: %s\n", ok ? "PASS" : "FAIL", what, detail.c_str());
  if (!ok) ++failures;
}

static bool identical(const PropagationResult& a, const PropagationResult& b) {
  // operator== on doubles: -0.0 == +0.0
  return a.status == b.status && a.rounds_executed == b.rounds_executed &&
         a.per_round_changes == b.per_round_changes && a.bounds.lower == b.bounds.lower &&
         a.bounds.upper == b.bounds.upper;
}

int main() {
  // the acceptance suite's instances (tests/acceptance.cpp:56-75)
  std::mt19937_64 rng(20240901);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  const EngineConfig cfg;
  GpuOptions par_mode;
  par_mode.row_check = false;
  int n = 0, bit_exact = 0, verdicts = 0, agree = 0, both = 0;
  for (int i = 0; i < 500; ++i) {
    RandomInstanceOptions o;
    o.num_rows = (int)std::exp(std::log(10.0) + unit(rng) * (std::log(2000.0) - std::log(10.0)));
    o.num_cols = (int)std::exp(std::log(10.0) + unit(rng) * (std::log(2000.0) - std::log(10.0)));
    o.seed = 1000 + (std::uint64_t)i;
    o.max_nnz = 50000;
    const ProblemInstance inst = gen_random(o);
    ++n;
    if (identical(propagate_gpu(inst, cfg, par_mode), propagate_parallel(inst, cfg))) ++bit_exact;
    const PropagationResult gpu = propagate_gpu(inst, cfg);  // default: row check on
    const PropagationResult seq = propagate_sequential(inst, cfg);
    if ((gpu.status == PropagationStatus::Infeasible) == (seq.status == PropagationStatus::Infeasible))
      ++verdicts;
    if (gpu.status == PropagationStatus::Converged && seq.status == PropagationStatus::Converged) {
      ++both;
      if (compare_results(seq, gpu, 1e-8, 1e-5).equal) ++agree;
    }
  }
  report("cpu_par bit-exact", bit_exact == n, std::to_string(bit_exact) + "/" + std::to_string(n));
  report("cpu_seq verdicts", verdicts == n, std::to_string(verdicts) + "/" + std::to_string(n));
  report("cpu_seq agreement (1e-8, 1e-5)", agree == both,
         std::to_string(agree) + "/" + std::to_string(both) + " both converged");

  bool casc = true;
  for (int m : {2, 10, 50}) {
    const auto r = propagate_gpu(gen_cascade(m), cfg, par_mode);
    casc = casc && r.status == PropagationStatus::Converged && r.rounds_executed == m + 1;
  }
  const auto lim = propagate_gpu(gen_cascade(200), cfg, par_mode);
  report("cascade rounds / round limit", casc && lim.status == PropagationStatus::RoundLimit &&
                                             lim.rounds_executed == 100, "m+1 rounds; 100 at m=200");

  bool threw = false;
  try {
    EngineConfig bad;
    bad.round_limit = 0;
    propagate_gpu(gen_cascade(3), bad);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  report("invalid config throws std::invalid_argument", threw, "round_limit = 0");

  RoundSnapshot snap;
  const ProblemInstance c3 = gen_cascade(3);
  snap.bounds_in = c3.bounds;
  const RoundOutcome o = propagate_round_gpu(c3, snap, partition_row_blocks(c3.matrix, cfg), cfg);
  report("one round (test_par_engine.cpp:102-116)",
         o.changed && !o.infeasible && o.changes == 1 && snap.bounds_out.upper[1] == 0.0,
         "1 change, ub[1] = 0");
  // csr_from_triplets (model.cpp:37-80): the reference's own builder vs the
  // device build on shuffled triplets with duplicates and cancelling pairs
  {
    RandomInstanceOptions ro;
    ro.num_rows = ro.num_cols = 20000;
    ro.seed = 7;
    ro.mean_row_nnz = 12.0;
    const ProblemInstance big = gen_random(ro);
    std::vector<std::tuple<int, int, double>> trip;
    for (int r = 0; r < big.matrix.num_rows; ++r)
      for (int k = big.matrix.row_ptr[r]; k < big.matrix.row_ptr[r + 1]; ++k) {
        trip.emplace_back(r, big.matrix.col_idx[k], big.matrix.values[k]);
        if (k % 5 == 0) trip.emplace_back(r, big.matrix.col_idx[k], 0.5);
        if (k % 11 == 0) trip.emplace_back(r, big.matrix.col_idx[k], -big.matrix.values[k]);
      }
    for (size_t i = trip.size() - 1; i > 0; --i) std::swap(trip[i], trip[(i * 2654435761u) % (i + 1)]);
    const SparseMatrix a = csr_from_triplets(trip, big.matrix.num_rows, big.matrix.num_cols);
    const SparseMatrix b = csr_from_triplets_gpu(trip, big.matrix.num_rows, big.matrix.num_cols);
    const bool same = a.row_ptr == b.row_ptr && a.col_idx == b.col_idx &&
                      a.values.size() == b.values.size() &&
                      std::memcmp(a.values.data(), b.values.data(), 8 * a.values.size()) == 0;
    report("csr_from_triplets on the device (model.cpp:37-80)", same,
           std::to_string(trip.size()) + " triplets -> " + std::to_string(a.values.size()) + " entries");
    bool oor = false;
    try {
      const std::vector<std::tuple<int, int, double>> bad = {{0, 0, 1.0}, {0, 5, 1.0}};
      csr_from_triplets_gpu(bad, 2, 2);
    } catch (const std::out_of_range& e) {
      oor = std::string(e.what()) == "triplet column index out of range";
    }
    report("bad triplet throws std::out_of_range", oor, "column 5 of 2");
  }
  std::printf("%d check(s) failed\n", failures);
  return failures;
}
