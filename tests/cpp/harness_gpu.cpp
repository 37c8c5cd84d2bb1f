// The reference's own bench harness driving the GPU engine (SURVEY.md 8(f)
// row 1).  Linked against the reference's harness.cpp with the EngineId::Gpu
// patch INTEGRATION.md describes (applied to a build-time copy by
// oracle/patch_harness.py; nothing of the reference is committed), so
// run_benchmark's best-of-N timing, exclusion of non-converged instances,
// speedup geomean / percentiles / size classes and bench_to_csv /
// bench_to_json are the reference's code (core/src/harness.cpp:124-213+).
//
// Instances: gen_cascade m in {2, 10, 50, 200}, the C1 configuration
// (gen_random 10k x 10k, mean 8, 50% integral) seeds 1-5, and any instance
// files given on the command line (.pgi: int64 m, n, nnz, then row_ptr,
// col_idx (i32), values, lhs, rhs, lower, upper (f64), integral (u8)), each
// written out with the reference's write_mps and read back with its
// parse_mps (the reference's MPS path), e.g. the 6 MPS fixtures.
// Engines {Seq, Par, Gpu}, baseline Seq.  Besides the tables, every GPU
// result is compared with the reference's compare_results (harness.cpp:
// 22-60) against cpu_par (bit-identical expected) and cpu_seq (the
// acceptance comparator, tests/acceptance.cpp:104-117).
//
// usage: harness_gpu OUT_PREFIX [file.pgi ...]   -> OUT_PREFIX.csv / .json
// exit code = number of failed checks
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "propgate/generators.hpp"
#include "propgate/harness.hpp"
#include "propgate/mps.hpp"
#include "propgate/par_engine.hpp"
#include "propgate/seq_engine.hpp"
#include "propgate_b200.hpp"

using namespace propgate;

// a raw instance file (written by tests/test_gpu_dropin.py)
static ProblemInstance read_pgi(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  int64_t h[3];
  in.read(reinterpret_cast<char*>(h), sizeof(h));
  ProblemInstance inst;
  inst.matrix.num_rows = (int)h[0];
  inst.matrix.num_cols = (int)h[1];
  auto rd = [&](auto& v, size_t n) {
    v.resize(n);
    in.read(reinterpret_cast<char*>(v.data()), (std::streamsize)(n * sizeof(v[0])));
  };
  rd(inst.matrix.row_ptr, (size_t)h[0] + 1);
  rd(inst.matrix.col_idx, (size_t)h[2]);
  rd(inst.matrix.values, (size_t)h[2]);
  rd(inst.lhs, (size_t)h[0]);
  rd(inst.rhs, (size_t)h[0]);
  rd(inst.bounds.lower, (size_t)h[1]);
  rd(inst.bounds.upper, (size_t)h[1]);
  rd(inst.integral, (size_t)h[1]);
  if (!in) throw std::runtime_error("short instance file " + path);
  // through the reference's MPS writer and parser
  std::stringstream mps;
  write_mps(inst, mps);
  return parse_mps(mps);
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s OUT_PREFIX [file.mps ...]\n", argv[0]);
    return 2;
  }
  const std::string out = argv[1];
  std::vector<BenchInput> inputs;
  for (int m : {2, 10, 50, 200}) inputs.push_back({"cascade" + std::to_string(m), gen_cascade(m)});
  for (int seed = 1; seed <= 5; ++seed) {
    RandomInstanceOptions o;
    o.num_rows = o.num_cols = 10000;
    o.seed = (std::uint64_t)seed;
    o.mean_row_nnz = 8.0;
    o.integral_fraction = 0.5;
    inputs.push_back({"c1_s" + std::to_string(seed), gen_random(o)});
  }
  for (int i = 2; i < argc; ++i) {
    std::string name = argv[i];
    const size_t slash = name.find_last_of('/');
    if (slash != std::string::npos) name = name.substr(slash + 1);
    inputs.push_back({name, read_pgi(argv[i])});
  }

  const EngineConfig cfg;
  int failures = 0;
  // agreement (acceptance.cpp:104-117 style): GPU vs cpu_par bit-identical,
  // GPU vs cpu_seq within the reference comparator (continuous bounds of
  // Jacobi vs Gauss-Seidel tails differ)
  for (const BenchInput& in : inputs) {
    const PropagationResult par = propagate_parallel(in.instance, cfg);
    const PropagationResult seq = propagate_sequential(in.instance, cfg);
    GpuOptions plain;
    plain.row_check = false;
    const PropagationResult g_par = propagate_gpu(in.instance, cfg, plain);
    const PropagationResult g = propagate_gpu(in.instance, cfg);
    const ComparisonReport rp = compare_results(par, g_par, 0.0, 0.0);
    const bool same_par = rp.equal && par.rounds_executed == g_par.rounds_executed &&
                          par.per_round_changes == g_par.per_round_changes;
    const bool inf_seq = seq.status == PropagationStatus::Infeasible;
    const bool inf_gpu = g.status == PropagationStatus::Infeasible;
    bool ok_seq = inf_seq == inf_gpu;
    if (ok_seq && seq.status == PropagationStatus::Converged &&
        g.status == PropagationStatus::Converged)
      ok_seq = compare_results(seq, g).equal;
    std::printf("%s  %-24s gpu(row check off) == cpu_par: %s; verdict/bounds vs cpu_seq: %s "
                "(%s, %d rounds)\n",
                same_par && ok_seq ? "PASS" : "FAIL", in.name.c_str(), same_par ? "yes" : "NO",
                ok_seq ? "yes" : "NO", inf_gpu ? "Infeasible" : "feasible", g.rounds_executed);
    failures += !same_par + !ok_seq;
  }

  const std::vector<EngineId> engines = {EngineId::Seq, EngineId::Par, EngineId::Gpu};
  BenchOptions opt;
  opt.repetitions = 3;
  opt.baseline = EngineId::Seq;
  const BenchTable table = run_benchmark(inputs, engines, cfg, opt);
  std::ofstream(out + ".csv") << bench_to_csv(table);
  std::ofstream(out + ".json") << bench_to_json(table);
  for (const EngineAggregate& a : table.aggregates)
    std::printf("engine %s: %d instances in the means, geomean speedup vs seq %.2f (p50 %.2f)\n",
                to_string(a.engine), a.included, a.geo_mean, a.p50);
  std::printf("excluded (not converged in every engine): %zu\n", table.excluded.size());
  bool has_gpu = false;
  for (const BenchRecord& r : table.records) has_gpu |= r.engine == EngineId::Gpu;
  if (!has_gpu) ++failures;
  std::printf("%d failed checks\n", failures);
  return failures;
}
