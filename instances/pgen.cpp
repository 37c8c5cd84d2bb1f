// pgen -- seeded synthetic instance generators (ingest side, untimed).
//
// Not on the propagation hot path: these build the inputs that both the GPU
// engine and the CPU reference consume, identically, from a seed.
//
//  * pgen_random   restates the reference's gen_random
//                  (/root/reference/proj/core/src/generators.cpp:46-168) with
//                  the same std:: engines and distributions, so a given
//                  RandomInstanceOptions yields bit-identical instances
//                  (checked against the compiled reference in tests).
//  * pgen_cascade  restates gen_cascade (generators.cpp:13-36).
//  * pgen_powerlaw config C2: Pareto row lengths.
//  * pgen_longrows config C3: 1% of rows with 100k-150k entries.
//  * pgen_setpart  config C5: planted set partitioning.
//  * pgen_nodes    config C4: branch-and-bound child-node bound vectors.
//
// C2/C3/C5 use a counter-based generator (splitmix64 streams keyed by
// seed/entity) so rows are generated in parallel yet independent of the
// thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <vector>

#include "../include/propgate_b200.h"

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct Instance {
  int32_t m = 0, n = 0;
  std::vector<int32_t> row_ptr{0};
  std::vector<int32_t> col_idx;
  std::vector<double> values, lhs, rhs, lower, upper;
  std::vector<uint8_t> integral;
};

// ---- counter-based RNG ---------------------------------------------------
inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
struct Stream {
  uint64_t s;
  Stream(uint64_t seed, uint64_t tag, uint64_t idx)
      : s(mix64(mix64(seed ^ (tag * 0xD1B54A32D192ED03ull)) ^ (idx * 0x8CB92BA72F3D8DD7ull))) {}
  uint64_t next() { return mix64(s += 0x9E3779B97F4A7C15ull); }
  double unit() { return (double)(next() >> 11) * 0x1.0p-53; }              // [0,1)
  double unit_open() { return ((double)(next() >> 11) + 1.0) * 0x1.0p-53; }  // (0,1]
  uint64_t below(uint64_t b) { return next() % b; }
};

enum : uint64_t { kTagCol = 1, kTagRow = 2, kTagLen = 3, kTagPerm = 4, kTagFix = 5, kTagNode = 6 };

// Column attributes following gen_random's recipe (generators.cpp:75-98):
// bounds U[-100,100] (integers rounded outward), infinite per side with
// probability inf_bound, interior point kept inside the bounds.
void column_attrs(Instance& in, std::vector<double>& point, uint64_t seed, double int_frac,
                  double inf_bound) {
  const int32_t n = in.n;
  in.lower.resize(n);
  in.upper.resize(n);
  in.integral.resize(n);
  point.resize(n);
#pragma omp parallel for schedule(static)
  for (int32_t j = 0; j < n; ++j) {
    Stream r(seed, kTagCol, (uint64_t)j);
    const bool integer = r.unit() < int_frac;
    double lo = -100.0 + 200.0 * r.unit();
    double up = -100.0 + 200.0 * r.unit();
    if (lo > up) std::swap(lo, up);
    if (integer) {
      lo = std::floor(lo);
      up = std::ceil(up);
    }
    if (r.unit() < inf_bound) lo = -kInf;
    if (r.unit() < inf_bound) up = kInf;
    double x;
    if (std::isfinite(lo) && std::isfinite(up))
      x = lo + r.unit() * (up - lo);
    else if (std::isfinite(lo))
      x = lo + 50.0 * r.unit();
    else if (std::isfinite(up))
      x = up - 50.0 * r.unit();
    else
      x = 100.0 * r.unit() - 50.0;
    if (integer) {
      x = std::round(x);
      if (std::isfinite(lo)) x = std::max(x, lo);
      if (std::isfinite(up)) x = std::min(x, up);
    }
    in.integral[j] = integer ? 1 : 0;
    in.lower[j] = lo;
    in.upper[j] = up;
    point[j] = x;
  }
}

// Sides around the interior point, as gen_random (generators.cpp:136-163):
// 25% infinite rhs, else 25% infinite lhs; finite sides t^2-scaled toward
// the activity bound.
void row_sides(Instance& in, const std::vector<double>& point, int32_t i, Stream& r,
               double inf_side) {
  const int64_t b = in.row_ptr[i], e = in.row_ptr[i + 1];
  double vp = 0.0, amin = 0.0, amax = 0.0;
  int imin = 0, imax = 0;
  for (int64_t k = b; k < e; ++k) {
    const int32_t j = in.col_idx[k];
    const double a = in.values[k];
    vp += a * point[j];
    const double bmin = a > 0 ? in.lower[j] : in.upper[j];
    const double bmax = a > 0 ? in.upper[j] : in.lower[j];
    if (std::isinf(bmin)) ++imin; else amin += a * bmin;
    if (std::isinf(bmax)) ++imax; else amax += a * bmax;
  }
  const double act_min = imin ? -kInf : amin;
  const double act_max = imax ? kInf : amax;
  const bool rhs_inf = r.unit() < inf_side;
  const bool lhs_inf = !rhs_inf && r.unit() < inf_side;
  if (rhs_inf) {
    in.rhs[i] = kInf;
  } else {
    const double t = r.unit();
    in.rhs[i] = std::isfinite(act_max) ? vp + t * t * (act_max - vp) : vp + 20.0 * t;
  }
  if (lhs_inf) {
    in.lhs[i] = -kInf;
  } else {
    const double t = r.unit();
    in.lhs[i] = std::isfinite(act_min) ? vp - t * t * (vp - act_min) : vp - 20.0 * t;
  }
}

// Fill rows whose lengths are already in row_ptr: distinct uniform columns
// (rejection with a per-thread mark array), sorted; coefficients U[-10,10]
// with |a| >= 0.1; then the sides.
void fill_random_rows(Instance& in, const std::vector<double>& point, uint64_t seed,
                      double inf_side) {
  const int32_t m = in.m, n = in.n;
  in.col_idx.resize(in.row_ptr[m]);
  in.values.resize(in.row_ptr[m]);
  in.lhs.resize(m);
  in.rhs.resize(m);
#pragma omp parallel
  {
    std::vector<uint8_t> used((size_t)n, 0);
#pragma omp for schedule(dynamic, 256)
    for (int32_t i = 0; i < m; ++i) {
      Stream r(seed, kTagRow, (uint64_t)i);
      const int64_t b = in.row_ptr[i], e = in.row_ptr[i + 1];
      int32_t* cols = in.col_idx.data() + b;
      const int64_t len = e - b;
      if (len * 2 > n) {
        // dense row: sample the complement, then list the rest in order
        std::fill(used.begin(), used.end(), 1);
        int64_t drop = n - len;
        while (drop > 0) {
          const int32_t j = (int32_t)r.below((uint64_t)n);
          if (used[j]) { used[j] = 0; --drop; }
        }
        int64_t c = 0;
        for (int32_t j = 0; j < n; ++j)
          if (used[j]) cols[c++] = j;
        std::fill(used.begin(), used.end(), 0);
      } else {
        int64_t c = 0;
        while (c < len) {
          const int32_t j = (int32_t)r.below((uint64_t)n);
          if (!used[j]) { used[j] = 1; cols[c++] = j; }
        }
        for (int64_t q = 0; q < len; ++q) used[cols[q]] = 0;
        std::sort(cols, cols + len);
      }
      for (int64_t k = b; k < e; ++k) {
        double a;
        do a = -10.0 + 20.0 * r.unit(); while (std::fabs(a) < 0.1);
        in.values[k] = a;
      }
      row_sides(in, point, i, r, inf_side);
    }
  }
}

void prefix(Instance& in, const std::vector<int64_t>& len) {
  in.row_ptr.assign((size_t)in.m + 1, 0);
  int64_t acc = 0;
  for (int32_t i = 0; i < in.m; ++i) {
    acc += len[i];
    in.row_ptr[i + 1] = (int32_t)acc;
  }
}

Instance* gen_random_restated(int32_t m, int32_t n, uint64_t seed, double mean_row_nnz,
                              double int_frac, double inf_bound, double inf_side,
                              int64_t max_nnz) {
  // generators.cpp:46-168, same RNG call order
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::uniform_real_distribution<double> coef_dist(-10.0, 10.0);
  std::uniform_real_distribution<double> bound_dist(-100.0, 100.0);
  auto* in = new Instance;
  in->m = m;
  in->n = n;
  in->lower.resize(n);
  in->upper.resize(n);
  in->integral.resize(n);
  std::vector<double> point(n);
  for (int32_t j = 0; j < n; ++j) {
    const bool integer = unit(rng) < int_frac;
    in->integral[j] = integer ? 1 : 0;
    double lo = bound_dist(rng);
    double up = bound_dist(rng);
    if (lo > up) std::swap(lo, up);
    if (integer) {
      lo = std::floor(lo);
      up = std::ceil(up);
    }
    if (unit(rng) < inf_bound) lo = -kInf;
    if (unit(rng) < inf_bound) up = kInf;
    in->lower[j] = lo;
    in->upper[j] = up;
    double x;
    if (std::isfinite(lo) && std::isfinite(up))
      x = lo + unit(rng) * (up - lo);
    else if (std::isfinite(lo))
      x = lo + 50.0 * unit(rng);
    else if (std::isfinite(up))
      x = up - 50.0 * unit(rng);
    else
      x = 100.0 * unit(rng) - 50.0;
    if (integer) {
      x = std::round(x);
      if (std::isfinite(lo)) x = std::max(x, lo);
      if (std::isfinite(up)) x = std::min(x, up);
    }
    point[j] = x;
  }
  const double p_stop = 1.0 / std::max(1.1, mean_row_nnz);
  std::geometric_distribution<int> extra(p_stop);
  std::vector<char> used(n, 0);
  std::vector<int32_t> row_cols;
  in->lhs.resize(m);
  in->rhs.resize(m);
  in->row_ptr.assign((size_t)m + 1, 0);
  int64_t nnz = 0;
  for (int32_t i = 0; i < m; ++i) {
    int len = 1 + extra(rng);
    len = std::min(len, n);
    if (max_nnz > 0 && nnz + len > max_nnz) len = (int)std::max<int64_t>(0, max_nnz - nnz);
    nnz += len;
    row_cols.clear();
    while ((int)row_cols.size() < len) {
      const int32_t j = (int32_t)(rng() % (uint64_t)n);
      if (!used[j]) {
        used[j] = 1;
        row_cols.push_back(j);
      }
    }
    for (int32_t j : row_cols) used[j] = 0;
    std::sort(row_cols.begin(), row_cols.end());
    double vp = 0.0, amin = 0.0, amax = 0.0;
    int imin = 0, imax = 0;
    for (int32_t j : row_cols) {
      double a = coef_dist(rng);
      while (std::fabs(a) < 0.1) a = coef_dist(rng);
      vp += a * point[j];
      in->col_idx.push_back(j);
      in->values.push_back(a);
    }
    // compute_row_activities over the sorted row (generators.cpp:139-142)
    for (size_t q = 0; q < row_cols.size(); ++q) {
      const int32_t j = row_cols[q];
      const double a = in->values[in->values.size() - row_cols.size() + q];
      const double bmin = a > 0 ? in->lower[j] : in->upper[j];
      const double bmax = a > 0 ? in->upper[j] : in->lower[j];
      if (std::isinf(bmin)) ++imin; else amin += a * bmin;
      if (std::isinf(bmax)) ++imax; else amax += a * bmax;
    }
    const double act_min = imin ? -kInf : amin;
    const double act_max = imax ? kInf : amax;
    const bool rhs_inf = unit(rng) < inf_side;
    const bool lhs_inf = !rhs_inf && unit(rng) < inf_side;
    if (rhs_inf) {
      in->rhs[i] = kInf;
    } else {
      const double t = unit(rng);
      in->rhs[i] = std::isfinite(act_max) ? vp + t * t * (act_max - vp) : vp + 20.0 * t;
    }
    if (lhs_inf) {
      in->lhs[i] = -kInf;
    } else {
      const double t = unit(rng);
      in->lhs[i] = std::isfinite(act_min) ? vp - t * t * (vp - act_min) : vp - 20.0 * t;
    }
    in->row_ptr[i + 1] = (int32_t)in->col_idx.size();
  }
  return in;
}

}  // namespace

extern "C" {

void pgen_view(void* h, pg_problem* p) {
  auto* in = static_cast<Instance*>(h);
  p->num_rows = in->m;
  p->num_cols = in->n;
  p->nnz = in->row_ptr[in->m];
  p->row_ptr = in->row_ptr.data();
  p->col_idx = in->col_idx.data();
  p->values = in->values.data();
  p->lhs = in->lhs.data();
  p->rhs = in->rhs.data();
  p->lower = in->lower.data();
  p->upper = in->upper.data();
  p->integral = in->integral.data();
}

void pgen_free(void* h) { delete static_cast<Instance*>(h); }

// Copy of caller arrays into a generator-owned instance (used to hand
// fixture data or modified bounds around with one lifetime).
void* pgen_from_arrays(const pg_problem* p) {
  auto* in = new Instance;
  in->m = p->num_rows;
  in->n = p->num_cols;
  in->row_ptr.assign(p->row_ptr, p->row_ptr + p->num_rows + 1);
  in->col_idx.assign(p->col_idx, p->col_idx + p->nnz);
  in->values.assign(p->values, p->values + p->nnz);
  in->lhs.assign(p->lhs, p->lhs + p->num_rows);
  in->rhs.assign(p->rhs, p->rhs + p->num_rows);
  in->lower.assign(p->lower, p->lower + p->num_cols);
  in->upper.assign(p->upper, p->upper + p->num_cols);
  in->integral.assign(p->integral, p->integral + p->num_cols);
  return in;
}

void* pgen_random(int32_t m, int32_t n, uint64_t seed, double mean_row_nnz, double int_frac,
                  double inf_bound, double inf_side, int64_t max_nnz) {
  if (m < 1 || n < 1) return nullptr;
  return gen_random_restated(m, n, seed, mean_row_nnz, int_frac, inf_bound, inf_side, max_nnz);
}

// gen_cascade (generators.cpp:13-36): x_k - x_{k-1} <= 0, x_0 in [0,0],
// the rest in [0, 1e6].
void* pgen_cascade(int32_t m) {
  if (m < 2) return nullptr;
  auto* in = new Instance;
  in->m = m;
  in->n = m + 1;
  in->row_ptr.resize(m + 1);
  for (int32_t k = 1; k <= m; ++k) {
    in->col_idx.push_back(k - 1);
    in->values.push_back(-1.0);
    in->col_idx.push_back(k);
    in->values.push_back(1.0);
    in->row_ptr[k] = 2 * k;
  }
  in->lhs.assign(m, -kInf);
  in->rhs.assign(m, 0.0);
  in->lower.assign(m + 1, 0.0);
  in->upper.assign(m + 1, 1e6);
  in->upper[0] = 0.0;
  in->integral.assign(m + 1, 0);
  return in;
}

// C2: power-law row lengths L = floor(x_min * U^(-1/beta)) clipped to
// [1, cap]; gen_random-style columns, coefficients and sides.
void* pgen_powerlaw(int32_t m, int32_t n, uint64_t seed, double x_min, double beta, int32_t cap,
                    double int_frac, double inf_bound, double inf_side) {
  if (m < 1 || n < 1) return nullptr;
  auto* in = new Instance;
  in->m = m;
  in->n = n;
  std::vector<double> point;
  column_attrs(*in, point, seed, int_frac, inf_bound);
  std::vector<int64_t> len(m);
  const int64_t lim = std::min<int64_t>(cap, n);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < m; ++i) {
    Stream r(seed, kTagLen, (uint64_t)i);
    const double L = std::floor(x_min * std::pow(r.unit_open(), -1.0 / beta));
    len[i] = (int64_t)std::min<double>(std::max(1.0, L), (double)lim);
  }
  prefix(*in, len);
  fill_random_rows(*in, point, seed, inf_side);
  return in;
}

// C3: every long_every-th row has U[long_min, long_max] entries, the rest
// 1 + geometric (mean mean_short), as gen_random's lengths.
void* pgen_longrows(int32_t m, int32_t n, uint64_t seed, int32_t long_every, int32_t long_min,
                    int32_t long_max, double mean_short, double int_frac, double inf_bound,
                    double inf_side) {
  if (m < 1 || n < 1 || long_every < 1) return nullptr;
  auto* in = new Instance;
  in->m = m;
  in->n = n;
  std::vector<double> point;
  column_attrs(*in, point, seed, int_frac, inf_bound);
  std::vector<int64_t> len(m);
  const double p = 1.0 / std::max(1.1, mean_short);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < m; ++i) {
    Stream r(seed, kTagLen, (uint64_t)i);
    int64_t L;
    if (i % long_every == 0)
      L = long_min + (int64_t)r.below((uint64_t)(long_max - long_min + 1));
    else
      L = 1 + (int64_t)std::floor(std::log(r.unit_open()) / std::log1p(-p));
    len[i] = std::min<int64_t>(std::max<int64_t>(L, 1), n);
  }
  prefix(*in, len);
  fill_random_rows(*in, point, seed, inf_side);
  return in;
}

// C5: planted set partitioning.  n1 = round(s1_frac * m) columns form S1
// (x* = 1); every row holds exactly one S1 column and per_row-1 distinct S0
// columns, coefficients 1, lhs = rhs = 1, all variables binary.  Column
// labels are a random permutation.  A fraction f_fixed of S1 columns starts
// with lb = 1.  infeasible != 0 also sets lb = 1 on one S0 column of a row
// whose S1 column is fixed.
void* pgen_setpart(int32_t m, int32_t n, int32_t per_row, double s1_frac, double f_fixed,
                   uint64_t seed, int32_t infeasible) {
  const int64_t n1 = std::max<int64_t>(1, std::llround(s1_frac * m));
  if (m < 1 || per_row < 1 || n1 >= n || per_row - 1 > n - n1) return nullptr;
  auto* in = new Instance;
  in->m = m;
  in->n = n;
  // label[c] for canonical column c: c < n1 is S1, else S0
  std::vector<int32_t> label(n);
  for (int32_t c = 0; c < n; ++c) label[c] = c;
  {
    Stream r(seed, kTagPerm, 0);
    for (int32_t c = n - 1; c > 0; --c) std::swap(label[c], label[(int32_t)r.below((uint64_t)c + 1)]);
  }
  in->row_ptr.resize((size_t)m + 1);
  for (int32_t i = 0; i <= m; ++i) in->row_ptr[i] = i * per_row;
  in->col_idx.resize((size_t)m * per_row);
  in->values.assign((size_t)m * per_row, 1.0);
  in->lhs.assign(m, 1.0);
  in->rhs.assign(m, 1.0);
  std::vector<int32_t> s1_of_row(m);
  const int64_t n0 = n - n1;
#pragma omp parallel
  {
    std::vector<uint8_t> used((size_t)n0, 0);
    std::vector<int32_t> tmp(per_row);
    std::vector<int64_t> picked(per_row);
#pragma omp for schedule(static)
    for (int32_t i = 0; i < m; ++i) {
      Stream r(seed, kTagRow, (uint64_t)i);
      const int32_t s1 = (int32_t)r.below((uint64_t)n1);
      s1_of_row[i] = s1;
      tmp[0] = label[s1];
      for (int32_t q = 1; q < per_row;) {
        const int64_t c0 = (int64_t)r.below((uint64_t)n0);
        if (!used[c0]) {
          used[c0] = 1;
          picked[q] = c0;
          tmp[q++] = label[n1 + c0];
        }
      }
      for (int32_t q = 1; q < per_row; ++q) used[picked[q]] = 0;
      std::sort(tmp.begin(), tmp.end());
      std::copy(tmp.begin(), tmp.end(), in->col_idx.begin() + (size_t)i * per_row);
    }
  }
  in->lower.assign(n, 0.0);
  in->upper.assign(n, 1.0);
  in->integral.assign(n, 1);
  std::vector<uint8_t> fixed(n1, 0);
  for (int64_t c = 0; c < n1; ++c) {
    Stream r(seed, kTagFix, (uint64_t)c);
    if (r.unit() < f_fixed) {
      fixed[c] = 1;
      in->lower[label[c]] = 1.0;
    }
  }
  if (infeasible) {
    for (int32_t i = 0; i < m; ++i) {
      if (!fixed[s1_of_row[i]]) continue;
      const int32_t s1col = label[s1_of_row[i]];
      for (int32_t q = 0; q < per_row; ++q) {
        const int32_t c = in->col_idx[(size_t)i * per_row + q];
        if (c != s1col) {
          in->lower[c] = 1.0;
          break;
        }
      }
      break;
    }
  }
  return in;
}

// C4: K child-node bound vectors (node-major [K * n]) from root bounds.
// Node k: stream (seed_base + k); depth d ~ U{dmin..dmax}; d distinct
// integer variables with finite root width >= 1; mid = floor((lb+ub)/2);
// down branch ub = mid or up branch lb = mid + 1 with p = 1/2.
int pgen_nodes(const pg_problem* p, const double* root_lo, const double* root_up, int32_t K,
               uint64_t seed_base, int32_t dmin, int32_t dmax, double* lo_out, double* up_out) {
  const int32_t n = p->num_cols;
  std::vector<int32_t> cand;
  for (int32_t j = 0; j < n; ++j)
    if (p->integral[j] && std::isfinite(root_lo[j]) && std::isfinite(root_up[j]) &&
        root_up[j] - root_lo[j] >= 1.0)
      cand.push_back(j);
#pragma omp parallel for schedule(static)
  for (int32_t k = 0; k < K; ++k) {
    double* lo = lo_out + (size_t)k * n;
    double* up = up_out + (size_t)k * n;
    std::memcpy(lo, root_lo, sizeof(double) * n);
    std::memcpy(up, root_up, sizeof(double) * n);
    if (cand.empty()) continue;
    Stream r(seed_base + (uint64_t)k, kTagNode, 0);
    const int32_t d = dmin + (int32_t)r.below((uint64_t)(dmax - dmin + 1));
    std::vector<int32_t> picked;
    for (int32_t t = 0; (int32_t)picked.size() < d && t < 64 * d; ++t) {
      const int32_t j = cand[r.below(cand.size())];
      if (std::find(picked.begin(), picked.end(), j) != picked.end()) continue;
      picked.push_back(j);
      const double mid = std::floor((root_lo[j] + root_up[j]) / 2.0);
      if (r.unit() < 0.5)
        up[j] = mid;
      else
        lo[j] = mid + 1.0;
    }
  }
  return 0;
}

}  // extern "C"

extern "C" {

// Instance sizes of the reference acceptance suite (tests/acceptance.cpp:56-75):
// log-uniform rows/cols in [10, 2000] from std::mt19937_64(20240901); seed
// 1000 + i; max_nnz 50000 (options otherwise default).
void pgen_acceptance_sizes(int32_t count, int32_t* rows, int32_t* cols) {
  std::mt19937_64 rng(20240901);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  for (int32_t i = 0; i < count; ++i) {
    rows[i] = (int32_t)std::exp(std::log(10.0) + unit(rng) * (std::log(2000.0) - std::log(10.0)));
    cols[i] = (int32_t)std::exp(std::log(10.0) + unit(rng) * (std::log(2000.0) - std::log(10.0)));
  }
}

}  // extern "C"
