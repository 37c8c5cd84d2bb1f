// nodes.cuh -- a batch of branch-and-bound nodes, one CTA per node.
//
// Config C4: K child nodes of a root fixpoint, node k = the root bounds with
// a few columns overridden.  Each node is an independent cpu_par solve
// (run_parallel, par_engine.cpp:203-273) from its start bounds; a node
// touches few rows, so a solve is run sparsely by one CTA, and many nodes
// run at once (one per resident CTA, nodes handed out by a ticket):
//   * the CTA's slot holds the round-input bounds and the merge keys of
//     every column (root values, with the node's changes applied and undone
//     afterwards -- no per-node O(n) reset);
//   * round r visits only the rows containing a column changed in round
//     r - 1 (round 1: the overridden columns).  Exact: a row none of whose
//     bounds changed produces the candidates it produced before, which were
//     rejected against the same bounds (the root's confirming round, or
//     round r - 1), the reference's marking argument (seq_engine.cpp:29,77);
//   * per dirty row, one thread: activity in entry order (chunked pairwise
//     sums for rows longer than nnz_budget, par_engine.cpp:99-123), row
//     check, exactness-preserving filters, the exact candidate pipeline
//     (propcore.hpp:78-208) and 64-bit atomic merges into the slot's keys;
//   * commit over the columns whose keys moved: change count, crossing
//     check, next round's rows (column index); then the round decision in
//     run_parallel's order (Infeasible, Converged, RoundLimit).
#pragma once

#include "kernels.cuh"

namespace pgb {

constexpr int kNodeThreads = 256;

struct NodeArgs {
  // matrix (sorted-row CSR) and its column index (column -> sorted rows)
  const int32_t* row_ptr;
  const int32_t* colx;
  const double* vals;
  const double* lhs;
  const double* rhs;
  const int32_t* col_ptr;
  const int32_t* col_row;
  int32_t m, n;
  // root fixpoint
  const double* root_lo;
  const double* root_up;
  // nodes
  int32_t K;
  const int32_t* node_ptr;
  const int32_t* vars;
  const double* nlo;
  const double* nup;
  int32_t* status;
  int32_t* rounds;
  double* lower_out;  // [K * n] or null
  double* upper_out;
  int32_t* ticket;
  // per-slot scratch, slot s at offset s * (n or m or parts)
  double* s_lo;
  double* s_up;
  longlong2* s_key;
  int32_t* s_cflag;  // bit 0: key moved this round, bit 1: on the undo list
  int32_t* s_touch;
  int32_t* s_undo;
  int32_t* s_rflag;
  int32_t* s_rows;   // two lists of m
  Act* s_part;       // chunk partials: kNodeThreads * maxc per slot
  int32_t maxc;
};

struct NodeSmem {
  int32_t nrows, nnext, ntouch, nundo;
  int32_t infeasible;
  unsigned long long changes;
  int32_t node;
};

// activity of sorted row r under the slot's bounds, in cpu_par's summation
// order; xmax = max |a| q over the row (filter)
__device__ __forceinline__ Act node_row_activity(const NodeArgs& N, int r, const double* lo,
                                                 const double* up, Act* part, const DevCfg& cfg,
                                                 double& xmax) {
  const int k0 = N.row_ptr[r], k1 = N.row_ptr[r + 1];
  const int chunk = cfg.chunk;
  xmax = -CUDART_INF;
  int np = 0;
  for (int b = k0; b < k1 || b == k0; b += chunk) {
    // one chain (compute_row_activities, propcore.hpp:45-65); a row of at
    // most nnz_budget entries is a single chain
    Act a = {0.0, 0.0, 0, 0};
    const int e1 = k1 - k0 <= chunk ? k1 : min(k1, b + chunk);
    for (int k = b; k < e1; ++k) {
      const double v = N.vals[k];
      const int32_t cx = N.colx[k];
      const int j = cx & 0x7fffffff;
      const double l = lo[j], u = up[j];
      const double bmin = v > 0 ? l : u;
      const double bmax = v > 0 ? u : l;
      if (isinf(bmin)) ++a.min_i; else a.min_f = __dadd_rn(a.min_f, __dmul_rn(v, bmin));
      if (isinf(bmax)) ++a.max_i; else a.max_f = __dadd_rn(a.max_f, __dmul_rn(v, bmax));
      xmax = fmax(xmax, fabs(v) * column_q(l, u, cx < 0, cfg));
    }
    if (k1 - k0 <= chunk) return a;
    part[np++] = a;
  }
  while (np > 1) {  // pairwise in chunk order (par_engine.cpp:117-121)
    int out = 0;
    for (int i = 0; i + 1 < np; i += 2) part[out++] = act_combine(part[i], part[i + 1]);
    if (np & 1) part[out++] = part[np - 1];
    np = out;
  }
  return part[0];
}

// one entry's candidates against the slot's bounds; merges into the slot's
// keys.  Returns bit 0 = EmptyDomain, bit 1 = a key moved
__device__ __forceinline__ int node_entry(const Act& act, double a, double lo, double up, double l,
                                          double h, int32_t cx, longlong2* key, const DevCfg& cfg) {
  double min_res, max_res, cl, cu;
  residual(act, a, lo, up, min_res, max_res);
  candidates(a, l, h, min_res, max_res, cx < 0, cfg, cl, cu);
  const int kind = tighten(lo, up, cl, cu, cfg);
  if (kind == 4) return 1;
  const int j = cx & 0x7fffffff;
  int moved = 0;
  if (kind & 1) {
    const long long k = key_enc(canon0(cl));
    long long* p = &key[j].x;
    if (ld_gpu(p) < k && atomicMax(p, k) < k) moved = 2;
  }
  if (kind & 2) {
    const long long k = -key_enc(canon0(cu));
    long long* p = &key[j].y;
    if (ld_gpu(p) < k && atomicMax(p, k) < k) moved = 2;
  }
  return moved;
}

template <bool kRowCheck>
__global__ void __launch_bounds__(kNodeThreads) k_nodes(const NodeArgs N, const DevCfg cfg) {
  __shared__ NodeSmem S;
  const int slot = blockIdx.x;
  double* lo = N.s_lo + (size_t)slot * N.n;
  double* up = N.s_up + (size_t)slot * N.n;
  longlong2* key = N.s_key + (size_t)slot * N.n;
  int32_t* cflag = N.s_cflag + (size_t)slot * N.n;
  int32_t* touch = N.s_touch + (size_t)slot * N.n;
  int32_t* undo = N.s_undo + (size_t)slot * N.n;
  int32_t* rflag = N.s_rflag + (size_t)slot * N.m;
  int32_t* rows[2] = {N.s_rows + (size_t)slot * 2 * N.m, N.s_rows + ((size_t)slot * 2 + 1) * N.m};
  Act* part = N.s_part + ((size_t)slot * kNodeThreads + threadIdx.x) * N.maxc;
  const int tid = threadIdx.x;

  // the slot starts as the root (once per launch)
  for (int j = tid; j < N.n; j += blockDim.x) {
    lo[j] = N.root_lo[j];
    up[j] = N.root_up[j];
    key[j] = make_longlong2(key_enc(N.root_lo[j]), -key_enc(N.root_up[j]));
    cflag[j] = 0;
  }
  for (int i = tid; i < N.m; i += blockDim.x) rflag[i] = 0;
  __syncthreads();

  for (;;) {
    if (tid == 0) {
      S.node = atomicAdd(N.ticket, 1);
      S.nrows = S.nnext = S.ntouch = S.nundo = 0;
      S.infeasible = 0;
    }
    __syncthreads();
    const int node = S.node;
    if (node >= N.K) break;
    int cur = 0;
    // start bounds: overrides (normalised like every start bound), crossing
    // check over them (the root is not crossed), their rows marked
    const int v0 = N.node_ptr[node], v1 = N.node_ptr[node + 1];
    for (int i = v0 + tid; i < v1; i += blockDim.x) {
      const int j = N.vars[i];
      double l = N.nlo[i], u = N.nup[i];
      l = l >= cfg.inf_thr ? CUDART_INF : (l <= -cfg.inf_thr ? -CUDART_INF : l);
      u = u >= cfg.inf_thr ? CUDART_INF : (u <= -cfg.inf_thr ? -CUDART_INF : u);
      lo[j] = l;
      up[j] = u;
      key[j] = make_longlong2(key_enc(l), -key_enc(u));
      if (!(atomicOr(&cflag[j], 2) & 2)) undo[atomicAdd(&S.nundo, 1)] = j;
      if (l > __dadd_rn(u, cfg.imp_abs)) S.infeasible = 1;  // engine_common.hpp:51-58
      for (int e = N.col_ptr[j]; e < N.col_ptr[j + 1]; ++e) {
        const int r = N.col_row[e];
        if (!atomicExch(&rflag[r], 1)) rows[cur][atomicAdd(&S.nrows, 1)] = r;
      }
    }
    __syncthreads();
    int status = -1, round = 0;
    if (S.infeasible) status = 2;  // PG_INFEASIBLE with 0 rounds
    while (status < 0) {
      ++round;
      // ---- the round's rows ---------------------------------------------------
      const int nr = S.nrows;
      for (int i = tid; i < nr; i += blockDim.x) {
        const int r = rows[cur][i];
        rflag[r] = 0;
        double xmax;
        const Act act = node_row_activity(N, r, lo, up, part, cfg, xmax);
        const double l = N.lhs[r], h = N.rhs[r];
        if (kRowCheck && row_infeasible(act, l, h, cfg)) S.infeasible = 1;
        const RowFilter f = row_filter(act, l, h);
        if (!row_may(f, xmax)) continue;
        for (int k = N.row_ptr[r]; k < N.row_ptr[r + 1]; ++k) {
          const double a = N.vals[k];
          const int32_t cx = N.colx[k];
          const int j = cx & 0x7fffffff;
          const double bl = lo[j], bu = up[j];
          const double bmin = a > 0 ? bl : bu;
          const double bmax = a > 0 ? bu : bl;
          if (!entry_may(f, fabs(a) * column_q(bl, bu, cx < 0, cfg), isinf(bmin), isinf(bmax)))
            continue;
          const int res = node_entry(act, a, bl, bu, l, h, cx, key, cfg);
          if (res & 1) S.infeasible = 1;
          if ((res & 2) && !(atomicOr(&cflag[j], 1) & 1)) touch[atomicAdd(&S.ntouch, 1)] = j;
        }
      }
      __syncthreads();
      // ---- commit (par_engine.cpp:191-197) -------------------------------------
      if (tid == 0) {
        S.changes = 0;
        S.nnext = 0;
      }
      __syncthreads();
      const int nt = S.ntouch;
      unsigned long long ch = 0;
      for (int i = tid; i < nt; i += blockDim.x) {
        const int j = touch[i];
        const longlong2 kk = key[j];
        const double nl = key_dec(kk.x), nu = key_dec(-kk.y);
        ch += (nl != lo[j]) + (nu != up[j]);
        lo[j] = nl;
        up[j] = nu;
        if (nl > __dadd_rn(nu, cfg.imp_abs)) S.infeasible = 1;
        if (!(atomicAnd(&cflag[j], ~1) & 2)) {
          atomicOr(&cflag[j], 2);
          undo[atomicAdd(&S.nundo, 1)] = j;
        }
        for (int e = N.col_ptr[j]; e < N.col_ptr[j + 1]; ++e) {
          const int r = N.col_row[e];
          if (!atomicExch(&rflag[r], 1)) rows[cur ^ 1][atomicAdd(&S.nnext, 1)] = r;
        }
      }
      if (ch) atomicAdd(&S.changes, ch);
      __syncthreads();
      // ---- decision (par_engine.cpp:248-266) -----------------------------------
      if (S.infeasible) status = 2;
      else if (S.changes == 0) status = 0;
      else if (round >= cfg.round_limit) status = 1;
      __syncthreads();
      if (tid == 0) {
        S.nrows = S.nnext;
        S.ntouch = 0;
      }
      cur ^= 1;
      __syncthreads();
    }
    // ---- results, then back to the root -------------------------------------------
    if (tid == 0) {
      N.status[node] = status;
      N.rounds[node] = round;
    }
    if (N.lower_out)
      for (int j = tid; j < N.n; j += blockDim.x) {
        N.lower_out[(size_t)node * N.n + j] = lo[j];
        N.upper_out[(size_t)node * N.n + j] = up[j];
      }
    __syncthreads();
    const int nu = S.nundo, nrem = S.nrows;
    for (int i = tid; i < nu; i += blockDim.x) {
      const int j = undo[i];
      lo[j] = N.root_lo[j];
      up[j] = N.root_up[j];
      key[j] = make_longlong2(key_enc(N.root_lo[j]), -key_enc(N.root_up[j]));
      cflag[j] = 0;
    }
    for (int i = tid; i < nrem; i += blockDim.x) rflag[rows[cur][i]] = 0;
    __syncthreads();
  }
}

}  // namespace pgb
