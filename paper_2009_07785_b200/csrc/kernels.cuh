// kernels.cuh -- the round-synchronous propagation round on sm_100a.
//
// One round (par_engine.cpp:174-200 run_round + process_block :126-171):
//   k_tiles        rows of <= long_t entries, CSR-stream tiles of <= 1024
//                  entries: coalesced loads of vals/col, one 16 B gather of
//                  the {lb,ub} key pair per entry, activities summed per row in
//                  entry order from shared memory (bit-exact with cpu_par),
//                  candidates + tighten vs the snapshot, 64-bit atomic
//                  max/min commit of accepted sides.
//   k_long_partial one warp per nnz_budget chunk of a long row: chunk
//                  partial activity in entry order (wide_row_activities,
//                  par_engine.cpp:99-123).
//   k_long_combine pairwise tree of the chunk partials in index order.
//   k_long_cand    one CTA per chunk: candidates of the long row.
//   k_commit       per variable: changes / crossing check / snapshot update
//                  (par_engine.cpp:191-197), then the last CTA takes the
//                  round decision (par_engine.cpp:248-266) and sets the CUDA
//                  graph's WHILE condition: no host round trip per round.
#pragma once

#include <math_constants.h>

#include "propcore.cuh"

namespace pgb {

constexpr int kTileNnz = 1024;
constexpr int kTileRows = 256;
constexpr int kTileThreads = 256;
constexpr int kItems = kTileNnz / kTileThreads;
constexpr int kCommitThreads = 256;

// Device-resident loop state.
struct DevState {
  unsigned long long round_changes;  // changes of the current round
  long long total_changes;
  int32_t infeasible;                // raised by any kernel of the current round
  int32_t round;                     // rounds executed
  int32_t status;                    // -1 running, else PG_* status
  int32_t done;
  uint32_t ticket;                   // last-CTA election in k_commit
  uint32_t ticket_reset;             // last-CTA election in k_reset
  int32_t crossed;
  int32_t pad;
};

struct LongChunk {
  int32_t slot;   // long-row slot
  int32_t k0;     // first entry
  int32_t k1;     // one past last entry
  int32_t pad;
};

// ---- helpers ------------------------------------------------------------------
__device__ __forceinline__ longlong2 ld_key(const longlong2* p) { return __ldg(p); }

__device__ __forceinline__ void commit_side(long long* key_out, int j, int kind, double cl,
                                            double cu) {
  // merge_lower / merge_upper (par_engine.cpp:56-71) as exact 64-bit max/min
  if (kind & 1) {
    const long long k = key_enc(canon0(cl));
    long long* p = key_out + 2 * (size_t)j;
    if (*((volatile long long*)p) < k) atomicMax(p, k);
  }
  if (kind & 2) {
    const long long k = key_enc(canon0(cu));
    long long* p = key_out + 2 * (size_t)j + 1;
    if (*((volatile long long*)p) > k) atomicMin(p, k);
  }
}

// ---- K1: tiles of short rows --------------------------------------------------
template <bool kRowCheck>
__global__ void __launch_bounds__(kTileThreads)
    k_tiles(const int2* __restrict__ tiles, const int32_t* __restrict__ row_ptr,
            const int32_t* __restrict__ colx, const double* __restrict__ vals,
            const double* __restrict__ lhs, const double* __restrict__ rhs,
            const longlong2* __restrict__ key_in, long long* __restrict__ key_out,
            DevState* __restrict__ st, const DevCfg cfg) {
  __shared__ double s_pmin[kTileNnz];
  __shared__ double s_pmax[kTileNnz];
  __shared__ Act s_act[kTileRows];
  __shared__ double s_lhs[kTileRows];
  __shared__ double s_rhs[kTileRows];
  __shared__ int32_t s_rp[kTileRows + 1];
  __shared__ uint8_t s_row[kTileNnz];
  __shared__ int32_t s_inf;

  const int tid = threadIdx.x;
  const int2 tl = tiles[blockIdx.x];
  const int r0 = tl.x;
  const int nr = tl.y - tl.x;
  if (tid == 0) s_inf = 0;
  for (int i = tid; i <= nr; i += kTileThreads) s_rp[i] = row_ptr[r0 + i];
  __syncthreads();
  const int k0 = s_rp[0];
  const int nz = s_rp[nr] - k0;

  // phase 1: coalesced entry loads + one 16 B snapshot gather per entry
  double a[kItems], lo[kItems], up[kItems];
  int32_t cx[kItems];
#pragma unroll
  for (int q = 0; q < kItems; ++q) {
    const int e = tid + q * kTileThreads;
    if (e < nz) {
      cx[q] = __ldg(colx + k0 + e);
      a[q] = __ldg(vals + k0 + e);
    }
  }
#pragma unroll
  for (int q = 0; q < kItems; ++q) {
    const int e = tid + q * kTileThreads;
    if (e < nz) {
      const longlong2 kk = ld_key(key_in + (cx[q] & 0x7fffffff));
      lo[q] = key_dec(kk.x);
      up[q] = key_dec(kk.y);
      double pmin, pmax;
      contrib(a[q], lo[q], up[q], pmin, pmax);
      s_pmin[e] = pmin;
      s_pmax[e] = pmax;
    }
  }
  __syncthreads();

  // phase 2: one thread per row, sum in entry order (propcore.hpp:50-63)
  for (int r = tid; r < nr; r += kTileThreads) {
    const int b = s_rp[r] - k0, e = s_rp[r + 1] - k0;
    Act act = {0.0, 0.0, 0, 0};
    for (int k = b; k < e; ++k) {
      act_add(act, s_pmin[k], s_pmax[k]);
      s_row[k] = (uint8_t)r;
    }
    s_act[r] = act;
    const double l = lhs[r0 + r], h = rhs[r0 + r];
    s_lhs[r] = l;
    s_rhs[r] = h;
    if (kRowCheck && row_infeasible(act, l, h, cfg)) s_inf = 1;
  }
  __syncthreads();

  // phase 3: candidates vs the frozen snapshot, atomic commit
#pragma unroll
  for (int q = 0; q < kItems; ++q) {
    const int e = tid + q * kTileThreads;
    if (e < nz) {
      const int r = s_row[e];
      const Act act = s_act[r];
      double min_res, max_res, cl, cu;
      residual(act, a[q], lo[q], up[q], min_res, max_res);
      candidates(a[q], s_lhs[r], s_rhs[r], min_res, max_res, cx[q] < 0, cfg, cl, cu);
      const int kind = tighten(lo[q], up[q], cl, cu, cfg);
      if (kind == 4) {
        s_inf = 1;  // EmptyDomain: flag, skip the merge (par_engine.cpp:163-166)
      } else if (kind) {
        commit_side(key_out, cx[q] & 0x7fffffff, kind, cl, cu);
      }
    }
  }
  __syncthreads();
  if (tid == 0 && s_inf) st->infeasible = 1;
}

// ---- long rows ----------------------------------------------------------------
// One warp per chunk; lanes load 32 entries at a time (coalesced) and the
// products are folded in entry order through warp shuffles.
__global__ void __launch_bounds__(256)
    k_long_partial(const LongChunk* __restrict__ chunks, int nchunks,
                   const int32_t* __restrict__ colx, const double* __restrict__ vals,
                   const longlong2* __restrict__ key_in, Act* __restrict__ partial) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nchunks) return;
  const LongChunk ch = chunks[w];
  Act acc = {0.0, 0.0, 0, 0};
  for (int base = ch.k0; base < ch.k1; base += 32) {
    const int k = base + lane;
    double pmin = 0.0, pmax = 0.0;
    if (k < ch.k1) {
      const int32_t c = __ldg(colx + k);
      const double a = __ldg(vals + k);
      const longlong2 kk = ld_key(key_in + (c & 0x7fffffff));
      contrib(a, key_dec(kk.x), key_dec(kk.y), pmin, pmax);
    }
    const int cnt = min(32, ch.k1 - base);
    for (int s = 0; s < cnt; ++s) {
      const double vmin = __shfl_sync(0xffffffffu, pmin, s);
      const double vmax = __shfl_sync(0xffffffffu, pmax, s);
      act_add(acc, vmin, vmax);
    }
  }
  if (lane == 0) partial[w] = acc;
}

// Pairwise tree over a long row's chunk partials in index order
// (par_engine.cpp:117-121); optional Step-2 row check.
template <bool kRowCheck>
__global__ void k_long_combine(const int32_t* __restrict__ long_rows,
                               const int32_t* __restrict__ long_first_chunk, int nlong,
                               Act* __restrict__ partial, Act* __restrict__ long_act,
                               const double* __restrict__ lhs, const double* __restrict__ rhs,
                               DevState* __restrict__ st, const DevCfg cfg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nlong) return;
  Act* P = partial + long_first_chunk[s];
  int np = long_first_chunk[s + 1] - long_first_chunk[s];
  while (np > 1) {
    int out = 0;
    for (int i = 0; i + 1 < np; i += 2) P[out++] = act_combine(P[i], P[i + 1]);
    if (np & 1) P[out++] = P[np - 1];
    np = out;
  }
  const Act act = P[0];
  long_act[s] = act;
  if (kRowCheck) {
    const int row = long_rows[s];
    if (row_infeasible(act, lhs[row], rhs[row], cfg)) st->infeasible = 1;
  }
}

__global__ void __launch_bounds__(256)
    k_long_cand(const LongChunk* __restrict__ chunks, const int32_t* __restrict__ long_rows,
                const Act* __restrict__ long_act, const int32_t* __restrict__ colx,
                const double* __restrict__ vals, const double* __restrict__ lhs,
                const double* __restrict__ rhs, const longlong2* __restrict__ key_in,
                long long* __restrict__ key_out, DevState* __restrict__ st, const DevCfg cfg) {
  __shared__ int32_t s_inf;
  const LongChunk ch = chunks[blockIdx.x];
  if (threadIdx.x == 0) s_inf = 0;
  __syncthreads();
  const Act act = long_act[ch.slot];
  const int row = long_rows[ch.slot];
  const double l = lhs[row], h = rhs[row];
  for (int k = ch.k0 + threadIdx.x; k < ch.k1; k += blockDim.x) {
    const int32_t c = __ldg(colx + k);
    const double a = __ldg(vals + k);
    const longlong2 kk = ld_key(key_in + (c & 0x7fffffff));
    const double lo = key_dec(kk.x), up = key_dec(kk.y);
    double min_res, max_res, cl, cu;
    residual(act, a, lo, up, min_res, max_res);
    candidates(a, l, h, min_res, max_res, c < 0, cfg, cl, cu);
    const int kind = tighten(lo, up, cl, cu, cfg);
    if (kind == 4) s_inf = 1;
    else if (kind) commit_side(key_out, c & 0x7fffffff, kind, cl, cu);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_inf) st->infeasible = 1;
}

// ---- commit + round decision --------------------------------------------------
template <int kThreads>
__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, int* flag_or,
                                                        int& f) {
  __shared__ unsigned long long s_sum[kThreads / 32];
  __shared__ int s_f[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    f |= __shfl_xor_sync(0xffffffffu, f, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_sum[w] = v;
    s_f[w] = f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    int ff = 0;
    for (int i = 0; i < kThreads / 32; ++i) {
      t += s_sum[i];
      ff |= s_f[i];
    }
    v = t;
    f = ff;
  }
  (void)flag_or;
  return v;
}

__global__ void __launch_bounds__(kCommitThreads)
    k_commit(longlong2* __restrict__ key_in, const longlong2* __restrict__ key_out, int n,
             DevState* __restrict__ st, long long* __restrict__ per_round, const DevCfg cfg,
             cudaGraphConditionalHandle cond, int use_graph) {
  unsigned long long changes = 0;
  int inf = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const longlong2 ki = key_in[j];
    const longlong2 ko = key_out[j];
    const int c = (ki.x != ko.x) + (ki.y != ko.y);
    if (c) {
      changes += c;
      key_in[j] = ko;
    }
    if (key_dec(ko.x) > __dadd_rn(key_dec(ko.y), cfg.imp_abs)) inf = 1;
  }
  changes = block_sum<kCommitThreads>(changes, nullptr, inf);
  if (threadIdx.x == 0) {
    if (changes) atomicAdd(&st->round_changes, changes);
    if (inf) st->infeasible = 1;
    __threadfence();
    const uint32_t t = atomicAdd(&st->ticket, 1u);
    if (t == gridDim.x - 1) {
      // last CTA: the round decision of run_parallel (par_engine.cpp:248-266)
      __threadfence();
      const long long ch = (long long)atomicAdd(&st->round_changes, 0ull);
      const int infeasible = atomicAdd(&st->infeasible, 0);
      const int r = st->round + 1;
      st->round = r;
      if (r - 1 < cfg.round_limit) per_round[r - 1] = ch;
      st->total_changes += ch;
      int status = -1;
      if (infeasible) status = 2;             // PG_INFEASIBLE
      else if (ch == 0) status = 0;           // PG_CONVERGED
      else if (r >= cfg.round_limit) status = 1;  // PG_ROUNDLIMIT
      st->status = status;
      st->done = status >= 0;
      st->round_changes = 0;
      st->infeasible = 0;
      st->ticket = 0;
      __threadfence();
      if (use_graph) cudaGraphSetConditional(cond, status >= 0 ? 0u : 1u);
    }
  }
}

// Start of a solve: keys from the (normalised) start bounds, state reset,
// bounds_crossed pre-check (engine_common.hpp:51-58).
__global__ void __launch_bounds__(kCommitThreads)
    k_reset(const double* __restrict__ lo0, const double* __restrict__ up0,
            longlong2* __restrict__ key_in, longlong2* __restrict__ key_out, int n,
            DevState* __restrict__ st, const DevCfg cfg, int check_crossed,
            cudaGraphConditionalHandle cond, int use_graph) {
  int crossed = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double l = lo0[j], u = up0[j];
    const longlong2 k = make_longlong2(key_enc(l), key_enc(u));
    key_in[j] = k;
    key_out[j] = k;
    if (l > __dadd_rn(u, cfg.imp_abs)) crossed = 1;
  }
  unsigned long long dummy = 0;
  block_sum<kCommitThreads>(dummy, nullptr, crossed);
  if (threadIdx.x == 0) {
    if (crossed) atomicOr(&st->crossed, 1);
    __threadfence();
    const uint32_t t = atomicAdd(&st->ticket_reset, 1u);
    if (t == gridDim.x - 1) {
      __threadfence();
      const int cr = check_crossed && atomicAdd(&st->crossed, 0);
      st->round_changes = 0;
      st->total_changes = 0;
      st->infeasible = 0;
      st->round = 0;
      st->status = cr ? 2 : -1;
      st->done = cr;
      st->ticket = 0;
      st->crossed = 0;
      st->ticket_reset = 0;
      __threadfence();
      if (use_graph) cudaGraphSetConditional(cond, cr ? 0u : 1u);
    }
  }
}

// keys -> doubles (result download)
__global__ void k_decode(const longlong2* __restrict__ key, double* __restrict__ lo,
                         double* __restrict__ up, int n) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const longlong2 k = key[j];
    lo[j] = key_dec(k.x);
    up[j] = key_dec(k.y);
  }
}

// |v| >= threshold -> +-inf (model.hpp:147-151), in place
__global__ void k_normalize(double* __restrict__ v, int n, double thr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = v[i];
    v[i] = x >= thr ? CUDART_INF : (x <= -thr ? -CUDART_INF : x);
  }
}

// integrality packed into bit 31 of the column index: no per-entry byte gather
__global__ void k_pack_cols(int32_t* __restrict__ colx, const uint8_t* __restrict__ integral,
                            long long nnz) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x) {
    const int32_t c = colx[k];
    colx[k] = integral[c] ? (int32_t)(c | 0x80000000u) : c;
  }
}

}  // namespace pgb
