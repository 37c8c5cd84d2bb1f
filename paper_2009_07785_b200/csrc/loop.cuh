// loop.cuh -- the whole round loop in one persistent kernel.
//
// For instances whose rounds are latency-bound (small matrices, and the
// sparse worklist rounds of branch-and-bound nodes) three or four launches
// per round cost more than the round itself.  k_loop runs run_parallel's
// loop (par_engine.cpp:228-267) inside one cooperative launch: every CTA is
// resident, and the phases of a round -- chains (sell.cuh), split-row
// candidates (cand.cuh), commit + decision, worklist marks -- are separated
// by grid barriers instead of kernel boundaries.  The phase bodies are the
// same device functions the per-phase kernels run, so results are identical.
#pragma once

#include "cand.cuh"
#include "sell.cuh"

namespace pgb {

// sense-free generation barrier over all CTAs of a cooperative launch
__device__ __forceinline__ void grid_barrier(DevState* st) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t* gen = &st->bar_gen;
    const uint32_t g = ld_gpu(gen);
    __threadfence();
    if (atomicAdd(&st->bar_count, 1u) == gridDim.x - 1) {
      st->bar_count = 0;
      __threadfence();
      atomicAdd(&st->bar_gen, 1u);
    } else {
      while (ld_gpu(gen) == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

union LoopSmem {
  SellWarpSmem sell[kSellWarps];
  CandWarpSmem cand[kCandWarps];
  SplitSmem<64> split[kSellWarps];
};

template <bool kRowCheck>
__global__ void __launch_bounds__(kSellThreads, PG_SELL_MINB)
    k_loop(const RoundArgsL A, const DevCfg cfg, Snap* __restrict__ snap, int n,
           long long* __restrict__ per_round, const int32_t* __restrict__ split, int nsplit) {
  extern __shared__ __align__(16) unsigned char loop_dyn[];  // LoopSmem
  LoopSmem& sm = *reinterpret_cast<LoopSmem*>(loop_dyn);
  longlong2* key_out = reinterpret_cast<longlong2*>(A.key_out);
  while (!ld_gpu(&A.st->done)) {
    const bool sparse = round_is_sparse(A.st, A.dirty);  // the round's kind, before any phase
    if (blockIdx.x == 0 && threadIdx.x == 0) A.st->sparse_round = sparse ? 1 : 0;  // for cand_sweep
    if (!sparse)
      sell_sweep<kRowCheck, true>(A, cfg, sm.sell);
    else
      sell_sweep<kRowCheck, false>(A, cfg, sm.sell);
    grid_barrier(A.st);
    if (nsplit) {
      split_finish_body<kRowCheck, 64>(A, split, nsplit, sm.split, cfg);
      grid_barrier(A.st);
    }
    // phase 2 of split rows: pieces of long rows AND batches of short split
    // rows (a row of nnz_budget < len <= kCandShort entries, nnz_budget < 32)
    if (ld_gpu(&A.st->wl_long) || ld_gpu(&A.st->wl_short)) {
      cand_sweep(A, cfg, sm.cand);
      grid_barrier(A.st);
    }
    if (sparse)
      commit_body<true>(snap, const_cast<double2*>(A.bnd), key_out, n, A.st, per_round, cfg, A.dirty,
                        0, 0, &A.touch);
    else
      commit_body(snap, const_cast<double2*>(A.bnd), key_out, n, A.st, per_round, cfg, A.dirty, 0, 0);
    grid_barrier(A.st);
    if (A.dirty.enabled) {
      mark_body(A.dirty, A.st);
      grid_barrier(A.st);
    }
  }
}

}  // namespace pgb
