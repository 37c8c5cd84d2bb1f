// split.cuh -- rows longer than nnz_budget: combine the chunk partials.
//
// wide_row_activities (par_engine.cpp:99-123): a row longer than
// nnz_budget is summed in nnz_budget chunks (one chain each, sell.cuh), and
// the chunk records are combined pairwise in index order, level by level,
// an odd last record carried up unpaired.  After the round's sweep, one
// warp per split row whose chunks all ran (row_done == chunks) loads the
// partials into shared memory and runs that tree level by level (lane i
// forms record i of the next level), then the row finish (row check, filter,
// queueing for k_cand).  All partial loads of a level are independent, so a
// row of P chunks costs ~log2(P) dependent steps instead of P.
#pragma once

#include "kernels.cuh"

namespace pgb {

constexpr int kSplitWarps = 4;

// per warp: two levels of up to MAXP partials
template <int MAXP>
struct SplitSmem {
  Act buf[2][MAXP];
};

template <bool kRowCheck, int MAXP>
__device__ __forceinline__ void split_finish_body(const RoundArgs& A, const int32_t* split,
                                                  int nsplit, SplitSmem<MAXP>* smem,
                                                  const DevCfg& cfg) {
  const int lane = threadIdx.x & 31;
  SplitSmem<MAXP>& S = smem[threadIdx.x >> 5];
  bool inf_flag = false;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int w = gw; w < nsplit; w += nw) {
    const int rs = split[w];
    const int first = A.sfirst[rs];
    const int np = A.sfirst[rs + 1] - first;
    if (ld_gpu(&A.row_done[rs]) != np) continue;  // not all chunks ran
    __syncwarp();
    if (lane == 0) A.row_done[rs] = 0;
    if (np > MAXP) {
      if (lane == 0) finish_split_row<kRowCheck>(A, rs, inf_flag, cfg);
      continue;
    }
    const SegPartial* P = A.partial + first;
    double xmax = -CUDART_INF;
    for (int i = lane; i < np; i += 32) {
      const SegPartial p = P[i];
      S.buf[0][i] = Act{p.min_f, p.max_f, p.min_i, p.max_i};
      xmax = fmax(xmax, p.xmax);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) xmax = fmax(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
    __syncwarp();
    int n = np, src = 0;
    while (n > 1) {
      const int out = (n + 1) >> 1;
      for (int i = lane; i < out; i += 32)
        S.buf[src ^ 1][i] =
            2 * i + 1 < n ? act_combine(S.buf[src][2 * i], S.buf[src][2 * i + 1]) : S.buf[src][2 * i];
      __syncwarp();
      src ^= 1;
      n = out;
    }
    if (lane == 0) finish_row<kRowCheck>(A, A.srow[rs], S.buf[src][0], xmax, inf_flag, cfg);
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
}

template <bool kRowCheck>
__global__ void __launch_bounds__(kSplitWarps * 32) k_split_finish(const RoundArgs A,
                                                                   const int32_t* split, int nsplit,
                                                                   const DevCfg cfg) {
  __shared__ SplitSmem<256> smem[kSplitWarps];
  pdl_begin();
  if (compute_off(A.st, cfg)) return;
  split_finish_body<kRowCheck, 256>(A, split, nsplit, smem, cfg);
}

// split-row slots (rows with more than one chunk), for k_split_finish
__global__ void k_split_list(const int32_t* __restrict__ sfirst, int nsrow,
                             int32_t* __restrict__ list, int32_t* __restrict__ count) {
  for (int rs = blockIdx.x * blockDim.x + threadIdx.x; rs < nsrow; rs += gridDim.x * blockDim.x)
    if (sfirst[rs + 1] - sfirst[rs] > 1) list[atomicAdd(count, 1)] = rs;
}

}  // namespace pgb
