// cand.cuh -- phase 2 of a round: candidates of the rows that may tighten.
//
// process_block's per-nonzero loop (par_engine.cpp:148-169):
// residual_activities -> compute_bound_candidates -> tighten against the
// round's input bounds -> merge (propcore.hpp:78-208, par_engine.cpp:56-71),
// for the rows phase 1 queued.  Work is spread over lanes by ENTRY, not by
// row, so a long row keeps a whole warp busy and a batch of short rows
// shares one:
//   * long queue: pieces of <= kCandPiece entries of one row, one warp each,
//     lanes over consecutive entries (coalesced CSR loads, 4 in flight per
//     lane);
//   * short queue: 32 rows of <= kCandShort entries per warp, their entries
//     flattened over the lanes (row found by a binary search over the
//     batch's prefix sums in shared memory).
// Every entry goes through the exactness-preserving filter (kernels.cuh);
// the survivors are compacted into a per-warp queue and run through the
// exact pipeline 32 at a time, so the expensive, branchy part is SIMT-dense.
#pragma once

#include "kernels.cuh"

namespace pgb {

constexpr int kCandThreads = 256;
constexpr int kCandWarps = kCandThreads / 32;
constexpr int kCandUnroll = 4;

struct CandWarpSmem {
  // per batch row (short queue) or the single row (long queue, slot 0)
  double min_f[32], max_f[32], lhs[32], rhs[32], tr[32], tl[32];
  int32_t min_i[32], max_i[32], start[33], k0[32];
  uint8_t mode[32];
  // surviving entries
  double qa[64], qlo[64], qup[64];
  int32_t qc[64];
  uint8_t qr[64];
};

__device__ __forceinline__ void cand_row_load(const RoundArgs& A, CandWarpSmem& W, int slot, int r) {
  const Act act = A.ract[r];
  const double l = A.lhs[r], h = A.rhs[r];
  const RowFilter f = row_filter(act, l, h);
  W.min_f[slot] = act.min_f;
  W.max_f[slot] = act.max_f;
  W.min_i[slot] = act.min_i;
  W.max_i[slot] = act.max_i;
  W.lhs[slot] = l;
  W.rhs[slot] = h;
  W.tr[slot] = f.tr;
  W.tl[slot] = f.tl;
  W.mode[slot] = f.mode;
}

// run the exact pipeline over queue entries [0, cnt), one per lane
__device__ __forceinline__ bool cand_drain(const CandWarpSmem& W, int cnt, int lane,
                                           long long* key_out, const DevCfg& cfg,
                                           const Touch* touch = nullptr) {
  bool inf_flag = false;
  if (lane < cnt) {
    const int r = W.qr[lane];
    const Act act = {W.min_f[r], W.max_f[r], W.min_i[r], W.max_i[r]};
    inf_flag = entry_pipeline(act, W.qa[lane], W.qlo[lane], W.qup[lane], W.lhs[r], W.rhs[r],
                              W.qc[lane], key_out, cfg, touch);
  }
  return inf_flag;
}

// append this lane's surviving entry (if any); drain full batches of 32
__device__ __forceinline__ void cand_push(CandWarpSmem& W, int& qn, bool pass, double a,
                                          double lo, double up, int32_t c, int slot, int lane,
                                          bool& inf_flag, long long* key_out, const DevCfg& cfg,
                                          const Touch* touch) {
  const unsigned m = __ballot_sync(0xffffffffu, pass);
  if (!m) return;
  if (pass) {
    const int k = qn + __popc(m & ((1u << lane) - 1u));
    W.qa[k] = a;
    W.qlo[k] = lo;
    W.qup[k] = up;
    W.qc[k] = c;
    W.qr[k] = (uint8_t)slot;
  }
  qn += __popc(m);
  if (qn >= 32) {
    __syncwarp();
    inf_flag |= cand_drain(W, 32, lane, key_out, cfg, touch);
    __syncwarp();
    qn -= 32;
    if (lane < qn) {
      W.qa[lane] = W.qa[32 + lane];
      W.qlo[lane] = W.qlo[32 + lane];
      W.qup[lane] = W.qup[32 + lane];
      W.qc[lane] = W.qc[32 + lane];
      W.qr[lane] = W.qr[32 + lane];
    }
    __syncwarp();
  }
}

// entry k of the row in slot `slot`: gather, filter
template <class RA>
__device__ __forceinline__ bool cand_entry(const RA& A, const CandWarpSmem& W, int slot,
                                           int k, double& a, double& lo, double& up, int32_t& c) {
  a = __ldg(A.vals + k);
  c = __ldg(A.colx + k);
  double q;
  if constexpr (coherent_v<RA>)
    ld_snap_coh(A.snap + (c & 0x7fffffff), lo, up, q);
  else
    ld_snap(A.snap + (c & 0x7fffffff), lo, up, q);
  const double bmin = a > 0 ? lo : up;
  const double bmax = a > 0 ? up : lo;
  const RowFilter f = {W.tr[slot], W.tl[slot], W.mode[slot]};
  return entry_may(f, fabs(a) * q, isinf(bmin), isinf(bmax));
}

template <class RA>
__device__ __forceinline__ void cand_sweep(const RA& A, const DevCfg& cfg,
                                           CandWarpSmem* smem) {
  const int lane = threadIdx.x & 31;
  CandWarpSmem& W = smem[threadIdx.x >> 5];
  const int nlong = ld_gpu(&A.st->wl_long);
  const int nshort = ld_gpu(&A.st->wl_short);
  const int nbatch = (nshort + 31) / 32;
  const Touch* touch = A.dirty.enabled && ld_gpu(&A.st->sparse_round) ? &A.touch : nullptr;
  bool inf_flag = false;
  for (;;) {
    int t = 0;
    if (lane == 0) t = ticket(&A.st->cand_work);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= nlong + nbatch) break;
    int qn = 0;
    if (t < nlong) {
      // one piece of a long row
      const CandItem it = A.wl_long[t];
      if (lane == 0) cand_row_load(A, W, 0, it.row);
      __syncwarp();
      for (int e0 = 0; e0 < it.len; e0 += 32 * kCandUnroll) {
        double a[kCandUnroll], lo[kCandUnroll], up[kCandUnroll];
        int32_t c[kCandUnroll];
        bool pass[kCandUnroll];
#pragma unroll
        for (int u = 0; u < kCandUnroll; ++u) {
          const int e = e0 + 32 * u + lane;
          pass[u] = e < it.len && cand_entry(A, W, 0, it.k0 + e, a[u], lo[u], up[u], c[u]);
        }
#pragma unroll
        for (int u = 0; u < kCandUnroll; ++u)
          cand_push(W, qn, pass[u], a[u], lo[u], up[u], c[u], 0, lane, inf_flag, A.key_out, cfg, touch);
      }
    } else {
      // a batch of up to 32 short rows, entries flattened over the lanes
      const int b = t - nlong;
      const int i = 32 * b + lane;
      int len = 0;
      if (i < nshort) {
        const int r = A.wl_short[i];
        cand_row_load(A, W, lane, r);
        const int k0 = A.row_ptr[r];
        len = A.row_ptr[r + 1] - k0;
        W.k0[lane] = k0;
      }
      int incl = len;  // inclusive warp scan of the lengths
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      W.start[lane + 1] = incl;
      if (lane == 0) W.start[0] = 0;
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      __syncwarp();
      for (int e0 = 0; e0 < total; e0 += 32 * kCandUnroll) {
        double a[kCandUnroll], lo[kCandUnroll], up[kCandUnroll];
        int32_t c[kCandUnroll];
        bool pass[kCandUnroll];
        int slot[kCandUnroll];
#pragma unroll
        for (int u = 0; u < kCandUnroll; ++u) {
          const int e = e0 + 32 * u + lane;
          pass[u] = false;
          slot[u] = 0;
          if (e < total) {
            // last slot whose start <= e
            int lo_s = 0, hi_s = 31;
            while (lo_s < hi_s) {
              const int mid = (lo_s + hi_s + 1) >> 1;
              if (W.start[mid] <= e) lo_s = mid; else hi_s = mid - 1;
            }
            slot[u] = lo_s;
            pass[u] = cand_entry(A, W, lo_s, W.k0[lo_s] + (e - W.start[lo_s]), a[u], lo[u], up[u],
                                 c[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < kCandUnroll; ++u)
          cand_push(W, qn, pass[u], a[u], lo[u], up[u], c[u], slot[u], lane, inf_flag, A.key_out,
                    cfg, touch);
      }
    }
    if (qn) {
      __syncwarp();
      inf_flag |= cand_drain(W, qn, lane, A.key_out, cfg, touch);
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, inf_flag) && lane == 0) A.st->infeasible = 1;
}

__global__ void __launch_bounds__(kCandThreads) k_cand(const RoundArgs A, const DevCfg cfg) {
  __shared__ CandWarpSmem smem[kCandWarps];
  pdl_begin();
  if (compute_off(A.st, cfg)) return;
  cand_sweep(A, cfg, smem);
}

}  // namespace pgb
