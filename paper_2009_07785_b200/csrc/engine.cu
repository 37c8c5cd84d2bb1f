// engine.cu -- host side of the B200 propagation engine and the C-ABI
// (include/propgate_b200.h).
//
// Session = one problem resident in HBM:
//   row_ptr  int32[m+1]     col  int32[nnz] (bit 31 = integral flag)
//   vals     f64[nnz]       lhs/rhs f64[m] (normalised to +-inf)
//   snap     Snap[n]        32 B snapshot record {lo, up, q, flags} per column
//   key_out  {i64,i64}[n]   merge target of the round (atomicMax/atomicMin on
//                           ordered-bits keys)
//   lo0/up0  f64[n]         normalised start bounds
// Rows are stored sorted by length.  Short rows (<= min(16, nnz_budget)
// entries) form warp tiles; longer rows are split into segments of
// nnz_budget entries (the chunks of cpu_par's wide-row sums).
//
// The round loop (par_engine.cpp:228-267) runs on the device: a CUDA graph
//   k_reset -> WHILE(cond) { k_round, k_seg_cand, k_commit }
// where k_commit's last CTA writes per_round_changes[r] and clears `cond`
// on Infeasible / Converged / RoundLimit.  One graph launch per solve; no
// host synchronisation per round.
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <cstdlib>
#include <limits>
#include <atomic>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/propgate_b200.h"
#include <cub/device/device_scan.cuh>

#include <cub/device/device_radix_sort.cuh>

#include "kernels.cuh"
#include "setup.cuh"
#include "sell.cuh"
#include "cand.cuh"
#include "loop.cuh"
#include "nodes.cuh"
#include "narrow.cuh"
#include "narrow_sell.cuh"
#include "ingest.cuh"
#include "mps_reader.h"

using namespace pgb;

namespace {

thread_local std::string g_err;

struct Error {
  int code;
  std::string msg;
};

#define PG_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw Error{e_ == cudaErrorMemoryAllocation ? PG_ENOMEM : PG_ECUDA,               \
                  std::string(#call) + ": " + cudaGetErrorString(e_)};                   \
  } while (0)

// Device memory comes from the device's stream-ordered pool with an infinite
// release threshold: repeated sessions (one-shot pg_propagate calls, B&B
// sessions) reuse it instead of paying cudaMalloc / cudaFree each time.
thread_local cudaStream_t t_alloc_stream = nullptr;
template <typename T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  PG_CUDA(cudaMallocAsync(&p, count * sizeof(T), t_alloc_stream));
  return static_cast<T*>(p);
}
inline void dfree(void* p) {
  if (p) cudaFreeAsync(p, t_alloc_stream);
}

// per-device properties, queried once (cudaGetDeviceProperties costs ms)
struct DevInfo {
  bool ok = false;
  int major = 0, minor = 0, sms = 0;
  std::string name;
};
DevInfo device_info(int dev) {
  static DevInfo cache[64];
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) return DevInfo{};
  if (!cache[dev].ok) {
    cudaDeviceProp prop;
    PG_CUDA(cudaGetDeviceProperties(&prop, dev));
    cache[dev] = DevInfo{true, prop.major, prop.minor, prop.multiProcessorCount, prop.name};
    cudaMemPool_t pool;
    PG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    PG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  return cache[dev];
}

int validate(const pg_config* c) {
  // EngineConfig::validate (core/src/model.cpp:21-35), same messages
  const char* m = nullptr;
  if (c->round_limit < 1) m = "round_limit must be >= 1";
  else if (!(c->infinity_threshold > 0)) m = "infinity_threshold must be positive";
  else if (!(c->improvement_abs > 0) || !(c->improvement_rel > 0))
    m = "improvement tolerances must be positive";
  else if (!(c->integrality_eps > 0)) m = "integrality_eps must be positive";
  else if (c->vector_threshold < 1) m = "vector_threshold must be >= 1";
  else if (c->nnz_budget < c->vector_threshold) m = "nnz_budget must be >= vector_threshold";
  else if (c->worker_count < 0) m = "worker_count must be >= 0";
  else if (c->scalar_mode != PG_WIDE64 && c->scalar_mode != PG_NARROW32)
    m = "scalar_mode must be Wide64 or Narrow32";
  else if (c->loop_mode != PG_LOOP_GRAPH && c->loop_mode != PG_LOOP_HOST)
    m = "loop_mode must be PG_LOOP_GRAPH or PG_LOOP_HOST";
  if (m) {
    g_err = m;
    return PG_EINVAL;
  }
  return PG_OK;
}

void check_problem(const pg_problem* p) {
  if (!p) throw Error{PG_EINVAL, "problem is NULL"};
  if (p->num_rows < 0 || p->num_cols < 0 || p->nnz < 0)
    throw Error{PG_EINVAL, "negative problem dimensions"};
  if (p->nnz > 0x7fffffffLL) throw Error{PG_EINVAL, "nnz exceeds int32 (reference uses int32 indices)"};
  if (!p->row_ptr || (p->num_rows && (!p->lhs || !p->rhs)) ||
      (p->num_cols && (!p->lower || !p->upper || !p->integral)) ||
      (p->nnz && (!p->col_idx || !p->values)))
    throw Error{PG_EINVAL, "problem array is NULL"};
  if (p->row_ptr[0] != 0 || p->row_ptr[p->num_rows] != p->nnz)
    throw Error{PG_EINVAL, "row_ptr must start at 0 and end at nnz"};
}

// PG_TIMING=1: phase times of session setup on stderr (e2e diagnostics)
struct PhaseTimer {
  bool on = getenv("PG_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[pg] %-24s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// PG_TIMING: device-side timeline of a one-shot call (events on the
// streams named at each mark), printed relative to the first mark
struct GpuTrace {
  bool on = getenv("PG_TIMING") != nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  void mark(const char* what, cudaStream_t q) {
    if (!on) return;
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, q);
    ev.emplace_back(what, e);
  }
  void dump() {
    if (!on || ev.empty()) return;
    for (auto& x : ev) {
      cudaEventSynchronize(x.second);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0].second, x.second);
      fprintf(stderr, "[pg gpu] %-28s %8.3f ms\n", x.first, ms);
    }
    for (auto& x : ev) cudaEventDestroy(x.second);
    ev.clear();
  }
};
thread_local GpuTrace g_trace;

// NCCL, loaded on first use (the single-GPU engine has no NCCL dependency).
// Values from nccl.h: ncclInt64 = 4, ncclMax = 2; ncclUniqueId = 128 bytes.
constexpr int kNcclInt64 = 4;
constexpr int kNcclMax = 2;
constexpr int kNcclInt32 = 2;
struct NcclUid {
  char internal[128];
};
struct Nccl {
  void* h = nullptr;
  int (*get_unique_id)(NcclUid*) = nullptr;
  int (*comm_init_rank)(void**, int, NcclUid, int) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*comm_abort)(void*) = nullptr;
  int (*all_reduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*all_gather_fn)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
  bool load() {
    if (h) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    get_unique_id = (int (*)(NcclUid*))dlsym(h, "ncclGetUniqueId");
    comm_init_rank = (int (*)(void**, int, NcclUid, int))dlsym(h, "ncclCommInitRank");
    comm_destroy = (int (*)(void*))dlsym(h, "ncclCommDestroy");
    comm_abort = (int (*)(void*))dlsym(h, "ncclCommAbort");
    all_reduce_fn = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
        h, "ncclAllReduce");
    all_gather_fn = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(
        h, "ncclAllGather");
    error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    return get_unique_id && comm_init_rank && comm_destroy && all_reduce_fn && all_gather_fn;
  }
  int all_reduce(const void* s, void* r, size_t count, int dt, int op, void* comm,
                 cudaStream_t st) const {
    return all_reduce_fn(s, r, count, dt, op, comm, st);
  }
  const char* error(int rc) const { return error_string ? error_string(rc) : "nccl error"; }
};
Nccl g_nccl;

}  // namespace

// Streams and events of finished sessions, kept per device for the next
// session (creating them costs ~0.1 ms per one-shot call).  Pending
// stream-ordered work on a returned stream simply precedes the next user's.
// The set also carries the session's pinned DevState mirror: cudaFreeHost
// synchronises the whole device, so a one-shot call's reaper freeing it
// would stall the next call's setup behind its own upload.
struct StreamSet {
  cudaStream_t st = nullptr, st2 = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, fork = nullptr, join = nullptr;
  DevState* h_st = nullptr;  // pinned
};
struct StreamPool {
  std::mutex mu;
  std::vector<StreamSet> free_sets[64];
  StreamSet get(int dev) {  // the caller has made `dev` current
    {
      std::lock_guard<std::mutex> lk(mu);
      if (dev >= 0 && dev < 64 && !free_sets[dev].empty()) {
        const StreamSet x = free_sets[dev].back();
        free_sets[dev].pop_back();
        return x;
      }
    }
    StreamSet x;
    PG_CUDA(cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking));
    PG_CUDA(cudaStreamCreateWithFlags(&x.st2, cudaStreamNonBlocking));
    PG_CUDA(cudaEventCreate(&x.ev0));
    PG_CUDA(cudaEventCreate(&x.ev1));
    PG_CUDA(cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming));
    PG_CUDA(cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming));
    PG_CUDA(cudaMallocHost(&x.h_st, sizeof(DevState)));
    return x;
  }
  void put(int dev, const StreamSet& x) {
    {
      std::lock_guard<std::mutex> lk(mu);
      if (dev >= 0 && dev < 64 && free_sets[dev].size() < 4 && x.st && x.st2 && x.ev0 && x.ev1 &&
          x.fork && x.join && x.h_st) {
        free_sets[dev].push_back(x);
        return;
      }
    }
    for (cudaEvent_t e : {x.ev0, x.ev1, x.fork, x.join})
      if (e) cudaEventDestroy(e);
    for (cudaStream_t q : {x.st, x.st2})
      if (q) cudaStreamDestroy(q);
    if (x.h_st) cudaFreeHost(x.h_st);
  }
  static StreamPool& get() {
    static StreamPool* p = new StreamPool;  // never destroyed (reaper thread)
    return *p;
  }
};

struct pg_session {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int32_t m = 0, n = 0;
  int64_t nnz = 0;
  pg_config cfg{};
  DevCfg dcfg{};
  int num_sms = 148;
  int sell_per_sm = 1;   // resident k_sell CTAs per SM
  int sell_dense_per_sm = 1;  // the same for the full sweep (less shared memory)
  int cand_per_sm = 1;   // resident k_cand CTAs per SM
  int loop_grid = 0;     // co-resident CTAs of the persistent loop kernel
  int nodes_per_sm = 1;  // resident k_nodes CTAs per SM
  int32_t max_row_len = -1;  // lazily: max_len()
  ActF* d_f32_part = nullptr;  // Narrow32: per-thread chunk partials (k_round_f32)
  ActF* d_ractf = nullptr;     // Narrow32 over the sliced-ELL copy: row records
  ActF* d_partf = nullptr;     //   and chunk partials (narrow_sell.cuh)
  int f32_maxc = 1;

  // device arrays
  int32_t* d_row_ptr = nullptr;
  int32_t* d_colx = nullptr;
  double* d_vals = nullptr;
  double* d_lhs = nullptr;
  double* d_rhs = nullptr;
  Snap* d_snap = nullptr;
  double2* d_bnd = nullptr;  // compact {lb, ub} records (sell.cuh gathers)
  float2* d_bf = nullptr;    // float {lb, ub} records (DevCfg::bf), when the bounds are floats
  uint8_t* d_integral = nullptr;
  int32_t* d_row_done = nullptr;
  longlong2* d_key_out = nullptr;
  double* d_lo0 = nullptr;
  double* d_up0 = nullptr;
  double* d_lo_res = nullptr;
  double* d_up_res = nullptr;
  SegDesc* d_segs = nullptr;
  int32_t* d_srow = nullptr;
  int32_t* d_sfirst = nullptr;
  SegPartial* d_partial = nullptr;
  Act* d_ract = nullptr;           // phase-2 queues
  int32_t* d_wl_short = nullptr;
  CandItem* d_wl_long = nullptr;
  // sliced-ELL copy of the matrix (sell.cuh)
  UnitDesc* d_units = nullptr;
  SliceDesc* d_slices = nullptr;
  double* d_sv = nullptr;
  int32_t* d_sc = nullptr;
  uint32_t* d_sw = nullptr;
  int32_t nunits = 0, nslices = 0, lg_min = 0, group_start = 0, lg0_ustart = 0, lg0_sstart = 0;
  int64_t sell_elems = 0;
  DevState* d_st = nullptr;
  long long* d_per_round = nullptr;
  // worklist index and dirty sets
  int32_t* d_col_ptr = nullptr;
  int32_t* d_col_item = nullptr;
  uint8_t* d_flags = nullptr;  // row marks, two buffers
  int32_t* d_chg = nullptr;    // changed-column lists, two buffers
  int32_t *d_row_unit = nullptr, *d_part_unit = nullptr, *d_unit_slice = nullptr;
  int32_t* d_wide_list = nullptr;
  int32_t* d_unit_list = nullptr;
  Dirty dirty{};
  Touch touch{};           // worklist rounds: merged-into columns
  uint32_t* d_tflag = nullptr;
  int32_t* d_tlist = nullptr;

  // host mirrors
  DevState* h_st = nullptr;  // pinned
  int32_t nseg = 0, nsrow = 0, nsplit = 0;
  int32_t* d_split = nullptr;  // split-row slots (k_split_finish)
  int64_t short_rows = 0, short_nnz = 0, seg_nnz = 0, wl_long_cap = 0;

  // graph
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t stream2 = nullptr;  // session setup: ordering overlapped with the upload
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void* comm = nullptr;  // NCCL communicator of the row-sharded mode
  std::atomic<bool> comm_aborted{false};  // another rank failed: the communicator was aborted
  int32_t rank = 0, world = 1;
  // sum(len^2) / (n nnz): how often consecutive entries of a row hit
  // neighbouring columns; dense rows gather the 16 B bounds records (two per
  // sector), sparse ones the 32 B snapshot records (filter coefficient q
  // precomputed, no per-entry recompute) when those fit in L2 beside the
  // streamed matrix
  double row_density = 0.0;
  // the 32 B records must also stay L2-resident next to the streamed matrix
  // (C5: 5M columns = 160 MB of snapshot records, 80 MB of bounds records)
  bool many_cols() const { return (double)n * sizeof(Snap) > 48e6; }
  // gather record of the round kernels (RoundArgsG): 0 = 32 B snapshot
  // records, 1 = 16 B bounds, 2 = 8 B float bounds (d_bf, kept when the
  // sampled start bounds are floats of integral columns, whose tightened
  // bounds stay integers; a bound that is not a float falls back to its
  // 16 B record, so the choice is a matter of speed only)
  int gather_kind() const {
    static const char* e = getenv("PG_SELL_GATHER");
    if (e) return atoi(e) == 8 && d_bf ? 2 : atoi(e) == 16 ? 1 : 0;
    if (many_cols() && d_bf) return 2;
    return row_density > 0.05 || many_cols() ? 1 : 0;
  }
  bool gather16() const { return gather_kind() != 0; }
  // sparse delta exchange (PG_FLAG_DELTA_EXCHANGE): this rank's items, every
  // rank's items, counts; rounds of the last solve that used it
  DeltaItem* d_delta = nullptr;
  DeltaItem* d_delta_all = nullptr;
  int* d_dcnt = nullptr;
  int* d_dcnt_all = nullptr;
  int* h_dcnt = nullptr;
  int32_t delta_cap = 0, delta_rounds = 0;
  // row shards in graph mode: graphs of kShardRounds unrolled rounds -- one
  // with the dense all-reduce, one per delta capacity tier (fixed-size
  // all-gathers) -- launched by the host, which reads the round state once
  // per graph (engine.cu run_shard_solve); no NCCL call sits inside a
  // conditional node
  static constexpr int kMaxTiers = 3;
  int shard_rounds = 4;
  bool unrolled = false;             // capturing / running the unrolled graphs
  cudaGraphExec_t shard_dense = nullptr;
  cudaGraphExec_t shard_delta[kMaxTiers] = {nullptr, nullptr, nullptr};
  int32_t delta_caps[kMaxTiers] = {0, 0, 0};
  int ntiers = 0;
  int64_t host_syncs = 0;            // host round trips of the last solve
  int64_t held_rounds = 0;           // delta rounds held by an overflow (resumed densely)
  int64_t delta_graphs = 0;          // graphs of delta rounds launched (the rest were dense)
  bool delta_mode() const { return comm && (cfg.flags & PG_FLAG_DELTA_EXCHANGE); }
  // branch-and-bound: the root fixpoint and the next solve's start control
  NodeCtl* d_ctl = nullptr;
  double* d_root_lo = nullptr;
  double* d_keep_lo = nullptr;  // pg_session_round: the session's start bounds, kept aside
  double* d_keep_up = nullptr;
  double* d_root_up = nullptr;
  bool has_root = false;
  bool l2_window = false;  // a persisting-L2 access window on the session stream

  ~pg_session() {
    if (dev >= 0) cudaSetDevice(dev);
    t_alloc_stream = stream;
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    destroy_shard_graphs();

    if (comm && !comm_aborted) g_nccl.comm_destroy(comm);  // an aborted one is freed already
    if (l2_window) {
      // the pooled stream must not carry this session's window into the next
      cudaStreamAttrValue av = {};
      av.accessPolicyWindow.num_bytes = 0;
      cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &av);
      cudaCtxResetPersistingL2Cache();
    }
    release_buffers();
    if (h_dcnt) cudaFreeHost(h_dcnt);
    StreamPool::get().put(dev, StreamSet{stream, stream2, ev0, ev1, ev_fork, ev_join, h_st});
  }

  // device buffers back to the pool (stream-ordered, no device sync; a few
  // microseconds of host time): a one-shot call does this itself so the next
  // call's allocations reuse the memory instead of growing the pool while
  // the reaper thread still holds the session
  void release_buffers() {
    t_alloc_stream = stream;
    void** ptrs[] = {
        (void**)&d_ctl, (void**)&d_root_lo, (void**)&d_root_up, (void**)&d_keep_lo, (void**)&d_keep_up,
        (void**)&d_delta, (void**)&d_delta_all, (void**)&d_dcnt, (void**)&d_dcnt_all, (void**)&d_row_ptr,
        (void**)&d_colx, (void**)&d_vals, (void**)&d_lhs, (void**)&d_rhs, (void**)&d_snap,
        (void**)&d_integral, (void**)&d_row_done, (void**)&d_key_out, (void**)&d_lo0, (void**)&d_up0,
        (void**)&d_lo_res, (void**)&d_up_res, (void**)&d_segs, (void**)&d_srow, (void**)&d_sfirst,
        (void**)&d_partial, (void**)&d_ract, (void**)&d_wl_short, (void**)&d_wl_long,
        (void**)&d_f32_part, (void**)&d_ractf, (void**)&d_partf, (void**)&d_split, (void**)&d_bnd, (void**)&d_bf,
        (void**)&d_units, (void**)&d_slices, (void**)&d_sv, (void**)&d_sc, (void**)&d_sw, (void**)&d_st,
        (void**)&d_per_round, (void**)&d_col_ptr, (void**)&d_col_item, (void**)&d_flags, (void**)&d_chg,
        (void**)&d_row_unit, (void**)&d_part_unit, (void**)&d_unit_slice, (void**)&d_wide_list,
        (void**)&d_unit_list, (void**)&d_tflag, (void**)&d_tlist};
    for (void** p : ptrs) {
      dfree(*p);
      *p = nullptr;
    }
  }

  int grid_for(int64_t items, int threads, int per_sm = 8) const {
    const int64_t g = (items + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms * per_sm));
  }

  // ---- one round of kernels, enqueued on `stream` ------------------------------
  RoundArgs round_args() const {
    RoundArgs A;
    A.slices = d_slices;
    A.nslices = nslices;
    A.group_start = group_start;
    A.lg0_ustart = lg0_ustart;
    A.lg0_sstart = lg0_sstart;
    A.nunits = nunits;
    A.units = d_units;
    A.sv = d_sv;
    A.sc = d_sc;
    A.sw = d_sw;
    A.pad_col = n;
    A.segs = d_segs;
    A.srow = d_srow;
    A.sfirst = d_sfirst;
    A.row_done = d_row_done;
    A.partial = d_partial;
    A.row_ptr = d_row_ptr;
    A.colx = d_colx;
    A.vals = d_vals;
    A.lhs = d_lhs;
    A.rhs = d_rhs;
    A.ract = d_ract;
    A.wl_short = d_wl_short;
    A.wl_long = d_wl_long;
    A.snap = d_snap;
    A.bnd = d_bnd;
    A.key_out = (long long*)d_key_out;
    A.st = d_st;
    A.dirty = dirty;
    A.touch = touch;
    return A;
  }

  // A round kernel on the session stream with programmatic dependent launch
  // (PG_PDL, default on; single-GPU sessions): its CTAs are scheduled while the previous
  // kernel's last CTAs run and wait for its completion in pdl_begin()
  // (kernels.cuh) -- the per-kernel launch gap of the round's chain
  static bool use_pdl() {
    static const bool on = !getenv("PG_PDL") || atoi(getenv("PG_PDL")) != 0;
    return on;
  }
  template <typename... KArgs, typename... Args>
  void pdl(void (*k)(KArgs...), int grid, int block, size_t smem, Args... args) {
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3((unsigned)grid);
    c.blockDim = dim3((unsigned)block);
    c.dynamicSmemBytes = smem;
    c.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = at;
    // not across a row shard's NCCL exchange: its collectives can only be
    // exercised at world 1 here, so those graphs keep plain stream order
    c.numAttrs = use_pdl() && !comm ? 1 : 0;
    PG_CUDA(cudaLaunchKernelEx(&c, k, args...));
  }

  // phase 1 over the sliced-ELL copy: the full sweep, and with the worklist
  // the worklist sweep (each returns at once when the round is of the other kind)
  template <int kB16>
  void launch_sell(const RoundArgsG<kB16>& G, int grid, bool rowcheck) {
    const int dgrid = std::max(1, std::min((nslices + 7) / 8, num_sms * sell_dense_per_sm));
    if (rowcheck)
      pdl(k_sell<true, true, kB16>, dgrid, kSellThreads, kSellSmemDense, G, dcfg);
    else
      pdl(k_sell<false, true, kB16>, dgrid, kSellThreads, kSellSmemDense, G, dcfg);
    if (dirty.enabled) {
      if (rowcheck)
        pdl(k_sell<true, false, kB16>, grid, kSellThreads, kSellSmem, G, dcfg);
      else
        pdl(k_sell<false, false, kB16>, grid, kSellThreads, kSellSmem, G, dcfg);
    }
  }

  // One round: phase 1 (k_sell), phase 2 (k_cand), [row shards: all-reduce],
  // commit + decision (k_commit), [worklist: k_mark].  k1_begin/k1_end
  // bracket the two compute phases (bench.py's roofline timing).
  // tier >= 0: an unrolled row-shard round exchanging sparse deltas at the
  // fixed capacity delta_caps[tier] (held on overflow, see k_delta_apply)
  void enqueue_round(bool use_graph, cudaEvent_t k1_begin = nullptr, cudaEvent_t k1_end = nullptr,
                     int tier = -1) {
    const bool rowcheck = (cfg.flags & PG_FLAG_ROWCHECK) != 0;
    const RoundArgs A = round_args();
    if (k1_begin) PG_CUDA(cudaEventRecord(k1_begin, stream));
    if (cfg.scalar_mode == PG_NARROW32 && nslices > 0 && d_ractf) {
      // float chains and candidates over the sliced-ELL copy (narrow_sell.cuh)
      const int grid = std::max(1, std::min((nslices + 7) / 8, num_sms * sell_per_sm));
      if (rowcheck)
        k_sellf_act<true><<<grid, kSellThreads, 0, stream>>>(A, dcfg, d_ractf, d_partf);
      else
        k_sellf_act<false><<<grid, kSellThreads, 0, stream>>>(A, dcfg, d_ractf, d_partf);
      if (nsplit > 0) {
        const int g = std::max(1, std::min((nsplit + 127) / 128, num_sms * 4));
        if (rowcheck)
          k_sellf_split<true><<<g, 128, 0, stream>>>(A, d_split, nsplit, d_ractf, d_partf, dcfg);
        else
          k_sellf_split<false><<<g, 128, 0, stream>>>(A, d_split, nsplit, d_ractf, d_partf, dcfg);
      }
      k_sellf_cand<<<grid, kSellThreads, 0, stream>>>(A, dcfg, d_ractf);
    } else if (cfg.scalar_mode == PG_NARROW32) {
      if (m > 0) {
        const int grid = grid_for(m, 256, 4);
        if (rowcheck)
          k_round_f32<true><<<grid, 256, 0, stream>>>(A, dcfg, m, d_f32_part, f32_maxc);
        else
          k_round_f32<false><<<grid, 256, 0, stream>>>(A, dcfg, m, d_f32_part, f32_maxc);
      }
    } else if (nslices > 0) {
      const int grid = std::max(1, std::min((nslices + 7) / 8, num_sms * sell_per_sm));
      switch (gather_kind()) {
        case 2: launch_sell(RoundArgsG<2>{A}, grid, rowcheck); break;
        case 1: launch_sell(RoundArgsG<1>{A}, grid, rowcheck); break;
        default: launch_sell(RoundArgsG<0>{A}, grid, rowcheck);
      }
      if (nsplit > 0) {
        const int g = std::max(1, std::min((nsplit + kSplitWarps - 1) / kSplitWarps, num_sms * 8));
        if (rowcheck)
          pdl(k_split_finish<true>, g, kSplitWarps * 32, 0, A, (const int32_t*)d_split, nsplit, dcfg);
        else
          pdl(k_split_finish<false>, g, kSplitWarps * 32, 0, A, (const int32_t*)d_split, nsplit, dcfg);
      }
      // phase 2 of split rows (their finisher queues them); none without
      if (nsplit > 0) pdl(k_cand, num_sms * cand_per_sm, kCandThreads, 0, A, dcfg);
    }
    if (k1_end) PG_CUDA(cudaEventRecord(k1_end, stream));
    bool dense_exchange = comm != nullptr;
    if (comm && tier >= 0) {
      const int cap = delta_caps[tier];
      PG_CUDA(cudaMemsetAsync(d_dcnt, 0, 2 * sizeof(int), stream));
      k_delta_compact<<<grid_for(n, 256, 8), 256, 0, stream>>>(d_bnd, d_key_out, n, d_st, d_delta,
                                                                cap, d_dcnt);
      PG_CUDA(cudaGetLastError());
      int rc = g_nccl.all_gather_fn(d_dcnt, d_dcnt_all, 2, kNcclInt32, comm, stream);
      if (rc != 0) throw Error{PG_ENCCL, std::string("ncclAllGather: ") + g_nccl.error(rc)};
      rc = g_nccl.all_gather_fn(d_delta, d_delta_all, 3 * (size_t)cap, kNcclInt64, comm, stream);
      if (rc != 0) throw Error{PG_ENCCL, std::string("ncclAllGather: ") + g_nccl.error(rc)};
      k_delta_apply<<<grid_for(cap, 256, 8), 256, 0, stream>>>(d_delta_all, d_dcnt_all, world, cap,
                                                               d_key_out, d_st, 1);
      PG_CUDA(cudaGetLastError());
      dense_exchange = false;
    } else if (comm && delta_mode() && !use_graph && !unrolled) {
      // sparse delta exchange: all-gather the
      // counts; when every rank changed at most delta_cap columns, all-gather
      // the (column, keys) items and max-merge them, else the dense all-reduce.
      // The choice reads the gathered counts, so every rank makes the same one.
      PG_CUDA(cudaMemsetAsync(d_dcnt, 0, 2 * sizeof(int), stream));
      k_delta_compact<<<grid_for(n, 256, 8), 256, 0, stream>>>(d_bnd, d_key_out, n, d_st, d_delta,
                                                                delta_cap, d_dcnt);
      PG_CUDA(cudaGetLastError());
      int rc = g_nccl.all_gather_fn(d_dcnt, d_dcnt_all, 2, kNcclInt32, comm, stream);
      if (rc != 0) throw Error{PG_ENCCL, std::string("ncclAllGather: ") + g_nccl.error(rc)};
      PG_CUDA(cudaMemcpyAsync(h_dcnt, d_dcnt_all, 2 * sizeof(int) * world, cudaMemcpyDeviceToHost,
                              stream));
      PG_CUDA(cudaStreamSynchronize(stream));
      int maxc = 0;
      for (int r = 0; r < world; ++r) maxc = std::max(maxc, h_dcnt[2 * r]);
      if (maxc <= delta_cap) {
        dense_exchange = false;
        ++delta_rounds;
        if (maxc > 0) {
          rc = g_nccl.all_gather_fn(d_delta, d_delta_all, 3 * (size_t)maxc, kNcclInt64, comm, stream);
          if (rc != 0) throw Error{PG_ENCCL, std::string("ncclAllGather: ") + g_nccl.error(rc)};
        }
        k_delta_apply<<<grid_for(std::max(maxc, 1), 256, 8), 256, 0, stream>>>(
            d_delta_all, d_dcnt_all, world, maxc, d_key_out, d_st, 0);
        PG_CUDA(cudaGetLastError());
      }
    }
    if (dense_exchange) {
      // row shards: merge every rank's bound keys (lb keys and negated ub keys)
      // and infeasibility with one max all-reduce; each rank then commits the
      // same merged bounds, so counts and decisions need no further exchange
      k_flag_to_slot<<<1, 32, 0, stream>>>(d_st, d_key_out + n);
      PG_CUDA(cudaGetLastError());
      const int rc = g_nccl.all_reduce(d_key_out, d_key_out, 2 * ((size_t)n + 1), kNcclInt64,
                                       kNcclMax, comm, stream);
      if (rc != 0) throw Error{PG_ENCCL, std::string("ncclAllReduce: ") + g_nccl.error(rc)};
    }
    // commit / list / mark grids per SM (env overrides: A/B experiments)
    static const int commit_per_sm = getenv("PG_COMMIT_PER_SM") ? atoi(getenv("PG_COMMIT_PER_SM")) : 2;
    static const int list_per_sm = getenv("PG_LIST_PER_SM") ? atoi(getenv("PG_LIST_PER_SM")) : 2;
    pdl(k_commit, grid_for(n, kCommitThreads, commit_per_sm), kCommitThreads, 0, d_snap, d_bnd,
        (const longlong2*)d_key_out, (int)n, d_st, d_per_round, dcfg, dirty, cond,
        use_graph && !unrolled ? 1 : 0, comm ? 0 : 1);
    if (dirty.enabled && !comm)
      pdl(k_commit_list, num_sms * list_per_sm, kCommitThreads, 0, d_snap, d_bnd,
          (const longlong2*)d_key_out, (int)n, d_st, d_per_round, dcfg, dirty, touch, cond,
          use_graph ? 1 : 0);
    if (dirty.enabled) pdl(k_mark, num_sms * list_per_sm, 256, 0, dirty, d_st);
    PG_CUDA(cudaGetLastError());
  }

  void enqueue_reset(bool use_graph, bool check_crossed) {
    k_reset<<<grid_for(n, kCommitThreads), kCommitThreads, 0, stream>>>(
        d_lo0, d_up0, d_integral, d_snap, d_bnd, d_key_out, n, d_st, dcfg, dirty, d_ctl,
        check_crossed ? 1 : 0, cond, use_graph ? 1 : 0);
    if (dirty.enabled) k_mark_vars<<<num_sms * 2, 256, 0, stream>>>(dirty, d_ctl, d_st);
    PG_CUDA(cudaGetLastError());
  }

  // longest row (computed on first use: Narrow32 scratch, B&B node scratch)
  int32_t max_len() {
    if (max_row_len >= 0) return max_row_len;
    int32_t* d = dalloc<int32_t>(1);
    PG_CUDA(cudaMemsetAsync(d, 0, sizeof(int32_t), stream));
    if (m) k_max_row_len<<<grid_for(m, 256), 256, 0, stream>>>(d_row_ptr, m, d);
    PG_CUDA(cudaMemcpyAsync(&max_row_len, d, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    PG_CUDA(cudaStreamSynchronize(stream));
    dfree(d);
    return max_row_len;
  }

  // column -> rows index over the sorted rows (device counting sort);
  // used by the worklist marks and the batched branch-and-bound nodes
  void ensure_col_index() {
    if (d_col_ptr) return;
    t_alloc_stream = stream;
    build_col_index(d_row_ptr, d_colx, nullptr, stream);
  }
  // rp/cols: a CSR whose row r is session row rowmap[r] (nullptr: r itself)
  void build_col_index(const int32_t* rp, const int32_t* cols, const int32_t* rowmap,
                       cudaStream_t st) {
    d_col_ptr = dalloc<int32_t>((size_t)n + 1);
    d_col_item = dalloc<int32_t>(nnz);
    int32_t* cnt = dalloc<int32_t>((size_t)n + 1);
    PG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ((size_t)n + 1), st));
    if (nnz) k_csc_count<<<grid_for(nnz, 256, 16), 256, 0, st>>>(cols, nnz, n, cnt);
    size_t tmp_bytes = 0;
    PG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, d_col_ptr, n + 1, st));
    void* tmp = dalloc<unsigned char>(tmp_bytes);
    PG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, d_col_ptr, n + 1, st));
    PG_CUDA(cudaMemcpyAsync(cnt, d_col_ptr, sizeof(int32_t) * ((size_t)n + 1),
                            cudaMemcpyDeviceToDevice, st));
    if (m) k_csc_fill<<<grid_for(nnz * 32 / kWalkChunk + 1, 256, 16), 256, 0, st>>>(rp, cols, m, n, cnt,
                                                                                   rowmap, d_col_item);
    PG_CUDA(cudaGetLastError());
    dfree(tmp);
    dfree(cnt);
    dirty.col_ptr = d_col_ptr;
    dirty.col_row = d_col_item;
  }

  // persistent round loop (loop.cuh): small instances and worklist solves,
  // whose rounds are launch-latency bound; never with a communicator (the
  // all-reduce is a host-enqueued NCCL call between phases)
  // the hybrid loop: per-kernel rounds while they are full sweeps, then the
  // persistent kernel for the worklist tail (instances above the persistent
  // threshold, worklist on; PG_HYBRID=1 enables)
  bool use_hybrid() const {
    // measured slower on C2 / C5 (1.61 -> 1.78 ms, 10.1 -> 14.5 ms): opt-in
    static const bool on = getenv("PG_HYBRID") && atoi(getenv("PG_HYBRID")) != 0;
    return on && !comm && loop_grid > 0 && cfg.scalar_mode != PG_NARROW32 && dirty.enabled &&
           !use_persistent();
  }

  bool use_persistent() const {
    if (comm || loop_grid <= 0 || cfg.scalar_mode == PG_NARROW32) return false;
    static const long long thr = [] {
      const char* e = getenv("PG_PERSIST_NNZ");
      return e ? atoll(e) : 8000000LL;
    }();
    return nnz <= thr;
  }

  void enqueue_persistent() {
    const RoundArgsL A{round_args()};
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(loop_grid);
    lc.blockDim = dim3(kSellThreads);
    lc.dynamicSmemBytes = sizeof(LoopSmem);
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    Snap* snap = d_snap;
    long long* pr = d_per_round;
    int nn = n;
    if (cfg.flags & PG_FLAG_ROWCHECK)
      PG_CUDA(cudaLaunchKernelEx(&lc, k_loop<true>, A, dcfg, snap, nn, pr,
                                 (const int32_t*)d_split, nsplit));
    else
      PG_CUDA(cudaLaunchKernelEx(&lc, k_loop<false>, A, dcfg, snap, nn, pr,
                                 (const int32_t*)d_split, nsplit));
  }

  // row shards: the unrolled round graphs (see shard_dense)
  void build_shard_graphs() {
    destroy_shard_graphs();
    if (const char* e = getenv("PG_SHARD_ROUNDS")) shard_rounds = std::max(1, atoi(e));
    unrolled = true;
    // the round kernels of these graphs check the device state first
    dcfg.flags |= kUnrolledFlag;
    dirty.unrolled = 1;
    struct Off {
      bool* f;
      ~Off() { *f = false; }
    } off{&unrolled};
    auto capture = [&](int tier) {
      cudaGraph_t g = nullptr;
      PG_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      for (int r = 0; r < shard_rounds; ++r) enqueue_round(false, nullptr, nullptr, tier);
      PG_CUDA(cudaStreamEndCapture(stream, &g));
      cudaGraphExec_t x = nullptr;
      const cudaError_t e = cudaGraphInstantiate(&x, g, 0);
      cudaGraphDestroy(g);
      PG_CUDA(e);
      return x;
    };
    shard_dense = capture(-1);
    if (delta_mode())
      for (int t = 0; t < ntiers; ++t) shard_delta[t] = capture(t);
  }
  void destroy_shard_graphs() {
    if (shard_dense) cudaGraphExecDestroy(shard_dense);
    shard_dense = nullptr;
    for (auto& x : shard_delta) {
      if (x) cudaGraphExecDestroy(x);
      x = nullptr;
    }
  }

  // A row-sharded solve in graph mode: reset, then graphs of shard_rounds
  // rounds until the (identical on every rank) state says done.  The first
  // rounds exchange densely; once a round changed few enough sides, the
  // smallest delta tier whose capacity covers that count (a rank's changed
  // columns never exceed the round's changed sides, and the next round's
  // rarely exceed this one's); a held round (overflow) is resumed densely.
  // Every rank reads the same merged state, so all pick the same graph.
  void run_shard_solve(bool check_crossed) {
    host_syncs = 0;
    held_rounds = 0;
    delta_graphs = 0;
    // test knob: always the given delta tier after the first graph (forces
    // overflows, i.e. held and resumed rounds)
    static const int force_tier = getenv("PG_SHARD_TIER") ? atoi(getenv("PG_SHARD_TIER")) : -1;
    enqueue_reset(false, check_crossed);
    h_st->done = 0;
    h_st->stall = 0;
    bool first = true;
    for (;;) {
      cudaGraphExec_t g = shard_dense;
      if (h_st->stall) {
        ++held_rounds;
        k_shard_resume<<<1, 32, 0, stream>>>(d_st);
        PG_CUDA(cudaGetLastError());
      } else if (!first && delta_mode() && force_tier >= 0 && force_tier < ntiers) {
        g = shard_delta[force_tier];
      } else if (!first && delta_mode()) {
        const long long want = h_st->last_changes;
        for (int t = ntiers - 1; t >= 0; --t)
          if (shard_delta[t] && want <= delta_caps[t]) {
            g = shard_delta[t];
            break;
          }
      }
      PG_CUDA(cudaGraphLaunch(g, stream));
      delta_graphs += g != shard_dense;
      PG_CUDA(cudaMemcpyAsync(h_st, d_st, sizeof(DevState), cudaMemcpyDeviceToHost, stream));
      PG_CUDA(cudaStreamSynchronize(stream));
      ++host_syncs;
      first = false;
      if (h_st->done) break;
    }
    delta_rounds = h_st->delta_rounds;
  }

  void build_graph() {
    if (comm) {
      build_shard_graphs();
      return;
    }
    PG_CUDA(cudaGraphCreate(&graph, 0));
    if (use_persistent()) {
      PG_CUDA(cudaStreamBeginCaptureToGraph(stream, graph, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal));
      enqueue_reset(false, true);
      enqueue_persistent();
      cudaGraph_t g2 = nullptr;
      PG_CUDA(cudaStreamEndCapture(stream, &g2));
      PG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      return;
    }
    PG_CUDA(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    // node 1: reset (+ warm-start marks), captured
    cudaGraphNode_t reset_node = nullptr;
    {
      cudaGraph_t g2 = nullptr;
      PG_CUDA(cudaStreamBeginCaptureToGraph(stream, graph, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal));
      enqueue_reset(true, true);
      PG_CUDA(cudaStreamEndCapture(stream, &g2));
      size_t count = 0;
      PG_CUDA(cudaGraphGetNodes(graph, nullptr, &count));
      std::vector<cudaGraphNode_t> nodes(count);
      PG_CUDA(cudaGraphGetNodes(graph, nodes.data(), &count));
      for (cudaGraphNode_t nd : nodes) {  // the sink of the captured chain
        size_t deps = 0;
        PG_CUDA(cudaGraphNodeGetDependentNodes(nd, nullptr, &deps));
        if (deps == 0) reset_node = nd;
      }
    }
    // node 2: WHILE(cond) { round }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t while_node;
    PG_CUDA(cudaGraphAddNode(&while_node, graph, &reset_node, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    PG_CUDA(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
    enqueue_round(true);
    const bool hybrid = use_hybrid();
    if (hybrid) {
      k_hybrid_decide<<<1, 32, 0, stream>>>(d_st, dirty, cond);
      PG_CUDA(cudaGetLastError());
    }
    cudaGraph_t body2 = nullptr;
    PG_CUDA(cudaStreamEndCapture(stream, &body2));
    if (hybrid) {
      // node 3: the persistent kernel finishes the solve (returns at once if done)
      cudaGraph_t g3 = nullptr;
      PG_CUDA(cudaStreamBeginCaptureToGraph(stream, graph, &while_node, nullptr, 1,
                                            cudaStreamCaptureModeThreadLocal));
      enqueue_persistent();
      PG_CUDA(cudaStreamEndCapture(stream, &g3));
    }
    PG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  }

  // Runs one full solve from lo0/up0.  Returns elapsed device ns.
  // res: download the bounds in the same pass (graph loop): the decode and
  // the copies are queued behind the solve and the host faults in the
  // result pages while the GPU works (a fresh pageable array costs a page
  // fault per 4 KB inside the copy otherwise)
  int64_t run_solve(bool check_crossed = true, pg_result* res = nullptr) {
    bounds_done = false;
    delta_rounds = 0;
    if (comm && cfg.loop_mode == PG_LOOP_GRAPH) {
      PG_CUDA(cudaEventRecord(ev0, stream));
      run_shard_solve(check_crossed);
      PG_CUDA(cudaEventRecord(ev1, stream));
    } else if (cfg.loop_mode == PG_LOOP_GRAPH && check_crossed && !delta_mode()) {
      PG_CUDA(cudaEventRecord(ev0, stream));
      g_trace.mark("solve start", stream);
      PG_CUDA(cudaGraphLaunch(exec, stream));
      PG_CUDA(cudaEventRecord(ev1, stream));
      g_trace.mark("solve end", stream);
      if (res && (res->lower || res->upper)) {
        k_decode<<<grid_for(n, 256), 256, 0, stream>>>(d_key_out, d_lo_res, d_up_res, n);
        PG_CUDA(cudaGetLastError());
        for (double* out : {res->lower, res->upper})
          if (out) {
            volatile char* b = reinterpret_cast<volatile char*>(out);
            for (size_t off = 0; off < sizeof(double) * n; off += 4096) b[off] = 0;
          }
        if (res->lower)
          PG_CUDA(cudaMemcpyAsync(res->lower, d_lo_res, sizeof(double) * n,
                                  cudaMemcpyDeviceToHost, stream));
        if (res->upper)
          PG_CUDA(cudaMemcpyAsync(res->upper, d_up_res, sizeof(double) * n,
                                  cudaMemcpyDeviceToHost, stream));
        bounds_done = true;
        g_trace.mark("download", stream);
      }
    } else {
      // host-driven loop: one sync per round (the paper's cpu_loop)
      PG_CUDA(cudaEventRecord(ev0, stream));
      enqueue_reset(false, check_crossed);
      PG_CUDA(cudaMemcpyAsync(h_st, d_st, sizeof(DevState), cudaMemcpyDeviceToHost, stream));
      PG_CUDA(cudaStreamSynchronize(stream));
      static const bool dbg = getenv("PG_DEBUG_ROUNDS") != nullptr;
      while (!h_st->done) {
        if (dbg)
          fprintf(stderr,
                  "[pg] round %d: full=%d nunit={%d,%d} nwide={%d,%d} nmid={%d,%d} nchg={%d,%d} "
                  "deg={%lld,%lld}\n",
                  h_st->round + 1, h_st->full, h_st->nunit[0], h_st->nunit[1], h_st->nwide[0],
                  h_st->nwide[1], h_st->nmid[0], h_st->nmid[1], h_st->nchg[0], h_st->nchg[1],
                  h_st->chg_deg[0], h_st->chg_deg[1]);
        enqueue_round(false);
        PG_CUDA(cudaMemcpyAsync(h_st, d_st, sizeof(DevState), cudaMemcpyDeviceToHost, stream));
        PG_CUDA(cudaStreamSynchronize(stream));
      }
      PG_CUDA(cudaEventRecord(ev1, stream));
    }
    PG_CUDA(cudaMemcpyAsync(h_st, d_st, sizeof(DevState), cudaMemcpyDeviceToHost, stream));
    PG_CUDA(cudaStreamSynchronize(stream));
    check_input();
    float ms = 0.f;
    PG_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    return (int64_t)((double)ms * 1e6);
  }

  bool bounds_done = false;  // run_solve already downloaded the bounds

  // a col_idx outside [0, n) found during setup (k_permute_rows); h_st fresh
  void check_input() const {
    if (h_st->bad_input) throw Error{PG_EINVAL, "col_idx entry outside [0, num_cols)"};
  }

  void fill_result(pg_result* res, int64_t elapsed) {
    res->status = h_st->status < 0 ? PG_ROUNDLIMIT : h_st->status;
    res->rounds_executed = h_st->round;
    res->total_bound_changes = h_st->total_changes;
    res->constraints_processed = (int64_t)h_st->round * m;
    res->elapsed_ns = elapsed;
    if (res->per_round_changes && res->per_round_capacity > 0 && h_st->round > 0) {
      const int cnt = std::min(res->per_round_capacity, h_st->round);
      PG_CUDA(cudaMemcpyAsync(res->per_round_changes, d_per_round, sizeof(long long) * cnt,
                              cudaMemcpyDeviceToHost, stream));
    }
    if ((res->lower || res->upper) && !bounds_done) {
      // returned bounds = last round's output (par_engine.cpp:271); after
      // the commit key_in == key_out; with 0 rounds they are the start bounds
      k_decode<<<grid_for(n, 256), 256, 0, stream>>>(d_key_out, d_lo_res, d_up_res, n);
      PG_CUDA(cudaGetLastError());
      if (res->lower)
        PG_CUDA(cudaMemcpyAsync(res->lower, d_lo_res, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                stream));
      if (res->upper)
        PG_CUDA(cudaMemcpyAsync(res->upper, d_up_res, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                stream));
    }
    PG_CUDA(cudaStreamSynchronize(stream));
  }

  void upload_bounds(const double* lo, const double* up) {
    PG_CUDA(cudaMemcpyAsync(d_lo0, lo, sizeof(double) * n, cudaMemcpyHostToDevice, stream));
    PG_CUDA(cudaMemcpyAsync(d_up0, up, sizeof(double) * n, cudaMemcpyHostToDevice, stream));
    normalize_bounds();
  }
  void normalize_bounds() {
    if (n) {
      k_normalize<<<grid_for(n, 256), 256, 0, stream>>>(d_lo0, n, cfg.infinity_threshold);
      k_normalize<<<grid_for(n, 256), 256, 0, stream>>>(d_up0, n, cfg.infinity_threshold);
      if (cfg.scalar_mode == PG_NARROW32) {
        k_to_f32<<<grid_for(n, 256), 256, 0, stream>>>(d_lo0, n);
        k_to_f32<<<grid_for(n, 256), 256, 0, stream>>>(d_up0, n);
      }
      PG_CUDA(cudaGetLastError());
    }
  }
};

namespace {

// Whether the round kernels should gather 8 B float bound records: at least
// 95 % of up to 4096 evenly spaced columns are integral with both start
// bounds floats (their tightened bounds stay integers).  Speed only: a
// column whose bounds are not floats is read from its exact record.
static bool float_bounds_sample(const pg_problem* p) {
  const int32_t n = p->num_cols;
  if (n <= 0) return false;
  const int32_t k = std::min<int32_t>(n, 4096);
  int32_t ok = 0;
  for (int32_t i = 0; i < k; ++i) {
    const int32_t j = (int32_t)((int64_t)i * n / k);
    const double l = p->lower[j], u = p->upper[j];
    ok += p->integral[j] && (double)(float)l == l && (double)(float)u == u;
  }
  return ok >= k - k / 20;
}

pg_session* create_session(const pg_problem* p, const pg_config* cfg) {
  PhaseTimer tm;
  check_problem(p);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error{PG_ENODEV, "no CUDA device visible (the B200 engine has no CPU fallback)"};
  if (cfg->device < 0 || cfg->device >= ndev) throw Error{PG_EINVAL, "device ordinal out of range"};
  const DevInfo prop = device_info(cfg->device);
  if (prop.major != 10)
    throw Error{PG_ENODEV, std::string("device is ") + prop.name + " (sm_" +
                               std::to_string(prop.major * 10 + prop.minor) +
                               "); this build targets sm_100a only"};

  tm.lap("device query");
  auto* s = new pg_session;
  try {
    s->dev = cfg->device;
    PG_CUDA(cudaSetDevice(s->dev));
    s->num_sms = prop.sms;
    {
      // kernel attributes and occupancies, once per device (they cost ~0.7 ms)
      struct Occ {
        bool ok = false;
        int sell = 1, sell_dense = 1, cand = 1, loop_grid = 0, nodes = 1;
      };
      static Occ occ[64];
      static std::mutex mu;
      std::lock_guard<std::mutex> lock(mu);
      Occ& o = occ[s->dev];
      if (!o.ok) {
        for (const void* f :
             {(const void*)k_sell<true, true, 1>, (const void*)k_sell<false, true, 1>,
              (const void*)k_sell<true, false, 1>, (const void*)k_sell<false, false, 1>,
              (const void*)k_sell<true, true, 0>, (const void*)k_sell<false, true, 0>,
              (const void*)k_sell<true, false, 0>, (const void*)k_sell<false, false, 0>,
              (const void*)k_sell<true, true, 2>, (const void*)k_sell<false, true, 2>,
              (const void*)k_sell<true, false, 2>, (const void*)k_sell<false, false, 2>})
          PG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSellSmem));
        for (const void* f : {(const void*)k_loop<true>, (const void*)k_loop<false>})
          PG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(LoopSmem)));
        int o16 = 0, o8 = 0, d32 = 0, d16 = 0, d8 = 0;
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.sell, k_sell<true, false, 0>,
                                                              kSellThreads, kSellSmem));
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o16, k_sell<true, false, 1>,
                                                              kSellThreads, kSellSmem));
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o8, k_sell<true, false, 2>,
                                                              kSellThreads, kSellSmem));
        o.sell = std::min(o.sell, std::min(o16, o8));
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d32, k_sell<true, true, 0>,
                                                              kSellThreads, kSellSmemDense));
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d16, k_sell<true, true, 1>,
                                                              kSellThreads, kSellSmemDense));
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d8, k_sell<true, true, 2>,
                                                              kSellThreads, kSellSmemDense));
        o.sell_dense = std::min(d32, std::min(d16, d8));
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.cand, k_cand, kCandThreads, 0));
        int per = 0, per2 = 0;
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_loop<true>, kSellThreads,
                                                              sizeof(LoopSmem)));
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_loop<false>, kSellThreads,
                                                              sizeof(LoopSmem)));
        o.loop_grid = std::min(per, per2) * s->num_sms;
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_nodes<true>, kNodeThreads, 0));
        o.nodes = per;
        o.ok = true;
      }
      s->sell_per_sm = std::max(1, o.sell);
      s->sell_dense_per_sm = std::max(1, o.sell_dense);
      // one k_cand CTA per SM: the queues are drained by tickets, and fewer
      // CTAs start and drain faster (A/B: 1 < 2 < full occupancy on C2/C5)
      s->cand_per_sm = 1;
      if (const char* e = getenv("PG_CAND_PER_SM")) s->cand_per_sm = std::max(1, atoi(e));
      s->loop_grid = o.loop_grid;
      s->nodes_per_sm = std::max(1, o.nodes);
    }

    s->m = p->num_rows;
    s->n = p->num_cols;
    s->nnz = p->nnz;
    s->cfg = *cfg;
    s->dcfg.inf_thr = cfg->infinity_threshold;
    s->dcfg.imp_abs = cfg->improvement_abs;
    s->dcfg.imp_rel = cfg->improvement_rel;
    s->dcfg.int_eps = cfg->integrality_eps;
    s->dcfg.chunk = cfg->nnz_budget;
    s->dcfg.round_limit = cfg->round_limit;
    s->dcfg.flags = cfg->flags;
    {
      const StreamSet x = StreamPool::get().get(s->dev);
      s->stream = x.st;
      s->stream2 = x.st2;
      s->ev0 = x.ev0;
      s->ev1 = x.ev1;
      s->ev_fork = x.fork;
      s->ev_join = x.join;
      s->h_st = x.h_st;
    }
    t_alloc_stream = s->stream;

    tm.lap("streams/attributes");
    const int32_t m = s->m, n = s->n;
    const int64_t nnz = s->nnz;
    const int32_t short_max = (int32_t)std::min<int64_t>(cfg->nnz_budget, kShortMax);
    const int32_t chunk = cfg->nnz_budget;
    cudaStream_t st = s->stream, s2 = s->stream2;

    // buffers: the caller's arrays staged in input row order, the ordering work
    int32_t* t_rp = dalloc<int32_t>((size_t)m + 1);
    int32_t* t_cols = dalloc<int32_t>(nnz);
    double* t_vals = dalloc<double>(nnz);
    double* t_lhs = dalloc<double>(m);
    double* t_rhs = dalloc<double>(m);
    s->d_integral = dalloc<uint8_t>(n);
    s->d_row_ptr = dalloc<int32_t>((size_t)m + 1 + 4);  // +16 B: bulk-copy tail
    uint8_t* key = dalloc<uint8_t>(m);
    uint8_t* key2 = dalloc<uint8_t>(m);
    int32_t* idx = dalloc<int32_t>(m);
    int32_t* t_perm = dalloc<int32_t>(m);
    int32_t* slen = dalloc<int32_t>((size_t)m + 1);
    int32_t* counts = dalloc<int32_t>(kMaxClasses + 5);  // + u64 sum of len^2 at [kMaxClasses + 2], bad row_ptr flag at [+4]
    g_trace.mark("start", st);
    // row_ptr first, on stream 2, and the rest of the upload (stream 1,
    // asynchronous from pinned memory) after it: stream 2's ordering starts
    // as soon as row_ptr is in.  (Without the wait the matrix copies may
    // reach the copy engine first and row_ptr lands behind all of them; an
    // event after a copy on stream 1 can also fire only after the copies
    // that follow it.)
    auto h2d = [&](void* dst, const void* src, size_t bytes, cudaStream_t q) {
      if (bytes) PG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, q));
    };
    PG_CUDA(cudaEventRecord(s->ev_fork, st));
    PG_CUDA(cudaStreamWaitEvent(s2, s->ev_fork, 0));
    h2d(t_rp, p->row_ptr, sizeof(int32_t) * ((size_t)m + 1), s2);
    PG_CUDA(cudaEventRecord(s->ev_join, s2));
    PG_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
    g_trace.mark("row_ptr arrived (s2)", s2);
    h2d(t_cols, p->col_idx, sizeof(int32_t) * nnz, st);
    cudaEvent_t ev_cols = nullptr;
    PG_CUDA(cudaEventCreateWithFlags(&ev_cols, cudaEventDisableTiming));
    PG_CUDA(cudaEventRecord(ev_cols, st));
    h2d(t_vals, p->values, sizeof(double) * nnz, st);
    h2d(t_lhs, p->lhs, sizeof(double) * m, st);
    h2d(t_rhs, p->rhs, sizeof(double) * m, st);
    h2d(s->d_integral, p->integral, n, st);
    g_trace.mark("h2d matrix done (st)", st);

    // stream 2, concurrently: row order.  Short rows (<= short_max entries)
    // grouped by exact length (stable radix sort), then the rows split into
    // segments in input order.  Row order is not observable -- candidates
    // merge by exact max/min and each row is summed on its own.
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    auto cub_tmp = [&](size_t need) {
      if (need > tmp_bytes) {
        cudaStream_t prev = t_alloc_stream;
        t_alloc_stream = s2;
        dfree(tmp);
        tmp = dalloc<unsigned char>(need);
        tmp_bytes = need;
        t_alloc_stream = prev;
      }
    };
    std::vector<int32_t> cls(kMaxClasses + 5, 0);
    if (m) {
      PG_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (kMaxClasses + 5), s2));
      k_row_keys<<<s->grid_for(m, 256), 256, 0, s2>>>(t_rp, m, nnz, short_max, key, idx,
                                                      counts + kMaxClasses + 4);
      size_t need = 0;
      PG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, idx, t_perm, m, 0, 5, s2));
      cub_tmp(need);
      PG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, need, key, key2, idx, t_perm, m, 0, 5, s2));
      g_trace.mark("row sort (s2)", s2);
      k_sorted_len<<<s->grid_for((int64_t)m + 1, 256), 256, 0, s2>>>(t_rp, t_perm, m, slen);
      PG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, slen, s->d_row_ptr, m + 1, s2));
      cub_tmp(need);
      PG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, need, slen, s->d_row_ptr, m + 1, s2));
      k_class_counts<<<s->grid_for(m, 256), 256, 0, s2>>>(key2, m, counts);
      auto* len2 = reinterpret_cast<unsigned long long*>(counts + kMaxClasses + 2);
      k_len2_sum<<<s->grid_for(m, 256), 256, 0, s2>>>(t_rp, m, len2);
      g_trace.mark("class counts (s2)", s2);
      PG_CUDA(cudaMemcpyAsync(cls.data(), counts, sizeof(int32_t) * (kMaxClasses + 5),
                              cudaMemcpyDeviceToHost, s2));
      g_trace.mark("counts d2h (s2)", s2);
      PG_CUDA(cudaStreamSynchronize(s2));
      unsigned long long l2 = 0;
      if (cls[kMaxClasses + 4])
        throw Error{PG_EINVAL, "row_ptr must be non-decreasing with entries in [0, nnz]"};
      std::memcpy(&l2, cls.data() + kMaxClasses + 2, sizeof(l2));
      s->row_density = (double)l2 / std::max(1.0, (double)n * (double)nnz);
    }
    TileLayout lay{};
    lay.nclass = short_max + 1;
    {
      int32_t row = 0;
      for (int32_t L = 0; L <= short_max; ++L) {
        lay.class_start[L] = row;
        row += cls[L];
      }
      lay.class_start[short_max + 1] = row;
      s->short_rows = row;
      s->nsrow = m - row;
    }
    // the ordering's buffers come from stream 2's allocation order, so it
    // never waits behind the upload on stream 1
    t_alloc_stream = s2;
    s->d_srow = dalloc<int32_t>(s->nsrow);
    s->d_sfirst = dalloc<int32_t>((size_t)s->nsrow + 1);
    int32_t* scnt = dalloc<int32_t>((size_t)s->nsrow + 1);
    int32_t h_nseg = 0;
    if (s->nsrow) {
      k_seg_counts<<<s->grid_for((int64_t)s->nsrow + 1, 256), 256, 0, s2>>>(
          s->d_row_ptr, (int)s->short_rows, s->nsrow, chunk, scnt, s->d_srow);
      size_t need = 0;
      PG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, scnt, s->d_sfirst, s->nsrow + 1, s2));
      cub_tmp(need);
      PG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, need, scnt, s->d_sfirst, s->nsrow + 1, s2));
      PG_CUDA(cudaMemcpyAsync(&h_nseg, s->d_sfirst + s->nsrow, sizeof(int32_t), cudaMemcpyDeviceToHost, s2));
      PG_CUDA(cudaStreamSynchronize(s2));
    }
    s->nseg = h_nseg;
    for (int32_t L = 0; L <= short_max; ++L) s->short_nnz += (int64_t)L * cls[L];
    s->seg_nnz = nnz - s->short_nnz;
    s->d_segs = dalloc<SegDesc>(s->nseg);
    SegDesc* segs_in = dalloc<SegDesc>(s->nseg);
    uint32_t* skey = dalloc<uint32_t>(s->nseg);
    uint32_t* skey2 = dalloc<uint32_t>(s->nseg);
    int32_t* sidx = dalloc<int32_t>(s->nseg);
    int32_t* sorder = dalloc<int32_t>(s->nseg);
    if (s->nseg) {
      k_emit_segs<<<s->grid_for((int64_t)s->nsrow * 32, 256, 16), 256, 0, s2>>>(
          s->d_row_ptr, s->d_sfirst, (int)s->short_rows, s->nsrow, chunk, segs_in, skey, sidx);
      int bits = 1;
      while (bits < 32 && (1u << bits) <= (uint32_t)chunk) ++bits;
      size_t need = 0;
      PG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, skey, skey2, sidx, sorder, s->nseg, 0,
                                              bits, s2));
      cub_tmp(need);
      PG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, need, skey, skey2, sidx, sorder, s->nseg, 0,
                                              bits, s2));
      k_order_segs<<<s->grid_for(s->nseg, 256), 256, 0, s2>>>(segs_in, sorder, s->nseg, s->d_segs);
    }
    PG_CUDA(cudaGetLastError());
    t_alloc_stream = st;
    tm.lap("ordering + tables (dev)");

    s->d_colx = dalloc<int32_t>(nnz + 4);  // +16 B: bulk copies round up to 16 B
    s->d_vals = dalloc<double>(nnz + 2);
    s->d_lhs = dalloc<double>((size_t)m + 2);
    s->d_rhs = dalloc<double>((size_t)m + 2);
    s->d_snap = dalloc<Snap>((size_t)n + 1);  // + the padding column of the sliced-ELL copy
    {
      // bounds [0, 0] (a padding entry adds +0.0) and q = -inf (its filter
      // term 0 * -inf is NaN, which fmax ignores)
      static const Snap pad = {0.0, 0.0, -std::numeric_limits<double>::infinity(), 0};
      PG_CUDA(cudaMemcpyAsync(s->d_snap + n, &pad, sizeof(Snap), cudaMemcpyHostToDevice, st));
      s->d_bnd = dalloc<double2>((size_t)n + 1);
      PG_CUDA(cudaMemsetAsync(s->d_bnd + n, 0, sizeof(double2), st));
      static const char* ge = getenv("PG_SELL_GATHER");  // "8": forced (tests, A/B)
      if ((ge && atoi(ge) == 8) || (s->many_cols() && float_bounds_sample(p))) {
        s->d_bf = dalloc<float2>((size_t)n + 1);
        PG_CUDA(cudaMemsetAsync(s->d_bf + n, 0, sizeof(float2), st));
        s->dcfg.bf = s->d_bf;
      }
    }
    s->d_key_out = dalloc<longlong2>((size_t)n + 1);  // + infeasibility slot
    s->d_lo0 = dalloc<double>(n);
    s->d_up0 = dalloc<double>(n);
    s->d_lo_res = dalloc<double>(n);
    s->d_up_res = dalloc<double>(n);
    s->d_partial = dalloc<SegPartial>(s->nseg);
    // phase-2 queues: every row at most once; a long row in pieces
    s->d_ract = dalloc<Act>(m);
    s->d_wl_short = dalloc<int32_t>(m);
    s->wl_long_cap = nnz / kCandShort + nnz / kCandPiece + 1;
    s->d_wl_long = dalloc<CandItem>(s->wl_long_cap);
    s->d_row_done = dalloc<int32_t>(s->nsrow);
    s->d_st = dalloc<DevState>(1);
    s->d_ctl = dalloc<NodeCtl>(1);
    s->d_per_round = dalloc<long long>(cfg->round_limit);
    PG_CUDA(cudaMemsetAsync(s->d_ctl, 0, sizeof(NodeCtl), st));  // cold starts
    PG_CUDA(cudaMemsetAsync(s->d_st, 0, sizeof(DevState), st));
    PG_CUDA(cudaMemsetAsync(s->d_row_done, 0, sizeof(int32_t) * std::max<int32_t>(1, s->nsrow), st));
    // the start bounds follow the matrix on the copy engine (stream 2) while
    // stream 1 permutes the matrix and fills the sliced-ELL copy
    cudaEvent_t ev_mat = nullptr, ev_bnd = nullptr;
    PG_CUDA(cudaEventCreateWithFlags(&ev_mat, cudaEventDisableTiming));
    PG_CUDA(cudaEventCreateWithFlags(&ev_bnd, cudaEventDisableTiming));
    PG_CUDA(cudaEventRecord(ev_mat, st));
    t_alloc_stream = s2;
    s->d_split = dalloc<int32_t>(std::max<int32_t>(1, s->nsrow) + 1);
    if (s->nsrow) {
      int32_t* cnt = s->d_split + s->nsrow;  // the count rides at the end
      PG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t), s2));
      k_split_list<<<s->grid_for(s->nsrow, 256), 256, 0, s2>>>(s->d_sfirst, s->nsrow, s->d_split, cnt);
      PG_CUDA(cudaMemcpyAsync(&s->nsplit, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, s2));
      PG_CUDA(cudaStreamSynchronize(s2));
    }
    t_alloc_stream = st;
    PG_CUDA(cudaMemsetAsync(s->d_colx, 0, sizeof(int32_t) * (nnz + 4), st));
    PG_CUDA(cudaMemsetAsync(s->d_vals, 0, sizeof(double) * (nnz + 2), st));
    // sliced-ELL tables (units, regions, slice descriptors) depend on the
    // ordering only: built on stream 2 while the upload is still running
    UnitDesc* u_in = nullptr;
    int32_t *k0_in = nullptr, *uk0 = nullptr, *uidx = nullptr, *uord = nullptr, *rcnt = nullptr;
    uint32_t *ukey = nullptr, *ukey2 = nullptr;
    long long *elems = nullptr, *soff = nullptr, total = 0;
    void *stmp = nullptr, *stmp2 = nullptr;
    t_alloc_stream = s2;
    // sliced-ELL copy (sell.cuh): units sorted by length, slices per
    // lanes-per-unit region, transposed fill
    s->nunits = s->nseg + (int32_t)s->short_rows;
    if (s->nunits) {
      const int32_t nu = s->nunits;
      u_in = dalloc<UnitDesc>(nu);
      k0_in = dalloc<int32_t>(nu);
      uk0 = dalloc<int32_t>(nu);
      ukey = dalloc<uint32_t>(nu);
      ukey2 = dalloc<uint32_t>(nu);
      uidx = dalloc<int32_t>(nu);
      uord = dalloc<int32_t>(nu);
      rcnt = dalloc<int32_t>(5);
      s->d_units = dalloc<UnitDesc>(nu);
      PG_CUDA(cudaMemsetAsync(rcnt, 0, sizeof(int32_t) * 5, s2));
      k_make_units<<<s->grid_for(nu, 256), 256, 0, s2>>>(s->d_segs, s->nseg, s->d_srow, s->d_sfirst,
                                                           lay, s->d_row_ptr, nu, chunk, u_in, k0_in,
                                                           ukey, uidx);
      int bits = 1;
      while (bits < 32 && (1u << bits) <= (uint32_t)chunk) ++bits;
      size_t need = 0;
      PG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, ukey, ukey2, uidx, uord, nu, 0, bits, s2));
      stmp = dalloc<unsigned char>(need);
      PG_CUDA(cub::DeviceRadixSort::SortPairs(stmp, need, ukey, ukey2, uidx, uord, nu, 0, bits, s2));
      k_order_units<<<s->grid_for(nu, 256), 256, 0, s2>>>(u_in, k0_in, uord, nu, s->d_units, uk0);
      // lanes per unit at least 2^lg_min: a small instance spreads its chains
      // so that about one slice per resident warp remains
      const int64_t resident = (int64_t)s->num_sms * s->sell_per_sm * kSellWarps;
      int lg_min = 0;
      while (lg_min < 3 && ((int64_t)nu << lg_min) < resident * 32) ++lg_min;
      s->lg_min = lg_min;
      k_unit_regions<<<s->grid_for(nu, 256), 256, 0, s2>>>(s->d_units, nu, lg_min, rcnt);
      int32_t hc[5] = {0, 0, 0, 0, 0};
      PG_CUDA(cudaMemcpyAsync(hc, rcnt, sizeof(hc), cudaMemcpyDeviceToHost, s2));
      PG_CUDA(cudaStreamSynchronize(s2));
      SellRegions R{};
      R.ustart[0] = 0;
      R.ustart[1] = hc[3];
      R.ustart[2] = std::max(hc[2], R.ustart[1]);
      R.ustart[3] = std::max(hc[1], R.ustart[2]);
      R.ustart[4] = nu;
      R.sstart[0] = 0;
      for (int k = 0; k < 4; ++k) {
        const int H = 32 >> (3 - k);
        R.sstart[k + 1] = R.sstart[k] + (R.ustart[k + 1] - R.ustart[k] + H - 1) / H;
      }
      s->nslices = R.sstart[4];
      s->lg0_ustart = R.ustart[3];
      s->lg0_sstart = R.sstart[3];
      // narrow one-lane slices are handed out in groups (sell_group): the
      // first slice of region 0 whose units are all <= PG_SELL_GROUPW long
      s->group_start = s->nslices;
      if (R.ustart[4] > R.ustart[3]) {
        const int ub = std::max(hc[4], R.ustart[3]);  // first unit <= the grouping width
        s->group_start = std::min(s->nslices, R.sstart[3] + (ub - R.ustart[3] + 31) / 32);
      }
      s->d_slices = dalloc<SliceDesc>(s->nslices);
      elems = dalloc<long long>((size_t)s->nslices + 1);
      soff = dalloc<long long>((size_t)s->nslices + 1);
      k_slice_desc<<<s->grid_for((int64_t)s->nslices + 1, 256), 256, 0, s2>>>(s->d_units, R,
                                                                              s->d_slices, elems);
      need = 0;
      PG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, elems, soff, s->nslices + 1, s2));
      stmp2 = dalloc<unsigned char>(need);
      PG_CUDA(cub::DeviceScan::ExclusiveSum(stmp2, need, elems, soff, s->nslices + 1, s2));
      total = 0;
      PG_CUDA(cudaMemcpyAsync(&total, soff + s->nslices, sizeof(long long), cudaMemcpyDeviceToHost, s2));
      PG_CUDA(cudaStreamSynchronize(s2));
    }
    t_alloc_stream = st;
    // worklist: the column index from the caller's row order (rows renamed
    // through the inverse permutation) on stream 2 as soon as the column
    // indices have arrived, while the values are still uploading
    if ((cfg->flags & PG_FLAG_WORKLIST) && m) {
      t_alloc_stream = s2;
      int32_t* inv = dalloc<int32_t>(m);
      k_invert_perm<<<s->grid_for(m, 256), 256, 0, s2>>>(t_perm, m, inv);
      g_trace.mark("ordering (s2)", s2);
      PG_CUDA(cudaStreamWaitEvent(s2, ev_cols, 0));
      g_trace.mark("cols arrived (s2)", s2);
      s->build_col_index(t_rp, t_cols, inv, s2);
      dfree(inv);
      t_alloc_stream = st;
    }
    // the ordering (stream 2) must be complete before the permutation
    g_trace.mark("ordering+colindex (s2)", s2);
    PG_CUDA(cudaEventRecord(s->ev_join, s2));
    PG_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
    PG_CUDA(cudaStreamWaitEvent(s2, ev_mat, 0));
    h2d(s->d_lo0, p->lower, sizeof(double) * n, s2);
    h2d(s->d_up0, p->upper, sizeof(double) * n, s2);
    g_trace.mark("bounds h2d (s2)", s2);
    PG_CUDA(cudaEventRecord(ev_bnd, s2));
    if (m) {
      k_permute_rows<<<s->grid_for(std::max<int64_t>(m, nnz * 32 / kWalkChunk + 1), 256, 16), 256, 0, st>>>(
          t_rp, t_cols, t_vals, t_lhs, t_rhs, t_perm, s->d_row_ptr, s->d_integral, s->d_colx,
          s->d_vals, s->d_lhs, s->d_rhs, m, n, cfg->infinity_threshold, s->d_st);
      PG_CUDA(cudaGetLastError());
    }
    g_trace.mark("permute", st);
    if (cfg->scalar_mode == PG_NARROW32) {
      // the float working copy (engine_common.hpp:24-38) and chunk scratch
      k_to_f32<<<s->grid_for(nnz, 256), 256, 0, st>>>(s->d_vals, nnz);
      k_to_f32<<<s->grid_for(m, 256), 256, 0, st>>>(s->d_lhs, m);
      k_to_f32<<<s->grid_for(m, 256), 256, 0, st>>>(s->d_rhs, m);
      // row records and chunk partials of the sliced-ELL float round
      // (PG_F32_ROWS=1: the one-thread-per-row kernel instead, for A/B)
      if (!getenv("PG_F32_ROWS")) {
        s->d_ractf = dalloc<ActF>(std::max<int32_t>(m, 1));
        s->d_partf = dalloc<ActF>(std::max<int32_t>(s->nseg, 1));
      } else {
        const int chunk = cfg->nnz_budget;
        s->f32_maxc = s->max_len() > chunk ? (s->max_len() + chunk - 1) / chunk : 1;
        s->d_f32_part = dalloc<ActF>((size_t)s->grid_for(m, 256, 4) * 256 * s->f32_maxc);
      }
      PG_CUDA(cudaGetLastError());
    }
    if (s->nunits) {
      s->sell_elems = total;
      s->d_sv = dalloc<double>((size_t)total + 1);
      s->d_sc = dalloc<int32_t>((size_t)total + 1);
      s->d_sw = dalloc<uint32_t>((size_t)total + 1);
      k_fill_sell<<<s->grid_for((int64_t)s->nslices * 32, 256, 16), 256, 0, st>>>(
          s->d_units, uk0, s->nslices, soff, s->d_vals, s->d_colx, n, s->d_slices, s->d_sv, s->d_sc);
      PG_CUDA(cudaGetLastError());
      for (void* q : {(void*)u_in, (void*)k0_in, (void*)uk0, (void*)ukey, (void*)ukey2, (void*)uidx,
                      (void*)uord, (void*)rcnt, (void*)elems, (void*)soff, stmp, stmp2})
        dfree(q);
    }
    for (void* q : {(void*)key, (void*)key2, (void*)idx, (void*)slen, (void*)counts, (void*)scnt,
                    (void*)segs_in, (void*)skey, (void*)skey2, (void*)sidx, (void*)sorder,
                    tmp})
      dfree(q);
    g_trace.mark("fill sell", st);
    tm.lap("H2D + permute (queued)");
    // worklist index: column -> work items (device counting sort by column)
    {
      Dirty& D = s->dirty;
      D.m = m;
      D.ms = (m + 15) & ~15;
      D.n = n;
      D.first_seg_row = (int32_t)s->short_rows;
      D.enabled = (cfg->flags & PG_FLAG_WORKLIST) != 0;
      s->d_flags = dalloc<uint8_t>(2 * (size_t)D.ms + 16);
      D.row_flag = s->d_flags;
      if (D.enabled) {
        s->d_chg = dalloc<int32_t>(2 * (size_t)n);
        D.chg_list = s->d_chg;
        s->ensure_col_index();
        // dirty-slice lists of worklist rounds (sell.cuh)
        s->d_row_unit = dalloc<int32_t>(m);
        s->d_part_unit = dalloc<int32_t>(s->nseg);
        s->d_unit_slice = dalloc<int32_t>(s->nunits);
        s->d_wide_list = dalloc<int32_t>(2 * (size_t)s->nunits);
        s->d_unit_list = dalloc<int32_t>(2 * (size_t)s->nunits);
        PG_CUDA(cudaMemsetAsync(s->d_row_unit, 0xff, sizeof(int32_t) * std::max<int32_t>(m, 1), st));
        // round-kind heuristics (tuned on C2 / C5; environment overrides for
        // A/B).  per = the changed columns that mark about every row (mean
        // column degree nnz / n).  The next round is a full sweep when more
        // than per / PG_DENSE_DIV columns changed, or when the changed
        // columns' entries times the mean unit weight exceed PG_DENSE_DEG x
        // the unit count (marks and marked rows are cheap for C5's mid-length
        // rows, dear for C2's lane units); a full sweep after more than
        // PG_LIST_GATE x per changes builds no changed-column list.
        const double per = (double)m * (double)n / (double)std::max<int64_t>(nnz, 1);
        auto envd = [](const char* k, double d) { return getenv(k) ? atof(getenv(k)) : d; };
        static const double div = envd("PG_DENSE_DIV", 1.0), fdeg = envd("PG_DENSE_DEG", 1.0),
                            gate = envd("PG_LIST_GATE", 1.0);
        D.dense_nchg = (int32_t)std::min<double>(2e9, per / div);
        D.dense_deg = fdeg * (double)m;  // compared with entries x wsum / nunits
        D.list_gate = (long long)std::min<double>(9e18, gate * per);
        D.mark_batch = getenv("PG_MARK_BATCH") ? std::max(1, atoi(getenv("PG_MARK_BATCH"))) : 1;
        // a worklist round while the marked lane, long and mid units, weighted,
        // stay below the weighted unit count (round_is_sparse)
        int w[4] = {8, 32, 2, 1};
        if (const char* e = getenv("PG_WL_WEIGHTS")) sscanf(e, "%d,%d,%d,%d", &w[0], &w[1], &w[2], &w[3]);
        D.w_lane = w[0];
        D.w_wide = w[1];
        D.w_mid = w[2];
        D.w_all = w[3];
        if (s->nunits) {
          k_unit_maps<<<s->grid_for(s->nunits, 256), 256, 0, st>>>(s->d_units, s->nunits, s->d_segs,
                                                                 s->d_row_unit, s->d_part_unit);
          k_slice_units<<<s->grid_for(s->nslices, 256), 256, 0, st>>>(
              s->d_slices, s->nslices, s->d_units, s->d_unit_slice, D, s->d_st);
        }
        PG_CUDA(cudaGetLastError());
        D.row_unit = s->d_row_unit;
        D.part_unit = s->d_part_unit;
        D.sfirst = s->d_sfirst;
        D.unit_slice = s->d_unit_slice;
        D.wide_list = s->d_wide_list;
        s->d_tflag = dalloc<uint32_t>(n);
        s->d_tlist = dalloc<int32_t>(n);
        PG_CUDA(cudaMemsetAsync(s->d_tflag, 0, sizeof(uint32_t) * std::max(n, 1), st));
        s->touch = Touch{s->d_tflag, s->d_tlist, &s->d_st->ntouch};
        D.nslices = s->nslices;
        D.unit_list = s->d_unit_list;
        D.nunits = s->nunits;
      }
    }
    g_trace.mark("worklist maps", st);
    PG_CUDA(cudaStreamWaitEvent(st, ev_bnd, 0));
    s->normalize_bounds();
    g_trace.mark("bounds normalised", st);
    PG_CUDA(cudaGetLastError());
    // everything after this point is ordered on the session stream: no host
    // sync (the graph is instantiated while the GPU finishes the setup)
    for (void* q : {(void*)t_rp, (void*)t_cols, (void*)t_vals, (void*)t_lhs, (void*)t_rhs,
                    (void*)t_perm})
      dfree(q);
    tm.lap("worklist/bounds (queued)");
    // keep the gathered records resident in a persisting L2 carve-out while
    // the matrix streams through: by default for the 8 B float records (C5:
    // a 40 MB window in a 42 MB carve-out, first round 931 -> 878 us, solve
    // 7.47 -> 7.20 ms; a 64 MB carve-out 7.77 ms; the
    // 32 B / 16 B records measured slower with one, section 4 of DESIGN.md)
    {
      size_t want = 0;
      if (const char* e = getenv("PG_L2_PERSIST_MB")) want = (size_t)atoi(e) << 20;
      else if (s->gather_kind() == 2) want = sizeof(float2) * ((size_t)n + 1) * 21 / 20;
      int maxp = 0, maxw = 0;
      PG_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, s->dev));
      PG_CUDA(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, s->dev));
      want = std::min(want, (size_t)std::min(maxp, maxw));
      if (want) {
        s->l2_window = true;
        PG_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
        cudaStreamAttrValue av = {};
        // the array the full sweep gathers from: 16 B bounds or 32 B records
        const int gk = s->gather_kind();
        av.accessPolicyWindow.base_ptr = gk == 2 ? (void*)s->d_bf : gk == 1 ? (void*)s->d_bnd : (void*)s->d_snap;
        av.accessPolicyWindow.num_bytes =
            std::min((gk == 2 ? sizeof(float2) : gk == 1 ? sizeof(double2) : sizeof(Snap)) * ((size_t)n + 1), want);
        av.accessPolicyWindow.hitRatio = 1.0f;
        av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        PG_CUDA(cudaStreamSetAttribute(s->stream, cudaStreamAttributeAccessPolicyWindow, &av));
      }
    }
    cudaEventDestroy(ev_cols);
    cudaEventDestroy(ev_mat);
    cudaEventDestroy(ev_bnd);
    if (cfg->loop_mode == PG_LOOP_GRAPH) s->build_graph();
    tm.lap("graph instantiate");
    return s;
  } catch (...) {
    delete s;
    throw;
  }
}

// One-shot calls (pg_propagate) hand their finished session to a reaper
// thread: graph, streams, events, pinned and pool memory are released off
// the caller's critical path (~0.3 ms).  At most a few sessions wait; beyond
// that the caller releases its own.  An atexit hook drains the queue on the
// main thread before the CUDA runtime shuts down.
struct Reaper {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<pg_session*> q;
  int busy = 0;
  bool started = false, stop = false;
  void run() {
    std::unique_lock<std::mutex> lk(mu);
    for (;;) {
      cv.wait(lk, [&] { return stop || !q.empty(); });
      if (q.empty()) return;
      pg_session* s = q.front();
      q.pop_front();
      ++busy;
      lk.unlock();
      delete s;
      lk.lock();
      --busy;
      cv.notify_all();
    }
  }
  bool push(pg_session* s) {
    std::lock_guard<std::mutex> lk(mu);
    if (stop || q.size() >= 2) return false;
    if (!started) {
      started = true;
      std::thread([this] { run(); }).detach();
      std::atexit([] { reaper().drain(); });
    }
    q.push_back(s);
    cv.notify_all();
    return true;
  }
  void drain() {
    std::unique_lock<std::mutex> lk(mu);
    stop = true;
    cv.notify_all();
    cv.wait(lk, [&] { return busy == 0; });
    while (!q.empty()) {
      pg_session* s = q.front();
      q.pop_front();
      delete s;
    }
  }
  static Reaper& reaper() {
    static Reaper* r = new Reaper;  // never destroyed: the detached thread may outlive statics
    return *r;
  }
};

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return PG_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PG_ECUDA;
  }
}

}  // namespace

extern "C" {

void pg_config_default(pg_config* c) {
  c->round_limit = 100;
  c->infinity_threshold = 1e20;
  c->improvement_abs = 1e-7;
  c->improvement_rel = 1e-7;
  c->integrality_eps = 1e-6;
  c->nnz_budget = 1024;
  c->vector_threshold = 64;
  c->worker_count = 0;
  c->scalar_mode = PG_WIDE64;
  c->device = 0;
  c->loop_mode = PG_LOOP_GRAPH;
  c->flags = PG_FLAG_ROWCHECK;
}

int pg_config_validate(const pg_config* cfg) {
  if (!cfg) {
    g_err = "config is NULL";
    return PG_EINVAL;
  }
  return validate(cfg);
}

namespace {
// session setup without the final wait: the one-shot calls (pg_propagate,
// pg_round) go straight on to the solve, which syncs before they return
int session_create_async(const pg_problem* p, const pg_config* cfg, pg_session** out) {
  if (!out) {
    g_err = "out is NULL";
    return PG_EINVAL;
  }
  *out = nullptr;
  const int rc = pg_config_validate(cfg);
  if (rc) return rc;
  return guarded([&] {
    *out = create_session(p, cfg);
    return PG_OK;
  });
}
}  // namespace

int pg_session_create(const pg_problem* p, const pg_config* cfg, pg_session** out) {
  int rc = session_create_async(p, cfg, out);
  if (rc) return rc;
  // the caller's arrays (pinned ones are copied asynchronously) may be freed
  // or reused as soon as this returns
  rc = guarded([&] {
    PG_CUDA(cudaStreamSynchronize((*out)->stream2));
    PG_CUDA(cudaStreamSynchronize((*out)->stream));
    return PG_OK;
  });
  if (rc) {
    pg_session_destroy(*out);
    *out = nullptr;
  }
  return rc;
}

void pg_session_destroy(pg_session* s) { delete s; }

int pg_session_run(pg_session* s, pg_result* res) {
  if (!s || !res) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  return guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    const int64_t ns = s->run_solve(true, res);
    s->fill_result(res, ns);
    return PG_OK;
  });
}

int pg_session_propagate(pg_session* s, const double* lower, const double* upper, pg_result* res) {
  if (!s || !res) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  return guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    if (lower || upper) {
      if (!lower || !upper) throw Error{PG_EINVAL, "lower and upper must both be given"};
      s->upload_bounds(lower, upper);
    }
    const int64_t ns = s->run_solve(true, res);
    s->fill_result(res, ns);
    return PG_OK;
  });
}

int pg_session_round(pg_session* s, const double* lb_in, const double* ub_in, double* lb_out,
                     double* ub_out, int32_t* changed, int32_t* infeasible, int64_t* changes) {
  // propagate_round_parallel (par_engine.cpp:277-312) on a resident session:
  // one round on the caller snapshot, no bounds_crossed pre-check, no row
  // check, in double; the matrix setup is paid once per session, not per call
  if (!s || !lb_in || !ub_in || !lb_out || !ub_out || !changed || !infeasible || !changes) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  if (s->cfg.scalar_mode != PG_WIDE64) {
    g_err = "pg_session_round needs a Wide64 session (propagate_round_parallel works in double)";
    return PG_EINVAL;
  }
  if (s->comm) {
    g_err = "pg_session_round: row-sharded sessions are not supported";
    return PG_EINVAL;
  }
  return guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    // the caller's snapshot replaces the start bounds for this round only:
    // later pg_session_run / propagate calls start from the session's own
    if (!s->d_keep_lo) {
      s->d_keep_lo = dalloc<double>(s->n);
      s->d_keep_up = dalloc<double>(s->n);
    }
    PG_CUDA(cudaMemcpyAsync(s->d_keep_lo, s->d_lo0, sizeof(double) * s->n, cudaMemcpyDeviceToDevice, s->stream));
    PG_CUDA(cudaMemcpyAsync(s->d_keep_up, s->d_up0, sizeof(double) * s->n, cudaMemcpyDeviceToDevice, s->stream));
    s->upload_bounds(lb_in, ub_in);
    const pg_config saved = s->cfg;
    const DevCfg dsaved = s->dcfg;
    s->cfg.flags &= ~PG_FLAG_ROWCHECK;
    s->dcfg.flags = s->cfg.flags;
    s->dcfg.round_limit = 1;
    struct Restore {
      pg_session* s;
      pg_config c;
      DevCfg d;
      ~Restore() {
        s->cfg = c;
        s->dcfg = d;
      }
    } restore{s, saved, dsaved};
    PG_CUDA(cudaMemsetAsync(s->d_ctl, 0, sizeof(NodeCtl), s->stream));  // a cold start
    s->enqueue_reset(false, false);
    s->enqueue_round(false);
    long long ch = 0;
    PG_CUDA(cudaMemcpyAsync(&ch, s->d_per_round, sizeof(long long), cudaMemcpyDeviceToHost, s->stream));
    PG_CUDA(cudaMemcpyAsync(s->h_st, s->d_st, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    k_decode<<<s->grid_for(s->n, 256), 256, 0, s->stream>>>(s->d_key_out, s->d_lo_res, s->d_up_res,
                                                            s->n);
    PG_CUDA(cudaGetLastError());
    PG_CUDA(cudaMemcpyAsync(lb_out, s->d_lo_res, sizeof(double) * s->n, cudaMemcpyDeviceToHost,
                            s->stream));
    PG_CUDA(cudaMemcpyAsync(ub_out, s->d_up_res, sizeof(double) * s->n, cudaMemcpyDeviceToHost,
                            s->stream));
    PG_CUDA(cudaMemcpyAsync(s->d_lo0, s->d_keep_lo, sizeof(double) * s->n, cudaMemcpyDeviceToDevice, s->stream));
    PG_CUDA(cudaMemcpyAsync(s->d_up0, s->d_keep_up, sizeof(double) * s->n, cudaMemcpyDeviceToDevice, s->stream));
    PG_CUDA(cudaStreamSynchronize(s->stream));
    s->check_input();
    *changes = ch;
    *changed = ch > 0;
    *infeasible = s->h_st->status == PG_INFEASIBLE;
    return PG_OK;
  });
}

int pg_propagate(const pg_problem* p, const pg_config* cfg, pg_result* res) {
  if (!res) {
    g_err = "result is NULL";
    return PG_EINVAL;
  }
  pg_session* s = nullptr;
  int rc = session_create_async(p, cfg, &s);
  if (rc) return rc;
  PhaseTimer tm;
  rc = pg_session_run(s, res);
  tm.lap("solve + download");
  g_trace.dump();
  s->release_buffers();
  if (!Reaper::reaper().push(s)) pg_session_destroy(s);
  tm.lap("destroy (handed off)");
  return rc;
}

int pg_round(const pg_problem* p, const pg_config* cfg, const double* lb_in, const double* ub_in,
             double* lb_out, double* ub_out, int32_t* changed, int32_t* infeasible,
             int64_t* changes) {
  if (!p || !cfg || !lb_in || !ub_in || !lb_out || !ub_out || !changed || !infeasible || !changes) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  int rc = pg_config_validate(cfg);
  if (rc) return rc;
  // propagate_round_parallel: one cpu_par round on the caller snapshot, no
  // bounds_crossed pre-check and no row check (par_engine.cpp:277-312)
  pg_config c = *cfg;
  c.round_limit = 1;
  c.loop_mode = PG_LOOP_HOST;
  c.scalar_mode = PG_WIDE64;  // propagate_round_parallel always works in double (par_engine.cpp:282)
  c.flags &= ~PG_FLAG_ROWCHECK;
  pg_problem q = *p;
  q.lower = lb_in;
  q.upper = ub_in;
  pg_session* s = nullptr;
  rc = session_create_async(&q, &c, &s);
  if (rc) return rc;
  rc = guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    s->run_solve(false);
    long long ch = 0;
    PG_CUDA(cudaMemcpy(&ch, s->d_per_round, sizeof(long long), cudaMemcpyDeviceToHost));
    pg_result r = {};
    r.lower = lb_out;
    r.upper = ub_out;
    s->fill_result(&r, 0);
    *changes = ch;
    *changed = ch > 0;
    *infeasible = r.status == PG_INFEASIBLE;
    return PG_OK;
  });
  pg_session_destroy(s);
  return rc;
}

int pg_csr_from_triplets(int32_t num_rows, int32_t num_cols, int64_t count, const int32_t* rows,
                         const int32_t* cols, const double* values, int32_t device,
                         int32_t* row_ptr, int32_t* col_idx, double* values_out, int64_t* nnz) {
  // csr_from_triplets (core/src/model.cpp:37-80) on the device (ingest.cuh)
  if (!row_ptr || !nnz || (count > 0 && (!rows || !cols || !values || !col_idx || !values_out))) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  if (num_rows < 0 || num_cols < 0 || count < 0 || count > 0x7fffffffLL) {
    g_err = "triplet count or dimensions out of the int32 range";
    return PG_EINVAL;
  }
  return guarded([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error{PG_ENODEV, "no CUDA device visible (the B200 engine has no CPU fallback)"};
    if (device < 0 || device >= ndev) throw Error{PG_EINVAL, "device ordinal out of range"};
    const DevInfo prop = device_info(device);
    PG_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    PG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    t_alloc_stream = st;
    std::vector<void*> owned;
    auto cleanup = [&] {
      for (void* q : owned) dfree(q);
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    };
    try {
      const int64_t m = num_rows;
      auto grid = [&](int64_t items) {
        return (int)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)prop.sms * 8));
      };
      auto alloc = [&](size_t bytes) {
        void* q = dalloc<unsigned char>(bytes);
        owned.push_back(q);
        return q;
      };
      int32_t* d_rows = (int32_t*)alloc(4 * (size_t)count);
      int32_t* d_cols = (int32_t*)alloc(4 * (size_t)count);
      double* d_vals = (double*)alloc(8 * (size_t)count);
      auto* d_bad = (unsigned long long*)alloc(8);
      int32_t* d_rcnt = (int32_t*)alloc(4 * ((size_t)m + 1));
      if (count) {
        PG_CUDA(cudaMemcpyAsync(d_rows, rows, 4 * (size_t)count, cudaMemcpyHostToDevice, st));
        PG_CUDA(cudaMemcpyAsync(d_cols, cols, 4 * (size_t)count, cudaMemcpyHostToDevice, st));
        PG_CUDA(cudaMemcpyAsync(d_vals, values, 8 * (size_t)count, cudaMemcpyHostToDevice, st));
      }
      PG_CUDA(cudaMemsetAsync(d_bad, 0xff, 8, st));
      PG_CUDA(cudaMemsetAsync(d_rcnt, 0, 4 * ((size_t)m + 1), st));
      unsigned long long bad = ~0ull;
      if (count) {
        k_trip_check<<<grid(count), 256, 0, st>>>(d_rows, d_cols, count, num_rows, num_cols, d_bad);
        PG_CUDA(cudaGetLastError());
        PG_CUDA(cudaMemcpyAsync(&bad, d_bad, 8, cudaMemcpyDeviceToHost, st));
        PG_CUDA(cudaStreamSynchronize(st));
      }
      if (bad != ~0ull) {
        // the reference checks the row of a triplet before its column
        const int32_t r = rows[bad];
        throw Error{PG_ERANGE, r < 0 || r >= num_rows ? "triplet row index out of range"
                                                      : "triplet column index out of range"};
      }
      int colbits = 1, rowbits = 1;
      while (colbits < 31 && (1ll << colbits) < num_cols) ++colbits;
      while (rowbits < 31 && (1ll << rowbits) < num_rows) ++rowbits;
      int64_t kept = 0;
      if (count) {
        auto* key = (unsigned long long*)alloc(8 * (size_t)count);
        auto* key2 = (unsigned long long*)alloc(8 * (size_t)count);
        double* val2 = (double*)alloc(8 * (size_t)count);
        double* sum = (double*)alloc(8 * (size_t)count);
        int32_t* keep = (int32_t*)alloc(4 * (size_t)count + 4);
        int32_t* pos = (int32_t*)alloc(4 * (size_t)count + 4);
        k_trip_keys<<<grid(count), 256, 0, st>>>(d_rows, d_cols, count, colbits, key);
        size_t need = 0;
        PG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, d_vals, val2, count, 0,
                                                colbits + rowbits, st));
        void* tmp = alloc(need);
        PG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, need, key, key2, d_vals, val2, count, 0,
                                                colbits + rowbits, st));
        k_trip_runs<<<grid(count), 256, 0, st>>>(key2, val2, count, colbits, sum, keep, d_rcnt);
        need = 0;
        PG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, keep, pos, count + 1, st));
        void* tmp2 = alloc(need);
        PG_CUDA(cudaMemsetAsync(keep + count, 0, 4, st));
        PG_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, need, keep, pos, count + 1, st));
        int32_t* d_ci = (int32_t*)alloc(4 * (size_t)count);
        double* d_v = (double*)alloc(8 * (size_t)count);
        k_trip_emit<<<grid(count), 256, 0, st>>>(key2, sum, keep, pos, count, colbits, d_ci, d_v);
        PG_CUDA(cudaGetLastError());
        int32_t k32 = 0;
        PG_CUDA(cudaMemcpyAsync(&k32, pos + count, 4, cudaMemcpyDeviceToHost, st));
        PG_CUDA(cudaStreamSynchronize(st));
        kept = k32;
        if (kept) {
          PG_CUDA(cudaMemcpyAsync(col_idx, d_ci, 4 * (size_t)kept, cudaMemcpyDeviceToHost, st));
          PG_CUDA(cudaMemcpyAsync(values_out, d_v, 8 * (size_t)kept, cudaMemcpyDeviceToHost, st));
        }
      }
      int32_t* d_rp = (int32_t*)alloc(4 * ((size_t)m + 1));
      size_t need = 0;
      PG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, d_rcnt, d_rp, m + 1, st));
      void* tmp3 = alloc(need);
      PG_CUDA(cub::DeviceScan::ExclusiveSum(tmp3, need, d_rcnt, d_rp, m + 1, st));
      PG_CUDA(cudaMemcpyAsync(row_ptr, d_rp, 4 * ((size_t)m + 1), cudaMemcpyDeviceToHost, st));
      PG_CUDA(cudaStreamSynchronize(st));
      *nnz = kept;
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
    return PG_OK;
  });
}

int pg_partition_row_blocks(const pg_problem* p, const pg_config* cfg, int32_t* starts,
                            int32_t* kinds, int32_t* num_blocks) {
  // partition_row_blocks (par_engine.cpp:14-41): greedy Stream blocks of
  // >= 2 rows within nnz_budget, lone rows Narrow/Wide by vector_threshold
  if (!p || !cfg || !starts || !kinds || !num_blocks) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  const int rc = pg_config_validate(cfg);
  if (rc) return rc;
  int32_t nb = 0, row = 0;
  starts[0] = 0;
  const int32_t* rp = p->row_ptr;
  while (row < p->num_rows) {
    int32_t end = row;
    int64_t acc = 0;
    while (end < p->num_rows && acc + (rp[end + 1] - rp[end]) <= cfg->nnz_budget) {
      acc += rp[end + 1] - rp[end];
      ++end;
    }
    if (end - row >= 2) {
      kinds[nb] = 0;
      starts[++nb] = end;
      row = end;
    } else {
      kinds[nb] = (rp[row + 1] - rp[row]) < cfg->vector_threshold ? 1 : 2;
      starts[++nb] = row + 1;
      ++row;
    }
  }
  *num_blocks = nb;
  return PG_OK;
}

int pg_session_propagate_batch(pg_session* s, int32_t K, const double* lower, const double* upper,
                               double* lower_out, double* upper_out, int32_t* status,
                               int32_t* rounds) {
  if (!s || K < 0 || (K && (!lower || !upper || !status || !rounds))) {
    g_err = "invalid batch arguments";
    return PG_EINVAL;
  }
  return guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    const size_t n = (size_t)s->n;
    for (int32_t k = 0; k < K; ++k) {
      s->upload_bounds(lower + k * n, upper + k * n);
      const int64_t ns = s->run_solve(true);
      pg_result r = {};
      r.lower = lower_out ? lower_out + k * n : nullptr;
      r.upper = upper_out ? upper_out + k * n : nullptr;
      s->fill_result(&r, ns);
      status[k] = r.status;
      rounds[k] = r.rounds_executed;
    }
    return PG_OK;
  });
}

int pg_session_set_root(pg_session* s, pg_result* res) {
  if (!s || !res) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  return guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    const int64_t ns = s->run_solve(true, res);
    s->fill_result(res, ns);
    s->has_root = res->status == PG_CONVERGED;
    if (s->has_root) {
      t_alloc_stream = s->stream;
      if (!s->d_root_lo) {
        s->d_root_lo = dalloc<double>(s->n);
        s->d_root_up = dalloc<double>(s->n);
      }
      k_decode<<<s->grid_for(s->n, 256), 256, 0, s->stream>>>(s->d_key_out, s->d_root_lo,
                                                              s->d_root_up, s->n);
      PG_CUDA(cudaGetLastError());
      PG_CUDA(cudaStreamSynchronize(s->stream));
    }
    return PG_OK;
  });
}

int pg_session_propagate_nodes(pg_session* s, int32_t K, const int32_t* node_ptr,
                               const int32_t* vars, const double* lo, const double* up,
                               int32_t* status, int32_t* rounds, double* lower_out,
                               double* upper_out, int64_t* elapsed_ns) {
  if (!s || K < 0 || (K && (!node_ptr || !status || !rounds))) {
    g_err = "invalid node arguments";
    return PG_EINVAL;
  }
  if (!s->has_root) {
    g_err = "pg_session_set_root must succeed (Converged) before propagating nodes";
    return PG_EINVAL;
  }
  return guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    t_alloc_stream = s->stream;
    const int32_t total = node_ptr[K];
    for (int32_t k = 0; k < K; ++k)
      if (node_ptr[k + 1] < node_ptr[k]) throw Error{PG_EINVAL, "node_ptr must be nondecreasing"};
    for (int32_t i = 0; i < total; ++i)
      if (vars[i] < 0 || vars[i] >= s->n) throw Error{PG_EINVAL, "node override column out of range"};
    int32_t* d_vars = dalloc<int32_t>(total);
    double* d_lo = dalloc<double>(total);
    double* d_up = dalloc<double>(total);
    NodeCtl* d_ctls = dalloc<NodeCtl>(K);
    int2* d_out = dalloc<int2>(K);
    cudaStream_t st = s->stream;
    if (total) {
      PG_CUDA(cudaMemcpyAsync(d_vars, vars, sizeof(int32_t) * total, cudaMemcpyHostToDevice, st));
      PG_CUDA(cudaMemcpyAsync(d_lo, lo, sizeof(double) * total, cudaMemcpyHostToDevice, st));
      PG_CUDA(cudaMemcpyAsync(d_up, up, sizeof(double) * total, cudaMemcpyHostToDevice, st));
    }
    std::vector<NodeCtl> ctls(K);
    for (int32_t k = 0; k < K; ++k)
      ctls[k] = NodeCtl{1, node_ptr[k + 1] - node_ptr[k], d_vars + node_ptr[k], d_lo + node_ptr[k],
                        d_up + node_ptr[k]};
    if (K) PG_CUDA(cudaMemcpyAsync(d_ctls, ctls.data(), sizeof(NodeCtl) * K, cudaMemcpyHostToDevice, st));
    const size_t n = (size_t)s->n;
    if (!getenv("PG_NODES_SERIAL") && s->cfg.scalar_mode == PG_WIDE64) {
      // batched: one CTA per node, many nodes at once (nodes.cuh)
      s->ensure_col_index();
      const size_t m = (size_t)s->m;
      const int chunk = s->cfg.nnz_budget;
      const int maxc = s->max_len() > chunk ? (s->max_len() + chunk - 1) / chunk : 1;
      const size_t per_slot = n * 44 + m * 12 + (size_t)kNodeThreads * maxc * sizeof(Act);
      size_t free_b = 0, total_b = 0;
      PG_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const size_t cap = std::max<size_t>(1, (free_b / 3) / std::max<size_t>(per_slot, 1));
      const int slots = (int)std::max<size_t>(1, std::min<size_t>(
          {(size_t)std::max(K, 1), (size_t)s->nodes_per_sm * s->num_sms, cap}));
      double* s_lo = dalloc<double>(n * slots);
      double* s_up = dalloc<double>(n * slots);
      longlong2* s_key = dalloc<longlong2>(n * slots);
      int32_t* s_cflag = dalloc<int32_t>(n * slots);
      int32_t* s_touch = dalloc<int32_t>(n * slots);
      int32_t* s_undo = dalloc<int32_t>(n * slots);
      int32_t* s_rflag = dalloc<int32_t>(m * slots);
      int32_t* s_rows = dalloc<int32_t>(2 * m * slots);
      Act* s_part = dalloc<Act>((size_t)slots * kNodeThreads * maxc);
      int32_t* d_res = dalloc<int32_t>(2 * (size_t)K + 1);
      // bound vectors, when asked for, in batches of at most ~1 GiB
      const bool want = lower_out || upper_out;
      const int32_t kb = want ? std::max<int32_t>(1, (int32_t)std::min<size_t>(
                                    K, (1ull << 30) / std::max<size_t>(16 * n, 1)))
                              : std::max(K, 1);
      double* d_blo = want ? dalloc<double>((size_t)kb * n) : nullptr;
      double* d_bup = want ? dalloc<double>((size_t)kb * n) : nullptr;
      std::vector<int32_t> hptr(node_ptr, node_ptr + K + 1);
      int32_t* d_ptr = dalloc<int32_t>((size_t)K + 1);
      PG_CUDA(cudaMemcpyAsync(d_ptr, hptr.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, st));
      PG_CUDA(cudaEventRecord(s->ev0, st));
      for (int32_t b0 = 0; b0 < K; b0 += kb) {
        const int32_t nb = std::min(kb, K - b0);
        NodeArgs N;
        N.row_ptr = s->d_row_ptr;
        N.colx = s->d_colx;
        N.vals = s->d_vals;
        N.lhs = s->d_lhs;
        N.rhs = s->d_rhs;
        N.col_ptr = s->d_col_ptr;
        N.col_row = s->d_col_item;
        N.m = s->m;
        N.n = s->n;
        N.root_lo = s->d_root_lo;
        N.root_up = s->d_root_up;
        N.K = nb;
        N.node_ptr = d_ptr + b0;
        N.vars = d_vars;
        N.nlo = d_lo;
        N.nup = d_up;
        N.status = d_res + b0;
        N.rounds = d_res + K + b0;
        N.lower_out = d_blo;
        N.upper_out = d_bup;
        N.ticket = d_res + 2 * K;
        N.s_lo = s_lo;
        N.s_up = s_up;
        N.s_key = s_key;
        N.s_cflag = s_cflag;
        N.s_touch = s_touch;
        N.s_undo = s_undo;
        N.s_rflag = s_rflag;
        N.s_rows = s_rows;
        N.s_part = s_part;
        N.maxc = maxc;
        PG_CUDA(cudaMemsetAsync(N.ticket, 0, sizeof(int32_t), st));
        const int grid = std::min(slots, std::max(nb, 1));
        if (s->cfg.flags & PG_FLAG_ROWCHECK)
          k_nodes<true><<<grid, kNodeThreads, 0, st>>>(N, s->dcfg);
        else
          k_nodes<false><<<grid, kNodeThreads, 0, st>>>(N, s->dcfg);
        PG_CUDA(cudaGetLastError());
        if (lower_out)
          PG_CUDA(cudaMemcpyAsync(lower_out + (size_t)b0 * n, d_blo, sizeof(double) * n * nb,
                                  cudaMemcpyDeviceToHost, st));
        if (upper_out)
          PG_CUDA(cudaMemcpyAsync(upper_out + (size_t)b0 * n, d_bup, sizeof(double) * n * nb,
                                  cudaMemcpyDeviceToHost, st));
      }
      PG_CUDA(cudaEventRecord(s->ev1, st));
      // the session's start bounds are the root fixpoint (as after serial nodes)
      PG_CUDA(cudaMemcpyAsync(s->d_lo0, s->d_root_lo, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      PG_CUDA(cudaMemcpyAsync(s->d_up0, s->d_root_up, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      std::vector<int32_t> res(2 * (size_t)K + 1);
      if (K) PG_CUDA(cudaMemcpyAsync(res.data(), d_res, sizeof(int32_t) * 2 * K, cudaMemcpyDeviceToHost, st));
      PG_CUDA(cudaStreamSynchronize(st));
      float ms = 0.f;
      PG_CUDA(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
      if (elapsed_ns) *elapsed_ns = (int64_t)((double)ms * 1e6);
      for (int32_t k = 0; k < K; ++k) {
        status[k] = res[k];
        rounds[k] = res[K + k];
      }
      t_alloc_stream = st;
      for (void* p : {(void*)s_lo, (void*)s_up, (void*)s_key, (void*)s_cflag, (void*)s_touch,
                      (void*)s_undo, (void*)s_rflag, (void*)s_rows, (void*)s_part, (void*)d_res,
                      (void*)d_blo, (void*)d_bup, (void*)d_ptr, (void*)d_vars, (void*)d_lo,
                      (void*)d_up, (void*)d_ctls, (void*)d_out})
        dfree(p);
      return PG_OK;
    }
    PG_CUDA(cudaEventRecord(s->ev0, st));
    for (int32_t k = 0; k < K; ++k) {
      // stream-ordered: root -> start bounds, overrides, warm control, solve
      PG_CUDA(cudaMemcpyAsync(s->d_lo0, s->d_root_lo, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      PG_CUDA(cudaMemcpyAsync(s->d_up0, s->d_root_up, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      PG_CUDA(cudaMemcpyAsync(s->d_ctl, d_ctls + k, sizeof(NodeCtl), cudaMemcpyDeviceToDevice, st));
      k_apply_node<<<4, 256, 0, st>>>(s->d_lo0, s->d_up0, s->d_ctl, s->cfg.infinity_threshold,
                                      s->cfg.scalar_mode == PG_NARROW32);
      PG_CUDA(cudaGetLastError());
      if (s->cfg.loop_mode == PG_LOOP_GRAPH) {
        PG_CUDA(cudaGraphLaunch(s->exec, st));
      } else {
        s->enqueue_reset(false, true);
        PG_CUDA(cudaMemcpyAsync(s->h_st, s->d_st, sizeof(DevState), cudaMemcpyDeviceToHost, st));
        PG_CUDA(cudaStreamSynchronize(st));
        while (!s->h_st->done) {
          s->enqueue_round(false);
          PG_CUDA(cudaMemcpyAsync(s->h_st, s->d_st, sizeof(DevState), cudaMemcpyDeviceToHost, st));
          PG_CUDA(cudaStreamSynchronize(st));
        }
      }
      // (status, round) of the node, stream-ordered, no host sync
      PG_CUDA(cudaMemcpyAsync(&d_out[k].x, &s->d_st->status, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
      PG_CUDA(cudaMemcpyAsync(&d_out[k].y, &s->d_st->round, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
      if (lower_out || upper_out) {
        k_decode<<<s->grid_for(s->n, 256), 256, 0, st>>>(s->d_key_out, s->d_lo_res, s->d_up_res, s->n);
        if (lower_out)
          PG_CUDA(cudaMemcpyAsync(lower_out + k * n, s->d_lo_res, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        if (upper_out)
          PG_CUDA(cudaMemcpyAsync(upper_out + k * n, s->d_up_res, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
      }
    }
    PG_CUDA(cudaEventRecord(s->ev1, st));
    PG_CUDA(cudaMemsetAsync(s->d_ctl, 0, sizeof(NodeCtl), st));  // later solves start cold
    // the session's start bounds are the root fixpoint again
    PG_CUDA(cudaMemcpyAsync(s->d_lo0, s->d_root_lo, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    PG_CUDA(cudaMemcpyAsync(s->d_up0, s->d_root_up, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    std::vector<int2> out(K);
    if (K) PG_CUDA(cudaMemcpyAsync(out.data(), d_out, sizeof(int2) * K, cudaMemcpyDeviceToHost, st));
    PG_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    PG_CUDA(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    if (elapsed_ns) *elapsed_ns = (int64_t)((double)ms * 1e6);
    for (int32_t k = 0; k < K; ++k) {
      status[k] = out[k].x < 0 ? PG_ROUNDLIMIT : out[k].x;
      rounds[k] = out[k].y;
    }
    t_alloc_stream = st;
    for (void* p : {(void*)d_vars, (void*)d_lo, (void*)d_up, (void*)d_ctls, (void*)d_out}) dfree(p);
    return PG_OK;
  });
}

int pg_session_time_round_kernel(pg_session* s, int32_t reps, double* mean_ns, double* bytes) {
  if (!s || !mean_ns || !bytes || reps < 1) {
    g_err = "invalid arguments";
    return PG_EINVAL;
  }
  return guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    cudaEvent_t b, e;
    PG_CUDA(cudaEventCreate(&b));
    PG_CUDA(cudaEventCreate(&e));
    double total = 0.0;
    s->enqueue_reset(false, false);
    for (int r = 0; r < reps; ++r) {
      s->enqueue_round(false, b, e);
      PG_CUDA(cudaEventSynchronize(e));
      float ms = 0.f;
      PG_CUDA(cudaEventElapsedTime(&ms, b, e));
      total += ms;
      // restore the snapshot so every launch sees the same input
      s->enqueue_reset(false, false);
    }
    PG_CUDA(cudaStreamSynchronize(s->stream));
    cudaEventDestroy(b);
    cudaEventDestroy(e);
    *mean_ns = total * 1e6 / reps;
    // algorithmic bytes of one k_tiles launch: vals+col per entry, row_ptr,
    // lhs/rhs per row, tile descriptors, one snapshot read per column
    // algorithmic bytes of one k_round launch (SURVEY.md 8(d) terms it owns):
    // vals + col per entry, row_ptr, lhs/rhs, one {lb, ub} read per column
    *bytes = 12.0 * (double)s->nnz + 4.0 * (double)(s->m + 1) + 16.0 * (double)s->m +
             16.0 * (double)s->n;
    return PG_OK;
  });
}

int pg_nccl_unique_id(uint8_t* out128) {
  if (!out128) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  if (!g_nccl.load()) {
    g_err = "libnccl.so.2 could not be loaded";
    return PG_ENCCL;
  }
  NcclUid uid;
  const int rc = g_nccl.get_unique_id(&uid);
  if (rc != 0) {
    g_err = std::string("ncclGetUniqueId: ") + g_nccl.error(rc);
    return PG_ENCCL;
  }
  std::memcpy(out128, uid.internal, 128);
  return PG_OK;
}

int pg_session_attach_comm(pg_session* s, const uint8_t* uid128, int32_t rank, int32_t world) {
  if (!s || !uid128 || world < 1 || rank < 0 || rank >= world) {
    g_err = "invalid communicator arguments";
    return PG_EINVAL;
  }
  return guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    if (!g_nccl.load()) throw Error{PG_ENCCL, "libnccl.so.2 could not be loaded"};
    NcclUid uid;
    std::memcpy(uid.internal, uid128, 128);
    void* comm = nullptr;
    const int rc = g_nccl.comm_init_rank(&comm, world, uid, rank);
    if (rc != 0) throw Error{PG_ENCCL, std::string("ncclCommInitRank: ") + g_nccl.error(rc)};
    if (s->comm && !s->comm_aborted) g_nccl.comm_destroy(s->comm);
    s->comm_aborted = false;
    s->comm = comm;
    s->rank = rank;
    s->world = world;
    t_alloc_stream = s->stream;
    for (void* p : {(void*)s->d_delta, (void*)s->d_delta_all, (void*)s->d_dcnt, (void*)s->d_dcnt_all})
      dfree(p);
    if (s->h_dcnt) cudaFreeHost(s->h_dcnt);
    // a round whose every rank changed at most n/16 columns goes sparse
    // (C5 changes <= 253k of 10M sides after round 1)
    s->delta_cap = std::max(1024, s->n / 16);
    // unrolled graphs all-gather a fixed capacity: tiers n/16, n/64, n/256
    s->ntiers = 0;
    for (int div : {16, 64, 256}) {
      const int c = std::max(1024, s->n / div);
      if (s->ntiers == 0 || c < s->delta_caps[s->ntiers - 1]) s->delta_caps[s->ntiers++] = c;
    }
    s->d_delta = dalloc<DeltaItem>(s->delta_cap);
    s->d_delta_all = dalloc<DeltaItem>((size_t)s->delta_cap * world);
    s->d_dcnt = dalloc<int>(2);
    s->d_dcnt_all = dalloc<int>(2 * (size_t)world);
    PG_CUDA(cudaMallocHost(&s->h_dcnt, 2 * sizeof(int) * world));
    // the device-resident loop now carries the all-reduce: rebuild the graph
    if (s->exec) {
      cudaGraphExecDestroy(s->exec);
      s->exec = nullptr;
    }
    if (s->graph) {
      cudaGraphDestroy(s->graph);
      s->graph = nullptr;
    }
    if (s->cfg.loop_mode == PG_LOOP_GRAPH) s->build_graph();
    return PG_OK;
  });
}

int pg_multi_propagate(const pg_problem* p, const pg_config* cfg, int32_t ngpus, int32_t mode,
                       pg_result* res) {
  // one host thread per GPU, each a row-shard session (nnz-balanced
  // contiguous rows, all columns) on its device, one NCCL communicator;
  // rank 0's result is returned (every rank holds the same bounds)
  if (!p || !cfg || !res) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  if (mode != PG_MULTI_ROWS) {
    g_err = "mode must be PG_MULTI_ROWS";
    return PG_EINVAL;
  }
  int rc = pg_config_validate(cfg);
  if (rc) return rc;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    g_err = "no CUDA device visible (the B200 engine has no CPU fallback)";
    return PG_ENODEV;
  }
  if (ngpus < 1 || cfg->device < 0 || cfg->device + ngpus > ndev) {
    g_err = "ngpus out of range (devices cfg->device .. cfg->device + ngpus - 1 must exist)";
    return PG_EINVAL;
  }
  if (!p->row_ptr || p->num_rows < 0) {
    g_err = "problem arrays are NULL";
    return PG_EINVAL;
  }
  uint8_t uid[128];
  if ((rc = pg_nccl_unique_id(uid))) return rc;
  const int32_t m = p->num_rows;
  // shard g: rows [r[g], r[g+1]), ~nnz / ngpus entries each
  std::vector<int32_t> r(ngpus + 1, 0);
  for (int g = 1; g < ngpus; ++g) {
    const int64_t target = p->nnz * g / ngpus;
    r[g] = (int32_t)(std::lower_bound(p->row_ptr, p->row_ptr + m + 1, target) - p->row_ptr);
    r[g] = std::max(r[g], r[g - 1]);
  }
  r[ngpus] = m;
  std::vector<std::vector<int32_t>> rps(ngpus);
  std::vector<int> rcs(ngpus, PG_OK), stage(ngpus, 0);
  std::vector<std::string> errs(ngpus);
  std::vector<pg_session*> ss(ngpus, nullptr);
  std::vector<pg_result> rr(ngpus);
  std::mutex mu;
  std::condition_variable cv;
  int created = 0;
  bool abort_all = false;
  auto work = [&](int g) {
    pg_problem q = *p;
    const int32_t k0 = p->row_ptr[r[g]];
    rps[g].resize((size_t)(r[g + 1] - r[g]) + 1);
    for (int32_t i = r[g]; i <= r[g + 1]; ++i) rps[g][i - r[g]] = p->row_ptr[i] - k0;
    q.num_rows = r[g + 1] - r[g];
    q.nnz = p->row_ptr[r[g + 1]] - k0;
    q.row_ptr = rps[g].data();
    q.col_idx = p->col_idx ? p->col_idx + k0 : nullptr;
    q.values = p->values ? p->values + k0 : nullptr;
    q.lhs = p->lhs ? p->lhs + r[g] : nullptr;
    q.rhs = p->rhs ? p->rhs + r[g] : nullptr;
    pg_config c = *cfg;
    c.device = cfg->device + g;
    int e = pg_session_create(&q, &c, &ss[g]);
    {
      // every rank must have a session before any enters the NCCL init
      std::unique_lock<std::mutex> lk(mu);
      if (e) abort_all = true;
      ++created;
      cv.notify_all();
      cv.wait(lk, [&] { return created == ngpus; });
      if (abort_all) {
        rcs[g] = e;
        errs[g] = e ? pg_last_error() : "";
        return;
      }
    }
    e = pg_session_attach_comm(ss[g], uid, g, ngpus);
    if (!e) {
      rr[g] = pg_result{};
      if (g == 0) rr[g] = *res;
      e = pg_session_propagate(ss[g], nullptr, nullptr, &rr[g]);
    }
    rcs[g] = e;
    if (e) {
      errs[g] = pg_last_error();
      // a failed rank must not leave the others waiting in a collective:
      // abort every attached communicator (ncclCommAbort is safe from
      // another thread and ends their in-flight NCCL work with an error)
      std::lock_guard<std::mutex> lk(mu);
      if (!abort_all && g_nccl.comm_abort) {
        abort_all = true;
        for (int k = 0; k < ngpus; ++k)
          if (k != g && ss[k] && ss[k]->comm && !ss[k]->comm_aborted.exchange(true))
            g_nccl.comm_abort(ss[k]->comm);
      }
    }
  };
  std::vector<std::thread> th;
  for (int g = 1; g < ngpus; ++g) th.emplace_back(work, g);
  work(0);
  for (auto& t : th) t.join();
  for (int g = 0; g < ngpus; ++g)
    if (ss[g]) pg_session_destroy(ss[g]);
  for (int g = 0; g < ngpus; ++g)
    if (rcs[g]) {
      g_err = "rank " + std::to_string(g) + ": " + errs[g];
      return rcs[g];
    }
  const pg_result out = rr[0];
  res->status = out.status;
  res->rounds_executed = out.rounds_executed;
  res->total_bound_changes = out.total_bound_changes;
  res->constraints_processed = (int64_t)out.rounds_executed * m;
  res->elapsed_ns = out.elapsed_ns;
  return PG_OK;
}

int pg_session_info(const pg_session* s, int64_t* info, int32_t n_info) {
  if (!s || !info) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  const int64_t v[] = {s->m, s->n, s->nnz, s->nslices, s->nsrow, s->nseg,
                       s->short_rows, s->short_nnz, s->seg_nnz, s->nunits, s->sell_elems,
                       s->nsplit, s->use_persistent() ? 1 : 0, s->delta_rounds,
                       s->host_syncs, s->held_rounds, s->shard_rounds, s->delta_graphs,
                       s->gather_kind() == 2 ? 8 : s->gather_kind() == 1 ? 16 : 32};
  for (int i = 0; i < n_info && i < (int)(sizeof(v) / sizeof(v[0])); ++i) info[i] = v[i];
  return PG_OK;
}

const char* pg_last_error(void) { return g_err.c_str(); }

int32_t pg_abi_version(void) { return PG_ABI_VERSION; }

}  // extern "C"

// ---- MPS ingest (mps_reader.h) -----------------------------------------------------
struct pg_mps {
  std::vector<char> text;
  pgmps::Problem p;
};

namespace {
int mps_parse(pg_mps* h, double thr, int32_t threads) {
  pgmps::Reader r;
  r.buf = h->text.data();
  r.size = (int64_t)h->text.size();
  r.thr = thr;
  const unsigned hw = std::thread::hardware_concurrency();
  r.threads = threads > 0 ? threads : (int)(hw ? hw : 1);
  try {
    r.run();
  } catch (const pgmps::Error& e) {
    g_err = "mps parse error at line " +
            std::to_string(pgmps::line_of(r.buf, r.size, e.offset)) + ": " + e.message;
    return PG_EPARSE;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory while parsing MPS";
    return PG_ENOMEM;
  }
  h->p = std::move(r.out);
  return PG_OK;
}
}  // namespace

int pg_mps_read_buffer(const char* text, int64_t size, double infinity_threshold, int32_t threads,
                       pg_mps** out) {
  if (!out || (size > 0 && !text) || size < 0) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  *out = nullptr;
  pg_mps* h = new (std::nothrow) pg_mps;
  if (!h) return PG_ENOMEM;
  h->text.assign(text, text + size);
  const int rc = mps_parse(h, infinity_threshold, threads);
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return PG_OK;
}

int pg_mps_read(const char* path, double infinity_threshold, int32_t threads, pg_mps** out) {
  // parse_mps_file (mps.cpp:409-420)
  if (!out || !path) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  *out = nullptr;
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) {
    g_err = std::string("cannot open '") + path + "'";
    return PG_EPARSE;
  }
  pg_mps* h = new (std::nothrow) pg_mps;
  if (!h) return PG_ENOMEM;
  const std::streamsize sz = in.tellg();
  in.seekg(0);
  h->text.resize((size_t)std::max<std::streamsize>(sz, 0));
  if (sz > 0 && !in.read(h->text.data(), sz)) {
    delete h;
    g_err = std::string("cannot read '") + path + "'";
    return PG_EPARSE;
  }
  const int rc = mps_parse(h, infinity_threshold, threads);
  if (rc) {
    delete h;
    return rc;
  }
  if (h->p.name.empty()) {
    const std::string sp(path);
    const size_t slash = sp.find_last_of('/');
    h->p.name = slash == std::string::npos ? sp : sp.substr(slash + 1);
  }
  *out = h;
  return PG_OK;
}

int pg_mps_dims(const pg_mps* h, int32_t* num_rows, int32_t* num_cols, int64_t* num_triplets) {
  if (!h || !num_rows || !num_cols || !num_triplets) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  *num_rows = h->p.m;
  *num_cols = h->p.n;
  *num_triplets = (int64_t)h->p.rows.size();
  return PG_OK;
}

const char* pg_mps_name(const pg_mps* h) { return h ? h->p.name.c_str() : ""; }

int pg_mps_arrays(const pg_mps* h, const int32_t** rows, const int32_t** cols, const double** values,
                  const double** lhs, const double** rhs, const double** lower, const double** upper,
                  const uint8_t** integral) {
  if (!h) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  if (rows) *rows = h->p.rows.data();
  if (cols) *cols = h->p.cols.data();
  if (values) *values = h->p.vals.data();
  if (lhs) *lhs = h->p.lhs.data();
  if (rhs) *rhs = h->p.rhs.data();
  if (lower) *lower = h->p.lower.data();
  if (upper) *upper = h->p.upper.data();
  if (integral) *integral = h->p.integral.data();
  return PG_OK;
}

int pg_mps_to_csr(const pg_mps* h, int32_t device, int32_t* row_ptr, int32_t* col_idx,
                  double* values, int64_t* nnz) {
  if (!h) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  return pg_csr_from_triplets(h->p.m, h->p.n, (int64_t)h->p.rows.size(), h->p.rows.data(),
                              h->p.cols.data(), h->p.vals.data(), device, row_ptr, col_idx, values,
                              nnz);
}

void pg_mps_free(pg_mps* h) { delete h; }
