// engine.cu -- host side of the B200 propagation engine and the C-ABI
// (include/propgate_b200.h).
//
// Session = one problem resident in HBM:
//   row_ptr  int32[m+1]     col  int32[nnz] (bit 31 = integral flag)
//   vals     f64[nnz]       lhs/rhs f64[m] (normalised to +-inf)
//   key_in   {i64,i64}[n]   snapshot bounds as ordered-bits keys
//   key_out  {i64,i64}[n]   merge target of the round (atomicMax/atomicMin)
//   lo0/up0  f64[n]         normalised start bounds
// plus the tile table of short rows and the chunk table of long rows.
//
// The round loop (par_engine.cpp:228-267) runs on the device: a CUDA graph
//   k_reset -> WHILE(cond) { k_tiles, k_long_*, k_commit }
// where k_commit's last CTA writes per_round_changes[r] and clears `cond`
// on Infeasible / Converged / RoundLimit.  One graph launch per solve; no
// host synchronisation per round.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/propgate_b200.h"
#include "kernels.cuh"

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

template <typename T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  PG_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return static_cast<T*>(p);
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

}  // namespace

struct pg_session {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int32_t m = 0, n = 0;
  int64_t nnz = 0;
  pg_config cfg{};
  DevCfg dcfg{};
  int num_sms = 148;

  // device arrays
  int32_t* d_row_ptr = nullptr;
  int32_t* d_colx = nullptr;
  double* d_vals = nullptr;
  double* d_lhs = nullptr;
  double* d_rhs = nullptr;
  longlong2* d_key_in = nullptr;
  longlong2* d_key_out = nullptr;
  double* d_lo0 = nullptr;
  double* d_up0 = nullptr;
  double* d_lo_res = nullptr;
  double* d_up_res = nullptr;
  int2* d_tiles = nullptr;
  LongChunk* d_chunks = nullptr;
  int32_t* d_long_rows = nullptr;
  int32_t* d_long_first = nullptr;
  Act* d_partial = nullptr;
  Act* d_long_act = nullptr;
  DevState* d_st = nullptr;
  long long* d_per_round = nullptr;

  // host mirrors
  DevState* h_st = nullptr;  // pinned
  int32_t num_tiles = 0, nlong = 0, nchunks = 0;
  int64_t tile_rows = 0, tile_nnz = 0, long_nnz = 0;

  // graph
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  ~pg_session() {
    if (dev >= 0) cudaSetDevice(dev);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    void* ptrs[] = {d_row_ptr, d_colx, d_vals, d_lhs, d_rhs, d_key_in, d_key_out, d_lo0, d_up0,
                    d_lo_res, d_up_res, d_tiles, d_chunks, d_long_rows, d_long_first, d_partial,
                    d_long_act, d_st, d_per_round};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (h_st) cudaFreeHost(h_st);
    if (stream) cudaStreamDestroy(stream);
  }

  int grid_for(int64_t items, int threads, int per_sm = 8) const {
    const int64_t g = (items + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms * per_sm));
  }

  // ---- one round of kernels, enqueued on `stream` ------------------------------
  void enqueue_round(bool use_graph, cudaEvent_t k1_begin = nullptr, cudaEvent_t k1_end = nullptr) {
    const bool rowcheck = (cfg.flags & PG_FLAG_ROWCHECK) != 0;
    if (k1_begin) PG_CUDA(cudaEventRecord(k1_begin, stream));
    if (num_tiles > 0) {
      if (rowcheck)
        k_tiles<true><<<num_tiles, kTileThreads, 0, stream>>>(d_tiles, d_row_ptr, d_colx, d_vals,
                                                              d_lhs, d_rhs, d_key_in,
                                                              (long long*)d_key_out, d_st, dcfg);
      else
        k_tiles<false><<<num_tiles, kTileThreads, 0, stream>>>(d_tiles, d_row_ptr, d_colx, d_vals,
                                                               d_lhs, d_rhs, d_key_in,
                                                               (long long*)d_key_out, d_st, dcfg);
    }
    if (k1_end) PG_CUDA(cudaEventRecord(k1_end, stream));
    if (nlong > 0) {
      k_long_partial<<<(nchunks * 32 + 255) / 256, 256, 0, stream>>>(d_chunks, nchunks, d_colx,
                                                                     d_vals, d_key_in, d_partial);
      if (rowcheck)
        k_long_combine<true><<<(nlong + 127) / 128, 128, 0, stream>>>(
            d_long_rows, d_long_first, nlong, d_partial, d_long_act, d_lhs, d_rhs, d_st, dcfg);
      else
        k_long_combine<false><<<(nlong + 127) / 128, 128, 0, stream>>>(
            d_long_rows, d_long_first, nlong, d_partial, d_long_act, d_lhs, d_rhs, d_st, dcfg);
      k_long_cand<<<nchunks, 256, 0, stream>>>(d_chunks, d_long_rows, d_long_act, d_colx, d_vals,
                                                d_lhs, d_rhs, d_key_in, (long long*)d_key_out,
                                                d_st, dcfg);
    }
    k_commit<<<grid_for(n, kCommitThreads), kCommitThreads, 0, stream>>>(
        d_key_in, d_key_out, n, d_st, d_per_round, dcfg, cond, use_graph ? 1 : 0);
    PG_CUDA(cudaGetLastError());
  }

  void enqueue_reset(bool use_graph, bool check_crossed) {
    k_reset<<<grid_for(n, kCommitThreads), kCommitThreads, 0, stream>>>(
        d_lo0, d_up0, d_key_in, d_key_out, n, d_st, dcfg, check_crossed ? 1 : 0, cond,
        use_graph ? 1 : 0);
    PG_CUDA(cudaGetLastError());
  }

  void build_graph() {
    PG_CUDA(cudaGraphCreate(&graph, 0));
    PG_CUDA(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    // node 1: reset (captured)
    cudaGraphNode_t reset_node;
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
      reset_node = nodes.back();
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
    cudaGraph_t body2 = nullptr;
    PG_CUDA(cudaStreamEndCapture(stream, &body2));
    PG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  }

  // Runs one full solve from lo0/up0.  Returns elapsed device ns.
  int64_t run_solve(bool check_crossed = true) {
    if (cfg.loop_mode == PG_LOOP_GRAPH && check_crossed) {
      PG_CUDA(cudaEventRecord(ev0, stream));
      PG_CUDA(cudaGraphLaunch(exec, stream));
      PG_CUDA(cudaEventRecord(ev1, stream));
    } else {
      // host-driven loop: one sync per round (the paper's cpu_loop)
      PG_CUDA(cudaEventRecord(ev0, stream));
      enqueue_reset(false, check_crossed);
      PG_CUDA(cudaMemcpyAsync(h_st, d_st, sizeof(DevState), cudaMemcpyDeviceToHost, stream));
      PG_CUDA(cudaStreamSynchronize(stream));
      while (!h_st->done) {
        enqueue_round(false);
        PG_CUDA(cudaMemcpyAsync(h_st, d_st, sizeof(DevState), cudaMemcpyDeviceToHost, stream));
        PG_CUDA(cudaStreamSynchronize(stream));
      }
      PG_CUDA(cudaEventRecord(ev1, stream));
    }
    PG_CUDA(cudaMemcpyAsync(h_st, d_st, sizeof(DevState), cudaMemcpyDeviceToHost, stream));
    PG_CUDA(cudaStreamSynchronize(stream));
    float ms = 0.f;
    PG_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    return (int64_t)((double)ms * 1e6);
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
    if (res->lower || res->upper) {
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
    if (n) {
      k_normalize<<<grid_for(n, 256), 256, 0, stream>>>(d_lo0, n, cfg.infinity_threshold);
      k_normalize<<<grid_for(n, 256), 256, 0, stream>>>(d_up0, n, cfg.infinity_threshold);
      PG_CUDA(cudaGetLastError());
    }
  }
};

namespace {

void build_tables(pg_session* s, const int32_t* rp, std::vector<int2>& tiles,
                  std::vector<LongChunk>& chunks, std::vector<int32_t>& long_rows,
                  std::vector<int32_t>& long_first) {
  const int64_t chunk = s->cfg.nnz_budget;
  const int64_t long_t = std::min<int64_t>(chunk, kTileNnz);
  int32_t i = 0;
  const int32_t m = s->m;
  while (i < m) {
    const int64_t len = (int64_t)rp[i + 1] - rp[i];
    if (len > long_t) {
      const int32_t slot = (int32_t)long_rows.size();
      long_rows.push_back(i);
      long_first.push_back((int32_t)chunks.size());
      for (int64_t k = rp[i]; k < rp[i + 1]; k += chunk)
        chunks.push_back({slot, (int32_t)k, (int32_t)std::min<int64_t>(k + chunk, rp[i + 1]), 0});
      s->long_nnz += len;
      ++i;
      continue;
    }
    const int32_t start = i;
    int64_t acc = 0;
    while (i < m && i - start < kTileRows) {
      const int64_t l = (int64_t)rp[i + 1] - rp[i];
      if (l > long_t || acc + l > kTileNnz) break;
      acc += l;
      ++i;
    }
    tiles.push_back(make_int2(start, i));
    s->tile_rows += i - start;
    s->tile_nnz += acc;
  }
  long_first.push_back((int32_t)chunks.size());
}

pg_session* create_session(const pg_problem* p, const pg_config* cfg) {
  check_problem(p);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error{PG_ENODEV, "no CUDA device visible (the B200 engine has no CPU fallback)"};
  if (cfg->device < 0 || cfg->device >= ndev) throw Error{PG_EINVAL, "device ordinal out of range"};
  cudaDeviceProp prop;
  PG_CUDA(cudaGetDeviceProperties(&prop, cfg->device));
  if (prop.major != 10)
    throw Error{PG_ENODEV, std::string("device is ") + prop.name + " (sm_" +
                               std::to_string(prop.major * 10 + prop.minor) +
                               "); this build targets sm_100a only"};
  if (cfg->scalar_mode != PG_WIDE64)
    throw Error{PG_EINVAL, "scalar_mode Narrow32 is not implemented on the GPU engine yet"};

  auto* s = new pg_session;
  try {
    s->dev = cfg->device;
    PG_CUDA(cudaSetDevice(s->dev));
    s->num_sms = prop.multiProcessorCount;
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
    PG_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    PG_CUDA(cudaEventCreate(&s->ev0));
    PG_CUDA(cudaEventCreate(&s->ev1));

    std::vector<int2> tiles;
    std::vector<LongChunk> chunks;
    std::vector<int32_t> long_rows, long_first;
    build_tables(s, p->row_ptr, tiles, chunks, long_rows, long_first);
    s->num_tiles = (int32_t)tiles.size();
    s->nlong = (int32_t)long_rows.size();
    s->nchunks = (int32_t)chunks.size();

    const int32_t m = s->m, n = s->n;
    const int64_t nnz = s->nnz;
    s->d_row_ptr = dalloc<int32_t>(m + 1);
    s->d_colx = dalloc<int32_t>(nnz);
    s->d_vals = dalloc<double>(nnz);
    s->d_lhs = dalloc<double>(m);
    s->d_rhs = dalloc<double>(m);
    s->d_key_in = dalloc<longlong2>(n);
    s->d_key_out = dalloc<longlong2>(n);
    s->d_lo0 = dalloc<double>(n);
    s->d_up0 = dalloc<double>(n);
    s->d_lo_res = dalloc<double>(n);
    s->d_up_res = dalloc<double>(n);
    s->d_tiles = dalloc<int2>(tiles.size());
    s->d_chunks = dalloc<LongChunk>(chunks.size());
    s->d_long_rows = dalloc<int32_t>(long_rows.size());
    s->d_long_first = dalloc<int32_t>(long_first.size());
    s->d_partial = dalloc<Act>(chunks.size());
    s->d_long_act = dalloc<Act>(long_rows.size());
    s->d_st = dalloc<DevState>(1);
    s->d_per_round = dalloc<long long>(cfg->round_limit);
    PG_CUDA(cudaMallocHost(&s->h_st, sizeof(DevState)));
    uint8_t* d_integral = dalloc<uint8_t>(n);

    cudaStream_t st = s->stream;
    PG_CUDA(cudaMemsetAsync(s->d_st, 0, sizeof(DevState), st));
    PG_CUDA(cudaMemcpyAsync(s->d_row_ptr, p->row_ptr, sizeof(int32_t) * (m + 1),
                            cudaMemcpyHostToDevice, st));
    if (nnz) {
      PG_CUDA(cudaMemcpyAsync(s->d_colx, p->col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
      PG_CUDA(cudaMemcpyAsync(s->d_vals, p->values, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
    }
    if (m) {
      PG_CUDA(cudaMemcpyAsync(s->d_lhs, p->lhs, sizeof(double) * m, cudaMemcpyHostToDevice, st));
      PG_CUDA(cudaMemcpyAsync(s->d_rhs, p->rhs, sizeof(double) * m, cudaMemcpyHostToDevice, st));
      k_normalize<<<s->grid_for(m, 256), 256, 0, st>>>(s->d_lhs, m, cfg->infinity_threshold);
      k_normalize<<<s->grid_for(m, 256), 256, 0, st>>>(s->d_rhs, m, cfg->infinity_threshold);
    }
    if (n) PG_CUDA(cudaMemcpyAsync(d_integral, p->integral, n, cudaMemcpyHostToDevice, st));
    if (nnz) k_pack_cols<<<s->grid_for(nnz, 256), 256, 0, st>>>(s->d_colx, d_integral, nnz);
    if (!tiles.empty())
      PG_CUDA(cudaMemcpyAsync(s->d_tiles, tiles.data(), sizeof(int2) * tiles.size(),
                              cudaMemcpyHostToDevice, st));
    if (!chunks.empty()) {
      PG_CUDA(cudaMemcpyAsync(s->d_chunks, chunks.data(), sizeof(LongChunk) * chunks.size(),
                              cudaMemcpyHostToDevice, st));
      PG_CUDA(cudaMemcpyAsync(s->d_long_rows, long_rows.data(), sizeof(int32_t) * long_rows.size(),
                              cudaMemcpyHostToDevice, st));
    }
    PG_CUDA(cudaMemcpyAsync(s->d_long_first, long_first.data(), sizeof(int32_t) * long_first.size(),
                            cudaMemcpyHostToDevice, st));
    s->upload_bounds(p->lower, p->upper);
    PG_CUDA(cudaGetLastError());
    PG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_integral);
    if (cfg->loop_mode == PG_LOOP_GRAPH) s->build_graph();
    return s;
  } catch (...) {
    delete s;
    throw;
  }
}

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

int pg_session_create(const pg_problem* p, const pg_config* cfg, pg_session** out) {
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

void pg_session_destroy(pg_session* s) { delete s; }

int pg_session_run(pg_session* s, pg_result* res) {
  if (!s || !res) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  return guarded([&] {
    PG_CUDA(cudaSetDevice(s->dev));
    const int64_t ns = s->run_solve(true);
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
    const int64_t ns = s->run_solve(true);
    s->fill_result(res, ns);
    return PG_OK;
  });
}

int pg_propagate(const pg_problem* p, const pg_config* cfg, pg_result* res) {
  if (!res) {
    g_err = "result is NULL";
    return PG_EINVAL;
  }
  pg_session* s = nullptr;
  int rc = pg_session_create(p, cfg, &s);
  if (rc) return rc;
  rc = pg_session_run(s, res);
  pg_session_destroy(s);
  return rc;
}

int pg_round(const pg_problem* p, const pg_config* cfg, const double* lb_in, const double* ub_in,
             double* lb_out, double* ub_out, int32_t* changed, int32_t* infeasible,
             int64_t* changes) {
  if (!cfg || !lb_in || !ub_in || !lb_out || !ub_out || !changed || !infeasible || !changes) {
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
  c.flags &= ~PG_FLAG_ROWCHECK;
  pg_problem q = *p;
  q.lower = lb_in;
  q.upper = ub_in;
  pg_session* s = nullptr;
  rc = pg_session_create(&q, &c, &s);
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
    *bytes = 12.0 * (double)s->tile_nnz + 4.0 * (double)(s->tile_rows + s->num_tiles) +
             16.0 * (double)s->tile_rows + 8.0 * s->num_tiles + 16.0 * (double)s->n;
    return PG_OK;
  });
}

int pg_session_info(const pg_session* s, int64_t* info, int32_t n_info) {
  if (!s || !info) {
    g_err = "NULL argument";
    return PG_EINVAL;
  }
  const int64_t v[] = {s->m, s->n, s->nnz, s->num_tiles, s->nlong, s->nchunks,
                       s->tile_rows, s->tile_nnz, s->long_nnz};
  for (int i = 0; i < n_info && i < (int)(sizeof(v) / sizeof(v[0])); ++i) info[i] = v[i];
  return PG_OK;
}

const char* pg_last_error(void) { return g_err.c_str(); }

int32_t pg_abi_version(void) { return PG_ABI_VERSION; }

}  // extern "C"
