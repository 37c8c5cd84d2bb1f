/*
 * propgate_b200.h -- C-ABI of the B200-native domain-propagation engine.
 *
 * This is the drop-in boundary for the round-synchronous ("GPU-atomic")
 * propagation path of the reference library `propgate` (arXiv 2009.07785).
 * Plain C: fixed-width integers, plain pointers and sizes, no CUDA or torch
 * types.  Every entry point cites the reference interface it replaces
 * (paths relative to /root/reference/proj).
 *
 * Ownership: all input pointers are borrowed host pointers and are read
 * during the call only (reference: `const ProblemInstance&`).  All output
 * arrays are caller-allocated.  Entry points return PG_OK (0) or a negative
 * error code; the message of the last error on the calling thread is
 * available from pg_last_error().  Infeasibility and the round limit are
 * *statuses* in pg_result, never errors (core/include/propgate/model.hpp:112).
 *
 * Threading: no global mutable state besides the thread-local error
 * message; distinct sessions may be used concurrently from distinct host
 * threads (reference: SPEC.md:379, engines are reentrant).
 */
#ifndef PROPGATE_B200_H
#define PROPGATE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PG_ABI_VERSION 1

/* ---- error codes ------------------------------------------------------ */
#define PG_OK 0
#define PG_EINVAL (-1)  /* config or shape invalid; reference throws std::invalid_argument (core/src/model.cpp:21-35) */
#define PG_ENOMEM (-2)  /* device or host allocation failed */
#define PG_ECUDA (-3)   /* CUDA runtime error */
#define PG_ENCCL (-4)   /* NCCL error (row-sharded multi-GPU path) */
#define PG_ENODEV (-5)  /* no usable sm_100 device */
#define PG_ERANGE (-6)  /* index out of range; reference throws std::out_of_range (core/src/model.cpp:40-45) */
#define PG_EPARSE (-7)  /* MPS parse / file error; reference throws MpsError / std::runtime_error (core/src/mps.cpp) */

/* ---- statuses: same order as propgate::PropagationStatus (model.hpp:112) */
#define PG_CONVERGED 0
#define PG_ROUNDLIMIT 1
#define PG_INFEASIBLE 2

/* ---- scalar modes: propgate::ScalarMode (model.hpp:129) ---------------- */
#define PG_WIDE64 0
#define PG_NARROW32 1

/* ---- loop modes (new; the reference has only its CPU round loop) ------- */
#define PG_LOOP_GRAPH 0 /* device-resident loop: CUDA graph with a conditional WHILE node */
#define PG_LOOP_HOST 1  /* host-driven loop, one stream sync per round (the paper's cpu_loop) */

/* ---- config flags ------------------------------------------------------ */
/* Step-2 row check of classify_constraint (core/include/propgate/propcore.hpp:138-158),
 * which cpu_seq runs (core/src/seq_engine.cpp:47-52) and cpu_par does not.
 * With it, infeasibility verdicts match cpu_seq. */
#define PG_FLAG_ROWCHECK 0x1u
/* Device-side worklist: a round only visits rows that contain a variable
 * whose bound changed in the previous round (exact under snapshot
 * semantics). */
#define PG_FLAG_WORKLIST 0x2u
/* Row-sharded sessions (pg_session_attach_comm): a round in which every rank
 * changed at most num_cols / 16 columns exchanges only those columns (NCCL
 * all-gather of (column, keys) items, max-merged on every rank) instead of
 * the dense all-reduce of every bound.  Results
 * are identical either way; the solve runs the host-driven loop (the choice
 * reads the gathered counts on the host each round). */
#define PG_FLAG_DELTA_EXCHANGE 0x4u

/* Problem in CSR form: the fields of propgate::ProblemInstance
 * (core/include/propgate/model.hpp:20-37, 68-79).  int32 row_ptr/col_idx,
 * fp64 values, canonical CSR (strictly increasing columns per row). */
typedef struct pg_problem {
  int32_t num_rows;
  int32_t num_cols;
  int64_t nnz;
  const int32_t* row_ptr; /* [num_rows + 1] */
  const int32_t* col_idx; /* [nnz] */
  const double* values;   /* [nnz] */
  const double* lhs;      /* [num_rows] */
  const double* rhs;      /* [num_rows] */
  const double* lower;    /* [num_cols] */
  const double* upper;    /* [num_cols] */
  const uint8_t* integral; /* [num_cols], nonzero = integer variable */
} pg_problem;

/* propgate::EngineConfig (model.hpp:131-144) plus GPU fields. */
typedef struct pg_config {
  int32_t round_limit;       /* 100 */
  double infinity_threshold; /* 1e20 */
  double improvement_abs;    /* 1e-7 */
  double improvement_rel;    /* 1e-7 */
  double integrality_eps;    /* 1e-6 */
  int32_t nnz_budget;        /* 1024: also the chunk length of long-row sums */
  int32_t vector_threshold;  /* 64 */
  int32_t worker_count;      /* 0; accepted and validated, unused on the GPU */
  int32_t scalar_mode;       /* PG_WIDE64 */
  int32_t device;            /* CUDA device ordinal, default 0 */
  int32_t loop_mode;         /* PG_LOOP_GRAPH */
  uint32_t flags;            /* PG_FLAG_ROWCHECK by default */
} pg_config;

/* propgate::PropagationResult (model.hpp:119-127).  `lower`/`upper` are
 * caller-allocated [num_cols]; `per_round_changes` is caller-allocated with
 * `per_round_capacity` entries (>= round_limit to receive all of them; may
 * be NULL).  elapsed_ns covers the round loop only, like the reference
 * (core/src/par_engine.cpp:228,268): device time from CUDA events. */
typedef struct pg_result {
  double* lower;
  double* upper;
  int64_t* per_round_changes;
  int32_t per_round_capacity;
  int32_t status;
  int32_t rounds_executed;
  int32_t _pad;
  int64_t total_bound_changes;
  int64_t constraints_processed;
  int64_t elapsed_ns;
} pg_result;

typedef struct pg_session pg_session;

/* Fills the reference defaults (model.hpp:131-140) and the GPU defaults. */
void pg_config_default(pg_config* cfg);

/* Mirrors EngineConfig::validate() (core/src/model.cpp:21-35). PG_EINVAL
 * with the reference's message on violation. */
int pg_config_validate(const pg_config* cfg);

/* Replaces propagate_parallel (core/include/propgate/par_engine.hpp:41-42,
 * core/src/par_engine.cpp:314-320) and, with PG_FLAG_ROWCHECK, carries
 * propagate_sequential's verdicts (seq_engine.hpp:15-16).  Uploads the
 * problem, runs the round loop to a fixpoint on the device, downloads the
 * bounds. */
int pg_propagate(const pg_problem* prob, const pg_config* cfg, pg_result* res);

/* Replaces propagate_round_parallel (par_engine.hpp:33-36,
 * par_engine.cpp:277-312): exactly one round on the caller's snapshot
 * (lb_in/ub_in), writing the merged bounds to lb_out/ub_out and the
 * RoundOutcome {changed, infeasible, changes} (par_engine.hpp:23-27). */
int pg_round(const pg_problem* prob, const pg_config* cfg, const double* lb_in,
             const double* ub_in, double* lb_out, double* ub_out,
             int32_t* changed, int32_t* infeasible, int64_t* changes);

/* Replaces partition_row_blocks (par_engine.hpp:12-13, par_engine.cpp:14-41)
 * for API completeness (the GPU uses its own length-binned tiling).
 * block_starts is caller-allocated [num_rows + 1], kinds [num_rows]
 * (0 Stream, 1 VectorNarrow, 2 VectorWide); *num_blocks receives the count. */
int pg_partition_row_blocks(const pg_problem* prob, const pg_config* cfg,
                            int32_t* block_starts, int32_t* kinds,
                            int32_t* num_blocks);

/* Replaces csr_from_triplets (core/include/propgate/model.hpp, core/src/model.cpp:37-80)
 * with an on-device build (on-device ingest): triplets
 * (row, col, value) stable-sorted by (row, col), duplicates summed in input
 * order, zero sums dropped.  PG_ERANGE with the reference's message
 * ("triplet row index out of range" / "triplet column index out of range")
 * for the first bad triplet.  row_ptr is caller-allocated [num_rows + 1],
 * col_idx / values_out [count] (the result has *nnz <= count entries). */
int pg_csr_from_triplets(int32_t num_rows, int32_t num_cols, int64_t count,
                         const int32_t* rows, const int32_t* cols, const double* values,
                         int32_t device, int32_t* row_ptr, int32_t* col_idx,
                         double* values_out, int64_t* nnz);

/* ---- sessions: matrix resident on the device ---------------------------
 * New capability (B&B warm start, SURVEY.md 5 "Checkpoint / resume"): the
 * reference re-reads the whole ProblemInstance on every call. */
int pg_session_create(const pg_problem* prob, const pg_config* cfg,
                      pg_session** out);
void pg_session_destroy(pg_session* s);

/* pg_session_create returns once the caller's arrays have been copied (they
 * may be freed or reused right away). */

/* pg_round on a resident session (propagate_round_parallel,
 * par_engine.hpp:33-36): one round on the snapshot lb_in/ub_in, the matrix
 * set up once per session instead of once per call (a branch-and-bound
 * caller of the one-round API).  Wide64 single-GPU sessions only
 * (PG_EINVAL otherwise). */
int pg_session_round(pg_session* s, const double* lb_in, const double* ub_in,
                     double* lb_out, double* ub_out, int32_t* changed,
                     int32_t* infeasible, int64_t* changes);

/* Propagate from new start bounds (NULL = the problem's own bounds), host
 * buffers in and out.  Same semantics as pg_propagate. */
int pg_session_propagate(pg_session* s, const double* lower,
                         const double* upper, pg_result* res);

/* Propagate from the device-resident start bounds already uploaded at
 * session creation: nothing crosses PCIe.  res->lower/upper may be NULL to
 * skip the download.  This is the device-resident timing path. */
int pg_session_run(pg_session* s, pg_result* res);

/* K independent node bound vectors over the shared matrix (config 4).
 * lower/upper are [K * num_cols] node-major; outputs likewise; status and
 * rounds are [K].  Each node follows propagate_parallel's semantics on its
 * own bounds. */
int pg_session_propagate_batch(pg_session* s, int32_t K, const double* lower,
                               const double* upper, double* lower_out,
                               double* upper_out, int32_t* status,
                               int32_t* rounds);

/* Timing helper for the roofline: runs `reps` isolated launches of the
 * fused round kernel(s) on the session's start bounds (no commit), and
 * returns the mean device time per launch in *mean_ns and the algorithmic
 * bytes of one launch in *bytes. */
int pg_session_time_round_kernel(pg_session* s, int32_t reps, double* mean_ns,
                                 double* bytes);

/* ---- branch-and-bound nodes (config 4) -----------------------------------
 * pg_session_set_root propagates the session's start bounds and, when the
 * result is Converged, keeps that fixpoint on the device as the root.
 * pg_session_propagate_nodes then solves K child nodes, each the root with a
 * few bounds overridden (node k: entries node_ptr[k]..node_ptr[k+1]-1 of
 * vars/lo/up), back to back in one stream with no host round trip per node.
 * With PG_FLAG_WORKLIST, a node's round 1 visits only the rows containing an
 * overridden column (exact: every other row's candidates were rejected
 * against the same bounds in the root's confirming round).  Per-node results
 * are those of pg_propagate on the node's full bounds; lower_out/upper_out
 * ([K * num_cols], node-major) may be NULL.  elapsed_ns: device time of all
 * K solves. */
int pg_session_set_root(pg_session* s, pg_result* res);
int pg_session_propagate_nodes(pg_session* s, int32_t K, const int32_t* node_ptr,
                               const int32_t* vars, const double* lo, const double* up,
                               int32_t* status, int32_t* rounds, double* lower_out,
                               double* upper_out, int64_t* elapsed_ns);

/* ---- row-sharded multi-GPU (config 5): one process per GPU --------------
 * New capability (the reference is single-process).  Each rank creates a
 * session over its contiguous row shard (all columns), rank 0 draws an NCCL
 * unique id, every rank attaches with it; each round then merges the shards'
 * bound keys and infeasibility with one NCCL max all-reduce over NVLink,
 * captured inside the device-resident loop.  Results are bit-identical to a
 * single GPU (exact max/min merges, rows never split). */
int pg_nccl_unique_id(uint8_t* out128);
int pg_session_attach_comm(pg_session* s, const uint8_t* uid128, int32_t rank,
                           int32_t world);

/* Single-process multi-GPU: one host thread per device
 * cfg->device .. cfg->device + ngpus - 1, each a row-shard session
 * (nnz-balanced contiguous rows, all columns) attached to one NCCL
 * communicator, solved together; same results and statuses as
 * pg_propagate (constraints_processed counts all rows).  mode:
 * PG_MULTI_ROWS (the only mode: a single instance shards by rows; node
 * batches use pg_session_propagate_nodes per process). */
#define PG_MULTI_ROWS 0
int pg_multi_propagate(const pg_problem* prob, const pg_config* cfg, int32_t ngpus,
                       int32_t mode, pg_result* res);

/* ---- MPS ingest ------------------------------------
 * Replaces parse_mps_file / parse_mps (core/include/propgate/mps.hpp:28-31,
 * core/src/mps.cpp:336-407): the same sections, row / bound semantics,
 * column numbering, integrality markers, infinity normalisation and error
 * messages ("mps parse error at line N: ...", PG_EPARSE).  The text is parsed
 * on host threads (threads <= 0: all hardware threads); the matrix comes out
 * as the triplets in file order, and pg_mps_to_csr builds the CSR on the
 * device (pg_csr_from_triplets: csr_from_triplets' order and sums).  A read
 * without a GPU is fine; only pg_mps_to_csr needs one. */
typedef struct pg_mps pg_mps;
int pg_mps_read(const char* path, double infinity_threshold, int32_t threads, pg_mps** out);
int pg_mps_read_buffer(const char* text, int64_t size, double infinity_threshold, int32_t threads,
                       pg_mps** out);
/* dimensions and the triplet count; the name (NAME section, else the file name) */
int pg_mps_dims(const pg_mps* h, int32_t* num_rows, int32_t* num_cols, int64_t* num_triplets);
const char* pg_mps_name(const pg_mps* h);
/* borrowed views, valid until pg_mps_free: triplets [num_triplets], lhs / rhs
 * [num_rows], lower / upper / integral [num_cols] */
int pg_mps_arrays(const pg_mps* h, const int32_t** rows, const int32_t** cols, const double** values,
                  const double** lhs, const double** rhs, const double** lower, const double** upper,
                  const uint8_t** integral);
/* CSR of the triplets on `device`: row_ptr [num_rows + 1], col_idx / values
 * [num_triplets] caller-allocated; *nnz receives the entry count */
int pg_mps_to_csr(const pg_mps* h, int32_t device, int32_t* row_ptr, int32_t* col_idx,
                  double* values, int64_t* nnz);
void pg_mps_free(pg_mps* h);

/* Session statistics, in this order: m, n, nnz, slices (sliced-ELL, 32
 * chains each), split-candidate rows (> 16 entries), segments (chains of
 * those rows), short rows, short-row entries, segment entries, chains,
 * sliced-ELL elements (entries + padding), split rows (> nnz_budget),
 * persistent loop (1: the whole solve is one cooperative kernel), rounds of
 * the last solve that used the sparse delta exchange, host round trips of
 * the last row-sharded solve (one per graph of unrolled rounds), delta
 * rounds held by a capacity overflow and resumed with the dense all-reduce,
 * rounds per unrolled graph, graphs of delta rounds launched, bytes of the
 * per-entry column record the round kernels gather (32, 16 or 8). */
int pg_session_info(const pg_session* s, int64_t* info, int32_t n_info);

/* Thread-local message of the last failed call on this thread. */
const char* pg_last_error(void);

/* ABI version (PG_ABI_VERSION) and the compiled device architecture. */
int32_t pg_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PROPGATE_B200_H */
