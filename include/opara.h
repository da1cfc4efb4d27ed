/*
 * opara.h — C ABI of libopara, the B200-native Opara operator-parallel DAG
 * executor.  Plain C types only: integers, doubles, pointers and sizes.  No C++
 * exceptions cross this boundary; every entry point returns an opara_status and
 * leaves a thread-local message in opara_last_error().
 *
 * The boundary replaces, entry for entry, the reference `opsched` package's
 * hot-path Python API (paths relative to /root/reference/pkg/src/opsched):
 *
 *   opara_dag_create          ComputationGraph.__init__ + _kahn   graph.py:110-153
 *   opara_dag_topo_sort       ComputationGraph.topo_sort          graph.py:193-195
 *   opara_dag_predecessors    ComputationGraph.predecessors       graph.py:179-184
 *   opara_dag_successors      ComputationGraph.successors         graph.py:186-191
 *   opara_allocate_streams    allocate_streams (Alg. 1)           allocator.py:43-67
 *   opara_single_stream_plan  single_stream_plan                  allocator.py:70-77
 *   opara_validate_plan       validate_plan                       allocator.py:80-109
 *   opara_dominant_share      dominant_share                      orderer.py:45-53
 *   opara_order               order_opara (Alg. 2) / order_baseline("sequential"|"dfs"|
 *                             "wavefront")                        orderer.py:60-153
 *   opara_linear_extensions   oracle.linear_extensions (every launch
 *                             order, lexicographic by id)         oracle.py:52-84
 *   opara_simulate            simulate (the reference "run": DES model),
 *                             bit-exact C++ port                  simulator.py:212-415
 *   opara_exec_*              the same "run" re-designed as a real multi-stream
 *                             CUDA Graph on the B200 (capture / replay / profile)
 *
 * Status codes map 1:1 onto the reference exception classes (errors.py:4-25);
 * the Python host re-raises the matching class with the message verbatim.
 */
#ifndef OPARA_H_
#define OPARA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */

typedef enum opara_status {
  OPARA_OK = 0,
  OPARA_ERR_FORMAT = 1,            /* FormatError          errors.py:8   */
  OPARA_ERR_GRAPH_VALIDATION = 2,  /* GraphValidationError errors.py:12  */
  OPARA_ERR_PLAN_VIOLATION = 3,    /* PlanViolationError   errors.py:16  */
  OPARA_ERR_COVERAGE = 4,          /* CoverageError        errors.py:20  */
  OPARA_ERR_INFEASIBLE_BLOCK = 5,  /* InfeasibleBlockError errors.py:24  */
  OPARA_ERR_CUDA = 6,              /* CUDA runtime / driver failure      */
  OPARA_ERR_INTERNAL = 7,          /* bug or resource exhaustion         */
  OPARA_ERR_VALUE = 8,             /* ValueError (bad config / policy)   */
  OPARA_ERR_KEY = 9,               /* KeyError ("unknown node id N")     */
  OPARA_ERR_CAPACITY = 10          /* caller buffer too small            */
} opara_status;

/* Message of the last failing call on this thread ("" after success). */
const char* opara_last_error(void);
/* Library version string, e.g. "0.1.0 sm_100a". */
const char* opara_version(void);

/* ---------------------------------------------------------- graph (L1) */

typedef enum opara_op_class { OPARA_COMPUTE = 0, OPARA_MEMORY = 1 } opara_op_class;

/* One operator's scheduling record: OperatorNode + ResourceDemand
 * (graph.py:55-99).  Demand fields are validated on the host side exactly as
 * the reference dataclasses do; the DAG stores them for Alg. 2. */
typedef struct opara_node {
  int64_t id;
  int32_t op_class;                /* opara_op_class */
  int32_t _pad;
  int64_t num_blocks;              /* ResourceDemand.num_blocks           */
  int64_t threads_per_block;       /* ResourceDemand.threads_per_block    */
  int64_t shared_mem_per_block;    /* ResourceDemand.shared_mem_per_block */
  int64_t registers_per_thread;    /* ResourceDemand.registers_per_thread */
} opara_node;

/* GpuConfig (simulator.py:42-59). */
typedef struct opara_gpu_config {
  int64_t num_sms;
  int64_t threads_per_sm;
  int64_t shared_mem_per_sm;
  int64_t registers_per_sm;
  int64_t max_blocks_per_sm;
  double same_class_slowdown;
} opara_gpu_config;

typedef struct opara_dag opara_dag;

/* Build and validate a DAG.  edges_uv holds m (u, v) pairs flattened.
 * Validation order and messages follow graph.py:111-152: duplicate node id
 * (ids scanned ascending) -> per edge in input order: unknown endpoint,
 * self-edge, duplicate edge -> cycle.  Errors: OPARA_ERR_GRAPH_VALIDATION. */
opara_status opara_dag_create(const opara_node* nodes, int64_t n, const int64_t* edges_uv,
                              int64_t m, opara_dag** out);
void opara_dag_destroy(opara_dag* dag);
int64_t opara_dag_num_nodes(const opara_dag* dag);
int64_t opara_dag_num_edges(const opara_dag* dag);
/* Node ids ascending (n entries). */
opara_status opara_dag_node_ids(const opara_dag* dag, int64_t* out);
/* Sorted unique edges, flattened (2*m entries). */
opara_status opara_dag_edges(const opara_dag* dag, int64_t* out_uv);
/* Lexicographically smallest topological order (Kahn, min-heap on id). */
opara_status opara_dag_topo_sort(const opara_dag* dag, int64_t* out);
/* Ascending-id adjacency; *count receives the degree.  Unknown id ->
 * OPARA_ERR_KEY "unknown node id N"; cap < degree -> OPARA_ERR_CAPACITY. */
opara_status opara_dag_predecessors(const opara_dag* dag, int64_t id, int64_t* out, int64_t cap,
                                    int64_t* count);
opara_status opara_dag_successors(const opara_dag* dag, int64_t id, int64_t* out, int64_t cap,
                                  int64_t* count);

/* ------------------------------------------------------ Alg. 1 (L2) */

/* stream_of[i] is the stream of the i-th node in ascending-id order;
 * sync_uv receives the sorted cross-stream edges (capacity 2*num_edges). */
opara_status opara_allocate_streams(const opara_dag* dag, int32_t* stream_of, int32_t* num_streams,
                                    int64_t* sync_uv, int64_t* num_sync);
opara_status opara_single_stream_plan(const opara_dag* dag, int32_t* stream_of,
                                      int32_t* num_streams);
/* Plan check.  The plan is given as (assigned_ids[k], streams[k]) pairs plus
 * its sync list.  Violations are written '\n'-separated into buf (reference
 * wording and order, allocator.py:84-108); *n_problems receives the count. */
opara_status opara_validate_plan(const opara_dag* dag, const int64_t* assigned_ids,
                                 const int64_t* streams, int64_t n_assigned, int64_t num_streams,
                                 const int64_t* sync_uv, int64_t n_sync, char* buf, int64_t buflen,
                                 int64_t* n_problems);

/* ------------------------------------------------------ Alg. 2 (L3) */

typedef enum opara_policy {
  OPARA_POLICY_OPARA = 0,
  OPARA_POLICY_SEQUENTIAL = 1,
  OPARA_POLICY_DFS = 2,
  OPARA_POLICY_WAVEFRONT = 3
} opara_policy;

/* IEEE-double dominant share, same operation order as orderer.py:48-53. */
opara_status opara_dominant_share(const opara_node* node, const opara_gpu_config* cfg, double* out);
/* Launch order (n node ids).  cfg may be NULL for the non-opara policies. */
opara_status opara_order(const opara_dag* dag, int32_t policy, const opara_gpu_config* cfg,
                         int64_t* out);

/* Every linear extension of the DAG in lexicographic order by node id (the
 * enumeration order of oracle.linear_extensions, oracle.py:52-84).  Skips the
 * first `skip` extensions, then writes up to `cap` orders of n ids each into
 * out[cap][n]; *written receives the number written and *exhausted 1 when the
 * enumeration ended inside this call (no extension after the last written). */
opara_status opara_linear_extensions(const opara_dag* dag, int64_t skip, int64_t cap, int64_t* out,
                                     int64_t* written, int32_t* exhausted);

/* -------------------------------------------- execution model (L4) */

typedef struct opara_sim_result {
  int64_t makespan_ns;
  int64_t blocked_ns;      /* sum of (first block placed - eligible) */
  int64_t sync_wait_ns;    /* sum of (eligible - reached stream head) */
  double sm_efficiency;    /* sum(sm busy) / (num_sms * makespan) */
} opara_sim_result;

/* The reference's discrete-event multi-SM execution model, bit-exact
 * (replaces simulate, simulator.py:212-415; semantics simulator.py:1-26).
 * Per-node arrays are in ascending-id order: block_duration_ns[i]
 * (OperatorNode.block_duration_ns), stream_of[i].  order = n node ids (a
 * linear extension), sync_uv = n_sync node-id pairs.  Optional outputs (NULL
 * to skip): op_start_ns / op_end_ns per node (first block placed / last block
 * done), sm_busy_ns[num_sms], block_log rows (op id, block index, sm, start,
 * end) up to block_log_cap rows; *n_blocks receives the placed-block count.
 * The host checks coverage / plan validity first (CoverageError,
 * PlanViolationError, InfeasibleBlockError wording of _check_inputs). */
opara_status opara_simulate(const opara_dag* dag, const int64_t* block_duration_ns, const int32_t* stream_of,
                            int32_t num_streams, const int64_t* order, const int64_t* sync_uv, int64_t n_sync,
                            const opara_gpu_config* cfg, opara_sim_result* out, int64_t* op_start_ns,
                            int64_t* op_end_ns, int64_t* sm_busy_ns, int64_t* block_log, int64_t block_log_cap,
                            int64_t* n_blocks);

/* ------------------------------------------- executor (subsystems 3 + 4) */

/* Operator kinds understood by the executor.  Parameter layout per kind is
 * documented in paper_2312_10351_b200/csrc/ops.h (struct opara_op.i[]). */
typedef enum opara_op_kind {
  OPARA_OP_NOP = 0,         /* join point without a kernel (eliminated concat):
                               capture only applies its waits and records      */
  OPARA_OP_CONV2D = 1,     /* NHWC implicit-GEMM conv + folded BN bias + ReLU, slice store */
  OPARA_OP_MAXPOOL2D = 2,   /* NHWC window max (ceil_mode aware)                          */
  OPARA_OP_AVGPOOL2D = 3,   /* NHWC window mean (count_include_pad aware)                 */
  OPARA_OP_GLOBAL_AVGPOOL = 4,
  OPARA_OP_LINEAR = 5,      /* y = act(x W^T + b), row-major                              */
  OPARA_OP_ADD = 6,         /* y = act(x0 + .. + x3) over channel views (csrc/elementwise.cu) */
  OPARA_OP_LAYERNORM = 7,   /* y = LN(x (+ residual))                                     */
  OPARA_OP_GELU = 8,
  OPARA_OP_EMBEDDING = 9,   /* row gather (+ position + type rows)                        */
  OPARA_OP_ATTENTION = 10,  /* softmax(Q K^T * scale + mask) V per head                   */
  OPARA_OP_COPY = 11,       /* strided channel-slice copy (+act)                          */
  OPARA_OP_FM = 12,         /* factorization-machine interaction      (csrc/deepfm.cu)    */
  OPARA_OP_DWCONV2D = 13,   /* depthwise conv, fused input ReLU       (csrc/dwconv.cu)    */
  OPARA_OP_RELU = 14,       /* unfused ReLU over a channel view                           */
  OPARA_OP_SOFTMAX = 15,    /* reserved                                                   */
  OPARA_OP_FIELD_EMBEDDING = 16, /* per-field embedding row gather into a slice (deepfm.cu) */
  OPARA_OP_FIRST_ORDER = 17, /* DeepFM linear part: sum of per-field weights + dense dot   */
  OPARA_OP_PACK_INPUT = 18  /* fp32 NCHW image -> NHWC bf16 with channels zero-padded to 8 */
} opara_op_kind;

#define OPARA_OP_MAX_INTS 40
#define OPARA_OP_MAX_PTRS 8

/* One kernel launch: a POD record the host fills in.  Pointers are device
 * addresses owned by the caller; the executor never frees them. */
typedef struct opara_op {
  int32_t kind;       /* opara_op_kind */
  int32_t variant;    /* kernel variant (tile shape, dtype, engine) */
  int64_t i[OPARA_OP_MAX_INTS];
  double f[4];
  void* p[OPARA_OP_MAX_PTRS];
} opara_op;

/* Per-op launch profile: the measured ResourceDemand plus isolated time. */
typedef struct opara_op_profile {
  int64_t num_blocks;
  int64_t threads_per_block;
  int64_t shared_mem_per_block;    /* static + dynamic bytes */
  int64_t registers_per_thread;
  double isolated_us;              /* median of in-stream event timings */
  int64_t tmem_columns;            /* TMEM columns one block allocates (0: none) */
  int64_t cluster_size;            /* thread-block cluster size (1: no cluster) */
} opara_op_profile;

typedef struct opara_exec opara_exec;

/* Create an executor for n ops on `device`.  The op records are copied. */
opara_status opara_exec_create(int32_t device, const opara_op* ops, int64_t n, opara_exec** out);
void opara_exec_destroy(opara_exec* ex);

/* Capture one multi-stream CUDA Graph into `slot`:
 *   stream_of[i]  plan stream of op i (dense 0..num_streams-1)
 *   order[k]      op indices in launch order (a linear extension)
 *   sync_uv       n_sync (u, v) op-index pairs; one event record after u and
 *                 one stream wait before v per pair (no coalescing)
 * Every plan stream forks from and joins back to the capture origin stream.
 * The sequential baseline is the same call with a single stream and the topo
 * order.  Errors: OPARA_ERR_COVERAGE / OPARA_ERR_PLAN_VIOLATION for bad plans. */
opara_status opara_exec_capture(opara_exec* ex, int32_t slot, const int32_t* stream_of,
                                int32_t num_streams, const int64_t* order, const int64_t* sync_uv,
                                int64_t n_sync);
/* Replay the graph in `slot` on a caller stream (cudaStream_t as void*; NULL =
 * the legacy default stream).  Asynchronous. */
/* Per-op CUDA scheduling priority for graphs captured afterwards (NULL clears):
 * lower = more urgent, clamped to cudaDeviceGetStreamPriorityRange; captured
 * graphs are instantiated with cudaGraphInstantiateFlagUseNodePriority. */
opara_status opara_exec_set_priorities(opara_exec* ex, const int32_t* prio);
opara_status opara_exec_replay(opara_exec* ex, int32_t slot, void* stream);
/* Launch every op eagerly in `order` on one stream (debugging / profiling). */
opara_status opara_exec_run_eager(opara_exec* ex, const int64_t* order, int64_t n, void* stream);
/* Measure each op alone: grid, block, registers, shared memory and the median
 * of `reps` event-timed launches. */
opara_status opara_exec_profile(opara_exec* ex, int32_t reps, opara_op_profile* out);
/* Replay `slot` once with kernel timestamps enabled: start_ns/end_ns[i] get
 * the earliest block start and latest block end (%globaltimer) of op i. */
opara_status opara_exec_trace(opara_exec* ex, int32_t slot, void* stream, int64_t* start_ns,
                              int64_t* end_ns);
/* Time `iters` replays of `slot` after `warmup` replays; out_ms receives per-
 * replay milliseconds (CUDA events on the replay stream, bracketing the replay
 * only).  When flush_bytes > 0 the device buffer `flush` is overwritten before
 * every replay (outside the timed bracket) so L2 starts cold each time. */
opara_status opara_exec_time(opara_exec* ex, int32_t slot, int32_t warmup, int32_t iters,
                             void* stream, void* flush, int64_t flush_bytes, float* out_ms);
/* Number of kernel launches one replay of `slot` performs. */
int64_t opara_exec_num_launches(const opara_exec* ex, int32_t slot);

/* ----------------------------------------------------------- device info */

/* Fill a GpuConfig from cudaGetDeviceProperties (the `b200` preset). */
opara_status opara_device_gpu_config(int32_t device, opara_gpu_config* out);

/* Launch configuration of one op without touching the device: grid blocks,
 * threads per block and dynamic+static shared memory (registers_per_thread
 * is filled only when a device is present, else 0).  Used to build the DAG's
 * ResourceDemand before profiling. */
opara_status opara_op_launch_config(const opara_op* op, opara_op_profile* out);

#ifdef __cplusplus
}
#endif

#endif /* OPARA_H_ */
