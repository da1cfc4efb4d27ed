// Executor half of libopara: multi-stream CUDA Graph capture of a (plan,
// launch order) pair with per-edge event fork/join, replay, per-op profiling
// and kernel timelines.
//
// Execution contract (simulator.py:5-18): every plan stream is a
// FIFO filled in launch order; a kernel waits for its stream predecessor and
// for every cross-stream producer (one event record after the producer, one
// stream wait before the consumer, per sync edge, no coalescing).  Capture
// records exactly those dependencies; cudaGraphInstantiate turns them into
// graph edges, so the replay honours the plan with zero host involvement.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "ops.h"
#include "status.h"

namespace opara {

opara_status cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return OPARA_OK;
  return fail(OPARA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                                  cudaGetErrorString(e) + ")");
}

// Per-launch scheduling priority applied by launch_kernel (0 = default); the
// capture sets it per op from opara_exec_set_priorities.
thread_local int g_launch_priority = 0;

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("OPARA_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

opara_status launch_kernel(const LaunchCfg& c, void** args, cudaStream_t s, unsigned cluster_z) {
  return launch_kernel_cluster(c, args, s, dim3(1, 1, cluster_z));
}

opara_status launch_kernel_cluster(const LaunchCfg& c, void** args, cudaStream_t s, dim3 cluster) {
  const unsigned cluster_z = cluster.x * cluster.y * cluster.z;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = c.grid;
  lc.blockDim = c.block;
  lc.dynamicSmemBytes = c.smem;
  lc.stream = s;
  cudaLaunchAttribute attr[3];
  unsigned n = 0;
  if (g_launch_priority != 0) {
    attr[n].id = cudaLaunchAttributePriority;
    attr[n].val.priority = g_launch_priority;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_z > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster.x;
    attr[n].val.clusterDim.y = cluster.y;
    attr[n].val.clusterDim.z = cluster.z;
    ++n;
  }
  lc.attrs = attr;
  lc.numAttrs = n;
  return cuda_fail(cudaLaunchKernelExC(&lc, c.func, args), "kernel launch");
}

opara_status launch_op(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                       LaunchCfg* cfg, bool dry) {
  switch (op.kind) {
    case OPARA_OP_NOP:
      if (cfg) *cfg = LaunchCfg{};
      return OPARA_OK;
    case OPARA_OP_CONV2D:
      return op.i[22] == 2   ? launch_conv2d_tc_bf16(op, s, trace, cfg, dry)
             : op.i[22] == 1 ? launch_conv2d_tc(op, s, trace, cfg, dry)
                             : launch_conv2d(op, s, trace, cfg, dry);
    case OPARA_OP_MAXPOOL2D:
    case OPARA_OP_AVGPOOL2D: return launch_pool2d(op, s, trace, cfg, dry);
    case OPARA_OP_GLOBAL_AVGPOOL: return launch_global_avgpool(op, s, trace, cfg, dry);
    case OPARA_OP_LINEAR: return launch_linear(op, s, trace, cfg, dry);
    case OPARA_OP_LAYERNORM:
    case OPARA_OP_EMBEDDING: return launch_rows(op, s, trace, cfg, dry);
    case OPARA_OP_ATTENTION: return launch_attention(op, s, trace, cfg, dry);
    case OPARA_OP_ADD:
    case OPARA_OP_COPY:
    case OPARA_OP_RELU: return launch_elementwise(op, s, trace, cfg, dry);
    case OPARA_OP_DWCONV2D: return launch_dwconv2d(op, s, trace, cfg, dry);
    case OPARA_OP_FIELD_EMBEDDING:
    case OPARA_OP_FIRST_ORDER:
    case OPARA_OP_FM: return launch_deepfm(op, s, trace, cfg, dry);
    case OPARA_OP_PACK_INPUT: return launch_pack_input(op, s, trace, cfg, dry);
    default: return fail(OPARA_ERR_VALUE, "unsupported op kind " + std::to_string(op.kind));
  }
}

}  // namespace opara

using opara::cuda_fail;
using opara::fail;

#define OPARA_CUDA(call)                                  \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
  } while (0)

struct opara_exec {
  struct Plan {
    std::vector<int32_t> stream_of;
    int32_t num_streams = 0;
    std::vector<int64_t> order;
    std::vector<int64_t> sync;  // flattened (u, v) op indices
  };
  struct Graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
  };
  int32_t device = 0;
  std::vector<opara_op> ops;
  std::vector<int32_t> prio;   // per-op CUDA priority for captured graphs (empty = none)
  std::map<int32_t, Plan> plans;
  std::map<int32_t, Graph> graphs;         // plain replay graphs
  std::map<int32_t, Graph> traced_graphs;  // same plan, kernels write timestamps
  unsigned long long* trace_buf = nullptr;  // 2 * ops.size()
  std::vector<void*> workspaces;

  ~opara_exec() {
    cudaSetDevice(device);
    for (void* w : workspaces) cudaFree(w);
    for (auto* m : {&graphs, &traced_graphs})
      for (auto& kv : *m) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
      }
    if (trace_buf) cudaFree(trace_buf);
  }
};

namespace {

opara_status check_plan(const opara_exec& ex, const opara_exec::Plan& p) {
  const int64_t n = static_cast<int64_t>(ex.ops.size());
  if (static_cast<int64_t>(p.stream_of.size()) != n || static_cast<int64_t>(p.order.size()) != n)
    return fail(OPARA_ERR_COVERAGE, "plan/order must cover every op exactly once");
  if (n > 0 && p.num_streams < 1) return fail(OPARA_ERR_PLAN_VIOLATION, "num_streams must be >= 1");
  std::vector<int64_t> pos(n, -1);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t v = p.order[k];
    if (v < 0 || v >= n || pos[v] >= 0)
      return fail(OPARA_ERR_COVERAGE, "launch order must cover the graph exactly");
    pos[v] = k;
  }
  for (int64_t i = 0; i < n; ++i)
    if (p.stream_of[i] < 0 || p.stream_of[i] >= p.num_streams)
      return fail(OPARA_ERR_PLAN_VIOLATION, "op " + std::to_string(i) + " has stream outside 0.." +
                                                std::to_string(p.num_streams - 1));
  for (size_t k = 0; k + 1 < p.sync.size(); k += 2) {
    const int64_t u = p.sync[k], v = p.sync[k + 1];
    if (u < 0 || u >= n || v < 0 || v >= n)
      return fail(OPARA_ERR_PLAN_VIOLATION, "sync event references an unknown op");
    if (p.stream_of[u] == p.stream_of[v])
      return fail(OPARA_ERR_PLAN_VIOLATION,
                  "sync event " + opara::py_pair(u, v) + " joins same-stream nodes");
    if (pos[u] >= pos[v])
      return fail(OPARA_ERR_COVERAGE, "launch order is not a linear extension of the graph");
  }
  return OPARA_OK;
}

opara_status capture(opara_exec& ex, const opara_exec::Plan& p, bool traced, opara_exec::Graph* out) {
  const int64_t n = static_cast<int64_t>(ex.ops.size());
  OPARA_CUDA(cudaSetDevice(ex.device));
  std::vector<std::vector<int64_t>> waits(n);
  std::vector<char> records(n, 0);
  for (size_t k = 0; k + 1 < p.sync.size(); k += 2) {
    waits[p.sync[k + 1]].push_back(p.sync[k]);
    records[p.sync[k]] = 1;
  }
  cudaStream_t origin = nullptr;
  std::vector<cudaStream_t> streams(p.num_streams, nullptr);
  std::vector<cudaEvent_t> done(n, nullptr), joins(p.num_streams, nullptr);
  cudaEvent_t fork = nullptr;
  opara_status st = OPARA_OK;
  auto cleanup = [&]() {
    for (auto e : done) if (e) cudaEventDestroy(e);
    for (auto e : joins) if (e) cudaEventDestroy(e);
    if (fork) cudaEventDestroy(fork);
    for (auto s : streams) if (s) cudaStreamDestroy(s);
    if (origin) cudaStreamDestroy(origin);
  };
#define CAP(call)                                 \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) {                      \
      st = cuda_fail(e_, #call);                  \
      goto abort_capture;                         \
    }                                             \
  } while (0)
  CAP(cudaStreamCreateWithFlags(&origin, cudaStreamNonBlocking));
  for (auto& s : streams) CAP(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  for (int64_t i = 0; i < n; ++i)
    if (records[i]) CAP(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
  for (auto& e : joins) CAP(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CAP(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));

  CAP(cudaStreamBeginCapture(origin, cudaStreamCaptureModeThreadLocal));
  CAP(cudaEventRecord(fork, origin));
  for (auto s : streams) CAP(cudaStreamWaitEvent(s, fork, 0));
  for (int64_t k = 0; k < n; ++k) {
    const int64_t v = p.order[k];
    cudaStream_t s = streams[p.stream_of[v]];
    for (int64_t u : waits[v]) CAP(cudaStreamWaitEvent(s, done[u], 0));
    opara::g_launch_priority = ex.prio.empty() ? 0 : ex.prio[v];
    st = opara::launch_op(ex.ops[v], s, traced ? ex.trace_buf + 2 * v : nullptr, nullptr, false);
    opara::g_launch_priority = 0;
    if (st != OPARA_OK) goto abort_capture;
    if (records[v]) CAP(cudaEventRecord(done[v], s));
  }
  for (int32_t k = 0; k < p.num_streams; ++k) {
    CAP(cudaEventRecord(joins[k], streams[k]));
    CAP(cudaStreamWaitEvent(origin, joins[k], 0));
  }
  {
    cudaGraph_t g = nullptr;
    CAP(cudaStreamEndCapture(origin, &g));
    out->graph = g;
    cudaError_t e = cudaGraphInstantiate(&out->exec, g, ex.prio.empty() ? 0 : cudaGraphInstantiateFlagUseNodePriority);
    if (e != cudaSuccess) {
      st = cuda_fail(e, "cudaGraphInstantiate");
      cudaGraphDestroy(g);
      out->graph = nullptr;
    }
  }
  cleanup();
  return st;
abort_capture : {
  cudaStreamCaptureStatus cs;
  if (origin && cudaStreamIsCapturing(origin, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(origin, &g);
    if (g) cudaGraphDestroy(g);
  }
  cudaGetLastError();
  cleanup();
  return st;
}
#undef CAP
}

opara_status ensure_graph(opara_exec& ex, int32_t slot, bool traced, opara_exec::Graph** out) {
  auto pit = ex.plans.find(slot);
  if (pit == ex.plans.end()) return fail(OPARA_ERR_VALUE, "slot " + std::to_string(slot) + " not captured");
  auto& m = traced ? ex.traced_graphs : ex.graphs;
  auto git = m.find(slot);
  if (git != m.end() && git->second.exec) {
    *out = &git->second;
    return OPARA_OK;
  }
  if (traced && !ex.trace_buf) {
    OPARA_CUDA(cudaSetDevice(ex.device));
    OPARA_CUDA(cudaMalloc(&ex.trace_buf, sizeof(unsigned long long) * 2 * std::max<size_t>(1, ex.ops.size())));
  }
  opara_exec::Graph g;
  opara_status st = capture(ex, pit->second, traced, &g);
  if (st != OPARA_OK) return st;
  m[slot] = g;
  *out = &m[slot];
  return OPARA_OK;
}

}  // namespace

extern "C" {

opara_status opara_exec_create(int32_t device, const opara_op* ops, int64_t n, opara_exec** out) {
  opara::g_last_error.clear();
  if (!out || n < 0 || (n && !ops)) return fail(OPARA_ERR_VALUE, "opara_exec_create: bad arguments");
  int count = 0;
  OPARA_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    return fail(OPARA_ERR_CUDA, "device " + std::to_string(device) + " not present");
  OPARA_CUDA(cudaSetDevice(device));
  auto* ex = new opara_exec();
  ex->device = device;
  ex->ops.assign(ops, ops + n);
  for (int64_t i = 0; i < n; ++i) {
    opara::LaunchCfg c;
    opara_status st = opara::launch_op(ex->ops[i], nullptr, nullptr, &c, true);
    if (st != OPARA_OK) {
      delete ex;
      return fail(st, "op " + std::to_string(i) + ": " + opara::g_last_error);
    }
    if (c.workspace > 0) {  // private per-op scratch: concurrent branches never share it
      void* ws = nullptr;
      cudaError_t e = cudaMalloc(&ws, c.workspace);
      if (e == cudaSuccess) e = cudaMemset(ws, 0, c.workspace);
      if (e != cudaSuccess) {
        delete ex;
        return cuda_fail(e, "workspace allocation");
      }
      ex->workspaces.push_back(ws);
      ex->ops[i].p[7] = ws;
    }
  }
  *out = ex;
  return OPARA_OK;
}

void opara_exec_destroy(opara_exec* ex) { delete ex; }

opara_status opara_exec_capture(opara_exec* ex, int32_t slot, const int32_t* stream_of,
                                int32_t num_streams, const int64_t* order, const int64_t* sync_uv,
                                int64_t n_sync) {
  if (!ex) return fail(OPARA_ERR_VALUE, "null executor");
  const int64_t n = static_cast<int64_t>(ex->ops.size());
  if (n && (!stream_of || !order)) return fail(OPARA_ERR_VALUE, "null plan");
  if (n_sync && !sync_uv) return fail(OPARA_ERR_VALUE, "null sync list");
  opara_exec::Plan p;
  p.stream_of.assign(stream_of, stream_of + n);
  p.num_streams = num_streams;
  p.order.assign(order, order + n);
  if (n_sync) p.sync.assign(sync_uv, sync_uv + 2 * n_sync);
  opara_status st = check_plan(*ex, p);
  if (st != OPARA_OK) return st;
  for (auto* m : {&ex->graphs, &ex->traced_graphs}) {
    auto it = m->find(slot);
    if (it != m->end()) {
      if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
      if (it->second.graph) cudaGraphDestroy(it->second.graph);
      m->erase(it);
    }
  }
  ex->plans[slot] = p;
  opara_exec::Graph* g = nullptr;
  st = ensure_graph(*ex, slot, false, &g);
  if (st != OPARA_OK) ex->plans.erase(slot);
  return st;
}

opara_status opara_exec_set_priorities(opara_exec* ex, const int32_t* prio) {
  if (!ex) return fail(OPARA_ERR_VALUE, "null executor");
  if (!prio) {
    ex->prio.clear();
    return OPARA_OK;
  }
  int lo = 0, hi = 0;
  OPARA_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));   // lo = least (0), hi = greatest (negative)
  ex->prio.assign(prio, prio + ex->ops.size());
  for (auto& p : ex->prio) p = std::max(hi, std::min(lo, p));
  return OPARA_OK;
}

opara_status opara_exec_replay(opara_exec* ex, int32_t slot, void* stream) {
  if (!ex) return fail(OPARA_ERR_VALUE, "null executor");
  auto it = ex->graphs.find(slot);
  if (it == ex->graphs.end()) return fail(OPARA_ERR_VALUE, "slot " + std::to_string(slot) + " not captured");
  OPARA_CUDA(cudaSetDevice(ex->device));
  OPARA_CUDA(cudaGraphLaunch(it->second.exec, static_cast<cudaStream_t>(stream)));
  return OPARA_OK;
}

opara_status opara_exec_run_eager(opara_exec* ex, const int64_t* order, int64_t n, void* stream) {
  if (!ex || (n && !order)) return fail(OPARA_ERR_VALUE, "null argument");
  OPARA_CUDA(cudaSetDevice(ex->device));
  for (int64_t k = 0; k < n; ++k) {
    const int64_t v = order[k];
    if (v < 0 || v >= static_cast<int64_t>(ex->ops.size())) return fail(OPARA_ERR_COVERAGE, "bad op index");
    opara_status st = opara::launch_op(ex->ops[v], static_cast<cudaStream_t>(stream), nullptr, nullptr, false);
    if (st != OPARA_OK) return st;
  }
  return OPARA_OK;
}

opara_status opara_op_launch_config(const opara_op* op, opara_op_profile* out) {
  if (!op || !out) return fail(OPARA_ERR_VALUE, "null argument");
  opara::LaunchCfg c;
  opara_status st = opara::launch_op(*op, nullptr, nullptr, &c, true);
  if (st != OPARA_OK) return st;
  out->num_blocks = static_cast<int64_t>(c.grid.x) * c.grid.y * c.grid.z;
  out->threads_per_block = static_cast<int64_t>(c.block.x) * c.block.y * c.block.z;
  out->shared_mem_per_block = static_cast<int64_t>(c.smem);
  out->registers_per_thread = 0;
  out->isolated_us = 0.0;
  out->tmem_columns = c.tmem_cols;
  out->cluster_size = c.cluster;
  int count = 0;
  if (c.func && cudaGetDeviceCount(&count) == cudaSuccess && count > 0) {
    cudaFuncAttributes attr;
    if (cudaFuncGetAttributes(&attr, c.func) == cudaSuccess) {
      out->registers_per_thread = attr.numRegs;
      out->shared_mem_per_block += static_cast<int64_t>(attr.sharedSizeBytes);
    }
  }
  cudaGetLastError();
  return OPARA_OK;
}

opara_status opara_exec_profile(opara_exec* ex, int32_t reps, opara_op_profile* out) {
  if (!ex || !out) return fail(OPARA_ERR_VALUE, "null argument");
  if (reps < 1) reps = 1;
  OPARA_CUDA(cudaSetDevice(ex->device));
  cudaStream_t s;
  OPARA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  opara_status st = OPARA_OK;
  for (size_t i = 0; i < ex->ops.size() && st == OPARA_OK; ++i) {
    opara::LaunchCfg c;
    st = opara::launch_op(ex->ops[i], s, nullptr, &c, true);
    if (st != OPARA_OK) break;
    if (!c.func) {  // NOP join: no kernel, no demand
      out[i] = opara_op_profile{1, 0, 0, 0, 0.0, 0, 1};
      continue;
    }
    cudaFuncAttributes attr;
    if (cudaFuncGetAttributes(&attr, c.func) != cudaSuccess) {
      st = fail(OPARA_ERR_CUDA, "cudaFuncGetAttributes failed");
      break;
    }
    opara_op_profile& p = out[i];
    p.num_blocks = static_cast<int64_t>(c.grid.x) * c.grid.y * c.grid.z;
    p.threads_per_block = static_cast<int64_t>(c.block.x) * c.block.y * c.block.z;
    p.shared_mem_per_block = static_cast<int64_t>(c.smem) + static_cast<int64_t>(attr.sharedSizeBytes);
    p.registers_per_thread = attr.numRegs;
    p.tmem_columns = c.tmem_cols;
    p.cluster_size = c.cluster;
    // In-graph duration: a graph of `reps` back-to-back launches of this op,
    // replayed three times; the median per-launch time is kept.
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      st = fail(OPARA_ERR_CUDA, "profile capture begin failed");
      break;
    }
    for (int r = 0; r < reps && st == OPARA_OK; ++r) st = opara::launch_op(ex->ops[i], s, nullptr, nullptr, false);
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (st != OPARA_OK) { if (g) cudaGraphDestroy(g); break; }
    if (e != cudaSuccess || cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
      st = fail(OPARA_ERR_CUDA, "profile graph instantiate failed");
      if (g) cudaGraphDestroy(g);
      break;
    }
    std::vector<float> ms;
    cudaGraphLaunch(ge, s);  // warm-up
    for (int t = 0; t < 3; ++t) {
      cudaEventRecord(a, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float x = 0.f;
      cudaEventElapsedTime(&x, a, b);
      ms.push_back(x);
    }
    std::sort(ms.begin(), ms.end());
    p.isolated_us = 1000.0 * ms[1] / reps;
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) st = cuda_fail(le, "profile");
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(s);
  return st;
}

opara_status opara_exec_trace(opara_exec* ex, int32_t slot, void* stream, int64_t* start_ns,
                              int64_t* end_ns) {
  if (!ex || !start_ns || !end_ns) return fail(OPARA_ERR_VALUE, "null argument");
  opara_exec::Graph* g = nullptr;
  opara_status st = ensure_graph(*ex, slot, true, &g);
  if (st != OPARA_OK) return st;
  const size_t n = ex->ops.size();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<unsigned long long> host(2 * n);
  for (size_t i = 0; i < n; ++i) {
    host[2 * i] = ~0ull;
    host[2 * i + 1] = 0ull;
  }
  // warm replays first: the first launch of a fresh executable graph uploads
  // it to the device and would stretch the timeline
  for (int w = 0; w < 3; ++w) OPARA_CUDA(cudaGraphLaunch(g->exec, s));
  OPARA_CUDA(cudaMemcpyAsync(ex->trace_buf, host.data(), sizeof(unsigned long long) * 2 * n,
                             cudaMemcpyHostToDevice, s));
  OPARA_CUDA(cudaGraphLaunch(g->exec, s));
  OPARA_CUDA(cudaMemcpyAsync(host.data(), ex->trace_buf, sizeof(unsigned long long) * 2 * n,
                             cudaMemcpyDeviceToHost, s));
  OPARA_CUDA(cudaStreamSynchronize(s));
  for (size_t i = 0; i < n; ++i) {
    start_ns[i] = static_cast<int64_t>(host[2 * i]);
    end_ns[i] = static_cast<int64_t>(host[2 * i + 1]);
  }
  return OPARA_OK;
}

opara_status opara_exec_time(opara_exec* ex, int32_t slot, int32_t warmup, int32_t iters,
                             void* stream, void* flush, int64_t flush_bytes, float* out_ms) {
  if (!ex || (iters > 0 && !out_ms)) return fail(OPARA_ERR_VALUE, "null argument");
  auto it = ex->graphs.find(slot);
  if (it == ex->graphs.end()) return fail(OPARA_ERR_VALUE, "slot " + std::to_string(slot) + " not captured");
  OPARA_CUDA(cudaSetDevice(ex->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int k = 0; k < warmup; ++k) OPARA_CUDA(cudaGraphLaunch(it->second.exec, s));
  std::vector<cudaEvent_t> ev(2 * std::max(iters, 0));
  for (auto& e : ev) OPARA_CUDA(cudaEventCreate(&e));
  opara_status st = OPARA_OK;
  for (int k = 0; k < iters && st == OPARA_OK; ++k) {
    if (flush && flush_bytes > 0) {
      cudaError_t e = cudaMemsetAsync(flush, k & 0xff, static_cast<size_t>(flush_bytes), s);
      if (e != cudaSuccess) st = cuda_fail(e, "flush");
    }
    cudaEventRecord(ev[2 * k], s);
    cudaError_t e = cudaGraphLaunch(it->second.exec, s);
    if (e != cudaSuccess) st = cuda_fail(e, "cudaGraphLaunch");
    cudaEventRecord(ev[2 * k + 1], s);
  }
  cudaError_t e = cudaStreamSynchronize(s);
  if (st == OPARA_OK && e != cudaSuccess) st = cuda_fail(e, "replay");
  for (int k = 0; k < iters && st == OPARA_OK; ++k)
    cudaEventElapsedTime(&out_ms[k], ev[2 * k], ev[2 * k + 1]);
  for (auto& x : ev) cudaEventDestroy(x);
  return st;
}

int64_t opara_exec_num_launches(const opara_exec* ex, int32_t slot) {
  if (!ex || !ex->plans.count(slot)) return 0;
  int64_t n = 0;
  for (const auto& op : ex->ops) n += op.kind != OPARA_OP_NOP;
  return n;
}

opara_status opara_device_gpu_config(int32_t device, opara_gpu_config* out) {
  if (!out) return fail(OPARA_ERR_VALUE, "null argument");
  cudaDeviceProp p;
  OPARA_CUDA(cudaGetDeviceProperties(&p, device));
  out->num_sms = p.multiProcessorCount;
  out->threads_per_sm = p.maxThreadsPerMultiProcessor;
  out->shared_mem_per_sm = static_cast<int64_t>(p.sharedMemPerMultiprocessor);
  out->registers_per_sm = p.regsPerMultiprocessor;
  out->max_blocks_per_sm = p.maxBlocksPerMultiProcessor;
  out->same_class_slowdown = 1.4;
  return OPARA_OK;
}

}  // extern "C"
