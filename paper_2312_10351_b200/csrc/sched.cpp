// Scheduler half of libopara: DAG model, Alg. 1 stream allocation, Alg. 2
// resource-aware launch order and the baseline orders, behind the C ABI in
// include/opara.h.  Host-only C++17; no CUDA here.
//
// Determinism contract: every tie breaks by
// ascending node id.  Nodes are stored sorted by id, so "ascending id" equals
// "ascending dense index" everywhere below and all heaps/sorts run on indices.
//
// Compile without -ffast-math and with -ffp-contract=off: dominant_share must
// reproduce Python's correctly-rounded int/int division bit for bit.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <functional>
#include <queue>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "opara.h"
#include "dag_internal.h"
#include "status.h"

namespace opara {

thread_local std::string g_last_error;

opara_status fail(opara_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

std::string py_int_list(const std::vector<int64_t>& v) {
  std::string s = "[";
  for (size_t k = 0; k < v.size(); ++k) {
    if (k) s += ", ";
    s += std::to_string(v[k]);
  }
  return s + "]";
}

std::string py_pair(int64_t u, int64_t v) {
  return "(" + std::to_string(u) + ", " + std::to_string(v) + ")";
}

}  // namespace opara

using opara::fail;


namespace {

// graph.py:138-153 — Kahn over a min-heap of ids.
bool lexicographic_topo(opara_dag& g, std::vector<int32_t>* stuck) {
  const int32_t n = g.n();
  std::vector<int32_t> missing(n);
  for (int32_t i = 0; i < n; ++i) missing[i] = g.pred_off[i + 1] - g.pred_off[i];
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> heap;
  for (int32_t i = 0; i < n; ++i)
    if (missing[i] == 0) heap.push(i);
  g.topo.clear();
  g.topo.reserve(n);
  while (!heap.empty()) {
    int32_t v = heap.top();
    heap.pop();
    g.topo.push_back(v);
    for (int32_t k = g.succ_off[v]; k < g.succ_off[v + 1]; ++k)
      if (--missing[g.succ[k]] == 0) heap.push(g.succ[k]);
  }
  if (static_cast<int32_t>(g.topo.size()) == n) return true;
  for (int32_t i = 0; i < n; ++i)
    if (missing[i] > 0) stuck->push_back(i);
  return false;
}

void build_csr(int32_t n, const std::vector<std::pair<int32_t, int32_t>>& e, bool by_target,
               std::vector<int32_t>* off, std::vector<int32_t>* adj) {
  off->assign(n + 1, 0);
  for (auto& uv : e) (*off)[(by_target ? uv.second : uv.first) + 1]++;
  for (int32_t i = 0; i < n; ++i) (*off)[i + 1] += (*off)[i];
  adj->assign(e.size(), 0);
  std::vector<int32_t> fill(off->begin(), off->end() - 1);
  // edges are sorted by (u, v): succ lists come out ascending; pred lists get
  // sorted explicitly below.
  for (auto& uv : e) {
    if (by_target)
      (*adj)[fill[uv.second]++] = uv.first;
    else
      (*adj)[fill[uv.first]++] = uv.second;
  }
  for (int32_t i = 0; i < n; ++i) std::sort(adj->begin() + (*off)[i], adj->begin() + (*off)[i + 1]);
}

double share_of(const opara_node& d, const opara_gpu_config& c) {
  // orderer.py:48-53: max(threads/tps, smem/smps, regs_per_block/rps) * blocks
  const double a = static_cast<double>(d.threads_per_block) / static_cast<double>(c.threads_per_sm);
  const double b =
      static_cast<double>(d.shared_mem_per_block) / static_cast<double>(c.shared_mem_per_sm);
  const double r = static_cast<double>(d.registers_per_thread * d.threads_per_block) /
                   static_cast<double>(c.registers_per_sm);
  double m = a;
  if (b > m) m = b;
  if (r > m) m = r;
  return m * static_cast<double>(d.num_blocks);
}

opara_status check_cfg(const opara_gpu_config* c) {
  if (!c) return fail(OPARA_ERR_VALUE, "gpu config is required for the opara policy");
  if (c->threads_per_sm < 1) return fail(OPARA_ERR_VALUE, "threads_per_sm must be >= 1");
  if (c->shared_mem_per_sm < 1) return fail(OPARA_ERR_VALUE, "shared_mem_per_sm must be >= 1");
  if (c->registers_per_sm < 1) return fail(OPARA_ERR_VALUE, "registers_per_sm must be >= 1");
  return OPARA_OK;
}

std::vector<int32_t> order_opara(const opara_dag& g, const opara_gpu_config& cfg) {
  // orderer.py:60-88 — two min-heaps keyed (share, id); memory first; after
  // each pop prefer the class NOT just launched.
  const int32_t n = g.n();
  std::vector<double> score(n);
  for (int32_t i = 0; i < n; ++i) score[i] = share_of(g.nodes[i], cfg);
  using Key = std::pair<double, int32_t>;
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap[2];
  std::vector<int32_t> missing(n);
  for (int32_t i = 0; i < n; ++i) {
    missing[i] = g.pred_off[i + 1] - g.pred_off[i];
    if (missing[i] == 0) heap[g.nodes[i].op_class].push({score[i], i});
  }
  std::vector<int32_t> out;
  out.reserve(n);
  int32_t want = OPARA_MEMORY;
  while (!heap[0].empty() || !heap[1].empty()) {
    const int32_t took = heap[want].empty() ? 1 - want : want;
    const int32_t v = heap[took].top().second;
    heap[took].pop();
    out.push_back(v);
    for (int32_t k = g.succ_off[v]; k < g.succ_off[v + 1]; ++k) {
      const int32_t s = g.succ[k];
      if (--missing[s] == 0) heap[g.nodes[s].op_class].push({score[s], s});
    }
    want = 1 - took;
  }
  return out;
}

std::vector<int32_t> order_dfs(const opara_dag& g) {
  // orderer.py:91-110 — emit a node when its last predecessor is emitted,
  // resuming each parent's successor scan where it stopped.
  const int32_t n = g.n();
  std::vector<int32_t> missing(n);
  for (int32_t i = 0; i < n; ++i) missing[i] = g.pred_off[i + 1] - g.pred_off[i];
  std::vector<int32_t> roots;
  for (int32_t i = 0; i < n; ++i)
    if (missing[i] == 0) roots.push_back(i);
  std::vector<int32_t> out;
  out.reserve(n);
  std::vector<std::pair<int32_t, int32_t>> stack;  // (node, next successor slot)
  for (int32_t r : roots) {
    out.push_back(r);
    stack.push_back({r, g.succ_off[r]});
    while (!stack.empty()) {
      auto& top = stack.back();
      const int32_t v = top.first;
      bool pushed = false;
      while (top.second < g.succ_off[v + 1]) {
        const int32_t s = g.succ[top.second++];
        if (--missing[s] == 0) {
          out.push_back(s);
          stack.push_back({s, g.succ_off[s]});  // invalidates `top`
          pushed = true;
          break;
        }
      }
      if (!pushed) stack.pop_back();
    }
  }
  return out;
}

std::vector<int32_t> order_wavefront(const opara_dag& g) {
  // orderer.py:113-118 — (level, id) ascending.
  const int32_t n = g.n();
  std::vector<int64_t> level(n, 0);
  for (int32_t v : g.topo) {
    int64_t lv = 0;
    for (int32_t k = g.pred_off[v]; k < g.pred_off[v + 1]; ++k)
      lv = std::max(lv, level[g.pred[k]] + 1);
    level[v] = lv;
  }
  std::vector<int32_t> out(n);
  for (int32_t i = 0; i < n; ++i) out[i] = i;
  std::stable_sort(out.begin(), out.end(),
                   [&](int32_t a, int32_t b) { return level[a] < level[b]; });
  return out;
}

}  // namespace

extern "C" {

const char* opara_last_error(void) { return opara::g_last_error.c_str(); }
#ifndef OPARA_SOURCE_HASH
#define OPARA_SOURCE_HASH "unknown"
#endif
// "<version> sm_100a src:<sha1 of every csrc/include source + nvcc flags>" (build.py
// source_hash): ties a loaded binary to the sources it was built from.
const char* opara_version(void) { return "0.1.0 sm_100a src:" OPARA_SOURCE_HASH; }

opara_status opara_dag_create(const opara_node* nodes, int64_t n, const int64_t* edges_uv,
                              int64_t m, opara_dag** out) {
  opara::g_last_error.clear();
  if (!out || (n > 0 && !nodes) || (m > 0 && !edges_uv) || n < 0 || m < 0)
    return fail(OPARA_ERR_VALUE, "opara_dag_create: bad arguments");
  if (n > INT32_MAX - 1) return fail(OPARA_ERR_VALUE, "opara_dag_create: too many nodes");
  try {
    auto* g = new opara_dag();
    g->nodes.assign(nodes, nodes + n);
    std::stable_sort(g->nodes.begin(), g->nodes.end(),
                     [](const opara_node& a, const opara_node& b) { return a.id < b.id; });
    g->index.reserve(static_cast<size_t>(n) * 2);
    for (int32_t i = 0; i < g->n(); ++i) {
      if (i > 0 && g->nodes[i].id == g->nodes[i - 1].id) {
        const int64_t dup = g->nodes[i].id;
        delete g;
        return fail(OPARA_ERR_GRAPH_VALIDATION, "duplicate node id " + std::to_string(dup));
      }
      g->index.emplace(g->nodes[i].id, i);
    }
    std::unordered_set<uint64_t> seen;
    seen.reserve(static_cast<size_t>(m) * 2);
    std::vector<std::pair<int32_t, int32_t>> e;
    e.reserve(m);
    for (int64_t k = 0; k < m; ++k) {
      const int64_t u = edges_uv[2 * k], v = edges_uv[2 * k + 1];
      auto iu = g->index.find(u), iv = g->index.find(v);
      if (iu == g->index.end() || iv == g->index.end()) {
        delete g;
        return fail(OPARA_ERR_GRAPH_VALIDATION,
                    "edge " + opara::py_pair(u, v) + " references an unknown node");
      }
      if (u == v) {
        delete g;
        return fail(OPARA_ERR_GRAPH_VALIDATION, "self-edge " + opara::py_pair(u, v));
      }
      const uint64_t key = (static_cast<uint64_t>(iu->second) << 32) | static_cast<uint32_t>(iv->second);
      if (!seen.insert(key).second) {
        delete g;
        return fail(OPARA_ERR_GRAPH_VALIDATION, "duplicate edge " + opara::py_pair(u, v));
      }
      e.push_back({iu->second, iv->second});
    }
    std::sort(e.begin(), e.end());
    g->edges = e;
    build_csr(g->n(), g->edges, false, &g->succ_off, &g->succ);
    build_csr(g->n(), g->edges, true, &g->pred_off, &g->pred);
    std::vector<int32_t> stuck;
    if (!lexicographic_topo(*g, &stuck)) {
      std::vector<int64_t> ids;
      for (int32_t i : stuck) ids.push_back(g->id(i));
      delete g;
      return fail(OPARA_ERR_GRAPH_VALIDATION, "cycle involving nodes " + opara::py_int_list(ids));
    }
    *out = g;
    return OPARA_OK;
  } catch (const std::exception& ex) {
    return fail(OPARA_ERR_INTERNAL, std::string("opara_dag_create: ") + ex.what());
  }
}

void opara_dag_destroy(opara_dag* dag) { delete dag; }
int64_t opara_dag_num_nodes(const opara_dag* dag) { return dag ? dag->n() : 0; }
int64_t opara_dag_num_edges(const opara_dag* dag) {
  return dag ? static_cast<int64_t>(dag->edges.size()) : 0;
}

opara_status opara_dag_node_ids(const opara_dag* g, int64_t* out) {
  if (!g || !out) return fail(OPARA_ERR_VALUE, "null argument");
  for (int32_t i = 0; i < g->n(); ++i) out[i] = g->id(i);
  return OPARA_OK;
}

opara_status opara_dag_edges(const opara_dag* g, int64_t* out) {
  if (!g || (!out && !g->edges.empty())) return fail(OPARA_ERR_VALUE, "null argument");
  for (size_t k = 0; k < g->edges.size(); ++k) {
    out[2 * k] = g->id(g->edges[k].first);
    out[2 * k + 1] = g->id(g->edges[k].second);
  }
  return OPARA_OK;
}

opara_status opara_dag_topo_sort(const opara_dag* g, int64_t* out) {
  if (!g || (!out && g->n())) return fail(OPARA_ERR_VALUE, "null argument");
  for (int32_t k = 0; k < g->n(); ++k) out[k] = g->id(g->topo[k]);
  return OPARA_OK;
}

static opara_status adjacency(const opara_dag* g, int64_t id, const std::vector<int32_t>& off,
                              const std::vector<int32_t>& adj, int64_t* out, int64_t cap,
                              int64_t* count) {
  if (!g || !count) return fail(OPARA_ERR_VALUE, "null argument");
  auto it = g->index.find(id);
  if (it == g->index.end()) return fail(OPARA_ERR_KEY, "unknown node id " + std::to_string(id));
  const int32_t i = it->second;
  const int64_t deg = off[i + 1] - off[i];
  *count = deg;
  if (deg > cap || (deg && !out)) return fail(OPARA_ERR_CAPACITY, "adjacency buffer too small");
  for (int64_t k = 0; k < deg; ++k) out[k] = g->id(adj[off[i] + k]);
  return OPARA_OK;
}

opara_status opara_dag_predecessors(const opara_dag* g, int64_t id, int64_t* out, int64_t cap,
                                    int64_t* count) {
  return g ? adjacency(g, id, g->pred_off, g->pred, out, cap, count)
           : fail(OPARA_ERR_VALUE, "null argument");
}

opara_status opara_dag_successors(const opara_dag* g, int64_t id, int64_t* out, int64_t cap,
                                  int64_t* count) {
  return g ? adjacency(g, id, g->succ_off, g->succ, out, cap, count)
           : fail(OPARA_ERR_VALUE, "null argument");
}

opara_status opara_allocate_streams(const opara_dag* g, int32_t* stream_of, int32_t* num_streams,
                                    int64_t* sync_uv, int64_t* num_sync) {
  // allocator.py:43-67 (Alg. 1).
  if (!g || !num_streams || !num_sync || (g->n() && !stream_of) || (!g->edges.empty() && !sync_uv))
    return fail(OPARA_ERR_VALUE, "null argument");
  const int32_t n = g->n();
  std::vector<char> donated(n, 0);
  int32_t next = 0;
  for (int32_t v : g->topo) {
    int32_t donor = -1;
    for (int32_t k = g->pred_off[v]; k < g->pred_off[v + 1]; ++k) {
      if (!donated[g->pred[k]]) {
        donor = g->pred[k];
        break;
      }
    }
    if (donor < 0) {
      stream_of[v] = next++;
    } else {
      stream_of[v] = stream_of[donor];
      donated[donor] = 1;
    }
  }
  int64_t s = 0;
  for (auto& uv : g->edges) {  // already sorted
    if (stream_of[uv.first] != stream_of[uv.second]) {
      sync_uv[2 * s] = g->id(uv.first);
      sync_uv[2 * s + 1] = g->id(uv.second);
      ++s;
    }
  }
  *num_streams = next;
  *num_sync = s;
  return OPARA_OK;
}

opara_status opara_single_stream_plan(const opara_dag* g, int32_t* stream_of,
                                      int32_t* num_streams) {
  // allocator.py:70-77.
  if (!g || !num_streams || (g->n() && !stream_of)) return fail(OPARA_ERR_VALUE, "null argument");
  for (int32_t i = 0; i < g->n(); ++i) stream_of[i] = 0;
  *num_streams = g->n() ? 1 : 0;
  return OPARA_OK;
}

opara_status opara_validate_plan(const opara_dag* g, const int64_t* assigned_ids,
                                 const int64_t* streams, int64_t n_assigned, int64_t num_streams,
                                 const int64_t* sync_uv, int64_t n_sync, char* buf, int64_t buflen,
                                 int64_t* n_problems) {
  // allocator.py:80-109, same checks, same order, same wording.
  if (!g || !n_problems || (n_assigned && (!assigned_ids || !streams)) || (n_sync && !sync_uv))
    return fail(OPARA_ERR_VALUE, "null argument");
  std::vector<std::string> probs;
  std::unordered_map<int64_t, int64_t> assign;
  assign.reserve(static_cast<size_t>(n_assigned) * 2);
  for (int64_t k = 0; k < n_assigned; ++k) assign[assigned_ids[k]] = streams[k];
  for (int32_t i = 0; i < g->n(); ++i)
    if (!assign.count(g->id(i))) probs.push_back("node " + std::to_string(g->id(i)) + " unassigned");
  std::vector<int64_t> aids;
  aids.reserve(assign.size());
  for (auto& kv : assign) aids.push_back(kv.first);
  std::sort(aids.begin(), aids.end());
  for (int64_t v : aids)
    if (!g->index.count(v)) probs.push_back("assigned node " + std::to_string(v) + " not in graph");
  std::vector<int64_t> used;
  for (auto& kv : assign) used.push_back(kv.second);
  std::sort(used.begin(), used.end());
  used.erase(std::unique(used.begin(), used.end()), used.end());
  bool dense = static_cast<int64_t>(used.size()) == std::max<int64_t>(num_streams, 0);
  for (size_t k = 0; dense && k < used.size(); ++k) dense = used[k] == static_cast<int64_t>(k);
  if (!used.empty() && !dense)
    probs.push_back("stream ids must be dense 0.." + std::to_string(num_streams - 1) + ", got " +
                    opara::py_int_list(used));
  if (assign.empty() && num_streams != 0)
    probs.push_back("num_streams must be 0 for an empty assignment");
  std::vector<std::pair<int64_t, int64_t>> sync;
  for (int64_t k = 0; k < n_sync; ++k) sync.push_back({sync_uv[2 * k], sync_uv[2 * k + 1]});
  std::sort(sync.begin(), sync.end());
  sync.erase(std::unique(sync.begin(), sync.end()), sync.end());
  auto is_edge = [&](int64_t u, int64_t v) {
    auto iu = g->index.find(u), iv = g->index.find(v);
    if (iu == g->index.end() || iv == g->index.end()) return false;
    return std::binary_search(g->edges.begin(), g->edges.end(),
                              std::make_pair(iu->second, iv->second));
  };
  for (auto& uv : sync)
    if (!is_edge(uv.first, uv.second))
      probs.push_back("sync event " + opara::py_pair(uv.first, uv.second) + " is not a graph edge");
  for (auto& e : g->edges) {
    const int64_t u = g->id(e.first), v = g->id(e.second);
    auto au = assign.find(u), av = assign.find(v);
    if (au == assign.end() || av == assign.end()) continue;
    const bool crosses = au->second != av->second;
    const bool synced = std::binary_search(sync.begin(), sync.end(), std::make_pair(u, v));
    if (crosses && !synced)
      probs.push_back("missing sync for cross-stream edge " + opara::py_pair(u, v));
    if (!crosses && synced)
      probs.push_back("sync event " + opara::py_pair(u, v) + " joins same-stream nodes");
  }
  std::string joined;
  for (size_t k = 0; k < probs.size(); ++k) {
    if (k) joined += '\n';
    joined += probs[k];
  }
  *n_problems = static_cast<int64_t>(probs.size());
  if (buf && buflen > 0) {
    if (static_cast<int64_t>(joined.size()) + 1 > buflen)
      return fail(OPARA_ERR_CAPACITY, "validate_plan message buffer too small (need " +
                                          std::to_string(joined.size() + 1) + ")");
    std::memcpy(buf, joined.c_str(), joined.size() + 1);
  }
  return OPARA_OK;
}

opara_status opara_dominant_share(const opara_node* node, const opara_gpu_config* cfg, double* out) {
  if (!node || !out) return fail(OPARA_ERR_VALUE, "null argument");
  opara_status st = check_cfg(cfg);
  if (st != OPARA_OK) return st;
  *out = share_of(*node, *cfg);
  return OPARA_OK;
}

opara_status opara_order(const opara_dag* g, int32_t policy, const opara_gpu_config* cfg,
                         int64_t* out) {
  if (!g || (!out && g->n())) return fail(OPARA_ERR_VALUE, "null argument");
  std::vector<int32_t> order;
  switch (policy) {
    case OPARA_POLICY_OPARA: {
      opara_status st = check_cfg(cfg);
      if (st != OPARA_OK) return st;
      order = order_opara(*g, *cfg);
      break;
    }
    case OPARA_POLICY_SEQUENTIAL: order = g->topo; break;
    case OPARA_POLICY_DFS: order = order_dfs(*g); break;
    case OPARA_POLICY_WAVEFRONT: order = order_wavefront(*g); break;
    default: return fail(OPARA_ERR_VALUE, "unknown policy " + std::to_string(policy));
  }
  for (size_t k = 0; k < order.size(); ++k) out[k] = g->id(order[k]);
  return OPARA_OK;
}

// Depth-first walk over ready sets kept sorted ascending, so extensions come
// out in lexicographic id order (oracle.py:52-84 enumerates the same way).
opara_status opara_linear_extensions(const opara_dag* g, int64_t skip, int64_t cap, int64_t* out,
                                     int64_t* written, int32_t* exhausted) {
  if (!g || !written || !exhausted || (cap > 0 && !out) || skip < 0 || cap < 0)
    return fail(OPARA_ERR_VALUE, "null argument");
  const int32_t n = g->n();
  std::vector<int32_t> indeg(n);
  for (int32_t v = 0; v < n; ++v) indeg[v] = g->pred_off[v + 1] - g->pred_off[v];
  std::vector<int32_t> prefix;
  prefix.reserve(n);
  std::vector<char> used(n, 0);
  int64_t seen = 0, nw = 0;
  bool stop = false;
  // ready set = {v : !used[v] && indeg[v] == 0}; scanning v ascending is the
  // lexicographic branch order (n is tiny: the space is up to n!)
  auto walk = [&](auto&& self) -> void {
    if (static_cast<int32_t>(prefix.size()) == n) {
      if (seen++ >= skip) {
        if (nw == cap) {
          stop = true;
          return;
        }
        for (int32_t k = 0; k < n; ++k) out[nw * n + k] = g->id(prefix[k]);
        ++nw;
      }
      return;
    }
    for (int32_t v = 0; v < n && !stop; ++v) {
      if (used[v] || indeg[v]) continue;
      used[v] = 1;
      prefix.push_back(v);
      for (int32_t e = g->succ_off[v]; e < g->succ_off[v + 1]; ++e) --indeg[g->succ[e]];
      self(self);
      for (int32_t e = g->succ_off[v]; e < g->succ_off[v + 1]; ++e) ++indeg[g->succ[e]];
      prefix.pop_back();
      used[v] = 0;
    }
  };
  if (cap > 0 || n == 0) walk(walk);
  else stop = true;
  *written = nw;
  *exhausted = stop ? 0 : 1;
  return OPARA_OK;
}

}  // extern "C"
