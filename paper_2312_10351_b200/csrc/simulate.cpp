// Execution model of the reference (`simulate`, simulator.py:212-415) in C++,
// bit-exact: the discrete-event multi-SM model the reference uses in place of
// a GPU.  On the B200 the real multi-stream CUDA Graph replaces it for
// execution; this port predicts a (plan, order) pair's makespan on a GpuConfig
// without a device, at native speed.
//
// Semantics kept exactly (simulator.py:1-26):
//   * every plan stream is a FIFO in launch order; a kernel is eligible once it
//     heads its stream and all its sync producers completed;
//   * eligible kernels queue in eligibility order: launch order at t = 0,
//     later simultaneous arrivals by stream id (sorted(newly, key=stream));
//   * head-of-line dispatch: the queue head places blocks one at a time on the
//     lowest-index SM with enough free threads, smem, registers and a slot;
//   * a block placed on an SM that holds a live block of the same class from a
//     different operator runs round(duration * slowdown) ns (Python round():
//     ties to even == std::nearbyint in the default rounding mode), decided
//     after the whole dispatch round so same-instant blocks see each other;
//   * completions pop in (end, placement token) order; integer nanoseconds.
// Compiled with -ffp-contract=off: base * slowdown is one IEEE multiply.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <queue>
#include <string>
#include <tuple>
#include <vector>

#include "dag_internal.h"
#include "opara.h"
#include "status.h"

using opara::fail;

namespace {

struct Event {
  int64_t end;
  int64_t token;
  int32_t op;  // dense index
  int32_t sm;
  bool operator>(const Event& o) const { return std::tie(end, token) > std::tie(o.end, o.token); }
};

struct LiveBlock {
  int64_t token;
  int32_t op;
};

}  // namespace

extern "C" {

opara_status opara_simulate(const opara_dag* g, const int64_t* block_duration_ns, const int32_t* stream_of,
                            int32_t num_streams, const int64_t* order, const int64_t* sync_uv, int64_t n_sync,
                            const opara_gpu_config* cfg, opara_sim_result* out, int64_t* op_start_ns,
                            int64_t* op_end_ns, int64_t* sm_busy_ns, int64_t* block_log, int64_t block_log_cap,
                            int64_t* n_blocks) {
  opara::g_last_error.clear();
  if (!g || !cfg || !out || (g->n() && (!block_duration_ns || !stream_of || !order)) || (n_sync && !sync_uv))
    return fail(OPARA_ERR_VALUE, "opara_simulate: null argument");
  if (cfg->num_sms < 1 || cfg->threads_per_sm < 1 || cfg->shared_mem_per_sm < 1 || cfg->registers_per_sm < 1 ||
      cfg->max_blocks_per_sm < 1)
    return fail(OPARA_ERR_VALUE, "GpuConfig capacities must be >= 1");
  if (cfg->same_class_slowdown < 1.0) return fail(OPARA_ERR_VALUE, "same_class_slowdown must be >= 1.0");
  const int32_t n = g->n();
  const int64_t S = cfg->num_sms;
  *out = opara_sim_result{0, 0, 0, 0.0};
  if (n_blocks) *n_blocks = 0;
  if (sm_busy_ns)
    for (int64_t i = 0; i < S; ++i) sm_busy_ns[i] = 0;
  if (n == 0) return OPARA_OK;

  // ---- inputs in dense-index space (validated by the host like _check_inputs)
  std::vector<int32_t> ord(n);
  std::vector<char> seen(n, 0);
  for (int32_t k = 0; k < n; ++k) {
    auto it = g->index.find(order[k]);
    if (it == g->index.end() || seen[it->second])
      return fail(OPARA_ERR_COVERAGE, "launch order must cover the graph exactly");
    seen[it->second] = 1;
    ord[k] = it->second;
  }
  std::vector<int64_t> dur(block_duration_ns, block_duration_ns + n);
  std::vector<int64_t> regs(n);
  for (int32_t i = 0; i < n; ++i) {
    const opara_node& d = g->nodes[i];
    regs[i] = d.registers_per_thread * d.threads_per_block;
    if (d.threads_per_block > cfg->threads_per_sm || d.shared_mem_per_block > cfg->shared_mem_per_sm ||
        regs[i] > cfg->registers_per_sm)
      return fail(OPARA_ERR_INFEASIBLE_BLOCK, "operator " + std::to_string(d.id) +
                                                  ": one block exceeds a single SM's capacity");
    if (stream_of[i] < 0 || stream_of[i] >= num_streams)
      return fail(OPARA_ERR_PLAN_VIOLATION, "stream id outside 0..num_streams-1");
  }
  std::vector<std::vector<int32_t>> stream_seq(num_streams);
  for (int32_t v : ord) stream_seq[stream_of[v]].push_back(v);
  std::vector<size_t> head_idx(num_streams, 0);
  std::vector<int32_t> pending(n, 0);
  std::vector<std::vector<int32_t>> consumers(n);
  for (int64_t k = 0; k < n_sync; ++k) {
    auto iu = g->index.find(sync_uv[2 * k]), iv = g->index.find(sync_uv[2 * k + 1]);
    if (iu == g->index.end() || iv == g->index.end())
      return fail(OPARA_ERR_PLAN_VIOLATION, "sync event references an unknown node");
    pending[iv->second] += 1;
    consumers[iu->second].push_back(iv->second);
  }

  // ---- state (simulator.py:242-266)
  const int64_t kUnset = -1;
  std::vector<int64_t> unplaced(n), running(n, 0), head_time(n, kUnset), eligible_time(n, kUnset),
      first_place(n, kUnset), op_end(n, kUnset), placed_index(n, 0);
  for (int32_t i = 0; i < n; ++i) unplaced[i] = g->nodes[i].num_blocks;
  std::vector<int64_t> free_thr(S, cfg->threads_per_sm), free_smem(S, cfg->shared_mem_per_sm),
      free_regs(S, cfg->registers_per_sm), free_slots(S, cfg->max_blocks_per_sm);
  std::vector<std::vector<LiveBlock>> live(S);
  std::vector<int64_t> busy(S, 0), busy_last(S, 0), busy_count(S, 0);
  std::priority_queue<std::pair<int64_t, int32_t>, std::vector<std::pair<int64_t, int32_t>>,
                      std::greater<std::pair<int64_t, int32_t>>>
      ee;  // (eligibility sequence, op)
  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> events;
  int64_t seq = 0, token = 0, completed = 0, logged = 0;
  const double slow = cfg->same_class_slowdown;

  auto touch = [&](int64_t sm, int64_t t) {
    if (busy_count[sm] > 0) busy[sm] += t - busy_last[sm];
    busy_last[sm] = t;
  };
  auto find_sm = [&](int32_t v) -> int64_t {
    const opara_node& d = g->nodes[v];
    for (int64_t i = 0; i < S; ++i)
      if (free_thr[i] >= d.threads_per_block && free_smem[i] >= d.shared_mem_per_block && free_regs[i] >= regs[v] &&
          free_slots[i] >= 1)
        return i;
    return -1;
  };
  auto make_eligible = [&](int32_t v, int64_t t) {
    eligible_time[v] = t;
    ee.push({seq++, v});
  };
  std::vector<std::tuple<int64_t, int32_t, int64_t>> round;  // (token, op, sm)
  auto dispatch = [&](int64_t t) {
    round.clear();
    while (!ee.empty()) {
      const int32_t v = ee.top().second;
      const opara_node& d = g->nodes[v];
      bool stuck = false;
      while (unplaced[v] > 0) {
        const int64_t sm = find_sm(v);
        if (sm < 0) {
          stuck = true;
          break;
        }
        free_thr[sm] -= d.threads_per_block;
        free_smem[sm] -= d.shared_mem_per_block;
        free_regs[sm] -= regs[v];
        free_slots[sm] -= 1;
        touch(sm, t);
        busy_count[sm] += 1;
        live[sm].push_back({token, v});
        round.emplace_back(token, v, sm);
        ++token;
        unplaced[v] -= 1;
        running[v] += 1;
        if (first_place[v] == kUnset) first_place[v] = t;
      }
      if (stuck) break;
      ee.pop();
    }
    // durations after the whole round: same-instant blocks see each other
    for (auto& [tok, v, sm] : round) {
      const int32_t cls = g->nodes[v].op_class;
      bool slowed = false;
      for (const LiveBlock& b : live[sm])
        if (b.token != tok && b.op != v && g->nodes[b.op].op_class == cls) {
          slowed = true;
          break;
        }
      const int64_t base = dur[v];
      const int64_t length = slowed ? static_cast<int64_t>(std::nearbyint(static_cast<double>(base) * slow)) : base;
      const int64_t end = t + length;
      const int64_t idx = placed_index[v]++;
      if (block_log && logged < block_log_cap) {
        int64_t* row = block_log + 5 * logged;
        row[0] = g->nodes[v].id;
        row[1] = idx;
        row[2] = sm;
        row[3] = t;
        row[4] = end;
      }
      ++logged;
      events.push({end, tok, v, static_cast<int32_t>(sm)});
    }
  };

  // time zero: stream heads in launch order (simulator.py:341-349)
  std::vector<char> at_head(n, 0);
  for (int32_t s = 0; s < num_streams; ++s)
    if (!stream_seq[s].empty()) {
      at_head[stream_seq[s][0]] = 1;
      head_time[stream_seq[s][0]] = 0;
    }
  for (int32_t v : ord)
    if (at_head[v] && pending[v] == 0) make_eligible(v, 0);
  dispatch(0);

  std::vector<int32_t> finished, newly;
  while (!events.empty()) {
    const int64_t t = events.top().end;
    finished.clear();
    while (!events.empty() && events.top().end == t) {
      const Event e = events.top();
      events.pop();
      const opara_node& d = g->nodes[e.op];
      touch(e.sm, t);
      busy_count[e.sm] -= 1;
      free_thr[e.sm] += d.threads_per_block;
      free_smem[e.sm] += d.shared_mem_per_block;
      free_regs[e.sm] += regs[e.op];
      free_slots[e.sm] += 1;
      auto& lv = live[e.sm];
      for (size_t k = 0; k < lv.size(); ++k)
        if (lv[k].token == e.token) {
          lv.erase(lv.begin() + static_cast<long>(k));
          break;
        }
      running[e.op] -= 1;
      if (running[e.op] == 0 && unplaced[e.op] == 0 && op_end[e.op] == kUnset) {
        op_end[e.op] = t;
        ++completed;
        finished.push_back(e.op);
      }
    }
    newly.clear();
    for (int32_t v : finished) {
      const int32_t s = stream_of[v];
      head_idx[s] += 1;
      if (head_idx[s] < stream_seq[s].size()) {
        const int32_t w = stream_seq[s][head_idx[s]];
        head_time[w] = t;
        if (pending[w] == 0) newly.push_back(w);
      }
      for (int32_t c : consumers[v]) {
        pending[c] -= 1;
        if (pending[c] == 0 && head_time[c] != kUnset && eligible_time[c] == kUnset) newly.push_back(c);
      }
    }
    std::stable_sort(newly.begin(), newly.end(), [&](int32_t a, int32_t b) { return stream_of[a] < stream_of[b]; });
    for (int32_t v : newly) make_eligible(v, t);
    dispatch(t);
  }
  if (completed != n) return fail(OPARA_ERR_INTERNAL, "simulation ended with unfinished operators");

  int64_t makespan = 0, blocked = 0, sync_wait = 0, busy_sum = 0;
  for (int32_t i = 0; i < n; ++i) {
    makespan = std::max(makespan, op_end[i]);
    blocked += first_place[i] - eligible_time[i];
    sync_wait += eligible_time[i] - head_time[i];
    if (op_start_ns) op_start_ns[i] = first_place[i];
    if (op_end_ns) op_end_ns[i] = op_end[i];
  }
  for (int64_t i = 0; i < S; ++i) {
    busy_sum += busy[i];
    if (sm_busy_ns) sm_busy_ns[i] = busy[i];
  }
  out->makespan_ns = makespan;
  out->blocked_ns = blocked;
  out->sync_wait_ns = sync_wait;
  out->sm_efficiency = makespan ? static_cast<double>(busy_sum) / static_cast<double>(S * makespan) : 0.0;
  if (n_blocks) *n_blocks = logged;
  if (block_log && logged > block_log_cap)
    return fail(OPARA_ERR_CAPACITY, "block log capacity " + std::to_string(block_log_cap) + " < " +
                                        std::to_string(logged) + " placed blocks");
  return OPARA_OK;
}

}  // extern "C"
