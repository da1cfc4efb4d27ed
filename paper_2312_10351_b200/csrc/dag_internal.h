// The DAG behind the opaque opara_dag handle, shared by the scheduler
// (sched.cpp) and the execution model (simulate.cpp).
#pragma once

#include <cstdint>
#include <unordered_map>
#include <utility>
#include <vector>

#include "opara.h"

struct opara_dag {
  std::vector<opara_node> nodes;                 // ascending id
  std::unordered_map<int64_t, int32_t> index;    // id -> dense index
  std::vector<int32_t> pred_off, pred;           // CSR, ascending index
  std::vector<int32_t> succ_off, succ;
  std::vector<std::pair<int32_t, int32_t>> edges;  // sorted, unique
  std::vector<int32_t> topo;                     // dense indices

  int32_t n() const { return static_cast<int32_t>(nodes.size()); }
  int64_t id(int32_t i) const { return nodes[i].id; }
};
