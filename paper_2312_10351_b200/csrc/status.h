// Internal error plumbing shared by the scheduler and the executor.
#pragma once

#include <string>
#include <vector>

#include "opara.h"

namespace opara {

extern thread_local std::string g_last_error;

// Record `msg` as this thread's last error and return `st`.
opara_status fail(opara_status st, const std::string& msg);

// Python repr of an int list / pair, for messages identical to the reference.
std::string py_int_list(const std::vector<int64_t>& v);
std::string py_pair(int64_t u, int64_t v);

}  // namespace opara
