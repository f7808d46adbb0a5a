// Internal plan / comm structures shared by planner.cpp and comm.cu.
// Not part of the ABI (include/themis.h is).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "themis.h"

namespace themis {

using u128 = unsigned __int128;

// Per-thread last-error message (themis_last_error).
void set_error(const std::string& msg);
themis_status_t fail(themis_status_t st, const std::string& msg);

struct Op {           // one (chunk, stage) of the plan
  int chunk, stage, dim;
  int phase;          // 0 = RS, 1 = AG
  uint32_t reduced_before;  // bitmask of dims reduce-scattered before this op
  u128 bytes_before;  // x byte_scale
  u128 volume;        // n_K^i x byte_scale
  u128 duration;      // time units
};

struct BindState;     // comm.cu

}  // namespace themis

struct themis_plan {
  themis_topology_t topo;
  themis_plan_req_t req;
  int D = 0, C = 0, P = 0, NS = 0;      // NS = stages per chunk
  int n_greedy = 0;
  std::vector<uint8_t> rs, ag;          // [C][D], 0xFF when absent
  std::vector<themis::Op> ops;          // [C][NS]
  std::vector<std::vector<uint32_t>> dim_ops;  // per dim: (chunk << 8) | stage
  std::vector<themis::u128> start, end; // [C][NS]
  std::vector<int32_t> server;          // [C][NS] pre-simulated server of each op
  std::vector<themis::u128> busy, idle, vol, load;
  themis::u128 makespan = 0, time_scale = 0, byte_scale = 0;
  uint64_t hash = 0;
  themis::BindState* bind = nullptr;    // set by themis_plan_bind
};
