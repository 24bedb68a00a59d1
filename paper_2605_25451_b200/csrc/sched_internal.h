// sched_internal.h -- the library-owned schedule object (opaque in bigmac.h).
#pragma once

#include <map>
#include <tuple>
#include <vector>

#include "../../include/bigmac.h"

struct bm_schedule {
  bm_sched_cfg cfg;
  std::vector<std::vector<bm_op>> ranks;
  std::vector<bm_sched_stats> stats;
  std::map<std::tuple<int, int, int>, std::pair<int, int>> rings;  // (src,dst,payload) -> (K, nmsg)
};

namespace bm {
namespace sched {
// rank that runs microbatch m's encoder (bm_sched_cfg.enc_exclude; R3, R22)
int enc_owner(const bm_sched_cfg& c, int m);
}  // namespace sched
}  // namespace bm
