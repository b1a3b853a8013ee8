// colosim/reclaim.hpp -- drop-in for /root/reference/proj/include/colosim/reclaim.hpp:12-37.
// Same types and free functions; the selection runs on the GPU (valve_select /
// valve_evicted_cost, sm_100a) over the instance uploaded as CSR.
#pragma once
#include <cstdint>
#include <map>
#include <vector>

#include "colosim/time.hpp"
#include "colosim/valve_detail.hpp"

namespace colosim {

struct ReclaimHandle {
  int id = 0;
  SimTime mapped_at = 0;              // allocation timestamp (FIFO order)
  std::vector<std::int64_t> requests;  // offline requests with >= 1 page on this handle
};

struct ReclaimInstance {
  std::vector<ReclaimHandle> handles;
  std::map<std::int64_t, std::int64_t> cost;  // request id -> recompute cost (tokens)
};

namespace valve_detail {
struct Csr {
  std::vector<int> ids, off;
  std::vector<std::int64_t> mapped, reqs, keys, vals;
  explicit Csr(const ReclaimInstance& inst) {
    off.push_back(0);
    for (const ReclaimHandle& h : inst.handles) {
      ids.push_back(h.id);
      mapped.push_back(h.mapped_at);
      reqs.insert(reqs.end(), h.requests.begin(), h.requests.end());
      off.push_back(static_cast<int>(reqs.size()));
    }
    for (const auto& [k, v] : inst.cost) {
      keys.push_back(k);
      vals.push_back(v);
    }
  }
  int n() const { return static_cast<int>(ids.size()); }
  int m() const { return static_cast<int>(keys.size()); }
};

inline std::vector<int> select(const ReclaimInstance& inst, int k, int mode) {
  Csr c(inst);
  std::vector<int> out(static_cast<std::size_t>(c.n()) + 1);
  int n_out = 0;
  check(valve_select(device(), c.n(), c.ids.data(), c.mapped.data(), c.off.data(), c.reqs.data(), c.m(),
                     c.keys.data(), c.vals.data(), k, mode, out.data(), &n_out));
  out.resize(static_cast<std::size_t>(n_out));
  return out;
}
}  // namespace valve_detail

// Union cost of a handle subset (reclaim.hpp:28-30).
inline std::int64_t evicted_cost(const ReclaimInstance& inst, const std::vector<int>& handle_ids) {
  valve_detail::Csr c(inst);
  std::int64_t cost = 0;
  valve_detail::check(valve_evicted_cost(device(), c.n(), c.ids.data(), c.off.data(), c.reqs.data(), c.m(),
                                         c.keys.data(), c.vals.data(), handle_ids.data(),
                                         static_cast<int>(handle_ids.size()), &cost));
  return cost;
}

// Algorithm 1 (reclaim.hpp:32-35).
inline std::vector<int> selective_reclaim(const ReclaimInstance& inst, int k) {
  return valve_detail::select(inst, k, VALVE_SELECT_SELECTIVE);
}
// Oldest first (reclaim.hpp:37-38).
inline std::vector<int> fifo_reclaim(const ReclaimInstance& inst, int k) {
  return valve_detail::select(inst, k, VALVE_SELECT_FIFO);
}
// Exhaustive minimum, <= 20 handles (reclaim.hpp:40-42).
inline std::vector<int> oracle_reclaim(const ReclaimInstance& inst, int k) {
  return valve_detail::select(inst, k, VALVE_SELECT_ORACLE);
}

}  // namespace colosim
