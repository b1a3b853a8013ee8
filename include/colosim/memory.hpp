// colosim/memory.hpp -- drop-in for /root/reference/proj/include/colosim/memory.hpp:19-146.
//
// MemoryPool keeps the reference's public API and value results, but its state lives in HBM
// and every mutating call is one sm_100a kernel launch through the C ABI (valve_pool_*).
// The counters (free/online/offline handles) are read from the pinned mirror each kernel
// publishes, so the reference's inline getters stay host-cheap.  ReservationController is the
// host fp64 control plane (valve_resctl_*), as the north star keeps it.
#pragma once
#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <utility>
#include <vector>

#include "colosim/reclaim.hpp"
#include "colosim/time.hpp"
#include "colosim/valve_detail.hpp"

namespace colosim {

class MemoryPool {
 public:
  enum class HandleState : std::uint8_t { kFree, kOnlineReserved, kOfflineMapped };

  MemoryPool(int total_handles, int handle_size_pages, int page_size_tokens)
      : total_(total_handles), hsz_(handle_size_pages), tok_(page_size_tokens) {
    valve_pool_config cfg;
    valve_pool_config_default(&cfg);
    cfg.device = device();
    cfg.total_handles = total_handles;
    cfg.handle_size_pages = handle_size_pages;
    cfg.page_size_tokens = page_size_tokens;
    if (total_handles > 0 && handle_size_pages > 0) {
      const std::int64_t pages = static_cast<std::int64_t>(total_handles) * handle_size_pages;
      cfg.max_pages_per_request = static_cast<int>(pages < 4096 ? pages : 4096);
    }
    valve_pool* p = nullptr;
    valve_detail::check(valve_pool_create_ex(&cfg, &p));
    pool_.reset(p);
  }

  // B200 addition: a pool with a page store / table sizes from a full device config
  explicit MemoryPool(const valve_pool_config& cfg)
      : total_(cfg.total_handles), hsz_(cfg.handle_size_pages), tok_(cfg.page_size_tokens) {
    valve_pool* p = nullptr;
    valve_detail::check(valve_pool_create_ex(&cfg, &p));
    pool_.reset(p);
  }

  int total_handles() const { return total_; }
  int handle_size_pages() const { return hsz_; }
  int page_size_tokens() const { return tok_; }
  int free_handles() const { return static_cast<int>(counts()[0]); }
  int online_handles() const { return static_cast<int>(counts()[1]); }
  int offline_handles() const { return static_cast<int>(counts()[2]); }

  std::int64_t quarantine_page_id() const { return static_cast<std::int64_t>(total_) * hsz_; }

  std::int64_t online_used_pages() const { return counts()[3]; }
  std::int64_t online_capacity_pages() const { return counts()[4]; }
  void online_grow(int k, SimTime t) { valve_detail::check(valve_pool_online_grow(pool_.get(), k, t)); }
  int online_release(int k) {
    int r = 0;
    valve_detail::check(valve_pool_online_release(pool_.get(), k, &r));
    return r;
  }
  void online_use_pages(std::int64_t n) { valve_detail::check(valve_pool_online_use_pages(pool_.get(), n)); }
  void online_free_pages(std::int64_t n) { valve_detail::check(valve_pool_online_free_pages(pool_.get(), n)); }

  bool offline_reserve(std::int64_t req, int pages, SimTime t, int max_offline_handles = -1) {
    int ok = 0;
    valve_detail::check(valve_pool_offline_reserve(pool_.get(), req, pages, t, max_offline_handles, &ok));
    return ok != 0;
  }
  void offline_release(std::int64_t req) { valve_detail::check(valve_pool_offline_release(pool_.get(), req)); }
  std::vector<std::int64_t> requests_on_handle(int handle) const {
    std::vector<std::int64_t> out(static_cast<std::size_t>(hsz_));
    int n = 0;
    valve_detail::check(valve_pool_requests_on_handle(pool_.get(), handle, out.data(), hsz_, &n));
    out.resize(static_cast<std::size_t>(n));
    return out;
  }
  std::vector<int> handles_of_request(std::int64_t req) const {
    std::vector<int> out(static_cast<std::size_t>(total_));
    int n = 0;
    valve_detail::check(valve_pool_handles_of_request(pool_.get(), req, out.data(), total_, &n));
    out.resize(static_cast<std::size_t>(n));
    return out;
  }
  int offline_pages_of(std::int64_t req) const {
    int n = 0;
    valve_detail::check(valve_pool_offline_pages_of(pool_.get(), req, &n));
    return n;
  }

  ReclaimInstance snapshot() const {
    int nh = 0, nr = 0;
    const int *ids = nullptr, *off = nullptr;
    const std::int64_t *mapped = nullptr, *reqs = nullptr;
    valve_detail::check(valve_pool_snapshot_view(pool_.get(), &ids, &mapped, &off, &reqs, &nh, &nr));
    ReclaimInstance inst;
    inst.handles.resize(static_cast<std::size_t>(nh));
    for (int i = 0; i < nh; ++i) {
      ReclaimHandle& h = inst.handles[static_cast<std::size_t>(i)];
      h.id = ids[i];
      h.mapped_at = mapped[i];
      h.requests.assign(reqs + off[i], reqs + off[i + 1]);
    }
    return inst;
  }

  struct ReclaimResult {
    std::vector<int> handles;
    std::vector<std::int64_t> evicted_requests;
    std::map<std::int64_t, std::vector<std::int64_t>> invalidated_pages;
  };
  ReclaimResult apply_reclaim(const std::vector<int>& handle_ids, SimTime t) {
    int nh = 0, ne = 0, np = 0;
    const int *handles = nullptr, *off = nullptr;
    const std::int64_t *ev = nullptr, *pages = nullptr;
    valve_detail::check(valve_pool_apply_reclaim_view(pool_.get(), handle_ids.data(),
                                                      static_cast<int>(handle_ids.size()), t, &handles, &nh, &ev,
                                                      &ne, &off, &pages, &np));
    ReclaimResult r;
    r.handles.assign(handles, handles + nh);
    r.evicted_requests.assign(ev, ev + ne);
    for (int i = 0; i < ne; ++i) r.invalidated_pages[ev[i]].assign(pages + off[i], pages + off[i + 1]);
    return r;
  }

  HandleState handle_state(int handle) const {
    int s = 0;
    valve_detail::check(valve_pool_handle_state(pool_.get(), handle, &s));
    return static_cast<HandleState>(s);
  }
  SimTime handle_mapped_at(int handle) const {
    std::int64_t t = 0;
    valve_detail::check(valve_pool_handle_mapped_at(pool_.get(), handle, &t));
    return t;
  }
  void check_invariants() const { valve_detail::check(valve_pool_check_invariants(pool_.get())); }

  // B200 additions
  valve_pool* native() const { return pool_.get(); }

 private:
  struct Del {
    void operator()(valve_pool* p) const { valve_pool_destroy(p); }
  };
  std::array<std::int64_t, 5> counts() const {
    std::array<std::int64_t, 5> c{};
    valve_pool_counts(pool_.get(), c.data());
    return c;
  }
  int total_, hsz_, tok_;
  std::unique_ptr<valve_pool, Del> pool_;
};

struct ReservationParams {
  double alpha = 1.5;
  double beta = 2.0;
  SimTime t_init_us = 1 * us_per_s;
  SimTime delta_us = 100 * us_per_ms;
  SimTime t_min_us = 100 * us_per_ms;
  SimTime t_max_us = 60 * us_per_s;
  SimTime window_us = 60 * us_per_s;
  double target_per_window = 1.0;
  int h_min = 1;
  double pressure_threshold = 0.9;
};

class ReservationController {
 public:
  explicit ReservationController(ReservationParams p) : params_(p) {
    valve_resparams c{p.alpha,     p.beta,      p.t_init_us,          p.delta_us, p.t_min_us,
                      p.t_max_us,  p.window_us, p.target_per_window, p.h_min,    p.pressure_threshold};
    valve_resctl* h = nullptr;
    valve_detail::check(valve_resctl_create(&c, &h));
    ctl_.reset(h);
  }
  SimTime interval() const { return valve_resctl_interval(ctl_.get()); }
  const ReservationParams& params() const { return params_; }
  std::int64_t pressure_events() const { return valve_resctl_pressure_events(ctl_.get()); }
  int grow_target(int h, int cap) const { return valve_resctl_grow_target(ctl_.get(), h, cap); }
  void record_pressure(SimTime t) { valve_resctl_record_pressure(ctl_.get(), t); }
  bool release_due(SimTime t, int h) const { return valve_resctl_release_due(ctl_.get(), t, h) != 0; }
  void note_tick(SimTime t) { valve_resctl_note_tick(ctl_.get(), t); }
  SimTime window_tick(SimTime t) { return valve_resctl_window_tick(ctl_.get(), t); }
  std::int64_t pressure_in_window(SimTime t) const { return valve_resctl_pressure_in_window(ctl_.get(), t); }

 private:
  struct Del {
    void operator()(valve_resctl* c) const { valve_resctl_destroy(c); }
  };
  ReservationParams params_;
  std::unique_ptr<valve_resctl, Del> ctl_;
};

}  // namespace colosim
