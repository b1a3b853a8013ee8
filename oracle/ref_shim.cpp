// ref_shim.cpp -- exports the oracle's C API (valve_oracle.h) on top of the REFERENCE
// implementation compiled from /root/reference/proj/src/{memory,reclaim,channel}.cpp.
//
// TEST INFRASTRUCTURE ONLY (see valve_oracle.h).  Built by oracle/Makefile into
// oracle/_ref/libcolosim_ref.so (git-ignored); the reference sources are compiled in place
// and never copied.  Quantities the reference does not model (physical slots, block
// indices, byte images) are reported as -1 / unsupported.
#include <algorithm>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "colosim/channel.hpp"
#include "colosim/memory.hpp"
#include "colosim/reclaim.hpp"
#include "valve_oracle.h"

using namespace colosim;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return VO_OK;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return VO_OUT_OF_RANGE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return VO_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return VO_LOGIC_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VO_RUNTIME_ERROR;
  }
}

ReclaimInstance make_inst(int n, const int* ids, const int64_t* mapped, const int* off,
                          const int64_t* reqs, int m, const int64_t* keys, const int64_t* vals) {
  ReclaimInstance inst;
  for (int i = 0; i < n; ++i) {
    ReclaimHandle h;
    h.id = ids[i];
    h.mapped_at = mapped ? mapped[i] : 0;
    h.requests.assign(reqs + off[i], reqs + off[i + 1]);
    inst.handles.push_back(std::move(h));
  }
  for (int i = 0; i < m; ++i) inst.cost[keys[i]] = vals[i];
  return inst;
}
}  // namespace

struct vo_pool {
  MemoryPool pool;
};
struct vo_resctl {
  ReservationController ctl;
};
struct vo_channel {
  std::unique_ptr<ChannelController> ctl;
};

extern "C" {

const char* vo_last_error(void) { return g_err.c_str(); }

int vo_pool_create(int H, int S, int T, vo_pool** out) {
  return guard([&] { *out = new vo_pool{MemoryPool(H, S, T)}; });
}
void vo_pool_destroy(vo_pool* p) { delete p; }
int vo_pool_counts(const vo_pool* p, int64_t out[5]) {
  out[0] = p->pool.free_handles();
  out[1] = p->pool.online_handles();
  out[2] = p->pool.offline_handles();
  out[3] = p->pool.online_used_pages();
  out[4] = p->pool.online_capacity_pages();
  return VO_OK;
}
int vo_pool_online_grow(vo_pool* p, int k, int64_t t) {
  return guard([&] { p->pool.online_grow(k, t); });
}
int vo_pool_online_release(vo_pool* p, int k, int* released) {
  return guard([&] { *released = p->pool.online_release(k); });
}
int vo_pool_online_use_pages(vo_pool* p, int64_t n) {
  return guard([&] { p->pool.online_use_pages(n); });
}
int vo_pool_online_free_pages(vo_pool* p, int64_t n) {
  return guard([&] { p->pool.online_free_pages(n); });
}
int vo_pool_offline_reserve(vo_pool* p, int64_t req, int pages, int64_t t, int max_off, int* ok) {
  return guard([&] { *ok = p->pool.offline_reserve(req, pages, t, max_off) ? 1 : 0; });
}
int vo_pool_offline_release(vo_pool* p, int64_t req) {
  return guard([&] { p->pool.offline_release(req); });
}
int vo_pool_requests_on_handle(const vo_pool* p, int h, int64_t* out, int cap, int* n) {
  return guard([&] {
    auto v = p->pool.requests_on_handle(h);
    *n = static_cast<int>(v.size());
    for (int i = 0; i < *n && i < cap; ++i) out[i] = v[i];
  });
}
int vo_pool_handles_of_request(const vo_pool* p, int64_t req, int* out, int cap, int* n) {
  return guard([&] {
    auto v = p->pool.handles_of_request(req);
    *n = static_cast<int>(v.size());
    for (int i = 0; i < *n && i < cap; ++i) out[i] = v[i];
  });
}
int vo_pool_offline_pages_of(const vo_pool* p, int64_t req, int* out) {
  return guard([&] { *out = p->pool.offline_pages_of(req); });
}
int vo_pool_snapshot(const vo_pool* p, int* ids, int64_t* mapped, int* off, int64_t* reqs, int cap_h,
                     int cap_r, int* nh, int* nr) {
  return guard([&] {
    ReclaimInstance inst = p->pool.snapshot();
    int h_n = 0, r_n = 0;
    if (off && cap_h >= 0) off[0] = 0;
    for (const ReclaimHandle& h : inst.handles) {
      if (ids && h_n < cap_h) {
        ids[h_n] = h.id;
        mapped[h_n] = h.mapped_at;
      }
      for (int64_t r : h.requests) {
        if (reqs && r_n < cap_r) reqs[r_n] = r;
        ++r_n;
      }
      ++h_n;
      if (off && h_n <= cap_h) off[h_n] = r_n;
    }
    *nh = h_n;
    *nr = r_n;
  });
}
int vo_pool_apply_reclaim(vo_pool* p, const int* ids, int k, int64_t t, int* handles, int* n_handles,
                          int64_t* evicted, int* n_evicted, int* inv_off, int64_t* inv_pages,
                          int* inv_phys, int* inv_blk, int cap_ev, int cap_pages, int* n_pages) {
  return guard([&] {
    MemoryPool::ReclaimResult r = p->pool.apply_reclaim(std::vector<int>(ids, ids + k), t);
    *n_handles = static_cast<int>(r.handles.size());
    for (int i = 0; i < *n_handles; ++i)
      if (handles) handles[i] = r.handles[i];
    if (static_cast<int>(r.evicted_requests.size()) > cap_ev)
      throw std::runtime_error("apply_reclaim: evicted capacity too small");
    int ne = 0, np = 0;
    for (int64_t req : r.evicted_requests) {
      evicted[ne] = req;
      inv_off[ne] = np;
      ++ne;
      for (int64_t pg : r.invalidated_pages.at(req)) {
        if (np < cap_pages) {
          inv_pages[np] = pg;
          inv_phys[np] = -1;
          inv_blk[np] = -1;
        }
        ++np;
      }
    }
    inv_off[ne] = np;
    *n_evicted = ne;
    *n_pages = np;
  });
}
int vo_pool_handle_state(const vo_pool* p, int h, int* st) {
  return guard([&] { *st = static_cast<int>(p->pool.handle_state(h)); });
}
int vo_pool_handle_mapped_at(const vo_pool* p, int h, int64_t* t) {
  return guard([&] { *t = p->pool.handle_mapped_at(h); });
}
int vo_pool_check_invariants(const vo_pool* p) {
  return guard([&] { p->pool.check_invariants(); });
}
int vo_pool_block_table(const vo_pool*, int64_t, int*, int, int* n) {
  *n = -1;
  g_err = "block tables are not modelled by the reference";
  return VO_RUNTIME_ERROR;
}

int vo_select(int n, const int* ids, const int64_t* mapped, const int* off, const int64_t* reqs, int m,
              const int64_t* keys, const int64_t* vals, int k, int mode, int* out, int* n_out) {
  return guard([&] {
    ReclaimInstance inst = make_inst(n, ids, mapped, off, reqs, m, keys, vals);
    std::vector<int> v = mode == 0   ? selective_reclaim(inst, k)
                         : mode == 1 ? fifo_reclaim(inst, k)
                                     : oracle_reclaim(inst, k);
    *n_out = static_cast<int>(v.size());
    std::copy(v.begin(), v.end(), out);
  });
}
int vo_evicted_cost(int n, const int* ids, const int* off, const int64_t* reqs, int m,
                    const int64_t* keys, const int64_t* vals, const int* pick, int n_pick,
                    int64_t* cost) {
  return guard([&] {
    ReclaimInstance inst = make_inst(n, ids, nullptr, off, reqs, m, keys, vals);
    *cost = evicted_cost(inst, std::vector<int>(pick, pick + n_pick));
  });
}

void vo_resparams_default(vo_resparams* o) {
  ReservationParams p;
  o->alpha = p.alpha;
  o->beta = p.beta;
  o->t_init_us = p.t_init_us;
  o->delta_us = p.delta_us;
  o->t_min_us = p.t_min_us;
  o->t_max_us = p.t_max_us;
  o->window_us = p.window_us;
  o->target_per_window = p.target_per_window;
  o->h_min = p.h_min;
  o->pressure_threshold = p.pressure_threshold;
}
int vo_resctl_create(const vo_resparams* o, vo_resctl** out) {
  return guard([&] {
    ReservationParams p;
    p.alpha = o->alpha;
    p.beta = o->beta;
    p.t_init_us = o->t_init_us;
    p.delta_us = o->delta_us;
    p.t_min_us = o->t_min_us;
    p.t_max_us = o->t_max_us;
    p.window_us = o->window_us;
    p.target_per_window = o->target_per_window;
    p.h_min = o->h_min;
    p.pressure_threshold = o->pressure_threshold;
    *out = new vo_resctl{ReservationController(p)};
  });
}
void vo_resctl_destroy(vo_resctl* c) { delete c; }
int64_t vo_resctl_interval(const vo_resctl* c) { return c->ctl.interval(); }
int64_t vo_resctl_pressure_events(const vo_resctl* c) { return c->ctl.pressure_events(); }
int vo_resctl_grow_target(const vo_resctl* c, int h, int cap) { return c->ctl.grow_target(h, cap); }
void vo_resctl_record_pressure(vo_resctl* c, int64_t t) { c->ctl.record_pressure(t); }
int vo_resctl_release_due(const vo_resctl* c, int64_t t, int h) { return c->ctl.release_due(t, h); }
void vo_resctl_note_tick(vo_resctl* c, int64_t t) { c->ctl.note_tick(t); }
int64_t vo_resctl_window_tick(vo_resctl* c, int64_t t) { return c->ctl.window_tick(t); }
int64_t vo_resctl_pressure_in_window(const vo_resctl* c, int64_t t) {
  return c->ctl.pressure_in_window(t);
}

int vo_channel_create(int64_t toggle, int64_t cooldown, const vo_channel_hooks* hk, vo_channel** out) {
  return guard([&] {
    vo_channel_hooks h = hk ? *hk : vo_channel_hooks{};
    ChannelController::Hooks hooks;
    hooks.schedule = [h](SimTime when, std::int64_t gen, bool cd) {
      if (h.schedule) h.schedule(h.user, when, gen, cd ? 1 : 0);
    };
    hooks.on_disabled = [h](SimTime t) {
      if (h.on_disabled) h.on_disabled(h.user, t);
    };
    hooks.on_enabled = [h](SimTime t) {
      if (h.on_enabled) h.on_enabled(h.user, t);
    };
    hooks.log = [h](SimTime t, ChannelLog what, SimTime aux, bool mem) {
      if (h.log) h.log(h.user, t, static_cast<int>(what), aux, mem ? 1 : 0);
    };
    auto* c = new vo_channel;
    c->ctl = std::make_unique<ChannelController>(toggle, cooldown, std::move(hooks));
    *out = c;
  });
}
void vo_channel_destroy(vo_channel* c) { delete c; }
int vo_channel_state(const vo_channel* c) { return static_cast<int>(c->ctl->state()); }
int vo_channel_offline_compute_allowed(const vo_channel* c) { return c->ctl->offline_compute_allowed(); }
int64_t vo_channel_disables_issued(const vo_channel* c) { return c->ctl->disables_issued(); }
int64_t vo_channel_pending_effective(const vo_channel* c) { return c->ctl->pending_effective(); }
void vo_channel_note_busy(vo_channel* c, int64_t t) { c->ctl->note_busy(t); }
void vo_channel_note_all_idle(vo_channel* c, int64_t t) { c->ctl->note_all_idle(t); }
int64_t vo_channel_ensure_disabled(vo_channel* c, int64_t t) { return c->ctl->ensure_disabled(t); }
void vo_channel_handle_toggle(vo_channel* c, int64_t t, int64_t gen) { c->ctl->handle_toggle(t, gen); }
void vo_channel_handle_cooldown(vo_channel* c, int64_t t, int64_t gen) {
  c->ctl->handle_cooldown(t, gen);
}

// Byte images are not a reference concept; the shim defers to nothing and reports zeros.
uint64_t vo_page_word(int64_t, int32_t, int64_t) { return 0; }
void vo_gather_images(const int64_t*, const int32_t*, int, int64_t, uint8_t*) {}
void vo_gather_memcpy(const uint8_t* src, int64_t slot_bytes, int64_t page_bytes, const int* phys,
                      int n_pages, uint8_t* dst, int) {
  for (int i = 0; i < n_pages; ++i)
    std::memcpy(dst + static_cast<int64_t>(i) * page_bytes,
                src + static_cast<int64_t>(phys[i]) * slot_bytes, static_cast<size_t>(page_bytes));
}

}  // extern "C"

// Draws of the reference's Rng (rng.hpp:31-58) so tests can pin their Python port of it.
#include "colosim/rng.hpp"
extern "C" void vr_rng_draws(uint64_t seed, const char* label, int n, uint64_t* out) {
  Rng rng = label ? Rng::substream(seed, label) : Rng(seed);
  for (int i = 0; i < n; ++i) out[i] = static_cast<uint64_t>(rng.uniform_int(0, INT64_MAX - 1));
}

// CPU baseline of the decision path, timed inside C++ (no ctypes in the timed region):
// snapshot + Cost(r) attach (sim.cpp:877-883) -> selective_reclaim (reclaim.cpp:33-67) ->
// apply_reclaim (memory.cpp:155-180), exactly what Sim::finish_op does per op.  Returns the
// invalidated logical page ids (report order) for the gather leg.
#include <chrono>
extern "C" int vr_time_reclaim(vo_pool* p, const int64_t* keys, const int64_t* vals, int m, int k,
                               int64_t t, double us_out[3], int64_t* pages_out, int cap,
                               int* n_pages) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    std::map<std::int64_t, std::int64_t> cost;
    for (int i = 0; i < m; ++i) cost[keys[i]] = vals[i];
    const auto t0 = clk::now();
    ReclaimInstance inst = p->pool.snapshot();
    for (const ReclaimHandle& h : inst.handles)
      for (std::int64_t r : h.requests) inst.cost[r] = cost.at(r);
    const auto t1 = clk::now();
    std::vector<int> chosen = selective_reclaim(inst, k);
    const auto t2 = clk::now();
    MemoryPool::ReclaimResult res = p->pool.apply_reclaim(chosen, t);
    const auto t3 = clk::now();
    us_out[0] = std::chrono::duration<double, std::micro>(t1 - t0).count();
    us_out[1] = std::chrono::duration<double, std::micro>(t2 - t1).count();
    us_out[2] = std::chrono::duration<double, std::micro>(t3 - t2).count();
    int n = 0;
    for (const auto& [req, pages] : res.invalidated_pages)
      for (std::int64_t pg : pages) {
        if (n < cap) pages_out[n] = pg;
        ++n;
      }
    *n_pages = n;
  });
}
