// colosim/channel.hpp -- drop-in for /root/reference/proj/include/colosim/channel.hpp:12-80.
// The state machine runs on the host (valve_channel_*) with the reference's hooks; on a pool
// with a device gate (bind_gate) the disable edge raises the HBM gate word that the gated
// offline kernels poll at every tile boundary, and the enable edge releases it.
#pragma once
#include <cstdint>
#include <functional>
#include <memory>

#include "colosim/time.hpp"
#include "colosim/valve_detail.hpp"

namespace colosim {

struct CooldownPolicy {
  SimTime max_gap_us = 0;
  SimTime cooldown_us() const { return 2 * max_gap_us; }  // T_cool = 2G
};

enum class ChannelLog : std::uint8_t {
  kDisableIssued,
  kDisabled,
  kEnableIssued,
  kEnabled,
  kCooldownScheduled,
  kCooldownCancelled,
};

class ChannelController {
 public:
  enum class State : std::uint8_t { kEnabled, kDisabling, kDisabled, kEnabling };

  struct Hooks {
    std::function<void(SimTime when, std::int64_t gen, bool cooldown)> schedule;
    std::function<void(SimTime t)> on_disabled;
    std::function<void(SimTime t)> on_enabled;
    std::function<void(SimTime t, ChannelLog what, SimTime aux, bool memory_cause)> log;
  };

  ChannelController(SimTime toggle_us, SimTime cooldown_us, Hooks hooks)
      : hooks_(std::make_unique<Hooks>(std::move(hooks))) {
    valve_channel_hooks c{};
    c.user = hooks_.get();
    c.schedule = [](void* u, std::int64_t when, std::int64_t gen, int cd) {
      auto* h = static_cast<Hooks*>(u);
      if (h->schedule) h->schedule(when, gen, cd != 0);
    };
    c.on_disabled = [](void* u, std::int64_t t) {
      auto* h = static_cast<Hooks*>(u);
      if (h->on_disabled) h->on_disabled(t);
    };
    c.on_enabled = [](void* u, std::int64_t t) {
      auto* h = static_cast<Hooks*>(u);
      if (h->on_enabled) h->on_enabled(t);
    };
    c.log = [](void* u, std::int64_t t, int what, std::int64_t aux, int mem) {
      auto* h = static_cast<Hooks*>(u);
      if (h->log) h->log(t, static_cast<ChannelLog>(what), aux, mem != 0);
    };
    valve_channel* ch = nullptr;
    valve_detail::check(valve_channel_create(toggle_us, cooldown_us, &c, &ch));
    ch_.reset(ch);
  }

  State state() const { return static_cast<State>(valve_channel_state(ch_.get())); }
  bool offline_compute_allowed() const { return valve_channel_offline_compute_allowed(ch_.get()) != 0; }
  std::int64_t disables_issued() const { return valve_channel_disables_issued(ch_.get()); }
  // Transitions that store to the bound device gate (disable raises it, enable releases it)
  // surface a failed store as std::runtime_error, after the state machine has moved -- the
  // reference's transitions cannot fail, so its callers never see this without a gate.
  void note_busy(SimTime t) {
    valve_channel_note_busy(ch_.get(), t);
    gate_check();
  }
  void note_all_idle(SimTime t) { valve_channel_note_all_idle(ch_.get(), t); }
  SimTime ensure_disabled(SimTime t) {
    const SimTime e = valve_channel_ensure_disabled(ch_.get(), t);
    gate_check();
    return e;
  }
  void handle_toggle(SimTime t, std::int64_t gen) {
    valve_channel_handle_toggle(ch_.get(), t, gen);
    gate_check();
  }
  void handle_cooldown(SimTime t, std::int64_t gen) {
    valve_channel_handle_cooldown(ch_.get(), t, gen);
    gate_check();
  }
  SimTime pending_effective() const { return valve_channel_pending_effective(ch_.get()); }

  // B200 addition: raise/release this device gate on the disable/enable edges.
  void bind_gate(valve_gate* g) { valve_detail::check(valve_channel_bind_gate(ch_.get(), g)); }
  void bind_gate(valve_gate* g, void* stream) {
    valve_detail::check(valve_channel_bind_gate_stream(ch_.get(), g, stream));
  }

 private:
  void gate_check() { valve_detail::check(valve_channel_gate_status(ch_.get())); }
  struct Del {
    void operator()(valve_channel* c) const { valve_channel_destroy(c); }
  };
  std::unique_ptr<Hooks> hooks_;  // stable address for the C trampolines
  std::unique_ptr<valve_channel, Del> ch_;
};

}  // namespace colosim
