// colosim_ops.cpp -- reclaim ops timed through the reference's C++ runtime API
// (colosim::MemoryPool::snapshot / selective_reclaim / apply_reclaim / offline_reserve /
// offline_release, /root/reference/proj/include/colosim/{memory,reclaim}.hpp).
//
// The same source is compiled twice:
//   tools/_bin/valve_ops  against the drop-in headers (include/colosim), linked to libvalve.so:
//                         every call runs on the B200 through the C ABI (paper_2604_07874_b200/
//                         csrc/Makefile)
//   oracle/_ref/ref_ops   against the reference's own headers and sources (oracle/Makefile; test
//                         / bench infrastructure, CPU)
//
//   ops table H k1,k2,..           per-op latency (median us): offline_reserve, offline_release,
//                                  and snapshot -> selective_reclaim -> apply_reclaim for each k;
//                                  valve_ops adds the fused device op (valve_pool_reclaim)
//   ops e2e H k steps warmup [tenant] (valve_ops) bench.py's e2e leg in C++: per op raise the gate and
//                                  wait for the offline decode pass to quiesce, snapshot, select,
//                                  apply, start the gather copy of the invalidated pages into
//                                  pinned host memory, re-admit; one copy queued behind the
//                                  running one.  Prints GB/s over the timed ops.
// Output: one JSON line.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "colosim/memory.hpp"
#include "colosim/reclaim.hpp"

using namespace colosim;
using clk = std::chrono::steady_clock;

namespace {

constexpr int kS = 64;              // pages per handle (SURVEY §8 geometry: 64 x 2 MiB slots)
constexpr std::int64_t kPage = 917504;  // Qwen2-7B 16-token KV page
constexpr std::int64_t kSlot = 2 << 20;

struct Rng {  // splitmix64: identical streams in both builds
  std::uint64_t s;
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  int range(int lo, int hi) { return lo + static_cast<int>(next() % static_cast<std::uint64_t>(hi - lo + 1)); }
};

double us(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); }

double median(std::vector<double> v) {
  if (v.empty()) return 0;
  std::sort(v.begin(), v.end());
  return v.size() % 2 ? v[v.size() / 2] : 0.5 * (v[v.size() / 2 - 1] + v[v.size() / 2]);
}

// The offline population of bench.py (C2): Qwen2-7B requests, input 2000-4000, output 100-200
// tokens, 16-token pages; cost = input + generated (requests.hpp:68-69).
struct Population {
  std::map<std::int64_t, std::pair<int, std::int64_t>> live;  // id -> (pages, cost)
  std::int64_t next_id = 0;
  SimTime t = 0;
  Rng rng{2604};

  bool admit(MemoryPool& pool) {
    const int in = rng.range(2000, 4000), out = rng.range(100, 200);
    const int pages = (in + out + 15) / 16;
    const std::int64_t cost = in + rng.range(0, out - 1);
    if (!pool.offline_reserve(next_id, pages, ++t)) return false;
    live[next_id++] = {pages, cost};
    return true;
  }
  void fill(MemoryPool& pool) {
    while (admit(pool)) {
    }
  }
  // after a reclaim of k handles: give them back, re-admit the evicted, top up (untimed)
  void restore(MemoryPool& pool, int k, const std::vector<std::int64_t>& evicted) {
    pool.online_release(k);
    for (std::int64_t r : evicted) {
      auto it = live.find(r);
      const auto pc = it->second;
      live.erase(it);
      if (pool.offline_reserve(r, pc.first, ++t)) live[r] = pc;
    }
    fill(pool);
  }
  ReclaimInstance instance(const MemoryPool& pool) const {
    ReclaimInstance inst = pool.snapshot();
    for (const ReclaimHandle& h : inst.handles)
      for (std::int64_t r : h.requests) inst.cost[r] = live.at(r).second;
    return inst;
  }
};

MemoryPool make_pool(int H, bool page_store) {
#ifdef VALVE_DROPIN
  valve_pool_config cfg;
  valve_pool_config_default(&cfg);
  cfg.device = device();
  cfg.total_handles = H;
  cfg.handle_size_pages = kS;
  cfg.page_size_tokens = 16;
  cfg.slot_bytes = page_store ? kSlot : 0;
  cfg.page_bytes = page_store ? kPage : 0;
  return MemoryPool(cfg);
#else
  (void)page_store;
  return MemoryPool(H, kS, 16);
#endif
}

void table(int H, const std::vector<int>& ks) {
  MemoryPool pool = make_pool(H, false);
  Population pop;
  pool.online_grow((H + 9) / 10, 0);
  pop.fill(pool);
#ifdef VALVE_DROPIN
  // the fused single-call path runs on its own pool + population, so the API-path sequence
  // (and every number it reports) stays call-for-call identical to the reference build's
  MemoryPool fpool = make_pool(H, false);
  Population fpop;
  fpool.online_grow((H + 9) / 10, 0);
  fpop.fill(fpool);
#endif
  // offline_release + offline_reserve of live requests (the re-admission path)
  std::vector<double> rel, res;
  std::vector<std::int64_t> ids;
  for (const auto& kv : pop.live) ids.push_back(kv.first);
  for (int i = 0; i < 200 && i < static_cast<int>(ids.size()); ++i) {
    const std::int64_t r = ids[static_cast<std::size_t>(i) * ids.size() / 200];
    const auto pc = pop.live.at(r);
    auto a = clk::now();
    pool.offline_release(r);
    auto b = clk::now();
    const bool ok = pool.offline_reserve(r, pc.first, ++pop.t);
    auto c = clk::now();
    rel.push_back(us(a, b));
    res.push_back(us(b, c));
    if (!ok) pop.live.erase(r);
  }
  std::printf("{\"build\": \"%s\", \"handles\": %d, \"slots_per_handle\": %d, \"live_requests\": %zu, "
              "\"offline_release_us\": %.2f, \"offline_reserve_us\": %.2f, \"reclaim\": [",
#ifdef VALVE_DROPIN
              "valve",
#else
              "reference",
#endif
              H, kS, pop.live.size(), median(rel), median(res));
  for (std::size_t ki = 0; ki < ks.size(); ++ki) {
    const int k = ks[ki];
    std::vector<double> snap, sel, app, tot, fused;
    std::int64_t pages = 0, pages_all = 0;
    const int reps = 15;
    for (int rep = 0; rep < reps + 2; ++rep) {
      auto a = clk::now();
      ReclaimInstance inst = pop.instance(pool);
      auto b = clk::now();
      std::vector<int> pick = selective_reclaim(inst, k);
      auto c = clk::now();
      MemoryPool::ReclaimResult rr = pool.apply_reclaim(pick, ++pop.t);
      auto d = clk::now();
      if (rep >= 2) {
        snap.push_back(us(a, b));
        sel.push_back(us(b, c));
        app.push_back(us(c, d));
        tot.push_back(us(a, d));
      }
      pages = 0;
      for (const auto& kv : rr.invalidated_pages) pages += static_cast<std::int64_t>(kv.second.size());
      pages_all += pages;
      pop.restore(pool, static_cast<int>(rr.handles.size()), rr.evicted_requests);
#ifdef VALVE_DROPIN
      // the B200 single call: snapshot + Algorithm 1 + apply on the device (costs kept with the rows)
      std::vector<std::int64_t> rq, cs;
      for (const auto& kv : fpop.live) rq.push_back(kv.first), cs.push_back(kv.second.second);
      valve_detail::check(valve_pool_set_costs(fpool.native(), static_cast<int>(rq.size()), rq.data(), cs.data()));
      int nh = 0, ne = 0, np = 0;
      auto e = clk::now();
      valve_detail::check(valve_pool_reclaim(fpool.native(), k, VALVE_SELECT_SELECTIVE, ++fpop.t, &nh, &ne, &np));
      auto f = clk::now();
      if (rep >= 2) fused.push_back(us(e, f));
      std::vector<int> hs(static_cast<std::size_t>(nh) + 1);
      std::vector<std::int64_t> ev(static_cast<std::size_t>(ne) + 1);
      valve_detail::check(valve_pool_last_reclaim(fpool.native(), hs.data(), ev.data(), nullptr, nullptr, nullptr,
                                                  nullptr, nh + 1, ne + 1, 0));
      ev.resize(static_cast<std::size_t>(ne));
      fpop.restore(fpool, nh, ev);
#endif
    }
    std::printf("%s{\"k\": %d, \"pages\": %lld, \"pages_all_reps\": %lld, \"snapshot_us\": %.2f, \"select_us\": %.2f, \"apply_us\": %.2f, "
                "\"api_total_us\": %.2f",
                ki ? ", " : "", k, static_cast<long long>(pages), static_cast<long long>(pages_all), median(snap), median(sel), median(app),
                median(tot));
#ifdef VALVE_DROPIN
    std::printf(", \"fused_us\": %.2f", median(fused));
#endif
    std::printf("}");
  }
  std::printf("]}\n");
}

#ifdef VALVE_DROPIN
void e2e(int H, int k, int steps, int warmup, bool tenant) {
  MemoryPool pool = make_pool(H, true);
  Population pop;
  pool.online_grow((H + 9) / 10, 0);
  pop.fill(pool);
  valve_detail::check(valve_pool_fill_pages(pool.native()));
  valve_gate* gate = nullptr;
  valve_detail::check(valve_gate_create(device(), &gate));
  void* off_stream = nullptr;
  valve_detail::check(valve_stream_create(device(), 0, &off_stream));
  const std::int64_t cap = static_cast<std::int64_t>(k) * kS * kPage;
  void* host[2] = {nullptr, nullptr};
  for (void*& h : host) valve_detail::check(valve_host_alloc(cap, &h));
  valve_copy_params cp;
  valve_copy_params_default(&cp);
  cp.ctas = 8;
  valve_offline_work w{};
  w.poll = 1;  // gated: stops claiming tiles once the gate is raised
  int in_flight = 0;
  std::int64_t bytes = 0, h2d = 0, d2h = 0;
  std::map<std::string, double> brk{{"quiesce", 0}, {"snapshot", 0}, {"select", 0}, {"apply", 0},
                                    {"copy_start", 0}, {"restore", 0}, {"copy_wait", 0}};
  auto drain = [&](int keep) {
    std::int64_t got = 0;
    while (in_flight > keep) {
      valve_copy_stats st{};
      valve_detail::check(valve_pool_reclaim_copy_wait(pool.native(), &st));
      got += st.bytes;
      --in_flight;
    }
    return got;
  };
  std::uint32_t gen = 0;
  const bool trace = std::getenv("VALVE_OPS_TRACE") != nullptr;
  auto mark = [&](int it, const char* what) {
    if (trace) std::fprintf(stderr, "e2e it %d: %s\n", it, what), std::fflush(stderr);
  };
  auto t_start = clk::now();
  for (int it = 0; it < warmup + steps; ++it) {
    if (it == warmup) {  // timed burst starts: drain the warm-up, reopen, preempt again
      drain(0);
      valve_detail::check(valve_gate_release(gate, gen, nullptr));
      valve_detail::check(valve_stream_synchronize(valve_gate_stream(gate)));
      bytes = h2d = d2h = 0;
      for (auto& kv : brk) kv.second = 0;
      t_start = clk::now();
    }
    ++gen;
    auto p0 = clk::now();
    if (tenant && (it == 0 || it == warmup)) {  // a burst's first op preempts the running offline tenant
      valve_detail::check(valve_offline_reset(gate));
      valve_detail::check(valve_offline_launch(gate, pool.native(), &w, off_stream));
    }
    mark(it, "raise");
    valve_detail::check(valve_gate_raise(gate, gen, nullptr));
    valve_detail::check(valve_gate_wait_quiesced(gate, gen, nullptr));
    valve_detail::check(valve_stream_synchronize(valve_gate_stream(gate)));
    mark(it, "quiesced");
    auto p1 = clk::now();
    ReclaimInstance inst = pop.instance(pool);
    auto p2 = clk::now();
    std::vector<int> pick = selective_reclaim(inst, k);
    auto p3 = clk::now();
    MemoryPool::ReclaimResult rr = pool.apply_reclaim(pick, ++pop.t);
    auto p4 = clk::now();
    mark(it, "applied");
    std::int64_t npg = 0;
    for (const auto& kv : rr.invalidated_pages) npg += static_cast<std::int64_t>(kv.second.size());
    valve_detail::check(valve_pool_reclaim_copy_start(pool.native(), host[it % 2], cap, &cp));
    ++in_flight;
    auto p5 = clk::now();
    pop.restore(pool, static_cast<int>(rr.handles.size()), rr.evicted_requests);
    auto p6 = clk::now();
    mark(it, "restored");
    bytes += drain(1);
    mark(it, "drained");
    auto p7 = clk::now();
    std::int64_t nnz = 0;
    for (const ReclaimHandle& h : inst.handles) nnz += static_cast<std::int64_t>(h.requests.size());
    const std::int64_t n = static_cast<std::int64_t>(inst.handles.size()), m = static_cast<std::int64_t>(inst.cost.size());
    // bytes crossing the link for this op (the C ABI's buffers): instance down, instance + ids
    // up for the selection, ids up / report down for apply, and the page bytes
    d2h += n * 16 + 4 + nnz * 8 + 4 * k + static_cast<std::int64_t>(rr.evicted_requests.size()) * 12 + npg * 16 +
           npg * kPage;
    h2d += n * 16 + 4 + nnz * 8 + m * 16 + 4 * k;
    brk["quiesce"] += us(p0, p1);
    brk["snapshot"] += us(p1, p2);
    brk["select"] += us(p2, p3);
    brk["apply"] += us(p3, p4);
    brk["copy_start"] += us(p4, p5);
    brk["restore"] += us(p5, p6);
    brk["copy_wait"] += us(p6, p7);
  }
  bytes += drain(0);
  const double secs = us(t_start, clk::now()) * 1e-6;
  valve_detail::check(valve_gate_release(gate, gen, nullptr));
  valve_detail::check(valve_offline_cancel(gate));
  valve_detail::check(valve_stream_synchronize(off_stream));
  valve_detail::check(valve_stream_synchronize(valve_gate_stream(gate)));
  std::printf("{\"build\": \"valve\", \"handles\": %d, \"k\": %d, \"steps\": %d, \"bytes\": %lld, \"seconds\": %.6f, "
              "\"gbs\": %.3f, \"h2d_bytes_per_step\": %lld, \"d2h_bytes_per_step\": %lld, \"breakdown_ms_per_step\": {",
              H, k, steps, static_cast<long long>(bytes), secs, bytes / secs / 1e9,
              static_cast<long long>(h2d / steps), static_cast<long long>(d2h / steps));
  bool first = true;
  for (const auto& kv : brk) {
    std::printf("%s\"%s\": %.3f", first ? "" : ", ", kv.first.c_str(), kv.second / steps / 1e3);
    first = false;
  }
  std::printf("}}\n");
  for (void* h : host) valve_host_free(h);
  valve_stream_destroy(off_stream);
  valve_gate_destroy(gate);
}
#endif

std::vector<int> parse_ks(const char* s) {
  std::vector<int> out;
  std::string cur;
  for (const char* p = s;; ++p) {
    if (*p == ',' || *p == 0) {
      if (!cur.empty()) out.push_back(std::atoi(cur.c_str()));
      cur.clear();
      if (!*p) break;
    } else {
      cur += *p;
    }
  }
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string mode = argc > 1 ? argv[1] : "table";
    if (mode == "table") {
      table(argc > 2 ? std::atoi(argv[2]) : 1024, parse_ks(argc > 3 ? argv[3] : "1,4,15,36,64"));
      return 0;
    }
#ifdef VALVE_DROPIN
    if (mode == "e2e") {
      e2e(argc > 2 ? std::atoi(argv[2]) : 1024, argc > 3 ? std::atoi(argv[3]) : 36, argc > 4 ? std::atoi(argv[4]) : 20,
          argc > 5 ? std::atoi(argv[5]) : 3, argc > 6 ? std::atoi(argv[6]) != 0 : true);
      return 0;
    }
#endif
    std::fprintf(stderr, "usage: %s table H k1,k2,.. | e2e H k steps warmup\n", argv[0]);
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
