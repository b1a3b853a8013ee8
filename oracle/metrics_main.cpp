// ref_metrics -- the reference's own report code (metrics.cpp build_report / ttft_increase /
// tpot_increase, log.cpp read_log_file; compiled unmodified from /root/reference/proj/src)
// applied to event logs.  TEST INFRASTRUCTURE ONLY: it recomputes the TTFT/TPOT deltas the
// real-time harness (paper_2604_07874_b200/realtime.py) reports, from the events.jsonl it wrote.
//
//   ref_metrics STANDALONE.jsonl COLOCATED.jsonl [NORMALIZATION_REFERENCE.jsonl]
//     -> {"ttft_mean_pct":..,"ttft_max_pct":..,"tpot_mean_pct":..,"tpot_max_pct":..,"pairs":..,
//         "tpot_pairs":..,"online_completed":..,"disables_issued":..,"reclaim_ops":..,"evictions":..,
//         "kills":..,"pressure_events":..,"offline_tokens_per_s":..,
//         "normalized_offline_throughput":..}   (the last with a third log: metrics.cpp:243-247,
//                                                e.g. the channel+prism run)
#include <cstdio>
#include <exception>

#include "colosim/log.hpp"
#include "colosim/metrics.hpp"

int main(int argc, char** argv) {
  if (argc != 3 && argc != 4) {
    std::fprintf(stderr, "usage: %s standalone.jsonl colocated.jsonl [reference.jsonl]\n", argv[0]);
    return 2;
  }
  try {
    const colosim::RunReport a = colosim::build_report(colosim::read_log_file(argv[1]));
    const colosim::RunReport b = colosim::build_report(colosim::read_log_file(argv[2]));
    const colosim::PairedIncrease t = colosim::ttft_increase(a, b);
    const colosim::PairedIncrease p = colosim::tpot_increase(a, b);
    double norm = -1.0;
    if (argc == 4) norm = colosim::normalized_offline_throughput(colosim::build_report(colosim::read_log_file(argv[3])), b);
    std::printf(
        "{\"ttft_mean_pct\":%.17g,\"ttft_max_pct\":%.17g,\"tpot_mean_pct\":%.17g,\"tpot_max_pct\":%.17g,"
        "\"pairs\":%lld,\"tpot_pairs\":%lld,\"online_completed\":%lld,\"disables_issued\":%lld,"
        "\"reclaim_ops\":%lld,\"evictions\":%lld,\"kills\":%lld,\"pressure_events\":%lld,"
        "\"offline_tokens_per_s\":%.17g,\"normalized_offline_throughput\":%.17g}\n",
        t.mean_pct, t.max_pct, p.mean_pct, p.max_pct, (long long)t.pairs, (long long)p.pairs,
        (long long)b.online_completed, (long long)b.disables_issued, (long long)b.reclaim_ops,
        (long long)b.evictions, (long long)b.kills, (long long)b.pressure_events, b.offline_tokens_per_s, norm);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_metrics: %s\n", e.what());
    return 1;
  }
  return 0;
}
