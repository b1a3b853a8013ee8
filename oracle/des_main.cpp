// des_main.cpp -- runs one scenario through the reference's discrete-event simulator and
// writes its event log (the reference's byte-stable JSONL, log.cpp:69-217).  TEST
// INFRASTRUCTURE: oracle/Makefile links it twice --
//   _ref/ref_des    reference sim + reference MemoryPool / selection / ChannelController
//   _ref/valve_des  reference sim compiled against include/colosim (the drop-in headers), so
//                   every pool, selection and channel call goes through libvalve.so on the GPU
// -- and tests/test_gpu_des.py requires the two logs to be byte-identical.
#include <cstdio>
#include <fstream>
#include <string>

#include "colosim/log.hpp"
#include "colosim/scenario.hpp"
#include "colosim/sim.hpp"

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s scenario.json out.jsonl [preset]\n", argv[0]);
    return 2;
  }
  try {
    colosim::Scenario sc = colosim::load_scenario_file(argv[1]);
    if (argc > 3) sc = colosim::with_preset(sc, argv[3]);
    colosim::SimOutput out = colosim::run_colocation(sc);
    std::ofstream f(argv[2]);
    colosim::write_log_jsonl(f, out.log);
    std::printf("records=%zu final_time=%lld\n", out.log.size(), static_cast<long long>(out.final_time));
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
