// colosim/valve_detail.hpp -- status -> C++ exception mapping shared by the drop-in headers.
// The C ABI (valve_cuda.h) never throws; these headers re-raise the reference's exception
// types (memory.cpp / reclaim.cpp / channel.cpp use invalid_argument, logic_error,
// out_of_range via std::vector::at, runtime_error for I/O).
#pragma once
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../valve_cuda.h"

namespace colosim::valve_detail {

inline void check(int rc) {
  if (rc == VALVE_OK) return;
  const std::string msg = valve_last_error();
  switch (rc) {
    case VALVE_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case VALVE_OUT_OF_RANGE: throw std::out_of_range(msg);
    case VALVE_LOGIC_ERROR: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// CUDA ordinal for pools and selection calls made through these headers:
// set_device(), else $VALVE_DEVICE, else 0.
inline int& device_slot() {
  static int dev = [] {
    const char* e = std::getenv("VALVE_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return dev;
}

}  // namespace colosim::valve_detail

namespace colosim {
inline void set_device(int ordinal) { valve_detail::device_slot() = ordinal; }
inline int device() { return valve_detail::device_slot(); }
}  // namespace colosim
