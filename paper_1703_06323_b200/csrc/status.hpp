// status.hpp — error plumbing for the C ABI: the reference's single error
// type with a code (common.hpp:24-46) becomes Failure inside the library and
// a cutbddc_status + thread-local message at the boundary (never thrown
// across it).
#pragma once

#include <stdexcept>
#include <string>

#include "cutbddc.h"

namespace cutbddc_b200 {

struct Failure : std::runtime_error {
  cutbddc_status code;
  Failure(cutbddc_status c, const std::string& w) : std::runtime_error(w), code(c) {}
};

void set_last_error(const std::string& msg);

template <typename F>
cutbddc_status guard(F&& f) {
  try {
    f();
    return CUTBDDC_OK;
  } catch (const Failure& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return CUTBDDC_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CUTBDDC_INTERNAL;
  }
}

}  // namespace cutbddc_b200
