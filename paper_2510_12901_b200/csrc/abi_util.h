// Internal helpers of libsimuli (host side): thread-local error text and argument checks.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/simuli.h"

namespace simuli {

void set_error(const char* fmt, ...);
void clear_error();

#define SIMULI_REQUIRE(cond, ...)                 \
  do {                                            \
    if (!(cond)) {                                \
      ::simuli::set_error(__VA_ARGS__);           \
      return SIMULI_ERR_INVALID_ARGUMENT;         \
    }                                             \
  } while (0)

}  // namespace simuli
