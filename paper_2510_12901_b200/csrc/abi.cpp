// libsimuli ABI plumbing: thread-local error text, version.
#include <cstdarg>
#include <cstdio>

#include "abi_util.h"

namespace simuli {
thread_local char g_error[512] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_error, sizeof(g_error), fmt, ap);
  va_end(ap);
}
void clear_error() { g_error[0] = '\0'; }
}  // namespace simuli

extern "C" const char* simuli_last_error(void) { return simuli::g_error; }
extern "C" int32_t simuli_abi_version(void) { return SIMULI_ABI_VERSION; }
