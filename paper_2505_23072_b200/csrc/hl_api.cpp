// hl_api.cpp — error reporting and version entry points of the C ABI.
#include <stdio.h>

#include "hl_internal.h"

namespace hl {
static thread_local char g_err[1024];

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

void clear_error() { g_err[0] = 0; }
}  // namespace hl

extern "C" const char* hl_last_error(void) { return hl::g_err; }
extern "C" int hl_abi_version(void) { return HL_ABI_VERSION; }
extern "C" const char* hl_version(void) { return "hbmload 0.1.0 (sm_100a)"; }
