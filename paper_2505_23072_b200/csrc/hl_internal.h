// hl_internal.h — shared helpers of libhbmload (not part of the ABI).
#pragma once
#include <stdarg.h>
#include <stdint.h>

#include "../../include/hbmload.h"

namespace hl {
// Record a thread-local error message and return `code` (negative hl_status).
int set_error(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
void clear_error();
}  // namespace hl
