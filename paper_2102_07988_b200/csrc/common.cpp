// common.cpp — tp_last_error() plumbing and the host-side parameter layout helpers.
#include "common.h"

#include <cstring>

namespace {
thread_local char g_err[1024] = "";
}

namespace tp {

tp_status fail(tp_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return st;
}

}  // namespace tp

extern "C" const char* tp_last_error(void) { return g_err; }
