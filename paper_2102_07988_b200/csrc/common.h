// common.h — error plumbing shared by the C-ABI implementation files (host side).
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "tp.h"

namespace tp {

// Sets the thread-local message returned by tp_last_error() and returns `st`.
tp_status fail(tp_status st, const char* fmt, ...);

}  // namespace tp

#define TP_CHECK_ARG(cond, ...)                         \
  do {                                                  \
    if (!(cond)) return ::tp::fail(TP_EINVAL, __VA_ARGS__); \
  } while (0)
