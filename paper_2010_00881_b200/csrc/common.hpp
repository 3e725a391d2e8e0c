// common.hpp -- error reporting shared by the C-ABI entry points.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

namespace fcm {

inline std::string& last_error() {
  thread_local std::string msg;
  return msg;
}
inline void clear_error() { last_error().clear(); }
inline int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return code;
}

}  // namespace fcm
