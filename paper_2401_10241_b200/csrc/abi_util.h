// Error plumbing shared by the extern "C" entry points: no exception crosses the ABI.
#pragma once
#include <new>
#include <stdexcept>
#include <string>

#include "zb.h"

namespace zb {
extern thread_local std::string g_last_error;

inline zb_status_t set_error(zb_status_t code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

struct Error : std::runtime_error {
  zb_status_t code;
  Error(zb_status_t c, const std::string& m) : std::runtime_error(m), code(c) {}
};
}  // namespace zb

#define ZB_TRY try
#define ZB_CATCH                                                              \
  catch (const ::zb::Error& e) {                                              \
    return ::zb::set_error(e.code, e.what());                                 \
  }                                                                           \
  catch (const std::bad_alloc& e) {                                           \
    return ::zb::set_error(ZB_ECAP, std::string("host allocation: ") + e.what()); \
  }                                                                           \
  catch (const std::invalid_argument& e) {                                    \
    return ::zb::set_error(ZB_EINVAL, e.what());                              \
  }                                                                           \
  catch (const std::exception& e) {                                           \
    return ::zb::set_error(ZB_ECUDA, e.what());                               \
  }                                                                           \
  catch (...) {                                                               \
    return ::zb::set_error(ZB_ECUDA, "unknown error");                        \
  }
