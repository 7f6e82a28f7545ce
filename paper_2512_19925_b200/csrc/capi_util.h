// Exception -> status-code translation for the C ABI (no exception crosses it).
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "hwwg.h"

namespace hwwg {

std::string& last_error_slot();

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct ApiError : std::runtime_error {
  int code;
  ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline int fail(int code, const std::string& msg) {
  last_error_slot() = msg;
  return code;
}

}  // namespace hwwg

#define HWWG_API_BEGIN try {
#define HWWG_API_END                                                         \
  }                                                                          \
  catch (const ::hwwg::ApiError& e) {                                        \
    return ::hwwg::fail(e.code, e.what());                                   \
  }                                                                          \
  catch (const ::hwwg::CudaError& e) {                                       \
    return ::hwwg::fail(HWWG_ECUDA, e.what());                               \
  }                                                                          \
  catch (const std::bad_alloc&) {                                            \
    return ::hwwg::fail(HWWG_ENOMEM, "device or host allocation failed");    \
  }                                                                          \
  catch (const std::exception& e) {                                          \
    return ::hwwg::fail(HWWG_EINVAL, e.what());                              \
  }
