// status.hpp — status-code exception and C-ABI guard macros (host + device TUs).
#pragma once
#include <stdexcept>
#include <string>

#include "qgnn_b200.h"

namespace qgnn_b200 {

// Status-carrying exception used inside the library; converted to a status
// code + thread-local message at every C-ABI boundary.
struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
int status_from_exception();

#define QGNN_REQUIRE(cond, code, msg)                         \
  do {                                                        \
    if (!(cond)) throw ::qgnn_b200::Status((code), (msg));    \
  } while (0)

#define QGNN_API_BEGIN try {
#define QGNN_API_END                            \
  return QGNN_OK;                               \
  }                                             \
  catch (...) {                                 \
    return ::qgnn_b200::status_from_exception(); \
  }

}  // namespace qgnn_b200
