// Shared host-side plumbing: status/exception mapping, CUDA checks.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "hetpar_b200.h"

namespace hp {

// Mirrors the reference error taxonomy (include/hetpar/common.hpp:14-34).
struct error : std::runtime_error {
  hp_status code;
  error(hp_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(hp_status c, const std::string& m) {
  static const char* prefix[] = {"", "shape: ", "config: ", "index: ", "io: ",
                                 "comm: ", "numeric: ", "cuda: "};
  throw error(c, std::string(prefix[c]) + m);
}

void set_last_error(const std::string& m);

}  // namespace hp

#define HP_CUDA(call)                                                          \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess)                                                     \
      ::hp::fail(HP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + \
                               " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define HP_NCCL(call)                                                          \
  do {                                                                         \
    ncclResult_t r_ = (call);                                                  \
    if (r_ != ncclSuccess)                                                     \
      ::hp::fail(HP_ECOMM, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// C-ABI guard: converts exceptions into statuses + thread-local message.
#define HP_API_BEGIN try {
#define HP_API_END                                                             \
  return HP_OK;                                                                \
  }                                                                            \
  catch (const ::hp::error& e) {                                               \
    ::hp::set_last_error(e.what());                                            \
    return e.code;                                                             \
  }                                                                            \
  catch (const std::exception& e) {                                            \
    ::hp::set_last_error(e.what());                                            \
    return HP_ECONFIG;                                                         \
  }
