// Internal helpers shared by the host runtime and the CUDA sources.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "dsinf.h"

namespace dsinf {

// infersim::ConfigError / InfeasibleError (errors.hpp:24-34) on the C++ side; the C ABI
// converts them into DSINF_ERR_CONFIG / DSINF_ERR_INFEASIBLE.
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
struct InfeasibleError : std::runtime_error {
  explicit InfeasibleError(const std::string& w) : std::runtime_error(w) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};
struct NcclError : std::runtime_error {
  explicit NcclError(const std::string& w) : std::runtime_error(w) {}
};

void set_last_error(const std::string& msg);

// Runs `fn`, mapping exceptions to status codes (exceptions never cross the C ABI).
template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return DSINF_OK;
  } catch (const ConfigError& e) {
    set_last_error(e.what());
    return DSINF_ERR_CONFIG;
  } catch (const InfeasibleError& e) {
    set_last_error(e.what());
    return DSINF_ERR_INFEASIBLE;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return DSINF_ERR_CUDA;
  } catch (const NcclError& e) {
    set_last_error(e.what());
    return DSINF_ERR_NCCL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return DSINF_ERR_INTERNAL;
  }
}

inline void require(bool ok, const char* msg) {
  if (!ok) throw ConfigError(msg);
}

}  // namespace dsinf

#define DSINF_CUDA_CHECK(expr)                                                          \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw ::dsinf::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" + \
                               __FILE__ + ":" + std::to_string(__LINE__) + ")");        \
  } while (0)
