// Internal error plumbing for libplora.  The exception types mirror the
// reference's (include/lorasim/errors.hpp:9-24); the C ABI maps them onto
// the status codes in include/plora.h and a thread-local message.
#pragma once

#include <atomic>
#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>

#include "plora.h"

namespace plora {

class ValidationError : public std::runtime_error {
 public:
  explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class ParseError : public std::runtime_error {
 public:
  explicit ParseError(const std::string& m) : std::runtime_error(m) {}
};
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

void set_last_error(const std::string& msg);
void count_launch(uint64_t n = 1);

// Runs f, translating exceptions into PLORA_E_* codes.  f returns int.
template <class F>
int guard(F&& f) noexcept {
  try {
    return f();
  } catch (const ValidationError& e) {
    set_last_error(e.what());
    return PLORA_E_VALIDATION;
  } catch (const ConfigError& e) {
    set_last_error(e.what());
    return PLORA_E_CONFIG;
  } catch (const ParseError& e) {
    set_last_error(e.what());
    return PLORA_E_PARSE;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return PLORA_E_CUDA;
  } catch (const std::logic_error& e) {
    set_last_error(e.what());
    return PLORA_E_LOGIC;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return PLORA_E_NOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PLORA_E_LOGIC;
  }
}

}  // namespace plora
