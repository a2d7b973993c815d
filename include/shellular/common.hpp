// common.hpp -- drop-in for /root/reference/proj/include/shellular/common.hpp
//
// Same error hierarchy (:25-48), thread resolution (:50-58), splitmix64 Rng
// (:86-127), Timer (:129-140) and StageTimings (:145-160).  Adds the device
// context plumbing: every call that does device work goes through one
// shl_ctx per (host thread, device) from include/shellular_cuda.h, and C-ABI
// status codes are rethrown as the reference's exception classes.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../shellular_cuda.h"
#include "linalg.hpp"

namespace shellular {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
class ValidationError : public Error {
 public:
  explicit ValidationError(const std::string& msg) : Error(msg) {}
};
class DegenerateDesignError : public Error {
 public:
  explicit DegenerateDesignError(const std::string& msg) : Error(msg) {}
};
class SolverError : public Error {
 public:
  explicit SolverError(const std::string& msg) : Error(msg) {}
};
class IoError : public Error {
 public:
  explicit IoError(const std::string& msg) : Error(msg) {}
};
// Device / driver failure; no reference analogue.
class DeviceError : public Error {
 public:
  explicit DeviceError(const std::string& msg) : Error(msg) {}
};

inline int resolve_threads(int requested) {
  if (requested > 0) return requested;
  if (const char* env = std::getenv("SHELL_THREADS")) {
    int n = std::atoi(env);
    if (n > 0) return n;
  }
  unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : static_cast<int>(hw);
}

// splitmix64 (common.hpp:86-104); Box-Muller normal() as the reference.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : state_(seed ? seed : 0x9e3779b97f4a7c15ull) {}
  std::uint64_t next_u64() {
    std::uint64_t z = (state_ += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  int uniform_int(int lo, int hi) {
    return lo + static_cast<int>(next_u64() % static_cast<std::uint64_t>(hi - lo + 1));
  }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    double u1 = 0.0;
    while (u1 <= 1e-300) u1 = uniform01();
    double u2 = uniform01();
    double r = std::sqrt(-2.0 * std::log(u1));
    double a = 2.0 * M_PI * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }

 private:
  std::uint64_t state_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

class Timer {
 public:
  Timer() : start_(clock::now()) {}
  double elapsed_ms() const {
    return std::chrono::duration<double, std::milli>(clock::now() - start_).count();
  }
  void reset() { start_ = clock::now(); }

 private:
  using clock = std::chrono::steady_clock;
  clock::time_point start_;
};

// Stage times in ms under the paper's Table 2 names; on the device path they
// are CUDA-event times of the corresponding kernels.
struct StageTimings {
  double t_field = 0.0, t_mesh = 0.0, t_PBC = 0.0, t_AS = 0.0, t_RHS = 0.0, t_solve = 0.0,
         t_C = 0.0, t_fwd = 0.0;

  std::map<std::string, double> to_map() const {
    return {{"t_field", t_field}, {"t_mesh", t_mesh}, {"t_PBC", t_PBC}, {"t_AS", t_AS},
            {"t_RHS", t_RHS},     {"t_solve", t_solve}, {"t_C", t_C},   {"t_fwd", t_fwd}};
  }
  std::string to_json() const {
    std::ostringstream os;
    os.precision(17);
    os << "{";
    bool first = true;
    for (const auto& [k, v] : to_map()) {
      os << (first ? "" : ", ") << '"' << k << "\": " << v;
      first = false;
    }
    os << "}";
    return os.str();
  }
};

namespace detail {

// Rethrow a C-ABI status as the reference exception class.
inline void check(int code, const shl_ctx* ctx) {
  if (code == SHL_OK) return;
  const std::string msg = shl_last_error(ctx);
  switch (code) {
    case SHL_VALIDATION: throw ValidationError(msg);
    case SHL_DEGENERATE: throw DegenerateDesignError(msg);
    case SHL_SOLVER: throw SolverError(msg);
    case SHL_IO: throw IoError(msg);
    case SHL_ERROR: throw Error(msg);
    default: throw DeviceError(msg);
  }
}

// One context per (host thread, device), created on first use.
class Context {
 public:
  explicit Context(int device) {
    shl_ctx* c = nullptr;
    check(shl_ctx_create(device, &c), nullptr);
    ctx_ = c;
  }
  ~Context() { shl_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  shl_ctx* get() const { return ctx_; }

 private:
  shl_ctx* ctx_ = nullptr;
};

inline int& current_device() {
  static thread_local int dev = [] {
    const char* e = std::getenv("SHELLULAR_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return dev;
}

inline shl_ctx* context() {
  static thread_local std::map<int, std::unique_ptr<Context>> ctxs;
  int dev = current_device();
  auto it = ctxs.find(dev);
  if (it == ctxs.end()) it = ctxs.emplace(dev, std::make_unique<Context>(dev)).first;
  return it->second->get();
}

}  // namespace detail

// Select the CUDA device used by the calling thread's subsequent calls.
inline void set_device(int device) { detail::current_device() = device; }

}  // namespace shellular
