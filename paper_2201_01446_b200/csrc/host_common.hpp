// Shared host-side helpers of the dp_b200 library: error classes mirroring the reference's
// (error.hpp:9-17), the C-ABI guard that maps them to return codes (dpmd.cpp:434-443), unit
// constants (units.hpp:9-18) and the smooth switch (switch_fn.hpp:11-25).
#pragma once

#include <algorithm>
#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

#include "dp_b200.h"

namespace dpb {

struct InputErr : std::runtime_error {
  explicit InputErr(const std::string& m) : std::runtime_error(m) {}
};
struct NumErr : std::runtime_error {
  explicit NumErr(const std::string& m) : std::runtime_error(m) {}
};
struct CudaErr : std::runtime_error {
  explicit CudaErr(const std::string& m) : std::runtime_error(m) {}
};

namespace units {
constexpr double K_B = 8.617333262e-5;
constexpr double MVV_TO_EV = 1.0e7 / (6.02214076e23 * 1.602176634e-19);
constexpr double EVA_PER_MASS_TO_ACC = 1.0 / MVV_TO_EV;
constexpr double EVA3_TO_BAR = 1.602176634e6;
} // namespace units

// Last error text of calls that have no handle (generators).
std::string& global_error();

template <class F>
int guard_call(std::string* err, F&& f) {
  std::string& e = err ? *err : global_error();
  try {
    f();
    return DP_OK;
  } catch (const InputErr& x) {
    e = x.what();
    return DP_INPUT_ERROR;
  } catch (const NumErr& x) {
    e = x.what();
    return DP_NUMERICAL_ERROR;
  } catch (const std::exception& x) {
    e = x.what();
    return DP_RUNTIME_ERROR;
  }
}

inline double switch_w(double r, double rs, double rc) {
  if (r >= rc) return 0.0;
  if (r <= rs) return 1.0;
  const double u = (r - rs) / (rc - rs);
  const double uu = u * u;
  return std::max(0.0, uu * u * (-6.0 * uu + 15.0 * u - 10.0) + 1.0);
}

// Offsets of every parameter array inside a model blob (dp_b200.h "Model flat layout").
struct ModelLayout {
  explicit ModelLayout(const dp_preset& s);
  std::vector<std::size_t> emb_off;
  std::vector<std::vector<std::size_t>> fit_w_off, fit_b_off;
  std::vector<std::size_t> fit_wout_off, fit_bout_off;
  std::size_t total = 0;
};

void check_shape(const dp_preset& s);

} // namespace dpb
