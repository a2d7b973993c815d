// internal.h -- declarations shared by the host code and the CUDA kernels of
// libshellular_cuda.so.  Not part of the public ABI (include/shellular_cuda.h).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/shellular_cuda.h"

namespace shl {

struct ShlError : std::runtime_error {
  int code;
  ShlError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Local corner order of the trilinear hex (fem.hpp:41-46, voxel.hpp:157-158).
constexpr int kCorner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                               {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

struct HostDesign {
  int symmetry = SHL_SYM_NONE;
  int K = 2;
  std::vector<double> pos;  // 3 per charge, wrapped into [0,1)
  std::vector<int> sign;
  std::vector<double> weights;  // (K+1)^3

  static HostDesign from_abi(const shl_design& d);
  void validate() const;
  HostDesign expanded() const;
  std::vector<double> grid_coefficients() const;
};

double basis_weight(int h, int k, int l);
std::vector<double> axis_tables(const HostDesign& expanded, int r);
void element_stiffness(double E, double nu, double edge, double* K);
HostDesign random_design(int sym, int n_pre, int K, double lo, double hi, uint64_t seed);

}  // namespace shl
