// fem.hpp -- drop-in for /root/reference/proj/include/shellular/fem.hpp
//
// BaseMaterial (:19-30), ElementStiffness / element_stiffness (:34-92),
// ElasticTensor (:96-125), unit_test_strains (:129-142), hex_corner_offsets
// (:41-46).  The reference's assembled master-slave system + sparse direct
// solve (build_periodic_system / solve_test_strains / effective_tensor,
// :144-428) is replaced by the device's matrix-free masked-torus PCG, which
// solves the same system; `effective_tensor(mesh, K0)` is the
// one-call equivalent.
#pragma once

#include <array>
#include <sstream>

#include "voxel.hpp"

namespace shellular {

struct BaseMaterial {
  double youngs = 1.0;
  double poisson = 0.3;
  void validate() const {
    if (!(youngs > 0.0)) throw ValidationError("Young's modulus must be positive");
    if (!(poisson > -1.0 && poisson < 0.5)) throw ValidationError("Poisson ratio must lie in (-1, 0.5)");
  }
  double lambda() const { return youngs * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)); }
  double mu() const { return youngs / (2.0 * (1.0 + poisson)); }
  double bulk() const { return youngs / (3.0 * (1.0 - 2.0 * poisson)); }
  shl_material abi() const { return {youngs, poisson}; }
};

using Mat24 = Matrix<double, 24, 24>;

struct ElementStiffness {
  Mat24 matrix = Mat24::Zero();
  double edge = 1.0;
  std::array<double, 576> row_major() const {
    std::array<double, 576> k{};
    for (int i = 0; i < 24; ++i)
      for (int j = 0; j < 24; ++j) k[i * 24 + j] = matrix(i, j);
    return k;
  }
};

inline const std::array<Vec3i, 8>& hex_corner_offsets() {
  static const std::array<Vec3i, 8> off = {Vec3i(0, 0, 0), Vec3i(1, 0, 0), Vec3i(1, 1, 0),
                                           Vec3i(0, 1, 0), Vec3i(0, 0, 1), Vec3i(1, 0, 1),
                                           Vec3i(1, 1, 1), Vec3i(0, 1, 1)};
  return off;
}

inline ElementStiffness element_stiffness(const BaseMaterial& mat, double edge) {
  double k[576];
  const shl_material m = mat.abi();
  detail::check(shl_element_stiffness(&m, edge, k), nullptr);
  ElementStiffness out;
  out.edge = edge;
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j) out.matrix(i, j) = k[i * 24 + j];
  return out;
}

struct ElasticTensor {
  Mat6 c = Mat6::Zero();
  static ElasticTensor isotropic(const BaseMaterial& mat) {
    ElasticTensor t;
    double la = mat.lambda(), mu = mat.mu();
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) t.c(a, b) = a == b ? la + 2.0 * mu : la;
    for (int a = 3; a < 6; ++a) t.c(a, a) = mu;
    return t;
  }
  std::string to_json() const {
    std::ostringstream os;
    os.precision(17);
    os << "[";
    for (int i = 0; i < 6; ++i) {
      os << (i ? ", [" : "[");
      for (int j = 0; j < 6; ++j) os << (j ? ", " : "") << c(i, j);
      os << "]";
    }
    os << "]";
    return os.str();
  }
};

inline const std::array<Mat3, 6>& unit_test_strains() {
  static const std::array<Mat3, 6> strains = [] {
    std::array<Mat3, 6> s;
    for (auto& m : s) m.setZero();
    s[0](0, 0) = 1.0;
    s[1](1, 1) = 1.0;
    s[2](2, 2) = 1.0;
    s[3](1, 2) = s[3](2, 1) = 0.5;
    s[4](0, 2) = s[4](2, 0) = 0.5;
    s[5](0, 1) = s[5](1, 0) = 0.5;
    return s;
  }();
  return strains;
}

// Device solve options shared by effective_tensor / GridSolver / homogenize.
struct DeviceSolveOptions {
  double tol = 1e-9;
  int max_iter = 0;
  int precision = SHL_PREC_AUTO;
  int preconditioner = SHL_PRECOND_AUTO;
  shl_solve_options abi() const { return {tol, max_iter, precision, 0, preconditioner}; }
};

// build_periodic_system + solve_test_strains + effective_tensor for `mesh`
// (fem.hpp:179-428) as one device solve; the gauge is node 0 (any corner
// gauge gives the same tensor, test_fem.cpp:234-247).
inline ElasticTensor effective_tensor(const VoxelMesh& mesh, const ElementStiffness& K0,
                                      const DeviceSolveOptions& opt = {},
                                      shl_stats* stats_out = nullptr) {
  const std::vector<double> beta = mesh.dense_beta();
  const auto k = K0.row_major();
  const shl_solve_options o = opt.abi();
  double C[36];
  shl_stats st{};
  shl_ctx* ctx = detail::context();
  detail::check(shl_grid_solve(ctx, mesh.resolution, beta.data(), k.data(), &o, C, &st), ctx);
  if (stats_out) *stats_out = st;
  ElasticTensor t;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) t.c(i, j) = C[i * 6 + j];
  return t;
}

}  // namespace shellular
