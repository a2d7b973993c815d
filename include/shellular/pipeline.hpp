// pipeline.hpp -- drop-in for /root/reference/proj/include/shellular/pipeline.hpp
//
// homogenize(params, sp, mat, r, opt) (:61-113) with the same signature and
// defaults; the whole pipeline (field, mask, six-load-case PCG, C^H) runs on
// the device through one shl_homogenize call.  Errors carry the reference's
// stage prefixes ("field: ", "mesh: ", "solve: ").  solver_used reports the
// device solver ("device_pcg_mixed" / "device_pcg_fp64" / ...) instead of
// "grid_cg" / "direct_ldlt" (solver-name contract).  Like the
// reference, the result carries the sampled grid and the reduced mesh (with
// its lattice topology); return_fields = false skips those readbacks.
#pragma once

#include <sstream>
#include <string>

#include "grid_solver.hpp"

namespace shellular {

enum class SolverKind { Auto, Direct, GridCG };

struct HomogenizeOptions {
  int threads = 1;                      // accepted, unused (device path)
  SolverKind solver = SolverKind::Auto;  // the device PCG; GridCG keeps the reference's full-grid check
  double residual_tol = 1e-9;
  int corner_gauge = 0;                 // any gauge gives the same tensor
  int precision = SHL_PREC_AUTO;        // device arithmetic (shellular_cuda.h)
  int max_iter = 0;
  int preconditioner = SHL_PRECOND_AUTO;  // multigrid V-cycle when r allows (shellular_cuda.h)
  bool return_fields = true;            // fill res.grid / res.mesh as the reference does (pipeline.hpp:70,74)
};

struct HomogenizationResult {
  ElasticTensor tensor;
  FieldGrid grid;   // samples when opt.return_fields (default)
  VoxelMesh mesh;   // resolution / full_fallback always; elements, beta, topology when return_fields
  StageTimings timings;
  double volume_ratio = 0.0;
  double element_fraction = 0.0;
  std::string solver_used;
  std::array<int, 6> iterations{};
  shl_stats stats{};

  std::string to_json() const {
    std::ostringstream os;
    os.precision(17);
    os << "{\"C\": " << tensor.to_json() << ", \"resolution\": " << grid.resolution
       << ", \"volume_ratio\": " << volume_ratio << ", \"element_fraction\": " << element_fraction
       << ", \"solver\": \"" << solver_used << "\", \"timings_ms\": " << timings.to_json() << "}";
    return os.str();
  }
};

inline HomogenizationResult homogenize(const DesignParams& params, const ShellParams& sp,
                                       const BaseMaterial& mat, int r,
                                       const HomogenizeOptions& opt = {}) {
  mat.validate();
  sp.validate();
  auto a = params.abi();
  const shl_shell_params spa = sp.abi();
  const shl_material ma = mat.abi();
  const shl_solve_options o{opt.residual_tol, opt.max_iter, opt.precision, 0, opt.preconditioner};
  HomogenizationResult res;
  double C[36];
  shl_ctx* ctx = detail::context();
  detail::check(shl_homogenize(ctx, &a.d, &spa, &ma, r, &o, C, &res.stats), ctx);
  // pipeline.hpp:81-88: the grid solver only accepts the full-grid fallback mesh
  if (opt.solver == SolverKind::GridCG && res.stats.full_fallback == 0)
    throw SolverError("solve: grid solver requires the full-grid fallback mesh");
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) res.tensor.c(i, j) = C[i * 6 + j];
  const shl_stats& st = res.stats;
  res.timings = {st.t_field, st.t_mesh, st.t_PBC, st.t_AS, st.t_RHS, st.t_solve, st.t_C, st.t_fwd};
  res.volume_ratio = st.volume_ratio;
  res.element_fraction = double(st.n_elements) / (double(r) * r * r);
  for (int s = 0; s < 6; ++s) res.iterations[s] = st.iterations[s];
  static const char* names[] = {"device_pcg_fp64", "device_pcg_mixed", "device_pcg_fp32"};
  res.solver_used = (st.precision >= 0 && st.precision <= 2) ? names[st.precision] : "device_pcg";
  res.grid.resolution = r;
  res.grid.norm = st.norm;
  res.mesh.resolution = r;
  res.mesh.full_fallback = st.full_fallback != 0;
  res.mesh.active_nodes = st.n_nodes;
  if (opt.return_fields) {
    res.grid = sample_grid(params, r);
    res.mesh = build_reduced_mesh(res.grid, sp);
    res.mesh.active_nodes = st.n_nodes;
  }
  return res;
}

}  // namespace shellular
