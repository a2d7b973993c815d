// grid_solver.hpp -- drop-in for /root/reference/proj/include/shellular/grid_solver.hpp
//
// Same constructor and solve() signature (:20, :37) and Result fields
// (:29-35).  The solve runs on the device (shl_grid_solve): lockstep 6-column
// block-Jacobi PCG, identical stopping rule and iteration accounting.  It
// also accepts masked beta arrays (beta == 0 = absent element), which the
// reference rejects by construction (it requires the full-grid fallback).
#pragma once

#include <array>

#include "fem.hpp"

namespace shellular {

class GridSolver {
 public:
  GridSolver(std::vector<double> beta, int r, const ElementStiffness& K0, int threads = 1)
      : beta_(std::move(beta)), r_(r), K0_(K0.row_major()) {
    (void)threads;
    if (static_cast<size_t>(r_) * r_ * r_ != beta_.size())
      throw ValidationError("beta array does not match resolution");
  }

  struct Result {
    ElasticTensor tensor;
    std::array<int, 6> iterations{};
    double t_rhs_ms = 0.0;
    double t_solve_ms = 0.0;
    double t_reduce_ms = 0.0;
    shl_stats stats{};
  };

  // precision: SHL_PREC_AUTO (FP64 below tol 1e-7), _FP64, _MIXED or _FP32
  Result solve(double tol = 1e-9, int max_iter = 0, int precision = SHL_PREC_AUTO,
               int preconditioner = SHL_PRECOND_JACOBI) {
    const shl_solve_options o{tol, max_iter, precision, 0, preconditioner};
    double C[36];
    Result res;
    shl_ctx* ctx = detail::context();
    detail::check(shl_grid_solve(ctx, r_, beta_.data(), K0_.data(), &o, C, &res.stats), ctx);
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) res.tensor.c(i, j) = C[i * 6 + j];
    for (int s = 0; s < 6; ++s) res.iterations[s] = res.stats.iterations[s];
    res.t_rhs_ms = res.stats.t_AS + res.stats.t_RHS;
    res.t_solve_ms = res.stats.t_solve;
    res.t_reduce_ms = res.stats.t_C;
    return res;
  }

 private:
  std::vector<double> beta_;
  int r_;
  std::array<double, 576> K0_;
};

}  // namespace shellular
