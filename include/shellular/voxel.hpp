// voxel.hpp -- drop-in for /root/reference/proj/include/shellular/voxel.hpp
//
// ShellParams (:18-34), step_function (:38-41), classify_surface_elements
// (:118-141) and build_reduced_mesh (:235-313) with the reference's
// semantics; the element selection and beta run on the device (identical
// element sets, beta within 1e-12 relative).  The node bookkeeping of
// build_topology (:147-228) is implicit on the device (active torus nodes);
// VoxelMesh therefore carries the element list, beta and counts but does not
// materialize node_coords / periodic_groups.
#pragma once

#include <fstream>
#include <vector>

#include "field.hpp"

namespace shellular {

struct ShellParams {
  double sharpness = 500.0;
  double floor_ratio = 1e-3;
  int expand_layers = 0;

  void validate() const {
    if (!(sharpness > 0.0)) throw ValidationError("sharpness must be positive");
    if (!(floor_ratio > 0.0 && floor_ratio < 1.0)) throw ValidationError("floor must lie in (0, 1)");
    if (expand_layers < 0) throw ValidationError("expand_layers must be >= 0");
  }
  int layers_for(int r) const {
    if (expand_layers > 0) return expand_layers;
    return std::max(1, static_cast<int>(std::lround(2.0 * r / 64.0)));
  }
  shl_shell_params abi() const { return {sharpness, floor_ratio, expand_layers}; }
};

inline double step_function(double v, const ShellParams& sp) {
  double v0 = 2.0 * (1.0 - sp.floor_ratio);
  return 1.0 + 0.5 * v0 - v0 / (1.0 + std::exp(-sp.sharpness * v * v));
}

struct VoxelMesh {
  int resolution = 0;
  std::vector<std::uint32_t> elements;  // sorted linear ids (k*r + j)*r + i
  std::vector<double> beta;             // per element
  bool full_fallback = false;
  std::int64_t active_nodes = 0;  // torus nodes touched by an element (device count)

  size_t num_elements() const { return elements.size(); }
  double element_fraction() const {
    return double(elements.size()) / (double(resolution) * resolution * resolution);
  }
  double volume_ratio() const {
    double s = 0.0;
    for (double b : beta) s += b;
    return s / (double(resolution) * resolution * resolution);
  }
  static std::uint32_t element_id(int i, int j, int k, int r) {
    return static_cast<std::uint32_t>((k * r + j) * r + i);
  }
  static Vec3i element_coords(std::uint32_t id, int r) {
    return Vec3i(static_cast<int>(id % r), static_cast<int>((id / r) % r), static_cast<int>(id / (r * r)));
  }
  // voxel.hpp:106-114: r^3 bytes, 0 = absent, 1..255 = quantized beta
  void write_raw(const std::string& path) const {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    std::vector<std::uint8_t> occ(static_cast<size_t>(resolution) * resolution * resolution, 0);
    for (size_t e = 0; e < elements.size(); ++e)
      occ[elements[e]] = static_cast<std::uint8_t>(1 + std::lround(beta[e] * 254.0));
    out.write(reinterpret_cast<const char*>(occ.data()), static_cast<std::streamsize>(occ.size()));
    if (!out) throw IoError("failed writing '" + path + "'");
  }
  // dense r^3 beta (0 = absent), the device solver's input
  std::vector<double> dense_beta() const {
    std::vector<double> b(static_cast<size_t>(resolution) * resolution * resolution, 0.0);
    for (size_t e = 0; e < elements.size(); ++e) b[elements[e]] = beta[e];
    return b;
  }
};

namespace detail {
inline shl_ctx* load_grid(const FieldGrid& grid) {
  shl_ctx* ctx = context();
  check(shl_load_grid(ctx, grid.resolution, grid.samples.data(), grid.corner_samples.data(), grid.norm),
        ctx);
  return ctx;
}
}  // namespace detail

inline std::vector<std::uint32_t> classify_surface_elements(const FieldGrid& grid) {
  if (grid.degenerate())
    throw DegenerateDesignError("cannot classify surface elements of a degenerate field");
  shl_ctx* ctx = detail::load_grid(grid);
  std::vector<std::uint32_t> out(static_cast<size_t>(grid.resolution) * grid.resolution * grid.resolution);
  std::int64_t n = 0;
  detail::check(shl_classify_surface(ctx, out.data(), &n), ctx);
  out.resize(static_cast<size_t>(n));
  return out;
}

inline VoxelMesh build_reduced_mesh(const FieldGrid& grid, const ShellParams& sp) {
  sp.validate();
  shl_ctx* ctx = detail::load_grid(grid);
  const int r = grid.resolution;
  VoxelMesh m;
  m.resolution = r;
  m.elements.resize(static_cast<size_t>(r) * r * r);
  m.beta.resize(m.elements.size());
  std::int64_t n = 0;
  std::int32_t ff = 0;
  const shl_shell_params p = sp.abi();
  detail::check(shl_build_reduced_mesh(ctx, &p, m.elements.data(), m.beta.data(), &n, &ff), ctx);
  m.elements.resize(static_cast<size_t>(n));
  m.beta.resize(static_cast<size_t>(n));
  m.full_fallback = ff != 0;
  return m;
}

inline VoxelMesh full_solid_mesh(int r, double beta_value = 1.0) {
  VoxelMesh m;
  m.resolution = r;
  const size_t total = static_cast<size_t>(r) * r * r;
  m.elements.resize(total);
  for (size_t e = 0; e < total; ++e) m.elements[e] = static_cast<std::uint32_t>(e);
  m.beta.assign(total, beta_value);
  m.full_fallback = true;
  m.active_nodes = static_cast<std::int64_t>(total);
  return m;
}

inline VoxelMesh full_field_mesh(const FieldGrid& grid, const ShellParams& sp) {
  sp.validate();
  if (grid.degenerate()) throw DegenerateDesignError("degenerate field");
  VoxelMesh m = full_solid_mesh(grid.resolution, 1.0);
  for (size_t e = 0; e < m.elements.size(); ++e) m.beta[e] = step_function(grid.samples[e] / grid.norm, sp);
  return m;
}

}  // namespace shellular
