// voxel.hpp -- drop-in for /root/reference/proj/include/shellular/voxel.hpp
//
// ShellParams (:18-34), step_function (:38-41), classify_surface_elements
// (:118-141) and build_reduced_mesh (:235-313) with the reference's
// semantics; the element selection and beta run on the device (identical
// element sets, beta within 1e-12 relative).  The device solver needs no
// lattice topology (active torus nodes are implicit), but the drop-in
// VoxelMesh carries the reference's: element_nodes, node_coords, node_class,
// periodic_groups and corner_group with build_topology's (:147-228) numbering,
// built on the host from the returned element list (detail::build_topology).
#pragma once

#include <algorithm>
#include <chrono>
#include <fstream>
#include <string>
#include <utility>
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

enum class NodeClass : std::uint8_t { Interior, Face, Edge, Corner };

struct PeriodicGroup {
  std::uint32_t master = 0;                             // node with all offsets zero
  std::vector<std::pair<std::uint32_t, Vec3i>> slaves;  // (node, lattice offset in {0,1}^3)
};

struct VoxelMesh {
  int resolution = 0;
  std::vector<std::uint32_t> elements;  // sorted linear ids (k*r + j)*r + i
  std::vector<double> beta;             // per element
  std::vector<std::uint32_t> element_nodes;  // 8 per element (voxel.hpp:147-228 numbering)
  std::vector<Vec3i> node_coords;            // lattice ints in [0, r]
  std::vector<NodeClass> node_class;
  std::vector<PeriodicGroup> periodic_groups;
  int corner_group = -1;  // index into periodic_groups, -1 if absent
  bool full_fallback = false;
  double t_select_ms = 0.0;    // element selection + beta (device)
  double t_topology_ms = 0.0;  // node numbering + periodic groups (host)
  std::int64_t active_nodes = 0;  // torus nodes touched by an element (device count)

  size_t num_elements() const { return elements.size(); }
  size_t num_nodes() const { return node_coords.size(); }
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
// The reference's lattice topology (voxel.hpp:147-228): nodes numbered in order
// of first use over the sorted element list (hex corner order of
// element_stiffness), boundary nodes grouped by lattice position mod r, groups
// in increasing key order, each group's members in node order; the same group
// checks and error messages.  A dense (r+1)^3 lattice index replaces the
// reference's hash maps (same result, linear time).
inline void build_topology(VoxelMesh& m) {
  const int r = m.resolution;
  const size_t r1 = static_cast<size_t>(r) + 1;
  static const int off[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
  std::vector<std::int32_t> id(r1 * r1 * r1, -1);
  m.element_nodes.assign(m.elements.size() * 8, 0);
  m.node_coords.clear();
  m.node_coords.reserve(m.elements.size() + m.elements.size() / 4);
  for (size_t e = 0; e < m.elements.size(); ++e) {
    const Vec3i c = VoxelMesh::element_coords(m.elements[e], r);
    for (int n = 0; n < 8; ++n) {
      const int i = c[0] + off[n][0], j = c[1] + off[n][1], k = c[2] + off[n][2];
      std::int32_t& slot = id[(static_cast<size_t>(k) * r1 + j) * r1 + i];
      if (slot < 0) {
        slot = static_cast<std::int32_t>(m.node_coords.size());
        m.node_coords.emplace_back(i, j, k);
      }
      m.element_nodes[e * 8 + n] = static_cast<std::uint32_t>(slot);
    }
  }
  const size_t nn = m.node_coords.size();
  m.node_class.assign(nn, NodeClass::Interior);
  std::vector<std::pair<std::uint64_t, std::uint32_t>> boundary;  // (key mod r, node)
  for (size_t n = 0; n < nn; ++n) {
    const Vec3i& c = m.node_coords[n];
    int b = 0;
    for (int a = 0; a < 3; ++a) b += (c[a] == 0 || c[a] == r);
    m.node_class[n] = static_cast<NodeClass>(b);
    if (b == 0) continue;
    const std::uint64_t key =
        (static_cast<std::uint64_t>(c[2] % r) * r1 + static_cast<std::uint64_t>(c[1] % r)) * r1 + (c[0] % r);
    boundary.emplace_back(key, static_cast<std::uint32_t>(n));
  }
  std::sort(boundary.begin(), boundary.end());  // by key, members in node order
  m.periodic_groups.clear();
  m.corner_group = -1;
  for (size_t a = 0; a < boundary.size();) {
    size_t b = a;
    while (b < boundary.size() && boundary[b].first == boundary[a].first) ++b;
    PeriodicGroup g;
    bool found_master = false;
    for (size_t q = a; q < b; ++q) {
      const std::uint32_t n = boundary[q].second;
      const Vec3i& c = m.node_coords[n];
      const Vec3i delta(c[0] == r, c[1] == r, c[2] == r);
      if (delta == Vec3i::Zero()) {
        g.master = n;
        found_master = true;
      } else {
        g.slaves.emplace_back(n, delta);
      }
    }
    if (!found_master)
      throw SolverError("periodic group without master node: mesh is not periodically complete");
    int axes = 0;
    for (int d = 0; d < 3; ++d) axes += (m.node_coords[g.master][d] % r == 0);
    const size_t expect = size_t(1) << axes;
    if (b - a != expect)
      throw SolverError("periodic group has " + std::to_string(b - a) + " members, expected " +
                        std::to_string(expect));
    if (axes == 3) m.corner_group = static_cast<int>(m.periodic_groups.size());
    m.periodic_groups.push_back(std::move(g));
    a = b;
  }
}

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
  const auto t0 = std::chrono::steady_clock::now();
  detail::check(shl_build_reduced_mesh(ctx, &p, m.elements.data(), m.beta.data(), &n, &ff), ctx);
  const auto t1 = std::chrono::steady_clock::now();
  m.elements.resize(static_cast<size_t>(n));
  m.beta.resize(static_cast<size_t>(n));
  m.full_fallback = ff != 0;
  detail::build_topology(m);
  m.t_select_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  m.t_topology_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
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
  detail::build_topology(m);
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
