// geomio.hpp -- drop-in for the mesh half of
// /root/reference/proj/include/shellular/geomio.hpp
//
//   TriMesh (:18-39), extract_isosurface (:45-108) on the device
//   (shl_extract_isosurface: identical vertices, triangles and their order),
//   MeshFormat / export_mesh (:272-316) on the host (same bytes).
// Tiling (TileSpec / TileField, :112-265) and export_solid_voxels (:318-371)
// are outside the C^H hot path (SURVEY.md §8 f lists only the isosurface and
// the raw voxel export) and are not provided.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "voxel.hpp"

namespace shellular {

struct TriMesh {
  std::vector<Vec3> vertices;
  std::vector<std::array<std::uint32_t, 3>> triangles;

  double area() const {
    double a = 0.0;
    for (const auto& t : triangles) {
      Vec3 e1 = vertices[t[1]] - vertices[t[0]];
      Vec3 e2 = vertices[t[2]] - vertices[t[0]];
      a += 0.5 * e1.cross(e2).norm();
    }
    return a;
  }
  double signed_volume() const {
    double v = 0.0;
    for (const auto& t : triangles) v += vertices[t[0]].dot(vertices[t[1]].cross(vertices[t[2]])) / 6.0;
    return v;
  }
};

// Marching cubes on the zero level set of the corner samples (device).
inline TriMesh extract_isosurface(const FieldGrid& grid) {
  if (grid.degenerate()) throw DegenerateDesignError("cannot extract isosurface of a degenerate field");
  shl_ctx* ctx = detail::load_grid(grid);
  std::int64_t nv = 0, nt = 0;
  detail::check(shl_extract_isosurface(ctx, nullptr, 0, nullptr, 0, &nv, &nt), ctx);
  std::vector<double> v(static_cast<size_t>(nv) * 3);
  std::vector<std::uint32_t> t(static_cast<size_t>(nt) * 3);
  detail::check(shl_extract_isosurface(ctx, v.data(), nv, t.data(), nt, &nv, &nt), ctx);
  TriMesh m;
  m.vertices.reserve(static_cast<size_t>(nv));
  for (std::int64_t i = 0; i < nv; ++i) m.vertices.emplace_back(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  m.triangles.resize(static_cast<size_t>(nt));
  for (std::int64_t i = 0; i < nt; ++i) m.triangles[i] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
  return m;
}

enum class MeshFormat { StlBinary, Obj };

// Binary STL (80-byte header, uint32 count, 50 bytes per triangle: float
// normal, three float vertices, zero attribute) or OBJ with 17-digit vertices.
inline void export_mesh(const TriMesh& mesh, const std::string& path, MeshFormat format) {
  if (mesh.triangles.empty()) throw ValidationError("refusing to export an empty mesh");
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open '" + path + "' for writing");
  if (format == MeshFormat::StlBinary) {
    char header[80] = {};
    std::strncpy(header, "shellular voxel cell export", sizeof(header) - 1);
    out.write(header, sizeof(header));
    const std::uint32_t count = static_cast<std::uint32_t>(mesh.triangles.size());
    out.write(reinterpret_cast<const char*>(&count), sizeof(count));
    for (const auto& t : mesh.triangles) {
      const Vec3& a = mesh.vertices[t[0]];
      const Vec3& b = mesh.vertices[t[1]];
      const Vec3& c = mesh.vertices[t[2]];
      Vec3 n = (b - a).cross(c - a);
      const double len = n.norm();
      if (len > 0.0) n /= len;
      const float rec[12] = {float(n[0]), float(n[1]), float(n[2]), float(a[0]), float(a[1]), float(a[2]),
                             float(b[0]), float(b[1]), float(b[2]), float(c[0]), float(c[1]), float(c[2])};
      out.write(reinterpret_cast<const char*>(rec), sizeof(rec));
      const std::uint16_t attr = 0;
      out.write(reinterpret_cast<const char*>(&attr), sizeof(attr));
    }
  } else {
    out.precision(17);
    for (const auto& v : mesh.vertices) out << "v " << v[0] << ' ' << v[1] << ' ' << v[2] << '\n';
    for (const auto& t : mesh.triangles) out << "f " << t[0] + 1 << ' ' << t[1] + 1 << ' ' << t[2] + 1 << '\n';
  }
  if (!out) throw IoError("failed writing '" + path + "'");
}

}  // namespace shellular
