// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Thin C ABI over the reference's OWN field/voxel/geomio code
// (/root/reference/proj/include/shellular/{common,field,voxel,geomio}.hpp, included
// unmodified; Eigen replaced by oracle/ref_shim).  Built by `make -C oracle ref`
// into oracle/_ref/ and used only to generate / check tests/golden fixtures and
// to pin the C++ restatement in oracle/shellular_oracle.cpp.
#include "shellular/field.hpp"
#include "shellular/voxel.hpp"

// geomio.hpp uses hex_corner_offsets, defined in fem.hpp (fem.hpp:41-46), which
// needs Eigen's sparse module and cannot be compiled here; the same eight
// offsets are declared for it.
namespace shellular {
inline const std::array<Vec3i, 8>& hex_corner_offsets() {
  static const std::array<Vec3i, 8> off = {Vec3i(0, 0, 0), Vec3i(1, 0, 0), Vec3i(1, 1, 0), Vec3i(0, 1, 0),
                                           Vec3i(0, 0, 1), Vec3i(1, 0, 1), Vec3i(1, 1, 1), Vec3i(0, 1, 1)};
  return off;
}
}  // namespace shellular

#include "shellular/geomio.hpp"

#include <cstring>
#include <string>

using namespace shellular;

namespace {
thread_local std::string g_err;

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 1;
  } catch (const DegenerateDesignError& e) {
    g_err = e.what();
    return 2;
  } catch (const SolverError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

DesignParams make(int sym, int K, int n, const double* pos, const int* sign, const double* w) {
  DesignParams p;
  p.symmetry = static_cast<Symmetry>(sym);
  p.truncation = K;
  int m = K + 1;
  p.weights.assign(w, w + m * m * m);
  for (int i = 0; i < n; ++i) p.charges.emplace_back(Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]), sign[i]);
  return p;
}

FieldGrid grid_from(int r, const double* centres, const double* corners, double norm) {
  FieldGrid g;
  g.resolution = r;
  g.samples.assign(centres, centres + size_t(r) * r * r);
  g.corner_samples.assign(corners, corners + size_t(r + 1) * (r + 1) * (r + 1));
  g.norm = norm;
  return g;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_random_design(int sym, int n_pre, int K, double lo, double hi, std::uint64_t seed,
                      double* pos_out, int* sign_out, double* w_out) {
  return guard([&] {
    RandomDesignSpec spec;
    spec.symmetry = static_cast<Symmetry>(sym);
    spec.n_charges_pre_expansion = n_pre;
    spec.truncation = K;
    spec.weight_lo = lo;
    spec.weight_hi = hi;
    DesignParams p = random_design(spec, seed);
    for (size_t i = 0; i < p.charges.size(); ++i) {
      for (int a = 0; a < 3; ++a) pos_out[3 * i + a] = p.charges[i].position[a];
      sign_out[i] = p.charges[i].sign;
    }
    std::memcpy(w_out, p.weights.data(), p.weights.size() * sizeof(double));
  });
}

int ref_expand_symmetry(int sym, int K, int n, const double* pos, const int* sign, const double* w,
                        double* pos_out, int* sign_out, int* n_out) {
  return guard([&] {
    DesignParams e = expand_symmetry(make(sym, K, n, pos, sign, w));
    for (size_t i = 0; i < e.charges.size(); ++i) {
      for (int a = 0; a < 3; ++a) pos_out[3 * i + a] = e.charges[i].position[a];
      sign_out[i] = e.charges[i].sign;
    }
    *n_out = static_cast<int>(e.charges.size());
  });
}

int ref_field_value(int sym, int K, int n, const double* pos, const int* sign, const double* w,
                    int npts, const double* pts, double* out) {
  return guard([&] {
    FieldEvaluator ev(make(sym, K, n, pos, sign, w));
    for (int i = 0; i < npts; ++i) out[i] = ev.value(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
  });
}

int ref_sample_grid(int sym, int K, int n, const double* pos, const int* sign, const double* w,
                    int r, int threads, double* centres, double* corners, double* norm) {
  return guard([&] {
    FieldGrid g = sample_grid(make(sym, K, n, pos, sign, w), r, threads);
    std::memcpy(centres, g.samples.data(), g.samples.size() * sizeof(double));
    std::memcpy(corners, g.corner_samples.data(), g.corner_samples.size() * sizeof(double));
    *norm = g.norm;
  });
}

int ref_classify(int r, const double* centres, const double* corners, double norm,
                 std::uint32_t* out, std::int64_t* count) {
  return guard([&] {
    auto s = classify_surface_elements(grid_from(r, centres, corners, norm));
    std::memcpy(out, s.data(), s.size() * sizeof(std::uint32_t));
    *count = static_cast<std::int64_t>(s.size());
  });
}

// info: [n_elements, n_nodes, n_groups, corner_group, full_fallback, corner_group_size]
int ref_build_reduced_mesh(int r, const double* centres, const double* corners, double norm,
                           double sharpness, double floor_ratio, int expand_layers,
                           std::uint32_t* elements, double* beta, std::int64_t* info) {
  return guard([&] {
    ShellParams sp;
    sp.sharpness = sharpness;
    sp.floor_ratio = floor_ratio;
    sp.expand_layers = expand_layers;
    VoxelMesh m = build_reduced_mesh(grid_from(r, centres, corners, norm), sp);
    std::memcpy(elements, m.elements.data(), m.elements.size() * sizeof(std::uint32_t));
    std::memcpy(beta, m.beta.data(), m.beta.size() * sizeof(double));
    info[0] = static_cast<std::int64_t>(m.elements.size());
    info[1] = static_cast<std::int64_t>(m.num_nodes());
    info[2] = static_cast<std::int64_t>(m.periodic_groups.size());
    info[3] = m.corner_group;
    info[4] = m.full_fallback ? 1 : 0;
    info[5] = m.corner_group >= 0 ? 1 + static_cast<std::int64_t>(m.periodic_groups[m.corner_group].slaves.size()) : 0;
  });
}

int ref_step_function(double v, double sharpness, double floor_ratio, double* out) {
  return guard([&] {
    ShellParams sp;
    sp.sharpness = sharpness;
    sp.floor_ratio = floor_ratio;
    *out = step_function(v, sp);
  });
}

// extract_isosurface (geomio.hpp:45-108); counts always, arrays when they fit
int ref_extract_isosurface(int r, const double* centres, const double* corners, double norm,
                           double* verts, std::int64_t vcap, std::uint32_t* tris, std::int64_t tcap,
                           std::int64_t* nv, std::int64_t* nt) {
  return guard([&] {
    TriMesh m = extract_isosurface(grid_from(r, centres, corners, norm));
    *nv = static_cast<std::int64_t>(m.vertices.size());
    *nt = static_cast<std::int64_t>(m.triangles.size());
    if (static_cast<std::int64_t>(m.vertices.size()) <= vcap)
      for (size_t i = 0; i < m.vertices.size(); ++i)
        for (int a = 0; a < 3; ++a) verts[3 * i + a] = m.vertices[i][a];
    if (static_cast<std::int64_t>(m.triangles.size()) <= tcap)
      for (size_t i = 0; i < m.triangles.size(); ++i)
        for (int a = 0; a < 3; ++a) tris[3 * i + a] = m.triangles[i][a];
  });
}

// VoxelMesh::write_raw (voxel.hpp:105-114) of build_reduced_mesh
int ref_write_raw(int r, const double* centres, const double* corners, double norm, double sharpness,
                  double floor_ratio, int expand_layers, const char* path) {
  return guard([&] {
    ShellParams sp;
    sp.sharpness = sharpness;
    sp.floor_ratio = floor_ratio;
    sp.expand_layers = expand_layers;
    build_reduced_mesh(grid_from(r, centres, corners, norm), sp).write_raw(path);
  });
}

// export_mesh (geomio.hpp:277-316); format 0 = binary STL, 1 = OBJ
int ref_export_mesh(const double* verts, std::int64_t nv, const std::uint32_t* tris, std::int64_t nt,
                    const char* path, int format) {
  return guard([&] {
    TriMesh m;
    for (std::int64_t i = 0; i < nv; ++i) m.vertices.emplace_back(verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]);
    for (std::int64_t i = 0; i < nt; ++i) m.triangles.push_back({tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]});
    export_mesh(m, path, format == 0 ? MeshFormat::StlBinary : MeshFormat::Obj);
  });
}

}  // extern "C"
