// test_dropin.cpp -- the reference's Catch2 hot-path tests (proj/tests/
// test_field.cpp, test_voxel.cpp, test_fem.cpp), restated against the C++
// drop-in headers include/shellular/*.hpp.  A minimal harness replaces
// Catch2 (absent).  Cases that need Eigen's eigen-solver or the sparse
// master-slave internals are covered in Python (tests/test_oracle_fem.py).
//
//   ./test_dropin            host + device cases (needs a GPU)
//   ./test_dropin --host     host-only cases (reference arithmetic in the
//                            library, no device work)
#include <cstdio>
#include <cstring>
#include <functional>
#include <set>
#include <string>
#include <vector>

#include "shellular/geomio.hpp"
#include "shellular/pipeline.hpp"

using namespace shellular;

namespace {

int g_checks = 0, g_failed = 0;
std::string g_case;

#define CHECK(cond)                                                                     \
  do {                                                                                  \
    ++g_checks;                                                                         \
    if (!(cond)) {                                                                      \
      ++g_failed;                                                                       \
      std::fprintf(stderr, "FAILED [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                   \
  } while (0)

#define CHECK_THROWS_AS(expr, type)   \
  do {                                \
    bool thrown_ = false;             \
    try {                             \
      (void)(expr);                   \
    } catch (const type&) {           \
      thrown_ = true;                 \
    } catch (...) {                   \
    }                                 \
    CHECK(thrown_ && #type);          \
  } while (0)

struct Case {
  const char* name;
  bool device;
  std::function<void()> fn;
};
std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, bool d, std::function<void()> f) { registry().push_back({n, d, std::move(f)}); }
};
#define HOST_CASE(id, name) \
  static void id();         \
  static Reg reg_##id(name, false, id); \
  static void id()
#define DEVICE_CASE(id, name) \
  static void id();           \
  static Reg reg_##id(name, true, id); \
  static void id()

bool approx(double a, double b, double rel, double abs_ = 0.0) {
  return std::abs(a - b) <= std::max(abs_, rel * std::max(std::abs(a), std::abs(b)));
}
double rel_diff(const Mat6& a, const Mat6& b) {
  return (a - b).cwiseAbs().maxCoeff() / b.cwiseAbs().maxCoeff();
}

DesignParams seeded_random(Symmetry sym, int n_pre, std::uint64_t seed) {
  RandomDesignSpec spec;
  spec.symmetry = sym;
  spec.n_charges_pre_expansion = n_pre;
  spec.truncation = 2;
  return random_design(spec, seed);
}
DesignParams seeded_design(std::uint64_t seed) { return seeded_random(Symmetry::CubicOctant, 4, seed); }

DesignParams plane_design(int axis, double shift) {  // test_voxel.cpp:15-24
  DesignParams p;
  p.symmetry = Symmetry::None;
  p.truncation = 2;
  p.weights.assign(27, 0.0);
  int h = axis == 0, k = axis == 1, l = axis == 2;
  p.weight(h, k, l) = 1.0;
  Vec3 a(0.5, 0.5, 0.5), b(0.5, 0.5, 0.5);
  a[axis] = 0.25 + shift;
  b[axis] = 0.75 + shift;
  p.charges.emplace_back(a, 1);
  p.charges.emplace_back(b, -1);
  return p;
}

// oracles.hpp:22-41 direct triple-loop Eq. 5
double direct_field_sum(const DesignParams& expanded, const Vec3& p) {
  double total = 0.0;
  int K = expanded.truncation;
  for (const auto& c : expanded.charges)
    for (int h = 0; h <= K; ++h)
      for (int k = 0; k <= K; ++k)
        for (int l = 0; l <= K; ++l) {
          if (!h && !k && !l) continue;
          int zeros = (h == 0) + (k == 0) + (l == 0);
          double w = zeros == 1 ? 0.5 : (zeros == 2 ? 0.25 : 1.0);
          double b = std::cos(2.0 * M_PI * h * (p[0] - c.position[0])) *
                     std::cos(2.0 * M_PI * k * (p[1] - c.position[1])) *
                     std::cos(2.0 * M_PI * l * (p[2] - c.position[2])) / double(h * h + k * k + l * l);
          total += c.sign * expanded.weight(h, k, l) * w * b;
        }
  return total;
}

// test_voxel.cpp:35-96 independent full-grid re-implementation
std::set<std::uint32_t> scan_oracle_elements(const FieldGrid& grid, const ShellParams& sp) {
  int r = grid.resolution;
  size_t total = size_t(r) * r * r;
  std::vector<std::uint8_t> in(total, 0);
  for (int k = 0; k < r; ++k)
    for (int j = 0; j < r; ++j)
      for (int i = 0; i < r; ++i) {
        int pos = 0, neg = 0, zero = 0;
        for (int d = 0; d < 8; ++d) {
          double v = grid.corner(i + (d & 1), j + ((d >> 1) & 1), k + ((d >> 2) & 1));
          (v > 0 ? pos : v < 0 ? neg : zero) = 1;
        }
        if (zero || (pos && neg)) in[VoxelMesh::element_id(i, j, k, r)] = 1;
      }
  for (int layer = 0; layer < sp.layers_for(r); ++layer) {
    std::vector<std::uint8_t> next = in;
    for (int k = 0; k < r; ++k)
      for (int j = 0; j < r; ++j)
        for (int i = 0; i < r; ++i) {
          if (in[VoxelMesh::element_id(i, j, k, r)]) continue;
          bool near = in[VoxelMesh::element_id((i + 1) % r, j, k, r)] ||
                      in[VoxelMesh::element_id((i + r - 1) % r, j, k, r)] ||
                      in[VoxelMesh::element_id(i, (j + 1) % r, k, r)] ||
                      in[VoxelMesh::element_id(i, (j + r - 1) % r, k, r)] ||
                      in[VoxelMesh::element_id(i, j, (k + 1) % r, r)] ||
                      in[VoxelMesh::element_id(i, j, (k + r - 1) % r, r)];
          if (near) next[VoxelMesh::element_id(i, j, k, r)] = 1;
        }
    in = std::move(next);
  }
  std::set<std::uint32_t> out;
  for (size_t e = 0; e < total; ++e)
    if (in[e]) out.insert(std::uint32_t(e));
  bool changed = true;
  while (changed) {
    changed = false;
    std::set<std::uint32_t> add;
    for (auto e : out) {
      Vec3i c = VoxelMesh::element_coords(e, r);
      for (int a = 0; a < 3; ++a)
        if (c[a] == 0 || c[a] == r - 1) {
          Vec3i q = c;
          q[a] = (c[a] == 0) ? r - 1 : 0;
          add.insert(VoxelMesh::element_id(q[0], q[1], q[2], r));
        }
    }
    for (auto e : add)
      if (out.insert(e).second) changed = true;
  }
  bool touches = false;
  for (auto e : out) {
    Vec3i c = VoxelMesh::element_coords(e, r);
    for (int a = 0; a < 3; ++a)
      if (c[a] == 0 || c[a] == r - 1) touches = true;
  }
  if (touches)
    for (int i : {0, r - 1})
      for (int j : {0, r - 1})
        for (int k : {0, r - 1}) out.insert(VoxelMesh::element_id(i, j, k, r));
  return out;
}

}  // namespace

// ============================ host cases ====================================
HOST_CASE(basis_weight_rule, "basis_weight follows the zero-index rule") {
  CHECK(basis_weight(1, 0, 0) == 0.25);
  CHECK(basis_weight(0, 0, 2) == 0.25);
  CHECK(basis_weight(1, 1, 0) == 0.5);
  CHECK(basis_weight(1, 2, 1) == 1.0);
  CHECK_THROWS_AS(basis_weight(0, 0, 0), ValidationError);
}

HOST_CASE(plane_antisymmetry, "mirror-antisymmetric two-charge design vanishes on x=0.5") {
  DesignParams p;
  p.symmetry = Symmetry::None;
  p.truncation = 2;
  p.weights.assign(27, 1.0);
  p.weights[0] = 0.0;
  p.charges.emplace_back(Vec3(0.25, 0.5, 0.5), 1);
  p.charges.emplace_back(Vec3(0.75, 0.5, 0.5), -1);
  FieldEvaluator ev(p);
  for (double y : {0.0, 0.31, 0.77})
    for (double z : {0.13, 0.5, 0.9}) CHECK(std::abs(ev.value(Vec3(0.5, y, z))) < 1e-12);
}

HOST_CASE(periodic, "field is periodic in every axis") {
  FieldEvaluator ev(seeded_random(Symmetry::None, 6, 991));
  Rng rng(7);
  for (int t = 0; t < 50; ++t) {
    Vec3 q(rng.uniform01(), rng.uniform01(), rng.uniform01());
    Vec3 shift(rng.uniform_int(-2, 2), rng.uniform_int(-2, 2), rng.uniform_int(-2, 2));
    double f0 = ev.value(q), f1 = ev.value(q + shift);
    CHECK(std::abs(f1 - f0) <= 1e-12 * std::max(1.0, std::abs(f0)));
  }
}

HOST_CASE(negate, "negating all signs negates the field") {
  DesignParams p = seeded_random(Symmetry::CubicOctant, 4, 55), f = p;
  for (auto& c : f.charges) c.sign = -c.sign;
  FieldEvaluator a(p), b(f);
  Rng rng(3);
  for (int t = 0; t < 20; ++t) {
    Vec3 q(rng.uniform01(), rng.uniform01(), rng.uniform01());
    CHECK(std::abs(a.value(q) + b.value(q)) < 1e-12 * std::max(1.0, std::abs(a.value(q))));
  }
}

HOST_CASE(evaluator_vs_direct, "evaluator matches the direct-summation oracle") {
  for (auto sym : {Symmetry::None, Symmetry::CubicOctant, Symmetry::Tetrahedral}) {
    DesignParams p = seeded_random(sym, 4, 1234 + int(sym));
    FieldEvaluator ev(p);
    DesignParams ex = expand_symmetry(p);
    Rng rng(99);
    for (int t = 0; t < 30; ++t) {
      Vec3 q(rng.uniform01(), rng.uniform01(), rng.uniform01());
      double want = direct_field_sum(ex, q);
      CHECK(std::abs(ev.value(q) - want) <= 1e-12 * std::max(1.0, std::abs(want)));
    }
  }
}

HOST_CASE(octant_expansion, "cubic octant expansion produces 8 images per charge") {
  DesignParams p;
  p.symmetry = Symmetry::CubicOctant;
  p.truncation = 2;
  p.weights.assign(27, 0.0);
  p.weights[1] = 1.0;
  p.charges.emplace_back(Vec3(0.2, 0.3, 0.1), 1);
  p.charges.emplace_back(Vec3(0.4, 0.1, 0.45), -1);
  DesignParams full = expand_symmetry(p);
  CHECK(full.charges.size() == 16);
  int plus = 0;
  for (const auto& c : full.charges) plus += c.sign == 1;
  CHECK(plus == 8);
  CHECK(full.symmetry == Symmetry::None);
}

HOST_CASE(identity_expansion, "expansion with symmetry None is the identity") {
  DesignParams p = seeded_random(Symmetry::None, 4, 5);
  DesignParams full = expand_symmetry(p);
  CHECK(full.charges.size() == p.charges.size());
  for (size_t i = 0; i < p.charges.size(); ++i) CHECK(full.charges[i].position == p.charges[i].position);
}

HOST_CASE(tetra_count, "tetrahedral orbit has 48 images per charge") {
  DesignParams p;
  p.symmetry = Symmetry::Tetrahedral;
  p.truncation = 2;
  p.weights.assign(27, 0.0);
  p.weights[1] = 1.0;
  p.charges.emplace_back(Vec3(0.3, 0.2, 0.1), 1);
  p.charges.emplace_back(Vec3(0.45, 0.25, 0.05), -1);
  CHECK(expand_symmetry(p).charges.size() == 96);
}

HOST_CASE(fbv_reject, "expansion rejects charges outside the fundamental volume") {
  DesignParams p;
  p.symmetry = Symmetry::CubicOctant;
  p.truncation = 2;
  p.weights.assign(27, 0.0);
  p.weights[1] = 1.0;
  p.charges.emplace_back(Vec3(0.7, 0.2, 0.2), 1);
  p.charges.emplace_back(Vec3(0.1, 0.1, 0.1), -1);
  CHECK_THROWS_AS(expand_symmetry(p), ValidationError);
}

HOST_CASE(random_det, "random designs are deterministic and well formed") {
  RandomDesignSpec spec;
  spec.symmetry = Symmetry::CubicOctant;
  spec.n_charges_pre_expansion = 2;
  DesignParams a = random_design(spec, 42), b = random_design(spec, 42);
  CHECK(a.charges.size() == 2);
  for (size_t i = 0; i < a.charges.size(); ++i) CHECK(a.charges[i].position == b.charges[i].position);
  CHECK(a.weights == b.weights);
  spec.symmetry = Symmetry::None;
  spec.n_charges_pre_expansion = 64;
  DesignParams c = random_design(spec, 1);
  int plus = 0;
  for (const auto& ch : c.charges) plus += ch.sign == 1;
  CHECK(c.charges.size() == 64 && plus == 32);
  CHECK_THROWS_AS(random_design(RandomDesignSpec{Symmetry::None, 3}, 1), ValidationError);
}

HOST_CASE(random_fbv, "random draws stay inside the fundamental volume and weight range") {
  for (auto sym : {Symmetry::None, Symmetry::CubicOctant, Symmetry::Tetrahedral}) {
    RandomDesignSpec spec;
    spec.symmetry = sym;
    spec.n_charges_pre_expansion = 4;
    spec.weight_lo = -0.5;
    spec.weight_hi = 2.0;
    for (std::uint64_t seed = 0; seed < 250; ++seed) {
      DesignParams p = random_design(spec, seed);
      for (const auto& c : p.charges) CHECK(in_fundamental_volume(sym, c.position));
      for (size_t w = 1; w < p.weights.size(); ++w) CHECK(p.weights[w] >= -0.5 && p.weights[w] <= 2.0);
    }
  }
}

HOST_CASE(step_anchor, "step function hits its anchor values") {
  ShellParams sp;
  CHECK(approx(step_function(0.0, sp), 1.0, 0.0, 1e-15));
  CHECK(approx(step_function(10.0, sp), 1e-3, 0.0, 1e-9));
  CHECK(approx(step_function(-10.0, sp), 1e-3, 0.0, 1e-9));
}

HOST_CASE(shell_validation, "shell parameter validation") {
  ShellParams sp;
  sp.floor_ratio = 1.5;
  CHECK_THROWS_AS(sp.validate(), ValidationError);
  sp.floor_ratio = 0.5;
  sp.sharpness = -1.0;
  CHECK_THROWS_AS(sp.validate(), ValidationError);
  CHECK(ShellParams{}.layers_for(64) == 2);
  CHECK(ShellParams{}.layers_for(32) == 1);
  CHECK(ShellParams{}.layers_for(8) == 1);
}

HOST_CASE(k0_rigid, "element stiffness annihilates rigid modes and is symmetric") {
  ElementStiffness K = element_stiffness(BaseMaterial{}, 0.25);
  double scale = K.matrix.cwiseAbs().maxCoeff();
  Matrix<double, 24, 1> t, rot;
  Vec3 w(0.2, -0.5, 1.0);
  const auto& off = hex_corner_offsets();
  for (int n = 0; n < 8; ++n) {
    Vec3 tr(0.3, -1.2, 0.7), ro = w.cross(off[n].cast<double>() * 0.25);
    for (int a = 0; a < 3; ++a) {
      t[3 * n + a] = tr[a];
      rot[3 * n + a] = ro[a];
    }
  }
  CHECK((K.matrix * t).cwiseAbs().maxCoeff() < 1e-12 * scale);
  CHECK((K.matrix * rot).cwiseAbs().maxCoeff() < 1e-12 * scale);
  CHECK((K.matrix - K.matrix.transpose()).cwiseAbs().maxCoeff() < 1e-12 * scale);
}

HOST_CASE(k0_scale, "element stiffness scales linearly with the edge") {
  BaseMaterial mat;
  mat.poisson = 0.25;
  Mat24 k1 = element_stiffness(mat, 1.0).matrix, kh = element_stiffness(mat, 0.5).matrix;
  CHECK((kh - 0.5 * k1).cwiseAbs().maxCoeff() < 1e-12 * k1.cwiseAbs().maxCoeff());
}

HOST_CASE(material_validation, "material validation") {
  BaseMaterial bad;
  bad.poisson = 0.5;
  CHECK_THROWS_AS(element_stiffness(bad, 1.0), ValidationError);
  bad.poisson = 0.3;
  bad.youngs = -1.0;
  CHECK_THROWS_AS(element_stiffness(bad, 1.0), ValidationError);
}

// =========================== device cases ===================================
DEVICE_CASE(grid_vs_pointwise, "grid sampling agrees with pointwise evaluation") {
  DesignParams p = seeded_random(Symmetry::CubicOctant, 4, 808);
  FieldGrid grid = sample_grid(p, 16);
  FieldEvaluator ev(p);
  Rng rng(2);
  for (int t = 0; t < 40; ++t) {
    int i = rng.uniform_int(0, 15), j = rng.uniform_int(0, 15), k = rng.uniform_int(0, 15);
    double want = ev.value(Vec3((i + 0.5) / 16.0, (j + 0.5) / 16.0, (k + 0.5) / 16.0));
    CHECK(std::abs(grid.center(i, j, k) - want) < 1e-12 * std::max(1.0, std::abs(want)));
    double wantc = ev.value(Vec3(i / 16.0, j / 16.0, k / 16.0));
    CHECK(std::abs(grid.corner(i, j, k) - wantc) < 1e-12 * std::max(1.0, std::abs(wantc)));
  }
  CHECK(grid.norm > 0.0 && !grid.degenerate());
}

DEVICE_CASE(zero_weights, "all-zero weights give a degenerate grid") {
  DesignParams p = seeded_random(Symmetry::None, 4, 11);
  std::fill(p.weights.begin(), p.weights.end(), 0.0);
  FieldGrid grid = sample_grid(p, 8);
  CHECK(grid.norm == 0.0 && grid.degenerate());
}

DEVICE_CASE(corner_closure, "corner samples close periodically") {
  FieldGrid grid = sample_grid(seeded_random(Symmetry::None, 4, 21), 8);
  for (int a = 0; a <= 8; ++a)
    for (int b = 0; b <= 8; ++b) {
      CHECK(grid.corner(8, a, b) == grid.corner(0, a % 8, b % 8));
      CHECK(grid.corner(a, 8, b) == grid.corner(a % 8, 0, b % 8));
    }
}

DEVICE_CASE(plane_slabs, "plane design classifies as two single-voxel slabs") {
  int r = 32;
  auto surf = classify_surface_elements(sample_grid(plane_design(2, 0.5 / r), r));
  CHECK(surf.size() == size_t(2 * r * r));
  std::set<int> layers;
  for (auto e : surf) layers.insert(VoxelMesh::element_coords(e, r)[2]);
  CHECK(layers.size() == 2);
}

DEVICE_CASE(no_surface, "all-positive field has no surface") {
  FieldGrid grid = sample_grid_fn([](const Vec3&) { return 1.0; }, 8);
  CHECK(classify_surface_elements(grid).empty());
  CHECK_THROWS_AS(build_reduced_mesh(grid, ShellParams{}), DegenerateDesignError);
}

DEVICE_CASE(schwarz_p, "schwarz-p classification matches the brute corner scan") {
  auto f = [](const Vec3& q) { return std::cos(2 * M_PI * q[0]) + std::cos(2 * M_PI * q[1]) + std::cos(2 * M_PI * q[2]); };
  int r = 32;
  FieldGrid grid = sample_grid_fn(f, r);
  auto surf = classify_surface_elements(grid);
  std::set<std::uint32_t> got(surf.begin(), surf.end()), want;
  for (int k = 0; k < r; ++k)
    for (int j = 0; j < r; ++j)
      for (int i = 0; i < r; ++i) {
        double mn = 1e300, mx = -1e300;
        for (int d = 0; d < 8; ++d) {
          double v = grid.corner(i + (d & 1), j + ((d >> 1) & 1), k + ((d >> 2) & 1));
          mn = std::min(mn, v);
          mx = std::max(mx, v);
        }
        if (mn <= 0.0 && mx >= 0.0) want.insert(VoxelMesh::element_id(i, j, k, r));
      }
  CHECK(got == want);
}

DEVICE_CASE(scan_oracle, "reduced mesh matches the independent scan oracle") {
  ShellParams sp;
  for (std::uint64_t seed : {3u, 12u}) {
    FieldGrid grid = sample_grid(seeded_design(seed), 16);
    VoxelMesh mesh = build_reduced_mesh(grid, sp);
    std::set<std::uint32_t> got(mesh.elements.begin(), mesh.elements.end());
    CHECK(got == scan_oracle_elements(grid, sp));
  }
  sp.expand_layers = 2;
  FieldGrid grid = sample_grid(seeded_design(2024), 64);
  VoxelMesh mesh = build_reduced_mesh(grid, sp);
  CHECK(mesh.element_fraction() >= 0.03 && mesh.element_fraction() <= 0.35);
  std::set<std::uint32_t> got(mesh.elements.begin(), mesh.elements.end());
  CHECK(got == scan_oracle_elements(grid, sp));
}

DEVICE_CASE(dilation_monotone, "dilation grows monotonically with the layer count") {
  FieldGrid grid = sample_grid(seeded_design(8), 16);
  ShellParams sp1, sp2;
  sp1.expand_layers = 1;
  sp2.expand_layers = 3;
  VoxelMesh m1 = build_reduced_mesh(grid, sp1), m2 = build_reduced_mesh(grid, sp2);
  std::set<std::uint32_t> s2(m2.elements.begin(), m2.elements.end());
  for (auto e : m1.elements) CHECK(s2.count(e) == 1);
}

DEVICE_CASE(completion, "completion is a fixpoint") {
  VoxelMesh mesh = build_reduced_mesh(sample_grid(seeded_design(21), 16), ShellParams{});
  int r = mesh.resolution;
  std::set<std::uint32_t> present(mesh.elements.begin(), mesh.elements.end());
  for (auto e : mesh.elements) {
    Vec3i c = VoxelMesh::element_coords(e, r);
    for (int a = 0; a < 3; ++a)
      if (c[a] == 0 || c[a] == r - 1) {
        Vec3i q = c;
        q[a] = (c[a] == 0) ? r - 1 : 0;
        CHECK(present.count(VoxelMesh::element_id(q[0], q[1], q[2], r)) == 1);
      }
  }
  for (int i : {0, r - 1})
    for (int j : {0, r - 1})
      for (int k : {0, r - 1}) CHECK(present.count(VoxelMesh::element_id(i, j, k, r)) == 1);
}

DEVICE_CASE(beta_bounds, "beta stays inside its bounds") {
  ShellParams sp;
  VoxelMesh mesh = build_reduced_mesh(sample_grid(seeded_design(77), 16), sp);
  for (double b : mesh.beta) CHECK(b >= sp.floor_ratio && b <= 1.0);
  CHECK(mesh.volume_ratio() > 0.0 && mesh.volume_ratio() <= 1.0);
}

DEVICE_CASE(full_fallback, "full fallback mesh is flagged") {
  ShellParams sp;
  sp.expand_layers = 8;
  VoxelMesh mesh = build_reduced_mesh(sample_grid(seeded_design(5), 8), sp);
  CHECK(mesh.full_fallback && mesh.elements.size() == 512);
  CHECK(full_solid_mesh(8).full_fallback);
}

DEVICE_CASE(raw_export, "raw export writes one byte per voxel") {
  VoxelMesh mesh = build_reduced_mesh(sample_grid(seeded_design(9), 8), ShellParams{});
  std::string path = "voxel_test_export.raw";
  mesh.write_raw(path);
  std::FILE* f = std::fopen(path.c_str(), "rb");
  CHECK(f != nullptr);
  std::vector<unsigned char> bytes(600);
  size_t n = std::fread(bytes.data(), 1, bytes.size(), f);
  std::fclose(f);
  std::remove(path.c_str());
  CHECK(n == 512);
  size_t nonzero = 0;
  for (size_t i = 0; i < n; ++i) nonzero += bytes[i] != 0;
  CHECK(nonzero == mesh.elements.size());
}

DEVICE_CASE(isotropic, "full solid homogenization reproduces the base isotropic tensor") {
  int r = 4;
  BaseMaterial mat;
  ElasticTensor C = effective_tensor(full_solid_mesh(r), element_stiffness(mat, 1.0 / r), {1e-12});
  ElasticTensor iso = ElasticTensor::isotropic(mat);
  CHECK(rel_diff(C.c, iso.c) < 1e-6);
  CHECK(approx(iso.c(0, 0), 1.34615384615, 1e-9));
  CHECK(approx(iso.c(0, 1), 0.57692307692, 1e-9));
  CHECK(approx(iso.c(3, 3), 0.38461538461, 1e-9));
}

DEVICE_CASE(laminate, "layered beta profile matches the exact laminate constants") {
  int r = 8;
  BaseMaterial mat;
  std::vector<double> layer = {1.0, 0.4, 1e-3, 0.02, 1.0, 0.7, 1e-3, 0.15};
  VoxelMesh mesh = full_solid_mesh(r);
  for (size_t e = 0; e < mesh.elements.size(); ++e) mesh.beta[e] = layer[VoxelMesh::element_coords(mesh.elements[e], r)[2]];
  ElasticTensor C = effective_tensor(mesh, element_stiffness(mat, 1.0 / r), {1e-12});
  // oracles.hpp:143-161
  double la = mat.lambda(), mu = mat.mu();
  auto mean = [&](auto f) {
    double s = 0.0;
    for (double b : layer) s += f(b * la, b * mu);
    return s / double(layer.size());
  };
  double inv_a = mean([](double l, double m) { return 1.0 / (l + 2 * m); });
  double loa = mean([](double l, double m) { return l / (l + 2 * m); });
  double C33 = 1.0 / inv_a, C13 = loa * C33;
  double C11 = mean([](double l, double m) { return 4 * m * (l + m) / (l + 2 * m); }) + loa * loa * C33;
  double C12 = mean([](double l, double m) { return 2 * m * l / (l + 2 * m); }) + loa * loa * C33;
  double C44 = 1.0 / mean([](double, double m) { return 1.0 / m; });
  double C66 = mean([](double, double m) { return m; });
  CHECK(approx(C.c(0, 0), C11, 1e-8));
  CHECK(approx(C.c(1, 1), C11, 1e-8));
  CHECK(approx(C.c(0, 1), C12, 1e-8));
  CHECK(approx(C.c(0, 2), C13, 1e-8));
  CHECK(approx(C.c(2, 2), C33, 1e-8));
  CHECK(approx(C.c(3, 3), C44, 1e-8));
  CHECK(approx(C.c(4, 4), C44, 1e-8));
  CHECK(approx(C.c(5, 5), C66, 1e-8));
}

DEVICE_CASE(grid_solver_api, "GridSolver keeps the reference signature and result fields") {
  int r = 8;
  Rng rng(31);
  std::vector<double> beta(size_t(r) * r * r);
  for (auto& b : beta) b = rng.uniform(0.05, 1.0);
  ElementStiffness K0 = element_stiffness(BaseMaterial{}, 1.0 / r);
  GridSolver solver(beta, r, K0);
  GridSolver::Result res = solver.solve(1e-11);
  for (int s = 0; s < 6; ++s) CHECK(res.iterations[s] > 0);
  CHECK(res.tensor.c(0, 0) > 0.0 && res.t_solve_ms > 0.0);
  CHECK_THROWS_AS(GridSolver(std::vector<double>(10, 1.0), r, K0), ValidationError);
}

DEVICE_CASE(modulus_scaling, "tensor scales exactly with the base modulus") {
  VoxelMesh mesh = build_reduced_mesh(sample_grid(seeded_design(21), 8), ShellParams{});
  BaseMaterial m1, m3;
  m3.youngs = 3.0;
  ElasticTensor c1 = effective_tensor(mesh, element_stiffness(m1, 1.0 / 8), {1e-12});
  ElasticTensor c3 = effective_tensor(mesh, element_stiffness(m3, 1.0 / 8), {1e-12});
  CHECK(rel_diff(c3.c, 3.0 * c1.c) < 1e-10);
}

DEVICE_CASE(homogenize_composition, "homogenize composes the stages and reports timings") {
  HomogenizationResult res = homogenize(seeded_design(5), ShellParams{}, BaseMaterial{}, 8);
  CHECK(res.tensor.c.cwiseAbs().maxCoeff() > 0.0);
  CHECK(res.volume_ratio > 0.0 && res.timings.t_fwd > 0.0);
  CHECK(res.mesh.full_fallback);  // r=8: one-layer dilation covers the cell
  HomogenizationResult res16 = homogenize(seeded_design(5), ShellParams{}, BaseMaterial{}, 16);
  CHECK(!res16.mesh.full_fallback);
  std::string j = res.to_json();
  for (const char* key : {"t_field", "t_mesh", "t_PBC", "t_AS", "t_RHS", "t_solve", "t_C", "t_fwd"})
    CHECK(j.find(key) != std::string::npos);
  DesignParams degenerate = seeded_design(5);
  std::fill(degenerate.weights.begin(), degenerate.weights.end(), 0.0);
  CHECK_THROWS_AS(homogenize(degenerate, ShellParams{}, BaseMaterial{}, 8), DegenerateDesignError);
  CHECK_THROWS_AS(homogenize(seeded_design(5), ShellParams{}, BaseMaterial{}, 3), ValidationError);
}

DEVICE_CASE(reduced_mesh_topology, "reduced mesh topology matches the reference's build_topology") {
  // node / periodic-group counts of the reference's own build_topology
  // (voxel.hpp:147-228) for these designs: tests/golden/reference_fixtures.npz
  // ("<name>/r<r>/info", written from oracle/_ref by make_golden.py)
  struct Want {
    std::uint64_t seed;
    int r;
    size_t nodes, groups;
  };
  for (const Want& w : {Want{3, 16, 3862, 544}, Want{12, 16, 3640, 416}}) {
    VoxelMesh m = build_reduced_mesh(sample_grid(seeded_design(w.seed), w.r), ShellParams{});
    CHECK(m.num_nodes() == w.nodes);
    CHECK(m.periodic_groups.size() == w.groups);
    CHECK(m.corner_group == 0 && m.periodic_groups[0].slaves.size() == 7);
    CHECK(m.element_nodes.size() == 8 * m.num_elements());
    for (size_t e = 0; e < m.num_elements(); ++e) {
      const Vec3i c = VoxelMesh::element_coords(m.elements[e], w.r);
      CHECK(m.node_coords[m.element_nodes[e * 8]] == c);
      CHECK(m.node_coords[m.element_nodes[e * 8 + 6]] == Vec3i(c[0] + 1, c[1] + 1, c[2] + 1));
    }
  }
  // the drop-in homogenize fills the grid and mesh like the reference (pipeline.hpp:70,74)
  HomogenizationResult res = homogenize(seeded_design(3), ShellParams{}, BaseMaterial{}, 16);
  CHECK(res.grid.samples.size() == size_t(16 * 16 * 16) && res.mesh.num_nodes() == 3862);
  CHECK(res.mesh.element_fraction() == res.element_fraction);
  // GridCG on a reduced mesh: the reference's SolverError (pipeline.hpp:86-88)
  HomogenizeOptions o;
  o.solver = SolverKind::GridCG;
  CHECK_THROWS_AS(homogenize(seeded_design(3), ShellParams{}, BaseMaterial{}, 16, o), SolverError);
  CHECK(res.stats.n_components >= 1 && res.stats.n_floating >= 0);
}

DEVICE_CASE(orthotropic, "plane design homogenizes to an orthotropic tensor") {
  DesignParams p = plane_design(2, 0.0);
  ShellParams sp;
  sp.sharpness = 100.0;
  HomogenizationResult res = homogenize(p, sp, BaseMaterial{}, 16);
  double c11 = res.tensor.c(0, 0);
  for (int i = 0; i < 3; ++i)
    for (int j = 3; j < 6; ++j) CHECK(std::abs(res.tensor.c(i, j)) < 1e-6 * c11);
}

DEVICE_CASE(void_floor, "void-dominant design stays under the floor bound") {
  ShellParams sp;
  sp.sharpness = 120.0;
  FieldGrid grid = sample_grid(plane_design(2, 0.0), 16);
  VoxelMesh mesh = full_field_mesh(grid, sp);
  ElasticTensor C = effective_tensor(mesh, element_stiffness(BaseMaterial{}, 1.0 / 16));
  CHECK(C.c.cwiseAbs().maxCoeff() <= 1e-2 * ElasticTensor::isotropic(BaseMaterial{}).c(0, 0));
}

DEVICE_CASE(self_convergence, "self convergence between r=8 and r=16") {
  HomogenizationResult a = homogenize(seeded_design(77), ShellParams{}, BaseMaterial{}, 8);
  HomogenizationResult b = homogenize(seeded_design(77), ShellParams{}, BaseMaterial{}, 16);
  CHECK(rel_diff(a.tensor.c, b.tensor.c) < 0.6);
}

// ---- geomio (SPEC.md geomio examples; geomio.hpp:45-108, :272-316) ----------
DEVICE_CASE(mc_sphere_area, "sphere-field isosurface area within 2% of analytic at r=64") {
  const double R = 0.3;
  FieldGrid grid = sample_grid_fn(
      [R](const Vec3& p) {
        Vec3 d = p - Vec3(0.5, 0.5, 0.5);
        return d.squaredNorm() - R * R;
      },
      64);
  TriMesh m = extract_isosurface(grid);
  const double exact = 4.0 * 3.14159265358979323846 * R * R;
  CHECK(std::abs(m.area() - exact) < 0.02 * exact);
  CHECK(std::abs(std::abs(m.signed_volume()) - 4.0 / 3.0 * 3.14159265358979323846 * R * R * R) < 0.02);
  for (const auto& t : m.triangles)
    for (int q = 0; q < 3; ++q) CHECK(t[q] < m.vertices.size());
}

DEVICE_CASE(mc_plane, "plane design isosurface lies within half a voxel of its plane") {
  const int r = 16;
  TriMesh m = extract_isosurface(sample_grid(plane_design(0, 0.0), r));
  CHECK(!m.triangles.empty());
  size_t near = 0;
  for (const auto& v : m.vertices) near += std::abs(std::abs(v[0] - 0.5) - 0.5) < 0.5 / r || std::abs(v[0] - 0.5) < 0.5 / r;
  CHECK(near == m.vertices.size());
}

DEVICE_CASE(mc_empty, "a field without zero crossing has no isosurface") {
  CHECK_THROWS_AS(extract_isosurface(sample_grid_fn([](const Vec3&) { return 1.0; }, 8)), Error);
  FieldGrid zero = sample_grid_fn([](const Vec3&) { return 0.0; }, 8);
  CHECK_THROWS_AS(extract_isosurface(zero), DegenerateDesignError);
}

DEVICE_CASE(stl_roundtrip, "binary STL byte layout reads back with an independent reader") {
  TriMesh m = extract_isosurface(sample_grid(seeded_design(3), 8));
  std::string path = "mc_test_export.stl";
  export_mesh(m, path, MeshFormat::StlBinary);
  std::FILE* f = std::fopen(path.c_str(), "rb");
  CHECK(f != nullptr);
  std::vector<unsigned char> bytes(84 + 50 * m.triangles.size() + 16);
  size_t n = std::fread(bytes.data(), 1, bytes.size(), f);
  std::fclose(f);
  std::remove(path.c_str());
  CHECK(n == 84 + 50 * m.triangles.size());
  std::uint32_t count = 0;
  std::memcpy(&count, bytes.data() + 80, 4);
  CHECK(count == m.triangles.size());
  size_t bad = 0;
  for (size_t t = 0; t < m.triangles.size(); ++t) {
    float rec[12];
    std::memcpy(rec, bytes.data() + 84 + 50 * t, 48);
    for (int q = 0; q < 3; ++q)
      for (int a = 0; a < 3; ++a) bad += rec[3 + 3 * q + a] != float(m.vertices[m.triangles[t][q]][a]);
  }
  CHECK(bad == 0);
  CHECK_THROWS_AS(export_mesh(TriMesh{}, path, MeshFormat::Obj), ValidationError);
}

int main(int argc, char** argv) {
  bool host_only = argc > 1 && std::strcmp(argv[1], "--host") == 0;
  int ran = 0;
  for (auto& c : registry()) {
    if (c.device && host_only) continue;
    g_case = c.name;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_failed;
      std::fprintf(stderr, "FAILED [%s] unexpected exception: %s\n", c.name, e.what());
    }
    ++ran;
  }
  std::printf("%d cases, %d checks, %d failed\n", ran, g_checks, g_failed);
  return g_failed ? 1 : 0;
}
