// shellular_oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A plain C++20 restatement (no Eigen) of the reference hot path of
// arxiv/paper_2511_04025 (`proj/include/shellular/*.hpp`), used as the checker
// for the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it.  The product library
// (paper_2511_04025_b200/libshellular_cuda.so) never links or calls it.
//
// Build flags follow the reference build (CMakeLists.txt:11, "-O2 -DNDEBUG",
// no -march => no FMA contraction): -O2 -ffp-contract=off.  Every
// floating-point expression on the bit-exact part (field sampling, mask) keeps
// the reference's operation order; each function cites the reference lines it
// restates.
//
// Pinning: the field/mask half is checked bit-for-bit against the reference
// headers themselves (oracle/_ref, built from /root/reference with a minimal
// Eigen shim) through tests/golden/*; the FEM half is pinned by the
// reference's known-answer tests (isotropic tensor, laminate closed form,
// dense KKT, direct master-slave solve) in tests/test_oracle_fem.py.

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

// the standard marching-cubes triangulation, packed (same data the product uses)
#include "../paper_2511_04025_b200/csrc/mc_table.h"

namespace orc {

// ---- errors (common.hpp:25-48) -------------------------------------------
enum Status { OK = 0, VALIDATION = 1, DEGENERATE = 2, SOLVER = 3, IO = 4, BASE = 6 };
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

static thread_local std::string g_last_error;

// ---- threads (common.hpp:50-82) ------------------------------------------
inline int resolve_threads(int requested) {
  if (requested > 0) return requested;
  if (const char* env = std::getenv("SHELL_THREADS")) {
    int n = std::atoi(env);
    if (n > 0) return n;
  }
  unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : static_cast<int>(hw);
}

inline void parallel_for(std::int64_t n, int threads,
                         const std::function<void(std::int64_t, std::int64_t)>& body) {
  if (n <= 0) return;
  int nt = resolve_threads(threads);
  if (nt > n) nt = static_cast<int>(n);
  if (nt <= 1) {
    body(0, n);
    return;
  }
  std::vector<std::thread> pool;
  std::int64_t chunk = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    std::int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&body, lo, hi] { body(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

// ---- splitmix64 Rng (common.hpp:86-113) ----------------------------------
struct Rng {
  std::uint64_t state;
  explicit Rng(std::uint64_t seed) : state(seed ? seed : 0x9e3779b97f4a7c15ull) {}
  std::uint64_t next_u64() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
};

// ---- design space (field.hpp:15-249) -------------------------------------
enum Symmetry { None = 0, CubicOctant = 1, Tetrahedral = 2 };

struct V3 {
  double v[3];
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};

// field.hpp:35-42
inline double basis_weight(int h, int k, int l) {
  if (h < 0 || k < 0 || l < 0) fail(VALIDATION, "basis_weight: negative index");
  int zeros = (h == 0) + (k == 0) + (l == 0);
  if (zeros == 3) fail(VALIDATION, "basis_weight: (0,0,0) term is excluded");
  if (zeros == 1) return 0.5;
  if (zeros == 2) return 0.25;
  return 1.0;
}

// field.hpp:49-56 (Charge ctor wrap)
inline V3 wrap_unit(const V3& p) {
  V3 q;
  for (int a = 0; a < 3; ++a) {
    double v = p[a] - std::floor(p[a]);
    if (v >= 1.0) v -= 1.0;
    q[a] = v;
  }
  return q;
}

// field.hpp:63-99: signed permutation matrices m(row, perm[row]) = sign[row]
struct SignedPerm {
  int perm[3];
  int sign[3];
};
inline std::vector<SignedPerm> symmetry_operators(int s) {
  std::vector<SignedPerm> ops;
  if (s == None) {
    ops.push_back({{0, 1, 2}, {1, 1, 1}});
  } else if (s == CubicOctant) {
    for (int sx : {1, -1})
      for (int sy : {1, -1})
        for (int sz : {1, -1}) ops.push_back({{0, 1, 2}, {sx, sy, sz}});
  } else {
    int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (auto& p : perms)
      for (int sx : {1, -1})
        for (int sy : {1, -1})
          for (int sz : {1, -1}) ops.push_back({{p[0], p[1], p[2]}, {sx, sy, sz}});
  }
  return ops;
}

// field.hpp:101-112
inline bool in_fundamental_volume(int s, const V3& p, double eps = 1e-9) {
  switch (s) {
    case None:
      return p[0] >= -eps && p[0] < 1.0 + eps && p[1] >= -eps && p[1] < 1.0 + eps &&
             p[2] >= -eps && p[2] < 1.0 + eps;
    case CubicOctant: {
      double mn = std::min(p[0], std::min(p[1], p[2]));
      double mx = std::max(p[0], std::max(p[1], p[2]));
      return mn >= -eps && mx <= 0.5 + eps;
    }
    default:
      return p[2] >= -eps && p[2] <= p[1] + eps && p[1] <= p[0] + eps && p[0] <= 0.5 + eps;
  }
}

// field.hpp:116-125
inline V3 fold_into_fbv(int s, const V3& p) {
  V3 q = p;
  for (int a = 0; a < 3; ++a) q[a] -= std::floor(q[a]);
  if (s == None) return q;
  for (int a = 0; a < 3; ++a)
    if (q[a] > 0.5) q[a] = 1.0 - q[a];
  if (s == CubicOctant) return q;
  std::sort(q.v, q.v + 3, std::greater<double>());
  return q;
}

struct Design {
  int symmetry = None;
  int K = 2;
  std::vector<V3> pos;  // wrapped into [0,1)
  std::vector<int> sign;
  std::vector<double> weights;  // (K+1)^3

  // field.hpp:149-172
  void validate() const {
    if (K < 0) fail(VALIDATION, "truncation order K must be >= 0");
    int n = K + 1;
    if (static_cast<int>(weights.size()) != n * n * n)
      fail(VALIDATION, "weights must have (K+1)^3 slots");
    if (weights[0] != 0.0) fail(VALIDATION, "the (0,0,0) weight must be zero");
    int plus = 0, minus = 0;
    for (size_t i = 0; i < pos.size(); ++i) {
      if (sign[i] == 1)
        ++plus;
      else if (sign[i] == -1)
        ++minus;
      else
        fail(VALIDATION, "charge sign must be +1 or -1");
      if (!in_fundamental_volume(symmetry, pos[i]))
        fail(VALIDATION, "charge lies outside the fundamental bounding volume");
    }
    if (plus != minus)
      fail(VALIDATION, "charge counts must balance: " + std::to_string(plus) + " positive vs " +
                           std::to_string(minus) + " negative");
  }
};

// field.hpp:236-249.  center + op*(p - center): the signed-permutation
// product contributes one nonzero term per row, so it is p'_i = 0.5 +
// s_i*(p_{perm_i} - 0.5) exactly; then the Charge ctor wrap.
inline Design expand_symmetry(const Design& d) {
  d.validate();
  if (d.symmetry == None) return d;
  auto ops = symmetry_operators(d.symmetry);
  Design out = d;
  out.symmetry = None;
  out.pos.clear();
  out.sign.clear();
  for (size_t c = 0; c < d.pos.size(); ++c)
    for (const auto& op : ops) {
      V3 rel;
      for (int a = 0; a < 3; ++a) rel[a] = d.pos[c][a] - 0.5;
      V3 img;
      for (int a = 0; a < 3; ++a) img[a] = 0.5 + op.sign[a] * rel[op.perm[a]];
      out.pos.push_back(wrap_unit(img));
      out.sign.push_back(d.sign[c]);
    }
  return out;
}

// field.hpp:569-593
inline Design random_design(int symmetry, int n_pre, int K, double lo, double hi_w,
                            std::uint64_t seed) {
  if (n_pre <= 0 || n_pre % 2 != 0)
    fail(VALIDATION, "pre-expansion charge count must be even and positive");
  if (K < 0) fail(VALIDATION, "truncation order K must be >= 0");
  Rng rng(seed);
  Design p;
  p.symmetry = symmetry;
  p.K = K;
  int n = K + 1;
  p.weights.assign(static_cast<size_t>(n) * n * n, 0.0);
  for (int h = 0; h < n; ++h)
    for (int k = 0; k < n; ++k)
      for (int l = 0; l < n; ++l) {
        if (h == 0 && k == 0 && l == 0) continue;
        p.weights[(h * n + k) * n + l] = rng.uniform(lo, hi_w);
      }
  double hi = symmetry == None ? 1.0 : 0.5;
  for (int i = 0; i < n_pre; ++i) {
    // field.hpp:587 builds Vec3(rng.uniform(..), rng.uniform(..), rng.uniform(..));
    // C++ leaves argument evaluation order unspecified and GCC (the
    // reference's toolchain) evaluates right to left, so the compiled
    // reference draws z, then y, then x.  Pinned against oracle/_ref.
    V3 q;
    q[2] = rng.uniform(0.0, hi);
    q[1] = rng.uniform(0.0, hi);
    q[0] = rng.uniform(0.0, hi);
    q = fold_into_fbv(symmetry, q);
    p.pos.push_back(wrap_unit(q));
    p.sign.push_back(i < n_pre / 2 ? 1 : -1);
  }
  p.validate();
  return p;
}

// ---- grid sampling (field.hpp:417-534) -----------------------------------
struct Grid {
  int r = 0;
  std::vector<double> samples;  // r^3 centres, x fastest
  std::vector<double> corners;  // (r+1)^3
  double norm = 0.0;
};

// field.hpp:492-500: coeff = (alpha * w) / d  (NOT FieldEvaluator's alpha*(w/d))
inline std::vector<double> grid_coefficients(const Design& d) {
  int n = d.K + 1;
  std::vector<double> coeff(static_cast<size_t>(n) * n * n, 0.0);
  for (int h = 0; h < n; ++h)
    for (int k = 0; k < n; ++k)
      for (int l = 0; l < n; ++l) {
        if (h == 0 && k == 0 && l == 0) continue;
        int idx = (h * n + k) * n + l;
        coeff[idx] = d.weights[idx] * basis_weight(h, k, l) / double(h * h + k * k + l * l);
      }
  return coeff;
}

// field.hpp:424-445: tab[c][axis][i][h], i < r centres, i >= r corners
inline std::vector<double> cos_tables(const Design& expanded, int K, int r) {
  int n = K + 1;
  size_t nc = expanded.pos.size();
  std::vector<double> tab(nc * 3 * (2 * static_cast<size_t>(r)) * n);
  for (size_t c = 0; c < nc; ++c)
    for (int axis = 0; axis < 3; ++axis) {
      double pos = expanded.pos[c][axis];
      for (int i = 0; i < 2 * r; ++i) {
        double t = (i < r) ? (i + 0.5) / r : double(i - r) / r;
        double* dst = tab.data() + (((c * 3 + axis) * (2 * r)) + i) * n;
        dst[0] = 1.0;
        if (n > 1) {
          double a = 2.0 * M_PI * (t - pos);
          double c1 = std::cos(a);
          dst[1] = c1;
          for (int h = 2; h < n; ++h) dst[h] = 2.0 * c1 * dst[h - 1] - dst[h - 2];
        }
      }
    }
  return tab;
}

// field.hpp:448-469
inline double eval_point(const std::vector<double>& tab, const std::vector<double>& coeff,
                         const std::vector<int>& sign, int n, int r, int ix, int iy, int iz) {
  double acc = 0.0;
  for (size_t c = 0; c < sign.size(); ++c) {
    const double* cx = tab.data() + (((c * 3 + 0) * (2 * r)) + ix) * n;
    const double* cy = tab.data() + (((c * 3 + 1) * (2 * r)) + iy) * n;
    const double* cz = tab.data() + (((c * 3 + 2) * (2 * r)) + iz) * n;
    double s = 0.0;
    for (int h = 0; h < n; ++h) {
      double sh = 0.0;
      const double* row = coeff.data() + h * n * n;
      for (int k = 0; k < n; ++k) {
        double sl = 0.0;
        const double* cell = row + k * n;
        for (int l = 0; l < n; ++l) sl += cell[l] * cz[l];
        sh += cy[k] * sl;
      }
      s += cx[h] * sh;
    }
    acc += sign[c] * s;
  }
  return acc;
}

// field.hpp:488-534
inline Grid sample_grid(const Design& params, int r, int threads) {
  if (r < 4) fail(VALIDATION, "grid resolution must be >= 4");
  Design ex = expand_symmetry(params);
  // FieldEvaluator ctor (field.hpp:266-279) evaluates basis_weight for every term
  std::vector<double> coeff = grid_coefficients(params);
  int n = params.K + 1;
  std::vector<double> tab = cos_tables(ex, params.K, r);
  Grid g;
  g.r = r;
  g.samples.assign(static_cast<size_t>(r) * r * r, 0.0);
  g.corners.assign(static_cast<size_t>(r + 1) * (r + 1) * (r + 1), 0.0);
  auto ci = [r](int i, int j, int k) { return (static_cast<size_t>(k) * (r + 1) + j) * (r + 1) + i; };
  parallel_for(r, threads, [&](std::int64_t k0, std::int64_t k1) {
    for (int k = int(k0); k < int(k1); ++k)
      for (int j = 0; j < r; ++j)
        for (int i = 0; i < r; ++i)
          g.samples[(static_cast<size_t>(k) * r + j) * r + i] =
              eval_point(tab, coeff, ex.sign, n, r, i, j, k);
  });
  parallel_for(r, threads, [&](std::int64_t k0, std::int64_t k1) {
    for (int k = int(k0); k < int(k1); ++k)
      for (int j = 0; j < r; ++j)
        for (int i = 0; i < r; ++i)
          g.corners[ci(i, j, k)] = eval_point(tab, coeff, ex.sign, n, r, r + i, r + j, r + k);
  });
  int r1 = r + 1;
  for (int k = 0; k < r1; ++k)
    for (int j = 0; j < r1; ++j)
      for (int i = 0; i < r1; ++i) {
        if (i < r && j < r && k < r) continue;
        g.corners[ci(i, j, k)] = g.corners[ci(i % r, j % r, k % r)];
      }
  double m = 0.0;
  for (double v : g.samples) m = std::max(m, std::abs(v));
  g.norm = m;
  return g;
}

// ---- voxelization (voxel.hpp:18-41, 118-141, 235-313) --------------------
struct Shell {
  double sharpness = 500.0;
  double floor_ratio = 1e-3;
  int expand_layers = 0;
  void validate() const {
    if (!(sharpness > 0.0)) fail(VALIDATION, "sharpness must be positive");
    if (!(floor_ratio > 0.0 && floor_ratio < 1.0)) fail(VALIDATION, "floor must lie in (0, 1)");
    if (expand_layers < 0) fail(VALIDATION, "expand_layers must be >= 0");
  }
  int layers_for(int r) const {
    if (expand_layers > 0) return expand_layers;
    return std::max(1, static_cast<int>(std::lround(2.0 * r / 64.0)));
  }
};

inline double step_function(double v, const Shell& sp) {
  double v0 = 2.0 * (1.0 - sp.floor_ratio);
  return 1.0 + 0.5 * v0 - v0 / (1.0 + std::exp(-sp.sharpness * v * v));
}

inline std::vector<std::uint32_t> classify_surface_elements(const Grid& g) {
  if (g.norm == 0.0) fail(DEGENERATE, "cannot classify surface elements of a degenerate field");
  int r = g.r;
  auto corner = [&](int i, int j, int k) {
    return g.corners[(static_cast<size_t>(k) * (r + 1) + j) * (r + 1) + i];
  };
  std::vector<std::uint32_t> out;
  for (int k = 0; k < r; ++k)
    for (int j = 0; j < r; ++j)
      for (int i = 0; i < r; ++i) {
        bool pos = false, neg = false, zero = false;
        for (int dk = 0; dk < 2; ++dk)
          for (int dj = 0; dj < 2; ++dj)
            for (int di = 0; di < 2; ++di) {
              double v = corner(i + di, j + dj, k + dk);
              if (v > 0.0)
                pos = true;
              else if (v < 0.0)
                neg = true;
              else
                zero = true;
            }
        if (zero || (pos && neg)) out.push_back(static_cast<std::uint32_t>((k * r + j) * r + i));
      }
  return out;
}

struct Mesh {
  int r = 0;
  std::vector<std::uint8_t> in;       // r^3 occupancy
  std::vector<std::uint32_t> elements;  // sorted
  std::vector<double> beta;            // per element
  bool full_fallback = false;
  std::size_t n_surface = 0;
  double t_select_ms = 0.0;
};

inline Mesh build_reduced_mesh(const Grid& g, const Shell& sp) {
  sp.validate();
  auto t0 = std::chrono::steady_clock::now();
  int r = g.r;
  std::vector<std::uint32_t> surface = classify_surface_elements(g);
  if (surface.empty()) fail(DEGENERATE, "field has no zero crossing: no surface to mesh");
  size_t total = static_cast<size_t>(r) * r * r;
  Mesh m;
  m.r = r;
  m.n_surface = surface.size();
  m.in.assign(total, 0);
  auto& in = m.in;
  std::vector<std::uint32_t> frontier = surface;
  for (auto e : surface) in[e] = 1;
  int layers = sp.layers_for(r);
  for (int layer = 0; layer < layers; ++layer) {
    std::vector<std::uint32_t> next;
    for (auto e : frontier) {
      int c[3] = {int(e % r), int((e / r) % r), int(e / (r * r))};
      for (int a = 0; a < 3; ++a)
        for (int d : {-1, 1}) {
          int q[3] = {c[0], c[1], c[2]};
          q[a] = (q[a] + d + r) % r;
          std::uint32_t id = static_cast<std::uint32_t>((q[2] * r + q[1]) * r + q[0]);
          if (!in[id]) {
            in[id] = 1;
            next.push_back(id);
          }
        }
    }
    frontier = std::move(next);
  }
  for (size_t e = 0; e < total; ++e) {
    if (!in[e]) continue;
    int c[3] = {int(e % r), int((e / r) % r), int(e / (size_t(r) * r))};
    int flips[3], nf = 0;
    for (int a = 0; a < 3; ++a)
      if (c[a] == 0 || c[a] == r - 1) flips[nf++] = a;
    for (int mask = 1; mask < (1 << nf); ++mask) {
      int q[3] = {c[0], c[1], c[2]};
      for (int b = 0; b < nf; ++b)
        if (mask & (1 << b)) q[flips[b]] = (q[flips[b]] == 0) ? r - 1 : 0;
      in[(size_t(q[2]) * r + q[1]) * r + q[0]] = 1;
    }
  }
  bool touches = false;
  for (size_t e = 0; e < total && !touches; ++e) {
    if (!in[e]) continue;
    int c[3] = {int(e % r), int((e / r) % r), int(e / (size_t(r) * r))};
    for (int a = 0; a < 3; ++a)
      if (c[a] == 0 || c[a] == r - 1) touches = true;
  }
  if (touches)
    for (int i : {0, r - 1})
      for (int j : {0, r - 1})
        for (int k : {0, r - 1}) in[(size_t(k) * r + j) * r + i] = 1;
  for (size_t e = 0; e < total; ++e)
    if (in[e]) m.elements.push_back(static_cast<std::uint32_t>(e));
  m.full_fallback = m.elements.size() == total;
  m.beta.resize(m.elements.size());
  for (size_t e = 0; e < m.elements.size(); ++e)
    m.beta[e] = step_function(g.samples[m.elements[e]] / g.norm, sp);
  m.t_select_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return m;
}

// ---- FEM (fem.hpp:19-92, 129-142) ----------------------------------------
static const int kOff[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                               {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

inline void validate_material(double E, double nu) {
  if (!(E > 0.0)) fail(VALIDATION, "Young's modulus must be positive");
  if (!(nu > -1.0 && nu < 0.5)) fail(VALIDATION, "Poisson ratio must lie in (-1, 0.5)");
}

// fem.hpp:50-92 ; K row-major 24x24
inline void element_stiffness(double E, double nu, double edge, double* K) {
  validate_material(E, nu);
  if (!(edge > 0.0)) fail(VALIDATION, "element edge must be positive");
  double la = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  double mu = E / (2.0 * (1.0 + nu));
  double D[6][6] = {};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) D[a][b] = a == b ? la + 2.0 * mu : la;
  for (int a = 3; a < 6; ++a) D[a][a] = mu;
  std::fill(K, K + 576, 0.0);
  const double g = 1.0 / std::sqrt(3.0);
  double detJ = edge * edge * edge / 8.0;
  double scale = 2.0 / edge;
  for (int gp = 0; gp < 8; ++gp) {
    double xi = g * (2 * ((gp >> 0) & 1) - 1);
    double eta = g * (2 * ((gp >> 1) & 1) - 1);
    double zeta = g * (2 * ((gp >> 2) & 1) - 1);
    double B[6][24] = {};
    for (int n = 0; n < 8; ++n) {
      double sx = 2.0 * kOff[n][0] - 1.0, sy = 2.0 * kOff[n][1] - 1.0, sz = 2.0 * kOff[n][2] - 1.0;
      double dNdx = 0.125 * sx * (1 + sy * eta) * (1 + sz * zeta) * scale;
      double dNdy = 0.125 * sy * (1 + sx * xi) * (1 + sz * zeta) * scale;
      double dNdz = 0.125 * sz * (1 + sx * xi) * (1 + sy * eta) * scale;
      int c = 3 * n;
      B[0][c + 0] = dNdx;
      B[1][c + 1] = dNdy;
      B[2][c + 2] = dNdz;
      B[3][c + 1] = dNdz;
      B[3][c + 2] = dNdy;
      B[4][c + 0] = dNdz;
      B[4][c + 2] = dNdx;
      B[5][c + 0] = dNdy;
      B[5][c + 1] = dNdx;
    }
    double DB[6][24];
    for (int a = 0; a < 6; ++a)
      for (int j = 0; j < 24; ++j) {
        double s = 0.0;
        for (int b = 0; b < 6; ++b) s += D[a][b] * B[b][j];
        DB[a][j] = s;
      }
    for (int i = 0; i < 24; ++i)
      for (int j = 0; j < 24; ++j) {
        double s = 0.0;
        for (int a = 0; a < 6; ++a) s += B[a][i] * DB[a][j];
        K[i * 24 + j] += detJ * s;
      }
  }
  for (int i = 0; i < 24; ++i)
    for (int j = i + 1; j < 24; ++j) {
      double s = 0.5 * (K[i * 24 + j] + K[j * 24 + i]);
      K[i * 24 + j] = K[j * 24 + i] = s;
    }
}

// fem.hpp:129-142: engineering shear (tensor component 1/2)
inline void unit_strain(int s, double e[3][3]) {
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) e[a][b] = 0.0;
  if (s < 3) e[s][s] = 1.0;
  if (s == 3) e[1][2] = e[2][1] = 0.5;
  if (s == 4) e[0][2] = e[2][0] = 0.5;
  if (s == 5) e[0][1] = e[1][0] = 0.5;
}

// ---- masked matrix-free PCG (grid_solver.hpp:18-207) ---------------------
// GridSolver generalized to a masked torus: elements with beta == 0 are
// absent, nodes touched by no present element carry no unknowns, torus node 0
// is pinned (the corner gauge, fem.hpp:190-203).  With beta > 0 everywhere it
// is exactly the reference GridSolver.
struct SolveResult {
  double C[36];
  int iterations[6];
  double t_rhs_ms, t_solve_ms, t_reduce_ms;
  std::int64_t n_nodes, n_elements;
  bool converged;
};

struct MaskedGridSolver {
  int r;
  int threads;
  std::vector<double> beta;  // r^3, 0 = absent
  double K0[576];
  size_t N;  // r^3 nodes
  std::vector<std::uint32_t> elem_nodes;
  std::vector<std::uint32_t> active;  // active element ids, grouped by z layer
  std::vector<size_t> layer_start;    // r+1
  std::vector<std::uint8_t> node_on;
  std::vector<double> dinv;  // 9 per node
  double T[24][6];
  // Diagonal ridge of the reference's singular-system path (fem.hpp:337-343):
  // 1e-11 * mean|diag(A)|.  The reduced shell systems are semidefinite
  // whenever a component floats; the ridge keeps p^T A p > 0 at
  // rounding level and moves C^H by O(1e-11).
  double ridge = 0.0;

  MaskedGridSolver(const std::vector<double>& b, int r_, const double* K, int thr)
      : r(r_), threads(thr), beta(b) {
    if (static_cast<size_t>(r) * r * r != beta.size())
      fail(VALIDATION, "beta array does not match resolution");
    std::memcpy(K0, K, sizeof(K0));
    N = static_cast<size_t>(r) * r * r;
    elem_nodes.resize(N * 8);
    node_on.assign(N, 0);
    layer_start.assign(r + 1, 0);
    for (int k = 0; k < r; ++k) {
      layer_start[k] = active.size();
      for (int j = 0; j < r; ++j)
        for (int i = 0; i < r; ++i) {
          size_t e = (static_cast<size_t>(k) * r + j) * r + i;
          for (int n = 0; n < 8; ++n)
            elem_nodes[e * 8 + n] = static_cast<std::uint32_t>(
                ((static_cast<size_t>((k + kOff[n][2]) % r) * r + (j + kOff[n][1]) % r) * r +
                 (i + kOff[n][0]) % r));
          if (beta[e] != 0.0) {
            active.push_back(static_cast<std::uint32_t>(e));
            for (int n = 0; n < 8; ++n) node_on[elem_nodes[e * 8 + n]] = 1;
          }
        }
    }
    layer_start[r] = active.size();
    // element-local affine displacements (grid_solver.hpp:119-126)
    for (int s = 0; s < 6; ++s) {
      double e[3][3];
      unit_strain(s, e);
      for (int n = 0; n < 8; ++n) {
        double y[3] = {kOff[n][0] / double(r), kOff[n][1] / double(r), kOff[n][2] / double(r)};
        for (int a = 0; a < 3; ++a) T[3 * n + a][s] = e[a][0] * y[0] + e[a][1] * y[1] + e[a][2] * y[2];
      }
    }
    // 3x3 block Jacobi (grid_solver.hpp:129-139)
    std::vector<double> diag(N * 9, 0.0);
    for (auto e : active) {
      double be = beta[e];
      for (int n = 0; n < 8; ++n) {
        double* d = &diag[elem_nodes[e * 8 + n] * 9];
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) d[a * 3 + b] += be * K0[(3 * n + a) * 24 + 3 * n + b];
      }
    }
    double dsum = 0.0;
    size_t ndof = 0;
    for (size_t n = 1; n < N; ++n)
      if (node_on[n]) {
        dsum += std::abs(diag[n * 9 + 0]) + std::abs(diag[n * 9 + 4]) + std::abs(diag[n * 9 + 8]);
        ndof += 3;
      }
    ridge = ndof ? 1e-11 * dsum / double(ndof) : 0.0;
    for (size_t n = 1; n < N; ++n)
      if (node_on[n]) {
        diag[n * 9 + 0] += ridge;
        diag[n * 9 + 4] += ridge;
        diag[n * 9 + 8] += ridge;
      }
    dinv.assign(N * 9, 0.0);
    for (size_t n = 0; n < N; ++n) {
      if (!node_on[n] || n == 0) continue;
      const double* m = &diag[n * 9];
      double c00 = m[4] * m[8] - m[5] * m[7], c01 = m[5] * m[6] - m[3] * m[8],
             c02 = m[3] * m[7] - m[4] * m[6];
      double det = m[0] * c00 + m[1] * c01 + m[2] * c02;
      double id = 1.0 / det;
      double* o = &dinv[n * 9];
      o[0] = c00 * id;
      o[1] = (m[2] * m[7] - m[1] * m[8]) * id;
      o[2] = (m[1] * m[5] - m[2] * m[4]) * id;
      o[3] = c01 * id;
      o[4] = (m[0] * m[8] - m[2] * m[6]) * id;
      o[5] = (m[2] * m[3] - m[0] * m[5]) * id;
      o[6] = c02 * id;
      o[7] = (m[1] * m[6] - m[0] * m[7]) * id;
      o[8] = (m[0] * m[4] - m[1] * m[3]) * id;
    }
  }

  // Blocks are node-major: v[(node*3 + comp)*6 + s]
  void rhs(std::vector<double>& F) const {  // grid_solver.hpp:141-152
    F.assign(N * 18, 0.0);
    double W[24][6];
    for (int i = 0; i < 24; ++i)
      for (int s = 0; s < 6; ++s) {
        double acc = 0.0;
        for (int j = 0; j < 24; ++j) acc += K0[i * 24 + j] * T[j][s];
        W[i][s] = acc;
      }
    for (auto e : active) {
      double be = beta[e];
      for (int n = 0; n < 8; ++n) {
        double* f = &F[elem_nodes[e * 8 + n] * 18];
        for (int a = 0; a < 3; ++a)
          for (int s = 0; s < 6; ++s) f[a * 6 + s] += -be * W[3 * n + a][s];
      }
    }
    for (int q = 0; q < 18; ++q) F[q] = 0.0;
  }

  void apply(const std::vector<double>& x, std::vector<double>& y) const {  // :154-176
    std::fill(y.begin(), y.end(), 0.0);
    auto work_layer = [&](int k) {
      double u[24][6], f[24][6];
      for (size_t q = layer_start[k]; q < layer_start[k + 1]; ++q) {
        std::uint32_t e = active[q];
        const std::uint32_t* nodes = &elem_nodes[size_t(e) * 8];
        for (int n = 0; n < 8; ++n)
          for (int a = 0; a < 3; ++a)
            for (int s = 0; s < 6; ++s) u[3 * n + a][s] = x[(nodes[n] * 3 + a) * 6 + s];
        double be = beta[e];
        for (int i = 0; i < 24; ++i) {
          double acc[6] = {0, 0, 0, 0, 0, 0};
          for (int j = 0; j < 24; ++j) {
            double kij = K0[i * 24 + j];
            for (int s = 0; s < 6; ++s) acc[s] += kij * u[j][s];
          }
          for (int s = 0; s < 6; ++s) f[i][s] = be * acc[s];
        }
        for (int n = 0; n < 8; ++n)
          for (int a = 0; a < 3; ++a)
            for (int s = 0; s < 6; ++s) y[(nodes[n] * 3 + a) * 6 + s] += f[3 * n + a][s];
      }
    };
    if (r % 2 == 0) {
      // two-phase z colouring (valid for even r only)
      for (int parity = 0; parity < 2; ++parity)
        parallel_for((r + 1) / 2, threads, [&](std::int64_t lo, std::int64_t hi) {
          for (std::int64_t idx = lo; idx < hi; ++idx) {
            int k = static_cast<int>(2 * idx + parity);
            if (k < r) work_layer(k);
          }
        });
    } else {
      for (int k = 0; k < r; ++k) work_layer(k);
    }
    if (ridge != 0.0)
      for (size_t q = 18; q < y.size(); ++q) y[q] += ridge * x[q];
    for (int q = 0; q < 18; ++q) y[q] = 0.0;
  }

  void precond(const std::vector<double>& rr, std::vector<double>& z) const {
    parallel_for(static_cast<std::int64_t>(N), threads, [&](std::int64_t lo, std::int64_t hi) {
      for (std::int64_t n = lo; n < hi; ++n) {
        const double* m = &dinv[n * 9];
        for (int a = 0; a < 3; ++a)
          for (int s = 0; s < 6; ++s)
            z[(n * 3 + a) * 6 + s] = m[a * 3 + 0] * rr[(n * 3 + 0) * 6 + s] +
                                     m[a * 3 + 1] * rr[(n * 3 + 1) * 6 + s] +
                                     m[a * 3 + 2] * rr[(n * 3 + 2) * 6 + s];
      }
    });
  }

  void reduce_tensor(const std::vector<double>& X, double* C) const {  // :183-197
    double acc[36] = {};
    double U[24][6], W[24][6];
    for (auto e : active) {
      const std::uint32_t* nodes = &elem_nodes[size_t(e) * 8];
      for (int n = 0; n < 8; ++n)
        for (int a = 0; a < 3; ++a)
          for (int s = 0; s < 6; ++s) U[3 * n + a][s] = X[(nodes[n] * 3 + a) * 6 + s] + T[3 * n + a][s];
      for (int i = 0; i < 24; ++i)
        for (int s = 0; s < 6; ++s) {
          double w = 0.0;
          for (int j = 0; j < 24; ++j) w += K0[i * 24 + j] * U[j][s];
          W[i][s] = w;
        }
      double be = beta[e];
      for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b) {
          double s = 0.0;
          for (int i = 0; i < 24; ++i) s += U[i][a] * W[i][b];
          acc[a * 6 + b] += be * s;
        }
    }
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) C[a * 6 + b] = 0.5 * (acc[a * 6 + b] + acc[b * 6 + a]);
  }

  // grid_solver.hpp:37-96 (lockstep 6 columns, per-column done flags)
  SolveResult solve(double tol, int max_iter, bool allow_unconverged, std::vector<double>* xout) {
    if (max_iter <= 0) max_iter = 20 * r + 2000;
    SolveResult res{};
    res.n_elements = static_cast<std::int64_t>(active.size());
    std::int64_t nn = 0;
    for (auto v : node_on) nn += v;
    res.n_nodes = nn;
    const size_t L = N * 18;
    std::vector<double> X(L, 0.0), R, P(L), AP(L), Z(L);
    auto t0 = std::chrono::steady_clock::now();
    rhs(R);
    auto t1 = std::chrono::steady_clock::now();
    res.t_rhs_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    auto colnorm = [&](const std::vector<double>& v, int s) {
      double acc = 0.0;
      for (size_t i = s; i < L; i += 6) acc += v[i] * v[i];
      return std::sqrt(acc);
    };
    auto coldot = [&](const std::vector<double>& a, const std::vector<double>& b, int s) {
      double acc = 0.0;
      for (size_t i = s; i < L; i += 6) acc += a[i] * b[i];
      return acc;
    };
    double bnorm[6], rz[6];
    for (int s = 0; s < 6; ++s) bnorm[s] = colnorm(R, s);
    precond(R, Z);
    P = Z;
    for (int s = 0; s < 6; ++s) rz[s] = coldot(R, Z, s);
    bool done[6] = {};
    int iters[6] = {};
    for (int s = 0; s < 6; ++s)
      if (bnorm[s] == 0.0) done[s] = true;
    int it = 0;
    while (it < max_iter) {
      bool all = true;
      for (int s = 0; s < 6; ++s) all = all && done[s];
      if (all) break;
      apply(P, AP);
      for (int s = 0; s < 6; ++s) {
        if (done[s]) continue;
        double pap = coldot(P, AP, s);
        if (pap <= 0.0) fail(SOLVER, "grid CG: operator lost positive definiteness");
        double alpha = rz[s] / pap;
        for (size_t i = s; i < L; i += 6) {
          X[i] += alpha * P[i];
          R[i] -= alpha * AP[i];
        }
        iters[s] = it + 1;
        if (colnorm(R, s) <= tol * bnorm[s]) {
          done[s] = true;
          for (size_t i = s; i < L; i += 6) P[i] = 0.0;
          continue;
        }
      }
      precond(R, Z);
      for (int s = 0; s < 6; ++s) {
        if (done[s]) continue;
        double rz_new = coldot(R, Z, s);
        double b = rz_new / rz[s];
        for (size_t i = s; i < L; i += 6) P[i] = Z[i] + b * P[i];
        rz[s] = rz_new;
      }
      ++it;
    }
    res.converged = true;
    for (int s = 0; s < 6; ++s)
      if (!done[s]) res.converged = false;
    if (!res.converged && !allow_unconverged)
      fail(SOLVER, "grid CG did not reach tolerance " + std::to_string(tol) + " in " +
                       std::to_string(max_iter) + " iterations");
    for (int s = 0; s < 6; ++s) res.iterations[s] = iters[s];
    auto t2 = std::chrono::steady_clock::now();
    res.t_solve_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
    reduce_tensor(X, res.C);
    res.t_reduce_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t2).count();
    if (xout) *xout = std::move(X);
    return res;
  }
};

// ---- marching cubes (geomio.hpp:45-108) ------------------------------------
// Sequential restatement: cells in grid order, edges in table order, vertices
// welded on (low lattice corner, axis) keys by a hash map -- the reference's
// own algorithm; the GPU replaces the map by owner-cell prefix sums.
struct TriMesh {
  std::vector<double> v;          // 3 per vertex
  std::vector<std::uint32_t> t;   // 3 per triangle
};

inline TriMesh extract_isosurface(const Grid& g) {
  static const std::uint64_t kTri[256] = SHL_MC_PACKED;
  static const int off[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
  if (g.norm == 0.0) fail(DEGENERATE, "cannot extract isosurface of a degenerate field");
  const int r = g.r, r1 = r + 1;
  TriMesh m;
  std::unordered_map<std::uint64_t, std::uint32_t> edge_vertex;
  auto corner = [&](int i, int j, int k) { return g.corners[(size_t(k) * r1 + j) * r1 + i]; };
  auto vertex_on_edge = [&](const int* lo, int axis, double va, double vb) {
    std::uint64_t key = ((std::uint64_t(lo[2]) * r1 + lo[1]) * r1 + lo[0]) * 4 + axis;
    auto it = edge_vertex.find(key);
    if (it != edge_vertex.end()) return it->second;
    double t = (va == vb) ? 0.5 : va / (va - vb);
    double p[3] = {double(lo[0]) / r, double(lo[1]) / r, double(lo[2]) / r};
    p[axis] += t / r;
    auto id = static_cast<std::uint32_t>(m.v.size() / 3);
    m.v.insert(m.v.end(), p, p + 3);
    edge_vertex.emplace(key, id);
    return id;
  };
  for (int k = 0; k < r; ++k)
    for (int j = 0; j < r; ++j)
      for (int i = 0; i < r; ++i) {
        double val[8];
        int cube = 0;
        for (int n = 0; n < 8; ++n) {
          val[n] = corner(i + off[n][0], j + off[n][1], k + off[n][2]);
          if (val[n] < 0.0) cube |= 1 << n;
        }
        std::uint32_t ev[12];
        bool any = false;
        for (int e = 0; e < 12; ++e) {
          const int a = shl::mc::edge_a(e), b = shl::mc::edge_b(e);
          if (!(((cube >> a) ^ (cube >> b)) & 1)) continue;  // kEdgeTable bit
          any = true;
          int ca[3], cb[3];
          for (int d = 0; d < 3; ++d) {
            ca[d] = (d == 0 ? i : d == 1 ? j : k) + off[a][d];
            cb[d] = (d == 0 ? i : d == 1 ? j : k) + off[b][d];
          }
          int axis = 0;
          for (int d = 0; d < 3; ++d)
            if (ca[d] != cb[d]) axis = d;
          const bool a_low = ca[axis] < cb[axis];
          ev[e] = vertex_on_edge(a_low ? ca : cb, axis, a_low ? val[a] : val[b], a_low ? val[b] : val[a]);
        }
        if (!any) continue;
        const std::uint64_t w = kTri[cube];
        for (int t = 0; t < int(w >> 60); ++t) {
          std::uint32_t tri[3];
          for (int q = 0; q < 3; ++q) tri[q] = ev[(w >> (12 * t + 4 * q)) & 15];
          if (tri[0] == tri[1] || tri[1] == tri[2] || tri[0] == tri[2]) continue;
          const double* v0 = &m.v[3 * size_t(tri[0])];
          const double* v1 = &m.v[3 * size_t(tri[1])];
          const double* v2 = &m.v[3 * size_t(tri[2])];
          double e1[3] = {v1[0] - v0[0], v1[1] - v0[1], v1[2] - v0[2]};
          double e2[3] = {v2[0] - v0[0], v2[1] - v0[1], v2[2] - v0[2]};
          double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2],
                 cz = e1[0] * e2[1] - e1[1] * e2[0];
          if (std::sqrt(cx * cx + cy * cy + cz * cz) < 1e-12) continue;
          m.t.insert(m.t.end(), tri, tri + 3);
        }
      }
  if (m.t.empty()) fail(BASE, "field has no zero crossing: empty isosurface");
  return m;
}

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return IO;
  }
}

inline Design make_design(int symmetry, int K, int n, const double* pos, const int* sign,
                          const double* weights) {
  Design d;
  d.symmetry = symmetry;
  d.K = K;
  if (K < 0) fail(VALIDATION, "truncation order K must be >= 0");
  int m = K + 1;
  d.weights.assign(weights, weights + m * m * m);
  for (int i = 0; i < n; ++i) {
    if (sign[i] != 1 && sign[i] != -1) fail(VALIDATION, "charge sign must be +1 or -1");
    d.pos.push_back(wrap_unit(V3{{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]}}));
    d.sign.push_back(sign[i]);
  }
  return d;
}

}  // namespace orc

// =========================== C ABI (test use) ==============================
extern "C" {

const char* orc_last_error() { return orc::g_last_error.c_str(); }

int orc_random_design(int symmetry, int n_pre, int K, double lo, double hi, std::uint64_t seed,
                      double* pos_out, int* sign_out, double* weights_out) {
  return orc::guard([&] {
    orc::Design d = orc::random_design(symmetry, n_pre, K, lo, hi, seed);
    for (int i = 0; i < n_pre; ++i) {
      for (int a = 0; a < 3; ++a) pos_out[3 * i + a] = d.pos[i][a];
      sign_out[i] = d.sign[i];
    }
    std::copy(d.weights.begin(), d.weights.end(), weights_out);
  });
}

// returns the number of expanded charges through *n_out
int orc_expand_symmetry(int symmetry, int K, int n, const double* pos, const int* sign,
                        const double* weights, double* pos_out, int* sign_out, int* n_out) {
  return orc::guard([&] {
    orc::Design d = orc::make_design(symmetry, K, n, pos, sign, weights);
    orc::Design e = orc::expand_symmetry(d);
    for (size_t i = 0; i < e.pos.size(); ++i) {
      for (int a = 0; a < 3; ++a) pos_out[3 * i + a] = e.pos[i][a];
      sign_out[i] = e.sign[i];
    }
    *n_out = static_cast<int>(e.pos.size());
  });
}

int orc_sample_grid(int symmetry, int K, int n, const double* pos, const int* sign,
                    const double* weights, int r, int threads, double* centres, double* corners,
                    double* norm) {
  return orc::guard([&] {
    orc::Design d = orc::make_design(symmetry, K, n, pos, sign, weights);
    orc::Grid g = orc::sample_grid(d, r, threads);
    std::copy(g.samples.begin(), g.samples.end(), centres);
    std::copy(g.corners.begin(), g.corners.end(), corners);
    *norm = g.norm;
  });
}

// Reduced mesh from a grid.  occupancy: r^3 bytes; beta_dense: r^3 (0 = absent).
int orc_build_reduced_mesh(int r, const double* centres, const double* corners, double norm,
                           double sharpness, double floor_ratio, int expand_layers,
                           std::uint8_t* occupancy, double* beta_dense, std::int64_t* n_elements,
                           std::int64_t* n_surface, int* full_fallback) {
  return orc::guard([&] {
    orc::Grid g;
    g.r = r;
    size_t n3 = size_t(r) * r * r, c3 = size_t(r + 1) * (r + 1) * (r + 1);
    g.samples.assign(centres, centres + n3);
    g.corners.assign(corners, corners + c3);
    g.norm = norm;
    orc::Shell sp{sharpness, floor_ratio, expand_layers};
    orc::Mesh m = orc::build_reduced_mesh(g, sp);
    std::copy(m.in.begin(), m.in.end(), occupancy);
    std::fill(beta_dense, beta_dense + n3, 0.0);
    for (size_t e = 0; e < m.elements.size(); ++e) beta_dense[m.elements[e]] = m.beta[e];
    *n_elements = static_cast<std::int64_t>(m.elements.size());
    *n_surface = static_cast<std::int64_t>(m.n_surface);
    *full_fallback = m.full_fallback ? 1 : 0;
  });
}

// extract_isosurface on a grid; counts always, arrays when they fit
int orc_extract_isosurface(int r, const double* corners, double norm, double* verts, std::int64_t vcap,
                           std::uint32_t* tris, std::int64_t tcap, std::int64_t* nv, std::int64_t* nt) {
  return orc::guard([&] {
    orc::Grid g;
    g.r = r;
    g.corners.assign(corners, corners + size_t(r + 1) * (r + 1) * (r + 1));
    g.norm = norm;
    orc::TriMesh m = orc::extract_isosurface(g);
    *nv = static_cast<std::int64_t>(m.v.size() / 3);
    *nt = static_cast<std::int64_t>(m.t.size() / 3);
    if (*nv <= vcap) std::copy(m.v.begin(), m.v.end(), verts);
    if (*nt <= tcap) std::copy(m.t.begin(), m.t.end(), tris);
  });
}

int orc_step_function(double v, double sharpness, double floor_ratio, double* out) {
  return orc::guard([&] {
    orc::Shell sp{sharpness, floor_ratio, 0};
    *out = orc::step_function(v, sp);
  });
}

int orc_element_stiffness(double E, double nu, double edge, double* K) {
  return orc::guard([&] { orc::element_stiffness(E, nu, edge, K); });
}

// Masked GridSolver.  stats: [t_rhs, t_solve, t_reduce, n_nodes, n_elements, converged]
int orc_grid_solve(int r, const double* beta_dense, const double* K0, double tol, int max_iter,
                   int threads, int allow_unconverged, double* C_out, int* iterations,
                   double* stats, double* x_out) {
  return orc::guard([&] {
    std::vector<double> b(beta_dense, beta_dense + size_t(r) * r * r);
    orc::MaskedGridSolver s(b, r, K0, threads);
    std::vector<double> X;
    orc::SolveResult res = s.solve(tol, max_iter, allow_unconverged != 0, x_out ? &X : nullptr);
    std::copy(res.C, res.C + 36, C_out);
    std::copy(res.iterations, res.iterations + 6, iterations);
    if (stats) {
      stats[0] = res.t_rhs_ms;
      stats[1] = res.t_solve_ms;
      stats[2] = res.t_reduce_ms;
      stats[3] = double(res.n_nodes);
      stats[4] = double(res.n_elements);
      stats[5] = res.converged ? 1.0 : 0.0;
    }
    if (x_out) std::copy(X.begin(), X.end(), x_out);
  });
}

// homogenize (pipeline.hpp:61-113) with the masked grid solver as the solve
// stage.  timings (ms): t_field, t_mesh, t_PBC, t_AS, t_RHS, t_solve, t_C, t_fwd
int orc_homogenize(int symmetry, int K, int n, const double* pos, const int* sign,
                   const double* weights, double sharpness, double floor_ratio, int expand_layers,
                   double E, double nu, int r, int threads, double tol, int max_iter,
                   int allow_unconverged, double* C_out, int* iterations, double* timings,
                   double* info /*[n_elements, n_nodes, volume_ratio, full_fallback, converged]*/) {
  return orc::guard([&] {
    orc::validate_material(E, nu);
    orc::Shell sp{sharpness, floor_ratio, expand_layers};
    sp.validate();
    auto T0 = std::chrono::steady_clock::now();
    orc::Design d = orc::make_design(symmetry, K, n, pos, sign, weights);
    orc::Grid g;
    try {
      g = orc::sample_grid(d, r, threads);
    } catch (const orc::Error& e) {
      orc::fail(e.code, std::string("field: ") + e.what());
    }
    auto T1 = std::chrono::steady_clock::now();
    if (g.norm == 0.0) orc::fail(orc::DEGENERATE, "field: design is degenerate (norm = 0)");
    orc::Mesh m;
    try {
      m = orc::build_reduced_mesh(g, sp);
    } catch (const orc::Error& e) {
      orc::fail(e.code, std::string("mesh: ") + e.what());
    }
    auto T2 = std::chrono::steady_clock::now();
    double K0[576];
    orc::element_stiffness(E, nu, 1.0 / r, K0);
    std::vector<double> beta(size_t(r) * r * r, 0.0);
    double vol = 0.0;
    for (size_t e = 0; e < m.elements.size(); ++e) {
      beta[m.elements[e]] = m.beta[e];
      vol += m.beta[e];
    }
    vol /= double(r) * r * r;
    orc::MaskedGridSolver s(beta, r, K0, threads);
    auto T3 = std::chrono::steady_clock::now();
    orc::SolveResult res;
    try {
      res = s.solve(tol, max_iter, allow_unconverged != 0, nullptr);
    } catch (const orc::Error& e) {
      orc::fail(e.code, std::string("solve: ") + e.what());
    }
    auto T4 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::copy(res.C, res.C + 36, C_out);
    std::copy(res.iterations, res.iterations + 6, iterations);
    timings[0] = ms(T0, T1);
    timings[1] = m.t_select_ms;
    timings[2] = ms(T1, T2) - m.t_select_ms;
    timings[3] = ms(T2, T3);
    timings[4] = res.t_rhs_ms;
    timings[5] = res.t_solve_ms;
    timings[6] = res.t_reduce_ms;
    timings[7] = ms(T0, T4);
    info[0] = double(res.n_elements);
    info[1] = double(res.n_nodes);
    info[2] = vol;
    info[3] = m.full_fallback ? 1.0 : 0.0;
    info[4] = res.converged ? 1.0 : 0.0;
  });
}

}  // extern "C"
