// field.hpp -- drop-in for /root/reference/proj/include/shellular/field.hpp
//
// Design space (Symmetry, basis_weight, Charge, symmetry operators, FBV,
// DesignParams, expand_symmetry), pointwise FieldEvaluator, FieldGrid,
// sample_grid (device, bit-identical FP64), sample_grid_fn and
// random_design, with the reference's names, signatures and defaults.
// Deviations: JSON (de)serialization uses strings (no nlohmann dependency);
// FieldEvaluator::gradient is not provided (it only feeds the spec-only
// fitting module).
#pragma once

#include <algorithm>
#include <array>
#include <functional>
#include <string>
#include <vector>

#include "common.hpp"

namespace shellular {

enum class Symmetry { None, CubicOctant, Tetrahedral };

inline std::string to_string(Symmetry s) {
  switch (s) {
    case Symmetry::None: return "none";
    case Symmetry::CubicOctant: return "cubic_octant";
    case Symmetry::Tetrahedral: return "tetrahedral";
  }
  return "none";
}

inline Symmetry symmetry_from_string(const std::string& s) {
  if (s == "none") return Symmetry::None;
  if (s == "cubic_octant") return Symmetry::CubicOctant;
  if (s == "tetrahedral") return Symmetry::Tetrahedral;
  throw ValidationError("unknown symmetry mode '" + s + "'");
}

// field.hpp:35-42
inline double basis_weight(int h, int k, int l) {
  if (h < 0 || k < 0 || l < 0) throw ValidationError("basis_weight: negative index");
  int zeros = (h == 0) + (k == 0) + (l == 0);
  if (zeros == 3) throw ValidationError("basis_weight: (0,0,0) term is excluded");
  if (zeros == 1) return 0.5;
  if (zeros == 2) return 0.25;
  return 1.0;
}

struct Charge {
  Vec3 position = Vec3::Zero();  // wrapped into [0,1)
  int sign = 1;

  Charge() = default;
  Charge(const Vec3& p, int s) : sign(s) {
    if (s != 1 && s != -1) throw ValidationError("charge sign must be +1 or -1");
    for (int a = 0; a < 3; ++a) {
      double v = p[a] - std::floor(p[a]);
      if (v >= 1.0) v -= 1.0;
      position[a] = v;
    }
  }
};

// field.hpp:63-99
inline const std::vector<Mat3>& symmetry_operators(Symmetry s) {
  static const std::vector<Mat3> identity = {Mat3::Identity()};
  static const std::vector<Mat3> octant = [] {
    std::vector<Mat3> ops;
    for (int sx : {1, -1})
      for (int sy : {1, -1})
        for (int sz : {1, -1}) {
          Mat3 m;
          m(0, 0) = sx;
          m(1, 1) = sy;
          m(2, 2) = sz;
          ops.push_back(m);
        }
    return ops;
  }();
  static const std::vector<Mat3> octahedral = [] {
    std::vector<Mat3> ops;
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (auto& p : perms)
      for (int sx : {1, -1})
        for (int sy : {1, -1})
          for (int sz : {1, -1}) {
            Mat3 m;
            m(0, p[0]) = sx;
            m(1, p[1]) = sy;
            m(2, p[2]) = sz;
            ops.push_back(m);
          }
    return ops;
  }();
  switch (s) {
    case Symmetry::None: return identity;
    case Symmetry::CubicOctant: return octant;
    case Symmetry::Tetrahedral: return octahedral;
  }
  return identity;
}

inline bool in_fundamental_volume(Symmetry s, const Vec3& p, double eps = 1e-9) {
  switch (s) {
    case Symmetry::None:
      return p[0] >= -eps && p[0] < 1.0 + eps && p[1] >= -eps && p[1] < 1.0 + eps &&
             p[2] >= -eps && p[2] < 1.0 + eps;
    case Symmetry::CubicOctant: return p.minCoeff() >= -eps && p.maxCoeff() <= 0.5 + eps;
    case Symmetry::Tetrahedral:
      return p[2] >= -eps && p[2] <= p[1] + eps && p[1] <= p[0] + eps && p[0] <= 0.5 + eps;
  }
  return false;
}

inline Vec3 fold_into_fbv(Symmetry s, const Vec3& p) {
  Vec3 q = p;
  for (int a = 0; a < 3; ++a) q[a] -= std::floor(q[a]);
  if (s == Symmetry::None) return q;
  for (int a = 0; a < 3; ++a)
    if (q[a] > 0.5) q[a] = 1.0 - q[a];
  if (s == Symmetry::CubicOctant) return q;
  std::sort(q.data(), q.data() + 3, std::greater<double>());
  return q;
}

struct DesignParams {
  Symmetry symmetry = Symmetry::None;
  int truncation = 2;  // K
  std::vector<Charge> charges;
  std::vector<double> weights;  // (K+1)^3, weights[0] == 0

  int weight_index(int h, int k, int l) const {
    int n = truncation + 1;
    return (h * n + k) * n + l;
  }
  double weight(int h, int k, int l) const { return weights[weight_index(h, k, l)]; }
  double& weight(int h, int k, int l) { return weights[weight_index(h, k, l)]; }
  int num_weight_terms() const {
    int n = truncation + 1;
    return n * n * n - 1;
  }

  void validate() const {  // field.hpp:149-172
    if (truncation < 0) throw ValidationError("truncation order K must be >= 0");
    int n = truncation + 1;
    if (static_cast<int>(weights.size()) != n * n * n)
      throw ValidationError("weights must have (K+1)^3 slots");
    if (weights[0] != 0.0) throw ValidationError("the (0,0,0) weight must be zero");
    int plus = 0, minus = 0;
    for (const auto& c : charges) {
      (c.sign == 1 ? plus : minus)++;
      if (!in_fundamental_volume(symmetry, c.position))
        throw ValidationError("charge lies outside the fundamental bounding volume");
    }
    if (plus != minus)
      throw ValidationError("charge counts must balance: " + std::to_string(plus) +
                            " positive vs " + std::to_string(minus) + " negative");
  }

  // ABI view; the returned holder owns the flat arrays.
  struct Abi {
    std::vector<double> pos;
    std::vector<int32_t> sign;
    shl_design d{};
  };
  Abi abi() const {
    Abi a;
    for (const auto& c : charges) {
      for (int i = 0; i < 3; ++i) a.pos.push_back(c.position[i]);
      a.sign.push_back(c.sign);
    }
    a.d.symmetry = static_cast<int>(symmetry);
    a.d.K = truncation;
    a.d.n_charges = static_cast<int>(charges.size());
    a.d.positions = a.pos.data();
    a.d.signs = a.sign.data();
    a.d.weights = weights.data();
    return a;
  }
};

// field.hpp:236-249 (host reference arithmetic inside the library)
inline DesignParams expand_symmetry(const DesignParams& params) {
  params.validate();
  if (params.symmetry == Symmetry::None) return params;
  auto a = params.abi();
  const size_t mult = symmetry_operators(params.symmetry).size();
  std::vector<double> pos(3 * params.charges.size() * mult);
  std::vector<int32_t> sg(params.charges.size() * mult);
  int32_t n = 0;
  detail::check(shl_expand_symmetry(&a.d, pos.data(), sg.data(), &n), nullptr);
  DesignParams out = params;
  out.symmetry = Symmetry::None;
  out.charges.clear();
  for (int i = 0; i < n; ++i) out.charges.emplace_back(Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]), sg[i]);
  return out;
}

// Pointwise evaluation of the truncated series (field.hpp:264-312); host,
// for fixtures and spot checks (the grid goes through the device).
class FieldEvaluator {
 public:
  explicit FieldEvaluator(const DesignParams& params)
      : expanded_(expand_symmetry(params)), K_(params.truncation) {
    int n = K_ + 1;
    coeff_.assign(static_cast<size_t>(n) * n * n, 0.0);
    for (int h = 0; h < n; ++h)
      for (int k = 0; k < n; ++k)
        for (int l = 0; l < n; ++l) {
          if (!h && !k && !l) continue;
          int idx = (h * n + k) * n + l;
          coeff_[idx] = params.weights[idx] * (basis_weight(h, k, l) / double(h * h + k * k + l * l));
        }
  }
  const DesignParams& expanded() const { return expanded_; }
  double value(const Vec3& p) const { return value(p[0], p[1], p[2]); }
  double value(double x, double y, double z) const {
    int n = K_ + 1;
    double acc = 0.0;
    std::vector<double> cx(n), cy(n), cz(n);
    for (const auto& c : expanded_.charges) {
      cosines(x - c.position[0], n, cx.data());
      cosines(y - c.position[1], n, cy.data());
      cosines(z - c.position[2], n, cz.data());
      double s = 0.0;
      for (int h = 0; h < n; ++h) {
        double sh = 0.0;
        for (int k = 0; k < n; ++k) {
          double sl = 0.0;
          for (int l = 0; l < n; ++l) sl += coeff_[(h * n + k) * n + l] * cz[l];
          sh += cy[k] * sl;
        }
        s += cx[h] * sh;
      }
      acc += c.sign * s;
    }
    return acc;
  }

 private:
  static void cosines(double d, int n, double* c) {
    c[0] = 1.0;
    if (n == 1) return;
    double c1 = std::cos(2.0 * M_PI * d);
    c[1] = c1;
    for (int h = 2; h < n; ++h) c[h] = 2.0 * c1 * c[h - 1] - c[h - 2];
  }
  DesignParams expanded_;
  int K_;
  std::vector<double> coeff_;
};

inline double eval_field(const DesignParams& params, const Vec3& p) {
  return FieldEvaluator(params).value(p);
}

struct FieldGrid {
  int resolution = 0;
  std::vector<double> samples;         // r^3 centres
  std::vector<double> corner_samples;  // (r+1)^3 incl. wrapped copies
  double norm = 0.0;

  bool degenerate() const { return norm == 0.0; }
  size_t cell_index(int i, int j, int k) const {
    int r = resolution;
    return (static_cast<size_t>(k) * r + j) * r + i;
  }
  size_t corner_index(int i, int j, int k) const {
    int r1 = resolution + 1;
    return (static_cast<size_t>(k) * r1 + j) * r1 + i;
  }
  double corner(int i, int j, int k) const { return corner_samples[corner_index(i, j, k)]; }
  double center(int i, int j, int k) const { return samples[cell_index(i, j, k)]; }
};

// field.hpp:488-534 -- on the device, bit-identical to the reference.  The
// `threads` argument is accepted for signature compatibility.
inline FieldGrid sample_grid(const DesignParams& params, int r, int threads = 0) {
  (void)threads;
  auto a = params.abi();
  FieldGrid g;
  g.resolution = r;
  if (r >= 4) {
    g.samples.resize(static_cast<size_t>(r) * r * r);
    g.corner_samples.resize(static_cast<size_t>(r + 1) * (r + 1) * (r + 1));
  }
  shl_ctx* ctx = detail::context();
  detail::check(shl_sample_grid(ctx, &a.d, r, g.samples.data(), g.corner_samples.data(), &g.norm),
                ctx);
  return g;
}

// field.hpp:538-559 (host)
template <class F>
inline FieldGrid sample_grid_fn(F&& fn, int r) {
  if (r < 4) throw ValidationError("grid resolution must be >= 4");
  FieldGrid g;
  g.resolution = r;
  g.samples.assign(static_cast<size_t>(r) * r * r, 0.0);
  g.corner_samples.assign(static_cast<size_t>(r + 1) * (r + 1) * (r + 1), 0.0);
  for (int k = 0; k < r; ++k)
    for (int j = 0; j < r; ++j)
      for (int i = 0; i < r; ++i)
        g.samples[g.cell_index(i, j, k)] = fn(Vec3((i + 0.5) / r, (j + 0.5) / r, (k + 0.5) / r));
  for (int k = 0; k <= r; ++k)
    for (int j = 0; j <= r; ++j)
      for (int i = 0; i <= r; ++i)
        g.corner_samples[g.corner_index(i, j, k)] = fn(Vec3(double(i) / r, double(j) / r, double(k) / r));
  double m = 0.0;
  for (double v : g.samples) m = std::max(m, std::abs(v));
  g.norm = m;
  return g;
}

struct RandomDesignSpec {
  Symmetry symmetry = Symmetry::CubicOctant;
  int n_charges_pre_expansion = 8;
  int truncation = 2;
  double weight_lo = -1.0;
  double weight_hi = 1.0;
};

// field.hpp:569-593 (bit-identical to the GCC-compiled reference)
inline DesignParams random_design(const RandomDesignSpec& spec, std::uint64_t seed) {
  const int npre = std::max(spec.n_charges_pre_expansion, 0);
  const int n = spec.truncation + 1;
  std::vector<double> pos(3 * static_cast<size_t>(npre));
  std::vector<int32_t> sg(npre);
  std::vector<double> w(static_cast<size_t>(std::max(n, 1)) * std::max(n, 1) * std::max(n, 1));
  detail::check(shl_random_design(static_cast<int>(spec.symmetry), spec.n_charges_pre_expansion,
                                  spec.truncation, spec.weight_lo, spec.weight_hi, seed, pos.data(),
                                  sg.data(), w.data()),
                nullptr);
  DesignParams p;
  p.symmetry = spec.symmetry;
  p.truncation = spec.truncation;
  p.weights = w;
  for (int i = 0; i < npre; ++i) p.charges.emplace_back(Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]), sg[i]);
  return p;
}

}  // namespace shellular
