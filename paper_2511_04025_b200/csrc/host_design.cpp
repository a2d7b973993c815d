// host_design.cpp -- host-side reference arithmetic for the device pipeline.
//
// Everything here runs once per design and feeds the kernels: symmetry
// expansion, series coefficients, the per-axis cosine tables, the element
// stiffness matrix and the seeded random designs.  It is compiled with
// -O2 -ffp-contract=off (no FMA contraction), matching the reference build
// (proj/CMakeLists.txt:11), because the FP64 field must reproduce the
// reference samples bit for bit: the tables use glibc cos exactly as
// field.hpp:424-445 does.
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <functional>
#include <stdexcept>

namespace shl {

namespace {

// splitmix64 (common.hpp:86-104)
struct SplitMix {
  uint64_t s;
  explicit SplitMix(uint64_t seed) : s(seed ? seed : 0x9e3779b97f4a7c15ull) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double range(double lo, double hi) { return lo + (hi - lo) * unit(); }
};

inline double wrap01(double x) {  // Charge ctor, field.hpp:51-54
  double v = x - std::floor(x);
  if (v >= 1.0) v -= 1.0;
  return v;
}

}  // namespace

double basis_weight(int h, int k, int l) {  // field.hpp:35-42
  if (h < 0 || k < 0 || l < 0) throw ShlError(SHL_VALIDATION, "basis_weight: negative index");
  const int zeros = (h == 0) + (k == 0) + (l == 0);
  switch (zeros) {
    case 3: throw ShlError(SHL_VALIDATION, "basis_weight: (0,0,0) term is excluded");
    case 2: return 0.25;
    case 1: return 0.5;
    default: return 1.0;
  }
}

bool inside_fbv(int sym, const double* p) {  // field.hpp:101-112
  const double eps = 1e-9;
  if (sym == SHL_SYM_NONE) {
    for (int a = 0; a < 3; ++a)
      if (!(p[a] >= -eps && p[a] < 1.0 + eps)) return false;
    return true;
  }
  if (sym == SHL_SYM_CUBIC_OCTANT)
    return std::min({p[0], p[1], p[2]}) >= -eps && std::max({p[0], p[1], p[2]}) <= 0.5 + eps;
  return p[2] >= -eps && p[2] <= p[1] + eps && p[1] <= p[0] + eps && p[0] <= 0.5 + eps;
}

HostDesign HostDesign::from_abi(const shl_design& d) {
  if (d.K < 0) throw ShlError(SHL_VALIDATION, "truncation order K must be >= 0");
  if (d.symmetry < SHL_SYM_NONE || d.symmetry > SHL_SYM_TETRAHEDRAL)
    throw ShlError(SHL_VALIDATION, "unknown symmetry mode");
  if (d.n_charges < 0 || (d.n_charges > 0 && (!d.positions || !d.signs)) || !d.weights)
    throw ShlError(SHL_VALIDATION, "design arrays missing");
  HostDesign h;
  h.symmetry = d.symmetry;
  h.K = d.K;
  const int n = d.K + 1;
  h.weights.assign(d.weights, d.weights + n * n * n);
  for (int c = 0; c < d.n_charges; ++c) {
    if (d.signs[c] != 1 && d.signs[c] != -1)
      throw ShlError(SHL_VALIDATION, "charge sign must be +1 or -1");
    for (int a = 0; a < 3; ++a) h.pos.push_back(wrap01(d.positions[3 * c + a]));
    h.sign.push_back(d.signs[c]);
  }
  return h;
}

void HostDesign::validate() const {  // field.hpp:149-172
  const int n = K + 1;
  if (K < 0) throw ShlError(SHL_VALIDATION, "truncation order K must be >= 0");
  if (static_cast<int>(weights.size()) != n * n * n)
    throw ShlError(SHL_VALIDATION, "weights must have (K+1)^3 slots");
  if (weights[0] != 0.0) throw ShlError(SHL_VALIDATION, "the (0,0,0) weight must be zero");
  int balance = 0;
  for (size_t c = 0; c < sign.size(); ++c) {
    balance += sign[c];
    if (!inside_fbv(symmetry, &pos[3 * c]))
      throw ShlError(SHL_VALIDATION, "charge lies outside the fundamental bounding volume");
  }
  if (balance != 0) throw ShlError(SHL_VALIDATION, "charge counts must balance");
}

// field.hpp:63-99 + 236-249: image = 0.5 + s_a * (p_{perm(a)} - 0.5) per row
// of a signed permutation (exactly the Eigen product: one nonzero per row),
// then the Charge wrap; order = charge-major, operator-minor.
HostDesign HostDesign::expanded() const {
  validate();
  if (symmetry == SHL_SYM_NONE) return *this;
  struct Op {
    int perm[3];
    int sgn[3];
  };
  std::vector<Op> ops;
  const int flips[2] = {1, -1};
  if (symmetry == SHL_SYM_CUBIC_OCTANT) {
    for (int sx : flips)
      for (int sy : flips)
        for (int sz : flips) ops.push_back({{0, 1, 2}, {sx, sy, sz}});
  } else {
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (const auto& p : perms)
      for (int sx : flips)
        for (int sy : flips)
          for (int sz : flips) ops.push_back({{p[0], p[1], p[2]}, {sx, sy, sz}});
  }
  HostDesign out = *this;
  out.symmetry = SHL_SYM_NONE;
  out.pos.clear();
  out.sign.clear();
  for (size_t c = 0; c < sign.size(); ++c) {
    double rel[3];
    for (int a = 0; a < 3; ++a) rel[a] = pos[3 * c + a] - 0.5;
    for (const Op& op : ops) {
      for (int a = 0; a < 3; ++a) out.pos.push_back(wrap01(0.5 + op.sgn[a] * rel[op.perm[a]]));
      out.sign.push_back(sign[c]);
    }
  }
  return out;
}

// field.hpp:492-500 -- (alpha * w) / d, the sampler's own rounding.
std::vector<double> HostDesign::grid_coefficients() const {
  const int n = K + 1;
  std::vector<double> coeff(static_cast<size_t>(n) * n * n, 0.0);
  for (int h = 0; h < n; ++h)
    for (int k = 0; k < n; ++k)
      for (int l = 0; l < n; ++l) {
        if (!h && !k && !l) continue;
        const int idx = (h * n + k) * n + l;
        coeff[idx] = weights[idx] * basis_weight(h, k, l) / double(h * h + k * k + l * l);
      }
  return coeff;
}

// field.hpp:424-445.  Layout [charge][axis][t][order]; t < r centres
// (i+1/2)/r, t >= r corners (t-r)/r.
std::vector<double> axis_tables(const HostDesign& ex, int r) {
  const int n = ex.K + 1;
  const size_t nc = ex.sign.size();
  std::vector<double> tab(nc * 3 * 2 * static_cast<size_t>(r) * n);
  for (size_t c = 0; c < nc; ++c)
    for (int axis = 0; axis < 3; ++axis) {
      const double p = ex.pos[3 * c + axis];
      for (int i = 0; i < 2 * r; ++i) {
        const double t = (i < r) ? (i + 0.5) / r : double(i - r) / r;
        double* out = &tab[(((c * 3 + axis) * 2 * r) + i) * n];
        out[0] = 1.0;
        if (n == 1) continue;
        const double c1 = std::cos(2.0 * M_PI * (t - p));
        out[1] = c1;
        for (int h = 2; h < n; ++h) out[h] = 2.0 * c1 * out[h - 1] - out[h - 2];
      }
    }
  return tab;
}

// fem.hpp:50-92: 8-node hex, 2x2x2 Gauss, Voigt (xx,yy,zz,yz,xz,xy).
void element_stiffness(double E, double nu, double edge, double* K) {
  if (!(E > 0.0)) throw ShlError(SHL_VALIDATION, "Young's modulus must be positive");
  if (!(nu > -1.0 && nu < 0.5)) throw ShlError(SHL_VALIDATION, "Poisson ratio must lie in (-1, 0.5)");
  if (!(edge > 0.0)) throw ShlError(SHL_VALIDATION, "element edge must be positive");
  const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double mu = E / (2.0 * (1.0 + nu));
  const double g = 1.0 / std::sqrt(3.0);
  const double detJ = edge * edge * edge / 8.0, scale = 2.0 / edge;
  std::fill(K, K + 576, 0.0);
  for (int gp = 0; gp < 8; ++gp) {
    const double q[3] = {g * (2 * ((gp >> 0) & 1) - 1), g * (2 * ((gp >> 1) & 1) - 1),
                         g * (2 * ((gp >> 2) & 1) - 1)};
    // shape-function gradients at this Gauss point
    double dN[8][3];
    for (int n = 0; n < 8; ++n) {
      const double s[3] = {2.0 * kCorner[n][0] - 1.0, 2.0 * kCorner[n][1] - 1.0,
                           2.0 * kCorner[n][2] - 1.0};
      dN[n][0] = 0.125 * s[0] * (1 + s[1] * q[1]) * (1 + s[2] * q[2]) * scale;
      dN[n][1] = 0.125 * s[1] * (1 + s[0] * q[0]) * (1 + s[2] * q[2]) * scale;
      dN[n][2] = 0.125 * s[2] * (1 + s[0] * q[0]) * (1 + s[1] * q[1]) * scale;
    }
    // B^T D B for isotropic D: row (a,i), col (b,j):
    //   lam dN_a[i] dN_b[j] + mu (dN_a[j] dN_b[i] + delta_ij dN_a . dN_b)
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b) {
        const double dot = dN[a][0] * dN[b][0] + dN[a][1] * dN[b][1] + dN[a][2] * dN[b][2];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double v = lam * dN[a][i] * dN[b][j] + mu * dN[a][j] * dN[b][i];
            if (i == j) v += mu * dot;
            K[(3 * a + i) * 24 + 3 * b + j] += detJ * v;
          }
      }
  }
  for (int i = 0; i < 24; ++i)
    for (int j = i + 1; j < 24; ++j) {
      const double s = 0.5 * (K[i * 24 + j] + K[j * 24 + i]);
      K[i * 24 + j] = K[j * 24 + i] = s;
    }
}

// field.hpp:569-593.  The reference builds each position as
// Vec3(rng.uniform(), rng.uniform(), rng.uniform()); GCC (its toolchain)
// evaluates those arguments right to left, so the draws land in z, y, x.
HostDesign random_design(int sym, int n_pre, int K, double lo, double hi, uint64_t seed) {
  if (n_pre <= 0 || n_pre % 2 != 0)
    throw ShlError(SHL_VALIDATION, "pre-expansion charge count must be even and positive");
  if (K < 0) throw ShlError(SHL_VALIDATION, "truncation order K must be >= 0");
  SplitMix rng(seed);
  HostDesign d;
  d.symmetry = sym;
  d.K = K;
  const int n = K + 1;
  d.weights.assign(static_cast<size_t>(n) * n * n, 0.0);
  for (int idx = 1; idx < n * n * n; ++idx) d.weights[idx] = rng.range(lo, hi);
  const double box = sym == SHL_SYM_NONE ? 1.0 : 0.5;
  for (int c = 0; c < n_pre; ++c) {
    double p[3];
    p[2] = rng.range(0.0, box);
    p[1] = rng.range(0.0, box);
    p[0] = rng.range(0.0, box);
    // fold_into_fbv (field.hpp:116-125)
    for (double& v : p) v -= std::floor(v);
    if (sym != SHL_SYM_NONE)
      for (double& v : p)
        if (v > 0.5) v = 1.0 - v;
    if (sym == SHL_SYM_TETRAHEDRAL) std::sort(p, p + 3, std::greater<double>());
    for (double v : p) d.pos.push_back(wrap01(v));
    d.sign.push_back(c < n_pre / 2 ? 1 : -1);
  }
  d.validate();
  return d;
}

}  // namespace shl
