// gmg_host.h -- host side of the geometric multigrid preconditioner, shared by
// the single-device solve (shl_api.cu) and the z-slab solve (slab.cu):
// parameters, hierarchy setup (levels 1..L on the full torus) and the V-cycle
// driver.  Internal; not part of the public ABI.
#pragma once

#include <cstdlib>
#include <vector>

#include "context.h"

namespace shl {
namespace host {

// ---- geometric multigrid hierarchy (gmg.cuh) ---------------------------------
struct GmgParams {
  int nu = 0;          // pre/post block-Jacobi sweeps; 0 = by operator precision:
                       // 1 with an FP64 operator (mixed, fp64), 2 with the FP32
                       // one (nu = 1 broke down on ~1.5% of 64^3 FP32 designs)
  double omega = 0.6;  // Jacobi damping (>= 0.7 loses smoother convergence: lambda_max(D^-1 A) ~ 2.9)
  int min_r = 8;       // coarsest grid (nodes per axis); r = 4 Galerkin levels of a thin shell
                       // made the V-cycle indefinite on half the designs tested
  int coarse_sweeps = 16;  // damped Jacobi sweeps on the coarsest level (128^3 sweep:
                           // 16 beats 10 by ~3 iterations, 24 gains nothing more)
  int max_levels = 8;
  double omega_c = 0.6;    // damping on the stored (Galerkin) levels
  int l1 = 0;              // l1-block-Jacobi on the stored levels
  int nu0 = 0;             // level-0 sweeps when > 0 (else nu)
  int nu_at(int l) const { return (l == 0 && nu0 > 0) ? nu0 : nu; }
};

inline GmgParams gmg_params() { return GmgParams{}; }

// Coarse levels 1..L: active set, ordered ids, Galerkin stencils, Dinv.
// Two passes so the host waits once, not once per level: the active sets and
// ids of every level depend only on the level above's node map, so they are
// all computed first and their sizes read back together; then the stencils.
// (With concurrent batch lanes every host wait also waits out whatever the
// other lanes have in flight on the GPU.)
template <typename TV>
int gmg_setup(shl_ctx* c, const GmgParams& gp, TV ridge) {
  int L = 0;
  {
    int rf = c->r;
    const int* map_f = c->node_map.as<int>();
    while (L < gp.max_levels && L < 32 && rf % 2 == 0 && rf / 2 >= gp.min_r) {
      const int rc = rf / 2;
      const int n3 = rc * rc * rc;
      if (static_cast<int>(c->gmg.size()) <= L) c->gmg.emplace_back();
      auto& Lv = c->gmg[L];
      Lv.flag.ensure(static_cast<size_t>(n3) * sizeof(int));
      Lv.off.ensure(static_cast<size_t>(n3) * sizeof(int));
      Lv.map.ensure(static_cast<size_t>(n3) * sizeof(int));
      Lv.list.ensure(static_cast<size_t>(n3) * sizeof(int));
      Lv.scan_tmp.ensure(shl::scan_temp_bytes(n3));
      shl::launch_coarse_flags(map_f, rf, rc, Lv.flag.as<int>(), c->stream);
      shl::launch_exclusive_scan(Lv.flag.as<int>(), Lv.off.as<int>(), n3, Lv.scan_tmp.p, Lv.scan_tmp.cap,
                                 c->stream);
      shl::launch_scatter_compact(Lv.flag.as<int>(), Lv.off.as<int>(), n3, Lv.map.as<int>(),
                                  Lv.list.as<int>(), c->stream);
      CK(cudaMemcpyAsync(&c->hlevels[2 * L], Lv.off.as<int>() + n3 - 1, sizeof(int), cudaMemcpyDeviceToHost,
                         c->stream));
      CK(cudaMemcpyAsync(&c->hlevels[2 * L + 1], Lv.flag.as<int>() + n3 - 1, sizeof(int), cudaMemcpyDeviceToHost,
                         c->stream));
      // active bricks of the level for the staged stored-level sweep (FP32; the
      // sizes where it beats the node-ordered sweeps, launch_level_sweep: ~32^3)
      c->hlevels[32 + 2 * L] = c->hlevels[32 + 2 * L + 1] = 0;
      if (sizeof(TV) == 4 && rc % 8 == 0 && rc >= 32 && rc <= 40 && L < 16) {
        const int nb = (rc / 8) * (rc / 4) * (rc / 4);
        Lv.bflag.ensure(static_cast<size_t>(nb) * sizeof(int));
        Lv.boff.ensure(static_cast<size_t>(nb) * sizeof(int));
        Lv.blist.ensure(static_cast<size_t>(nb) * sizeof(int));
        shl::launch_coarse_brick_flags(Lv.map.as<int>(), rc, Lv.bflag.as<int>(), c->stream);
        shl::launch_exclusive_scan(Lv.bflag.as<int>(), Lv.boff.as<int>(), nb, Lv.scan_tmp.p, Lv.scan_tmp.cap,
                                   c->stream);
        shl::launch_scatter_compact(Lv.bflag.as<int>(), Lv.boff.as<int>(), nb, nullptr, Lv.blist.as<int>(),
                                    c->stream);
        CK(cudaMemcpyAsync(&c->hlevels[32 + 2 * L], Lv.boff.as<int>() + nb - 1, sizeof(int),
                           cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&c->hlevels[32 + 2 * L + 1], Lv.bflag.as<int>() + nb - 1, sizeof(int),
                           cudaMemcpyDeviceToHost, c->stream));
      }
      Lv.r = rc;
      map_f = Lv.map.as<int>();
      rf = rc;
      ++L;
    }
  }
  c->sync();
  int rf = c->r;
  const int* map_f = c->node_map.as<int>();
  const TV* beta_f = sizeof(TV) == 8 ? reinterpret_cast<const TV*>(c->beta64.p)
                                     : reinterpret_cast<const TV*>(c->beta32.p);
  const TV* stencil_f = nullptr;
  for (int l = 0; l < L; ++l) {
    auto& Lv = c->gmg[l];
    const int rc = Lv.r;
    Lv.n = c->hlevels[2 * l] + c->hlevels[2 * l + 1];
    Lv.nab = c->hlevels[32 + 2 * l] + c->hlevels[32 + 2 * l + 1];
    Lv.ld = round_up(Lv.n + 1, 32);
    Lv.stencil.ensure(static_cast<size_t>(243) * Lv.ld * sizeof(TV));
    Lv.dinv.ensure(static_cast<size_t>(6) * Lv.ld * sizeof(TV));
    Lv.vec.ensure(static_cast<size_t>(4) * 18 * Lv.ld * sizeof(TV));
    CK(cudaMemsetAsync(Lv.vec.p, 0, static_cast<size_t>(4) * 18 * Lv.ld * sizeof(TV), c->stream));
    shl::launch_galerkin<TV>(Lv.list.as<int>(), Lv.n, rc, map_f, rf, l == 0 ? beta_f : nullptr, stencil_f,
                             l == 0 ? ridge : TV(0), Lv.stencil.as<TV>(), c->stream);
    shl::launch_coarse_dinv<TV>(Lv.list.as<int>(), Lv.n, Lv.stencil.as<TV>(), Lv.dinv.as<TV>(), gp.l1, c->stream);
    c->launches += 5;
    CK(cudaGetLastError());
    map_f = Lv.map.as<int>();
    stencil_f = Lv.stencil.as<TV>();
    rf = rc;
  }
  return L;
}

// Symmetric V(nu, nu) cycle: z = M r on level 0, written by the last level-0
// sweep into zout (type TO).
template <typename TX, typename TV, typename TO>
struct Vcycle {
  shl_ctx* c;
  GmgParams gp;
  int L = 0;
  std::vector<shl::GmgLevelView<TV>> view;  // 0..L
  std::vector<TV*> b, xa, xb, res;          // per level (b[0] unused: level-0 rhs is r)
  shl::PcgState* st;
  double* partials;
  int64_t launches = 0;
  TO* zout = nullptr;
  cudaStream_t s = nullptr;  // launch stream (the capture stream while recording the iteration graph)

  int grid(int n) const { return shl::apply_grid(n, c->num_sms); }

  // first_done: the restriction into b[l] already wrote x = omega Dinv b[l]
  // into xa[l] (restrict_kernel's fused first sweep)
  TV* level(int l, const TX* b0, int init, bool first_done = false) {
    const auto& V = view[l];
    const bool fine = l == 0;
    const TV w = static_cast<TV>(fine ? gp.omega : gp.omega_c);
    TV* cur = xa[l];
    TV* oth = xb[l];
    auto sweep = [&](TV* xin, TV* xout, int mode) {
      if (fine)
        shl::launch_level_sweep<TX, TV>(V, true, b0, xin, xout, w, mode, st, partials, init, grid(V.n), s);
      else
        shl::launch_level_sweep<TV, TV>(V, false, b[l], xin, xout, w, mode, st, partials, init, grid(V.n),
                                        s);
      ++launches;
    };
    if (l == L && l > 0 && shl::launch_coarsest<TV>(V, b[l], cur, w, gp.coarse_sweeps, st, s)) {
      ++launches;
      return cur;
    }
    if (!fine && !first_done) {
      shl::launch_jacobi_first<TV, TV>(V, b[l], cur, w, st, s);
      ++launches;
    }  // level 0: the update kernel already wrote w Dinv r into xa[0]
    const int nu = gp.nu_at(l);
    const int pre = (l == L) ? gp.coarse_sweeps : nu;  // coarsest: damped Jacobi solve
    for (int k = 1; k < pre; ++k) {
      sweep(cur, oth, 0);
      std::swap(cur, oth);
    }
    if (l == L) return cur;
    sweep(cur, res[l], 1);
    // the child's first sweep rides on the restriction, except on an 8^3
    // coarsest level (its cluster kernel starts from b itself)
    const bool fuse = !(l + 1 == L && view[l + 1].r == 8);
    shl::launch_restrict<TV>(view[l + 1], V, res[l], b[l + 1], st, s, fuse ? xa[l + 1] : nullptr,
                             static_cast<TV>(gp.omega_c));
    TV* xc = level(l + 1, b0, init, fuse);
    shl::launch_prolong<TV>(V, view[l + 1], xc, cur, st, s);
    launches += 2;
    for (int k = 1; k <= nu; ++k) {
      if (fine && k == nu) {
        shl::launch_level_sweep_out<TX, TV, TO>(V, b0, cur, zout, w, st, partials, init, grid(V.n), s);
        launches += V.bricks.nab > 0 ? 2 : 1;  // (brick sweep + its r.z reduction)
        return nullptr;
      }
      sweep(cur, oth, 0);
      std::swap(cur, oth);
    }
    return cur;
  }
};


}  // namespace host
}  // namespace shl
