// context.h -- the shl_ctx device context and the host-side stage helpers
// shared by shl_api.cu (single-device pipeline) and slab.cu (z-slab
// decomposition).  Internal; not part of the public ABI.
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "device.cuh"
#include "internal.h"
#include "solver.cuh"

using shl::ShlError;


#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw ShlError(SHL_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace shl {
namespace host {

extern thread_local std::string g_thread_error;
// Stream of the context the calling thread is working in (set by guarded()):
// workspaces grow with stream-ordered cudaMallocAsync / cudaFreeAsync on it, so
// a growing buffer never synchronizes the device (and with it the other batch
// lanes), as cudaFree would.
extern thread_local cudaStream_t g_alloc_stream;

// Owning device allocation that only grows.  Move-only: a copied raw pointer
// would be freed twice (e.g. when a std::vector of levels reallocates).
struct DevBuf;

// NVTX range for one pipeline stage (header-only nvtx3: a no-op unless a
// profiler's injection library is attached).  Host-side ranges: with
// asynchronous launches they bracket the enqueueing of the stage's work.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), cap(o.cap) {
    o.p = nullptr;
    o.cap = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      if (p) cudaFree(p);
      p = o.p;
      cap = o.cap;
      o.p = nullptr;
      o.cap = 0;
    }
    return *this;
  }
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    const cudaStream_t as = g_alloc_stream;
    if (p) {
      if (as)
        CK(cudaFreeAsync(p, as));
      else
        cudaFree(p);
    }
    p = nullptr;
    cap = 0;
    size_t want = bytes + bytes / 8 + 256;
    if (as) {
      CK(cudaMallocAsync(&p, want, as));
      // host-synchronous copies (legacy stream) may touch it next
      CK(cudaStreamSynchronize(as));
    } else {
      CK(cudaMalloc(&p, want));
    }
    cap = want;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// Small device-side bookkeeping block, mirrored into pinned host memory.
struct Misc {
  unsigned long long norm_bits;
  int n_surface;
  int touches;
  int n_nodes;
  int n_elem;
  int n_bricks;  // active level-0 bricks (brick numbering)
  int node0_active;
  double beta_sum;
  int n_components;  // mechanical components of the element set (fem.hpp:288-317)
  int n_floating;    // ... without an element at torus node 0
  double pad[3];
};

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

}  // namespace host
}  // namespace shl

struct shl_ctx {
  using DevBuf = shl::host::DevBuf;
  using Misc = shl::host::Misc;
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t cap_stream = nullptr;  // only ever in capture mode (iteration graph)
  bool high_priority = false;         // lane 0 of a batch under SHL_LANE_PRIO (A/B)
  std::string err;
  bool profiling = false;
  int64_t launches = 0;
  int64_t h2d = 0, d2h = 0;  // bytes across PCIe (counted at each copy)

  // resident grid
  int r = 0;
  bool grid_ready = false, mesh_ready = false;
  double norm = 0.0;
  DevBuf tab, coeff, sl, sign8, centres, corners, csign, misc;
  // mesh + topology
  DevBuf occ0, occ1, beta64, beta32, elem_flag, node_flag, off, node_map, node_list, elem_list,
      scan_tmp, beta_partials;
  // brick-major level-0 numbering (brick.cuh): padded flags / offsets, brick
  // activity / index, active brick table
  DevBuf bflag, boff, bact, bidx, bcoord, bstart;
  int n_bricks = 0;
  DevBuf cc_parent, cc_corner;  // union-find workspaces (launch_components)
  int n_components = 0, n_floating = 0;
  shl::BrickView brick_view() const {
    shl::BrickView v;
    const shl::BrickDims d = shl::brick_dims(r);
    v.bcoord = bcoord.as<int>();
    v.bstart = bstart.as<int>();
    v.nab = n_bricks;
    v.nbx = d.nbx;
    v.nby = d.nby;
    v.n_nodes = n_nodes;
    return v;
  }
  int64_t n_surface = 0, n_elem = 0;
  int n_nodes = 0, full_fallback = 0, node0_active = 0;
  double volume_ratio = 0.0, beta_sum = 0.0;
  // solver
  DevBuf vec, partials, state, cout;
  // multigrid hierarchy (levels >= 1; level 0 aliases the solver's buffers)
  struct GmgLevel {
    int r = 0, n = 0, ld = 0;
    DevBuf flag, off, map, list, stencil, dinv, vec, scan_tmp;
    DevBuf bflag, boff, blist;  // active 8x4x4 bricks (stencil_brick_sweep), r % 8 == 0 and r >= 16
    int nab = 0;
    shl::BrickView brick_view() const {
      shl::BrickView v;
      if (nab > 0) {
        v.bcoord = blist.as<int>();
        v.nab = nab;
        v.nbx = r / 8;
        v.nby = r / 4;
      }
      return v;
    }
  };
  std::vector<GmgLevel> gmg;
  DevBuf gmg0;  // level-0 V-cycle work vectors (xa, xb, res)
  // marching cubes / raw export (geom.cu)
  DevBuf mc_owned, mc_cnt, mc_verts, mc_tris;
  Misc* hmisc = nullptr;
  int* hlevels = nullptr;  // pinned: per multigrid level (last scan offset, last flag)
  shl::PcgState* hstate = nullptr;
  double* hC = nullptr;
  cudaEvent_t ev[12] = {};  // 0 field | 1 mesh select | 7 topology | 2 solve: 3 AS | 8 RHS | 9 AS | 4 | 5 C | 6
  void* nccl = nullptr;  // z-slab communicator (slab.cu), created on demand
  void (*nccl_deleter)(void*) = nullptr;
  std::vector<cudaEvent_t> prof_ev;
  // concurrent batch lanes (shl_homogenize_batch): sub-contexts on the same
  // device, each with its own stream and workspaces, driven by one host thread
  int n_lanes = 1;
  std::vector<shl_ctx*> lanes;

  // Host waits block (yield the core) instead of spinning: batch lanes each
  // wait on their own stream, and spinning threads starved the other lanes'
  // host work (graph launches, polls) when the process has few cores.
  cudaEvent_t sync_ev = nullptr;
  void sync() {
    if (!sync_ev) {
      CK(cudaStreamSynchronize(stream));
      return;
    }
    CK(cudaEventRecord(sync_ev, stream));
    CK(cudaEventSynchronize(sync_ev));
  }
  float ms(int a, int b) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, ev[a], ev[b]));
    return t;
  }
};

namespace shl {
namespace host {

template <class Fn>
int guarded(shl_ctx* ctx, Fn&& fn) {
  struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
    ~StreamScope() { g_alloc_stream = prev; }
  } scope(ctx ? ctx->stream : nullptr);
  try {
    if (ctx) CK(cudaSetDevice(ctx->device));
    fn();
    if (ctx) ctx->err.clear();
    return SHL_OK;
  } catch (const ShlError& e) {
    if (ctx) ctx->err = e.what();
    g_thread_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    g_thread_error = e.what();
    return SHL_IO;
  }
}

template <class Fn>
auto tagged(const char* stage, Fn&& fn) {
  try {
    return fn();
  } catch (const ShlError& e) {
    if (e.code == SHL_CUDA || e.code == SHL_IO) throw;
    throw ShlError(e.code, std::string(stage) + ": " + e.what());
  }
}

struct FieldInputs {
  int r = 0, nc = 0, n = 0;
  std::vector<double> coeff, tab;
  std::vector<int8_t> sign;
  size_t h2d_bytes() const { return (coeff.size() + tab.size()) * sizeof(double) + sign.size(); }
};

void require_r(int r);
void alloc_grid(shl_ctx* c, int r);
FieldInputs prepare_field(const HostDesign& d, int r);
void run_field(shl_ctx* c, const FieldInputs& f);
void read_norm(shl_ctx* c);
void build_topology(shl_ctx* c);
void run_mesh(shl_ctx* c, const shl_shell_params& sp);
int resolve_precision(const shl_solve_options& o);
void element_loads(const double* K0, int r, double* T, double* W);
void fill_mesh_stats(shl_ctx* c, shl_stats* st);
shl_solve_options default_opts(const shl_solve_options* o);
void validate_inputs(const shl_design* design, const shl_shell_params* sp, const shl_material* mat,
                     int r, double* K0_out);

}  // namespace host
}  // namespace shl
