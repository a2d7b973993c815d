// geom.cu -- the export formats either side of the hot path (SURVEY.md §8 f,
// N4) on the resident grid / mesh:
//
//   shl_extract_isosurface <- extract_isosurface   geomio.hpp:45-108
//   shl_voxel_raw          <- VoxelMesh::write_raw  voxel.hpp:105-114 (the bytes)
//
// Marching cubes reproduces the reference's output exactly, including vertex
// and triangle ORDER, without its sequential hash map.  The reference visits
// cells in grid order (x fastest), and within a cell the 12 edges in table
// order, creating a vertex the first time an edge is met.  A cut edge with low
// lattice corner L and direction a is shared by up to four cells; the first of
// them in grid order -- its "owner" -- has coordinate L_a along a and
// L_b - (L_b >= 1) across (each axis independent, cells stop at r-1).  So
//   vertex id = (# vertices owned by earlier cells) + (rank of the edge among
//               the owner's owned cut edges in edge order)
// and triangle ids are the same kind of prefix over per-cell kept counts.
// Three passes: count (owned-cut mask, vertex and kept-triangle counts per
// cell) -> two exclusive scans -> emit.  Vertex coordinates use the
// reference's FP64 expressions (t = va/(va-vb), p_a = L_a/r + t/r) with
// explicit round-to-nearest intrinsics, so every coordinate is bit-identical
// and the degenerate-triangle test (|e1 x e2| < 1e-12) decides identically.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "context.h"
#include "mc_table.h"

namespace shl {
namespace {

__constant__ uint64_t c_mc[256] = SHL_MC_PACKED;

// local corner offsets (fem.hpp:41-46 hex_corner_offsets)
__device__ __forceinline__ int cx_(int n) { return (n == 1 || n == 2 || n == 5 || n == 6) ? 1 : 0; }
__device__ __forceinline__ int cy_(int n) { return (n == 2 || n == 3 || n == 6 || n == 7) ? 1 : 0; }
__device__ __forceinline__ int cz_(int n) { return n >= 4 ? 1 : 0; }

struct EdgeGeom {
  int axis;
  int lo[3];    // low lattice corner (cell-local offset 0/1 added)
  bool a_low;   // corner a of the edge is the low one
};

__device__ __forceinline__ EdgeGeom edge_geom(int e, int i, int j, int k) {
  const int a = mc::edge_a(e), b = mc::edge_b(e);
  const int ca[3] = {i + cx_(a), j + cy_(a), k + cz_(a)};
  const int cb[3] = {i + cx_(b), j + cy_(b), k + cz_(b)};
  EdgeGeom g;
  g.axis = ca[0] != cb[0] ? 0 : (ca[1] != cb[1] ? 1 : 2);
  g.a_low = ca[g.axis] < cb[g.axis];
#pragma unroll
  for (int d = 0; d < 3; ++d) g.lo[d] = g.a_low ? ca[d] : cb[d];
  return g;
}

// grid.corner(i, j, k) for i, j, k in [0, r]: index r is the wrapped copy of 0
__device__ __forceinline__ double corner_val(const double* __restrict__ cor, int r, int x, int y, int z) {
  x -= x == r ? r : 0;
  y -= y == r ? r : 0;
  z -= z == r ? r : 0;
  return cor[(static_cast<size_t>(z) * r + y) * r + x];
}

struct Cell {
  double val[8];
  int cube;
};

__device__ __forceinline__ void load_cell(const double* __restrict__ cor, int r, int i, int j, int k, Cell& c) {
  c.cube = 0;
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    c.val[n] = corner_val(cor, r, i + cx_(n), j + cy_(n), k + cz_(n));
    if (c.val[n] < 0.0) c.cube |= 1 << n;
  }
}

// edges whose corners fall on different sides (== mc::kEdgeTable[cube])
__device__ __forceinline__ int cut_edges(int cube) {
  int m = 0;
#pragma unroll
  for (int e = 0; e < 12; ++e)
    if (((cube >> mc::edge_a(e)) ^ (cube >> mc::edge_b(e))) & 1) m |= 1 << e;
  return m;
}

__device__ __forceinline__ bool owns(const EdgeGeom& g, int i, int j, int k) {
  const int c[3] = {i, j, k};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int o = d == g.axis ? g.lo[d] : g.lo[d] - (g.lo[d] >= 1 ? 1 : 0);
    if (o != c[d]) return false;
  }
  return true;
}

// vertex_on_edge (geomio.hpp:58-67): t = va/(va-vb) (0.5 if equal), p = L/r, p_a += t/r
__device__ __forceinline__ void edge_point(const EdgeGeom& g, const Cell& c, int e, int r, double (&p)[3]) {
  const int a = mc::edge_a(e), b = mc::edge_b(e);
  const double va = g.a_low ? c.val[a] : c.val[b];
  const double vb = g.a_low ? c.val[b] : c.val[a];
  const double t = (va == vb) ? 0.5 : __ddiv_rn(va, __dsub_rn(va, vb));
  const double rd = static_cast<double>(r);
#pragma unroll
  for (int d = 0; d < 3; ++d) p[d] = __ddiv_rn(static_cast<double>(g.lo[d]), rd);
  p[g.axis] = __dadd_rn(p[g.axis], __ddiv_rn(t, rd));
}

// |e1 x e2| < 1e-12 with e1 = v1 - v0, e2 = v2 - v0 (geomio.hpp:101-103), no FMA
__device__ __forceinline__ bool degenerate_tri(const double (&v0)[3], const double (&v1)[3], const double (&v2)[3]) {
  double e1[3], e2[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    e1[d] = __dsub_rn(v1[d], v0[d]);
    e2[d] = __dsub_rn(v2[d], v0[d]);
  }
  const double x = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
  const double y = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
  const double z = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
  const double s = __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
  return __dsqrt_rn(s) < 1e-12;
}

// Pass 1: per cell the owned cut-edge mask, #vertices it creates, #triangles kept.
__global__ void mc_count_kernel(const double* __restrict__ cor, int r, uint16_t* __restrict__ owned,
                                int* __restrict__ nvert, int* __restrict__ ntri) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  const size_t cell = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (cell >= n3) return;
  const int i = static_cast<int>(cell % r), j = static_cast<int>((cell / r) % r),
            k = static_cast<int>(cell / (static_cast<size_t>(r) * r));
  Cell c;
  load_cell(cor, r, i, j, k, c);
  const int cut = cut_edges(c.cube);
  int own = 0, kept = 0;
  if (cut) {
    double pts[12][3];
#pragma unroll
    for (int e = 0; e < 12; ++e) {
      if (!((cut >> e) & 1)) continue;
      const EdgeGeom g = edge_geom(e, i, j, k);
      if (owns(g, i, j, k)) own |= 1 << e;
      edge_point(g, c, e, r, pts[e]);
    }
    const uint64_t w = c_mc[c.cube];
    const int nt = static_cast<int>(w >> 60);
    for (int t = 0; t < nt; ++t) {
      const int a = (w >> (12 * t)) & 15, b = (w >> (12 * t + 4)) & 15, d = (w >> (12 * t + 8)) & 15;
      if (!degenerate_tri(pts[a], pts[b], pts[d])) ++kept;
    }
  }
  owned[cell] = static_cast<uint16_t>(own);
  nvert[cell] = __popc(own);
  ntri[cell] = kept;
}

// global id of the vertex on cut edge e of cell (i, j, k)
__device__ __forceinline__ uint32_t vertex_id(const EdgeGeom& g, int r, const uint16_t* __restrict__ owned,
                                              const int* __restrict__ voff) {
  int o[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) o[d] = d == g.axis ? g.lo[d] : g.lo[d] - (g.lo[d] >= 1 ? 1 : 0);
  const size_t oc = (static_cast<size_t>(o[2]) * r + o[1]) * r + o[0];
  // the same edge seen from the owner: local edge index with matching axis and low corner
  int le = 0;
#pragma unroll
  for (int e = 0; e < 12; ++e) {
    const EdgeGeom h = edge_geom(e, o[0], o[1], o[2]);
    if (h.axis == g.axis && h.lo[0] == g.lo[0] && h.lo[1] == g.lo[1] && h.lo[2] == g.lo[2]) le = e;
  }
  const int m = owned[oc];
  return static_cast<uint32_t>(voff[oc] + __popc(m & ((1 << le) - 1)));
}

// Pass 3: write this cell's vertices and kept triangles at their prefix offsets.
__global__ void mc_emit_kernel(const double* __restrict__ cor, int r, const uint16_t* __restrict__ owned,
                               const int* __restrict__ voff, const int* __restrict__ toff,
                               double* __restrict__ verts, uint32_t* __restrict__ tris) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  const size_t cell = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (cell >= n3) return;
  const int i = static_cast<int>(cell % r), j = static_cast<int>((cell / r) % r),
            k = static_cast<int>(cell / (static_cast<size_t>(r) * r));
  Cell c;
  load_cell(cor, r, i, j, k, c);
  const int cut = cut_edges(c.cube);
  if (!cut) return;
  const int own = owned[cell];
  double pts[12][3];
  uint32_t ids[12];
  int nv = voff[cell];
#pragma unroll
  for (int e = 0; e < 12; ++e) {
    if (!((cut >> e) & 1)) continue;
    const EdgeGeom g = edge_geom(e, i, j, k);
    edge_point(g, c, e, r, pts[e]);
    if ((own >> e) & 1) {
      ids[e] = static_cast<uint32_t>(nv);
      verts[3 * static_cast<size_t>(nv) + 0] = pts[e][0];
      verts[3 * static_cast<size_t>(nv) + 1] = pts[e][1];
      verts[3 * static_cast<size_t>(nv) + 2] = pts[e][2];
      ++nv;
    } else {
      ids[e] = vertex_id(g, r, owned, voff);
    }
  }
  const uint64_t w = c_mc[c.cube];
  const int nt = static_cast<int>(w >> 60);
  size_t out = toff[cell];
  for (int t = 0; t < nt; ++t) {
    const int a = (w >> (12 * t)) & 15, b = (w >> (12 * t + 4)) & 15, d = (w >> (12 * t + 8)) & 15;
    if (degenerate_tri(pts[a], pts[b], pts[d])) continue;
    tris[3 * out + 0] = ids[a];
    tris[3 * out + 1] = ids[b];
    tris[3 * out + 2] = ids[d];
    ++out;
  }
}

// write_raw bytes: 0 absent, 1 + lround(254 beta) present (voxel.hpp:108-110)
__global__ void raw_kernel(const int* __restrict__ elem_list, int64_t n_elem, const double* __restrict__ beta64,
                           uint8_t* __restrict__ occ) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= n_elem) return;
  const int e = elem_list[t];
  occ[e] = static_cast<uint8_t>(1 + llround(__dmul_rn(beta64[e], 254.0)));
}

}  // namespace
}  // namespace shl

using namespace shl::host;

extern "C" {

int shl_extract_isosurface(shl_ctx* c, double* vertices, int64_t vertex_cap, uint32_t* triangles,
                           int64_t triangle_cap, int64_t* n_vertices, int64_t* n_triangles) {
  if (!c) return SHL_VALIDATION;
  return guarded(c, [&] {
    if (!c->grid_ready) throw ShlError(SHL_VALIDATION, "no resident grid: call shl_sample_grid first");
    if (c->norm == 0.0) throw ShlError(SHL_DEGENERATE, "cannot extract isosurface of a degenerate field");
    const int r = c->r;
    const size_t n3 = static_cast<size_t>(r) * r * r;
    c->mc_owned.ensure(n3 * sizeof(uint16_t));
    c->mc_cnt.ensure(n3 * sizeof(int) * 4);
    int* nv = c->mc_cnt.as<int>();
    int* nt = nv + n3;
    int* voff = nt + n3;
    int* toff = voff + n3;
    c->scan_tmp.ensure(shl::scan_temp_bytes(static_cast<int>(n3)));
    const unsigned blocks = static_cast<unsigned>((n3 + 255) / 256);
    shl::mc_count_kernel<<<blocks, 256, 0, c->stream>>>(c->corners.as<double>(), r, c->mc_owned.as<uint16_t>(), nv,
                                                        nt);
    shl::launch_exclusive_scan(nv, voff, static_cast<int>(n3), c->scan_tmp.p, c->scan_tmp.cap, c->stream);
    shl::launch_exclusive_scan(nt, toff, static_cast<int>(n3), c->scan_tmp.p, c->scan_tmp.cap, c->stream);
    CK(cudaGetLastError());
    int last[4];
    CK(cudaMemcpyAsync(&last[0], voff + n3 - 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&last[1], nv + n3 - 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&last[2], toff + n3 - 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&last[3], nt + n3 - 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    const int64_t V = static_cast<int64_t>(last[0]) + last[1], T = static_cast<int64_t>(last[2]) + last[3];
    c->launches += 3;
    if (n_vertices) *n_vertices = V;
    if (n_triangles) *n_triangles = T;
    if (T == 0) throw ShlError(SHL_ERROR, "field has no zero crossing: empty isosurface");
    if (!vertices || !triangles || vertex_cap < V || triangle_cap < T) return;  // sizes only
    c->mc_verts.ensure(static_cast<size_t>(V) * 3 * sizeof(double));
    c->mc_tris.ensure(static_cast<size_t>(T) * 3 * sizeof(uint32_t));
    shl::mc_emit_kernel<<<blocks, 256, 0, c->stream>>>(c->corners.as<double>(), r, c->mc_owned.as<uint16_t>(), voff,
                                                       toff, c->mc_verts.as<double>(), c->mc_tris.as<uint32_t>());
    CK(cudaGetLastError());
    c->launches += 1;
    CK(cudaMemcpyAsync(vertices, c->mc_verts.p, static_cast<size_t>(V) * 3 * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaMemcpyAsync(triangles, c->mc_tris.p, static_cast<size_t>(T) * 3 * sizeof(uint32_t),
                       cudaMemcpyDeviceToHost, c->stream));
    c->d2h += V * 3 * 8 + T * 3 * 4;
    c->sync();
  });
}

int shl_voxel_raw(shl_ctx* c, uint8_t* occ) {
  if (!c || !occ) return SHL_VALIDATION;
  return guarded(c, [&] {
    if (!c->mesh_ready) throw ShlError(SHL_VALIDATION, "no resident mesh: call shl_build_reduced_mesh");
    const int r = c->r;
    const size_t n3 = static_cast<size_t>(r) * r * r;
    c->occ1.ensure(n3);
    CK(cudaMemsetAsync(c->occ1.p, 0, n3, c->stream));
    if (c->n_elem > 0)
      shl::raw_kernel<<<static_cast<unsigned>((c->n_elem + 255) / 256), 256, 0, c->stream>>>(
          c->elem_list.as<int>(), c->n_elem, c->beta64.as<double>(), c->occ1.as<uint8_t>());
    CK(cudaGetLastError());
    c->launches += 1;
    CK(cudaMemcpyAsync(occ, c->occ1.p, n3, cudaMemcpyDeviceToHost, c->stream));
    c->d2h += static_cast<int64_t>(n3);
    c->sync();
  });
}

}  // extern "C"
