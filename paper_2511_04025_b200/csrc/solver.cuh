// solver.cuh -- argument blocks and launchers of the PCG kernels (solver.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "device.cuh"

namespace shl {

template <typename TV>
struct ApplyArgs {
  const int* node_list;  // active node -> grid id
  const int* node_map;   // r^3 -> active node id or -1
  const TV* beta;        // r^3 dense, 0 = absent
  const TV* z;           // 18 planes, slot n is a zero row
  TV* p;
  TV* q;
  double* partials;
  PcgState* state;
  int r;
  int n;
  int ld;
};

template <typename TX, typename TV>
struct UpdateArgs {
  TX* x;
  TX* r;
  const TV* p;
  const TV* q;
  TV* z;
  const TV* dinv;
  double* partials;
  PcgState* state;
  int n;
  int ld;
  int init;
};

template <typename TX>
struct ChomArgs {
  const int* elem_list;
  const int* node_map;
  const double* beta64;
  const TX* x;
  double* partials;
  double* C_out;
  PcgState* state;
  int n_elem;
  int r;
  int ld;
};

void upload_element_constants(const double* K0, const double* W, const double* T, cudaStream_t s);
template <typename TX, typename TV>
void launch_setup(const int* node_list, int n_nodes, int ld, int r, const double* beta64,
                  double ridge, TX* rvec, TV* dinv, cudaStream_t s);
template <typename TV>
void launch_apply(const ApplyArgs<TV>& a, int grid, cudaStream_t s);
template <typename TX, typename TV>
void launch_update(const UpdateArgs<TX, TV>& u, int grid, cudaStream_t s);
template <typename TX>
void launch_chom(const ChomArgs<TX>& c, int grid, cudaStream_t s);

}  // namespace shl
