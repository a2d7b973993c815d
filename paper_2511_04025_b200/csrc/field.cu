// field.cu -- K1: periodic charge-potential field on the r^3 grid (sm_100a).
//
// Replaces the two parallel_for sweeps of sample_grid (field.hpp:488-534)
// over GridSampler::eval (field.hpp:448-469).  FP64, bit-identical to the
// reference: the cosine tables come from the host (glibc cos, field.hpp:
// 424-445) and every product/sum below is an explicit round-to-nearest
// intrinsic in the reference's order (no FMA contraction):
//
//   sl(c,z,h,k) = sum_l coeff[h][k][l] * cz[l]          (starts at 0.0)
//   sh(c,y,z,h) = sum_k cy[k] * sl(c,z,h,k)
//   s(c,x,y,z)  = sum_h cx[h] * sh(c,y,z,h)
//   F(x,y,z)    = sum_c sign_c * s                       (charges in expanded order)
//
// sl depends on (charge, z) and sh on (charge, y, z) only, so they are hoisted
// with identical rounding and the per-sample cost drops from 80 to 7 flops
// per charge.  One block owns kFieldRows (y,z)-rows of one sample set
// (centres, table coords [0,r); or corners, [r,2r)); the sh values of its rows
// live in shared memory, each thread keeps one x abscissa's cx in registers
// and accumulates the kFieldRows samples of its column.
#include "device.cuh"

namespace shl {

namespace {

__global__ void field_sl_kernel(const double* __restrict__ tab, const double* __restrict__ coeff,
                                double* __restrict__ sl, int nc, int r, int n) {
  // one thread per (charge, table coordinate t along z)
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int twor = 2 * r;
  if (tid >= nc * twor) return;
  const int c = tid / twor, t = tid % twor;
  const double* cz = tab + ((static_cast<size_t>(c) * 3 + 2) * twor + t) * n;
  double* out = sl + static_cast<size_t>(tid) * n * n;
  for (int h = 0; h < n; ++h)
    for (int k = 0; k < n; ++k) {
      const double* cell = coeff + (h * n + k) * n;
      double acc = 0.0;
      for (int l = 0; l < n; ++l) acc = __dadd_rn(acc, __dmul_rn(cell[l], cz[l]));
      out[h * n + k] = acc;
    }
}

template <int N>
__global__ void __launch_bounds__(kFieldThreads)
    field_samples_kernel(const double* __restrict__ tab, const double* __restrict__ sl,
                         const int8_t* __restrict__ sign, int nc, int r, int n_rt,
                         double* __restrict__ centres, double* __restrict__ corners,
                         int8_t* __restrict__ corner_sign, unsigned long long* norm_bits) {
  const int n = N > 0 ? N : n_rt;
  extern __shared__ double sh_s[];  // [kFieldRows][chunk][n]
  const int set = blockIdx.z;       // 0 centres, 1 corners
  const int tz = blockIdx.y;
  const int ty0 = blockIdx.x * kFieldRows;
  const int nrows = min(kFieldRows, r - ty0);
  const int twor = 2 * r;
  const int toff = set ? r : 0;
  double* out = set ? corners : centres;
  double vmax = 0.0;

  for (int x0 = 0; x0 < r; x0 += kFieldThreads) {
    const int tx = x0 + threadIdx.x;
    double acc[kFieldRows];
#pragma unroll
    for (int q = 0; q < kFieldRows; ++q) acc[q] = 0.0;
    for (int c0 = 0; c0 < nc; c0 += kFieldChargeChunk) {
      const int cn = min(kFieldChargeChunk, nc - c0);
      __syncthreads();
      // sh for this block's rows and charge chunk (field.hpp:458-463 inner two loops)
      for (int w = threadIdx.x; w < nrows * cn * n; w += blockDim.x) {
        const int h = w % n;
        const int c = (w / n) % cn;
        const int q = w / (n * cn);
        const int cg = c0 + c;
        const double* cy = tab + ((static_cast<size_t>(cg) * 3 + 1) * twor + toff + ty0 + q) * n;
        const double* slc = sl + (static_cast<size_t>(cg) * twor + toff + tz) * n * n + h * n;
        double s = 0.0;
        for (int k = 0; k < n; ++k) s = __dadd_rn(s, __dmul_rn(cy[k], slc[k]));
        sh_s[(q * kFieldChargeChunk + c) * n + h] = s;
      }
      __syncthreads();
      if (tx < r) {
        for (int c = 0; c < cn; ++c) {
          const int cg = c0 + c;
          const double* cx = tab + ((static_cast<size_t>(cg) * 3 + 0) * twor + toff + tx) * n;
          double cxr[N > 0 ? N : 17];
#pragma unroll
          for (int h = 0; h < (N > 0 ? N : 17); ++h)
            if (h < n) cxr[h] = __ldg(cx + h);
          const bool neg = sign[cg] < 0;
#pragma unroll
          for (int q = 0; q < kFieldRows; ++q) {
            const double* shq = sh_s + (q * kFieldChargeChunk + c) * n;
            double s = 0.0;
#pragma unroll
            for (int h = 0; h < (N > 0 ? N : 17); ++h)
              if (h < n) s = __dadd_rn(s, __dmul_rn(cxr[h], shq[h]));
            // acc += sign * s  (sign = +-1.0, the product is exact)
            acc[q] = __dadd_rn(acc[q], neg ? -s : s);
          }
        }
      }
    }
    if (tx < r) {
      for (int q = 0; q < nrows; ++q) {
        const size_t g = (static_cast<size_t>(tz) * r + (ty0 + q)) * r + tx;
        out[g] = acc[q];
        if (set) {
          corner_sign[g] = acc[q] > 0.0 ? 1 : (acc[q] < 0.0 ? -1 : 0);
        } else {
          vmax = fmax(vmax, fabs(acc[q]));
        }
      }
    }
  }
  if (!set) {
    // norm = max |centre| (field.hpp:530-532); max is order independent
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    if ((threadIdx.x & 31) == 0 && vmax > 0.0)
      atomicMax(norm_bits, static_cast<unsigned long long>(__double_as_longlong(vmax)));
  }
}

}  // namespace

void launch_field_sl(const double* tab, const double* coeff, double* sl, int nc, int r, int n,
                     cudaStream_t s) {
  const int total = nc * 2 * r;
  if (total == 0) return;
  field_sl_kernel<<<(total + 255) / 256, 256, 0, s>>>(tab, coeff, sl, nc, r, n);
}

void launch_field_samples(const double* tab, const double* sl, const int8_t* sign, int nc, int r,
                          int n, double* centres, double* corners, int8_t* corner_sign,
                          unsigned long long* norm_bits, cudaStream_t s) {
  dim3 grid((r + kFieldRows - 1) / kFieldRows, r, 2);
  const size_t smem = sizeof(double) * kFieldRows * kFieldChargeChunk * n;
  if (n == 3) {
    cudaFuncSetAttribute(field_samples_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    field_samples_kernel<3><<<grid, kFieldThreads, smem, s>>>(tab, sl, sign, nc, r, n, centres,
                                                              corners, corner_sign, norm_bits);
  } else {
    cudaFuncSetAttribute(field_samples_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    field_samples_kernel<0><<<grid, kFieldThreads, smem, s>>>(tab, sl, sign, nc, r, n, centres,
                                                              corners, corner_sign, norm_bits);
  }
}

}  // namespace shl
