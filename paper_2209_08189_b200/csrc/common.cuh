// Shared device/host helpers for libvelreg_b200 (sm_100a only).
//
// Layout convention (mirrors /root/reference/pkg/src/velreg/grid.py:3-5,99):
//   scalar field  : float[n1][n2][n3], C order, x1 outermost, x3 contiguous
//   vector field  : float[3][n1][n2][n3] (SoA, one component after another)
//   characteristic: float[3][n1][n2][n3] displacement in INDEX units, i.e. the
//                   departure point of voxel (i,j,k) is (i-d1, j-d2, k-d3).
//   spectrum      : complex[n1][n2][n3/2+1] (numpy rfftn layout,
//                   /root/reference/pkg/src/velreg/diffops.py:34-38)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define VR_OK 0
#define VR_ERR_ARG -1
#define VR_ERR_DIMS -2
#define VR_ERR_LAUNCH -3
#define VR_ERR_ALLOC -4
#define VR_ERR_UNSUPPORTED -5

#define VR_CHECK_LAUNCH()                                   \
  do {                                                      \
    cudaError_t e__ = cudaGetLastError();                   \
    if (e__ != cudaSuccess) return VR_ERR_LAUNCH;           \
  } while (0)

namespace vr {

constexpr double kTwoPi = 6.283185307179586476925286766559;

struct Dims {
  int n1, n2, n3;
  __host__ __device__ int64_t n() const { return (int64_t)n1 * n2 * n3; }
};

inline int dims_from(const int64_t* d, Dims* out) {
  if (!d) return VR_ERR_ARG;
  for (int a = 0; a < 3; ++a)
    if (d[a] < 1 || d[a] > (1 << 20)) return VR_ERR_DIMS;
  int64_t n = d[0] * d[1] * d[2];
  // per-field element offsets are 32-bit on the device
  if (n >= (int64_t(1) << 31)) return VR_ERR_DIMS;
  out->n1 = (int)d[0];
  out->n2 = (int)d[1];
  out->n3 = (int)d[2];
  return VR_OK;
}

__device__ __forceinline__ int wrap_idx(int i, int n) {
  int r = i % n;
  return r < 0 ? r + n : r;
}

__device__ __forceinline__ int next_wrap(int i, int n) { return (i + 1 == n) ? 0 : i + 1; }

// Split a departure coordinate q = base - d into (floor index, fraction).
// Exact for |d| < 2^23: the fraction is computed from d alone, so its
// precision is that of the small displacement, not of the absolute index.
__device__ __forceinline__ void split_coord(int base, float d, int& i0, float& t) {
  float nd = -d;
  float fl = floorf(nd);
  t = nd - fl;           // exact (Sterbenz)
  i0 = base + (int)fl;
  if (t >= 1.0f) { t = 0.0f; i0 += 1; }  // guards -0 / rounding at the top
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline unsigned grid_for(int64_t n, int threads, int64_t cap = (int64_t)1 << 30) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

}  // namespace vr
