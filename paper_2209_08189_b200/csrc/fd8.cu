// 8th-order centred finite differences with periodic wrap
// (/root/reference/pkg/src/velreg/diffops.py:84-105, coefficients :20).
//
// The arithmetic sequence is the reference's, in fp32, without FMA contraction:
//   out = 0; for o in 1..4: out += c_o * (f[i+o] - f[i-o]);  out /= h
// so fp32 inputs give bit-identical outputs to numpy's fp32 evaluation.
// divergence: out = d1 v1; out += d2 v2; out += d3 v3   (diffops.py:102-104)
//
// Tiling: one CTA = a (TY x 32) tile of one x1-plane; each thread walks NX
// consecutive x1-planes keeping the 9-deep x1 stencil window in registers and
// reading the y/z halos from shared memory (4-plane halo on each side).
#include "common.cuh"
#include "../../include/velreg_b200.h"

namespace vr {

// numpy evaluates `c * (...)` on fp32 arrays with c rounded to fp32 from the
// Python float (NEP 50), hence the double -> float conversions.
__constant__ float kFd8[4] = {(float)(4.0 / 5.0), (float)(-1.0 / 5.0), (float)(4.0 / 105.0),
                              (float)(-1.0 / 280.0)};

// d/dx_axis at a point given the 8 neighbours m[0..3] = f[-1..-4], p[0..3] = f[+1..+4]
__device__ __forceinline__ float fd8_combine(const float p[4], const float m[4], float h) {
  float out = 0.0f;
#pragma unroll
  for (int o = 0; o < 4; ++o) out = __fadd_rn(out, __fmul_rn(kFd8[o], __fsub_rn(p[o], m[o])));
  return __fdiv_rn(out, h);
}

constexpr int TZ = 32, TY = 8, HALO = 4;

// Loads a (TY+8) x (TZ+8) plane tile of `f` at x1-plane `i` into smem.
__device__ __forceinline__ void load_tile(float (*tile)[TZ + 2 * HALO + 1], const float* __restrict__ f,
                                          const Dims& d, int i, int j0, int k0) {
  const int W = TZ + 2 * HALO, H = TY + 2 * HALO;
  const float* plane = f + (int64_t)i * d.n2 * d.n3;
  for (int t = threadIdx.y * TZ + threadIdx.x; t < W * H; t += TZ * TY) {
    int yy = t / W, zz = t - yy * W;
    int j = j0 + yy - HALO, k = k0 + zz - HALO;
    j = j < 0 ? j + d.n2 : (j >= d.n2 ? j - d.n2 : j);
    k = k < 0 ? k + d.n3 : (k >= d.n3 ? k - d.n3 : k);
    tile[yy][zz] = __ldg(plane + j * d.n3 + k);
  }
}

// MODE 0: gradient of a scalar (3 outputs); MODE 1: divergence of a vector.
// SLAB: the input is an x1 slab with `xoff` (>= 4) ghost planes per side and
// component stride `cs`; d = local (output) dims, no x1 wrap.
// SLAB: the x1 window reads ghost planes from lo (4 planes before the slab) /
// hi (4 planes after); y/z tiles only ever read the local plane.
template <int MODE, bool SLAB>
__global__ void __launch_bounds__(TZ* TY) fd8_kernel(const float* __restrict__ f, const float* __restrict__ lo,
                                                     const float* __restrict__ hi, Dims d, float h1, float h2,
                                                     float h3, float* __restrict__ out, int nx) {
  __shared__ float tile[TY + 2 * HALO][TZ + 2 * HALO + 1];
  const int64_t N = d.n();
  const int64_t cs = N;
  const int psz = d.n2 * d.n3;
  const int k0 = blockIdx.x * TZ, j0 = blockIdx.y * TY;
  const int i_begin = blockIdx.z * nx;
  const int i_end = min(i_begin + nx, d.n1);
  const int k = k0 + threadIdx.x, j = j0 + threadIdx.y;
  const bool active = (k < d.n3) && (j < d.n2);
  // x1 window: w[0..8] = f[i-4 .. i+4] (component 0 for divergence)
  const float* fx = f;  // component used along x1
  float w[9];
  if (active) {
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      int ii = i_begin - HALO + o;
      const float* pl;
      if (SLAB) {
        pl = ii < 0 ? lo + (int64_t)(ii + HALO) * psz : (ii >= d.n1 ? hi + (int64_t)(ii - d.n1) * psz
                                                                    : fx + (int64_t)ii * psz);
      } else {
        ii = ii < 0 ? ii + d.n1 : (ii >= d.n1 ? ii - d.n1 : ii);  // n1 >= 9 (caller)
        pl = fx + (int64_t)ii * psz;
      }
      w[o] = __ldg(pl + j * d.n3 + k);
    }
  }
  for (int i = i_begin; i < i_end; ++i) {
    if (active) {
      int ii = i + HALO;
      const float* pl;
      if (SLAB) {
        pl = ii >= d.n1 ? hi + (int64_t)(ii - d.n1) * psz : fx + (int64_t)ii * psz;
      } else {
        ii = ii >= d.n1 ? ii - d.n1 : ii;
        pl = fx + (int64_t)ii * psz;
      }
      w[8] = __ldg(pl + j * d.n3 + k);
    }
    float g1 = 0.f;
    if (active) {
      float p[4] = {w[5], w[6], w[7], w[8]}, m[4] = {w[3], w[2], w[1], w[0]};
      g1 = fd8_combine(p, m, h1);
    }
    const int64_t o = ((int64_t)i * d.n2 + j) * d.n3 + k;
    if (MODE == 0) {
      __syncthreads();
      load_tile(tile, f, d, i, j0, k0);
      __syncthreads();
      if (active) {
        const int ty = threadIdx.y + HALO, tz = threadIdx.x + HALO;
        float p[4], m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { p[q] = tile[ty + q + 1][tz]; m[q] = tile[ty - q - 1][tz]; }
        const float g2 = fd8_combine(p, m, h2);
#pragma unroll
        for (int q = 0; q < 4; ++q) { p[q] = tile[ty][tz + q + 1]; m[q] = tile[ty][tz - q - 1]; }
        const float g3 = fd8_combine(p, m, h3);
        out[o] = g1;
        out[N + o] = g2;
        out[2 * N + o] = g3;
      }
    } else {
      __syncthreads();
      load_tile(tile, f + cs, d, i, j0, k0);
      __syncthreads();
      float acc = g1;
      if (active) {
        const int ty = threadIdx.y + HALO, tz = threadIdx.x + HALO;
        float p[4], m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { p[q] = tile[ty + q + 1][tz]; m[q] = tile[ty - q - 1][tz]; }
        acc = __fadd_rn(acc, fd8_combine(p, m, h2));
      }
      __syncthreads();
      load_tile(tile, f + 2 * cs, d, i, j0, k0);
      __syncthreads();
      if (active) {
        const int ty = threadIdx.y + HALO, tz = threadIdx.x + HALO;
        float p[4], m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { p[q] = tile[ty][tz + q + 1]; m[q] = tile[ty][tz - q - 1]; }
        acc = __fadd_rn(acc, fd8_combine(p, m, h3));
        out[o] = acc;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = w[q + 1];
  }
}

}  // namespace vr

using namespace vr;

// lo/hi == nullptr: periodic; otherwise a slab with 4-plane ghost blocks
static int fd8_launch(int mode, const float* in, const float* lo, const float* hi, const int64_t dims[3],
                      int64_t n1_global, float* out, void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!in || !out || in == out) return VR_ERR_ARG;
  const bool slab = lo != nullptr;
  if (slab && !hi) return VR_ERR_ARG;
  if ((!slab && d.n1 < 9) || d.n2 < 9 || d.n3 < 9 || n1_global < 9) return VR_ERR_DIMS;  // diffops.py:21,77-81
  if (slab && d.n1 < HALO) return VR_ERR_DIMS;
  const float h1 = (float)(kTwoPi / n1_global), h2 = (float)(kTwoPi / d.n2), h3 = (float)(kTwoPi / d.n3);
  const int nx = 16;
  dim3 grid((d.n3 + TZ - 1) / TZ, (d.n2 + TY - 1) / TY, (d.n1 + nx - 1) / nx);
  dim3 block(TZ, TY);
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0 && slab)
    fd8_kernel<0, true><<<grid, block, 0, s>>>(in, lo, hi, d, h1, h2, h3, out, nx);
  else if (mode == 0)
    fd8_kernel<0, false><<<grid, block, 0, s>>>(in, nullptr, nullptr, d, h1, h2, h3, out, nx);
  else if (slab)
    fd8_kernel<1, true><<<grid, block, 0, s>>>(in, lo, hi, d, h1, h2, h3, out, nx);
  else
    fd8_kernel<1, false><<<grid, block, 0, s>>>(in, nullptr, nullptr, d, h1, h2, h3, out, nx);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

extern "C" {
int vr_fd8_grad(const float* f, const int64_t dims[3], float* out3, void* stream) {
  return fd8_launch(0, f, nullptr, nullptr, dims, dims ? dims[0] : 0, out3, stream);
}
int vr_fd8_div(const float* v3, const int64_t dims[3], float* out, void* stream) {
  return fd8_launch(1, v3, nullptr, nullptr, dims, dims ? dims[0] : 0, out, stream);
}
int vr_fd8_grad_slab(const float* f, const float* f_lo, const float* f_hi, const int64_t dims[3], int64_t n1_global,
                     float* out3, void* stream) {
  if (!f_lo || !f_hi) return VR_ERR_ARG;
  return fd8_launch(0, f, f_lo, f_hi, dims, n1_global, out3, stream);
}
int vr_fd8_div_slab(const float* v3, const float* v1_lo, const float* v1_hi, const int64_t dims[3],
                    int64_t n1_global, float* out, void* stream) {
  if (!v1_lo || !v1_hi) return VR_ERR_ARG;
  return fd8_launch(1, v3, v1_lo, v1_hi, dims, n1_global, out, stream);
}
}
