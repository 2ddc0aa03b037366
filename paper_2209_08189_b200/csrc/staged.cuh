// Shared-memory-staged tricubic sweeps ("z-quad" staging) -- EXPERIMENT, not
// built into libvelreg_b200 (no .cu includes it).  Correct (passed the full
// GPU parity suite when wired into vr_advect / vr_incstate_step / labels) but
// measured 0.385 ms vs 0.33 ms for the direct lean gather at 256^3 (B200):
// the staged path is latency-bound (3 CTAs / SM by 64 KB smem, serialized
// load -> reduce -> stage -> gather phases; ncu: long_scoreboard stalls,
// 67 % L1tex throughput).  Kept for a persistent, double-buffered revisit.
//
// One CTA owns a TX x TY x TZ = 4 x 8 x 32 tile of arrival voxels (256 threads:
// lanes along x3, warps along x2, 4 x1 planes per thread).  It reads the tile's
// displacements, reduces the floor-index bounding box of the departure points,
// and stages the source box -- stencil included -- in shared memory as
// overlapping float4 quads Q[row][c] = (f[c], f[c+1], f[c+2], f[c+3]) along x3.
// Every stencil row of a tricubic tap set is then ONE 16-byte shared load:
// 16 LDS.128 per point instead of 64 scattered LDG, which makes the gather
// shared-memory-bandwidth bound (~2 clk/point/SM) instead of L1/LSU bound.
// Smooth characteristics keep the box small (C2: ~8 x 12 x 36 quads = 55 KB for
// 1024 points, ~3.4 L1-resident loads per point to stage).  A tile whose box
// exceeds the budget (rough velocity, tiny grid) uses the direct gather --
// same arithmetic, same results.  Sources: periodic fields or x1 slabs with
// ghost blocks (PlaneSrc); the label-indicator source converts while staging.
#pragma once
#include <climits>
#include "interp.cuh"

namespace vr {
namespace staged {

constexpr int TZ = 32, TY = 8, TX = 4;
constexpr int QCAP = 4096;                       // float4 quads per CTA (64 KB)
constexpr size_t kSmem = sizeof(float4) * QCAP;

// source adaptors for staging: value at (x1 plane, in-plane offset)
template <bool SLAB>
struct FieldSrc {
  PlaneSrc<1, SLAB> p;
  __device__ __forceinline__ const float* plane(int x, int psz) const { return p.plane(0, x, psz); }
  __device__ __forceinline__ float at(const float* pl, int off) const { return __ldg(pl + off); }
};

struct LabelSrc {  // indicator of one label id (synth.py:125), periodic only
  const int* lab;
  int id;
  __device__ __forceinline__ const int* plane(int x, int psz) const { return lab + (int64_t)x * psz; }
  __device__ __forceinline__ float at(const int* pl, int off) const { return __ldg(pl + off) == id ? 1.0f : 0.0f; }
};

// direct (unstaged) tricubic gather through the same adaptor, periodic / slab x1
template <bool SLAB, class S>
__device__ __forceinline__ float direct_cubic(const S& src, const Dims& d, int w, int L1, int ix, int iy, int iz,
                                              float tx, float ty, float tz) {
  float wx[4], wy[4], wz[4];
  lagrange4(tx, wx);
  lagrange4(ty, wy);
  lagrange4(tz, wz);
  const int psz = d.n2 * d.n3;
  int xo[4], yo[4], zo[4];
  if (SLAB) {
    const int i0 = clampi(ix, 1 - w, L1 + w - 3);
    xo[0] = i0 - 1; xo[1] = i0; xo[2] = i0 + 1; xo[3] = i0 + 2;
  } else {
    cubic_idx(wrap_idx(ix, d.n1), d.n1, xo);
  }
  cubic_idx(wrap_idx(iy, d.n2), d.n2, yo);
  cubic_idx(wrap_idx(iz, d.n3), d.n3, zo);
  float acc = 0.0f;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const auto pl = src.plane(xo[a], psz);
    float sa = 0.0f;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = yo[b] * d.n3;
      sa += wy[b] * (wz[0] * src.at(pl, r + zo[0]) + wz[1] * src.at(pl, r + zo[1]) + wz[2] * src.at(pl, r + zo[2]) +
                     wz[3] * src.at(pl, r + zo[3]));
    }
    acc += wx[a] * sa;
  }
  return acc;
}

// Generic staged tricubic sweep: out voxel idx <- epi(idx, interp(src, departure(idx)))
// over output x1 planes [x_begin, x_begin + x_count) of the (local) dims d.
template <bool SLAB, class S, class Epi>
__global__ void __launch_bounds__(256, 3) quad_sweep_kernel(S src, Dims d, int w, int x_begin, int x_count,
                                                            const float* __restrict__ disp, Epi epi) {
  extern __shared__ float4 quads[];
  __shared__ int ext[6];
  const int64_t N = d.n();
  const int L1 = d.n1;
  const int z0 = blockIdx.x * TZ, y0 = blockIdx.y * TY, x0 = x_begin + blockIdx.z * TX;
  const int x_end = x_begin + x_count;
  const int k = z0 + threadIdx.x, j = y0 + threadIdx.y;
  const int tid = threadIdx.y * TZ + threadIdx.x;
  if (tid < 6) ext[tid] = (tid < 3) ? INT_MAX : INT_MIN;
  int ix[TX], iy[TX], iz[TX];
  float fx[TX], fy[TX], fz[TX];
  int mn0 = INT_MAX, mn1 = INT_MAX, mn2 = INT_MAX, mx0 = INT_MIN, mx1 = INT_MIN, mx2 = INT_MIN;
  const bool inyz = (j < d.n2) && (k < d.n3);
#pragma unroll
  for (int u = 0; u < TX; ++u) {
    const int i = x0 + u;
    ix[u] = iy[u] = iz[u] = 0;
    fx[u] = fy[u] = fz[u] = 0.0f;
    if (inyz && i < x_end) {
      const int idx = (i * d.n2 + j) * d.n3 + k;
      split_coord(i, __ldg(disp + idx), ix[u], fx[u]);
      split_coord(j, __ldg(disp + N + idx), iy[u], fy[u]);
      split_coord(k, __ldg(disp + 2 * N + idx), iz[u], fz[u]);
      if (SLAB) ix[u] = clampi(ix[u], 1 - w, L1 + w - 3);
      mn0 = min(mn0, ix[u]); mx0 = max(mx0, ix[u]);
      mn1 = min(mn1, iy[u]); mx1 = max(mx1, iy[u]);
      mn2 = min(mn2, iz[u]); mx2 = max(mx2, iz[u]);
    }
  }
  mn0 = __reduce_min_sync(0xffffffffu, mn0);
  mn1 = __reduce_min_sync(0xffffffffu, mn1);
  mn2 = __reduce_min_sync(0xffffffffu, mn2);
  mx0 = __reduce_max_sync(0xffffffffu, mx0);
  mx1 = __reduce_max_sync(0xffffffffu, mx1);
  mx2 = __reduce_max_sync(0xffffffffu, mx2);
  __syncthreads();
  if ((tid & 31) == 0) {
    atomicMin(&ext[0], mn0); atomicMin(&ext[1], mn1); atomicMin(&ext[2], mn2);
    atomicMax(&ext[3], mx0); atomicMax(&ext[4], mx1); atomicMax(&ext[5], mx2);
  }
  __syncthreads();
  // box of stencil rows: x1 [lo0-1, hi0+2], x2 [lo1-1, hi1+2]; quads start at x3 lo2-1 .. hi2-1
  const int bx0 = ext[0] - 1, by0 = ext[1] - 1, qz0 = ext[2] - 1;
  const int BX = ext[3] - ext[0] + 4, BY = ext[4] - ext[1] + 4, QZ = ext[5] - ext[2] + 1;
  const bool use_box = BX <= d.n1 + (SLAB ? 2 * w : 0) && BY <= d.n2 && QZ + 3 <= d.n3 && QZ <= 2 * 29 &&
                       (int64_t)BX * BY * QZ <= QCAP;
  const int psz = d.n2 * d.n3;
  if (use_box) {
    // staging: warp w owns box x1 rows a = w, w+8, ... (one plane pointer each)
    // and walks its x2 rows 4 at a time with an incremental conditional wrap; a
    // row is read in 29-quad windows -- lane l loads f[c0+l] once (coalesced)
    // and lanes l < 29 assemble quad (f[l], f[l+1], f[l+2], f[l+3]) with
    // shuffles, so every float is loaded once and 8 loads are in flight.
    const int warp = tid >> 5, lane = tid & 31;
    constexpr int RPI = 4, WPR = 2, QW = 29;
    int z_lo[WPR];
#pragma unroll
    for (int q = 0; q < WPR; ++q) {   // x3 index of this lane's element in window q
      int z = wrap_idx(qz0, d.n3) + q * QW + lane;
      z = z >= d.n3 ? z - d.n3 : z;
      z_lo[q] = z >= d.n3 ? z - d.n3 : z;
    }
    const int gy0 = wrap_idx(by0, d.n2);
    for (int a = warp; a < BX; a += 8) {
      const int gx = SLAB ? bx0 + a : wrap_idx(bx0 + a, d.n1);
      const auto pl = src.plane(gx, psz);
      for (int b0 = 0; b0 < BY; b0 += RPI) {
        float v[RPI][WPR];
#pragma unroll
        for (int r = 0; r < RPI; ++r) {
          int gy = gy0 + b0 + r;
          gy = gy >= d.n2 ? gy - d.n2 : gy;
          const bool rok = b0 + r < BY;
          const int rbase = (rok ? gy : 0) * d.n3;
#pragma unroll
          for (int q = 0; q < WPR; ++q)
            v[r][q] = (rok && q * QW + lane < QZ + 3) ? src.at(pl, rbase + z_lo[q]) : 0.0f;
        }
#pragma unroll
        for (int r = 0; r < RPI; ++r) {
          float4* qrow = quads + (a * BY + b0 + r) * QZ;
#pragma unroll
          for (int q = 0; q < WPR; ++q) {
            const float x0v = v[r][q];
            const float x1v = __shfl_down_sync(0xffffffffu, x0v, 1);
            const float x2v = __shfl_down_sync(0xffffffffu, x0v, 2);
            const float x3v = __shfl_down_sync(0xffffffffu, x0v, 3);
            const int c = q * QW + lane;
            if (b0 + r < BY && lane < QW && c < QZ) qrow[c] = make_float4(x0v, x1v, x2v, x3v);
          }
        }
      }
    }
    __syncthreads();
  }
  const int sa_row = BY * QZ;  // x1 stride in quads
#pragma unroll
  for (int u = 0; u < TX; ++u) {
    const int i = x0 + u;
    if (!(inyz && i < x_end)) continue;
    float o;
    if (use_box) {
      float wx[4], wy[4], wz[4];
      lagrange4(fx[u], wx);
      lagrange4(fy[u], wy);
      lagrange4(fz[u], wz);
      const float4* q = quads + ((ix[u] - 1 - bx0) * BY + (iy[u] - 1 - by0)) * QZ + (iz[u] - 1 - qz0);
      float acc = 0.0f;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        float sa = 0.0f;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const float4 v = q[a * sa_row + b * QZ];
          sa += wy[b] * (wz[0] * v.x + wz[1] * v.y + wz[2] * v.z + wz[3] * v.w);
        }
        acc += wx[a] * sa;
      }
      o = acc;
    } else {
      o = direct_cubic<SLAB>(src, d, w, L1, ix[u], iy[u], iz[u], fx[u], fy[u], fz[u]);
    }
    epi((i * d.n2 + j) * d.n3 + k, o);
  }
}

// ---- epilogues ---------------------------------------------------------------------
struct EpiStore {  // state / adjoint / Jacobian step: dst = interp [* fac]
  float* __restrict__ dst;
  const float* __restrict__ fac;
  int* flag;
  __device__ __forceinline__ void operator()(int idx, float o) const {
    if (fac) o *= __ldg(fac + idx);
    dst[idx] = o;
    if (flag && !isfinite(o)) atomicOr(flag, 1);
  }
};

struct EpiInc {  // incremental state step (transport.py:174-183)
  const float* __restrict__ vt;
  const float* __restrict__ g;
  int64_t N;
  float half;
  int last;
  float* __restrict__ dst;
  int* flag;
  __device__ __forceinline__ void operator()(int idx, float o) const {
    const float s = -(__ldg(vt + idx) * __ldg(g + idx) + __ldg(vt + N + idx) * __ldg(g + N + idx) +
                      __ldg(vt + 2 * N + idx) * __ldg(g + 2 * N + idx));
    const float hs = half * s;
    float m = o + hs;
    if (last == 0) m = m + hs;
    else if (last == 2) m = -m;
    dst[idx] = m;
    if (flag && !isfinite(m)) atomicOr(flag, 1);
  }
};

struct EpiLabel {  // label transport: float indicator or thresholded label write
  float* __restrict__ dst;
  int* __restrict__ lab_out;
  int id;
  __device__ __forceinline__ void operator()(int idx, float o) const {
    if (lab_out) {
      if (o >= 0.5f) lab_out[idx] = id;
    } else {
      dst[idx] = o;
    }
  }
};

inline dim3 sweep_grid(const Dims& d, int nplanes) {
  return dim3((d.n3 + TZ - 1) / TZ, (d.n2 + TY - 1) / TY, (nplanes + TX - 1) / TX);
}
inline dim3 sweep_block() { return dim3(TZ, TY); }

}  // namespace staged
}  // namespace vr
