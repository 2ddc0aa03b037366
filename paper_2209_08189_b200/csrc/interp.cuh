// Periodic trilinear / tricubic-Lagrange gathers (device side).
//
// Semantics follow /root/reference/pkg/src/velreg/interp.py:
//   trilinear  : interp.py:19-44 (8 taps, z innermost, then y, then x)
//   tricubic   : interp.py:47-103 (Lagrange weights on offsets {-1,0,1,2},
//                weights interp.py:61-72, z-fastest accumulation :73-103)
// Indices are wrapped periodically (Python `%` semantics, never negative).
// Arithmetic is fp32 here (the reference uses f64 internally); the measured
// difference is ~1e-7 relative, far inside the 1e-5 operator tolerance.
#pragma once
#include "common.cuh"

namespace vr {

enum { ORDER_LINEAR = 1, ORDER_CUBIC = 3 };

// Source adaptors: value at flat voxel index `idx` of component `c`.
struct SrcF32 {
  const float* __restrict__ p[3];
  int64_t stride;  // component stride (unused for 1-component sources)
  __device__ __forceinline__ float operator()(int c, int idx) const { return __ldg(p[c] + idx); }
};

// Indicator of one label id read straight from an int32 label map
// (pkg/synth.py:125: (labels == lab).astype(float)).
struct SrcLabel {
  const int* __restrict__ lab;
  int id;
  __device__ __forceinline__ float operator()(int, int idx) const {
    return __ldg(lab + idx) == id ? 1.0f : 0.0f;
  }
};

__device__ __forceinline__ void lagrange4(float t, float w[4]) {
  // interp.py:61-64
  const float tm1 = t - 1.0f, tm2 = t - 2.0f, tp1 = t + 1.0f;
  w[0] = -t * tm1 * tm2 * (1.0f / 6.0f);
  w[1] = (t * t - 1.0f) * tm2 * 0.5f;
  w[2] = -t * tp1 * tm2 * 0.5f;
  w[3] = t * (t * t - 1.0f) * (1.0f / 6.0f);
}

// wrapped neighbour offsets i0-1 .. i0+2 for a base index already in [0,n)
__device__ __forceinline__ void cubic_idx(int i0, int n, int o[4]) {
  int m = i0 - 1;
  o[0] = m < 0 ? m + n : m;
  o[1] = i0;
  int p = i0 + 1;
  o[2] = p >= n ? p - n : p;
  int q = i0 + 2;
  o[3] = q >= n ? q - n : q;
}

// NC components sharing one set of weights (the RK2 trace interpolates all
// three velocity components at the same point, pkg/transport.py:74).
template <int NC, class Src>
__device__ __forceinline__ void gather_linear(const Src& src, const Dims& d, int ix, int iy, int iz,
                                              float tx, float ty, float tz, float* out) {
  const int i0 = wrap_idx(ix, d.n1), j0 = wrap_idx(iy, d.n2), k0 = wrap_idx(iz, d.n3);
  const int i1 = next_wrap(i0, d.n1), j1 = next_wrap(j0, d.n2), k1 = next_wrap(k0, d.n3);
  const int r00 = (i0 * d.n2 + j0) * d.n3, r01 = (i0 * d.n2 + j1) * d.n3;
  const int r10 = (i1 * d.n2 + j0) * d.n3, r11 = (i1 * d.n2 + j1) * d.n3;
  const float sz = 1.0f - tz, sy = 1.0f - ty, sx = 1.0f - tx;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float c00 = src(c, r00 + k0) * sz + src(c, r00 + k1) * tz;
    float c01 = src(c, r01 + k0) * sz + src(c, r01 + k1) * tz;
    float c10 = src(c, r10 + k0) * sz + src(c, r10 + k1) * tz;
    float c11 = src(c, r11 + k0) * sz + src(c, r11 + k1) * tz;
    float c0 = c00 * sy + c01 * ty;
    float c1 = c10 * sy + c11 * ty;
    out[c] = c0 * sx + c1 * tx;
  }
}

template <int NC, class Src>
__device__ __forceinline__ void gather_cubic(const Src& src, const Dims& d, int ix, int iy, int iz,
                                             float tx, float ty, float tz, float* out) {
  float wx[4], wy[4], wz[4];
  lagrange4(tx, wx);
  lagrange4(ty, wy);
  lagrange4(tz, wz);
  int xo[4], yo[4], zo[4];
  cubic_idx(wrap_idx(ix, d.n1), d.n1, xo);
  cubic_idx(wrap_idx(iy, d.n2), d.n2, yo);
  cubic_idx(wrap_idx(iz, d.n3), d.n3, zo);
  float acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0f;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int xa = xo[a] * d.n2;
    float sa[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) sa[c] = 0.0f;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int row = (xa + yo[b]) * d.n3;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        float sb = wz[0] * src(c, row + zo[0]) + wz[1] * src(c, row + zo[1]) +
                   wz[2] * src(c, row + zo[2]) + wz[3] * src(c, row + zo[3]);
        sa[c] += wy[b] * sb;
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] += wx[a] * sa[c];
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) out[c] = acc[c];
}

// 3-component source interleaved as float4 (v1, v2, v3, -): one 16-byte load
// per tap instead of three scalar loads from three planes (the RK2 trace's
// velocity gathers).  The arithmetic is gather_cubic / gather_linear's,
// component by component, so the results are identical.
struct SrcAoS4 {
  const float4* __restrict__ q;
  __device__ __forceinline__ float4 operator()(int idx) const { return __ldg(q + idx); }
};

template <int ORDER>
__device__ __forceinline__ void gather_aos3(const SrcAoS4& src, const Dims& d, int ix, int iy, int iz, float tx,
                                            float ty, float tz, float* out) {
  if (ORDER == ORDER_LINEAR) {
    const int i0 = wrap_idx(ix, d.n1), j0 = wrap_idx(iy, d.n2), k0 = wrap_idx(iz, d.n3);
    const int i1 = next_wrap(i0, d.n1), j1 = next_wrap(j0, d.n2), k1 = next_wrap(k0, d.n3);
    const int r00 = (i0 * d.n2 + j0) * d.n3, r01 = (i0 * d.n2 + j1) * d.n3;
    const int r10 = (i1 * d.n2 + j0) * d.n3, r11 = (i1 * d.n2 + j1) * d.n3;
    const float sz = 1.0f - tz, sy = 1.0f - ty, sx = 1.0f - tx;
    const float4 a00 = src(r00 + k0), b00 = src(r00 + k1), a01 = src(r01 + k0), b01 = src(r01 + k1);
    const float4 a10 = src(r10 + k0), b10 = src(r10 + k1), a11 = src(r11 + k0), b11 = src(r11 + k1);
    const float A00[3] = {a00.x, a00.y, a00.z}, B00[3] = {b00.x, b00.y, b00.z};
    const float A01[3] = {a01.x, a01.y, a01.z}, B01[3] = {b01.x, b01.y, b01.z};
    const float A10[3] = {a10.x, a10.y, a10.z}, B10[3] = {b10.x, b10.y, b10.z};
    const float A11[3] = {a11.x, a11.y, a11.z}, B11[3] = {b11.x, b11.y, b11.z};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float c00 = A00[c] * sz + B00[c] * tz;
      const float c01 = A01[c] * sz + B01[c] * tz;
      const float c10 = A10[c] * sz + B10[c] * tz;
      const float c11 = A11[c] * sz + B11[c] * tz;
      const float c0 = c00 * sy + c01 * ty;
      const float c1 = c10 * sy + c11 * ty;
      out[c] = c0 * sx + c1 * tx;
    }
  } else {
    float wx[4], wy[4], wz[4];
    lagrange4(tx, wx);
    lagrange4(ty, wy);
    lagrange4(tz, wz);
    int xo[4], yo[4], zo[4];
    cubic_idx(wrap_idx(ix, d.n1), d.n1, xo);
    cubic_idx(wrap_idx(iy, d.n2), d.n2, yo);
    cubic_idx(wrap_idx(iz, d.n3), d.n3, zo);
    float acc[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int xa = xo[a] * d.n2;
      float sa[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int row = (xa + yo[b]) * d.n3;
        const float4 t0 = src(row + zo[0]), t1 = src(row + zo[1]), t2 = src(row + zo[2]), t3 = src(row + zo[3]);
        const float T0[3] = {t0.x, t0.y, t0.z}, T1[3] = {t1.x, t1.y, t1.z};
        const float T2[3] = {t2.x, t2.y, t2.z}, T3[3] = {t3.x, t3.y, t3.z};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float sb = wz[0] * T0[c] + wz[1] * T1[c] + wz[2] * T2[c] + wz[3] * T3[c];
          sa[c] += wy[b] * sb;
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] += wx[a] * sa[c];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) out[c] = acc[c];
  }
}

template <int ORDER, int NC, class Src>
__device__ __forceinline__ void gather(const Src& src, const Dims& d, int ix, int iy, int iz, float tx,
                                       float ty, float tz, float* out) {
  if (ORDER == ORDER_LINEAR)
    gather_linear<NC>(src, d, ix, iy, iz, tx, ty, tz, out);
  else
    gather_cubic<NC>(src, d, ix, iy, iz, tx, ty, tz, out);
}

// ---- lean gather for the transport sweeps --------------------------------------
// Same arithmetic as gather<> but instruction-lean: the base index is wrapped
// with one conditional per axis, every stencil row gets one row pointer and its
// taps are immediate-offset loads unless the x3 window wraps at the end of the
// row.  SLAB: the source is this rank's x1 slab (L1 planes) plus separate
// ghost blocks of w planes before (lo) and after (hi) it, filled by the host's
// halo exchange (dist.py); x1 is never wrapped and is clamped into [-w, L1+w).
__device__ __forceinline__ int wrap1(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }
__device__ __forceinline__ int clampi(int i, int lo, int hi) { return i < lo ? lo : (i > hi ? hi : i); }

// Component c of every block lives at base + c * stride (vector fields are
// SoA: (3, L1, N2, N3) local, (3, w, N2, N3) ghosts).
template <int NC, bool SLAB>
struct PlaneSrc {
  const float* mid;      // local field (periodic case: the whole field)
  const float* lo;       // SLAB: ghost planes [-w, 0)
  const float* hi;       // SLAB: ghost planes [L1, L1 + w)
  int64_t mid_cs, ghost_cs;
  int w, L1;
  __device__ __forceinline__ const float* plane(int c, int x, int psz) const {
    if (!SLAB) return mid + c * mid_cs + (int64_t)x * psz;
    if (x < 0) return lo + c * ghost_cs + (int64_t)(x + w) * psz;
    if (x < L1) return mid + c * mid_cs + (int64_t)x * psz;
    return hi + c * ghost_cs + (int64_t)(x - L1) * psz;
  }
};

template <int ORDER, int NC, bool SLAB>
__device__ __forceinline__ void gather_lean(const PlaneSrc<NC, SLAB>& src, const Dims& d, int ix, int iy, int iz,
                                            float tx, float ty, float tz, float* out) {
  // d = arrival dims (for SLAB d.n1 = L1); ix is a local x1 index
  const int psz = d.n2 * d.n3;
  if (ORDER == ORDER_LINEAR) {
    const int i0 = SLAB ? clampi(ix, -src.w, src.L1 + src.w - 2) : wrap1(ix, d.n1);
    const int j0 = wrap1(iy, d.n2), k0 = wrap1(iz, d.n3);
    const int i1 = SLAB ? i0 + 1 : next_wrap(i0, d.n1), j1 = next_wrap(j0, d.n2);
    const bool zin = k0 + 1 < d.n3;
    const int dk = zin ? 1 : 1 - d.n3;
    const int r0 = j0 * d.n3 + k0, r1 = j1 * d.n3 + k0;
    const float sz = 1.0f - tz, sy = 1.0f - ty, sx = 1.0f - tx;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const float* b0 = src.plane(c, i0, psz);
      const float* b1 = src.plane(c, i1, psz);
      const float c00 = __ldg(b0 + r0) * sz + __ldg(b0 + r0 + dk) * tz;
      const float c01 = __ldg(b0 + r1) * sz + __ldg(b0 + r1 + dk) * tz;
      const float c10 = __ldg(b1 + r0) * sz + __ldg(b1 + r0 + dk) * tz;
      const float c11 = __ldg(b1 + r1) * sz + __ldg(b1 + r1 + dk) * tz;
      const float c0 = c00 * sy + c01 * ty;
      const float c1 = c10 * sy + c11 * ty;
      out[c] = c0 * sx + c1 * tx;
    }
  } else {
    float wx[4], wy[4], wz[4];
    lagrange4(tx, wx);
    lagrange4(ty, wy);
    lagrange4(tz, wz);
    const int j0 = wrap1(iy, d.n2), k0 = wrap1(iz, d.n3);
    int xo[4], yo[4];
    if (SLAB) {
      const int i0 = clampi(ix, 1 - src.w, src.L1 + src.w - 3);
      xo[0] = i0 - 1; xo[1] = i0; xo[2] = i0 + 1; xo[3] = i0 + 2;
    } else {
      cubic_idx(wrap1(ix, d.n1), d.n1, xo);
    }
    cubic_idx(j0, d.n2, yo);
    float acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0f;
    if (k0 >= 1 && k0 + 2 < d.n3) {  // x3 window inside the row: immediate-offset taps
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        float sa[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) sa[c] = 0.0f;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const float* r = src.plane(c, xo[a], psz) + (yo[b] * d.n3 + k0 - 1);
            const float sb = wz[0] * __ldg(r) + wz[1] * __ldg(r + 1) + wz[2] * __ldg(r + 2) + wz[3] * __ldg(r + 3);
            sa[c] += wy[b] * sb;
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] += wx[a] * sa[c];
      }
    } else {
      int zo[4];
      cubic_idx(k0, d.n3, zo);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        float sa[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) sa[c] = 0.0f;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const float* row = src.plane(c, xo[a], psz) + yo[b] * d.n3;
            const float sb = wz[0] * __ldg(row + zo[0]) + wz[1] * __ldg(row + zo[1]) + wz[2] * __ldg(row + zo[2]) +
                             wz[3] * __ldg(row + zo[3]);
            sa[c] += wy[b] * sb;
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] += wx[a] * sa[c];
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) out[c] = acc[c];
  }
}

// Departure point of arrival voxel (i,j,k) displaced by -(d1,d2,d3); huge
// displacements (|d| >= n - 4) are pre-wrapped with a full modulo.
template <int ORDER, int NC, bool SLAB>
__device__ __forceinline__ void gather_disp_lean(const PlaneSrc<NC, SLAB>& src, const Dims& d, int i, int j, int k,
                                                 float d1, float d2, float d3, float* out) {
  int ix, iy, iz;
  float tx, ty, tz;
  split_coord(i, d1, ix, tx);
  split_coord(j, d2, iy, ty);
  split_coord(k, d3, iz, tz);
  if (!SLAB && !(fabsf(d1) < d.n1 - 4)) ix = wrap_idx(ix, d.n1);
  if (!(fabsf(d2) < d.n2 - 4)) iy = wrap_idx(iy, d.n2);
  if (!(fabsf(d3) < d.n3 - 4)) iz = wrap_idx(iz, d.n3);
  gather_lean<ORDER, NC, SLAB>(src, d, ix, iy, iz, tx, ty, tz, out);
}

// Gather at voxel (i,j,k) displaced by -(d1,d2,d3) index units.
template <int ORDER, int NC, class Src>
__device__ __forceinline__ void gather_disp(const Src& src, const Dims& d, int i, int j, int k, float d1,
                                            float d2, float d3, float* out) {
  int ix, iy, iz;
  float tx, ty, tz;
  split_coord(i, d1, ix, tx);
  split_coord(j, d2, iy, ty);
  split_coord(k, d3, iz, tz);
  gather<ORDER, NC>(src, d, ix, iy, iz, tx, ty, tz, out);
}

}  // namespace vr
