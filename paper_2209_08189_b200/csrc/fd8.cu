// 8th-order centred finite differences with periodic wrap
// (/root/reference/pkg/src/velreg/diffops.py:84-105, coefficients :20).
//
// The arithmetic sequence is the reference's, in fp32, without FMA contraction:
//   out = 0; for o in 1..4: out += c_o * (f[i+o] - f[i-o]);  out /= h
// so fp32 inputs give bit-identical outputs to numpy's fp32 evaluation.
// divergence: out = d1 v1; out += d2 v2; out += d3 v3   (diffops.py:102-104)
//
// Tiling: one CTA (16 x 16 threads) = a 32 x 32 (x2, x3) tile; each thread owns
// a 2 (x3) x 2 (x2) micro-tile and walks nx consecutive x1-planes keeping the
// 9-deep x1 stencil windows in registers.  The x2/x3 halos come from per-plane
// shared-memory tiles filled by 8-byte cp.async copies NS-1 planes ahead
// (a ring of NS stages), read back as aligned float2.
#include <algorithm>
#include "common.cuh"
#include "../../include/velreg_b200.h"

namespace vr {

// numpy evaluates `c * (...)` on fp32 arrays with c rounded to fp32 from the
// Python float (NEP 50), hence the double -> float conversions.
__constant__ float kFd8[4] = {(float)(4.0 / 5.0), (float)(-1.0 / 5.0), (float)(4.0 / 105.0),
                              (float)(-1.0 / 280.0)};

// x / h correctly rounded from the precomputed r = RN(1/h) (Markstein):
// q = RN(x r) is within 1 ulp of x/h, e = x - q h is exact by FMA, and
// RN(q + e r) = RN(x/h) -- the same bits as IEEE division, in 3 instructions.
// tools/recip_div_check.cu verifies this exhaustively over all 2^32 float32
// x for every h = fp32(2 pi / n), n even in [10, 8192]: every mismatch has
// |x| < 2^-102 or |x| >= 2^117.  Outside [2^-60, 2^60) (zero excepted) the
// kernel therefore takes IEEE division.
__device__ __forceinline__ float div_fast(float x, float h, float r) {
  const float q = __fmul_rn(x, r);
  const float e = __fmaf_rn(-q, h, x);
  return __fmaf_rn(e, r, q);
}
// |x| outside [2^-60, 2^60) and not 0: take IEEE division
__device__ __forceinline__ bool div_needs_ieee(float x, unsigned lo, unsigned span) {
  const unsigned u = __float_as_uint(x) & 0x7fffffffu;
  return u != 0u && (u - lo) >= span;
}

// c1*(p1-m1) + c2*(p2-m2) + c3*(p3-m3) + c4*(p4-m4) in the reference's order
// (before the division by h).  The reference starts from out = 0 and adds
// c1*(p1-m1) first; 0 + x == x bit for bit because c1 > 0 and p1 - m1 is never
// -0 under RN.
__device__ __forceinline__ float fd8_sum(float p0, float p1, float p2, float p3, float m0, float m1, float m2,
                                         float m3) {
  float out = __fmul_rn(kFd8[0], __fsub_rn(p0, m0));
  out = __fadd_rn(out, __fmul_rn(kFd8[1], __fsub_rn(p1, m1)));
  out = __fadd_rn(out, __fmul_rn(kFd8[2], __fsub_rn(p2, m2)));
  out = __fadd_rn(out, __fmul_rn(kFd8[3], __fsub_rn(p3, m3)));
  return out;
}

// The 12 sums of one micro-tile step (x1 / x2 / x3 derivative, 4 voxels each)
// divided by h: IEEE division where the reciprocal form is not proven exact.
struct F12 {
  float v[12];
};
__device__ __noinline__ F12 fd8_div_ieee(F12 s, float h1, float h2, float h3, float r1, float r2, float r3,
                                         unsigned dlo, unsigned dspan) {
  // Tiny sums with a normal quotient (2^-125 <= |x/h|, |x| < 2^-100) are
  // scaled by 2^64 into the verified range first: both scalings are exact.
  const bool verified = dlo == 0x0d800000u;
  F12 o;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    const float h = i < 4 ? h1 : (i < 8 ? h2 : h3), r = i < 4 ? r1 : (i < 8 ? r2 : r3);
    const float x = s.v[i], ax = fabsf(x);
    if (!div_needs_ieee(x, dlo, dspan))
      o.v[i] = div_fast(x, h, r);
    else if (verified && ax < 0x1p-100f && ax >= 0x1p-125f * h)
      o.v[i] = __fmul_rn(div_fast(__fmul_rn(x, 0x1p64f), h, r), 0x1p-64f);
    else
      o.v[i] = __fdiv_rn(x, h);
  }
  return o;
}

template <int V>
struct IC {
  static constexpr int value = V;
};

// Thread micro-tile: 2 consecutive x3 voxels x RY consecutive x2 rows, walked
// along x1.  CTA = TXB x TYB threads = a TY x TZ (x2, x3) tile.
constexpr int TXB = 16, TYB = 16, RY = 2, TZ = 2 * TXB, TY = RY * TYB, HALO = 4, NTHR = TXB * TYB;
constexpr int NS = 4;  // cp.async ring depth (plane steps in flight)

// One plane step in shared memory.  MODE 0 (gradient): a (TY+8) x (TZ+8) tile
// of f.  MODE 1 (divergence): a (TY+8) x TZ tile of v2 (x2 halo only) and a
// TY x (TZ+8) tile of v3 (x3 halo only).  Both carry the TY x TZ x1-values of
// the plane 4 ahead (the leading edge of the x1 register windows).  Rows are
// unpadded: every access is an aligned float2 and a warp reads two whole rows.
template <int MODE> struct Fd8Stage;
template <> struct Fd8Stage<0> {
  static constexpr int H = TY + 2 * HALO, W = TZ + 2 * HALO;
  static constexpr int PAIRS = H * W / 2, EPT = (PAIRS + NTHR - 1) / NTHR;
  float a[H * W];
  float xc[TY * TZ];
};
template <> struct Fd8Stage<1> {
  static constexpr int HY = TY + 2 * HALO, WY = TZ, HZ = TY, WZ = TZ + 2 * HALO;
  static constexpr int PAIRS = (HY * WY + HZ * WZ) / 2, EPT = (PAIRS + NTHR - 1) / NTHR;
  float y[HY * WY];
  float z[HZ * WZ];
  float xc[TY * TZ];
};

__device__ __forceinline__ int wrapmod(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

__device__ __forceinline__ void cp8(float* dst, const float* src) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ float2 lds2(const float* p) { return *reinterpret_cast<const float2*>(p); }

// MODE 0: gradient of a scalar (3 outputs); MODE 1: divergence of a vector.
// SLAB: f is this rank's x1 slab (d = local dims, no x1 wrap); the x1 windows
// read the 4 ghost planes before (lo) / after (hi) it.  The x2/x3 tiles only
// ever read local planes.  Requires N3 even (the reference grid's dims are).
template <int MODE, bool SLAB>
__global__ void __launch_bounds__(NTHR, 2) fd8_kernel(const float* __restrict__ f, const float* __restrict__ lo,
                                                      const float* __restrict__ hi, Dims d, float h1, float h2,
                                                      float h3, float r1, float r2, float r3, unsigned dlo,
                                                      unsigned dspan,
                                                      float* __restrict__ out, int nchunk) {
  using T = Fd8Stage<MODE>;
  constexpr int EPT = T::EPT;
  extern __shared__ __align__(16) unsigned char fd8_smem[];
  T* ring = reinterpret_cast<T*>(fd8_smem);
  const int64_t N = d.n();
  const int psz = d.n2 * d.n3;
  // CTA b = (tile b % ntiles, x1 chunk b / ntiles): the CTAs resident at the
  // same time sweep the same x1 planes in step, so the x2/x3 halo rows one
  // tile reads are still in L2 when its neighbour tiles read them.
  const int tiles_z = (d.n3 + TZ - 1) / TZ, tiles_y = (d.n2 + TY - 1) / TY;
  const int ntiles = tiles_z * tiles_y;
  for (int b = blockIdx.x; b < ntiles * nchunk; b += gridDim.x) {
    const int tile = b % ntiles, chunk = b / ntiles;
    const int i_begin = (int)((int64_t)d.n1 * chunk / nchunk);
    const int i_end = (int)((int64_t)d.n1 * (chunk + 1) / nchunk);
    if (i_begin >= i_end) continue;
    __syncthreads();  // previous segment's readers are done with the ring
    const int k0 = (tile % tiles_z) * TZ, j0 = (tile / tiles_z) * TY;
    const int tid = threadIdx.y * TXB + threadIdx.x;
    const int zl = 2 * threadIdx.x, yl = RY * threadIdx.y;  // tile-local x3 / x2 of the micro-tile
    const int k = k0 + zl;

    // ---- per-thread tile pair map (plane-invariant) ----
    int goff[EPT];  // plane offset of the pair (+ component * N for MODE 1), or -1
    int slot[EPT];  // float index within a stage
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int t = tid + e * NTHR;
      goff[e] = -1;
      slot[e] = 0;
      if (t >= T::PAIRS) continue;
      int yy, zz, jo, ko, comp, sidx;
      if constexpr (MODE == 0) {
        yy = t / (T::W / 2); zz = 2 * (t - yy * (T::W / 2));
        comp = 0; jo = yy - HALO; ko = zz - HALO;
        sidx = yy * T::W + zz;
      } else {
        if (t < T::HY * T::WY / 2) {
          yy = t / (T::WY / 2); zz = 2 * (t - yy * (T::WY / 2));
          comp = 1; jo = yy - HALO; ko = zz;
          sidx = yy * T::WY + zz;
        } else {
          const int u = t - T::HY * T::WY / 2;
          yy = u / (T::WZ / 2); zz = 2 * (u - yy * (T::WZ / 2));
          comp = 2; jo = yy; ko = zz - HALO;
          sidx = T::HY * T::WY + yy * T::WZ + zz;
        }
      }
      const int jr = j0 + jo, kr = k0 + ko;
      if (jr >= d.n2 + HALO || kr >= d.n3 + HALO) continue;  // read by no active output
      goff[e] = wrapmod(jr, d.n2) * d.n3 + wrapmod(kr, d.n3);
      slot[e] = sidx | (comp << 24);
    }

    bool act[RY];
    int rowoff[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const int j = j0 + yl + r;
      act[r] = k < d.n3 && j < d.n2;
      rowoff[r] = act[r] ? j * d.n3 + k : 0;
    }
    auto xplane = [&](int ii) -> const float* {  // component 0, plane ii in [-4, L1 + 4)
      if (SLAB) return ii < 0 ? lo + (int64_t)(ii + HALO) * psz
                              : (ii >= d.n1 ? hi + (int64_t)(ii - d.n1) * psz : f + (int64_t)ii * psz);
      ii = ii < 0 ? ii + d.n1 : (ii >= d.n1 ? ii - d.n1 : ii);  // n1 >= 9 (caller)
      return f + (int64_t)ii * psz;
    };
    // plane step p: x2/x3 tile(s) of plane p + x1 values of plane p + 4
    auto issue = [&](int p) {
      T& st = ring[p % NS];
      float* sf = reinterpret_cast<float*>(&st);
      const float* pl = f + (int64_t)p * psz;
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        if (goff[e] < 0) continue;
        cp8(sf + (slot[e] & 0xffffff), pl + (int64_t)(slot[e] >> 24) * N + goff[e]);
      }
      const float* xp = xplane(p + HALO);
#pragma unroll
      for (int r = 0; r < RY; ++r)
        if (act[r]) cp8(st.xc + (yl + r) * TZ + zl, xp + rowoff[r]);
    };

    // x1 windows: logical o (plane i-4+o) of row r, x3 column c lives in
    // w[r][c][(S + o) % 9] at unrolled step S -- a compile-time rotation, no moves.
    float w[RY][2][9];
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const float* pl = xplane(i_begin - HALO + o);
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const float2 v = act[r] ? __ldg(reinterpret_cast<const float2*>(pl + rowoff[r])) : make_float2(0.f, 0.f);
        w[r][0][o] = v.x;
        w[r][1][o] = v.y;
      }
    }
#pragma unroll
    for (int q = 0; q < NS - 1; ++q) {
      if (i_begin + q < i_end) issue(i_begin + q);
      cp_commit();
    }
    float* op = out + (int64_t)i_begin * psz;

    auto step = [&](auto S_, int i) {
      constexpr int S = decltype(S_)::value;
      __syncthreads();  // every reader of the stage about to be refilled is done
      if (i + NS - 1 < i_end) issue(i + NS - 1);
      cp_commit();
      cp_wait<NS - 1>();
      __syncthreads();
      const T& st = ring[i % NS];
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const float2 v = lds2(st.xc + (yl + r) * TZ + zl);
        w[r][0][(S + 8) % 9] = v.x;
        w[r][1][(S + 8) % 9] = v.y;
      }
      float g1[RY][2], g2[RY][2], g3[RY][2];
#pragma unroll
      for (int r = 0; r < RY; ++r) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float* x = w[r][c];
          g1[r][c] = fd8_sum(x[(S + 5) % 9], x[(S + 6) % 9], x[(S + 7) % 9], x[(S + 8) % 9], x[(S + 3) % 9],
                             x[(S + 2) % 9], x[(S + 1) % 9], x[S % 9]);
        }
      }
      // x2: rows yl-4 .. yl+RY+3 of the two x3 columns
      {
        const float* ybase;
        int ys;
        if constexpr (MODE == 0) { ybase = st.a + HALO; ys = T::W; }
        else { ybase = st.y; ys = T::WY; }
        float Y[RY + 8][2];
#pragma unroll
        for (int q = 0; q < RY + 8; ++q) {
          const float2 v = lds2(ybase + (yl + q) * ys + zl);
          Y[q][0] = v.x;
          Y[q][1] = v.y;
        }
#pragma unroll
        for (int r = 0; r < RY; ++r) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int m = r + HALO;
            g2[r][c] = fd8_sum(Y[m + 1][c], Y[m + 2][c], Y[m + 3][c], Y[m + 4][c], Y[m - 1][c], Y[m - 2][c],
                               Y[m - 3][c], Y[m - 4][c]);
          }
        }
      }
      // x3: columns zl-4 .. zl+5 of each row
      {
        const float* zbase;
        int zs;
        if constexpr (MODE == 0) { zbase = st.a + HALO * T::W; zs = T::W; }
        else { zbase = st.z; zs = T::WZ; }
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          float Z[10];
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            const float2 v = lds2(zbase + (yl + r) * zs + zl + 2 * q);
            Z[2 * q] = v.x;
            Z[2 * q + 1] = v.y;
          }
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int m = c + HALO;
            g3[r][c] = fd8_sum(Z[m + 1], Z[m + 2], Z[m + 3], Z[m + 4], Z[m - 1], Z[m - 2], Z[m - 3], Z[m - 4]);
          }
        }
      }
      // out /= h (diffops.py:96): reciprocal division unless an operand is extreme
      bool ieee = false;
#pragma unroll
      for (int r = 0; r < RY; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          ieee |= div_needs_ieee(g1[r][c], dlo, dspan) | div_needs_ieee(g2[r][c], dlo, dspan) |
                  div_needs_ieee(g3[r][c], dlo, dspan);
      if (ieee) {  // rare: out of line, so the 9 unrolled steps stay compact
        F12 sv;
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            sv.v[r * 2 + c] = g1[r][c];
            sv.v[4 + r * 2 + c] = g2[r][c];
            sv.v[8 + r * 2 + c] = g3[r][c];
          }
        sv = fd8_div_ieee(sv, h1, h2, h3, r1, r2, r3, dlo, dspan);
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            g1[r][c] = sv.v[r * 2 + c];
            g2[r][c] = sv.v[4 + r * 2 + c];
            g3[r][c] = sv.v[8 + r * 2 + c];
          }
      } else {
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            g1[r][c] = div_fast(g1[r][c], h1, r1);
            g2[r][c] = div_fast(g2[r][c], h2, r2);
            g3[r][c] = div_fast(g3[r][c], h3, r3);
          }
      }
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        if (!act[r]) continue;
        float2* o = reinterpret_cast<float2*>(op + rowoff[r]);
        if constexpr (MODE == 0) {
          o[0] = make_float2(g1[r][0], g1[r][1]);
          o[N / 2] = make_float2(g2[r][0], g2[r][1]);
          o[N] = make_float2(g3[r][0], g3[r][1]);
        } else {
          o[0] = make_float2(__fadd_rn(__fadd_rn(g1[r][0], g2[r][0]), g3[r][0]),
                             __fadd_rn(__fadd_rn(g1[r][1], g2[r][1]), g3[r][1]));
        }
      }
      op += psz;
    };
#define VR_FD8_STEP(S)        \
    if (i >= i_end) break;      \
    step(IC<S>{}, i);           \
    ++i;
    for (int i = i_begin;;) {
      VR_FD8_STEP(0) VR_FD8_STEP(1) VR_FD8_STEP(2) VR_FD8_STEP(3) VR_FD8_STEP(4)
      VR_FD8_STEP(5) VR_FD8_STEP(6) VR_FD8_STEP(7) VR_FD8_STEP(8)
    }
#undef VR_FD8_STEP
    cp_wait<0>();
  }
}

template <int MODE, bool SLAB>
void fd8_run(dim3 block, cudaStream_t s, const float* in, const float* lo, const float* hi, Dims d,
             float h1, float h2, float h3, float r1, float r2, float r3, unsigned dlo, unsigned dspan,
             float* out) {
  const size_t smem = sizeof(Fd8Stage<MODE>) * NS;
  static int slots = 0;  // resident CTAs per GPU
  if (!slots) {
    cudaFuncSetAttribute(fd8_kernel<MODE, SLAB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fd8_kernel<MODE, SLAB>, NTHR, smem);
    slots = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int ntiles = ((d.n3 + TZ - 1) / TZ) * ((d.n2 + TY - 1) / TY);
  int nchunk = std::max(1, std::min(slots / ntiles, d.n1 / 8));
  const int grid = std::min(ntiles * nchunk, std::max(slots, ntiles));
  fd8_kernel<MODE, SLAB><<<grid, block, smem, s>>>(in, lo, hi, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out,
                                                     nchunk);
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
  if (d.n3 % 2) return VR_ERR_DIMS;  // float2 rows; the reference grid has even dims (grid.py)
  if (((uintptr_t)in | (uintptr_t)out | (uintptr_t)lo | (uintptr_t)hi) & 7) return VR_ERR_ARG;
  const float h1 = (float)(kTwoPi / n1_global), h2 = (float)(kTwoPi / d.n2), h3 = (float)(kTwoPi / d.n3);
  const float r1 = 1.0f / h1, r2 = 1.0f / h2, r3 = 1.0f / h3;  // fp32 IEEE: RN(1/h)
  // reciprocal-division range, float bit patterns (see div_fast)
  const bool verified = n1_global <= 8192 && d.n2 <= 8192 && d.n3 <= 8192;
  const unsigned dlo = verified ? 0x0d800000u : 0x21800000u;            // 2^-100 / 2^-60
  const unsigned dspan = (verified ? 0x79800000u : 0x5d800000u) - dlo;  // 2^116 / 2^60
  dim3 block(TXB, TYB);
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0 && slab)
    fd8_run<0, true>(block, s, in, lo, hi, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out);
  else if (mode == 0)
    fd8_run<0, false>(block, s, in, nullptr, nullptr, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out);
  else if (slab)
    fd8_run<1, true>(block, s, in, lo, hi, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out);
  else
    fd8_run<1, false>(block, s, in, nullptr, nullptr, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out);
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
