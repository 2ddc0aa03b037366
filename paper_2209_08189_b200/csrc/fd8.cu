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
// div_fast for |x| in [2^-124, 2^116) (the verified sizes' inline range): sums
// below 2^-100 are scaled by 2^64 into the exhaustively verified reciprocal
// range and back -- both scalings exact, the quotient stays normal
// (|x / h| > 2^-124 for h < 1) -- so tiny far-field values no longer leave the
// unrolled loop for the out-of-line IEEE branch
__device__ __forceinline__ float div_fast_s(float x, float h, float r) {
  const bool tiny = fabsf(x) < 0x1p-100f;
  const float q = div_fast(tiny ? __fmul_rn(x, 0x1p64f) : x, h, r);
  return tiny ? __fmul_rn(q, 0x1p-64f) : q;
}
// |x| outside [lo, lo + span) (as float bits) and not 0: take IEEE division
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
  const bool verified = dlo == 0x01800000u;
  F12 o;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    const float h = i < 4 ? h1 : (i < 8 ? h2 : h3), r = i < 4 ? r1 : (i < 8 ? r2 : r3);
    const float x = s.v[i], ax = fabsf(x);
    if (!div_needs_ieee(x, dlo, dspan))
      o.v[i] = div_fast_s(x, h, r);
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
#ifndef VR_FD8_CTAS
#define VR_FD8_CTAS 2      // resident CTAs / SM (3, at 80 registers: divergence 0.100 vs 0.085 ms)
#endif

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
__global__ void __launch_bounds__(NTHR, VR_FD8_CTAS) fd8_kernel(const float* __restrict__ f, const float* __restrict__ lo,
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
            g1[r][c] = div_fast_s(g1[r][c], h1, r1);
            g2[r][c] = div_fast_s(g2[r][c], h2, r2);
            g3[r][c] = div_fast_s(g3[r][c], h3, r3);
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

// ---- row-tile FD8 with bulk-copy plane staging (N3 in {128, 256, 512}) -------
// One CTA = TY whole x2 rows (every x3 voxel) walked along a chunk of x1
// planes.  Each plane step is staged in shared memory by ONE bulk copy per
// row (cp.async.bulk, 0.5-2 KB contiguous, completion on an mbarrier): the
// x2-halo'd rows of plane p (x2 / x3 derivatives) and the TY centre rows of
// plane p + 4 (the leading edge of the x1 register windows), NS plane steps in
// flight.  A row tile spans the whole x3 extent, so the x3 stencil wraps
// inside the staged row and only the x2 halo rows ever wrap (done by the
// producer's row addresses).  Thread = 4 consecutive x3 voxels (float4) x RY
// rows; arithmetic and division exactly as fd8_kernel (bit-identical).
// MODE 0: gradient of f; MODE 1: divergence of v (v2 halo'd rows, v3 and the
// plane-ahead v1 centre rows).
template <int N3> struct RowCfg;
template <> struct RowCfg<128> { static constexpr int TPR = 32, RPP = 8, RY = 1, TY = 8, NS = 4; };
template <> struct RowCfg<256> { static constexpr int TPR = 64, RPP = 4, RY = 2, TY = 8, NS = 4; };
template <> struct RowCfg<512> { static constexpr int TPR = 128, RPP = 2, RY = 2, TY = 4, NS = 3; };

template <int MODE, int N3> struct RowStage {
  using C = RowCfg<N3>;
  // row blocks: [0, TY+8) x2-halo'd rows (f or v2); then TY centre rows of the
  // plane 4 ahead (f or v1); MODE 1 adds TY centre rows of v3
  static constexpr int ROWS = C::TY + 8 + C::TY + (MODE == 1 ? C::TY : 0);
  static constexpr int HALO_ROW = 0, XC_ROW = C::TY + 8, Z_ROW = 2 * C::TY + 8;
  static constexpr size_t BYTES = sizeof(float) * ROWS * N3;
};

__device__ __forceinline__ unsigned fd8_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int MODE, bool SLAB, int N3>
__global__ void __launch_bounds__(256, 2) fd8_rows_kernel(const float* __restrict__ f, const float* __restrict__ lo,
                                                          const float* __restrict__ hi, Dims d, float h1, float h2,
                                                          float h3, float r1, float r2, float r3, unsigned dlo,
                                                          unsigned dspan, float* __restrict__ out, int nchunk) {
  using C = RowCfg<N3>;
  using St = RowStage<MODE, N3>;
  constexpr int TY = C::TY, RY = C::RY, RPP = C::RPP, NS = C::NS, TPR = C::TPR;
  extern __shared__ __align__(128) float rows_smem[];
  __shared__ __align__(8) unsigned long long full[NS];
  const int64_t N = d.n();
  const int psz = d.n2 * N3;
  const int ntiles = d.n2 / TY;
  const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
  const int i_begin = (int)((int64_t)d.n1 * chunk / nchunk);
  const int i_end = (int)((int64_t)d.n1 * (chunk + 1) / nchunk);
  const int j0 = tile * TY;
  const int tid = threadIdx.x, lane = tid & 31;
  const int tc = tid % TPR, ty = tid / TPR;      // float4 column, first tile row of the thread
  const int k = 4 * tc;
  if (tid < NS) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fd8_smem_u32(&full[tid])) : "memory");
  }
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (i_begin >= i_end) return;

  auto plane = [&](const float* base, int ii) -> const float* {   // plane ii in [-4, L1 + 4)
    if (SLAB) return ii < 0 ? lo + (int64_t)(ii + HALO) * psz
                            : (ii >= d.n1 ? hi + (int64_t)(ii - d.n1) * psz : base + (int64_t)ii * psz);
    ii = ii < 0 ? ii + d.n1 : (ii >= d.n1 ? ii - d.n1 : ii);
    return base + (int64_t)ii * psz;
  };
  // component bases: MODE 0 f; MODE 1 v1 = f, v2 = f + N, v3 = f + 2N (ghosts only for v1)
  const float* fx = f;                              // x1 windows
  const float* fy = MODE == 0 ? f : f + N;          // x2 halo'd rows
  // producer: warp 0, one bulk copy per staged row
  auto issue = [&](int p) {
    if (tid >= 32) return;
    const int s = p % NS;
    float* st = rows_smem + (size_t)s * St::ROWS * N3;
    const unsigned bar = fd8_smem_u32(&full[s]);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((unsigned)St::BYTES)
                   : "memory");
    __syncwarp();
    for (int r = lane; r < St::ROWS; r += 32) {
      const float* src;
      if (r < TY + 8) {                       // x2-halo'd rows of plane p (x1 local: never a ghost for x2/x3)
        int jr = j0 - HALO + r;
        jr = jr < 0 ? jr + d.n2 : (jr >= d.n2 ? jr - d.n2 : jr);
        src = fy + (int64_t)p * psz + (int64_t)jr * N3;
      } else if (r < 2 * TY + 8) {            // centre rows of plane p + 4 (x1 window, may be a ghost)
        src = plane(fx, p + HALO) + (int64_t)(j0 + r - (TY + 8)) * N3;
      } else {                                // MODE 1: centre rows of v3, plane p
        src = f + 2 * N + (int64_t)p * psz + (int64_t)(j0 + r - (2 * TY + 8)) * N3;
      }
      const unsigned dst = fd8_smem_u32(st + (size_t)r * N3);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src), "r"((unsigned)(N3 * 4)), "r"(bar) : "memory");
    }
  };

  // x1 windows: plane i-4+o of row r, column c in w[r][c][(S + o) % 9]
  float w[RY][4][9];
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    const float* pl = plane(fx, i_begin - HALO + o);
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(pl + (int64_t)(j0 + ty + r * RPP) * N3 + k));
      w[r][0][o] = v.x; w[r][1][o] = v.y; w[r][2][o] = v.z; w[r][3][o] = v.w;
    }
  }
#pragma unroll
  for (int q = 0; q < NS - 1; ++q)
    if (i_begin + q < i_end) issue(i_begin + q);

  auto step = [&](auto S_, int i) {
    constexpr int S = decltype(S_)::value;
    const int s = i % NS;
    if (i + NS - 1 < i_end) issue(i + NS - 1);   // stage (i - 1) % NS: released by the barrier below
    {
      const unsigned bar = fd8_smem_u32(&full[s]);
      const unsigned par = (unsigned)((i - i_begin) / NS) & 1u;
      asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\t"
                   "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
                   ::"r"(bar), "r"(par) : "memory");
    }
    const float* st = rows_smem + (size_t)s * St::ROWS * N3;
    // window leading edge (plane i + 4)
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(st + (size_t)(St::XC_ROW + ty + r * RPP) * N3 + k);
      w[r][0][(S + 8) % 9] = v.x; w[r][1][(S + 8) % 9] = v.y;
      w[r][2][(S + 8) % 9] = v.z; w[r][3][(S + 8) % 9] = v.w;
    }
    float g1[RY][4], g2[RY][4], g3[RY][4];
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float* x = w[r][c];
        g1[r][c] = fd8_sum(x[(S + 5) % 9], x[(S + 6) % 9], x[(S + 7) % 9], x[(S + 8) % 9], x[(S + 3) % 9],
                           x[(S + 2) % 9], x[(S + 1) % 9], x[S % 9]);
      }
    // x2: halo'd rows ty + r RPP - 4 .. + 4 (staged row index = tile row + 4)
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      float Y[9][4];
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        if (q == 4) continue;
        const float4 v = *reinterpret_cast<const float4*>(st + (size_t)(ty + r * RPP + q) * N3 + k);
        Y[q][0] = v.x; Y[q][1] = v.y; Y[q][2] = v.z; Y[q][3] = v.w;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
        g2[r][c] = fd8_sum(Y[5][c], Y[6][c], Y[7][c], Y[8][c], Y[3][c], Y[2][c], Y[1][c], Y[0][c]);
    }
    // x3: columns k-4 .. k+7 of the row, wrapped inside the staged row
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const float* row = MODE == 0 ? st + (size_t)(ty + r * RPP + HALO) * N3
                                   : st + (size_t)(St::Z_ROW + ty + r * RPP) * N3;
      const int km = k == 0 ? N3 - 4 : k - 4, kp = k + 4 == N3 ? 0 : k + 4;
      const float4 a = *reinterpret_cast<const float4*>(row + km);
      const float4 b = *reinterpret_cast<const float4*>(row + k);
      const float4 e = *reinterpret_cast<const float4*>(row + kp);
      const float Z[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, e.x, e.y, e.z, e.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int m = c + HALO;
        g3[r][c] = fd8_sum(Z[m + 1], Z[m + 2], Z[m + 3], Z[m + 4], Z[m - 1], Z[m - 2], Z[m - 3], Z[m - 4]);
      }
    }
    __syncthreads();   // every reader of stage s is done: the next issue() may refill it
    bool ieee = false;
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        ieee |= div_needs_ieee(g1[r][c], dlo, dspan) | div_needs_ieee(g2[r][c], dlo, dspan) |
                div_needs_ieee(g3[r][c], dlo, dspan);
    if (ieee) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        F12 sv;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          sv.v[c] = g1[r][c];
          sv.v[4 + c] = g2[r][c];
          sv.v[8 + c] = g3[r][c];
        }
        sv = fd8_div_ieee(sv, h1, h2, h3, r1, r2, r3, dlo, dspan);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          g1[r][c] = sv.v[c];
          g2[r][c] = sv.v[4 + c];
          g3[r][c] = sv.v[8 + c];
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < RY; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          g1[r][c] = div_fast_s(g1[r][c], h1, r1);
          g2[r][c] = div_fast_s(g2[r][c], h2, r2);
          g3[r][c] = div_fast_s(g3[r][c], h3, r3);
        }
    }
    float* op = out + (int64_t)i * psz;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      float4* o = reinterpret_cast<float4*>(op + (int64_t)(j0 + ty + r * RPP) * N3 + k);
      if constexpr (MODE == 0) {
        o[0] = make_float4(g1[r][0], g1[r][1], g1[r][2], g1[r][3]);
        o[N / 4] = make_float4(g2[r][0], g2[r][1], g2[r][2], g2[r][3]);
        o[N / 2] = make_float4(g3[r][0], g3[r][1], g3[r][2], g3[r][3]);
      } else {
        float4 q;
        q.x = __fadd_rn(__fadd_rn(g1[r][0], g2[r][0]), g3[r][0]);
        q.y = __fadd_rn(__fadd_rn(g1[r][1], g2[r][1]), g3[r][1]);
        q.z = __fadd_rn(__fadd_rn(g1[r][2], g2[r][2]), g3[r][2]);
        q.w = __fadd_rn(__fadd_rn(g1[r][3], g2[r][3]), g3[r][3]);
        o[0] = q;
      }
    }
  };
#define VR_FD8R_STEP(S)        \
  if (i >= i_end) break;       \
  step(IC<S>{}, i);            \
  ++i;
  for (int i = i_begin;;) {
    VR_FD8R_STEP(0) VR_FD8R_STEP(1) VR_FD8R_STEP(2) VR_FD8R_STEP(3) VR_FD8R_STEP(4)
    VR_FD8R_STEP(5) VR_FD8R_STEP(6) VR_FD8R_STEP(7) VR_FD8R_STEP(8)
  }
#undef VR_FD8R_STEP
}

template <int MODE, bool SLAB, int N3>
void fd8_rows_run(cudaStream_t s, const float* in, const float* lo, const float* hi, Dims d, float h1, float h2,
                  float h3, float r1, float r2, float r3, unsigned dlo, unsigned dspan, float* out) {
  using C = RowCfg<N3>;
  const size_t smem = RowStage<MODE, N3>::BYTES * C::NS;
  static int slots = 0;   // resident CTAs per GPU (per instantiation)
  if (!slots) {
    cudaFuncSetAttribute(fd8_rows_kernel<MODE, SLAB, N3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fd8_rows_kernel<MODE, SLAB, N3>, 256, smem);
    slots = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int ntiles = d.n2 / C::TY;
  // ~2 waves of CTAs, chunks of >= 8 planes (the 8-plane window preload is amortised)
  const int nchunk = std::max(1, std::min((2 * slots + ntiles - 1) / ntiles, d.n1 / 8));
  fd8_rows_kernel<MODE, SLAB, N3><<<ntiles * nchunk, 256, smem, s>>>(in, lo, hi, d, h1, h2, h3, r1, r2, r3, dlo,
                                                                    dspan, out, nchunk);
}

// 0 (default): cp.async tile kernel; 1: row-tile bulk-copy kernel where it applies
// (N3 in {128, 256}).  Measured on B200 at 256^3 with the L2 flushed: row
// kernel gradient 0.092 ms / divergence 0.145 ms vs tile kernel 0.084 / 0.085 ms
// (one barrier + mbarrier wait per plane for all 8 warps, and the 8-plane
// window preload per 16-plane chunk), so the tile kernel stays the default.
// (A per-element inline IEEE-division select was also measured: 0.094 ms, and
// an inline f64 division for flagged micro-tiles 0.146 vs 0.120 ms on the C2
// state series -- the out-of-line one-branch-per-micro-tile form below is
// faster on the common path.)
static int g_fd8_mode = 0;

template <int MODE, bool SLAB>
bool fd8_rows_dispatch(cudaStream_t s, const float* in, const float* lo, const float* hi, Dims d, float h1,
                       float h2, float h3, float r1, float r2, float r3, unsigned dlo, unsigned dspan, float* out) {
  if (!g_fd8_mode || (((uintptr_t)in | (uintptr_t)out | (uintptr_t)lo | (uintptr_t)hi) & 15)) return false;
  if (d.n1 < 8) return false;
  switch (d.n3) {
    case 128: if (d.n2 % RowCfg<128>::TY) return false;
      fd8_rows_run<MODE, SLAB, 128>(s, in, lo, hi, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out); return true;
    case 256: if (d.n2 % RowCfg<256>::TY) return false;
      fd8_rows_run<MODE, SLAB, 256>(s, in, lo, hi, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out); return true;
    default: return false;
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
  if (d.n3 % 2) return VR_ERR_DIMS;  // float2 rows; the reference grid has even dims (grid.py)
  if (((uintptr_t)in | (uintptr_t)out | (uintptr_t)lo | (uintptr_t)hi) & 7) return VR_ERR_ARG;
  const float h1 = (float)(kTwoPi / n1_global), h2 = (float)(kTwoPi / d.n2), h3 = (float)(kTwoPi / d.n3);
  const float r1 = 1.0f / h1, r2 = 1.0f / h2, r3 = 1.0f / h3;  // fp32 IEEE: RN(1/h)
  // reciprocal-division range, float bit patterns (see div_fast)
  const bool verified = n1_global <= 8192 && d.n2 <= 8192 && d.n3 <= 8192;
  const unsigned dlo = verified ? 0x01800000u : 0x21800000u;            // 2^-124 / 2^-60
  const unsigned dspan = (verified ? 0x79800000u : 0x5d800000u) - dlo;  // 2^116 / 2^60
  dim3 block(TXB, TYB);
  cudaStream_t s = (cudaStream_t)stream;
  bool done;
  if (mode == 0 && slab) done = fd8_rows_dispatch<0, true>(s, in, lo, hi, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out);
  else if (mode == 0) done = fd8_rows_dispatch<0, false>(s, in, nullptr, nullptr, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out);
  else if (slab) done = fd8_rows_dispatch<1, true>(s, in, lo, hi, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out);
  else done = fd8_rows_dispatch<1, false>(s, in, nullptr, nullptr, d, h1, h2, h3, r1, r2, r3, dlo, dspan, out);
  if (done) {
    VR_CHECK_LAUNCH();
    return VR_OK;
  }
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
int vr_set_fd8_mode(int mode) {
  const int prev = g_fd8_mode;
  g_fd8_mode = mode;
  return prev;
}
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
