// Separable f64 line engine for A = |k|^2 (diffops.py:116-118).
//
// The symbol of A is a SUM of one-axis symbols, |k|^2 = k1^2 + k2^2 + k3^2, and
// each k_a^2 is real and even, so
//     irfftn(|k|^2 rfftn(v)) = D11 v + D22 v + D33 v,
//     D_aa = ifft_a(k_a^2 fft_a(.))   (one 1-D transform pair per line),
// exactly (both sides are the same Fourier multiplier; the x3 Nyquist bin of a
// real line is real, so dropping its imaginary part in irfft changes nothing).
// This matters for precision and traffic:
//   * |k|^2 amplifies the absolute rounding of a forward transform at high k.
//     A 3-D f32 transform cannot meet the 1e-5 operator bar at 256^3 (SURVEY §7:
//     3-5e-5), which is why the 3-D path stores its forward half in f64 (2.8 GB
//     of pass traffic per A at 256^3).  Here a line is loaded from the f32
//     field and forward-transformed and multiplied in f64 registers; the
//     inverse runs in f32 (its rounding is relative to the output), and the
//     three partial sums are f32 -- every rounding after the multiply is
//     relative to |A v| (~1e-7).
//   * Traffic: three passes (x3, x2, x1), each reading v once and the running
//     partial sum, 32-36 B/voxel per component instead of ~55 B (3-D, f64).
// Two real lines travel as one complex line (a + i b): the symbol is real and
// even, so ifft(s fft(a + i b)) = D a + i D b.
//
// Line FFT = the four-step register FFT of spectral_4step.cuh (L = 16 R2,
// R2 in {8, 16}: R2 threads per line, 16 values per thread, one shared
// transpose).  Its output order (thread t owns X[t + 16 u]) is a permutation
// of its input order (thread t owns x[t + R2 m]), so the inverse transform
// runs on the multiplied spectrum in place.
//
// Passes (all components in one launch, grid.y = component):
//   ROWS     x3 lines (contiguous):      acc  = D33 v
//   STRIDED  x2 lines (stride n3):       acc += D22 v
//   STRIDED  x1 lines (stride n2 n3):    out  = alpha (acc + D11 v) + add
#pragma once

namespace vr {
namespace d2 {

// input slot of the forward line FFT for the value thread t holds at output
// position u (see fs::out_freq): identity for R2 = 16, interleave for R2 = 8
template <int R2, typename C>
__device__ __forceinline__ void to_input_order(C (&v)[16]) {
  if constexpr (R2 == 8) {
    C w[16];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      w[2 * u] = v[u];
      w[2 * u + 1] = v[8 + u];
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = w[u];
  }
}

// forward line FFT (f64) -> multiply by scale * k^2 (k = fftfreq * L) ->
// inverse (f32: after the multiply every value is O(|D x|), so the inverse's
// rounding is relative to the output, as in the 3-D engine's inverse half).
// Values enter as x[t + R2 m] (f64) and leave as y[out_freq(t, u)] (f32).
template <int R2>
__device__ __forceinline__ void line_d2(double2 (&v)[16], float2 (&y)[16], int t, double2* sm,
                                        const double2* __restrict__ tw, double scale) {
  constexpr int L = 16 * R2;
  fs::line_fft<double2, R2>(v, t, sm, tw, false);
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int k = fs::out_freq<R2>(t, u);
    const double f = (double)(k < L / 2 ? k : k - L);
    const double m = f * f * scale;
    y[u] = make_float2((float)(v[u].x * m), (float)(v[u].y * m));
  }
  to_input_order<R2>(y);
  __syncthreads();   // the transpose scratch is reused by the inverse
  fs::line_fft<float2, R2>(y, t, reinterpret_cast<float2*>(sm), tw, true);
}

// x3 lines: one complex line = rows (2p, 2p+1) of the flattened (n1 n2, n3)
// row array; R2 threads per line, lane = t + R2 q.  acc = D33 v.
template <int R2, int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 4) rows_kernel(const float* __restrict__ v, float* __restrict__ acc,
                                                      int npairs, int64_t cstride, const double2* __restrict__ tw,
                                                      double scale) {
  constexpr int L = 16 * R2, LPB = NT / R2;
  extern __shared__ __align__(16) unsigned char d2_smem[];
  double2* smem = reinterpret_cast<double2*>(d2_smem);
  const int t = threadIdx.x % R2, q = threadIdx.x / R2;
  const int p = blockIdx.x * LPB + q;
  const bool ok = p < npairs;
  const float* ra = v + blockIdx.y * cstride + (int64_t)(ok ? p : 0) * 2 * L;
  const float* rb = ra + L;
  double2 x[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) x[m] = make_double2(__ldg(ra + t + R2 * m), __ldg(rb + t + R2 * m));
  float2 y[16];
  line_d2<R2>(x, y, t, smem + q * fs::line_smem<R2>(), tw, scale);
  if (ok) {
    float* wa = acc + blockIdx.y * cstride + (int64_t)p * 2 * L;
    float* wb = wa + L;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int k = fs::out_freq<R2>(t, u);
      wa[k] = y[u].x;
      wb[k] = y[u].y;
    }
  }
}

// Strided lines (x2: es = n3, outer = x1 plane; x1: es = n2 n3, outer = x2 row).
// One complex line = columns (k0 + 2q, k0 + 2q + 1); NB = NT / R2 lines per
// CTA (NT threads) cover 2 NB consecutive x3 columns, lane = q + NB t, so every warp load is
// a contiguous 2 NB-float run.  FINAL = false: acc += D v; FINAL = true:
// out = alpha (acc + D v) (+ add).  acc may alias out (same element, same thread).
template <int R2, bool FINAL, int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 4) strided_kernel(const float* __restrict__ v, float* acc,
                                                         const float* __restrict__ add, float* out, int n3, int es,
                                                         int outer_stride, int64_t cstride,
                                                         const double2* __restrict__ tw, double scale, double alpha) {
  constexpr int NB = NT / R2;
  extern __shared__ __align__(16) unsigned char d2_smem[];
  double2* smem = reinterpret_cast<double2*>(d2_smem);
  const int q = threadIdx.x % NB, t = threadIdx.x / NB;
  const int nchunks = n3 / (2 * NB);
  const int o = blockIdx.x / nchunks, k0 = (blockIdx.x - o * nchunks) * 2 * NB;
  // 64-bit component base, 32-bit offsets inside a component (< 2^31 voxels)
  const int64_t cb = blockIdx.y * cstride;
  const int base = o * outer_stride + k0 + 2 * q;
  const float2* vb = reinterpret_cast<const float2*>(v + cb);
  double2 x[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const float2 a = __ldg(vb + ((base + (t + R2 * m) * es) >> 1));
    x[m] = make_double2(a.x, a.y);
  }
  float2 y[16];
  line_d2<R2>(x, y, t, smem + q * fs::line_smem<R2>(), tw, scale);
  float2* ab = reinterpret_cast<float2*>(acc + cb);
  float2* ob = reinterpret_cast<float2*>(out + cb);
  const float2* db = add ? reinterpret_cast<const float2*>(add + cb) : nullptr;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int e = (base + fs::out_freq<R2>(t, u) * es) >> 1;
    const float2 s = ab[e];
    float2 r;
    if (FINAL) {
      r.x = (float)(alpha * ((double)s.x + (double)y[u].x));
      r.y = (float)(alpha * ((double)s.y + (double)y[u].y));
      if (db) {
        const float2 b = __ldg(db + e);
        r.x += b.x;
        r.y += b.y;
      }
      ob[e] = r;
    } else {
      r.x = s.x + y[u].x;
      r.y = s.y + y[u].y;
      ab[e] = r;
    }
  }
}

template <int R2, int NT> constexpr size_t smem_bytes() { return sizeof(double2) * (NT / R2) * fs::line_smem<R2>(); }

}  // namespace d2
}  // namespace vr
