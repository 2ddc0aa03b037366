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
// x1 lines of 512 / 1024 / 2048 (long_kernel) use the three-step register FFT
// of spectral_4step.cuh (fs::lf3) instead of the four-step one.
//
// On x1 slabs (one rank per GPU, D2Peer) the x3 and x2 passes are local; the
// rows pass also stores every slab row into the block buffer of the rank that
// owns its x2 chunk (the transpose as the pass's second output), the x1 pass
// runs on the received block [N1][L2][N3] and stores D11 v into the owning
// rank's back buffer [L1][N2][N3], and final_kernel forms
// alpha (acc + back) (+ add) with the same arithmetic as the FINAL strided
// epilogue -- identical results to the single-domain operator.
#pragma once

namespace vr {
namespace d2 {

// peer destinations of the distributed passes (symmetric buffers, per rank)
struct D2Peer {
  void* dst[8];
  const float* back;   // MODE 3: this rank's back buffer (D11 values, slab layout)
  int me;              // this rank
  int l1, l2;          // x1 planes per rank, x2 rows per block
  int n1, n2;          // global N1, N2
};

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

// pe.dst[r] by a select chain (select_ptr): a dynamically indexed parameter
// array would be copied to local memory (ptxas: 88-byte stack frame)
__device__ __forceinline__ float* peer_dst(const D2Peer& pe, int r) {
  return reinterpret_cast<float*>(select_ptr(pe.dst, r));
}

// D11 v at (x1 = i, block row jl, columns k, k + 1) -> rank i / l1's back
// buffer [c][i - x0][me * l2 + jl][k]
__device__ __forceinline__ void store_back(const D2Peer& pe, int c, int i, int jl, int k, int n3, float2 val) {
  const int owner = i / pe.l1, il = i - owner * pe.l1;
  float* b = peer_dst(pe, owner) + (((int64_t)c * pe.l1 + il) * pe.n2 + (int64_t)pe.me * pe.l2 + jl) * n3 + k;
  *reinterpret_cast<float2*>(b) = val;
}

// the final epilogue's arithmetic (strided MODE 1, long_kernel MODE 1, final_kernel)
__device__ __forceinline__ float final_value(float acc, float d, double alpha) {
  return (float)(alpha * ((double)acc + (double)d));
}

// x3 lines: one complex line = rows (2p, 2p+1) of the flattened (n1 n2, n3)
// row array; R2 threads per line, lane = t + R2 q.  acc = D33 v.
template <int R2, int NT, bool PEER = false>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 4) rows_kernel(const float* __restrict__ v, float* __restrict__ acc,
                                                      int npairs, int64_t cstride, const double2* __restrict__ tw,
                                                      double scale, D2Peer pe) {
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
  if (PEER && ok) {
    // rows (i, j), (i, j + 1) of the slab -> rows (x0 + i, jl), (x0 + i, jl + 1)
    // of the block of rank j / l2 (l2 even: a pair never straddles two blocks)
    const int r0 = 2 * p, i = r0 / pe.n2, j = r0 - i * pe.n2;
    const int owner = j / pe.l2, jl = j - owner * pe.l2;
    float* b = peer_dst(pe, owner) + (((int64_t)blockIdx.y * pe.n1 + (int64_t)pe.me * pe.l1 + i) * pe.l2 + jl) * L;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      b[t + R2 * m] = (float)x[m].x;
      b[L + t + R2 * m] = (float)x[m].y;
    }
  }
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
// a contiguous 2 NB-float run.  MODE 0: acc += D v; MODE 1 (final):
// out = alpha (acc + D v) (+ add), acc may alias out (same element, same
// thread); MODE 2: x1 lines of a distributed block, D v -> the owning rank's
// back buffer (pe); MODE 3: out = alpha ((acc + D v) + back) (+ add).
template <int R2, int MODE, int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 4) strided_kernel(const float* __restrict__ v, float* acc,
                                                         const float* __restrict__ add, float* out, int n3, int es,
                                                         int outer_stride, int64_t cstride,
                                                         const double2* __restrict__ tw, double scale, double alpha,
                                                         D2Peer pe) {
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
  if constexpr (MODE == 2) {
#pragma unroll
    for (int u = 0; u < 16; ++u) store_back(pe, blockIdx.y, fs::out_freq<R2>(t, u), o, k0 + 2 * q, n3, y[u]);
    return;
  }
  float2* ab = reinterpret_cast<float2*>(acc + cb);
  float2* ob = reinterpret_cast<float2*>(out + cb);
  const float2* db = add ? reinterpret_cast<const float2*>(add + cb) : nullptr;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int e = (base + fs::out_freq<R2>(t, u) * es) >> 1;
    const float2 s = ab[e];
    float2 r;
    if (MODE == 1) {
      r.x = final_value(s.x, y[u].x, alpha);
      r.y = final_value(s.y, y[u].y, alpha);
      if (db) {
        const float2 b = __ldg(db + e);
        r.x += b.x;
        r.y += b.y;
      }
      ob[e] = r;
    } else if (MODE == 3) {
      // distributed x2 pass after the x1 exchange: the MODE 0 sum, then the
      // final epilogue with the received D11 values (same roundings as the
      // single-domain MODE 0 -> MODE 1 sequence)
      const float2 bk = __ldg(reinterpret_cast<const float2*>(pe.back + cb) + e);
      r.x = final_value(s.x + y[u].x, bk.x, alpha);
      r.y = final_value(s.y + y[u].y, bk.y, alpha);
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

// Strided x1 lines of L = 256 R3 (512 / 1024 / 2048): the strided kernel's
// column pairing and epilogues (MODE 1 / 2) around the three-step register
// FFT (f64 forward, k1^2 / L, f32 inverse).  NB complex lines per CTA,
// lane = q + NB u.
template <int R3, int NB> constexpr size_t long_smem_bytes() {
  return sizeof(double2) * NB * fs::lf3::smem_elems<R3>();
}
template <int R3, int NB, int MODE>
__global__ void __launch_bounds__(NB * 16 * R3, 1) long_kernel(const float* __restrict__ v, const float* acc,
                                                               const float* __restrict__ add, float* out, int n3,
                                                               int es, int outer_stride, int64_t cstride,
                                                               const double2* __restrict__ twL, double scale,
                                                               double alpha, D2Peer pe) {
  constexpr int Tn = fs::lf3::T<R3>(), L = 256 * R3, LS = fs::lf3::smem_elems<R3>();
  extern __shared__ __align__(16) unsigned char d2_smem[];
  const int q = threadIdx.x % NB, u = threadIdx.x / NB;
  const int nchunks = n3 / (2 * NB);
  const int o = blockIdx.x / nchunks, k0 = (blockIdx.x - o * nchunks) * 2 * NB;
  const int64_t cb = blockIdx.y * cstride;
  const int64_t base = (int64_t)o * outer_stride + k0 + 2 * q;
  const float2* vb = reinterpret_cast<const float2*>(v + cb);
  double2 x[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const float2 a = __ldg(vb + ((base + (int64_t)(u + Tn * m) * es) >> 1));
    x[m] = make_double2(a.x, a.y);
  }
  fs::lf3::forward<double2, R3>(x, u, reinterpret_cast<double2*>(d2_smem) + q * LS, twL);
  float2 y[16];
#pragma unroll
  for (int idx = 0; idx < 16; ++idx) {
    const int k = fs::lf3::freq<R3>(u, idx);
    const double f = (double)(k < L / 2 ? k : k - L);
    const double m = f * f * scale;
    y[idx] = make_float2((float)(x[idx].x * m), (float)(x[idx].y * m));
  }
  __syncthreads();   // the shared buffer is reused by the f32 inverse
  fs::lf3::inverse<float2, R3>(y, u, reinterpret_cast<float2*>(d2_smem) + q * LS, twL);
  if constexpr (MODE == 2) {
#pragma unroll
    for (int m = 0; m < 16; ++m) store_back(pe, blockIdx.y, u + Tn * m, o, k0 + 2 * q, n3, y[m]);
  } else {
    const float2* ab = reinterpret_cast<const float2*>(acc + cb);
    float2* ob = reinterpret_cast<float2*>(out + cb);
    const float2* db = add ? reinterpret_cast<const float2*>(add + cb) : nullptr;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int64_t e = (base + (int64_t)(u + Tn * m) * es) >> 1;
      const float2 s = ab[e];
      float2 r = make_float2(final_value(s.x, y[m].x, alpha), final_value(s.y, y[m].y, alpha));
      if (db) {
        const float2 b = __ldg(db + e);
        r.x += b.x;
        r.y += b.y;
      }
      ob[e] = r;
    }
  }
}

// distributed final: out = alpha (acc + back) (+ add), n4 float4s
__global__ void __launch_bounds__(256) final_kernel(const float4* __restrict__ acc, const float4* __restrict__ back,
                                                    const float4* add, float4* out,
                                                    int64_t n4, double alpha) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = acc[e], b = __ldg(back + e);
    float4 r = make_float4(final_value(a.x, b.x, alpha), final_value(a.y, b.y, alpha), final_value(a.z, b.z, alpha),
                           final_value(a.w, b.w, alpha));
    if (add) {
      const float4 d = __ldg(add + e);
      r.x += d.x;
      r.y += d.y;
      r.z += d.z;
      r.w += d.w;
    }
    out[e] = r;
  }
}

template <int R2, int NT> constexpr size_t smem_bytes() { return sizeof(double2) * (NT / R2) * fs::line_smem<R2>(); }

}  // namespace d2
}  // namespace vr
