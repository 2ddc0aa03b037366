// Four-step register FFTs for the power-of-two fast path (L = 16 x R2, R2 in {8, 16}).
//
// The Stockham engine (spectral_fast.cuh) round-trips every radix-8 stage
// through shared memory: ~8 shared accesses per element per line FFT, and the
// passes measured 92-97 % of the L1/shared data pipe (profiles/r1_ncu_spectral_fast.txt).
// Here a line of L = 16 * R2 elements is held by R2 threads:
//   thread t owns x[t + R2 m], m = 0..15        (strided, coalesced across lines)
//   1. DFT-16 over m in registers                -> y_t[k1]
//   2. twiddle y_t[k1] *= W_L^{t k1}             (from the plan's W_L table)
//   3. one shared-memory transpose (row t, column k1; rows padded to 17)
//   4. DFT-R2 over t for each k1 the thread owns -> X[k1 + 16 k2]
// so a line FFT costs one shared write + one shared read per element.  Lines
// of a CTA are interleaved so that consecutive lanes are consecutive lines:
// every global load / store of a warp is a contiguous run along the line index.
// Inverse = conjugate twiddles (unnormalised, like the Stockham engine).
#pragma once

// resident CTAs / SM the f32 256-point line passes are compiled for (4, at 64
// registers with small spills, measured 0.663 vs 0.656 ms per shifted inverse)
#ifndef VR_F32_CTAS
#define VR_F32_CTAS 3
#endif

namespace vr {
namespace fs {

// W_16^m constants (forward sign), m = 0..15
__device__ __forceinline__ double w16c(int m) {
  constexpr double c[16] = {1.0, 0.92387953251128673848, 0.70710678118654752440, 0.38268343236508977173,
                            0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128673848,
                            -1.0, -0.92387953251128673848, -0.70710678118654752440, -0.38268343236508977173,
                            0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128673848};
  return c[m & 15];
}
__device__ __forceinline__ double w16s(int m) { return -w16c((m + 12) & 15); }   // -sin(2 pi m / 16)

template <typename C>
__device__ __forceinline__ C w16(int m, bool inv) {
  C w;
  w.x = (decltype(w.x))w16c(m);
  const double s = w16s(m);
  w.y = (decltype(w.y))(inv ? -s : s);
  return w;
}

// in-place DFT-16, natural order in and out
template <typename C>
__device__ __forceinline__ void dft16(C (&v)[16], bool inv) {
  // n = 4 n1 + n2, k = k1 + 4 k2
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4(v[n2], v[4 + n2], v[8 + n2], v[12 + n2], inv);   // v[4 k1 + n2]
#pragma unroll
  for (int k1 = 1; k1 < 4; ++k1)
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2) {
      const int m = k1 * n2;
      C& a = v[4 * k1 + n2];
      if (m == 4) a = rot(a, inv);   // W16^4 = -i
      else a = cmul(a, w16<C>(m, inv));
    }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3], inv);   // v[4 k1 + k2]
  C o[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) o[k1 + 4 * k2] = v[4 * k1 + k2];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = o[k];
}

// in-place DFT-8, natural order
template <typename C>
__device__ __forceinline__ void dft8(C (&v)[8], bool inv) {
  C e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  C o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4(e0, e1, e2, e3, inv);
  dft4(o0, o1, o2, o3, inv);
  o1 = cmul(o1, w16<C>(2, inv));
  o2 = rot(o2, inv);
  o3 = cmul(o3, w16<C>(6, inv));
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
}

template <int R2> __host__ __device__ constexpr int line_smem() { return R2 * 17 + 1; }   // elements, odd

// Steps 1-4 for one line held by R2 threads (thread t, 16 values x[t + R2 m] in v).
// `sm` = this line's shared scratch (line_smem<R2>() elements); `tw` = W_L table
// (L = 16 R2 entries, forward sign).  The CTA must __syncthreads() between calls
// that reuse `sm` (the caller owns the barrier because lines span warps).
// On return the thread owns X[k1 + 16 k2] for its k1 set:
//   R2 = 16: k1 = t, k2 = 0..15 -> v[k2]
//   R2 =  8: k1 = t and t + 8, k2 = 0..7 -> v[k2] (k1 = t), v[8 + k2] (k1 = t + 8)
template <typename C, int R2>
__device__ __forceinline__ void line_fft(C (&v)[16], int t, C* sm, const double2* __restrict__ tw, bool inv) {
  constexpr int L = 16 * R2;
  dft16(v, inv);
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) {
    double2 w = __ldg(tw + ((t * k1) & (L - 1)));
    if (inv) w.y = -w.y;
    v[k1] = cmul(v[k1], cvt<C>(w));
  }
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) sm[t * 17 + k1] = v[k1];
  __syncthreads();
  if constexpr (R2 == 16) {
#pragma unroll
    for (int s = 0; s < 16; ++s) v[s] = sm[s * 17 + t];
    dft16(v, inv);
  } else {
    C a[8], b[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      a[s] = sm[s * 17 + t];
      b[s] = sm[s * 17 + t + 8];
    }
    dft8(a, inv);
    dft8(b, inv);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      v[s] = a[s];
      v[8 + s] = b[s];
    }
  }
}

// output frequency of v[u] for thread t (see line_fft)
template <int R2>
__device__ __forceinline__ int out_freq(int t, int u) {
  if constexpr (R2 == 16) return t + 16 * u;
  else return (u < 8) ? t + 16 * u : t + 8 + 16 * (u - 8);
}

// ---- strided axis pass (x2 or plain x1), L = 256: NB lines (consecutive kz) per CTA,
// 16 threads per line, lane = line + NB * t.  grid (n_outer * nchunks, ncomp)
template <typename C, bool INV>
__global__ void __launch_bounds__(256, sizeof(C) == 8 ? VR_F32_CTAS : 2) axis256(C* __restrict__ S, int64_t es, int n_outer, int64_t outer_stride,
                                               int64_t comp_stride, int n3h, const double2* __restrict__ tw) {
  constexpr int R2 = 16, NB = 16;
  extern __shared__ __align__(16) unsigned char fs_smem[];
  C* smem = reinterpret_cast<C*>(fs_smem);
  const int q = threadIdx.x % NB, t = threadIdx.x / NB;
  const int nchunks = (n3h + NB - 1) / NB;
  const int o = blockIdx.x / nchunks, kz0 = (blockIdx.x - o * nchunks) * NB;
  const bool ok = kz0 + q < n3h;
  C* base = S + blockIdx.y * comp_stride + o * outer_stride + kz0 + q;
  C v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    if (ok) v[m] = base[(int64_t)(t + R2 * m) * es];
    else { v[m].x = 0; v[m].y = 0; }
  }
  line_fft<C, R2>(v, t, smem + q * line_smem<R2>(), tw, INV);
  if (ok) {
#pragma unroll
    for (int u = 0; u < 16; ++u) base[(int64_t)out_freq<R2>(t, u) * es] = v[u];
  }
}

// ---- X pass for 3-component operators, L = n1 = 256: forward (CF) -> symbol (f64)
// -> inverse (f32) -> T.  One CTA = fixed x2 row j, XB consecutive kz, all 3
// components: 3 * XB lines of 16 threads, lane = q + XB * (t + 16 c).
// The forward spectrum goes through one shared tile (per line, natural
// frequency order) so the symbol sees the 3 components of a wavenumber
// together (the Leray / K blend couples them); the inverse runs in f32 (its
// rounding is relative to the output, like the x2 / x3 inverse passes).
template <typename CF, int XB>
__global__ void __launch_bounds__(3 * XB * 16, (sizeof(CF) == 8 ? 20 : 12) / XB) xop256(const CF* __restrict__ S, float2* __restrict__ T, int n2,
                                                              int n3, int n3h, const double2* __restrict__ tw,
                                                              SpecOp op) {
  constexpr int R2 = 16, L = 256, LS = line_smem<R2>() > L ? line_smem<R2>() : L;
  extern __shared__ __align__(16) unsigned char fs_smem[];
  CF* tile = reinterpret_cast<CF*>(fs_smem);             // [c][q] lines of LS elements
  const int q = threadIdx.x % XB, t = (threadIdx.x / XB) % 16, c = threadIdx.x / (16 * XB);
  const int nchunks = (n3h + XB - 1) / XB;
  const int j = blockIdx.x / nchunks, kz0 = (blockIdx.x - j * nchunks) * XB;
  const bool ok = kz0 + q < n3h;
  const int64_t lstride = (int64_t)n2 * n3h;
  const CF* sb = S + (int64_t)j * n3h + kz0 + q;
  CF* line = tile + (c * XB + q) * LS;
  CF v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    if (ok) v[m] = sb[op.xoff(c, t + R2 * m, lstride)];
    else { v[m].x = 0; v[m].y = 0; }
  }
  line_fft<CF, R2>(v, t, line, tw, false);
  __syncthreads();   // every line finished reading its transpose scratch
#pragma unroll
  for (int u = 0; u < 16; ++u) line[out_freq<R2>(t, u)] = v[u];
  __syncthreads();
  // symbol at (k1 = freq along x1, k2 = row j, k3 = kz) for the 3 components
  const double k2 = (double)signed_freq(j + op.j0, op.n2g);
  for (int e = threadIdx.x; e < XB * L; e += blockDim.x) {
    const int qq = e / L, m = e - qq * L;
    double2 vals[3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) vals[cc] = to_d(tile[(cc * XB + qq) * LS + m]);
    apply_symbol(op, (double)signed_freq(m, L), k2, (double)(kz0 + qq), vals);
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) tile[(cc * XB + qq) * LS + m] = cvt<CF>(vals[cc]);
  }
  __syncthreads();
  float2 w[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const CF a = line[t + R2 * m];
    w[m] = make_float2((float)a.x, (float)a.y);
  }
  __syncthreads();   // the tile is reused as f32 transpose scratch
  float2* fline = reinterpret_cast<float2*>(fs_smem) + (c * XB + q) * LS;
  line_fft<float2, R2>(w, t, fline, tw, true);
  if (ok) {
    const int64_t rowoff = (int64_t)j * n3h + kz0 + q;
#pragma unroll
    for (int u = 0; u < 16; ++u) *op.out_at(T, c, out_freq<R2>(t, u), lstride, rowoff) = w[u];
  }
}

// ---- X pass for component-DIAGONAL symbols (A, shifted inverses, Gaussian),
// L = n1 = 256: one component per CTA row of the grid, NB = 16 consecutive kz
// per CTA (lane = q + NB t: every warp access is a 128-B contiguous run of
// float2, 256 B of double2), forward (CF) -> symbol in registers -> inverse
// (f32) -> T.  No shared tile: a line's spectrum never leaves its 16 threads
// (the symbol of a diagonal operator needs no other component), so the pass
// costs the two line FFTs' transposes only.  grid (n2 * nchunks, ncomp).
template <int R2>
__device__ __forceinline__ void diag_symbol_at(const SpecOp& op, int k1, double k2, double k3, double2& v) {
  double2 vals[1] = {v};
  SpecOp o1 = op;
  o1.ncomp = 1;
  apply_symbol(o1, (double)k1, k2, k3, vals);
  v = vals[0];
}

// FLAT: the CTA's NB lines are NB consecutive positions p = j n3h + kz of the
// (x2, kz) plane instead of NB kz of one x2 row -- every line load is one
// aligned 128-byte segment and no CTA idles on the odd n3h = n3 / 2 + 1
// (with 16 kz per row, 129 columns take 9 chunks, the last holding one).
template <typename CF, bool FLAT = false>
__global__ void __launch_bounds__(256, sizeof(CF) == 8 ? VR_F32_CTAS : 2) xdiag256(const CF* __restrict__ S,
                                                                      float2* __restrict__ T, int n2, int n3h,
                                                                      const double2* __restrict__ tw, SpecOp op) {
  constexpr int R2 = 16, NB = 16, L = 256;
  extern __shared__ __align__(16) unsigned char fs_smem[];
  const int q = threadIdx.x % NB, t = threadIdx.x / NB;
  int j, kz;
  bool ok;
  if (FLAT) {
    const int p = blockIdx.x * NB + q;
    ok = p < n2 * n3h;
    j = p / n3h;
    kz = p - j * n3h;
  } else {
    const int nchunks = (n3h + NB - 1) / NB;
    j = blockIdx.x / nchunks;
    kz = (blockIdx.x - j * nchunks) * NB + q;
    ok = kz < n3h;
  }
  const int c = blockIdx.y;
  const int64_t lstride = (int64_t)n2 * n3h;
  const CF* sb = S + (int64_t)j * n3h + kz;
  CF v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    if (ok) v[m] = sb[op.xoff(c, t + R2 * m, lstride)];
    else { v[m].x = 0; v[m].y = 0; }
  }
  CF* sm = reinterpret_cast<CF*>(fs_smem) + q * line_smem<R2>();
  line_fft<CF, R2>(v, t, sm, tw, false);
  const double k2 = (double)signed_freq(j + op.j0, op.n2g), k3 = (double)kz;
  float2 w[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    double2 a = to_d(v[u]);
    diag_symbol_at<R2>(op, signed_freq(out_freq<R2>(t, u), L), k2, k3, a);
    w[u] = make_float2((float)a.x, (float)a.y);
  }
  __syncthreads();   // transpose scratch reused by the inverse
  line_fft<float2, R2>(w, t, reinterpret_cast<float2*>(fs_smem) + q * line_smem<R2>(), tw, true);
  if (ok) {
    const int64_t rowoff = (int64_t)j * n3h + kz;
#pragma unroll
    for (int u = 0; u < 16; ++u) *op.out_at(T, c, out_freq<R2>(t, u), lstride, rowoff) = w[u];
  }
}

// ---- distributed x2 passes with the transpose fused in (L = n2 = 256) -------
// Between the slab layout [c][i][j][kz] and the rank-blocked transpose layout
// [r][c][i][jl][kz] (j = r L2 + jl, r = the x2 block's owner):
//   forward (INV = false): x2 FFT of the slab spectrum `in`; output row j is
//     stored straight into rank r = j / L2's receive buffer dst[r] at the
//     sender's block `me` (NVLink stores: pack + all-to-all are this kernel's
//     epilogue);
//   inverse (INV = true): rows loaded from this rank's receive buffer `in` in
//     the blocked layout (unpack fused into the loads), x2 inverse FFT, stored
//     to the slab spectrum `out`.
struct X2Peer {
  void* dst[8];
  int me, l2shift, ncomp;
};

template <typename C, bool INV>
__global__ void __launch_bounds__(256, sizeof(C) == 8 ? 3 : 2) axis256_dist(const C* __restrict__ in,
                                                                          C* __restrict__ out, X2Peer pe, int L1,
                                                                          int n3h, const double2* __restrict__ tw) {
  constexpr int R2 = 16, NB = 16, N2 = 256;
  extern __shared__ __align__(16) unsigned char fs_smem[];
  C* smem = reinterpret_cast<C*>(fs_smem);
  const int q = threadIdx.x % NB, t = threadIdx.x / NB;
  const int nchunks = (n3h + NB - 1) / NB;
  const int i = blockIdx.x / nchunks, kz0 = (blockIdx.x - i * nchunks) * NB, c = blockIdx.y;
  const bool ok = kz0 + q < n3h;
  const int L2 = N2 >> pe.l2shift, jshift = 8 - pe.l2shift;   // row j -> (r, jl) = (j >> jshift, j & (L2-1))
  auto slab_off = [&](int j) -> int64_t { return (((int64_t)c * L1 + i) * N2 + j) * n3h + kz0 + q; };
  auto blk_off = [&](int r, int jl) -> int64_t {
    return ((((int64_t)r * pe.ncomp + c) * L1 + i) * L2 + jl) * n3h + kz0 + q;
  };
  C v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int j = t + R2 * m;
    if (ok) v[m] = INV ? in[blk_off(j >> jshift, j & (L2 - 1))] : in[slab_off(j)];
    else { v[m].x = 0; v[m].y = 0; }
  }
  line_fft<C, R2>(v, t, smem + q * line_smem<R2>(), tw, INV);
  if (ok) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int j = out_freq<R2>(t, u);
      if (INV) out[slab_off(j)] = v[u];
      else reinterpret_cast<C*>(select_ptr(pe.dst, j >> jshift))[blk_off(pe.me, j & (L2 - 1))] = v[u];
    }
  }
  // (no per-thread system fence: the completion flag is stored by a kernel
  // ordered behind this one on the stream, after its own fence.sys -- a
  // per-thread fence here measured 0.185 vs ~0.12 ms per component)
}

}  // namespace fs
}  // namespace vr

// ---------------------------------------------------------------------------------
// Three-step register FFT for long lines, L = 16 x 16 x R3 (R3 in {2, 4, 8}:
// L = 512 / 1024 / 2048 -- the x1 lines of the transposed block in an x1-slab
// run on 2 / 4 / 8 GPUs).  T = 16 R3 threads per line, 16 values per thread:
//   forward  x[t + T m] -[DFT-16 over m]-[x W_L^{t k1}]-> transpose 1
//            -[DFT-16 over t_hi (t = t_lo + R3 t_hi)]-[x W_T^{t_lo k1'}]-> transpose 2
//            -[DFT-R3 over t_lo]-> X[k1 + 16 (k1' + 16 k2')]
//   inverse  the same stages run BACKWARD with conjugate twiddles (the DFT is
//            unitary up to scale: F^H = D1^H W1^H P1^T D2^H W2^H P2^T D3^H), so
//            the spectrum never needs reordering and the result lands back in
//            the input layout x[t + T m] (unnormalised, like the other engines).
// Two shared transposes per transform (the Stockham radix-8 path needs one
// round trip per stage) and -- with NB lines interleaved per CTA -- 128-B
// coalesced row segments for the strided x1 lines.
namespace vr {
namespace fs {
namespace lf3 {

template <int R3> __host__ __device__ constexpr int T() { return 16 * R3; }
// per-line shared elements, odd so that interleaved lines start on distinct banks
template <int R3> __host__ __device__ constexpr int smem_elems() {
  return ((16 * R3 * 17) > (256 * (R3 + 1)) ? (16 * R3 * 17) : (256 * (R3 + 1))) | 1;
}

// in-register DFT of R3 (2 / 4 / 8) values, natural order
template <typename C, int R>
__device__ __forceinline__ void dft_r(C (&v)[R], bool inv) {
  if constexpr (R == 2) {
    const C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    dft4(v[0], v[1], v[2], v[3], inv);
  } else {
    dft8(v, inv);
  }
}

template <typename C>
__device__ __forceinline__ C tw_at(const double2* __restrict__ tw, int idx, bool inv) {
  double2 w = __ldg(tw + idx);
  if (inv) w.y = -w.y;
  return cvt<C>(w);
}

// pair p = (k1, k1') of stage 3 owned by thread u: p = u + T s, s < 16 / R3
// forward: v holds x[t + T m] on entry, on exit v[s * R3 + k2'] = X[k1 + 16 (k1' + 16 k2')]
// twiddles come from the W_L table: W_T^m = W_L^(16 m)
template <typename C, int R3>
__device__ __forceinline__ void forward(C (&v)[16], int u, C* sm, const double2* __restrict__ twL) {
  constexpr int Tn = T<R3>(), L = 256 * R3;
  dft16(v, false);
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) v[k1] = cmul(v[k1], tw_at<C>(twL, (u * k1) & (L - 1), false));
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) sm[u * 17 + k1] = v[k1];
  __syncthreads();
  {
    const int k1 = u / R3, tlo = u - (u / R3) * R3;   // stage-2 pair (k1, t_lo)
#pragma unroll
    for (int th = 0; th < 16; ++th) v[th] = sm[(tlo + R3 * th) * 17 + k1];
    dft16(v, false);
#pragma unroll
    for (int q = 1; q < 16; ++q) v[q] = cmul(v[q], tw_at<C>(twL, 16 * ((tlo * q) & (Tn - 1)), false));
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) sm[(k1 * 16 + q) * (R3 + 1) + tlo] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 16 / R3; ++s) {
    const int p = u + Tn * s;
    C r[R3];
#pragma unroll
    for (int tl = 0; tl < R3; ++tl) r[tl] = sm[p * (R3 + 1) + tl];
    dft_r<C, R3>(r, false);
#pragma unroll
    for (int k2 = 0; k2 < R3; ++k2) v[s * R3 + k2] = r[k2];
  }
}

// frequency of v[s * R3 + k2] after forward (pair p = u + T s = k1 * 16 + k1')
template <int R3>
__device__ __forceinline__ int freq(int u, int idx) {
  const int s = idx / R3, k2 = idx - s * R3;
  const int p = u + T<R3>() * s, k1 = p >> 4, k1p = p & 15;
  return k1 + 16 * (k1p + 16 * k2);
}

// inverse: the forward's stages backward with conjugate twiddles (layouts as
// produced by forward); on exit v holds x[t + T m] (times L)
template <typename C, int R3>
__device__ __forceinline__ void inverse(C (&v)[16], int u, C* sm, const double2* __restrict__ twL) {
  constexpr int Tn = T<R3>(), L = 256 * R3;
#pragma unroll
  for (int s = 0; s < 16 / R3; ++s) {
    const int p = u + Tn * s;
    C r[R3];
#pragma unroll
    for (int k2 = 0; k2 < R3; ++k2) r[k2] = v[s * R3 + k2];
    dft_r<C, R3>(r, true);
#pragma unroll
    for (int tl = 0; tl < R3; ++tl) sm[p * (R3 + 1) + tl] = r[tl];
  }
  __syncthreads();
  const int k1 = u / R3, tlo = u - (u / R3) * R3;
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = sm[(k1 * 16 + q) * (R3 + 1) + tlo];
#pragma unroll
  for (int q = 1; q < 16; ++q) v[q] = cmul(v[q], tw_at<C>(twL, 16 * ((tlo * q) & (Tn - 1)), true));
  dft16(v, true);
  __syncthreads();
#pragma unroll
  for (int th = 0; th < 16; ++th) sm[(tlo + R3 * th) * 17 + k1] = v[th];
  __syncthreads();
#pragma unroll
  for (int k1b = 0; k1b < 16; ++k1b) v[k1b] = sm[u * 17 + k1b];
#pragma unroll
  for (int k1b = 1; k1b < 16; ++k1b) v[k1b] = cmul(v[k1b], tw_at<C>(twL, (u * k1b) & (L - 1), true));
  dft16(v, true);
}

}  // namespace lf3

// X pass for component-diagonal symbols on long lines (L = 256 R3): NB
// consecutive kz per CTA (lane = q + NB u), one component per grid row;
// forward in CF, symbol, inverse in f32 -> T (or the peer destinations).
// FLAT: lines over the flat (x2, kz) plane, as xdiag256<., true>
template <typename CF, int R3, int NB, bool FLAT = false>
__global__ void __launch_bounds__(NB * 16 * R3, 1) xdiag_long(const CF* __restrict__ S, float2* __restrict__ T,
                                                              int n2, int n3h, const double2* __restrict__ twL,
                                                              SpecOp op) {
  constexpr int Tn = lf3::T<R3>(), L = 256 * R3, LS = lf3::smem_elems<R3>();
  extern __shared__ __align__(16) unsigned char fs_smem[];
  const int q = threadIdx.x % NB, u = threadIdx.x / NB;
  int j, kz;
  bool ok;
  if (FLAT) {
    const int p = blockIdx.x * NB + q;
    ok = p < n2 * n3h;
    j = p / n3h;
    kz = p - j * n3h;
  } else {
    const int nchunks = (n3h + NB - 1) / NB;
    j = blockIdx.x / nchunks;
    kz = (blockIdx.x - j * nchunks) * NB + q;
    ok = kz < n3h;
  }
  const int c = blockIdx.y;
  const int64_t lstride = (int64_t)n2 * n3h;
  const CF* sb = S + (int64_t)j * n3h + kz;
  CF v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    if (ok) v[m] = sb[op.xoff(c, u + Tn * m, lstride)];
    else { v[m].x = 0; v[m].y = 0; }
  }
  lf3::forward<CF, R3>(v, u, reinterpret_cast<CF*>(fs_smem) + q * LS, twL);
  const double k2 = (double)signed_freq(j + op.j0, op.n2g), k3 = (double)kz;
  float2 w[16];
#pragma unroll
  for (int idx = 0; idx < 16; ++idx) {
    double2 a = to_d(v[idx]);
    diag_symbol_at<16>(op, signed_freq(lf3::freq<R3>(u, idx), L), k2, k3, a);
    w[idx] = make_float2((float)a.x, (float)a.y);
  }
  __syncthreads();   // the shared buffer is reused by the f32 inverse
  lf3::inverse<float2, R3>(w, u, reinterpret_cast<float2*>(fs_smem) + q * LS, twL);
  if (ok) {
    const int64_t rowoff = (int64_t)j * n3h + kz;
#pragma unroll
    for (int m = 0; m < 16; ++m) *op.out_at(T, c, u + Tn * m, lstride, rowoff) = w[m];
  }
}

}  // namespace fs
}  // namespace vr

namespace vr {
namespace fs {

// ---- the coupled K symbol on long x1 lines: three passes through a scratch
// spectrum W ([c][k][j][kz], natural frequency order), since a 3-component
// register tile of 512-2048-point lines does not fit:
//   xfwd_long (per component) -> xsym3 (elementwise, couples the components)
//   -> xinv_long (per component, loads each thread's frequencies, backward stages)
template <int R3, int NB>
__global__ void __launch_bounds__(NB * 16 * R3, 1) xfwd_long(const float2* __restrict__ S, float2* __restrict__ W,
                                                             int n2, int n3h, const double2* __restrict__ twL,
                                                             SpecOp op) {
  constexpr int Tn = lf3::T<R3>(), L = 256 * R3, LS = lf3::smem_elems<R3>();
  extern __shared__ __align__(16) unsigned char fs_smem[];
  const int q = threadIdx.x % NB, u = threadIdx.x / NB;
  const int nchunks = (n3h + NB - 1) / NB;
  const int j = blockIdx.x / nchunks, kz0 = (blockIdx.x - j * nchunks) * NB, c = blockIdx.y;
  const bool ok = kz0 + q < n3h;
  const int64_t lstride = (int64_t)n2 * n3h;
  const float2* sb = S + (int64_t)j * n3h + kz0 + q;
  float2 v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    if (ok) v[m] = sb[op.xoff(c, u + Tn * m, lstride)];
    else v[m] = make_float2(0.f, 0.f);
  }
  lf3::forward<float2, R3>(v, u, reinterpret_cast<float2*>(fs_smem) + q * LS, twL);
  if (ok) {
    float2* wb = W + ((int64_t)c * L * n2 + j) * n3h + kz0 + q;
#pragma unroll
    for (int idx = 0; idx < 16; ++idx) wb[(int64_t)lf3::freq<R3>(u, idx) * lstride] = v[idx];
  }
}

// K (apply_symbol, 3 components) at every (k1, j, kz) of W, in place
__global__ void __launch_bounds__(256) xsym3(float2* __restrict__ W, int L, int n2, int n3h, SpecOp op) {
  const int64_t per = (int64_t)L * n2 * n3h;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per) return;
  const int kz = (int)(e % n3h);
  const int64_t r = e / n3h;
  const int j = (int)(r % n2), k = (int)(r / n2);
  double2 vals[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) vals[c] = to_d(W[c * per + e]);
  apply_symbol(op, (double)signed_freq(k, L), (double)signed_freq(j + op.j0, op.n2g), (double)kz, vals);
#pragma unroll
  for (int c = 0; c < 3; ++c) W[c * per + e] = make_float2((float)vals[c].x, (float)vals[c].y);
}

template <int R3, int NB>
__global__ void __launch_bounds__(NB * 16 * R3, 1) xinv_long(const float2* __restrict__ W, float2* __restrict__ T,
                                                             int n2, int n3h, const double2* __restrict__ twL,
                                                             SpecOp op) {
  constexpr int Tn = lf3::T<R3>(), L = 256 * R3, LS = lf3::smem_elems<R3>();
  extern __shared__ __align__(16) unsigned char fs_smem[];
  const int q = threadIdx.x % NB, u = threadIdx.x / NB;
  const int nchunks = (n3h + NB - 1) / NB;
  const int j = blockIdx.x / nchunks, kz0 = (blockIdx.x - j * nchunks) * NB, c = blockIdx.y;
  const bool ok = kz0 + q < n3h;
  const int64_t lstride = (int64_t)n2 * n3h;
  const float2* wb = W + ((int64_t)c * L * n2 + j) * n3h + kz0 + q;
  float2 v[16];
#pragma unroll
  for (int idx = 0; idx < 16; ++idx) v[idx] = ok ? wb[(int64_t)lf3::freq<R3>(u, idx) * lstride] : make_float2(0.f, 0.f);
  lf3::inverse<float2, R3>(v, u, reinterpret_cast<float2*>(fs_smem) + q * LS, twL);
  if (ok) {
    const int64_t rowoff = (int64_t)j * n3h + kz0 + q;
#pragma unroll
    for (int m = 0; m < 16; ++m) *op.out_at(T, c, u + Tn * m, lstride, rowoff) = v[m];
  }
}

}  // namespace fs
}  // namespace vr

namespace vr {
namespace fs {

// ---- x3 passes for 256-point real rows: two rows as one complex line --------
// Forward: z = a + i b (rows 2p, 2p+1), four-step line FFT, then the two half
// spectra from Z and its mirror (A_k = (Z_k + conj Z_{N-k}) / 2,
// B_k = (Z_k - conj Z_{N-k}) / 2i); the mirror Z_{N-k} of thread t's Z_{t+16u}
// lives in thread (16 - t) & 15 at u' = 15 - u (thread 0: its own (16 - u) & 15),
// fetched with one shuffle per value.  Inverse: Z_k = A_k + i B_k with the
// Hermitian mirror for k > 128 (DC / Nyquist imaginary parts dropped, as
// pocketfft's c2r does), inverse line FFT, a = Re, b = Im (+ addend).
// 16 threads per pair, 16 pairs per 256-thread CTA, grid (pairs / 16, ncomp).
template <typename CF>
__global__ void __launch_bounds__(256, sizeof(CF) == 8 ? 3 : 2) zfwd256_pair(const float* __restrict__ in, int npairs,
                                                                          int64_t nvox, int64_t nspec,
                                                                          const double2* __restrict__ tw,
                                                                          CF* __restrict__ S) {
  constexpr int L = 256, NH = 129;
  extern __shared__ __align__(16) unsigned char fs_smem[];
  const int t = threadIdx.x & 15, q = threadIdx.x >> 4;
  const int pr = blockIdx.x * 16 + q;
  const bool ok = pr < npairs;
  const float* ra = in + blockIdx.y * nvox + (int64_t)(ok ? pr : 0) * 2 * L;
  const float* rb = ra + L;
  CF v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    v[m].x = __ldg(ra + t + 16 * m);
    v[m].y = __ldg(rb + t + 16 * m);
  }
  line_fft<CF, 16>(v, t, reinterpret_cast<CF*>(fs_smem) + q * line_smem<16>(), tw, false);
  // thread t holds Z[t + 16 u] in v[u]
  using R = decltype(v[0].x);
  const int lane = threadIdx.x & 31, base = lane & 16;
  const int partner = base + ((16 - t) & 15);
  CF* da = S + blockIdx.y * nspec + (int64_t)(ok ? pr : 0) * 2 * NH;
  CF* db = da + NH;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    CF m;
    m.x = __shfl_sync(0xffffffffu, v[15 - u].x, partner);
    m.y = __shfl_sync(0xffffffffu, v[15 - u].y, partner);
    if (t == 0) m = v[(16 - u) & 15];
    const int k = t + 16 * u;
    if (ok && k <= 128) {
      CF A, B;
      A.x = R(0.5) * (v[u].x + m.x);
      A.y = R(0.5) * (v[u].y - m.y);
      B.x = R(0.5) * (v[u].y + m.y);
      B.y = R(-0.5) * (v[u].x - m.x);
      da[k] = A;
      db[k] = B;
    }
  }
}

__global__ void __launch_bounds__(256, 3) zinv256_pair(const float2* __restrict__ T, int npairs, int64_t nvox,
                                                      int64_t nspec, const double2* __restrict__ tw,
                                                      float* __restrict__ out, const float* __restrict__ add) {
  constexpr int L = 256, NH = 129;
  extern __shared__ __align__(16) unsigned char fs_smem[];
  const int t = threadIdx.x & 15, q = threadIdx.x >> 4;
  const int pr = blockIdx.x * 16 + q;
  const bool ok = pr < npairs;
  const float2* sa = T + blockIdx.y * nspec + (int64_t)(ok ? pr : 0) * 2 * NH;
  const float2* sb = sa + NH;
  float2 v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int k = t + 16 * m;
    const bool mir = k > 128;
    const int kk = mir ? L - k : k;
    float2 A = __ldg(sa + kk), B = __ldg(sb + kk);
    if (kk == 0 || kk == 128) { A.y = 0.f; B.y = 0.f; }   // c2r ignores Im of DC / Nyquist
    if (mir) { A.y = -A.y; B.y = -B.y; }
    v[m] = make_float2(A.x - B.y, A.y + B.x);               // Z = A + i B
  }
  line_fft<float2, 16>(v, t, reinterpret_cast<float2*>(fs_smem) + q * line_smem<16>(), tw, true);
  if (ok) {
    float* oa = out + blockIdx.y * nvox + (int64_t)pr * 2 * L;
    float* ob = oa + L;
    const float* aa = add ? add + blockIdx.y * nvox + (int64_t)pr * 2 * L : nullptr;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int x = t + 16 * u;
      float ya = v[u].x, yb = v[u].y;
      if (aa) {
        ya += __ldg(aa + x);
        yb += __ldg(aa + L + x);
      }
      oa[x] = ya;
      ob[x] = yb;
    }
  }
}

}  // namespace fs
}  // namespace vr
