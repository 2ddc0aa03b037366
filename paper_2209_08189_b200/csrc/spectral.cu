// Spectral operators on hand-written batched mixed-radix FFT stages.
//
// Reference: /root/reference/pkg/src/velreg/diffops.py
//   SpectralWorkspace (:24-55)  -> vr_spec_plan (wavenumbers, rfft layout, multiplicity)
//   apply_A (:116-118)          -> SPEC_A      symbol |k|^2
//   apply_inv_shifted_A (:121)  -> SPEC_INVSHIFT symbol 1/(beta_v |k|^2 + shift)
//   apply_K (:129-146)          -> SPEC_K      Leray blend (couples the 3 components)
//   h1_energy (:149-154)        -> vr_h1_energy (forward transform + weighted reduction)
// numpy's rfftn/irfftn(s=dims) are pocketfft; this file re-derives the same
// transforms as a 3-pass pipeline per component:
//   Z  : real rows (x3) -> half spectrum (n3/2+1), f64           [fwd_z_kernel]
//   Y  : c2c along x2 (strided tiles staged in smem), f64         [y_kernel]
//   X  : c2c along x1 forward, operator multiply, c2c inverse, all
//        in one kernel (the operator is diagonal in k)             [x_op_kernel]
//   Y' : c2c inverse along x2, f32                                [y_kernel]
//   Z' : Hermitian c2r along x3 (imag of DC/Nyquist dropped, as pocketfft's
//        c2r does), f32, with a fused "+ addend" epilogue        [inv_z_kernel]
// The forward half runs in f64 (storage + arithmetic): the |k|^2 symbol
// amplifies absolute rounding at high k, and an f32 forward path cannot meet the
// 1e-5 operator tolerance at 256^3.  After the multiply the
// output is O(|A v|) so the inverse half runs in f32.
//
// Each line FFT is an out-of-place Stockham DIT over shared memory; radices
// 8/4/2 (powers of two), 3/5/7 (register butterflies) and any other prime via a
// direct O(R) stage, so every even grid size the reference accepts works
// (e.g. the CLARITY sizes 2816 = 2^8*11, 3016 = 2^3*13*29, 1162 = 2*7*83).
#include <vector>
#include <new>
#include <type_traits>
#include <algorithm>
#include <mutex>
#include <utility>
#include "common.cuh"
#include "../../include/velreg_b200.h"

namespace vr {

struct RadixPlan {
  int L;
  int ns;
  int r[24];
};

static RadixPlan make_radix_plan(int L) {
  RadixPlan p{};
  p.L = L;
  int m = L;
  const int pref[3] = {8, 4, 2};
  for (int q : pref)
    while (m % q == 0) { p.r[p.ns++] = q; m /= q; }
  for (int q = 3; m > 1; q += 2)
    while (m % q == 0) { p.r[p.ns++] = q; m /= q; }
  return p;
}

// ---- complex helpers -------------------------------------------------------
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <typename C> __device__ __forceinline__ C cvt(double2 w);
template <> __device__ __forceinline__ double2 cvt<double2>(double2 w) { return w; }
template <> __device__ __forceinline__ float2 cvt<float2>(double2 w) { return make_float2((float)w.x, (float)w.y); }
template <typename C> __device__ __forceinline__ C cvt_from(double2 w) { return cvt<C>(w); }
__device__ __forceinline__ double2 to_d(float2 a) { return make_double2(a.x, a.y); }
__device__ __forceinline__ double2 to_d(double2 a) { return a; }
// multiply by -i (forward) or +i (inverse)
template <typename C> __device__ __forceinline__ C rot(C a, bool inv) {
  C r;
  if (inv) { r.x = -a.y; r.y = a.x; } else { r.x = a.y; r.y = -a.x; }
  return r;
}
// twiddle W^m (forward e^{-2 pi i m/L}; inverse is the conjugate)
template <typename C> __device__ __forceinline__ C twid(const double2* tw, int m, bool inv) {
  double2 w = tw[m];
  if (inv) w.y = -w.y;
  return cvt<C>(w);
}

template <typename C>
__device__ __forceinline__ void dft4(C& a0, C& a1, C& a2, C& a3, bool inv) {
  C t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = rot(csub(a1, a3), inv);
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

template <typename C, int R>
__device__ __forceinline__ void dft_reg(C* v, const double2* tw, int L, bool inv) {
  if (R == 2) {
    C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if (R == 4) {
    dft4(v[0], v[1], v[2], v[3], inv);
  } else if (R == 8) {
    C e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    C o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4(e0, e1, e2, e3, inv);
    dft4(o0, o1, o2, o3, inv);
    const double s = 0.70710678118654752440;
    // W8^1 = s(1 -+ i), W8^2 = -+i, W8^3 = s(-1 -+ i)
    C w1, w3;
    w1.x = s; w1.y = inv ? s : -s;
    w3.x = -s; w3.y = inv ? s : -s;
    o1 = cmul(o1, w1);
    o2 = rot(o2, inv);
    o3 = cmul(o3, w3);
    v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
    v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
    v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
    v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
  } else {
    // small odd radix: direct DFT with the line's twiddle table (W_R = W_L^(L/R))
    C out[R];
    const int st = L / R;
#pragma unroll
    for (int s = 0; s < R; ++s) {
      C acc = v[0];
#pragma unroll
      for (int r = 1; r < R; ++r) acc = cadd(acc, cmul(v[r], twid<C>(tw, ((r * s) % R) * st, inv)));
      out[s] = acc;
    }
#pragma unroll
    for (int s = 0; s < R; ++s) v[s] = out[s];
  }
}

template <typename C, int R>
__device__ __forceinline__ void stage_reg(const C* __restrict__ src, C* __restrict__ dst, int L, int nb, int j,
                                          int Ns, const double2* tw, bool inv) {
  const int k = j % Ns;
  const int st = L / (Ns * R);
  C v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    v[r] = src[j + r * nb];
    if (r > 0 && k > 0) v[r] = cmul(v[r], twid<C>(tw, r * k * st, inv));
  }
  dft_reg<C, R>(v, tw, L, inv);
  const int idxD = (j / Ns) * Ns * R + k;
#pragma unroll
  for (int r = 0; r < R; ++r) dst[idxD + r * Ns] = v[r];
}

template <typename C>
__device__ void stage_generic(const C* __restrict__ src, C* __restrict__ dst, int L, int R, int nb, int j, int Ns,
                              const double2* tw, bool inv) {
  const int k = j % Ns;
  const int st = L / (Ns * R);
  const int sR = L / R;
  const int idxD = (j / Ns) * Ns * R + k;
  for (int s = 0; s < R; ++s) {
    C acc = src[j];
    for (int r = 1; r < R; ++r) {
      C x = src[j + r * nb];
      if (k > 0) x = cmul(x, twid<C>(tw, r * k * st, inv));
      acc = cadd(acc, cmul(x, twid<C>(tw, ((r * s) % R) * sR, inv)));
    }
    dst[idxD + s * Ns] = acc;
  }
}

// nl lines of length L (line stride ls) in `a`; `b` is scratch of the same
// shape.  Returns the buffer holding the (naturally ordered) result.
template <typename C>
__device__ C* line_fft(C* a, C* b, int ls, int nl, const RadixPlan& rp, const double2* tw, bool inv) {
  const int L = rp.L;
  int Ns = 1;
  for (int s = 0; s < rp.ns; ++s) {
    const int R = rp.r[s];
    const int nb = L / R;
    const int total = nl * nb;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int line = t / nb, j = t - line * nb;
      const C* src = a + line * ls;
      C* dst = b + line * ls;
      switch (R) {
        case 2: stage_reg<C, 2>(src, dst, L, nb, j, Ns, tw, inv); break;
        case 4: stage_reg<C, 4>(src, dst, L, nb, j, Ns, tw, inv); break;
        case 8: stage_reg<C, 8>(src, dst, L, nb, j, Ns, tw, inv); break;
        case 3: stage_reg<C, 3>(src, dst, L, nb, j, Ns, tw, inv); break;
        case 5: stage_reg<C, 5>(src, dst, L, nb, j, Ns, tw, inv); break;
        case 7: stage_reg<C, 7>(src, dst, L, nb, j, Ns, tw, inv); break;
        default: stage_generic<C>(src, dst, L, R, nb, j, Ns, tw, inv); break;
      }
    }
    __syncthreads();
    C* t = a; a = b; b = t;
    Ns *= R;
  }
  return a;
}

__device__ __forceinline__ void load_twiddles(double2* tw_s, const double2* __restrict__ tw, int L) {
  for (int t = threadIdx.x; t < L; t += blockDim.x) tw_s[t] = tw[t];
}

// ptrs[r] for a per-rank pointer array held in kernel parameters, by a select
// chain: dynamic indexing would copy the array to local memory (ptxas stack)
__device__ __forceinline__ void* select_ptr(void* const (&ptrs)[8], int r) {
  void* d = ptrs[0];
#pragma unroll
  for (int q = 1; q < 8; ++q)
    if (r == q) d = ptrs[q];
  return d;
}

// ---- operator symbols (applied between the forward and inverse x1 passes) ----
struct SpecOp {
  int kind;
  int ncomp;
  double beta_v, beta_w, shift, scale, sigma;
  int j0, n2g;   // x2 offset / global x2 size of this tile (distributed transposed X pass)
  int xblk;      // x1 rows per rank block: element (c, x1 = p*xblk + i) lives at
                 // ((p*ncomp + c)*xblk + i) * lstride  (xblk = n1 for a single domain)
  __host__ __device__ int64_t xoff(int c, int i, int64_t lstride) const {
    const int p = i / xblk;
    return ((int64_t)(p * ncomp + c) * xblk + (i - p * xblk)) * lstride;
  }
  // distributed X pass with peer output (spectral transposes over NVLink):
  // block p (x1 rows [p xblk, (p+1) xblk)) is stored straight into rank p's
  // receive buffer pdst[p] at the sender's block `me` ([me][c][il][jl][kz]).
  void* pdst[8] = {};
  int me = 0;
  __device__ __forceinline__ float2* out_at(float2* T, int c, int i, int64_t lstride, int64_t rowoff) const {
    const int p = i / xblk;
    if (pdst[0])
      return reinterpret_cast<float2*>(select_ptr(pdst, p)) + ((int64_t)(me * ncomp + c) * xblk + (i - p * xblk)) * lstride +
             rowoff;
    return T + xoff(c, i, lstride) + rowoff;
  }
};

__device__ __forceinline__ int signed_freq(int m, int n) { return m < n / 2 ? m : m - n; }  // fftfreq*n

// vals[c] for c < op.ncomp at wavenumber (k1,k2,k3); result in place.
__device__ __forceinline__ void apply_symbol(const SpecOp& op, double k1, double k2, double k3, double2* vals) {
  const double ksq = k1 * k1 + k2 * k2 + k3 * k3;  // diffops.py:38 (exact integers)
  switch (op.kind) {
    case VR_SPEC_A: {  // diffops.py:116-118
      const double m = ksq * op.scale;
      for (int c = 0; c < op.ncomp; ++c) { vals[c].x *= m; vals[c].y *= m; }
    } break;
    case VR_SPEC_INVSHIFT: {  // diffops.py:121-126
      const double m = (1.0 / (op.beta_v * ksq + op.shift)) * op.scale;
      for (int c = 0; c < op.ncomp; ++c) { vals[c].x *= m; vals[c].y *= m; }
    } break;
    case VR_SPEC_K: {  // diffops.py:129-146
      if (ksq > 0.0) {
        const double a = ksq, b = 1.0 + ksq;
        const double cb = (op.beta_w * b) / (op.beta_v * a + op.beta_w * b);
        const double2 kd = make_double2(k1 * vals[0].x + k2 * vals[1].x + k3 * vals[2].x,
                                        k1 * vals[0].y + k2 * vals[1].y + k3 * vals[2].y);
        const double f = cb * (1.0 / ksq);
        const double2 sc = make_double2(f * kd.x, f * kd.y);
        const double kk[3] = {k1, k2, k3};
        for (int c = 0; c < 3; ++c) {
          vals[c].x = (vals[c].x - kk[c] * sc.x) * op.scale;
          vals[c].y = (vals[c].y - kk[c] * sc.y) * op.scale;
        }
      } else {
        for (int c = 0; c < 3; ++c) { vals[c].x *= op.scale; vals[c].y *= op.scale; }
      }
    } break;
    case VR_SPEC_GAUSS: {  // Gaussian smoothing exp(-sigma^2 |k|^2 / 2) (north-star extra)
      const double m = exp(-0.5 * op.sigma * op.sigma * ksq) * op.scale;
      for (int c = 0; c < op.ncomp; ++c) { vals[c].x *= m; vals[c].y *= m; }
    } break;
    case VR_SPEC_A2: {  // H2 seminorm operator, symbol |k|^4 (north-star extra)
      const double m = ksq * ksq * op.scale;
      for (int c = 0; c < op.ncomp; ++c) { vals[c].x *= m; vals[c].y *= m; }
    } break;
    case VR_SPEC_INVSHIFT2: {  // inverse of beta_v A2 + shift
      const double m = (1.0 / (op.beta_v * ksq * ksq + op.shift)) * op.scale;
      for (int c = 0; c < op.ncomp; ++c) { vals[c].x *= m; vals[c].y *= m; }
    } break;
    default: {  // VR_SPEC_IDENTITY: pure round trip
      for (int c = 0; c < op.ncomp; ++c) { vals[c].x *= op.scale; vals[c].y *= op.scale; }
    }
  }
}

// ---- pass kernels ---------------------------------------------------------------
// Z forward: real rows -> half spectrum (f64).  grid (ceil(rows/RB), ncomp)
__global__ void __launch_bounds__(256) fwd_z_kernel(const float* __restrict__ in, Dims d, int n3h, RadixPlan rp,
                                                    const double2* __restrict__ tw, int RB,
                                                    double2* __restrict__ S) {
  extern __shared__ double2 smd[];
  const int L = d.n3, ls = L + 1;
  double2* tw_s = smd;
  double2* a = tw_s + L;
  double2* b = a + RB * ls;
  load_twiddles(tw_s, tw, L);
  const int nrows = d.n1 * d.n2;
  const int row0 = blockIdx.x * RB;
  const int nr = min(RB, nrows - row0);
  const int c = blockIdx.y;
  const float* src = in + (int64_t)c * d.n() + (int64_t)row0 * L;
  for (int t = threadIdx.x; t < nr * L; t += blockDim.x) {
    const int r = t / L, k = t - r * L;
    a[r * ls + k] = make_double2((double)__ldg(src + t), 0.0);
  }
  __syncthreads();
  double2* res = line_fft<double2>(a, b, ls, nr, rp, tw_s, false);
  double2* dst = S + (int64_t)c * d.n1 * d.n2 * n3h + (int64_t)row0 * n3h;
  for (int t = threadIdx.x; t < nr * n3h; t += blockDim.x) {
    const int r = t / n3h, k = t - r * n3h;
    dst[t] = res[r * ls + k];
  }
}

// Strided-axis c2c pass in place on C-typed spectra (the Y pass, and the plain
// X pass used by resampling).  Lines of length L with element stride `es`;
// `n_outer` independent line sets `outer_stride` apart; B consecutive kz per
// CTA so the global reads are B*sizeof(C)-byte contiguous segments.
// grid (n_outer*nchunks, ncomp)
template <typename C>
__global__ void __launch_bounds__(256) axis_kernel(C* __restrict__ S, int L, int64_t es, int n_outer,
                                                   int64_t outer_stride, int64_t comp_stride, int n3h,
                                                   RadixPlan rp, const double2* __restrict__ tw, int B, int inv) {
  extern __shared__ double2 smd[];
  const int ls = L + 1;
  double2* tw_s = smd;
  C* a = reinterpret_cast<C*>(tw_s + L);
  C* b = a + B * ls;
  load_twiddles(tw_s, tw, L);
  const int nchunks = (n3h + B - 1) / B;
  const int o = blockIdx.x / nchunks, kz0 = (blockIdx.x - o * nchunks) * B;
  const int nb = min(B, n3h - kz0);
  C* base = S + blockIdx.y * comp_stride + o * outer_stride + kz0;
  for (int t = threadIdx.x; t < L * nb; t += blockDim.x) {
    const int j = t / nb, q = t - j * nb;
    a[q * ls + j] = base[j * es + q];
  }
  __syncthreads();
  C* res = line_fft<C>(a, b, ls, nb, rp, tw_s, inv != 0);
  for (int t = threadIdx.x; t < L * nb; t += blockDim.x) {
    const int j = t / nb, q = t - j * nb;
    base[j * es + q] = res[q * ls + j];
  }
}

// Spectral zero-padding for prolongation (grid.py:181-208): every fine mode
// takes the coarse mode it maps to along each axis, halving at the two split
// Nyquist positions; the x3 (half) axis keeps only the positive Nyquist half,
// its mirror being implied by Hermitian symmetry in the c2r pass.  Scaled by
// 1/N_coarse (= N_t/N_s product scale times the 1/N_t inverse normalisation).
__device__ __forceinline__ int pad_src(int t, int ns, int nt, double& w) {
  w = 1.0;
  if (nt == ns) return t;
  const int half = ns / 2;
  if (t < half) return t;
  if (t == half || t == nt - half) { w = 0.5; return half; }
  if (t > nt - half) return t - nt + ns;
  w = 0.0;
  return 0;
}

__global__ void pad_kernel(const double2* __restrict__ Sc, Dims dc, int n3hc, float2* __restrict__ Tf, Dims df,
                           int n3hf, int ncomp, double scale) {
  const int64_t nspec_f = (int64_t)df.n1 * df.n2 * n3hf;
  const int64_t nspec_c = (int64_t)dc.n1 * dc.n2 * n3hc;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nspec_f * ncomp;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / nspec_f);
    int64_t r = e - c * nspec_f;
    const int kz = (int)(r % n3hf);
    r /= n3hf;
    const int j = (int)(r % df.n2), i = (int)(r / df.n2);
    double w1, w2, w3 = 1.0;
    const int si = pad_src(i, dc.n1, df.n1, w1), sj = pad_src(j, dc.n2, df.n2, w2);
    int sk = kz;
    if (df.n3 != dc.n3) {
      const int half = dc.n3 / 2;
      if (kz < half) sk = kz;
      else if (kz == half) { sk = half; w3 = 0.5; }
      else { sk = 0; w3 = 0.0; }
    }
    const double w = w1 * w2 * w3 * scale;
    float2 out = make_float2(0.f, 0.f);
    if (w != 0.0) {
      const double2 v = Sc[c * nspec_c + ((int64_t)si * dc.n2 + sj) * n3hc + sk];
      out = make_float2((float)(w * v.x), (float)(w * v.y));
    }
    Tf[e] = out;
  }
}

// X pass: forward c2c (f64) -> symbol -> inverse c2c (f64) -> store f32 into T.
// REDUCE: instead, accumulate the H1 energy sum mult*(1+|k|^2)*|F|^2 (diffops.py:149-154).
template <bool REDUCE>
__global__ void __launch_bounds__(256) x_op_kernel(const double2* __restrict__ S, float2* __restrict__ T, Dims d,
                                                   int n3h, RadixPlan rp, const double2* __restrict__ tw, int B,
                                                   SpecOp op, double* __restrict__ partials) {
  extern __shared__ double2 smd[];
  const int L = d.n1, ls = L + 1, NC = op.ncomp;
  double2* tw_s = smd;
  double2* a = tw_s + L;
  double2* b = a + NC * B * ls;
  load_twiddles(tw_s, tw, L);
  const int nchunks = (n3h + B - 1) / B;
  const int j = blockIdx.x / nchunks, kz0 = (blockIdx.x - j * nchunks) * B;
  const int nb = min(B, n3h - kz0);
  const int64_t cstride = (int64_t)d.n1 * d.n2 * n3h;
  const int64_t lstride = (int64_t)d.n2 * n3h;
  const double2* sbase = S + (int64_t)j * n3h + kz0;
  for (int t = threadIdx.x; t < NC * L * nb; t += blockDim.x) {
    const int c = t / (L * nb);
    const int r = t - c * L * nb;
    const int i = r / nb, q = r - i * nb;
    a[(c * B + q) * ls + i] = sbase[op.xoff(c, i, lstride) + q];
  }
  // unused lines (q >= nb) are left untouched; they never reach memory
  __syncthreads();
  double2* res = line_fft<double2>(a, b, ls, NC * B, rp, tw_s, false);
  double2* other = (res == a) ? b : a;
  const double k2 = (double)signed_freq(j + op.j0, op.n2g);
  if (REDUCE) {
    double acc = 0.0;
    for (int t = threadIdx.x; t < L * nb; t += blockDim.x) {
      const int q = t / L, m = t - q * L;
      const double k1 = (double)signed_freq(m, d.n1), k3 = (double)(kz0 + q);
      const double ksq = k1 * k1 + k2 * k2 + k3 * k3;
      const int kz = kz0 + q;
      const double mult = (kz == 0 || (d.n3 % 2 == 0 && kz == n3h - 1)) ? 1.0 : 2.0;  // diffops.py:45-49
      const double2 v = res[q * ls + m];
      acc += mult * (1.0 + ksq) * (v.x * v.x + v.y * v.y);
    }
    // deterministic block reduction
    __shared__ double red[32];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      double x = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      x = warp_sum(x);
      if (threadIdx.x == 0) partials[blockIdx.x] = x;
    }
    return;
  }
  for (int t = threadIdx.x; t < L * nb; t += blockDim.x) {
    const int q = t / L, m = t - q * L;
    const double k1 = (double)signed_freq(m, d.n1), k3 = (double)(kz0 + q);
    double2 vals[3];
    for (int c = 0; c < NC; ++c) vals[c] = res[(c * B + q) * ls + m];
    apply_symbol(op, k1, k2, k3, vals);
    for (int c = 0; c < NC; ++c) res[(c * B + q) * ls + m] = vals[c];
  }
  __syncthreads();
  double2* out = line_fft<double2>(res, other, ls, NC * B, rp, tw_s, true);
  for (int t = threadIdx.x; t < NC * L * nb; t += blockDim.x) {
    const int c = t / (L * nb);
    const int r = t - c * L * nb;
    const int i = r / nb, q = r - i * nb;
    const double2 v = out[(c * B + q) * ls + i];
    *op.out_at(T, c, i, lstride, (int64_t)j * n3h + kz0 + q) = make_float2((float)v.x, (float)v.y);
  }
}

// Z inverse: Hermitian half rows (f32) -> real rows, out = x (+ add).
__global__ void __launch_bounds__(256) inv_z_kernel(const float2* __restrict__ T, Dims d, int n3h, RadixPlan rp,
                                                    const double2* __restrict__ tw, int RB,
                                                    float* __restrict__ out, const float* __restrict__ add) {
  extern __shared__ double2 smd[];
  const int L = d.n3, ls = L + 1;
  double2* tw_s = smd;
  float2* a = reinterpret_cast<float2*>(tw_s + L);
  float2* b = a + RB * ls;
  load_twiddles(tw_s, tw, L);
  const int nrows = d.n1 * d.n2;
  const int row0 = blockIdx.x * RB;
  const int nr = min(RB, nrows - row0);
  const int c = blockIdx.y;
  const float2* src = T + (int64_t)c * nrows * n3h + (int64_t)row0 * n3h;
  for (int t = threadIdx.x; t < nr * n3h; t += blockDim.x) {
    const int r = t / n3h, k = t - r * n3h;
    float2 v = src[t];
    if (k == 0 || (k == n3h - 1 && (L % 2 == 0))) v.y = 0.0f;  // c2r ignores imag of DC/Nyquist
    a[r * ls + k] = v;
    if (k > 0 && L - k > k) a[r * ls + (L - k)] = make_float2(v.x, -v.y);
  }
  __syncthreads();
  float2* res = line_fft<float2>(a, b, ls, nr, rp, tw_s, true);
  const int64_t off = (int64_t)c * d.n() + (int64_t)row0 * L;
  for (int t = threadIdx.x; t < nr * L; t += blockDim.x) {
    const int r = t / L, k = t - r * L;
    float v = res[r * ls + k].x;
    if (add) v += __ldg(add + off + t);
    out[off + t] = v;
  }
}

__global__ void finalize_sum_kernel(const double* __restrict__ partials, int n, double scale,
                                    double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) acc += partials[t];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double x = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    x = warp_sum(x);
    if (threadIdx.x == 0) *out = x * scale;
  }
}

}  // namespace vr

#include "spectral_fast.cuh"
#include "spectral_4step.cuh"
#include "spectral_d2.cuh"

// Four-step register FFT kernels (spectral_4step.cuh) for the line lengths they
// cover; vr_set_fft_mode(0) selects the Stockham engine for A/B checks.
static int g_fft_mode = 1;
// A = |k|^2 through the separable f64 line engine (spectral_d2.cuh) where the
// line lengths allow; vr_set_spec_a_mode(0) selects the 3-D f64 path.
static int g_a_mode = 1;
// x1 pass of component-diagonal symbols without the 3-component shared tile
// (fs::xdiag256); vr_set_fft_mode(2) turns it off for A/B checks.
static bool g_xdiag = true;
// diagonal symbols on 3-component fields: one component at a time (L2 reuse of
// the half spectrum).  Measured slower on B200 at 256^3 (shifted inverse 0.714
// vs 0.656 ms, A 3-D 0.898 vs 0.841 ms: three times the launches and tails for
// no DRAM saving), so off by default; kept as an A/B switch.
static int g_percomp = 0;

using namespace vr;


struct vr_spec_plan {
  Dims d;
  int n3h;
  int64_t nspec;  // n1*n2*n3h
  bool fast;      // n1, n2, n3/2 powers of two in [8, 2048]
  RadixPlan rp1, rp2, rp3;
  double2 *tw1, *tw2, *tw3, *tw3h;  // W_n1, W_n2, W_n3, W_{n3/2}
  double2 *stw1, *stw2, *stw3h;     // fast path: per-stage tables (2L entries)
  double2* S;      // 3 * nspec (forward, f64)
  float2* T;       // 3 * nspec (inverse, f32)
  double* partials;
  int RBz, RBzi, Bx1, Bx3;
  size_t smz, smzi, smx1, smx3;
  int device;
};

namespace {

int pow2_floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

bool is_pow2_in(int x, int lo, int hi) { return x >= lo && x <= hi && (x & (x - 1)) == 0; }

int choose_lines(int L, int ncomp, size_t elem, size_t budget, int cap) {
  int B = (int)(budget / (2 * (size_t)ncomp * (L + 1) * elem));
  if (B < 1) B = 1;
  B = pow2_floor(B);
  return B > cap ? cap : B;
}

int upload_twiddles(int L, double2** out) {
  std::vector<double2> h(L);
  for (int m = 0; m < L; ++m) {
    double ang = -kTwoPi * (double)m / (double)L;
    h[m] = make_double2(cos(ang), sin(ang));
  }
  if (cudaMalloc(out, sizeof(double2) * L) != cudaSuccess) return VR_ERR_ALLOC;
  if (cudaMemcpy(*out, h.data(), sizeof(double2) * L, cudaMemcpyHostToDevice) != cudaSuccess) return VR_ERR_ALLOC;
  return VR_OK;
}

// Per-stage twiddles of the fast Stockham engine: entry NS + k = W_{NS R}^k for
// every stage (span NS > 1, radix R = min(8, L / NS)); stages are powers of 8
// apart, so the ranges [NS, 2 NS) are disjoint and lanes read consecutive slots.
int upload_stage_twiddles(int L, double2** out) {
  std::vector<double2> h(2 * (size_t)L, make_double2(1.0, 0.0));
  for (int ns = 8; ns < L; ns *= 8) {
    const int R = std::min(8, L / ns);
    for (int k = 0; k < ns; ++k) {
      double ang = -kTwoPi * (double)k / (double)(ns * R);
      h[ns + k] = make_double2(cos(ang), sin(ang));
    }
  }
  if (cudaMalloc(out, sizeof(double2) * h.size()) != cudaSuccess) return VR_ERR_ALLOC;
  if (cudaMemcpy(*out, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return VR_ERR_ALLOC;
  return VR_OK;
}

const size_t kSmemBudget = 200 * 1024;

// ---- fast-path launch helpers (compile-time sizes) ---------------------------------
#define VR_POW2_SWITCH(L, CASE)                                                                  \
  switch (L) {                                                                                   \
    case 8: CASE(8); break;                                                                      \
    case 16: CASE(16); break;                                                                    \
    case 32: CASE(32); break;                                                                    \
    case 64: CASE(64); break;                                                                    \
    case 128: CASE(128); break;                                                                  \
    case 256: CASE(256); break;                                                                  \
    case 512: CASE(512); break;                                                                  \
    case 1024: CASE(1024); break;                                                                \
    case 2048: CASE(2048); break;                                                                \
    default: break;                                                                              \
  }

template <int L> constexpr size_t fast_lines() { return 2048 / L; }
constexpr size_t padl(size_t L) { return L + L / 8 + 1; }

size_t sm_z(int M, size_t elem) { return sizeof(double2) * (3 * (size_t)M + 1) + elem * (2048 / M) * padl(M); }
size_t sm_zi(int M) { return sizeof(double2) * 2 * M + sizeof(float2) * (2048 / M) * padl(M); }
size_t sm_axis(int L, size_t elem) { return sizeof(double2) * 2 * L + elem * (2048 / L) * padl(L); }
int xb(int L, int nc) { return (nc == 3 ? 1024 : 2048) / L; }
size_t sm_x(int L, int nc, size_t elem) { return sizeof(double2) * 2 * L + elem * nc * xb(L, nc) * padl(L); }

template <typename F> void set_smem(F* f, size_t bytes) {
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void fast_attributes(int n1, int n2, int M) {
#define A_Z(MM)                                               \
  set_smem(fast::zfwd_fast<MM, double2>, sm_z(MM, 16));       \
  set_smem(fast::zfwd_fast<MM, float2>, sm_z(MM, 8));         \
  set_smem(fast::zinv_fast<MM>, sm_zi(MM));
#define A_AX(LL)                                              \
  set_smem(fast::axis_fast<double2, LL, false>, sm_axis(LL, 16)); \
  set_smem(fast::axis_fast<double2, LL, true>, sm_axis(LL, 16));  \
  set_smem(fast::axis_fast<float2, LL, false>, sm_axis(LL, 8));   \
  set_smem(fast::axis_fast<float2, LL, true>, sm_axis(LL, 8));
#define A_X(LL)                                                        \
  A_AX(LL)                                                             \
  set_smem(fast::xop_fast<LL, 3, false, double2>, sm_x(LL, 3, 16));    \
  set_smem(fast::xop_fast<LL, 3, false, float2>, sm_x(LL, 3, 8));      \
  set_smem(fast::xop_fast<LL, 1, false, double2>, sm_x(LL, 1, 16));    \
  set_smem(fast::xop_fast<LL, 1, false, float2>, sm_x(LL, 1, 8));      \
  set_smem(fast::xop_fast<LL, 1, true, double2>, sm_x(LL, 1, 16));
  VR_POW2_SWITCH(M, A_Z)
  VR_POW2_SWITCH(n2, A_AX)
  VR_POW2_SWITCH(n1, A_X)
#undef A_Z
#undef A_AX
#undef A_X
}

// Operators whose symbol amplifies high wavenumbers (|k|^2, |k|^4, the H1
// weights) need the forward transform in f64; bounded symbols
// (shifted inverses, K, Gaussian) run the forward half in f32.
bool needs_f64(int kind) { return kind == VR_SPEC_A || kind == VR_SPEC_A2; }

}  // namespace

extern "C" {

int vr_set_fft_mode(int mode) {
  // 0: Stockham only; 1 (default): four-step kernels incl. the diagonal x1 pass;
  // 2: four-step kernels with the 3-component x1 tile for every symbol
  const int prev = g_fft_mode == 0 ? 0 : (g_xdiag ? 1 : 2);
  g_fft_mode = mode != 0;
  g_xdiag = mode == 1;
  return prev;
}


int vr_spec_plan_create(const int64_t dims[3], vr_spec_plan** out) {
  if (!out) return VR_ERR_ARG;
  *out = nullptr;
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (d.n1 < 2 || d.n2 < 2 || d.n3 < 2 || (d.n3 % 2)) return VR_ERR_DIMS;
  vr_spec_plan* p = new (std::nothrow) vr_spec_plan();
  if (!p) return VR_ERR_ALLOC;
  p->d = d;
  p->n3h = d.n3 / 2 + 1;
  p->nspec = (int64_t)d.n1 * d.n2 * p->n3h;
  p->fast = is_pow2_in(d.n1, 8, 2048) && is_pow2_in(d.n2, 8, 2048) && is_pow2_in(d.n3 / 2, 8, 2048);
  p->rp1 = make_radix_plan(d.n1);
  p->rp2 = make_radix_plan(d.n2);
  p->rp3 = make_radix_plan(d.n3);
  cudaGetDevice(&p->device);
  rc = upload_twiddles(d.n1, &p->tw1);
  if (!rc) rc = upload_twiddles(d.n2, &p->tw2);
  if (!rc) rc = upload_twiddles(d.n3, &p->tw3);
  if (!rc) rc = upload_twiddles(d.n3 / 2, &p->tw3h);
  if (!rc && p->fast) rc = upload_stage_twiddles(d.n1, &p->stw1);
  if (!rc && p->fast) rc = upload_stage_twiddles(d.n2, &p->stw2);
  if (!rc && p->fast) rc = upload_stage_twiddles(d.n3 / 2, &p->stw3h);
  // S / T (the 3-component spectrum scratch, 36 B per voxel) are allocated on
  // first use (ensure_scratch): the transposed-block plan of the peer path
  // never touches them -- its input is the receive buffer and its output goes
  // straight to the peers
  const int maxblk = d.n2 * p->n3h + 1024;
  if (!rc && cudaMalloc(&p->partials, sizeof(double) * maxblk) != cudaSuccess) rc = VR_ERR_ALLOC;
  if (rc) {
    vr_spec_plan_destroy(p);
    return rc;
  }
  // generic path tile shapes: ~2-4K complex elements per CTA within the smem budget
  const size_t kLines = 4096;
  p->RBz = (int)std::max<size_t>(1, std::min<size_t>(16, kLines / d.n3));
  p->RBzi = p->RBz;
  p->smz = sizeof(double2) * (d.n3 + 2 * (size_t)p->RBz * (d.n3 + 1));
  p->smzi = sizeof(double2) * d.n3 + sizeof(float2) * 2 * (size_t)p->RBzi * (d.n3 + 1);
  p->Bx3 = std::min(choose_lines(d.n1, 3, sizeof(double2), 110 * 1024, 8), pow2_floor(p->n3h));
  p->Bx1 = std::min(choose_lines(d.n1, 1, sizeof(double2), 110 * 1024, 16), pow2_floor(p->n3h));
  p->smx3 = sizeof(double2) * (d.n1 + 2 * 3 * (size_t)p->Bx3 * (d.n1 + 1));
  p->smx1 = sizeof(double2) * (d.n1 + 2 * 1 * (size_t)p->Bx1 * (d.n1 + 1));
  const size_t sy = sizeof(double2) * (d.n2 + 2 * (size_t)choose_lines(d.n2, 1, sizeof(double2), 110 * 1024, 16) *
                                                 (d.n2 + 1));
  // (a 3-component x1 tile over budget only rules out the coupled K on this
  // plan -- vr_spec_apply / vr_dspec_xpass report VR_ERR_UNSUPPORTED for it)
  if (!p->fast && (p->smz > kSmemBudget || p->smzi > kSmemBudget || sy > kSmemBudget || p->smx1 > kSmemBudget)) {
    vr_spec_plan_destroy(p);
    return VR_ERR_UNSUPPORTED;
  }
  cudaFuncSetAttribute(fwd_z_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
  cudaFuncSetAttribute(inv_z_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
  cudaFuncSetAttribute(axis_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
  cudaFuncSetAttribute(axis_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
  cudaFuncSetAttribute(x_op_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
  cudaFuncSetAttribute(x_op_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
  if (p->fast) fast_attributes(d.n1, d.n2, d.n3 / 2);
  *out = p;
  return VR_OK;
}

int vr_spec_plan_destroy(vr_spec_plan* p) {
  if (!p) return VR_OK;
  cudaFree(p->tw1);
  cudaFree(p->tw2);
  cudaFree(p->tw3);
  cudaFree(p->tw3h);
  cudaFree(p->stw1);
  cudaFree(p->stw2);
  cudaFree(p->stw3h);
  cudaFree(p->S);
  cudaFree(p->T);
  cudaFree(p->partials);
  delete p;
  return VR_OK;
}

}  // extern "C"

// stream-ordered scratch stays in the default pool between calls (release
// threshold 0 would hand it back to the OS at every synchronisation)
static void keep_default_pool() {
  static thread_local int done_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

// Opt a kernel into `bytes` of dynamic shared memory once per (device, kernel,
// size).  Keyed on the kernel's address: template instances that differ only
// in non-type parameters share a function TYPE, so a per-type static flag
// would skip the opt-in for all but the first of them.
template <typename F> static void smem_optin(F* f, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, size_t>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const std::pair<const void*, int> key{reinterpret_cast<const void*>(f), dev};
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : done)
    if (e.first == key && e.second >= bytes) return;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  done.push_back({key, bytes});
}

// strided c2c pass along x1 (axis 1) or x2 (axis 2) over ncomp spectra
template <typename C>
static void launch_axis(vr_spec_plan* p, C* buf, int axis, int ncomp, int inv, cudaStream_t s) {
  const Dims& d = p->d;
  const bool ax2 = axis == 2;
  const int L = ax2 ? d.n2 : d.n1;
  const int64_t es = ax2 ? (int64_t)p->n3h : (int64_t)d.n2 * p->n3h;
  const int n_outer = ax2 ? d.n1 : d.n2;
  const int64_t outer_stride = ax2 ? (int64_t)d.n2 * p->n3h : (int64_t)p->n3h;
  if (p->fast && g_fft_mode && L == 256) {
    const int nchunks = (p->n3h + 15) / 16;
    const size_t sm = sizeof(C) * 16 * fs::line_smem<16>();
    const double2* twL = ax2 ? p->tw2 : p->tw1;
    if (inv) {
      smem_optin(fs::axis256<C, true>, sm);
      fs::axis256<C, true><<<dim3(n_outer * nchunks, ncomp), 256, sm, s>>>(buf, es, n_outer, outer_stride, p->nspec,
                                                                          p->n3h, twL);
    } else {
      smem_optin(fs::axis256<C, false>, sm);
      fs::axis256<C, false><<<dim3(n_outer * nchunks, ncomp), 256, sm, s>>>(buf, es, n_outer, outer_stride, p->nspec,
                                                                           p->n3h, twL);
    }
    return;
  }
  if (p->fast) {
    const double2* tw = ax2 ? p->stw2 : p->stw1;
#define L_AX(LL)                                                                                      \
  {                                                                                                   \
    const int B = (int)fast_lines<LL>();                                                              \
    const int nchunks = (p->n3h + B - 1) / B;                                                         \
    if (inv)                                                                                          \
      fast::axis_fast<C, LL, true><<<dim3(n_outer * nchunks, ncomp), 256, sm_axis(LL, sizeof(C)), s>>>( \
          buf, es, n_outer, outer_stride, p->nspec, p->n3h, tw);                                      \
    else                                                                                              \
      fast::axis_fast<C, LL, false><<<dim3(n_outer * nchunks, ncomp), 256, sm_axis(LL, sizeof(C)), s>>>( \
          buf, es, n_outer, outer_stride, p->nspec, p->n3h, tw);                                      \
  }
    VR_POW2_SWITCH(L, L_AX)
#undef L_AX
    return;
  }
  const int B = std::min(choose_lines(L, 1, sizeof(C), 110 * 1024, 16), pow2_floor(p->n3h));
  const size_t sm = sizeof(double2) * L + sizeof(C) * 2 * (size_t)B * (L + 1);
  const int nchunks = (p->n3h + B - 1) / B;
  axis_kernel<C><<<dim3(n_outer * nchunks, ncomp), 256, sm, s>>>(buf, L, es, n_outer, outer_stride, p->nspec,
                                                                 p->n3h, ax2 ? p->rp2 : p->rp1,
                                                                 ax2 ? p->tw2 : p->tw1, B, inv);
}

static int ensure_scratch(vr_spec_plan* p, bool need_s = true, bool need_t = true) {
  if (need_s && !p->S && cudaMalloc(&p->S, sizeof(double2) * 3 * p->nspec) != cudaSuccess) return VR_ERR_ALLOC;
  if (need_t && !p->T && cudaMalloc(&p->T, sizeof(float2) * 3 * p->nspec) != cudaSuccess) return VR_ERR_ALLOC;
  return VR_OK;
}

// forward Z + Y passes into p->S (as double2, or as float2 when !f64 on the fast path)
// x3 passes of 256-point rows as paired-row four-step kernels (fs::zfwd256_pair /
// zinv256_pair); vr_set_spectral_tuning(2, 0) selects the Stockham kernels
static int g_zpair = 1;
static int g_xflat = 1;   // vr_set_spectral_tuning(4, .): x1 passes (xdiag256 / xdiag_long) over the flat (x2, kz) plane
static bool zpair_ok(const vr_spec_plan* p) {
  return g_zpair && g_fft_mode && p->fast && p->d.n3 == 256 && (p->d.n1 * p->d.n2) % 2 == 0;
}
template <typename CF>
static void zfwd_pair(vr_spec_plan* p, const float* in, int ncomp, cudaStream_t s) {
  const int npairs = p->d.n1 * p->d.n2 / 2;
  const size_t sm = sizeof(CF) * 16 * fs::line_smem<16>();
  smem_optin(fs::zfwd256_pair<CF>, sm);
  fs::zfwd256_pair<CF><<<dim3((npairs + 15) / 16, ncomp), 256, sm, s>>>(in, npairs, p->d.n(), p->nspec, p->tw3,
                                                                        reinterpret_cast<CF*>(p->S));
}
static void zinv_pair(vr_spec_plan* p, int ncomp, const float* add, float* out, cudaStream_t s) {
  const int npairs = p->d.n1 * p->d.n2 / 2;
  const size_t sm = sizeof(float2) * 16 * fs::line_smem<16>();
  smem_optin(fs::zinv256_pair, sm);
  fs::zinv256_pair<<<dim3((npairs + 15) / 16, ncomp), 256, sm, s>>>(p->T, npairs, p->d.n(), p->nspec, p->tw3, out,
                                                                    add);
}

static int spec_forward(vr_spec_plan* p, const float* in, int ncomp, cudaStream_t s, bool f64 = true) {
  const Dims& d = p->d;
  const int nrows = d.n1 * d.n2;
  if (p->fast && zpair_ok(p)) {
    if (f64) {
      zfwd_pair<double2>(p, in, ncomp, s);
      launch_axis<double2>(p, p->S, 2, ncomp, 0, s);
    } else {
      zfwd_pair<float2>(p, in, ncomp, s);
      launch_axis<float2>(p, reinterpret_cast<float2*>(p->S), 2, ncomp, 0, s);
    }
    VR_CHECK_LAUNCH();
    return VR_OK;
  }
  if (p->fast) {
    const int M = d.n3 / 2;
#define L_Z(MM)                                                                                            \
  {                                                                                                        \
    const dim3 g((nrows + (int)fast_lines<MM>() - 1) / (int)fast_lines<MM>(), ncomp);                     \
    if (f64)                                                                                               \
      fast::zfwd_fast<MM, double2><<<g, 256, sm_z(MM, 16), s>>>(in, nrows, d.n(), p->nspec, p->stw3h, p->tw3, \
                                                                p->S);                                     \
    else                                                                                                   \
      fast::zfwd_fast<MM, float2><<<g, 256, sm_z(MM, 8), s>>>(in, nrows, d.n(), p->nspec, p->stw3h, p->tw3,  \
                                                              reinterpret_cast<float2*>(p->S));            \
  }
    VR_POW2_SWITCH(M, L_Z)
#undef L_Z
    if (f64)
      launch_axis<double2>(p, p->S, 2, ncomp, 0, s);
    else
      launch_axis<float2>(p, reinterpret_cast<float2*>(p->S), 2, ncomp, 0, s);
    VR_CHECK_LAUNCH();
    return VR_OK;
  } else {
    fwd_z_kernel<<<dim3((nrows + p->RBz - 1) / p->RBz, ncomp), 256, p->smz, s>>>(in, d, p->n3h, p->rp3, p->tw3,
                                                                                 p->RBz, p->S);
  }
  launch_axis<double2>(p, p->S, 2, ncomp, 0, s);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// Z forward pass only (fast path) into p->S
static void spec_forward_z(vr_spec_plan* p, const float* in, int ncomp, cudaStream_t s, bool f64) {
  if (zpair_ok(p)) {
    if (f64) zfwd_pair<double2>(p, in, ncomp, s);
    else zfwd_pair<float2>(p, in, ncomp, s);
    return;
  }
  const Dims& d = p->d;
  const int nrows = d.n1 * d.n2;
  const int M = d.n3 / 2;
#define L_Z(MM)                                                                                            \
  {                                                                                                        \
    const dim3 g((nrows + (int)fast_lines<MM>() - 1) / (int)fast_lines<MM>(), ncomp);                     \
    if (f64)                                                                                               \
      fast::zfwd_fast<MM, double2><<<g, 256, sm_z(MM, 16), s>>>(in, nrows, d.n(), p->nspec, p->stw3h, p->tw3, \
                                                                p->S);                                     \
    else                                                                                                   \
      fast::zfwd_fast<MM, float2><<<g, 256, sm_z(MM, 8), s>>>(in, nrows, d.n(), p->nspec, p->stw3h, p->tw3,  \
                                                              reinterpret_cast<float2*>(p->S));            \
  }
  VR_POW2_SWITCH(M, L_Z)
#undef L_Z
}

// Z inverse pass only (fast path): p->T -> out (+ add)
static void spec_inverse_z(vr_spec_plan* p, int ncomp, const float* add, float* out, cudaStream_t s) {
  if (zpair_ok(p)) {
    zinv_pair(p, ncomp, add, out, s);
    return;
  }
  const Dims& d = p->d;
  const int nrows = d.n1 * d.n2;
  const int M = d.n3 / 2;
#define L_ZI(MM)                                                                                          \
  fast::zinv_fast<MM><<<dim3((nrows + (int)fast_lines<MM>() - 1) / (int)fast_lines<MM>(), ncomp), 256,    \
                        sm_zi(MM), s>>>(p->T, nrows, d.n(), p->nspec, p->stw3h, p->tw3, out, add);
  VR_POW2_SWITCH(M, L_ZI)
#undef L_ZI
}

static void spec_inverse_yz(vr_spec_plan* p, int ncomp, const float* add, float* out, cudaStream_t s) {
  const Dims& d = p->d;
  launch_axis<float2>(p, p->T, 2, ncomp, 1, s);
  if (zpair_ok(p)) {
    zinv_pair(p, ncomp, add, out, s);
    return;
  }
  const int nrows = d.n1 * d.n2;
  if (p->fast) {
    const int M = d.n3 / 2;
#define L_ZI(MM)                                                                                          \
  fast::zinv_fast<MM><<<dim3((nrows + (int)fast_lines<MM>() - 1) / (int)fast_lines<MM>(), ncomp), 256,    \
                        sm_zi(MM), s>>>(p->T, nrows, d.n(), p->nspec, p->stw3h, p->tw3, out, add);
    VR_POW2_SWITCH(M, L_ZI)
#undef L_ZI
    return;
  }
  inv_z_kernel<<<dim3((nrows + p->RBzi - 1) / p->RBzi, ncomp), 256, p->smzi, s>>>(p->T, d, p->n3h, p->rp3, p->tw3,
                                                                                  p->RBzi, out, add);
}

// X pass: fwd -> op -> inv (or the H1 reduction); returns number of CTAs
static int spec_xpass(vr_spec_plan* p, const SpecOp& op, bool reduce, cudaStream_t s, bool f64 = true,
                      const void* Sext = nullptr, float2* Text = nullptr) {
  const Dims& d = p->d;
  const int nc = op.ncomp;
  const double2* Sd = Sext ? reinterpret_cast<const double2*>(Sext) : p->S;
  float2* Tt = Text ? Text : p->T;
  if (p->fast && g_fft_mode && d.n1 == 256 && !reduce && op.kind != VR_SPEC_K && g_xdiag) {
    // component-diagonal symbol: one component per CTA row, no shared tile
    const int nchunks = (p->n3h + 15) / 16;
    const dim3 g(g_xflat ? (d.n2 * p->n3h + 15) / 16 : d.n2 * nchunks, nc);
#define XD256(CF, FL)                                                                                         \
  {                                                                                                          \
    const size_t sm = sizeof(CF) * 16 * fs::line_smem<16>();                                                 \
    smem_optin(fs::xdiag256<CF, FL>, sm);                                                                    \
    fs::xdiag256<CF, FL><<<g, 256, sm, s>>>(reinterpret_cast<const CF*>(Sd), Tt, d.n2, p->n3h, p->tw1, op); \
  }
    if (f64 && g_xflat) XD256(double2, true)
    else if (f64) XD256(double2, false)
    else if (g_xflat) XD256(float2, true)
    else XD256(float2, false)
#undef XD256
    return g.x;
  }
  if (p->fast && g_fft_mode && g_xdiag && !reduce && op.kind != VR_SPEC_K &&
      (d.n1 == 512 || d.n1 == 1024 || d.n1 == 2048)) {
    // long x1 lines (the transposed block of a 2 / 4 / 8-rank x1-slab run):
    // three-step register FFT, one component per grid row
#define XLONG_LAUNCH(CF, R3, NB, FL)                                                                          \
  {                                                                                                          \
    const int nblk = FL ? (d.n2 * p->n3h + NB - 1) / NB : d.n2 * ((p->n3h + NB - 1) / NB);                   \
    const size_t sm = sizeof(CF) * NB * fs::lf3::smem_elems<R3>();                                           \
    smem_optin(fs::xdiag_long<CF, R3, NB, FL>, sm);                                                          \
    fs::xdiag_long<CF, R3, NB, FL><<<dim3(nblk, nc), NB * 16 * R3, sm, s>>>(                                 \
        reinterpret_cast<const CF*>(Sd), Tt, d.n2, p->n3h, p->tw1, op);                                      \
    return nblk;                                                                                             \
  }
#define XLONG(R3, NBF, NBD)                                                                                  \
  {                                                                                                          \
    if (f64 && g_xflat) XLONG_LAUNCH(double2, R3, NBD, true)                                                 \
    else if (f64) XLONG_LAUNCH(double2, R3, NBD, false)                                                      \
    else if (g_xflat) XLONG_LAUNCH(float2, R3, NBF, true)                                                    \
    else XLONG_LAUNCH(float2, R3, NBF, false)                                                                \
  }
    if (d.n1 == 512) XLONG(2, 16, 8)
    if (d.n1 == 1024) XLONG(4, 8, 8)
    XLONG(8, 4, 4)
#undef XLONG
#undef XLONG_LAUNCH
  }
  if (p->fast && g_fft_mode && g_xdiag && !reduce && op.kind == VR_SPEC_K && nc == 3 && !f64 &&
      (d.n1 == 512 || d.n1 == 1024 || d.n1 == 2048)) {
    // the coupled K on long x1 lines: forward per component into a scratch
    // spectrum W (natural frequency order), the 3-component symbol
    // elementwise, inverse per component (fs::xfwd_long / xsym3 / xinv_long)
    const int64_t wn = 3 * (int64_t)d.n1 * d.n2 * p->n3h;
    float2* W = nullptr;
    keep_default_pool();
    if (cudaMallocAsync((void**)&W, sizeof(float2) * wn, s) != cudaSuccess) return -1;
    const float2* S32 = reinterpret_cast<const float2*>(Sd);
    int nblk = 0;
#define KLONG(R3, NB)                                                                                        \
  {                                                                                                          \
    const int nch = (p->n3h + NB - 1) / NB;                                                                  \
    const size_t sm = sizeof(float2) * NB * fs::lf3::smem_elems<R3>();                                       \
    smem_optin(fs::xfwd_long<R3, NB>, sm);                                                                   \
    smem_optin(fs::xinv_long<R3, NB>, sm);                                                                   \
    fs::xfwd_long<R3, NB><<<dim3(d.n2 * nch, 3), NB * 16 * R3, sm, s>>>(S32, W, d.n2, p->n3h, p->tw1, op);   \
    const int64_t per = (int64_t)d.n1 * d.n2 * p->n3h;                                                      \
    fs::xsym3<<<(unsigned)((per + 255) / 256), 256, 0, s>>>(W, d.n1, d.n2, p->n3h, op);                      \
    fs::xinv_long<R3, NB><<<dim3(d.n2 * nch, 3), NB * 16 * R3, sm, s>>>(W, Tt, d.n2, p->n3h, p->tw1, op);    \
    nblk = d.n2 * nch;                                                                                       \
  }
    if (d.n1 == 512) KLONG(2, 16)
    else if (d.n1 == 1024) KLONG(4, 8)
    else KLONG(8, 4)
#undef KLONG
    cudaFreeAsync(W, s);
    return nblk;
  }
  if (p->fast && nc == 3 && !reduce && xb(d.n1, 3) == 0) {
    // x1 lines of 2048: no 3-component tile fits; component-diagonal symbols run
    // one component at a time (the coupled K symbol is rejected by the callers)
    SpecOp o1 = op;
    o1.ncomp = 1;
    const int64_t cstride = (int64_t)d.n1 * d.n2 * p->n3h;   // single-domain layout [c][i][j][kz]
    const size_t esz = f64 ? sizeof(double2) : sizeof(float2);
    int nblk = 0;
    for (int c = 0; c < 3; ++c)
      nblk = spec_xpass(p, o1, false, s, f64, reinterpret_cast<const char*>(Sd) + c * cstride * esz, Tt + c * cstride);
    return nblk;
  }
  if (p->fast && g_fft_mode && d.n1 == 256 && nc == 3 && !reduce) {
    constexpr int LS = 273;
#define XOP4(XB)                                                                                             \
  {                                                                                                          \
    const int nblk = d.n2 * ((p->n3h + XB - 1) / XB);                                                        \
    if (f64) {                                                                                               \
      const size_t sm = sizeof(double2) * 3 * XB * LS;                                                       \
      smem_optin(fs::xop256<double2, XB>, sm);                                                               \
      fs::xop256<double2, XB><<<nblk, 3 * XB * 16, sm, s>>>(Sd, Tt, d.n2, d.n3, p->n3h, p->tw1, op);         \
    } else {                                                                                                 \
      const size_t sm = sizeof(float2) * 3 * XB * LS;                                                        \
      smem_optin(fs::xop256<float2, XB>, sm);                                                                \
      fs::xop256<float2, XB><<<nblk, 3 * XB * 16, sm, s>>>(reinterpret_cast<const float2*>(Sd), Tt, d.n2,    \
                                                           d.n3, p->n3h, p->tw1, op);                        \
    }                                                                                                        \
    return nblk;                                                                                             \
  }
    XOP4(4)   // 4 kz columns x 3 components per CTA (register-limited to 2 CTAs / SM)
#undef XOP4
  }
  if (p->fast) {
    int nblk = 0;
    const float2* S32 = reinterpret_cast<const float2*>(Sd);
#define L_X(LL)                                                                                              \
  {                                                                                                          \
    const int B3 = xb(LL, 3), B1 = xb(LL, 1);                                                                \
    const int B = (nc == 3 && !reduce) ? B3 : B1;                                                            \
    nblk = d.n2 * ((p->n3h + B - 1) / B);                                                                    \
    if (reduce)                                                                                              \
      fast::xop_fast<LL, 1, true, double2><<<nblk, B1 * LL / 8, sm_x(LL, 1, 16), s>>>(                        \
          Sd, Tt, d.n2, d.n3, p->n3h, p->nspec, p->stw1, op, p->partials);                                   \
    else if (nc == 3 && f64)                                                                                 \
      fast::xop_fast<LL, 3, false, double2><<<nblk, 3 * B3 * LL / 8, sm_x(LL, 3, 16), s>>>(                  \
          Sd, Tt, d.n2, d.n3, p->n3h, p->nspec, p->stw1, op, nullptr);                                       \
    else if (nc == 3)                                                                                        \
      fast::xop_fast<LL, 3, false, float2><<<nblk, 3 * B3 * LL / 8, sm_x(LL, 3, 8), s>>>(                    \
          S32, Tt, d.n2, d.n3, p->n3h, p->nspec, p->stw1, op, nullptr);                                      \
    else if (f64)                                                                                            \
      fast::xop_fast<LL, 1, false, double2><<<nblk, B1 * LL / 8, sm_x(LL, 1, 16), s>>>(                      \
          Sd, Tt, d.n2, d.n3, p->n3h, p->nspec, p->stw1, op, nullptr);                                       \
    else                                                                                                     \
      fast::xop_fast<LL, 1, false, float2><<<nblk, B1 * LL / 8, sm_x(LL, 1, 8), s>>>(                        \
          S32, Tt, d.n2, d.n3, p->n3h, p->nspec, p->stw1, op, nullptr);                                      \
  }
    VR_POW2_SWITCH(d.n1, L_X)
#undef L_X
    return nblk;
  }
  const int B = nc == 3 ? p->Bx3 : p->Bx1;
  const size_t sm = nc == 3 ? p->smx3 : p->smx1;
  const int ncx = (p->n3h + B - 1) / B;
  const int nblk = d.n2 * ncx;
  if (reduce)
    x_op_kernel<true><<<nblk, 256, sm, s>>>(Sd, Tt, d, p->n3h, p->rp1, p->tw1, B, op, p->partials);
  else
    x_op_kernel<false><<<nblk, 256, sm, s>>>(Sd, Tt, d, p->n3h, p->rp1, p->tw1, B, op, nullptr);
  return nblk;
}

// ---- A via the separable line engine (spectral_d2.cuh) ------------------------------
static int d2_r2(int L) { return L == 256 ? 16 : (L == 128 ? 8 : 0); }
// CTA size of the line passes: 128 threads capped at 128 registers -> 4 CTAs / SM
// (measured at 256^3: 0.703 ms per A; 3 CTAs / SM at 160 registers 0.818 ms;
// 5 CTAs / SM at 102 registers 0.837 ms; 256-thread CTAs at 2 / SM 0.757 ms)
static int g_d2_threads = 128;

// x1 lines of 512 / 1024 / 2048 take the three-step long_kernel
static int d2_r3(int L) { return L == 512 ? 2 : (L == 1024 ? 4 : (L == 2048 ? 8 : 0)); }

static bool d2_ok(const vr_spec_plan* p) {
  const Dims& d = p->d;
  const int r1 = d2_r2(d.n1) || d2_r3(d.n1), r2 = d2_r2(d.n2), r3 = d2_r2(d.n3);
  return g_a_mode && r1 && r2 && r3 && d.n3 % 64 == 0 && d.n2 % 2 == 0;
}

template <int R2, int NT, bool PEER = false>
static void d2_rows(vr_spec_plan* p, const float* in, float* acc, int ncomp, cudaStream_t s,
                    const d2::D2Peer& pe = d2::D2Peer{}) {
  const Dims& d = p->d;
  constexpr size_t sm = d2::smem_bytes<R2, NT>();
  smem_optin(d2::rows_kernel<R2, NT, PEER>, sm);
  const int npairs = d.n1 * d.n2 / 2, lpb = NT / R2;
  d2::rows_kernel<R2, NT, PEER><<<dim3((npairs + lpb - 1) / lpb, ncomp), NT, sm, s>>>(in, acc, npairs, d.n(),
                                                                                      p->tw3, 1.0 / d.n3, pe);
}

template <int R2, int MODE, int NT>
static void d2_strided(vr_spec_plan* p, int axis, const float* in, float* acc, const float* add, float* out,
                       int ncomp, double alpha, cudaStream_t s, const d2::D2Peer& pe = d2::D2Peer{}) {
  const Dims& d = p->d;
  constexpr size_t sm = d2::smem_bytes<R2, NT>();
  smem_optin(d2::strided_kernel<R2, MODE, NT>, sm);
  const bool ax2 = axis == 2;
  const int L = ax2 ? d.n2 : d.n1;
  const int es = ax2 ? d.n3 : d.n2 * d.n3;
  const int n_outer = ax2 ? d.n1 : d.n2;
  const int outer_stride = ax2 ? d.n2 * d.n3 : d.n3;
  const int nchunks = d.n3 / (2 * (NT / R2));
  d2::strided_kernel<R2, MODE, NT><<<dim3(n_outer * nchunks, ncomp), NT, sm, s>>>(
      in, acc, add, out, d.n3, es, outer_stride, d.n(), ax2 ? p->tw2 : p->tw1, 1.0 / L, alpha, pe);
}

// x1 lines of 512 / 1024 / 2048 (MODE 1: final epilogue, MODE 2: peer store)
template <int MODE>
static void d2_long(vr_spec_plan* p, const float* in, const float* acc, const float* add, float* out, int ncomp,
                    double alpha, cudaStream_t s, const d2::D2Peer& pe = d2::D2Peer{}) {
  const Dims& d = p->d;
#define D2LONG(R3, NB)                                                                                         {                                                                                                              constexpr size_t sm = d2::long_smem_bytes<R3, NB>();                                                         smem_optin(d2::long_kernel<R3, NB, MODE>, sm);                                                               d2::long_kernel<R3, NB, MODE><<<dim3(d.n2 * (d.n3 / (2 * NB)), ncomp), NB * 16 * R3, sm, s>>>(                    in, acc, add, out, d.n3, d.n2 * d.n3, d.n3, d.n(), p->tw1, 1.0 / d.n1, alpha, pe);                     }
  // 256-thread CTAs: the f64 line (16 double2 per thread) needs more than the
  // 128 registers a 512-thread CTA leaves (spills at R3 = 4 / 8 measured in ptxas)
  if (d.n1 == 512) D2LONG(2, 8)
  else if (d.n1 == 1024) D2LONG(4, 4)
  else D2LONG(8, 2)
#undef D2LONG
}

template <int NT>
static void spec_apply_A_d2_nt(vr_spec_plan* p, const float* in, int ncomp, double alpha, const float* add,
                               float* out, float* acc, cudaStream_t s) {
  const Dims& d = p->d;
  if (d.n3 == 256) d2_rows<16, NT>(p, in, acc, ncomp, s); else d2_rows<8, NT>(p, in, acc, ncomp, s);
  if (d.n2 == 256) d2_strided<16, 0, NT>(p, 2, in, acc, nullptr, nullptr, ncomp, 1.0, s);
  else d2_strided<8, 0, NT>(p, 2, in, acc, nullptr, nullptr, ncomp, 1.0, s);
  if (d.n1 == 256) d2_strided<16, 1, NT>(p, 1, in, acc, add, out, ncomp, alpha, s);
  else if (d.n1 == 128) d2_strided<8, 1, NT>(p, 1, in, acc, add, out, ncomp, alpha, s);
  else d2_long<1>(p, in, acc, add, out, ncomp, alpha, s);
}

// out = alpha * (D33 + D22 + D11) in (+ add); the partial sums live in p->T
static int spec_apply_A_d2(vr_spec_plan* p, const float* in, int ncomp, double alpha, const float* add, float* out,
                           cudaStream_t s) {
  float* acc = reinterpret_cast<float*>(p->T);   // 3 * nspec float2 >= 3 * N floats
  if (g_d2_threads == 256) spec_apply_A_d2_nt<256>(p, in, ncomp, alpha, add, out, acc, s);
  else spec_apply_A_d2_nt<128>(p, in, ncomp, alpha, add, out, acc, s);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

extern "C" {

// kernel launches one vr_spec_apply(p, kind, ., ncomp, ...) makes (bench accounting)
int vr_spec_apply_launches(const vr_spec_plan* p, int kind, int ncomp) {
  if (!p) return 0;
  if (kind == VR_SPEC_A && d2_ok(p)) return 3;
  if (kind == VR_SPEC_K && p->fast && g_fft_mode && g_xdiag &&
      (p->d.n1 == 512 || p->d.n1 == 1024 || p->d.n1 == 2048))
    return 7;   // z, y, xfwd_long, xsym3, xinv_long, y', z
  const bool x3split = p->fast && ncomp == 3 && xb(p->d.n1, 3) == 0 && !(g_fft_mode && p->d.n1 == 256);
  const int per = 5 + (x3split ? 2 : 0);
  if (ncomp == 3 && kind != VR_SPEC_K && g_percomp) return 15;
  return per;
}

int vr_set_spectral_tuning(int key, int value) {
  // key 1: per-component scheduling of diagonal symbols (1 = on, 0 = all components per pass)
  // key 2: paired-row four-step x3 passes for 256-point rows (1 = on, 0 = Stockham)
  // key 4: x1 pass (xdiag256) over the flat (x2, kz) plane (1) or 16 kz of one x2 row per CTA (0)
  if (key == 4) {
    const int prev = g_xflat;
    g_xflat = value;
    return prev;
  }
  if (key == 2) {
    const int prev = g_zpair;
    g_zpair = value;
    return prev;
  }
  if (key == 1) {
    const int prev = g_percomp;
    g_percomp = value;
    return prev;
  }
  return VR_ERR_ARG;
}

int vr_set_spec_a_mode(int mode) {
  // 0: 3-D f64 path; 1: separable engine (128-thread CTAs); 2: separable, 256-thread CTAs
  const int prev = g_a_mode == 0 ? 0 : (g_d2_threads == 256 ? 2 : 1);
  g_a_mode = mode != 0;
  g_d2_threads = mode == 2 ? 256 : 128;
  return prev;
}

// out = alpha * IFFT(symbol * FFT(in)) [+ add], component-wise or coupled (K).
// alpha is folded into the f64 symbol (e.g. beta_v * A v + body in one call).
int vr_spec_apply(vr_spec_plan* p, int kind, const float* in, int ncomp, double beta_v, double beta_w,
                  double shift, double sigma, double alpha, const float* add, float* out, void* stream) {
  if (!p || !in || !out || (ncomp != 1 && ncomp != 3)) return VR_ERR_ARG;
  if (kind == VR_SPEC_K && ncomp != 3) return VR_ERR_ARG;
  if (kind == VR_SPEC_K && p->fast && xb(p->d.n1, 3) == 0 && !(g_fft_mode && g_xdiag && p->d.n1 == 2048))
    return VR_ERR_UNSUPPORTED;   // N1 > 2048 (2048: the long-line K passes)
  if (kind == VR_SPEC_K && !p->fast && p->smx3 > kSmemBudget) return VR_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  const Dims& d = p->d;
  const bool sep = kind == VR_SPEC_A && d2_ok(p);
  if (int rc = ensure_scratch(p, !sep, true)) return rc;
  if (sep) return spec_apply_A_d2(p, in, ncomp, alpha, add, out, s);
  const bool f64 = needs_f64(kind);
  if (ncomp == 3 && kind != VR_SPEC_K && g_percomp) {
    // component-diagonal symbol: run the five passes one component at a time
    // on the same spectrum buffer, so a component's half spectrum (67.6 MB in
    // f32 at 256^3) is still in L2 when the next pass reads it
    const int64_t n = d.n();
    SpecOp op{kind, 1, beta_v, beta_w, shift, alpha / (double)n, sigma, 0, d.n2, d.n1};
    for (int c = 0; c < 3; ++c) {
      int rc = spec_forward(p, in + c * n, 1, s, f64);
      if (rc) return rc;
      spec_xpass(p, op, false, s, f64);
      spec_inverse_yz(p, 1, add ? add + c * n : nullptr, out + c * n, s);
    }
    VR_CHECK_LAUNCH();
    return VR_OK;
  }
  int rc = spec_forward(p, in, ncomp, s, f64);
  if (rc) return rc;
  SpecOp op{kind, ncomp, beta_v, beta_w, shift, alpha / (double)d.n(), sigma, 0, d.n2, d.n1};
  spec_xpass(p, op, false, s, f64);
  spec_inverse_yz(p, ncomp, add, out, s);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// prolong_spectral (grid.py:181-226): coarse rfftn -> Nyquist-split zero pad ->
// fine irfftn, all on the device; `in` lives on pc's grid, `out` on pf's.
int vr_prolong_spectral(vr_spec_plan* pc, vr_spec_plan* pf, const float* in, int ncomp, float* out,
                        void* stream) {
  if (!pc || !pf || !in || !out || (ncomp != 1 && ncomp != 3)) return VR_ERR_ARG;
  if (pf->d.n1 < pc->d.n1 || pf->d.n2 < pc->d.n2 || pf->d.n3 < pc->d.n3) return VR_ERR_DIMS;
  if (pc->d.n1 % 2 || pc->d.n2 % 2 || pc->d.n3 % 2) return VR_ERR_DIMS;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = ensure_scratch(pc);
  if (!rc) rc = ensure_scratch(pf);
  if (!rc) rc = spec_forward(pc, in, ncomp, s);
  if (rc) return rc;
  launch_axis<double2>(pc, pc->S, 1, ncomp, 0, s);
  const int64_t n = pf->nspec * ncomp;
  pad_kernel<<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(pc->S, pc->d, pc->n3h, pf->T, pf->d, pf->n3h, ncomp,
                                                          1.0 / (double)pc->d.n());
  launch_axis<float2>(pf, pf->T, 1, ncomp, 1, s);
  spec_inverse_yz(pf, ncomp, nullptr, out, s);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// (2 pi)^3 * sum mult (1+|k|^2) |F/N|^2  -> *out_dev (device f64)
int vr_h1_energy(vr_spec_plan* p, const float* f, double* out_dev, void* stream) {
  if (!p || !f || !out_dev) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const Dims& d = p->d;
  int rc = ensure_scratch(p);
  if (!rc) rc = spec_forward(p, f, 1, s);
  if (rc) return rc;
  SpecOp op{VR_SPEC_IDENTITY, 1, 0, 0, 0, 1.0, 0, 0, d.n2, d.n1};
  const int nblk = spec_xpass(p, op, true, s);
  const double n = (double)d.n();
  finalize_sum_kernel<<<1, 1024, 0, s>>>(p->partials, nblk, kTwoPi * kTwoPi * kTwoPi / (n * n), out_dev);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_spec_plan_dims(const vr_spec_plan* p, int64_t dims_out[3]) {
  if (!p || !dims_out) return VR_ERR_ARG;
  dims_out[0] = p->d.n1;
  dims_out[1] = p->d.n2;
  dims_out[2] = p->d.n3;
  return VR_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------
// Distributed (x1-slab) spectral operators.  A rank owns x1 planes [r L1, (r+1) L1)
// of the real fields.  Forward: x3 and x2 passes on the local slab, then the
// half spectrum is packed per destination rank q (x2 block [q L2, (q+1) L2)) so
// that ONE all-to-all per component (torch.distributed / NCCL, issued by the
// host) delivers complete x1 lines: recv[c][x1 = p L1 + i][jl][kz].  The X pass
// (forward, symbol, inverse) runs on that transposed block with the x2
// wavenumber offset j0 = r L2; its output is already contiguous per destination
// for the inverse all-to-all; the receiver unpacks and runs the x2 / x3 inverse
// passes.  Requires the power-of-two fast path on both plans.
// ---------------------------------------------------------------------------------
namespace vr {

// Rank-blocked transpose layout [q][c][i][jl][kz] <-> slab layout [c][i][j][kz]
// (j = q * L2 + jl).  One warp moves one contiguous kz row: a single 32-bit
// index decomposition per row instead of 64-bit divisions per element.
template <typename C, bool PACK>
__global__ void __launch_bounds__(256) rowmove_kernel(const C* __restrict__ src, C* __restrict__ dst, int ncomp,
                                                      int L1, int N2, int n3h, int P) {
  const int L2 = N2 / P;
  const int rows = ncomp * L1 * N2;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int j = row % N2, ci = row / N2;   // slab row (c, i, j)
  const int i = ci % L1, c = ci / L1;
  const int q = j / L2, jl = j - q * L2;
  const int64_t slab = (int64_t)row * n3h;
  const int64_t blk = ((((int64_t)q * ncomp + c) * L1 + i) * L2 + jl) * n3h;
  const C* a = src + (PACK ? slab : blk);
  C* b = dst + (PACK ? blk : slab);
  for (int kz = lane; kz < n3h; kz += 32) b[kz] = a[kz];
}

}  // namespace vr

extern "C" {

// Z + Y forward passes of `in` (local slab, ncomp components) and pack into
// sendbuf ([q][c][i][jl][kz], complex128 if f64 else complex64).
int vr_dspec_forward(vr_spec_plan* pl, const float* in, int ncomp, int f64, int nranks, void* sendbuf, void* stream) {
  if (!pl || !in || !sendbuf || nranks < 1 || (ncomp != 1 && ncomp != 3)) return VR_ERR_ARG;
  if (pl->d.n2 % nranks) return VR_ERR_UNSUPPORTED;
  // the generic mixed-radix path (non-power-of-two sizes, e.g. the CLARITY
  // shape 2816 x 3016 x 1162) always forward-transforms in f64
  if (!pl->fast) f64 = 1;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = ensure_scratch(pl);
  if (!rc) rc = spec_forward(pl, in, ncomp, s, f64 != 0);
  if (rc) return rc;
  const int64_t n = pl->nspec * ncomp;
  const unsigned g = (unsigned)((ncomp * pl->d.n1 * pl->d.n2 + 7) / 8);
  (void)n;
  if (f64)
    rowmove_kernel<double2, true><<<g, 256, 0, s>>>(pl->S, reinterpret_cast<double2*>(sendbuf), ncomp, pl->d.n1,
                                                    pl->d.n2, pl->n3h, nranks);
  else
    rowmove_kernel<float2, true><<<g, 256, 0, s>>>(reinterpret_cast<const float2*>(pl->S),
                                                   reinterpret_cast<float2*>(sendbuf), ncomp, pl->d.n1, pl->d.n2,
                                                   pl->n3h, nranks);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// X pass on the transposed block (px dims = {N1, L2, N3}); recv / xout are
// [p][c][il][jl][kz] (x1 = p*L1 + il: what one all-to-all delivers / sends);
// n_global = N1*N2*N3 for the inverse normalisation.
int vr_dspec_xpass(vr_spec_plan* px, int kind, int ncomp, int f64, double beta_v, double beta_w, double shift,
                   double sigma, double alpha, int64_t n_global, int j0, int n2_global, int l1, const void* recv,
                   void* xout, void* stream) {
  if (!px || !recv || !xout || (ncomp != 1 && ncomp != 3) || l1 < 1 || px->d.n1 % l1) return VR_ERR_ARG;
  if (kind == VR_SPEC_K && ncomp != 3) return VR_ERR_ARG;
  if (px->fast && ncomp == 3 && xb(px->d.n1, 3) == 0 && !(g_fft_mode && g_xdiag && px->d.n1 == 2048))
    return VR_ERR_UNSUPPORTED;   // N1 > 2048: 3-component tiles do not fit
  if (!px->fast && ncomp == 3 && px->smx3 > kSmemBudget) return VR_ERR_UNSUPPORTED;
  if (!px->fast) f64 = 1;   // generic path: f64 forward (see vr_dspec_forward)
  if (!px->fast)
    if (int rc = ensure_scratch(px)) return rc;
  SpecOp op{kind, ncomp, beta_v, beta_w, shift, alpha / (double)n_global, sigma, j0, n2_global, l1};
  spec_xpass(px, op, false, (cudaStream_t)stream, f64 != 0, recv, reinterpret_cast<float2*>(xout));
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// H1 partial sum over this rank's transposed block -> *out_dev = scale * sum
int vr_dspec_h1_partial(vr_spec_plan* px, const void* recv, int j0, int n2_global, int l1, double scale,
                        double* out_dev, void* stream) {
  if (!px || !recv || !out_dev || l1 < 1 || px->d.n1 % l1) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (!px->fast)
    if (int rc = ensure_scratch(px)) return rc;
  SpecOp op{VR_SPEC_IDENTITY, 1, 0, 0, 0, 1.0, 0, j0, n2_global, l1};
  const int nblk = spec_xpass(px, op, true, s, true, recv, nullptr);
  finalize_sum_kernel<<<1, 1024, 0, s>>>(px->partials, nblk, scale, out_dev);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// unpack the inverse all-to-all result ([c][q][i][jl][kz], complex64) and run the
// Y / Z inverse passes into `out` (+ add) on the local slab
int vr_dspec_inverse(vr_spec_plan* pl, const void* recv_inv, int ncomp, int nranks, const float* add, float* out,
                     void* stream) {
  if (!pl || !recv_inv || !out || (ncomp != 1 && ncomp != 3)) return VR_ERR_ARG;
  if (pl->d.n2 % nranks) return VR_ERR_UNSUPPORTED;
  if (int rc = ensure_scratch(pl)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = pl->nspec * ncomp;
  (void)n;
  rowmove_kernel<float2, false><<<(unsigned)((ncomp * pl->d.n1 * pl->d.n2 + 7) / 8), 256, 0, s>>>(
      reinterpret_cast<const float2*>(recv_inv), pl->T, ncomp, pl->d.n1, pl->d.n2, pl->n3h, nranks);
  spec_inverse_yz(pl, ncomp, add, out, s);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// ---- peer variants: the transposes fused into the x2 / x1 passes (NVLink stores) ----
static bool peer_ok(const vr_spec_plan* pl, int nranks) {
  return pl && pl->fast && g_fft_mode && pl->d.n2 == 256 && nranks >= 1 && nranks <= 8 &&
         (nranks & (nranks - 1)) == 0;
}

static int log2i(int x) {
  int s = 0;
  while ((1 << s) < x) ++s;
  return s;
}

// Z + Y forward of `in`; the Y pass stores row j straight into rank j / L2's
// receive buffer dst[j / L2] (host array of device pointers) at block `me`.
int vr_dspec_forward_peer(vr_spec_plan* pl, const float* in, int ncomp, int f64, int nranks, int me,
                          void* const* dst, void* stream) {
  if (!in || !dst || (ncomp != 1 && ncomp != 3) || me < 0 || me >= nranks) return VR_ERR_ARG;
  if (!peer_ok(pl, nranks)) return VR_ERR_UNSUPPORTED;
  if (int rc = ensure_scratch(pl)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  spec_forward_z(pl, in, ncomp, s, f64 != 0);
  fs::X2Peer pe{};
  for (int r = 0; r < nranks; ++r) pe.dst[r] = dst[r];
  pe.me = me;
  pe.l2shift = log2i(nranks);
  pe.ncomp = ncomp;
  const int nchunks = (pl->n3h + 15) / 16;
  const dim3 g(pl->d.n1 * nchunks, ncomp);
  if (f64) {
    const size_t sm = sizeof(double2) * 16 * fs::line_smem<16>();
    smem_optin(fs::axis256_dist<double2, false>, sm);
    fs::axis256_dist<double2, false><<<g, 256, sm, s>>>(pl->S, nullptr, pe, pl->d.n1, pl->n3h, pl->tw2);
  } else {
    const size_t sm = sizeof(float2) * 16 * fs::line_smem<16>();
    smem_optin(fs::axis256_dist<float2, false>, sm);
    fs::axis256_dist<float2, false><<<g, 256, sm, s>>>(reinterpret_cast<const float2*>(pl->S), nullptr, pe,
                                                       pl->d.n1, pl->n3h, pl->tw2);
  }
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// X pass on the transposed block with its output stored straight into rank
// p's inverse receive buffer dst[p] (block `me`); arguments as vr_dspec_xpass.
int vr_dspec_xpass_peer(vr_spec_plan* px, int kind, int ncomp, int f64, double beta_v, double beta_w, double shift,
                        double sigma, double alpha, int64_t n_global, int j0, int n2_global, int l1, const void* recv,
                        int nranks, int me, void* const* dst, void* stream) {
  if (!px || !recv || !dst || (ncomp != 1 && ncomp != 3) || l1 < 1 || px->d.n1 % l1) return VR_ERR_ARG;
  if (nranks < 1 || nranks > 8 || me < 0 || me >= nranks || px->d.n1 / l1 != nranks) return VR_ERR_ARG;
  if (kind == VR_SPEC_K && ncomp != 3) return VR_ERR_ARG;
  if (!px->fast) return VR_ERR_UNSUPPORTED;
  if (ncomp == 3 && xb(px->d.n1, 3) == 0 && !(g_fft_mode && g_xdiag && px->d.n1 == 2048)) return VR_ERR_UNSUPPORTED;
  SpecOp op{kind, ncomp, beta_v, beta_w, shift, alpha / (double)n_global, sigma, j0, n2_global, l1};
  for (int p = 0; p < nranks; ++p) op.pdst[p] = dst[p];
  op.me = me;
  spec_xpass(px, op, false, (cudaStream_t)stream, f64 != 0, recv, nullptr);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// inverse: Y inverse reading the blocked receive buffer (unpack fused), Z inverse -> out (+ add)
int vr_dspec_inverse_peer(vr_spec_plan* pl, const void* recv_inv, int ncomp, int nranks, const float* add,
                          float* out, void* stream) {
  if (!recv_inv || !out || (ncomp != 1 && ncomp != 3)) return VR_ERR_ARG;
  if (!peer_ok(pl, nranks)) return VR_ERR_UNSUPPORTED;
  if (int rc = ensure_scratch(pl)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  fs::X2Peer pe{};
  pe.l2shift = log2i(nranks);
  pe.ncomp = ncomp;
  const int nchunks = (pl->n3h + 15) / 16;
  const size_t sm = sizeof(float2) * 16 * fs::line_smem<16>();
  smem_optin(fs::axis256_dist<float2, true>, sm);
  fs::axis256_dist<float2, true><<<dim3(pl->d.n1 * nchunks, ncomp), 256, sm, s>>>(
      reinterpret_cast<const float2*>(recv_inv), pl->T, pe, pl->d.n1, pl->n3h, pl->tw2);
  spec_inverse_z(pl, ncomp, add, out, s);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// ---- A on x1 slabs through the separable engine ---------------------------------
// pl: the slab plan {L1, N2, N3}; px: the block plan {N1, L2, N3}, L2 = N2 / P.
// blk[q] / back[q]: rank q's block buffer [c][N1][L2][N3] and back buffer
// [c][L1][N2][N3] (f32, symmetric).  The partial sums live in pl's T.
static bool dsep_ok(const vr_spec_plan* pl, const vr_spec_plan* px, int nranks) {
  if (!pl || !px || nranks < 1 || nranks > 8 || !g_a_mode) return false;
  const Dims &a = pl->d, &b = px->d;
  const int L2 = b.n2;
  return d2_r2(a.n3) && d2_r2(a.n2) && (d2_r2(b.n1) || d2_r3(b.n1)) && a.n3 % 64 == 0 && b.n3 == a.n3 &&
         L2 * nranks == a.n2 && L2 % 2 == 0 && a.n1 * nranks == b.n1;
}

static d2::D2Peer dsep_peer(const vr_spec_plan* pl, const vr_spec_plan* px, int nranks, int me, void* const* dst) {
  d2::D2Peer pe{};
  for (int q = 0; q < nranks; ++q) pe.dst[q] = dst[q];
  pe.me = me;
  pe.l1 = pl->d.n1;
  pe.l2 = px->d.n2;
  pe.n1 = px->d.n1;
  pe.n2 = pl->d.n2;
  return pe;
}

int vr_dspec_a_ok(const vr_spec_plan* pl, const vr_spec_plan* px, int nranks) {
  return dsep_ok(pl, px, nranks) ? 1 : 0;
}

// acc = D33 in on the slab; every slab row also goes to blk[j / L2]
int vr_dspec_a_rows(vr_spec_plan* pl, vr_spec_plan* px, const float* in, int ncomp, int nranks, int me,
                    void* const* blk, void* stream) {
  if (!in || !blk || (ncomp != 1 && ncomp != 3) || me < 0 || me >= nranks) return VR_ERR_ARG;
  if (!dsep_ok(pl, px, nranks)) return VR_ERR_UNSUPPORTED;
  if (int rc = ensure_scratch(pl, false, true)) return rc;
  const d2::D2Peer pe = dsep_peer(pl, px, nranks, me, blk);
  float* acc = reinterpret_cast<float*>(pl->T);
  cudaStream_t s = (cudaStream_t)stream;
  if (pl->d.n3 == 256) d2_rows<16, 128, true>(pl, in, acc, ncomp, s, pe);
  else d2_rows<8, 128, true>(pl, in, acc, ncomp, s, pe);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// acc += D22 in (local x2 lines)
int vr_dspec_a_x2(vr_spec_plan* pl, const float* in, int ncomp, void* stream) {
  if (!pl || !in || (ncomp != 1 && ncomp != 3) || !pl->T || !d2_r2(pl->d.n2)) return VR_ERR_ARG;
  float* acc = reinterpret_cast<float*>(pl->T);
  cudaStream_t s = (cudaStream_t)stream;
  if (pl->d.n2 == 256) d2_strided<16, 0, 128>(pl, 2, in, acc, nullptr, nullptr, ncomp, 1.0, s);
  else d2_strided<8, 0, 128>(pl, 2, in, acc, nullptr, nullptr, ncomp, 1.0, s);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// out = alpha ((acc + D22 in) + back) (+ add): the x2 pass and the final in
// one kernel (after the x1 exchange), instead of vr_dspec_a_x2 + vr_dspec_a_final
int vr_dspec_a_x2_final(vr_spec_plan* pl, const float* in, const float* back_local, int ncomp, double alpha,
                        const float* add, float* out, void* stream) {
  if (!pl || !in || !back_local || !out || (ncomp != 1 && ncomp != 3) || !pl->T || !d2_r2(pl->d.n2))
    return VR_ERR_ARG;
  float* acc = reinterpret_cast<float*>(pl->T);
  cudaStream_t s = (cudaStream_t)stream;
  d2::D2Peer pe{};
  pe.back = back_local;
  if (pl->d.n2 == 256) d2_strided<16, 3, 128>(pl, 2, in, acc, add, out, ncomp, alpha, s, pe);
  else d2_strided<8, 3, 128>(pl, 2, in, acc, add, out, ncomp, alpha, s, pe);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// D11 of the received block's x1 lines -> back[i / L1]
int vr_dspec_a_x1_peer(vr_spec_plan* pl, vr_spec_plan* px, const float* blk_local, int ncomp, int nranks, int me,
                       void* const* back, void* stream) {
  if (!blk_local || !back || (ncomp != 1 && ncomp != 3) || me < 0 || me >= nranks) return VR_ERR_ARG;
  if (!dsep_ok(pl, px, nranks)) return VR_ERR_UNSUPPORTED;
  const d2::D2Peer pe = dsep_peer(pl, px, nranks, me, back);
  cudaStream_t s = (cudaStream_t)stream;
  const int n1 = px->d.n1;
  if (n1 == 256) d2_strided<16, 2, 128>(px, 1, blk_local, nullptr, nullptr, nullptr, ncomp, 1.0, s, pe);
  else if (n1 == 128) d2_strided<8, 2, 128>(px, 1, blk_local, nullptr, nullptr, nullptr, ncomp, 1.0, s, pe);
  else d2_long<2>(px, blk_local, nullptr, nullptr, nullptr, ncomp, 1.0, s, pe);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// out = alpha (acc + back) (+ add) on the slab
int vr_dspec_a_final(vr_spec_plan* pl, const float* back_local, int ncomp, double alpha, const float* add,
                     float* out, void* stream) {
  if (!pl || !back_local || !out || (ncomp != 1 && ncomp != 3) || !pl->T) return VR_ERR_ARG;
  const int64_t n4 = (int64_t)ncomp * pl->d.n() / 4;
  d2::final_kernel<<<grid_for(n4, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(pl->T), reinterpret_cast<const float4*>(back_local),
      reinterpret_cast<const float4*>(add), reinterpret_cast<float4*>(out), n4, alpha);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_spec_plan_is_fast(const vr_spec_plan* p) { return p && p->fast ? 1 : 0; }

}  // extern "C"
