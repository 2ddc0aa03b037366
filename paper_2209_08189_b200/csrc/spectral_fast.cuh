// Fast path of the spectral engine for power-of-two line lengths (8..4096).
//
// Line FFT: compile-time in-place Stockham DIT with radix 8 (and one final
// radix 2/4).  Every lane owns exactly 8 elements per stage, so a line of
// length L is processed by LP = L/8 lanes: several lines per warp for L < 256,
// one warp for L = 256, a named-barrier group of L/256 warps above.  Stages
// synchronise only the lanes of a line (__syncwarp / bar.sync id, LP), never
// the CTA.  Shared memory is padded (one slot per 8) to break the power-of-two
// bank strides of the Stockham writes.
//
// The x3 (contiguous, real) axis uses the half-length packing trick: a real
// row of 2M samples is FFT'd as M complex samples z[m] = x[2m] + i x[2m+1] and
// post-processed (forward) / pre-processed (inverse) into the n3/2+1 Hermitian
// half spectrum, halving both the arithmetic and the shared-memory footprint.
#pragma once

namespace vr {
namespace fast {

__device__ __forceinline__ int padi(int i) { return i + (i >> 3); }
// odd line stride: consecutive lines land in different shared-memory banks
template <int L> __host__ __device__ constexpr int padlen() { return L + L / 8 + 1; }

template <typename C> struct Real;
template <> struct Real<double2> { using T = double; };
template <> struct Real<float2> { using T = float; };

template <typename C> __device__ __forceinline__ C mk(double x, double y) {
  C r;
  r.x = (typename Real<C>::T)x;
  r.y = (typename Real<C>::T)y;
  return r;
}

template <int L>
__device__ __forceinline__ void gsync(int gid) {
  constexpr int LP = L / 8;
  if constexpr (LP <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(gid + 1), "r"(LP) : "memory");
  }
}

template <typename C, int R>
__device__ __forceinline__ void dft(C* v, bool inv) {
  if constexpr (R == 2) {
    C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    dft4(v[0], v[1], v[2], v[3], inv);
  } else {
    C e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    C o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4(e0, e1, e2, e3, inv);
    dft4(o0, o1, o2, o3, inv);
    const double s = 0.70710678118654752440;
    const C w1 = mk<C>(s, inv ? s : -s), w3 = mk<C>(-s, inv ? s : -s);
    o1 = cmul(o1, w1);
    o2 = rot(o2, inv);
    o3 = cmul(o3, w3);
    v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
    v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
    v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
    v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
  }
}

// one in-place Stockham stage; twiddle powers W^{r k} by recurrence from W^k
// (one table read per butterfly instead of R-1 bank-conflicting ones)
template <typename C, int L, int R, int NS, bool INV>
__device__ __forceinline__ void stage(C* line, int lane, const double2* tw, int gid) {
  constexpr int LP = L / 8, NB = L / R, PER = 8 / R;
  C v[8];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = lane + q * LP;
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = line[padi(j + r * NB)];
  }
  gsync<L>(gid);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = lane + q * LP;
    const int k = j & (NS - 1);
    C* u = v + q * R;
    if constexpr (NS > 1) {
      const C w1 = twid<C>(tw, NS + k, INV);   // per-stage table: tw[NS + k] = W_{NS R}^k
      C w = w1;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        u[r] = cmul(u[r], w);
        if (r + 1 < R) w = cmul(w, w1);
      }
    }
    dft<C, R>(u, INV);
    const int idxD = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) line[padi(idxD + r * NS)] = u[r];
  }
  gsync<L>(gid);
}

template <typename C, int L, int NS, bool INV>
__device__ __forceinline__ void stages(C* line, int lane, const double2* tw, int gid) {
  if constexpr (NS < L) {
    constexpr int REM = L / NS;
    constexpr int R = REM >= 8 ? 8 : REM;
    stage<C, L, R, NS, INV>(line, lane, tw, gid);
    stages<C, L, NS * R, INV>(line, lane, tw, gid);
  }
}

// thread -> (line, lane); every thread of the CTA takes part (nlines * L/8 == blockDim)
template <typename C, int L, bool INV>
__device__ __forceinline__ void fft_tile(C* tile, const double2* tw) {
  constexpr int LP = L / 8;
  const int line = threadIdx.x / LP, lane = threadIdx.x % LP;
  const int gid = threadIdx.x / (LP > 32 ? LP : 32);
  stages<C, L, 1, INV>(tile + line * padlen<L>(), lane, tw, gid);
}

template <typename C, typename D> __device__ __forceinline__ C convert(D a) { return mk<C>(a.x, a.y); }

// ---- Z forward: real rows (2M) -> half spectrum (M+1) in precision CF ----------------
// block = 256 threads, 2048/M rows per CTA (8 input float2 per thread). grid (rows/LINES, ncomp)
template <int M, typename CF>
__global__ void __launch_bounds__(256, 3) zfwd_fast(const float* __restrict__ in, int nrows, int64_t nvox,
                                                 int64_t nspec, const double2* __restrict__ twM,
                                                 const double2* __restrict__ twL, CF* __restrict__ S) {
  constexpr int LINES = 2048 / M, PL = padlen<M>();
  extern __shared__ double2 smd[];
  double2* tw_s = smd;             // M entries
  double2* twl_s = tw_s + 2 * M;   // M+1 entries of W_{2M}^k
  CF* tile = reinterpret_cast<CF*>(twl_s + M + 1);   // LINES x PL
  for (int t = threadIdx.x; t < 2 * M; t += 256) tw_s[t] = twM[t];
  for (int t = threadIdx.x; t <= M; t += 256) twl_s[t] = twL[t];
  const int row0 = blockIdx.x * LINES;
  const int nr = min(LINES, nrows - row0);
  const float2* src = reinterpret_cast<const float2*>(in + (int64_t)blockIdx.y * nvox) + (int64_t)row0 * M;
  float2 x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * 256;
    x[u] = (e < nr * M) ? __ldg(src + e) : make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * 256;
    const int r = e / M, m = e - r * M;
    tile[r * PL + padi(m)] = mk<CF>(x[u].x, x[u].y);
  }
  __syncthreads();
  fft_tile<CF, M, false>(tile, tw_s);
  __syncthreads();
  CF* dst = S + blockIdx.y * nspec + (int64_t)row0 * (M + 1);
  using R = typename Real<CF>::T;
  for (int e = threadIdx.x; e < nr * (M + 1); e += 256) {
    const int r = e / (M + 1), k = e - r * (M + 1);
    const CF* line = tile + r * PL;
    const CF zk = line[padi(k & (M - 1))];
    const CF zm = line[padi((M - k) & (M - 1))];
    // E = (Z[k] + conj Z[M-k]) / 2 ;  O = (Z[k] - conj Z[M-k]) / (2i)
    CF E, O;
    E.x = R(0.5) * (zk.x + zm.x);
    E.y = R(0.5) * (zk.y - zm.y);
    O.x = R(0.5) * (zk.y + zm.y);
    O.y = R(-0.5) * (zk.x - zm.x);
    dst[e] = cadd(E, cmul(convert<CF>(twl_s[k]), O));
  }
}

// ---- Z inverse: half spectrum (M+1, f32) -> real rows (2M), out = x (+ add) -------
template <int M>
__global__ void __launch_bounds__(256) zinv_fast(const float2* __restrict__ T, int nrows, int64_t nvox,
                                                 int64_t nspec, const double2* __restrict__ twM,
                                                 const double2* __restrict__ twL, float* __restrict__ out,
                                                 const float* __restrict__ add) {
  constexpr int LINES = 2048 / M, PL = padlen<M>();
  extern __shared__ double2 smd[];
  double2* tw_s = smd;
  float2* tile = reinterpret_cast<float2*>(tw_s + 2 * M);
  for (int t = threadIdx.x; t < 2 * M; t += 256) tw_s[t] = twM[t];
  const int row0 = blockIdx.x * LINES;
  const int nr = min(LINES, nrows - row0);
  const float2* src = T + blockIdx.y * nspec + (int64_t)row0 * (M + 1);
  float2 xk[8], xm[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * 256;
    const int r = e / M, k = e - r * M;
    const bool ok = e < nr * M;
    xk[u] = ok ? src[r * (M + 1) + k] : make_float2(0.f, 0.f);
    xm[u] = ok ? src[r * (M + 1) + M - k] : make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * 256;
    const int r = e / M, k = e - r * M;
    float2 a = xk[u], b = xm[u];
    if (k == 0) { a.y = 0.f; b.y = 0.f; }   // c2r drops imag of DC and Nyquist
    // E2 = X[k] + conj X[M-k];  O2 = (X[k] - conj X[M-k]) * conj(W_2M^k);  Z = E2 + i O2
    const double2 wd = twL[k];
    const float2 wc = make_float2((float)wd.x, (float)-wd.y);
    const float2 E = make_float2(a.x + b.x, a.y - b.y);
    const float2 O = cmul(make_float2(a.x - b.x, a.y + b.y), wc);
    tile[r * PL + padi(k)] = make_float2(E.x - O.y, E.y + O.x);
  }
  __syncthreads();
  fft_tile<float2, M, true>(tile, tw_s);
  __syncthreads();
  const int64_t off = blockIdx.y * nvox + (int64_t)row0 * 2 * M;
  float2* dst = reinterpret_cast<float2*>(out + off);
  const float2* ad = add ? reinterpret_cast<const float2*>(add + off) : nullptr;
  float2 a[8];
  if (ad) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = threadIdx.x + u * 256;
      a[u] = (e < nr * M) ? __ldg(ad + e) : make_float2(0.f, 0.f);
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * 256;
    if (e < nr * M) {
      const int r = e / M, m = e - r * M;
      float2 z = tile[r * PL + padi(m)];
      if (ad) {
        z.x += a[u].x;
        z.y += a[u].y;
      }
      dst[e] = z;
    }
  }
}

// ---- strided axis pass (x2, or plain x1): B = 2048/L columns of length L per CTA --------
// 256 threads, 8 elements per thread each way.  grid (n_outer*nchunks, ncomp)
template <typename C, int L, bool INV>
__global__ void __launch_bounds__(256, 3) axis_fast(C* __restrict__ S, int64_t es, int n_outer,
                                                 int64_t outer_stride, int64_t comp_stride, int n3h,
                                                 const double2* __restrict__ tw) {
  constexpr int PL = padlen<L>(), B = 2048 / L;
  extern __shared__ double2 smd[];
  double2* tw_s = smd;
  C* tile = reinterpret_cast<C*>(tw_s + 2 * L);
  for (int t = threadIdx.x; t < 2 * L; t += 256) tw_s[t] = tw[t];
  const int nchunks = (n3h + B - 1) / B;
  const int o = blockIdx.x / nchunks, kz0 = (blockIdx.x - o * nchunks) * B;
  const int nb = min(B, n3h - kz0);
  C* base = S + blockIdx.y * comp_stride + o * outer_stride + kz0;
  C x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * 256;
    const int j = e / B, q = e - j * B;
    x[u] = (q < nb) ? base[j * es + q] : mk<C>(0.0, 0.0);
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * 256;
    const int j = e / B, q = e - j * B;
    tile[q * PL + padi(j)] = x[u];
  }
  __syncthreads();
  fft_tile<C, L, INV>(tile, tw_s);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * 256;
    const int j = e / B, q = e - j * B;
    if (q < nb) base[j * es + q] = tile[q * PL + padi(j)];
  }
}

// ---- X pass: fwd -> symbol (f64) -> inv -> c64 store; or the H1 reduction -----
// precision CF for the line FFTs; lines = NC*B with B = 1024/L (NC = 3) or 2048/L (NC = 1);
// threads = NC*B*L/8 (8 elements per thread each way)
template <int L, int NC, bool REDUCE, typename CF>
__global__ void __launch_bounds__(NC == 3 ? 384 : 256, NC == 3 ? 2 : 3) xop_fast(const CF* __restrict__ S, float2* __restrict__ T, int n2,
                                                     int n3, int n3h, int64_t nspec,
                                                     const double2* __restrict__ tw, SpecOp op,
                                                     double* __restrict__ partials) {
  constexpr int PL = padlen<L>(), B = (NC == 3 ? 1024 : 2048) / L, NT = NC * B * L / 8;
  extern __shared__ double2 smd[];
  double2* tw_s = smd;
  CF* tile = reinterpret_cast<CF*>(tw_s + 2 * L);
  for (int t = threadIdx.x; t < 2 * L; t += NT) tw_s[t] = tw[t];
  const int nchunks = (n3h + B - 1) / B;
  const int j = blockIdx.x / nchunks, kz0 = (blockIdx.x - j * nchunks) * B;
  const int nb = min(B, n3h - kz0);
  const int64_t lstride = (int64_t)n2 * n3h;
  const CF* sbase = S + (int64_t)j * n3h + kz0;
  CF x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * NT;       // e = (c*L + i)*B + q
    const int q = e % B, ci = e / B;
    const int c = ci / L, i = ci - c * L;
    x[u] = (q < nb) ? sbase[op.xoff(c, i, lstride) + q] : mk<CF>(0.0, 0.0);
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * NT;
    const int q = e % B, ci = e / B;
    const int c = ci / L, i = ci - c * L;
    tile[(c * B + q) * PL + padi(i)] = x[u];
  }
  __syncthreads();
  fft_tile<CF, L, false>(tile, tw_s);
  __syncthreads();
  const double k2 = (double)signed_freq(j + op.j0, op.n2g);
  if constexpr (REDUCE) {
    double acc = 0.0;
    for (int t = threadIdx.x; t < L * nb; t += NT) {
      const int q = t / L, m = t - q * L;
      const double k1 = (double)signed_freq(m, L);
      const int kz = kz0 + q;
      const double k3 = (double)kz;
      const double ksq = k1 * k1 + k2 * k2 + k3 * k3;
      const double mult = (kz == 0 || (n3 % 2 == 0 && kz == n3h - 1)) ? 1.0 : 2.0;
      const CF v = tile[q * PL + padi(m)];
      acc += mult * (1.0 + ksq) * ((double)v.x * v.x + (double)v.y * v.y);
    }
    __shared__ double red[32];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      double y = threadIdx.x < (NT >> 5) ? red[threadIdx.x] : 0.0;
      y = warp_sum(y);
      if (threadIdx.x == 0) partials[blockIdx.x] = y;
    }
    return;
  } else {
    for (int t = threadIdx.x; t < L * B; t += NT) {
      const int q = t / L, m = t - q * L;
      const double k1 = (double)signed_freq(m, L), k3 = (double)(kz0 + q);
      double2 vals[3];
#pragma unroll
      for (int c = 0; c < NC; ++c) vals[c] = to_d(tile[(c * B + q) * PL + padi(m)]);
      apply_symbol(op, k1, k2, k3, vals);
#pragma unroll
      for (int c = 0; c < NC; ++c) tile[(c * B + q) * PL + padi(m)] = convert<CF>(vals[c]);
    }
    __syncthreads();
    fft_tile<CF, L, true>(tile, tw_s);
    __syncthreads();

#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = threadIdx.x + u * NT;
      const int q = e % B, ci = e / B;
      const int c = ci / L, i = ci - c * L;
      if (q < nb) {
        const CF v = tile[(c * B + q) * PL + padi(i)];
        *op.out_at(T, c, i, lstride, (int64_t)j * n3h + kz0 + q) = make_float2((float)v.x, (float)v.y);
      }
    }
  }
}

}  // namespace fast
}  // namespace vr
