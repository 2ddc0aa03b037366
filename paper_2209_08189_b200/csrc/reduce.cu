// Deterministic reductions and fused vector updates for the GN / PCG loop.
//
// Reference call sites (/root/reference/pkg/src/velreg/):
//   inner / weighted_norm     optim.py:80-85   (np.dot * cell volume)
//   PCG dots and norms        optim.py:231-246 (unweighted np.dot / np.linalg.norm)
//   relative_residual         optim.py:252-258
//   _intensity_shift          optim.py:261-268 (min / max over both images)
//   max_pointwise_norm (CFL)  grid.py:129-130, transport.py:53-54
//   J extrema                 optim.py:362-363
//   non-finite guards         transport.py:57-59,119-121; optim.py:157,179
//   Dice counts               metrics.py:45-57,72-73 (exact integers)
// Every sum accumulates in f64; the tree is fixed (grid-stride partials per
// CTA, then one CTA sums the partials in index order), so results are
// bit-reproducible run to run -- the analogue of the reference's
// "reproducible" serial kernels (runtime.py:1-17).
#include <climits>
#include "common.cuh"
#include "../../include/velreg_b200.h"

namespace vr {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 148 * 4;  // one wave of 4 CTAs per SM

// NaN-propagating min / max (numpy .min() / .max() return NaN when any entry
// is NaN; fmin / fmax would skip it and let a NaN Jacobian pass in_bounds)
__device__ __forceinline__ double nmin(double x, double y) { return x != x ? x : (y != y ? y : fmin(x, y)); }
__device__ __forceinline__ double nmax(double x, double y) { return x != x ? x : (y != y ? y : fmax(x, y)); }

template <int K>
__device__ __forceinline__ void block_reduce_store(double (&v)[K], double* __restrict__ dst, int mode) {
  __shared__ double red[K][kRedThreads / 32];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    double x = v[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double y = __shfl_xor_sync(0xffffffffu, x, o);
      x = (mode == VR_RED_SUM) ? x + y : (((q & 1) == 0) ? nmin(x, y) : nmax(x, y));
    }
    if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < K; ++q) {
      double x = red[q][0];
      for (int w = 1; w < kRedThreads / 32; ++w)
        x = (mode == VR_RED_SUM) ? x + red[q][w] : (((q & 1) == 0) ? nmin(x, red[q][w]) : nmax(x, red[q][w]));
      dst[q] = x;
    }
  }
}

// K sums of products  sum_i a_q[i] * b_q[i]   (b_q == nullptr -> a_q itself squared
// is NOT implied; pass the same pointer twice for norms)
struct DotArgs {
  const float* a[4];
  const float* b[4];
  int k;
};

template <int K>
__global__ void __launch_bounds__(kRedThreads) dot_partials_kernel(DotArgs args, int64_t n,
                                                                   double* __restrict__ partials) {
  double acc[K];
#pragma unroll
  for (int q = 0; q < K; ++q) acc[q] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] += (double)__ldg(args.a[q] + i) * (double)__ldg(args.b[q] + i);
  }
  block_reduce_store<K>(acc, partials + (int64_t)blockIdx.x * K, VR_RED_SUM);
}

// The same sums with every distinct operand array loaded once per element:
// PCG's (r.z, z.z) and the norms (g.g) name an array twice, and a load per
// operand re-reads it (a dot is HBM-bound).  Same products, same order: the
// results equal dot_partials_kernel's bit for bit.
struct DotArgsU {
  const float* src[8];
  int ia[4], ib[4];
};

template <int K, int NS>
__global__ void __launch_bounds__(kRedThreads) dotu_partials_kernel(DotArgsU args, int64_t n,
                                                                    double* __restrict__ partials) {
  double acc[K];
#pragma unroll
  for (int q = 0; q < K; ++q) acc[q] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v[NS];
#pragma unroll
    for (int u = 0; u < NS; ++u) v[u] = (double)__ldg(args.src[u] + i);
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] += v[args.ia[q]] * v[args.ib[q]];
  }
  block_reduce_store<K>(acc, partials + (int64_t)blockIdx.x * K, VR_RED_SUM);
}

// sum (a-b)^2 and sum (c-b)^2 in one pass (relative residual numerator/denominator)
__global__ void __launch_bounds__(kRedThreads) sqdiff_partials_kernel(const float* __restrict__ a,
                                                                      const float* __restrict__ b,
                                                                      const float* __restrict__ c, int64_t n,
                                                                      double* __restrict__ partials) {
  double acc[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double bb = __ldg(b + i);
    const double x = (double)__ldg(a + i) - bb;
    acc[0] += x * x;
    if (c) {
      const double y = (double)__ldg(c + i) - bb;
      acc[1] += y * y;
    }
  }
  block_reduce_store<2>(acc, partials + (int64_t)blockIdx.x * 2, VR_RED_SUM);
}

// min/max of up to two arrays -> (min0, max0, min1, max1); also counts
// non-finite entries of array 0 in slot 4 (as a sum of 0/1)
__global__ void __launch_bounds__(kRedThreads) minmax_partials_kernel(const float* __restrict__ a,
                                                                      const float* __restrict__ b, int64_t n,
                                                                      double* __restrict__ partials) {
  double acc[4] = {INFINITY, -INFINITY, INFINITY, -INFINITY};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = __ldg(a + i);
    acc[0] = nmin(acc[0], x);
    acc[1] = nmax(acc[1], x);
    if (b) {
      const double y = __ldg(b + i);
      acc[2] = nmin(acc[2], y);
      acc[3] = nmax(acc[3], y);
    }
  }
  block_reduce_store<4>(acc, partials + (int64_t)blockIdx.x * 4, VR_RED_MINMAX);
}

// max_x |v(x)|^2 over a 3-component field, plus count of non-finite values and
// count of non-zero values (np.any)
__global__ void __launch_bounds__(kRedThreads) vecstats_partials_kernel(const float* __restrict__ v, int64_t n,
                                                                        double* __restrict__ partials) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // [maxnorm2 (as max, slot1), ...]
  double mx = 0.0, nonfinite = 0.0, nonzero = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = __ldg(v + i), y = __ldg(v + n + i), z = __ldg(v + 2 * n + i);
    const double s = x * x + y * y + z * z;
    if (isfinite(s)) mx = fmax(mx, s);
    nonfinite += (!isfinite(x)) + (!isfinite(y)) + (!isfinite(z));
    nonzero += (x != 0.0) + (y != 0.0) + (z != 0.0);
  }
  // slots: 0 = -maxnorm2 (min-reduced), 1 = maxnorm2 (max-reduced) -- reuse the
  // min/max tree for the max; the counts go through a second (sum) tree.
  acc[0] = -mx;
  acc[1] = mx;
  acc[2] = INFINITY;
  acc[3] = -INFINITY;
  block_reduce_store<4>(acc, partials + (int64_t)blockIdx.x * 8, VR_RED_MINMAX);
  __syncthreads();
  double cnt[2] = {nonfinite, nonzero};
  block_reduce_store<2>(cnt, partials + (int64_t)blockIdx.x * 8 + 4, VR_RED_SUM);
}

// one CTA folds nblk x K partials (stride `stride`) in index order
__global__ void fold_partials_kernel(const double* __restrict__ partials, int nblk, int stride, int k, int mode,
                                     double* __restrict__ out) {
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int q = 0; q < k; ++q) {
    const bool isMin = (mode == VR_RED_MINMAX) && ((q & 1) == 0);
    double x = (mode == VR_RED_SUM) ? 0.0 : (isMin ? INFINITY : -INFINITY);
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
      const double y = partials[(int64_t)b * stride + q];
      x = (mode == VR_RED_SUM) ? x + y : (isMin ? nmin(x, y) : nmax(x, y));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, x, o);
      x = (mode == VR_RED_SUM) ? x + y : (isMin ? nmin(x, y) : nmax(x, y));
    }
    if (lane == 0) red[q][w] = x;
  }
  __syncthreads();
  if (threadIdx.x < k) {
    const int q = threadIdx.x;
    const bool isMin = (mode == VR_RED_MINMAX) && ((q & 1) == 0);
    double x = red[q][0];
    for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww)
      x = (mode == VR_RED_SUM) ? x + red[q][ww] : (isMin ? nmin(x, red[q][ww]) : nmax(x, red[q][ww]));
    out[q] = x;
  }
}

// ---- fused vector updates (f64 arithmetic on f32 storage) ----------------------
// out = a*x + b*y   (y may be null -> out = a*x)
__global__ void __launch_bounds__(256) axpby_kernel(int64_t n, double a, const float* __restrict__ x, double b,
                                                    const float* __restrict__ y, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double r = a * (double)x[i];
    if (y) r += b * (double)y[i];
    out[i] = (float)r;
  }
}

// PCG step (optim.py:241-242): x += alpha p; r -= alpha hp
__global__ void __launch_bounds__(256) pcg_update_kernel(int64_t n, double alpha, const float* __restrict__ p,
                                                         const float* __restrict__ hp, float* __restrict__ x,
                                                         float* __restrict__ r) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = (float)((double)x[i] + alpha * (double)p[i]);
    r[i] = (float)((double)r[i] - alpha * (double)hp[i]);
  }
}

// PCG step with the step length formed on the device, alpha = rz / php (f64,
// the host's Python division bit for bit), from separate inputs into separate
// outputs so the caller can still return the previous iterate when php <= 0
// (optim.py:238-240 negative-curvature exit) after reading both scalars with
// the next host read.
__global__ void __launch_bounds__(256) pcg_update2_kernel(int64_t n, const double* __restrict__ rz,
                                                          const double* __restrict__ php,
                                                          const float* __restrict__ p, const float* __restrict__ hp,
                                                          const float* x, const float* r, float* xo, float* ro) {
  const double alpha = __ldg(rz) / __ldg(php);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    xo[i] = (float)((double)x[i] + alpha * (double)p[i]);
    ro[i] = (float)((double)r[i] - alpha * (double)hp[i]);
  }
}

__global__ void __launch_bounds__(256) fill_kernel(int64_t n, float v, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

// ---- Dice counts (metrics.py:45-57,72-73) ---------------------------------------
// counts[3*id + {0,1,2}] += |l0==id|, |l1==id|, |l0==id & l1==id| for id <= max_id
__global__ void __launch_bounds__(256) label_counts_kernel(const int* __restrict__ l0, const int* __restrict__ l1,
                                                           int64_t n, int max_id,
                                                           unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned int hist[];
  const int nb = 3 * (max_id + 1);
  for (int t = threadIdx.x; t < nb; t += blockDim.x) hist[t] = 0u;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int a = __ldg(l0 + i), b = __ldg(l1 + i);
    if (a >= 0 && a <= max_id) atomicAdd(&hist[3 * a], 1u);
    if (b >= 0 && b <= max_id) atomicAdd(&hist[3 * b + 1], 1u);
    if (a == b && a >= 0 && a <= max_id) atomicAdd(&hist[3 * a + 2], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nb; t += blockDim.x)
    if (hist[t]) atomicAdd(counts + t, (unsigned long long)hist[t]);
}

// (min l0, max l0, min l1, max l1) of one or two int32 label maps in one pass:
// validates label ids (grid.py LabelMap: non-negative) and sizes the label
// histogram with a single host read.  Integer min / max atomics are
// order-independent, so the result is deterministic.
__global__ void label_range_init_kernel(int* __restrict__ out) {
  if (threadIdx.x < 4) out[threadIdx.x] = (threadIdx.x & 1) ? INT_MIN : INT_MAX;
}

__global__ void __launch_bounds__(256) label_range_kernel(const int* __restrict__ l0, const int* __restrict__ l1,
                                                          int64_t n, int* __restrict__ out) {
  int a0 = INT_MAX, a1 = INT_MIN, b0 = INT_MAX, b1 = INT_MIN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int a = __ldg(l0 + i);
    a0 = min(a0, a);
    a1 = max(a1, a);
    if (l1) {
      const int b = __ldg(l1 + i);
      b0 = min(b0, b);
      b1 = max(b1, b);
    }
  }
  a0 = __reduce_min_sync(~0u, a0);
  a1 = __reduce_max_sync(~0u, a1);
  b0 = __reduce_min_sync(~0u, b0);
  b1 = __reduce_max_sync(~0u, b1);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, a0);
    atomicMax(out + 1, a1);
    if (l1) {
      atomicMin(out + 2, b0);
      atomicMax(out + 3, b1);
    }
  }
}

}  // namespace vr

using namespace vr;

namespace {
unsigned red_blocks(int64_t n) {
  int64_t b = (n + kRedThreads - 1) / kRedThreads;
  return (unsigned)(b < kRedBlocks ? (b < 1 ? 1 : b) : kRedBlocks);
}
}  // namespace

extern "C" {

int vr_reduce_scratch_doubles(void) { return kRedBlocks * 8 + 64; }

int vr_dots(int k, const float* const* a, const float* const* b, int64_t n, double* scratch, double* out,
            void* stream) {
  if (k < 1 || k > 4 || !a || !b || !scratch || !out || n < 0) return VR_ERR_ARG;
  DotArgs args{};
  args.k = k;
  for (int q = 0; q < k; ++q) {
    if (!a[q] || !b[q]) return VR_ERR_ARG;
    args.a[q] = a[q];
    args.b[q] = b[q];
  }
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned nb = red_blocks(n);
  // distinct operand arrays
  DotArgsU u{};
  int ns = 0;
  auto slot = [&](const float* ptr) {
    for (int t = 0; t < ns; ++t)
      if (u.src[t] == ptr) return t;
    u.src[ns] = ptr;
    return ns++;
  };
  for (int q = 0; q < k; ++q) {
    u.ia[q] = slot(a[q]);
    u.ib[q] = slot(b[q]);
  }
  if (ns < 2 * k && ns <= 3 && k <= 2) {   // an array is named twice: load it once
#define VR_DOTU(KK, NN) dotu_partials_kernel<KK, NN><<<nb, kRedThreads, 0, s>>>(u, n, scratch)
    if (k == 1) VR_DOTU(1, 1);
    else if (ns == 2) VR_DOTU(2, 2);
    else VR_DOTU(2, 3);
#undef VR_DOTU
    fold_partials_kernel<<<1, 256, 0, s>>>(scratch, nb, k, k, VR_RED_SUM, out);
    VR_CHECK_LAUNCH();
    return VR_OK;
  }
  switch (k) {
    case 1: dot_partials_kernel<1><<<nb, kRedThreads, 0, s>>>(args, n, scratch); break;
    case 2: dot_partials_kernel<2><<<nb, kRedThreads, 0, s>>>(args, n, scratch); break;
    case 3: dot_partials_kernel<3><<<nb, kRedThreads, 0, s>>>(args, n, scratch); break;
    default: dot_partials_kernel<4><<<nb, kRedThreads, 0, s>>>(args, n, scratch); break;
  }
  fold_partials_kernel<<<1, 256, 0, s>>>(scratch, nb, k, k, VR_RED_SUM, out);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_sqdiff(const float* a, const float* b, const float* c, int64_t n, double* scratch, double* out2,
              void* stream) {
  if (!a || !b || !scratch || !out2 || n < 0) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned nb = red_blocks(n);
  sqdiff_partials_kernel<<<nb, kRedThreads, 0, s>>>(a, b, c, n, scratch);
  fold_partials_kernel<<<1, 256, 0, s>>>(scratch, nb, 2, 2, VR_RED_SUM, out2);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_minmax(const float* a, const float* b, int64_t n, double* scratch, double* out4, void* stream) {
  if (!a || !scratch || !out4 || n < 1) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned nb = red_blocks(n);
  minmax_partials_kernel<<<nb, kRedThreads, 0, s>>>(a, b, n, scratch);
  fold_partials_kernel<<<1, 256, 0, s>>>(scratch, nb, 4, 4, VR_RED_MINMAX, out4);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// out4 = {-max|v|^2, max|v|^2, nonfinite count, nonzero count}
int vr_vecstats(const float* v, int64_t n, double* scratch, double* out4, void* stream) {
  if (!v || !scratch || !out4 || n < 1) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned nb = red_blocks(n);
  vecstats_partials_kernel<<<nb, kRedThreads, 0, s>>>(v, n, scratch);
  fold_partials_kernel<<<1, 256, 0, s>>>(scratch, nb, 8, 2, VR_RED_MINMAX, out4);
  fold_partials_kernel<<<1, 256, 0, s>>>(scratch + 4, nb, 8, 2, VR_RED_SUM, out4 + 2);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_axpby(int64_t n, double a, const float* x, double b, const float* y, float* out, void* stream) {
  if (!x || !out || n < 0) return VR_ERR_ARG;
  if (n == 0) return VR_OK;
  axpby_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(n, a, x, b, y, out);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_pcg_update(int64_t n, double alpha, const float* p, const float* hp, float* x, float* r, void* stream) {
  if (!p || !hp || !x || !r || n < 0) return VR_ERR_ARG;
  if (n == 0) return VR_OK;
  pcg_update_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(n, alpha, p, hp, x, r);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_pcg_update2(int64_t n, const double* rz_dev, const double* php_dev, const float* p, const float* hp,
                   const float* x, const float* r, float* x_out, float* r_out, void* stream) {
  if (!rz_dev || !php_dev || !p || !hp || !x || !r || !x_out || !r_out || n < 0) return VR_ERR_ARG;
  if (n == 0) return VR_OK;
  pcg_update2_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(n, rz_dev, php_dev, p, hp, x, r,
                                                                                 x_out, r_out);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_fill(int64_t n, float value, float* out, void* stream) {
  if (!out || n < 0) return VR_ERR_ARG;
  if (n == 0) return VR_OK;
  fill_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(n, value, out);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_label_range(const int* l0, const int* l1, int64_t n, int* out, void* stream) {
  if (!l0 || !out || n < 0) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  label_range_init_kernel<<<1, 32, 0, s>>>(out);
  if (n > 0) label_range_kernel<<<red_blocks(n), 256, 0, s>>>(l0, l1, n, out);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_label_counts(const int* l0, const int* l1, int64_t n, int max_id, unsigned long long* counts,
                    void* stream) {
  if (!l0 || !l1 || !counts || n < 0 || max_id < 0 || max_id > 8191) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t sm = sizeof(unsigned) * 3 * (size_t)(max_id + 1);
  if (cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * 3 * (max_id + 1), s) != cudaSuccess)
    return VR_ERR_LAUNCH;
  if (n == 0) return VR_OK;
  if (sm > 48 * 1024)
    cudaFuncSetAttribute(label_counts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  label_counts_kernel<<<red_blocks(n), 256, sm, s>>>(l0, l1, n, max_id, counts);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

}  // extern "C"
