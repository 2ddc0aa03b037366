// Shared-memory-staged semi-Lagrangian gathers.
//
// One CTA owns a TX x TY x TZ tile of arrival voxels (4 x 8 x 32; 256 threads,
// each thread 4 voxels along x1).  It reads the tile's departure points (the
// displacement field, coalesced), reduces their floor-index bounding box, and
// stages that box of the source volume -- plus the interpolation stencil --
// into shared memory with coalesced x3-row loads (periodic wrap applied while
// loading).  All 8 (trilinear) / 64 (tricubic) taps per point are then read
// from shared memory instead of issuing scattered L1/L2 gathers.  Smooth
// characteristics make the box only slightly larger than the tile
// (~3.7 source voxels staged per arrival voxel for C2); a tile whose box
// exceeds the budget (rough velocity, tiny grid) falls back to direct gathers
// -- same arithmetic, same results.
#pragma once
#include <climits>
#include "interp.cuh"

namespace vr {
namespace staged {

constexpr int TZ = 32, TY = 8, TX = 4;
constexpr int CAP = 12032;  // staged floats per CTA (47 KB), 4 CTAs per SM

__device__ __forceinline__ void voxel_of(int idx, const Dims& d, int& i, int& j, int& k) {
  k = idx % d.n3;
  const int r = idx / d.n3;
  j = r % d.n2;
  i = r / d.n2;
}

// interpolation from the staged box; (lx, ly, lz) = floor index minus box origin
// (the box origin already includes the cubic stencil's -1)
__device__ __forceinline__ void cp_async4(float* smem, const float* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// how a source is staged: raw fp32 fields go through cp.async (no register
// round trip, every copy in flight at once); label indicators are converted.
template <class Src> struct Stager;
template <> struct Stager<SrcF32> {
  __device__ __forceinline__ static void put(const SrcF32& s, float* dst, int idx) { cp_async4(dst, s.p[0] + idx); }
};
template <> struct Stager<SrcLabel> {
  __device__ __forceinline__ static void put(const SrcLabel& s, float* dst, int idx) { *dst = s(0, idx); }
};

template <int ORDER>
__device__ __forceinline__ float gather_box(const float* __restrict__ box, int by, int bz, int lx, int ly, int lz,
                                            float tx, float ty, float tz) {
  if (ORDER == ORDER_LINEAR) {
    const int r00 = (lx * by + ly) * bz + lz, r01 = r00 + bz;
    const int r10 = r00 + by * bz, r11 = r10 + bz;
    const float sz = 1.0f - tz, sy = 1.0f - ty, sx = 1.0f - tx;
    const float c00 = box[r00] * sz + box[r00 + 1] * tz;
    const float c01 = box[r01] * sz + box[r01 + 1] * tz;
    const float c10 = box[r10] * sz + box[r10 + 1] * tz;
    const float c11 = box[r11] * sz + box[r11 + 1] * tz;
    const float c0 = c00 * sy + c01 * ty;
    const float c1 = c10 * sy + c11 * ty;
    return c0 * sx + c1 * tx;
  } else {
    float wx[4], wy[4], wz[4];
    lagrange4(tx, wx);
    lagrange4(ty, wy);
    lagrange4(tz, wz);
    float acc = 0.0f;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      float sa = 0.0f;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float* row = box + ((lx + a) * by + (ly + b)) * bz + lz;
        const float sb = wz[0] * row[0] + wz[1] * row[1] + wz[2] * row[2] + wz[3] * row[3];
        sa += wy[b] * sb;
      }
      acc += wx[a] * sa;
    }
    return acc;
  }
}

// Generic staged sweep: out voxel idx <- epi(idx, interp(src, departure(idx)))
template <int ORDER, class Src, class Epi>
__global__ void __launch_bounds__(256, 4) sweep_kernel(Src src, Dims d, const float* __restrict__ disp, Epi epi) {
  extern __shared__ float box[];
  __shared__ int ext[6];
  const int64_t N = d.n();
  const int z0 = blockIdx.x * TZ, y0 = blockIdx.y * TY, x0 = blockIdx.z * TX;
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
    if (inyz && i < d.n1) {
      const int idx = (i * d.n2 + j) * d.n3 + k;
      split_coord(i, __ldg(disp + idx), ix[u], fx[u]);
      split_coord(j, __ldg(disp + N + idx), iy[u], fy[u]);
      split_coord(k, __ldg(disp + 2 * N + idx), iz[u], fz[u]);
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
  const int lo_off = (ORDER == ORDER_CUBIC) ? 1 : 0, hi_off = (ORDER == ORDER_CUBIC) ? 2 : 1;
  const int lox = ext[0] - lo_off, loy = ext[1] - lo_off, loz = ext[2] - lo_off;
  const int bx = ext[3] + hi_off - lox + 1, by = ext[4] + hi_off - loy + 1, bz = ext[5] + hi_off - loz + 1;
  const bool use_box = bx <= d.n1 && by <= d.n2 && bz <= d.n3 && (int64_t)bx * by * ((bz + 31) & ~31) <= CAP;
  const int bzp = (bz + 31) & ~31;  // x3 row pitch in the box
  if (use_box) {
    // stage: one x3 row of the box per warp iteration, lanes along x3 (coalesced);
    // all copies are issued before the single wait
    const int warp = tid >> 5, lane = tid & 31;
    const int lzw = wrap_idx(loz, d.n3);
    const int nrows = bx * by;
    int a = warp / by, b = warp - a * by;
    for (int row = warp; row < nrows; row += 8) {
      const int gi = wrap_idx(lox + a, d.n1), gj = wrap_idx(loy + b, d.n2);
      const int rbase = (gi * d.n2 + gj) * d.n3;
      float* dst = box + row * bzp;
      for (int c = lane; c < bz; c += 32) {
        int gk = lzw + c;
        gk = gk >= d.n3 ? gk - d.n3 : gk;
        Stager<Src>::put(src, dst + c, rbase + gk);
      }
      b += 8;
      while (b >= by) { b -= by; ++a; }
    }
    cp_async_wait_all();
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < TX; ++u) {
    const int i = x0 + u;
    if (!(inyz && i < d.n1)) continue;
    float o;
    if (use_box) {
      o = gather_box<ORDER>(box, by, bzp, ix[u] - lox - lo_off, iy[u] - loy - lo_off, iz[u] - loz - lo_off, fx[u],
                            fy[u], fz[u]);
    } else {
      gather<ORDER, 1>(src, d, ix[u], iy[u], iz[u], fx[u], fy[u], fz[u], &o);
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

inline dim3 sweep_grid(const Dims& d) {
  return dim3((d.n3 + TZ - 1) / TZ, (d.n2 + TY - 1) / TY, (d.n1 + TX - 1) / TX);
}
inline dim3 sweep_block() { return dim3(TZ, TY); }
constexpr size_t kSweepSmem = sizeof(float) * CAP;

}  // namespace staged
}  // namespace vr
